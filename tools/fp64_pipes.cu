// Microbenchmark: FP64 vector (DFMA) vs FP64 tensor (DMMA m8n8k4) throughput on
// one B200, alone and interleaved. Decides whether the 1D sum-factorization
// passes should move to mma.sync f64.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters)
{
  double a[8];
  for (int i = 0; i < 8; ++i)
    a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 8; ++i)
    s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FP32 FFMA peak (the fp32 roofline denominator of the c5f32 line)
__global__ void ffma_kernel(float *out, int iters)
{
  float a[16];
  for (int i = 0; i < 16; ++i)
    a[i] = threadIdx.x * 1e-3f + i;
  const float b = 1.0000001f, c = 1e-9f;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i)
      a[i] = fmaf(a[i], b, c);
  float s = 0;
  for (int i = 0; i < 16; ++i)
    s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double *out, int iters)
{
  double d[8][2];
  for (int i = 0; i < 8; ++i)
    d[i][0] = d[i][1] = 0;
  const double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      dmma(d[i][0], d[i][1], a, b);
  double s = 0;
  for (int i = 0; i < 8; ++i)
    s += d[i][0] + d[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void both_kernel(double *out, int iters)
{
  double d[4][2], x[8];
  for (int i = 0; i < 4; ++i)
    d[i][0] = d[i][1] = 0;
  for (int i = 0; i < 8; ++i)
    x[i] = threadIdx.x * 1e-3 + i;
  const double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it)
    {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        dmma(d[i][0], d[i][1], a, b);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        x[i] = fma(x[i], 1.0000001, 1e-9);
    }
  double s = 0;
  for (int i = 0; i < 4; ++i)
    s += d[i][0] + d[i][1];
  for (int i = 0; i < 8; ++i)
    s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  double *out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const double warps = (double)blocks * threads / 32;
  for (int rep = 0; rep < 2; ++rep)
    {
      cudaEventRecord(e0);
      dfma_kernel<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double dfma_tf = 2.0 * blocks * threads * 8.0 * iters / (ms * 1e-3) / 1e12;
      cudaEventRecord(e0);
      dmma_kernel<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double dmma_tf = 2.0 * 256 * warps * 8.0 * iters / (ms * 1e-3) / 1e12;
      cudaEventRecord(e0);
      both_kernel<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double both_tf =
        (2.0 * 256 * warps * 4.0 * iters + 2.0 * blocks * threads * 8.0 * iters) /
        (ms * 1e-3) / 1e12;
      cudaEventRecord(e0);
      ffma_kernel<<<blocks, threads>>>(reinterpret_cast<float *>(out), iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double ffma_tf = 2.0 * blocks * threads * 16.0 * iters / (ms * 1e-3) / 1e12;
      std::printf("DFMA %.1f TFLOP/s  DMMA %.1f TFLOP/s  interleaved %.1f TFLOP/s  FFMA %.1f TFLOP/s\n",
                  dfma_tf, dmma_tf, both_tf, ffma_tf);
    }
  return 0;
}

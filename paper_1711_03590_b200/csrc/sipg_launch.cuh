// Per-basis constant tables and launch dispatch of the fused SIPG apply
// kernel. Included once per basis by sipg_gl.cu / sipg_gauss.cu /
// sipg_hermite.cu with DGX_BASIS set: every translation unit owns its
// TU-local __constant__ tables (sipg_kernel.cuh), so each basis has its own
// 64 KB constant bank and the three compile in parallel.
#pragma once
#include "device.hpp"
#include "setup.hpp"
#include "sipg_kernel.cuh"
#include "sipg_pairs.cuh"
#include "sipg_cart.cuh"
#include "sipg_rhs.cuh"
#include "sipg_adv.cuh"

#include <algorithm>
#include <cmath>
#include <mutex>
#include <vector>
#include <set>
#include <tuple>

#ifndef DGX_BASIS
#error "define DGX_BASIS (0 GL, 1 Gauss, 2 Hermite-like) before including sipg_launch.cuh"
#endif

namespace dgx
{
namespace
{

// Even-odd halves [CE][CE] of a mirror-(skew-)symmetric K x K matrix M
// (reference basis.cpp:182-221 packing, in the padded layout the device
// routines eo_sym / eo_skew index).
void eo_halves(const std::vector<double> &M, int K, double *E, double *O)
{
  const int H = K / 2, CE = (K + 1) / 2;
  for (int q = 0; q < CE; ++q)
    for (int j = 0; j < CE; ++j)
      {
        E[q * CE + j] = j < H ? 0.5 * (M[q * K + j] + M[q * K + (K - 1 - j)])
                              : M[q * K + j];
        O[q * CE + j] = j < H ? 0.5 * (M[q * K + j] - M[q * K + (K - 1 - j)]) : 0.0;
      }
}

std::vector<double> transpose(const std::vector<double> &M, int K)
{
  std::vector<double> t(K * K);
  for (int i = 0; i < K; ++i)
    for (int j = 0; j < K; ++j)
      t[i * K + j] = M[j * K + i];
  return t;
}

std::vector<double> build_table(int K)
{
  const Tables1D t = make_tables(K - 1, DGX_BASIS);
  const int CE = (K + 1) / 2;
  std::vector<double> tab(dev::tab_size(K), 0.0);
  double *b = tab.data();
  const int c2 = CE * CE;
  eo_halves(t.S, K, b + 0 * c2, b + 1 * c2);
  eo_halves(transpose(t.S, K), K, b + 2 * c2, b + 3 * c2);
  eo_halves(t.Dco, K, b + 4 * c2, b + 5 * c2);
  eo_halves(transpose(t.Dco, K), K, b + 6 * c2, b + 7 * c2);
  double *o = b + 8 * c2;
  for (int i = 0; i < K * K; ++i)
    o[i] = t.S[i];
  o += K * K;
  for (int i = 0; i < K * K; ++i)
    o[i] = t.Dco[i];
  o += K * K;
  for (int s = 0; s < 2; ++s)
    for (int j = 0; j < K; ++j)
      o[s * K + j] = t.Sf[s][j];
  o += 2 * K;
  for (int s = 0; s < 2; ++s)
    for (int j = 0; j < K; ++j)
      o[s * K + j] = t.Df[s][j];
  o += 2 * K;
  for (int s = 0; s < 2; ++s)
    for (int j = 0; j < K; ++j)
      o[s * K + j] = t.rf[s][j];
  o += 2 * K;
  for (int j = 0; j < K; ++j)
    o[j] = t.qw[j];
  o += K;
  // rows (rf_s Dco)[j] = sum_q rf_s[q] Dco[q][j]: own normal-derivative
  // trace from collocation values, and (Dco^T rf_s^T) for its transpose
  for (int s = 0; s < 2; ++s)
    for (int j = 0; j < K; ++j)
      {
        double acc = 0.0;
        for (int q = 0; q < K; ++q)
          acc += t.rf[s][q] * t.Dco[q * K + j];
        o[s * K + j] = acc;
      }
  o += 2 * K;
  eo_halves(t.D, K, o, o + c2); // nodal derivative D (basis.cpp:277-278)
  o += 2 * c2;
  for (int i = 0; i < K * K; ++i) // and plainly (row-dot neighbour traces, sipg_pairs.cuh)
    o[i] = t.D[i];
  o += K * K;
  // 1D mass and stiffness matrices of the k-point Gauss rule (sipg_cart.cuh)
  std::vector<double> M1(K * K, 0.0), K1(K * K, 0.0);
  for (int i = 0; i < K; ++i)
    for (int j = 0; j < K; ++j)
      for (int q = 0; q < K; ++q)
        {
          M1[i * K + j] += t.S[q * K + i] * t.qw[q] * t.S[q * K + j];
          K1[i * K + j] += t.D[q * K + i] * t.qw[q] * t.D[q * K + j];
        }
  eo_halves(M1, K, o, o + c2);
  o += 2 * c2;
  // M1^{-1} [K1 | Sf_0^T Sf_1^T Df_0^T Df_1^T]: Gaussian elimination with
  // partial pivoting on the augmented system (M1 is s.p.d., k <= 11)
  const int NR = K + 4;
  std::vector<double> aug(K * (K + NR), 0.0);
  for (int i = 0; i < K; ++i)
    {
      for (int j = 0; j < K; ++j)
        {
          aug[i * (K + NR) + j] = M1[i * K + j];
          aug[i * (K + NR) + K + j] = K1[i * K + j];
        }
      for (int s = 0; s < 2; ++s)
        {
          aug[i * (K + NR) + 2 * K + s] = t.Sf[s][i];
          aug[i * (K + NR) + 2 * K + 2 + s] = t.Df[s][i];
        }
    }
  for (int c = 0; c < K; ++c)
    {
      int piv = c;
      for (int r = c + 1; r < K; ++r)
        if (std::fabs(aug[r * (K + NR) + c]) > std::fabs(aug[piv * (K + NR) + c]))
          piv = r;
      if (piv != c)
        for (int j = 0; j < K + NR; ++j)
          std::swap(aug[c * (K + NR) + j], aug[piv * (K + NR) + j]);
      const double d = aug[c * (K + NR) + c];
      for (int j = 0; j < K + NR; ++j)
        aug[c * (K + NR) + j] /= d;
      for (int r = 0; r < K; ++r)
        if (r != c)
          {
            const double f = aug[r * (K + NR) + c];
            if (f != 0.0)
              for (int j = 0; j < K + NR; ++j)
                aug[r * (K + NR) + j] -= f * aug[c * (K + NR) + j];
          }
    }
  std::vector<double> MK(K * K);
  for (int i = 0; i < K; ++i)
    for (int j = 0; j < K; ++j)
      MK[i * K + j] = aug[i * (K + NR) + K + j];
  // symmetrise the mirror pairs (the even-odd halves assume exact mirror symmetry)
  for (int i = 0; i < K; ++i)
    for (int j = 0; j < K; ++j)
      {
        const double a = 0.5 * (MK[i * K + j] + MK[(K - 1 - i) * K + (K - 1 - j)]);
        MK[i * K + j] = MK[(K - 1 - i) * K + (K - 1 - j)] = a;
      }
  // Hermite-like basis: cond(M1) grows to 1e6 at p = 10 (the nodal bases stay
  // below 20), so that kernel keeps K1 itself and two mass products per axis
#if DGX_BASIS == 2
  eo_halves(K1, K, o, o + c2);
#else
  eo_halves(MK, K, o, o + c2);
#endif
  o += 2 * c2;
  for (int s = 0; s < 2; ++s)
    for (int i = 0; i < K; ++i)
      {
        o[s * K + i] = aug[i * (K + NR) + 2 * K + s];           // M1^{-1} Sf_s^T
        o[2 * K + s * K + i] = aug[i * (K + NR) + 2 * K + 2 + s]; // M1^{-1} Df_s^T
      }
  return tab;
}

std::mutex g_mutex;
std::set<std::tuple<int, int>> g_uploaded; // (device, K)

template <typename KERN>
void set_smem_once(KERN kern, size_t smem, std::set<int> &configured);

#ifndef DGX_PAIRS
#define DGX_PAIRS 1 // 3D fp64, even K: the pencil-pair kernel (sipg_pairs.cuh)
#endif
#ifndef DGX_PAIRS_ODD
#define DGX_PAIRS_ODD 0 // odd K through the padded pair kernel: correct, measured slower (C3 15.7 vs 17.6, C5 19.0 vs 23.7 GDoF/s)
#endif

template <int K, bool C>
void launch_pairs(const dev::ApplyParams<double> &prm, cudaStream_t s)
{
  using L = dev::PL<K>;
#ifndef DGX_EXP_SMEM_PAD
#define DGX_EXP_SMEM_PAD 0 // occupancy ablation: unused extra shared memory per CTA
#endif
  const size_t smem = (size_t)L::SMEM_REALS * sizeof(double) + DGX_EXP_SMEM_PAD;
  auto kern = dev::sipg_pairs_kernel<K, C, DGX_BASIS>;
  static std::set<int> configured;
  set_smem_once(kern, smem, configured);
  static int resident[64] = {0}; // CTAs resident on the whole device, per device
  int devid = 0;
  cuda_check(cudaGetDevice(&devid), "cudaGetDevice");
  if (devid >= 0 && devid < 64 && resident[devid] == 0)
    {
      int per_sm = 0, sms = 0;
      cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L::THREADS, smem),
                 "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
      cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, devid),
                 "cudaDeviceGetAttribute");
      resident[devid] = per_sm * sms > 0 ? per_sm * sms : 1;
    }
  dev::ApplyParams<double> p2 = prm;
  p2.ahead = ((devid >= 0 && devid < 64) ? resident[devid] : 1) * L::NC;
  const int grid = (prm.n_tasks + L::NC - 1) / L::NC;
  if (grid > 0)
    kern<<<grid, L::THREADS, smem, s>>>(p2);
  cuda_check(cudaGetLastError(), "sipg_pairs_kernel launch");
}

// Axis-aligned affine records, nodal bases: the tensor-product kernel
// (sipg_cart.cuh); prm.cart == 2
template <typename Real, int D, int K>
void launch_cart(const dev::ApplyParams<Real> &prm, cudaStream_t s)
{
  using CS = dev::CartShape<Real, D, K, DGX_BASIS == 2>;
  const size_t smem = (size_t)CS::SMEM_REALS * sizeof(Real);
  auto kern = dev::sipg_cart_kernel<Real, D, K, DGX_BASIS>;
  static std::set<int> configured;
  set_smem_once(kern, smem, configured);
  const int grid = (prm.n_tasks + CS::NC - 1) / CS::NC;
  if (grid > 0)
    kern<<<grid, CS::THREADS, smem, s>>>(prm);
  cuda_check(cudaGetLastError(), "sipg_cart_kernel launch");
}

#ifndef DGX_CART_PAIRS
#define DGX_CART_PAIRS 1 // even K, 3D fp64 Cartesian: 1 = the general pair kernel, 0 = the single-pencil CART kernel
#endif

template <typename Real, int D, int K, bool C, bool CART = false>
void launch_one(const dev::ApplyParams<Real> &prm, cudaStream_t s)
{
  if constexpr (C && !CART)
    if (prm.cart == 2)
      {
        launch_cart<Real, D, K>(prm, s);
        return;
      }
  if constexpr (C && !CART)
    if (prm.cart && !(DGX_CART_PAIRS && DGX_PAIRS && D == 3 && sizeof(Real) == 8 && K % 2 == 0))
      {
        launch_one<Real, D, K, C, true>(prm, s);
        return;
      }
  if constexpr (!CART && DGX_PAIRS && D == 3 && sizeof(Real) == 8 && (K % 2 == 0 || DGX_PAIRS_ODD))
    {
      launch_pairs<K, C>(prm, s);
      return;
    }
  using KS = dev::KernelShape<D, K, true, CART>;
  const size_t smem = (size_t)KS::SMEM_REALS * sizeof(Real);
  auto kern = dev::sipg_apply_kernel<Real, D, K, C, DGX_BASIS, CART>;
  static std::set<int> configured;
  int devid = 0;
  cuda_check(cudaGetDevice(&devid), "cudaGetDevice");
  {
    std::lock_guard<std::mutex> lk(g_mutex);
    if (!configured.count(devid))
      {
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem),
                   "cudaFuncSetAttribute");
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        cudaSharedmemCarveoutMaxShared),
                   "cudaFuncSetAttribute(carveout)");
        configured.insert(devid);
      }
  }
  const int grid = (prm.n_tasks + KS::NC - 1) / KS::NC;
  if (grid > 0)
    kern<<<grid, KS::THREADS, smem, s>>>(prm);
  cuda_check(cudaGetLastError(), "sipg_apply_kernel launch");
}

template <typename Real, int D, int K>
void launch_k(bool compressed, const dev::ApplyParams<Real> &prm, cudaStream_t s)
{
  if (compressed)
    launch_one<Real, D, K, true>(prm, s);
  else
    launch_one<Real, D, K, false>(prm, s);
}

template <typename Real, int D>
void launch_d(int K, bool compressed, const dev::ApplyParams<Real> &prm, cudaStream_t s)
{
  switch (K)
    {
#ifdef DGX_DEV_K
    // kernel-experiment builds (tools/expbuild.sh): one 3D degree only
    case DGX_DEV_K:
      if constexpr (D == 3)
        launch_k<Real, D, DGX_DEV_K>(compressed, prm, s);
      break;
#else
#if DGX_BASIS != 2
    case 2: launch_k<Real, D, 2>(compressed, prm, s); break;
    case 3: launch_k<Real, D, 3>(compressed, prm, s); break;
#endif
    case 4: launch_k<Real, D, 4>(compressed, prm, s); break;
    case 5: launch_k<Real, D, 5>(compressed, prm, s); break;
    case 6: launch_k<Real, D, 6>(compressed, prm, s); break;
    case 7: launch_k<Real, D, 7>(compressed, prm, s); break;
    case 8: launch_k<Real, D, 8>(compressed, prm, s); break;
    case 9: launch_k<Real, D, 9>(compressed, prm, s); break;
    case 10: launch_k<Real, D, 10>(compressed, prm, s); break;
    case 11: launch_k<Real, D, 11>(compressed, prm, s); break;
#endif
    default: fail(Code::invalid_argument, "sipg apply: unsupported k");
    }
}

template <typename KERN>
void set_smem_once(KERN kern, size_t smem, std::set<int> &configured)
{
  int devid = 0;
  cuda_check(cudaGetDevice(&devid), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_mutex);
  if (!configured.count(devid))
    {
      cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem),
                 "cudaFuncSetAttribute");
      cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      cudaSharedmemCarveoutMaxShared),
                 "cudaFuncSetAttribute(carveout)");
      configured.insert(devid);
    }
}

template <int D, int K, bool C>
void launch_adv_one(const dev::AdvParams<double> &prm, cudaStream_t s)
{
  using KS = dev::KernelShape<D, K>;
  const size_t smem = (size_t)KS::SMEM_REALS * sizeof(double);
  auto kern = dev::sipg_adv_kernel<double, D, K, C, DGX_BASIS>;
  static std::set<int> configured;
  set_smem_once(kern, smem, configured);
  const int grid = (prm.n_tasks + KS::NC - 1) / KS::NC;
  if (grid > 0)
    kern<<<grid, KS::THREADS, smem, s>>>(prm);
  cuda_check(cudaGetLastError(), "sipg_adv_kernel launch");
}

template <int D>
void launch_adv_d(int K, bool compressed, const dev::AdvParams<double> &prm, cudaStream_t s)
{
  switch (K)
    {
#define DGX_ADV_K(KK)                                                                      \
  case KK:                                                                                 \
    if (compressed)                                                                        \
      launch_adv_one<D, KK, true>(prm, s);                                                 \
    else                                                                                   \
      launch_adv_one<D, KK, false>(prm, s);                                                \
    break;
#ifdef DGX_DEV_K
      DGX_ADV_K(DGX_DEV_K)
#else
      DGX_ADV_K(2) DGX_ADV_K(3) DGX_ADV_K(4) DGX_ADV_K(5) DGX_ADV_K(6) DGX_ADV_K(7)
      DGX_ADV_K(8) DGX_ADV_K(9) DGX_ADV_K(10) DGX_ADV_K(11)
#endif
#undef DGX_ADV_K
    default: fail(Code::invalid_argument, "advection: unsupported k");
    }
}

template <int D, int K, bool C, bool ADV>
void launch_rhs_one(const dev::RhsParams<double> &prm, cudaStream_t s)
{
  using KS = dev::KernelShape<D, K>;
  const size_t smem = (size_t)KS::SMEM_REALS * sizeof(double);
  auto kern = dev::sipg_rhs_kernel<double, D, K, C, DGX_BASIS, ADV>;
  static std::set<int> configured;
  int devid = 0;
  cuda_check(cudaGetDevice(&devid), "cudaGetDevice");
  {
    std::lock_guard<std::mutex> lk(g_mutex);
    if (!configured.count(devid))
      {
        cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem),
                   "cudaFuncSetAttribute");
        configured.insert(devid);
      }
  }
  const int grid = (prm.n_tasks + KS::NC - 1) / KS::NC;
  if (grid > 0)
    kern<<<grid, KS::THREADS, smem, s>>>(prm);
  cuda_check(cudaGetLastError(), "sipg_rhs_kernel launch");
}

template <int D, bool ADV>
void launch_rhs_d(int K, bool compressed, const dev::RhsParams<double> &prm, cudaStream_t s)
{
  switch (K)
    {
#define DGX_RHS_K(KK)                                                                      \
  case KK:                                                                                 \
    if (compressed)                                                                        \
      launch_rhs_one<D, KK, true, ADV>(prm, s);                                            \
    else                                                                                   \
      launch_rhs_one<D, KK, false, ADV>(prm, s);                                           \
    break;
#ifdef DGX_DEV_K
      DGX_RHS_K(DGX_DEV_K)
#else
#if DGX_BASIS != 2
      DGX_RHS_K(2) DGX_RHS_K(3)
#endif
      DGX_RHS_K(4) DGX_RHS_K(5) DGX_RHS_K(6) DGX_RHS_K(7) DGX_RHS_K(8) DGX_RHS_K(9)
      DGX_RHS_K(10) DGX_RHS_K(11)
#endif
#undef DGX_RHS_K
    default: fail(Code::invalid_argument, "assemble_rhs: unsupported k");
    }
}

} // namespace

void DGX_FN(launch_rhs)(int D, int K, bool compressed, bool adv,
                        const dev::RhsParams<double> &prm, cudaStream_t s)
{
  if (adv)
    {
      if (D == 2)
        launch_rhs_d<2, true>(K, compressed, prm, s);
      else
        launch_rhs_d<3, true>(K, compressed, prm, s);
      return;
    }
  if (D == 2)
    launch_rhs_d<2, false>(K, compressed, prm, s);
  else
    launch_rhs_d<3, false>(K, compressed, prm, s);
}

void DGX_FN(launch_adv)(int D, int K, bool compressed, const dev::AdvParams<double> &prm,
                        cudaStream_t s)
{
#if DGX_BASIS == 2
  (void)D, (void)K, (void)compressed, (void)prm, (void)s;
  fail(Code::invalid_argument,
       "advection: the Hermite-like basis is not implemented for advection on the device");
#else
  if (D == 2)
    launch_adv_d<2>(K, compressed, prm, s);
  else
    launch_adv_d<3>(K, compressed, prm, s);
#endif
}

// Line permutations of the tensor-product kernel (sipg_cart.cuh): thread t of
// a cell owns, in the x- and y-phases, a line whose first entry lies in bank
// (t + beta) mod #banks -- lines are handed out greedily by bank residue, the
// few that do not fit the run fill the gaps.
template <typename Real, int K>
void cart_perm_host(unsigned char (&out)[2][128])
{
  using CS = dev::CartShape<Real, 3, K>;
  constexpr int P = K * K, NB = CS::NBANK;
  for (int A = 0; A < 2; ++A)
    {
      std::vector<int> res(P);
      for (int l = 0; l < P; ++l)
        {
          const int i = l % K, j = l / K;
          res[l] = (A == 0 ? CS::S1 * i + CS::S2 * j : i + CS::S2 * j) % NB;
        }
      int best_bad = 1 << 30, beta = 0;
      for (int b = 0; b < NB; ++b)
        {
          std::vector<int> need(NB, 0), have(NB, 0);
          for (int t = 0; t < P; ++t)
            {
              ++need[(t + b) % NB];
              ++have[res[t]];
            }
          int bad = 0;
          for (int r = 0; r < NB; ++r)
            bad += std::max(0, need[r] - have[r]);
          if (bad < best_bad)
            {
              best_bad = bad;
              beta = b;
            }
        }
      std::vector<int> line_of(P, -1);
      std::vector<char> used(P, 0);
      for (int t = 0; t < P; ++t)
        for (int l = 0; l < P; ++l)
          if (!used[l] && res[l] == (t + beta) % NB)
            {
              line_of[t] = l;
              used[l] = 1;
              break;
            }
      int next = 0;
      for (int t = 0; t < P; ++t)
        if (line_of[t] < 0)
          {
            while (used[next])
              ++next;
            line_of[t] = next;
            used[next] = 1;
          }
      for (int t = 0; t < 128; ++t)
        out[A][t] = static_cast<unsigned char>(t < P ? line_of[t] : 0);
    }
}

template <int K>
void upload_cart_perm()
{
  unsigned char h[2][128];
  cart_perm_host<double, K>(h);
  cuda_check(cudaMemcpyToSymbol(dev::c_cart_perm, h, sizeof h, (size_t)(0 * (dev::kMaxK + 1) + K) * sizeof h),
             "upload line permutations");
  cart_perm_host<float, K>(h);
  cuda_check(cudaMemcpyToSymbol(dev::c_cart_perm, h, sizeof h, (size_t)(1 * (dev::kMaxK + 1) + K) * sizeof h),
             "upload line permutations");
}

void DGX_FN(upload_tables)(int K)
{
  int devid = 0;
  cuda_check(cudaGetDevice(&devid), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_mutex);
  if (g_uploaded.count({devid, K}))
    return;
  const std::vector<double> t = build_table(K);
  std::vector<float> tf(t.begin(), t.end());
  cuda_check(cudaMemcpyToSymbol(dev::c_tab_d, t.data(), t.size() * sizeof(double),
                                dev::tab_offset(K) * sizeof(double)),
             "upload tables");
  cuda_check(cudaMemcpyToSymbol(dev::c_tab_f, tf.data(), tf.size() * sizeof(float),
                                dev::tab_offset(K) * sizeof(float)),
             "upload tables");
  switch (K)
    {
#define DGX_PERM_K(KK)                                                                     \
  case KK: upload_cart_perm<KK>(); break;
      DGX_PERM_K(2) DGX_PERM_K(3) DGX_PERM_K(4) DGX_PERM_K(5) DGX_PERM_K(6) DGX_PERM_K(7)
      DGX_PERM_K(8) DGX_PERM_K(9) DGX_PERM_K(10) DGX_PERM_K(11)
#undef DGX_PERM_K
    default: break;
    }
  g_uploaded.insert({devid, K});
}

template <typename Real>
void DGX_FN(launch_apply)(int D, int K, bool compressed, const dev::ApplyParams<Real> &prm,
                          cudaStream_t s)
{
  if (D == 2)
    launch_d<Real, 2>(K, compressed, prm, s);
  else
    launch_d<Real, 3>(K, compressed, prm, s);
}

template void DGX_FN(launch_apply)<double>(int, int, bool, const dev::ApplyParams<double> &,
                                           cudaStream_t);
#ifdef DGX_WITH_FP32
template void DGX_FN(launch_apply)<float>(int, int, bool, const dev::ApplyParams<float> &,
                                          cudaStream_t);
#endif

} // namespace dgx

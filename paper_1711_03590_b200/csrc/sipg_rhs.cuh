// Right-hand side kernel (RankOperator::assemble_rhs, reference
// operators.cpp:266-282): forcing (add_forcing, :1115-1145) and the
// Dirichlet data moved to the right-hand side by the boundary face kernel in
// rhs mode (process_boundary_batch, :1033-1111):
//   rv = 2 tau g JxW_f,  rw_b = -g JxW_f (n.J^{-T})_b on every boundary face,
//   then the face test (w = rv + sum_t Dco_t^T rw_t, normal part rw_A) and
//   the forcing values f det(J) w_q, all in collocation space, followed by
//   the transposed interpolation S^T x S^T x S^T -- the same test-side
//   algebra as the apply kernel with the trial side replaced by data.
// Included by sipg_launch.cuh (per-basis constant tables).
#pragma once

namespace dgx
{
namespace dev
{

// ADV: the advection operator's boundary data term, (|c.n| - c.n) g JxW_f
// (inflow only, operators.cpp:1053-1060), from the advection face records.
template <typename Real, int D, int K, bool COMPRESSED, int BASIS, bool ADV>
__global__ void __launch_bounds__(KernelShape<D, K>::THREADS)
  sipg_rhs_kernel(const RhsParams<Real> prm)
{
  using KS = KernelShape<D, K>;
  using L = SL<D, K>;
  using T = TabLayout<K>;
  constexpr int P = L::P, NQ = L::NQ, NC = KS::NC, FP = L::FP, NL = L::NL;
  constexpr bool HERM = BASIS == 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Real *smem = reinterpret_cast<Real *>(smem_raw);
  const int lc = threadIdx.x / P;
  const int p = threadIdx.x - lc * P;
  const int task = blockIdx.x * NC + lc;
  const bool active = task < prm.n_tasks;
  Real *cell = smem + lc * L::SM_CELL;
  Real *val = cell;
  const int slot = active ? prm.task_slot[task] : 0;
  const int fp = fpt<D, K>(p);

  // ---- boundary faces: data terms at face point p, per axis ------------
  Real wf = Real(1);
  if constexpr (COMPRESSED)
    {
      int idx = p;
#pragma unroll
      for (int t = 0; t < D - 1; ++t)
        {
          const int qt = idx % K;
          idx /= K;
          Real wa = Real(0);
#pragma unroll
          for (int i = 0; i < K; ++i)
            wa = (qt == i) ? tab<Real, K>(T::oW + i) : wa;
          wf *= wa;
        }
    }
#pragma unroll
  for (int A = 0; A < D; ++A)
    {
      Real *OUT = cell + L::OFF_OUT + (2 * A) * 2 * FP;
      Real *DT = cell + L::OFF_DT;
#pragma unroll
      for (int s = 0; s < 2; ++s)
        {
          Real rv = Real(0), gd[D];
#pragma unroll
          for (int b = 0; b < D; ++b)
            gd[b] = Real(0);
          const int2 tf = active ? prm.task_face[task * 2 * D + 2 * A + s] : make_int2(-2, 0);
          if (tf.x == -1 && prm.g)
            {
              const int fid = tf.y & 0x3fffffff;
              if constexpr (ADV)
                {
                  Real jxw, cn;
                  if constexpr (COMPRESSED)
                    {
                      jxw = prm.face_geo[(long long)fid * 2] * wf;
                      cn = prm.face_geo[(long long)fid * 2 + 1];
                    }
                  else
                    {
                      jxw = prm.face_geo[(long long)fid * 2 * P + p];
                      cn = prm.face_geo[(long long)fid * 2 * P + P + p];
                    }
                  rv = (fabs(cn) - cn) * prm.g[(long long)fid * P + p] * jxw;
                }
              else
                {
                  Real jxw, jo[D];
                  if constexpr (COMPRESSED)
                    {
                      const Real *fg = prm.face_geo + (long long)fid * (2 * D + 1);
                      jxw = fg[0] * wf;
#pragma unroll
                      for (int b = 0; b < D; ++b)
                        jo[b] = fg[1 + b];
                    }
                  else
                    {
                      const Real *fg = prm.face_geo + (long long)fid * (2 * D + 1) * P + p;
                      jxw = fg[0];
#pragma unroll
                      for (int b = 0; b < D; ++b)
                        jo[b] = fg[(1 + b) * P];
                    }
                  const Real gb = prm.g[(long long)fid * P + p] * jxw;
                  rv = gb * prm.penalty[fid] * Real(2);
#pragma unroll
                  for (int b = 0; b < D; ++b)
                    gd[b] = -gb * jo[b];
                }
            }
          OUT[(2 * s) * FP + fp] = rv;
          OUT[(2 * s + 1) * FP + fp] = gd[A];
#pragma unroll
          for (int t = 0; t < D - 1; ++t)
            DT[(2 * t + s) * FP + fp] = gd[t < A ? t : t + 1];
        }
      __syncthreads();
      for (int t = p; t < 2 * NL; t += P)
        {
          const int s = t / NL, l = t - s * NL;
          line_op<Real, D, K, 0, 3>(OUT + 2 * s * FP, DT + s * FP, l);
        }
      if constexpr (D == 3)
        {
          __syncthreads();
          for (int t = p; t < 2 * NL; t += P)
            {
              const int s = t / NL, l = t - s * NL;
              line_op<Real, D, K, 1, 3>(OUT + 2 * s * FP, DT + (2 + s) * FP, l);
            }
        }
      __syncthreads();
    }

  // ---- forcing values + face terms, then S^T in every direction ---------
  {
    Real x[K], z[K], v[K];
#pragma unroll
    for (int m = 0; m < K; ++m)
      {
        const long long q = (long long)slot * NQ + p + P * m; // pencil along D-1
        v[m] = (active && prm.f) ? prm.f[q] * prm.detw[q] : Real(0);
      }
    add_face_terms<Real, D, K, D - 1>(cell, p, v);
    store_pencil<Real, D, K, D - 1>(val, p, v);
    __syncthreads();
    if constexpr (D == 3)
      {
        load_pencil<Real, D, K, 1>(val, p, v);
        add_face_terms<Real, D, K, 1>(cell, p, v);
        store_pencil<Real, D, K, 1>(val, p, v);
        __syncthreads();
      }
    load_pencil<Real, D, K, 0>(val, p, v);
    add_face_terms<Real, D, K, 0>(cell, p, v);
    apply_St<Real, K>(v, z);
    store_pencil<Real, D, K, 0>(val, p, z);
    __syncthreads();
    if constexpr (D == 3)
      {
        load_pencil<Real, D, K, 1>(val, p, x);
        apply_St<Real, K>(x, z);
        store_pencil<Real, D, K, 1>(val, p, z);
        __syncthreads();
      }
    load_pencil<Real, D, K, D - 1>(val, p, x);
    apply_St<Real, K>(x, z);
    if (active)
      {
        Real sp = Real(1);
        if constexpr (HERM)
          {
            sp = hsign<Real, K>(p % K);
            if constexpr (D == 3)
              sp *= hsign<Real, K>(p / K);
          }
        Real *yc = prm.y + (long long)slot * NQ;
#pragma unroll
        for (int m = 0; m < K; ++m)
          yc[p + P * m] = HERM ? z[m] * (sp * hsign<Real, K>(m)) : z[m];
      }
  }
}

} // namespace dev
} // namespace dgx

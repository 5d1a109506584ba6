// Fused cell-centric apply of the advection operator (the paper's other
// operator): OperatorKind::advection of the
// reference, cell term -(c u, grad v) (cell_advection, operators.cpp:634-667)
// and the upwind flux 1/2 c.n (u- + u+) + 1/2 |c.n| (u- - u+) on interior
// faces (:942-960), |c.n| u- on boundary faces (mirror u+ = -u-, :1040-1052).
// Same task lists, thread layout and collocation-space algebra as the
// Laplacian kernel (sipg_kernel.cuh), values only on the faces:
//   forward   val = (S x S x S) u
//   faces     own trace rf.val along the normal, neighbour trace from its
//             nodal face layer (Sf row; one layer for nodal-on-faces bases,
//             read_face_dofs) and two tangential S passes; flux; w = rv
//   cell      t_b = -coef_b val with coef = J^{-1} c det(J) w precomputed
//             (the reference's g3 algebra folded once, its g4 coefficient)
//   backward  S^T x S^T x S^T (sum_b Dco_b^T t_b + rf^T w)
// Included by sipg_launch.cuh (per-basis constant tables). Nodal and generic
// bases only (the reference uses Gauss-Lobatto for advection,
// make_operator_config, operators.cpp:27-41).
#pragma once

namespace dgx
{
namespace dev
{

// One face axis A of every cell in the CTA: both faces' flux values w into
// OUT (values only; the rgn slots are zeroed for the shared backward pass).
template <typename Real, int D, int K, int A, bool COMPRESSED, bool NODAL>
__device__ __forceinline__ void adv_face_axis(const AdvParams<Real> &prm, Real *cell, bool active,
                                              int p, Real wf)
{
  using L = SL<D, K>;
  using T = TabLayout<K>;
  constexpr int P = L::P, NQ = L::NQ, FP = L::FP, NL = L::NL;
  const Real *val = cell;
  Real *NB = cell + L::OFF_NB;
  const int fp = fpt<D, K>(p);
  const int2 *tfs = reinterpret_cast<const int2 *>(cell + L::OFF_TF);
  int2 tf[2] = {make_int2(-2, 0), make_int2(-2, 0)};
  if (active)
    {
      tf[0] = tfs[2 * A];
      tf[1] = tfs[2 * A + 1];
    }
  Real jxw[2], cn[2];
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      jxw[s] = cn[s] = Real(0);
      if (tf[s].x != -2)
        {
          const int fid = tf[s].y & 0x3fffffff;
          if constexpr (COMPRESSED)
            {
              const Real *fr = prm.face + (long long)fid * 2;
              jxw[s] = __ldg(fr) * wf;
              cn[s] = __ldg(fr + 1);
            }
          else
            {
              const Real *fr = prm.face + (long long)fid * 2 * P + p;
              jxw[s] = __ldg(fr);
              cn[s] = __ldg(fr + P);
            }
        }
    }
  // neighbour value layer (own low face meets the neighbour's high face)
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      Real nu = Real(0);
      if (tf[s].x >= 0)
        {
          const Real *un = prm.u + (long long)tf[s].x * NQ;
          const int ro = s == 0 ? K : 0;
          if constexpr (NODAL)
            {
              const int me = s == 0 ? K - 1 : 0;
              nu = tab<Real, K>(T::oSf + ro + me) * __ldg(un + gidx<D, K, A>(p, me));
            }
          else
            {
              Real x[K];
#pragma unroll
              for (int m = 0; m < K; ++m)
                x[m] = __ldg(un + gidx<D, K, A>(p, m));
              nu = s == 0 ? dot_row<Real, K, T::oSf + K>(x) : dot_row<Real, K, T::oSf>(x);
            }
        }
      NB[s * FP + fp] = nu;
    }
  Real own[2];
  {
    Real x[K];
    load_pencil<Real, D, K, A>(val, p, x);
    own[0] = dot_row<Real, K, T::oRf>(x);
    own[1] = dot_row<Real, K, T::oRf + K>(x);
  }
  __syncthreads();
  // tangential interpolation of the neighbour layer to the face points
  if constexpr (D == 3)
    {
      for (int t = p; t < 2 * NL; t += P)
        {
          const int f = t / NL, l = t - f * NL;
          line_op<Real, D, K, 1, 0>(NB + f * FP, nullptr, l);
        }
      __syncthreads();
      for (int t = p; t < 2 * NL; t += P)
        {
          const int f = t / NL, l = t - f * NL;
          line_op<Real, D, K, 0, 0>(NB + f * FP, nullptr, l);
        }
    }
  else
    {
      for (int t = p; t < 2; t += P)
        line_op<Real, D, K, 0, 0>(NB + t * FP, nullptr, 0);
    }
  __syncthreads();
  Real *OUT = cell + L::OFF_OUT + (2 * A) * 2 * FP;
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      Real rv = Real(0);
      if (tf[s].x == -1)
        {
          // mirror u+ = -u-: the flux reduces to |c.n| u-
          rv = fabs(cn[s]) * own[s] * jxw[s];
        }
      else if (tf[s].x >= 0)
        {
          const int side = (tf[s].y >> 30) & 1;
          const Real nu = NB[s * FP + fp];
          const Real um = side == 0 ? own[s] : nu, up = side == 0 ? nu : own[s];
          // advection_numerical_flux (geometry.cpp, operators.cpp:949-957)
          const Real flux = Real(0.5) * cn[s] * (um + up) + Real(0.5) * fabs(cn[s]) * (um - up);
          rv = (side == 0 ? flux : -flux) * jxw[s];
        }
      OUT[(2 * s) * FP + fp] = rv;
      OUT[(2 * s + 1) * FP + fp] = Real(0);
    }
  // NB is rewritten by the next axis only after its own first barrier
}

template <typename Real, int D, int K, bool COMPRESSED, int BASIS>
__global__ void __launch_bounds__(KernelShape<D, K>::THREADS, KernelShape<D, K>::MIN_BLOCKS)
  sipg_adv_kernel(const AdvParams<Real> prm)
{
  using KS = KernelShape<D, K>;
  using L = SL<D, K>;
  using T = TabLayout<K>;
  constexpr int P = L::P, NQ = L::NQ, NC = KS::NC, FS = L::FS;
  // nodal on faces: the value trace reads one layer (read_face_dofs)
  constexpr bool NODAL = BASIS == 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Real *smem = reinterpret_cast<Real *>(smem_raw);

  const int lc = threadIdx.x / P;
  const int p = threadIdx.x - lc * P;
  const int task = blockIdx.x * NC + lc;
  const bool active = task < prm.n_tasks;
  Real *cell = smem + lc * L::SM_CELL;
  Real *val = cell;
  Real *G = cell + L::OFF_G;
  Real *NB = cell + L::OFF_NB;
  const int slot = active ? prm.task_slot[task] : 0;
  const int geo = active ? prm.task_geo[task] : -1;
  const int fp = fpt<D, K>(p);

  unsigned gmask = (1u << K) - 1u;
  if (active)
    {
      for (int i = p; i < 2 * D; i += P)
        reinterpret_cast<int2 *>(cell + L::OFF_TF)[i] = prm.task_face[task * 2 * D + i];
      if (NODAL && slot >= prm.n_owned)
        {
          // ghost cell: only the face layers the exchange ships
          int2 tf[2 * D];
#pragma unroll
          for (int phi = 0; phi < 2 * D; ++phi)
            tf[phi] = prm.task_face[task * 2 * D + phi];
          gmask = ghost_layer_mask<D, K, 1>(tf, p);
        }
    }

  // ---- forward: val = (S x S x S) u --------------------------------------
  {
    Real x[K], z[K];
    const Real *uc = prm.u + (long long)slot * NQ;
#pragma unroll
    for (int m = 0; m < K; ++m)
      x[m] = (active && ((gmask >> m) & 1u)) ? __ldg(uc + p + P * m) : Real(0);
    apply_S<Real, K>(x, z);
    store_pencil<Real, D, K, D - 1>(val, p, z);
    __syncthreads();
    load_pencil<Real, D, K, 0>(val, p, x);
    apply_S<Real, K>(x, z);
    store_pencil<Real, D, K, 0>(val, p, z);
    if constexpr (D == 3)
      {
        __syncthreads();
        load_pencil<Real, D, K, 1>(val, p, x);
        apply_S<Real, K>(x, z);
        store_pencil<Real, D, K, 1>(val, p, z);
      }
  }
  __syncthreads();

  // ---- faces -------------------------------------------------------------
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
  adv_face_axis<Real, D, K, 0, COMPRESSED, NODAL>(prm, cell, active, p, wf);
  adv_face_axis<Real, D, K, 1, COMPRESSED, NODAL>(prm, cell, active, p, wf);
  if constexpr (D == 3)
    adv_face_axis<Real, D, K, 2, COMPRESSED, NODAL>(prm, cell, active, p, wf);

  // ---- cell term t_b = -coef_b u at every quadrature point ----------------
  {
    constexpr int NG = D;
    const Real *cg = prm.cell + (long long)(geo >= 0 ? geo : 0) * NG * (COMPRESSED ? 1 : NQ);
    Real wxy = Real(1);
    if constexpr (COMPRESSED)
      {
        const int qa0 = p % K;
        Real wa = Real(0);
#pragma unroll
        for (int i = 0; i < K; ++i)
          wa = (qa0 == i) ? tab<Real, K>(T::oW + i) : wa;
        wxy *= wa;
        if constexpr (D == 3)
          {
            const int qa1 = p / K;
            wa = Real(0);
#pragma unroll
            for (int i = 0; i < K; ++i)
              wa = (qa1 == i) ? tab<Real, K>(T::oW + i) : wa;
            wxy *= wa;
          }
      }
#pragma unroll
    for (int m = 0; m < K; ++m)
      {
        const int q = pidx<D, K, D - 1>(p, m);
        const Real uq = val[q];
#pragma unroll
        for (int b = 0; b < D; ++b)
          {
            Real c = Real(0);
            if (geo >= 0)
              c = COMPRESSED ? __ldg(cg + b) * (wxy * tab<Real, K>(T::oW + m))
                             : __ldcs(cg + b * NQ + p + P * m);
            G[b * FS + q] = -(c * uq);
          }
      }
  }
  __syncthreads();

  // ---- backward: y = (S^T x S^T x S^T)(sum_b Dco_b^T t_b + rf^T w) ---------
  {
    Real x[K], z[K], v[K];
    if constexpr (D == 3)
      {
        load_pencil<Real, D, K, 2>(G + 2 * FS, p, x);
        apply_Dt<Real, K>(x, v);
        add_face_terms<Real, D, K, 2>(cell, p, v);
        store_pencil<Real, D, K, 2>(val, p, v);
        __syncthreads();
        load_pencil<Real, D, K, 1>(G + FS, p, x);
        apply_Dt<Real, K>(x, z);
        load_pencil<Real, D, K, 1>(val, p, v);
#pragma unroll
        for (int m = 0; m < K; ++m)
          v[m] += z[m];
      }
    else
      {
        load_pencil<Real, D, K, 1>(G + FS, p, x);
        apply_Dt<Real, K>(x, v);
      }
    add_face_terms<Real, D, K, 1>(cell, p, v);
    store_pencil<Real, D, K, 1>(val, p, v);
    __syncthreads();
    load_pencil<Real, D, K, 0>(G, p, x);
    apply_Dt<Real, K>(x, z);
    load_pencil<Real, D, K, 0>(val, p, v);
#pragma unroll
    for (int m = 0; m < K; ++m)
      v[m] += z[m];
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
        Real *yc = prm.y + (long long)slot * NQ;
#pragma unroll
        for (int m = 0; m < K; ++m)
          yc[p + P * m] = ((gmask >> m) & 1u) ? z[m] : Real(0);
      }
  }
}

} // namespace dev
} // namespace dgx

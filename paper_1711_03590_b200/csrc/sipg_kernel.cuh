// Fused cell-centric SIPG-Laplacian apply for sm_100a.
//
// One task = one cell slot of the rank-local vector. A task computes
//   (a) the cell integral (J^{-1}J^{-T} grad u, grad v) JxW
//       (reference operators.cpp:669-749, tensor_kernels.hpp:334-416), and
//   (b) its own side of every face integral that this rank computes and
//       that touches the cell (operators.cpp:933-1111),
// and writes y for the cell exactly once: no atomics, no read-modify-write
// of y in HBM, deterministic.
//
// Everything happens in collocation space (Gauss points). With S the k x k
// nodal-to-Gauss interpolation, val = (S x S x S) u and g_b = Dco_b val.
// Own face traces are 1D row contractions of (val, g) along the face normal
// with rf = Sf S^{-1} (Lagrange extrapolation from the Gauss points); their
// transposes add the face residuals into the collocation test arrays. The
// neighbour trace is evaluated reference-style from its nodal values
// (Sf/Df row along the normal, S sweeps and Dco along the face), so a
// neighbour costs O(k^d) reads and O(k^d) flops instead of a full transform.
// Both forms are algebraically identical to the reference's (S invertible,
// all interpolations exact on the polynomial space); only round-off differs.
//
// Thread layout: P = K^{D-1} "pencil" threads per cell, NC cells per CTA.
// A pass along axis a: thread p owns the 1D line ("pencil") along a through
// the other coordinates p, keeps K values in registers and applies the 1D
// matrix in even-odd form (reference tensor_kernels.hpp:54-137, Eq. 8 of
// the paper) with the matrix entries as constant-bank operands.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace dgx
{
namespace dev
{

constexpr int ipow_c(int b, int e) { return e == 0 ? 1 : b * ipow_c(b, e - 1); }

// ---- per-K 1D tables in constant memory ---------------------------------

template <int K>
struct TabLayout
{
  static constexpr int CE = (K + 1) / 2;
  static constexpr int H = K / 2;
  // even-odd halves, each [CE][CE] (zero padded), of S, S^T, Dco, Dco^T
  static constexpr int oSE = 0, oSO = oSE + CE * CE;
  static constexpr int oStE = oSO + CE * CE, oStO = oStE + CE * CE;
  static constexpr int oDE = oStO + CE * CE, oDO = oDE + CE * CE;
  static constexpr int oDtE = oDO + CE * CE, oDtO = oDtE + CE * CE;
  static constexpr int oS = oDtO + CE * CE;  // plain S, K x K
  static constexpr int oD = oS + K * K;      // plain Dco, K x K
  static constexpr int oSf = oD + K * K;     // Sf[2][K]
  static constexpr int oDf = oSf + 2 * K;    // Df[2][K]
  static constexpr int oRf = oDf + 2 * K;    // rf[2][K]
  static constexpr int oW = oRf + 2 * K;     // Gauss weights [K]
  static constexpr int size = oW + K;
};

constexpr int tab_size(int K) { return 8 * ((K + 1) / 2) * ((K + 1) / 2) + 2 * K * K + 7 * K; }
// offset of the table for K (K >= 2) inside the per-precision constant block
constexpr int tab_offset(int K) { return K <= 2 ? 0 : tab_offset(K - 1) + tab_size(K - 1); }
constexpr int kMaxK = 11;
constexpr int kTabTotal = tab_offset(kMaxK + 1);

extern __constant__ double c_tab_d[kTabTotal];
extern __constant__ float c_tab_f[kTabTotal];

template <typename Real>
__device__ __forceinline__ const Real *tab_base();
template <>
__device__ __forceinline__ const double *tab_base<double>() { return c_tab_d; }
template <>
__device__ __forceinline__ const float *tab_base<float>() { return c_tab_f; }

template <typename Real, int K>
__device__ __forceinline__ Real tab(int i) { return tab_base<Real>()[tab_offset(K) + i]; }

// ---- 1D operators in registers -------------------------------------------

// y = M x, M mirror-symmetric (M[q][j] = M[K-1-q][K-1-j]).
template <typename Real, int K, int OE, int OO>
__device__ __forceinline__ void eo_sym(const Real (&x)[K], Real (&y)[K])
{
  constexpr int H = K / 2, CE = (K + 1) / 2;
  Real xe[CE], xo[H > 0 ? H : 1];
#pragma unroll
  for (int j = 0; j < H; ++j)
    {
      xe[j] = x[j] + x[K - 1 - j];
      xo[j] = x[j] - x[K - 1 - j];
    }
  if (K & 1)
    xe[H] = x[H];
#pragma unroll
  for (int q = 0; q < H; ++q)
    {
      Real e = xe[0] * tab<Real, K>(OE + q * CE);
#pragma unroll
      for (int j = 1; j < CE; ++j)
        e += xe[j] * tab<Real, K>(OE + q * CE + j);
      Real o = xo[0] * tab<Real, K>(OO + q * CE);
#pragma unroll
      for (int j = 1; j < H; ++j)
        o += xo[j] * tab<Real, K>(OO + q * CE + j);
      y[q] = e + o;
      y[K - 1 - q] = e - o;
    }
  if (K & 1)
    {
      Real e = xe[0] * tab<Real, K>(OE + H * CE);
#pragma unroll
      for (int j = 1; j < CE; ++j)
        e += xe[j] * tab<Real, K>(OE + H * CE + j);
      y[H] = e;
    }
}

// y = M x, M mirror-skew (M[q][j] = -M[K-1-q][K-1-j]).
template <typename Real, int K, int OE, int OO>
__device__ __forceinline__ void eo_skew(const Real (&x)[K], Real (&y)[K])
{
  constexpr int H = K / 2, CE = (K + 1) / 2;
  Real xe[CE], xo[H > 0 ? H : 1];
#pragma unroll
  for (int j = 0; j < H; ++j)
    {
      xe[j] = x[j] + x[K - 1 - j];
      xo[j] = x[j] - x[K - 1 - j];
    }
  if (K & 1)
    xe[H] = x[H];
#pragma unroll
  for (int q = 0; q < H; ++q)
    {
      Real a = xo[0] * tab<Real, K>(OO + q * CE);
#pragma unroll
      for (int j = 1; j < H; ++j)
        a += xo[j] * tab<Real, K>(OO + q * CE + j);
      Real b = xe[0] * tab<Real, K>(OE + q * CE);
#pragma unroll
      for (int j = 1; j < CE; ++j)
        b += xe[j] * tab<Real, K>(OE + q * CE + j);
      y[q] = a + b;
      y[K - 1 - q] = a - b;
    }
  if (K & 1)
    {
      Real a = xo[0] * tab<Real, K>(OO + H * CE);
#pragma unroll
      for (int j = 1; j < H; ++j)
        a += xo[j] * tab<Real, K>(OO + H * CE + j);
      y[H] = a;
    }
}

template <typename Real, int K>
__device__ __forceinline__ void apply_S(const Real (&x)[K], Real (&y)[K])
{
  eo_sym<Real, K, TabLayout<K>::oSE, TabLayout<K>::oSO>(x, y);
}
template <typename Real, int K>
__device__ __forceinline__ void apply_St(const Real (&x)[K], Real (&y)[K])
{
  eo_sym<Real, K, TabLayout<K>::oStE, TabLayout<K>::oStO>(x, y);
}
template <typename Real, int K>
__device__ __forceinline__ void apply_D(const Real (&x)[K], Real (&y)[K])
{
  eo_skew<Real, K, TabLayout<K>::oDE, TabLayout<K>::oDO>(x, y);
}
template <typename Real, int K>
__device__ __forceinline__ void apply_Dt(const Real (&x)[K], Real (&y)[K])
{
  eo_skew<Real, K, TabLayout<K>::oDtE, TabLayout<K>::oDtO>(x, y);
}

template <typename Real, int K, int OFF>
__device__ __forceinline__ Real dot_row(const Real (&x)[K])
{
  Real s = x[0] * tab<Real, K>(OFF);
#pragma unroll
  for (int m = 1; m < K; ++m)
    s += x[m] * tab<Real, K>(OFF + m);
  return s;
}

// ---- pencil indexing ---------------------------------------------------

// Cell-local linear index of the m-th entry along axis A of pencil p (the
// remaining axes enumerated ascending, lowest fastest: identical to the
// reference face quadrature-point order, geometry.cpp:423-431).
template <int D, int K, int A>
__device__ __forceinline__ int pidx(int p, int m)
{
  if constexpr (A == 0)
    return m + K * p;
  else if constexpr (D == 2)
    return p + K * m;
  else if constexpr (A == 1)
    return (p % K) + K * m + K * K * (p / K);
  else
    return p + K * K * m;
}

// Index on the (D-1)-dimensional face grid of the i-th point along the
// tangential direction T (0 or 1) through face point p.
template <int D, int K, int T>
__device__ __forceinline__ int fidx(int p, int i)
{
  if constexpr (D == 2)
    return i;
  else if constexpr (T == 0)
    return i + K * (p / K);
  else
    return (p % K) + K * i;
}
template <int D, int K, int T>
__device__ __forceinline__ int fcoord(int p)
{
  if constexpr (D == 2)
    return p;
  else if constexpr (T == 0)
    return p % K;
  else
    return p / K;
}

// ---- kernel parameters ---------------------------------------------------

// task_face[t * 2D + phi]: x = neighbour slot, or -1 (boundary face), or -2
// (face not computed on this rank: its contribution arrives by compress);
// y = local face record | (own side << 30).
template <typename Real>
struct ApplyParams
{
  const Real *u;
  Real *y;
  const Real *cell_geo; // [geo][D*D+1][NQ] or compressed [geo][D*D+1]
  const Real *face_geo; // [face][2D+1][P]: JxW_f, n.J^{-T}(e-), n.J^{-T}(e+)
  const Real *penalty;  // [face]
  const int *task_slot;
  const int *task_geo;  // cell geometry record, -1: no cell integral
  const int2 *task_face;
  int n_tasks;
};

template <int D, int K>
struct KernelShape
{
  static constexpr int P = ipow_c(K, D - 1);
  static constexpr int NQ = ipow_c(K, D);
  // shared doubles per cell: val + D gradient fields + 4 face fields
  static constexpr int SM_CELL = (D + 1) * NQ + 4 * P;
  static constexpr int NC_THREADS = (256 / P) > 0 ? 256 / P : 1;
  static constexpr int NC_SMEM = (96 * 1024 / 8) / SM_CELL > 0 ? (96 * 1024 / 8) / SM_CELL : 1;
  static constexpr int NC = NC_THREADS < NC_SMEM ? NC_THREADS : NC_SMEM;
  static constexpr int THREADS = NC * P;
};

template <typename Real, int D, int K, int A>
__device__ __forceinline__ void load_pencil(const Real *arr, int p, Real (&x)[K])
{
#pragma unroll
  for (int m = 0; m < K; ++m)
    x[m] = arr[pidx<D, K, A>(p, m)];
}
template <typename Real, int D, int K, int A>
__device__ __forceinline__ void store_pencil(Real *arr, int p, const Real (&x)[K])
{
#pragma unroll
  for (int m = 0; m < K; ++m)
    arr[pidx<D, K, A>(p, m)] = x[m];
}

// Own-side residuals of one face: value test rv and gradient test rg[D]
template <typename Real, int D>
struct FaceRes
{
  Real rv;
  Real rg[D];
};

// Neighbour trace of u across the face of axis A, then the face integral
// flux; writes the own residuals. F: 4 x P shared scratch of this cell.
template <typename Real, int D, int K, int A>
__device__ __forceinline__ void face_axis(const ApplyParams<Real> &prm,
                                          const Real *val, const Real *G,
                                          Real *F, int task, bool active,
                                          int p, FaceRes<Real, D> (&res)[2])
{
  constexpr int P = KernelShape<D, K>::P;
  constexpr int NQ = KernelShape<D, K>::NQ;
  using L = TabLayout<K>;

  // own traces: value and reference gradient at the face points of both
  // faces (x_A = 0: s = 0, x_A = 1: s = 1), rf-extrapolated
  Real own_u[2], own_g[2][D];
  {
    Real x[K];
    load_pencil<Real, D, K, A>(val, p, x);
    own_u[0] = dot_row<Real, K, L::oRf>(x);
    own_u[1] = dot_row<Real, K, L::oRf + K>(x);
#pragma unroll
    for (int b = 0; b < D; ++b)
      {
        load_pencil<Real, D, K, A>(G + b * NQ, p, x);
        own_g[0][b] = dot_row<Real, K, L::oRf>(x);
        own_g[1][b] = dot_row<Real, K, L::oRf + K>(x);
      }
  }

  // neighbour nodal traces: value row Sf and normal derivative row Df of
  // the neighbour's opposite face (neighbour face number = phi ^ 1)
  int2 tf[2] = {make_int2(-2, 0), make_int2(-2, 0)};
  if (active)
    {
      tf[0] = prm.task_face[task * 2 * D + 2 * A];
      tf[1] = prm.task_face[task * 2 * D + 2 * A + 1];
    }
  Real nu[2], nw[2];
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      nu[s] = Real(0);
      nw[s] = Real(0);
      if (tf[s].x >= 0)
        {
          const Real *un = prm.u + (long long)tf[s].x * NQ;
          Real x[K];
#pragma unroll
          for (int m = 0; m < K; ++m)
            x[m] = __ldg(un + pidx<D, K, A>(p, m));
          // own low face (s = 0) meets the neighbour's high face (1) and
          // vice versa
          if (s == 0)
            {
              nu[s] = dot_row<Real, K, L::oSf + K>(x);
              nw[s] = dot_row<Real, K, L::oDf + K>(x);
            }
          else
            {
              nu[s] = dot_row<Real, K, L::oSf>(x);
              nw[s] = dot_row<Real, K, L::oDf>(x);
            }
        }
    }

  // tangential S sweeps of (nu, nw) for both faces on the face grid, then
  // tangential Dco derivatives of nu (operators.cpp:766-788)
  Real *F0 = F, *F1 = F + P, *F2 = F + 2 * P, *F3 = F + 3 * P;
  F0[p] = nu[0];
  F1[p] = nw[0];
  F2[p] = nu[1];
  F3[p] = nw[1];
  __syncthreads();
  Real dt[2][D > 1 ? D - 1 : 1];
  {
    // sweep along tangential direction 0
    const int i0 = fcoord<D, K, 0>(p);
    Real t0 = 0, t1 = 0, t2 = 0, t3 = 0;
#pragma unroll
    for (int m = 0; m < K; ++m)
      {
        const Real s = tab<Real, K>(L::oS + i0 * K + m);
        const int f = fidx<D, K, 0>(p, m);
        t0 += s * F0[f];
        t1 += s * F1[f];
        t2 += s * F2[f];
        t3 += s * F3[f];
      }
    __syncthreads();
    F0[p] = t0;
    F1[p] = t1;
    F2[p] = t2;
    F3[p] = t3;
    __syncthreads();
    if constexpr (D == 3)
      {
        const int i1 = fcoord<D, K, 1>(p);
        t0 = t1 = t2 = t3 = 0;
#pragma unroll
        for (int m = 0; m < K; ++m)
          {
            const Real s = tab<Real, K>(L::oS + i1 * K + m);
            const int f = fidx<D, K, 1>(p, m);
            t0 += s * F0[f];
            t1 += s * F1[f];
            t2 += s * F2[f];
            t3 += s * F3[f];
          }
        __syncthreads();
        F0[p] = t0;
        F1[p] = t1;
        F2[p] = t2;
        F3[p] = t3;
        __syncthreads();
      }
    nu[0] = t0;
    nw[0] = t1;
    nu[1] = t2;
    nw[1] = t3;
    // tangential derivatives of nu
#pragma unroll
    for (int t = 0; t < D - 1; ++t)
      {
        Real a0 = 0, a1 = 0;
        if (t == 0)
          {
            const int i = fcoord<D, K, 0>(p);
#pragma unroll
            for (int m = 0; m < K; ++m)
              {
                const Real dd = tab<Real, K>(L::oD + i * K + m);
                a0 += dd * F0[fidx<D, K, 0>(p, m)];
                a1 += dd * F2[fidx<D, K, 0>(p, m)];
              }
          }
        else
          {
            const int i = fcoord<D, K, (D == 3 ? 1 : 0)>(p);
#pragma unroll
            for (int m = 0; m < K; ++m)
              {
                const Real dd = tab<Real, K>(L::oD + i * K + m);
                a0 += dd * F0[fidx<D, K, (D == 3 ? 1 : 0)>(p, m)];
                a1 += dd * F2[fidx<D, K, (D == 3 ? 1 : 0)>(p, m)];
              }
          }
        dt[0][t] = a0;
        dt[1][t] = a1;
      }
  }

  // flux (operators.cpp:977-1003 interior, 1069-1089 boundary)
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      res[s].rv = Real(0);
#pragma unroll
      for (int b = 0; b < D; ++b)
        res[s].rg[b] = Real(0);
      if (tf[s].x == -2)
        continue;
      const int fid = tf[s].y & 0x3fffffff;
      const int side = (tf[s].y >> 30) & 1;
      const Real *fg = prm.face_geo + (long long)fid * (2 * D + 1) * P;
      const Real jxw = fg[p];
      Real jni[D], jne[D];
#pragma unroll
      for (int b = 0; b < D; ++b)
        {
          jni[b] = fg[(1 + b) * P + p];
          jne[b] = fg[(1 + D + b) * P + p];
        }
      const Real tau = prm.penalty[fid];
      Real jo[D], jnb[D];
#pragma unroll
      for (int b = 0; b < D; ++b)
        {
          jo[b] = side == 0 ? jni[b] : jne[b];
          jnb[b] = side == 0 ? jne[b] : jni[b];
        }
      Real dn_own = own_g[s][0] * jo[0];
#pragma unroll
      for (int b = 1; b < D; ++b)
        dn_own += own_g[s][b] * jo[b];
      Real g;
      if (tf[s].x == -1)
        {
          res[s].rv = (own_u[s] * tau * Real(2) - dn_own) * jxw;
          g = -(own_u[s] * jxw);
        }
      else
        {
          // neighbour reference gradient: normal comp A = nw, tangential = dt
          Real dn_nb = Real(0);
#pragma unroll
          for (int b = 0; b < D; ++b)
            dn_nb += (b == A ? nw[s] : dt[s][b < A ? b : b - 1]) * jnb[b];
          const Real um = side == 0 ? own_u[s] : nu[s];
          const Real up = side == 0 ? nu[s] : own_u[s];
          const Real dm = side == 0 ? dn_own : dn_nb;
          const Real dp = side == 0 ? dn_nb : dn_own;
          const Real jump = um - up;
          const Real r0 = (jump * tau - (dm + dp) * Real(0.5)) * jxw;
          res[s].rv = side == 0 ? r0 : -r0;
          g = -(jump * jxw * Real(0.5));
        }
#pragma unroll
      for (int b = 0; b < D; ++b)
        res[s].rg[b] = g * jo[b];
    }
}

// Transposed face trace: add rf^T rv into the value test field and
// rf^T rg[b] into the gradient test fields along pencils of axis A.
template <typename Real, int D, int K, int A>
__device__ __forceinline__ void face_distribute(Real *val, Real *G, int p,
                                                const FaceRes<Real, D> (&res)[2])
{
  constexpr int NQ = KernelShape<D, K>::NQ;
  using L = TabLayout<K>;
#pragma unroll
  for (int m = 0; m < K; ++m)
    {
      const int i = pidx<D, K, A>(p, m);
      const Real r0 = tab<Real, K>(L::oRf + m), r1 = tab<Real, K>(L::oRf + K + m);
      val[i] += r0 * res[0].rv + r1 * res[1].rv;
#pragma unroll
      for (int b = 0; b < D; ++b)
        G[b * NQ + i] += r0 * res[0].rg[b] + r1 * res[1].rg[b];
    }
}

template <typename Real, int D, int K, bool COMPRESSED>
__global__ void __launch_bounds__(KernelShape<D, K>::THREADS)
  sipg_apply_kernel(const ApplyParams<Real> prm)
{
  using KS = KernelShape<D, K>;
  constexpr int P = KS::P, NQ = KS::NQ, NC = KS::NC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Real *smem = reinterpret_cast<Real *>(smem_raw);

  const int lc = threadIdx.x / P;
  const int p = threadIdx.x - lc * P;
  const int task = blockIdx.x * NC + lc;
  const bool active = task < prm.n_tasks;
  Real *val = smem + lc * KS::SM_CELL;
  Real *G = val + NQ;
  Real *F = G + D * NQ;

  const int slot = active ? prm.task_slot[task] : 0;
  const int geo = active ? prm.task_geo[task] : -1;

  // 1. own values; thread p reads the pencil along axis D-1 (coalesced) and
  //    interpolates it to the Gauss points in registers
  {
    Real x[K], z[K];
    const Real *uc = prm.u + (long long)slot * NQ;
#pragma unroll
    for (int m = 0; m < K; ++m)
      x[m] = active ? __ldg(uc + p + P * m) : Real(0);
    apply_S<Real, K>(x, z);
    store_pencil<Real, D, K, D - 1>(val, p, z);
  }
  __syncthreads();
  // 2. remaining interpolation passes
#pragma unroll
  for (int a = 0; a < D - 1; ++a)
    {
      Real x[K], z[K];
      if (a == 0)
        {
          load_pencil<Real, D, K, 0>(val, p, x);
          apply_S<Real, K>(x, z);
          store_pencil<Real, D, K, 0>(val, p, z);
        }
      else
        {
          load_pencil<Real, D, K, 1>(val, p, x);
          apply_S<Real, K>(x, z);
          store_pencil<Real, D, K, 1>(val, p, z);
        }
      __syncthreads();
    }
  // 3. reference gradient in collocation space: G[b] = Dco_b val
  {
    Real x[K], z[K];
    load_pencil<Real, D, K, 0>(val, p, x);
    apply_D<Real, K>(x, z);
    store_pencil<Real, D, K, 0>(G, p, z);
    load_pencil<Real, D, K, 1>(val, p, x);
    apply_D<Real, K>(x, z);
    store_pencil<Real, D, K, 1>(G + NQ, p, z);
    if constexpr (D == 3)
      {
        load_pencil<Real, D, K, 2>(val, p, x);
        apply_D<Real, K>(x, z);
        store_pencil<Real, D, K, 2>(G + 2 * NQ, p, z);
      }
  }
  __syncthreads();

  // 4. faces, axis by axis; own residuals stay in registers
  FaceRes<Real, D> r0[2], r1[2], r2[2];
  face_axis<Real, D, K, 0>(prm, val, G, F, task, active, p, r0);
  face_axis<Real, D, K, 1>(prm, val, G, F, task, active, p, r1);
  if constexpr (D == 3)
    face_axis<Real, D, K, 2>(prm, val, G, F, task, active, p, r2);
  __syncthreads();

  // 5. quadrature-point operation t = J^{-1} J^{-T} g JxW
  //    (operators.cpp:669-709); thread p handles the points p + P m
#pragma unroll
  for (int m = 0; m < K; ++m)
    {
      const int q = p + P * m;
      Real g[D];
#pragma unroll
      for (int b = 0; b < D; ++b)
        g[b] = G[b * NQ + q];
      Real t[D];
      if (geo >= 0)
        {
          Real jit[D * D], jxw;
          if constexpr (COMPRESSED)
            {
              const Real *cg = prm.cell_geo + (long long)geo * (D * D + 1);
#pragma unroll
              for (int c = 0; c < D * D; ++c)
                jit[c] = __ldg(cg + c);
              // wq_cell[q] = prod_a w[q_a] (geometry.cpp:285-296)
              Real w = Real(1);
              int idx = q;
#pragma unroll
              for (int a = 0; a < D; ++a)
                {
                  int qa = idx % K;
                  idx /= K;
                  Real wa = Real(0);
#pragma unroll
                  for (int i = 0; i < K; ++i)
                    wa = (qa == i) ? tab<Real, K>(TabLayout<K>::oW + i) : wa;
                  w *= wa;
                }
              jxw = __ldg(cg + D * D) * w;
            }
          else
            {
              const Real *cg = prm.cell_geo + (long long)geo * (D * D + 1) * NQ + q;
#pragma unroll
              for (int c = 0; c < D * D; ++c)
                jit[c] = __ldg(cg + c * NQ);
              jxw = __ldg(cg + D * D * NQ);
            }
          Real ph[D];
#pragma unroll
          for (int i = 0; i < D; ++i)
            {
              Real acc = jit[i * D] * g[0];
#pragma unroll
              for (int j = 1; j < D; ++j)
                acc += jit[i * D + j] * g[j];
              ph[i] = acc;
            }
#pragma unroll
          for (int i = 0; i < D; ++i)
            {
              Real acc = jit[i] * ph[0];
#pragma unroll
              for (int j = 1; j < D; ++j)
                acc += jit[j * D + i] * ph[j];
              t[i] = acc * jxw;
            }
        }
      else
        {
#pragma unroll
          for (int b = 0; b < D; ++b)
            t[b] = Real(0);
        }
#pragma unroll
      for (int b = 0; b < D; ++b)
        G[b * NQ + q] = t[b];
      val[q] = Real(0);
    }
  __syncthreads();

  // 6. face residuals into the collocation test fields
  face_distribute<Real, D, K, 0>(val, G, p, r0);
  __syncthreads();
  face_distribute<Real, D, K, 1>(val, G, p, r1);
  __syncthreads();
  if constexpr (D == 3)
    {
      face_distribute<Real, D, K, 2>(val, G, p, r2);
      __syncthreads();
    }

  // 7. val += sum_b Dco_b^T G[b]
  {
    Real x[K], z[K], v[K];
    load_pencil<Real, D, K, 0>(G, p, x);
    apply_Dt<Real, K>(x, z);
    load_pencil<Real, D, K, 0>(val, p, v);
#pragma unroll
    for (int m = 0; m < K; ++m)
      v[m] += z[m];
    store_pencil<Real, D, K, 0>(val, p, v);
    __syncthreads();
    load_pencil<Real, D, K, 1>(G + NQ, p, x);
    apply_Dt<Real, K>(x, z);
    load_pencil<Real, D, K, 1>(val, p, v);
#pragma unroll
    for (int m = 0; m < K; ++m)
      v[m] += z[m];
    if constexpr (D == 3)
      {
        store_pencil<Real, D, K, 1>(val, p, v);
        __syncthreads();
        load_pencil<Real, D, K, 2>(G + 2 * NQ, p, x);
        apply_Dt<Real, K>(x, z);
        load_pencil<Real, D, K, 2>(val, p, v);
#pragma unroll
        for (int m = 0; m < K; ++m)
          v[m] += z[m];
        // axis 2 is the last S^T pass as well: keep it in registers below
        apply_St<Real, K>(v, z);
        store_pencil<Real, D, K, 2>(val, p, z);
      }
    else
      {
        apply_St<Real, K>(v, z);
        store_pencil<Real, D, K, 1>(val, p, z);
      }
    __syncthreads();
  }
  // 8. remaining S^T passes; the last one goes straight to y (pencil along
  //    axis D-1 first was done above, so here axes 0 .. D-2)
  {
    Real x[K], z[K];
    if constexpr (D == 3)
      {
        load_pencil<Real, D, K, 1>(val, p, x);
        apply_St<Real, K>(x, z);
        store_pencil<Real, D, K, 1>(val, p, z);
        __syncthreads();
      }
    // axis 0 pencil; thread p then writes its own pencil along axis 0
    load_pencil<Real, D, K, 0>(val, p, x);
    apply_St<Real, K>(x, z);
    store_pencil<Real, D, K, 0>(val, p, z);
    __syncthreads();
    if (active)
      {
        Real *yc = prm.y + (long long)slot * NQ;
#pragma unroll
        for (int m = 0; m < K; ++m)
          yc[p + P * m] = val[p + P * m];
      }
  }
}

} // namespace dev
} // namespace dgx

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
  static constexpr int oRD = oW + K;         // (rf Dco)[2][K] = (Dco^T rf^T)
  static constexpr int size = oRD + 2 * K;
};

constexpr int tab_size(int K) { return 8 * ((K + 1) / 2) * ((K + 1) / 2) + 2 * K * K + 9 * K; }
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

// ---- shared-memory layout -------------------------------------------------

// Volume fields use a padded row stride S1 (odd for even K) so pencils along
// axis 0 -- consecutive threads K entries apart -- are free of fp64 bank
// conflicts; face fields (k^{d-1} points) likewise use row stride FK.
// Global (HBM) cell data stays unpadded lexicographic, axis 0 fastest.
template <int D, int K>
struct SL
{
  static constexpr int P = ipow_c(K, D - 1);
  static constexpr int NQ = ipow_c(K, D);
  static constexpr int S1 = K + ((K % 2 == 0) ? 1 : 0);
  static constexpr int S2 = S1 * K;
  static constexpr int FS = D == 2 ? S1 * K : S2 * K; // padded volume field
  static constexpr int FK = D == 3 ? S1 : K;          // face row stride
  static constexpr int FP = D == 3 ? FK * K : K;      // padded face field
  static constexpr int NL = P / K;                    // lines per face field
  static constexpr int OFF_G = FS;                    // D gradient / test fields
  static constexpr int OFF_OUT = (D + 1) * FS;        // 2D faces x (w, rgn)
  static constexpr int OFF_NB = OFF_OUT + 4 * D * FP; // nu_lo, nw_lo, nu_hi, nw_hi
  static constexpr int OFF_OWN = OFF_NB + 4 * FP;     // ou_lo, ou_hi
  static constexpr int OFF_DT = OFF_OWN + 2 * FP;     // 4(D-1) derivative fields
  static constexpr int SM_CELL = OFF_DT + 4 * (D - 1) * FP;
};

// index of the m-th entry along axis A of pencil p (remaining axes
// ascending, lowest fastest: the reference face quadrature-point order,
// geometry.cpp:423-431); S1/S2 = row/plane strides
template <int D, int K, int A, int S1, int S2>
__device__ __forceinline__ int lidx(int p, int m)
{
  if constexpr (D == 2)
    return A == 0 ? m + S1 * p : p + S1 * m;
  else if constexpr (A == 0)
    return m + S1 * (p % K) + S2 * (p / K);
  else if constexpr (A == 1)
    return (p % K) + S1 * m + S2 * (p / K);
  else
    return (p % K) + S1 * (p / K) + S2 * m;
}
template <int D, int K, int A>
__device__ __forceinline__ int pidx(int p, int m) // shared (padded)
{
  return lidx<D, K, A, SL<D, K>::S1, SL<D, K>::S2>(p, m);
}
template <int D, int K, int A>
__device__ __forceinline__ int gidx(int p, int m) // global (unpadded)
{
  return lidx<D, K, A, K, K * K>(p, m);
}
// face field: point p, and the m-th point of line l along tangential dir T
template <int D, int K>
__device__ __forceinline__ int fpt(int p)
{
  if constexpr (D == 2)
    return p;
  else
    return (p % K) + SL<D, K>::FK * (p / K);
}
template <int D, int K, int T>
__device__ __forceinline__ int fln(int l, int m)
{
  if constexpr (D == 2)
    return m;
  else if constexpr (T == 0)
    return m + SL<D, K>::FK * l;
  else
    return l + SL<D, K>::FK * m;
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
  using L = SL<D, K>;
  static constexpr int P = L::P;
  static constexpr int NQ = L::NQ;
  static constexpr int SM_CELL = L::SM_CELL;
  // ~160-256 threads per CTA and <= ~72 KB of fp64 shared memory, so that
  // three CTAs share one SM (228 KB)
  static constexpr int NC_THREADS = (192 / P) > 0 ? 192 / P : 1;
  static constexpr int NC_SMEM = (72 * 1024 / 8) / SM_CELL > 0 ? (72 * 1024 / 8) / SM_CELL : 1;
  static constexpr int NC = NC_THREADS < NC_SMEM ? NC_THREADS : NC_SMEM;
  static constexpr int THREADS = NC * P;
  static constexpr int SMEM_REALS = NC * SM_CELL;
  static constexpr int MIN_BLOCKS = (D == 2 && K >= 7) ? 2 : ((65536 / (THREADS * 3)) >= 96 ? 3 : 2);
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
template <typename Real, int D, int K, int T>
__device__ __forceinline__ void load_line(const Real *f, int l, Real (&x)[K])
{
#pragma unroll
  for (int m = 0; m < K; ++m)
    x[m] = f[fln<D, K, T>(l, m)];
}
template <typename Real, int D, int K, int T>
__device__ __forceinline__ void store_line(Real *f, int l, const Real (&x)[K])
{
#pragma unroll
  for (int m = 0; m < K; ++m)
    f[fln<D, K, T>(l, m)] = x[m];
}

// Line operations on face fields along tangential direction T: each task is
// one line of K face points held in registers (even-odd 1D kernels with
// constant-bank matrices). op 0: x <- S x; op 1: y <- Dco x; op 2: S then
// y <- Dco(S x) as well; op 3: x += Dco^T y.
template <typename Real, int D, int K, int T, int OP>
__device__ __forceinline__ void line_op(Real *x, Real *y, int l)
{
  Real a[K], b[K];
  load_line<Real, D, K, T>(x, l, a);
  if constexpr (OP == 0)
    {
      apply_S<Real, K>(a, b);
      store_line<Real, D, K, T>(x, l, b);
    }
  else if constexpr (OP == 1)
    {
      apply_D<Real, K>(a, b);
      store_line<Real, D, K, T>(y, l, b);
    }
  else if constexpr (OP == 2)
    {
      apply_S<Real, K>(a, b);
      store_line<Real, D, K, T>(x, l, b);
      apply_D<Real, K>(b, a);
      store_line<Real, D, K, T>(y, l, a);
    }
  else
    {
      Real c[K];
      load_line<Real, D, K, T>(y, l, c);
      apply_Dt<Real, K>(c, b);
#pragma unroll
      for (int m = 0; m < K; ++m)
        a[m] += b[m];
      store_line<Real, D, K, T>(x, l, a);
    }
}

// ---- faces of one axis -----------------------------------------------------

// Both faces of axis A of every cell in the CTA:
//  own traces      u and dn/dxi_A from the collocation values (rows rf and
//                  rf Dco along the normal), tangential derivatives Dco_t u;
//  neighbour trace nodal Sf/Df rows of the neighbour's opposite face, S
//                  sweeps and Dco along the face (operators.cpp:794-858,
//                  766-788);
//  SIPG flux       operators.cpp:977-1003 (interior), 1069-1089 (boundary);
//  test side       w = rv + sum_t Dco_t^T rg_t on the face
//                  (face_tangential_integrate, :782-788) and rg_A, stored to
//                  OUT for the backward pass.
template <typename Real, int D, int K, int A>
__device__ __forceinline__ void face_axis(const ApplyParams<Real> &prm, Real *cell, int task,
                                          bool active, int p)
{
  using L = SL<D, K>;
  using T = TabLayout<K>;
  constexpr int P = L::P, NQ = L::NQ, FP = L::FP, NL = L::NL;
  const Real *val = cell;
  Real *NB = cell + L::OFF_NB;
  Real *OW = cell + L::OFF_OWN;
  Real *DT = cell + L::OFF_DT; // nb_t0 lo,hi | nb_t1 lo,hi | own_t0 lo,hi | own_t1 lo,hi
  Real *OUT = cell + L::OFF_OUT + (2 * A) * 2 * FP; // face lo: w, rgn | face hi: w, rgn
  const int fp = fpt<D, K>(p);

  int2 tf[2] = {make_int2(-2, 0), make_int2(-2, 0)};
  if (active)
    {
      tf[0] = prm.task_face[task * 2 * D + 2 * A];
      tf[1] = prm.task_face[task * 2 * D + 2 * A + 1];
    }
  // face geometry of face point p (issued first: longest latency)
  Real jxw[2], tau[2], jo[2][D], jb[2][D];
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      jxw[s] = tau[s] = Real(0);
#pragma unroll
      for (int b = 0; b < D; ++b)
        jo[s][b] = jb[s][b] = Real(0);
      if (tf[s].x != -2)
        {
          const int fid = tf[s].y & 0x3fffffff;
          const int side = (tf[s].y >> 30) & 1;
          const Real *fg = prm.face_geo + (long long)fid * (2 * D + 1) * P + p;
          jxw[s] = __ldg(fg);
#pragma unroll
          for (int b = 0; b < D; ++b)
            {
              jo[s][b] = __ldg(fg + (1 + side * D + b) * P);
              jb[s][b] = __ldg(fg + (1 + (1 - side) * D + b) * P);
            }
          tau[s] = __ldg(prm.penalty + fid);
        }
    }
  // neighbour pencils -> nodal traces (own low face meets the neighbour's
  // high face, row index 1, and vice versa)
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      Real nu = Real(0), nw = Real(0);
      if (tf[s].x >= 0)
        {
          const Real *un = prm.u + (long long)tf[s].x * NQ;
          Real x[K];
#pragma unroll
          for (int m = 0; m < K; ++m)
            x[m] = __ldg(un + gidx<D, K, A>(p, m));
          if (s == 0)
            {
              nu = dot_row<Real, K, T::oSf + K>(x);
              nw = dot_row<Real, K, T::oDf + K>(x);
            }
          else
            {
              nu = dot_row<Real, K, T::oSf>(x);
              nw = dot_row<Real, K, T::oDf>(x);
            }
        }
      NB[(2 * s) * FP + fp] = nu;
      NB[(2 * s + 1) * FP + fp] = nw;
    }
  // own traces from the collocation values along the normal
  Real own_u[2], own_n[2];
  {
    Real x[K];
    load_pencil<Real, D, K, A>(val, p, x);
    own_u[0] = dot_row<Real, K, T::oRf>(x);
    own_u[1] = dot_row<Real, K, T::oRf + K>(x);
    own_n[0] = dot_row<Real, K, T::oRD>(x);
    own_n[1] = dot_row<Real, K, T::oRD + K>(x);
    OW[fp] = own_u[0];
    OW[FP + fp] = own_u[1];
  }
  __syncthreads();

  if constexpr (D == 3)
    {
      // (a) along t0: S on the 4 neighbour fields; Dco on the 2 own fields
      for (int t = p; t < 6 * NL; t += P)
        {
          const int f = t / NL, l = t - f * NL;
          if (f < 4)
            line_op<Real, D, K, 0, 0>(NB + f * FP, nullptr, l);
          else
            line_op<Real, D, K, 0, 1>(OW + (f - 4) * FP, DT + (4 + (f - 4)) * FP, l);
        }
      __syncthreads();
      // (b) along t1: S on nw fields; S then Dco on nu fields; Dco on own
      for (int t = p; t < 6 * NL; t += P)
        {
          const int f = t / NL, l = t - f * NL;
          if (f < 4)
            {
              if ((f & 1) == 0) // nu_lo (0), nu_hi (2)
                line_op<Real, D, K, 1, 2>(NB + f * FP, DT + (2 + f / 2) * FP, l);
              else
                line_op<Real, D, K, 1, 0>(NB + f * FP, nullptr, l);
            }
          else
            line_op<Real, D, K, 1, 1>(OW + (f - 4) * FP, DT + (6 + (f - 4)) * FP, l);
        }
      __syncthreads();
      // (c) along t0: Dco on the interpolated neighbour values
      for (int t = p; t < 2 * NL; t += P)
        {
          const int f = t / NL, l = t - f * NL;
          line_op<Real, D, K, 0, 1>(NB + 2 * f * FP, DT + f * FP, l);
        }
      __syncthreads();
    }
  else
    {
      for (int t = p; t < 6; t += P)
        {
          if (t < 4)
            {
              if ((t & 1) == 0)
                line_op<Real, D, K, 0, 2>(NB + t * FP, DT + (t / 2) * FP, 0);
              else
                line_op<Real, D, K, 0, 0>(NB + t * FP, nullptr, 0);
            }
          else
            line_op<Real, D, K, 0, 1>(OW + (t - 4) * FP, DT + (2 + (t - 4)) * FP, 0);
        }
      __syncthreads();
    }

  // (d) flux at face point p for both faces
  constexpr int NT = D - 1; // tangential directions
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      Real rv = Real(0), g = Real(0);
      if (tf[s].x != -2)
        {
          const int side = (tf[s].y >> 30) & 1;
          // own reference gradient: normal comp own_n, tangential DT own
          Real dn_own = Real(0);
#pragma unroll
          for (int b = 0; b < D; ++b)
            {
              const Real gb = b == A ? own_n[s]
                                     : DT[(2 * NT + 2 * (b < A ? b : b - 1) + s) * FP + fp];
              dn_own += gb * jo[s][b];
            }
          if (tf[s].x == -1)
            {
              // mirror principle u+ = -u-, dn+ = dn- (operators.cpp:1069-1089)
              rv = (own_u[s] * tau[s] * Real(2) - dn_own) * jxw[s];
              g = -(own_u[s] * jxw[s]);
            }
          else
            {
              const Real nu = NB[(2 * s) * FP + fp], nw = NB[(2 * s + 1) * FP + fp];
              Real dn_nb = Real(0);
#pragma unroll
              for (int b = 0; b < D; ++b)
                {
                  const Real gb = b == A ? nw : DT[(2 * (b < A ? b : b - 1) + s) * FP + fp];
                  dn_nb += gb * jb[s][b];
                }
              // side 0: own = e-, side 1: own = e+ (jump = u- - u+)
              const Real sgn = side == 0 ? Real(1) : Real(-1);
              const Real delta = own_u[s] - nu;
              rv = (delta * tau[s] - sgn * ((dn_own + dn_nb) * Real(0.5))) * jxw[s];
              g = -(sgn * delta * jxw[s] * Real(0.5));
            }
        }
      OUT[(2 * s) * FP + fp] = rv;
      OUT[(2 * s + 1) * FP + fp] = g * jo[s][A];
      // tangential test components into the (now free) neighbour slots
#pragma unroll
      for (int t = 0; t < NT; ++t)
        DT[(2 * t + s) * FP + fp] = g * jo[s][t < A ? t : t + 1];
    }
  __syncthreads();
  // (e) w = rv + sum_t Dco_t^T rg_t, one tangential direction at a time
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

// Backward step along axis A: v (pencil) += rf_s w_s + (Dco^T rf_s) rgn_s
// for both faces of the axis (the transposed own traces, folded as rank-1
// updates into the pass that already holds the pencil).
template <typename Real, int D, int K, int A>
__device__ __forceinline__ void add_face_terms(const Real *cell, int p, Real (&v)[K])
{
  using L = SL<D, K>;
  using T = TabLayout<K>;
  constexpr int FP = L::FP;
  const Real *OUT = cell + L::OFF_OUT + (2 * A) * 2 * FP;
  const int fp = fpt<D, K>(p);
  const Real w0 = OUT[fp], r0 = OUT[FP + fp], w1 = OUT[2 * FP + fp], r1 = OUT[3 * FP + fp];
#pragma unroll
  for (int m = 0; m < K; ++m)
    v[m] += tab<Real, K>(T::oRf + m) * w0 + tab<Real, K>(T::oRf + K + m) * w1 +
            tab<Real, K>(T::oRD + m) * r0 + tab<Real, K>(T::oRD + K + m) * r1;
}

template <typename Real, int D, int K, bool COMPRESSED>
__global__ void __launch_bounds__(KernelShape<D, K>::THREADS, KernelShape<D, K>::MIN_BLOCKS)
  sipg_apply_kernel(const ApplyParams<Real> prm)
{
  using KS = KernelShape<D, K>;
  using L = SL<D, K>;
  using T = TabLayout<K>;
  constexpr int P = L::P, NQ = L::NQ, NC = KS::NC, FS = L::FS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Real *smem = reinterpret_cast<Real *>(smem_raw);

  const int lc = threadIdx.x / P;
  const int p = threadIdx.x - lc * P;
  const int task = blockIdx.x * NC + lc;
  const bool active = task < prm.n_tasks;
  Real *cell = smem + lc * L::SM_CELL;
  Real *val = cell;
  Real *G = cell + L::OFF_G;

  const int slot = active ? prm.task_slot[task] : 0;
  const int geo = active ? prm.task_geo[task] : -1;

  // ---- forward: val = (S x S x S) u, G_b = Dco_b val ----------------------
  {
    Real x[K], z[K];
    const Real *uc = prm.u + (long long)slot * NQ;
#pragma unroll
    for (int m = 0; m < K; ++m)
      x[m] = active ? __ldg(uc + p + P * m) : Real(0); // pencil along D-1
    apply_S<Real, K>(x, z);
    store_pencil<Real, D, K, D - 1>(val, p, z);
    __syncthreads();
    load_pencil<Real, D, K, 0>(val, p, x);
    apply_S<Real, K>(x, z);
    if constexpr (D == 3)
      {
        store_pencil<Real, D, K, 0>(val, p, z);
        __syncthreads();
        load_pencil<Real, D, K, 1>(val, p, x);
        apply_S<Real, K>(x, z);
        store_pencil<Real, D, K, 1>(val, p, z);
        apply_D<Real, K>(z, x);
        store_pencil<Real, D, K, 1>(G + FS, p, x);
        __syncthreads();
        load_pencil<Real, D, K, 0>(val, p, x);
        apply_D<Real, K>(x, z);
        store_pencil<Real, D, K, 0>(G, p, z);
        load_pencil<Real, D, K, 2>(val, p, x);
        apply_D<Real, K>(x, z);
        store_pencil<Real, D, K, 2>(G + 2 * FS, p, z);
      }
    else
      {
        store_pencil<Real, D, K, 0>(val, p, z);
        apply_D<Real, K>(z, x);
        store_pencil<Real, D, K, 0>(G, p, x);
        __syncthreads();
        load_pencil<Real, D, K, 1>(val, p, x);
        apply_D<Real, K>(x, z);
        store_pencil<Real, D, K, 1>(G + FS, p, z);
      }
  }
  __syncthreads();

  // ---- quadrature-point operation t = J^{-1} J^{-T} g JxW ------------------
  //      (operators.cpp:669-709); thread p: the points of its pencil along
  //      axis D-1 (coalesced geometry reads, [geo][comp][q] layout)
  {
#pragma unroll
    for (int m = 0; m < K; ++m)
      {
        const int q = pidx<D, K, D - 1>(p, m);
        Real t[D];
        if (geo >= 0)
          {
            Real jit[D * D], jw;
            if constexpr (COMPRESSED)
              {
                const Real *cg = prm.cell_geo + (long long)geo * (D * D + 1);
#pragma unroll
                for (int c = 0; c < D * D; ++c)
                  jit[c] = __ldg(cg + c);
                // wq_cell[q] = prod_a w[q_a] in axis order (geometry.cpp:285-296)
                Real wt = Real(1);
                const int qa0 = p % K;
                Real wa = Real(0);
#pragma unroll
                for (int i = 0; i < K; ++i)
                  wa = (qa0 == i) ? tab<Real, K>(T::oW + i) : wa;
                wt *= wa;
                if constexpr (D == 3)
                  {
                    const int qa1 = p / K;
                    wa = Real(0);
#pragma unroll
                    for (int i = 0; i < K; ++i)
                      wa = (qa1 == i) ? tab<Real, K>(T::oW + i) : wa;
                    wt *= wa;
                  }
                jw = __ldg(cg + D * D) * (wt * tab<Real, K>(T::oW + m));
              }
            else
              {
                const Real *cg = prm.cell_geo + (long long)geo * (D * D + 1) * NQ + p + P * m;
#pragma unroll
                for (int c = 0; c < D * D; ++c)
                  jit[c] = __ldg(cg + c * NQ);
                jw = __ldg(cg + D * D * NQ);
              }
            Real g[D], ph[D];
#pragma unroll
            for (int b = 0; b < D; ++b)
              g[b] = G[b * FS + q];
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
                t[i] = acc * jw;
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
          G[b * FS + q] = t[b];
      }
  }
  // (no barrier: the face phase reads val only, and its first barrier
  //  orders these G writes before the backward pass)

  // ---- faces ------------------------------------------------------------
  face_axis<Real, D, K, 0>(prm, cell, task, active, p);
  face_axis<Real, D, K, 1>(prm, cell, task, active, p);
  if constexpr (D == 3)
    face_axis<Real, D, K, 2>(prm, cell, task, active, p);

  // ---- backward: y = (S^T x S^T x S^T)(sum_b Dco_b^T t_b + face terms) ----
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
          yc[p + P * m] = z[m];
      }
  }
}

} // namespace dev
} // namespace dgx

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

#include "sipg_params.hpp"

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
  static constexpr int oDnE = oRD + 2 * K;   // even-odd halves of the nodal D
  static constexpr int oDnO = oDnE + CE * CE;
  static constexpr int oDn = oDnO + CE * CE; // plain nodal D, K x K (Gauss point, node)
  // the tensor-product Cartesian kernel (sipg_cart.cuh): 1D mass M1 = S^T W S
  // of the k-point Gauss rule, and the line operator premultiplied by its
  // inverse: M1^{-1} K1 with the stiffness K1 = D^T W D (both mirror-symmetric,
  // even-odd halves), M1^{-1} Sf_s^T and M1^{-1} Df_s^T (the face lifts)
  static constexpr int oM1E = oDn + K * K, oM1O = oM1E + CE * CE;
  static constexpr int oK1E = oM1O + CE * CE, oK1O = oK1E + CE * CE;
  static constexpr int oLS = oK1O + CE * CE; // [2][K]
  static constexpr int oLD = oLS + 2 * K;    // [2][K]
  static constexpr int size = oLD + 2 * K;
};

constexpr int tab_size(int K) { return 14 * ((K + 1) / 2) * ((K + 1) / 2) + 3 * K * K + 13 * K; }
// offset of the table for K (K >= 2) inside the per-precision constant block
constexpr int tab_offset(int K) { return K <= 2 ? 0 : tab_offset(K - 1) + tab_size(K - 1); }
constexpr int kMaxK = 11;
constexpr int kTabTotal = tab_offset(kMaxK + 1);

// Defined here (internal linkage) and used only by sipg.cu.
static __constant__ double c_tab_d[kTabTotal];
static __constant__ float c_tab_f[kTabTotal];

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

template <typename Real, int K>
__device__ __forceinline__ void apply_Dn(const Real (&x)[K], Real (&y)[K])
{
  eo_skew<Real, K, TabLayout<K>::oDnE, TabLayout<K>::oDnO>(x, y);
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

// Hermite-like basis, stored sign-flipped (setup.hpp Tables1D): sigma_j.
template <typename Real, int K>
__device__ __forceinline__ Real hsign(int j)
{
  return j == K - 2 ? Real(-1) : Real(1);
}

// Dofs of a ghost cell that a face evaluation may read: NLAY layers next to
// every face this rank computes for it (two for the Hermite-like basis, one
// for values on a nodal basis; read_face_dofs / mark_face_dofs,
// dof_layout.hpp:291-336, ghost_exchange.cpp:46-70): bit m set if the dof
// (thread pencil p, index m along axis D-1) is one of them. Ghost data
// outside these layers is never shipped and must not be read.
template <int D, int K, int NLAY>
__device__ __forceinline__ unsigned ghost_layer_mask(const int2 *tf, int p)
{
  constexpr unsigned ALL = (1u << K) - 1u, LOW = (1u << NLAY) - 1u;
  unsigned keep = 0;
#pragma unroll
  for (int phi = 0; phi < 2 * D; ++phi)
    {
      if (tf[phi].x == -2)
        continue;
      const int a = phi / 2, side = phi % 2;
      if (a == D - 1)
        keep |= side == 0 ? LOW : (LOW << (K - NLAY));
      else
        {
          const int c = (D == 2 || a == 0) ? p % K : p / K;
          if (side == 0 ? c < NLAY : c >= K - NLAY)
            keep = ALL;
        }
    }
  return keep;
}

// ---- shared-memory layout -------------------------------------------------

// Volume fields use a padded row stride S1 (odd for even K) so pencils along
// axis 0 -- consecutive threads K entries apart -- are free of fp64 bank
// conflicts; face fields (k^{d-1} points) likewise use row stride FK.
// Global (HBM) cell data stays unpadded lexicographic, axis 0 fastest.
#ifndef DGX_V4_W1
#define DGX_V4_W1 1
#endif

// CART: axis-aligned affine (Cartesian) records -- J^{-T} diagonal, face
// normals n.J^{-T} along the face axis only (checked at setup): the face
// phase needs no tangential derivatives (no DT fields, no W1 test fields)
template <int D, int K, bool CART = false>
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
  static constexpr int OFF_DT = OFF_NB + 4 * FP;      // 2(D-1) derivative fields
  // 2D int2 face entries (16 D bytes, fp32 or fp64); even offset so that
  // they stay 8-byte aligned in fp32 too
  static constexpr int OFF_TF = (OFF_DT + (CART ? 0 : 2 * (D - 1) * FP) + 1) / 2 * 2;
  static constexpr int SM_CELL = OFF_TF + 4 * D;
  // apply kernel, 3D: the t1 test parts Dco_t1^T rg_t1 (3 axes x 2 faces)
  // after the common layout, so that both test-side passes of a face axis
  // run in one phase (sipg_faces.cuh); the advection / rhs kernels do not
  // carry it
  static constexpr int OFF_W1 = (SM_CELL + 1) / 2 * 2;
  static constexpr int SM_CELL_APPLY = OFF_W1 + (D == 3 && DGX_V4_W1 && !CART ? 6 * FP : 0);
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

template <int D, int K, bool APPLY = false, bool CART = false>
struct KernelShape
{
  using L = SL<D, K, CART>;
  static constexpr int P = L::P;
  static constexpr int NQ = L::NQ;
  static constexpr int SM_CELL = APPLY ? L::SM_CELL_APPLY : L::SM_CELL;
  // ~160-256 threads per CTA and <= 74 KB of fp64 shared memory, so that
  // three CTAs share one SM (228 KB)
  static constexpr int NC_THREADS = (192 / P) > 0 ? 192 / P : 1;
  // CART cells are smaller: four CTAs per SM (4 x 55 KB)
  static constexpr int SMEM_CAP = (CART ? 55 : 74) * 1024 / 8;
  static constexpr int NC_SMEM = SMEM_CAP / SM_CELL > 0 ? SMEM_CAP / SM_CELL : 1;
  // 3D, k = 5 (C3): one cell = 25 threads = one warp per CTA. The barriers of a
  // one-warp CTA cost nothing, which outweighs the 7 idle lanes: measured on C3,
  // 7 cells x 3 CTAs/SM 1.768 ms, 6 x 4 1.707, 5 x 4 1.691, 4 x 6 1.824,
  // 1 x 16 1.608, 1 x 20 1.552, 1 x 22 1.545, 1 x 24 1.548 (Hermite-like basis alike).
  // k = 7 (two warps per cell) and k = 9 lose with one cell per CTA (5.15 vs 5.06,
  // 5.18 vs 4.91 ms on the sweep meshes).
  static constexpr bool K5 = APPLY && !CART && D == 3 && K == 5;
#ifdef DGX_SP_NC // kernel experiments: cells per CTA / CTAs per SM of the single-pencil kernels
  static constexpr int NC = DGX_SP_NC;
#else
  static constexpr int NC = K5 ? 1 : (NC_THREADS < NC_SMEM ? NC_THREADS : NC_SMEM);
#endif
  static constexpr int THREADS = NC * P;
  static constexpr int SMEM_REALS = NC * SM_CELL;
  static constexpr int MIN_BLOCKS =
#ifdef DGX_SP_MINB
    DGX_SP_MINB > 0 ? DGX_SP_MINB :
#endif
    K5 ? 22 :
    (D == 2 && K >= 7) ? 2
                       : ((CART && 65536 / (THREADS * 4) >= 96 && 4 * SMEM_REALS * 8 + 4096 <= 228 * 1024)
                            ? 4
                            : ((65536 / (THREADS * 3)) >= 96 ? 3 : 2));
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
  else if constexpr (OP == 3)
    {
      Real c[K];
      load_line<Real, D, K, T>(y, l, c);
      apply_Dt<Real, K>(c, b);
#pragma unroll
      for (int m = 0; m < K; ++m)
        a[m] += b[m];
      store_line<Real, D, K, T>(x, l, a);
    }
  else
    {
      // OP 4: x <- Dco^T y
      Real c[K];
      load_line<Real, D, K, T>(y, l, c);
      apply_Dt<Real, K>(c, b);
      store_line<Real, D, K, T>(x, l, b);
    }
}

// Backward step along axis A: v (pencil) += rf_s w_s + (Dco^T rf_s) rgn_s
// for both faces of the axis (the transposed own traces, folded as rank-1
// updates into the pass that already holds the pencil).
template <typename Real, int D, int K, int A, bool USE_W1 = false, bool CART = false>
__device__ __forceinline__ void add_face_terms(const Real *cell, int p, Real (&v)[K])
{
  using L = SL<D, K, CART>;
  using T = TabLayout<K>;
  constexpr int FP = L::FP;
  const Real *OUT = cell + L::OFF_OUT + (2 * A) * 2 * FP;
  const int fp = fpt<D, K>(p);
  Real w0 = OUT[fp], r0 = OUT[FP + fp], w1 = OUT[2 * FP + fp], r1 = OUT[3 * FP + fp];
  if constexpr (D == 3 && DGX_V4_W1 && USE_W1)
    {
      const Real *W1 = cell + L::OFF_W1 + (2 * A) * FP;
      w0 += W1[fp];
      w1 += W1[FP + fp];
    }
#pragma unroll
  for (int m = 0; m < K; ++m)
    v[m] += tab<Real, K>(T::oRf + m) * w0 + tab<Real, K>(T::oRf + K + m) * w1 +
            tab<Real, K>(T::oRD + m) * r0 + tab<Real, K>(T::oRD + K + m) * r1;
}

} // namespace dev
} // namespace dgx
#include "sipg_faces.cuh"
namespace dgx
{
namespace dev
{

// BASIS 2 (Hermite-like): 2-layer neighbour reads, per-dof sign of the
// sign-flipped functions, masked ghost cells; otherwise (nodal or generic
// bases) the neighbour's whole pencil. BASIS is a template argument also so
// that the instantiations of the per-basis translation units (each with its
// own constant tables) are distinct kernels, not one weak host stub.
// One task (cell slot) per group of P threads.
template <typename Real, int D, int K, bool COMPRESSED, int BASIS, bool CART = false>
__device__ __forceinline__ void sipg_task(const ApplyParams<Real> &prm, Real *cell, int p,
                                          int task)
{
  constexpr bool HERM = BASIS == 2;
  static_assert(!CART || COMPRESSED, "CART records are compressed");
  using L = SL<D, K, CART>;
  using T = TabLayout<K>;
  constexpr int P = L::P, NQ = L::NQ, FS = L::FS;
  const bool active = task < prm.n_tasks;
  Real *val = cell;
  Real *G = cell + L::OFF_G;

  const int slot = active ? prm.task_slot[task] : 0;
  const int geo = active ? prm.task_geo[task] : -1;

  // ---- L2 prefetch of everything this cell reads later: the geometry
  //      record (read in the quadrature-point phase), its face records and
  //      the neighbour cells (read in the face phase). Issued now, the HBM
  //      latency overlaps the forward pass instead of stalling later.
  if (active)
    {
      constexpr int LINE = 128;
      // doubles per point of the cell record: g3 J^{-T} + JxW, g4 the
      // merged symmetric coefficient
      const int ncg = prm.sym ? D * (D + 1) / 2 : D * D + 1;
#ifndef DGX_EXP_PF
#define DGX_EXP_PF 3 // bit 0: cell record, bit 1: face records, bit 2: neighbours (measured: bits 0+1 best, neighbour prefetch costs 2%)
#endif
      if ((DGX_EXP_PF & 1) && geo >= 0)
        {
          const char *gp = reinterpret_cast<const char *>(
            prm.cell_geo + (long long)geo * ncg * (COMPRESSED ? 1 : NQ));
          const int bytes = ncg * (COMPRESSED ? 1 : NQ) * (int)sizeof(Real);
          for (int off = p * LINE; off < bytes; off += P * LINE)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(gp + off));
        }
      // the task's face entries, read again by every face axis: kept in
      // shared memory (one L2 round trip less per axis)
      for (int i = p; i < 2 * D; i += P) // P may be smaller than 2D (2D, K=2)
        reinterpret_cast<int2 *>(cell + L::OFF_TF)[i] = prm.task_face[task * 2 * D + i];
#pragma unroll
      for (int phi = 0; phi < 2 * D; ++phi)
        {
          const int2 tf = prm.task_face[task * 2 * D + phi];
          if (tf.x == -2 || !(DGX_EXP_PF & 6))
            continue;
          constexpr int FREC = COMPRESSED ? 1 : P;
          const char *fp = reinterpret_cast<const char *>(
            prm.face_geo + (long long)(tf.y & 0x3fffffff) * (2 * D + 1) * FREC);
          constexpr int fbytes = (2 * D + 1) * FREC * (int)sizeof(Real);
          if (DGX_EXP_PF & 2)
            for (int off = p * LINE; off < fbytes; off += P * LINE)
              asm volatile("prefetch.global.L2 [%0];" ::"l"(fp + off));
          if ((DGX_EXP_PF & 4) && tf.x >= 0)
            {
              const char *np = reinterpret_cast<const char *>(prm.u + (long long)tf.x * NQ);
              constexpr int nbytes = NQ * (int)sizeof(Real);
              for (int off = p * LINE; off < nbytes; off += P * LINE)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(np + off));
            }
        }
    }

  // sign of the tangential indices of this thread's pencils (Hermite)
  Real sp = Real(1);
  unsigned gmask = (1u << K) - 1u;
  if constexpr (HERM)
    {
      sp = hsign<Real, K>(p % K);
      if constexpr (D == 3)
        sp *= hsign<Real, K>(p / K);
      if (active && slot >= prm.n_owned)
        {
          int2 tf[2 * D];
#pragma unroll
          for (int phi = 0; phi < 2 * D; ++phi)
            tf[phi] = prm.task_face[task * 2 * D + phi];
          gmask = ghost_layer_mask<D, K, 2>(tf, p);
        }
    }

  // ---- forward: val = (S x S x S) u, G_b = Dco_b val ----------------------
  {
    Real x[K], z[K];
    const Real *uc = prm.u + (long long)slot * NQ;
#pragma unroll
    for (int m = 0; m < K; ++m)
      {
        x[m] = active ? __ldg(uc + p + P * m) : Real(0); // pencil along D-1
        if constexpr (HERM)
          x[m] = ((gmask >> m) & 1u) ? x[m] * (sp * hsign<Real, K>(m)) : Real(0);
      }
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
  // neighbour pencils of the first face axis, in flight across the barrier
  Real xnb[2][K];
  if constexpr (!HERM)
    nb_fetch_v4<Real, D, K, 0, CART>(prm, cell, active, p, xnb);
  __syncthreads();

  // ---- faces ------------------------------------------------------------
#ifndef DGX_EXP_NO_FACE
  {
    // tangential quadrature weight of face point p, prod_t w[q_t] in axis
    // order (wq_face, geometry.cpp:298-308), for compressed face records
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
    if constexpr (CART)
      {
        face_axis_cart<Real, D, K, 0, HERM, BASIS == 0>(prm, cell, active, p, wf, sp, xnb, [&] {
          if constexpr (!HERM)
            nb_fetch_v4<Real, D, K, 1, CART>(prm, cell, active, p, xnb);
        });
        face_axis_cart<Real, D, K, 1, HERM, BASIS == 0>(prm, cell, active, p, wf, sp, xnb, [&] {
          if constexpr (!HERM && D == 3)
            nb_fetch_v4<Real, D, K, 2, CART>(prm, cell, active, p, xnb);
        });
        if constexpr (D == 3)
          face_axis_cart<Real, D, K, 2, HERM, BASIS == 0>(prm, cell, active, p, wf, sp, xnb, [] {});
      }
    else
      {
        face_axis_v4<Real, D, K, 0, COMPRESSED, HERM, BASIS == 0>(prm, cell, task, active, p, wf, sp, xnb, [&] {
          if constexpr (!HERM)
            nb_fetch_v4<Real, D, K, 1>(prm, cell, active, p, xnb);
        });
        face_axis_v4<Real, D, K, 1, COMPRESSED, HERM, BASIS == 0>(prm, cell, task, active, p, wf, sp, xnb, [&] {
          if constexpr (!HERM && D == 3)
            nb_fetch_v4<Real, D, K, 2>(prm, cell, active, p, xnb);
        });
        if constexpr (D == 3)
          face_axis_v4<Real, D, K, 2, COMPRESSED, HERM, BASIS == 0>(prm, cell, task, active, p, wf, sp, xnb, [] {});
      }
  }
#else
  {
    Real *OUT = cell + L::OFF_OUT;
    for (int i = p; i < 4 * D * L::FP; i += P)
      OUT[i] = Real(0);
    __syncthreads();
  }
#endif

  // ---- quadrature-point operation t = J^{-1} J^{-T} g JxW ------------------
  //      (operators.cpp:669-709); thread p: the points of its pencil along
  //      axis D-1 (coalesced geometry reads, [geo][comp][q] layout)
  {
    // 3D: t_2 of the thread's own z-pencil stays in registers and the first
    // backward pass (along z, same pencil) follows without a barrier
    Real tz[K];
#pragma unroll
    for (int m = 0; m < K; ++m)
      {
        const int q = pidx<D, K, D - 1>(p, m);
        Real t[D];
        if (geo >= 0 && prm.sym)
          {
            // g4: t = C g with the merged symmetric coefficient
            // (laplacian_coefficient, operators.cpp:712-733)
            constexpr int NS = D * (D + 1) / 2;
            Real cf[NS];
            if constexpr (COMPRESSED)
              {
                const Real *cg = prm.cell_geo + (long long)geo * NS;
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
                const Real w = wt * tab<Real, K>(T::oW + m);
#pragma unroll
                for (int e = 0; e < NS; ++e)
                  cf[e] = __ldg(cg + e) * w;
              }
            else
              {
                const Real *cg = prm.cell_geo + (long long)geo * NS * NQ + p + P * m;
#pragma unroll
                for (int e = 0; e < NS; ++e)
                  cf[e] = __ldcs(cg + e * NQ);
              }
            Real g[D];
#pragma unroll
            for (int b = 0; b < D; ++b)
              g[b] = G[b * FS + q];
            if constexpr (D == 3)
              {
                t[0] = cf[0] * g[0] + cf[3] * g[1] + cf[4] * g[2];
                t[1] = cf[3] * g[0] + cf[1] * g[1] + cf[5] * g[2];
                t[2] = cf[4] * g[0] + cf[5] * g[1] + cf[2] * g[2];
              }
            else
              {
                t[0] = cf[0] * g[0] + cf[2] * g[1];
                t[1] = cf[2] * g[0] + cf[1] * g[1];
              }
          }
        else if (geo >= 0)
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
                // read-once stream: evict-first, keep L2 for the reused
                // neighbour cells and face records
#ifdef DGX_EXP_NO_GEO
#pragma unroll
                for (int c = 0; c < D * D; ++c)
                  jit[c] = (c % (D + 1) == 0) ? Real(1) : Real(0);
                jw = Real(1e-3) * (Real)(geo & 7);
                (void)cg;
#else
#pragma unroll
                for (int c = 0; c < D * D; ++c)
                  jit[c] = __ldcs(cg + c * NQ);
                jw = __ldcs(cg + D * D * NQ);
#endif
              }
            Real g[D], ph[D];
#pragma unroll
            for (int b = 0; b < D; ++b)
              g[b] = G[b * FS + q];
            if constexpr (CART)
              {
                // diagonal J^{-T} (off-diagonal round-off <= 1e-13 relative, dropped)
                (void)ph;
#pragma unroll
                for (int i = 0; i < D; ++i)
                  t[i] = (jit[i * D + i] * (jit[i * D + i] * g[i])) * jw;
              }
            else
              {
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
          }
        else
          {
#pragma unroll
            for (int b = 0; b < D; ++b)
              t[b] = Real(0);
          }
#pragma unroll
        for (int b = 0; b < (D == 3 ? 2 : D); ++b)
          G[b * FS + q] = t[b];
        tz[m] = t[D - 1];
      }
    if constexpr (D == 3)
      {
        // ---- backward, first pass (z): v = Dco_z^T t_2 + z-face terms
        Real v[K];
        apply_Dt<Real, K>(tz, v);
        add_face_terms<Real, D, K, 2, !CART, CART>(cell, p, v);
        store_pencil<Real, D, K, 2>(val, p, v);
      }
  }
  __syncthreads();

  // ---- backward: y = (S^T x S^T x S^T)(sum_b Dco_b^T t_b + face terms) ----
  {
    Real x[K], z[K], v[K];
    if constexpr (D == 3)
      {
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
    add_face_terms<Real, D, K, 1, !CART, CART>(cell, p, v);
    store_pencil<Real, D, K, 1>(val, p, v);
    __syncthreads();
    load_pencil<Real, D, K, 0>(G, p, x);
    apply_Dt<Real, K>(x, z);
    load_pencil<Real, D, K, 0>(val, p, v);
#pragma unroll
    for (int m = 0; m < K; ++m)
      v[m] += z[m];
    add_face_terms<Real, D, K, 0, !CART, CART>(cell, p, v);
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
          {
            if constexpr (HERM)
              z[m] = ((gmask >> m) & 1u) ? z[m] * (sp * hsign<Real, K>(m)) : Real(0);
            __stcs(yc + p + P * m, z[m]); // y is not read again (streaming)
          }
      }
  }
}

template <typename Real, int D, int K, bool COMPRESSED, int BASIS, bool CART = false>
__global__ void __launch_bounds__(KernelShape<D, K, true, CART>::THREADS, KernelShape<D, K, true, CART>::MIN_BLOCKS)
  sipg_apply_kernel(const ApplyParams<Real> prm)
{
  using KS = KernelShape<D, K, true, CART>;
  using L = SL<D, K, CART>;
  constexpr int P = L::P, NC = KS::NC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Real *smem = reinterpret_cast<Real *>(smem_raw);
  const int lc = threadIdx.x / P;
  const int p = threadIdx.x - lc * P;
  Real *cell = smem + lc * KS::SM_CELL;
  sipg_task<Real, D, K, COMPRESSED, BASIS, CART>(prm, cell, p, blockIdx.x * NC + lc);
}

} // namespace dev
} // namespace dgx

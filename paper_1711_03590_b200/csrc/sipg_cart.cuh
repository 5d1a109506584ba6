// SIPG-Laplacian apply on axis-aligned affine (Cartesian) records as a sum of
// tensor products of 1D matrices (included by sipg_launch.cuh after
// sipg_kernel.cuh; BASELINE configs C1, C2 and C5).
//
// With a constant diagonal J^{-T}, constant det J and constant face records
// (geometry.cpp:267-275 compression; checked at setup, Operator::cart_) the
// reference's discrete operator factorises exactly. Its cell integral
// (operators.cpp:669-749 with tensor_kernels.hpp:334-416) is
//   sum_a  (J^{-T}_aa)^2 det J  [K1 along a] x [M1 along the other axes],
// M1 = S^T W S, K1 = D^T W D (S, D: nodal values / derivatives in the k Gauss
// points, W the Gauss weights), and every face integral along axis a
// (operators.cpp:933-1111) is M1 in the tangential directions times a rank-2
// update along the normal line: the flux (interior :977-1003, boundary
// mirror rule :1069-1089) only needs the face value Sf.u and the normal
// derivative Df.u of the two nodal lines that meet in the face point. So
//   y = sum_a (M1 x M1)_tangential(a)  L_a u,
//   L_a u = c_a K1 u_line + sum_{faces s of a} rv_s Sf_s^T + g_s jo_s Df_s^T
// on every nodal line along a: no quadrature-point fields, no face fields,
// no tangential interpolation of the neighbour. Same quadrature as the
// reference (the k-point Gauss rule is inside M1 and K1), so the results agree
// to round-off; the sum order differs like in the collocation kernels.
//
// The kernel evaluates it as
//   y = (M1 x M1 x M1) w,   w = sum_a M1^{-1} L_a u   (M1^{-1} along a),
// with the 1D tables M1^{-1} K1, M1^{-1} Sf^T, M1^{-1} Df^T built on the host
// (sipg_launch.cuh): the three line results add up point by point in one field
// and three mass products follow, instead of two mass products per axis.
// cond(M1) <= 20 for the Gauss-Lobatto basis and <= 5 for the Lagrange-Gauss
// basis at p <= 10, so the inverse costs a digit at most (tests: <= 1e-12 in
// fp64, <= 1e-5 in fp32 up to p = 10). The Hermite-like basis (cond(M1) = 1e3
// at p = 3, 1e6 at p = 10) keeps the direct form: t_a = L_a u with K1 itself
// and two mass products per axis,
//   z: t_z -> C;  x: t_x -> A, C <- M_x C;  y: t_y -> B, A <- M_y A,
//   C <- M_y C;  x: A <- A + M_x B;  z: y = M_z A + C      (17 field passes).
//
// P = K^{D-1} threads per cell; a thread holds one nodal line along the
// current axis in registers; the 1D matrices are mirror-symmetric and applied
// in even-odd form from the constant bank; end-point rows are used for the low
// end only and mirrored for the high end (fewer constants in flight: ptxas
// keeps them in uniform registers and spills those first).
//   3D:  z: C = L~_z u;  x: C += L~_x u;  y: w = C + L~_y u, C = M_y w;
//        x: C = M_x C;  z: y = M_z C        (L~ = M1^{-1} L)
// 11 shared-memory field passes and 6 1D products per cell (+ the staging of
// the neighbour cells), against 59 passes, 12 products and the face phase of
// the collocation kernels.
//
// The kernel is bound by the L1 / shared-memory data pipe (ncu: 91% busy in
// its first version), so the layout is built around wavefronts:
// * every global access is coalesced: the own cell and all 2D neighbour cells
//   are read as flat runs (thread t reads elements t + P m); the cells across
//   the x- and y-faces are staged in shared memory and the thread then reads
//   its neighbour lines from there (a thread-contiguous x-line read from HBM
//   costs one sector per lane and request); an x-neighbour that is the CTA's
//   adjacent task (tasks run along x) is read from that cell's own field;
// * volume fields have row stride K and a plane stride S2 = K^2 + pad chosen
//   per K and word size so that the bank residues of the lines along x and
//   along y are (nearly) evenly spread; a per-axis permutation of the lines
//   over the threads (host-built, constant memory) then makes the residue of
//   thread t equal t + beta mod #banks, and a cell stride = P mod #banks
//   continues that run across the cells of a CTA: consecutive lanes hit
//   consecutive banks for every axis, whatever the warp alignment.
// * each neighbour line is reduced at once to the two scalars a face needs,
//   and the per-face constants to three flux coefficients (cart_face).
// Hermite-like basis: the sign-flipped tables (mirror-symmetric M1, K1), the
// sign applied to u and y; value and derivative at a face live on the two dofs
// next to it, so traces, lifts and neighbour reads touch two values per line
// (only those layers are shipped for a ghost cell); masked ghost cells.
#pragma once

namespace dgx
{
namespace dev
{

// plane-stride padding (3D) per K = 2..11 for 8-byte and 4-byte words (16 / 32
// banks): offline search for evenly spread line residues, pad <= 8
constexpr int cart_pad(int K, int wbytes)
{
  constexpr int p8[10] = {0, 5, 3, 5, 3, 1, 7, 1, 3, 4};
  constexpr int p4[10] = {0, 5, 3, 3, 1, 3, 7, 3, 3, 0};
  return (K < 2 || K > 11) ? 0 : (wbytes == 8 ? p8[K - 2] : p4[K - 2]);
}

template <typename Real, int D, int K, bool HERM = false>
struct CartShape
{
  static constexpr int P = ipow_c(K, D - 1);
  static constexpr int NBANK = 128 / (int)sizeof(Real); // banks of one word
  // 3D: rows dense (x + K y = the thread index of a z-line), padded planes;
  // 2D: odd row stride
  static constexpr int S1 = D == 3 ? K : K + ((K % 2 == 0) ? 1 : 0);
  static constexpr int S2 = D == 3 ? K * K + cart_pad(K, (int)sizeof(Real)) : 0;
  static constexpr int FS = D == 3 ? S2 * K : S1 * K;
  // U, A, B, C (+ two more neighbour staging fields in 3D)
  static constexpr int NF = D == 3 ? 6 : 4;
  // per-cell constants behind the fields: three flux coefficients per face
  // (cart_face), per axis the cell coefficient
  static constexpr int OFF_FC = NF * FS;
  static constexpr int OFF_CC = OFF_FC + 6 * D;
  static constexpr int SM_MIN = OFF_CC + D;
  // cell stride = P mod #banks (3D): the bank run continues across cells
  static constexpr int SM_CELL = D == 3 ? SM_MIN + ((P % NBANK) - (SM_MIN % NBANK) + NBANK) % NBANK
                                        : (SM_MIN + 1) / 2 * 2;
#ifdef DGX_CART_NC // kernel experiments
  static constexpr int NC = DGX_CART_NC;
#else
  // about 192 threads per CTA; 3D k = 7 in fp64 with a nodal basis (C5): 4 cells
  // (196 threads, 3 CTAs per SM; more x-neighbours inside the CTA): 15.96 ms
  // against 16.59 (3 cells, 4 CTAs), 19.7 (5 cells, 2 CTAs), 19.1 (6 cells,
  // 2 CTAs). fp32 (9.97 vs 9.03 ms) and the Hermite-like basis, which does not
  // share x-neighbours (16.86 vs 16.03 ms), stay at 3 cells.
  // 2D: one warp per CTA (32 / K cells, barriers cost nothing): C2 p = 2 / 5 / 8
  // 18.3 / 32.9 / 82 us -> 17.0 / 32.8 / 74 us
#ifndef DGX_CART_2D_WARP
#define DGX_CART_2D_WARP 1
#endif
  static constexpr int NC =
    (D == 2 && DGX_CART_2D_WARP) ? (32 / P > 0 ? 32 / P : 1)
    : (D == 3 && K == 7 && sizeof(Real) == 8 && !HERM) ? 4
    // 3D k = 4 (C1, 16 threads per cell): 4 cells = two warps per CTA, 10.4 us
    // against 12.2 (12 cells), 11.4 (2), 10.8 (3), 10.5 (6, 8)
    : (D == 3 && K == 4) ? 4 : ((192 / P) > 0 ? 192 / P : 1);
#endif
  static constexpr int THREADS = NC * P;
  static constexpr int SMEM_REALS = NC * SM_CELL;
  // registers: two lines of K values and the neighbour scalars (measured at
  // k = 7, C5: 4 CTAs per SM 19.8 ms, 3 CTAs 23.6 ms, 5 CTAs (spills) 21.9 ms)
  static constexpr int REGS = (2 * K + 4 * D) * (int)(sizeof(Real) / 4) + 40;
  static constexpr int WARP_THREADS = (THREADS + 31) / 32 * 32;
  static constexpr int MB_REGS = 65536 / (WARP_THREADS * REGS) - (K >= 9 && sizeof(Real) == 8 ? 1 : 0);
  static constexpr int MB_SMEM = (220 * 1024) / (SMEM_REALS * (int)sizeof(Real) + 1024);
  static constexpr int MB0 = MB_REGS < MB_SMEM ? MB_REGS : MB_SMEM;
#ifdef DGX_CART_MINB
  static constexpr int MINB = DGX_CART_MINB;
#else
  static constexpr int MINB =
    (D == 2 && DGX_CART_2D_WARP) ? (K >= 9 && sizeof(Real) == 8 ? 12 : 16) : (MB0 < 1 ? 1 : (MB0 > 8 ? 8 : MB0));
#endif
};

// line permutations of the 3D kernel, [fp64 / fp32][K][axis 0 / 1][thread]
static __constant__ unsigned char c_cart_perm[2][kMaxK + 1][2][128];

// shared-memory offset of entry m of line l along axis A
template <typename Real, int D, int K, int A>
__device__ __forceinline__ int cidx(int l, int m)
{
  using CS = CartShape<Real, D, K>;
  return lidx<D, K, A, CS::S1, CS::S2>(l, m);
}
template <typename Real, int D, int K, int A>
__device__ __forceinline__ void cload(const Real *f, int l, Real (&x)[K])
{
#pragma unroll
  for (int m = 0; m < K; ++m)
    x[m] = f[cidx<Real, D, K, A>(l, m)];
}
template <typename Real, int D, int K, int A>
__device__ __forceinline__ void cstore(Real *f, int l, const Real (&x)[K])
{
#pragma unroll
  for (int m = 0; m < K; ++m)
    f[cidx<Real, D, K, A>(l, m)] = x[m];
}

template <typename Real, int K>
__device__ __forceinline__ void apply_M1(const Real (&x)[K], Real (&y)[K])
{
  eo_sym<Real, K, TabLayout<K>::oM1E, TabLayout<K>::oM1O>(x, y);
}

// The neighbour's face value and normal derivative on the nodal line p along
// axis A, for both faces of the axis: everything a face needs from the cell
// across it. Issued for all axes at task start (every global load of the
// task is in flight at once).
// End-point value and derivative of a nodal line at its low (index 0) and
// high (index 1) end from the rows of the low end only: the basis is
// mirror-symmetric, Sf_1[j] = Sf_0[K-1-j] and Df_1[j] = -Df_0[K-1-j] (half the
// constants in flight).
template <typename Real, int K, bool GLN, bool HERM>
__device__ __forceinline__ void cart_ends(const Real (&u)[K], Real (&val)[2], Real (&der)[2])
{
  using T = TabLayout<K>;
  if constexpr (HERM)
    {
      // Hermite-like: value and derivative at an end point live on the two
      // dofs next to it (the other entries of Sf, Df are zero)
      const Real s0 = tab<Real, K>(T::oSf), s1 = tab<Real, K>(T::oSf + 1);
      const Real d0 = tab<Real, K>(T::oDf), d1 = tab<Real, K>(T::oDf + 1);
      val[0] = s0 * u[0] + s1 * u[1];
      val[1] = s0 * u[K - 1] + s1 * u[K - 2];
      der[0] = d0 * u[0] + d1 * u[1];
      der[1] = -(d0 * u[K - 1] + d1 * u[K - 2]);
    }
  else
    {
      Real a = Real(0), b = Real(0), c = Real(0), d = Real(0);
#pragma unroll
      for (int m = 0; m < K; ++m)
        {
          const Real df = tab<Real, K>(T::oDf + m);
          c += df * u[m];
          d += df * u[K - 1 - m];
          if constexpr (!GLN)
            {
              const Real sf = tab<Real, K>(T::oSf + m);
              a += sf * u[m];
              b += sf * u[K - 1 - m];
            }
        }
      // Gauss-Lobatto: Sf rows are exact unit vectors (the end nodes)
      val[0] = GLN ? u[0] : a;
      val[1] = GLN ? u[K - 1] : b;
      der[0] = c;
      der[1] = -d;
    }
}

// The neighbours' face value and normal derivative on the nodal line l along
// axis A, for both faces of the axis: everything a face needs from the cell
// across it. Direct global reads (the last axis: coalesced; and every axis
// when staging is off).
template <typename Real, int D, int K, int A, bool GLN, bool HERM>
__device__ __forceinline__ void cart_nb(const ApplyParams<Real> &prm, const int2 (&tf)[2 * D], int l, Real sp,
                                        Real (&nu)[2], Real (&nd)[2])
{
  constexpr int NQ = ipow_c(K, D);
  Real xn[2][K];
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      const int nbs = tf[2 * A + s].x;
      const Real *un = prm.u + (long long)(nbs >= 0 ? nbs : 0) * NQ;
#pragma unroll
      for (int m = 0; m < K; ++m)
        {
          // Hermite-like: only the two layers next to the face carry a value
          // or a normal derivative there (read_face_dofs, dof_layout.hpp:291-336)
          // -- and only they are shipped for a ghost neighbour
          const bool need = !HERM || (s == 0 ? m >= K - 2 : m < 2);
          xn[s][m] = (need && nbs >= 0) ? __ldg(un + gidx<D, K, A>(l, m)) : Real(0);
          if constexpr (HERM)
            xn[s][m] *= sp * hsign<Real, K>(m);
        }
    }
  // face 0 (low side) meets the neighbour's high end, and vice versa
  Real v[2], d[2];
  cart_ends<Real, K, GLN, HERM>(xn[0], v, d);
  nu[0] = v[1];
  nd[0] = d[1];
  cart_ends<Real, K, GLN, HERM>(xn[1], v, d);
  nu[1] = v[0];
  nd[1] = d[0];
}

// The same two scalars from neighbour cells staged in shared memory (fields
// F0: across the low face, F1: across the high face; line l along A, sp: the
// Hermite-like sign of the line)
template <typename Real, int D, int K, int A, bool GLN, bool HERM>
__device__ __forceinline__ void cart_nb_staged(const Real *F0, const Real *F1, int l, Real sp, Real (&nu)[2],
                                               Real (&nd)[2], bool own0 = false, bool own1 = false)
{
  // own0 / own1: the field is a CTA partner's own U, which holds the
  // sign-flipped Hermite-like coefficients already
  Real xn[2][K];
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      const Real *F = s == 0 ? F0 : F1;
      const bool own = s == 0 ? own0 : own1;
#pragma unroll
      for (int m = 0; m < K; ++m)
        {
          const bool need = !HERM || (s == 0 ? m >= K - 2 : m < 2);
          xn[s][m] = need ? F[cidx<Real, D, K, A>(l, m)] : Real(0);
          if constexpr (HERM)
            xn[s][m] *= own ? Real(1) : sp * hsign<Real, K>(m);
        }
    }
  Real v[2], d[2];
  cart_ends<Real, K, GLN, HERM>(xn[0], v, d);
  nu[0] = v[1];
  nd[0] = d[1];
  cart_ends<Real, K, GLN, HERM>(xn[1], v, d);
  nu[1] = v[0];
  nd[1] = d[0];
}

// t = M1^{-1} L_A u (Hermite-like basis: L_A u) for one nodal line along axis A
// of the task's cell: c_A M1^{-1} K1 u plus both faces of the axis. u: own nodal line; nu, nd: the
// neighbours' face value and normal derivative (reference coordinates) on the
// same line (zeros without a neighbour). The per-face constants are folded at
// task start into three coefficients that cover the interior flux
// (operators.cpp:977-1003), the boundary mirror rule (:1069-1089) and faces not
// computed on this rank (all zero) without a branch:
//   rv = A1 (uf - nu) + A2 Df.u + A3 nd,   g jo = A2 (uf - nu)
//   interior: A1 = tau JxW, A2 = -sgn jo JxW / 2, A3 = -sgn jb JxW / 2
//   boundary: A1 = 2 tau JxW, A2 = -jo JxW, A3 = 0
// and the result rv Sf^T + g jo Df^T is lifted with M1^{-1} (tables of the low
// end, mirrored for the high end).
template <typename Real, int D, int K, int A, bool GLN, bool HERM>
__device__ __forceinline__ void cart_line(const Real *cell, const Real (&u)[K], const Real (&nu)[2],
                                          const Real (&nd)[2], Real (&t)[K])
{
  using T = TabLayout<K>;
  using CS = CartShape<Real, D, K>;
  const Real c = cell[CS::OFF_CC + A];
  eo_sym<Real, K, T::oK1E, T::oK1O>(u, t);
  Real uf[2], dno[2], rv[2], gj[2];
  cart_ends<Real, K, GLN, HERM>(u, uf, dno);
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      const Real *fc = cell + CS::OFF_FC + 3 * (2 * A + s);
      const Real delta = uf[s] - nu[s];
      rv[s] = fc[0] * delta + fc[1] * dno[s] + fc[2] * nd[s];
      gj[s] = fc[1] * delta;
    }
  if constexpr (HERM)
    {
      // Hermite-like (no M1^{-1}: t = L_A u): rv Sf^T + g jo Df^T lives on the
      // two dofs next to each end
      const Real s0 = tab<Real, K>(T::oSf), s1 = tab<Real, K>(T::oSf + 1);
      const Real d0 = tab<Real, K>(T::oDf), d1 = tab<Real, K>(T::oDf + 1);
#pragma unroll
      for (int m = 0; m < K; ++m)
        t[m] *= c;
      t[0] += rv[0] * s0 + gj[0] * d0;
      t[1] += rv[0] * s1 + gj[0] * d1;
      t[K - 1] += rv[1] * s0 - gj[1] * d0;
      t[K - 2] += rv[1] * s1 - gj[1] * d1;
    }
  else
    {
#pragma unroll
      for (int m = 0; m < K; ++m)
        {
          const Real ls = tab<Real, K>(T::oLS + m), ld = tab<Real, K>(T::oLD + m);
          t[m] = c * t[m] + (rv[0] * ls + gj[0] * ld);
        }
#pragma unroll
      for (int m = 0; m < K; ++m)
        {
          const Real ls = tab<Real, K>(T::oLS + m), ld = tab<Real, K>(T::oLD + m);
          t[K - 1 - m] += rv[1] * ls - gj[1] * ld;
        }
    }
}

template <typename Real, int D, int K, int BASIS>
__global__ void __launch_bounds__(CartShape<Real, D, K, BASIS == 2>::THREADS,
                                  CartShape<Real, D, K, BASIS == 2>::MINB)
  sipg_cart_kernel(const ApplyParams<Real> prm)
{
  constexpr bool GLN = BASIS == 0, HERM = BASIS == 2;
  using CS = CartShape<Real, D, K, HERM>;
  constexpr int P = CS::P, NQ = P * K, FS = CS::FS, NC = CS::NC;
  // neighbour cells across the x- / y-faces staged in shared memory (the L1
  // data pipe binds in both precisions: C5 fp64 19.8 -> 19.3 ms, fp32 10.8 ->
  // 10.4 ms); the two-value Hermite-like reads go to HBM / L2 directly
#ifndef DGX_CART_STAGE
#define DGX_CART_STAGE 4
#endif
  constexpr bool STAGE = (int)sizeof(Real) >= DGX_CART_STAGE;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Real *smem = reinterpret_cast<Real *>(smem_raw);
  const int lc = threadIdx.x / P;
  const int p = threadIdx.x - lc * P;
  const int task = blockIdx.x * NC + lc;
  const bool active = task < prm.n_tasks;
  Real *U = smem + lc * CS::SM_CELL;
  Real *Af = U + FS;      // staging: cell across the low x-face; then t_x, ...
  Real *Bf = Af + FS;     // staging: cell across the high x-face; then t_y
  Real *Cf = Bf + FS;     // t of the last axis
  const int slot = active ? prm.task_slot[task] : 0;
  const int geo = active ? prm.task_geo[task] : -1;
  const int2 *tfp = prm.task_face + (long long)(active ? task : 0) * 2 * D;

  // the lines this thread owns in the x- and y-phases (bank-spreading
  // permutations, 3D), and in the last-axis phases: line p
  int p0 = p, p1 = p;
  if constexpr (D == 3)
    {
      p0 = c_cart_perm[sizeof(Real) == 8 ? 0 : 1][K][0][p];
      p1 = c_cart_perm[sizeof(Real) == 8 ? 0 : 1][K][1][p];
    }

  // ---- every global load of the task: face entries, own cell, neighbour
  //      cells (coalesced; reduced to two scalars per line), constants -------
  int2 tf[2 * D];
#pragma unroll
  for (int phi = 0; phi < 2 * D; ++phi)
    tf[phi] = active ? __ldg(tfp + phi) : make_int2(-2, 0);
  // Hermite-like basis (tables of the sign-flipped functions, setup.hpp
  // Tables1D): sign of a line's two tangential indices -- the digits of its
  // line number -- and, for a ghost-side task, the layers that were shipped
  Real sp = Real(1), sp0 = Real(1), sp1 = Real(1);
  unsigned gmask = (1u << K) - 1u;
  if constexpr (HERM)
    {
      sp = hsign<Real, K>(p % K);
      sp0 = hsign<Real, K>(p0 % K);
      sp1 = hsign<Real, K>(p1 % K);
      if constexpr (D == 3)
        {
          sp *= hsign<Real, K>(p / K);
          sp0 *= hsign<Real, K>(p0 / K);
          sp1 *= hsign<Real, K>(p1 / K);
        }
      if (active && slot >= prm.n_owned)
        gmask = ghost_layer_mask<D, K, 2>(tf, p);
    }
  Real x[K], t[K];
  {
    // last axis: the thread's line is contiguous across threads in HBM
    const Real *uc = prm.u + (long long)slot * NQ;
#pragma unroll
    for (int m = 0; m < K; ++m)
      {
        x[m] = active ? __ldg(uc + p + P * m) : Real(0);
        if constexpr (HERM)
          x[m] = ((gmask >> m) & 1u) ? x[m] * (sp * hsign<Real, K>(m)) : Real(0);
      }
  }
  // x-neighbours that are the CTA's previous / next task (Hermite-like: owned
  // cells only -- a ghost cell's U is masked to the shipped layers)
  bool xin[2] = {false, false};
  if constexpr (STAGE)
    {
      xin[0] = active && lc > 0 && tf[0].x >= 0 && tf[0].x == __ldg(prm.task_slot + task - 1) &&
               (!HERM || tf[0].x < prm.n_owned);
      xin[1] = active && lc + 1 < NC && task + 1 < prm.n_tasks && tf[1].x >= 0 &&
               tf[1].x == __ldg(prm.task_slot + task + 1) && (!HERM || tf[1].x < prm.n_owned);
    }
  Real nu[D][2], nd[D][2];
  cart_nb<Real, D, K, D - 1, GLN, HERM>(prm, tf, p, sp, nu[D - 1], nd[D - 1]);
  if constexpr (!STAGE)
    {
      cart_nb<Real, D, K, 0, GLN, HERM>(prm, tf, p0, sp0, nu[0], nd[0]);
      if constexpr (D == 3)
        cart_nb<Real, D, K, 1, GLN, HERM>(prm, tf, p1, sp1, nu[1], nd[1]);
    }
  else
    {
      // the cells across the x- (and y-) faces, staged like U -- unless the
      // cell is the task next door in this CTA (consecutive tasks run along
      // x): its own field U is read instead
#pragma unroll
      for (int phi = 0; phi < 2 * (D - 1); ++phi)
        {
          Real *F = phi < 2 ? Af + phi * FS : Cf + (phi - 1) * FS; // 3D: fields 4, 5 behind C
          const int nbs = tf[phi].x;
          if (phi < 2 && xin[phi])
            continue; // the CTA partner
          const Real *un = prm.u + (long long)(nbs >= 0 ? nbs : 0) * NQ;
          Real v[K];
#pragma unroll
          for (int m = 0; m < K; ++m)
            v[m] = nbs >= 0 ? __ldg(un + p + P * m) : Real(0); // zeros without a neighbour
          cstore<Real, D, K, D - 1>(F, p, v);
        }
    }
  cstore<Real, D, K, D - 1>(U, p, x);
  for (int phi = p; phi < 2 * D; phi += P)
    {
      int2 f = make_int2(-2, 0);
#pragma unroll
      for (int i = 0; i < 2 * D; ++i)
        f = (i == phi) ? tf[i] : f;
      Real a1 = Real(0), a2 = Real(0), a3 = Real(0);
      if (f.x != -2)
        {
          const int fid = f.y & 0x3fffffff;
          const int side = (f.y >> 30) & 1;
          const int a = phi / 2;
          const Real *fg = prm.face_geo + (long long)fid * (2 * D + 1);
          const Real jx = __ldg(fg);
          const Real jo = __ldg(fg + 1 + side * D + a);
          const Real tau = __ldg(prm.penalty + fid);
          if (f.x == -1)
            {
              a1 = Real(2) * tau * jx;
              a2 = -(jo * jx);
            }
          else
            {
              const Real jb = __ldg(fg + 1 + (1 - side) * D + a);
              const Real hs = side == 0 ? Real(0.5) : Real(-0.5);
              a1 = tau * jx;
              a2 = -(hs * jo * jx);
              a3 = -(hs * jb * jx);
            }
        }
      Real *fc = U + CS::OFF_FC + 3 * phi;
      fc[0] = a1;
      fc[1] = a2;
      fc[2] = a3;
    }
  for (int a = p; a < D; a += P)
    {
      Real c = Real(0);
      if (geo >= 0)
        {
          // (J^{-T}_aa)^2 det J; off-diagonal round-off (<= 1e-13 relative) dropped
          const Real *cg = prm.cell_geo + (long long)geo * (D * D + 1);
          const Real j = __ldg(cg + a * D + a);
          c = (j * j) * __ldg(cg + D * D);
        }
      U[CS::OFF_CC + a] = c;
    }
  __syncthreads();

  if constexpr (HERM)
    {
      // y = M_x M_y t_z + M_z (M_y t_x + M_x t_y), t_a = L_a u (two mass products
      // per axis; no inverse of the ill-conditioned Hermite-like mass matrix)
      cart_line<Real, D, K, D - 1, GLN, HERM>(U, x, nu[D - 1], nd[D - 1], t);
      cstore<Real, D, K, D - 1>(Cf, p, t); // t of the last axis
      if constexpr (STAGE)
        cart_nb_staged<Real, D, K, 0, GLN, HERM>(xin[0] ? U - CS::SM_CELL : Af, xin[1] ? U + CS::SM_CELL : Bf,
                                                 p0, sp0, nu[0], nd[0], xin[0], xin[1]);
      cload<Real, D, K, 0>(U, p0, x);
      cart_line<Real, D, K, 0, GLN, HERM>(U, x, nu[0], nd[0], t); // t_x, kept in registers
      __syncthreads(); // staging fields free, C complete
      if constexpr (D == 3)
        {
          cstore<Real, D, K, 0>(Af, p0, t); // t_x
          cload<Real, D, K, 0>(Cf, p0, x);
          apply_M1<Real, K>(x, t);
          cstore<Real, D, K, 0>(Cf, p0, t); // M_x t_z
          __syncthreads();
          if constexpr (STAGE)
            cart_nb_staged<Real, D, K, 1, GLN, HERM>(Cf + FS, Cf + 2 * FS, p1, sp1, nu[1], nd[1]);
          cload<Real, D, K, 1>(U, p1, x);
          cart_line<Real, D, K, 1, GLN, HERM>(U, x, nu[1], nd[1], t);
          cstore<Real, D, K, 1>(Bf, p1, t); // t_y
          cload<Real, D, K, 1>(Af, p1, x);
          apply_M1<Real, K>(x, t);
          cstore<Real, D, K, 1>(Af, p1, t); // M_y t_x
          cload<Real, D, K, 1>(Cf, p1, x);
          apply_M1<Real, K>(x, t);
          cstore<Real, D, K, 1>(Cf, p1, t); // M_y M_x t_z
          __syncthreads();
          cload<Real, D, K, 0>(Bf, p0, x);
          apply_M1<Real, K>(x, t);
          cload<Real, D, K, 0>(Af, p0, x);
#pragma unroll
          for (int m = 0; m < K; ++m)
            t[m] += x[m];
          cstore<Real, D, K, 0>(Af, p0, t); // M_y t_x + M_x t_y
          __syncthreads();
          cload<Real, D, K, 2>(Af, p, x);
          apply_M1<Real, K>(x, t);
          cload<Real, D, K, 2>(Cf, p, x);
        }
      else
        {
          cstore<Real, D, K, 0>(Bf, p0, t); // t_x
          cload<Real, D, K, 0>(Cf, p0, x);
          apply_M1<Real, K>(x, t);
          cstore<Real, D, K, 0>(Cf, p0, t); // M_x t_y
          __syncthreads();
          cload<Real, D, K, 1>(Bf, p, x);
          apply_M1<Real, K>(x, t);
          cload<Real, D, K, 1>(Cf, p, x);
        }
#pragma unroll
      for (int m = 0; m < K; ++m)
        t[m] += x[m];
    }
  else
    {
      // last axis (line p, in registers since the load): C = M^{-1} L u along it
      cart_line<Real, D, K, D - 1, GLN, HERM>(U, x, nu[D - 1], nd[D - 1], t);
      cstore<Real, D, K, D - 1>(Cf, p, t);
      if constexpr (STAGE)
        {
          cart_nb_staged<Real, D, K, 0, GLN, HERM>(xin[0] ? U - CS::SM_CELL : Af, xin[1] ? U + CS::SM_CELL : Bf, p0,
                                                   sp0, nu[0], nd[0]);
          // (the y-neighbours' fields are not reused: their scalars are taken in
          // the y-phase, which keeps four values out of the registers until then)
        }
      cload<Real, D, K, 0>(U, p0, x);
      cart_line<Real, D, K, 0, GLN, HERM>(U, x, nu[0], nd[0], t); // along x, kept in registers
      __syncthreads(); // C complete
      cload<Real, D, K, 0>(Cf, p0, x);
#pragma unroll
      for (int m = 0; m < K; ++m)
        t[m] += x[m];
      if constexpr (D == 3)
        {
          cstore<Real, D, K, 0>(Cf, p0, t); // sum over z and x
          __syncthreads();
          if constexpr (STAGE)
            cart_nb_staged<Real, D, K, 1, GLN, HERM>(Cf + FS, Cf + 2 * FS, p1, sp1, nu[1], nd[1]);
          cload<Real, D, K, 1>(U, p1, x);
          cart_line<Real, D, K, 1, GLN, HERM>(U, x, nu[1], nd[1], t);
          cload<Real, D, K, 1>(Cf, p1, x);
#pragma unroll
          for (int m = 0; m < K; ++m)
            x[m] += t[m]; // w = sum_a M_a^{-1} L_a u on this y-line
          apply_M1<Real, K>(x, t);
          cstore<Real, D, K, 1>(Cf, p1, t); // M_y w
          __syncthreads();
          cload<Real, D, K, 0>(Cf, p0, x);
          apply_M1<Real, K>(x, t);
          cstore<Real, D, K, 0>(Cf, p0, t); // M_x M_y w
          __syncthreads();
          cload<Real, D, K, 2>(Cf, p, x);
          apply_M1<Real, K>(x, t); // y = M_z M_x M_y w
        }
      else
        {
          apply_M1<Real, K>(t, x);
          cstore<Real, D, K, 0>(Cf, p0, x); // M_x w
          __syncthreads();
          cload<Real, D, K, 1>(Cf, p, x);
          apply_M1<Real, K>(x, t); // y = M_y M_x w
        }
    }
  if (active)
    {
      Real *yc = prm.y + (long long)slot * NQ;
#pragma unroll
      for (int m = 0; m < K; ++m)
        {
          Real v = t[m];
          if constexpr (HERM)
            v = ((gmask >> m) & 1u) ? v * (sp * hsign<Real, K>(m)) : Real(0);
          __stcs(yc + p + P * m, v); // y is not read again (streaming)
        }
    }
}

} // namespace dev
} // namespace dgx

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
// Thread layout as sipg_apply_kernel: P = K^{D-1} threads per cell, thread p
// holds one nodal line along the current axis in registers; 1D matrices are
// mirror-symmetric and applied in even-odd form from the constant bank.
//   3D:  z: t_z -> C;  x: t_x -> A, C <- M_x C;  y: t_y -> B, A <- M_y A,
//        C <- M_y C;  x: A <- A + M_x B;  z: y = M_z A + C.
// 17 shared-memory field passes and 9 1D products per cell, against 59 and 12
// (+ the face phase) of the collocation kernels.
#pragma once

namespace dgx
{
namespace dev
{

template <typename Real, int D, int K>
struct CartShape
{
  using L = SL<D, K>;
  static constexpr int P = L::P;
  static constexpr int FS = L::FS;
  static constexpr int NF = D == 3 ? 4 : 3; // U, A, B (, C)
  static constexpr int SM_CELL = NF * FS;
  static constexpr int NC = (192 / P) > 0 ? 192 / P : 1;
  static constexpr int THREADS = NC * P;
  static constexpr int SMEM_REALS = NC * SM_CELL;
  // registers: four lines of K values (own, result, two neighbours)
  static constexpr int REGS = 4 * K * (int)(sizeof(Real) / 4) + 40;
  static constexpr int WARP_THREADS = (THREADS + 31) / 32 * 32;
  static constexpr int MB_REGS = 65536 / (WARP_THREADS * REGS);
  static constexpr int MB_SMEM = (220 * 1024) / (SMEM_REALS * (int)sizeof(Real) + 1024);
  static constexpr int MB0 = MB_REGS < MB_SMEM ? MB_REGS : MB_SMEM;
  static constexpr int MINB = MB0 < 1 ? 1 : (MB0 > 6 ? 6 : MB0);
};

template <typename Real, int K>
__device__ __forceinline__ void apply_M1(const Real (&x)[K], Real (&y)[K])
{
  eo_sym<Real, K, TabLayout<K>::oM1E, TabLayout<K>::oM1O>(x, y);
}

// One face (side S of the line's axis A) of the line operator: adds
// rv Sf_S^T + g jo Df_S^T to t. u: own nodal line, xn: the neighbour's line
// through the same face point (zeros if there is none).
template <typename Real, int D, int K, int A, int S, bool GLN>
__device__ __forceinline__ void cart_face(const ApplyParams<Real> &prm, const int2 tf,
                                          const Real (&u)[K], const Real (&xn)[K], Real (&t)[K])
{
  using T = TabLayout<K>;
  if (tf.x == -2)
    return; // not computed on this rank (arrives by compress)
  const int fid = tf.y & 0x3fffffff;
  const int side = (tf.y >> 30) & 1;
  const Real *fg = prm.face_geo + (long long)fid * (2 * D + 1);
  const Real jx = __ldg(fg);
  const Real jo = __ldg(fg + 1 + side * D + A);
  const Real tau = __ldg(prm.penalty + fid);
  const Real uf = GLN ? (S == 0 ? u[0] : u[K - 1]) : dot_row<Real, K, T::oSf + S * K>(u);
  const Real dno = dot_row<Real, K, T::oDf + S * K>(u) * jo;
  Real rv, g;
  if (tf.x == -1)
    {
      // boundary face, mirror rule (operators.cpp:1069-1089)
      rv = (uf * tau * Real(2) - dno) * jx;
      g = -(uf * jx);
    }
  else
    {
      const Real jb = __ldg(fg + 1 + (1 - side) * D + A);
      const Real nu = GLN ? (S == 0 ? xn[K - 1] : xn[0]) : dot_row<Real, K, T::oSf + (1 - S) * K>(xn);
      const Real dnb = dot_row<Real, K, T::oDf + (1 - S) * K>(xn) * jb;
      const Real sgn = side == 0 ? Real(1) : Real(-1);
      const Real delta = uf - nu;
      rv = (delta * tau - sgn * ((dno + dnb) * Real(0.5))) * jx;
      g = -(sgn * delta * jx * Real(0.5));
    }
  const Real gj = g * jo;
  if constexpr (GLN)
    {
      // Gauss-Lobatto: Sf rows are exact unit vectors (the end nodes)
      t[S == 0 ? 0 : K - 1] += rv;
#pragma unroll
      for (int m = 0; m < K; ++m)
        t[m] += gj * tab<Real, K>(T::oDf + S * K + m);
    }
  else
    {
#pragma unroll
      for (int m = 0; m < K; ++m)
        t[m] += rv * tab<Real, K>(T::oSf + S * K + m) + gj * tab<Real, K>(T::oDf + S * K + m);
    }
}

// t = L_A u for the nodal line p along axis A of the task's cell
template <typename Real, int D, int K, int A, bool GLN>
__device__ __forceinline__ void cart_line(const ApplyParams<Real> &prm, bool active, const int2 *tfp,
                                          int geo, int p, const Real (&u)[K], Real (&t)[K])
{
  using T = TabLayout<K>;
  constexpr int NQ = ipow_c(K, D);
  int2 tf[2];
  Real xn[2][K];
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      tf[s] = active ? __ldg(tfp + 2 * A + s) : make_int2(-2, 0);
      const bool nb = tf[s].x >= 0;
      const Real *un = prm.u + (long long)(nb ? tf[s].x : 0) * NQ;
#pragma unroll
      for (int m = 0; m < K; ++m)
        xn[s][m] = nb ? __ldg(un + gidx<D, K, A>(p, m)) : Real(0);
    }
  Real c = Real(0);
  if (geo >= 0)
    {
      const Real *cg = prm.cell_geo + (long long)geo * (D * D + 1);
      const Real j = __ldg(cg + A * D + A);
      c = (j * j) * __ldg(cg + D * D);
    }
  eo_sym<Real, K, T::oK1E, T::oK1O>(u, t);
#pragma unroll
  for (int m = 0; m < K; ++m)
    t[m] *= c;
  cart_face<Real, D, K, A, 0, GLN>(prm, tf[0], u, xn[0], t);
  cart_face<Real, D, K, A, 1, GLN>(prm, tf[1], u, xn[1], t);
}

template <typename Real, int D, int K, int BASIS>
__global__ void __launch_bounds__(CartShape<Real, D, K>::THREADS, CartShape<Real, D, K>::MINB)
  sipg_cart_kernel(const ApplyParams<Real> prm)
{
  static_assert(BASIS != 2, "the Hermite-like basis runs the collocation kernels");
  using CS = CartShape<Real, D, K>;
  using L = SL<D, K>;
  constexpr int P = L::P, NQ = L::NQ, FS = L::FS, NC = CS::NC;
  constexpr bool GLN = BASIS == 0;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Real *smem = reinterpret_cast<Real *>(smem_raw);
  const int lc = threadIdx.x / P;
  const int p = threadIdx.x - lc * P;
  const int task = blockIdx.x * NC + lc;
  const bool active = task < prm.n_tasks;
  Real *U = smem + lc * CS::SM_CELL;
  Real *Af = U + FS;
  Real *Bf = Af + FS;
  const int slot = active ? prm.task_slot[task] : 0;
  const int geo = active ? prm.task_geo[task] : -1;
  const int2 *tfp = prm.task_face + (long long)(active ? task : 0) * 2 * D;

  Real x[K], t[K];
  // last axis: the thread's line is contiguous across threads in HBM
  {
    const Real *uc = prm.u + (long long)slot * NQ;
#pragma unroll
    for (int m = 0; m < K; ++m)
      x[m] = active ? __ldg(uc + p + P * m) : Real(0);
  }
  cart_line<Real, D, K, D - 1, GLN>(prm, active, tfp, geo, p, x, t);
  store_pencil<Real, D, K, D - 1>(U, p, x);
  if constexpr (D == 3)
    {
      Real *Cf = Bf + FS;
      store_pencil<Real, D, K, 2>(Cf, p, t); // t_z
      __syncthreads();
      load_pencil<Real, D, K, 0>(U, p, x);
      cart_line<Real, D, K, 0, GLN>(prm, active, tfp, geo, p, x, t);
      store_pencil<Real, D, K, 0>(Af, p, t); // t_x
      load_pencil<Real, D, K, 0>(Cf, p, x);
      apply_M1<Real, K>(x, t);
      store_pencil<Real, D, K, 0>(Cf, p, t); // M_x t_z
      __syncthreads();
      load_pencil<Real, D, K, 1>(U, p, x);
      cart_line<Real, D, K, 1, GLN>(prm, active, tfp, geo, p, x, t);
      store_pencil<Real, D, K, 1>(Bf, p, t); // t_y
      load_pencil<Real, D, K, 1>(Af, p, x);
      apply_M1<Real, K>(x, t);
      store_pencil<Real, D, K, 1>(Af, p, t); // M_y t_x
      load_pencil<Real, D, K, 1>(Cf, p, x);
      apply_M1<Real, K>(x, t);
      store_pencil<Real, D, K, 1>(Cf, p, t); // M_y M_x t_z
      __syncthreads();
      load_pencil<Real, D, K, 0>(Bf, p, x);
      apply_M1<Real, K>(x, t);
      load_pencil<Real, D, K, 0>(Af, p, x);
#pragma unroll
      for (int m = 0; m < K; ++m)
        t[m] += x[m];
      store_pencil<Real, D, K, 0>(Af, p, t); // M_y t_x + M_x t_y
      __syncthreads();
      load_pencil<Real, D, K, 2>(Af, p, x);
      apply_M1<Real, K>(x, t);
      load_pencil<Real, D, K, 2>(Cf, p, x);
    }
  else
    {
      store_pencil<Real, D, K, 1>(Af, p, t); // t_y
      __syncthreads();
      load_pencil<Real, D, K, 0>(U, p, x);
      cart_line<Real, D, K, 0, GLN>(prm, active, tfp, geo, p, x, t);
      store_pencil<Real, D, K, 0>(Bf, p, t); // t_x
      load_pencil<Real, D, K, 0>(Af, p, x);
      apply_M1<Real, K>(x, t);
      store_pencil<Real, D, K, 0>(Af, p, t); // M_x t_y
      __syncthreads();
      load_pencil<Real, D, K, 1>(Bf, p, x);
      apply_M1<Real, K>(x, t);
      load_pencil<Real, D, K, 1>(Af, p, x);
    }
  if (active)
    {
      Real *yc = prm.y + (long long)slot * NQ;
#pragma unroll
      for (int m = 0; m < K; ++m)
        __stcs(yc + p + P * m, t[m] + x[m]); // y is not read again (streaming)
    }
}

} // namespace dev
} // namespace dgx

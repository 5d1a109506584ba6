// Face phase of the fused SIPG apply (included by sipg_kernel.cuh).
#pragma once

namespace dgx
{
namespace dev
{

// Global load of two consecutive dofs (m, m+1) of the pencil along axis A
// through face point p. Along axis 0 they are adjacent in memory (the
// pencil is K contiguous values at K p), and for even K and fp64 16-byte
// aligned: one vector load instead of two strided scalar ones (halves the
// L1 sectors of the x-neighbour reads).
template <typename Real, int D, int K, int A>
__device__ __forceinline__ void ldg_pair(const Real *un, int p, int m, Real &a, Real &b)
{
  if constexpr (A == 0 && sizeof(Real) == 8 && K % 2 == 0)
    {
      const double2 v = __ldg(reinterpret_cast<const double2 *>(un + gidx<D, K, A>(p, m)));
      a = v.x;
      b = v.y;
    }
  else
    {
      a = __ldg(un + gidx<D, K, A>(p, m));
      b = __ldg(un + gidx<D, K, A>(p, m + 1));
    }
}

// The neighbour pencils through face point p of both faces of axis A
// (nodal bases), fetched one phase early (across the forward pass's last
// barrier for axis 0, during the previous axis's test-side passes otherwise)
template <typename Real, int D, int K, int A, bool CART = false>
__device__ __forceinline__ void nb_fetch_v4(const ApplyParams<Real> &prm, const Real *cell, bool active, int p,
                                            Real (&x)[2][K])
{
  using L = SL<D, K, CART>;
  constexpr int NQ = L::NQ;
  int2 tf[2] = {make_int2(-2, 0), make_int2(-2, 0)};
  if (active)
    {
      const int2 *tfs = reinterpret_cast<const int2 *>(cell + L::OFF_TF);
      tf[0] = tfs[2 * A];
      tf[1] = tfs[2 * A + 1];
    }
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      const Real *un = prm.u + (long long)(tf[s].x >= 0 ? tf[s].x : 0) * NQ;
#pragma unroll
      for (int m = 0; m + 1 < K; m += 2)
        {
          ldg_pair<Real, D, K, A>(un, p, m, x[s][m], x[s][m + 1]);
          if (tf[s].x < 0)
            x[s][m] = x[s][m + 1] = Real(0);
        }
      if constexpr (K % 2 == 1)
        x[s][K - 1] = tf[s].x >= 0 ? __ldg(un + gidx<D, K, A>(p, K - 1)) : Real(0);
    }
}

// Both faces of axis A of every cell in the CTA (runs before the
// quadrature-point phase, so G still holds the reference gradient):
//  own traces      value and reference gradient at the face points from the
//                  collocation fields: u = rf val, g_b = rf G_b along the
//                  normal (exact: rf extrapolates polynomials of degree < k);
//  neighbour trace nodal Sf/Df rows of the neighbour's opposite face, then
//                  two tangential passes: along t1 (S and the nodal
//                  derivative D on the value layer, S on the normal
//                  derivative), along t0 (S on all, D on the value) --
//                  the same algebra as face_eval + face_tangential_derivative
//                  (operators.cpp:794-858, 766-788) in two passes;
//  SIPG flux       operators.cpp:977-1003 (interior), 1069-1089 (boundary);
//  test side       w = rv + sum_t Dco_t^T rg_t on the face
//                  (face_tangential_integrate, :782-788) and rg_A, stored to
//                  OUT for the backward pass.
template <typename Real, int D, int K, int A, bool COMPRESSED, bool HERM, bool GLN, typename HOOK>
__device__ __forceinline__ void face_axis_v4(const ApplyParams<Real> &prm, Real *cell, int task,
                                             bool active, int p, Real wf, Real sp,
                                             const Real (&xnb)[2][K], HOOK &&before_wpass)
{
  using L = SL<D, K>;
  using T = TabLayout<K>;
  constexpr int P = L::P, NQ = L::NQ, FP = L::FP, NL = L::NL, FS = L::FS;
  const Real *val = cell;
  const Real *G = cell + L::OFF_G;
  Real *NB = cell + L::OFF_NB;  // face s: nu (2s), nw (2s+1)
  Real *DT = cell + L::OFF_DT;  // neighbour d/dt0 (s), d/dt1 (2 + s)
  Real *OUT = cell + L::OFF_OUT + (2 * A) * 2 * FP; // face s: w (2s), rgn (2s+1)
  const int fp = fpt<D, K>(p);

  int2 tf[2] = {make_int2(-2, 0), make_int2(-2, 0)};
  if (active)
    {
      // stashed by the prologue (ordered by the forward-pass barriers)
      const int2 *tfs = reinterpret_cast<const int2 *>(cell + L::OFF_TF);
      tf[0] = tfs[2 * A];
      tf[1] = tfs[2 * A + 1];
    }
  // face geometry at face point p (issued first: longest latency)
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
          if constexpr (COMPRESSED)
            {
              // Cartesian: one record per face, JxW_f = det |J^{-T} e| w_q
              const Real *fg = prm.face_geo + (long long)fid * (2 * D + 1);
              jxw[s] = __ldg(fg) * wf;
#pragma unroll
              for (int b = 0; b < D; ++b)
                {
                  jo[s][b] = __ldg(fg + 1 + side * D + b);
                  jb[s][b] = __ldg(fg + 1 + (1 - side) * D + b);
                }
            }
          else
            {
              const Real *fg = prm.face_geo + (long long)fid * (2 * D + 1) * P + p;
              jxw[s] = __ldg(fg);
#pragma unroll
              for (int b = 0; b < D; ++b)
                {
                  jo[s][b] = __ldg(fg + (1 + side * D + b) * P);
                  jb[s][b] = __ldg(fg + (1 + (1 - side) * D + b) * P);
                }
            }
          tau[s] = __ldg(prm.penalty + fid);
        }
    }
  // own traces from the collocation fields along the normal (first: their
  // shared-memory loads overlap the arrival of the neighbour pencils)
  Real own_u[2], own_g[2][D];
  {
    Real x[K];
    load_pencil<Real, D, K, A>(val, p, x);
    own_u[0] = dot_row<Real, K, T::oRf>(x);
    own_u[1] = dot_row<Real, K, T::oRf + K>(x);
#pragma unroll
    for (int b = 0; b < D; ++b)
      {
        load_pencil<Real, D, K, A>(G + b * FS, p, x);
        own_g[0][b] = dot_row<Real, K, T::oRf>(x);
        own_g[1][b] = dot_row<Real, K, T::oRf + K>(x);
      }
  }
  // neighbour pencils -> nodal value / normal-derivative layer (own low face
  // meets the neighbour's high face, row index 1, and vice versa). Both
  // neighbours' loads are issued before either is used: one memory latency
  // per axis, not two.
  if constexpr (HERM)
    {
      // two layers: value and derivative live on the edge layer and its
      // inner neighbour (read_face_dofs, dof_layout.hpp:291-336)
      Real xe[2], xi[2];
#pragma unroll
      for (int s = 0; s < 2; ++s)
        {
          xe[s] = xi[s] = Real(0);
          if (tf[s].x >= 0)
            {
              const Real *un = prm.u + (long long)tf[s].x * NQ;
              if (s == 0)
                ldg_pair<Real, D, K, A>(un, p, K - 2, xi[s], xe[s]);
              else
                ldg_pair<Real, D, K, A>(un, p, 0, xe[s], xi[s]);
            }
        }
#pragma unroll
      for (int s = 0; s < 2; ++s)
        {
          const int me = s == 0 ? K - 1 : 0, mi = s == 0 ? K - 2 : 1;
          const int ro = s == 0 ? K : 0;
          const Real ve = xe[s] * (sp * hsign<Real, K>(me));
          const Real vi = xi[s] * (sp * hsign<Real, K>(mi));
          NB[(2 * s) * FP + fp] =
            tab<Real, K>(T::oSf + ro + me) * ve + tab<Real, K>(T::oSf + ro + mi) * vi;
          NB[(2 * s + 1) * FP + fp] =
            tab<Real, K>(T::oDf + ro + me) * ve + tab<Real, K>(T::oDf + ro + mi) * vi;
        }
    }
  else
    {
      const Real(&x)[2][K] = xnb; // fetched one phase early (nb_fetch_v4)
      // Gauss-Lobatto nodes: the value rows Sf are exact unit vectors
      NB[fp] = GLN ? x[0][K - 1] : dot_row<Real, K, T::oSf + K>(x[0]);
      NB[FP + fp] = dot_row<Real, K, T::oDf + K>(x[0]);
      NB[2 * FP + fp] = GLN ? x[1][0] : dot_row<Real, K, T::oSf>(x[1]);
      NB[3 * FP + fp] = dot_row<Real, K, T::oDf>(x[1]);
    }
  __syncthreads();

  if constexpr (D == 3)
    {
      // pass 1, along t1: nu -> (S nu, D nu -> DT[2+s]); nw -> S nw
      for (int t = p; t < 4 * NL; t += P)
        {
          const int f = t / NL, l = t - f * NL;
          Real a[K], b[K];
          load_line<Real, D, K, 1>(NB + f * FP, l, a);
          apply_S<Real, K>(a, b);
          store_line<Real, D, K, 1>(NB + f * FP, l, b);
          if ((f & 1) == 0)
            {
              apply_Dn<Real, K>(a, b);
              store_line<Real, D, K, 1>(DT + (2 + f / 2) * FP, l, b);
            }
        }
      __syncthreads();
      // pass 2, along t0: nu -> (S nu, D nu -> DT[s]); nw, dt1 -> S
      for (int t = p; t < 6 * NL; t += P)
        {
          const int f = t / NL, l = t - f * NL;
          Real *fld = f < 4 ? NB + f * FP : DT + (2 + (f - 4)) * FP;
          Real a[K], b[K];
          load_line<Real, D, K, 0>(fld, l, a);
          apply_S<Real, K>(a, b);
          store_line<Real, D, K, 0>(fld, l, b);
          if (f < 4 && (f & 1) == 0)
            {
              apply_Dn<Real, K>(a, b);
              store_line<Real, D, K, 0>(DT + (f / 2) * FP, l, b);
            }
        }
      __syncthreads();
    }
  else
    {
      for (int t = p; t < 4; t += P)
        {
          Real a[K], b[K];
          load_line<Real, D, K, 0>(NB + t * FP, 0, a);
          apply_S<Real, K>(a, b);
          store_line<Real, D, K, 0>(NB + t * FP, 0, b);
          if ((t & 1) == 0)
            {
              apply_Dn<Real, K>(a, b);
              store_line<Real, D, K, 0>(DT + (t / 2) * FP, 0, b);
            }
        }
      __syncthreads();
    }

  // flux at face point p for both faces
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      Real rv = Real(0), g = Real(0);
      if (tf[s].x != -2)
        {
          const int side = (tf[s].y >> 30) & 1;
          Real dn_own = own_g[s][0] * jo[s][0];
#pragma unroll
          for (int b = 1; b < D; ++b)
            dn_own += own_g[s][b] * jo[s][b];
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
      // tangential test components into the neighbour-derivative slots
      // (each thread overwrites only the entries it has just read)
#pragma unroll
      for (int t = 0; t < D - 1; ++t)
        DT[(2 * t + s) * FP + fp] = g * jo[s][t < A ? t : t + 1];
    }
  __syncthreads();
  before_wpass();
  // w = rv + sum_t Dco_t^T rg_t, one tangential direction at a time
  if constexpr (D == 3 && DGX_V4_W1)
    {
      // both directions in one phase: rows accumulate into OUT, columns go
      // to W1 (summed in add_face_terms)
      Real *W1 = cell + L::OFF_W1 + (2 * A) * FP;
      for (int t = p; t < 4 * NL; t += P)
        {
          const int s = (t / NL) & 1, l = t % NL;
          if (t < 2 * NL)
            line_op<Real, D, K, 0, 3>(OUT + 2 * s * FP, DT + s * FP, l);
          else
            line_op<Real, D, K, 1, 4>(W1 + s * FP, DT + (2 + s) * FP, l);
        }
      return;
    }
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
  // no trailing barrier: the next axis's first step touches only NB and
  // reads val/G, disjoint from OUT/DT used above, and its own barrier orders
  // everything after it; the quadrature-point phase that follows the last
  // axis writes only G and is followed by a barrier before OUT is read
}

// Both faces of axis A on axis-aligned affine records (CART: J^{-T}
// diagonal and constant per cell, n.J^{-T} = (0, .., j_A, .., 0) per face,
// verified at setup to 1e-13 relative: a box mesh's Jacobian carries
// off-axis round-off of ~1e-17). The general phase above multiplies the
// tangential derivatives and tangential test components by these (near)
// zeros; here they are skipped: dn = j_A g_A on each side
// (operators.cpp:977-1003, 1069-1089 without the off-axis terms), so only
// the value and normal-derivative traces of the neighbour are interpolated
// (two S passes each) and the test side is w = rv, rg_A = g j_A (no
// tangential Dco^T passes). Results differ from the general path by the
// dropped round-off terms (relative ~1e-16), far inside the 1e-12 parity
// tolerance.
template <typename Real, int D, int K, int A, bool HERM, bool GLN, typename HOOK>
__device__ __forceinline__ void face_axis_cart(const ApplyParams<Real> &prm, Real *cell, bool active, int p,
                                               Real wf, Real sp, const Real (&xnb)[2][K], HOOK &&after_flux)
{
  using L = SL<D, K, true>;
  using T = TabLayout<K>;
  constexpr int NQ = L::NQ, FP = L::FP, NL = L::NL, FS = L::FS;
  const Real *val = cell;
  const Real *G = cell + L::OFF_G;
  Real *NB = cell + L::OFF_NB;  // face s: nu (2s), nw (2s+1)
  Real *OUT = cell + L::OFF_OUT + (2 * A) * 2 * FP; // face s: w (2s), rgn (2s+1)
  const int fp = fpt<D, K>(p);

  int2 tf[2] = {make_int2(-2, 0), make_int2(-2, 0)};
  if (active)
    {
      const int2 *tfs = reinterpret_cast<const int2 *>(cell + L::OFF_TF);
      tf[0] = tfs[2 * A];
      tf[1] = tfs[2 * A + 1];
    }
  Real jxw[2], tau[2], jo[2], jb[2];
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      jxw[s] = tau[s] = jo[s] = jb[s] = Real(0);
      if (tf[s].x != -2)
        {
          const int fid = tf[s].y & 0x3fffffff;
          const int side = (tf[s].y >> 30) & 1;
          const Real *fg = prm.face_geo + (long long)fid * (2 * D + 1);
          jxw[s] = __ldg(fg) * wf;
          jo[s] = __ldg(fg + 1 + side * D + A);
          jb[s] = __ldg(fg + 1 + (1 - side) * D + A);
          tau[s] = __ldg(prm.penalty + fid);
        }
    }
  // own value and normal-gradient traces (rf rows along the normal)
  Real own_u[2], own_g[2];
  {
    Real x[K];
    load_pencil<Real, D, K, A>(val, p, x);
    own_u[0] = dot_row<Real, K, T::oRf>(x);
    own_u[1] = dot_row<Real, K, T::oRf + K>(x);
    load_pencil<Real, D, K, A>(G + A * FS, p, x);
    own_g[0] = dot_row<Real, K, T::oRf>(x);
    own_g[1] = dot_row<Real, K, T::oRf + K>(x);
  }
  if constexpr (HERM)
    {
      Real xe[2], xi[2];
#pragma unroll
      for (int s = 0; s < 2; ++s)
        {
          xe[s] = xi[s] = Real(0);
          if (tf[s].x >= 0)
            {
              const Real *un = prm.u + (long long)tf[s].x * NQ;
              if (s == 0)
                ldg_pair<Real, D, K, A>(un, p, K - 2, xi[s], xe[s]);
              else
                ldg_pair<Real, D, K, A>(un, p, 0, xe[s], xi[s]);
            }
        }
#pragma unroll
      for (int s = 0; s < 2; ++s)
        {
          const int me = s == 0 ? K - 1 : 0, mi = s == 0 ? K - 2 : 1;
          const int ro = s == 0 ? K : 0;
          const Real ve = xe[s] * (sp * hsign<Real, K>(me));
          const Real vi = xi[s] * (sp * hsign<Real, K>(mi));
          NB[(2 * s) * FP + fp] =
            tab<Real, K>(T::oSf + ro + me) * ve + tab<Real, K>(T::oSf + ro + mi) * vi;
          NB[(2 * s + 1) * FP + fp] =
            tab<Real, K>(T::oDf + ro + me) * ve + tab<Real, K>(T::oDf + ro + mi) * vi;
        }
    }
  else
    {
      const Real(&x)[2][K] = xnb;
      NB[fp] = GLN ? x[0][K - 1] : dot_row<Real, K, T::oSf + K>(x[0]);
      NB[FP + fp] = dot_row<Real, K, T::oDf + K>(x[0]);
      NB[2 * FP + fp] = GLN ? x[1][0] : dot_row<Real, K, T::oSf>(x[1]);
      NB[3 * FP + fp] = dot_row<Real, K, T::oDf>(x[1]);
    }
  __syncthreads();
  // neighbour value / normal derivative to the face Gauss points: S along
  // every tangential direction (face_eval's sweeps, operators.cpp:835-858)
  if constexpr (D == 3)
    {
      for (int t = p; t < 4 * NL; t += L::P)
        line_op<Real, D, K, 1, 0>(NB + (t / NL) * FP, nullptr, t % NL);
      __syncthreads();
    }
  for (int t = p; t < 4 * NL; t += L::P)
    line_op<Real, D, K, 0, 0>(NB + (t / NL) * FP, nullptr, t % NL);
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      Real rv = Real(0), g = Real(0);
      if (tf[s].x != -2)
        {
          const int side = (tf[s].y >> 30) & 1;
          const Real dn_own = own_g[s] * jo[s];
          if (tf[s].x == -1)
            {
              rv = (own_u[s] * tau[s] * Real(2) - dn_own) * jxw[s];
              g = -(own_u[s] * jxw[s]);
            }
          else
            {
              const Real nu = NB[(2 * s) * FP + fp], nw = NB[(2 * s + 1) * FP + fp];
              const Real dn_nb = nw * jb[s];
              const Real sgn = side == 0 ? Real(1) : Real(-1);
              const Real delta = own_u[s] - nu;
              rv = (delta * tau[s] - sgn * ((dn_own + dn_nb) * Real(0.5))) * jxw[s];
              g = -(sgn * delta * jxw[s] * Real(0.5));
            }
        }
      OUT[(2 * s) * FP + fp] = rv;
      OUT[(2 * s + 1) * FP + fp] = g * jo[s];
    }
  after_flux();
  // no trailing barrier: the next axis's first writes are NB at this
  // thread's own face point (read above by this thread only), and the
  // quadrature-point phase after the last axis is followed by a barrier
  // before OUT is read
}

} // namespace dev
} // namespace dgx

// Fused SIPG apply, "pencil-pair" kernel for 3D, even K, fp64 (included by
// sipg_launch.cuh after sipg_kernel.cuh; same algorithm and reference
// citations as sipg_apply_kernel, only the thread mapping and the
// shared-memory layout differ).
//
// Why: the single-pencil kernel is bound by the L1/shared data pipe (ncu:
// 81% busy, shared wavefronts 1.7x the conflict-free ideal, because 8-byte
// accesses are served per half-warp and 36-thread cells straddle
// half-warps). Here every thread owns TWO adjacent pencils, so every shared
// and global access of the kernel is a 16-byte vector of the pair: 16-byte
// accesses are served per quarter-warp (8 lanes x 16 B = 128 B), and the
// strides below make the quarter-warps conflict-free for the z- and
// y-pencil passes and for every face-point access.
//
// Thread t of a cell (P2 = K^2/2 threads), (c, w) = (t % H, t / H):
//   z pass: pencils (x = 2c, 2c+1; y = w)   -- pair adjacent along x
//   y pass: pencils (x = 2c, 2c+1; z = w)   -- pair adjacent along x
//   x pass: pencils (y = 2c, 2c+1; z = w)   -- each pencil contiguous
//   face axis A: face points (t0 = 2c, 2c+1; t1 = w), i.e. exactly the two
//   pencils along A of the pass above through those points.
// Shared volume fields: (x, y, z) at x + K y + S2 z with (S2/2) = H mod 8
// (z and y pair accesses hit quad t + const); face fields: (t0, t1) at
// t0 + K t1. Cell stride CS with (CS/2) = P2 mod 8, so quads stay
// t_global + const across the cells of a CTA.
#pragma once

// One warp per cell (DGX_PAIRS_WARP): a cell's threads are one warp, so every
// synchronisation is a __syncwarp and the cells of a CTA run independently
#ifndef DGX_PAIRS_WARP
#define DGX_PAIRS_WARP 0
#endif
#ifndef DGX_PAIRS_W1
#define DGX_PAIRS_W1 1
#endif
#ifndef DGX_EXP_NO_CELL_PF
#define DGX_EXP_NO_CELL_PF 0
#endif
#ifndef DGX_EXP_NO_META_PF
#define DGX_EXP_NO_META_PF 0
#endif
// own value and normal-gradient traces of every face axis computed in the
// forward pass, from the pencils the thread holds in registers there (val
// along y after S_y, along x / z in the G_0 / G_2 steps, and the G_A output
// of each): the face phase then loads only the two tangential gradient
// fields along A (2 instead of 4 volume-field loads per axis); the x-face
// points of a thread become its permuted x-pass pair (cx, wx)
#ifndef DGX_PAIRS_FWDTRACE
#define DGX_PAIRS_FWDTRACE 0
#endif
// neighbour trace along t0 as row dot products at the thread's own face
// points, fused with the flux (no row pass, one barrier less per axis)
#ifndef DGX_PAIRS_ROWDOT
#define DGX_PAIRS_ROWDOT 0 // measured (C4): 21.43 vs 20.99 ms (divergent constant loads, 168 registers)
#endif

namespace dgx
{
namespace dev
{

constexpr int pr_stride(int lo, int h) // smallest even s >= lo with (s/2) % 8 == h % 8
{
  return ((lo + 1) / 2 * 2 / 2 % 8 == h % 8) ? (lo + 1) / 2 * 2 : pr_stride((lo + 1) / 2 * 2 + 2, h);
}

template <int K>
struct PL
{
  // odd K: shared rows padded to KP = K + 1 (the second pencil of the last
  // pair is a dummy living in the padding: x = K for z/y pairs, y = K for
  // x pairs, t0 = K on faces); global accesses are then 8-byte scalars
  static constexpr bool ODD = (K & 1) != 0;
  static constexpr int KP = K + (K & 1);
  static constexpr int H = KP / 2;
  static constexpr int P2 = K * H;
  static constexpr int NQ = K * K * K;
  static constexpr int S2 = pr_stride(KP * (ODD ? KP : K), H); // volume plane stride
  static constexpr int FS = S2 * K;              // volume field (even)
  static constexpr int FK = KP;                  // face row stride
  // face field stride: K = 6 dense (FP/2 = 2 mod 8: the row passes and the
  // f-fastest column passes below are conflict-free)
  static constexpr int FP = K == 6 ? 36 : pr_stride(KP * K, H);
  static constexpr int OFF_G = FS;
#ifdef DGX_EXP_PAIRS_NO_FACE_SMALL // ablation: cell integral only, no face storage at all
  static constexpr int OFF_OUT = 4 * FS, OFF_W1 = OFF_OUT, OFF_NB = OFF_OUT, OFF_DT = OFF_OUT,
                       OFF_RG1 = OFF_OUT, OFF_TF = OFF_OUT;
#else
  static constexpr int OFF_OUT = 4 * FS;         // 3 axes x (w0, w1, rgn0, rgn1)
  // W1: the t1 part Dco_t1^T rg_t1 of the face test values, 3 axes x 2
  // faces, so that the row and column test passes run in one phase
  static constexpr int OFF_W1 = OFF_OUT + 12 * FP;
  static constexpr int OFF_NB = OFF_W1 + (DGX_PAIRS_W1 ? 6 * FP : 0);
  static constexpr int OFF_DT = OFF_NB + 4 * FP;
  static constexpr int OFF_RG1 = OFF_DT + 4 * FP; // row-dot variant: rg along t1, 2 faces
  static constexpr int OFF_TF = OFF_RG1 + (DGX_PAIRS_ROWDOT ? 2 * FP : 0); // 6 int2 face entries
#endif
  // threads per cell: P2 (option: rounded up to whole quarter-warps, so that
  // no quarter-warp mixes two cells; lanes >= P2 duplicate the last pair and
  // take line-operation tasks)
  static constexpr bool WARP = DGX_PAIRS_WARP && P2 <= 32;
#if DGX_PAIRS_WARP
  static constexpr int G = WARP ? 32 : P2;
#elif defined(DGX_PAIRS_PAD) // measured (C4): conflicts halve but the duplicated lanes cost more
  static constexpr int G = (P2 + 7) / 8 * 8;
#else
  static constexpr int G = P2;
#endif
  static constexpr int SM_CELL = pr_stride(OFF_TF + 7, G); // + the task's slot
  static constexpr int NC_THREADS = (160 / G) > 0 ? 160 / G : 1;
  static constexpr int NC_SMEM = (74 * 1024 / 8) / SM_CELL > 0 ? (74 * 1024 / 8) / SM_CELL : 1;
  // Brick CTAs: the CTA's cells form a 2x2x2 (BRICK 8) or 2x2x1 (BRICK 4)
  // brick of the task order (Operator::build_tasks); a face between two
  // cells of the brick takes the partner's own trace from shared memory
  // instead of re-evaluating it from the partner's nodal values.
#ifndef DGX_PAIRS_BRICK
#define DGX_PAIRS_BRICK 1 // measured (C4, 21.6 -> 21.1 ms); 2x2x2 and 2x2x1 bricks need NC = 8 or 4: slower (23.6, 22.1 ms)
#endif
  // BRICK 1: no reordering; consecutive tasks of the CTA that are
  // x-neighbours (the tiled task order runs along x) share their x-face.
#if DGX_PAIRS_WARP
  static constexpr int BRICK = 0; // cells do not synchronise with each other
#else
  static constexpr int BRICK = (DGX_PAIRS_BRICK == 1 || (DGX_PAIRS_BRICK > 1 && DGX_PAIRS_BRICK * SM_CELL * 8 <= 113 * 1024))
                                 ? DGX_PAIRS_BRICK : 0;
#endif
  // k = 4: 8 threads per cell; 4 cells = one warp per CTA (barriers are free)
  // and 8 CTAs per SM -- sweep p = 3 (117^3): 10 cells x 3 CTAs 4.68 ms,
  // 16 x 2 4.99, 8 x 4 4.52, 4 x 8 4.36
#ifdef DGX_PAIRS_NC
  static constexpr int NC = DGX_PAIRS_NC;
#else
  static constexpr int NC = BRICK > 1 ? BRICK : (K == 4 ? 4 : (NC_THREADS < NC_SMEM ? NC_THREADS : NC_SMEM));
#endif
  static constexpr int THREADS = NC * G;
#ifdef DGX_PAIRS_MINB
  static constexpr int MINB = DGX_PAIRS_MINB;
#else
  static constexpr int MINB = (K == 4 && !(BRICK > 1)) ? 8 : (220 * 1024) / (NC * SM_CELL * 8 + 1024) >= 3 ? 3 : 2; // CTAs per SM
#endif
  static constexpr int SMEM_REALS = NC * SM_CELL;
};

// timing ablation only (wrong results): face records / neighbour cells
// remapped into a small window that stays cache-resident
#ifdef DGX_EXP_FACE_RESIDENT
#define DGX_EXP_FID(f) ((f) & 1023)
#define DGX_EXP_NBSLOT(x) ((x) & 1023)
#else
#define DGX_EXP_FID(f) (f)
#define DGX_EXP_NBSLOT(x) (x)
#endif
template <int K>
__device__ __forceinline__ void pr_sync()
{
  if constexpr (PL<K>::WARP)
    __syncwarp();
  else
    __syncthreads();
}
// timing ablation only (wrong results): face-phase barriers removed
#ifdef DGX_EXP_NO_FACE_SYNC
#define DGX_EXP_FSYNC() ((void)0)
#else
#define DGX_EXP_FSYNC() pr_sync<K>()
#endif

__device__ __forceinline__ double2 lds2(const double *p) { return *reinterpret_cast<const double2 *>(p); }
__device__ __forceinline__ void sts2(double *p, double a, double b)
{
  *reinterpret_cast<double2 *>(p) = make_double2(a, b);
}

// offset of element m of pencil e (e = 0, 1) of the pair (c, w) along axis A
// in a volume array with row stride RS and plane stride PS
template <int K, int A, int RS, int PS>
__device__ __forceinline__ int pr_el(int c, int w, int e, int m)
{
  if constexpr (A == 2)
    return 2 * c + e + RS * w + PS * m;
  else if constexpr (A == 1)
    return 2 * c + e + RS * m + PS * w;
  else
    return m + RS * (2 * c + e) + PS * w;
}
// shared (padded) and global (unpadded, K^3 per cell) offsets
template <int K, int A>
__device__ __forceinline__ int pr_sh(int c, int w, int e, int m)
{
  return pr_el<K, A, PL<K>::KP, PL<K>::S2>(c, w, e, m);
}
template <int K, int A>
__device__ __forceinline__ int pr_gl(int c, int w, int e, int m)
{
  return pr_el<K, A, K, K * K>(c, w, e, m);
}

// load / store the pencil pair (c, w) along A in shared memory: x[e][m]
template <int K, int A>
__device__ __forceinline__ void pr_load(const double *f, int c, int w, double (&x)[2][K])
{
  constexpr int H = PL<K>::H;
  if constexpr (A == 0)
    {
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int j = 0; j < H; ++j)
          {
            const double2 v = lds2(f + pr_sh<K, A>(c, w, e, 2 * j));
            x[e][2 * j] = v.x;
            if (2 * j + 1 < K)
              x[e][2 * j + 1] = v.y;
          }
    }
  else
    {
#pragma unroll
      for (int m = 0; m < K; ++m)
        {
          const double2 v = lds2(f + pr_sh<K, A>(c, w, 0, m));
          x[0][m] = v.x;
          x[1][m] = v.y;
        }
    }
}
template <int K, int A>
__device__ __forceinline__ void pr_store(double *f, int c, int w, const double (&x)[2][K])
{
  constexpr int H = PL<K>::H;
  if constexpr (A == 0)
    {
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int j = 0; j < H; ++j)
          sts2(f + pr_sh<K, A>(c, w, e, 2 * j), x[e][2 * j], 2 * j + 1 < K ? x[e][2 * j + 1] : 0.0);
    }
  else
    {
#pragma unroll
      for (int m = 0; m < K; ++m)
        sts2(f + pr_sh<K, A>(c, w, 0, m), x[0][m], x[1][m]);
    }
}

// global (read-only path), predicated (branch-free: the loads of both faces
// stay in flight together); zeros where !pred and for the dummy pencil of
// an odd K. Even K: 16-byte pair loads; odd K: 8-byte loads (the pairs are
// not 16-byte aligned in the unpadded global layout)
template <int K, int A>
__device__ __forceinline__ void pr_ldg_if(bool pred, const double *f, int c, int w, double (&x)[2][K])
{
  const double2 z = make_double2(0.0, 0.0);
  if constexpr (!PL<K>::ODD)
    {
      if constexpr (A == 0)
        {
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int j = 0; j < K / 2; ++j)
              {
                const double2 v =
                  pred ? __ldg(reinterpret_cast<const double2 *>(f + pr_gl<K, A>(c, w, e, 2 * j))) : z;
                x[e][2 * j] = v.x;
                x[e][2 * j + 1] = v.y;
              }
        }
      else
        {
#pragma unroll
          for (int m = 0; m < K; ++m)
            {
              const double2 v = pred ? __ldg(reinterpret_cast<const double2 *>(f + pr_gl<K, A>(c, w, 0, m))) : z;
              x[0][m] = v.x;
              x[1][m] = v.y;
            }
        }
    }
  else
    {
      const bool p1 = pred && 2 * c + 1 < K;
#pragma unroll
      for (int m = 0; m < K; ++m)
        {
          x[0][m] = pred ? __ldg(f + pr_gl<K, A>(c, w, 0, m)) : 0.0;
          x[1][m] = p1 ? __ldg(f + pr_gl<K, A>(c, w, 1, m)) : 0.0;
        }
    }
}
template <int K, int A>
__device__ __forceinline__ void pr_ldg(const double *f, int c, int w, double (&x)[2][K])
{
  pr_ldg_if<K, A>(true, f, c, w, x);
}

// elements m and m+1 of both pencils of the pair along A (global)
template <int K, int A>
__device__ __forceinline__ void pr_ldg_two(const double *f, int c, int w, int m, double (&lo)[2],
                                           double (&hi)[2])
{
  if constexpr (PL<K>::ODD)
    {
      const bool p1 = 2 * c + 1 < K;
      lo[0] = __ldg(f + pr_gl<K, A>(c, w, 0, m));
      hi[0] = __ldg(f + pr_gl<K, A>(c, w, 0, m + 1));
      lo[1] = p1 ? __ldg(f + pr_gl<K, A>(c, w, 1, m)) : 0.0;
      hi[1] = p1 ? __ldg(f + pr_gl<K, A>(c, w, 1, m + 1)) : 0.0;
    }
  else if constexpr (A == 0)
    {
#pragma unroll
      for (int e = 0; e < 2; ++e)
        {
          const double2 v = __ldg(reinterpret_cast<const double2 *>(f + pr_gl<K, A>(c, w, e, m)));
          lo[e] = v.x;
          hi[e] = v.y;
        }
    }
  else
    {
      const double2 a = __ldg(reinterpret_cast<const double2 *>(f + pr_gl<K, A>(c, w, 0, m)));
      const double2 b = __ldg(reinterpret_cast<const double2 *>(f + pr_gl<K, A>(c, w, 0, m + 1)));
      lo[0] = a.x;
      lo[1] = a.y;
      hi[0] = b.x;
      hi[1] = b.y;
    }
}

// two values at global offset o (pair element e = 0) and o + 1 (e = 1; the
// dummy of an odd K reads nothing)
template <int K, bool LDCS = false>
__device__ __forceinline__ double2 pr_ldg_pt(const double *f, bool p1)
{
  if constexpr (!PL<K>::ODD)
    return LDCS ? __ldcs(reinterpret_cast<const double2 *>(f)) : __ldg(reinterpret_cast<const double2 *>(f));
  else
    return make_double2(LDCS ? __ldcs(f) : __ldg(f), p1 ? (LDCS ? __ldcs(f + 1) : __ldg(f + 1)) : 0.0);
}

template <int K, int A>
__device__ __forceinline__ void pr_apply(const double (&x)[2][K], double (&y)[2][K]);

// Hermite-like ghost layers kept for the pencil along z at (x, y)
// (ghost_layer_mask of the single-pencil kernel, explicit coordinates)
template <int K, int NLAY>
__device__ __forceinline__ unsigned pr_ghost_mask(const int2 *tf, int x, int y)
{
  constexpr unsigned ALL = (1u << K) - 1u, LOW = (1u << NLAY) - 1u;
  unsigned keep = 0;
#pragma unroll
  for (int phi = 0; phi < 6; ++phi)
    {
      if (tf[phi].x == -2)
        continue;
      const int a = phi / 2, side = phi % 2;
      if (a == 2)
        keep |= side == 0 ? LOW : (LOW << (K - NLAY));
      else
        {
          const int cc = a == 0 ? x : y;
          if (side == 0 ? cc < NLAY : cc >= K - NLAY)
            keep = ALL;
        }
    }
  return keep;
}

// Backward step along A for the pair: v[e] += rf_s w_s + (Dco^T rf_s) rgn_s
template <int K, int A>
__device__ __forceinline__ void pr_face_terms(const double *cell, int c, int w, double (&v)[2][K])
{
#ifdef DGX_EXP_PAIRS_NO_FACE_SMALL
  return;
#endif
  using L = PL<K>;
  using T = TabLayout<K>;
  const double *OUT = cell + L::OFF_OUT + (2 * A) * 2 * L::FP;
  const int fp = 2 * c + L::FK * w;
  double2 w0 = lds2(OUT + fp), w1 = lds2(OUT + L::FP + fp);
  const double2 r0 = lds2(OUT + 2 * L::FP + fp), r1 = lds2(OUT + 3 * L::FP + fp);
  if constexpr (DGX_PAIRS_W1)
    {
      const double *W1 = cell + L::OFF_W1 + (2 * A) * L::FP;
      const double2 u0 = lds2(W1 + fp), u1 = lds2(W1 + L::FP + fp);
      w0.x += u0.x;
      w0.y += u0.y;
      w1.x += u1.x;
      w1.y += u1.y;
    }
#pragma unroll
  for (int m = 0; m < K; ++m)
    {
      const double a0 = tab<double, K>(T::oRf + m), a1 = tab<double, K>(T::oRf + K + m);
      const double b0 = tab<double, K>(T::oRD + m), b1 = tab<double, K>(T::oRD + K + m);
      v[0][m] += a0 * w0.x + a1 * w1.x + b0 * r0.x + b1 * r1.x;
      v[1][m] += a0 * w0.y + a1 * w1.y + b0 * r0.y + b1 * r1.y;
    }
}

// Face entries of axis A from the stash, and which of the two faces is
// shared with the CTA partner (x-rows, BRICK 1; bricks, BRICK 4 / 8); PNB:
// the partner's NB fields.
template <int K, int A>
__device__ __forceinline__ void pr_axis_faces(const double *cell, bool active, int lc, int2 (&tf)[2],
                                              bool (&inr)[2], const double *(&PNB)[2])
{
  using L = PL<K>;
  tf[0] = tf[1] = make_int2(-2, 0);
  if (active)
    {
      const int2 *tfs = reinterpret_cast<const int2 *>(cell + L::OFF_TF);
      tf[0] = tfs[2 * A];
      tf[1] = tfs[2 * A + 1];
    }
  inr[0] = inr[1] = false;
  PNB[0] = PNB[1] = cell + L::OFF_NB;
  if constexpr (L::BRICK == 8 || (L::BRICK == 4 && A < 2))
    {
      const int lp = lc ^ (1 << A);
      const double *pcell = cell + (lp - lc) * L::SM_CELL;
      PNB[0] = PNB[1] = pcell + L::OFF_NB;
      const int pslot = reinterpret_cast<const int *>(pcell + L::OFF_TF)[12];
#pragma unroll
      for (int s = 0; s < 2; ++s)
        inr[s] = tf[s].x >= 0 && tf[s].x == pslot;
    }
  if constexpr (L::BRICK == 1 && A == 0)
    {
#pragma unroll
      for (int s = 0; s < 2; ++s)
        {
          const int lp = lc + (s == 0 ? -1 : 1);
          if (lp >= 0 && lp < L::NC)
            {
              const double *pcell = cell + (lp - lc) * L::SM_CELL;
              PNB[s] = pcell + L::OFF_NB;
              inr[s] = tf[s].x >= 0 && tf[s].x == reinterpret_cast<const int *>(pcell + L::OFF_TF)[12];
            }
        }
    }
}

// The neighbour pencils through the thread's two face points of axis A
// (nodal bases): issued one phase early so that their latency overlaps the
// previous phase (the forward pass's last barrier for axis 0, the test-side
// passes of axis A-1 otherwise).
template <int K, int A>
__device__ __forceinline__ void pr_nb_fetch(const ApplyParams<double> &prm, const double *cell, bool active,
                                            int c, int w, int lc, double (&x)[2][2][K])
{
  int2 tf[2];
  bool inr[2];
  const double *PNB[2];
  pr_axis_faces<K, A>(cell, active, lc, tf, inr, PNB);
#pragma unroll
  for (int s = 0; s < 2; ++s)
    pr_ldg_if<K, A>(tf[s].x >= 0 && !inr[s], prm.u + (long long)DGX_EXP_NBSLOT(tf[s].x >= 0 ? tf[s].x : 0) * PL<K>::NQ,
                    c, w, x[s]);
}

// Both faces of axis A (same algebra as face_axis_v4, sipg_faces.cuh, with
// the pair mapping): own traces, neighbour trace, SIPG flux
// (operators.cpp:977-1003 interior, 1069-1089 boundary), test side.
template <int K, int A, bool COMPRESSED, bool HERM, bool GLN, typename HOOK>
__device__ __forceinline__ void pr_face_axis(const ApplyParams<double> &prm, double *cell, bool active,
                                             int c, int w, int t, int lc, const double (&wf)[2],
                                             const double (&sp)[2], const double (&xnb)[2][2][K],
                                             const double (&trc)[2][2][2], HOOK &&before_wpass)
{
  using L = PL<K>;
  using T = TabLayout<K>;
  constexpr int P = K * K, NQ = L::NQ, FP = L::FP, FK = L::FK, H = L::H, FS = L::FS;
  const double *val = cell;
  const double *G = cell + L::OFF_G;
  double *NB = cell + L::OFF_NB;
  double *DT = cell + L::OFF_DT;
  double *OUT = cell + L::OFF_OUT + (2 * A) * 2 * FP;
  const int fp = 2 * c + FK * w;     // shared face fields
  const int fpg = 2 * c + K * w;     // global face records (unpadded)
  const bool p1 = 2 * c + 1 < K;     // second point of the pair real (odd K: last pair)

  // face entries; faces shared with the CTA partner (its own trace and
  // normal derivative are in its NB slots of the opposite side after the
  // barrier)
  int2 tf[2];
  bool inr[2];
  const double *PNB[2];
  pr_axis_faces<K, A>(cell, active, lc, tf, inr, PNB);
  // own side n.J^{-T} at the two points (issued first: used right after the
  // own traces, as dn_own = n.J^{-T} grad u)
  double jo[2][2][3], dn_own[2][2];
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int b = 0; b < 3; ++b)
          jo[s][e][b] = 0.0;
      if (tf[s].x != -2)
        {
          const int fid = DGX_EXP_FID(tf[s].y & 0x3fffffff);
          const int side = (tf[s].y >> 30) & 1;
          if constexpr (COMPRESSED)
            {
              const double *fg = prm.face_geo + (long long)fid * 7;
#pragma unroll
              for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int b = 0; b < 3; ++b)
                  jo[s][e][b] = __ldg(fg + 1 + side * 3 + b);
            }
          else
            {
              const double *fg = prm.face_geo + (long long)fid * 7 * P + fpg;
#pragma unroll
              for (int b = 0; b < 3; ++b)
                {
                  const double2 o = pr_ldg_pt<K>(fg + (1 + side * 3 + b) * P, p1);
                  jo[s][0][b] = o.x;
                  jo[s][1][b] = o.y;
                }
            }
        }
    }
  // own traces from the collocation fields along the normal (first: their
  // shared-memory loads overlap the arrival of the neighbour pencils)
  double own_u[2][2], own_g[2][2][3];
  {
    double x[2][K];
#if DGX_PAIRS_FWDTRACE
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        {
          own_u[s][e] = trc[s][e][0];
          own_g[s][e][A] = trc[s][e][1];
        }
#else
    (void)trc;
    pr_load<K, A>(val, c, w, x);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      {
        own_u[0][e] = dot_row<double, K, T::oRf>(x[e]);
        own_u[1][e] = dot_row<double, K, T::oRf + K>(x[e]);
      }
#endif
#pragma unroll
    for (int b = 0; b < 3; ++b)
      {
        if (DGX_PAIRS_FWDTRACE && b == A)
          continue;
        pr_load<K, A>(G + b * FS, c, w, x);
#pragma unroll
        for (int e = 0; e < 2; ++e)
          {
            own_g[0][e][b] = dot_row<double, K, T::oRf>(x[e]);
            own_g[1][e][b] = dot_row<double, K, T::oRf + K>(x[e]);
          }
      }
  }
  // neighbour nodal value / normal-derivative layers at the two points
  if constexpr (HERM)
    {
      double xe[2][2], xi[2][2];
#pragma unroll
      for (int s = 0; s < 2; ++s)
        {
#pragma unroll
          for (int e = 0; e < 2; ++e)
            xe[s][e] = xi[s][e] = 0.0;
          if (tf[s].x >= 0 && !inr[s])
            {
              const double *un = prm.u + (long long)tf[s].x * NQ;
              if (s == 0)
                pr_ldg_two<K, A>(un, c, w, K - 2, xi[s], xe[s]);
              else
                pr_ldg_two<K, A>(un, c, w, 0, xe[s], xi[s]);
            }
        }
#pragma unroll
      for (int s = 0; s < 2; ++s)
        {
          const int me = s == 0 ? K - 1 : 0, mi = s == 0 ? K - 2 : 1;
          const int ro = s == 0 ? K : 0;
          double nu[2], nw[2];
#pragma unroll
          for (int e = 0; e < 2; ++e)
            {
              const double ve = xe[s][e] * (sp[e] * hsign<double, K>(me));
              const double vi = xi[s][e] * (sp[e] * hsign<double, K>(mi));
              nu[e] = tab<double, K>(T::oSf + ro + me) * ve + tab<double, K>(T::oSf + ro + mi) * vi;
              nw[e] = tab<double, K>(T::oDf + ro + me) * ve + tab<double, K>(T::oDf + ro + mi) * vi;
            }
          sts2(NB + (2 * s) * FP + fp, nu[0], nu[1]);
          sts2(NB + (2 * s + 1) * FP + fp, nw[0], nw[1]);
        }
    }
  else
    {
      const double(&x)[2][2][K] = xnb; // fetched one phase early (pr_nb_fetch)
      // Gauss-Lobatto nodes: the value rows Sf are exact unit vectors (the
      // end nodes), so the neighbour's face value is its end-node value
      if constexpr (GLN)
        sts2(NB + fp, x[0][0][K - 1], x[0][1][K - 1]);
      else
        sts2(NB + fp, dot_row<double, K, T::oSf + K>(x[0][0]), dot_row<double, K, T::oSf + K>(x[0][1]));
      sts2(NB + FP + fp, dot_row<double, K, T::oDf + K>(x[0][0]), dot_row<double, K, T::oDf + K>(x[0][1]));
      if constexpr (GLN)
        sts2(NB + 2 * FP + fp, x[1][0][0], x[1][1][0]);
      else
        sts2(NB + 2 * FP + fp, dot_row<double, K, T::oSf>(x[1][0]), dot_row<double, K, T::oSf>(x[1][1]));
      sts2(NB + 3 * FP + fp, dot_row<double, K, T::oDf>(x[1][0]), dot_row<double, K, T::oDf>(x[1][1]));
    }
  // the own gradient trace is only needed projected on n.J^{-T} (dn_own),
  // which frees its registers early
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
#pragma unroll
      for (int e = 0; e < 2; ++e)
        dn_own[s][e] = own_g[s][e][0] * jo[s][e][0] + own_g[s][e][1] * jo[s][e][1] +
                       own_g[s][e][2] * jo[s][e][2];
      if (inr[s])
        {
          // n^- . J^{-T} grad u on this side: the partner's neighbour term
          sts2(NB + (2 * s) * FP + fp, own_u[s][0], own_u[s][1]);
          sts2(NB + (2 * s + 1) * FP + fp, dn_own[s][0], dn_own[s][1]);
        }
    }
  DGX_EXP_FSYNC();

  // pass 1, along t1 (column pairs): nu -> (S nu, D nu -> DT[2+s]); nw -> S nw
  for (int tk = t; tk < 4 * H; tk += L::G)
    {
      const int a = tk / 4, f = tk - a * 4; // field fastest (conflict-free)
      if ((f < 2) ? inr[0] : inr[1])
        continue;
      double *fld = NB + f * FP + 2 * a;
      double x[2][K], y[2][K];
#pragma unroll
      for (int m = 0; m < K; ++m)
        {
          const double2 v = lds2(fld + FK * m);
          x[0][m] = v.x;
          x[1][m] = v.y;
        }
#pragma unroll
      for (int e = 0; e < 2; ++e)
        apply_S<double, K>(x[e], y[e]);
#pragma unroll
      for (int m = 0; m < K; ++m)
        sts2(fld + FK * m, y[0][m], y[1][m]);
      if ((f & 1) == 0)
        {
#pragma unroll
          for (int e = 0; e < 2; ++e)
            apply_Dn<double, K>(x[e], y[e]);
          double *dt = DT + (2 + f / 2) * FP + 2 * a;
#pragma unroll
          for (int m = 0; m < K; ++m)
            sts2(dt + FK * m, y[0][m], y[1][m]);
        }
    }
  DGX_EXP_FSYNC();
  // rest of the face geometry (L2-resident: prefetched at task start;
  // issued here so that pass 2 overlaps the latency)
  double jxw[2][2], tau[2], jb[2][2][3];
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      tau[s] = 0.0;
#pragma unroll
      for (int e = 0; e < 2; ++e)
        {
          jxw[s][e] = 0.0;
#pragma unroll
          for (int b = 0; b < 3; ++b)
            jb[s][e][b] = 0.0;
        }
      if (tf[s].x != -2)
        {
          const int fid = DGX_EXP_FID(tf[s].y & 0x3fffffff);
          const int side = (tf[s].y >> 30) & 1;
          if constexpr (COMPRESSED)
            {
              const double *fg = prm.face_geo + (long long)fid * 7;
              const double j0 = __ldg(fg);
#pragma unroll
              for (int e = 0; e < 2; ++e)
                {
                  jxw[s][e] = j0 * wf[e];
#pragma unroll
                  for (int b = 0; b < 3; ++b)
                    jb[s][e][b] = __ldg(fg + 1 + (1 - side) * 3 + b);
                }
            }
          else
            {
              const double *fg = prm.face_geo + (long long)fid * 7 * P + fpg;
              const double2 j2 = pr_ldg_pt<K>(fg, p1);
              jxw[s][0] = j2.x;
              jxw[s][1] = j2.y;
#pragma unroll
              for (int b = 0; b < 3; ++b)
                {
                  const double2 n = !inr[s] ? pr_ldg_pt<K>(fg + (1 + (1 - side) * 3 + b) * P, p1)
                                            : make_double2(0.0, 0.0);
                  jb[s][0][b] = n.x;
                  jb[s][1][b] = n.y;
                }
            }
          tau[s] = __ldg(prm.penalty + fid);
        }
    }
#if !DGX_PAIRS_ROWDOT
  // pass 2, along t0 (rows): nu -> (S nu, D nu -> DT[s]); nw, dt1 -> S
  for (int tk = t; tk < 6 * K; tk += L::G)
    {
      const int f = tk / K, r = tk - f * K;
      if ((f < 2 || f == 4) ? inr[0] : inr[1])
        continue;
      double *fld = (f < 4 ? NB + f * FP : DT + (2 + (f - 4)) * FP) + FK * r;
      double x[K], y[K];
#pragma unroll
      for (int j = 0; j < H; ++j)
        {
          const double2 v = lds2(fld + 2 * j);
          x[2 * j] = v.x;
          if (2 * j + 1 < K)
            x[2 * j + 1] = v.y;
        }
      apply_S<double, K>(x, y);
#pragma unroll
      for (int j = 0; j < H; ++j)
        sts2(fld + 2 * j, y[2 * j], 2 * j + 1 < K ? y[2 * j + 1] : 0.0);
      if (f < 4 && (f & 1) == 0)
        {
          apply_Dn<double, K>(x, y);
          double *dt = DT + (f / 2) * FP + FK * r;
#pragma unroll
          for (int j = 0; j < H; ++j)
            sts2(dt + 2 * j, y[2 * j], 2 * j + 1 < K ? y[2 * j + 1] : 0.0);
        }
    }
  DGX_EXP_FSYNC();
#endif

  // flux at the two face points of both faces
#pragma unroll
  for (int s = 0; s < 2; ++s)
    {
      double rv[2] = {0.0, 0.0}, g[2] = {0.0, 0.0};
      if (tf[s].x != -2)
        {
          const int side = (tf[s].y >> 30) & 1;
          if (tf[s].x == -1)
            {
#pragma unroll
              for (int e = 0; e < 2; ++e)
                {
                  rv[e] = (own_u[s][e] * tau[s] * 2.0 - dn_own[s][e]) * jxw[s][e];
                  g[e] = -(own_u[s][e] * jxw[s][e]);
                }
            }
          else if (inr[s])
            {
              const double2 nu = lds2(PNB[s] + (2 * (1 - s)) * FP + fp);
              const double2 dn = lds2(PNB[s] + (2 * (1 - s) + 1) * FP + fp);
              const double nuv[2] = {nu.x, nu.y}, dnv[2] = {dn.x, dn.y};
              const double sgn = side == 0 ? 1.0 : -1.0;
#pragma unroll
              for (int e = 0; e < 2; ++e)
                {
                  const double delta = own_u[s][e] - nuv[e];
                  rv[e] = (delta * tau[s] - sgn * ((dn_own[s][e] + dnv[e]) * 0.5)) * jxw[s][e];
                  g[e] = -(sgn * delta * jxw[s][e] * 0.5);
                }
            }
          else
            {
#if DGX_PAIRS_ROWDOT
              // rows w of the t1-interpolated fields (value, normal derivative,
              // t1-derivative), contracted along t0 at the two points:
              // u+ = S nu, d/dt0 u+ = D nu, nw+ = S nw, d/dt1 u+ = S dt1
              double rnu[K], rnw[K], rd1[K];
              {
                const double *r0 = NB + (2 * s) * FP + FK * w, *r1 = NB + (2 * s + 1) * FP + FK * w;
                const double *r2 = DT + (2 + s) * FP + FK * w;
#pragma unroll
                for (int j = 0; j < H; ++j)
                  {
                    const double2 a0 = lds2(r0 + 2 * j), a1 = lds2(r1 + 2 * j), a2 = lds2(r2 + 2 * j);
                    rnu[2 * j] = a0.x;
                    rnw[2 * j] = a1.x;
                    rd1[2 * j] = a2.x;
                    if (2 * j + 1 < K)
                      {
                        rnu[2 * j + 1] = a0.y;
                        rnw[2 * j + 1] = a1.y;
                        rd1[2 * j + 1] = a2.y;
                      }
                  }
              }
              double nuv[2], nwv[2], dt0[2], dt1[2];
#pragma unroll
              for (int e = 0; e < 2; ++e)
                {
                  const int qr = (2 * c + e < K ? 2 * c + e : K - 1) * K;
                  double a = 0.0, b = 0.0, cc = 0.0, dd = 0.0;
#pragma unroll
                  for (int j = 0; j < K; ++j)
                    {
                      const double sj = tab<double, K>(T::oS + qr + j), dj = tab<double, K>(T::oDn + qr + j);
                      a += sj * rnu[j];
                      b += dj * rnu[j];
                      cc += sj * rnw[j];
                      dd += sj * rd1[j];
                    }
                  nuv[e] = a;
                  dt0[e] = b;
                  nwv[e] = cc;
                  dt1[e] = dd;
                }
#else
              const double2 nu = lds2(NB + (2 * s) * FP + fp), nw = lds2(NB + (2 * s + 1) * FP + fp);
              const double2 d0 = lds2(DT + s * FP + fp), d1 = lds2(DT + (2 + s) * FP + fp);
              const double nuv[2] = {nu.x, nu.y}, nwv[2] = {nw.x, nw.y};
              const double dt0[2] = {d0.x, d0.y}, dt1[2] = {d1.x, d1.y};
#endif
              const double sgn = side == 0 ? 1.0 : -1.0;
#pragma unroll
              for (int e = 0; e < 2; ++e)
                {
                  double dn_nb = 0.0;
#pragma unroll
                  for (int b = 0; b < 3; ++b)
                    {
                      const double gb = b == A ? nwv[e] : ((b < A ? b : b - 1) == 0 ? dt0[e] : dt1[e]);
                      dn_nb += gb * jb[s][e][b];
                    }
                  const double delta = own_u[s][e] - nuv[e];
                  rv[e] = (delta * tau[s] - sgn * ((dn_own[s][e] + dn_nb) * 0.5)) * jxw[s][e];
                  g[e] = -(sgn * delta * jxw[s][e] * 0.5);
                }
            }
        }
      sts2(OUT + s * FP + fp, rv[0], rv[1]);
      sts2(OUT + (2 + s) * FP + fp, g[0] * jo[s][0][A], g[1] * jo[s][1][A]);
      // rg along t0 -> DT[s]; along t1 -> DT[2 + s] (row-dot: RG1[s], since
      // DT[2 + s] rows are still being read by the other threads of the row)
      sts2(DT + s * FP + fp, g[0] * jo[s][0][A == 0 ? 1 : 0], g[1] * jo[s][1][A == 0 ? 1 : 0]);
      sts2((DGX_PAIRS_ROWDOT ? cell + L::OFF_RG1 + s * FP : DT + (2 + s) * FP) + fp,
           g[0] * jo[s][0][A == 2 ? 1 : 2], g[1] * jo[s][1][A == 2 ? 1 : 2]);
    }
  DGX_EXP_FSYNC();
  before_wpass();
  // w = rv + Dco_t0^T rg_t0 (rows) ... [W1: and the column tasks below in
  // the same phase, into W1]
  for (int tk = t; tk < 2 * K + (DGX_PAIRS_W1 ? 2 * H : 0); tk += L::G)
    {
      if (DGX_PAIRS_W1 && tk >= 2 * K)
        {
          const int tc = tk - 2 * K;
          const int s = tc / H, a2 = tc - s * H;
          double *xo = cell + L::OFF_W1 + (2 * A + s) * FP + 2 * a2;
          const double *yo = DT + (2 + s) * FP + 2 * a2;
          double y[2][K], b[2][K];
#pragma unroll
          for (int m = 0; m < K; ++m)
            {
              const double2 u = lds2(yo + FK * m);
              y[0][m] = u.x;
              y[1][m] = u.y;
            }
#pragma unroll
          for (int e = 0; e < 2; ++e)
            apply_Dt<double, K>(y[e], b[e]);
#pragma unroll
          for (int m = 0; m < K; ++m)
            sts2(xo + FK * m, b[0][m], b[1][m]);
          continue;
        }
      const int s = tk / K, r = tk - s * K;
      double *xo = OUT + s * FP + FK * r;
      const double *yo = DT + s * FP + FK * r;
      double a[K], b[K], y[K];
#pragma unroll
      for (int j = 0; j < H; ++j)
        {
          const double2 v = lds2(xo + 2 * j), u = lds2(yo + 2 * j);
          a[2 * j] = v.x;
          y[2 * j] = u.x;
          if (2 * j + 1 < K)
            {
              a[2 * j + 1] = v.y;
              y[2 * j + 1] = u.y;
            }
        }
      apply_Dt<double, K>(y, b);
#pragma unroll
      for (int j = 0; j < H; ++j)
        sts2(xo + 2 * j, a[2 * j] + b[2 * j], 2 * j + 1 < K ? a[2 * j + 1] + b[2 * j + 1] : 0.0);
    }
  if constexpr (DGX_PAIRS_W1)
    return; // no trailing barrier (below)
  pr_sync<K>();
  // ... + Dco_t1^T rg_t1 (column pairs)
  for (int tk = t; tk < 2 * H; tk += L::G)
    {
      const int s = tk / H, a2 = tk - s * H;
      double *xo = OUT + s * FP + 2 * a2;
      const double *yo = (DGX_PAIRS_ROWDOT ? cell + L::OFF_RG1 + s * FP : DT + (2 + s) * FP) + 2 * a2;
      double a[2][K], y[2][K], b[2][K];
#pragma unroll
      for (int m = 0; m < K; ++m)
        {
          const double2 v = lds2(xo + FK * m), u = lds2(yo + FK * m);
          a[0][m] = v.x;
          a[1][m] = v.y;
          y[0][m] = u.x;
          y[1][m] = u.y;
        }
#pragma unroll
      for (int e = 0; e < 2; ++e)
        apply_Dt<double, K>(y[e], b[e]);
#pragma unroll
      for (int m = 0; m < K; ++m)
        sts2(xo + FK * m, a[0][m] + b[0][m], a[1][m] + b[1][m]);
    }
  // no trailing barrier (as face_axis_v4): the next axis touches NB first
  // after reading val/G, and its own barriers order the rest; DT/OUT reuse
  // by the next axis happens after its first barrier
}

template <int K, bool COMPRESSED, int BASIS>
__global__ void __launch_bounds__(PL<K>::THREADS, PL<K>::MINB)
  sipg_pairs_kernel(const ApplyParams<double> prm)
{
  constexpr bool HERM = BASIS == 2;
  using L = PL<K>;
  using T = TabLayout<K>;
  constexpr int H = L::H, P2 = L::P2, NQ = L::NQ, FS = L::FS, S2 = L::S2, NC = L::NC;
  constexpr int P = K * K;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *smem = reinterpret_cast<double *>(smem_raw);

  constexpr int GS = L::G;
  const int lc = threadIdx.x / GS;
  const int t = threadIdx.x - lc * GS;   // lane in the cell's group
  const int tp = t < P2 ? t : P2 - 1;   // pencil pair (padding lanes duplicate the last)
  const int c = tp % H, w = tp / H;
  // x-pass pairs: for K = 6 a permutation of the pairs that makes the
  // quarter-warps conflict-free for the contiguous x-pencils (quad
  // 3 (2c + w) = 3 (t + 4) mod 8); natural order otherwise
  int cx = c, wx = w;
  if constexpr (K == 6)
    {
      const unsigned long long tb = tp < 12 ? 0x5a14749860835ecull : 0xa22062eull;
      const int px = (int)((tb >> (5 * (tp < 12 ? tp : tp - 12))) & 31u);
      cx = px % H;
      wx = px / H;
    }
  const int task = blockIdx.x * NC + lc;
  const bool active = task < prm.n_tasks;
  double *cell = smem + lc * L::SM_CELL;
  double *val = cell;
  double *G = cell + L::OFF_G;

  const int slot = active ? prm.task_slot[task] : 0;
  const int geo = active ? prm.task_geo[task] : -1;
  if (!active && t == 0)
    reinterpret_cast<int *>(cell + L::OFF_TF)[12] = -3; // no brick partner here

  // task metadata of the CTAs one and two generations ahead (prm.ahead =
  // tasks resident on the device): the first link of their prologue's
  // dependent-load chain becomes an L2 hit
  if (!DGX_EXP_NO_META_PF && threadIdx.x < 6 && prm.ahead > 0)
    {
      const long long t2 = (long long)(blockIdx.x * NC) + (long long)prm.ahead * (1 + threadIdx.x % 2);
      if (t2 < prm.n_tasks)
        {
          const int which = threadIdx.x / 2;
          const char *a = which == 0 ? reinterpret_cast<const char *>(prm.task_slot + t2)
                        : which == 1 ? reinterpret_cast<const char *>(prm.task_geo + t2)
                                     : reinterpret_cast<const char *>(prm.task_face + t2 * 6);
          asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
          if (which == 2)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a + 128));
        }
    }

  // L2 prefetch of the cell record (measured essential: 20.5 -> 22.5 ms
  // without), face entries stashed in shared memory
  if (active)
    {
      constexpr int LINE = 128;
      const int ncg = prm.sym ? 6 : 10;
      if (geo >= 0 && !DGX_EXP_NO_CELL_PF)
        {
          const char *gp = reinterpret_cast<const char *>(
            prm.cell_geo + (long long)geo * ncg * (COMPRESSED ? 1 : NQ));
          const int bytes = ncg * (COMPRESSED ? 1 : NQ) * 8;
          for (int off = t * LINE; off < bytes; off += GS * LINE)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(gp + off));
        }
      for (int i = t; i < 6; i += GS)
        reinterpret_cast<int2 *>(cell + L::OFF_TF)[i] = prm.task_face[task * 6 + i];
      if (t == 0)
        reinterpret_cast<int *>(cell + L::OFF_TF)[12] = slot;
      // (no L2 prefetch of the face records: measured 20.72 -> 20.55 ms
      // without it once the neighbour pencils are fetched one phase early)
    }

  // face points of axis 0 (FWDTRACE: the permuted x-pass pair)
  const int c0 = DGX_PAIRS_FWDTRACE ? cx : c, w0 = DGX_PAIRS_FWDTRACE ? wx : w;
  // own traces per axis, [A][face s][pencil e][value, normal gradient]
  double tr[3][2][2][2];
  (void)tr;
  // Hermite-like: sign of the tangential indices of the two face points /
  // z-pencils (x = 2c + e, y = w), and the ghost layers of a ghost-side task
  double sp0[2] = {1.0, 1.0};
  if constexpr (HERM)
#pragma unroll
    for (int e = 0; e < 2; ++e)
      sp0[e] = hsign<double, K>(2 * c0 + e) * hsign<double, K>(w0);
  double sp[2] = {1.0, 1.0};
  unsigned gmask[2] = {(1u << K) - 1u, (1u << K) - 1u};
  if constexpr (HERM)
    {
#pragma unroll
      for (int e = 0; e < 2; ++e)
        sp[e] = hsign<double, K>(2 * c + e) * hsign<double, K>(w);
      if (active && slot >= prm.n_owned)
        {
          int2 tf[6];
#pragma unroll
          for (int phi = 0; phi < 6; ++phi)
            tf[phi] = prm.task_face[task * 6 + phi];
#pragma unroll
          for (int e = 0; e < 2; ++e)
            gmask[e] = pr_ghost_mask<K, 2>(tf, 2 * c + e, w);
        }
    }

  // neighbour pencils of the first face axis: issued with the cell's own u
  // (the stashed face entries are visible after the forward's first barrier,
  // so the fetch happens right after it), in flight across the forward pass
  double xnb[2][2][K];
  // ---- forward: val = (S x S x S) u, G_b = Dco_b val ----------------------
  {
    double x[2][K], z[2][K];
    const double *uc = prm.u + (long long)slot * NQ;
    if (active)
      pr_ldg<K, 2>(uc, c, w, x);
    else
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int m = 0; m < K; ++m)
          x[e][m] = 0.0;
    if constexpr (HERM)
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int m = 0; m < K; ++m)
          x[e][m] = ((gmask[e] >> m) & 1u) ? x[e][m] * (sp[e] * hsign<double, K>(m)) : 0.0;
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_S<double, K>(x[e], z[e]);
    pr_store<K, 2>(val, c, w, z);
    pr_sync<K>();
#ifndef DGX_EXP_PAIRS_NO_FACE
    if constexpr (!HERM)
      pr_nb_fetch<K, 0>(prm, cell, active, c0, w0, lc, xnb);
#endif
    pr_load<K, 0>(val, cx, wx, x);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_S<double, K>(x[e], z[e]);
    pr_store<K, 0>(val, cx, wx, z);
    pr_sync<K>();
    // own value / normal-gradient traces of axis A from the pencils along A
    // held here (val in v, G_A in g): rf rows (operators.cpp:794-858 own side)
    auto traces = [&](int a, const double(&v)[2][K], const double(&g)[2][K]) {
#pragma unroll
      for (int e = 0; e < 2; ++e)
        {
          tr[a][0][e][0] = dot_row<double, K, T::oRf>(v[e]);
          tr[a][1][e][0] = dot_row<double, K, T::oRf + K>(v[e]);
          tr[a][0][e][1] = dot_row<double, K, T::oRf>(g[e]);
          tr[a][1][e][1] = dot_row<double, K, T::oRf + K>(g[e]);
        }
    };
    (void)traces;
    pr_load<K, 1>(val, c, w, x);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_S<double, K>(x[e], z[e]);
    pr_store<K, 1>(val, c, w, z);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_D<double, K>(z[e], x[e]);
    pr_store<K, 1>(G + FS, c, w, x);
    if constexpr (DGX_PAIRS_FWDTRACE)
      traces(1, z, x);
    pr_sync<K>();
    pr_load<K, 0>(val, cx, wx, x);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_D<double, K>(x[e], z[e]);
    pr_store<K, 0>(G, cx, wx, z);
    if constexpr (DGX_PAIRS_FWDTRACE)
      traces(0, x, z);
    pr_load<K, 2>(val, c, w, x);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_D<double, K>(x[e], z[e]);
    pr_store<K, 2>(G + 2 * FS, c, w, z);
    if constexpr (DGX_PAIRS_FWDTRACE)
      traces(2, x, z);
  }
  pr_sync<K>();

  // cell record of the quadrature-point operation: its first point layers
  // are loaded before the last face axis's test-side passes, so their latency
  // overlaps face work
  const bool sym = prm.sym != 0;
  const int ncg = sym ? 6 : 10;
  const double *cgb = prm.cell_geo + (long long)(geo >= 0 ? geo : 0) * ncg * (COMPRESSED ? 1 : NQ);
#ifndef DGX_PAIRS_QDEPTH
#define DGX_PAIRS_QDEPTH 2
#endif
  constexpr int QD = DGX_PAIRS_QDEPTH; // layers in flight
  double2 gn[QD][10];
  auto load_layer = [&](int m) {
    if constexpr (!COMPRESSED)
      {
        const double *cg = cgb + 2 * c + K * w + K * K * m;
#pragma unroll
        for (int i = 0; i < 10; ++i)
          gn[m % QD][i] = (geo >= 0 && i < ncg) ? pr_ldg_pt<K, true>(cg + i * NQ, 2 * c + 1 < K)
                                                : make_double2(0.0, 0.0);
      }
  };

  // ---- faces ------------------------------------------------------------
  {
    // tangential weight prod_t w[q_t] of the two face points (compressed)
    double wf[2] = {1.0, 1.0}, wf0[2] = {1.0, 1.0};
    if constexpr (COMPRESSED)
      {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          {
            const int q0 = 2 * c + e, q00 = 2 * c0 + e;
            double wa = 0.0, wb = 0.0, wa0 = 0.0, wb0 = 0.0;
#pragma unroll
            for (int i = 0; i < K; ++i)
              {
                wa = (q0 == i) ? tab<double, K>(T::oW + i) : wa;
                wb = (w == i) ? tab<double, K>(T::oW + i) : wb;
                wa0 = (q00 == i) ? tab<double, K>(T::oW + i) : wa0;
                wb0 = (w0 == i) ? tab<double, K>(T::oW + i) : wb0;
              }
            wf[e] = (1.0 * wa) * wb;
            wf0[e] = (1.0 * wa0) * wb0;
          }
      }
    auto none = [] {};
#ifdef DGX_EXP_PAIRS_NO_FACE // ablation: cell integral only
#ifndef DGX_EXP_PAIRS_NO_FACE_SMALL
    for (int i = t; i < 12 * L::FP; i += L::G)
      cell[L::OFF_OUT + i] = 0.0;
#endif
    pr_sync<K>();
    (void)none;
    (void)wf;
    (void)xnb;
    if (false)
#endif
    {
    pr_face_axis<K, 0, COMPRESSED, HERM, BASIS == 0>(prm, cell, active, c0, w0, t, lc, wf0, sp0, xnb, tr[0], [&] {
      if constexpr (!HERM)
        pr_nb_fetch<K, 1>(prm, cell, active, c, w, lc, xnb);
    });
    pr_face_axis<K, 1, COMPRESSED, HERM, BASIS == 0>(prm, cell, active, c, w, t, lc, wf, sp, xnb, tr[1], [&] {
      if constexpr (!HERM)
        pr_nb_fetch<K, 2>(prm, cell, active, c, w, lc, xnb);
    });
    pr_face_axis<K, 2, COMPRESSED, HERM, BASIS == 0>(prm, cell, active, c, w, t, lc, wf, sp, xnb, tr[2], [&] {
#pragma unroll
      for (int m = 0; m < QD - 1; ++m)
        load_layer(m);
    });
    }
#ifdef DGX_EXP_PAIRS_NO_FACE
#pragma unroll
    for (int m = 0; m < QD - 1; ++m)
      load_layer(m);
#endif
  }

  // ---- quadrature-point operation (operators.cpp:669-733), z-pencil pairs;
  //      the cell record of point layer m+1 is loaded while layer m computes
  {
    double wxy[2] = {1.0, 1.0};
    if constexpr (COMPRESSED)
      {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          {
            const int q0 = 2 * c + e;
            double wa = 0.0, wb = 0.0;
#pragma unroll
            for (int i = 0; i < K; ++i)
              {
                wa = (q0 == i) ? tab<double, K>(T::oW + i) : wa;
                wb = (w == i) ? tab<double, K>(T::oW + i) : wb;
              }
            wxy[e] = (1.0 * wa) * wb;
          }
      }
#ifndef DGX_PAIRS_FUSEQ
#define DGX_PAIRS_FUSEQ 1
#endif
    // t_2 of the thread's own z-pencil pair stays in registers: the first
    // backward pass (along z, same pencils) follows without a barrier
    double t2r[2][K];
#pragma unroll
    for (int m = 0; m < K; ++m)
      {
        const int q = 2 * c + L::KP * w + S2 * m; // shared
        if (m + QD - 1 < K)
          load_layer(m + QD - 1);
        double2 gc[10];
#pragma unroll
        for (int i = 0; i < 10; ++i)
          gc[i] = gn[m % QD][i];
        double gg[3][2], tt[3][2];
#pragma unroll
        for (int b = 0; b < 3; ++b)
          {
            const double2 v = lds2(G + b * FS + q);
            gg[b][0] = v.x;
            gg[b][1] = v.y;
          }
        if (geo >= 0 && sym)
          {
            double cf[6][2];
            if constexpr (COMPRESSED)
              {
#pragma unroll
                for (int e = 0; e < 2; ++e)
                  {
                    const double wq = wxy[e] * tab<double, K>(T::oW + m);
#pragma unroll
                    for (int i = 0; i < 6; ++i)
                      cf[i][e] = __ldg(cgb + i) * wq;
                  }
              }
            else
              {
#pragma unroll
                for (int i = 0; i < 6; ++i)
                  {
                    cf[i][0] = gc[i].x;
                    cf[i][1] = gc[i].y;
                  }
              }
#pragma unroll
            for (int e = 0; e < 2; ++e)
              {
                tt[0][e] = cf[0][e] * gg[0][e] + cf[3][e] * gg[1][e] + cf[4][e] * gg[2][e];
                tt[1][e] = cf[3][e] * gg[0][e] + cf[1][e] * gg[1][e] + cf[5][e] * gg[2][e];
                tt[2][e] = cf[4][e] * gg[0][e] + cf[5][e] * gg[1][e] + cf[2][e] * gg[2][e];
              }
          }
        else if (geo >= 0)
          {
            double jit[9][2], jw[2];
            if constexpr (COMPRESSED)
              {
#pragma unroll
                for (int e = 0; e < 2; ++e)
                  {
#pragma unroll
                    for (int i = 0; i < 9; ++i)
                      jit[i][e] = __ldg(cgb + i);
                    jw[e] = __ldg(cgb + 9) * (wxy[e] * tab<double, K>(T::oW + m));
                  }
              }
            else
              {
#pragma unroll
                for (int i = 0; i < 9; ++i)
                  {
                    jit[i][0] = gc[i].x;
                    jit[i][1] = gc[i].y;
                  }
                jw[0] = gc[9].x;
                jw[1] = gc[9].y;
              }
#pragma unroll
            for (int e = 0; e < 2; ++e)
              {
                double ph[3];
#pragma unroll
                for (int i = 0; i < 3; ++i)
                  ph[i] = jit[i * 3][e] * gg[0][e] + jit[i * 3 + 1][e] * gg[1][e] +
                          jit[i * 3 + 2][e] * gg[2][e];
#pragma unroll
                for (int i = 0; i < 3; ++i)
                  tt[i][e] = (jit[i][e] * ph[0] + jit[3 + i][e] * ph[1] + jit[6 + i][e] * ph[2]) * jw[e];
              }
          }
        else
          {
#pragma unroll
            for (int b = 0; b < 3; ++b)
              tt[b][0] = tt[b][1] = 0.0;
          }
#pragma unroll
        for (int b = 0; b < (DGX_PAIRS_FUSEQ ? 2 : 3); ++b)
          sts2(G + b * FS + q, tt[b][0], tt[b][1]);
        t2r[0][m] = tt[2][0];
        t2r[1][m] = tt[2][1];
      }
#if DGX_PAIRS_FUSEQ
    // ---- backward, first pass (z): v = Dco_z^T t_2 + z-face terms
    double v[2][K];
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_Dt<double, K>(t2r[e], v[e]);
    pr_face_terms<K, 2>(cell, c, w, v);
    pr_store<K, 2>(val, c, w, v);
#endif
  }
  pr_sync<K>();

  // ---- backward: y = (S^T x S^T x S^T)(sum_b Dco_b^T t_b + face terms) ----
  {
    double x[2][K], z[2][K], v[2][K];
#if !DGX_PAIRS_FUSEQ
    pr_load<K, 2>(G + 2 * FS, c, w, x);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_Dt<double, K>(x[e], v[e]);
    pr_face_terms<K, 2>(cell, c, w, v);
    pr_store<K, 2>(val, c, w, v);
    pr_sync<K>();
#endif
    pr_load<K, 1>(G + FS, c, w, x);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_Dt<double, K>(x[e], z[e]);
    pr_load<K, 1>(val, c, w, v);
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int m = 0; m < K; ++m)
        v[e][m] += z[e][m];
    pr_face_terms<K, 1>(cell, c, w, v);
    pr_store<K, 1>(val, c, w, v);
    pr_sync<K>();
    pr_load<K, 0>(G, cx, wx, x);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_Dt<double, K>(x[e], z[e]);
    pr_load<K, 0>(val, cx, wx, v);
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int m = 0; m < K; ++m)
        v[e][m] += z[e][m];
    pr_face_terms<K, 0>(cell, cx, wx, v);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_St<double, K>(v[e], z[e]);
    pr_store<K, 0>(val, cx, wx, z);
    pr_sync<K>();
    pr_load<K, 1>(val, c, w, x);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_St<double, K>(x[e], z[e]);
    pr_store<K, 1>(val, c, w, z);
    pr_sync<K>();
    pr_load<K, 2>(val, c, w, x);
#pragma unroll
    for (int e = 0; e < 2; ++e)
      apply_St<double, K>(x[e], z[e]);
    if (active && t < P2)
      {
        double *yc = prm.y + (long long)slot * NQ;
#pragma unroll
        for (int m = 0; m < K; ++m)
          {
            double a = z[0][m], b = z[1][m];
            if constexpr (HERM)
              {
                a = ((gmask[0] >> m) & 1u) ? a * (sp[0] * hsign<double, K>(m)) : 0.0;
                b = ((gmask[1] >> m) & 1u) ? b * (sp[1] * hsign<double, K>(m)) : 0.0;
              }
            if constexpr (L::ODD)
              {
                yc[pr_gl<K, 2>(c, w, 0, m)] = a;
                if (2 * c + 1 < K)
                  yc[pr_gl<K, 2>(c, w, 1, m)] = b;
              }
            else
              // streaming store: y is not read again, keep L2 for u and the
              // face records (measured 20.82 -> 20.72 ms on C4)
              __stcs(reinterpret_cast<double2 *>(yc + pr_gl<K, 2>(c, w, 0, m)), make_double2(a, b));
          }
      }
  }
}

} // namespace dev
} // namespace dgx

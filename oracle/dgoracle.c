/* CPU restatement of the reference SIPG-Laplacian apply path.
 * TEST INFRASTRUCTURE ONLY -- see dgoracle.h. Compiled with
 * -ffp-contract=off like the reference (CMakeLists.txt:33-39) so that the
 * setup routines (quadrature, shape matrices, geometry) reproduce the
 * reference bit for bit; the apply itself is an independent table-based
 * (non sum-factorized) evaluation of the same weak form. */
#include "dgoracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static char g_err[256];
static int fail(const char *msg)
{
  snprintf(g_err, sizeof g_err, "%s", msg);
  return -1;
}
const char *dgo_last_error(void) { return g_err; }

static int64_t ipow64(int b, int e)
{
  int64_t r = 1;
  while (e-- > 0)
    r *= b;
  return r;
}

/* ---------------------------------------------------------------- RNG --- */
/* std::mt19937 (MT19937, 32 bit) and libstdc++'s generate_canonical<double,
 * 53> with two 32-bit draws, then a + (b - a) r (tests/test_helpers.hpp). */
typedef struct
{
  uint32_t mt[624];
  int idx;
} mt19937_t;

static void mt_seed(mt19937_t *g, uint32_t s)
{
  g->mt[0] = s;
  for (int i = 1; i < 624; ++i)
    g->mt[i] = 1812433253u * (g->mt[i - 1] ^ (g->mt[i - 1] >> 30)) + (uint32_t)i;
  g->idx = 624;
}

static uint32_t mt_next(mt19937_t *g)
{
  if (g->idx >= 624)
    {
      for (int i = 0; i < 624; ++i)
        {
          uint32_t y = (g->mt[i] & 0x80000000u) | (g->mt[(i + 1) % 624] & 0x7fffffffu);
          g->mt[i] = g->mt[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
      g->idx = 0;
    }
  uint32_t y = g->mt[g->idx++];
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}

int dgo_random_vector(int64_t n, uint32_t seed, double *out)
{
  mt19937_t g;
  mt_seed(&g, seed);
  for (int64_t i = 0; i < n; ++i)
    {
      double sum = 0.0, tmp = 1.0;
      for (int k = 0; k < 2; ++k)
        {
          sum += (double)mt_next(&g) * tmp;
          tmp *= 4294967296.0;
        }
      double r = sum / tmp;
      if (r >= 1.0)
        r = nextafter(1.0, 0.0);
      out[i] = r * 2.0 + (-1.0);
    }
  return 0;
}

/* --------------------------------------------------------- quadrature --- */
/* quadrature.cpp:15-35 */
static void legendre(int n, double x, double *p, double *dp)
{
  double p0 = 1.0, p1 = x;
  if (n == 0)
    {
      *p = 1.0;
      *dp = 0.0;
      return;
    }
  for (int m = 2; m <= n; ++m)
    {
      const double p2 = ((2 * m - 1) * x * p1 - (m - 1) * p0) / m;
      p0 = p1;
      p1 = p2;
    }
  *p = p1;
  if (fabs(x) == 1.0)
    *dp = (n % 2 == 0 ? x : 1.0) * n * (n + 1) / 2.0;
  else
    *dp = n * (x * p1 - p0) / (x * x - 1.0);
}

/* quadrature.cpp:38-53 */
static void symmetrize(int n, double *pts, double *w)
{
  for (int i = 0; i < n / 2; ++i)
    {
      const int j = n - 1 - i;
      const double p = 0.5 * (pts[i] + (1.0 - pts[j]));
      pts[i] = p;
      pts[j] = 1.0 - p;
      const double ww = 0.5 * (w[i] + w[j]);
      w[i] = ww;
      w[j] = ww;
    }
  if (n % 2 == 1)
    pts[n / 2] = 0.5;
}

/* quadrature.cpp:56-127 */
int dgo_gauss(int n, int lobatto, double *pts, double *w)
{
  if (!lobatto)
    {
      if (n < 1)
        return fail("gauss: need at least one point");
      for (int i = 0; i < n; ++i)
        {
          double x = cos(M_PI * (i + 0.75) / (n + 0.5));
          double p = 0, dp = 1;
          for (int it = 0; it < 100; ++it)
            {
              legendre(n, x, &p, &dp);
              const double dx = p / dp;
              x -= dx;
              if (fabs(dx) < 1e-15)
                break;
            }
          legendre(n, x, &p, &dp);
          pts[n - 1 - i] = 0.5 * (x + 1.0);
          w[n - 1 - i] = 1.0 / ((1.0 - x * x) * dp * dp);
        }
    }
  else
    {
      if (n < 2)
        return fail("gauss_lobatto: need at least two points");
      const int m = n - 1;
      for (int i = 0; i < n; ++i)
        {
          double x;
          if (i == 0)
            x = -1.0;
          else if (i == m)
            x = 1.0;
          else
            {
              x = cos(M_PI * (m - i) / m);
              for (int it = 0; it < 100; ++it)
                {
                  double p, dp;
                  legendre(m, x, &p, &dp);
                  const double d2p = (2.0 * x * dp - m * (m + 1) * p) / (1.0 - x * x);
                  const double dx = dp / d2p;
                  x -= dx;
                  if (fabs(dx) < 1e-15)
                    break;
                }
            }
          double p, dp;
          legendre(m, x, &p, &dp);
          pts[i] = 0.5 * (x + 1.0);
          w[i] = 1.0 / (m * (m + 1) * p * p);
        }
    }
  symmetrize(n, pts, w);
  return 0;
}

/* -------------------------------------------------------------- basis --- */
/* basis.cpp:15-47 */
static double lag_value(const double *nodes, int n, int j, double x)
{
  double v = 1.0;
  for (int m = 0; m < n; ++m)
    if (m != j)
      v *= (x - nodes[m]) / (nodes[j] - nodes[m]);
  return v;
}

static double lag_derivative(const double *nodes, int n, int j, double x)
{
  double sum = 0.0;
  for (int i = 0; i < n; ++i)
    {
      if (i == j)
        continue;
      double v = 1.0 / (nodes[j] - nodes[i]);
      for (int m = 0; m < n; ++m)
        if (m != j && m != i)
          v *= (x - nodes[m]) / (nodes[j] - nodes[m]);
      sum += v;
    }
  return sum;
}

/* GL nodes of degree p, make_basis (basis.cpp:128-132) */
static void gl_nodes(int p, double *nodes)
{
  if (p == 0)
    {
      nodes[0] = 0.5;
      return;
    }
  double w[64];
  dgo_gauss(p + 1, 1, nodes, w);
}

/* Values and derivatives of the shifted Legendre polynomials P_m(2x-1),
 * m = 0..n-1, by the three-term recurrence (basis.cpp:40-62). */
static void shifted_legendre(int n, double x, double *p, double *dp)
{
  const double t = 2.0 * x - 1.0;
  for (int m = 0; m < n; ++m)
    {
      if (m == 0)
        {
          p[0] = 1.0;
          dp[0] = 0.0;
        }
      else if (m == 1)
        {
          p[1] = t;
          dp[1] = 2.0;
        }
      else
        {
          p[m] = ((2 * m - 1) * t * p[m - 1] - (m - 1) * p[m - 2]) / m;
          dp[m] = dp[m - 2] + 2.0 * (2 * m - 1) * p[m - 1];
        }
    }
}

/* One-dimensional basis of make_basis (basis.cpp:116-180): kind 0 Lagrange
 * in the Gauss-Lobatto points, 1 Lagrange in the Gauss points, 2 Hermite-like
 * (value/derivative at 0 carried by functions 0/1, derivative/value at 1 by
 * k-2/k-1, values in k-4 interior Chebyshev points; Legendre coefficients
 * from the interpolation conditions by Gaussian elimination with partial
 * pivoting). */
typedef struct
{
  int kind, k;
  double nodes[64];
  double coef[32 * 32]; /* hermite: coef[j*k+m] of P_m in function j */
} basis1d_t;

static int basis_init(basis1d_t *b, int kind, int p)
{
  const int k = p + 1;
  b->kind = kind;
  b->k = k;
  if (kind == 0)
    gl_nodes(p, b->nodes);
  else if (kind == 1)
    {
      double w[64];
      dgo_gauss(k, 0, b->nodes, w);
    }
  else if (kind == 2)
    {
      if (p < 3)
        return fail("make_basis: hermite_like requires cubic or higher degree");
      if (k > 32)
        return fail("make_basis: degree too high");
      double c[32 * 32], a[32 * 32], pv[32], dv[32];
      for (int m = 0; m < k; ++m)
        {
          shifted_legendre(k, 0.0, pv, dv);
          c[0 * k + m] = pv[m];
          c[1 * k + m] = dv[m];
          shifted_legendre(k, 1.0, pv, dv);
          c[(k - 2) * k + m] = dv[m];
          c[(k - 1) * k + m] = pv[m];
          for (int t = 0; t < k - 4; ++t)
            {
              const double xi = 0.5 * (1.0 - cos(M_PI * (t + 1) / (k - 3)));
              shifted_legendre(k, xi, pv, dv);
              c[(2 + t) * k + m] = pv[m];
            }
        }
      /* a = c^{-1}: Gauss-Jordan with partial pivoting on [c | I] */
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j)
          a[i * k + j] = i == j ? 1.0 : 0.0;
      for (int col = 0; col < k; ++col)
        {
          int piv = col;
          for (int r = col + 1; r < k; ++r)
            if (fabs(c[r * k + col]) > fabs(c[piv * k + col]))
              piv = r;
          for (int j = 0; j < k; ++j)
            {
              double t = c[col * k + j];
              c[col * k + j] = c[piv * k + j];
              c[piv * k + j] = t;
              t = a[col * k + j];
              a[col * k + j] = a[piv * k + j];
              a[piv * k + j] = t;
            }
          const double inv = 1.0 / c[col * k + col];
          for (int j = 0; j < k; ++j)
            {
              c[col * k + j] *= inv;
              a[col * k + j] *= inv;
            }
          for (int r = 0; r < k; ++r)
            if (r != col && c[r * k + col] != 0.0)
              {
                const double f = c[r * k + col];
                for (int j = 0; j < k; ++j)
                  {
                    c[r * k + j] -= f * c[col * k + j];
                    a[r * k + j] -= f * a[col * k + j];
                  }
              }
        }
      /* basis function j has the Legendre coefficients of column j */
      for (int j = 0; j < k; ++j)
        for (int m = 0; m < k; ++m)
          b->coef[j * k + m] = a[m * k + j];
    }
  else
    return fail("make_basis: unknown basis kind");
  return 0;
}

static void basis_eval(const basis1d_t *b, int j, double x, double *v, double *dv)
{
  if (b->kind != 2)
    {
      *v = lag_value(b->nodes, b->k, j, x);
      *dv = lag_derivative(b->nodes, b->k, j, x);
      return;
    }
  double pv[32], pd[32];
  shifted_legendre(b->k, x, pv, pd);
  double s = 0.0, sd = 0.0;
  for (int m = 0; m < b->k; ++m)
    {
      s += b->coef[j * b->k + m] * pv[m];
      sd += b->coef[j * b->k + m] * pd[m];
    }
  *v = s;
  *dv = sd;
}

/* face rows (basis.cpp:288-309): the Hermite interpolation conditions pin
 * the value / derivative rows at the end points exactly */
static void basis_face_rows(const basis1d_t *b, double *vf, double *gf)
{
  const int k = b->k;
  for (int f = 0; f < 2; ++f)
    for (int j = 0; j < k; ++j)
      basis_eval(b, j, f ? 1.0 : 0.0, &vf[f * k + j], &gf[f * k + j]);
  if (b->kind == 2)
    {
      for (int i = 0; i < 2 * k; ++i)
        vf[i] = gf[i] = 0.0;
      vf[0] = 1.0;
      gf[1] = 1.0;
      vf[k + k - 1] = 1.0;
      gf[k + k - 2] = 1.0;
    }
}

/* pack_even_odd + unpack_even_odd (basis.cpp:182-259): the plain matrices
 * are re-expanded from their packed halves (basis.cpp:311-323). */
static void even_odd_roundtrip(double *m, int rows, int cols, int skew)
{
  const int rh = rows / 2, ch = cols / 2;
  const int re = skew ? rh : (rows + 1) / 2;
  const int ro = skew ? (rows + 1) / 2 : rh;
  const int ce = (cols + 1) / 2;
  double be[64 * 64], bo[64 * 64];
  for (int q = 0; q < re; ++q)
    for (int j = 0; j < ce; ++j)
      be[q * ce + j] = j < ch ? 0.5 * (m[q * cols + j] + m[q * cols + (cols - 1 - j)])
                              : m[q * cols + j];
  for (int q = 0; q < ro; ++q)
    for (int j = 0; j < ch; ++j)
      bo[q * ch + j] = 0.5 * (m[q * cols + j] - m[q * cols + (cols - 1 - j)]);

  const double sign = skew ? -1.0 : 1.0;
  for (int i = 0; i < rows * cols; ++i)
    m[i] = 0.0;
  for (int q = 0; q < rh; ++q)
    for (int j = 0; j < cols; ++j)
      {
        const int jm = j < cols - 1 - j ? j : cols - 1 - j;
        const double e = be[q * ce + jm];
        const double o = jm < ch ? bo[q * ch + jm] : 0.0;
        const double v = j < ch ? e + o : (j == jm ? e : e - o);
        m[q * cols + j] = v;
        m[(rows - 1 - q) * cols + (cols - 1 - j)] = sign * v;
      }
  if (rows % 2 == 1)
    {
      const int q = rh;
      for (int j = 0; j < cols; ++j)
        {
          const int jm = j < cols - 1 - j ? j : cols - 1 - j;
          if (!skew)
            m[q * cols + j] = be[q * ce + jm];
          else
            m[q * cols + j] = jm < ch ? (j < ch ? bo[q * ch + jm] : -bo[q * ch + jm]) : 0.0;
        }
    }
}

/* shape_matrices, basis.cpp:261-325 (l = k Gauss points); even-odd
 * round trip only for the mirror-symmetric bases (basis.cpp:311-323) */
int dgo_shape(int p, int basis, double *S, double *D, double *Dco, double *Sf, double *Df)
{
  const int k = p + 1;
  if (k > 32)
    return fail("dgo_shape: degree too high");
  basis1d_t b;
  if (basis_init(&b, basis, p))
    return -1;
  double qp[64], qw[64];
  dgo_gauss(k, 0, qp, qw);
  for (int q = 0; q < k; ++q)
    {
      for (int j = 0; j < k; ++j)
        basis_eval(&b, j, qp[q], &S[q * k + j], &D[q * k + j]);
      for (int j = 0; j < k; ++j)
        Dco[q * k + j] = lag_derivative(qp, k, j, qp[q]);
    }
  basis_face_rows(&b, Sf, Df);
  if (basis != 2)
    {
      even_odd_roundtrip(S, k, k, 0);
      even_odd_roundtrip(D, k, k, 1);
      even_odd_roundtrip(Dco, k, k, 1);
    }
  return 0;
}

/* --------------------------------------------------------------- mesh --- */
static int n_cells_of(int d, const int *cells)
{
  int n = 1;
  for (int a = 0; a < d; ++a)
    n *= cells[a];
  return n;
}

static void multi_index(int d, const int *cells, int c, int *m)
{
  m[0] = m[1] = m[2] = 0;
  for (int a = 0; a < d; ++a)
    {
      m[a] = c % cells[a];
      c /= cells[a];
    }
}

static int cell_index(int d, const int *cells, const int *m)
{
  int c = 0;
  for (int a = d - 1; a >= 0; --a)
    c = c * cells[a] + m[a];
  return c;
}

/* enumerate_faces, mesh.cpp:70-132 (make_box_mesh: dirichlet id = side) */
int64_t dgo_faces(int d, const int *cells, int periodic, uint32_t *fi,
                  uint32_t *fe, uint8_t *ni, uint8_t *ne)
{
  const int nc = n_cells_of(d, cells);
  int64_t n = 0;
#define PUSH(I, E, NI, NE)                                                    \
  do                                                                          \
    {                                                                         \
      if (fi)                                                                 \
        {                                                                     \
          fi[n] = (I);                                                        \
          fe[n] = (E);                                                        \
          ni[n] = (uint8_t)(NI);                                              \
          ne[n] = (uint8_t)(NE);                                              \
        }                                                                     \
      ++n;                                                                    \
    }                                                                         \
  while (0)
  for (int a = 0; a < d; ++a)
    for (int c = 0; c < nc; ++c)
      {
        int m[3];
        multi_index(d, cells, c, m);
        if (m[a] == 0 && !periodic)
          PUSH((uint32_t)c, 0xffffffffu, 2 * a, 2 * a);
        if (m[a] == cells[a] - 1)
          {
            if (!periodic)
              PUSH((uint32_t)c, 0xffffffffu, 2 * a + 1, 2 * a + 1);
            else
              {
                int mn[3] = {m[0], m[1], m[2]};
                mn[a] = 0;
                PUSH((uint32_t)cell_index(d, cells, mn), (uint32_t)c, 2 * a, 2 * a + 1);
              }
          }
        else
          {
            int mn[3] = {m[0], m[1], m[2]};
            mn[a] = m[a] + 1;
            PUSH((uint32_t)c, (uint32_t)cell_index(d, cells, mn), 2 * a + 1, 2 * a);
          }
      }
#undef PUSH
  return n;
}

/* partition_cells, mesh.cpp:134-155 */
int dgo_partition(int n, int n_ranks, int *owner, int *ranges)
{
  if (n_ranks < 1 || n_ranks > n)
    return fail("partition: rank count must be in [1, n_cells]");
  const int base = n / n_ranks, extra = n % n_ranks;
  int begin = 0;
  for (int r = 0; r < n_ranks; ++r)
    {
      const int size = base + (r < extra ? 1 : 0);
      ranges[2 * r] = begin;
      ranges[2 * r + 1] = begin + size;
      for (int c = begin; c < begin + size; ++c)
        owner[c] = r;
      begin += size;
    }
  return 0;
}

typedef struct
{
  int64_t key; /* ra * 2^20 + rb */
  int64_t face;
} iface_t;

static int cmp_iface(const void *a, const void *b)
{
  const iface_t *x = a, *y = b;
  if (x->key != y->key)
    return x->key < y->key ? -1 : 1;
  return x->face < y->face ? -1 : (x->face > y->face);
}

/* assign_face_owners, mesh.cpp:157-232 */
int dgo_face_owners(int64_t nf, const uint32_t *fi, const uint32_t *fe,
                    const int *owner, int *face_owner)
{
  iface_t *list = malloc(sizeof(iface_t) * (nf > 0 ? nf : 1));
  int64_t nl = 0;
  uint32_t max_cell = 0;
  for (int64_t i = 0; i < nf; ++i)
    {
      if (fi[i] > max_cell)
        max_cell = fi[i];
      if (fe[i] != 0xffffffffu && fe[i] > max_cell)
        max_cell = fe[i];
      face_owner[i] = -1;
      const int ri = owner[fi[i]];
      if (fe[i] == 0xffffffffu)
        {
          face_owner[i] = ri;
          continue;
        }
      const int re = owner[fe[i]];
      if (ri == re)
        face_owner[i] = ri;
      else
        {
          const int lo = ri < re ? ri : re, hi = ri < re ? re : ri;
          list[nl].key = (int64_t)lo * (1 << 20) + hi;
          list[nl].face = i;
          ++nl;
        }
    }
  qsort(list, nl, sizeof(iface_t), cmp_iface);
  int *mult = calloc(max_cell + 1, sizeof(int));
  int *group = malloc(sizeof(int) * (max_cell + 1));
  for (uint32_t c = 0; c <= max_cell; ++c)
    group[c] = -1;
  int64_t s = 0;
  while (s < nl)
    {
      int64_t e = s;
      while (e < nl && list[e].key == list[s].key)
        ++e;
      const int ra = (int)(list[s].key >> 20), rb = (int)(list[s].key & ((1 << 20) - 1));
      for (int64_t t = s; t < e; ++t)
        {
          ++mult[fi[list[t].face]];
          ++mult[fe[list[t].face]];
        }
      int count_a = 0, count_b = 0, n_groups = 0;
      int64_t *singles = malloc(sizeof(int64_t) * (e - s));
      int64_t ns = 0;
      for (int64_t t = s; t < e; ++t)
        {
          const int64_t i = list[t].face;
          const uint32_t ca = owner[fi[i]] == ra ? fi[i] : fe[i];
          const uint32_t cb = ca == fi[i] ? fe[i] : fi[i];
          const int ma = mult[ca], mb = mult[cb];
          int r = -1;
          if (ma >= 2 && mb < 2)
            r = rb;
          else if (mb >= 2 && ma < 2)
            r = ra;
          else if (ma >= 2 && mb >= 2)
            {
              if (group[ca] < 0)
                {
                  group[ca] = n_groups % 2 == 0 ? rb : ra;
                  ++n_groups;
                }
              r = group[ca];
            }
          else
            singles[ns++] = i;
          if (r >= 0)
            {
              face_owner[i] = r;
              if (r == ra)
                ++count_a;
              else
                ++count_b;
            }
        }
      for (int64_t t = 0; t < ns; ++t)
        {
          const int r = count_a <= count_b ? ra : rb;
          face_owner[singles[t]] = r;
          if (r == ra)
            ++count_a;
          else
            ++count_b;
        }
      free(singles);
      for (int64_t t = s; t < e; ++t)
        {
          mult[fi[list[t].face]] = 0;
          mult[fe[list[t].face]] = 0;
          group[fi[list[t].face]] = -1;
          group[fe[list[t].face]] = -1;
        }
      s = e;
    }
  free(mult);
  free(group);
  free(list);
  return 0;
}

static int cmp_u32(const void *a, const void *b)
{
  const uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
  return x < y ? -1 : (x > y);
}

/* ghost cells, dof_layout.cpp:191-213 */
int64_t dgo_ghosts(int rank, int64_t nf, const uint32_t *fi, const uint32_t *fe,
                   const int *face_owner, const int *owner, uint32_t *ghosts)
{
  uint32_t *tmp = malloc(sizeof(uint32_t) * (2 * nf + 1));
  int64_t n = 0;
  for (int64_t i = 0; i < nf; ++i)
    {
      if (face_owner[i] != rank)
        continue;
      if (owner[fi[i]] != rank)
        tmp[n++] = fi[i];
      if (fe[i] != 0xffffffffu && owner[fe[i]] != rank)
        tmp[n++] = fe[i];
    }
  qsort(tmp, n, sizeof(uint32_t), cmp_u32);
  int64_t u = 0;
  for (int64_t i = 0; i < n; ++i)
    if (u == 0 || tmp[u - 1] != tmp[i])
      tmp[u++] = tmp[i];
  if (ghosts)
    memcpy(ghosts, tmp, sizeof(uint32_t) * u);
  free(tmp);
  return u;
}

/* ---------------------------------------------------- support points --- */
/* build_mapping (geometry.cpp:36-63) with Mesh::map_point (mesh.cpp:11-26)
 * on the unit box. */
int dgo_support_reference(int d, const int *cells, double amp, int m,
                          double *sup)
{
  double nodes[64];
  gl_nodes(m, nodes);
  const int nc = n_cells_of(d, cells);
  const int64_t pp = ipow64(m + 1, d);
  double *out = sup;
  for (int c = 0; c < nc; ++c)
    {
      int mi[3];
      multi_index(d, cells, c, mi);
      for (int64_t s = 0; s < pp; ++s)
        {
          double xi[3] = {0, 0, 0};
          int64_t idx = s;
          for (int a = 0; a < d; ++a)
            {
              xi[a] = nodes[idx % (m + 1)];
              idx /= (m + 1);
            }
          double y[3] = {0, 0, 0};
          for (int a = 0; a < d; ++a)
            y[a] = (mi[a] + xi[a]) / cells[a];
          double bump = amp;
          for (int a = 0; a < d; ++a)
            bump *= sin(M_PI * y[a]);
          for (int a = 0; a < d; ++a)
            *out++ = 0.0 + (1.0 - 0.0) * (y[a] + bump);
        }
    }
  return 0;
}

/* BASELINE.json configs[2..3]: vertices x + eps*h*sin(2 pi x)sin(2 pi y)
 * [sin(2 pi z)] per component; cells are trilinear between their vertices. */
int dgo_support_vertex_bump(int d, const int *cells, double eps, double *sup)
{
  const int nc = n_cells_of(d, cells);
  const int pp = 1 << d;
  double *out = sup;
  for (int c = 0; c < nc; ++c)
    {
      int mi[3];
      multi_index(d, cells, c, mi);
      for (int s = 0; s < pp; ++s)
        {
          double x[3];
          for (int a = 0; a < d; ++a)
            x[a] = (double)(mi[a] + ((s >> a) & 1)) / cells[a];
          double bump = 1.0;
          for (int a = 0; a < d; ++a)
            bump *= sin(2.0 * M_PI * x[a]);
          for (int a = 0; a < d; ++a)
            *out++ = x[a] + eps * (1.0 / cells[a]) * bump;
        }
    }
  return 0;
}

/* ----------------------------------------------------------- geometry --- */
typedef struct
{
  int m, n;
  double nodes[16];
} mapbasis_t;

/* mapping_point_jacobian, geometry.cpp:65-116 */
static void map_point_jac(const mapbasis_t *mb, int d, const double *sp,
                          const double *xi, double *x_out, double *jac)
{
  const int n = mb->n;
  double val[3][16], der[3][16];
  for (int a = 0; a < d; ++a)
    for (int j = 0; j < n; ++j)
      {
        val[a][j] = lag_value(mb->nodes, n, j, xi[a]);
        der[a][j] = lag_derivative(mb->nodes, n, j, xi[a]);
      }
  if (x_out)
    for (int i = 0; i < d; ++i)
      x_out[i] = 0.0;
  for (int i = 0; i < d * d; ++i)
    jac[i] = 0.0;
  const int64_t np = ipow64(n, d);
  for (int64_t s = 0; s < np; ++s)
    {
      double shape = 1.0, dshape[3];
      int64_t idx = s;
      int loc[3] = {0, 0, 0};
      for (int a = 0; a < d; ++a)
        {
          loc[a] = (int)(idx % n);
          idx /= n;
          shape *= val[a][loc[a]];
        }
      for (int a = 0; a < d; ++a)
        {
          double p = der[a][loc[a]];
          for (int b = 0; b < d; ++b)
            if (b != a)
              p *= val[b][loc[b]];
          dshape[a] = p;
        }
      const double *xs = sp + s * d;
      if (x_out)
        for (int i = 0; i < d; ++i)
          x_out[i] += shape * xs[i];
      for (int i = 0; i < d; ++i)
        for (int a = 0; a < d; ++a)
          jac[i * d + a] += dshape[a] * xs[i];
    }
}

/* invert_jacobian, geometry.cpp:118-150 */
static double invert_jac(int d, const double *jac, double *jit)
{
  if (d == 2)
    {
      const double a = jac[0], b = jac[1], c = jac[2], e = jac[3];
      const double det = a * e - b * c;
      const double inv = 1.0 / det;
      jit[0] = e * inv;
      jit[1] = -c * inv;
      jit[2] = -b * inv;
      jit[3] = a * inv;
      return det;
    }
  const double *j = jac;
  double cof[9];
  cof[0] = j[4] * j[8] - j[5] * j[7];
  cof[1] = j[5] * j[6] - j[3] * j[8];
  cof[2] = j[3] * j[7] - j[4] * j[6];
  cof[3] = j[2] * j[7] - j[1] * j[8];
  cof[4] = j[0] * j[8] - j[2] * j[6];
  cof[5] = j[1] * j[6] - j[0] * j[7];
  cof[6] = j[1] * j[5] - j[2] * j[4];
  cof[7] = j[2] * j[3] - j[0] * j[5];
  cof[8] = j[0] * j[4] - j[1] * j[3];
  const double det = j[0] * cof[0] + j[1] * cof[1] + j[2] * cof[2];
  const double inv = 1.0 / det;
  for (int i = 0; i < 9; ++i)
    jit[i] = cof[i] * inv;
  return det;
}

static double coef_a(const double *x)
{
  return 1.0 + 0.5 * sin(M_PI * x[0]) * cos(M_PI * x[1]);
}

/* precompute_geometry, geometry.cpp:248-522, g3 + Laplacian */
int dgo_geometry(int d, const int *cells, int m, const double *support, int k,
                 int compress, int coefficient, int64_t nfaces,
                 const uint32_t *fi, const uint32_t *fe, const uint8_t *ni,
                 const uint8_t *ne, double *inv_jac_t, double *jxw,
                 double *face_jxw, double *face_jni, double *face_jne,
                 double *penalty, double *cell_volume)
{
  if (m < 1 || m > 15)
    return fail("dgo_geometry: mapping degree out of range");
  if (compress && coefficient)
    return fail("dgo_geometry: a(x) folding needs per-point storage");
  const int l = k;
  double qp[64], qw[64];
  dgo_gauss(l, 0, qp, qw);
  mapbasis_t mb;
  mb.m = m;
  mb.n = m + 1;
  gl_nodes(m, mb.nodes);
  const int nc = n_cells_of(d, cells);
  const int64_t nq = ipow64(l, d), nqf = ipow64(l, d - 1);
  const int64_t pp = ipow64(m + 1, d);
  double *wq = malloc(sizeof(double) * nq), *wqf = malloc(sizeof(double) * nqf);
  for (int64_t q = 0; q < nq; ++q)
    {
      double w = 1.0;
      int64_t idx = q;
      for (int a = 0; a < d; ++a)
        {
          w *= qw[idx % l];
          idx /= l;
        }
      wq[q] = w;
    }
  for (int64_t q = 0; q < nqf; ++q)
    {
      double w = 1.0;
      int64_t idx = q;
      for (int a = 0; a < d - 1; ++a)
        {
          w *= qw[idx % l];
          idx /= l;
        }
      wqf[q] = w;
    }
  const int64_t nrec = compress ? 1 : nq;
  int status = 0;
  for (int c = 0; c < nc && status == 0; ++c)
    {
      const double *sp = support + (int64_t)c * pp * d;
      for (int64_t rec = 0; rec < nrec; ++rec)
        {
          double xi[3] = {0.5, 0.5, 0.5};
          if (!compress)
            {
              int64_t idx = rec;
              for (int a = 0; a < d; ++a)
                {
                  xi[a] = qp[idx % l];
                  idx /= l;
                }
            }
          double x[3], jac[9], jit[9];
          map_point_jac(&mb, d, sp, xi, x, jac);
          const double det = invert_jac(d, jac, jit);
          if (!(det > 0.0))
            {
              status = fail("precompute_geometry: non-positive mapping Jacobian");
              break;
            }
          double det_jxw = compress ? det : det * wq[rec];
          if (coefficient)
            det_jxw *= coef_a(x);
          for (int i = 0; i < d * d; ++i)
            inv_jac_t[((int64_t)c * nrec + rec) * d * d + i] = jit[i];
          jxw[(int64_t)c * nrec + rec] = det_jxw;
        }
      if (compress)
        {
          double v = 1.0;
          for (int a = 0; a < d; ++a)
            v *= (1.0 - 0.0) / cells[a];
          cell_volume[c] = v;
        }
      else
        {
          cell_volume[c] = 0.0;
          for (int64_t q = 0; q < nq; ++q)
            {
              double xi[3] = {0, 0, 0};
              int64_t idx = q;
              for (int a = 0; a < d; ++a)
                {
                  xi[a] = qp[idx % l];
                  idx /= l;
                }
              double jac[9], jit[9];
              map_point_jac(&mb, d, sp, xi, NULL, jac);
              cell_volume[c] += invert_jac(d, jac, jit) * wq[q];
            }
        }
    }
  double *av = malloc(sizeof(double) * nqf);
  for (int64_t f = 0; f < nfaces && status == 0; ++f)
    {
      const int axis = ni[f] / 2;
      int tang[2], nt = 0;
      for (int a = 0; a < d; ++a)
        if (a != axis)
          tang[nt++] = a;
      const int boundary = fe[f] == 0xffffffffu;
      double area = 0.0;
      for (int64_t q = 0; q < nqf; ++q)
        {
          double tc[2] = {0.5, 0.5};
          int64_t idx = q;
          for (int t = 0; t < nt; ++t)
            {
              tc[t] = qp[idx % l];
              idx /= l;
            }
          double xi[3] = {0, 0, 0};
          for (int t = 0; t < nt; ++t)
            xi[tang[t]] = tc[t];
          xi[axis] = ni[f] % 2 ? 1.0 : 0.0;
          double xq[3], jac[9], jit[9];
          map_point_jac(&mb, d, support + (int64_t)fi[f] * pp * d, xi, xq, jac);
          const double det = invert_jac(d, jac, jit);
          if (!(det > 0.0))
            {
              status = fail("precompute_geometry: non-positive Jacobian on a face");
              break;
            }
          const double sign = ni[f] % 2 ? 1.0 : -1.0;
          double nvec[3], nrm = 0, normal[3];
          for (int i = 0; i < d; ++i)
            {
              nvec[i] = jit[i * d + axis];
              nrm += nvec[i] * nvec[i];
            }
          nrm = sqrt(nrm);
          for (int i = 0; i < d; ++i)
            normal[i] = sign * nvec[i] / nrm;
          const int64_t base = f * nqf + q;
          face_jxw[base] = det * nrm * wqf[q];
          area += face_jxw[base];
          av[q] = coefficient ? coef_a(xq) : 1.0;
          for (int j = 0; j < d; ++j)
            {
              double s = 0;
              for (int i = 0; i < d; ++i)
                s += normal[i] * jit[i * d + j];
              face_jni[base * d + j] = s;
            }
          if (boundary)
            for (int j = 0; j < d; ++j)
              face_jne[base * d + j] = face_jni[base * d + j];
          else
            {
              double xie[3] = {0, 0, 0};
              for (int t = 0; t < nt; ++t)
                xie[tang[t]] = tc[t];
              xie[axis] = ne[f] % 2 ? 1.0 : 0.0;
              double jace[9], jite[9];
              map_point_jac(&mb, d, support + (int64_t)fe[f] * pp * d, xie, NULL, jace);
              if (!(invert_jac(d, jace, jite) > 0.0))
                {
                  status = fail("precompute_geometry: non-positive Jacobian on a face");
                  break;
                }
              for (int j = 0; j < d; ++j)
                {
                  double s = 0;
                  for (int i = 0; i < d; ++i)
                    s += normal[i] * jite[i * d + j];
                  face_jne[base * d + j] = s;
                }
            }
        }
      if (status)
        break;
      const double p1sq = (double)k * k;
      if (boundary)
        penalty[f] = p1sq * area / cell_volume[fi[f]];
      else
        penalty[f] = p1sq * 0.5 * (area / cell_volume[fi[f]] + area / cell_volume[fe[f]]);
      if (coefficient)
        {
          double abar = 0.0;
          for (int64_t q = 0; q < nqf; ++q)
            {
              abar += av[q];
              for (int j = 0; j < d; ++j)
                {
                  face_jni[(f * nqf + q) * d + j] *= av[q];
                  face_jne[(f * nqf + q) * d + j] *= av[q];
                }
            }
          penalty[f] *= abar / (double)nqf;
        }
    }
  free(av);
  free(wq);
  free(wqf);
  return status;
}

/* -------------------------------------------------------------- apply --- */
static int64_t local_cell(uint32_t g, int begin, int end, int64_t ng,
                          const uint32_t *ghosts)
{
  if ((int64_t)g >= begin && (int64_t)g < end)
    return (int64_t)g - begin;
  int64_t lo = 0, hi = ng;
  while (lo < hi)
    {
      const int64_t mid = (lo + hi) / 2;
      if (ghosts[mid] < g)
        lo = mid + 1;
      else
        hi = mid;
    }
  if (lo < ng && ghosts[lo] == g)
    return (end - begin) + lo;
  return -1;
}

/* Table-based evaluation of the SIP weak form (oracle.cpp:205-426 applied
 * matrix-free; flux algebra of operators.cpp:933-1111). */
int dgo_apply_rank(int d, int k, int n_cells, int compress,
                   const double *inv_jac_t, const double *jxw, int64_t nf,
                   const uint32_t *fi, const uint32_t *fe, const uint8_t *ni,
                   const uint8_t *ne, const double *face_jxw,
                   const double *face_jni, const double *face_jne,
                   const double *penalty, int rank, const int *face_owner,
                   int begin, int end, int64_t ng, const uint32_t *ghosts,
                   const double *u, double *y, int basis)
{
  (void)n_cells;
  if (k > 16)
    return fail("dgo_apply_rank: k too large for the table oracle");
  basis1d_t bas;
  if (basis_init(&bas, basis, k - 1))
    return -1;
  double qp[64], qw[64];
  dgo_gauss(k, 0, qp, qw);
  double v[16 * 16], g[16 * 16], vf[2][16], gf[2][16];
  for (int q = 0; q < k; ++q)
    for (int j = 0; j < k; ++j)
      basis_eval(&bas, j, qp[q], &v[q * k + j], &g[q * k + j]);
  {
    double rv[32], rg[32];
    basis_face_rows(&bas, rv, rg);
    for (int f = 0; f < 2; ++f)
      for (int j = 0; j < k; ++j)
        {
          vf[f][j] = rv[f * k + j];
          gf[f][j] = rg[f * k + j];
        }
  }
  const int64_t nj = ipow64(k, d), nq = nj, nqf = ipow64(k, d - 1);
  double *wq = malloc(sizeof(double) * nq);
  for (int64_t q = 0; q < nq; ++q)
    {
      double w = 1.0;
      int64_t idx = q;
      for (int a = 0; a < d; ++a)
        {
          w *= qw[idx % k];
          idx /= k;
        }
      wq[q] = w;
    }
  /* cell tables, oracle.cpp:79-122 */
  double *dphi = malloc(sizeof(double) * nq * nj * d);
  for (int64_t q = 0; q < nq; ++q)
    for (int64_t j = 0; j < nj; ++j)
      {
        int qm[3], jm[3];
        int64_t qq = q, jj = j;
        for (int a = 0; a < d; ++a)
          {
            qm[a] = (int)(qq % k);
            qq /= k;
            jm[a] = (int)(jj % k);
            jj /= k;
          }
        for (int a = 0; a < d; ++a)
          {
            double dp = g[qm[a] * k + jm[a]];
            for (int b = 0; b < d; ++b)
              if (b != a)
                dp *= v[qm[b] * k + jm[b]];
            dphi[(q * nj + j) * d + a] = dp;
          }
      }
  /* face tables, oracle.cpp:134-201 */
  double *fphi = malloc(sizeof(double) * 2 * d * nqf * nj);
  double *fdphi = malloc(sizeof(double) * 2 * d * nqf * nj * d);
  for (int fn = 0; fn < 2 * d; ++fn)
    {
      const int axis = fn / 2, side = fn % 2;
      int tang[2], nt = 0;
      for (int a = 0; a < d; ++a)
        if (a != axis)
          tang[nt++] = a;
      for (int64_t q = 0; q < nqf; ++q)
        {
          int qm[3] = {0, 0, 0};
          int64_t qq = q;
          for (int t = 0; t < nt; ++t)
            {
              qm[tang[t]] = (int)(qq % k);
              qq /= k;
            }
          for (int64_t j = 0; j < nj; ++j)
            {
              int jm[3];
              int64_t jj = j;
              for (int a = 0; a < d; ++a)
                {
                  jm[a] = (int)(jj % k);
                  jj /= k;
                }
              double fac[3];
              for (int a = 0; a < d; ++a)
                fac[a] = a == axis ? vf[side][jm[a]] : v[qm[a] * k + jm[a]];
              double p = 1.0;
              for (int a = 0; a < d; ++a)
                p *= fac[a];
              fphi[((int64_t)fn * nqf + q) * nj + j] = p;
              for (int a = 0; a < d; ++a)
                {
                  double dp = a == axis ? gf[side][jm[a]] : g[qm[a] * k + jm[a]];
                  for (int b = 0; b < d; ++b)
                    if (b != a)
                      dp *= fac[b];
                  fdphi[(((int64_t)fn * nqf + q) * nj + j) * d + a] = dp;
                }
            }
        }
    }

  const int64_t n_local = (int64_t)(end - begin) + ng;
  memset(y, 0, sizeof(double) * n_local * nj);
  double *gr = malloc(sizeof(double) * nq * 3);
  /* cell integrals: (J^{-1}J^{-T} grad u, grad v) JxW, geometry.cpp:189-209 */
  for (int c = begin; c < end; ++c)
    {
      const double *uc = u + (int64_t)(c - begin) * nj;
      double *yc = y + (int64_t)(c - begin) * nj;
      for (int64_t q = 0; q < nq; ++q)
        {
          double gref[3] = {0, 0, 0};
          for (int64_t j = 0; j < nj; ++j)
            for (int a = 0; a < d; ++a)
              gref[a] += dphi[(q * nj + j) * d + a] * uc[j];
          const int64_t rec = compress ? c : (int64_t)c * nq + q;
          const double *jit = inv_jac_t + rec * d * d;
          const double jw = compress ? jxw[c] * wq[q] : jxw[rec];
          double gp[3], t[3];
          for (int i = 0; i < d; ++i)
            {
              double s = 0;
              for (int j = 0; j < d; ++j)
                s += jit[i * d + j] * gref[j];
              gp[i] = s;
            }
          for (int i = 0; i < d; ++i)
            {
              double s = 0;
              for (int j = 0; j < d; ++j)
                s += jit[j * d + i] * gp[j];
              t[i] = s * jw;
            }
          for (int a = 0; a < d; ++a)
            gr[q * 3 + a] = t[a];
        }
      for (int64_t i = 0; i < nj; ++i)
        {
          double s = 0;
          for (int64_t q = 0; q < nq; ++q)
            for (int a = 0; a < d; ++a)
              s += dphi[(q * nj + i) * d + a] * gr[q * 3 + a];
          yc[i] = s;
        }
    }
  /* face integrals, operators.cpp:977-1003 (interior), 1069-1089 (boundary) */
  int status = 0;
  for (int64_t f = 0; f < nf; ++f)
    {
      if (face_owner && face_owner[f] != rank)
        continue;
      const int boundary = fe[f] == 0xffffffffu;
      const int nsides = boundary ? 1 : 2;
      int64_t lc[2];
      const int fn[2] = {ni[f], ne[f]};
      const uint32_t gc[2] = {fi[f], fe[f]};
      for (int s = 0; s < nsides; ++s)
        {
          lc[s] = local_cell(gc[s], begin, end, ng, ghosts);
          if (lc[s] < 0)
            {
              status = fail("dgo_apply_rank: face references an absent cell");
              break;
            }
        }
      if (status)
        break;
      const double tau = penalty[f];
      for (int64_t q = 0; q < nqf; ++q)
        {
          const int64_t base = f * nqf + q;
          const double jw = face_jxw[base];
          double uq[2] = {0, 0}, dn[2] = {0, 0};
          const double *jn[2] = {face_jni + base * d, face_jne + base * d};
          for (int s = 0; s < nsides; ++s)
            {
              const double *us = u + lc[s] * nj;
              const double *ph = fphi + ((int64_t)fn[s] * nqf + q) * nj;
              const double *dph = fdphi + ((int64_t)fn[s] * nqf + q) * nj * d;
              double val = 0, gref[3] = {0, 0, 0};
              for (int64_t j = 0; j < nj; ++j)
                {
                  val += ph[j] * us[j];
                  for (int a = 0; a < d; ++a)
                    gref[a] += dph[j * d + a] * us[j];
                }
              uq[s] = val;
              double acc = 0;
              for (int a = 0; a < d; ++a)
                acc += gref[a] * jn[s][a];
              dn[s] = acc;
            }
          double rv[2], gg;
          if (boundary)
            {
              rv[0] = (uq[0] * tau * 2.0 - dn[0]) * jw;
              gg = -(uq[0] * jw);
            }
          else
            {
              const double jump = uq[0] - uq[1];
              const double r0 = (jump * tau - (dn[0] + dn[1]) * 0.5) * jw;
              rv[0] = r0;
              rv[1] = -r0;
              gg = -(jump * jw * 0.5);
            }
          for (int s = 0; s < nsides; ++s)
            {
              double *ys = y + lc[s] * nj;
              const double *ph = fphi + ((int64_t)fn[s] * nqf + q) * nj;
              const double *dph = fdphi + ((int64_t)fn[s] * nqf + q) * nj * d;
              double rg[3];
              for (int a = 0; a < d; ++a)
                rg[a] = gg * jn[s][a];
              for (int64_t j = 0; j < nj; ++j)
                {
                  double acc = ph[j] * rv[s];
                  for (int a = 0; a < d; ++a)
                    acc += dph[j * d + a] * rg[a];
                  ys[j] += acc;
                }
            }
        }
    }
  free(gr);
  free(fphi);
  free(fdphi);
  free(dphi);
  free(wq);
  return status;
}

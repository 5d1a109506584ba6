// Host setup: see setup.hpp. Built with -ffp-contract=off so the 1D tables
// match the reference's bit for bit (reference CMakeLists.txt:33-39).
#include "setup.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <tuple>

namespace dgx
{

namespace
{

// Legendre P_n and P_n' on [-1,1] by the three-term recurrence
// (quadrature.cpp:15-35).
void legendre(int n, double x, double &p, double &dp)
{
  double p0 = 1.0, p1 = x;
  if (n == 0)
    {
      p = 1.0;
      dp = 0.0;
      return;
    }
  for (int m = 2; m <= n; ++m)
    {
      const double p2 = ((2 * m - 1) * x * p1 - (m - 1) * p0) / m;
      p0 = p1;
      p1 = p2;
    }
  p = p1;
  if (std::abs(x) == 1.0)
    dp = (n % 2 == 0 ? x : 1.0) * n * (n + 1) / 2.0;
  else
    dp = n * (x * p1 - p0) / (x * x - 1.0);
}

void symmetrize(Quad1D &q)
{
  const int n = static_cast<int>(q.points.size());
  for (int i = 0; i < n / 2; ++i)
    {
      const int j = n - 1 - i;
      const double p = 0.5 * (q.points[i] + (1.0 - q.points[j]));
      q.points[i] = p;
      q.points[j] = 1.0 - p;
      const double w = 0.5 * (q.weights[i] + q.weights[j]);
      q.weights[i] = w;
      q.weights[j] = w;
    }
  if (n % 2 == 1)
    q.points[n / 2] = 0.5;
}

double lagrange_value(const std::vector<double> &x, int j, double t)
{
  double v = 1.0;
  for (int m = 0; m < static_cast<int>(x.size()); ++m)
    if (m != j)
      v *= (t - x[m]) / (x[j] - x[m]);
  return v;
}

double lagrange_derivative(const std::vector<double> &x, int j, double t)
{
  double sum = 0.0;
  const int n = static_cast<int>(x.size());
  for (int i = 0; i < n; ++i)
    {
      if (i == j)
        continue;
      double v = 1.0 / (x[j] - x[i]);
      for (int m = 0; m < n; ++m)
        if (m != j && m != i)
          v *= (t - x[m]) / (x[j] - x[m]);
      sum += v;
    }
  return sum;
}

// Mirror (even-odd) form and back: the reference stores the plain matrices
// re-expanded from their packed halves (basis.cpp:182-259,311-323); doing
// the same keeps our tables bitwise equal to the reference's.
void mirror_roundtrip(std::vector<double> &m, int n, bool skew)
{
  const int rh = n / 2, ch = n / 2;
  const int re = skew ? rh : (n + 1) / 2, ro = skew ? (n + 1) / 2 : rh;
  const int ce = (n + 1) / 2;
  std::vector<double> be(re * ce), bo(ro * ch);
  for (int q = 0; q < re; ++q)
    for (int j = 0; j < ce; ++j)
      be[q * ce + j] = j < ch ? 0.5 * (m[q * n + j] + m[q * n + (n - 1 - j)])
                              : m[q * n + j];
  for (int q = 0; q < ro; ++q)
    for (int j = 0; j < ch; ++j)
      bo[q * ch + j] = 0.5 * (m[q * n + j] - m[q * n + (n - 1 - j)]);
  const double sign = skew ? -1.0 : 1.0;
  std::fill(m.begin(), m.end(), 0.0);
  for (int q = 0; q < rh; ++q)
    for (int j = 0; j < n; ++j)
      {
        const int jm = std::min(j, n - 1 - j);
        const double e = be[q * ce + jm];
        const double o = jm < ch ? bo[q * ch + jm] : 0.0;
        const double v = j < ch ? e + o : (j == jm ? e : e - o);
        m[q * n + j] = v;
        m[(n - 1 - q) * n + (n - 1 - j)] = sign * v;
      }
  if (n % 2 == 1)
    {
      const int q = rh;
      for (int j = 0; j < n; ++j)
        {
          const int jm = std::min(j, n - 1 - j);
          if (!skew)
            m[q * n + j] = be[q * ce + jm];
          else
            m[q * n + j] = jm < ch ? (j < ch ? bo[q * ch + jm] : -bo[q * ch + jm]) : 0.0;
        }
    }
}

} // namespace

Quad1D gauss(int n)
{
  if (n < 1)
    fail(Code::invalid_argument, "gauss: need at least one point");
  Quad1D q;
  q.points.resize(n);
  q.weights.resize(n);
  for (int i = 0; i < n; ++i)
    {
      double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
      double p = 0, dp = 1;
      for (int it = 0; it < 100; ++it)
        {
          legendre(n, x, p, dp);
          const double dx = p / dp;
          x -= dx;
          if (std::abs(dx) < 1e-15)
            break;
        }
      legendre(n, x, p, dp);
      q.points[n - 1 - i] = 0.5 * (x + 1.0);
      q.weights[n - 1 - i] = 1.0 / ((1.0 - x * x) * dp * dp);
    }
  symmetrize(q);
  return q;
}

Quad1D gauss_lobatto(int n)
{
  if (n < 2)
    fail(Code::invalid_argument, "gauss_lobatto: need at least two points");
  Quad1D q;
  q.points.resize(n);
  q.weights.resize(n);
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
          x = std::cos(M_PI * (m - i) / m);
          for (int it = 0; it < 100; ++it)
            {
              double p, dp;
              legendre(m, x, p, dp);
              const double d2p = (2.0 * x * dp - m * (m + 1) * p) / (1.0 - x * x);
              const double dx = dp / d2p;
              x -= dx;
              if (std::abs(dx) < 1e-15)
                break;
            }
        }
      double p, dp;
      legendre(m, x, p, dp);
      q.points[i] = 0.5 * (x + 1.0);
      q.weights[i] = 1.0 / (m * (m + 1) * p * p);
    }
  symmetrize(q);
  return q;
}

namespace
{
// Values and derivatives of the shifted Legendre polynomials P_m(2x-1),
// m = 0..n-1 (basis.cpp:40-62).
void shifted_legendre(int n, double x, double *p, double *dp)
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

// Legendre coefficients of the Hermite-like basis (basis.cpp:139-177):
// functions 0/1 carry value/derivative at 0, k-2/k-1 derivative/value at 1,
// the others interpolate k-4 interior Chebyshev points. Column j of the
// inverse of the condition matrix (Gauss-Jordan, partial pivoting).
std::vector<double> hermite_coefficients(int k)
{
  std::vector<double> c(k * k), a(k * k, 0.0), pv(k), dv(k);
  for (int m = 0; m < k; ++m)
    {
      shifted_legendre(k, 0.0, pv.data(), dv.data());
      c[0 * k + m] = pv[m];
      c[1 * k + m] = dv[m];
      shifted_legendre(k, 1.0, pv.data(), dv.data());
      c[(k - 2) * k + m] = dv[m];
      c[(k - 1) * k + m] = pv[m];
      for (int t = 0; t < k - 4; ++t)
        {
          const double xi = 0.5 * (1.0 - std::cos(M_PI * (t + 1) / (k - 3)));
          shifted_legendre(k, xi, pv.data(), dv.data());
          c[(2 + t) * k + m] = pv[m];
        }
    }
  for (int i = 0; i < k; ++i)
    a[i * k + i] = 1.0;
  for (int col = 0; col < k; ++col)
    {
      int piv = col;
      for (int r = col + 1; r < k; ++r)
        if (std::abs(c[r * k + col]) > std::abs(c[piv * k + col]))
          piv = r;
      for (int j = 0; j < k; ++j)
        {
          std::swap(c[col * k + j], c[piv * k + j]);
          std::swap(a[col * k + j], a[piv * k + j]);
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
  std::vector<double> coef(k * k); // coef[j * k + m]: P_m in function j
  for (int j = 0; j < k; ++j)
    for (int m = 0; m < k; ++m)
      coef[j * k + m] = a[m * k + j];
  return coef;
}
} // namespace

int hermite_sign(int k, int j) { return j == k - 2 ? -1 : 1; }

Tables1D make_tables(int p, int basis)
{
  if (p < 1 || p > 10)
    fail(Code::invalid_argument, "dgx: supported degrees are 1..10");
  if (basis < 0 || basis > 2)
    fail(Code::invalid_argument, "RankOperator: unknown basis kind");
  if (basis == 2 && p < 3)
    fail(Code::invalid_argument, "RankOperator: the Hermite-type basis needs degree >= 3");
  const int k = p + 1;
  const Quad1D qg = gauss(k);
  Tables1D t;
  t.k = k;
  t.basis = basis;
  t.qw = qg.weights;
  t.S.resize(k * k);
  t.Dco.resize(k * k);
  t.D.resize(k * k);
  // basis function j: value and derivative at x
  std::vector<double> nodes, coef;
  if (basis == 0)
    nodes = gauss_lobatto(k).points;
  else if (basis == 1)
    nodes = qg.points;
  else
    coef = hermite_coefficients(k);
  std::vector<double> pv(k), dv(k);
  auto eval = [&](int j, double x, double &v, double &dvx) {
    if (basis != 2)
      {
        v = lagrange_value(nodes, j, x);
        dvx = lagrange_derivative(nodes, j, x);
        return;
      }
    // sign-flipped Hermite function psi_j = sigma_j phi_j, sigma_{k-2} = -1:
    // psi_{k-1-j}(x) = psi_j(1-x), so S, D admit the even-odd form
    shifted_legendre(k, x, pv.data(), dv.data());
    double s = 0.0, sd = 0.0;
    for (int m = 0; m < k; ++m)
      {
        s += coef[j * k + m] * pv[m];
        sd += coef[j * k + m] * dv[m];
      }
    v = hermite_sign(k, j) * s;
    dvx = hermite_sign(k, j) * sd;
  };
  for (int q = 0; q < k; ++q)
    for (int j = 0; j < k; ++j)
      {
        eval(j, qg.points[q], t.S[q * k + j], t.D[q * k + j]);
        t.Dco[q * k + j] = lagrange_derivative(qg.points, j, qg.points[q]);
      }
  mirror_roundtrip(t.S, k, false);
  mirror_roundtrip(t.Dco, k, true);
  mirror_roundtrip(t.D, k, true);
  for (int s = 0; s < 2; ++s)
    {
      const double x = s ? 1.0 : 0.0;
      t.Sf[s].resize(k);
      t.Df[s].resize(k);
      t.rf[s].resize(k);
      for (int j = 0; j < k; ++j)
        {
          eval(j, x, t.Sf[s][j], t.Df[s][j]);
          t.rf[s][j] = lagrange_value(qg.points, j, x);
        }
    }
  if (basis == 2)
    {
      // pinned by the interpolation conditions (basis.cpp:298-309), in the
      // sign-flipped functions
      for (int s = 0; s < 2; ++s)
        std::fill(t.Sf[s].begin(), t.Sf[s].end(), 0.0), std::fill(t.Df[s].begin(), t.Df[s].end(), 0.0);
      t.Sf[0][0] = 1.0;
      t.Df[0][1] = 1.0;
      t.Sf[1][k - 1] = 1.0;
      t.Df[1][k - 2] = hermite_sign(k, k - 2);
    }
  return t;
}

// ------------------------------------------------------------ mesh ------

void MeshDesc::check() const
{
  if (d != 2 && d != 3)
    fail(Code::invalid_argument, "mesh: dimension must be 2 or 3");
  for (int a = 0; a < d; ++a)
    {
      if (cells[a] < 1)
        fail(Code::invalid_argument, "mesh: need at least one cell");
      if (hi[a] <= lo[a])
        fail(Code::invalid_argument, "mesh: non-positive extent");
    }
  if (n_cells() >= (1ll << 31))
    fail(Code::invalid_argument, "mesh: cell count exceeds int32 indexing");
}

std::vector<RawFace> enumerate_faces(const MeshDesc &m)
{
  m.check();
  std::vector<RawFace> faces;
  const int d = m.d;
  const long long nc = m.n_cells();
  long long nf = 0;
  for (int a = 0; a < d; ++a)
    nf += nc + (m.periodic[a] ? 0 : nc / m.cells[a]);
  faces.reserve(nf);
  for (int a = 0; a < d; ++a)
    {
      const bool periodic = m.periodic[a];
      const int na = m.cells[a];
      long long stride = 1;
      for (int b = 0; b < a; ++b)
        stride *= m.cells[b];
      for (long long c = 0; c < nc; ++c)
        {
          const int ia = static_cast<int>((c / stride) % na);
          if (ia == 0 && !periodic)
            {
              RawFace f;
              f.interior_cell = static_cast<std::uint32_t>(c);
              f.interior_face_number = static_cast<std::uint8_t>(2 * a);
              f.exterior_face_number = static_cast<std::uint8_t>(m.dirichlet_id[2 * a]);
              faces.push_back(f);
            }
          if (ia == na - 1)
            {
              RawFace f;
              if (!periodic)
                {
                  f.interior_cell = static_cast<std::uint32_t>(c);
                  f.interior_face_number = static_cast<std::uint8_t>(2 * a + 1);
                  f.exterior_face_number =
                    static_cast<std::uint8_t>(m.dirichlet_id[2 * a + 1]);
                }
              else
                {
                  // wrap-around face: the low-side cell becomes e-
                  f.interior_cell = static_cast<std::uint32_t>(c - (long long)ia * stride);
                  f.exterior_cell = static_cast<std::uint32_t>(c);
                  f.interior_face_number = static_cast<std::uint8_t>(2 * a);
                  f.exterior_face_number = static_cast<std::uint8_t>(2 * a + 1);
                }
              faces.push_back(f);
            }
          else
            {
              RawFace f;
              f.interior_cell = static_cast<std::uint32_t>(c);
              f.exterior_cell = static_cast<std::uint32_t>(c + stride);
              f.interior_face_number = static_cast<std::uint8_t>(2 * a + 1);
              f.exterior_face_number = static_cast<std::uint8_t>(2 * a);
              faces.push_back(f);
            }
        }
    }
  return faces;
}

Partition make_partition(const MeshDesc &m, const std::vector<RawFace> &faces,
                         int n_ranks)
{
  const long long n = m.n_cells();
  if (n_ranks < 1 || n_ranks > n)
    fail(Code::invalid_argument, "partition_cells: rank count must be in [1, n_cells]");
  Partition p;
  p.n_ranks = n_ranks;
  p.cell_owner.resize(n);
  const long long base = n / n_ranks, extra = n % n_ranks;
  long long begin = 0;
  for (int r = 0; r < n_ranks; ++r)
    {
      const long long size = base + (r < extra ? 1 : 0);
      p.ranges.emplace_back(static_cast<int>(begin), static_cast<int>(begin + size));
      std::fill(p.cell_owner.begin() + begin, p.cell_owner.begin() + begin + size, r);
      begin += size;
    }
  assign_face_owners(faces, p);
  return p;
}

// assign_face_owners (mesh.cpp:157-232): interface faces split between the
// two ranks; a cell touching several interface faces sends all of them to
// the opposite rank so its data crosses only once.
void assign_face_owners(const std::vector<RawFace> &faces, Partition &part)
{
  part.face_owner.assign(faces.size(), -1);
  std::map<std::pair<int, int>, std::vector<std::size_t>> iface;
  for (std::size_t i = 0; i < faces.size(); ++i)
    {
      const RawFace &f = faces[i];
      const int ri = part.cell_owner[f.interior_cell];
      if (f.at_boundary())
        {
          part.face_owner[i] = ri;
          continue;
        }
      const int re = part.cell_owner[f.exterior_cell];
      if (ri == re)
        part.face_owner[i] = ri;
      else
        iface[{std::min(ri, re), std::max(ri, re)}].push_back(i);
    }
  for (auto &[pair, list] : iface)
    {
      const int ra = pair.first, rb = pair.second;
      std::map<std::uint32_t, int> mult;
      for (std::size_t i : list)
        {
          ++mult[faces[i].interior_cell];
          ++mult[faces[i].exterior_cell];
        }
      int count_a = 0, count_b = 0;
      auto assign = [&](std::size_t i, int r) {
        part.face_owner[i] = r;
        (r == ra ? count_a : count_b) += 1;
      };
      std::map<std::uint32_t, int> group;
      std::vector<std::size_t> singles;
      for (std::size_t i : list)
        {
          const RawFace &f = faces[i];
          const std::uint32_t ca =
            part.cell_owner[f.interior_cell] == ra ? f.interior_cell : f.exterior_cell;
          const std::uint32_t cb = ca == f.interior_cell ? f.exterior_cell : f.interior_cell;
          const int ma = mult[ca], mb = mult[cb];
          if (ma >= 2 && mb < 2)
            assign(i, rb);
          else if (mb >= 2 && ma < 2)
            assign(i, ra);
          else if (ma >= 2 && mb >= 2)
            {
              auto it = group.find(ca);
              if (it == group.end())
                it = group.emplace(ca, group.size() % 2 == 0 ? rb : ra).first;
              assign(i, it->second);
            }
          else
            singles.push_back(i);
        }
      for (std::size_t i : singles)
        assign(i, count_a <= count_b ? ra : rb);
    }
}

long long RankLayout::slot(std::uint32_t g) const
{
  if (g >= owned_begin && g < owned_begin + n_owned)
    return g - owned_begin;
  auto it = std::lower_bound(ghosts.begin(), ghosts.end(), g);
  if (it == ghosts.end() || *it != g)
    return -1;
  return (long long)n_owned + (it - ghosts.begin());
}

RankLayout build_layout(const MeshDesc &m, const std::vector<RawFace> &faces,
                        const Partition &p, int rank, int k, int basis, int kind)
{
  if (rank < 0 || rank >= p.n_ranks)
    fail(Code::invalid_argument, "build_dof_layout: rank out of range");
  RankLayout l;
  l.rank = rank;
  long long dpc = 1;
  for (int a = 0; a < m.d; ++a)
    dpc *= k;
  l.dofs_per_cell = dpc;
  l.owned_begin = static_cast<std::uint32_t>(p.ranges[rank].first);
  l.n_owned = static_cast<std::uint32_t>(p.ranges[rank].second - p.ranges[rank].first);
  if ((long long)(l.n_owned) * dpc >= (1ll << 32))
    fail(Code::invalid_argument, "layout: rank-local size exceeds uint32 indexing");
  // ghosts: every non-owned cell of a face this rank computes
  // (dof_layout.cpp:191-213)
  std::vector<std::uint32_t> g;
  for (std::uint32_t i = 0; i < faces.size(); ++i)
    {
      if (p.face_owner[i] != rank)
        continue;
      l.my_faces.push_back(i);
      for (std::uint32_t c : {faces[i].interior_cell, faces[i].exterior_cell})
        if (c != invalid_cell && p.cell_owner[c] != rank)
          g.push_back(c);
    }
  std::sort(g.begin(), g.end());
  g.erase(std::unique(g.begin(), g.end()), g.end());
  l.ghosts = g;
  for (std::uint32_t c : g)
    l.ghost_owner.push_back(p.cell_owner[c]);
  // exchange plans (ghost_exchange.cpp:100-144): one face side whose cell is
  // owned elsewhere than the face contributes that cell, with the dofs the
  // face evaluation reads (mark_face_dofs, :46-70): two layers next to the
  // face for the Hermite-like basis, the whole cell otherwise
  // one layer for values on a nodal basis, two for the Hermite-like basis,
  // the whole cell otherwise (mark_face_dofs, ghost_exchange.cpp:46-70)
  const int nl = basis == 2 ? 2 : (basis == 0 && kind == 1 ? 1 : 0);
  auto mark = [&](std::vector<char> &mask, int face_number) {
    if (mask.empty())
      mask.assign((size_t)dpc, 0);
    if (nl == 0)
      {
        std::fill(mask.begin(), mask.end(), 1);
        return;
      }
    const int axis = face_number / 2, side = face_number % 2;
    long long inner = 1;
    for (int a = 0; a < axis; ++a)
      inner *= k;
    for (long long j = 0; j < dpc; ++j)
      {
        const int ja = static_cast<int>((j / inner) % k);
        if (side == 0 ? ja < nl : ja >= k - nl)
          mask[j] = 1;
      }
  };
  std::map<int, std::map<std::uint32_t, std::vector<char>>> send, recv;
  for (std::size_t fid = 0; fid < faces.size(); ++fid)
    {
      const RawFace &f = faces[fid];
      const int w = p.face_owner[fid];
      const std::uint32_t cells[2] = {f.interior_cell, f.exterior_cell};
      const int fns[2] = {f.interior_face_number, f.exterior_face_number};
      for (int s = 0; s < (f.at_boundary() ? 1 : 2); ++s)
        {
          const int o = p.cell_owner[cells[s]];
          if (o == w)
            continue;
          if (o == rank)
            mark(send[w][cells[s]], fns[s]);
          else if (w == rank)
            mark(recv[o][cells[s]], fns[s]);
        }
    }
  for (auto *mp : {&send, &recv})
    for (auto &[nb, cm] : *mp)
      {
        NeighborPlan np;
        np.neighbor = nb;
        np.dof_offsets.push_back(0);
        for (auto &[c, mask] : cm)
          {
            np.cells.push_back(c);
            for (long long j = 0; j < dpc; ++j)
              if (mask[j])
                np.dofs.push_back(static_cast<std::uint32_t>(j));
            np.dof_offsets.push_back(static_cast<std::uint32_t>(np.dofs.size()));
            if (np.dof_offsets.back() - np.dof_offsets[np.dof_offsets.size() - 2] != dpc)
              l.whole_cells = false;
          }
        (mp == &send ? l.send : l.recv).push_back(std::move(np));
      }
  return l;
}

// ------------------------------------------------------ support points --

std::vector<double> reference_support(const MeshDesc &m,
                                      const std::vector<std::uint32_t> &cells)
{
  const int d = m.d, mm = m.mapping_degree;
  const std::vector<double> nodes = gauss_lobatto(mm + 1).points;
  long long pp = 1;
  for (int a = 0; a < d; ++a)
    pp *= mm + 1;
  std::vector<double> out(cells.size() * pp * d);
  double *o = out.data();
  for (std::uint32_t c : cells)
    {
      long long cc = c;
      int mi[3] = {0, 0, 0};
      for (int a = 0; a < d; ++a)
        {
          mi[a] = static_cast<int>(cc % m.cells[a]);
          cc /= m.cells[a];
        }
      for (long long s = 0; s < pp; ++s)
        {
          double xi[3] = {0, 0, 0};
          long long idx = s;
          for (int a = 0; a < d; ++a)
            {
              xi[a] = nodes[idx % (mm + 1)];
              idx /= (mm + 1);
            }
          double y[3] = {0, 0, 0};
          for (int a = 0; a < d; ++a)
            y[a] = (mi[a] + xi[a]) / m.cells[a];
          double bump = m.amplitude;
          for (int a = 0; a < d; ++a)
            bump *= std::sin(M_PI * y[a]);
          for (int a = 0; a < d; ++a)
            *o++ = m.lo[a] + (m.hi[a] - m.lo[a]) * (y[a] + bump);
        }
    }
  return out;
}

std::vector<double> vertex_bump_support(const MeshDesc &m, double eps,
                                        const std::vector<std::uint32_t> &cells)
{
  const int d = m.d, pp = 1 << d;
  std::vector<double> out(cells.size() * pp * d);
  double *o = out.data();
  for (std::uint32_t c : cells)
    {
      long long cc = c;
      int mi[3] = {0, 0, 0};
      for (int a = 0; a < d; ++a)
        {
          mi[a] = static_cast<int>(cc % m.cells[a]);
          cc /= m.cells[a];
        }
      for (int s = 0; s < pp; ++s)
        {
          double x[3];
          for (int a = 0; a < d; ++a)
            x[a] = m.lo[a] + (m.hi[a] - m.lo[a]) *
                               ((double)(mi[a] + ((s >> a) & 1)) / m.cells[a]);
          double bump = 1.0;
          for (int a = 0; a < d; ++a)
            bump *= std::sin(2.0 * M_PI * x[a]);
          for (int a = 0; a < d; ++a)
            *o++ = x[a] + eps * ((m.hi[a] - m.lo[a]) / m.cells[a]) * bump;
        }
    }
  return out;
}

} // namespace dgx

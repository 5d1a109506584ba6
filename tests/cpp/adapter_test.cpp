// The reference's own fixtures with the B200 operator swapped in:
// dgx_ref::RankOperator (include/dgx_rank_operator.hpp) against
// dg::RankOperator on SingleRankOp-style single-rank applies
// (proj/tests/test_operators.cpp:26-52) and on the threaded GhostExchanger
// transport (proj/tests/test_ghost_exchange.cpp:63-87). Exit 0 = all pass.
#include <dg/ghost_exchange.hpp>
#include <dg/operators.hpp>

#include <dgx_rank_operator.hpp>

#include <cmath>
#include <cstdio>
#include <random>

using namespace dg;

static std::vector<double> random_vector(std::size_t n, unsigned seed)
{
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  std::vector<double> v(n);
  for (auto &x : v)
    x = dist(rng);
  return v;
}

static double rel_linf(const std::vector<double> &a, const std::vector<double> &b)
{
  double diff = 0, scale = 0;
  for (std::size_t i = 0; i < a.size(); ++i)
    {
      diff = std::max(diff, std::abs(a[i] - b[i]));
      scale = std::max(scale, std::abs(b[i]));
    }
  return diff / std::max(scale, 1e-300);
}

template <typename Op>
static std::vector<double> distributed_apply(std::vector<std::unique_ptr<Op>> &ops,
                                             const std::vector<RawFace> &faces,
                                             const Partition &part, const OperatorConfig &cfg,
                                             const std::vector<double> &x)
{
  const int nr = static_cast<int>(ops.size());
  TransportHub hub(nr);
  std::vector<std::vector<double>> partial(nr, std::vector<double>(x.size(), 0.0));
  const FaceAccess access = make_basis(cfg.basis, cfg.p).face_access;
  run_ranks(nr, [&](int r) {
    GhostExchanger ex(build_exchange_plan(ops[r]->layout(), faces, part, access,
                                          ghost_need(cfg.kind)),
                      &ops[r]->layout(), &hub);
    ExchangeHooks hooks = ex.hooks();
    GhostedVector u = ops[r]->layout().make_vector();
    GhostedVector y = ops[r]->layout().make_vector();
    from_canonical(ops[r]->layout(), x, u);
    ops[r]->apply(u, y, nr > 1 ? &hooks : nullptr);
    to_canonical(ops[r]->layout(), y, partial[r]);
  });
  std::vector<double> out(x.size(), 0.0);
  for (int r = 0; r < nr; ++r)
    for (std::size_t i = 0; i < x.size(); ++i)
      out[i] += partial[r][i];
  return out;
}

// op: 0 Laplacian with the Gauss-Lobatto basis (BASELINE), 1 the reference
// default configuration (Hermite-like basis for p >= 3), 2 advection
static int run_case(int d, int cells, int p, double amp, bool periodic, int m, int nr, int op = 0)
{
  const Mesh mesh = make_box_mesh(d, cells, amp, periodic, m);
  OperatorConfig cfg = make_operator_config(op == 2 ? OperatorKind::advection : OperatorKind::laplacian,
                                            d, p, 1, GeometryVariant::g3);
  if (op == 0)
    cfg.basis = BasisKind::lagrange_gauss_lobatto;
  if (op == 2)
    cfg.velocity.constant = {0.85, -0.6, 0.35};
  const auto faces = enumerate_faces(mesh);
  Partition part = partition_cells(mesh, nr);
  assign_face_owners(mesh, faces, part);
  auto geom = std::make_shared<GeometryCache>(
    precompute_geometry(mesh, faces, cfg.k(), cfg.k(), cfg.geometry, cfg.equation(),
                        cfg.velocity));
  std::vector<std::unique_ptr<RankOperator>> ref;
  std::vector<std::unique_ptr<dgx_ref::RankOperator>> gpu;
  for (int r = 0; r < nr; ++r)
    {
      ref.push_back(std::make_unique<RankOperator>(mesh, part, faces, geom, cfg, r));
      gpu.push_back(std::make_unique<dgx_ref::RankOperator>(mesh, part, faces, geom, cfg, r));
    }
  const long long n = static_cast<long long>(mesh.n_cells()) * ref[0]->layout().dofs_per_cell;
  const auto x = random_vector(n, 1234 + p + 7 * d);
  const auto y_ref = distributed_apply(ref, faces, part, cfg, x);
  const auto y_gpu = distributed_apply(gpu, faces, part, cfg, x);
  const double err = rel_linf(y_gpu, y_ref);
  const bool ok = err < 1e-12;
  std::printf("%s op=%d d=%d cells=%d p=%d amp=%.2f periodic=%d m=%d ranks=%d rel_linf=%.2e\n",
              ok ? "PASS" : "FAIL", op, d, cells, p, amp, periodic, m, nr, err);
  // a ghosted layout without hooks is a logic error (operators.cpp:238-240)
  if (nr > 1)
    {
      GhostedVector u = gpu[0]->layout().make_vector(), y = gpu[0]->layout().make_vector();
      bool threw = false;
      try
        {
          gpu[0]->apply(u, y);
        }
      catch (const std::logic_error &)
        {
          threw = true;
        }
      std::printf("%s ghosted layout without hooks throws std::logic_error\n",
                  threw ? "PASS" : "FAIL");
      if (!threw)
        return 1;
    }
  return ok ? 0 : 1;
}

int main()
{
  int fails = 0;
  fails += run_case(2, 3, 3, 0.07, false, 3, 1);
  fails += run_case(3, 2, 3, 0.05, false, 2, 1);
  fails += run_case(3, 4, 4, 0.0, true, 1, 1);
  fails += run_case(2, 4, 2, 0.05, true, 2, 2);
  fails += run_case(2, 5, 5, 0.04, false, 2, 4);
  fails += run_case(3, 3, 3, 0.06, false, 3, 3);
  fails += run_case(3, 3, 5, 0.05, false, 2, 3, 1); // reference default: Hermite-like
  fails += run_case(2, 5, 4, 0.04, true, 2, 2, 1);
  fails += run_case(3, 3, 3, 0.05, false, 2, 3, 2); // advection
  fails += run_case(2, 6, 5, 0.0, true, 1, 2, 2);
  std::printf("%s\n", fails ? "FAILED" : "ALL PASS");
  return fails ? 1 : 0;
}

// extern "C" entry points of include/dgx.h. Exceptions never cross the ABI:
// they are mapped onto dgx_status codes (reference exception classes) and
// the message is kept per thread for dgx_last_error().
#include "../../include/dgx.h"
#include "nccl_exchange.hpp"
#include "operator.hpp"

#include <cstring>
#include <random>
#include <string>

struct dgx_op
{
  std::unique_ptr<dgx::Operator> impl;
};
struct dgx_exchanger
{
  std::unique_ptr<dgx::Exchanger> impl;
};

namespace
{
thread_local std::string g_err;

template <typename F>
dgx_status guard(F &&f)
{
  try
    {
      f();
      return DGX_OK;
    }
  catch (const dgx::Error &e)
    {
      g_err = e.what();
      return static_cast<dgx_status>(e.code);
    }
  catch (const std::invalid_argument &e)
    {
      g_err = e.what();
      return DGX_INVALID_ARGUMENT;
    }
  catch (const std::logic_error &e)
    {
      g_err = e.what();
      return DGX_LOGIC_ERROR;
    }
  catch (const std::exception &e)
    {
      g_err = e.what();
      return DGX_RUNTIME_ERROR;
    }
  catch (...)
    {
      g_err = "unknown error";
      return DGX_RUNTIME_ERROR;
    }
}

dgx::MeshDesc mesh_desc(const dgx_mesh *m)
{
  if (!m)
    dgx::fail(dgx::Code::invalid_argument, "null mesh");
  dgx::MeshDesc md;
  md.d = m->d;
  for (int a = 0; a < 3; ++a)
    {
      md.cells[a] = a < m->d ? m->cells_per_dim[a] : 1;
      md.lo[a] = m->lo[a];
      md.hi[a] = m->hi[a];
      md.periodic[a] = m->periodic[a] != 0;
    }
  md.amplitude = m->deform_amplitude;
  md.mapping_degree = m->mapping_degree < 1 ? 1 : m->mapping_degree;
  for (int s = 0; s < 6; ++s)
    md.dirichlet_id[s] = m->dirichlet_id[s];
  md.check();
  return md;
}

dgx::Operator &op_of(const dgx_op *op)
{
  if (!op || !op->impl)
    dgx::fail(dgx::Code::invalid_argument, "null operator");
  return *op->impl;
}
} // namespace

namespace dgx
{
void set_last_error(const char *msg) { g_err = msg ? msg : ""; }
} // namespace dgx

extern "C" {

const char *dgx_last_error(void) { return g_err.c_str(); }
const char *dgx_version(void)
{
  return "dgx 0.2 (sm_100a, fp64/fp32, GL / Gauss / Hermite-like bases, g3)";
}

dgx_status dgx_enumerate_faces(const dgx_mesh *mesh, dgx_raw_face *faces, int64_t *n_faces)
{
  return guard([&] {
    const auto f = dgx::enumerate_faces(mesh_desc(mesh));
    if (n_faces)
      *n_faces = static_cast<int64_t>(f.size());
    if (faces)
      std::memcpy(faces, f.data(), sizeof(dgx_raw_face) * f.size());
  });
}

dgx_status dgx_partition(const dgx_mesh *mesh, const dgx_raw_face *faces, int64_t n_faces,
                         int n_ranks, int *cell_owner, int *rank_cell_range, int *face_owner)
{
  return guard([&] {
    const dgx::MeshDesc md = mesh_desc(mesh);
    std::vector<dgx::RawFace> f(n_faces);
    if (n_faces > 0)
      std::memcpy(f.data(), faces, sizeof(dgx_raw_face) * n_faces);
    const dgx::Partition p = dgx::make_partition(md, f, n_ranks);
    if (cell_owner)
      std::memcpy(cell_owner, p.cell_owner.data(), sizeof(int) * p.cell_owner.size());
    if (rank_cell_range)
      for (int r = 0; r < n_ranks; ++r)
        {
          rank_cell_range[2 * r] = p.ranges[r].first;
          rank_cell_range[2 * r + 1] = p.ranges[r].second;
        }
    if (face_owner)
      std::memcpy(face_owner, p.face_owner.data(), sizeof(int) * p.face_owner.size());
  });
}

dgx_status dgx_create(const dgx_setup *setup, int device, dgx_op **op)
{
  return guard([&] {
    if (!setup || !op)
      dgx::fail(dgx::Code::invalid_argument, "dgx_create: null argument");
    auto o = std::make_unique<dgx_op>();
    o->impl = std::make_unique<dgx::Operator>(*setup, device);
    *op = o.release();
  });
}

dgx_status dgx_destroy(dgx_op *op)
{
  return guard([&] { delete op; });
}

dgx_status dgx_get_layout(const dgx_op *op, dgx_layout *out)
{
  return guard([&] {
    const dgx::RankLayout &l = op_of(op).layout();
    out->owned_cell_begin = l.owned_begin;
    out->n_owned_cells = l.n_owned;
    out->n_ghost_cells = (int64_t)l.ghosts.size();
    out->dofs_per_cell = l.dofs_per_cell;
    out->owned_size = l.owned_size();
    out->total_size = l.total_size();
  });
}

dgx_status dgx_get_ghost_cells(const dgx_op *op, uint32_t *cells, int *owners)
{
  return guard([&] {
    const dgx::RankLayout &l = op_of(op).layout();
    for (std::size_t i = 0; i < l.ghosts.size(); ++i)
      {
        if (cells)
          cells[i] = l.ghosts[i];
        if (owners)
          owners[i] = l.ghost_owner[i];
      }
  });
}

dgx_status dgx_get_plan(const dgx_op *op, int which, int idx, int *n_plans, int *neighbor,
                        int64_t *n_cells, uint32_t *cells)
{
  return guard([&] {
    const dgx::RankLayout &l = op_of(op).layout();
    const auto &v = which == 0 ? l.send : l.recv;
    if (n_plans)
      *n_plans = (int)v.size();
    if (idx < 0)
      return;
    if (idx >= (int)v.size())
      dgx::fail(dgx::Code::invalid_argument, "dgx_get_plan: index out of range");
    if (neighbor)
      *neighbor = v[idx].neighbor;
    if (n_cells)
      *n_cells = (int64_t)v[idx].cells.size();
    if (cells)
      std::memcpy(cells, v[idx].cells.data(), 4 * v[idx].cells.size());
  });
}

dgx_status dgx_get_plan_dofs(const dgx_op *op, int which, int idx, uint32_t *dof_offsets,
                             int64_t *n_dofs, uint32_t *dofs)
{
  return guard([&] {
    const dgx::RankLayout &l = op_of(op).layout();
    const auto &v = which == 0 ? l.send : l.recv;
    if (idx < 0 || idx >= (int)v.size())
      dgx::fail(dgx::Code::invalid_argument, "dgx_get_plan_dofs: index out of range");
    const dgx::NeighborPlan &np = v[idx];
    if (n_dofs)
      *n_dofs = (int64_t)np.dofs.size();
    if (dof_offsets)
      std::memcpy(dof_offsets, np.dof_offsets.data(), 4 * np.dof_offsets.size());
    if (dofs)
      std::memcpy(dofs, np.dofs.data(), 4 * np.dofs.size());
  });
}

dgx_status dgx_apply(dgx_op *op, double *u, double *y, const dgx_hooks *hooks, void *stream)
{
  return guard([&] {
    op_of(op).apply(u, y, hooks, static_cast<cudaStream_t>(stream), false);
  });
}

dgx_status dgx_apply_f32(dgx_op *op, float *u, float *y, const dgx_hooks *hooks, void *stream)
{
  return guard([&] {
    op_of(op).apply(u, y, hooks, static_cast<cudaStream_t>(stream), true);
  });
}

dgx_status dgx_apply_host(dgx_op *op, const double *u, double *y)
{
  return guard([&] {
    op_of(op).apply_host(u, y);
  });
}

dgx_status dgx_apply_phase(dgx_op *op, int phase, const void *u, void *y, void *stream)
{
  return guard([&] {
    dgx::Operator &o = op_of(op);
    o.apply_phase(phase, u, y, static_cast<cudaStream_t>(stream), o.precision() == 1);
  });
}

dgx_status dgx_accumulate_plan(dgx_op *op, int idx, const double *contrib, double *y,
                               void *stream)
{
  return guard([&] {
    op_of(op).accumulate_plan(idx, contrib, y, static_cast<cudaStream_t>(stream));
  });
}

dgx_status dgx_get_quadrature_points(dgx_op *op, int which, double *out, int64_t *n)
{
  return guard([&] {
    const std::vector<double> v = op_of(op).quadrature_points(which);
    if (n)
      *n = (int64_t)v.size();
    if (out)
      std::memcpy(out, v.data(), 8 * v.size());
  });
}

dgx_status dgx_set_velocity(dgx_op *op, const double *c_cells, const double *c_faces,
                            void *stream)
{
  return guard([&] {
    op_of(op).set_velocity(c_cells, c_faces, static_cast<cudaStream_t>(stream));
  });
}

dgx_status dgx_assemble_rhs(dgx_op *op, const double *f, const double *g, double *rhs,
                            void *stream)
{
  return guard([&] {
    op_of(op).assemble_rhs(f, g, rhs, static_cast<cudaStream_t>(stream));
  });
}

dgx_status dgx_conjugate_gradient(dgx_op *op, const double *b, double *x, double rel_tol,
                                  int max_iterations, dgx_solve_report *report, void *stream)
{
  return guard([&] {
    const dgx_solve_report r = dgx::conjugate_gradient(op_of(op), b, x, rel_tol, max_iterations,
                                                       static_cast<cudaStream_t>(stream));
    if (report)
      *report = r;
  });
}

dgx_status dgx_nccl_unique_id(void *id128)
{
  return guard([&] { dgx::nccl_unique_id(id128); });
}

dgx_status dgx_exchanger_create(dgx_op *op, const void *id128, dgx_exchanger **ex)
{
  return guard([&] {
    dgx::Operator &o = op_of(op);
    if (!id128 || !ex)
      dgx::fail(dgx::Code::invalid_argument, "dgx_exchanger_create: null argument");
    auto e = std::make_unique<dgx_exchanger>();
    e->impl = std::make_unique<dgx::Exchanger>(
      &o, dgx::make_nccl_transport(id128, o.n_ranks(), o.layout().rank));
    *ex = e.release();
  });
}

struct dgx_loopback
{
  std::shared_ptr<dgx::LoopbackWorld> world;
};

dgx_status dgx_loopback_create(int n_ranks, dgx_loopback **world)
{
  return guard([&] {
    if (!world)
      dgx::fail(dgx::Code::invalid_argument, "dgx_loopback_create: null argument");
    auto w = std::make_unique<dgx_loopback>();
    w->world = dgx::make_loopback_world(n_ranks);
    *world = w.release();
  });
}

dgx_status dgx_loopback_destroy(dgx_loopback *world)
{
  return guard([&] { delete world; });
}

dgx_status dgx_exchanger_create_loopback(dgx_op *op, dgx_loopback *world, dgx_exchanger **ex)
{
  return guard([&] {
    dgx::Operator &o = op_of(op);
    if (!world || !ex)
      dgx::fail(dgx::Code::invalid_argument, "dgx_exchanger_create_loopback: null argument");
    auto e = std::make_unique<dgx_exchanger>();
    e->impl = std::make_unique<dgx::Exchanger>(&o, dgx::make_loopback_transport(world->world, o.layout().rank));
    *ex = e.release();
  });
}

dgx_status dgx_exchanger_hooks(dgx_exchanger *ex, dgx_hooks *hooks)
{
  return guard([&] {
    if (!ex || !hooks)
      dgx::fail(dgx::Code::invalid_argument, "null exchanger");
    *hooks = ex->impl->hooks();
  });
}

dgx_status dgx_exchanger_destroy(dgx_exchanger *ex)
{
  return guard([&] { delete ex; });
}

dgx_status dgx_get_geometry(const dgx_op *op, int which, double *out, int64_t *n)
{
  return guard([&] {
    const std::vector<double> v = op_of(op).geometry(which);
    if (n)
      *n = (int64_t)v.size();
    if (out)
      std::memcpy(out, v.data(), 8 * v.size());
  });
}

dgx_status dgx_get_tasks(const dgx_op *op, int64_t *n_tasks, int64_t *n_inner, int *slot,
                         int *geo, int *face_entries)
{
  return guard([&] {
    const dgx::Operator &o = op_of(op);
    if (n_tasks)
      *n_tasks = (int64_t)o.host_task_slot().size();
    if (n_inner)
      *n_inner = o.n_inner();
    if (slot)
      std::memcpy(slot, o.host_task_slot().data(), 4 * o.host_task_slot().size());
    if (geo)
      std::memcpy(geo, o.host_task_geo().data(), 4 * o.host_task_geo().size());
    if (face_entries)
      std::memcpy(face_entries, o.host_task_face().data(), 8 * o.host_task_face().size());
  });
}

dgx_status dgx_get_stats(const dgx_op *op, dgx_stats *out)
{
  return guard([&] { *out = op_of(op).stats(); });
}

dgx_status dgx_random_uniform(double *out, int64_t n, uint32_t seed)
{
  return guard([&] {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (int64_t i = 0; i < n; ++i)
      out[i] = dist(rng);
  });
}

} // extern "C"

/* dgx.h -- C ABI of the B200-native matrix-free SIPG-Laplacian apply.
 *
 * Drop-in boundary for the reference operator path (arXiv 1711.03590 CPU
 * reference, /root/reference/proj). Every entry point cites the reference
 * interface it replaces (paths relative to proj/). Plain pointers and sizes
 * only; no torch or CUDA types in the signatures (streams are void*).
 *
 * Status codes map 1:1 onto the reference's exception classes
 * (SURVEY.md s.8b): DGX_INVALID_ARGUMENT <-> std::invalid_argument,
 * DGX_LOGIC_ERROR <-> std::logic_error, DGX_RUNTIME_ERROR <->
 * std::runtime_error. dgx_last_error() returns the message of the last
 * failure on the calling thread.
 *
 * Vector layout: the reference rank-local layout with W = 1
 * (dof_layout.cpp:50-65,170-253): owned cells cell-major (k^d dofs each,
 * lexicographic, axis 0 fastest), then the ghost cells in ascending global
 * id. Single rank: canonical cell-major numbering. Indices are uint32 as in
 * the reference (dof_layout.hpp:46-50).
 */
#ifndef DGX_H
#define DGX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dgx_status
{
  DGX_OK = 0,
  DGX_INVALID_ARGUMENT = 1,
  DGX_LOGIC_ERROR = 2,
  DGX_RUNTIME_ERROR = 3,
  DGX_CUDA_ERROR = 4
} dgx_status;

/* Replaces dg::RawFace (include/dg/mesh.hpp:80-93); identical 12-byte layout
 * so a std::vector<dg::RawFace>::data() can be passed unchanged. */
typedef struct dgx_raw_face
{
  uint32_t interior_cell;
  uint32_t exterior_cell; /* 0xffffffff on the boundary */
  uint8_t interior_face_number;
  uint8_t exterior_face_number; /* boundary id on boundary faces */
  uint8_t subface_index;
  uint8_t face_orientation;
} dgx_raw_face;

/* Replaces dg::Mesh (include/dg/mesh.hpp:24-60) + dg::BoundarySpec. */
typedef struct dgx_mesh
{
  int d;
  int cells_per_dim[3];
  double lo[3], hi[3];
  double deform_amplitude; /* x = y + a prod sin(pi y_i), mesh.cpp:11-26 */
  int mapping_degree;
  int periodic[3];
  int dirichlet_id[6];
} dgx_mesh;

const char *dgx_last_error(void);
const char *dgx_version(void);

/* ---- mesh topology, bit-exact with the reference ------------------------ */

/* Replaces dg::enumerate_faces (mesh.hpp:97, mesh.cpp:70-132). faces may be
 * NULL to query the count. */
dgx_status dgx_enumerate_faces(const dgx_mesh *mesh, dgx_raw_face *faces,
                               int64_t *n_faces);

/* Replaces dg::partition_cells + dg::assign_face_owners (mesh.hpp:102-118,
 * mesh.cpp:134-232). cell_owner: n_cells; rank_cell_range: 2*n_ranks
 * [begin,end); face_owner: n_faces. */
dgx_status dgx_partition(const dgx_mesh *mesh, const dgx_raw_face *faces,
                         int64_t n_faces, int n_ranks, int *cell_owner,
                         int *rank_cell_range, int *face_owner);

/* ---- operator ----------------------------------------------------------- */

typedef enum dgx_geometry_source
{
  /* deformation of the reference mesh (Mesh::map_point, mesh.cpp:11-26),
   * mapping of degree mesh.mapping_degree, precomputed on the device */
  DGX_GEOMETRY_MESH = 0,
  /* BASELINE.json vertex deformation x + eps h prod_a sin(2 pi x_a), cells
   * trilinear between their displaced vertices (mapping degree 1) */
  DGX_GEOMETRY_VERTEX_BUMP = 1,
  /* caller-supplied mapping support points [n_cells][(m+1)^d][d] on the
   * Gauss-Lobatto nodes of degree m (dg::MappingEval, geometry.hpp:62-76) */
  DGX_GEOMETRY_SUPPORT = 2,
  /* the reference GeometryCache arrays (geometry.hpp:94-147), variant g3 */
  DGX_GEOMETRY_HOST_ARRAYS = 3
} dgx_geometry_source;

typedef struct dgx_geometry
{
  int source;      /* dgx_geometry_source */
  int coefficient; /* 0: none; 1: a(x) = 1 + 0.5 sin(pi x) cos(pi y) folded
                      into JxW, n.J^{-T} and the penalty */
  double vertex_bump_eps;        /* VERTEX_BUMP */
  const double *support_points;  /* SUPPORT */
  int support_degree;            /* SUPPORT: m */
  int cartesian;                 /* SUPPORT: compress to one record per cell */
  int compressed;                /* HOST_ARRAYS: GeometryCache::compressed() */
  const double *inv_jac_t, *jxw; /* HOST_ARRAYS, [cell][q][d*d], [cell][q] */
  const double *face_jxw, *face_jni, *face_jne, *penalty; /* HOST_ARRAYS */
  const double *face_normal; /* HOST_ARRAYS, advection: GeometryCache::face_normal
                                [face][qf][d] */
  const double *coeff;       /* HOST_ARRAYS, g4: GeometryCache::coeff [cell][q][d(d+1)/2] */
} dgx_geometry;

/* Replaces dg::OperatorConfig (operators.hpp:26-51) for this path: the
 * Laplacian, the nodal Gauss-Lobatto basis, k = p+1 Gauss points, g3. */
typedef struct dgx_config
{
  int d;
  int p;                /* 1..10 */
  int W;                /* accepted for API parity; the layout is W = 1 */
  int basis;            /* BasisKind (basis.hpp:10-15): 0 lagrange_gauss_lobatto,
                           1 lagrange_gauss, 2 hermite_like (p >= 3; the
                           reference default for the Laplacian at p >= 3,
                           make_operator_config, operators.cpp:27-41) */
  int geometry_variant; /* 3: g3 (J^{-T} and JxW per point), 4: g4 (the merged
                           coefficient J^{-1}J^{-T} det(J) w, geometry.cpp:219-246,
                           370-388); others rejected */
  int precision;        /* 0: fp64, 1: fp32 */
  int kind;             /* OperatorKind: 0 laplacian, 1 advection (fp64, nodal or
                           Lagrange-Gauss basis) */
  double velocity[3];   /* advection: VelocityField::constant */
  int variable_velocity; /* advection: 1 = VelocityField::field, values given per
                            quadrature point by dgx_set_velocity (no Cartesian
                            compression, geometry.cpp:267-271) */
} dgx_config;

/* Replaces the RankOperator constructor arguments (operators.hpp:72-75):
 * (Mesh, Partition, faces, GeometryCache, OperatorConfig, rank). */
typedef struct dgx_setup
{
  dgx_mesh mesh;
  const dgx_raw_face *faces; /* enumerate_faces order */
  int64_t n_faces;
  int n_ranks;
  const int *cell_owner;      /* dg::Partition::cell_owner */
  const int *rank_cell_range; /* 2*n_ranks */
  const int *face_owner;
  int rank;
  dgx_config config;
  dgx_geometry geometry;
} dgx_setup;

typedef struct dgx_op dgx_op;

/* Replaces RankOperator::RankOperator (operators.hpp:72-75,
 * operators.cpp:89-198, 1202-1209). Builds the layout, the task lists and
 * the device geometry on `device`. device < 0 builds a host-only operator
 * (layout, plans and task lists; no GPU needed, apply is refused). */
dgx_status dgx_create(const dgx_setup *setup, int device, dgx_op **op);
dgx_status dgx_destroy(dgx_op *op);

/* Replaces RankOperator::layout() (operators.hpp:79; DoFLayout,
 * dof_layout.hpp:110-155). */
typedef struct dgx_layout
{
  int64_t owned_cell_begin, n_owned_cells, n_ghost_cells;
  int64_t dofs_per_cell, owned_size, total_size;
} dgx_layout;
dgx_status dgx_get_layout(const dgx_op *op, dgx_layout *out);
/* DoFLayout::ghost_global_cells / ghost_owner (dof_layout.hpp:124-125) */
dgx_status dgx_get_ghost_cells(const dgx_op *op, uint32_t *cells, int *owners);
/* ExchangePlan send (which=0) / recv (which=1) neighbour plans
 * (ghost_exchange.hpp:29-52): neighbour and ascending cells. */
dgx_status dgx_get_plan(const dgx_op *op, int which, int idx, int *n_plans,
                        int *neighbor, int64_t *n_cells, uint32_t *cells);
/* NeighborPlan::dof_offsets (n_cells + 1) and dofs (cell-local, ascending per
 * cell) of plan idx (build_exchange_plan, ghost_exchange.cpp:100-144): whole
 * cells for the nodal / generic bases, the two layers next to every coupled
 * face for hermite_like. Pass NULL arrays to query n_dofs. */
dgx_status dgx_get_plan_dofs(const dgx_op *op, int which, int idx, uint32_t *dof_offsets,
                             int64_t *n_dofs, uint32_t *dofs);

/* Physical quadrature points of the operator's mapping (the reference
 * evaluates forcing and Dirichlet data there, operators.cpp:545-560,
 * 1115-1145; unavailable for DGX_GEOMETRY_HOST_ARRAYS): which 0: owned cells
 * [cell][q][d] (q lexicographic, axis 0 fastest); 1: the faces this rank
 * computes [face][qf][d] (GeometryCache::face_qpoints order, dgx_get_geometry
 * which=3 gives their global ids); 2: boundary flag (0/1) per computed face.
 * Pass out=NULL to query n. */
dgx_status dgx_get_quadrature_points(dgx_op *op, int which, double *out, int64_t *n);
/* Advection with a variable velocity: c at the owned cells' quadrature points
 * [cell][q][d] and at the computed faces' quadrature points [face][qf][d]
 * (device arrays, dgx_get_quadrature_points order); replaces the field
 * evaluation of load_cell_geometry / load_face_geometry (operators.cpp:
 * 397-545). Also accepted for a constant velocity config (overrides it). */
dgx_status dgx_set_velocity(dgx_op *op, const double *c_cells, const double *c_faces,
                            void *stream);
/* RankOperator::assemble_rhs (operators.cpp:266-282): rhs = forcing
 * (f det(J) w_q tested with the basis, :1115-1145) + the Dirichlet data moved
 * to the right-hand side by the boundary faces (:1033-1111). f: device
 * [owned cell][q] values f(x_q), g: device [computed face][qf] values g(x_qf)
 * (only boundary faces are read); either may be NULL (zero). rhs: device,
 * layout total_size, overwritten; the ghost region is zero. fp64 only. */
dgx_status dgx_assemble_rhs(dgx_op *op, const double *f, const double *g, double *rhs,
                            void *stream);

/* Replaces dg::ExchangeHooks (operators.hpp:61-66). Each hook receives the
 * device vector and the stream of the apply; it must leave its work ordered
 * on that stream. */
typedef dgx_status (*dgx_hook_fn)(void *ctx, void *vector, void *stream);
typedef struct dgx_hooks
{
  void *ctx;
  dgx_hook_fn start_ghost_update;
  dgx_hook_fn finish_ghost_update;
  dgx_hook_fn compress;
} dgx_hooks;

/* Replaces RankOperator::apply (operators.hpp:85-86, operators.cpp:217-264):
 * y = A u. u, y: device pointers of layout.total_size values each (u's ghost
 * region is written by the update hooks). Without hooks the layout must
 * have no ghosts (DGX_LOGIC_ERROR otherwise, operators.cpp:238-240). On
 * return without a compress hook, y's ghost region holds the contributions
 * to remote cells; with one, y is clean and its ghost region zero. */
dgx_status dgx_apply(dgx_op *op, double *u, double *y, const dgx_hooks *hooks,
                     void *stream);
/* fp32 variant (config.precision = 1). */
dgx_status dgx_apply_f32(dgx_op *op, float *u, float *y, const dgx_hooks *hooks,
                         void *stream);
/* Host pointers (layout.total_size values each): H2D, apply, D2H. For a
 * ghosted layout u's ghost region must already hold the neighbour values
 * (the caller ran its update) and y returns with the contributions to remote
 * cells in its ghost region (the caller compresses), i.e. the state between
 * finish_ghost_update and compress of operators.cpp:245-262. */
dgx_status dgx_apply_host(dgx_op *op, const double *u, double *y);

/* Split phases for external transports (the two loops of
 * operators.cpp:245-258): phase 1 = cells none of whose computed faces
 * read ghosts; phase 2 = ghost-coupled cells plus the ghost-side residuals
 * written into y's ghost region. */
dgx_status dgx_apply_phase(dgx_op *op, int phase, const void *u, void *y,
                           void *stream);

/* Compress accumulation for external transports (ghost_exchange.cpp:
 * 376-395): y[owned cells of send plan idx] += contributions (plan order). */
dgx_status dgx_accumulate_plan(dgx_op *op, int idx, const double *contrib,
                               double *y, void *stream);

/* ---- solver around the apply (caller of RankOperator::apply) ------------ */

/* Replaces dg::SolveReport (solvers.hpp:17-22). */
typedef struct dgx_solve_report
{
  int converged;
  int iterations;
  double relative_residual;
} dgx_solve_report;

/* Replaces conjugate_gradient(make_apply(op), b, x, rel_tol, max_iterations)
 * (solvers.cpp:24-68,189-206) on the device: b, x device pointers of
 * layout.owned_size values; single-rank operators only (make_apply's
 * contract, DGX_INVALID_ARGUMENT otherwise); a non-positive p.Ap raises
 * DGX_RUNTIME_ERROR as the reference does. */
dgx_status dgx_conjugate_gradient(dgx_op *op, const double *b, double *x, double rel_tol,
                                  int max_iterations, dgx_solve_report *report, void *stream);

/* ---- native exchanger (replaces GhostExchanger, ghost_exchange.hpp:96-128,
 * update_ghost_values / compress ghost_exchange.cpp:300-398) ---------------
 * Pack, in-place ghost receives, compress and the ascending-rank
 * accumulation run on the device over a transport: NCCL send/recv between
 * the GPUs of one box (one process per GPU), or an in-process loopback
 * (R rank operators in one process -- one host thread per rank calling
 * dgx_apply -- whose messages become cudaMemcpyAsync between the ranks'
 * device buffers; the reference's run_ranks + in-process queues,
 * ghost_exchange.cpp:409-430). dgx_apply with an exchanger's hooks
 * overlaps the exchange with the inner cells: the ghost-coupled cells run
 * on a high-priority stream as soon as the update lands and their
 * contributions are sent back while the inner cells still run. */
typedef struct dgx_exchanger dgx_exchanger;
typedef struct dgx_loopback dgx_loopback;
dgx_status dgx_nccl_unique_id(void *id128);
dgx_status dgx_exchanger_create(dgx_op *op, const void *nccl_id128,
                                dgx_exchanger **ex);
dgx_status dgx_loopback_create(int n_ranks, dgx_loopback **world);
dgx_status dgx_loopback_destroy(dgx_loopback *world);
dgx_status dgx_exchanger_create_loopback(dgx_op *op, dgx_loopback *world,
                                         dgx_exchanger **ex);
dgx_status dgx_exchanger_hooks(dgx_exchanger *ex, dgx_hooks *hooks);
dgx_status dgx_exchanger_destroy(dgx_exchanger *ex);

/* ---- introspection ------------------------------------------------------ */

/* Device geometry in the device layout: which 0 cell records
 * [cell][d*d+1][k^d | 1], 1 face records [face][2d+1][k^{d-1}], 2 penalty,
 * 3 face ids (int64 as double) of the face records. out may be NULL. */
dgx_status dgx_get_geometry(const dgx_op *op, int which, double *out, int64_t *n);

/* Cell task lists (host copy): slot, cell-geometry record (-1: ghost-side
 * task), and 2d int2 face entries per task (x: neighbour slot | -1 boundary
 * | -2 not computed here; y: face record | own side << 30). Tasks
 * [0, n_inner) form phase 1. Arrays may be NULL to query the counts. */
dgx_status dgx_get_tasks(const dgx_op *op, int64_t *n_tasks, int64_t *n_inner,
                         int *slot, int *geo, int *face_entries);

typedef struct dgx_stats
{
  int64_t n_tasks_inner, n_tasks_coupled, n_faces;
  int64_t kernel_launches_per_apply;
  double bytes_vectors, bytes_cell_geometry, bytes_face_geometry; /* per apply */
  int cells_per_cta, threads_per_cta;
  int cartesian; /* axis-aligned affine records: 2 the tensor-product kernel runs,
                    1 the collocation CART kernels (DGX_NO_TENSOR set at creation) */
} dgx_stats;
dgx_status dgx_get_stats(const dgx_op *op, dgx_stats *out);

/* std::mt19937(seed) + uniform_real_distribution<double>(-1,1), the
 * reference input convention (tests/test_helpers.hpp:11-19). */
dgx_status dgx_random_uniform(double *out, int64_t n, uint32_t seed);

#ifdef __cplusplus
}
#endif
#endif /* DGX_H */

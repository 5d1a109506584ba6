/* CPU restatement of the reference SIPG-Laplacian apply path (TEST
 * INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the checker; never linked by the product).
 *
 * Plain C, fp64, scalar. Every function cites the reference file:line it
 * restates (paths relative to /root/reference/proj). Parity of this
 * restatement is pinned against the reference itself (oracle/_ref/libdgref.so
 * built from the unmodified sources) and the golden fixtures under
 * tests/golden/ that the reference generated (tests/golden/make_golden.py).
 *
 * Conventions: canonical numbering = cell * k^d + lexicographic local index
 * (axis 0 fastest), operators.hpp:108-114. Indices uint32 (dof_layout.hpp:46),
 * counts int64.
 */
#ifndef DGORACLE_H
#define DGORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char *dgo_last_error(void);

/* std::mt19937(seed) + std::uniform_real_distribution<double>(-1,1) as
 * libstdc++ implements it (tests/test_helpers.hpp:11-19). */
int dgo_random_vector(int64_t n, uint32_t seed, double *out);

/* quadrature.cpp:56-127 */
int dgo_gauss(int n, int lobatto, double *points, double *weights);

/* Shape matrices on k = p+1 Gauss points: basis.cpp:116-180,182-325.
 * basis: 0 lagrange_gauss_lobatto, 1 lagrange_gauss, 2 hermite_like.
 * S, D, Dco: k*k row-major (quadrature index = row); Sf, Df: 2*k. */
int dgo_shape(int p, int basis, double *S, double *D, double *Dco, double *Sf,
              double *Df);

/* enumerate_faces, mesh.cpp:70-132. n_faces first (pass NULL arrays). */
int64_t dgo_faces(int d, const int *cells, int periodic, uint32_t *interior,
                  uint32_t *exterior, uint8_t *fn_int, uint8_t *fn_ext);

/* partition_cells, mesh.cpp:134-155; ranges: 2*n_ranks [begin,end). */
int dgo_partition(int n_cells, int n_ranks, int *cell_owner, int *ranges);

/* assign_face_owners, mesh.cpp:157-232. */
int dgo_face_owners(int64_t n_faces, const uint32_t *interior,
                    const uint32_t *exterior, const int *cell_owner,
                    int *face_owner);

/* Ghost cells of one rank, ascending (dof_layout.cpp:191-213). Returns the
 * count; ghosts may be NULL to query. */
int64_t dgo_ghosts(int rank, int64_t n_faces, const uint32_t *interior,
                   const uint32_t *exterior, const int *face_owner,
                   const int *cell_owner, uint32_t *ghosts);

/* Mapping support points, [cell][(m+1)^d][d] on GL(m) nodes:
 * reference box deformation (build_mapping + Mesh::map_point,
 * geometry.cpp:36-63, mesh.cpp:11-26), unit box. */
int dgo_support_reference(int d, const int *cells, double amplitude, int m,
                          double *support);
/* BASELINE.json vertex deformation x + eps*h*prod_a sin(2 pi x_a) per
 * component (m = 1, trilinear cells). h per axis = 1/cells[a]. */
int dgo_support_vertex_bump(int d, const int *cells, double eps,
                            double *support);

/* precompute_geometry for g3 + Laplacian (geometry.cpp:248-522).
 * compress: 1 record per cell (jxw = det) -- caller decides (cartesian).
 * coefficient: 0 none, 1 = a(x) = 1 + 0.5 sin(pi x) cos(pi y) folded into
 * jxw, face_jni/jne and penalty (SURVEY.md s.8c folding definition).
 * Output sizes: inv_jac_t n_rec*d*d, jxw n_rec, face_* n_faces*nqf(*d),
 * penalty n_faces, cell_volume n_cells; n_rec = cells * (compress?1:k^d). */
int dgo_geometry(int d, const int *cells, int m, const double *support,
                 int k, int compress, int coefficient, int64_t n_faces,
                 const uint32_t *interior, const uint32_t *exterior,
                 const uint8_t *fn_int, const uint8_t *fn_ext,
                 double *inv_jac_t, double *jxw, double *face_jxw,
                 double *face_jni, double *face_jne, double *penalty,
                 double *cell_volume);

/* Rank-local SIPG apply, matrix-free but WITHOUT sum factorization: full
 * tensor basis tables as in the dense oracle (oracle.cpp:79-201,205-426),
 * evaluated per cell / per face instead of assembled.
 *   cells in [cell_begin, cell_end) are owned; ghosts[n_ghost] ascending;
 *   faces with face_owner[f] == rank are computed (face_owner NULL: all).
 *   u, y: rank-local W=1 layout (owned cells then ghost cells, k^d each),
 *   y fully overwritten (ghost slots receive the remote contributions,
 *   i.e. the state before compress, ghost_exchange.cpp:359-398).
 * basis as for dgo_shape (the reference reads any basis through full tables).
 * Single rank: cell_begin=0, cell_end=n_cells, n_ghost=0, face_owner NULL. */
int dgo_apply_rank(int d, int k, int n_cells, int compress,
                   const double *inv_jac_t, const double *jxw,
                   int64_t n_faces, const uint32_t *interior,
                   const uint32_t *exterior, const uint8_t *fn_int,
                   const uint8_t *fn_ext, const double *face_jxw,
                   const double *face_jni, const double *face_jne,
                   const double *penalty, int rank, const int *face_owner,
                   int cell_begin, int cell_end, int64_t n_ghost,
                   const uint32_t *ghosts, const double *u, double *y,
                   int basis);

#ifdef __cplusplus
}
#endif
#endif

// Rank operator: setup (layout, cell tasks, device geometry) and apply.
// Mirrors RankOperator / OperatorImpl (reference operators.cpp:89-264).
#include "operator.hpp"
#include "nccl_exchange.hpp"

#include "sipg_params.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace dgx
{

namespace
{
MeshDesc to_mesh(const dgx_mesh &m)
{
  MeshDesc md;
  md.d = m.d;
  for (int a = 0; a < 3; ++a)
    {
      md.cells[a] = a < m.d ? m.cells_per_dim[a] : 1;
      md.lo[a] = m.lo[a];
      md.hi[a] = m.hi[a];
      md.periodic[a] = m.periodic[a] != 0;
    }
  md.amplitude = m.deform_amplitude;
  md.mapping_degree = std::max(1, m.mapping_degree);
  for (int s = 0; s < 6; ++s)
    md.dirichlet_id[s] = m.dirichlet_id[s];
  md.check();
  return md;
}
} // namespace

Operator::Operator(const dgx_setup &s, int device) : device_(device)
{
  const dgx_config &c = s.config;
  if (c.geometry_variant != 3 && c.geometry_variant != 4)
    fail(Code::invalid_argument,
         "RankOperator: geometry variants g3 and g4 are implemented on the device");
  sym_ = c.geometry_variant == 4;
  if (sym_ && c.kind == 1)
    fail(Code::invalid_argument, "RankOperator: advection runs with geometry variant g3");
  if (c.d != s.mesh.d)
    fail(Code::invalid_argument, "RankOperator: mesh dimension mismatch");
  if (c.W != 1 && c.W != 2 && c.W != 4 && c.W != 8)
    fail(Code::invalid_argument, "RankOperator: unsupported lane count");
  if (c.precision != 0 && c.precision != 1)
    fail(Code::invalid_argument, "RankOperator: precision must be 0 (fp64) or 1 (fp32)");
  mesh_ = to_mesh(s.mesh);
  d_ = c.d;
  p_ = c.p;
  k_ = c.p + 1;
  if (c.p < 1 || c.p > 10)
    fail(Code::invalid_argument, "RankOperator: supported degrees are 1..10");
  if (c.basis < 0 || c.basis > 2)
    fail(Code::invalid_argument, "RankOperator: unknown basis kind");
  if (c.basis == 2 && c.p < 3)
    fail(Code::invalid_argument, "RankOperator: the Hermite-type basis needs degree >= 3");
  basis_ = c.basis;
  if (c.kind != 0 && c.kind != 1)
    fail(Code::invalid_argument, "RankOperator: unknown operator kind");
  kind_ = c.kind;
  if (kind_ == 1)
    {
      if (c.precision != 0)
        fail(Code::invalid_argument, "RankOperator: advection runs in fp64 only");
      if (c.basis == 2)
        fail(Code::invalid_argument,
             "RankOperator: advection with the Hermite-like basis is not implemented");
      for (int a = 0; a < 3; ++a)
        velocity_[a] = c.velocity[a];
      variable_velocity_ = c.variable_velocity != 0;
    }
  precision_ = c.precision;
  nq_ = 1;
  for (int a = 0; a < d_; ++a)
    nq_ *= k_;
  nqf_ = nq_ / k_;

  host_only_ = device_ < 0;
  if (!host_only_)
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");

  if (!s.faces || s.n_faces <= 0)
    fail(Code::invalid_argument, "RankOperator: empty face list");
  std::vector<RawFace> faces(s.n_faces);
  std::memcpy(faces.data(), s.faces, sizeof(RawFace) * s.n_faces);
  const long long nc = mesh_.n_cells();
  for (const RawFace &f : faces)
    if (f.interior_cell >= nc || (!f.at_boundary() && f.exterior_cell >= nc) ||
        f.interior_face_number >= 2 * d_ ||
        (!f.at_boundary() && f.exterior_face_number >= 2 * d_))
      fail(Code::invalid_argument, "RankOperator: face references an invalid cell or face");

  Partition part;
  if (s.n_ranks < 1)
    fail(Code::invalid_argument, "RankOperator: n_ranks must be >= 1");
  if (s.cell_owner && s.rank_cell_range && s.face_owner)
    {
      part.n_ranks = s.n_ranks;
      part.cell_owner.assign(s.cell_owner, s.cell_owner + nc);
      for (int r = 0; r < s.n_ranks; ++r)
        part.ranges.emplace_back(s.rank_cell_range[2 * r], s.rank_cell_range[2 * r + 1]);
      part.face_owner.assign(s.face_owner, s.face_owner + s.n_faces);
    }
  else
    part = make_partition(mesh_, faces, s.n_ranks);
  n_ranks_ = part.n_ranks;
  layout_ = build_layout(mesh_, faces, part, s.rank, k_, basis_, kind_);

  build_tasks(faces, part);
  if (host_only_)
    return;
  build_geometry(s, faces);
  upload_tables(k_, basis_);
  if (kind_ == 1)
    set_velocity(nullptr, nullptr, nullptr);
}

// Task lists. Owned cells whose computed faces never read a ghost form the
// inner phase (overlappable with the ghost update, operators.cpp:314-317);
// owned cells with a ghost-reading face and one "ghost-side" task per ghost
// cell (the remote side of the faces this rank computes, later compressed
// to the owner) form the coupled phase.
void Operator::build_tasks(const std::vector<RawFace> &faces, const Partition &part)
{
  const int nfpc = 2 * d_;
  const long long n_owned = layout_.n_owned;
  const long long n_slots = n_owned + (long long)layout_.ghosts.size();
  std::vector<long long> face_of(n_slots * nfpc, -1);
  for (std::size_t f = 0; f < faces.size(); ++f)
    {
      const RawFace &rf = faces[f];
      const long long s0 = layout_.slot(rf.interior_cell);
      if (s0 >= 0)
        face_of[s0 * nfpc + rf.interior_face_number] = (long long)f;
      if (!rf.at_boundary())
        {
          const long long s1 = layout_.slot(rf.exterior_cell);
          if (s1 >= 0)
            face_of[s1 * nfpc + rf.exterior_face_number] = (long long)f;
        }
    }
  std::vector<int> face_local(faces.size(), -1);
  for (std::size_t i = 0; i < layout_.my_faces.size(); ++i)
    face_local[layout_.my_faces[i]] = static_cast<int>(i);

  std::vector<int> slot_inner, slot_coupled, geo_inner, geo_coupled;
  std::vector<int2> tf_inner, tf_coupled;
  auto make_task = [&](long long slot, bool owned, std::vector<int2> &tf) {
    bool coupled = false;
    const std::uint32_t gcell =
      owned ? layout_.owned_begin + (std::uint32_t)slot : layout_.ghosts[slot - n_owned];
    for (int phi = 0; phi < nfpc; ++phi)
      {
        const long long f = face_of[slot * nfpc + phi];
        int2 e = make_int2(-2, 0);
        if (f < 0)
          {
            if (owned)
              fail(Code::logic_error, "layout: owned cell without a face on every side");
          }
        else if (part.face_owner[f] == layout_.rank)
          {
            const RawFace &rf = faces[f];
            const int side =
              (rf.interior_cell == gcell && rf.interior_face_number == phi) ? 0 : 1;
            if (rf.at_boundary())
              e.x = -1;
            else
              {
                const std::uint32_t other = side == 0 ? rf.exterior_cell : rf.interior_cell;
                const long long os = layout_.slot(other);
                if (os < 0)
                  fail(Code::logic_error, "layout: face neighbour absent on this rank");
                e.x = static_cast<int>(os);
                if (os >= n_owned)
                  coupled = true;
              }
            e.y = face_local[f] | (side << 30);
          }
        tf.push_back(e);
      }
    return coupled;
  };

  // Task order = traversal order of the owned cells. Lexicographic order
  // puts the z-neighbour one cell layer (n_x n_y tasks) away, far beyond
  // what L2 retains while the read-once geometry streams through it. Sweep
  // z inside tiles of full x-rows and TILE_Y y-rows instead: the z-neighbour
  // (and the shared face record) is then n_x TILE_Y tasks away and still in
  // L2; only neighbours across the y tile edges are read twice from HBM.
  //
  // Brick CTAs (the pencil-pair kernel, sipg_pairs.cuh): the same sweep in
  // 2x2x2 (or 2x2x1) bricks of consecutive tasks, one brick per CTA, so that
  // the faces inside a brick take the partner's trace from shared memory.
  // A brick goes whole into one phase list (coupled if any of its cells
  // reads a ghost) so that the CTA groups stay aligned; cells of incomplete
  // bricks follow as single tasks.
  std::vector<std::vector<long long>> groups;
  {
    const int nx = mesh_.cells[0], ny = d_ == 3 ? mesh_.cells[1] : 1;
    const long long layer = (long long)nx * ny;
    const long long b = layout_.owned_begin, e = b + n_owned;
    int tile_y = d_ == 3 ? 8 : 1 << 30;
    if (const char *e = std::getenv("DGX_TILE_Y")) // traversal experiments
      if (d_ == 3 && std::atoi(e) > 0)
        tile_y = std::atoi(e);
    const int brick0 = (d_ == 3 && precision_ == 0) ? kernel_brick(d_, k_) : 0;
    const int brick = brick0 >= 4 ? brick0 : 0; // 1: x-rows, no reordering
    auto in_range = [&](long long z, int y, int x) {
      const long long c = z * layer + (long long)y * nx + x;
      return x < nx && y < ny && c >= b && c < e;
    };
    if (d_ == 3 && brick > 0)
      {
        const int bz = brick == 8 ? 2 : 1;
        std::vector<char> used(n_owned, 0);
        const long long z0 = b / layer, z1 = (e + layer - 1) / layer;
        for (int ty = 0; ty < ny; ty += tile_y)
          for (long long z = z0; z < z1; z += bz)
            for (int y = ty; y < std::min(ny, ty + tile_y); y += 2)
              for (int x = 0; x < nx; x += 2)
                {
                  std::vector<long long> g;
                  for (int iz = 0; iz < bz; ++iz)
                    for (int iy = 0; iy < 2; ++iy)
                      for (int ix = 0; ix < 2; ++ix)
                        if (y + iy < std::min(ny, ty + tile_y) && in_range(z + iz, y + iy, x + ix))
                          g.push_back((z + iz) * layer + (long long)(y + iy) * nx + x + ix - b);
                  if ((int)g.size() == brick)
                    {
                      for (long long c : g)
                        used[c] = 1;
                      groups.push_back(g);
                    }
                }
        for (int ty = 0; ty < ny; ty += tile_y)
          for (long long z = z0; z < z1; ++z)
            for (int y = ty; y < std::min(ny, ty + tile_y); ++y)
              for (int x = 0; x < nx; ++x)
                if (in_range(z, y, x))
                  {
                    const long long c = z * layer + (long long)y * nx + x - b;
                    if (!used[c])
                      groups.push_back({c});
                  }
      }
    else if (d_ == 3)
      {
        const long long z0 = b / layer, z1 = (e + layer - 1) / layer;
        for (int ty = 0; ty < ny; ty += tile_y)
          for (long long z = z0; z < z1; ++z)
            for (int y = ty; y < std::min(ny, ty + tile_y); ++y)
              for (int x = 0; x < nx; ++x)
                if (in_range(z, y, x))
                  groups.push_back({z * layer + (long long)y * nx + x - b});
      }
    else
      for (long long s = 0; s < n_owned; ++s)
        groups.push_back({s});
  }
  // whole bricks first in each phase list, single tasks after them
  for (int pass = 0; pass < 2; ++pass)
    for (const auto &g : groups)
      {
        if ((pass == 0) != (g.size() > 1))
          continue;
        std::vector<std::vector<int2>> tfs(g.size());
        bool coupled = false;
        for (std::size_t i = 0; i < g.size(); ++i)
          coupled = make_task(g[i], true, tfs[i]) || coupled;
        auto &sl = coupled ? slot_coupled : slot_inner;
        auto &gl = coupled ? geo_coupled : geo_inner;
        auto &fl = coupled ? tf_coupled : tf_inner;
        for (std::size_t i = 0; i < g.size(); ++i)
          {
            sl.push_back(static_cast<int>(g[i]));
            gl.push_back(static_cast<int>(g[i]));
            fl.insert(fl.end(), tfs[i].begin(), tfs[i].end());
          }
      }
  for (long long s = n_owned; s < n_slots; ++s)
    {
      std::vector<int2> tf;
      make_task(s, false, tf);
      slot_coupled.push_back(static_cast<int>(s));
      geo_coupled.push_back(-1);
      tf_coupled.insert(tf_coupled.end(), tf.begin(), tf.end());
    }
  n_inner_ = static_cast<int>(slot_inner.size());
  n_coupled_ = static_cast<int>(slot_coupled.size());
  slot_inner.insert(slot_inner.end(), slot_coupled.begin(), slot_coupled.end());
  geo_inner.insert(geo_inner.end(), geo_coupled.begin(), geo_coupled.end());
  tf_inner.insert(tf_inner.end(), tf_coupled.begin(), tf_coupled.end());
  if (!host_only_)
    {
      task_slot_.upload(slot_inner);
      task_geo_.upload(geo_inner);
      task_face_.upload(tf_inner);
    }
  host_task_slot_ = slot_inner;
  host_task_geo_ = geo_inner;
  host_task_face_ = tf_inner;

  // exchange plans flattened to value indices (plan order: ascending cells,
  // ascending dofs, pack_plan_values, ghost_exchange.cpp:240-295)
  auto flatten = [&](const std::vector<NeighborPlan> &plans, std::vector<long long> &idx,
                     std::vector<long long> &offs) {
    offs.assign(1, 0);
    for (const NeighborPlan &np : plans)
      {
        for (std::size_t i = 0; i < np.cells.size(); ++i)
          {
            const long long sl = layout_.slot(np.cells[i]);
            if (sl < 0)
              fail(Code::logic_error, "exchange plan: cell absent from the layout");
            for (std::uint32_t j = np.dof_offsets[i]; j < np.dof_offsets[i + 1]; ++j)
              idx.push_back(sl * nq_ + np.dofs[j]);
          }
        offs.push_back((long long)idx.size());
      }
  };
  std::vector<long long> si, ri;
  flatten(layout_.send, si, send_offsets_);
  flatten(layout_.recv, ri, recv_offsets_);
  // in place: whole ghost cells, concatenated receive plans = ghost region
  recv_in_place_ = layout_.whole_cells &&
                   (long long)ri.size() == (long long)layout_.ghosts.size() * nq_;
  for (std::size_t i = 0; recv_in_place_ && i < ri.size(); ++i)
    if (ri[i] != layout_.owned_size() + (long long)i)
      recv_in_place_ = false;
  if (!host_only_)
    {
      send_index_.upload(si);
      recv_index_.upload(ri);
    }
  // whole-cell send plans as cell slot lists (pack / accumulate per cell)
  send_cell_offsets_.assign(1, 0);
  if (layout_.whole_cells)
    {
      std::vector<int> sc;
      for (const NeighborPlan &np : layout_.send)
        {
          for (std::uint32_t c : np.cells)
            sc.push_back(static_cast<int>(layout_.slot(c)));
          send_cell_offsets_.push_back((long long)sc.size());
        }
      if (!host_only_)
        send_slots_.upload(sc);
    }
}

void Operator::build_geometry(const dgx_setup &s, const std::vector<RawFace> &faces)
{
  face_boundary_.resize(layout_.my_faces.size());
  for (std::size_t i = 0; i < layout_.my_faces.size(); ++i)
    face_boundary_[i] = faces[layout_.my_faces[i]].at_boundary() ? 1 : 0;
  const dgx_geometry &g = s.geometry;
  const long long n_owned = layout_.n_owned;
  const long long n_slots = n_owned + (long long)layout_.ghosts.size();
  const long long nmy = (long long)layout_.my_faces.size();
  // g3: J^{-T} (d^2) and JxW; g4: the d(d+1)/2 merged coefficients
  const int ncomp = sym_ ? d_ * (d_ + 1) / 2 : d_ * d_ + 1;
  std::vector<std::uint32_t> slot_cells(n_slots);
  for (long long i = 0; i < n_owned; ++i)
    slot_cells[i] = layout_.owned_begin + (std::uint32_t)i;
  for (std::size_t i = 0; i < layout_.ghosts.size(); ++i)
    slot_cells[n_owned + i] = layout_.ghosts[i];

  if (g.source == DGX_GEOMETRY_HOST_ARRAYS)
    {
      if (g.coefficient)
        fail(Code::invalid_argument, "geometry: fold the coefficient into the host arrays");
      if ((sym_ ? !g.coeff : (!g.inv_jac_t || !g.jxw)) || !g.face_jxw || !g.face_jni ||
          !g.face_jne || !g.penalty)
        fail(Code::invalid_argument, "geometry: missing host arrays");
      compressed_ = g.compressed != 0;
      const long long nrec = compressed_ ? 1 : nq_;
      std::vector<double> cg((size_t)n_owned * ncomp * nrec);
      for (long long c = 0; c < n_owned; ++c)
        {
          const long long gc = layout_.owned_begin + c;
          for (long long r = 0; r < nrec; ++r)
            {
              if (sym_)
                {
                  // GeometryCache::coeff [cell][q][d(d+1)/2]
                  for (int i = 0; i < ncomp; ++i)
                    cg[(c * ncomp + i) * nrec + r] = g.coeff[(gc * nrec + r) * ncomp + i];
                  continue;
                }
              const double *jit = g.inv_jac_t + (gc * nrec + r) * d_ * d_;
              for (int i = 0; i < d_ * d_; ++i)
                cg[(c * ncomp + i) * nrec + r] = jit[i];
              cg[(c * ncomp + d_ * d_) * nrec + r] = g.jxw[gc * nrec + r];
            }
        }
      // Cartesian caches: faces compress like the cells (one record, JxW_f
      // weight applied on the fly); the reference stores them in full, so
      // check that they are constant per face
      const long long nrf = compressed_ ? 1 : nqf_;
      std::vector<double> wqf(nqf_, 1.0);
      {
        const Quad1D qg = gauss(k_);
        for (long long q = 0; q < nqf_; ++q)
          {
            long long idx = q;
            for (int a = 0; a < d_ - 1; ++a)
              {
                wqf[q] *= qg.weights[idx % k_];
                idx /= k_;
              }
          }
      }
      std::vector<double> fg((size_t)nmy * (2 * d_ + 1) * nrf), pen(nmy);
      for (long long i = 0; i < nmy; ++i)
        {
          const long long f = layout_.my_faces[i];
          for (long long q = 0; q < nqf_; ++q)
            {
              const double jw = g.face_jxw[f * nqf_ + q];
              const double *jni = g.face_jni + (f * nqf_ + q) * d_;
              const double *jne = g.face_jne + (f * nqf_ + q) * d_;
              if (!compressed_)
                {
                  double *o = fg.data() + i * (2 * d_ + 1) * nqf_ + q;
                  o[0] = jw;
                  for (int b = 0; b < d_; ++b)
                    {
                      o[(1 + b) * nqf_] = jni[b];
                      o[(1 + d_ + b) * nqf_] = jne[b];
                    }
                  continue;
                }
              double *o = fg.data() + i * (2 * d_ + 1);
              if (q == 0)
                {
                  o[0] = jw / wqf[0];
                  for (int b = 0; b < d_; ++b)
                    {
                      o[1 + b] = jni[b];
                      o[1 + d_ + b] = jne[b];
                    }
                }
              double scale = 0.0;
              for (int b = 0; b < d_; ++b)
                scale = std::max({scale, std::abs(jni[b]), std::abs(jne[b])});
              bool same = std::abs(jw - o[0] * wqf[q]) <= 1e-12 * std::abs(jw);
              for (int b = 0; b < d_; ++b)
                same = same && std::abs(jni[b] - o[1 + b]) <= 1e-12 * scale &&
                       std::abs(jne[b] - o[1 + d_ + b]) <= 1e-12 * scale;
              if (!same)
                fail(Code::invalid_argument,
                     "geometry: compressed (Cartesian) cache with non-constant face data");
            }
          pen[i] = g.penalty[f];
        }
      cell_geo_.upload(cg);
      face_geo_.upload(fg);
      penalty_.upload(pen);
      if (kind_ == 1)
        {
          if (!g.face_normal)
            fail(Code::invalid_argument, "geometry: advection needs the face normals");
          if (compressed_ && variable_velocity_)
            fail(Code::invalid_argument,
                 "geometry: a variable velocity needs an uncompressed geometry cache");
          std::vector<double> nv((size_t)nmy * d_ * nrf);
          for (long long i = 0; i < nmy; ++i)
            {
              const long long f = layout_.my_faces[i];
              for (long long q = 0; q < nrf; ++q)
                for (int b = 0; b < d_; ++b)
                  nv[(i * d_ + b) * nrf + q] = g.face_normal[(f * nqf_ + q) * d_ + b];
            }
          normals_.upload(nv);
        }
    }
  else
    {
      std::vector<double> support;
      int m = 1;
      bool cartesian = false;
      switch (g.source)
        {
        case DGX_GEOMETRY_MESH:
          m = mesh_.mapping_degree;
          support = reference_support(mesh_, slot_cells);
          cartesian = mesh_.amplitude == 0.0;
          break;
        case DGX_GEOMETRY_VERTEX_BUMP:
          m = 1;
          support = vertex_bump_support(mesh_, g.vertex_bump_eps, slot_cells);
          cartesian = g.vertex_bump_eps == 0.0;
          break;
        case DGX_GEOMETRY_SUPPORT:
          {
            if (!g.support_points)
              fail(Code::invalid_argument, "geometry: missing support points");
            m = std::max(1, g.support_degree);
            long long pp = 1;
            for (int a = 0; a < d_; ++a)
              pp *= m + 1;
            support.resize((size_t)n_slots * pp * d_);
            for (long long i = 0; i < n_slots; ++i)
              std::memcpy(support.data() + i * pp * d_,
                          g.support_points + (long long)slot_cells[i] * pp * d_,
                          sizeof(double) * pp * d_);
            cartesian = g.cartesian != 0;
            break;
          }
        default:
          fail(Code::invalid_argument, "geometry: unknown source");
        }
      if (g.coefficient != 0 && g.coefficient != 1)
        fail(Code::invalid_argument, "geometry: unknown coefficient");
      compressed_ = cartesian && !g.coefficient && !variable_velocity_;
      DeviceArray<double> &dsup = support_;
      dsup.upload(support);
      has_mapping_ = true;
      map_degree_ = m;
      std::vector<int4> fl(nmy);
      for (long long i = 0; i < nmy; ++i)
        {
          const RawFace &rf = faces[layout_.my_faces[i]];
          fl[i] = make_int4(static_cast<int>(layout_.slot(rf.interior_cell)),
                            rf.at_boundary() ? -1 : static_cast<int>(layout_.slot(rf.exterior_cell)),
                            rf.interior_face_number, rf.exterior_face_number);
        }
      DeviceArray<int4> &dfl = face_list_;
      dfl.upload(fl);
      DeviceArray<double> vol(n_slots);
      cell_geo_.resize((size_t)n_owned * ncomp * (compressed_ ? 1 : nq_));
      face_geo_.resize((size_t)nmy * (2 * d_ + 1) * (compressed_ ? 1 : nqf_));
      penalty_.resize(nmy);
      GeometryJob job;
      job.d = d_;
      job.k = k_;
      job.m = m;
      job.compress = compressed_;
      job.coefficient = g.coefficient;
      job.g4 = sym_;
      if (cartesian)
        {
          double v = 1.0;
          for (int a = 0; a < d_; ++a)
            v *= (mesh_.hi[a] - mesh_.lo[a]) / mesh_.cells[a];
          job.cart_volume = v;
        }
      job.support = dsup.get();
      job.n_slots = static_cast<int>(n_slots);
      job.n_geo_cells = static_cast<int>(n_owned);
      job.n_faces = nmy;
      job.faces = dfl.get();
      job.cell_geo = cell_geo_.get();
      job.face_geo = face_geo_.get();
      job.penalty = penalty_.get();
      job.volume = vol.get();
      if (kind_ == 1)
        {
          normals_.resize((size_t)nmy * d_ * (compressed_ ? 1 : nqf_));
          job.face_normal = normals_.get();
        }
      run_geometry(job, nullptr);
    }
  // axis-aligned affine records (every Cartesian box mesh): the CART
  // kernels skip the tangential face terms, which are exact zeros here
  cart_ = false;
  if (compressed_ && kind_ == 0 && !sym_ && !host_only_ && !std::getenv("DGX_NO_CART"))
    {
      std::vector<signed char> ax(nmy);
      for (long long i = 0; i < nmy; ++i)
        ax[i] = static_cast<signed char>(faces[layout_.my_faces[i]].interior_face_number / 2);
      DeviceArray<signed char> dax;
      dax.upload(ax);
      cuda_check(cudaDeviceSynchronize(), "geometry setup");
      cart_ = count_non_axis_records(d_, cell_geo_.get(), n_owned, face_geo_.get(), dax.get(), nmy) == 0;
    }
  // the tensor-product kernel (sipg_cart.cuh) instead of the collocation
  // CART kernels
  tensor_ = cart_ && !std::getenv("DGX_NO_TENSOR");
  if (precision_ == 1)
    {
      cell_geo_f_.resize(cell_geo_.size());
      face_geo_f_.resize(face_geo_.size());
      penalty_f_.resize(penalty_.size());
      launch_convert<float>(cell_geo_.get(), cell_geo_f_.get(), cell_geo_.size(), nullptr);
      launch_convert<float>(face_geo_.get(), face_geo_f_.get(), face_geo_.size(), nullptr);
      launch_convert<float>(penalty_.get(), penalty_f_.get(), penalty_.size(), nullptr);
      cuda_check(cudaDeviceSynchronize(), "convert geometry");
    }
  cuda_check(cudaDeviceSynchronize(), "geometry setup");
}

void Operator::set_velocity(const double *c_cells, const double *c_faces, cudaStream_t s)
{
  if (kind_ != 1)
    fail(Code::invalid_argument, "set_velocity: not an advection operator");
  if (host_only_)
    return;
  if (compressed_ && (c_cells || c_faces))
    fail(Code::invalid_argument,
         "set_velocity: per-point velocities need variable_velocity = 1 (uncompressed geometry)");
  if (variable_velocity_ && (!c_cells || !c_faces) && adv_cell_.size() > 0)
    fail(Code::invalid_argument, "set_velocity: missing per-point velocity arrays");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  const long long nrec = compressed_ ? 1 : nq_, nrf = compressed_ ? 1 : nqf_;
  const long long nmy = (long long)layout_.my_faces.size();
  adv_cell_.resize((size_t)layout_.n_owned * d_ * nrec);
  adv_face_.resize((size_t)nmy * 2 * nrf);
  run_adv_coefficients(d_, k_, compressed_, layout_.n_owned, nmy, cell_geo_.get(),
                       face_geo_.get(), normals_.get(), velocity_, c_cells, c_faces,
                       adv_cell_.get(), adv_face_.get(), s);
}

template <typename Real>
void Operator::launch_range(int begin, int count, const Real *u, Real *y, cudaStream_t s)
{
  launch_tasks(task_slot_.get() + begin, task_geo_.get() + begin,
               task_face_.get() + (long long)begin * 2 * d_, count, u, y, s);
}

template <typename Real>
void Operator::launch_tasks(const int *tslot, const int *tgeo, const int2 *tface, int count,
                            const Real *u, Real *y, cudaStream_t s)
{
  if (count <= 0)
    return;
  if (kind_ == 1)
    {
      if constexpr (sizeof(Real) == 8)
        {
          dev::AdvParams<double> ap;
          ap.u = u;
          ap.y = y;
          ap.cell = adv_cell_.get();
          ap.face = adv_face_.get();
          ap.task_slot = tslot;
          ap.task_geo = tgeo;
          ap.task_face = tface;
          ap.n_tasks = count;
          ap.n_owned = static_cast<int>(layout_.n_owned);
          launch_adv(d_, k_, basis_, compressed_, ap, s);
        }
      else
        fail(Code::invalid_argument, "advection: fp64 only");
      return;
    }
  dev::ApplyParams<Real> prm;
  prm.u = u;
  prm.y = y;
  if constexpr (sizeof(Real) == 8)
    {
      prm.cell_geo = cell_geo_.get();
      prm.face_geo = face_geo_.get();
      prm.penalty = penalty_.get();
    }
  else
    {
      prm.cell_geo = cell_geo_f_.get();
      prm.face_geo = face_geo_f_.get();
      prm.penalty = penalty_f_.get();
    }
  prm.task_slot = tslot;
  prm.task_geo = tgeo;
  prm.task_face = tface;
  prm.n_tasks = count;
  prm.n_owned = static_cast<int>(layout_.n_owned);
  prm.sym = sym_ ? 1 : 0;
  prm.ahead = 0;
  prm.cart = cart_ ? (tensor_ ? 2 : 1) : 0;
  launch_apply<Real>(d_, k_, basis_, compressed_, prm, s);
}

// argument checks of an apply (operators.cpp:220-222 checks before any hook)
void Operator::check_apply_args(const void *u, const void *y, bool fp32) const
{
  if (fp32 != (precision_ == 1))
    fail(Code::invalid_argument, "apply: precision does not match the operator config");
  if (host_only_)
    fail(Code::invalid_argument, "apply: operator was created host-only (device < 0)");
  if (u == y)
    fail(Code::invalid_argument, "apply: source and destination must differ");
}

void Operator::apply_phase(int phase, const void *u, void *y, cudaStream_t s, bool fp32)
{
  check_apply_args(u, y, fp32);
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  const int b = phase == 1 ? 0 : n_inner_;
  const int n = phase == 1 ? n_inner_ : n_coupled_;
  if (phase != 1 && phase != 2)
    fail(Code::invalid_argument, "apply_phase: phase must be 1 or 2");
  if (fp32)
    {
#ifdef DGX_WITH_FP32
      launch_range<float>(b, n, static_cast<const float *>(u), static_cast<float *>(y), s);
#else
      fail(Code::invalid_argument, "apply: library built without fp32 kernels");
#endif
    }
  else
    launch_range<double>(b, n, static_cast<const double *>(u), static_cast<double *>(y), s);
}

// RankOperator::apply (operators.cpp:217-264) with the exchange hooks.
void Operator::apply(void *u, void *y, const dgx_hooks *hooks, cudaStream_t s, bool fp32)
{
  // every argument error is raised before a hook posts any communication
  // (a failing apply must not leave the exchanger in flight)
  check_apply_args(u, y, fp32);
  const bool have_ghosts = !layout_.ghosts.empty();
  if (Exchanger *ex = native_exchanger(hooks); ex && ex->op() == this && n_coupled_ > 0)
    {
      // The native exchanger takes compress off the critical path: the
      // ghost-coupled tasks run first on a high-priority stream as soon as
      // the update has landed, their ghost contributions leave while the
      // inner tasks still run on the caller's stream, and only the
      // accumulation waits for both (same hooks, same results: the phases
      // write disjoint cells, the accumulation order is unchanged).
      cuda_check(cudaSetDevice(device_), "cudaSetDevice");
      cudaStream_t sg = ghost_stream();
      ex->start_update(u, s);
      ex->finish_update(u, sg);
      apply_phase(2, u, y, sg, fp32);
      ex->compress_post(y, sg);
      apply_phase(1, u, y, s, fp32);
      ex->compress_finish(y, s);
      return;
    }
  auto call = [&](dgx_hook_fn fn, void *v, const char *what) {
    const dgx_status st = fn(hooks->ctx, v, static_cast<void *>(s));
    if (st != DGX_OK)
      fail(static_cast<Code>(st), std::string(what) + " hook failed");
  };
  if (hooks && hooks->start_ghost_update)
    call(hooks->start_ghost_update, u, "start_ghost_update");
  else if (have_ghosts)
    fail(Code::logic_error, "apply: layout has ghost cells but no exchange hooks were given");
  apply_phase(1, u, y, s, fp32);
  if (n_coupled_ > 0)
    {
      if (hooks && hooks->finish_ghost_update)
        call(hooks->finish_ghost_update, u, "finish_ghost_update");
      else if (have_ghosts)
        fail(Code::logic_error,
             "apply: ghost-coupled face reached without a way to finish the ghost update");
      apply_phase(2, u, y, s, fp32);
    }
  if (hooks && hooks->compress)
    call(hooks->compress, y, "compress");
}

cudaStream_t Operator::ghost_stream()
{
  if (!ghost_stream_)
    {
      int lo = 0, hi = 0;
      cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
      cuda_check(cudaStreamCreateWithPriority(&ghost_stream_, cudaStreamNonBlocking, hi),
                 "cudaStreamCreateWithPriority");
    }
  return ghost_stream_;
}

Operator::~Operator()
{
  if (ghost_stream_)
    {
      cudaSetDevice(device_);
      cudaStreamDestroy(ghost_stream_);
    }
  if (pipe_.sh || pipe_.sc || pipe_.sd)
    {
      cudaSetDevice(device_);
      for (cudaEvent_t e : pipe_.ev_h)
        cudaEventDestroy(e);
      for (cudaEvent_t e : pipe_.ev_c)
        cudaEventDestroy(e);
      cudaStreamDestroy(pipe_.sh);
      cudaStreamDestroy(pipe_.sc);
      cudaStreamDestroy(pipe_.sd);
    }
}

// z-slab chunks of the owned cells (single rank: slot = global cell), task
// lists reordered chunk by chunk (stable: the traversal order inside a chunk
// is the apply's own)
void Operator::build_host_pipe()
{
  HostPipe &P = pipe_;
  P.built = true;
  const long long n = layout_.total_size();
  P.du.resize(n);
  P.dy.resize(n);
  P.pipelined = d_ == 3 && n_ranks_ == 1 && layout_.ghosts.empty() && n_coupled_ == 0 &&
                precision_ == 0 && mesh_.cells[2] >= 4;
  cuda_check(cudaStreamCreateWithFlags(&P.sh, cudaStreamNonBlocking), "cudaStreamCreate");
  cuda_check(cudaStreamCreateWithFlags(&P.sc, cudaStreamNonBlocking), "cudaStreamCreate");
  cuda_check(cudaStreamCreateWithFlags(&P.sd, cudaStreamNonBlocking), "cudaStreamCreate");
  if (!P.pipelined)
    return;
  const int nz = mesh_.cells[2];
  const long long layer = (long long)mesh_.cells[0] * mesh_.cells[1];
  P.nchunk = std::min(64, nz / 2); // measured (C4 e2e): 16 / 32 / 64 slabs 5.51 / 5.80 / 5.84 GDoF/s
  if (const char *e = std::getenv("DGX_HOST_CHUNKS"))
    P.nchunk = std::max(2, std::min(nz, std::atoi(e)));
  P.periodic_z = mesh_.periodic[2] != 0;
  P.cell_begin.resize(P.nchunk + 1);
  for (int k = 0; k <= P.nchunk; ++k)
    P.cell_begin[k] = (long long)(nz * (long long)k / P.nchunk) * layer;
  std::vector<std::vector<int>> idx(P.nchunk);
  const int nt = n_inner_;
  for (int i = 0; i < nt; ++i)
    {
      const long long c = host_task_slot_[i];
      int k = (int)(c / layer * P.nchunk / nz);
      while (k + 1 < P.nchunk && c >= P.cell_begin[k + 1])
        ++k;
      while (k > 0 && c < P.cell_begin[k])
        --k;
      idx[k].push_back(i);
    }
  std::vector<int> sl, ge;
  std::vector<int2> fa;
  P.task_begin.assign(1, 0);
  for (int k = 0; k < P.nchunk; ++k)
    {
      for (int i : idx[k])
        {
          sl.push_back(host_task_slot_[i]);
          ge.push_back(host_task_geo_[i]);
          for (int f = 0; f < 2 * d_; ++f)
            fa.push_back(host_task_face_[(size_t)i * 2 * d_ + f]);
        }
      P.task_begin.push_back((int)sl.size());
    }
  P.slot.upload(sl);
  P.geo.upload(ge);
  P.face.upload(fa);
  P.ev_h.resize(P.nchunk);
  P.ev_c.resize(P.nchunk);
  for (int k = 0; k < P.nchunk; ++k)
    {
      cuda_check(cudaEventCreateWithFlags(&P.ev_h[k], cudaEventDisableTiming), "cudaEventCreate");
      cuda_check(cudaEventCreateWithFlags(&P.ev_c[k], cudaEventDisableTiming), "cudaEventCreate");
    }
}

void Operator::apply_host(const double *u, double *y)
{
  if (precision_ != 0)
    fail(Code::invalid_argument, "dgx_apply_host: fp64 operators only");
  if (host_only_)
    fail(Code::invalid_argument, "apply: operator was created host-only (device < 0)");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  if (!pipe_.built)
    build_host_pipe();
  HostPipe &P = pipe_;
  const long long n = layout_.total_size();
  double *du = P.du.get(), *dy = P.dy.get();
  if (!P.pipelined)
    {
      // ghosted layouts: the caller has completed the ghost update on the
      // host side; both phases, y returns the ghost contributions
      cuda_check(cudaMemcpyAsync(du, u, n * 8, cudaMemcpyHostToDevice, P.sc), "h2d");
      apply_phase(1, du, dy, P.sc, false);
      apply_phase(2, du, dy, P.sc, false);
      cuda_check(cudaMemcpyAsync(y, dy, n * 8, cudaMemcpyDeviceToHost, P.sc), "d2h");
      cuda_check(cudaStreamSynchronize(P.sc), "apply_host");
      return;
    }
  const long long nq = nq_;
  const int S = P.nchunk;
  for (int k = 0; k < S; ++k)
    {
      const long long c0 = P.cell_begin[k], c1 = P.cell_begin[k + 1];
      cuda_check(cudaMemcpyAsync(du + c0 * nq, u + c0 * nq, (c1 - c0) * nq * 8, cudaMemcpyHostToDevice,
                                 P.sh),
                 "h2d");
      cuda_check(cudaEventRecord(P.ev_h[k], P.sh), "cudaEventRecord");
    }
  // a chunk reads its neighbours' u across z: wait for the H2D of the chunk
  // above (in-order copies imply the ones below); with periodic z chunk 0
  // also reads the last chunk, so it runs last
  std::vector<int> order;
  for (int k = P.periodic_z ? 1 : 0; k < S; ++k)
    order.push_back(k);
  if (P.periodic_z)
    order.push_back(0);
  for (int k : order)
    {
      const int need = P.periodic_z && k == 0 ? S - 1 : std::min(k + 1, S - 1);
      cuda_check(cudaStreamWaitEvent(P.sc, P.ev_h[need], 0), "cudaStreamWaitEvent");
      launch_tasks(P.slot.get() + P.task_begin[k], P.geo.get() + P.task_begin[k],
                   P.face.get() + (long long)P.task_begin[k] * 2 * d_, P.task_begin[k + 1] - P.task_begin[k],
                   du, dy, P.sc);
      cuda_check(cudaEventRecord(P.ev_c[k], P.sc), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(P.sd, P.ev_c[k], 0), "cudaStreamWaitEvent");
      const long long c0 = P.cell_begin[k], c1 = P.cell_begin[k + 1];
      cuda_check(cudaMemcpyAsync(y + c0 * nq, dy + c0 * nq, (c1 - c0) * nq * 8, cudaMemcpyDeviceToHost,
                                 P.sd),
                 "d2h");
    }
  cuda_check(cudaStreamSynchronize(P.sd), "apply_host");
  cuda_check(cudaStreamSynchronize(P.sc), "apply_host");
}

void Operator::accumulate_plan(int idx, const double *contrib, double *y, cudaStream_t s)
{
  if (idx < 0 || idx >= (int)layout_.send.size())
    fail(Code::invalid_argument, "accumulate_plan: plan index out of range");
  const long long b = send_offsets_[idx], e = send_offsets_[idx + 1];
  launch_scatter_add_values(y, send_index_.get() + b, e - b, contrib, s);
}

GeometryJob Operator::mapping_job() const
{
  if (!has_mapping_)
    fail(Code::invalid_argument,
         "quadrature points: the geometry came as host arrays, there is no mapping");
  GeometryJob job;
  job.d = d_;
  job.k = k_;
  job.m = map_degree_;
  job.support = support_.get();
  job.n_geo_cells = static_cast<int>(layout_.n_owned);
  job.n_faces = (long long)layout_.my_faces.size();
  job.faces = face_list_.get();
  return job;
}

std::vector<double> Operator::quadrature_points(int which)
{
  if (host_only_)
    fail(Code::invalid_argument, "quadrature points: operator was created host-only");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  if (which == 2)
    return std::vector<double>(face_boundary_.begin(), face_boundary_.end());
  if (which != 0 && which != 1)
    fail(Code::invalid_argument, "quadrature points: unknown set");
  const GeometryJob job = mapping_job();
  DeviceArray<double> x(which == 0 ? (size_t)layout_.n_owned * nq_ * d_
                                   : layout_.my_faces.size() * (size_t)nqf_ * d_);
  run_qpoints(job, which == 0 ? x.get() : nullptr, nullptr, which == 1 ? x.get() : nullptr,
              nullptr);
  return x.download();
}

void Operator::ensure_detw()
{
  if (cell_detw_.size() == (size_t)layout_.n_owned * nq_)
    return;
  cell_detw_.resize((size_t)layout_.n_owned * nq_);
  if (has_mapping_)
    {
      run_qpoints(mapping_job(), nullptr, cell_detw_.get(), nullptr, nullptr);
      return;
    }
  // host-array geometry (the reference's GeometryCache, no coefficient):
  // JxW is det(J) w_q, or det(J) for a compressed record
  if (sym_)
    fail(Code::invalid_argument,
         "assemble_rhs: a g4 host-array cache carries no JxW for the forcing");
  const std::vector<double> cg = cell_geo_.download();
  const int ncomp = d_ * d_ + 1;
  const Quad1D qg = gauss(k_);
  std::vector<double> dw((size_t)layout_.n_owned * nq_);
  for (long long c = 0; c < (long long)layout_.n_owned; ++c)
    for (long long q = 0; q < nq_; ++q)
      {
        if (!compressed_)
          dw[c * nq_ + q] = cg[(c * ncomp + d_ * d_) * nq_ + q];
        else
          {
            double w = 1.0;
            long long idx = q;
            for (int a = 0; a < d_; ++a)
              {
                w *= qg.weights[idx % k_];
                idx /= k_;
              }
            dw[c * nq_ + q] = cg[c * ncomp + d_ * d_] * w;
          }
      }
  cell_detw_.upload(dw);
}

void Operator::assemble_rhs(const double *f, const double *g, double *rhs, cudaStream_t s)
{
  if (host_only_)
    fail(Code::invalid_argument, "assemble_rhs: operator was created host-only");
  if (precision_ != 0)
    fail(Code::invalid_argument, "assemble_rhs: fp64 operators only");
  if (!rhs)
    fail(Code::invalid_argument, "assemble_rhs: null right-hand side");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  if (f)
    ensure_detw();
  // std::fill(rhs, 0) (operators.cpp:270-272): the ghost region stays zero
  cuda_check(cudaMemsetAsync(rhs, 0, sizeof(double) * layout_.total_size(), s), "memset");
  dev::RhsParams<double> prm;
  prm.f = f;
  prm.detw = cell_detw_.get();
  prm.g = g;
  prm.y = rhs;
  prm.face_geo = kind_ == 1 ? adv_face_.get() : face_geo_.get();
  prm.penalty = penalty_.get();
  prm.task_slot = task_slot_.get();
  prm.task_face = task_face_.get();
  prm.n_tasks = static_cast<int>(layout_.n_owned); // owned tasks come first
  launch_rhs(d_, k_, basis_, compressed_, kind_ == 1, prm, s);
}

std::vector<double> Operator::geometry(int which) const
{
  if (host_only_ && which != 3)
    fail(Code::invalid_argument, "geometry: operator was created host-only");
  switch (which)
    {
    case 0: return cell_geo_.download();
    case 1: return face_geo_.download();
    case 2: return penalty_.download();
    case 3:
      {
        std::vector<double> v(layout_.my_faces.begin(), layout_.my_faces.end());
        return v;
      }
    default: fail(Code::invalid_argument, "geometry: unknown array");
    }
}

dgx_stats Operator::stats() const
{
  dgx_stats st{};
  st.n_tasks_inner = n_inner_;
  st.n_tasks_coupled = n_coupled_;
  st.n_faces = (long long)layout_.my_faces.size();
  st.kernel_launches_per_apply = (n_inner_ > 0) + (n_coupled_ > 0);
  const double es = precision_ == 1 ? 4.0 : 8.0;
  st.bytes_vectors = 2.0 * es * (double)layout_.owned_size();
  st.bytes_cell_geometry = es * (double)(kind_ == 1 ? adv_cell_.size() : cell_geo_.size());
  st.bytes_face_geometry =
    es * (double)(kind_ == 1 ? adv_face_.size() : face_geo_.size() + penalty_.size());
  long long P = nq_ / k_;
  if (tensor_)
    {
      // dev::CartShape<Real, D, K, HERM>::NC
      st.cells_per_cta = d_ == 2 ? static_cast<int>(32 / P > 0 ? 32 / P : 1)
                         : ((k_ == 7 && precision_ == 0 && basis_ != 2) || k_ == 4)
                           ? 4
                           : static_cast<int>(192 / P > 0 ? 192 / P : 1);
      st.cartesian = 2;
    }
  else
    {
      st.cells_per_cta = kernel_cells_per_cta(d_, k_, cart_);
      st.cartesian = cart_ ? 1 : 0;
    }
  st.threads_per_cta = static_cast<int>(st.cells_per_cta * P);
  return st;
}

} // namespace dgx

// Host-side integer topology of the AIMx setup (S0): mesh validation, RWG
// basis, AIM grid, stencil anchors, near-region CSR, occupied-node map.
//
// P:177-178 RWG basis on pairs of adjacent triangles; P:188 regular grid on the
// bounding box; P:576 (n+1)^3 stencil; P:192 near-region entries.  Readings
// R2-R5 of DESIGN.md (RWG order/sign, grid rule, anchor rule, near metric).
// Compiled with -ffp-contract=off: the anchor arithmetic is one IEEE op at a
// time so that anchors are reproducible bit for bit.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "aimx_internal.h"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace aimx {

static void mesh_error(const std::string& m) { throw Error(AIMX_E_MESH, m); }
static void grid_error(const std::string& m) { throw Error(AIMX_E_GRID, m); }

static double tri_area2(const double* V, const int32_t* t) {
  const double* a = V + 3 * (int64_t)t[0];
  const double* b = V + 3 * (int64_t)t[1];
  const double* c = V + 3 * (int64_t)t[2];
  double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  double n0 = e1[1] * e2[2] - e1[2] * e2[1];
  double n1 = e1[2] * e2[0] - e1[0] * e2[2];
  double n2 = e1[0] * e2[1] - e1[1] * e2[0];
  return std::sqrt(n0 * n0 + n1 * n1 + n2 * n2);
}

void build_topology(const aimx_mesh_desc* mesh, const aimx_grid_desc* grid, Topology& t) {
  if (!mesh || !grid || !mesh->vertices || !mesh->triangles)
    throw Error(AIMX_E_INVALID_ARG, "null mesh or grid descriptor");
  if (mesh->nv <= 0 || mesh->nt <= 0) mesh_error("empty mesh");
  if (mesh->nt > (int64_t)INT32_MAX / 3 || mesh->nv > (int64_t)INT32_MAX)
    mesh_error("mesh too large for 32-bit indices");
  t.nv = mesh->nv;
  t.nt = mesh->nt;
  t.V.assign(mesh->vertices, mesh->vertices + 3 * t.nv);
  t.T.assign(mesh->triangles, mesh->triangles + 3 * t.nt);
  for (int64_t i = 0; i < 3 * t.nv; ++i)
    if (!std::isfinite(t.V[i])) mesh_error("non-finite vertex coordinate");
  for (int64_t f = 0; f < t.nt; ++f) {
    const int32_t* tr = &t.T[3 * f];
    for (int k = 0; k < 3; ++k)
      if (tr[k] < 0 || tr[k] >= t.nv) mesh_error("triangle index out of range");
    if (tr[0] == tr[1] || tr[1] == tr[2] || tr[0] == tr[2]) mesh_error("triangle with repeated vertex");
    if (!(tri_area2(t.V.data(), tr) > 0.0)) mesh_error("degenerate (zero-area) triangle");
  }

  // ---- RWG basis (reading R2) -----------------------------------------------
  struct DEdge { int32_t lo, hi; uint8_t back; int32_t tri, free; };
  std::vector<DEdge> de(3 * t.nt);
  for (int64_t f = 0; f < t.nt; ++f) {
    const int32_t* tr = &t.T[3 * f];
    for (int k = 0; k < 3; ++k) {
      int32_t u = tr[k], v = tr[(k + 1) % 3], w = tr[(k + 2) % 3];
      de[3 * f + k] = {std::min(u, v), std::max(u, v), (uint8_t)(u < v ? 0 : 1), (int32_t)f, w};
    }
  }
  std::sort(de.begin(), de.end(), [](const DEdge& a, const DEdge& b) {
    if (a.lo != b.lo) return a.lo < b.lo;
    if (a.hi != b.hi) return a.hi < b.hi;
    if (a.back != b.back) return a.back < b.back;
    return a.tri < b.tri;
  });
  for (size_t i = 0; i < de.size();) {
    size_t j = i;
    while (j < de.size() && de[j].lo == de[i].lo && de[j].hi == de[i].hi) ++j;
    size_t cnt = j - i;
    if (cnt > 2) mesh_error("non-manifold edge (more than two triangles)");
    if (cnt == 2) {
      if (de[i].back == de[i + 1].back) mesh_error("inconsistent triangle orientation");
      t.ea.push_back(de[i].lo);
      t.eb.push_back(de[i].hi);
      t.tp.push_back(de[i].tri);       // a->b
      t.pp.push_back(de[i].free);
      t.tm.push_back(de[i + 1].tri);   // b->a
      t.pm.push_back(de[i + 1].free);
    }
    i = j;
  }
  t.nb = (int64_t)t.ea.size();
  if (t.nb == 0) mesh_error("mesh has no interior edge (no RWG unknowns)");

  // ---- grid (reading R3) --------------------------------------------------------
  t.order = grid->order;
  t.near_cells = grid->near_cells;
  if (t.order < 1 || t.order > 3) grid_error("stencil order must be 1..3");
  if (t.near_cells < 0 || t.near_cells > 8) grid_error("near threshold must be 0..8 cells");
  t.p = t.order + 1;
  t.p3 = t.p * t.p * t.p;
  for (int a = 0; a < 3; ++a) {
    t.n[a] = grid->n[a];
    if (t.n[a] < t.p) grid_error("grid has fewer points than the stencil");
  }
  if ((int64_t)t.n[0] * t.n[1] * t.n[2] > (int64_t)INT32_MAX / 64) grid_error("grid too large");
  if (grid->h > 0.0) {
    t.h = grid->h;
    for (int a = 0; a < 3; ++a) t.origin[a] = grid->origin[a];
  } else {
    const int m = (t.order + 1) / 2;
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) { lo[a] = t.V[a]; hi[a] = t.V[a]; }
    for (int64_t i = 0; i < t.nv; ++i)
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], t.V[3 * i + a]);
        hi[a] = std::max(hi[a], t.V[3 * i + a]);
      }
    double h = 0.0;
    for (int a = 0; a < 3; ++a) {
      double ext = hi[a] - lo[a];
      int span = t.n[a] - 1 - 2 * m;
      if (ext > 0.0) {
        if (span <= 0) grid_error("grid too small for the mesh extent");
        h = std::max(h, ext / (double)span);
      }
    }
    if (!(h > 0.0)) grid_error("zero-extent mesh");
    t.h = h;
    for (int a = 0; a < 3; ++a) t.origin[a] = lo[a] - (double)m * h;
  }

  // ---- stencil anchors (reading R4; no FMA contraction in this file) --------------
  t.anchor.resize(3 * t.nb);
  const int half = t.order / 2;
  for (int64_t e = 0; e < t.nb; ++e) {
    for (int a = 0; a < 3; ++a) {
      double s1 = t.V[3 * (int64_t)t.ea[e] + a] + t.V[3 * (int64_t)t.eb[e] + a];
      s1 = s1 * 2.0;
      double s2 = t.V[3 * (int64_t)t.pp[e] + a] + t.V[3 * (int64_t)t.pm[e] + a];
      double c = s1 + s2;
      c = c / 6.0;
      double u = (c - t.origin[a]) / t.h;
      double A = (t.order % 2 == 0) ? std::floor(u + 0.5) - (double)half
                                    : std::floor(u) - (double)((t.order - 1) / 2);
      if (!(A >= 0.0) || A > (double)(t.n[a] - 1 - t.order))
        grid_error("stencil does not fit in the grid (RWG " + std::to_string(e) + ")");
      t.anchor[3 * e + a] = (int32_t)A;
    }
  }

  // ---- near-region CSR (reading R5): bucket RWGs by anchor cell ---------------------
  const int Nx = t.n[0], Ny = t.n[1], Nz = t.n[2];
  const int64_t ncell = (int64_t)Nx * Ny * Nz;
  std::vector<int32_t> cell_ptr(ncell + 1, 0), cell_rwg(t.nb);
  for (int64_t e = 0; e < t.nb; ++e) {
    int64_t c = t.anchor[3 * e] + (int64_t)Nx * (t.anchor[3 * e + 1] + (int64_t)Ny * t.anchor[3 * e + 2]);
    cell_ptr[c + 1]++;
  }
  for (int64_t c = 0; c < ncell; ++c) cell_ptr[c + 1] += cell_ptr[c];
  {
    std::vector<int32_t> fill(cell_ptr.begin(), cell_ptr.end() - 1);
    for (int64_t e = 0; e < t.nb; ++e) {
      int64_t c = t.anchor[3 * e] + (int64_t)Nx * (t.anchor[3 * e + 1] + (int64_t)Ny * t.anchor[3 * e + 2]);
      cell_rwg[fill[c]++] = (int32_t)e;   // ascending e within a cell
    }
  }
  const int R = t.order + t.near_cells;
  const int T2 = t.near_cells * t.near_cells;
  const int nthreads =
#ifdef _OPENMP
      omp_get_max_threads();
#else
      1;
#endif
  // two passes over rows in contiguous chunks: count, then fill sorted columns
  t.rowptr.assign(t.nb + 1, 0);
  auto row_cols = [&](int64_t m, std::vector<int32_t>& out) {
    out.clear();
    const int32_t* Am = &t.anchor[3 * m];
    for (int dz = -R; dz <= R; ++dz) {
      int z = Am[2] + dz;
      if (z < 0 || z >= Nz) continue;
      int gz = std::max(0, std::abs(dz) - t.order);
      for (int dy = -R; dy <= R; ++dy) {
        int y = Am[1] + dy;
        if (y < 0 || y >= Ny) continue;
        int gy = std::max(0, std::abs(dy) - t.order);
        for (int dx = -R; dx <= R; ++dx) {
          int x = Am[0] + dx;
          if (x < 0 || x >= Nx) continue;
          int gx = std::max(0, std::abs(dx) - t.order);
          if (gx * gx + gy * gy + gz * gz > T2) continue;
          int64_t c = x + (int64_t)Nx * (y + (int64_t)Ny * z);
          for (int32_t k = cell_ptr[c]; k < cell_ptr[c + 1]; ++k) out.push_back(cell_rwg[k]);
        }
      }
    }
    std::sort(out.begin(), out.end());
  };
#pragma omp parallel num_threads(nthreads)
  {
    std::vector<int32_t> buf;
#pragma omp for schedule(dynamic, 256)
    for (int64_t m = 0; m < t.nb; ++m) {
      row_cols(m, buf);
      t.rowptr[m + 1] = (int64_t)buf.size();
    }
  }
  for (int64_t m = 0; m < t.nb; ++m) t.rowptr[m + 1] += t.rowptr[m];
  const int64_t nnz = t.rowptr[t.nb];
  if (nnz > (int64_t)INT32_MAX) grid_error("near-region matrix exceeds 2^31 entries");
  t.col.resize(nnz);
#pragma omp parallel num_threads(nthreads)
  {
    std::vector<int32_t> buf;
#pragma omp for schedule(dynamic, 256)
    for (int64_t m = 0; m < t.nb; ++m) {
      row_cols(m, buf);
      std::copy(buf.begin(), buf.end(), t.col.begin() + t.rowptr[m]);
    }
  }
}

// Overlapping pairs for the linear-term modification (reading R21):
// n is listed in row m when the supports of f_m and f_n share a triangle.
// A triangle carries at most 3 RWGs, so a row holds at most 1 + 2 + 2 columns.
void build_overlap(const Topology& t, std::vector<int32_t>& cols) {
  std::vector<int32_t> cnt(t.nt + 1, 0);
  for (int64_t e = 0; e < t.nb; ++e) { ++cnt[t.tp[e] + 1]; ++cnt[t.tm[e] + 1]; }
  for (int64_t i = 0; i < t.nt; ++i) cnt[i + 1] += cnt[i];
  std::vector<int32_t> by_tri(cnt[t.nt]), fill(cnt.begin(), cnt.end() - 1);
  for (int64_t e = 0; e < t.nb; ++e) {
    by_tri[fill[t.tp[e]]++] = (int32_t)e;
    by_tri[fill[t.tm[e]]++] = (int32_t)e;
  }
  cols.assign((size_t)t.nb * kLinW, -1);
  std::vector<int32_t> u;
  for (int64_t e = 0; e < t.nb; ++e) {
    u.clear();
    for (int32_t tri : {t.tp[e], t.tm[e]})
      for (int32_t k = cnt[tri]; k < cnt[tri + 1]; ++k) u.push_back(by_tri[k]);
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    if ((int)u.size() > kLinW) throw Error(AIMX_E_MESH, "more than 3 RWG edges on a triangle");
    std::copy(u.begin(), u.end(), cols.begin() + e * kLinW);
  }
}

void build_nodemap(const Topology& t, const std::vector<uint8_t>& nz_slot, NodeMap& m) {
  const int Nx = t.n[0], Ny = t.n[1], Nz = t.n[2];
  const int p = t.p, p3 = t.p3;
  const int64_t ng = (int64_t)Nx * Ny * Nz;
  std::vector<int32_t> cnt(ng + 1, 0);
  auto node_of = [&](int64_t e, int s) -> int64_t {
    int i = s % p, j = (s / p) % p, k = s / (p * p);
    const int32_t* A = &t.anchor[3 * e];
    return (A[0] + i) + (int64_t)Nx * ((A[1] + j) + (int64_t)Ny * (A[2] + k));
  };
  for (int64_t e = 0; e < t.nb; ++e)
    for (int s = 0; s < p3; ++s)
      if (nz_slot[e * p3 + s]) cnt[node_of(e, s) + 1]++;
  for (int64_t q = 0; q < ng; ++q) cnt[q + 1] += cnt[q];
  const int64_t nent = cnt[ng];
  std::vector<int32_t> er(nent), es(nent);
  {
    std::vector<int32_t> fill(cnt.begin(), cnt.end() - 1);
    for (int64_t e = 0; e < t.nb; ++e)
      for (int s = 0; s < p3; ++s)
        if (nz_slot[e * p3 + s]) {
          int64_t q = node_of(e, s);
          er[fill[q]] = (int32_t)e;
          es[fill[q]] = s;
          fill[q]++;
        }
  }
  m.node_lin.clear();
  m.node_ptr.clear();
  m.node_line.clear();
  m.line_id.clear();
  m.line_ptr.clear();
  m.zplanes.clear();
  m.line_occ.assign((size_t)Ny * Nz, 0);
  m.node_ptr.push_back(0);
  for (int64_t q = 0; q < ng; ++q) {
    if (cnt[q + 1] == cnt[q]) continue;
    int32_t line = (int32_t)(q / Nx);
    if (m.line_id.empty() || m.line_id.back() != line) {
      m.line_id.push_back(line);
      m.line_ptr.push_back((int32_t)m.node_lin.size());
      m.line_occ[line] = 1;
      int z = line / Ny;
      if (m.zplanes.empty() || m.zplanes.back() != z) m.zplanes.push_back(z);
    }
    m.node_lin.push_back((int32_t)q);
    m.node_line.push_back((int32_t)m.line_id.size() - 1);
    m.node_ptr.push_back(cnt[q + 1]);
  }
  m.line_ptr.push_back((int32_t)m.node_lin.size());
  m.ent_rwg.swap(er);
  m.ent_slot.swap(es);
  (void)Nz;
}

}  // namespace aimx

namespace aimx {

// ---- near matrix in row-group form (hot-path layout of C) ----
// Rows (testing RWGs) are ordered spatially by their stencil anchor and cut
// into groups of R consecutive rows.  A group stores the sorted union of its
// rows' near columns once; each union entry carries R (C_A, C_rho) pairs, zero
// where the pair (row, column) is not near.  A column's x values are then read
// once for R rows.  Near-ness depends only on the anchors (reading R5), so rows
// with close anchors have nearly equal column sets.

static uint32_t spread3(uint32_t v) {   // 10 bits -> every third bit
  v &= 0x3ff;
  v = (v | (v << 16)) & 0x030000ff;
  v = (v | (v << 8)) & 0x0300f00f;
  v = (v | (v << 4)) & 0x030c30c3;
  v = (v | (v << 2)) & 0x09249249;
  return v;
}

// rows (a subset of the RWGs, all if `sub` is empty) ordered by anchor key
static std::vector<int32_t> row_order(const Topology& t, int kind, const std::vector<int32_t>& sub) {
  std::vector<int32_t> p;
  if (sub.empty()) {
    p.resize(t.nb);
    std::iota(p.begin(), p.end(), 0);
  } else {
    p = sub;
  }
  auto key = [&](int32_t e) -> int64_t {
    const int32_t* A = &t.anchor[3 * (int64_t)e];
    return kind == 0 ? (int64_t)A[0] + (int64_t)t.n[0] * ((int64_t)A[1] + (int64_t)t.n[1] * A[2])
                     : (int64_t)(spread3(A[0]) | (spread3(A[1]) << 1) | (spread3(A[2]) << 2));
  };
  std::stable_sort(p.begin(), p.end(), [&](int32_t a, int32_t b) { return key(a) < key(b); });
  return p;
}

static void group_union(const Topology& t, const std::vector<int32_t>& p, int64_t g, int R,
                        std::vector<int32_t>& u) {
  u.clear();
  const int64_t nr = (int64_t)p.size();
  for (int r = 0; r < R; ++r) {
    const int64_t i = g * R + r;
    if (i >= nr) break;
    const int32_t m = p[i];
    u.insert(u.end(), t.col.begin() + t.rowptr[m], t.col.begin() + t.rowptr[m + 1]);
  }
  std::sort(u.begin(), u.end());
  u.erase(std::unique(u.begin(), u.end()), u.end());
}

void build_near_groups(const Topology& t, const std::vector<uint8_t>& nz_slot, NearGroups& ng,
                       const std::vector<int32_t>& rows) {
  const int64_t nb = rows.empty() ? t.nb : (int64_t)rows.size();   // rows in the groups
  // candidate (ordering, R): union sizes estimated on a sample of groups, cost
  // model = HBM bytes + FMA issue + x-row loads of a 16-column c64 SpMM
  int best_kind = 0, best_R = 8;
  double best = 1e300;
  const char* eR = std::getenv("AIMX_NEAR_R");
  const char* eK = std::getenv("AIMX_NEAR_ORDER");
  std::vector<int32_t> perm[2] = {row_order(t, 0, rows), row_order(t, 1, rows)};
  // every anchor in one z plane (planar meshes, cfg5): the linear order, a
  // band of grid rows per round of groups, measured faster than Morton order
  // (cfg5, 32 columns: S4+S5 0.783 -> 0.748 ms in the serial stage profile,
  // bench step 3.93 -> 3.87 ms)
  bool one_plane = true;
  for (int64_t e = 1; e < t.nb && one_plane; ++e) one_plane = t.anchor[3 * e + 2] == t.anchor[2];
  for (int kind = 0; kind < 2; ++kind) {
    if (eK ? std::atoi(eK) != kind : (one_plane && kind == 1)) continue;
    for (int R : {4, 8, 16}) {
      if (eR ? std::atoi(eR) != R : R == 16) continue;   // 16: opt-in (AIMX_NEAR_R=16)
      const int64_t ngrp = (nb + R - 1) / R;
      const int64_t stride = std::max<int64_t>(1, ngrp / 4096);
      int64_t U = 0, ns = 0;
#pragma omp parallel reduction(+ : U, ns)
      {
        std::vector<int32_t> u;
#pragma omp for schedule(dynamic, 16)
        for (int64_t g = 0; g < ngrp; g += stride) {
          group_union(t, perm[kind], g, R, u);
          U += (int64_t)u.size();
          ns += 1;
        }
      }
      const double Ue = (double)U * (double)ngrp / (double)std::max<int64_t>(ns, 1);
      // Morton order keeps the gathered x / potential rows of a CTA's groups
      // local in 2-D and 3-D, which the union size does not see: measured,
      // it wins whenever its union is within ~4% (cfg3, cfg5), not at 5%
      // (cfg2's strips)
      const double cost = (Ue * (4.0 + 8.0 * R) / 6.0 + Ue * R * 48.0 / 18.0 + Ue * 128.0 / 18.0) *
                          (kind == 1 ? 0.96 : 1.0);
      if (cost < best) { best = cost; best_kind = kind; best_R = R; }
    }
  }
  const int R = best_R;
  const std::vector<int32_t>& p = perm[best_kind];
  const int64_t ngrp = (nb + R - 1) / R;
  const int Nx = t.n[0], Ny = t.n[1], pp = t.p, p3 = t.p3;
  ng.R = R;
  ng.order_kind = best_kind;
  ng.ngrp = ngrp;
  ng.rows.assign(ngrp * R, -1);
  for (int64_t i = 0; i < nb; ++i) ng.rows[i] = p[i];
  // stencil node (linear grid index) of slot s of RWG e
  auto node_of = [&](int64_t e, int sl) -> int32_t {
    const int32_t* A = &t.anchor[3 * e];
    return (A[0] + sl % pp) + Nx * ((A[1] + (sl / pp) % pp) + Ny * (A[2] + sl / (pp * pp)));
  };
  auto w_union = [&](int64_t g, std::vector<int32_t>& u) {
    u.clear();
    for (int r = 0; r < R; ++r) {
      const int64_t i = g * R + r;
      if (i >= nb) break;
      const int32_t m = p[i];
      for (int sl = 0; sl < p3; ++sl)
        if (nz_slot[(int64_t)m * p3 + sl]) u.push_back(node_of(m, sl));
    }
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
  };
  ng.ptr.assign(ngrp + 1, 0);
  ng.wptr.assign(ngrp + 1, 0);
#pragma omp parallel
  {
    std::vector<int32_t> u;
#pragma omp for schedule(dynamic, 64)
    for (int64_t g = 0; g < ngrp; ++g) {
      group_union(t, p, g, R, u);
      ng.ptr[g + 1] = (int64_t)u.size();
      w_union(g, u);
      ng.wptr[g + 1] = (int64_t)u.size();
    }
  }
  // unions padded to a multiple of 4 entries (16-byte aligned index blocks;
  // padding entries carry zero coefficients)
  for (int64_t g = 0; g < ngrp; ++g) {
    ng.ptr[g + 1] = ng.ptr[g] + ((ng.ptr[g + 1] + 3) & ~(int64_t)3);
    ng.wptr[g + 1] = ng.wptr[g] + ((ng.wptr[g + 1] + 3) & ~(int64_t)3);
  }
  const int64_t U = ng.ptr[ngrp], Uw = ng.wptr[ngrp];
  if (U * R > (int64_t)INT32_MAX * 4) throw Error(AIMX_E_GRID, "near matrix too large for the row-group layout");
  ng.ucol.resize(U);
  ng.slot.assign(t.rowptr[t.nb], -1);
  ng.wnode.resize(Uw);
  ng.wslot.assign(t.nb * p3, -1);
#pragma omp parallel
  {
    std::vector<int32_t> u;
#pragma omp for schedule(dynamic, 64)
    for (int64_t g = 0; g < ngrp; ++g) {
      group_union(t, p, g, R, u);
      const int64_t u0 = ng.ptr[g];
      std::copy(u.begin(), u.end(), ng.ucol.begin() + u0);
      std::fill(ng.ucol.begin() + u0 + (int64_t)u.size(), ng.ucol.begin() + ng.ptr[g + 1], u.empty() ? 0 : u[0]);
      for (int r = 0; r < R; ++r) {
        const int64_t i = g * R + r;
        if (i >= nb) break;
        const int32_t m = p[i];
        size_t pos = 0;
        for (int64_t k = t.rowptr[m]; k < t.rowptr[m + 1]; ++k) {   // both sorted: two pointers
          while (u[pos] != t.col[k]) ++pos;
          ng.slot[k] = (u0 + (int64_t)pos) * R + r;
        }
      }
      w_union(g, u);
      const int64_t w0 = ng.wptr[g];
      std::copy(u.begin(), u.end(), ng.wnode.begin() + w0);
      std::fill(ng.wnode.begin() + w0 + (int64_t)u.size(), ng.wnode.begin() + ng.wptr[g + 1], u.empty() ? 0 : u[0]);
      for (int r = 0; r < R; ++r) {
        const int64_t i = g * R + r;
        if (i >= nb) break;
        const int32_t m = p[i];
        for (int sl = 0; sl < p3; ++sl)
          if (nz_slot[(int64_t)m * p3 + sl]) {
            const int64_t pos = std::lower_bound(u.begin(), u.end(), node_of(m, sl)) - u.begin();
            ng.wslot[(int64_t)m * p3 + sl] = (w0 + pos) * R + r;
          }
      }
    }
  }
}

void build_near_chunks(const NearGroups& ng, int chw, int chc, int cs, NearChunks& ck,
                       const std::vector<int64_t>& order) {
  // chunk list in `order` (all groups, each once): the group's W
  // (interpolation) chunks, then its C (near) chunks; every group gets at
  // least one chunk (its epilogue).
  const int R = ng.R;
  if ((int64_t)order.size() != ng.ngrp) throw Error(AIMX_E_INTERNAL, "near group order");
  ck.chunks.clear();
  ck.gfirst.assign(ng.ngrp + 1, 0);
  ck.cost.assign(ng.ngrp, 0.0);
  ck.uoff_c.assign(ng.ptr[ng.ngrp], 0);
  ck.uoff_w.assign(ng.wptr[ng.ngrp], 0);
  int64_t off = 0;   // payload bytes so far
  std::vector<int64_t> poff;
  auto pad16 = [](int64_t x) { return (x + 15) & ~(int64_t)15; };
  for (int64_t gi = 0; gi < ng.ngrp; ++gi) {
    const int64_t g = order[gi];
    ck.gfirst[g] = (int64_t)ck.chunks.size() / 4;
    const int64_t n0 = ck.chunks.size();
    for (int kind = 0; kind < 2; ++kind) {
      const int64_t b = kind ? ng.ptr[g] : ng.wptr[g], e = kind ? ng.ptr[g + 1] : ng.wptr[g + 1];
      const int ch = kind ? chc : chw;
      const int eb = R * (kind ? cs : 2 * cs);   // coefficient bytes per entry
      for (int64_t u = b; u < e; u += ch) {
        const int64_t n = std::min<int64_t>(ch, e - u);
        for (int64_t i = 0; i < n; ++i) (kind ? ck.uoff_c : ck.uoff_w)[u + i] = off + i * eb;
        ck.chunks.insert(ck.chunks.end(), {(int32_t)g, kind, (int32_t)u, (int32_t)n});
        poff.push_back(off);
        off += n * eb + pad16(4 * n) + 16;
      }
    }
    if ((int64_t)ck.chunks.size() == n0) {
      ck.chunks.insert(ck.chunks.end(), {(int32_t)g, 1, 0, 0});
      poff.push_back(off);
      off += 16;
    }
    ck.chunks[n0 + 1] |= 2;                          // first chunk of the group
    ck.chunks[ck.chunks.size() - 3] |= 4;            // last chunk of the group
    ck.cost[g] = 4.0 * (ng.wptr[g + 1] - ng.wptr[g]) + (ng.ptr[g + 1] - ng.ptr[g]) + 32.0;
  }
  ck.nchunk = (int64_t)ck.chunks.size() / 4;
  if (off / 16 > (int64_t)INT32_MAX) throw Error(AIMX_E_GRID, "near matrix payload too large");
  // payload: per chunk [coefficients | row indices (16-byte padded) | descriptor of chunk + kNearD]
  const int64_t nchunk = (int64_t)ck.chunks.size() / 4;
  ck.payload.assign(off, 0);
  for (int64_t c = 0; c < nchunk; ++c) {
    const int32_t* d = &ck.chunks[4 * c];
    const int kind = d[1] & 1;
    const int64_t n = d[3];
    const int eb = R * (kind ? cs : 2 * cs);
    unsigned char* p = ck.payload.data() + poff[c] + n * eb;
    const int32_t* src = (kind ? ng.ucol.data() : ng.wnode.data()) + d[2];
    std::memcpy(p, src, 4 * n);
    p += pad16(4 * n);
    if (c + kNearD < nchunk) {
      int32_t nd[4] = {ck.chunks[4 * (c + kNearD)], ck.chunks[4 * (c + kNearD) + 1],
                       (int32_t)(poff[c + kNearD] / 16), ck.chunks[4 * (c + kNearD) + 3]};
      std::memcpy(p, nd, 16);
    }
  }
  for (int64_t c = 0; c < nchunk; ++c) ck.chunks[4 * c + 2] = (int32_t)(poff[c] / 16);
}

std::vector<int64_t> near_round_order(int64_t ngrp, int ncta, std::vector<int64_t>& cta_begin) {
  // Groups are spatially ordered (anchor Morton code or linear index), so a
  // run of consecutive groups shares most of its stencil nodes and near
  // columns.  Round r = groups [r ncta, (r + 1) ncta); CTA k takes the k-th
  // group of every round.  All CTAs advance through the rounds together, so
  // the gathered rows in use at any time (x: B columns per RWG, phi: 4 B per
  // node) are one round's neighbourhood and stay in L2, whatever B is; with
  // contiguous per-CTA ranges the CTAs would touch the whole grid at once
  // (cfg5 at 32 columns: 2.3 GB of DRAM reads against 1.2 GB of coefficients).
  ncta = (int)std::max<int64_t>(1, std::min<int64_t>(ncta, ngrp));
  std::vector<int64_t> order;
  order.reserve(ngrp);
  cta_begin.assign(ncta + 1, 0);
  for (int k = 0; k < ncta; ++k) {
    cta_begin[k] = (int64_t)order.size();
    for (int64_t g = k; g < ngrp; g += ncta) order.push_back(g);
  }
  cta_begin[ncta] = ngrp;
  return order;
}


// Nodes of rows [y0, y1) only, lines renumbered locally: (y - y0) + (y1 - y0) z.
void nodemap_rows(const Topology& t, const NodeMap& full, int y0, int y1, NodeMap& m) {
  const int Nx = t.n[0], Ny = t.n[1], Nz = t.n[2], ny = y1 - y0;
  m = NodeMap{};
  m.line_occ.assign((size_t)ny * Nz, 0);
  m.node_ptr.push_back(0);
  for (size_t q = 0; q < full.node_lin.size(); ++q) {
    const int32_t lin = full.node_lin[q];
    const int y = (lin / Nx) % Ny, z = lin / (Nx * Ny);
    if (y < y0 || y >= y1) continue;
    const int32_t line = (y - y0) + ny * z;
    if (m.line_id.empty() || m.line_id.back() != line) {
      m.line_id.push_back(line);
      m.line_ptr.push_back((int32_t)m.node_lin.size());
      m.line_occ[line] = 1;
      if (m.zplanes.empty() || m.zplanes.back() != z) m.zplanes.push_back(z);
    }
    m.node_lin.push_back(lin);
    m.node_line.push_back((int32_t)m.line_id.size() - 1);
    for (int32_t e = full.node_ptr[q]; e < full.node_ptr[q + 1]; ++e) {
      m.ent_rwg.push_back(full.ent_rwg[e]);
      m.ent_slot.push_back(full.ent_slot[e]);
    }
    m.node_ptr.push_back((int32_t)m.ent_rwg.size());
  }
  m.line_ptr.push_back((int32_t)m.node_lin.size());
}

}  // namespace aimx

extern "C" aimx_status aimx_slab_plan(const int32_t n[3], int32_t order, int32_t world, int32_t rank,
                                      int32_t out[6]) {
  if (!n || !out || world < 1 || rank < 0 || rank >= world || order < 1) return AIMX_E_INVALID_ARG;
  const int Lx = 2 * n[0];
  if (Lx % world != 0 || ((Lx / world) & (Lx / world - 1)) != 0) return AIMX_E_UNSUPPORTED;
  if (n[1] < world) return AIMX_E_UNSUPPORTED;
  // rows: contiguous near-equal blocks of the unpadded y axis; phi rows extend
  // `order` rows past the block (stencils of RWGs anchored in it); kx: equal slabs
  const int base = n[1] / world, rem = n[1] % world;
  const int y0 = rank * base + (rank < rem ? rank : rem);
  const int y1 = y0 + base + (rank < rem ? 1 : 0);
  out[0] = y0;
  out[1] = y1;
  out[2] = y1 + order < n[1] ? y1 + order : n[1];
  out[3] = rank * (Lx / world);
  out[4] = (rank + 1) * (Lx / world);
  out[5] = 0;
  return AIMX_OK;
}

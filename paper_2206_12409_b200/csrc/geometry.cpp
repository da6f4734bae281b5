// RWG extraction and source tables (PAPER.md P:78 RWG basis on a triangular
// tessellation; P:106 Petrov-Galerkin coupling; SURVEY §8c-L10 canonical order,
// §8c-E source nodes and moment vectors, §8c-L18 non-singular check).
#include "geometry.hpp"

#include <algorithm>
#include <cmath>
#include <string>

namespace vsie {

GridDesc make_grid(const vsie_grid* g) {
  VSIE_REQUIRE(g != nullptr, VSIE_ERR_ARG, "grid is NULL");
  GridDesc d;
  for (int a = 0; a < 3; ++a) {
    VSIE_REQUIRE(g->n[a] > 0, VSIE_ERR_ARG, "grid n must be > 0");
    VSIE_REQUIRE(g->h[a] > 0 && std::isfinite(g->h[a]), VSIE_ERR_ARG, "grid h must be > 0");
    VSIE_REQUIRE(std::isfinite(g->origin[a]), VSIE_ERR_ARG, "grid origin must be finite");
    d.n[a] = g->n[a];
    d.h[a] = g->h[a];
    d.origin[a] = g->origin[a];
  }
  return d;
}

namespace {

struct EdgeRec {
  uint64_t key;  // (min vid << 32) | max vid
  int64_t tri;
  int64_t opp;   // vertex opposite the edge in `tri`
};

}  // namespace

std::vector<RwgRec> extract_rwgs(const vsie_mesh& mesh) {
  VSIE_REQUIRE(mesh.xyz != nullptr && mesh.tri != nullptr, VSIE_ERR_ARG, "mesh arrays are NULL");
  VSIE_REQUIRE(mesh.n_vertices >= 3 && mesh.n_triangles >= 1, VSIE_ERR_ARG, "mesh too small");
  VSIE_REQUIRE(mesh.n_vertices < (int64_t(1) << 31), VSIE_ERR_ARG, "too many vertices");
  const double* X = mesh.xyz;
  const int32_t* T = mesh.tri;
  const int64_t nt = mesh.n_triangles, nv = mesh.n_vertices;
  for (int64_t i = 0; i < 3 * nv; ++i)
    VSIE_REQUIRE(std::isfinite(X[i]), VSIE_ERR_GEOMETRY, "non-finite vertex coordinate");
  std::vector<EdgeRec> recs;
  recs.reserve(3 * nt);
  for (int64_t t = 0; t < nt; ++t) {
    int64_t v[3] = {T[3 * t], T[3 * t + 1], T[3 * t + 2]};
    for (int k = 0; k < 3; ++k)
      VSIE_REQUIRE(v[k] >= 0 && v[k] < nv, VSIE_ERR_GEOMETRY,
                   "triangle " + std::to_string(t) + " has a vertex id out of range");
    double e1[3], e2[3];
    for (int c = 0; c < 3; ++c) {
      e1[c] = X[3 * v[1] + c] - X[3 * v[0] + c];
      e2[c] = X[3 * v[2] + c] - X[3 * v[0] + c];
    }
    double cx = e1[1] * e2[2] - e1[2] * e2[1];
    double cy = e1[2] * e2[0] - e1[0] * e2[2];
    double cz = e1[0] * e2[1] - e1[1] * e2[0];
    double area2 = std::sqrt(cx * cx + cy * cy + cz * cz);
    VSIE_REQUIRE(area2 > 0, VSIE_ERR_GEOMETRY, "degenerate triangle " + std::to_string(t));
    for (int k = 0; k < 3; ++k) {
      uint64_t a = (uint64_t)v[(k + 1) % 3], b = (uint64_t)v[(k + 2) % 3];
      VSIE_REQUIRE(a != b, VSIE_ERR_GEOMETRY, "repeated vertex in triangle " + std::to_string(t));
      uint64_t lo = std::min(a, b), hi = std::max(a, b);
      recs.push_back({(lo << 32) | hi, t, v[k]});
    }
  }
  std::sort(recs.begin(), recs.end(), [](const EdgeRec& p, const EdgeRec& q) {
    return p.key != q.key ? p.key < q.key : p.tri < q.tri;
  });
  std::vector<RwgRec> out;
  size_t i = 0;
  while (i < recs.size()) {
    size_t j = i + 1;
    while (j < recs.size() && recs[j].key == recs[i].key) ++j;
    VSIE_REQUIRE(j - i <= 2, VSIE_ERR_GEOMETRY, "edge shared by more than two triangles");
    if (j - i == 2) {
      const EdgeRec& P = recs[i];      // T+ : smaller triangle id
      const EdgeRec& M = recs[i + 1];  // T-
      out.push_back({P.tri, M.tri, P.opp, M.opp, (int64_t)(P.key >> 32), (int64_t)(P.key & 0xffffffffu)});
    }
    i = j;
  }
  return out;
}

namespace {

void append_mesh(const vsie_mesh& mesh, std::vector<double>& table, int tri_points) {
  const double* X = mesh.xyz;
  const int32_t* T = mesh.tri;
  // barycentric interior rule (2/3, 1/6, 1/6) and permutations
  const double b_hi = 2.0 / 3.0, b_lo = 1.0 / 6.0;
  for (const RwgRec& r : extract_rwgs(mesh)) {
    double l = 0;
    for (int c = 0; c < 3; ++c) {
      double d = X[3 * r.a + c] - X[3 * r.b + c];
      l += d * d;
    }
    l = std::sqrt(l);
    const double coef = l / 6.0;
    double rec[kSrcStride];
    if (tri_points == 1) {
      // one point per triangle (the paper's far-block rule): the centroid with the
      // whole triangle's weight, J = +-(l/2)(r_c - p); records 0 (T+) and 1 (T-), the other
      // four records carry J = 0 (the kernel reads only the first two, EntryGeom::nsrc)
      for (int side = 0; side < 2; ++side) {
        const int64_t tri = side == 0 ? r.tp : r.tm, opp = side == 0 ? r.pp : r.pm;
        double* o = rec + 6 * side;
        for (int c = 0; c < 3; ++c) {
          const double rr = (X[3 * T[3 * tri] + c] + X[3 * T[3 * tri + 1] + c] + X[3 * T[3 * tri + 2] + c]) / 3.0;
          const double p = X[3 * opp + c];
          o[c] = rr;
          o[3 + c] = side == 0 ? 0.5 * l * (rr - p) : 0.5 * l * (p - rr);
        }
      }
      for (int q = 2; q < kSrcPerRwg; ++q)
        for (int c = 0; c < 6; ++c) rec[6 * q + c] = c < 3 ? rec[c] : 0.0;
      table.insert(table.end(), rec, rec + kSrcStride);
      continue;
    }
    for (int side = 0; side < 2; ++side) {
      const int64_t tri = side == 0 ? r.tp : r.tm, opp = side == 0 ? r.pp : r.pm;
      const int64_t v0 = T[3 * tri], v1 = T[3 * tri + 1], v2 = T[3 * tri + 2];
      for (int q = 0; q < 3; ++q) {
        const double w0 = q == 0 ? b_hi : b_lo, w1 = q == 1 ? b_hi : b_lo, w2 = q == 2 ? b_hi : b_lo;
        double* o = rec + 6 * (3 * side + q);
        for (int c = 0; c < 3; ++c) {
          const double rr = w0 * X[3 * v0 + c] + w1 * X[3 * v1 + c] + w2 * X[3 * v2 + c];
          const double p = X[3 * opp + c];
          o[c] = rr;
          o[3 + c] = side == 0 ? coef * (rr - p) : coef * (p - rr);  // J+ = l/6 (r - p+), J- = l/6 (p- - r)
        }
      }
    }
    table.insert(table.end(), rec, rec + kSrcStride);
  }
}

}  // namespace

Sources build_rwg_sources(const vsie_mesh* meshes, int n_meshes, int tri_points) {
  VSIE_REQUIRE(meshes != nullptr && n_meshes >= 1, VSIE_ERR_ARG, "no meshes");
  VSIE_REQUIRE(tri_points == 3 || tri_points == 1, VSIE_ERR_ARG, "triangle rule must have 3 or 1 points");
  Sources s;
  for (int k = 0; k < n_meshes; ++k) append_mesh(meshes[k], s.table, tri_points);
  s.m = (int64_t)(s.table.size() / kSrcStride);
  VSIE_REQUIRE(s.m >= 1, VSIE_ERR_GEOMETRY, "meshes have no interior edge (no RWG function)");
  return s;
}

double max_edge_length(const vsie_mesh* meshes, int n_meshes) {
  double best = 0;
  for (int k = 0; k < n_meshes; ++k) {
    const double* X = meshes[k].xyz;
    const int32_t* T = meshes[k].tri;
    for (int64_t t = 0; t < meshes[k].n_triangles; ++t)
      for (int e = 0; e < 3; ++e) {
        const int64_t a = T[3 * t + e], b = T[3 * t + (e + 1) % 3];
        double d2 = 0;
        for (int c = 0; c < 3; ++c) d2 += (X[3 * a + c] - X[3 * b + c]) * (X[3 * a + c] - X[3 * b + c]);
        best = std::max(best, std::sqrt(d2));
      }
  }
  return best;
}

Sources build_sources(const vsie_mesh* meshes, int n_meshes, const GridDesc& grid, int tri_points) {
  Sources s = build_rwg_sources(meshes, n_meshes, tri_points);
  // Non-singular rule (reading R-L18): every source node must be at
  // least 10 max(h) away from the bounding box of the voxel quadrature nodes.
  double lo[3], hi[3], hmax = 0;
  for (int a = 0; a < 3; ++a) {
    const double off = grid.h[a] / (2.0 * std::sqrt(3.0));
    lo[a] = grid.origin[a] - off;
    hi[a] = grid.origin[a] + (grid.n[a] - 1) * grid.h[a] + off;
    hmax = std::max(hmax, grid.h[a]);
  }
  double best = 1e300;
  for (int64_t n = 0; n < s.m; ++n) {
    for (int q = 0; q < kSrcPerRwg; ++q) {
      const double* r = &s.table[kSrcStride * n + 6 * q];
      double d2 = 0;
      for (int a = 0; a < 3; ++a) {
        double d = std::max(0.0, std::max(lo[a] - r[a], r[a] - hi[a]));
        d2 += d * d;
      }
      best = std::min(best, std::sqrt(d2));
    }
  }
  s.min_box_distance = best;
  VSIE_REQUIRE(best >= 10.0 * hmax, VSIE_ERR_GEOMETRY,
               "source nodes closer than 10 max(h) to the voxel grid (non-singular quadrature rule)");
  return s;
}

}  // namespace vsie

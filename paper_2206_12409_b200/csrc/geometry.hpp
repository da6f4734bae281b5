// Host-side geometry preprocessing: RWG extraction from the
// far-domain triangle meshes and the per-RWG source table uploaded to HBM.
#pragma once

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace vsie {

// 6 source nodes per RWG (3 on T+, 3 on T-), each (r_x, r_y, r_z, J_x, J_y, J_z):
// 36 doubles = 288 bytes per RWG, RWG-major (AoS) so that one entry's sources
// are 2.25 contiguous 128-B lines.
constexpr int kSrcPerRwg = 6;
constexpr int kSrcStride = 36;

struct Sources {
  int64_t m = 0;
  std::vector<double> table;     // [m][36]
  double min_box_distance = 0;   // to the voxel-node bounding box
};

struct GridDesc {
  int n[3];
  double h[3];
  double origin[3];
  int64_t nv() const { return (int64_t)n[0] * n[1] * n[2]; }
};

// Validates and converts the public structs; throws Error(VSIE_ERR_ARG / VSIE_ERR_GEOMETRY).
GridDesc make_grid(const vsie_grid* g);
// tri_points: 3 (interior rule, default) or 1 (centroid; the paper's far-block rule)
Sources build_sources(const vsie_mesh* meshes, int n_meshes, const GridDesc& grid, int tri_points = 3);
// One RWG function of a mesh (canonical order): T+ / T- triangle ids, the
// vertices opposite the shared edge (p+, p-) and the shared edge's vertices (a < b).
struct RwgRec {
  int64_t tp, tm, pp, pm, a, b;
};
// Validates one mesh (degenerate / non-manifold -> VSIE_ERR_GEOMETRY) and lists its RWGs.
std::vector<RwgRec> extract_rwgs(const vsie_mesh& mesh);
// The RWG table alone (no voxel-grid check): the surface-surface blocks (farnear.cu).
Sources build_rwg_sources(const vsie_mesh* meshes, int n_meshes, int tri_points = 3);
// Longest triangle edge of the meshes (validated by build_rwg_sources first).
double max_edge_length(const vsie_mesh* meshes, int n_meshes);

}  // namespace vsie

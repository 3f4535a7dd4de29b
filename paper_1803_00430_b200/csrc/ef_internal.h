// Internal structures shared by the host builder and the CUDA kernels.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/echoforge_b200.h"

namespace ef {

constexpr int kMaxBands = 8;
constexpr int kMaxOrder = 4;
constexpr int kBruteMaxTris = 512;   // scene.py:29
constexpr double kRayEps = 1e-4;     // scene.py:22
constexpr int kStackSize = 64;
constexpr int kMaxLeaf = 4;

// Two-child BVH node, 64 bytes (four 16-byte vectors):
//   a = (c0.lo.x, c0.hi.x, c0.lo.y, c0.hi.y)
//   b = (c1.lo.x, c1.hi.x, c1.lo.y, c1.hi.y)
//   c = (c0.lo.z, c0.hi.z, c1.lo.z, c1.hi.z)
//   d = (child0, child1, -, -)  child >= 0: inner node index,
//                               child <  0: leaf ~((start << 3) | (count - 1))
struct alignas(16) GpuNode {
    float a[4];
    float b[4];
    float c[4];
    int32_t d[4];
};
static_assert(sizeof(GpuNode) == 64, "node must be 64 bytes");

// f64 triangle payload in BVH leaf order, 80 bytes = 5 x double2:
// v0.xyz e1.xyz e2.xyz and the original triangle id (as int64 bits).
struct alignas(16) GpuTri {
    double v[9];
    int64_t id;
};
static_assert(sizeof(GpuTri) == 80, "tri must be 80 bytes");

struct HostBvh {
    std::vector<GpuNode> nodes;
    std::vector<int64_t> order;  // leaf-order position -> original triangle id
    int max_depth = 0;
    int max_leaf = 0;
};

// Builds a binned-SAH BVH2 with conservative f32 boxes over the triangles
// (v0, v0+e1, v0+e2).  Throws std::runtime_error on failure.
void build_bvh(const double* v0, const double* e1, const double* e2, int64_t n, HostBvh& out);

}  // namespace ef

struct ef_scene {
    int64_t n_tri = 0;
    int32_t n_bands = 0;
    int32_t n_mat = 0;
    int64_t n_nodes = 0;
    int32_t max_depth = 0;
    int32_t max_leaf = 0;
    int64_t device_bytes = 0;
    // device buffers
    ef::GpuNode* nodes = nullptr;      // (n_nodes)
    ef::GpuTri* tris = nullptr;        // (n_tri) leaf order
    double* tris_by_id = nullptr;      // (n_tri, 9) original order (all-pairs path)
    double* normals = nullptr;         // (n_tri, 3) original order
    int32_t* mat = nullptr;            // (n_tri)
    float* fd = nullptr;               // (n_mat, n_bands) diffuse reflection factor
    float* fs = nullptr;               // (n_mat, n_bands) specular reflection factor
    double* pdiff = nullptr;           // (n_mat) probability of a diffuse bounce
};

// error plumbing (ef_api.cpp)
namespace ef {
int set_error(int code, const std::string& msg);
int check_cuda(int err, const char* what);
void count_launch(uint64_t n = 1);
}  // namespace ef

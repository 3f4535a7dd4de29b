// Internal structures shared by the host builder and the CUDA kernels.
#pragma once
#include <climits>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/echoforge_b200.h"

namespace ef {

constexpr int kMaxBands = 8;
constexpr int kMaxOrder = 4;
constexpr int kBruteMaxTris = 512;   // scene.py:29
constexpr double kRayEps = 1e-4;     // scene.py:22
constexpr int kStackSize = 96;
constexpr int kMaxLeaf = 4;
constexpr int kTailMaxTris = 4096;   // scenes small enough for the CTA-wide tail sweep
#ifndef EF_TAIL_CLUSTER
#define EF_TAIL_CLUSTER 16
#endif
constexpr int kTailCluster = EF_TAIL_CLUSTER;   // leaf-order triangles per tail-sweep cluster

// Four-child BVH node, 128 bytes = four 32-byte sectors, child boxes in
// structure-of-arrays form so one node visit is three 256-bit loads (x, y, z
// planes), one 128-bit load (children) and four independent slab tests:
//   lox, hix, loy, hiy, loz, hiz : float[4]  (conservative f32 child boxes)
//   child : int32[4]  >= 0 inner node index,
//                     <  0 leaf ~((start << 3) | (count - 1)),
//                     kEmptyChild = unused slot
struct alignas(32) GpuNode {
    float lox[4], hix[4], loy[4], hiy[4], loz[4], hiz[4];
    int32_t child[4];
    int32_t pad[4];
};
static_assert(sizeof(GpuNode) == 128, "node must be 128 bytes");

// The traversal copy of a GpuNode (ef_scene.cu encode_nodes, after every
// build / rebuild / refit): each child box as a centre and a half extent
// per axis, cx[k] +- ex[k] enclosing [lox[k], hix[k]] (e rounded up), so a
// ray's slab distances are m = c * (1/d) - o/d, near = m - e |1/d|, far =
// m + e |1/d|: three FMAs per axis, packed two children per FFMA2, and no
// min/max ordering of the two planes.  Same 128-byte sector
// layout as GpuNode.  Built with EF_SLAB_CE=0 (A/B) it holds lo / hi.
#ifndef EF_SLAB_CE
#define EF_SLAB_CE 1
#endif
// EF_QNODE = 1 (default): the traversal copy is 64 bytes, two 256-bit loads
// per node visit instead of four loads.  Every plane of the four child
// boxes is a 16-bit coordinate on a grid over the scene's bounds (TravGrid,
// stored in the slot before node 0): word k of an axis = lo | hi << 16 of
// child k, lo rounded down and hi up to the grid and each widened by one
// more cell, which covers the rounding of the ray-space evaluation (one
// PRMT per plane builds the float 2^23 + q, one FMA maps it to the ray
// parameter).  An empty slot is lo = 65535, hi = 0 on every
// axis (near > far for every direction).
#ifndef EF_QNODE
#define EF_QNODE 1
#endif
#if EF_QNODE
struct alignas(32) TravNode {
    uint32_t px[4], py[4], pz[4];
    int32_t child[4];
};
static_assert(sizeof(TravNode) == 64, "node must be 64 bytes");
// the grid: plane q of axis a lies at lo[a] + q * cell[a]
struct alignas(32) TravGrid {
    float lo[3], pad0;
    float cell[3], pad1;
    float fill[8];
};
static_assert(sizeof(TravGrid) == sizeof(TravNode), "the grid takes one node slot");
constexpr uint32_t kEmptyPlanes = 0x0000ffffu;
#else
struct alignas(32) TravNode {
    float cx[4], ex[4], cy[4], ey[4], cz[4], ez[4];
    int32_t child[4];
    int32_t pad[4];
};
static_assert(sizeof(TravNode) == 128, "node must be 128 bytes");
#endif
constexpr int32_t kEmptyChild = INT32_MIN;

// f64 triangle payload in BVH leaf order, 96 bytes = three 32-byte sectors
// read by three 256-bit loads (LDG.E.256: one sector each, no half-used
// sectors as with 16-byte loads of an 80-byte record):
// v0.xyz e1.xyz e2.xyz, the original triangle id (as int64 bits), padding.
struct alignas(32) GpuTri {
    double v[9];
    int64_t id;
    int64_t pad[2];
};
static_assert(sizeof(GpuTri) == 96, "tri must be 96 bytes");

// Per-triangle shading record by original id, 48 bytes: the normal, the
// diffuse probability p_m of its material and the material index -- one
// level of loads per reflection instead of material -> p_m.
// EF_SHADE64 = 1 (default): 64-byte records, the normal and p_m in one
// 256-bit load (+0.3% on C3 / C5 against two 128-bit loads of a 48-byte
// record).
#ifndef EF_SHADE64
#define EF_SHADE64 1
#endif
#if EF_SHADE64
struct alignas(32) GpuShade {
    double n[3];
    double p;
    int32_t m;
    int32_t pad[7];
};
static_assert(sizeof(GpuShade) == 64, "shade record must be 64 bytes");
#else
struct alignas(16) GpuShade {
    double n[3];
    double p;
    int32_t m;
    int32_t pad[3];
};
static_assert(sizeof(GpuShade) == 48, "shade record must be 48 bytes");
#endif

// The builder's binary tree (kept on request: tools/sim_bottomup.cpp studies
// other collapse widths with it).
struct HostBinNode {
    double lo[3], hi[3];
    int32_t left, right;     // -1: leaf
    int64_t start, count;    // leaf: range of `order`
};

struct HostBvh {
    bool keep_binary = false;
    std::vector<HostBinNode> binary;    // keep_binary: the binary tree, root binary_root
    int32_t binary_root = 0;
    std::vector<GpuNode> nodes;
    std::vector<int32_t> level_nodes;   // node indices grouped by depth (root level first)
    std::vector<int64_t> level_start;   // offsets into level_nodes, size levels + 1
    double pad = 0.0;                   // absolute box padding used by the build
    std::vector<int64_t> order;  // leaf-order position -> original triangle id (repeats
                                 // where spatial splits share a triangle between leaves)
    int max_depth = 0;           // of the 4-wide tree
    int max_leaf = 0;
    int max_stack = 0;           // bound on traversal stack entries
};

// Builds a binned-SAH BVH2 with conservative f32 boxes over the triangles
// (v0, v0+e1, v0+e2).  Throws std::runtime_error on failure.
void build_bvh(const double* v0, const double* e1, const double* e2, int64_t n, HostBvh& out);

}  // namespace ef

struct ef_scene;
typedef struct CUstream_st* cudaStream_t;
namespace ef {
// LBVH on the device (bvh_device.cu) from DEVICE triangle rows `stride`
// doubles apart; replaces the scene's nodes, leaf order and refit schedule.
int device_build_bvh(ef_scene* s, const double* v0, const double* e1, const double* e2,
                     int64_t stride, cudaStream_t st);
// (Re)computes s->shade from s->normals, s->mat and s->pdiff, and s->tri_box
// from s->tris_by_id and s->pad (ef_scene.cu).
int update_shade(ef_scene* s, cudaStream_t st);
// (Re)computes s->tnodes, the traversal form of s->nodes (ef_scene.cu).
int encode_nodes(ef_scene* s, cudaStream_t st);

}  // namespace ef

struct ef_scene {
    int64_t n_tri = 0;
    int64_t n_refs = 0;                // triangle references in leaf order (>= n_tri with spatial splits)
    int32_t n_bands = 0;
    int32_t n_mat = 0;
    int64_t n_nodes = 0;
    int32_t max_depth = 0;
    int32_t max_leaf = 0;
    int64_t device_bytes = 0;
    // device buffers
    ef::GpuNode* nodes = nullptr;      // (n_nodes) build / refit form
    ef::TravNode* tnodes = nullptr;    // (n_nodes) traversal form (encode_nodes); EF_QNODE: tnodes[-1]
                                       // holds the TravGrid (tnodes_base is the allocation)
    ef::TravNode* tnodes_base = nullptr;
    int64_t n_tnodes_cap = 0;
    ef::GpuTri* tris = nullptr;        // (n_refs) leaf order
    double* tris_by_id = nullptr;      // (n_tri, 9) original order (all-pairs path)
    double* normals = nullptr;         // (n_tri, 3) original order
    int32_t* mat = nullptr;            // (n_tri)
    float* fd = nullptr;               // (n_mat, n_bands) diffuse reflection factor
    float* fs = nullptr;               // (n_mat, n_bands) specular reflection factor
    double* pdiff = nullptr;           // (n_mat) probability of a diffuse bounce
    float* fr = nullptr;               // (n_mat, n_bands) (1 - a) * s for diffuse rain
    ef::GpuShade* shade = nullptr;     // (n_tri) shading records, original order
    float* tri_box = nullptr;          // (n_tri, 8) padded f32 triangle boxes lo.xyz hi.xyz,
                                       // scenes of <= kTailMaxTris triangles (tail_kernel)
    float* clu_box = nullptr;          // (n_clu, 8) unions of kTailCluster consecutive leaf-order boxes
    int32_t* clu_ids = nullptr;        // (n_tri) triangle ids in leaf order, each once
    int64_t n_clu = 0;
    std::vector<int32_t> clu_order;    // host builds: that order (spatial splits repeat ids
                                       // in the leaves); empty: the device tree's leaf order
    // refit support (dynamic scenes)
    int64_t* leaf_order = nullptr;     // (n_refs) leaf position -> original id
    int32_t* level_nodes = nullptr;    // node indices grouped by depth
    int64_t n_nodes_cap = 0;           // allocated nodes (device builds over-allocate)
    int64_t level_nodes_len = 0;
    std::vector<int64_t> level_start;  // host copy of the level offsets
    double pad = 0.0;
};

// error plumbing (ef_api.cpp)
namespace ef {
int set_error(int code, const std::string& msg);
int check_cuda(int err, const char* what);
void count_launch(uint64_t n = 1);
void keep_pool_memory();   // default mempool keeps its memory (cudaMallocAsync scratch)
}  // namespace ef

/*
 * echoforge_b200.h -- C ABI of the B200-native hot path of the echoforge
 * reference (arXiv 1803.00430; /root/reference/pkg/src/echoforge).
 *
 * The reference has no FFI: its boundary is the Python call signatures of
 * scene.py / bvh.py / sh.py plus the SPEC-only propagation and ir-analysis
 * operations.  Every entry point below replaces one of them (cited per
 * function); the Python package paper_1803_00430_b200 binds them with ctypes
 * and keeps the reference signatures.
 *
 * Conventions
 *   - Plain pointers and sizes; no torch types.  "host" pointers are CPU
 *     memory, "device" pointers are CUDA global memory on the current device.
 *   - Every call is stream-ordered on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and never blocks the host unless documented.
 *   - Return 0 (EF_OK) or a negative status; never throws, never exits.  The
 *     message of the last failure on the calling thread is available through
 *     ef_last_error().  Contract violations -> EF_EINVAL (Python: ValueError),
 *     CUDA failures -> EF_ECUDA (Python: RuntimeError).
 *   - Stream-ordered scratch comes from the device's default memory pool
 *     (cudaMallocAsync); the library sets that pool's release threshold to
 *     "keep everything" so per-frame scratch is not re-mapped at every
 *     synchronisation.
 *   - ef_scene handles are immutable after ef_scene_create and may be used
 *     concurrently from several streams.
 */
#ifndef ECHOFORGE_B200_H
#define ECHOFORGE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EF_OK 0
#define EF_EINVAL (-1)
#define EF_ECUDA (-2)
#define EF_ENOMEM (-3)
#define EF_EUNSUPPORTED (-4)
#define EF_ENCCL (-5)

#define EF_ABI_VERSION 1

/* Per-source trace counters (u64), index into the stats array. */
enum {
    EF_ST_PATHS = 0,       /* primary rays traced                               */
    EF_ST_SEGMENTS,        /* closest-hit queries (the throughput unit)         */
    EF_ST_REFLECTIONS,     /* segments that ended on a surface                  */
    EF_ST_ARRIVALS,        /* listener-sphere crossings                         */
    EF_ST_DIRECT,          /* crossings before any reflection (-> Dir)          */
    EF_ST_DROPPED,         /* late arrivals past the IR length    */
    EF_ST_ESCAPED,         /* paths that left the scene                         */
    EF_ST_NODES,           /* BVH nodes visited (device tree)                   */
    EF_ST_TRIS,            /* exact triangle tests (device tree / all-pairs)    */
    EF_ST_TAIL,            /* segments run by the frame-tail kernel (subset of  */
                           /* EF_ST_SEGMENTS; scenes of 513-4,096 triangles)    */
    EF_ST_COUNT = 10
};

/* Per-(source, band) analysis outputs (f64), index into params. */
enum {
    EF_P_RT60 = 0,         /* s, clamped to [0.05, max_rt]   */
    EF_P_GAIN,             /* g_reverb                        */
    EF_P_DRR_DB,           /* 10 log10(E_dir / E_reverb), +-99 dB clamps        */
    EF_P_TOTAL,            /* sum_t I_b(t)                                      */
    EF_P_DIRECT,           /* E_dir,b                                           */
    EF_P_SILENT,           /* 1.0 if the band is silent / indeterminate         */
    EF_P_FIT_N,            /* bins used by the decay regression                 */
    EF_P_SLOPE,            /* dB/s                                              */
    EF_P_FIRST_BIN,        /* first bin with I_b > 0, -1 if none                */
    EF_P_LAST_BIN,         /* last bin with I_b > 0, -1 if none                 */
    EF_P_COUNT = 10
};
/* Per-source analysis outputs (f64). */
enum {
    EF_S_PREDELAY = 0,     /* s, -1 when silent               */
    EF_S_MFP,              /* mean free path, m               */
    EF_S_SILENT,
    EF_S_COUNT = 4
};

typedef struct ef_scene ef_scene;

/* ---- library -------------------------------------------------------- */
int ef_abi_version(void);
/* Copies the calling thread's last error message (NUL-terminated). */
int ef_last_error(char* buf, size_t n);
/* Number of CUDA kernels this library launched since load (all threads). */
uint64_t ef_launch_count(void);

/* ---- scene ------------------------------------------------------------
 * Replaces SceneModel.__init__ (scene.py:149-171) and BVH.__init__
 * (bvh.py:51-128).  All inputs are HOST arrays, copied: v0/e1/e2/normals
 * (n_tri,3) f64 exactly as the reference stores them (scene.py:152-166),
 * material_index (n_tri,) i64, absorption/scattering (n_materials, n_bands)
 * f64 in [0,1] (scene.py:167-170; n_bands generalised from 4 to 1..8).
 * Builds the device BVH (binned SAH, four-child nodes with conservative f32
 * boxes, re-encoded for traversal as 64-byte nodes of 16-bit planes on a
 * grid over the scene bounds) and uploads the f64 triangle payload in leaf
 * order. */
int ef_scene_create(const double* v0, const double* e1, const double* e2,
                    const double* normals, const int64_t* material_index, int64_t n_tri,
                    const double* absorption, const double* scattering,
                    int32_t n_materials, int32_t n_bands, ef_scene** out);
/* Same, with build flags: EF_SCENE_DEVICE_BUILD builds the tree on the GPU
 * (linear BVH over 63-bit Morton codes collapsed to the same four-child
 * nodes; milliseconds instead of seconds for 10^6 triangles, looser than
 * SAH).  Hit results do not depend on the tree. */
#define EF_SCENE_DEVICE_BUILD 1u
int ef_scene_create_ex(const double* v0, const double* e1, const double* e2,
                       const double* normals, const int64_t* material_index, int64_t n_tri,
                       const double* absorption, const double* scattering,
                       int32_t n_materials, int32_t n_bands, uint32_t flags, ef_scene** out);
int ef_scene_destroy(ef_scene* scene);
/* Dynamic geometry: replace the triangle
 * data of a scene (same triangle count and ids; DEVICE v0/e1/e2/normals
 * (n_tri,3) f64) and refit the device BVH bottom-up, one kernel per level.
 * Stream-ordered; the tree topology is kept, boxes stay conservative. */
int ef_scene_refit(ef_scene* scene, const double* v0, const double* e1, const double* e2,
                   const double* normals, void* stream);
/* Dynamic geometry with a new topology: replace the triangle data (DEVICE
 * arrays as ef_scene_refit) and rebuild the tree on the GPU (the
 * EF_SCENE_DEVICE_BUILD builder).  For motion that a refit would leave with
 * loose boxes.  Returns after the build (one stream synchronisation). */
int ef_scene_rebuild(ef_scene* scene, const double* v0, const double* e1, const double* e2,
                     const double* normals, void* stream);
/* out[0]=n_tri out[1]=n_nodes out[2]=max_depth out[3]=device bytes
 * out[4]=max leaf size out[5]=n_bands out[6]=n_materials
 * out[7]=triangle references in the leaves (> n_tri where spatial splits
 * share a triangle between leaves) */
int ef_scene_info(const ef_scene* scene, int64_t* out8);

/* ---- ray queries ------------------------------------------------------
 * Replaces SceneModel.intersect_batch (scene.py:208-230), BVH.intersect
 * (bvh.py:130-160, one ray per row) and SceneModel.intersect_brute
 * (scene.py:194-206).  DEVICE arrays: origins, dirs (n,3) f64; t_max (n,)
 * f64 or NULL (= +inf); outputs t (n,) f64 (+inf on miss), tri (n,) i64 (-1),
 * hit (n,) u8.  mode: 0 = reference dispatch (all-pairs for n_tri <= 512,
 * else BVH), 1 = all triangles, 2 = BVH.  Ties in t resolve to the lowest
 * triangle id (the reference's all-pairs rule, scene.py:220). */
int ef_intersect_batch(const ef_scene* scene, const double* origins, const double* dirs,
                       int64_t n, double t_min, const double* t_max, int32_t mode,
                       double* t_out, int64_t* tri_out, uint8_t* hit_out, void* stream);

/* Replaces SceneModel.occluded_batch (scene.py:232-252): DEVICE origins,
 * targets (n,3) f64 -> out (n,) u8, 1 where the segment is blocked. */
int ef_occluded_batch(const ef_scene* scene, const double* origins, const double* targets,
                      int64_t n, uint8_t* out, void* stream);

/* Replaces ray_triangles (bvh.py:11-28) and ray_triangles_batch
 * (bvh.py:31-45): every ray against every triangle.  DEVICE origins, dirs
 * (n_rays,3); v0, e1, e2 (n_tri,3) f64; t_max (n_rays,) or NULL (= none, the
 * batch form).  Outputs t (n_rays, n_tri) f64 -- including the reference's
 * values for invalid pairs (0 when |det| <= 1e-14) -- and valid (n_rays,
 * n_tri) u8 = barycentric test && t > t_min && t <= t_max. */
int ef_ray_triangles(const double* origins, const double* dirs, int64_t n_rays,
                     const double* v0, const double* e1, const double* e2, int64_t n_tri,
                     double t_min, const double* t_max, double* t_out, uint8_t* valid_out,
                     void* stream);

/* ---- spherical harmonics ---------------------------------------------
 * Replaces eval_sh_batch (sh.py:86-126): DEVICE dirs (n,3) f64 -> out
 * (n,(order+1)^2) f64, bit-identical to the reference; order 0..4. */
int ef_eval_sh_batch(const double* dirs, int64_t n, int32_t order, double* out, void* stream);

/* Replaces directional_loudness_matrix (sh.py:240-253) for n
 * distributions: DEVICE avg (n,(order+1)^2) f64, design (n_design,3) f64 ->
 * out (n, nk, nk) f64 = (4 pi / N) B^T diag(max(0, B avg)) B. */
int ef_loudness_batch(const double* avg, int64_t n, int32_t order, const double* design,
                      int32_t n_design, double* out, void* stream);

/* ---- propagation ------------------------------------------------------
 * Replaces trace_frame for n_sources sources in one
 * launch (forward tracing from point sources to a listener sphere, the
 * BASELINE.json configs).  Bounce model pinned in DESIGN.md section 3. */
typedef struct {
    int32_t n_sources;
    int32_t order;          /* SH order of the histogram, 0..4              */
    int32_t n_bins;         /* IR length in bins                           */
    int32_t max_bounces;    /* reflections per path                        */
    int64_t n_rays;         /* rays per source traced by this call         */
    uint32_t ray0;          /* global index of the first ray (sharding)    */
    uint32_t seed;          /* Philox key word 0                           */
    uint32_t frame;         /* Philox counter word 3                       */
    int32_t mode;           /* 0 reference dispatch, 1 all-pairs, 2 BVH     */
    double bin_len;         /* metres of path per bin = c * bin_seconds    */
    double listener[3];
    double radius;          /* listener sphere radius, m                   */
    float e0;               /* initial energy per band of every path       */
    int32_t record_ids;     /* nonzero: write per-segment hit ids          */
    int32_t clear_outputs;  /* nonzero: zero H, Dir, stats, sum_t first    */
    int32_t diffuse_rain;   /* nonzero: next-event connection from every
                               diffuse bounce; segments
                               leaving a diffuse bounce then skip the
                               sphere test                  */
    int32_t er_max_order;   /* arrivals of order 1..er_max_order (<= 2) go
                               to the early-reflection list, not to H       */
    int64_t er_capacity;    /* entries available at er_entries             */
    void* er_entries;       /* DEVICE ef_er_entry[er_capacity] or NULL      */
    uint32_t* er_count;     /* DEVICE counter, ACCUMULATED (caller zeroes)  */
} ef_trace_config;

/* One early-reflection arrival (PathList source data). */
typedef struct {
    int32_t src, order;     /* source index in the launch, reflections     */
    int32_t tri0, tri1;     /* first two reflecting triangles (-1: none)   */
    double dist;            /* path length to the listener, m              */
    float dir[3];           /* arrival direction (towards the source side) */
    float pad;
    float energy[8];        /* per-band energy (intensity units of H)      */
} ef_er_entry;

/* DEVICE arrays:
 *   src_pos  (n_sources,3) f64      src_key (n_sources,) u32 Philox key word 1
 *   ray_ids  (n_rays,) u32 or NULL: explicit global ray indices (subsets)
 *   H        (n_sources, n_bins, n_bands, nk) f32, ACCUMULATED (caller zeroes)
 *   Dir      (n_sources, n_bands, nk) f32, ACCUMULATED direct arrivals
 *   stats    (n_sources, EF_ST_COUNT) u64, ACCUMULATED
 *   sum_t    (n_sources,) f64, ACCUMULATED reflected segment lengths
 *   path_nseg (n_sources*n_rays,) i32 or NULL: segments per path
 *   path_ids (n_sources*n_rays, max_bounces) i32 or NULL: hit ids (-1 escape)
 * nk = (order+1)^2. */
int ef_trace(const ef_scene* scene, const ef_trace_config* cfg, const double* src_pos,
             const uint32_t* src_key, const uint32_t* ray_ids, float* H, float* Dir,
             unsigned long long* stats, double* sum_t, int32_t* path_nseg, int32_t* path_ids,
             void* stream);

/* ---- multi-GPU: trace fused with the histogram reduce-scatter ---------
 * One process per GPU, rays sharded by global index (ray0).  Instead of a
 * local (n_sources, ...) histogram followed by a reduce-scatter, every splat
 * of global source g is added straight into the block g % sources_per_rank
 * of rank g / sources_per_rank: hist_peers / dir_peers are HOST arrays of
 * n_sources / sources_per_rank (<= 8) DEVICE pointers, rank r's entries
 * -> (sources_per_rank, n_bins, n_bands, nk) f32 and
 * (sources_per_rank, n_bands, nk) f32, mapped with ef_peer_open (remote
 * atomics over NVLink/NVSwitch).  The blocks are ACCUMULATED and owned by
 * their rank: clear_outputs clears only the local stats / sum_t, and the
 * caller orders "owner zeroed" before and "all ranks done" after the launch
 * (distributed.PeerHistograms double-buffers so one barrier per frame
 * suffices).  Replaces bench.py's ef_trace + reduce_scatter_tensor pair. */
int ef_trace_fused(const ef_scene* scene, const ef_trace_config* cfg, const double* src_pos,
                   const uint32_t* src_key, const uint32_t* ray_ids, float* const* hist_peers,
                   float* const* dir_peers, int32_t sources_per_rank, unsigned long long* stats,
                   double* sum_t, int32_t* path_nseg, int32_t* path_ids, void* stream);

#define EF_IPC_HANDLE_BYTES 64
/* cudaMalloc'd, zeroed device buffer of `bytes` and its IPC handle
 * (EF_IPC_HANDLE_BYTES bytes written to ipc_handle). */
int ef_peer_alloc(int64_t bytes, void** dev_ptr, void* ipc_handle);
int ef_peer_free(void* dev_ptr);
/* Map another process's ef_peer_alloc buffer (same node). */
int ef_peer_open(const void* ipc_handle, void** dev_ptr);
int ef_peer_close(void* dev_ptr);

/* ---- scene ingestion --------------------------
 * Replaces _parse_obj (scene.py:255-280): positions only, fan triangulation,
 * 1-based / negative indices, the current g / o / usemtl name per triangle;
 * numbers parsed like Python's float() / int().  Malformed lines and
 * out-of-range indices -> EF_EINVAL with file:line.  ef_mesh_info: out4 =
 * n_verts, n_tris, n_groups, bytes of the NUL-separated group names;
 * ef_mesh_arrays fills HOST verts (V,3) f64, tris (T,3) i64 0-based,
 * tri_group (T) i32 and the names (any pointer may be NULL). */
typedef struct ef_mesh ef_mesh;
int ef_obj_parse(const char* path, ef_mesh** out);
int ef_mesh_info(const ef_mesh* mesh, int64_t* out4);
int ef_mesh_arrays(const ef_mesh* mesh, double* verts, int64_t* tris, int32_t* tri_group, char* names,
                   int64_t names_bytes);
int ef_mesh_destroy(ef_mesh* mesh);

/* ---- unfused histogram exchange over NCCL -------
 * Replaces the reference-side reduction of per-worker partial IRs (the
 * paper's multi-threaded tracer sums per-thread IRs; SPEC.md:247-248 splits
 * a frame over primary rays).  Rank g traces rays [g R/N, (g+1) R/N) of every
 * source into local partial histograms with ef_trace; ef_nccl_reduce_hist
 * then sums them:
 *   EF_NCCL_REDUCE_SCATTER  partial = N * owned_count f32 (sources ordered
 *                           by owner rank); owned = this rank's S/N sources,
 *                           summed over ranks (K4 then runs on them);
 *   EF_NCCL_ALLREDUCE       owned = sum of partial (owned_count f32; may alias);
 *   EF_NCCL_REDUCE          the sum on rank 0.
 * The communicator comes from ef_nccl_comm_create (unique id from
 * ef_nccl_unique_id on one rank, shared out of band).  libnccl.so.2 is
 * resolved at first use (dlopen); failures -> EF_ENCCL. */
#define EF_NCCL_REDUCE_SCATTER 0
#define EF_NCCL_ALLREDUCE 1
#define EF_NCCL_REDUCE 2
int ef_nccl_unique_id(uint8_t* out128);
int ef_nccl_comm_create(int32_t world, int32_t rank, const uint8_t* id128, int32_t device, void** comm);
int ef_nccl_comm_destroy(void* comm);
int ef_nccl_reduce_hist(void* comm, const float* partial, float* owned, int64_t owned_count, int32_t mode,
                        void* stream);

/* ---- ir-analysis ------------------------------------------------------
 * Replaces estimate_rt60, reverb_gain (290),
 * estimate_predelay (299), average_directivity (308) and
 * directional_loudness_matrix (sh.py:240-253), batched over sources and
 * bands.  DEVICE inputs are ef_trace's outputs; design (n_design,3) f64 is
 * the t-design of design_for_order(order) (tdesigns.py:360).
 * Outputs (DEVICE): params (n_sources, n_bands, EF_P_COUNT) f64,
 * src_params (n_sources, EF_S_COUNT) f64, avg_dir (n_sources, n_bands, nk)
 * f64, loudness (n_sources, n_bands, nk, nk) f64 or NULL. */
typedef struct {
    int32_t n_sources, n_bins, n_bands, order;
    double bin_s;           /* seconds per bin                             */
    double max_rt;          /* RT60 clamp upper bound, s                   */
} ef_analysis_config;

int ef_analyze(const ef_analysis_config* cfg, const float* H, const float* Dir,
               const unsigned long long* stats, const double* sum_t, const double* design,
               int32_t n_design, double* params, double* src_params, double* avg_dir,
               double* loudness, void* stream);

/* Replaces acoustic_metrics: DEVICE
 * energy (n_series, n_bins) f64 per-bin energy, direct_index (n_series) i32
 * or NULL (= 0); e_ref = free-field direct energy at 10 m.  out (n_series, 5)
 * f64 = RT60 (-1 when silent), C80 dB (+99 sentinel), D50, TS s, G dB. */
int ef_acoustic_metrics(const double* energy, int64_t n_series, int32_t n_bins, double bin_s,
                        const int32_t* direct_index, double e_ref, double max_rt, double* out,
                        void* stream);

/* Replaces accumulate_ir: DEVICE f32 arrays of n
 * elements, out = alpha * frame + (1 - alpha) * cache (out may alias). */
int ef_blend(const float* cache, const float* frame, int64_t n, double alpha, float* out,
             void* stream);

/* ---- SH-domain auralization (BASELINE config C4) ---------------------
 * Replaces the SPEC-only reverb renderer (C4's 16-line FDN
 * per band) and spatialize_hrtf.  Semantics: DESIGN.md 3.7.
 * ef_audio_create takes HOST parameter arrays (copied):
 *   sos (4 bands, 5 biquads, b0 b1 b2 a1 a2) f32; Y (S,16) f32 direct SH
 *   encoding; d_int/d_w (S) direct delay = d_int + 1 - d_w samples; gain (S,4)
 *   direct gain per band; p_int/p_w (S) predelay likewise; fdn_delay (S,16)
 *   i32 line delays in (512, line_len]; g_line (S,4,16) f32 line gains;
 *   M (S,4,16,16) f32 line -> SH matrices; hrtf_spec (16,2,513) complex f32
 *   rFFT(1024) of the zero-padded 2-ear filters.
 * ef_audio_process renders one 512-sample block: x (S,512) f32 DEVICE input,
 * bus_out (16,512) f32 DEVICE or NULL, out (2,512) f32 DEVICE binaural. */
typedef struct {
    int32_t n_sources;
    int32_t hist_len;   /* band history ring length, power of two       */
    int32_t line_len;   /* FDN line ring length, power of two            */
    int32_t reserved;
} ef_audio_config;

typedef struct ef_audio ef_audio;

int ef_audio_create(const ef_audio_config* cfg, const float* sos, const float* Y,
                    const int32_t* d_int, const float* d_w, const float* gain,
                    const int32_t* p_int, const float* p_w, const int32_t* fdn_delay,
                    const float* g_line, const float* M, const float* hrtf_spec, ef_audio** out);
int ef_audio_destroy(ef_audio* audio);
/* update_params: swap the per-source parameters at a block
 * boundary -- HOST arrays laid out as in ef_audio_create (NULL = keep):
 * Y, d_int/d_w, gain, p_int/p_w, g_line, M.  Stream-ordered on `stream`
 * (blocks enqueued before render with the old values); returns after the
 * copies complete.  Line delays and HRTF are fixed at create. */
int ef_audio_update(ef_audio* audio, const float* Y, const int32_t* d_int, const float* d_w,
                    const float* gain, const int32_t* p_int, const float* p_w, const float* g_line,
                    const float* M, void* stream);
/* out[0]=n_sources out[1]=device bytes out[2]=next sample index out[3]=grid */
int ef_audio_info(const ef_audio* audio, int64_t* out4);
int ef_audio_process(ef_audio* audio, const float* x, float* bus_out, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ECHOFORGE_B200_H */

/*
 * oracle/efo.c -- CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the checker or the CPU
 * baseline.  The product path (paper_1803_00430_b200/) never links it.
 *
 * This is a plain-C restatement of the reference's hot path
 * (/root/reference/pkg/src/echoforge, "echoforge" 0.1.0):
 *   - Moeller-Trumbore exactly as bvh.py:11-28 (scalar) and bvh.py:31-45
 *     (all-pairs), with numpy's evaluation order: np.cross is a1*b2-a2*b1
 *     per component, every 3-term einsum dot is (p0+p2)+p1, no FMA.
 *     Pinned bit-for-bit against the reference by tests/golden (see
 *     oracle/gen_golden.py).
 *   - the binned-SAH BVH build of bvh.py:51-128 (same node numbering, same
 *     tri_order, same split choices) and the stack traversal of
 *     bvh.py:130-160 (right child popped first, ties -> last visited).
 *   - SceneModel.intersect_batch dispatch (scene.py:208-230): brute force for
 *     T <= 512 (lowest id wins ties, scene.py:216-223), else per-ray BVH.
 *   - the bounce loop, listener-sphere receiver and SH histogram that the
 *     reference only specifies; the choices are pinned in
 *     DESIGN.md section 3 and restated independently in the CUDA kernel.
 *
 * Parity of the SPEC-only parts (bounce loop, histogram) is pinned only by
 * this restatement and its own known-answer tests: "parity unpinned" for
 * those rows in the sense of the task statement (no reference code exists).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, no -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EFO_BARY_EPS 1e-10   /* bvh.py:8 */
#define EFO_LEAF_SIZE 4      /* bvh.py:6 */
#define EFO_N_BINS 16        /* bvh.py:7 */
#define EFO_BRUTE_MAX 512    /* scene.py:29 */
#define EFO_RAY_EPS 1e-4     /* scene.py:22 */
#define EFO_MAX_BANDS 8
#define EFO_MAX_NK 25

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al. 2011), counter-based RNG               */
/* ------------------------------------------------------------------ */
void efo_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* 53-bit uniform in [0,1) from two 32-bit words (exact in binary64). */
static inline double u53(uint32_t a, uint32_t b) {
    return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}

static inline void draw2(uint32_t ray, uint32_t bounce, uint32_t draw, uint32_t frame,
                         uint32_t seed, uint32_t src, double* u1, double* u2) {
    uint32_t c[4] = {ray, bounce, draw, frame}, k[2] = {seed, src}, o[4];
    efo_philox(c, k, o);
    *u1 = u53(o[0], o[1]);
    *u2 = u53(o[2], o[3]);
}

/* Uniform direction on the sphere by Marsaglia (1972) rejection.
 * Only + - * sqrt: reproducible bit-for-bit on host and device. */
void efo_sample_sphere(uint32_t seed, uint32_t src, uint32_t ray, uint32_t frame, double d[3]) {
    for (uint32_t j = 0; j < 64; ++j) {
        double u1, u2;
        draw2(ray, 0u, j, frame, seed, src, &u1, &u2);
        double a = 2.0 * u1 - 1.0;
        double b = 2.0 * u2 - 1.0;
        double s = a * a + b * b;
        if (s >= 1.0) continue;
        double f = 2.0 * sqrt(1.0 - s);
        d[0] = a * f;
        d[1] = b * f;
        d[2] = 1.0 - 2.0 * s;
        return;
    }
    d[0] = 0.0; d[1] = 0.0; d[2] = 1.0;
}

/* Cosine-weighted hemisphere about unit n (disk rejection, Malley) with the
 * Duff et al. (2017) branchless orthonormal basis. */
void efo_sample_cosine(uint32_t seed, uint32_t src, uint32_t ray, uint32_t bounce,
                       uint32_t frame, const double n[3], double d[3]) {
    for (uint32_t j = 0; j < 64; ++j) {
        double u1, u2;
        draw2(ray, bounce, 1u + j, frame, seed, src, &u1, &u2);
        double a = 2.0 * u1 - 1.0;
        double b = 2.0 * u2 - 1.0;
        double s = a * a + b * b;
        if (s >= 1.0) continue;
        double z = sqrt(1.0 - s);
        double sg = copysign(1.0, n[2]);
        double aa = -1.0 / (sg + n[2]);
        double bb = n[0] * n[1] * aa;
        double t1x = 1.0 + sg * n[0] * n[0] * aa, t1y = sg * bb, t1z = -sg * n[0];
        double t2x = bb, t2y = sg + n[1] * n[1] * aa, t2z = -n[1];
        d[0] = (a * t1x + b * t2x) + z * n[0];
        d[1] = (a * t1y + b * t2y) + z * n[1];
        d[2] = (a * t1z + b * t2z) + z * n[2];
        return;
    }
    d[0] = n[0]; d[1] = n[1]; d[2] = n[2];
}

/* ------------------------------------------------------------------ */
/* numpy-order vector helpers                                          */
/* ------------------------------------------------------------------ */
/* np.einsum 3-term dot: (p0 + p2) + p1 (measured) */
static inline double dot3(const double* a, const double* b) {
    return (a[0] * b[0] + a[2] * b[2]) + a[1] * b[1];
}
/* np.cross (numpy/_core/numeric.py): cp0 = a1*b2 - a2*b1, ... */
static inline void cross3(const double* a, const double* b, double* o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
/* OpenBLAS dgemv order for `qvec @ direction` (bvh.py:24) as measured on
 * the survey host (DYNAMIC_ARCH, x86-64): host dependent, used only to pin
 * the reference's own BVH path bit-for-bit in tests. */
static inline double dot3_blas(const double* q, const double* d, int k_rows) {
    if (k_rows == 1) return fma(q[2], d[2], fma(q[1], d[1], q[0] * d[0]));
    return fma(q[2], d[2], fma(q[0], d[0], q[1] * d[1]));
}

/* One Moeller-Trumbore test, bvh.py:17-27 (scalar) == bvh.py:33-44 (batch).
 * Returns validity (without the t window), writes t, u, v. */
static inline int mt_test(const double* o, const double* d, const double* v0,
                          const double* e1, const double* e2, int vmode, int k_rows,
                          double* t_out, double* u_out, double* v_out) {
    double pvec[3], tvec[3], qvec[3];
    cross3(d, e2, pvec);
    double det = dot3(e1, pvec);
    int valid = fabs(det) > 1e-14;
    double inv = valid ? 1.0 / det : 0.0;
    tvec[0] = o[0] - v0[0];
    tvec[1] = o[1] - v0[1];
    tvec[2] = o[2] - v0[2];
    double u = dot3(tvec, pvec) * inv;
    cross3(tvec, e1, qvec);
    double vd = vmode ? dot3_blas(qvec, d, k_rows) : dot3(qvec, d);
    double v = vd * inv;
    double t = dot3(e2, qvec) * inv;
    valid = valid && (u >= -EFO_BARY_EPS) && (v >= -EFO_BARY_EPS) && (u + v <= 1.0 + EFO_BARY_EPS);
    *t_out = t; *u_out = u; *v_out = v;
    return valid;
}

/* ------------------------------------------------------------------ */
/* Scene + reference BVH (bvh.py:51-128)                               */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t n_tri;
    const double *v0, *e1, *e2, *normals; /* borrowed, (T,3) row-major */
    const int64_t* mat;                    /* borrowed, (T,) */
    int n_bands, n_mat;
    /* reflection factors per material: diffuse / specular, f32 */
    float* fd;
    float* fs;
    float* fr;     /* (1 - a) * s: diffusely reflected fraction (diffuse rain) */
    double* pdiff;
    /* reference BVH */
    int64_t n_nodes, cap_nodes;
    double* node_min; /* (N,3) */
    double* node_max;
    int64_t* node_left;
    int64_t* node_start;
    int64_t* node_count;
    int64_t* tri_order;
    double* tri_min;
    double* tri_max;
    double* cen;
} efo_scene;

static int64_t add_node(efo_scene* s) {
    if (s->n_nodes == s->cap_nodes) {
        int64_t nc = s->cap_nodes ? 2 * s->cap_nodes : 64;
        s->node_min = realloc(s->node_min, sizeof(double) * 3 * nc);
        s->node_max = realloc(s->node_max, sizeof(double) * 3 * nc);
        s->node_left = realloc(s->node_left, sizeof(int64_t) * nc);
        s->node_start = realloc(s->node_start, sizeof(int64_t) * nc);
        s->node_count = realloc(s->node_count, sizeof(int64_t) * nc);
        s->cap_nodes = nc;
    }
    int64_t i = s->n_nodes++;
    s->node_left[i] = -1;
    s->node_start[i] = -1;
    s->node_count[i] = 0;
    return i;
}

/* np.sum of a 3-vector: sequential (measured) */
static inline double area_of(const double* a, const double* b) {
    double d0 = b[0] - a[0], d1 = b[1] - a[1], d2 = b[2] - a[2];
    /* (b-a) * np.roll(b-a, 1) = [d0*d2, d1*d0, d2*d1] */
    return (d0 * d2 + d1 * d0) + d2 * d1;
}

typedef struct { int64_t* buf; int64_t* tmp; } build_ws;

static void build_rec(efo_scene* s, build_ws* ws, int64_t idx, int64_t lo, int64_t hi) {
    int64_t* order = s->tri_order;
    double bmin[3] = {INFINITY, INFINITY, INFINITY}, bmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = lo; i < hi; ++i) {
        int64_t t = order[i];
        for (int k = 0; k < 3; ++k) {
            double a = s->tri_min[3 * t + k], b = s->tri_max[3 * t + k];
            if (a < bmin[k]) bmin[k] = a;
            if (b > bmax[k]) bmax[k] = b;
        }
    }
    memcpy(&s->node_min[3 * idx], bmin, sizeof bmin);
    memcpy(&s->node_max[3 * idx], bmax, sizeof bmax);
    int64_t count = hi - lo;
    if (count <= EFO_LEAF_SIZE) {
        s->node_start[idx] = lo;
        s->node_count[idx] = count;
        return;
    }
    double cmin[3] = {INFINITY, INFINITY, INFINITY}, cmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = lo; i < hi; ++i) {
        const double* c = &s->cen[3 * order[i]];
        for (int k = 0; k < 3; ++k) {
            if (c[k] < cmin[k]) cmin[k] = c[k];
            if (c[k] > cmax[k]) cmax[k] = c[k];
        }
    }
    double ext[3] = {cmax[0] - cmin[0], cmax[1] - cmin[1], cmax[2] - cmin[2]};
    int axis = 0; /* np.argmax: first maximum */
    if (ext[1] > ext[axis]) axis = 1;
    if (ext[2] > ext[axis]) axis = 2;
    if (ext[axis] <= 1e-12) {
        s->node_start[idx] = lo;
        s->node_count[idx] = count;
        return;
    }
    int64_t* bins = ws->buf + lo; /* per-triangle bin, aligned with order[lo:hi] */
    int64_t bcount[EFO_N_BINS] = {0};
    double bbmin[EFO_N_BINS][3], bbmax[EFO_N_BINS][3];
    for (int b = 0; b < EFO_N_BINS; ++b)
        for (int k = 0; k < 3; ++k) { bbmin[b][k] = INFINITY; bbmax[b][k] = -INFINITY; }
    double cm = cmin[axis], ea = ext[axis];
    for (int64_t i = lo; i < hi; ++i) {
        int64_t t = order[i];
        double rel = (s->cen[3 * t + axis] - cm) / ea;
        int64_t b = (int64_t)(EFO_N_BINS * rel);
        if (b > EFO_N_BINS - 1) b = EFO_N_BINS - 1;
        bins[i - lo] = b;
        bcount[b]++;
        for (int k = 0; k < 3; ++k) {
            double a = s->tri_min[3 * t + k], c = s->tri_max[3 * t + k];
            if (a < bbmin[b][k]) bbmin[b][k] = a;
            if (c > bbmax[b][k]) bbmax[b][k] = c;
        }
    }
    /* prefix / suffix bounds: min/max are exact, so this equals the
     * reference's per-split recomputation (bvh.py:94-106) */
    double lmin[EFO_N_BINS + 1][3], lmax[EFO_N_BINS + 1][3], rmin[EFO_N_BINS + 1][3], rmax[EFO_N_BINS + 1][3];
    int64_t lcnt[EFO_N_BINS + 1];
    for (int k = 0; k < 3; ++k) { lmin[0][k] = INFINITY; lmax[0][k] = -INFINITY; rmin[EFO_N_BINS][k] = INFINITY; rmax[EFO_N_BINS][k] = -INFINITY; }
    lcnt[0] = 0;
    for (int b = 0; b < EFO_N_BINS; ++b) {
        lcnt[b + 1] = lcnt[b] + bcount[b];
        for (int k = 0; k < 3; ++k) {
            lmin[b + 1][k] = bbmin[b][k] < lmin[b][k] ? bbmin[b][k] : lmin[b][k];
            lmax[b + 1][k] = bbmax[b][k] > lmax[b][k] ? bbmax[b][k] : lmax[b][k];
        }
    }
    for (int b = EFO_N_BINS - 1; b >= 0; --b)
        for (int k = 0; k < 3; ++k) {
            rmin[b][k] = bbmin[b][k] < rmin[b + 1][k] ? bbmin[b][k] : rmin[b + 1][k];
            rmax[b][k] = bbmax[b][k] > rmax[b + 1][k] ? bbmax[b][k] : rmax[b + 1][k];
        }
    double best_cost = INFINITY;
    int best_split = -1;
    for (int split = 1; split < EFO_N_BINS; ++split) {
        int64_t nl = lcnt[split];
        if (nl == 0 || nl == count) continue;
        double cost = area_of(lmin[split], lmax[split]) * (double)nl +
                      area_of(rmin[split], rmax[split]) * (double)(count - nl);
        if (cost < best_cost) { best_cost = cost; best_split = split; }
    }
    int64_t mid;
    int64_t* tmp = ws->tmp;
    if (best_split < 0) {
        /* stable argsort of centroids along axis (bvh.py:108-111) */
        int64_t n = count;
        for (int64_t i = 0; i < n; ++i) tmp[i] = order[lo + i];
        /* stable merge sort by key */
        int64_t* a = tmp; int64_t* b = ws->buf + lo; /* bins no longer needed */
        for (int64_t w = 1; w < n; w *= 2) {
            for (int64_t i = 0; i < n; i += 2 * w) {
                int64_t m = i + w < n ? i + w : n, e = i + 2 * w < n ? i + 2 * w : n;
                int64_t p = i, q = m, o = i;
                while (p < m && q < e) {
                    double kp = s->cen[3 * a[p] + axis], kq = s->cen[3 * a[q] + axis];
                    if (kq < kp) b[o++] = a[q++]; else b[o++] = a[p++];
                }
                while (p < m) b[o++] = a[p++];
                while (q < e) b[o++] = a[q++];
            }
            int64_t* sw = a; a = b; b = sw;
        }
        for (int64_t i = 0; i < n; ++i) order[lo + i] = a[i];
        mid = lo + count / 2;
    } else {
        int64_t o = 0;
        for (int64_t i = lo; i < hi; ++i) if (bins[i - lo] < best_split) tmp[o++] = order[i];
        int64_t nl = o;
        for (int64_t i = lo; i < hi; ++i) if (bins[i - lo] >= best_split) tmp[o++] = order[i];
        for (int64_t i = 0; i < count; ++i) order[lo + i] = tmp[i];
        mid = lo + nl;
    }
    int64_t li = add_node(s);
    add_node(s);
    s->node_left[idx] = li;
    build_rec(s, ws, li, lo, mid);
    build_rec(s, ws, li + 1, mid, hi);
}

static float f32_of(double x) { return (float)x; }

/* Material reflection factors: E_b *= (1 - alpha_b) * w_b with
 * w_b = s_b / p (diffuse) or (1 - s_b) / (1 - p) (specular),
 * p = mean_b(s_b) summed sequentially. */
static void material_tables(efo_scene* s, const double* absorption, const double* scattering) {
    int nb = s->n_bands;
    s->fd = calloc((size_t)s->n_mat * nb, sizeof(float));
    s->fs = calloc((size_t)s->n_mat * nb, sizeof(float));
    s->fr = calloc((size_t)s->n_mat * nb, sizeof(float));
    s->pdiff = calloc((size_t)s->n_mat, sizeof(double));
    for (int m = 0; m < s->n_mat; ++m) {
        double p = 0.0;
        for (int b = 0; b < nb; ++b) p += scattering[m * nb + b];
        p = p / (double)nb;
        s->pdiff[m] = p;
        for (int b = 0; b < nb; ++b) {
            double keep = 1.0 - absorption[m * nb + b];
            double sb = scattering[m * nb + b];
            s->fd[m * nb + b] = p > 0.0 ? f32_of(keep * (sb / p)) : 0.0f;
            s->fs[m * nb + b] = p < 1.0 ? f32_of(keep * ((1.0 - sb) / (1.0 - p))) : 0.0f;
            s->fr[m * nb + b] = f32_of(keep * sb);
        }
    }
}

efo_scene* efo_scene_create(const double* v0, const double* e1, const double* e2,
                            const double* normals, const int64_t* mat, int64_t n_tri,
                            const double* absorption, const double* scattering,
                            int n_mat, int n_bands) {
    efo_scene* s = calloc(1, sizeof(efo_scene));
    s->n_tri = n_tri; s->v0 = v0; s->e1 = e1; s->e2 = e2; s->normals = normals; s->mat = mat;
    s->n_bands = n_bands; s->n_mat = n_mat;
    material_tables(s, absorption, scattering);
    if (n_tri == 0) return s;
    s->tri_min = malloc(sizeof(double) * 3 * n_tri);
    s->tri_max = malloc(sizeof(double) * 3 * n_tri);
    s->cen = malloc(sizeof(double) * 3 * n_tri);
    for (int64_t t = 0; t < n_tri; ++t) {
        for (int k = 0; k < 3; ++k) {
            double a = v0[3 * t + k];
            double b = a + e1[3 * t + k];
            double c = a + e2[3 * t + k];
            double mn = a < b ? a : b; mn = mn < c ? mn : c;   /* np.minimum(np.minimum(v0, v0+e1), v0+e2) */
            double mx = a > b ? a : b; mx = mx > c ? mx : c;
            s->tri_min[3 * t + k] = mn;
            s->tri_max[3 * t + k] = mx;
            s->cen[3 * t + k] = (mn + mx) * 0.5;
        }
    }
    s->tri_order = malloc(sizeof(int64_t) * n_tri);
    for (int64_t t = 0; t < n_tri; ++t) s->tri_order[t] = t;
    build_ws ws;
    ws.buf = malloc(sizeof(int64_t) * n_tri);
    ws.tmp = malloc(sizeof(int64_t) * n_tri);
    int64_t root = add_node(s);
    build_rec(s, &ws, root, 0, n_tri);
    free(ws.buf); free(ws.tmp);
    return s;
}

void efo_scene_destroy(efo_scene* s) {
    if (!s) return;
    free(s->fd); free(s->fs); free(s->fr); free(s->pdiff);
    free(s->node_min); free(s->node_max); free(s->node_left); free(s->node_start); free(s->node_count);
    free(s->tri_order); free(s->tri_min); free(s->tri_max); free(s->cen);
    free(s);
}

int64_t efo_scene_n_nodes(const efo_scene* s) { return s->n_nodes; }

/* Copy out the reference BVH arrays (for pinning against bvh.py). */
void efo_scene_bvh(const efo_scene* s, double* nmin, double* nmax, int64_t* left,
                   int64_t* start, int64_t* count, int64_t* order) {
    memcpy(nmin, s->node_min, sizeof(double) * 3 * s->n_nodes);
    memcpy(nmax, s->node_max, sizeof(double) * 3 * s->n_nodes);
    memcpy(left, s->node_left, sizeof(int64_t) * s->n_nodes);
    memcpy(start, s->node_start, sizeof(int64_t) * s->n_nodes);
    memcpy(count, s->node_count, sizeof(int64_t) * s->n_nodes);
    memcpy(order, s->tri_order, sizeof(int64_t) * s->n_tri);
}

void efo_material_tables(const efo_scene* s, float* fd, float* fs, double* pdiff) {
    memcpy(fd, s->fd, sizeof(float) * s->n_mat * s->n_bands);
    memcpy(fs, s->fs, sizeof(float) * s->n_mat * s->n_bands);
    memcpy(pdiff, s->pdiff, sizeof(double) * s->n_mat);
}

/* ------------------------------------------------------------------ */
/* Queries                                                              */
/* ------------------------------------------------------------------ */
typedef struct {
    double t, u, v;
    int64_t tri;
    int64_t n_nodes, n_tris; /* work counters (reference algorithm) */
    int tie;                 /* an exactly equal t was seen for the winner */
} hit_info;

/* np.minimum / np.maximum / .max / .min propagate NaN */
static inline double np_min(double a, double b) { return (isnan(a) || isnan(b)) ? NAN : (a < b ? a : b); }
static inline double np_max(double a, double b) { return (isnan(a) || isnan(b)) ? NAN : (a > b ? a : b); }

/* BVH.intersect, bvh.py:130-160 */
static void bvh_intersect(const efo_scene* s, const double* o, const double* d, double t_min,
                          double t_max, int vmode, hit_info* h, int64_t* stack) {
    h->t = INFINITY; h->tri = -1; h->u = h->v = 0.0; h->n_nodes = 0; h->n_tris = 0; h->tie = 0;
    if (s->n_tri == 0) return;
    double inv[3];
    for (int k = 0; k < 3; ++k) inv[k] = fabs(d[k]) > 1e-300 ? 1.0 / d[k] : INFINITY;
    double best_t = t_max, bu = 0.0, bv = 0.0;
    int64_t best_tri = -1;
    int tie = 0;
    int64_t sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        int64_t node = stack[--sp];
        h->n_nodes++;
        const double* mn = &s->node_min[3 * node];
        const double* mx = &s->node_max[3 * node];
        double nr = 0.0, fr = 0.0;
        for (int k = 0; k < 3; ++k) {
            double t0 = (mn[k] - o[k]) * inv[k];
            double t1 = (mx[k] - o[k]) * inv[k];
            double lo = np_min(t0, t1), hi = np_max(t0, t1);
            nr = k == 0 ? lo : np_max(nr, lo);
            fr = k == 0 ? hi : np_min(fr, hi);
        }
        if (nr > fr || fr < t_min || nr > best_t) continue;
        if (s->node_left[node] < 0) {
            int64_t st = s->node_start[node], cnt = s->node_count[node];
            /* ray_triangles over the leaf with t_max = best_t, then argmin */
            double lt = INFINITY, lu = 0.0, lv = 0.0;
            int64_t lk = -1;
            int ltie = 0;
            for (int64_t i = 0; i < cnt; ++i) {
                int64_t id = s->tri_order[st + i];
                double t, u, v;
                h->n_tris++;
                int ok = mt_test(o, d, &s->v0[3 * id], &s->e1[3 * id], &s->e2[3 * id], vmode, (int)cnt, &t, &u, &v);
                ok = ok && (t > t_min) && (t <= best_t);
                if (!ok) continue;
                if (t < lt) { lt = t; lu = u; lv = v; lk = id; ltie = 0; }
                else if (t == lt) ltie = 1;
            }
            if (lk >= 0) {
                tie = (lt == best_t && best_tri >= 0) || ltie;
                best_t = lt; best_tri = lk; bu = lu; bv = lv;
            }
        } else {
            stack[sp++] = s->node_left[node];
            stack[sp++] = s->node_left[node] + 1;
        }
    }
    if (best_tri < 0) return;
    h->t = best_t; h->tri = best_tri; h->u = bu; h->v = bv; h->tie = tie;
}

/* brute all-triangle closest hit, as intersect_batch for T <= 512
 * (scene.py:216-223): t > t_min, no t_max, argmin -> lowest id on ties */
static void brute_intersect(const efo_scene* s, const double* o, const double* d, double t_min,
                            hit_info* h) {
    h->t = INFINITY; h->tri = -1; h->u = h->v = 0.0; h->n_nodes = 0; h->n_tris = s->n_tri; h->tie = 0;
    for (int64_t i = 0; i < s->n_tri; ++i) {
        double t, u, v;
        int ok = mt_test(o, d, &s->v0[3 * i], &s->e1[3 * i], &s->e2[3 * i], 0, 1, &t, &u, &v);
        if (!(ok && t > t_min)) continue;
        if (t < h->t) { h->t = t; h->tri = i; h->u = u; h->v = v; h->tie = 0; }
        else if (t == h->t) h->tie = 1;
    }
}

/* SceneModel.intersect_batch (scene.py:208-230).  mode: 0 = the
 * reference dispatch (brute <= 512 else BVH), 1 = force brute, 2 = force BVH. */
void efo_intersect_batch(const efo_scene* s, const double* o, const double* d, int64_t n,
                         double t_min, const double* t_max, int mode, int vmode,
                         double* t_out, int64_t* tri_out, uint8_t* hit_out,
                         int64_t* n_nodes, int64_t* n_tris) {
    int64_t* stack = malloc(sizeof(int64_t) * 4096);
    int brute = mode == 1 || (mode == 0 && s->n_tri <= EFO_BRUTE_MAX);
    for (int64_t i = 0; i < n; ++i) {
        hit_info h;
        if (brute) brute_intersect(s, &o[3 * i], &d[3 * i], t_min, &h);
        else bvh_intersect(s, &o[3 * i], &d[3 * i], t_min, t_max ? t_max[i] : INFINITY, vmode, &h, stack);
        t_out[i] = h.t; tri_out[i] = h.tri; hit_out[i] = h.tri >= 0;
        if (n_nodes) n_nodes[i] = h.n_nodes;
        if (n_tris) n_tris[i] = h.n_tris;
    }
    free(stack);
}

/* ------------------------------------------------------------------ */
/* SH evaluation, sh.py:86-126 (same expression trees)                 */
/* ------------------------------------------------------------------ */
static const double C0 = 0.28209479177387814;
static const double C1 = 0.4886025119029199;
static const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                             -1.0925484305920792, 0.5462742152960396};
static const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                             0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                             -0.5900435899266435};
static const double C4[9] = {2.5033429417967046, -1.7701307697799304, 0.9461746957575601,
                             -0.6690465435572892, 0.10578554691520431, -0.6690465435572892,
                             0.47308734787878004, -1.7701307697799304, 0.6258357354491761};

void efo_eval_sh(const double* dir, int order, double* out) {
    double x = dir[0], y = dir[1], z = dir[2];
    out[0] = C0;
    if (order >= 1) {
        out[1] = -C1 * y;
        out[2] = C1 * z;
        out[3] = -C1 * x;
    }
    if (order >= 2) {
        double xx = x * x, yy = y * y, zz = z * z;
        out[4] = C2[0] * x * y;
        out[5] = C2[1] * y * z;
        out[6] = C2[2] * (2.0 * zz - xx - yy);
        out[7] = C2[3] * x * z;
        out[8] = C2[4] * (xx - yy);
        if (order >= 3) {
            out[9] = C3[0] * y * (3.0 * xx - yy);
            out[10] = C3[1] * x * y * z;
            out[11] = C3[2] * y * (4.0 * zz - xx - yy);
            out[12] = C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            out[13] = C3[4] * x * (4.0 * zz - xx - yy);
            out[14] = C3[5] * z * (xx - yy);
            out[15] = C3[6] * x * (xx - 3.0 * yy);
        }
        if (order >= 4) {
            out[16] = C4[0] * x * y * (xx - yy);
            out[17] = C4[1] * y * z * (3.0 * xx - yy);
            out[18] = C4[2] * x * y * (7.0 * zz - 1.0);
            out[19] = C4[3] * y * z * (7.0 * zz - 3.0);
            out[20] = C4[4] * (zz * (35.0 * zz - 30.0) + 3.0);
            out[21] = C4[5] * x * z * (7.0 * zz - 3.0);
            out[22] = C4[6] * (xx - yy) * (7.0 * zz - 1.0);
            out[23] = C4[7] * x * z * (xx - 3.0 * yy);
            out[24] = C4[8] * (xx * (xx - 3.0 * yy) - yy * (3.0 * xx - yy));
        }
    }
}

void efo_eval_sh_batch(const double* dirs, int64_t n, int order, double* out) {
    int nk = (order + 1) * (order + 1);
    for (int64_t i = 0; i < n; ++i) efo_eval_sh(&dirs[3 * i], order, &out[i * nk]);
}

/* ------------------------------------------------------------------ */
/* Bounce loop (pinned in DESIGN.md 3)       */
/* ------------------------------------------------------------------ */
enum { ST_PATHS = 0, ST_SEGMENTS, ST_REFLECTIONS, ST_ARRIVALS, ST_DIRECT, ST_DROPPED, ST_ESCAPED,
       ST_NODES, ST_TRIS, ST_NEARTIE_PATHS, ST_COUNT };

typedef struct {
    int32_t n_bands, order, n_bins, max_bounces;
    double bin_len;        /* meters per IR bin = c * bin_s */
    double listener[3];
    double radius;
    uint32_t seed, frame;
    int32_t vmode;         /* 1: OpenBLAS order for v on BVH leaves (pin only) */
    int32_t mode;          /* 0 reference dispatch, 1 brute, 2 bvh */
    float e0;              /* initial per-band energy of every path */
    int32_t rain;          /* diffuse rain */
    int32_t er_max_order;  /* arrivals of order 1..er_max_order -> ER list */
} efo_trace_cfg;

typedef struct {
    int32_t src, order, tri0, tri1;
    double dist;
    float dir[3];
    float pad;
    float energy[8];
} efo_er_entry;

typedef struct {
    double* H;
    double* Dir;
    uint64_t* stats;
    efo_er_entry* er;
    int64_t er_cap;
    int64_t* er_count;
} efo_sink;

/* one arrival: order 0 -> Dir, 1..er_max_order -> ER list, else H bin */
static void commit(const efo_trace_cfg* cfg, efo_sink* k, uint32_t src_key, int order, int tri0,
                   int tri1, double dist, double ux, double uy, double uz, const float* c) {
    const int nb = cfg->n_bands;
    const int nk = (cfg->order + 1) * (cfg->order + 1);
    k->stats[ST_ARRIVALS]++;
    double* dst = NULL;
    if (order == 0) {
        k->stats[ST_DIRECT]++;
        dst = k->Dir;
    } else if (order <= cfg->er_max_order) {
        if (*k->er_count < k->er_cap) {
            efo_er_entry* e = &k->er[*k->er_count];
            e->src = (int32_t)src_key; e->order = order; e->tri0 = tri0; e->tri1 = tri1;
            e->dist = dist;
            e->dir[0] = (float)ux; e->dir[1] = (float)uy; e->dir[2] = (float)uz; e->pad = 0.f;
            for (int b = 0; b < 8; ++b) e->energy[b] = b < nb ? c[b] : 0.f;
        }
        (*k->er_count)++;
        return;
    } else {
        double q = dist / cfg->bin_len;
        if (q < (double)cfg->n_bins) dst = &k->H[(int64_t)q * nb * nk];
        else k->stats[ST_DROPPED]++;
    }
    if (dst) {
        double dir[3] = {ux, uy, uz}, Y[EFO_MAX_NK];
        efo_eval_sh(dir, cfg->order, Y);
        for (int b = 0; b < nb; ++b)
            for (int kk = 0; kk < nk; ++kk) dst[b * nk + kk] += (double)(c[b] * (float)Y[kk]);
    }
}


/* Trace rays ray_ids[0..n) (or ray0 + i when ray_ids is NULL) of one source.
 * H: (n_bins, n_bands, nk) f64 accumulator, Dir: (n_bands, nk) f64.
 * stats: u64[ST_COUNT]; sum_t: f64 sum of reflected segment lengths.
 * Optional per-path outputs: nseg[i]; ids[i*max_bounces + j] = hit triangle
 * of segment j (-1 = escape); first_tie[i] = first segment index whose hit is
 * a documented near-tie (min(u,v,1-u-v) < 1e-6 or an exact t tie), else -1. */
void efo_trace(const efo_scene* s, const efo_trace_cfg* cfg, uint32_t src_key,
               const double* src_pos, const uint32_t* ray_ids, uint32_t ray0, int64_t n,
               double* H, double* Dir, uint64_t* stats, double* sum_t,
               int32_t* nseg_out, int32_t* ids_out, int32_t* first_tie_out,
               efo_er_entry* er, int64_t er_cap, int64_t* er_count) {
    int64_t er_dummy = 0;
    efo_sink sink = {H, Dir, stats, er, er_cap, er_count ? er_count : &er_dummy};
    const int nb = cfg->n_bands;
    int64_t* stack = malloc(sizeof(int64_t) * 4096);
    int brute = cfg->mode == 1 || (cfg->mode == 0 && s->n_tri <= EFO_BRUTE_MAX);
    const double r2 = cfg->radius * cfg->radius;
    for (int64_t i = 0; i < n; ++i) {
        uint32_t ray = ray_ids ? ray_ids[i] : ray0 + (uint32_t)i;
        double o[3] = {src_pos[0], src_pos[1], src_pos[2]};
        double d[3];
        efo_sample_sphere(cfg->seed, src_key, ray, cfg->frame, d);
        float E[EFO_MAX_BANDS];
        for (int b = 0; b < nb; ++b) E[b] = cfg->e0;
        double plen = 0.0;
        int nrefl = 0, nseg = 0, first_tie = -1;
        int tri0 = -1, tri1 = -1, last_diffuse = 0;
        stats[ST_PATHS]++;
        for (;;) {
            hit_info h;
            if (brute) brute_intersect(s, o, d, EFO_RAY_EPS, &h);
            else bvh_intersect(s, o, d, EFO_RAY_EPS, INFINITY, cfg->vmode, &h, stack);
            stats[ST_NODES] += (uint64_t)h.n_nodes;
            stats[ST_TRIS] += (uint64_t)h.n_tris;
            int hit = h.tri >= 0;
            if (hit && first_tie < 0) {
                double w = 1.0 - h.u - h.v;
                double m = h.u < h.v ? h.u : h.v;
                m = m < w ? m : w;
                if (m < 1e-6 || h.tie) first_tie = nseg;
            }
            if (ids_out) ids_out[i * cfg->max_bounces + nseg] = (int32_t)h.tri;
            /* listener sphere receiver (skipped after a diffuse bounce when
             * diffuse rain is the listener connection) */
            if (!(cfg->rain && last_diffuse)) {
                double Lo[3] = {cfg->listener[0] - o[0], cfg->listener[1] - o[1], cfg->listener[2] - o[2]};
                double tc = dot3(Lo, d);
                double tlim = hit ? h.t : INFINITY;
                if (tc > 0.0 && tc < tlim) {
                    double dist2 = dot3(Lo, Lo);
                    double perp2 = dist2 - tc * tc;
                    if (perp2 <= r2) commit(cfg, &sink, src_key, nrefl, tri0, tri1, plen + tc,
                                            -d[0], -d[1], -d[2], E);
                }
            }
            nseg++;
            stats[ST_SEGMENTS]++;
            if (!hit) { stats[ST_ESCAPED]++; break; }
            /* reflection */
            double t = h.t;
            plen += t;
            *sum_t += t;
            o[0] = o[0] + t * d[0];
            o[1] = o[1] + t * d[1];
            o[2] = o[2] + t * d[2];
            nrefl++;
            if (nrefl == 1) tri0 = (int)h.tri;
            if (nrefl == 2) tri1 = (int)h.tri;
            stats[ST_REFLECTIONS]++;
            int64_t m = s->mat[h.tri];
            const double* nrm = &s->normals[3 * h.tri];
            double u1, u2;
            draw2(ray, (uint32_t)nrefl, 0u, cfg->frame, cfg->seed, src_key, &u1, &u2);
            int diffuse = u1 < s->pdiff[m];
            double nd = dot3(nrm, d);
            if (cfg->rain && diffuse) {
                /* diffuse rain: c_b = E_b (1-a_b) s_b cos r^2 / d^2 if visible */
                double sg = nd > 0.0 ? -1.0 : 1.0;
                double L[3] = {cfg->listener[0] - o[0], cfg->listener[1] - o[1], cfg->listener[2] - o[2]};
                double d2 = dot3(L, L);
                double dd = sqrt(d2);
                double sn[3] = {sg * nrm[0], sg * nrm[1], sg * nrm[2]};
                double cosv = dot3(sn, L) / dd;
                if (cosv > 0.0 && dd > EFO_RAY_EPS) {
                    double e[3] = {L[0] / dd, L[1] / dd, L[2] / dd};
                    double limit = dd - EFO_RAY_EPS;
                    hit_info sh;
                    if (brute) {
                        brute_intersect(s, o, e, EFO_RAY_EPS, &sh);
                        if (sh.tri >= 0 && !(sh.t <= limit)) sh.tri = -1;
                    } else {
                        bvh_intersect(s, o, e, EFO_RAY_EPS, limit, cfg->vmode, &sh, stack);
                    }
                    if (sh.tri < 0) {
                        float gf = (float)(cosv * r2 / d2);
                        float c[EFO_MAX_BANDS];
                        for (int b = 0; b < nb; ++b) c[b] = E[b] * s->fr[m * nb + b] * gf;
                        commit(cfg, &sink, src_key, nrefl, tri0, tri1, plen + dd, -e[0], -e[1], -e[2], c);
                    }
                }
            }
            last_diffuse = diffuse;
            const float* f = diffuse ? &s->fd[m * nb] : &s->fs[m * nb];
            for (int b = 0; b < nb; ++b) E[b] = E[b] * f[b];
            if (diffuse) {
                double nn[3] = {nrm[0], nrm[1], nrm[2]};
                if (nd > 0.0) { nn[0] = -nn[0]; nn[1] = -nn[1]; nn[2] = -nn[2]; }
                efo_sample_cosine(cfg->seed, src_key, ray, (uint32_t)nrefl, cfg->frame, nn, d);
            } else {
                double k2 = 2.0 * nd;
                d[0] = d[0] - k2 * nrm[0];
                d[1] = d[1] - k2 * nrm[1];
                d[2] = d[2] - k2 * nrm[2];
            }
            if (nrefl >= cfg->max_bounces) break;
        }
        if (first_tie >= 0) stats[ST_NEARTIE_PATHS]++;
        if (nseg_out) nseg_out[i] = nseg;
        if (first_tie_out) first_tie_out[i] = first_tie;
    }
    free(stack);
}

// Uniform grid over the triangles, used by the warp-cooperative tail mode of
// the trace kernel: when a warp has one or two live paths left,
// all 32 lanes answer each closest-hit query together by walking the grid
// cells along the ray (3-D DDA) and testing a cell's triangles 32 at a time.
//
// Triangles are registered in every cell their padded bounding box overlaps,
// so a hit that rounding pushes just past a cell's exit distance is found
// again in the next cell.  Cell lists store leaf-order triangle positions
// (the GpuTri payload the BVH path reads).
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

#include "ef_internal.h"

namespace ef {

void build_grid(const double* v0, const double* e1, const double* e2, int64_t n,
                const std::vector<int64_t>& leaf_order, double pad, HostGrid& g) {
    if (n <= 0) throw std::runtime_error("build_grid: empty scene");
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    std::vector<double> tlo(3 * n), thi(3 * n);
    for (int64_t t = 0; t < n; ++t)
        for (int k = 0; k < 3; ++k) {
            const double a = v0[3 * t + k], b = a + e1[3 * t + k], c = a + e2[3 * t + k];
            tlo[3 * t + k] = std::min(a, std::min(b, c)) - pad;
            thi[3 * t + k] = std::max(a, std::max(b, c)) + pad;
            lo[k] = std::min(lo[k], tlo[3 * t + k]);
            hi[k] = std::max(hi[k], thi[3 * t + k]);
        }
    // about kCellsPerTri cells per triangle, cubic-ish cells, each axis >= 1
    double ext[3], vol = 1.0;
    for (int k = 0; k < 3; ++k) {
        ext[k] = std::max(hi[k] - lo[k], 1e-6);
        lo[k] -= 1e-6 * ext[k];
        ext[k] *= 1.0 + 2e-6;
        vol *= ext[k];
    }
    const double target = std::min<double>(kGridCellsPerTri * (double)n, (double)kGridMaxCells);
    const double cell = std::cbrt(vol / target);
    for (int k = 0; k < 3; ++k) {
        g.dims[k] = (int32_t)std::max(1.0, std::min(std::ceil(ext[k] / cell), 2048.0));
        g.lo[k] = lo[k];
        g.cell[k] = ext[k] / g.dims[k];
    }
    const int64_t ncell = (int64_t)g.dims[0] * g.dims[1] * g.dims[2];
    std::vector<uint32_t> count(ncell + 1, 0);
    std::vector<int64_t> pos_of(n);
    for (int64_t i = 0; i < n; ++i) pos_of[leaf_order[i]] = i;
    auto cell_range = [&](int64_t t, int c0[3], int c1[3]) {
        for (int k = 0; k < 3; ++k) {
            c0[k] = std::max(0, std::min(g.dims[k] - 1, (int)std::floor((tlo[3 * t + k] - g.lo[k]) / g.cell[k])));
            c1[k] = std::max(0, std::min(g.dims[k] - 1, (int)std::floor((thi[3 * t + k] - g.lo[k]) / g.cell[k])));
        }
    };
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
            uint32_t acc = 0;
            for (int64_t c = 0; c < ncell; ++c) {
                const uint32_t v = count[c];
                count[c] = acc;
                acc += v;
            }
            count[ncell] = acc;
            g.cell_start.assign(count.begin(), count.end());
            g.cell_tris.assign(acc, 0);
        }
        std::vector<uint32_t> fill = pass == 1 ? count : std::vector<uint32_t>();
        for (int64_t t = 0; t < n; ++t) {
            int c0[3], c1[3];
            cell_range(t, c0, c1);
            for (int z = c0[2]; z <= c1[2]; ++z)
                for (int y = c0[1]; y <= c1[1]; ++y)
                    for (int x = c0[0]; x <= c1[0]; ++x) {
                        const int64_t c = ((int64_t)z * g.dims[1] + y) * g.dims[0] + x;
                        if (pass == 0) ++count[c];
                        else g.cell_tris[fill[c]++] = (uint32_t)pos_of[t];
                    }
        }
        if (pass == 0 && [&] {
                uint64_t tot = 0;
                for (int64_t c = 0; c < ncell; ++c) tot += count[c];
                return tot > (uint64_t)kGridMaxRefs;
            }())
            throw std::runtime_error("build_grid: too many cell references");
    }
    // keep every cell list sorted by leaf position (deterministic order)
    for (int64_t c = 0; c < ncell; ++c)
        std::sort(g.cell_tris.begin() + g.cell_start[c], g.cell_tris.begin() + g.cell_start[c + 1]);
}

}  // namespace ef

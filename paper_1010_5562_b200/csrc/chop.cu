// chop.cu — a layout's rects cut into T x T tiles (NEXT-3, the paper's flow: "chops polygons and places
// them in their corresponding tiles. Each tile is then transformed individually"; reading
// A17 of DESIGN.md).  The tiles then go through fcfs_vertices_from_rects / fcfs_coeffs_batched as a
// batch of clips with variable K.
//
//   1. k_chop_count: thread per rect: range check, number of overlapped tiles;
//   2. CUB exclusive scan: each rect's first piece;
//   3. k_chop_emit: thread per rect: one (tile id, rect index) pair per overlapped tile, ty-major;
//   4. CUB radix sort of the pairs by tile id — stable, so pieces stay in rect order within a tile;
//   5. k_chop_gather: each sorted pair's piece (the rect cut to its tile, tile-local) in tile order;
//      k_chop_tile_ptr: CSR over tiles by lower_bound.
// One stream sync (the piece count).
#include <cub/cub.cuh>

#include "common.cuh"

namespace fcfs {

struct ChopWs {
    int64_t *cnt, *off;
    uint32_t *key_a, *key_b;
    int32_t *idx_a, *idx_b;
    int64_t *n;
    int32_t *err;
    void *cub_tmp;
    size_t cub_bytes;
};

__global__ void k_chop_count(const int4 *__restrict__ rects, int64_t R, int32_t T, int32_t tiles_x, int32_t tiles_y,
                             int64_t *cnt, int32_t *err) {
    const int64_t W = (int64_t)tiles_x * T, H = (int64_t)tiles_y * T;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
        const int4 q = rects[r];
        if (q.x < 0 || q.y < 0 || q.z > W || q.w > H || q.x >= q.z || q.y >= q.w) {
            atomicOr(err, 1);
            cnt[r] = 0;
            continue;
        }
        const int64_t nx = (q.z - 1) / T - q.x / T + 1, ny = (q.w - 1) / T - q.y / T + 1;
        cnt[r] = nx * ny;
    }
}

__global__ void k_chop_emit(const int4 *__restrict__ rects, int64_t R, int32_t T, int32_t tiles_x,
                            const int64_t *__restrict__ cnt, const int64_t *__restrict__ off, int64_t cap,
                            uint32_t *keys, int32_t *idx) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R; r += (int64_t)gridDim.x * blockDim.x) {
        if (cnt[r] == 0) continue;
        const int4 q = rects[r];
        int64_t o = off[r];
        for (int32_t ty = q.y / T; (int64_t)ty * T < q.w; ++ty)
            for (int32_t tx = q.x / T; (int64_t)tx * T < q.z; ++tx, ++o) {
                if (o >= cap) return;
                keys[o] = (uint32_t)ty * (uint32_t)tiles_x + (uint32_t)tx;
                idx[o] = (int32_t)r;
            }
    }
}

// piece i of the tile order: rect idx[i] cut to tile keys[i], in tile-local coordinates
__global__ void k_chop_gather(const int4 *__restrict__ rects, const uint32_t *__restrict__ keys,
                              const int32_t *__restrict__ idx, int64_t n, int32_t T, int32_t tiles_x, int4 *out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int4 q = rects[idx[i]];
        const uint32_t t = keys[i];
        const int32_t ax = (int32_t)(t % (uint32_t)tiles_x) * T, ay = (int32_t)(t / (uint32_t)tiles_x) * T;
        out[i] = make_int4(max(q.x, ax) - ax, max(q.y, ay) - ay, min(q.z, ax + T) - ax, min(q.w, ay + T) - ay);
    }
}

// tile_ptr[t] = first sorted piece with tile id >= t, t in [0, tiles]
__global__ void k_chop_tile_ptr(const uint32_t *__restrict__ keys, int64_t n, int64_t tiles, int64_t *tile_ptr) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= tiles; t += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if ((int64_t)keys[mid] < t) lo = mid + 1; else hi = mid;
        }
        tile_ptr[t] = lo;
    }
}

static int key_bits(int64_t tiles) {
    int b = 1;
    while ((int64_t(1) << b) < tiles) ++b;
    return b;
}

static size_t chop_cub_bytes(int64_t R, int64_t cap, int64_t tiles) {
    size_t a = 0, b = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, a, (int64_t *)nullptr, (int64_t *)nullptr, (int)(R > 0 ? R : 1));
    cub::DeviceRadixSort::SortPairs(nullptr, b, (uint32_t *)nullptr, (uint32_t *)nullptr, (int32_t *)nullptr,
                                    (int32_t *)nullptr, (int)(cap > 0 ? cap : 1), 0, key_bits(tiles));
    return a > b ? a : b;
}

static void carve_chop(Carver &cv, int64_t R, int64_t cap, int64_t tiles, ChopWs &w) {
    const size_t r1 = (size_t)(R > 0 ? R : 1), c1 = (size_t)(cap > 0 ? cap : 1);
    w.cnt = cv.take<int64_t>(r1);
    w.off = cv.take<int64_t>(r1);
    w.key_a = cv.take<uint32_t>(c1);
    w.key_b = cv.take<uint32_t>(c1);
    w.idx_a = cv.take<int32_t>(c1);
    w.idx_b = cv.take<int32_t>(c1);
    w.n = cv.take<int64_t>(1);
    w.err = cv.take<int32_t>(4);
    w.cub_bytes = chop_cub_bytes(R, cap, tiles);
    w.cub_tmp = cv.take<char>(w.cub_bytes);
}

size_t chop_workspace_bytes(int64_t R, int64_t cap, int64_t tiles) {
    Carver cv(nullptr, 0);
    ChopWs w;
    carve_chop(cv, R, cap, tiles, w);
    return cv.used();
}

fcfs_status chop_rects(const int32_t *rects, int64_t R, int32_t T, int32_t tiles_x, int32_t tiles_y,
                       int32_t *out, int64_t cap, int64_t *tile_ptr, int64_t *n_host, void *ws, size_t ws_bytes,
                       cudaStream_t s) {
    const int64_t tiles = (int64_t)tiles_x * tiles_y;
    Carver cv(ws, ws_bytes);
    ChopWs W;
    carve_chop(cv, R, cap, tiles, W);
    if (!cv.fits()) {
        set_error("fcfs_chop_rects: workspace %zu < %zu bytes", ws_bytes, cv.used());
        return FCFS_E_WORKSPACE;
    }
    FCFS_TRY_CUDA(cudaMemsetAsync(W.err, 0, 4 * sizeof(int32_t), s));
    FCFS_TRY_CUDA(cudaMemsetAsync(W.n, 0, sizeof(int64_t), s));
    const int threads = 256;
    int64_t blocks = (R + threads - 1) / threads;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    int64_t n = 0;
    if (R > 0) {
        k_chop_count<<<(unsigned)blocks, threads, 0, s>>>((const int4 *)rects, R, T, tiles_x, tiles_y, W.cnt, W.err);
        FCFS_CHECK_LAUNCH("k_chop_count");
        size_t tb = W.cub_bytes;
        FCFS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(W.cub_tmp, tb, W.cnt, W.off, (int)R, s));
        count_launch(1);
        int64_t last[2] = {0, 0};
        FCFS_TRY_CUDA(cudaMemcpyAsync(&last[0], W.off + R - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        FCFS_TRY_CUDA(cudaMemcpyAsync(&last[1], W.cnt + R - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        int32_t errh = 0;
        FCFS_TRY_CUDA(cudaMemcpyAsync(&errh, W.err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        FCFS_TRY_CUDA(cudaStreamSynchronize(s));
        n = last[0] + last[1];
        if (n_host) *n_host = n;
        if (errh & 1) {
            set_error("fcfs_chop_rects: a rect lies outside the layout or is empty");
            return FCFS_E_RANGE;
        }
        if (n > cap) {
            set_error("fcfs_chop_rects: %lld pieces > cap=%lld", (long long)n, (long long)cap);
            return FCFS_E_CAPACITY;
        }
        k_chop_emit<<<(unsigned)blocks, threads, 0, s>>>((const int4 *)rects, R, T, tiles_x, W.cnt, W.off, cap,
                                                         W.key_a, W.idx_a);
        FCFS_CHECK_LAUNCH("k_chop_emit");
        tb = W.cub_bytes;
        FCFS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(W.cub_tmp, tb, W.key_a, W.key_b, W.idx_a, W.idx_b, (int)n, 0,
                                                      key_bits(tiles), s));
        count_launch(4);
        int64_t gb = (n + threads - 1) / threads;
        if (gb > 148 * 16) gb = 148 * 16;
        if (gb < 1) gb = 1;
        k_chop_gather<<<(unsigned)gb, threads, 0, s>>>((const int4 *)rects, W.key_b, W.idx_b, n, T, tiles_x,
                                                       (int4 *)out);
        FCFS_CHECK_LAUNCH("k_chop_gather");
    } else if (n_host) {
        *n_host = 0;
    }
    int64_t pb = (tiles + 1 + threads - 1) / threads;
    if (pb > 148 * 8) pb = 148 * 8;
    k_chop_tile_ptr<<<(unsigned)pb, threads, 0, s>>>(W.key_b, n, tiles, tile_ptr);
    FCFS_CHECK_LAUNCH("k_chop_tile_ptr");
    return FCFS_OK;
}

}  // namespace fcfs

// extract.cu — a1: vertex extraction, rects -> canonical signed corners + exact area.
//
// Follows Alg. 2 lines 1-14 re-expressed on signed corners:
// the +1/-1 entries of V^KL/S^KL at the ends of horizontal edges are the
// mixed difference w = f(x,y) - f(x-1,y) - f(x,y-1) + f(x-1,y-1) of the cell mask f
// (Prop. 1, half-open convention P:398-402).  Step 1's area is
// sum_k w_k x_k y_k, accumulated exactly in int64.
//
// Pipeline (all on the caller's stream, one host sync at the end for K):
//   1. raw corners:  singleton groups -> 4 corners per rect (thread per rect);
//                    unions -> one CTA per group: coordinate compression, 2-D difference
//                    array of the coverage count on the compressed grid in SMEM, prefix
//                    sums, union indicator, mixed difference, append non-zeros.
//   2. CUB radix sort of 64-bit keys (clip<<42 | y<<21 | x) with int32 weights.
//   3. CUB reduce-by-key (sum weights of equal keys; groups are SUMMED, reading A5).
//   4. drop zero weights: flag + exclusive scan + scatter into x, y, w; int64 area atomics.
//   5. corner_ptr by lower_bound of b<<42 in the compacted keys.
// Batched clips of singleton groups take the per-clip paths below (one CTA per clip, SMEM sort,
// look-back offsets, direct output) instead.
#include <cub/cub.cuh>
#include <utility>

#include "common.cuh"

namespace fcfs {

static constexpr int kCoordBits = 21;
static constexpr unsigned long long kSentinel = ~0ull;
static constexpr int kMaxGroup = 100;

struct ExtractWs {
    unsigned long long *keys_a, *keys_b;
    int32_t *w_a, *w_b;
    int32_t *flags, *pos;
    int64_t *num_runs, *K;
    int32_t *err;
    void *cub_tmp;
    size_t cub_bytes;
    int64_t cap_raw;
};

// key = clip | y | x with cb = coord_bits(T) bits per coordinate (0..T): the radix sort runs over
// 2 cb + clip_bits(B) bits only (c2, T = 4096: 27 bits, 4 onesweep passes instead of 6)
__host__ __device__ inline int coord_bits(int32_t T) {
    int b = 1;
    while ((int64_t(1) << b) <= (int64_t)T) ++b;
    return b;
}

__device__ __forceinline__ unsigned long long make_key(int64_t clip, int32_t y, int32_t x, int cb) {
    return ((unsigned long long)clip << (2 * cb)) | ((unsigned long long)y << cb) | (unsigned long long)x;
}

__device__ __forceinline__ int64_t find_clip(const int64_t *clip_ptr, int64_t B, int64_t g) {
    if (clip_ptr == nullptr) return 0;
    // last b with clip_ptr[b] <= g
    int64_t lo = 0, hi = B - 1;
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) >> 1;
        if (clip_ptr[mid] <= g) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ bool rect_ok(int4 q, int32_t T) {
    return q.x >= 0 && q.y >= 0 && q.z <= T && q.w <= T && q.x < q.z && q.y < q.w;
}

// one thread per rect, every rect its own group (group_ptr == NULL)
__global__ void k_singleton_corners(const int4 *__restrict__ rects, int64_t R,
                                    const int64_t *__restrict__ clip_ptr, int64_t B, int32_t T,
                                    unsigned long long *keys, int32_t *wts, int32_t *err) {
    const int cb = coord_bits(T);
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
         r += (int64_t)gridDim.x * blockDim.x) {
        int4 q = rects[r];
        int64_t b = find_clip(clip_ptr, B, r);
        if (!rect_ok(q, T)) {
            atomicOr(err, 1);
            q = make_int4(0, 0, 0, 0);
        }
        keys[4 * r + 0] = make_key(b, q.y, q.x, cb); wts[4 * r + 0] = 1;
        keys[4 * r + 1] = make_key(b, q.y, q.z, cb); wts[4 * r + 1] = -1;
        keys[4 * r + 2] = make_key(b, q.w, q.x, cb); wts[4 * r + 2] = -1;
        keys[4 * r + 3] = make_key(b, q.w, q.z, cb); wts[4 * r + 3] = 1;
        if (q.x == q.z) { wts[4 * r + 0] = wts[4 * r + 1] = wts[4 * r + 2] = wts[4 * r + 3] = 0; }
    }
}

// sort v[0..n) (stable rank sort, O(n) per thread) and unique it into uniq[0..*nu) (each distinct
// value's slot = number of distinct values before it, O(n) per thread: no serial pass)
__device__ __forceinline__ void compress(const int32_t *v, int n, int32_t *tmp, int32_t *uniq, int32_t *nu) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int32_t vi = v[i];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            int32_t vj = v[j];
            rank += (vj < vi) || (vj == vi && j < i);
        }
        tmp[rank] = vi;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const bool first = i == 0 || tmp[i] != tmp[i - 1];
        if (!first && i != n - 1) continue;
        int c = 0;
        for (int j = 1; j <= i; ++j) c += tmp[j] != tmp[j - 1];
        if (first) uniq[c] = tmp[i];
        if (i == n - 1) *nu = c + 1;
    }
    __syncthreads();
}

__device__ __forceinline__ int find_sorted(const int32_t *u, int n, int32_t key) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (u[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// one CTA per group: union of the group's rects on its compressed grid
__global__ void k_group_corners(const int4 *__restrict__ rects, const int64_t *__restrict__ group_ptr,
                                int64_t G, const int64_t *__restrict__ clip_ptr, int64_t B, int32_t T,
                                unsigned long long *keys, int32_t *wts, int64_t cap_raw,
                                unsigned long long *raw_count, int32_t *err) {
    const int cb = coord_bits(T);
    extern __shared__ __align__(16) unsigned char smem[];
    int4 *sr = (int4 *)smem;                                  // [kMaxGroup]
    int32_t *vx = (int32_t *)(sr + kMaxGroup);                // [2*kMaxGroup]
    int32_t *vy = vx + 2 * kMaxGroup;                         // [2*kMaxGroup]
    int32_t *ux = vy + 2 * kMaxGroup;                         // [2*kMaxGroup]
    int32_t *uy = ux + 2 * kMaxGroup;                         // [2*kMaxGroup]
    int32_t *tmp = uy + 2 * kMaxGroup;                        // [2*kMaxGroup]
    int32_t *nxy = tmp + 2 * kMaxGroup;                       // [2]
    int32_t *grid = nxy + 2;                                  // [nx*ny] (dynamic extent)

    for (int64_t g = blockIdx.x; g < G; g += gridDim.x) {
        int64_t r0 = group_ptr[g], r1 = group_ptr[g + 1];
        int n = (int)(r1 - r0);
        if (n <= 0) continue;
        if (n > kMaxGroup) {
            if (threadIdx.x == 0) atomicOr(err, 2);
            continue;
        }
        int64_t b = find_clip(clip_ptr, B, g);
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            int4 q = rects[r0 + i];
            if (!rect_ok(q, T)) { atomicOr(err, 1); q = make_int4(0, 0, 0, 0); }
            sr[i] = q;
            vx[2 * i] = q.x; vx[2 * i + 1] = q.z;
            vy[2 * i] = q.y; vy[2 * i + 1] = q.w;
        }
        __syncthreads();
        compress(vx, 2 * n, tmp, ux, &nxy[0]);
        compress(vy, 2 * n, tmp, uy, &nxy[1]);
        const int nx = nxy[0], ny = nxy[1];
        // difference array of the coverage count at grid points (i, j), i < nx, j < ny
        for (int t = threadIdx.x; t < nx * ny; t += blockDim.x) grid[t] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            int4 q = sr[i];
            if (q.x == q.z) continue;   // invalid rect, already flagged
            int i0 = find_sorted(ux, nx, q.x), i1 = find_sorted(ux, nx, q.z);
            int j0 = find_sorted(uy, ny, q.y), j1 = find_sorted(uy, ny, q.w);
            atomicAdd(&grid[i0 * ny + j0], 1);
            atomicAdd(&grid[i1 * ny + j0], -1);
            atomicAdd(&grid[i0 * ny + j1], -1);
            atomicAdd(&grid[i1 * ny + j1], 1);
        }
        __syncthreads();
        // prefix sums (warp per line, shuffle scans): along j for each i, then along i for each j ->
        // coverage count of cell (i, j), kept as the union indicator
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int i = warp; i < nx; i += nw) {
            int carry = 0;
            for (int j0 = 0; j0 < ny; j0 += 32) {
                const int j = j0 + lane;
                int v = j < ny ? grid[i * ny + j] : 0;
                for (int d = 1; d < 32; d <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, v, d);
                    if (lane >= d) v += u;
                }
                if (j < ny) grid[i * ny + j] = carry + v;
                carry += __shfl_sync(0xffffffffu, v, 31);
            }
        }
        __syncthreads();
        for (int j = warp; j < ny; j += nw) {
            int carry = 0;
            for (int i0 = 0; i0 < nx; i0 += 32) {
                const int i = i0 + lane;
                int v = i < nx ? grid[i * ny + j] : 0;
                for (int d = 1; d < 32; d <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, v, d);
                    if (lane >= d) v += u;
                }
                if (i < nx) grid[i * ny + j] = carry + v > 0 ? 1 : 0;
                carry += __shfl_sync(0xffffffffu, v, 31);
            }
        }
        __syncthreads();
        // mixed difference of the union indicator at every grid point; one slot reservation per warp
        for (int t0 = warp * 32; t0 < nx * ny; t0 += blockDim.x) {
            const int t = t0 + lane;
            int wv = 0, i = 0, j = 0;
            if (t < nx * ny) {
                i = t / ny; j = t - i * ny;
                const int c00 = grid[t];
                const int cm0 = i > 0 ? grid[t - ny] : 0;
                const int c0m = j > 0 ? grid[t - 1] : 0;
                const int cmm = (i > 0 && j > 0) ? grid[t - ny - 1] : 0;
                wv = c00 - cm0 - c0m + cmm;
            }
            const unsigned m = __ballot_sync(0xffffffffu, wv != 0);
            if (m == 0) continue;
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(raw_count, (unsigned long long)__popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (wv != 0) {
                const unsigned long long slot = base + __popc(m & ((1u << lane) - 1u));
                if ((int64_t)slot < cap_raw) {
                    keys[slot] = make_key(b, uy[j], ux[i], cb);
                    wts[slot] = wv;
                } else {
                    atomicOr(err, 4);
                }
            }
        }
        __syncthreads();
    }
}

// Polygon vertex lists (the paper's input, Alg. 2): one warp per polygon.  Every vertex
// is the end of its incoming edge and the start of its outgoing one, so with s = +1 for a clockwise
// (y up) list and -1 for a counter-clockwise one (sign of the vertex-form area sum_h y_a (x_b - x_a),
// reading A16), Alg. 2 lines 9-10 ("+1 at the end, -1 at the start of each horizontal edge",
// P:945-946) give vertex i the raw weight s ([edge i-1 horizontal] - [edge i horizontal]): one raw
// corner per vertex, no counting pass.  Collinear vertices get 0.  A diagonal or zero-length edge
// sets err bit 16, a vertex outside [0,T]^2 bit 1; the polygon then contributes nothing.
__global__ void k_polygon_corners(const int32_t *__restrict__ vx, const int32_t *__restrict__ vy,
                                  const int64_t *__restrict__ poly_ptr, int64_t P,
                                  const int64_t *__restrict__ clip_ptr, int64_t B, int32_t T,
                                  unsigned long long *keys, int32_t *wts, int32_t *err) {
    const int cb = coord_bits(T);
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P; p += nwarps) {
        const int64_t v0 = poly_ptr[p];
        const int64_t n = poly_ptr[p + 1] - v0;
        if (n <= 0) continue;
        const int64_t b = find_clip(clip_ptr, B, p);
        long long A = 0;
        bool bad = false, range = false;
        for (int64_t i = lane; i < n; i += 32) {
            const int64_t j = i + 1 == n ? 0 : i + 1;
            const int32_t xi = vx[v0 + i], yi = vy[v0 + i], xj = vx[v0 + j], yj = vy[v0 + j];
            range |= xi < 0 || yi < 0 || xi > T || yi > T;
            const bool hor = yi == yj && xi != xj, ver = xi == xj && yi != yj;
            bad |= !(hor || ver);
            if (hor) A += (long long)yi * (long long)(xj - xi);
        }
        for (int o = 16; o > 0; o >>= 1) A += __shfl_xor_sync(0xffffffffu, A, o);
        bad = __any_sync(0xffffffffu, bad);
        range = __any_sync(0xffffffffu, range);
        if (lane == 0 && (bad || range)) atomicOr(err, (bad ? 16 : 0) | (range ? 1 : 0));
        const int s = A < 0 ? -1 : 1;
        for (int64_t i = lane; i < n; i += 32) {
            const int64_t h = i == 0 ? n - 1 : i - 1, j = i + 1 == n ? 0 : i + 1;
            const int32_t xi = vx[v0 + i], yi = vy[v0 + i];
            const bool hin = vy[v0 + h] == yi && vx[v0 + h] != xi;
            const bool hout = vy[v0 + j] == yi && vx[v0 + j] != xi;
            const bool ok = !(bad || range);
            keys[v0 + i] = ok ? make_key(b, yi, xi, cb) : make_key(b, 0, 0, cb);
            wts[v0 + i] = ok ? s * ((int)hin - (int)hout) : 0;
        }
    }
}

__global__ void k_fill_sentinel(unsigned long long *keys, int32_t *wts, int64_t n,
                                const unsigned long long *raw_count) {
    int64_t start = raw_count ? (int64_t)*raw_count : 0;
    for (int64_t i = start + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = kSentinel;
        wts[i] = 0;
    }
}

// y-band of one clip (fcfs_vertices_from_rects_band): the raw corners with y in [y_lo, y_hi) are
// compacted (warp-aggregated append, any order: the sort follows) so that the sort and merge run over
// the band's share only.  A canonical corner is a sum over the raw corners of one (x, y) key, so the
// band's canonical corners are exactly the unbanded ones with y in the band.
__global__ void k_band_compact(const unsigned long long *__restrict__ keys, const int32_t *__restrict__ wts, int64_t n,
                               int cb, int32_t y_lo, int32_t y_hi, unsigned long long *okeys, int32_t *owts,
                               unsigned long long *count) {
    const unsigned long long mask = (1ull << cb) - 1;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); i0 < n; i0 += stride) {
        const int64_t i = i0 + lane;
        bool keep = false;
        unsigned long long k = kSentinel;
        int32_t wv = 0;
        if (i < n) {
            k = keys[i];
            wv = wts[i];
            const int32_t yy = (int32_t)((k >> cb) & mask);
            keep = k != kSentinel && wv != 0 && yy >= y_lo && yy < y_hi;
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (m == 0) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(count, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
            const unsigned long long slot = base + __popc(m & ((1u << lane) - 1u));
            FCFS_DCHECK((int64_t)slot < n);
            okeys[slot] = k;
            owts[slot] = wv;
        }
    }
}

__global__ void k_flags(const int32_t *wts, const int64_t *num_runs, int64_t n, int32_t *flags) {
    int64_t nr = *num_runs;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        flags[i] = (i < nr && wts[i] != 0) ? 1 : 0;
}

__global__ void k_scatter(const unsigned long long *ukeys, const int32_t *agg, const int32_t *flags,
                          const int32_t *pos, int64_t n, int64_t cap, int32_t *x, int32_t *y, int32_t *w,
                          unsigned long long *ckeys, int64_t *area, int64_t *K, int cb) {
    // warp-uniform loop: the area is reduced over the warp before the atomic (corners are sorted by
    // clip, so a warp nearly always holds one clip: one atomic per warp instead of one per corner)
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // lane 0 carries the warp's running area of one clip across iterations (one atomic per warp and clip
    // run instead of per iteration: a single large clip otherwise serialises ~K/32 atomics on area[0])
    int64_t acc_b = -1;
    long long acc_a = 0;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); i0 < n; i0 += stride) {
        const int64_t i = i0 + lane;
        const bool valid = i < n;
        long long a = 0;
        int64_t b = -1;
        if (valid) {
            if (i == n - 1) *K = (int64_t)pos[i] + flags[i];
            const unsigned long long key = ukeys[i];
            b = (int64_t)(key >> (2 * cb));
            if (flags[i]) {
                const int32_t xx = (int32_t)(key & ((1ull << cb) - 1));
                const int32_t yy = (int32_t)((key >> cb) & ((1ull << cb) - 1));
                const int64_t p = pos[i];
                ckeys[p] = key;
                if (p < cap) { x[p] = xx; y[p] = yy; w[p] = agg[i]; }
                a = (long long)agg[i] * (long long)xx * (long long)yy;
            }
        }
        const int64_t b0 = __shfl_sync(0xffffffffu, b, 0);
        if (__all_sync(0xffffffffu, !valid || b == b0)) {
            for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (lane == 0 && a != 0) {
                if (b0 != acc_b) {
                    if (acc_a != 0) atomicAdd((unsigned long long *)&area[acc_b], (unsigned long long)acc_a);
                    acc_b = b0;
                    acc_a = 0;
                }
                acc_a += a;
            }
        } else if (valid && a != 0) {
            atomicAdd((unsigned long long *)&area[b], (unsigned long long)a);
        }
    }
    if (lane == 0 && acc_a != 0) atomicAdd((unsigned long long *)&area[acc_b], (unsigned long long)acc_a);
}

__global__ void k_corner_ptr(const unsigned long long *ckeys, const int64_t *K, int64_t B, int64_t *corner_ptr,
                             int cb) {
    int64_t n = *K;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= B;
         b += (int64_t)gridDim.x * blockDim.x) {
        if (b == B) { corner_ptr[b] = n; continue; }
        unsigned long long target = (unsigned long long)b << (2 * cb);
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (ckeys[mid] < target) lo = mid + 1; else hi = mid;
        }
        corner_ptr[b] = lo;
    }
}

// ------------------------------------------------------------------------------------------
// Per-clip fast path (every rect its own group, clips of <= kClipRects rects, T < 2^16): one
// CTA per clip builds the clip's 4n raw corners with 32-bit keys (y << 16 | x), sorts them in
// shared memory (CUB BlockRadixSort), merges equal keys with a segmented block scan, drops zero
// weights, finds its output offset by a decoupled look-back over the clips before it
// (clip_lookback: corner_ptr without a separate scan) and writes the compacted clip straight
// into x, y, w, with its exact int64 area.  Same canonical (clip, y, x) order as the global path.
// ------------------------------------------------------------------------------------------
static constexpr int kClipThreads = 512;
static constexpr int kClipItems = 16;
static constexpr int kClipRects = kClipThreads * kClipItems / 4;   // 2048 rects -> 8192 corners
static_assert(kClipRects == 512 * 4, "bucket path: 4 rects per thread");

struct SegSum {
    int head;   // a segment starts at or before this element
    int val;
};
struct SegSumOp {
    __device__ __forceinline__ SegSum operator()(const SegSum &a, const SegSum &b) const {
        SegSum r;
        r.head = a.head | b.head;
        r.val = b.head ? b.val : a.val + b.val;
        return r;
    }
};

// Output offset of clip b by a decoupled look-back over the clips before it (one CTA per clip,
// CTAs dispatched in clip order, so every predecessor is resident or done): publish this clip's
// count, add predecessors' counts until one with a published inclusive prefix, publish ours.
// Writes corner_ptr[b] (and corner_ptr[B] for the last clip).  Thread 0 only.
static constexpr unsigned long long kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbMask = (1ull << 62) - 1;
__device__ int64_t clip_lookback(unsigned long long *status, int64_t b, int64_t B, int64_t count,
                                 int64_t *corner_ptr) {
    volatile unsigned long long *st = status;
    int64_t prefix = 0;
    if (b > 0) {
        st[b] = kLbAgg | (unsigned long long)count;
        __threadfence();
        for (int64_t j = b - 1;; --j) {
            unsigned long long v;
            do { v = st[j]; } while ((v >> 62) == 0);
            prefix += (int64_t)(v & kLbMask);
            if ((v >> 62) == 2) break;
        }
    }
    st[b] = kLbInc | (unsigned long long)(prefix + count);
    __threadfence();
    corner_ptr[b] = prefix;
    if (b == B - 1) corner_ptr[B] = prefix + count;
    return prefix;
}

// The same look-back walked by a whole warp (all 32 lanes call it; every lane returns the prefix): each
// step reads 32 predecessors' status words at once (lane l: clip j - l) instead of one, so a clip whose
// recent predecessors have only published their counts waits for one L2 round trip per 32 clips
// rather than per clip.  Same status protocol (mixes with clip_lookback).
// agg_published: the caller already stored this clip's aggregate (clip_publish_count), earlier in its
// work, so that its successors' walks do not wait for the rest of it.
__device__ __forceinline__ void clip_publish_count(unsigned long long *status, int64_t b, int64_t count) {
    if (b > 0) {
        volatile unsigned long long *st = status;
        st[b] = kLbAgg | (unsigned long long)count;
        __threadfence();
    }
}
__device__ int64_t clip_lookback_warp(unsigned long long *status, int64_t b, int64_t B, int64_t count,
                                      int64_t *corner_ptr, bool agg_published = false) {
    volatile unsigned long long *st = status;
    const int lane = threadIdx.x & 31;
    int64_t prefix = 0;
    if (b > 0) {
        if (lane == 0 && !agg_published) {
            st[b] = kLbAgg | (unsigned long long)count;
            __threadfence();
        }
        __syncwarp();
        for (int64_t j = b - 1;; j -= 32) {
            const int64_t idx = j - lane;
            unsigned long long v = kLbInc;                  // before clip 0: an inclusive prefix of 0
            if (idx >= 0) {
                do { v = st[idx]; } while ((v >> 62) == 0);
            }
            const unsigned inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
            // lanes up to (and including) the nearest inclusive predecessor contribute
            const int stop = inc ? __ffs(inc) - 1 : 31;
            long long c = lane <= stop ? (long long)(v & kLbMask) : 0;
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            prefix += c;
            if (inc) break;
        }
    }
    if (lane == 0) {
        st[b] = kLbInc | (unsigned long long)(prefix + count);
        __threadfence();
        corner_ptr[b] = prefix;
        if (b == B - 1) corner_ptr[B] = prefix + count;
    }
    __syncwarp();
    return prefix;
}

__global__ void __launch_bounds__(kClipThreads, 1)
k_clip_corners(const int4 *__restrict__ rects, const int64_t *__restrict__ clip_ptr, int64_t B, int64_t R,
               int32_t T, int32_t *xs, int32_t *ys, int32_t *ws, int64_t cap, int64_t *corner_ptr,
               unsigned long long *status, int64_t *area, int32_t *err) {
    typedef cub::BlockRadixSort<uint32_t, kClipThreads, kClipItems, int32_t> Sort;
    typedef cub::BlockScan<SegSum, kClipThreads> SegScan;
    typedef cub::BlockScan<int, kClipThreads> IntScan;
    typedef cub::BlockReduce<long long, kClipThreads> Red;
    __shared__ union {
        typename Sort::TempStorage sort;
        typename SegScan::TempStorage seg;
        typename IntScan::TempStorage scan;
        typename Red::TempStorage red;
    } tmp;
    __shared__ uint32_t edge_first[kClipThreads], edge_last[kClipThreads];
    __shared__ int64_t s_off;
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
        const int64_t r0 = clip_ptr ? clip_ptr[b] : 0, r1 = clip_ptr ? clip_ptr[b + 1] : R;
        const int n = (int)(r1 - r0);
        if (n > kClipRects) {
            // the caller falls back to the general path; the clip still publishes a count (0) so
            // that the look-back of the clips after it completes
            if (threadIdx.x == 0) { atomicOr(err, 8); area[b] = 0; clip_lookback(status, b, B, 0, corner_ptr); }
            continue;
        }
        uint32_t key[kClipItems];
        int32_t val[kClipItems];
#pragma unroll
        for (int j = 0; j < kClipItems / 4; ++j) {
            const int r = threadIdx.x * (kClipItems / 4) + j;
            int4 q = make_int4(0, 0, 0, 0);
            bool ok = r < n;
            if (ok) {
                q = rects[r0 + r];
                if (!rect_ok(q, T)) { atomicOr(err, 1); ok = false; }
            }
            const uint32_t kx0 = (uint32_t)q.x, kx1 = (uint32_t)q.z, ky0 = (uint32_t)q.y, ky1 = (uint32_t)q.w;
            key[4 * j + 0] = ok ? (ky0 << 16) | kx0 : 0xFFFFFFFFu; val[4 * j + 0] = ok ? 1 : 0;
            key[4 * j + 1] = ok ? (ky0 << 16) | kx1 : 0xFFFFFFFFu; val[4 * j + 1] = ok ? -1 : 0;
            key[4 * j + 2] = ok ? (ky1 << 16) | kx0 : 0xFFFFFFFFu; val[4 * j + 2] = ok ? -1 : 0;
            key[4 * j + 3] = ok ? (ky1 << 16) | kx1 : 0xFFFFFFFFu; val[4 * j + 3] = ok ? 1 : 0;
        }
        __syncthreads();
        Sort(tmp.sort).Sort(key, val);   // blocked: thread t holds sorted items 16 t .. 16 t + 15
        __syncthreads();
        // heads: key differs from the previous item (previous thread's last key via SMEM)
        edge_first[threadIdx.x] = key[0];
        edge_last[threadIdx.x] = key[kClipItems - 1];
        __syncthreads();
        SegSum seg[kClipItems];
#pragma unroll
        for (int j = 0; j < kClipItems; ++j) {
            const uint32_t prev = j ? key[j - 1] : (threadIdx.x ? edge_last[threadIdx.x - 1] : 0xFFFFFFFEu);
            seg[j].head = key[j] != prev;
            seg[j].val = val[j];
        }
        SegScan(tmp.seg).InclusiveScan(seg, seg, SegSumOp());
        __syncthreads();
        // tails: key differs from the next item; keep a tail whose run sum is non-zero
        int keep[kClipItems], pos[kClipItems];
        long long a = 0;
#pragma unroll
        for (int j = 0; j < kClipItems; ++j) {
            const bool last = (j + 1 == kClipItems) && (threadIdx.x + 1 == kClipThreads);
            const uint32_t nxt = j + 1 < kClipItems ? key[j + 1] : (last ? 0u : edge_first[threadIdx.x + 1]);
            const bool tail = last || key[j] != nxt;
            keep[j] = (tail && key[j] != 0xFFFFFFFFu && seg[j].val != 0) ? 1 : 0;
            if (keep[j]) a += (long long)seg[j].val * (long long)(key[j] & 0xFFFFu) * (long long)(key[j] >> 16);
        }
        __syncthreads();   // edge_key reads above complete before it is reused next clip
        int total = 0;
        IntScan(tmp.scan).ExclusiveSum(keep, pos, total);
        __syncthreads();
        if (threadIdx.x < 32) {
            const int64_t pre = clip_lookback_warp(status, b, B, total, corner_ptr);
            if (threadIdx.x == 0) s_off = pre;
        }
        __syncthreads();
        const int64_t base = s_off;
#pragma unroll
        for (int j = 0; j < kClipItems; ++j) {
            if (keep[j] && base + pos[j] < cap) {
                xs[base + pos[j]] = (int32_t)(key[j] & 0xFFFFu);
                ys[base + pos[j]] = (int32_t)(key[j] >> 16);
                ws[base + pos[j]] = seg[j].val;
            }
        }
        const long long asum = Red(tmp.red).Sum(a);
        if (threadIdx.x == 0) area[b] = asum;
        __syncthreads();
    }
}

// Per-clip bucket path (every rect its own group, T <= kBucketMaxT, clips <= kClipRects rects):
// one CTA per clip counting-sorts the clip's 4n corners by y into T+1 SMEM buckets (atomics);
// then every corner finds its rank inside its (short) bucket by x, the first of equal (y, x)
// carries the summed weight (groups are summed, reading A5), a block scan over the sorted
// positions drops zero weights, and the clip is written in canonical (y, x) order straight to its
// CSR position (look-back offset, coalesced), with its exact int64 area.  O(n * bucket) with all
// threads busy, instead of a radix sort of 4n keys.
static constexpr int kBucketThreads = 512;
static constexpr int kBucketMaxT = 8191;
static constexpr int kBucketCap = 4 * kClipRects;
static constexpr int kSmallRects = 448 * 3;        // the small per-clip bucket variant (3 CTAs / SM)

// exclusive scan of the nb bucket sizes in hist (thread t owns buckets [t*per, (t+1)*per)); ends
// with a __syncthreads
template <int kNT>
__device__ __forceinline__ void bucket_scan(int32_t *hist, int nb, int32_t *wsum) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int per = (nb + kNT - 1) / kNT;
    const int lo = threadIdx.x * per, hi = min(lo + per, nb);
    int sown = 0;
    for (int i = lo; i < hi; ++i) sown += hist[i];
    int incl = sown;
    for (int o = 1; o < 32; o <<= 1) { int v = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += v; }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int run = incl - sown;
    for (int i = 0; i < wid; ++i) run += wsum[i];
    for (int i = lo; i < hi; ++i) { const int c = hist[i]; hist[i] = run; run += c; }
    __syncthreads();
}

// Second half of the per-clip bucket paths (shared by rects and polygons): the clip's nv corners sit
// in y buckets (bxw = x << 16 | w & 0xFFFF, by = y; hist[y] = end of bucket y).  Every corner finds
// its rank inside its (short) bucket by x, the first of equal (y, x) carries the summed weight
// (groups / polygons are summed), a block scan over the sorted positions drops zero weights, and the
// clip is written in canonical (y, x) order straight to its CSR position (look-back offset,
// coalesced), with its exact int64 area.  Ends with a __syncthreads.
template <bool kPaired, int kNT>
__device__ __forceinline__ void bucket_emit(int64_t b, int64_t B, int nb, uint32_t *bxw, uint32_t *syx, int16_t *by,
                                            int16_t *sw, int32_t *hist, int32_t *wsum, long long *asum,
                                            int *tot_s, int64_t *s_off, int32_t *xs, int32_t *ys, int32_t *ws,
                                            int64_t cap, int64_t *corner_ptr, unsigned long long *status,
                                            int64_t *area) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nv = hist[nb - 1];                    // valid corners (invalid rects skipped)
    if constexpr (kPaired) {
        // rects: every bucket holds whole edges, (x0, w) (x1, -w) at an even position, so a thread takes
        // one edge and ranks both of its corners in one pass over the bucket's edges (8-byte loads; four
        // compares per load instead of one)
        for (int t = threadIdx.x; 2 * t < nv; t += kNT) {
            const int i0 = 2 * t;
            const int y = by[i0];
            const int st = y ? hist[y - 1] : 0, en = hist[y];
            FCFS_DCHECK((st & 1) == 0 && (en & 1) == 0 && st <= i0 && i0 + 1 < en);
            const uint2 me = *(const uint2 *)(bxw + i0);
            const uint32_t xa = me.x >> 16, xb = me.y >> 16;
            int ra = 0, rb = 0, wa = 0, wb = 0;
            bool fa = true, fb = true;
            for (int j = st; j < en; j += 2) {
                const uint2 v = *(const uint2 *)(bxw + j);
                const uint32_t x0 = v.x >> 16, x1 = v.y >> 16;
                const int w0 = (int)(int16_t)(v.x & 0xFFFFu), w1 = (int)(int16_t)(v.y & 0xFFFFu);
                const bool a0 = x0 == xa, a1 = x1 == xa, b0 = x0 == xb, b1 = x1 == xb;
                // entry j is before i0 iff j < i0 (then j + 1 < i0 too); entry j + 1 is before i1 iff j < i0
                // or j == i0; i0 itself is before i1
                const bool pa = j < i0, pb = j <= i0;
                ra += (int)((x0 < xa) | (a0 & pa)) + (int)((x1 < xa) | (a1 & pa));
                rb += (int)((x0 < xb) | (b0 & pb)) + (int)((x1 < xb) | (b1 & pa));
                wa += (a0 ? w0 : 0) + (a1 ? w1 : 0);
                wb += (b0 ? w0 : 0) + (b1 ? w1 : 0);
                fa &= !(a0 & pa) & !(a1 & pa);
                fb &= !(b0 & pb) & !(b1 & pa);
            }
            syx[st + ra] = ((uint32_t)y << 16) | xa;
            sw[st + ra] = fa ? (int16_t)wa : (int16_t)0;
            syx[st + rb] = ((uint32_t)y << 16) | xb;
            sw[st + rb] = fb ? (int16_t)wb : (int16_t)0;
        }
    } else
    // rank inside the bucket by x (ties by index); the first of equal x carries the run sum
    for (int i = threadIdx.x; i < nv; i += kNT) {
        const int y = by[i];
        const int st = y ? hist[y - 1] : 0, en = hist[y];
        const uint32_t xi = bxw[i] >> 16;
        int rank = 0, wv = 0;
        bool first = true;
#pragma unroll 2
        for (int j = st; j < en; ++j) {
            const uint32_t v = bxw[j];
            const uint32_t xj = v >> 16;
            const bool eq = xj == xi, before = j < i;
            rank += (xj < xi) | (eq & before);
            wv += eq ? (int)(int16_t)(v & 0xFFFFu) : 0;
            first &= !(eq & before);
        }
        syx[st + rank] = ((uint32_t)y << 16) | xi;
        sw[st + rank] = first ? (int16_t)wv : (int16_t)0;
    }
    __syncthreads();
    // compact the non-zero sorted entries: thread t owns sorted positions [t*pp, (t+1)*pp)
    const int pp = (nv + kNT - 1) / kNT;
    const int lo = threadIdx.x * pp, hi = min(lo + pp, nv);
    int cnt = 0;
    long long a = 0;
    for (int i = lo; i < hi; ++i) {
        const int16_t wv = sw[i];
        if (wv != 0) {
            ++cnt;
            a += (long long)wv * (long long)(syx[i] & 0xFFFFu) * (long long)(syx[i] >> 16);
        }
    }
    int incl = cnt;
    for (int o = 1; o < 32; o <<= 1) { int v = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += v; }
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    __syncthreads();                                // wsum reuse; bxw / by are free from here
    if (lane == 31) wsum[wid] = incl;
    if (lane == 0) asum[wid] = a;
    __syncthreads();
    int outp = incl - cnt;
    for (int i = 0; i < wid; ++i) outp += wsum[i];
    int total = 0;
    if (wid == 0) {   // the clip's count is known: publish it before the compaction (successors' walks)
        for (int i = 0; i < (kNT >> 5); ++i) total += wsum[i];
        if (lane == 0) clip_publish_count(status, b, total);
    }
    for (int i = lo; i < hi; ++i) {
        const int16_t wv = sw[i];
        if (wv != 0) { bxw[outp] = syx[i]; by[outp] = wv; ++outp; }
    }
    if (wid == 0) {   // the look-back walk of warp 0 overlaps the other warps' compaction
        const int64_t pre = clip_lookback_warp(status, b, B, total, corner_ptr, true);
        if (lane == 0) { *s_off = pre; *tot_s = total; }
    }
    __syncthreads();
    total = *tot_s;
    const int64_t base = *s_off;
    for (int i = threadIdx.x; i < total; i += kNT) {   // coalesced stores, final positions
        if (base + i >= cap) break;
        const uint32_t yx = bxw[i];
        xs[base + i] = (int32_t)(yx & 0xFFFFu);
        ys[base + i] = (int32_t)(yx >> 16);
        ws[base + i] = by[i];
    }
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int i = 0; i < (kNT >> 5); ++i) t += asum[i];
        area[b] = t;
    }
    __syncthreads();
}


// kThr threads x kRPT rects per thread per clip (corner capacity 4 kThr kRPT, 12 B per corner of
// shared memory): <448, 3> (1344 rects, 72 KB: 3 CTAs / SM) runs first, <512, 4> (2048 rects) if a
// clip is larger
template <int kThr, int kRPT>
__global__ void __launch_bounds__(kThr, 3)
k_clip_corners_bucket(const int4 *__restrict__ rects, const int64_t *__restrict__ clip_ptr, int64_t B, int64_t R,
                      int32_t T, int32_t *xs, int32_t *ys, int32_t *ws, int64_t cap, int64_t *corner_ptr,
                      unsigned long long *status, int64_t *area, int32_t *err) {
    constexpr int kCap = 4 * kThr * kRPT;
    extern __shared__ __align__(16) unsigned char bsm[];
    uint32_t *bxw = (uint32_t *)bsm;                    // [cap] bucketed (x << 16 | w & 0xFFFF); later compacted (y << 16 | x)
    uint32_t *syx = bxw + kCap;                         // [cap] sorted (y << 16 | x)
    int16_t *by = (int16_t *)(syx + kCap);              // [cap] bucket y; later compacted weights
    int16_t *sw = by + kCap;                            // [cap] sorted merged weight (0 = dropped)
    int32_t *hist = (int32_t *)(sw + kCap);             // [T + 2]: bucket start, then bucket end
    __shared__ int32_t wsum[kThr / 32];
    __shared__ long long asum[kThr / 32];
    __shared__ int tot_s;
    __shared__ int64_t s_off;
    const int nb = T + 1;                               // buckets y = 0..T
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
        const int64_t r0 = clip_ptr ? clip_ptr[b] : 0, r1 = clip_ptr ? clip_ptr[b + 1] : R;
        const int n = (int)(r1 - r0);
        if (n > kThr * kRPT) {
            // the caller falls back to the general path; the clip still publishes a count (0) so
            // that the look-back of the clips after it completes
            if (threadIdx.x == 0) { atomicOr(err, 8); area[b] = 0; clip_lookback(status, b, B, 0, corner_ptr); }
            continue;
        }
        // all of this thread's rects are loaded up front (independent loads in flight)
        int4 rq[kRPT];
        bool rok[kRPT];
#pragma unroll
        for (int j = 0; j < kRPT; ++j) {
            const int r = threadIdx.x + j * kThr;
            rok[j] = r < n;
            rq[j] = rok[j] ? rects[r0 + r] : make_int4(0, 0, 0, 0);
        }
        for (int i = threadIdx.x; i < nb + 1; i += kThr) hist[i] = 0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kRPT; ++j) {
            if (!rok[j]) continue;
            if (!rect_ok(rq[j], T)) { atomicOr(err, 1); rok[j] = false; continue; }
            atomicAdd(&hist[rq[j].y], 2);
            atomicAdd(&hist[rq[j].w], 2);
        }
        __syncthreads();
        bucket_scan<kThr>(hist, nb, wsum);
        // scatter into buckets: afterwards hist[y] = end of bucket y (= start of bucket y + 1)
#pragma unroll
        for (int j = 0; j < kRPT; ++j) {
            if (!rok[j]) continue;
            const int4 q = rq[j];
            int p = atomicAdd(&hist[q.y], 2);
            FCFS_DCHECK(p >= 0 && p + 1 < kCap);
            bxw[p] = ((uint32_t)q.x << 16) | 0x0001u;       by[p] = (int16_t)q.y;
            bxw[p + 1] = ((uint32_t)q.z << 16) | 0xFFFFu;   by[p + 1] = (int16_t)q.y;
            p = atomicAdd(&hist[q.w], 2);
            FCFS_DCHECK(p >= 0 && p + 1 < kCap);
            bxw[p] = ((uint32_t)q.x << 16) | 0xFFFFu;       by[p] = (int16_t)q.w;
            bxw[p + 1] = ((uint32_t)q.z << 16) | 0x0001u;   by[p + 1] = (int16_t)q.w;
        }
        __syncthreads();
        bucket_emit<true, kThr>(b, B, nb, bxw, syx, by, sw, hist, wsum, asum, &tot_s, &s_off, xs, ys, ws, cap, corner_ptr,
                    status, area);
    }
}

static constexpr int kSmallPoly = 32;                          // thread per polygon up to this size
static constexpr int kMaxLarge = kBucketCap / kSmallPoly + 1;  // longer polygons of one clip (warp each)

// Per-clip bucket path for polygon vertex lists (T <= kBucketMaxT, <= kBucketCap vertices per clip):
// a thread (a warp for polygons of > kSmallPoly vertices) per polygon computes the orientation (sign of the vertex-form area, reading A16), checks the
// edges and writes every vertex's raw weight s ([edge i-1 horizontal] - [edge i horizontal]) (Alg. 2
// lines 9-10) into shared memory; the non-zero ones are counting-sorted into y buckets,
// then bucket_emit as for rects.
__global__ void __launch_bounds__(kBucketThreads, 2)
k_clip_polygons_bucket(const int32_t *__restrict__ vx, const int32_t *__restrict__ vy,
                       const int64_t *__restrict__ poly_ptr, int64_t P, const int64_t *__restrict__ clip_ptr,
                       int64_t B, int32_t T, int32_t *xs, int32_t *ys, int32_t *ws, int64_t cap, int64_t *corner_ptr,
                       unsigned long long *status, int64_t *area, int32_t *err) {
    extern __shared__ __align__(16) unsigned char bsm[];
    uint32_t *bxw = (uint32_t *)bsm;                    // [cap] bucketed (x << 16 | w & 0xFFFF)
    uint32_t *syx = bxw + kBucketCap;                   // [cap] raw (y << 16 | x), then sorted
    int16_t *by = (int16_t *)(syx + kBucketCap);        // [cap] bucket y
    int16_t *sw = by + kBucketCap;                      // [cap] raw weight, then sorted merged weight
    int32_t *hist = (int32_t *)(sw + kBucketCap);       // [T + 2]
    __shared__ int32_t wsum[kBucketThreads / 32];
    __shared__ long long asum[kBucketThreads / 32];
    __shared__ int tot_s;
    __shared__ int64_t s_off;
    __shared__ int n_large;
    __shared__ int32_t large[kMaxLarge];
    const int nb = T + 1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
        const int64_t p0 = clip_ptr ? clip_ptr[b] : 0, p1 = clip_ptr ? clip_ptr[b + 1] : P;
        const int64_t vbase = poly_ptr[p0];
        const int64_t nvr = poly_ptr[p1] - vbase;       // raw corners = vertices of the clip
        if (nvr > kBucketCap) {
            if (threadIdx.x == 0) { atomicOr(err, 8); area[b] = 0; clip_lookback(status, b, B, 0, corner_ptr); }
            continue;
        }
        for (int i = threadIdx.x; i < nb + 1; i += kBucketThreads) hist[i] = 0;
        if (threadIdx.x == 0) n_large = 0;
        __syncthreads();
        // raw corners: thread per polygon of <= kSmallPoly vertices (two passes over its vertices:
        // orientation + edge checks, then weights); longer polygons are queued for warps
        for (int64_t p = p0 + threadIdx.x; p < p1; p += kBucketThreads) {
            const int64_t v0 = poly_ptr[p];
            const int n = (int)(poly_ptr[p + 1] - v0);
            if (n > kSmallPoly) {
                const int q = atomicAdd(&n_large, 1);
                if (q < kMaxLarge) large[q] = (int32_t)(p - p0);
                continue;
            }
            if (n == 0) continue;
            long long A = 0;
            bool bad = false, range = false;
            int32_t xf = vx[v0], yf = vy[v0], xi = xf, yi = yf;
            for (int i = 0; i < n; ++i) {
                const int32_t xj = i + 1 < n ? vx[v0 + i + 1] : xf, yj = i + 1 < n ? vy[v0 + i + 1] : yf;
                range |= xi < 0 || yi < 0 || xi > T || yi > T;
                const bool hor = yi == yj && xi != xj, ver = xi == xj && yi != yj;
                bad |= !(hor || ver);
                if (hor) A += (long long)yi * (long long)(xj - xi);
                xi = xj; yi = yj;
            }
            if (bad || range) atomicOr(err, (bad ? 16 : 0) | (range ? 1 : 0));
            const int sg = A < 0 ? -1 : 1;
            const bool ok = !(bad || range);
            int32_t xh = vx[v0 + n - 1], yh = vy[v0 + n - 1];
            xi = xf; yi = yf;
            for (int i = 0; i < n; ++i) {
                const int32_t xj = i + 1 < n ? vx[v0 + i + 1] : xf, yj = i + 1 < n ? vy[v0 + i + 1] : yf;
                const bool hin = yh == yi && xh != xi, hout = yj == yi && xj != xi;
                const int64_t o = v0 + i - vbase;
                syx[o] = ok ? ((uint32_t)yi << 16) | (uint32_t)xi : 0u;
                sw[o] = ok ? (int16_t)(sg * ((int)hin - (int)hout)) : (int16_t)0;
                xh = xi; yh = yi; xi = xj; yi = yj;
            }
        }
        __syncthreads();
        if (n_large > kMaxLarge) {   // cannot happen (kMaxLarge * kSmallPoly >= kBucketCap); guard anyway
            if (threadIdx.x == 0) atomicOr(err, 8);
        }
        // long polygons: warp per polygon
        for (int q = wid; q < min(n_large, kMaxLarge); q += kBucketThreads / 32) {
            const int64_t p = p0 + large[q];
            const int64_t v0 = poly_ptr[p];
            const int n = (int)(poly_ptr[p + 1] - v0);
            long long A = 0;
            bool bad = false, range = false;
            for (int i = lane; i < n; i += 32) {
                const int j = i + 1 == n ? 0 : i + 1;
                const int32_t xi = vx[v0 + i], yi = vy[v0 + i], xj = vx[v0 + j], yj = vy[v0 + j];
                range |= xi < 0 || yi < 0 || xi > T || yi > T;
                const bool hor = yi == yj && xi != xj, ver = xi == xj && yi != yj;
                bad |= !(hor || ver);
                if (hor) A += (long long)yi * (long long)(xj - xi);
            }
            for (int o = 16; o > 0; o >>= 1) A += __shfl_xor_sync(0xffffffffu, A, o);
            bad = __any_sync(0xffffffffu, bad);
            range = __any_sync(0xffffffffu, range);
            if (lane == 0 && (bad || range)) atomicOr(err, (bad ? 16 : 0) | (range ? 1 : 0));
            const int sg = A < 0 ? -1 : 1;
            const bool ok = !(bad || range);
            for (int i = lane; i < n; i += 32) {
                const int h = i == 0 ? n - 1 : i - 1, j = i + 1 == n ? 0 : i + 1;
                const int32_t xi = vx[v0 + i], yi = vy[v0 + i];
                const bool hin = vy[v0 + h] == yi && vx[v0 + h] != xi;
                const bool hout = vy[v0 + j] == yi && vx[v0 + j] != xi;
                const int64_t o = v0 + i - vbase;
                syx[o] = ok ? ((uint32_t)yi << 16) | (uint32_t)xi : 0u;
                sw[o] = ok ? (int16_t)(sg * ((int)hin - (int)hout)) : (int16_t)0;
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nvr; i += kBucketThreads)
            if (sw[i] != 0) atomicAdd(&hist[syx[i] >> 16], 1);
        __syncthreads();
        bucket_scan<kBucketThreads>(hist, nb, wsum);
        for (int i = threadIdx.x; i < nvr; i += kBucketThreads) {
            const int16_t wv = sw[i];
            if (wv == 0) continue;
            const uint32_t yx = syx[i];
            const int p = atomicAdd(&hist[yx >> 16], 1);
            bxw[p] = ((yx & 0xFFFFu) << 16) | ((uint32_t)(int32_t)wv & 0xFFFFu);
            by[p] = (int16_t)(yx >> 16);
        }
        __syncthreads();
        bucket_emit<false, kBucketThreads>(b, B, nb, bxw, syx, by, sw, hist, wsum, asum, &tot_s, &s_off, xs, ys, ws, cap, corner_ptr,
                    status, area);
    }
}

struct ClipWs {
    unsigned long long *status;   // [B] look-back words (flag << 62 | count)
    int32_t *err;
};

static void carve_clip(Carver &cv, int64_t R, int64_t B, ClipWs &w) {
    (void)R;
    w.status = cv.take<unsigned long long>(B);
    w.err = cv.take<int32_t>(4);
}

size_t extract_clip_workspace_bytes(int64_t R, int64_t B) {
    Carver cv(nullptr, 0);
    ClipWs w;
    carve_clip(cv, R, B, w);
    return cv.used();
}

// outcome of the sync-free per-clip path: K = corner_ptr[B]; the err bits of the per-clip kernels
// (1 a bad rect, 8 a clip above the launched variant's capacity) become an fcfs_status word
__global__ void k_clips_status(const int64_t *corner_ptr, int64_t B, const int32_t *err, int64_t cap, int64_t *K_dev,
                               int32_t *status) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int64_t k = corner_ptr[B];
    const int32_t e = *err;
    *K_dev = k;
    *status = (e & 8) ? FCFS_E_UNSUPPORTED : (e & 1) ? FCFS_E_RANGE : (k > cap ? FCFS_E_CAPACITY : FCFS_OK);
}

static fcfs_status clips_result(int64_t Kh, int32_t errh, int64_t cap, int64_t *K_host) {
    if (errh & 8) {
        set_error("a clip has more than %d rects", kClipRects);
        return FCFS_E_UNSUPPORTED;
    }
    if (K_host) *K_host = Kh;
    if (errh & 1) {
        set_error("fcfs_vertices_from_rects: a rect lies outside [0,T]^2 or is empty");
        return FCFS_E_RANGE;
    }
    if (Kh > cap) {
        set_error("fcfs_vertices_from_rects: K=%lld > cap=%lld", (long long)Kh, (long long)cap);
        return FCFS_E_CAPACITY;
    }
    return FCFS_OK;
}

// returns FCFS_E_UNSUPPORTED (after a sync) if a clip exceeds kClipRects: the caller falls back
// The per-clip bucket path with no host synchronisation (batched clips of singleton groups): the caller
// bounds the rects per clip (max_clip_rects <= kClipRects), which picks the variant up front instead of
// a read-back of the overflow bit; K and the outcome stay on the device (K_dev, status_dev).
fcfs_status extract_clips_async(const int32_t *rects, int64_t R, const int64_t *clip_ptr, int64_t B, int32_t T,
                                int64_t max_clip_rects, int32_t *x, int32_t *y, int32_t *w, int64_t cap,
                                int64_t *corner_ptr, int64_t *area, int64_t *K_dev, int32_t *status_dev, void *ws,
                                size_t ws_bytes, cudaStream_t s) {
    if (max_clip_rects < 0 || max_clip_rects > kClipRects || T > 65534) {
        set_error("fcfs_vertices_from_clips_async: max_clip_rects=%lld (<= %d) or T=%d (<= 65534) unsupported",
                  (long long)max_clip_rects, kClipRects, T);
        return FCFS_E_UNSUPPORTED;
    }
    Carver cv(ws, ws_bytes);
    ClipWs W;
    carve_clip(cv, R, B, W);
    if (!cv.fits()) {
        set_error("fcfs_vertices_from_clips_async: workspace %zu < %zu bytes", ws_bytes, cv.used());
        return FCFS_E_WORKSPACE;
    }
    FCFS_TRY_CUDA(cudaMemsetAsync(W.err, 0, 4 * sizeof(int32_t), s));
    FCFS_TRY_CUDA(cudaMemsetAsync(W.status, 0, B * sizeof(unsigned long long), s));
    const int64_t grid = B;
    if (T <= kBucketMaxT) {
        if (max_clip_rects <= kSmallRects) {
            FCFS_TRY(ensure_smem((const void *)k_clip_corners_bucket<448, 3>,
                                 4 * kSmallRects * 12 + (kBucketMaxT + 2) * 4, true));
            const size_t bsmem = 4 * kSmallRects * 12 + (size_t)(T + 2) * 4;
            k_clip_corners_bucket<448, 3><<<(unsigned)grid, 448, bsmem, s>>>((const int4 *)rects, clip_ptr, B, R, T, x,
                                                                            y, w, cap, corner_ptr, W.status, area,
                                                                            W.err);
        } else {
            FCFS_TRY(ensure_smem((const void *)k_clip_corners_bucket<512, 4>, kBucketCap * 12 + (kBucketMaxT + 2) * 4,
                                 true));
            const size_t bsmem = kBucketCap * 12 + (size_t)(T + 2) * 4;
            k_clip_corners_bucket<512, 4><<<(unsigned)grid, 512, bsmem, s>>>((const int4 *)rects, clip_ptr, B, R, T, x,
                                                                            y, w, cap, corner_ptr, W.status, area,
                                                                            W.err);
        }
        FCFS_CHECK_LAUNCH("k_clip_corners_bucket");
    } else {
        k_clip_corners<<<(unsigned)grid, kClipThreads, 0, s>>>((const int4 *)rects, clip_ptr, B, R, T, x, y, w, cap,
                                                               corner_ptr, W.status, area, W.err);
        FCFS_CHECK_LAUNCH("k_clip_corners");
    }
    k_clips_status<<<1, 32, 0, s>>>(corner_ptr, B, W.err, cap, K_dev, status_dev);
    FCFS_CHECK_LAUNCH("k_clips_status");
    return FCFS_OK;
}

fcfs_status extract_clips(const int32_t *rects, int64_t R, const int64_t *clip_ptr, int64_t B, int32_t T,
                          int32_t *x, int32_t *y, int32_t *w, int64_t cap, int64_t *corner_ptr, int64_t *area,
                          int64_t *K_host, void *ws, size_t ws_bytes, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    ClipWs W;
    carve_clip(cv, R, B, W);
    if (!cv.fits()) {
        set_error("fcfs_vertices_from_rects: workspace %zu < %zu bytes", ws_bytes, cv.used());
        return FCFS_E_WORKSPACE;
    }
    FCFS_TRY_CUDA(cudaMemsetAsync(W.err, 0, 4 * sizeof(int32_t), s));
    FCFS_TRY_CUDA(cudaMemsetAsync(W.status, 0, B * sizeof(unsigned long long), s));
    // one CTA per clip (the look-back needs every predecessor clip's CTA dispatched before it)
    const int64_t grid = B;
    if (T <= kBucketMaxT) {
        // the 1344-rect variant (3 CTAs / SM) unless the average clip is larger; if a clip overflows it,
        // the 2048-rect variant reruns the batch (same outputs), and beyond that the general path
        const bool small = R <= (int64_t)kSmallRects * B;
        FCFS_TRY(ensure_smem((const void *)k_clip_corners_bucket<512, 4>, kBucketCap * 12 + (kBucketMaxT + 2) * 4,
                             true));
        FCFS_TRY(ensure_smem((const void *)k_clip_corners_bucket<448, 3>,
                             4 * kSmallRects * 12 + (kBucketMaxT + 2) * 4, true));
        auto launch = [&](bool large) -> fcfs_status {
            if (large) {
                const size_t bsmem = kBucketCap * 12 + (size_t)(T + 2) * 4;
                k_clip_corners_bucket<512, 4><<<(unsigned)grid, 512, bsmem, s>>>((const int4 *)rects, clip_ptr, B, R,
                                                                                T, x, y, w, cap, corner_ptr, W.status,
                                                                                area, W.err);
            } else {
                const size_t bsmem = 4 * kSmallRects * 12 + (size_t)(T + 2) * 4;
                k_clip_corners_bucket<448, 3><<<(unsigned)grid, 448, bsmem, s>>>((const int4 *)rects, clip_ptr, B, R,
                                                                                T, x, y, w, cap, corner_ptr, W.status,
                                                                                area, W.err);
            }
            FCFS_CHECK_LAUNCH("k_clip_corners_bucket");
            return FCFS_OK;
        };
        fcfs_status st = launch(!small);
        if (st != FCFS_OK) return st;
        if (small) {
            // the result read-back below syncs once; only if the small variant overflowed (err bit 8)
            // does the batch rerun with the large one
            int64_t Kh = 0;
            int32_t errh = 0;
            FCFS_TRY_CUDA(cudaMemcpyAsync(&Kh, corner_ptr + B, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            FCFS_TRY_CUDA(cudaMemcpyAsync(&errh, W.err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            FCFS_TRY_CUDA(cudaStreamSynchronize(s));
            if (!(errh & 8)) return clips_result(Kh, errh, cap, K_host);
            FCFS_TRY_CUDA(cudaMemsetAsync(W.err, 0, 4 * sizeof(int32_t), s));
            FCFS_TRY_CUDA(cudaMemsetAsync(W.status, 0, B * sizeof(unsigned long long), s));
            st = launch(true);
            if (st != FCFS_OK) return st;
        }
    } else {
        k_clip_corners<<<(unsigned)grid, kClipThreads, 0, s>>>((const int4 *)rects, clip_ptr, B, R, T, x, y, w, cap,
                                                               corner_ptr, W.status, area, W.err);
        FCFS_CHECK_LAUNCH("k_clip_corners");
    }
    int64_t Kh = 0;
    int32_t errh = 0;
    FCFS_TRY_CUDA(cudaMemcpyAsync(&Kh, corner_ptr + B, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    FCFS_TRY_CUDA(cudaMemcpyAsync(&errh, W.err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    FCFS_TRY_CUDA(cudaStreamSynchronize(s));
    return clips_result(Kh, errh, cap, K_host);
}

// steps 2-5 of the general path on the raw (key, weight) list in W.keys_a / W.w_a: sort, merge
// equal keys (sum), drop zeros, scatter + area, corner_ptr; one stream sync for K and the error bits
// the sync-free path's ending: K and the error bits become a device status word (fcfs_status codes)
__global__ void k_extract_status(const int64_t *K, const int32_t *err, int64_t cap, int64_t *K_dev, int32_t *status) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int64_t k = *K;
    const int32_t e = *err;
    *K_dev = k;
    *status = (e & 1) ? FCFS_E_RANGE : (e & 2) ? FCFS_E_UNSUPPORTED : (e & 4) ? FCFS_E_WORKSPACE
                                                                  : (k > cap ? FCFS_E_CAPACITY : FCFS_OK);
}

static fcfs_status finish_corners(ExtractWs &W, int64_t cap_raw, int cb, int end_bit, int64_t B, int64_t cap, int32_t *x,
                                  int32_t *y, int32_t *w, int64_t *corner_ptr, int64_t *area, int64_t &Kh,
                                  int32_t &errh, cudaStream_t s, int64_t *K_dev = nullptr, int32_t *status_dev = nullptr) {
    const int threads = 256;
    size_t tb = W.cub_bytes;
    FCFS_TRY_CUDA(cub::DeviceRadixSort::SortPairs(W.cub_tmp, tb, W.keys_a, W.keys_b, W.w_a, W.w_b, (int)cap_raw,
                                                  0, end_bit, s));
    count_launch(4);
    tb = W.cub_bytes;
    FCFS_TRY_CUDA(cub::DeviceReduce::ReduceByKey(W.cub_tmp, tb, W.keys_b, W.keys_a, W.w_b, W.w_a, W.num_runs,
                                                 cub::Sum(), (int)cap_raw, s));
    count_launch(2);
    int64_t blocks = (cap_raw + threads - 1) / threads;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_flags<<<(unsigned)blocks, threads, 0, s>>>(W.w_a, W.num_runs, cap_raw, W.flags);
    FCFS_CHECK_LAUNCH("k_flags");
    tb = W.cub_bytes;
    FCFS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(W.cub_tmp, tb, W.flags, W.pos, (int)cap_raw, s));
    count_launch(2);
    k_scatter<<<(unsigned)blocks, threads, 0, s>>>(W.keys_a, W.w_a, W.flags, W.pos, cap_raw, cap, x, y, w,
                                                   W.keys_b, area, W.K, cb);
    FCFS_CHECK_LAUNCH("k_scatter");
    int64_t pb = (B + 1 + threads - 1) / threads;
    k_corner_ptr<<<(unsigned)(pb < 1024 ? pb : 1024), threads, 0, s>>>(W.keys_b, W.K, B, corner_ptr, cb);
    FCFS_CHECK_LAUNCH("k_corner_ptr");
    if (K_dev) {   // sync-free: K and the status stay on the device
        k_extract_status<<<1, 32, 0, s>>>(W.K, W.err, cap, K_dev, status_dev);
        FCFS_CHECK_LAUNCH("k_extract_status");
        return FCFS_OK;
    }
    FCFS_TRY_CUDA(cudaMemcpyAsync(&Kh, W.K, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    FCFS_TRY_CUDA(cudaMemcpyAsync(&errh, W.err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    FCFS_TRY_CUDA(cudaStreamSynchronize(s));
    return FCFS_OK;
}

static int64_t raw_capacity(int64_t R, int64_t max_group, bool singleton) {
    if (singleton) return 4 * R;
    int64_t g = max_group < 1 ? 1 : max_group;
    return 4 * R * g;   // a union of g rects has at most (2g)^2 grid points: sum_g 4 g^2 <= 4 R gmax
}

static size_t cub_bytes_for(int64_t n, int end_bit) {
    size_t a = 0, b = 0, c = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                    (int32_t *)nullptr, (int32_t *)nullptr, (int)n, 0, end_bit);
    cub::DeviceReduce::ReduceByKey(nullptr, b, (unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                   (int32_t *)nullptr, (int32_t *)nullptr, (int64_t *)nullptr,
                                   cub::Sum(), (int)n);
    cub::DeviceScan::ExclusiveSum(nullptr, c, (int32_t *)nullptr, (int32_t *)nullptr, (int)n);
    size_t m = a > b ? a : b;
    return m > c ? m : c;
}

static int clip_bits(int64_t B) {
    int bits = 1;
    while ((int64_t(1) << bits) <= B) ++bits;
    return bits;
}

static void carve(Carver &cv, int64_t cap_raw, size_t cub_bytes, ExtractWs &w) {
    w.cap_raw = cap_raw;
    w.keys_a = cv.take<unsigned long long>(cap_raw);
    w.keys_b = cv.take<unsigned long long>(cap_raw);
    w.w_a = cv.take<int32_t>(cap_raw);
    w.w_b = cv.take<int32_t>(cap_raw);
    w.flags = cv.take<int32_t>(cap_raw);
    w.pos = cv.take<int32_t>(cap_raw);
    w.num_runs = cv.take<int64_t>(1);
    w.K = cv.take<int64_t>(1);
    w.err = cv.take<int32_t>(4);
    w.cub_tmp = cv.take<char>(cub_bytes);
    w.cub_bytes = cub_bytes;
}

size_t extract_workspace_bytes(int64_t R, int64_t G, int64_t B, int64_t max_group, bool singleton) {
    int64_t cap = raw_capacity(R, max_group, singleton);
    if (cap < 1) cap = 1;
    Carver cv(nullptr, 0);
    ExtractWs w;
    carve(cv, cap, cub_bytes_for(cap, 2 * kCoordBits + clip_bits(B)), w);
    size_t a = cv.used();
    size_t b = singleton ? extract_clip_workspace_bytes(R, B) : 0;
    return a > b ? a : b;
}

fcfs_status extract(const int32_t *rects, int64_t R, const int64_t *group_ptr, int64_t G,
                    const int64_t *clip_ptr, int64_t B, int32_t T, int64_t max_group, int32_t *x,
                    int32_t *y, int32_t *w, int64_t cap, int64_t *corner_ptr, int64_t *area,
                    int64_t *K_host, void *ws, size_t ws_bytes, cudaStream_t s, int32_t y_lo, int32_t y_hi,
                    int64_t *K_dev, int32_t *status_dev) {
    const bool singleton = (group_ptr == nullptr);
    const bool band = y_lo > 0 || y_hi <= T;
    const bool async = K_dev != nullptr;   // sync-free: the general path, K and the status on the device
    if (async && band) {
        set_error("fcfs_vertices_from_rects: a band extraction is not available sync-free");
        return FCFS_E_INVALID;
    }
    if (!async && !band && singleton && T <= 65534 && (clip_ptr != nullptr || R <= kClipRects)) {
        fcfs_status st = extract_clips(rects, R, clip_ptr, B, T, x, y, w, cap, corner_ptr, area, K_host, ws,
                                       ws_bytes, s);
        if (st != FCFS_E_UNSUPPORTED) return st;   // else: a clip is too large for the per-clip path
    }
    if (!singleton && max_group > kMaxGroup) {
        set_error("fcfs_vertices_from_rects: max_group=%lld exceeds this build's limit %d",
                  (long long)max_group, kMaxGroup);
        return FCFS_E_UNSUPPORTED;
    }
    int64_t cap_raw = raw_capacity(R, max_group, singleton);
    if (cap_raw < 1) cap_raw = 1;
    if (cap_raw >= (int64_t(1) << 31)) {
        set_error("fcfs_vertices_from_rects: %lld raw corners exceed 2^31", (long long)cap_raw);
        return FCFS_E_UNSUPPORTED;
    }
    int cb = coord_bits(T), end_bit = 2 * cb + clip_bits(B);
    const size_t cub_max = cub_bytes_for(cap_raw, 2 * kCoordBits + clip_bits(B));   // as the size query
    if (cub_bytes_for(cap_raw, end_bit) > cub_max) { cb = kCoordBits; end_bit = 2 * cb + clip_bits(B); }
    Carver cv(ws, ws_bytes);
    ExtractWs W;
    carve(cv, cap_raw, cub_max, W);
    if (!cv.fits()) {
        set_error("fcfs_vertices_from_rects: workspace %zu < %zu bytes", ws_bytes, cv.used());
        return FCFS_E_WORKSPACE;
    }
    FCFS_TRY_CUDA(cudaMemsetAsync(W.err, 0, 4 * sizeof(int32_t), s));
    FCFS_TRY_CUDA(cudaMemsetAsync(W.num_runs, 0, 2 * sizeof(int64_t), s));
    FCFS_TRY_CUDA(cudaMemsetAsync(area, 0, B * sizeof(int64_t), s));
    unsigned long long *raw_count = (unsigned long long *)W.num_runs;   // reused before reduce
    const int threads = 256;
    if (singleton) {
        if (R > 0) {
            int64_t blocks = (R + threads - 1) / threads;
            if (blocks > 148 * 32) blocks = 148 * 32;
            k_singleton_corners<<<(unsigned)blocks, threads, 0, s>>>((const int4 *)rects, R, clip_ptr, B, T,
                                                                      W.keys_a, W.w_a, W.err);
            FCFS_CHECK_LAUNCH("k_singleton_corners");
        }
        if (cap_raw > 4 * R) {
            k_fill_sentinel<<<1, 32, 0, s>>>(W.keys_a + 4 * R, W.w_a + 4 * R, cap_raw - 4 * R, nullptr);
            FCFS_CHECK_LAUNCH("k_fill_sentinel");
        }
    } else {
        int mg = (int)(max_group < 1 ? 1 : max_group);
        size_t smem = sizeof(int4) * kMaxGroup + sizeof(int32_t) * (10 * kMaxGroup + 2) +
                      sizeof(int32_t) * (size_t)(2 * mg) * (2 * mg) + 16;
        FCFS_TRY(ensure_smem((const void *)k_group_corners, 210 * 1024));
        if (G > 0) {
            int64_t blocks = G < 148 * 8 ? G : 148 * 8;
            const int gthreads = mg <= 8 ? 128 : (mg <= 32 ? 256 : 512);   // (2 mg)^2 grid cells per group
            k_group_corners<<<(unsigned)blocks, gthreads, smem, s>>>((const int4 *)rects, group_ptr, G, clip_ptr, B, T,
                                                                 W.keys_a, W.w_a, cap_raw, raw_count, W.err);
            FCFS_CHECK_LAUNCH("k_group_corners");
        }
        k_fill_sentinel<<<148 * 4, 256, 0, s>>>(W.keys_a, W.w_a, cap_raw, raw_count);
        FCFS_CHECK_LAUNCH("k_fill_sentinel");
    }
    if (band) {
        // compact the band's raw corners into keys_b / w_b, then sort only those (one extra host read of
        // the count: the sort sizes are host-side)
        unsigned long long *cnt = (unsigned long long *)W.K;
        FCFS_TRY_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
        int64_t blocks = (cap_raw + threads - 1) / threads;
        if (blocks > 148 * 16) blocks = 148 * 16;
        k_band_compact<<<(unsigned)blocks, threads, 0, s>>>(W.keys_a, W.w_a, cap_raw, cb, y_lo, y_hi, W.keys_b,
                                                            W.w_b, cnt);
        FCFS_CHECK_LAUNCH("k_band_compact");
        unsigned long long nb = 0;
        FCFS_TRY_CUDA(cudaMemcpyAsync(&nb, cnt, sizeof(nb), cudaMemcpyDeviceToHost, s));
        FCFS_TRY_CUDA(cudaStreamSynchronize(s));
        if (nb == 0) {   // an empty band: one sentinel so the tail runs on a non-empty list
            k_fill_sentinel<<<1, 32, 0, s>>>(W.keys_b, W.w_b, 1, nullptr);
            FCFS_CHECK_LAUNCH("k_fill_sentinel");
            nb = 1;
        }
        std::swap(W.keys_a, W.keys_b);
        std::swap(W.w_a, W.w_b);
        cap_raw = (int64_t)nb;
        FCFS_TRY_CUDA(cudaMemsetAsync(W.num_runs, 0, 2 * sizeof(int64_t), s));
    }
    int64_t Kh = 0;
    int32_t errh = 0;
    fcfs_status st = finish_corners(W, cap_raw, cb, end_bit, B, cap, x, y, w, corner_ptr, area, Kh, errh, s, K_dev,
                                    status_dev);
    if (st != FCFS_OK || async) return st;
    if (K_host) *K_host = Kh;
    if (errh & 1) {
        set_error("fcfs_vertices_from_rects: a rect lies outside [0,T]^2 or is empty");
        return FCFS_E_RANGE;
    }
    if (errh & 2) {
        set_error("fcfs_vertices_from_rects: a group has more than %d rects", kMaxGroup);
        return FCFS_E_UNSUPPORTED;
    }
    if (errh & 4) {
        set_error("fcfs_vertices_from_rects: raw corner capacity exceeded (max_group too small?)");
        return FCFS_E_WORKSPACE;
    }
    if (Kh > cap) {
        set_error("fcfs_vertices_from_rects: K=%lld > cap=%lld", (long long)Kh, (long long)cap);
        return FCFS_E_CAPACITY;
    }
    return FCFS_OK;
}

size_t extract_polygons_workspace_bytes(int64_t V, int64_t B) {
    const int64_t cap = V < 1 ? 1 : V;
    Carver cv(nullptr, 0);
    ExtractWs w;
    carve(cv, cap, cub_bytes_for(cap, 2 * kCoordBits + clip_bits(B)), w);
    const size_t a = cv.used(), b = extract_clip_workspace_bytes(0, B);
    return a > b ? a : b;
}

// per-clip bucket path for polygons; FCFS_E_UNSUPPORTED (after its sync) if a clip has more than
// kBucketCap vertices: the caller falls back to the general path
static fcfs_status extract_polygon_clips(const int32_t *vx, const int32_t *vy, const int64_t *poly_ptr, int64_t P,
                                         const int64_t *clip_ptr, int64_t B, int32_t T, int32_t *x, int32_t *y,
                                         int32_t *w, int64_t cap, int64_t *corner_ptr, int64_t *area,
                                         int64_t *K_host, void *ws, size_t ws_bytes, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    ClipWs W;
    carve_clip(cv, 0, B, W);
    if (!cv.fits()) {
        set_error("fcfs_vertices_from_polygons: workspace %zu < %zu bytes", ws_bytes, cv.used());
        return FCFS_E_WORKSPACE;
    }
    FCFS_TRY_CUDA(cudaMemsetAsync(W.err, 0, 4 * sizeof(int32_t), s));
    FCFS_TRY_CUDA(cudaMemsetAsync(W.status, 0, B * sizeof(unsigned long long), s));
    const size_t bsmem = kBucketCap * 12 + (size_t)(T + 2) * 4;
    FCFS_TRY(ensure_smem((const void *)k_clip_polygons_bucket, kBucketCap * 12 + (kBucketMaxT + 2) * 4, true));
    // one CTA per clip (the look-back needs every predecessor clip's CTA dispatched before it)
    k_clip_polygons_bucket<<<(unsigned)B, kBucketThreads, bsmem, s>>>(vx, vy, poly_ptr, P, clip_ptr, B, T, x, y, w,
                                                                      cap, corner_ptr, W.status, area, W.err);
    FCFS_CHECK_LAUNCH("k_clip_polygons_bucket");
    int64_t Kh = 0;
    int32_t errh = 0;
    FCFS_TRY_CUDA(cudaMemcpyAsync(&Kh, corner_ptr + B, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    FCFS_TRY_CUDA(cudaMemcpyAsync(&errh, W.err, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    FCFS_TRY_CUDA(cudaStreamSynchronize(s));
    if (errh & 8) {
        set_error("a clip has more than %d vertices", kBucketCap);
        return FCFS_E_UNSUPPORTED;
    }
    if (K_host) *K_host = Kh;
    if (errh & 16) {
        set_error("fcfs_vertices_from_polygons: a polygon edge is diagonal or of zero length");
        return FCFS_E_INVALID;
    }
    if (errh & 1) {
        set_error("fcfs_vertices_from_polygons: a vertex lies outside [0,T]^2");
        return FCFS_E_RANGE;
    }
    if (Kh > cap) {
        set_error("fcfs_vertices_from_polygons: K=%lld > cap=%lld", (long long)Kh, (long long)cap);
        return FCFS_E_CAPACITY;
    }
    return FCFS_OK;
}

// polygon vertex lists -> canonical corners: one raw corner per vertex (k_polygon_corners), then the
// general path's sort / merge / compaction (polygons of a clip are summed)
fcfs_status extract_polygons(const int32_t *vx, const int32_t *vy, int64_t V, const int64_t *poly_ptr, int64_t P,
                             const int64_t *clip_ptr, int64_t B, int32_t T, int32_t *x, int32_t *y, int32_t *w,
                             int64_t cap, int64_t *corner_ptr, int64_t *area, int64_t *K_host, void *ws,
                             size_t ws_bytes, cudaStream_t s) {
    if (T <= kBucketMaxT && B >= 1 && V > 0 && (clip_ptr != nullptr || V <= kBucketCap)) {
        fcfs_status st = extract_polygon_clips(vx, vy, poly_ptr, P, clip_ptr, B, T, x, y, w, cap, corner_ptr, area,
                                               K_host, ws, ws_bytes, s);
        if (st != FCFS_E_UNSUPPORTED) return st;   // else: a clip is too large for the per-clip path
    }
    const int64_t cap_raw = V < 1 ? 1 : V;
    if (cap_raw >= (int64_t(1) << 31)) {
        set_error("fcfs_vertices_from_polygons: %lld vertices exceed 2^31", (long long)V);
        return FCFS_E_UNSUPPORTED;
    }
    int cb = coord_bits(T), end_bit = 2 * cb + clip_bits(B);
    const size_t cub_max = cub_bytes_for(cap_raw, 2 * kCoordBits + clip_bits(B));   // as the size query
    if (cub_bytes_for(cap_raw, end_bit) > cub_max) { cb = kCoordBits; end_bit = 2 * cb + clip_bits(B); }
    Carver cv(ws, ws_bytes);
    ExtractWs W;
    carve(cv, cap_raw, cub_max, W);
    if (!cv.fits()) {
        set_error("fcfs_vertices_from_polygons: workspace %zu < %zu bytes", ws_bytes, cv.used());
        return FCFS_E_WORKSPACE;
    }
    FCFS_TRY_CUDA(cudaMemsetAsync(W.err, 0, 4 * sizeof(int32_t), s));
    FCFS_TRY_CUDA(cudaMemsetAsync(W.num_runs, 0, 2 * sizeof(int64_t), s));
    FCFS_TRY_CUDA(cudaMemsetAsync(area, 0, B * sizeof(int64_t), s));
    // sentinels first: vertices outside every polygon's CSR range are never visited
    k_fill_sentinel<<<(unsigned)(cap_raw < 148 * 4 * 256 ? (cap_raw + 255) / 256 : 148 * 4), 256, 0, s>>>(
        W.keys_a, W.w_a, cap_raw, nullptr);
    FCFS_CHECK_LAUNCH("k_fill_sentinel");
    if (P > 0 && V > 0) {
        int64_t blocks = (P + 7) / 8;   // 8 warps (polygons) per block
        if (blocks > 148 * 16) blocks = 148 * 16;
        k_polygon_corners<<<(unsigned)blocks, 256, 0, s>>>(vx, vy, poly_ptr, P, clip_ptr, B, T, W.keys_a, W.w_a,
                                                           W.err);
        FCFS_CHECK_LAUNCH("k_polygon_corners");
    }
    int64_t Kh = 0;
    int32_t errh = 0;
    fcfs_status st = finish_corners(W, cap_raw, cb, end_bit, B, cap, x, y, w, corner_ptr, area, Kh, errh, s);
    if (st != FCFS_OK) return st;
    if (K_host) *K_host = Kh;
    if (errh & 16) {
        set_error("fcfs_vertices_from_polygons: a polygon edge is diagonal or of zero length");
        return FCFS_E_INVALID;
    }
    if (errh & 1) {
        set_error("fcfs_vertices_from_polygons: a vertex lies outside [0,T]^2");
        return FCFS_E_RANGE;
    }
    if (Kh > cap) {
        set_error("fcfs_vertices_from_polygons: K=%lld > cap=%lld", (long long)Kh, (long long)cap);
        return FCFS_E_CAPACITY;
    }
    return FCFS_OK;
}

}  // namespace fcfs

// buckets.cu — row buckets of the signed corner list: the row structure of Step 4.
//
// Step 4 of the paper evaluates the interior coefficients of Eq. Fkl
// as DFTs of the sparse image f~_xy whose non-zeros sit on horizontal
// edges: corners that share a row y share the factor E_y[n, y].  Grouping them,
//     sum_k w_k E_x[m,k] E_y[n,k] = sum_rows E_y[n, y_r] * G[m, r],
//     G[m, r] = sum_{k in row r} w_k E_x[m, x_k]            (a sparse row DFT)
// so the tensor-core contraction runs over R rows instead of K corners (K/R = 3.7 for
// BASELINE.json configs[2], 15 for configs[3]).  The axis sums (Eqs. Fk0/F0l) group the
// same way: sum_k w_k y_k E_x = sum_r y_r G[m, r], sum_k w_k x_k E_y = sum_r E_y (sum w x).
//
// A bucket is a maximal run of CONSECUTIVE corners with equal y, cut
//   - at every clip start (buckets never cross clips),
//   - at every kSeg-corner segment boundary (one CTA per segment, no cross-CTA state),
//   - every `cap` corners inside a run (bounded per-bucket work for the producers).
// Any corner order is valid (an unsorted list just yields shorter buckets); the
// canonical (clip, y, x) order of fcfs_vertices_from_rects gives the longest ones.
//
// Outputs (workspace): bptr[nb+1] (global corner index of each bucket start, bptr[nb] =
// k_hi), by[nb] (the bucket's y), clip_bptr[B+1] (CSR of buckets per clip).
#include <cub/cub.cuh>

#include "common.cuh"

namespace fcfs {
namespace bk {
constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kSeg = kThreads * kItems;   // 4096 corners per segment
}  // namespace bk

struct BucketSegInfo {
    const int32_t *y;
    const int64_t *corner_ptr;   // [B+1] or nullptr (one range)
    int64_t B, k_lo, k_hi;
    int32_t cap;
};

// flags of the kItems corners of this thread (bit j = corner ks + 16 t + j starts a bucket); shared
// by the count and the write pass so both see identical buckets.  Each thread loads its 16
// consecutive y with vector loads; the previous corner's y comes from the neighbouring lane (or
// warp); clip starts come from a per-thread binary search of corner_ptr.
template <class Scan>
__device__ __forceinline__ uint32_t bucket_flags(const BucketSegInfo &a, int64_t ks, int n, int32_t (&yv)[bk::kItems],
                                                 int32_t *warp_last, typename Scan::TempStorage &tmp) {
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int j0 = t * bk::kItems;
    const int64_t k0 = ks + j0;
    // vector loads only where the address itself is 16-byte aligned (the caller's y may start anywhere)
    if (j0 + bk::kItems <= n && (((uintptr_t)(a.y + k0)) & 15u) == 0) {
        const int4 *p = (const int4 *)(a.y + k0);
#pragma unroll
        for (int v = 0; v < bk::kItems / 4; ++v) {
            const int4 q = __ldg(p + v);
            yv[4 * v] = q.x; yv[4 * v + 1] = q.y; yv[4 * v + 2] = q.z; yv[4 * v + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < bk::kItems; ++i) yv[i] = j0 + i < n ? __ldg(a.y + k0 + i) : 0;
    }
    int prev = __shfl_up_sync(0xffffffffu, yv[bk::kItems - 1], 1);
    if (lane == 31) warp_last[wid] = yv[bk::kItems - 1];
    // clip starts inside this thread's corners: first b with corner_ptr[b] >= k0
    uint32_t cs = 0;
    if (a.corner_ptr && j0 < n) {
        int64_t lo = 0, hi = a.B;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (__ldg(a.corner_ptr + mid) < k0) lo = mid + 1; else hi = mid;
        }
        for (int64_t b = lo; b <= a.B; ++b) {
            const int64_t c = __ldg(a.corner_ptr + b);
            if (c >= k0 + bk::kItems) break;
            cs |= 1u << (int)(c - k0);
        }
    }
    __syncthreads();
    if (lane == 0 && wid > 0) prev = warp_last[wid - 1];
    // run starts (segment start, clip start, y change) and the last run start before each corner
    uint32_t rs = 0;
    int last = -1;
#pragma unroll
    for (int i = 0; i < bk::kItems; ++i) {
        const int j = j0 + i;
        const int py = i ? yv[i - 1] : prev;
        if (j < n && (j == 0 || (cs & (1u << i)) || yv[i] != py)) { rs |= 1u << i; last = j; }
    }
    int before;
    Scan(tmp).ExclusiveScan(last, before, cub::Max());
    if (t == 0) before = 0;
    uint32_t bf = 0;
    int run = before;
#pragma unroll
    for (int i = 0; i < bk::kItems; ++i) {
        const int j = j0 + i;
        if (j >= n) break;
        if (rs & (1u << i)) run = j;
        if ((j - run) % a.cap == 0) bf |= 1u << i;
    }
    return bf;
}

__global__ void __launch_bounds__(bk::kThreads) k_bucket_count(BucketSegInfo a, int32_t *counts) {
    typedef cub::BlockScan<int, bk::kThreads> Scan;
    typedef cub::BlockReduce<int, bk::kThreads> Red;
    __shared__ int32_t warp_last[bk::kThreads / 32];
    __shared__ union {
        typename Scan::TempStorage scan;
        typename Red::TempStorage red;
    } tmp;
    const int64_t ks = a.k_lo + (int64_t)blockIdx.x * bk::kSeg;
    const int n = (int)min((int64_t)bk::kSeg, a.k_hi - ks);
    int32_t yv[bk::kItems];
    const uint32_t bf = bucket_flags<Scan>(a, ks, n, yv, warp_last, tmp.scan);
    __syncthreads();
    const int c = Red(tmp.red).Sum(__popc(bf));
    if (threadIdx.x == 0) counts[blockIdx.x] = c;
}

__global__ void __launch_bounds__(bk::kThreads) k_bucket_write(BucketSegInfo a, const int32_t *__restrict__ offs,
                                                               int32_t *bptr, int32_t *by) {
    typedef cub::BlockScan<int, bk::kThreads> Scan;
    __shared__ int32_t warp_last[bk::kThreads / 32];
    __shared__ typename Scan::TempStorage tmp;
    const int64_t ks = a.k_lo + (int64_t)blockIdx.x * bk::kSeg;
    const int n = (int)min((int64_t)bk::kSeg, a.k_hi - ks);
    int32_t yv[bk::kItems];
    const uint32_t bf = bucket_flags<Scan>(a, ks, n, yv, warp_last, tmp);
    __syncthreads();
    int pos;
    Scan(tmp).ExclusiveSum(__popc(bf), pos);
    pos += offs[blockIdx.x];
#pragma unroll
    for (int i = 0; i < bk::kItems; ++i) {
        if (!(bf & (1u << i))) continue;
        bptr[pos] = (int32_t)(ks + threadIdx.x * bk::kItems + i);
        by[pos] = yv[i];
        ++pos;
    }
}

// clip_bptr[b] = number of buckets starting before corner_ptr[b] (every clip start is a bucket
// start, so this is also the clip's first bucket); bptr[nb] = k_hi
__global__ void k_bucket_clips(const int64_t *__restrict__ corner_ptr, int64_t B, const int32_t *__restrict__ offs,
                               int64_t nseg, int64_t k_hi, int32_t *bptr, int64_t *clip_bptr) {
    const int64_t nb = offs[nseg];
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i == 0) bptr[nb] = (int32_t)k_hi;
    if (corner_ptr == nullptr) {
        if (i == 0) { clip_bptr[0] = 0; clip_bptr[1] = nb; }
        return;
    }
    if (i > B) return;
    const int64_t c = corner_ptr[i];
    int64_t lo = 0, hi = nb;   // first bucket with start >= c
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (bptr[mid] < c) lo = mid + 1; else hi = mid;
    }
    clip_bptr[i] = lo;
}

static int64_t nsegments(int64_t n) { return (n + bk::kSeg - 1) / bk::kSeg; }

size_t buckets_workspace_bytes(int64_t K, int64_t B) {
    Carver cv(nullptr, 0);
    BucketWs w;
    carve_buckets(cv, K, B, w);
    return cv.used();
}

void carve_buckets(Carver &cv, int64_t K, int64_t B, BucketWs &w) {
    const int64_t nseg = nsegments(K);
    w.bptr = cv.take<int32_t>(K + nseg + 16);   // nb <= K (+ sentinel, + copy padding)
    w.by = cv.take<int32_t>(K + nseg + 16);
    w.clip_bptr = cv.take<int64_t>(B + 1);
    w.counts = cv.take<int32_t>(nseg + 1);
    w.offs = cv.take<int32_t>(nseg + 1);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, (int32_t *)nullptr, (int32_t *)nullptr, (int)(nseg + 1));
    w.cub_tmp = cv.take<char>(tb + 16);
    w.cub_bytes = tb + 16;
}

fcfs_status run_buckets(const int32_t *y, const int64_t *corner_ptr, int64_t B, int64_t k_lo, int64_t k_hi,
                        int32_t cap, const BucketWs &w, cudaStream_t s) {
    if (k_hi - k_lo >= (int64_t(1) << 31) - 64 || k_hi >= (int64_t(1) << 31) - 64) {
        set_error("row buckets: corner index range [%lld, %lld) exceeds int32", (long long)k_lo, (long long)k_hi);
        return FCFS_E_UNSUPPORTED;
    }
    BucketSegInfo a;
    a.y = y; a.corner_ptr = corner_ptr; a.B = B; a.k_lo = k_lo; a.k_hi = k_hi; a.cap = cap;
    const int64_t nseg = nsegments(k_hi - k_lo);
    FCFS_TRY_CUDA(cudaMemsetAsync(w.counts, 0, sizeof(int32_t) * (nseg + 1), s));
    if (nseg > 0) {
        k_bucket_count<<<(unsigned)nseg, bk::kThreads, 0, s>>>(a, w.counts);
        FCFS_CHECK_LAUNCH("k_bucket_count");
    }
    size_t tb = w.cub_bytes;
    FCFS_TRY_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.counts, w.offs, (int)(nseg + 1), s));
    count_launch();
    if (nseg > 0) {
        k_bucket_write<<<(unsigned)nseg, bk::kThreads, 0, s>>>(a, w.offs, w.bptr, w.by);
        FCFS_CHECK_LAUNCH("k_bucket_write");
    }
    const int64_t nthreads = corner_ptr ? B + 1 : 1;
    k_bucket_clips<<<(unsigned)((nthreads + 255) / 256), 256, 0, s>>>(corner_ptr, B, w.offs, nseg, k_hi, w.bptr,
                                                                       w.clip_bptr);
    FCFS_CHECK_LAUNCH("k_bucket_clips");
    return FCFS_OK;
}

}  // namespace fcfs

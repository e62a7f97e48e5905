// haar.cu — the continuous Haar transform of clips (the paper's CHT / PCHT,
// P:453-480).  Basis (reading A18 of DESIGN.md): phi_{j,kx,ky} = (2^j / T) 1[cell],
// psi^{(ab)} = sum_{n,m} a_n b_m phi_{j+1,2kx+n,2ky+m}, g = (1,1)/sqrt2, h = (1,-1)/sqrt2, J = log2 T.
//
// The paper's PCHT recurses over the quadtree and intersects each boundary cell with the polygons
// (Alg. 1).  Here the same coefficients come straight from the signed corners, f = sum_k w_k H(x-x_k)
// H(y-y_k), because the basis is separable (Lemma polyip):
//
//   C^{(ab)}_{j,kx,ky} = (2^j / T) sum_k w_k I_a(x_k) I_b(y_k),
//   I_g(x) = integral of H(. - x) over the cell's x-range = clamp(a2 - max(a1, x)),
//   I_h(x) = (left half) - (right half) = -tent(x): -(x - a1) on [a1, mid], -(a2 - x) on [mid, a2], else 0.
//
// I_h is supported inside the cell, so a corner touches ONE cell per level through an h factor: the
// hh numerators are a scatter of the corners; hg (h in x, g in y) = the corner's own cell (partial
// g = b2 - y) plus, for every cell above it in its column, s I_h(x) (full g): a column prefix sum of
// per-cell totals; gh likewise along rows.  That is the pruning of the PCHT — only cells crossed by
// the boundary get non-zero details — without a recursion: O(K J) atomics + O(T^2) prefix sums and
// output writes.  Every numerator is an exact integer (int64 atomics: order-independent), every
// coefficient an integer times 2^j / T: the FP64 output is exact.
#include "common.cuh"

namespace fcfs {

namespace haar {

constexpr int kThreads = 256;
#ifndef HAAR_UC
#define HAAR_UC 8
#endif
#ifndef HAAR_UR
#define HAAR_UR 4
#endif

// scratch per clip: for each level j (n = 2^j cells per side) five int64 n x n arrays at
// level_off(j) = 5 (4^j - 1) / 3: [0] hh, [1] hg partial, [2] hg column totals, [3] gh partial,
// [4] gh row totals
__host__ __device__ inline int64_t level_off(int j) { return 5 * ((((int64_t)1) << (2 * j)) - 1) / 3; }
__host__ __device__ inline int64_t clip_scratch(int J) { return level_off(J); }

__device__ __forceinline__ void add64(int64_t *p, int64_t v) {
    if (v) atomicAdd((unsigned long long *)p, (unsigned long long)v);
}

// thread per (corner, level)
__global__ void k_haar_scatter(const int32_t *__restrict__ x, const int32_t *__restrict__ y,
                               const int32_t *__restrict__ w, const int64_t *__restrict__ corner_ptr, int64_t B,
                               int64_t K, int32_t T, int J, int64_t *scratch, const int32_t *unsorted) {
    if (!*unsorted) return;   // y-sorted clips take the band sweep (k_haar_band)
    const int64_t total = K * J;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / J;
        const int j = (int)(i - k * J);
        const int32_t xk = x[k], yk = y[k];
        if (xk >= T || yk >= T) continue;   // corners on x = T or y = T touch no cell
        // clip of corner k (last b with corner_ptr[b] <= k)
        int64_t b = 0;
        if (corner_ptr) {
            int64_t lo = 0, hi = B - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (corner_ptr[mid] <= k) lo = mid; else hi = mid - 1;
            }
            b = lo;
        }
        const int64_t wk = w[k];
        const int sh = J - j;                      // cell side s = 2^sh
        const int32_t s = 1 << sh, hs = s >> 1;
        const int32_t kx = xk >> sh, ky = yk >> sh;
        const int32_t ax = kx * s, ay = ky * s;
        const int32_t dx = xk - ax, dy = yk - ay;  // in [0, s)
        const int64_t ihx = -(int64_t)(dx <= hs ? dx : s - dx), ihy = -(int64_t)(dy <= hs ? dy : s - dy);
        const int64_t igx = s - dx, igy = s - dy;  // own-cell partial g
        const int64_t n = (int64_t)1 << j;
        int64_t *L = scratch + b * clip_scratch(J) + level_off(j);
        const int64_t c = (int64_t)ky * n + kx;
        add64(L + 0 * n * n + c, wk * ihx * ihy);
        add64(L + 1 * n * n + c, wk * ihx * igy);
        add64(L + 2 * n * n + c, wk * ihx);
        add64(L + 3 * n * n + c, wk * igx * ihy);
        add64(L + 4 * n * n + c, wk * ihy);
    }
}

// (clip, level, line) of the flattened line index r in [0, B (T - 1)): level j has 2^j lines
__device__ __forceinline__ void line_of(int64_t i, int32_t T, int64_t &b, int &j, int64_t &line) {
    const int64_t per_clip = T - 1;
    b = i / per_clip;
    int64_t r = i - b * per_clip;
    j = 0;
    while (r >= ((int64_t)1 << j)) { r -= (int64_t)1 << j; ++j; }
    line = r;
}

// thread per (clip, level, column kx): hg = own-cell partial + s x (exclusive prefix over ky of the
// column totals), scaled by 2^j / T (exact); consecutive threads write consecutive columns
__global__ void k_haar_cols(const int64_t *scratch, const int64_t *__restrict__ area, int64_t B,
                            int32_t T, int J, double *out, const int32_t *unsorted) {
    if (!*unsorted) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B * (int64_t)(T - 1);
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t b, kx;
        int j;
        line_of(i, T, b, j, kx);
        const int64_t n = (int64_t)1 << j, s = (int64_t)T >> j;
        const double scale = (double)n / (double)T;
        const int64_t *L = scratch + b * clip_scratch(J) + level_off(j);
        double *o = out + b * (int64_t)T * T;
        if (j == 0) o[0] = (double)area[b] / (double)T;   // X_{0,0,0}
        int64_t *Lw = const_cast<int64_t *>(L);
        int64_t run = 0;
        // kU rows per step, all loads first: the loads of a step are independent, and issuing them
        // together hides the latency that a load -> store -> next load walk would expose per row
        constexpr int kU = HAAR_UC;
        for (int64_t k0 = 0; k0 < n; k0 += kU) {
            int64_t part[kU], tot[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t c = (k0 + u) * n + kx;
                const bool ok = k0 + u < n;
                part[u] = ok ? L[1 * n * n + c] : 0;
                tot[u] = ok ? L[2 * n * n + c] : 0;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t ky = k0 + u;
                if (ky >= n) break;
                const int64_t c = ky * n + kx;
                o[ky * T + n + kx] = (double)(part[u] + s * run) * scale;
                run += tot[u];
                if (part[u]) Lw[1 * n * n + c] = 0;   // leave the scratch zero for the next call (sparse clears)
                if (tot[u]) Lw[2 * n * n + c] = 0;
            }
        }
    }
}

// warp per (clip, level, row ky): gh = own-cell partial + s x (exclusive prefix over kx of the row
// totals; warp scan, 32 columns at a time, coalesced) and hh, scaled by 2^j / T
__global__ void k_haar_rows(const int64_t *scratch, int64_t B, int32_t T, int J, double *out,
                            const int32_t *unsorted) {
    if (!*unsorted) return;
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < B * (int64_t)(T - 1); i += nwarps) {
        int64_t b, ky;
        int j;
        line_of(i, T, b, j, ky);
        const int64_t n = (int64_t)1 << j, s = (int64_t)T >> j;
        const double scale = (double)n / (double)T;
        const int64_t *L = scratch + b * clip_scratch(J) + level_off(j);
        double *o = out + b * (int64_t)T * T + (n + ky) * T;
        int64_t carry = 0;
        constexpr int kU = HAAR_UR;   // 32-column chunks per step, all loads first (independent: latency overlapped)
        for (int64_t k00 = 0; k00 < n; k00 += 32 * kU) {
            int64_t tot[kU], part[kU], hh[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t kx = k00 + 32 * u + lane;
                const bool ok = kx < n;
                const int64_t c = ky * n + kx;
                tot[u] = ok ? L[4 * n * n + c] : 0;
                part[u] = ok ? L[3 * n * n + c] : 0;
                hh[u] = ok ? L[0 * n * n + c] : 0;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t k0 = k00 + 32 * u;
                if (k0 >= n) break;   // uniform
                const int64_t kx = k0 + lane;
                const bool ok = kx < n;
                const int64_t c = ky * n + kx;
                int64_t inc = tot[u];
                for (int d = 1; d < 32; d <<= 1) {
                    const int64_t v = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc += v;
                }
                if (ok) {
                    o[kx] = (double)(part[u] + s * (carry + inc - tot[u])) * scale;
                    o[n + kx] = (double)hh[u] * scale;
                    int64_t *Lw = const_cast<int64_t *>(L);
                    if (tot[u]) Lw[4 * n * n + c] = 0;
                    if (part[u]) Lw[3 * n * n + c] = 0;
                    if (hh[u]) Lw[0 * n * n + c] = 0;
                }
                carry += __shfl_sync(0xffffffffu, inc, 31);
            }
        }
    }
}


// ---------------------------------------------------------------- band sweep (y-sorted clips)
//
// For clips whose corners are sorted by y (as fcfs_vertices_from_* emit them) the coefficients are
// computed without the global scratch: a CTA owns (clip, level j, a block of kRB cell rows).  It first
// sums the column totals w I_h(x) of every corner in the cell rows above the block (the hg column prefix),
// then walks its rows in order: the corners of cell row ky are one contiguous range of the sorted list
// (yptr), their five per-cell terms go into shared-memory row arrays, a block scan gives the gh row
// prefix, and the row's hg / gh / hh outputs are written once, coalesced.  Traffic: the corners (once per
// level and block above) and the outputs; no O(T^2) scratch reads.  Integer arithmetic: bit-identical
// to the scatter path.

constexpr int kBT = 128;   // threads per band CTA
constexpr int kRB = 32;    // cell rows per band CTA

// yptr[b][v] = #corners of clip b with y < v (v = 0..T), by binary search; unsorted = 1 if y decreases
// inside a clip (then the scatter path runs instead)
__global__ void k_haar_yptr(const int32_t *__restrict__ y, const int64_t *__restrict__ corner_ptr, int64_t B,
                            int64_t K, int32_t T, int32_t *yptr, int32_t *unsorted) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nv = (int64_t)T + 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B * nv; i += stride) {
        const int64_t b = i / nv;
        const int32_t v = (int32_t)(i - b * nv);
        const int64_t k0 = corner_ptr ? corner_ptr[b] : 0, k1 = corner_ptr ? corner_ptr[b + 1] : K;
        int64_t lo = k0, hi = k1;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (__ldg(y + mid) < v) lo = mid + 1; else hi = mid;
        }
        yptr[i] = (int32_t)(lo - k0);
    }
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1; k < K; k += stride) {
        if (__ldg(y + k - 1) <= __ldg(y + k)) continue;
        int64_t lo = 0, hi = corner_ptr ? B : 0;   // a decrease is allowed only where a clip starts
        if (!corner_ptr) { *unsorted = 1; continue; }
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (corner_ptr[mid] < k) lo = mid + 1; else hi = mid;
        }
        if (lo > B || corner_ptr[lo] != k) *unsorted = 1;
    }
}

__host__ __device__ inline int64_t band_tasks_per_clip(int J) {
    int64_t t = 0;
    for (int j = 0; j < J; ++j) t += (((int64_t)1 << j) + kRB - 1) / kRB;
    return t;
}

__global__ void __launch_bounds__(kBT) k_haar_band(const int32_t *__restrict__ x, const int32_t *__restrict__ y,
                                                   const int32_t *__restrict__ w, const int64_t *__restrict__ corner_ptr,
                                                   int64_t B, int32_t T, int J, const int64_t *__restrict__ area,
                                                   const int32_t *__restrict__ yptr, const int32_t *unsorted,
                                                   double *out) {
    if (*unsorted) return;   // the scatter path runs instead
    extern __shared__ __align__(16) unsigned char hb_smem[];
    const int nmax = T >> 1;
    long long *colp = (long long *)hb_smem;   // hg column prefix (cell rows above the current one)
    long long *phg = colp + nmax, *thg = phg + nmax, *pgh = thg + nmax, *tgh = pgh + nmax, *hhv = tgh + nmax;
    __shared__ long long wsum[kBT / 32];
    __shared__ int32_t rb[kRB + 1];
    // task -> (clip, level, block): big levels first (their blocks are the long ones)
    int64_t t = blockIdx.x;
    int j = J - 1;
    int64_t nb = 0;
    for (; j >= 0; --j) {
        nb = (((int64_t)1 << j) + kRB - 1) / kRB;
        if (t < B * nb) break;
        t -= B * nb;
    }
    if (j < 0) return;
    const int64_t b = t / nb;
    const int blk = (int)(t - b * nb);
    const int n = 1 << j, sh = J - j;
    const int32_t s = 1 << sh, hs = s >> 1;
    const double scale = (double)n / (double)T;
    const int ky0 = blk * kRB, ky1 = min(n, ky0 + kRB);
    const int64_t k0 = corner_ptr ? corner_ptr[b] : 0;
    const int32_t *yp = yptr + b * ((int64_t)T + 1);
    double *o = out + b * (int64_t)T * T;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < 6 * n; i += kBT) {
        const int a = i / n, c = i - a * n;
        colp[a * nmax + c] = 0;
    }
    for (int i = tid; i <= ky1 - ky0; i += kBT) rb[i] = yp[(ky0 + i) << sh];
    if (j == 0 && tid == 0) o[0] = (double)area[b] / (double)T;   // X_{0,0,0}
    __syncthreads();
    // hg column prefix of the rows above the block
    for (int64_t k = k0 + tid; k < k0 + rb[0]; k += kBT) {
        const int32_t xk = __ldg(x + k);
        if (xk >= T) continue;
        const int32_t kx = xk >> sh, dx = xk - (kx << sh);
        const long long ihx = -(long long)(dx <= hs ? dx : s - dx);
        const long long v = (long long)__ldg(w + k) * ihx;
        if (v) atomicAdd((unsigned long long *)&colp[kx], (unsigned long long)v);
    }
    const int per = (n + kBT - 1) / kBT;   // scan: thread tid owns cells [tid per, (tid + 1) per)
    // this thread's first corner of the current row, loaded one row ahead (the loads overlap the previous
    // row's scan and outputs instead of stalling every row at the barrier after the scatter)
    int32_t px = T, py = 0, pw = 0;
    if (ky0 < ky1 && k0 + rb[0] + tid < k0 + rb[1]) {
        const int64_t k = k0 + rb[0] + tid;
        px = __ldg(x + k); py = __ldg(y + k); pw = __ldg(w + k);
    }
    for (int ky = ky0; ky < ky1; ++ky) {
        // the corners of cell row ky: one contiguous range of the y-sorted list
        const int64_t pa = k0 + rb[ky - ky0], pe = k0 + rb[ky - ky0 + 1];
        auto add = [&](int32_t xk, int32_t yk, int32_t wi) {
            if (xk >= T) return;
            const long long wk = wi;
            const int32_t kx = xk >> sh, dx = xk - (kx << sh), dy = yk - (ky << sh);
            const long long ihx = -(long long)(dx <= hs ? dx : s - dx), ihy = -(long long)(dy <= hs ? dy : s - dy);
            const long long igx = s - dx, igy = s - dy;
            atomicAdd((unsigned long long *)&phg[kx], (unsigned long long)(wk * ihx * igy));
            atomicAdd((unsigned long long *)&thg[kx], (unsigned long long)(wk * ihx));
            atomicAdd((unsigned long long *)&pgh[kx], (unsigned long long)(wk * igx * ihy));
            atomicAdd((unsigned long long *)&tgh[kx], (unsigned long long)(wk * ihy));
            atomicAdd((unsigned long long *)&hhv[kx], (unsigned long long)(wk * ihx * ihy));
        };
        if (pa + tid < pe) add(px, py, pw);
        for (int64_t k = pa + tid + kBT; k < pe; k += kBT) add(__ldg(x + k), __ldg(y + k), __ldg(w + k));
        if (ky + 1 < ky1) {
            const int64_t qe = k0 + rb[ky - ky0 + 2];
            if (pe + tid < qe) { px = __ldg(x + pe + tid); py = __ldg(y + pe + tid); pw = __ldg(w + pe + tid); }
        }
        __syncthreads();
        // exclusive prefix of the gh row totals over kx, in place
        {
            const int lo = tid * per, hi = min(lo + per, n);
            long long own = 0;
            for (int c = lo; c < hi; ++c) own += tgh[c];
            long long inc = own;
            for (int d = 1; d < 32; d <<= 1) {
                const long long v = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += v;
            }
            if (lane == 31) wsum[wid] = inc;
            __syncthreads();
            long long run = inc - own;
            for (int i = 0; i < wid; ++i) run += wsum[i];
            for (int c = lo; c < hi; ++c) { const long long v = tgh[c]; tgh[c] = run; run += v; }
        }
        __syncthreads();
        double *o_hg = o + (int64_t)ky * T + n, *o_gh = o + (int64_t)(n + ky) * T;
        for (int c = tid; c < n; c += kBT) {
            o_hg[c] = (double)(phg[c] + (long long)s * colp[c]) * scale;
            o_gh[c] = (double)(pgh[c] + (long long)s * tgh[c]) * scale;
            o_gh[n + c] = (double)hhv[c] * scale;
            colp[c] += thg[c];
            phg[c] = 0; thg[c] = 0; pgh[c] = 0; tgh[c] = 0; hhv[c] = 0;
        }
        __syncthreads();
    }
}

}  // namespace haar

static int log2_exact(int32_t T) {
    int J = 0;
    while ((1 << J) < T) ++J;
    return (1 << J) == T ? J : -1;
}

size_t haar_workspace_bytes(int64_t B, int32_t T) {
    const int J = log2_exact(T);
    if (J < 1 || B < 1) return 0;
    Carver cv(nullptr, 0);
    cv.take<int64_t>((size_t)(B * haar::clip_scratch(J)));
    cv.take<int32_t>((size_t)(B * ((int64_t)T + 1)));   // yptr
    cv.take<int32_t>(1);                                 // unsorted flag
    return cv.used();
}

fcfs_status haar_clips(const int32_t *x, const int32_t *y, const int32_t *w, const int64_t *corner_ptr, int64_t B,
                       int64_t K, const int64_t *area, int32_t T, double *out, void *ws, size_t ws_bytes,
                       cudaStream_t s) {
    const int J = log2_exact(T);
    Carver cv(ws, ws_bytes);
    int64_t *scratch = cv.take<int64_t>((size_t)(B * haar::clip_scratch(J)));
    int32_t *yptr = cv.take<int32_t>((size_t)(B * ((int64_t)T + 1)));
    int32_t *unsorted = cv.take<int32_t>(1);
    if (!cv.fits()) {
        set_error("fcfs_haar: workspace %zu < %zu bytes", ws_bytes, cv.used());
        return FCFS_E_WORKSPACE;
    }
    // y-sorted clips (the extraction's output) take the band sweep; any other order the scatter path.
    // Both are launched; each checks the device flag first, so the call needs no host sync.
    FCFS_TRY_CUDA(cudaMemsetAsync(unsorted, 0, sizeof(int32_t), s));
    {
        const int64_t work = B * ((int64_t)T + 1) > K ? B * ((int64_t)T + 1) : K;
        int64_t blocks = (work + 255) / 256;
        if (blocks > 148 * 32) blocks = 148 * 32;
        haar::k_haar_yptr<<<(unsigned)blocks, 256, 0, s>>>(y, corner_ptr, B, K, T, yptr, unsorted);
        FCFS_CHECK_LAUNCH("k_haar_yptr");
    }
    {
        const int64_t tasks = B * haar::band_tasks_per_clip(J);
        const size_t smem = (size_t)6 * (size_t)(T / 2) * sizeof(long long);
        FCFS_TRY(ensure_smem((const void *)haar::k_haar_band, smem, false));
        haar::k_haar_band<<<(unsigned)tasks, haar::kBT, smem, s>>>(x, y, w, corner_ptr, B, T, J, area, yptr, unsorted,
                                                                   out);
        FCFS_CHECK_LAUNCH("k_haar_band");
    }
    // the scratch is zero on entry (caller contract: zero-initialised once; every call clears the
    // entries it used, so no O(T^2) memset per call)
    if (K > 0) {
        int64_t blocks = (K * J + haar::kThreads - 1) / haar::kThreads;
        if (blocks > 148 * 32) blocks = 148 * 32;
        haar::k_haar_scatter<<<(unsigned)blocks, haar::kThreads, 0, s>>>(x, y, w, corner_ptr, B, K, T, J, scratch,
                                                                          unsorted);
        FCFS_CHECK_LAUNCH("k_haar_scatter");
    }
    const int64_t lines = B * (int64_t)(T - 1);
    int64_t lb = (lines + 127) / 128;
    if (lb > 148 * 32) lb = 148 * 32;
    haar::k_haar_cols<<<(unsigned)lb, 128, 0, s>>>(scratch, area, B, T, J, out, unsorted);
    FCFS_CHECK_LAUNCH("k_haar_cols");
    int64_t rb = (lines * 32 + 255) / 256;
    if (rb > 148 * 32) rb = 148 * 32;
    haar::k_haar_rows<<<(unsigned)rb, 256, 0, s>>>(scratch, B, T, J, out, unsorted);
    FCFS_CHECK_LAUNCH("k_haar_rows");
    return FCFS_OK;
}

}  // namespace fcfs

// small.cu — the latency path for ONE SMALL CLIP (c1-size): a1-a5 in a single kernel launch with no
// host synchronisation, so a step is capturable in a CUDA graph (fcfs_small_clip; SURVEY §7 H4,
// §8(b) "device-side K").  This is the paper's regime of "only a few CFS coefficients", evaluated
// directly, Goertzel-like, term by term instead of through a GEMM or FFT.
//
// Every CTA redoes the (tiny) extraction in shared memory — union of each group's rects on its
// compressed grid (Prop. 1: the mixed difference of the union indicator), block radix sort
// of the raw corners by (y, x), merge of equal keys (groups SUMMED, reading A5), zero weights dropped —
// then computes its share of the half window:
//
//   row m >= 1:  A_k = w_k E(m x_k);  F[m, n] = -S / (4 pi^2 m n),  S = sum_k A_k E(n y_k)      (Eq. Fkl)
//                F[m, 0] = i sum_k A_k y_k / (2 pi m T)                                          (Eq. Fk0)
//   row m = 0:   F[0, n] = i sum_k w_k x_k E(n y_k) / (2 pi n T)                                  (Eq. F0l)
//                F[0, 0] = area / T^2                                                             (Eq. Fdc)
//   E(v) = e^{-2 pi i v / T} from an FP64 table over the exact integer phase (m x_k) mod T;
//   F[-m, -n] = conj F[m, n], written bit-exactly.
//
// All arithmetic is FP64 whatever the precision argument (the result meets every contract); the split
// precisions only select complex64 output.  One CTA per (row m, block of n); warp per output n, lanes
// over the corners, FP64 shuffle reduction.
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "coeff.cuh"

namespace fcfs {
namespace sm {

constexpr int kThreads = 512;              // 1024 measured slower (64-register cap, idle warps in the output phase)
constexpr int kItems = 4;
constexpr int kMaxRaw = kThreads * kItems;   // 2048 raw corners per clip
constexpr int kMaxGroup = 100;
constexpr int kMaxT = 8192;
constexpr int kNBlk = 4;                     // CTAs per output row (blocks of n)
constexpr uint32_t kKeyBits = 14;            // x, y in [0, 8192]
constexpr int kMaxN = 4096;                  // |n| <= 4096: n y < 2^25, exact in 32-bit phase arithmetic
constexpr uint32_t kSentinel = 0xFFFFFFFFu;

struct Args {
    const int4 *rects;
    int64_t R;
    const int64_t *group_ptr;
    int64_t G;
    int32_t T, M, N, layout, mg;
    double r2;
    int32_t out_f32;
    void *F;
    int64_t *K_out;
    int32_t *status;
};

using Sort = cub::BlockRadixSort<uint32_t, kThreads, kItems, int32_t>;
using Sort1 = cub::BlockRadixSort<uint32_t, kThreads, 1, int32_t>;    // <= kThreads raw corners
using Scan = cub::BlockScan<int32_t, kThreads>;
struct Shared;

struct Shared {   // head of the dynamic shared memory; after it: the group scratch, then the twiddle table
    union {
        typename Sort::TempStorage sort;
        typename Sort1::TempStorage sort1;
        typename Scan::TempStorage scan;
    } cub;
    uint32_t key[kMaxRaw];
    int32_t wt[kMaxRaw];
    int32_t cx[kMaxRaw], cy[kMaxRaw], cw[kMaxRaw];   // canonical corners
    int32_t nraw, K, err, nxy[2];
    long long asum[kThreads / 32];
    int32_t rowoff[2 * 64 + 2];
};

constexpr size_t kSharedBytes = (sizeof(Shared) + 255) & ~(size_t)255;

__device__ __forceinline__ bool rect_ok_s(int4 q, int32_t T) {
    return q.x >= 0 && q.y >= 0 && q.z <= T && q.w <= T && q.x < q.z && q.y < q.w;
}

__device__ __forceinline__ void push_raw(Shared &S, int32_t x, int32_t y, int32_t w) {
    const int p = atomicAdd(&S.nraw, 1);
    if (p < kMaxRaw) { S.key[p] = ((uint32_t)y << kKeyBits) | (uint32_t)x; S.wt[p] = w; }
}

// stable rank sort + unique of v[0..n) (n <= 2 kMaxGroup <= kThreads / 2) into u, count in *nu: two
// threads per value rank it over half the array each, a block scan of the run heads places the uniques
__device__ void compress_s(const int32_t *v, int n, int32_t *tmp, int32_t *u, int32_t *nu,
                           typename Scan::TempStorage &scan) {
    {
        const int i = threadIdx.x >> 1, half = threadIdx.x & 1;
        int rank = 0;
        int32_t vi = 0;
        if (i < n) {
            vi = v[i];
            const int j0 = half ? n / 2 : 0, j1 = half ? n : n / 2;
            for (int j = j0; j < j1; ++j) rank += (v[j] < vi) || (v[j] == vi && j < i);
        }
        rank += __shfl_xor_sync(0xffffffffu, rank, 1);
        if (i < n && !half) tmp[rank] = vi;
    }
    __syncthreads();
    const int i = threadIdx.x;
    const int head = (i < n && (i == 0 || tmp[i] != tmp[i - 1])) ? 1 : 0;
    int pos, total;
    Scan(scan).ExclusiveSum(head, pos, total);
    if (head) u[pos] = tmp[i];
    if (i == 0) *nu = total;
    __syncthreads();
}

__device__ __forceinline__ int find_s(const int32_t *u, int n, int32_t key) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (u[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// union of one group's rects (n <= kMaxGroup) on its compressed grid -> raw corners
__device__ void group_union(Shared &S, uint8_t *dyn, const int4 *rects, int n, int32_t T) {
    int4 *sr = (int4 *)dyn;
    int32_t *vx = (int32_t *)(sr + kMaxGroup);
    int32_t *vy = vx + 2 * kMaxGroup;
    int32_t *ux = vy + 2 * kMaxGroup;
    int32_t *uy = ux + 2 * kMaxGroup;
    int32_t *tmp = uy + 2 * kMaxGroup;
    int32_t *grid = tmp + 2 * kMaxGroup;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int4 q = rects[i];
        if (!rect_ok_s(q, T)) { atomicOr(&S.err, 1); q = make_int4(0, 0, 0, 0); }
        sr[i] = q;
        vx[2 * i] = q.x; vx[2 * i + 1] = q.z;
        vy[2 * i] = q.y; vy[2 * i + 1] = q.w;
    }
    __syncthreads();
    compress_s(vx, 2 * n, tmp, ux, &S.nxy[0], S.cub.scan);
    compress_s(vy, 2 * n, tmp, uy, &S.nxy[1], S.cub.scan);
    const int nx = S.nxy[0], ny = S.nxy[1];
    FCFS_DCHECK(nx >= 1 && ny >= 1 && nx <= 2 * n && ny <= 2 * n);
    // row stride ny + 1 (odd): the column pass (lanes along i) hits 32 distinct banks, not one
    const int ld = ny + 1;
    for (int t = threadIdx.x; t < nx * ld; t += blockDim.x) grid[t] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int4 q = sr[i];
        if (q.x == q.z) continue;
        const int i0 = find_s(ux, nx, q.x), i1 = find_s(ux, nx, q.z);
        const int j0 = find_s(uy, ny, q.y), j1 = find_s(uy, ny, q.w);
        atomicAdd(&grid[i0 * ld + j0], 1);
        atomicAdd(&grid[i1 * ld + j0], -1);
        atomicAdd(&grid[i0 * ld + j1], -1);
        atomicAdd(&grid[i1 * ld + j1], 1);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = warp; i < nx; i += nw) {          // prefix along j, then along i: coverage count
        int carry = 0;
        for (int j0 = 0; j0 < ny; j0 += 32) {
            const int j = j0 + lane;
            int v = j < ny ? grid[i * ld + j] : 0;
            for (int d = 1; d < 32; d <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, v, d);
                if (lane >= d) v += u;
            }
            if (j < ny) grid[i * ld + j] = carry + v;
            carry += __shfl_sync(0xffffffffu, v, 31);
        }
    }
    __syncthreads();
    for (int j = warp; j < ny; j += nw) {
        int carry = 0;
        for (int i0 = 0; i0 < nx; i0 += 32) {
            const int i = i0 + lane;
            int v = i < nx ? grid[i * ld + j] : 0;
            for (int d = 1; d < 32; d <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, v, d);
                if (lane >= d) v += u;
            }
            if (i < nx) grid[i * ld + j] = carry + v > 0 ? 1 : 0;   // union indicator
            carry += __shfl_sync(0xffffffffu, v, 31);
        }
    }
    __syncthreads();
    for (int i = warp; i < nx; i += nw)                           // mixed difference
        for (int j = lane; j < ny; j += 32) {
        const int t = i * ld + j;
        const int c00 = grid[t];
        const int cm0 = i > 0 ? grid[t - ld] : 0;
        const int c0m = j > 0 ? grid[t - 1] : 0;
        const int cmm = (i > 0 && j > 0) ? grid[t - ld - 1] : 0;
        const int wv = c00 - cm0 - c0m + cmm;
        if (wv != 0) push_raw(S, ux[i], uy[j], wv);
        }
    __syncthreads();
}

// v mod T for 0 <= v < 2^25, T <= 8192: float quotient estimate (off by at most one) + correction
__device__ __forceinline__ int32_t mod_t(int32_t v, int32_t T, float rT) {
    int32_t r = v - (int32_t)((float)v * rT) * T;
    if (r < 0) r += T;
    if (r >= T) r -= T;
    return r;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ void put(const Args &A, int64_t o, double2 v) {
    if (A.out_f32) ((float2 *)A.F)[o] = make_float2((float)v.x, (float)v.y);
    else ((double2 *)A.F)[o] = v;
}

__global__ void __launch_bounds__(kThreads, 1) k_small_clip(Args A) {
    extern __shared__ __align__(16) uint8_t dyn_raw[];
    Shared &S = *(Shared *)dyn_raw;
    uint8_t *dyn = dyn_raw + kSharedBytes;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int32_t T = A.T;
    if (tid == 0) { S.nraw = 0; S.err = 0; }
    __syncthreads();
    // ---------------- a1: raw corners
    if (A.group_ptr == nullptr) {
        for (int64_t r = tid; r < A.R; r += kThreads) {
            int4 q = A.rects[r];
            if (!rect_ok_s(q, T)) { atomicOr(&S.err, 1); continue; }
            push_raw(S, q.x, q.y, 1); push_raw(S, q.z, q.y, -1);
            push_raw(S, q.x, q.w, -1); push_raw(S, q.z, q.w, 1);
        }
    } else {
        for (int64_t g = 0; g < A.G; ++g) {
            const int64_t r0 = A.group_ptr[g], r1 = A.group_ptr[g + 1];
            const int n = (int)(r1 - r0);
            if (n <= 0) continue;
            if (n > A.mg) { if (tid == 0) atomicOr(&S.err, 2); continue; }
            group_union(S, dyn, A.rects + r0, n, T);
        }
    }
    __syncthreads();
    const int nraw = S.nraw;
    if (nraw > kMaxRaw) S.err |= 4;   // (every thread reads the same value)
    if (S.err) {
        if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0)
            *A.status = (S.err & 1) ? FCFS_E_RANGE : FCFS_E_UNSUPPORTED;
        return;
    }
    // ---------------- sort by (y, x), merge equal keys, drop zeros
    {
        uint32_t k[kItems];
        int32_t v[kItems];
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const int p = tid * kItems + i;
            k[i] = p < nraw ? S.key[p] : kSentinel;
            v[i] = p < nraw ? S.wt[p] : 0;
        }
        __syncthreads();
        const int end_bit = kKeyBits + 32 - __clz((unsigned)T);   // y bits above the 14 x bits
        if (nraw <= kThreads) {   // one key per thread (c1-size clips): the same sort, 1/kItems the work
            uint32_t k1[1] = {tid < nraw ? S.key[tid] : kSentinel};
            int32_t v1[1] = {tid < nraw ? S.wt[tid] : 0};
            __syncthreads();
            Sort1(S.cub.sort1).Sort(k1, v1, 0, end_bit);
            __syncthreads();
            S.key[tid] = k1[0]; S.wt[tid] = v1[0];
#pragma unroll
            for (int i = 1; i < kItems; ++i) { S.key[i * kThreads + tid] = kSentinel; S.wt[i * kThreads + tid] = 0; }
        } else {
            Sort(S.cub.sort).Sort(k, v, 0, end_bit);
            __syncthreads();
#pragma unroll
            for (int i = 0; i < kItems; ++i) { S.key[tid * kItems + i] = k[i]; S.wt[tid * kItems + i] = v[i]; }
        }
        __syncthreads();
        int32_t keep[kItems], tot[kItems];
        int cnt = 0;
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const int p = tid * kItems + i;
            const uint32_t kp = S.key[p];
            keep[i] = 0; tot[i] = 0;
            if (kp != kSentinel && (p == 0 || S.key[p - 1] != kp)) {   // run head: sum the run
                int32_t s = 0;
                for (int q = p; q < kMaxRaw && S.key[q] == kp; ++q) s += S.wt[q];
                tot[i] = s;
                keep[i] = s != 0;
            }
            cnt += keep[i];
        }
        int pos, total;
        Scan(S.cub.scan).ExclusiveSum(cnt, pos, total);
        long long a = 0;
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            if (!keep[i]) continue;
            const uint32_t kp = S.key[tid * kItems + i];
            const int32_t xx = (int32_t)(kp & ((1u << kKeyBits) - 1)), yy = (int32_t)(kp >> kKeyBits);
            S.cx[pos] = xx; S.cy[pos] = yy; S.cw[pos] = tot[i];
            a += (long long)tot[i] * xx * yy;
            ++pos;
        }
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) S.asum[warp] = a;
        if (tid == 0) S.K = total;
        __syncthreads();
    }
    const int K = S.K;
    long long area = 0;
    for (int i = 0; i < kThreads / 32; ++i) area += S.asum[i];
    if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
        if (A.K_out) *A.K_out = K;
        *A.status = FCFS_OK;
    }
    // ---------------- a2-a5: twiddle table (overlays the group scratch), this CTA's outputs
    double2 *tab = (double2 *)dyn;                    // (cos, sin)(2 pi v / T), v < T
    double2 *Ak = tab + T;                            // [K] A_k = w_k E(m x_k) (row m >= 1) or w_k x_k (m = 0)
    {   // two-level: E(v) = E(32 h) E(l), v = 32 h + l: T / 32 + 32 sincospi per CTA, then one complex
        // product per entry (a few ulp: far inside the FP64 contract)
        double2 *lo = Ak;                              // scratch [32 + T/32 + 1] before A is written
        double2 *hi = Ak + 32;
        const int nh = (T + 31) / 32;
        for (int i = tid; i < 32 + nh; i += kThreads) {
            const int v = i < 32 ? i : 32 * (i - 32);
            double sn, cs;
            sincospi(2.0 * (double)v / (double)T, &sn, &cs);
            (i < 32 ? lo[i] : hi[i - 32]) = make_double2(cs, sn);
        }
        __syncthreads();
        for (int v = tid; v < T; v += kThreads) {
            const double2 a = hi[v >> 5], b = lo[v & 31];
            tab[v] = make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);   // cos / sin of the sum
        }
        __syncthreads();
    }
    const int m = blockIdx.x;
    if (tid == 0) {   // output row offsets (pupil rows / dense rows)
        int32_t off = 0;
        for (int i = 0; i <= 2 * A.M; ++i) {
            S.rowoff[i] = off;
            const int c = A.layout == FCFS_LAYOUT_PUPIL ? pupil_nmax(i - A.M, A.r2, A.N) : A.N;
            off += c < 0 ? 0 : 2 * c + 1;
        }
        S.rowoff[2 * A.M + 1] = off;   // the window size (bounds checks)
    }
    __syncthreads();
    const float rT = 1.0f / (float)T;
    for (int k = tid; k < K; k += kThreads) {
        if (m == 0) {
            Ak[k] = make_double2((double)S.cw[k] * (double)S.cx[k], 0.0);
        } else {
            FCFS_DCHECK(mod_t(m * S.cx[k], T, rT) >= 0 && mod_t(m * S.cx[k], T, rT) < T);
            const double2 e = tab[mod_t(m * S.cx[k], T, rT)];
            Ak[k] = make_double2((double)S.cw[k] * e.x, -(double)S.cw[k] * e.y);   // w e^{-i theta}
        }
    }
    __syncthreads();
    const int nm = A.layout == FCFS_LAYOUT_PUPIL ? pupil_nmax(m, A.r2, A.N) : A.N;
    if (nm < 0) return;
    const bool dmask = A.layout == FCFS_LAYOUT_DENSE && A.r2 >= 0.0;
    const int n_first = m == 0 ? 0 : -nm, n_cnt = nm - n_first + 1;
    const int nb0 = (int)((int64_t)n_cnt * blockIdx.y / gridDim.y), nb1 = (int)((int64_t)n_cnt * (blockIdx.y + 1) / gridDim.y);
    const double pi = 3.141592653589793238462643383279502884;
    const int64_t op = S.rowoff[A.M + m] + nm;                                   // (m, 0)
    const int64_t on = S.rowoff[A.M - m] + (A.layout == FCFS_LAYOUT_PUPIL ? pupil_nmax(-m, A.r2, A.N) : A.N);  // (-m, 0)
    for (int t = nb0 + warp; t < nb1; t += kThreads / 32) {
        const int n = n_first + t;
        double2 s = make_double2(0.0, 0.0);
        if (n == 0) {
            if (m == 0) continue;
            for (int k = lane; k < K; k += 32) {                          // sum_k A_k y_k
                const double yk = (double)S.cy[k];
                s.x = fma(Ak[k].x, yk, s.x);
                s.y = fma(Ak[k].y, yk, s.y);
            }
        } else {
            const int32_t an = n < 0 ? -n : n;
            const double sg = n < 0 ? -1.0 : 1.0;   // E(-v) = conj E(v)
            for (int k = lane; k < K; k += 32) {
                FCFS_DCHECK(mod_t(an * S.cy[k], T, rT) >= 0 && mod_t(an * S.cy[k], T, rT) < T);
                double2 e = tab[mod_t(an * S.cy[k], T, rT)];
                e.y *= sg;
                s = make_double2(fma(Ak[k].x, e.x, fma(Ak[k].y, e.y, s.x)),   // A * (c - i s)
                                 fma(Ak[k].y, e.x, fma(-Ak[k].x, e.y, s.y)));
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
            s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
        }
        if (lane != 0) continue;
        double2 f;
        if (m == 0) {                      // F[0, n] = i S / (2 pi n T)
            const double d = 2.0 * pi * (double)n * (double)T;
            f = make_double2(-s.y / d, s.x / d);
        } else if (n == 0) {               // F[m, 0] = i S_ax / (2 pi m T)
            const double d = 2.0 * pi * (double)m * (double)T;
            f = make_double2(-s.y / d, s.x / d);
        } else {                           // F = -S / (4 pi^2 m n)
            const double d = -4.0 * pi * pi * (double)m * (double)n;
            f = make_double2(s.x / d, s.y / d);
        }
        if (dmask && (double)m * m + (double)n * n > A.r2) f = make_double2(0.0, 0.0);
        FCFS_DCHECK(op + n >= 0 && on - n >= 0 && op + n < S.rowoff[2 * A.M + 1] && on - n < S.rowoff[2 * A.M + 1]);
        put(A, op + n, f);
        put(A, on - n, make_double2(f.x, -f.y));   // F[-m, -n] = conj F[m, n]
    }
    if (m == 0 && blockIdx.y == 0 && tid == 0) {  // DC (Eq. Fdc)
        const double dc = (double)area / ((double)T * (double)T);
        put(A, op, make_double2(dc, 0.0));
    }
}

}  // namespace sm

size_t small_clip_smem_bytes(int32_t T, int64_t max_group) {
    const int64_t mg = max_group < 1 ? 1 : max_group;
    const size_t scratch = sizeof(int4) * sm::kMaxGroup + sizeof(int32_t) * 10 * sm::kMaxGroup +
                           sizeof(int32_t) * (size_t)(2 * mg) * (size_t)(2 * mg + 1);
    const size_t table = sizeof(double2) * ((size_t)T + sm::kMaxRaw);
    return sm::kSharedBytes + (scratch > table ? scratch : table);
}

bool small_clip_eligible(int64_t R, int64_t G, int32_t T, int64_t max_group, int32_t M, int32_t N, bool grouped) {
    if (T > sm::kMaxT || M > 63 || N > sm::kMaxN || max_group > sm::kMaxGroup) return false;
    if (!grouped && 4 * R > sm::kMaxRaw) return false;
    if (grouped && R > 4 * sm::kMaxRaw) return false;
    return small_clip_smem_bytes(T, max_group) <= 227 * 1024;
}

fcfs_status launch_small_clip(const int32_t *rects, int64_t R, const int64_t *group_ptr, int64_t G, int32_t T,
                              int64_t max_group, const fcfs_window &win, int32_t out_f32, void *F, int64_t *K_dev,
                              int32_t *status_dev, cudaStream_t s) {
    sm::Args a{};
    a.rects = (const int4 *)rects;
    a.R = R; a.group_ptr = group_ptr; a.G = G; a.T = T;
    a.M = win.M; a.N = win.N; a.layout = win.layout; a.r2 = win.pupil_r2;
    a.mg = (int32_t)(max_group < 1 ? 1 : max_group);
    a.out_f32 = out_f32; a.F = F; a.K_out = K_dev; a.status = status_dev;
    const size_t smem = small_clip_smem_bytes(T, max_group);
    FCFS_TRY(ensure_smem((const void *)sm::k_small_clip, smem));
    dim3 grid((unsigned)(win.M + 1), sm::kNBlk);
    sm::k_small_clip<<<grid, sm::kThreads, smem, s>>>(a);
    FCFS_CHECK_LAUNCH("k_small_clip");
    return FCFS_OK;
}

}  // namespace fcfs

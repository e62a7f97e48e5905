// fft_route.cu — SURVEY §8(f) NEXT-2: the lattice-FFT route for one clip in FP64.
//
// Step 4 of the paper evaluates the interior coefficients as DFTs of the sparse image f~_xy
// (P:890-904).  The vertices lie on the integer lattice, so along y these are length-T
// DFTs, which the paper's TD-FFT route does with FFTs.  For a window
// |n| <= N this route computes, per row |m|:
//
//   G[m, y] = sum_{k: y_k = y (mod T)} w_k e^{-2 pi i m x_k / T}          (row sums over the corners)
//   S[m, n] = sum_y G[m, y] e^{-2 pi i n y / T}                           (length-T DFT along y)
//           = sum_{y1 < T1} e^{-2 pi i n y1 / T} Z_{y1}[n mod T2],  Z_{y1} = DFT_T2(G[m, y1 + T1 y2])
//
// with T = T1 T2 and T2 >= 2N+1 (an output-pruned two-step split: distinct n stay distinct mod T2),
// i.e. T1 FFTs of length T2 and (2N+1) T1 twiddled adds per row, instead of the 2N R MACs per row of
// the row-bucket GEMM (R = distinct rows, about T on configs[3] / [4]).  Then (Prop. 3)
//
//   F[m, n] = -S[m, n] / (4 pi^2 m n)                                     (Eq. Fkl, alpha case 4)
//   F[m, 0] = i / (2 pi m T) * sum_k w_k y_k e^{-2 pi i m x_k / T}        (Eq. Fk0; raw y_k: a corner
//             at y = T counts with T although its phase wraps to 0, reading A7)
//   F[0, n] = i / (2 pi n T) * DFT(G0)[n],  G0[y] = sum_{k: y_k = y} w_k x_k   (Eq. F0l)
//   F[0, 0] = area / T^2,  F[-m, -n] = conj F[m, n] (bitwise).
//
// Kernels: k_fr_yptr (CSR of the y-sorted corner list over y, sortedness flag), k_fr_table (the
// two-level e^{-2 pi i p / T} table), k_fr_row0 / k_fr_rows (G, thread = one y and 16 consecutive m:
// two exact-phase lookups per corner and the angle-addition recurrence over 16 m; written in the
// [row][y1][y2] order the FFT reads), k_fr_fft2 (CTA per (row, range of sub-rows), 2 CTAs / SM: each
// sub-row arrives by a TMA bulk copy into one padded shared buffer, is transformed in place by Stockham
// passes (radix 2/4/8 lead, then radix 16), and the outer twiddled sum accumulates X[n] in shared memory)
// and k_fr_epilogue (window / pupil / rows, axes, DC, mirror).
// Error (FP64): the FFT's is ~log2(T2) u ||G||_2 per output and ||G|| <= sum |w| (the L1 bound B up
// to the 1/(4 pi^2 m n) factor), far inside 1e-12 B.
#include <cstdlib>
#include <cstring>

#include "coeff.cuh"

namespace fcfs {
namespace fr {

constexpr int kThreads = 256;
constexpr int kRowsPerThread = 16;  // consecutive m per k_fr_rows thread (recurrence length)
constexpr int kMaxT2 = 4096;

struct Geo {
    int32_t T, T1, T2;
    int32_t t1bits, t2bits;
    int32_t lbits, nhi;     // two-level table of T: hi[p >> lbits] * lo[p & (2^lbits - 1)]
    int32_t b2, nhi2;       // two-level table of T2
};

// complex arithmetic on double2 (FP64 route) and float2 (FP32 route of the split precisions)
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }   // a * (-i)
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }

template <class V> struct Cx;
template <> struct Cx<double2> {
    using S = double;
    static __device__ __forceinline__ double2 mk(double a, double b) { return make_double2(a, b); }
};
template <> struct Cx<float2> {
    using S = float;
    static __device__ __forceinline__ float2 mk(double a, double b) { return make_float2((float)a, (float)b); }
};
template <class V>
__device__ __forceinline__ double2 to_d(V a) { return make_double2((double)a.x, (double)a.y); }

// e^{-2 pi i p / T} from a two-level table holding e^{-2 pi i j / T} (already conjugated)
template <class V>
__device__ __forceinline__ V tw_ldg(const V *tab, uint32_t p, int lbits, int nhi) {
    return cmul(__ldg(tab + (p >> lbits)), __ldg(tab + nhi + (p & ((1u << lbits) - 1u))));
}
template <class V>
__device__ __forceinline__ V tw_smem(const V *tab, uint32_t p, int lbits, int nhi) {
    return cmul(tab[p >> lbits], tab[nhi + (p & ((1u << lbits) - 1u))]);
}

// two-level table of e^{-2 pi i j / L}: entries [0, nhi) = hi steps (j << lbits), [nhi, nhi + 2^lbits) = lo
// (FP64 sincospi, rounded once to the route's precision)
template <class V>
__device__ __forceinline__ V tw_entry(int i, int L, int lbits, int nhi) {
    const int64_t j = i < nhi ? ((int64_t)i << lbits) : (int64_t)(i - nhi);
    double s, c;
    sincospi(2.0 * (double)j / (double)L, &s, &c);
    return Cx<V>::mk(c, -s);
}

template <class V>
__global__ void k_fr_table(V *tab, Geo g) {
    const int n = g.nhi + (1 << g.lbits);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        tab[i] = tw_entry<V>(i, g.T, g.lbits, g.nhi);
}

// yptr[v] = #corners in [k_lo, k_hi) with y < v, v in [0, T+1]; flag = 1 if y decreases somewhere.
// K_dev != NULL: the corner count comes from device memory (the sync-free path; K <= the planned cap)
__global__ void k_fr_yptr(const int32_t *__restrict__ y, int64_t k_lo, int64_t K, int32_t T, int32_t *yptr,
                          int32_t *flag, const int64_t *K_dev) {
    if (K_dev) K = *K_dev;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= (int64_t)T + 1; v += stride) {
        int64_t lo = 0, hi = K;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (y[k_lo + mid] < v) lo = mid + 1; else hi = mid;
        }
        yptr[v] = (int32_t)lo;
    }
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1; k < K; k += stride)
        if (y[k_lo + k] < y[k_lo + k - 1]) *flag = 1;
}

// Load balance of the row-sum kernels: within each sub-row y1 the T2 columns y2 (y = y1 + T1 y2) are
// stored in decreasing order of their corner-run length, so the 32 lanes of a warp get runs of about
// the same length (the y runs of the configs are uneven: a warp of 32 consecutive y2 idles ~45% of its
// lanes).  perm[y1 T2 + pos] = y2 and pinv[y1 T2 + y2] = pos (int16: T2 <= 4096); the FFT reads each
// sub-row back in y2 order through pinv.  G[m, y] does not depend on the thread that computes it, so
// the order changes no result bit (counting sort by run length with shared atomics, not stable).
__global__ void __launch_bounds__(kThreads)
k_fr_perm(const int32_t *__restrict__ yptr, Geo g, int16_t *perm, int16_t *pinv) {
    constexpr int kBins = 64;   // run lengths >= 63 share the first bin
    __shared__ int32_t cnt[kBins];
    const int y1 = blockIdx.x;
    if (threadIdx.x < kBins) cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int y2 = threadIdx.x; y2 < g.T2; y2 += kThreads) {
        const int32_t y = y1 + (y2 << g.t1bits);
        const int len = yptr[y + 1] - yptr[y];
        atomicAdd(&cnt[kBins - 1 - min(len, kBins - 1)], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int b = 0; b < kBins; ++b) { const int c = cnt[b]; cnt[b] = run; run += c; }
    }
    __syncthreads();
    for (int y2 = threadIdx.x; y2 < g.T2; y2 += kThreads) {
        const int32_t y = y1 + (y2 << g.t1bits);
        const int len = yptr[y + 1] - yptr[y];
        const int pos = atomicAdd(&cnt[kBins - 1 - min(len, kBins - 1)], 1);
        perm[(int64_t)y1 * g.T2 + pos] = (int16_t)y2;
        pinv[(int64_t)y1 * g.T2 + y2] = (int16_t)pos;
    }
}

// y of storage index t = y1 T2 + pos (pos = the permuted column of sub-row y1): y = y1 + T1 perm[t]
__device__ __forceinline__ int32_t y_of(int64_t t, const Geo &g, const int16_t *__restrict__ perm) {
    return (int32_t)((t >> g.t2bits) + ((int32_t)(uint16_t)__ldg(perm + t) << g.t1bits));
}

// the x-weighted row G0[y] = sum_{y_k = y mod T} w_k x_k (exact integer sum), as complex (row 0); the
// y = T run is added by k_fr_row0T
template <class V>
__global__ void k_fr_row0(const int32_t *__restrict__ x, const int32_t *__restrict__ w, int64_t k_lo,
                          const int32_t *__restrict__ yptr, const int16_t *__restrict__ perm, Geo g, V *Gd) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < g.T; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t yv = y_of(t, g, perm);
        long long s = 0;
        for (int32_t k = yptr[yv]; k < yptr[yv + 1]; ++k) s += (long long)w[k_lo + k] * x[k_lo + k];
        Gd[t] = Cx<V>::mk((double)s, 0.0);
    }
}

// one block: the y = T run's sum of w x (exact, int64) added into G0 at y = 0 (storage slot pinv[0]);
// the run holds thousands of corners on the configs (lines clipped at the tile edge)
template <class V>
__global__ void __launch_bounds__(kThreads)
k_fr_row0T(const int32_t *__restrict__ x, const int32_t *__restrict__ w, int64_t k_lo,
           const int32_t *__restrict__ yptr, const int16_t *__restrict__ pinv, Geo g, V *Gd) {
    __shared__ long long red[kThreads / 32];
    long long s = 0;
    for (int32_t k = yptr[g.T] + (int32_t)threadIdx.x; k < yptr[g.T + 1]; k += kThreads)
        s += (long long)w[k_lo + k] * x[k_lo + k];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long a = 0;
        for (int i = 0; i < kThreads / 32; ++i) a += red[i];
        const int64_t t0 = (uint16_t)pinv[0];
        const V v = Gd[t0];
        // both integers below 2^53: the FP64 sum is exact (FP32 route: rounded once)
        Gd[t0] = Cx<V>::mk((double)v.x + (double)a, 0.0);
    }
}

// rows m = m0 .. m0+15 (m0 = m_first + 16 blockIdx.y, up to m_last) of G, written to Gd rows
// row_off + 16 blockIdx.y + j.  Two corners per iteration (independent recurrence chains).
template <class V>
__global__ void __launch_bounds__(kThreads, sizeof(V) == 16 ? 2 : 3)
k_fr_rows(const int32_t *__restrict__ x, const int32_t *__restrict__ w, int64_t k_lo,
          const int32_t *__restrict__ yptr, const int16_t *__restrict__ perm, const V *__restrict__ tab, Geo g,
          int32_t m_first, int32_t m_last, int32_t row_off, V *Gd) {
    using S = typename Cx<V>::S;
    // the two-level table in shared memory (<= 32 KB): its lookups are the kernel's latency chain
    extern __shared__ __align__(16) unsigned char fr_rows_smem[];
    V *stab = (V *)fr_rows_smem;
    for (int i = threadIdx.x; i < g.nhi + (1 << g.lbits); i += blockDim.x) stab[i] = tab[i];
    __syncthreads();
    const int32_t m0 = m_first + kRowsPerThread * (int32_t)blockIdx.y;
    const uint32_t mask = (uint32_t)g.T - 1u;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < g.T; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t yv = y_of(t, g, perm);
        V acc[kRowsPerThread];
#pragma unroll
        for (int j = 0; j < kRowsPerThread; ++j) acc[j] = Cx<V>::mk(0.0, 0.0);
        auto run = [&](int32_t k0, int32_t k1) {
            int32_t k = k0;
            // corner coordinates / weights one pair ahead (their loads overlap the current pair's math)
            uint32_t nxa = 0, nxb = 0;
            int32_t nwa = 0, nwb = 0;
            if (k + 1 < k1) {
                nxa = (uint32_t)__ldg(x + k_lo + k); nxb = (uint32_t)__ldg(x + k_lo + k + 1);
                nwa = __ldg(w + k_lo + k); nwb = __ldg(w + k_lo + k + 1);
            }
            for (; k + 1 < k1; k += 2) {
                const uint32_t xa = nxa, xb = nxb;
                const S wa = (S)nwa, wb = (S)nwb;
                if (k + 3 < k1) {
                    nxa = (uint32_t)__ldg(x + k_lo + k + 2); nxb = (uint32_t)__ldg(x + k_lo + k + 3);
                    nwa = __ldg(w + k_lo + k + 2); nwb = __ldg(w + k_lo + k + 3);
                }
                V ea = tw_smem(stab, ((uint32_t)m0 * xa) & mask, g.lbits, g.nhi);
                V eb = tw_smem(stab, ((uint32_t)m0 * xb) & mask, g.lbits, g.nhi);
                if constexpr (sizeof(S) == 8) {
                    // FP64: the second-order recurrence E_{m+1} = 2 cos(theta) E_m - E_{m-1} (2 FMA per step
                    // instead of a complex multiply's 4); its error grows as ~m^2/2 ulp: < 130 ulp over 16 rows
                    V pa = tw_smem(stab, ((uint32_t)(m0 + 1) * xa) & mask, g.lbits, g.nhi);
                    V pb = tw_smem(stab, ((uint32_t)(m0 + 1) * xb) & mask, g.lbits, g.nhi);
                    const S ta = 2 * fma(pa.x, ea.x, pa.y * ea.y), tb = 2 * fma(pb.x, eb.x, pb.y * eb.y);   // 2 Re(E_{m+1} conj E_m)
                    acc[0].x = fma(wa, ea.x, fma(wb, eb.x, acc[0].x));
                    acc[0].y = fma(wa, ea.y, fma(wb, eb.y, acc[0].y));
                    acc[1].x = fma(wa, pa.x, fma(wb, pb.x, acc[1].x));
                    acc[1].y = fma(wa, pa.y, fma(wb, pb.y, acc[1].y));
#pragma unroll
                    for (int j = 2; j < kRowsPerThread; ++j) {
                        const V na = Cx<V>::mk(fma(ta, pa.x, -ea.x), fma(ta, pa.y, -ea.y));
                        const V nb = Cx<V>::mk(fma(tb, pb.x, -eb.x), fma(tb, pb.y, -eb.y));
                        ea = pa; pa = na; eb = pb; pb = nb;
                        acc[j].x = fma(wa, pa.x, fma(wb, pb.x, acc[j].x));
                        acc[j].y = fma(wa, pa.y, fma(wb, pb.y, acc[j].y));
                    }
                } else {
                    const V sa = tw_smem(stab, xa & mask, g.lbits, g.nhi), sb = tw_smem(stab, xb & mask, g.lbits, g.nhi);
#pragma unroll
                    for (int j = 0; j < kRowsPerThread; ++j) {
                        if (j) { ea = cmul(ea, sa); eb = cmul(eb, sb); }
                        acc[j].x = fma(wa, ea.x, fma(wb, eb.x, acc[j].x));
                        acc[j].y = fma(wa, ea.y, fma(wb, eb.y, acc[j].y));
                    }
                }
            }
            if (k < k1) {
                const uint32_t xa = (uint32_t)__ldg(x + k_lo + k);
                const S wa = (S)__ldg(w + k_lo + k);
                V ea = tw_smem(stab, ((uint32_t)m0 * xa) & mask, g.lbits, g.nhi);
                const V sa = tw_smem(stab, xa & mask, g.lbits, g.nhi);
#pragma unroll
                for (int j = 0; j < kRowsPerThread; ++j) {
                    if (j) ea = cmul(ea, sa);
                    acc[j].x = fma(wa, ea.x, acc[j].x);
                    acc[j].y = fma(wa, ea.y, acc[j].y);
                }
            }
        };
        FCFS_DCHECK(yv >= 0 && yv < g.T && yptr[yv] <= yptr[yv + 1]);
        run(yptr[yv], yptr[yv + 1]);   // the y = T run (phase of row 0) is added by k_fr_rowsT
#pragma unroll
        for (int j = 0; j < kRowsPerThread; ++j) {
            if (m0 + j > m_last) break;
            Gd[(row_off + kRowsPerThread * (int64_t)blockIdx.y + j) * g.T + t] = acc[j];
        }
    }
}

// the y = T run (its phase wraps to row y = 0; the axis sum weights it with T): block per 16 rows,
// threads over the run's corners (the run can hold thousands of corners: the lines clipped at the
// tile edge), block reduction; GT[row] = its share, added into G[m, 0]
template <class V>
__global__ void __launch_bounds__(kThreads)
k_fr_rowsT(const int32_t *__restrict__ x, const int32_t *__restrict__ w, int64_t k_lo,
           const int32_t *__restrict__ yptr, const int16_t *__restrict__ pinv, const V *__restrict__ tab, Geo g,
           int32_t m_first, int32_t m_last, int32_t row_off, V *Gd, double2 *GT) {
    using S = typename Cx<V>::S;
    __shared__ V red[kThreads / 32][kRowsPerThread];
    const int32_t m0 = m_first + kRowsPerThread * (int32_t)blockIdx.x;
    const uint32_t mask = (uint32_t)g.T - 1u;
    V acc[kRowsPerThread];
#pragma unroll
    for (int j = 0; j < kRowsPerThread; ++j) acc[j] = Cx<V>::mk(0.0, 0.0);
    for (int32_t k = yptr[g.T] + (int32_t)threadIdx.x; k < yptr[g.T + 1]; k += kThreads) {
        const uint32_t xa = (uint32_t)x[k_lo + k];
        const S wa = (S)w[k_lo + k];
        V e = tw_ldg(tab, ((uint32_t)m0 * xa) & mask, g.lbits, g.nhi);
        const V st = tw_ldg(tab, xa & mask, g.lbits, g.nhi);
#pragma unroll
        for (int j = 0; j < kRowsPerThread; ++j) {
            if (j) e = cmul(e, st);
            acc[j].x = fma(wa, e.x, acc[j].x);
            acc[j].y = fma(wa, e.y, acc[j].y);
        }
    }
#pragma unroll
    for (int j = 0; j < kRowsPerThread; ++j) {
        for (int o = 16; o > 0; o >>= 1) {
            acc[j].x += __shfl_xor_sync(0xffffffffu, acc[j].x, o);
            acc[j].y += __shfl_xor_sync(0xffffffffu, acc[j].y, o);
        }
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][j] = acc[j];
    }
    __syncthreads();
    const int j = threadIdx.x;
    if (j < kRowsPerThread && m0 + j <= m_last) {
        V a = Cx<V>::mk(0.0, 0.0);
        for (int i = 0; i < kThreads / 32; ++i) a = cadd(a, red[i][j]);
        const int64_t row = row_off + kRowsPerThread * (int64_t)blockIdx.x + j;
        GT[row] = to_d(a);
        const int64_t t0 = (uint16_t)pinv[0];   // storage slot of y = 0
        Gd[row * g.T + t0] = cadd(Gd[row * g.T + t0], a);
    }
}

// ---------------------------------------------------------------- the per-row FFT

template <class V>
__device__ __forceinline__ V w16(int q) {   // e^{-2 pi i q / 16}, q in [0, 8)
    const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, h = 0.70710678118654752440;
    switch (q) {
        case 0: return Cx<V>::mk(1.0, 0.0);
        case 1: return Cx<V>::mk(c1, -s1);
        case 2: return Cx<V>::mk(h, -h);
        case 3: return Cx<V>::mk(s1, -c1);
        case 4: return Cx<V>::mk(0.0, -1.0);
        case 5: return Cx<V>::mk(-s1, -c1);
        case 6: return Cx<V>::mk(-h, -h);
        default: return Cx<V>::mk(-c1, -s1);
    }
}

// radix-4 butterfly in place: (a0..a3) -> DFT_4
template <class V>
__device__ __forceinline__ void bfly4(V &a0, V &a1, V &a2, V &a3) {
    const V b0 = cadd(a0, a2), b1 = csub(a0, a2), b2 = cadd(a1, a3), b3 = mul_mi(csub(a1, a3));
    a0 = cadd(b0, b2); a2 = csub(b0, b2); a1 = cadd(b1, b3); a3 = csub(b1, b3);
}

// in-register DFT of size R (natural order in and out): R = 2, 4, or the four-step split
// R = 4 x 4 (16) / 2 x 4 (8) with the W_R^{r0 k1} twiddles as constants
template <int R, class V>
__device__ __forceinline__ void dft(V (&v)[R]) {
    if constexpr (R == 2) {
        const V a = v[0];
        v[0] = cadd(a, v[1]); v[1] = csub(a, v[1]);
    } else if constexpr (R == 4) {
        bfly4(v[0], v[1], v[2], v[3]);
    } else if constexpr (R == 8) {
        // x[r0 + 2 r1]: DFT_4 over r1 for r0 = 0, 1; twiddle W8^{r0 k1}; DFT_2 over r0
        V e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
        bfly4(e[0], e[1], e[2], e[3]);
        bfly4(o[0], o[1], o[2], o[3]);
        o[1] = cmul(o[1], w16<V>(2)); o[2] = mul_mi(o[2]); o[3] = cmul(o[3], w16<V>(6));
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) { v[k1] = cadd(e[k1], o[k1]); v[k1 + 4] = csub(e[k1], o[k1]); }
    } else {
        static_assert(R == 16, "radix");
        // x[r0 + 4 r1]: DFT_4 over r1 for each r0; twiddle W16^{r0 k1}; DFT_4 over r0 -> X[k1 + 4 k2]
        V y[4][4];
#pragma unroll
        for (int r0 = 0; r0 < 4; ++r0) {
            y[r0][0] = v[r0]; y[r0][1] = v[r0 + 4]; y[r0][2] = v[r0 + 8]; y[r0][3] = v[r0 + 12];
            bfly4(y[r0][0], y[r0][1], y[r0][2], y[r0][3]);
        }
        y[1][1] = cmul(y[1][1], w16<V>(1)); y[1][2] = cmul(y[1][2], w16<V>(2)); y[1][3] = cmul(y[1][3], w16<V>(3));
        y[2][1] = cmul(y[2][1], w16<V>(2)); y[2][2] = mul_mi(y[2][2]);            y[2][3] = cmul(y[2][3], w16<V>(6));
        y[3][1] = cmul(y[3][1], w16<V>(3)); y[3][2] = cmul(y[3][2], w16<V>(6));
        const V w9 = w16<V>(1);
        y[3][3] = cmul(y[3][3], Cx<V>::mk(-(double)w9.x, -(double)w9.y));       // W16^9 = -W16^1
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            bfly4(y[0][k1], y[1][k1], y[2][k1], y[3][k1]);
            v[k1] = y[0][k1]; v[k1 + 4] = y[1][k1]; v[k1 + 8] = y[2][k1]; v[k1 + 12] = y[3][k1];
        }
    }
}

// shared-memory FFT buffers hold element i at i + i/16 (one pad slot per 16): the first pass's
// radix-16 stores (stride 16 elements) then fall on distinct banks; the TMA-filled input is unpadded
__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// In-place Stockham pass (all reads, barrier, all writes) of radix R over length L <= R * kThreads;
// the first pass (Ns == 1) reads the unpadded TMA layout and accumulates sum_y y G[y] (axis)
template <int R, class V>
__device__ __forceinline__ void pass_inplace(V *buf, int L, int Ns, const V *tw2, const Geo &g, int y1,
                                             double2 &ax, const int16_t *pv) {
    const int nb = L / R;
    const int i = threadIdx.x;
    V v[R];
    const int k = i & (Ns - 1);
    if (i < nb) {   // read and transform; the barrier orders every read before any write
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = buf[Ns == 1 ? (int)(uint16_t)pv[i + r * nb] : pad(i + r * nb)];
        if (Ns == 1) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double yy = (double)(y1 + ((i + r * nb) << g.t1bits));
                ax.x = fma(yy, (double)v[r].x, ax.x); ax.y = fma(yy, (double)v[r].y, ax.y);
            }
        } else {
            const V w1 = tw_smem(tw2, (uint32_t)(k * (L / (Ns * R))), g.b2, g.nhi2);
            if constexpr (R == 16) {
                // powers by a tree of depth 4 (w2 = w1^2, w4 = w2^2, w8 = w4^2; w_r = w_{r & 8} w_{r & 4} ...)
                // instead of a chain of 14 dependent products
                const V w2 = cmul(w1, w1);
                const V w3 = cmul(w2, w1);
                const V w4 = cmul(w2, w2);
                const V w8 = cmul(w4, w4);
                v[1] = cmul(v[1], w1); v[2] = cmul(v[2], w2); v[3] = cmul(v[3], w3); v[4] = cmul(v[4], w4);
                v[8] = cmul(v[8], w8);
                v[5] = cmul(v[5], cmul(w4, w1)); v[6] = cmul(v[6], cmul(w4, w2)); v[7] = cmul(v[7], cmul(w4, w3));
                const V w12 = cmul(w8, w4);
                v[9] = cmul(v[9], cmul(w8, w1)); v[10] = cmul(v[10], cmul(w8, w2)); v[11] = cmul(v[11], cmul(w8, w3));
                v[12] = cmul(v[12], w12);
                v[13] = cmul(v[13], cmul(w12, w1)); v[14] = cmul(v[14], cmul(w12, w2)); v[15] = cmul(v[15], cmul(w12, w3));
            } else {
                V wr = w1;
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    v[r] = cmul(v[r], wr);
                    if (r + 1 < R) wr = cmul(wr, w1);
                }
            }
        }
        dft<R>(v);
    }
    __syncthreads();
    if (i < nb) {
        const int j = (i - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) buf[pad(j + r * Ns)] = v[r];
    }
    __syncthreads();
}

// CTA per (row, sub-row range blockIdx.y of gridDim.y) (2 CTAs / SM): one padded work buffer that the TMA bulk copy fills with the next
// sub-row and the passes transform in place; X[n] accumulates in shared memory
template <class V>
__global__ void __launch_bounds__(kThreads, 2)
k_fr_fft2(const V *__restrict__ Gd, const double2 *__restrict__ GT, const V *__restrict__ tabT,
          const int16_t *__restrict__ pinv, Geo g, int32_t N, int32_t r_first, int32_t nr, double2 *Xs,
          double2 *Axis) {
    extern __shared__ __align__(16) unsigned char fsm_raw[];
    const int LP = g.T2 + g.T2 / 16;
    const int nn = 2 * N + 1;
    // [buf: LP x V][X: nn x double2 (the outer sum in FP64 for both routes)][tw2: V][pinv row: T2 x int16]
    V *buf = (V *)fsm_raw;
    double2 *X = (double2 *)(fsm_raw + (size_t)LP * sizeof(V));
    V *tw2 = (V *)(X + nn);
    int16_t *pv = (int16_t *)(tw2 + g.nhi2 + (1 << g.b2));
    __shared__ __align__(8) unsigned long long bar;
    __shared__ double2 red[kThreads / 32];
    const int r = blockIdx.x;
    const V *grow = Gd + (int64_t)r * g.T;
    const int ntw = g.nhi2 + (1 << g.b2);
    for (int i = threadIdx.x; i < ntw; i += kThreads) tw2[i] = tw_entry<V>(i, g.T2, g.b2, g.nhi2);
    for (int o = threadIdx.x; o < nn; o += kThreads) X[o] = make_double2(0.0, 0.0);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t bytes = (uint32_t)(g.T2 * sizeof(V)), pbytes = (uint32_t)g.T2 * 2u;
    FCFS_DCHECK(((su32(buf) | su32(pv)) & 15u) == 0 && (bytes & 15u) == 0 && (pbytes & 15u) == 0);
    double2 ax = make_double2(0.0, 0.0);
    const uint32_t maskT = (uint32_t)g.T - 1u;
    const int lead = g.t2bits & 3;
    const int ya = (int)((int64_t)g.T1 * blockIdx.y / gridDim.y), yb = (int)((int64_t)g.T1 * (blockIdx.y + 1) / gridDim.y);
    for (int y1 = ya; y1 < yb; ++y1) {
        if (threadIdx.x == 0) {
            const uint32_t b = su32(&bar);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes + pbytes)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(buf)), "l"(grow + (int64_t)y1 * g.T2), "r"(bytes), "r"(b)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(pv)), "l"(pinv + (int64_t)y1 * g.T2), "r"(pbytes), "r"(b)
                         : "memory");
        }
        {
            const uint32_t b = su32(&bar), par = (uint32_t)((y1 - ya) & 1);
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                             " selp.u32 %0, 1, 0, p;\n}"
                             : "=r"(ok) : "r"(b), "r"(par) : "memory");
        }
        int Ns = 1;
        if (lead == 1) { pass_inplace<2>(buf, g.T2, Ns, tw2, g, y1, ax, pv); Ns = 2; }
        else if (lead == 2) { pass_inplace<4>(buf, g.T2, Ns, tw2, g, y1, ax, pv); Ns = 4; }
        else if (lead == 3) { pass_inplace<8>(buf, g.T2, Ns, tw2, g, y1, ax, pv); Ns = 8; }
        for (; Ns < g.T2; Ns <<= 4) pass_inplace<16>(buf, g.T2, Ns, tw2, g, y1, ax, pv);
        // outer step: X[n] += e^{-2 pi i n y1 / T} Z[n mod T2]
        if constexpr (sizeof(typename Cx<V>::S) == 8) {
            // FP64: a thread's outputs are kThreads apart: its first twiddle from the table (exact integer
            // phase), the rest by the step e^{-2 pi i kThreads y1 / T} (<= 16 products: error ~16 u)
            const int o0 = threadIdx.x;
            V e = tw_ldg(tabT, ((uint32_t)(o0 - N + g.T) * (uint32_t)y1) & maskT, g.lbits, g.nhi);
            const V step = tw_ldg(tabT, ((uint32_t)kThreads * (uint32_t)y1) & maskT, g.lbits, g.nhi);
            for (int o = o0; o < nn; o += kThreads) {
                const int n = o - N;
                FCFS_DCHECK(pad(n >= 0 ? n : n + g.T2) < LP && (n >= 0 ? n : n + g.T2) < g.T2);
                const V z = buf[pad(n >= 0 ? n : n + g.T2)];
                X[o] = cadd(X[o], to_d(cmul(e, z)));
                e = cmul(e, step);
            }
        } else
        // FP32 route: every twiddle from the table (a recurrence in FP32 would spend the split contract's
        // error budget)
        for (int o = threadIdx.x; o < nn; o += kThreads) {
            const int n = o - N;
            FCFS_DCHECK(pad(n >= 0 ? n : n + g.T2) < LP && (n >= 0 ? n : n + g.T2) < g.T2);
            const V z = buf[pad(n >= 0 ? n : n + g.T2)];
            const uint32_t ph = ((uint32_t)(n + g.T) * (uint32_t)y1) & maskT;
            X[o] = cadd(X[o], to_d(cmul(tw_ldg(tabT, ph, g.lbits, g.nhi), z)));
        }

        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
    }
    const int64_t rg = (int64_t)blockIdx.y * nr + r_first + r;   // partial of range blockIdx.y
    for (int o = threadIdx.x; o < nn; o += kThreads) Xs[rg * nn + o] = X[o];
    for (int o = 16; o > 0; o >>= 1) {
        ax.x += __shfl_xor_sync(0xffffffffu, ax.x, o);
        ax.y += __shfl_xor_sync(0xffffffffu, ax.y, o);
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ax;
    __syncthreads();
    if (threadIdx.x == 0) {
        double2 a = make_double2(0.0, 0.0);
        for (int i = 0; i < kThreads / 32; ++i) a = cadd(a, red[i]);
        const double2 gt = blockIdx.y == 0 ? GT[r] : make_double2(0.0, 0.0);
        Axis[rg] = make_double2(fma((double)g.T, gt.x, a.x), fma((double)g.T, gt.y, a.y));
    }
}

// outputs of rows m in [m_lo, m_hi]: grid.x = rows; Xs row of |m|: 0 -> row 0 (if present), else
// row0 + (|m| - mA); each row is the sum of the sp sub-row-range partials
__device__ __forceinline__ double2 psum(const double2 *__restrict__ a, int64_t i, int64_t stride, int sp) {
    double2 v = a[i];
    for (int q = 1; q < sp; ++q) v = cadd(v, a[i + q * stride]);   // fixed order: deterministic
    return v;
}

__global__ void k_fr_epilogue(const double2 *__restrict__ Xs, const double2 *__restrict__ Axis, EpiArgs ea,
                              int32_t row0, int32_t mA, int32_t nr, int32_t sp, void *F) {
    const int m = ea.m_lo + (int)blockIdx.x;
    if (m > ea.m_hi) return;
    const double pi = 3.141592653589793238462643383279502884;
    const int64_t area = ea.area_dev ? ea.area_dev[0] : ea.area_host;
    const double dc = (double)area / ((double)ea.T * (double)ea.T);
    const int nn = 2 * ea.N + 1;
    int64_t off;
    int nlo, nhi;
    if (ea.layout == FCFS_LAYOUT_PUPIL) {
        off = 0;
        for (int mm = -ea.M; mm < m; ++mm) {
            const int c = pupil_nmax(mm, ea.r2, ea.N);
            off += c < 0 ? 0 : 2 * c + 1;
        }
        const int c = pupil_nmax(m, ea.r2, ea.N);
        if (c < 0) return;
        nlo = -c; nhi = c;
    } else {
        off = (int64_t)(m - ea.m_lo) * nn;
        nlo = -ea.N; nhi = ea.N;
    }
    for (int n = nlo + (int)threadIdx.x; n <= nhi; n += blockDim.x) {
        double2 v = make_double2(0.0, 0.0);
        const bool keep = !(ea.layout == FCFS_LAYOUT_DENSE && ea.r2 >= 0.0 &&
                            (double)m * (double)m + (double)n * (double)n > ea.r2);
        if (keep) {
            if (m == 0 && n == 0) {
                v = make_double2(dc, 0.0);
            } else {
                int mp = m, np = n;
                const bool neg = (m < 0) || (m == 0 && n < 0);
                if (neg) { mp = -m; np = -n; }
                double re, im;
                if (mp == 0) {              // F[0, n] = i S0[n] / (2 pi n T)
                    const double2 s = psum(Xs, np + ea.N, (int64_t)nr * nn, sp);
                    const double d = 2.0 * pi * (double)np * (double)ea.T;
                    re = -s.y / d; im = s.x / d;
                } else {
                    const int64_t row = row0 + (mp - mA);
                    if (np == 0) {          // F[m, 0] = i (sum_k w y E_x) / (2 pi m T)
                        const double2 s = psum(Axis, row, nr, sp);
                        const double d = 2.0 * pi * (double)mp * (double)ea.T;
                        re = -s.y / d; im = s.x / d;
                    } else {                // F[m, n] = -S[m, n] / (4 pi^2 m n)
                        const double2 s = psum(Xs, row * nn + np + ea.N, (int64_t)nr * nn, sp);
                        const double d = -4.0 * pi * pi * (double)mp * (double)np;
                        re = s.x / d; im = s.y / d;
                    }
                }
                v = make_double2(re, neg ? -im : im);
            }
        }
        store_row_out(ea, F, off + (n - nlo), m, n, v);
    }
    if (ea.peer_n) __threadfence_system();   // peer stores performed before the kernel's completion is seen
}

}  // namespace fr

// ---------------------------------------------------------------- host side

static int ilog2_exact(int64_t v) {
    int b = 0;
    while ((int64_t(1) << b) < v) ++b;
    return b;
}

static fr::Geo make_geo(int32_t T, int32_t T2) {
    fr::Geo g;
    g.T = T; g.T2 = T2; g.T1 = T / T2;
    g.t2bits = ilog2_exact(T2); g.t1bits = ilog2_exact(g.T1);
    const int tb = ilog2_exact(T);
    g.lbits = (tb + 1) / 2;
    g.nhi = (int32_t)((T + (1 << g.lbits) - 1) >> g.lbits);
    g.b2 = (g.t2bits + 1) / 2;
    g.nhi2 = (int32_t)((T2 + (1 << g.b2) - 1) >> g.b2);
    return g;
}

// geometry + cost model; route (fcfs_options.route) = FCFS_ROUTE_FFT / FCFS_ROUTE_GEMM forces the choice
// where possible.  f32: the FP32 variant for the split precisions (same 1e-5 B contract as their tensor GEMM)
bool fft_route_plan(int32_t T, int32_t M, int32_t N, int32_t m_lo, int32_t m_hi, int64_t K, bool f32, FftPlan &p,
                    int32_t route) {
    p = FftPlan{};
    if (T < 64 || (T & (T - 1)) != 0 || K <= 0 || K >= (int64_t(1) << 31)) return false;
    int64_t T2 = 64;
    while (T2 < 2 * (int64_t)N + 1) T2 <<= 1;
    if (T2 > fr::kMaxT2 || T2 > T) return false;
    p.T = T; p.T2 = (int32_t)T2; p.N = N; p.f32 = f32 ? 1 : 0;
    p.row0 = (m_lo <= 0 && 0 <= m_hi) ? 1 : 0;
    int32_t a, b;
    if (m_lo > 0) { a = m_lo; b = m_hi; }
    else if (m_hi < 0) { a = -m_hi; b = -m_lo; }
    else { a = 1; b = (-m_lo > m_hi) ? -m_lo : m_hi; }
    p.mA = a;
    p.nm = b >= a ? b - a + 1 : 0;
    p.nr = p.row0 + p.nm;
    // rows per chunk: the G rows of a chunk (8 or 16 T bytes each) within ~4.5 GB, a multiple of 8
    int64_t rc = (int64_t)(4.5e9 / ((f32 ? 8.0 : 16.0) * (double)T));
    rc = rc / 8 * 8;
    if (rc < 8) rc = 8;
    p.rc = rc;
    // sub-row ranges per row: ~4 waves of 2 x 148 CTAs when there are few rows, >= 2 sub-rows each
    {
        const int64_t rows = rc < p.nr ? rc : p.nr;
        int64_t sp = rows > 0 ? (4 * 2 * 148) / rows : 1;
        const int64_t t1h = (T / T2) / 2;
        if (sp > t1h) sp = t1h;
        if (sp > 16) sp = 16;
        if (sp < 1) sp = 1;
        p.sp = (int32_t)sp;
    }
    if (route == FCFS_ROUTE_GEMM) return false;
    if (route == FCFS_ROUTE_FFT) return true;
    const double lg = log2((double)T2);
    const double fft = (double)p.nr * ((double)T * (5.0 * lg + 16.0) + (double)(T / T2) * (2.0 * N + 1) * 8.0) +
                       9.0 * (double)K * (double)p.nm;
    const double rows = (double)(K < (int64_t)T + 1 ? K : (int64_t)T + 1);
    const double gemm = 8.0 * (double)p.nm * (double)N * rows;
    // the tensor GEMMs run ~2x (DMMA vs FP64 route) / ~3x (split tcgen05 vs FP32 route) more flop/s
    return fft * (f32 ? 3.0 : 2.0) < gemm;
}

struct FftWs {
    int32_t *yptr, *flag;
    int16_t *perm, *pinv;
    void *tab, *Gd;      // double2 (FP64 route) or float2 (FP32 route)
    double2 *GT, *Xs, *Axis;
};

static void carve_fft(Carver &cv, const FftPlan &p, FftWs &w) {
    const fr::Geo g = make_geo(p.T, p.T2);
    const int64_t rc = p.rc < p.nr ? p.rc : p.nr;
    const size_t vb = p.f32 ? sizeof(float2) : sizeof(double2);
    w.yptr = cv.take<int32_t>((size_t)p.T + 2);
    w.flag = cv.take<int32_t>(1);
    w.perm = cv.take<int16_t>((size_t)p.T);
    w.pinv = cv.take<int16_t>((size_t)p.T);
    w.tab = cv.take<char>(vb * ((size_t)g.nhi + ((size_t)1 << g.lbits)));
    w.Gd = cv.take<char>(vb * (size_t)(rc > 0 ? rc : 1) * (size_t)p.T);
    w.GT = cv.take<double2>((size_t)(rc > 0 ? rc : 1));
    w.Xs = cv.take<double2>((size_t)p.sp * (size_t)(p.nr > 0 ? p.nr : 1) * (size_t)(2 * p.N + 1));
    w.Axis = cv.take<double2>((size_t)p.sp * (size_t)(p.nr > 0 ? p.nr : 1));
}

size_t fft_route_ws_bytes(const FftPlan &p) {
    Carver cv(nullptr, 0);
    FftWs w;
    carve_fft(cv, p, w);
    return cv.used();
}

// y-CSR of the corner range and whether its y are non-decreasing (one stream sync)
fcfs_status fft_route_prepare(const int32_t *y, int64_t k_lo, int64_t K, const FftPlan &p, void *ws, size_t ws_bytes,
                              bool &sorted, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    FftWs W;
    carve_fft(cv, p, W);
    if (!cv.fits()) { set_error("fft route: workspace %zu < %zu", ws_bytes, cv.used()); return FCFS_E_WORKSPACE; }
    FCFS_TRY_CUDA(cudaMemsetAsync(W.flag, 0, sizeof(int32_t), s));
    int64_t n = (int64_t)p.T + 2 > K ? (int64_t)p.T + 2 : K;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    fr::k_fr_yptr<<<(unsigned)blocks, 256, 0, s>>>(y, k_lo, K, p.T, W.yptr, W.flag, nullptr);
    FCFS_CHECK_LAUNCH("k_fr_yptr");
    int32_t f = 0;
    FCFS_TRY_CUDA(cudaMemcpyAsync(&f, W.flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    FCFS_TRY_CUDA(cudaStreamSynchronize(s));
    sorted = f == 0;
    return FCFS_OK;
}

// the sync-free variant: K from device memory (<= K_cap, the planned size), the sortedness flag turned
// into a device status instead of a host read (the corners of fcfs_vertices_from_rects_async are sorted)
__global__ void k_fr_status(const int32_t *flag, const int64_t *K_dev, int64_t K_cap, int32_t *status) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && *status == FCFS_OK)
        *status = *flag ? FCFS_E_INVALID : (*K_dev > K_cap ? FCFS_E_CAPACITY : FCFS_OK);
}

fcfs_status fft_route_prepare_dev(const int32_t *y, const int64_t *K_dev, int64_t K_cap, const FftPlan &p, void *ws,
                                  size_t ws_bytes, int32_t *status_dev, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    FftWs W;
    carve_fft(cv, p, W);
    if (!cv.fits()) { set_error("fft route: workspace %zu < %zu", ws_bytes, cv.used()); return FCFS_E_WORKSPACE; }
    FCFS_TRY_CUDA(cudaMemsetAsync(W.flag, 0, sizeof(int32_t), s));
    int64_t n = (int64_t)p.T + 2 > K_cap ? (int64_t)p.T + 2 : K_cap;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    fr::k_fr_yptr<<<(unsigned)blocks, 256, 0, s>>>(y, 0, K_cap, p.T, W.yptr, W.flag, K_dev);
    FCFS_CHECK_LAUNCH("k_fr_yptr");
    k_fr_status<<<1, 32, 0, s>>>(W.flag, K_dev, K_cap, status_dev);
    FCFS_CHECK_LAUNCH("k_fr_status");
    return FCFS_OK;
}

template <class V>
static fcfs_status run_route(const int32_t *x, const int32_t *w, int64_t k_lo, const FftPlan &p, FftWs &W,
                             const EpiArgs &ea, void *F, cudaStream_t s) {
    const fr::Geo g = make_geo(p.T, p.T2);
    V *tab = (V *)W.tab, *Gd = (V *)W.Gd;
    const int ntab = g.nhi + (1 << g.lbits);
    fr::k_fr_table<V><<<(unsigned)((ntab + 255) / 256), 256, 0, s>>>(tab, g);
    FCFS_CHECK_LAUNCH("k_fr_table");
    fr::k_fr_perm<<<(unsigned)g.T1, fr::kThreads, 0, s>>>(W.yptr, g, W.perm, W.pinv);
    FCFS_CHECK_LAUNCH("k_fr_perm");
    const size_t fsmem2 = (size_t)(p.T2 + p.T2 / 16 + g.nhi2 + (1 << g.b2)) * sizeof(V) +
                          (size_t)(2 * p.N + 1) * sizeof(double2) + (size_t)p.T2 * sizeof(int16_t);
    FCFS_TRY(ensure_smem((const void *)fr::k_fr_fft2<V>, fsmem2, true));
    int64_t tblocks = p.T / 256;
    if (tblocks > 512) tblocks = 512;
    if (tblocks < 1) tblocks = 1;
    for (int64_t c0 = 0; c0 < p.nr; c0 += p.rc) {
        const int64_t c1 = c0 + p.rc < p.nr ? c0 + p.rc : p.nr;
        FCFS_TRY_CUDA(cudaMemsetAsync(W.GT, 0, sizeof(double2) * (size_t)(c1 - c0), s));
        if (c0 == 0 && p.row0) {
            fr::k_fr_row0<V><<<(unsigned)tblocks, 256, 0, s>>>(x, w, k_lo, W.yptr, W.perm, g, Gd);
            FCFS_CHECK_LAUNCH("k_fr_row0");
            fr::k_fr_row0T<V><<<1, fr::kThreads, 0, s>>>(x, w, k_lo, W.yptr, W.pinv, g, Gd);
            FCFS_CHECK_LAUNCH("k_fr_row0T");
        }
        const int64_t ra = c0 > p.row0 ? c0 : p.row0;   // first |m| >= 1 row of the chunk
        if (ra < c1) {
            const int32_t m_first = p.mA + (int32_t)(ra - p.row0), m_last = p.mA + (int32_t)(c1 - 1 - p.row0);
            const int64_t rb = (m_last - m_first + fr::kRowsPerThread) / fr::kRowsPerThread;
            dim3 grid((unsigned)tblocks, (unsigned)rb);
            const size_t rsmem = sizeof(V) * (size_t)(g.nhi + (1 << g.lbits));
            fr::k_fr_rows<V><<<grid, fr::kThreads, rsmem, s>>>(x, w, k_lo, W.yptr, W.perm, tab, g, m_first, m_last,
                                                           (int32_t)(ra - c0), Gd);
            FCFS_CHECK_LAUNCH("k_fr_rows");
            fr::k_fr_rowsT<V><<<(unsigned)rb, fr::kThreads, 0, s>>>(x, w, k_lo, W.yptr, W.pinv, tab, g, m_first,
                                                                    m_last, (int32_t)(ra - c0), Gd, W.GT);
            FCFS_CHECK_LAUNCH("k_fr_rowsT");
        }
        dim3 fgrid((unsigned)(c1 - c0), (unsigned)p.sp);
        fr::k_fr_fft2<V><<<fgrid, fr::kThreads, fsmem2, s>>>(Gd, W.GT, tab, W.pinv, g, p.N, (int32_t)c0,
                                                             (int32_t)(p.nr > 0 ? p.nr : 1), W.Xs, W.Axis);
        FCFS_CHECK_LAUNCH("k_fr_fft");
    }
    const int rows = ea.m_hi - ea.m_lo + 1;
    if (rows > 0) {
        fr::k_fr_epilogue<<<(unsigned)rows, 128, 0, s>>>(W.Xs, W.Axis, ea, p.row0, p.mA,
                                                        (int32_t)(p.nr > 0 ? p.nr : 1), p.sp, F);
        FCFS_CHECK_LAUNCH("k_fr_epilogue");
    }
    return FCFS_OK;
}

fcfs_status fft_route_run(const int32_t *x, const int32_t *w, int64_t k_lo, const FftPlan &p, void *ws,
                          size_t ws_bytes, const EpiArgs &ea, void *F, cudaStream_t s) {
    Carver cv(ws, ws_bytes);
    FftWs W;
    carve_fft(cv, p, W);
    if (!cv.fits()) { set_error("fft route: workspace %zu < %zu", ws_bytes, cv.used()); return FCFS_E_WORKSPACE; }
    return p.f32 ? run_route<float2>(x, w, k_lo, p, W, ea, F, s) : run_route<double2>(x, w, k_lo, p, W, ea, F, s);
}

}  // namespace fcfs

// contract_fp64.cu — a2 + a3 (FP64): generated-operand real GEMM over ROW BUCKETS.
//
// The interior coefficients of Eq. Fkl are the 2-D DFT of the
// sparse +-1 image f~_xy (Step 4), evaluated directly ("Goertzel-like",
// P:917-920) on a low-pass window.  Writing E = c - i s, the complex sum
// sum_k w_k E_x[m,k] E_y[n,k] for (m, +-n) is recombined from the four real quadrant
// products P_cc, P_cs, P_sc, P_ss.  Step 4's row structure (corners on one row y share
// E_y[n, y]) turns the sum over K corners into a sum over the R row buckets of buckets.cu:
//     A[2j  ,b] = sum_{k in b} w_k cos(2 pi m_j x_k / T),  A[2j+1,b] = sum_{k in b} w_k sin(...),
//     A[2nf ,b] = sum_{k in b} w_k x_k
//     B[2j  ,b] = cos(2 pi n_j y_b / T),  B[2j+1,b] = sin(...),  B[2nf,b] = y_b
// (the last rows carry the axis sums of Eqs. Fk0/F0l, Steps 2-3 P:870-888), so the GEMM has
// inner dimension R instead of K (K/R = 15 on BASELINE.json configs[3]).
//
// a2 (twiddles) is fused: each CTA generates its bucket slab of A and B in shared memory
// from the integer phase r = (m x) mod T (exact, lattice vertices P:860-862) through a
// two-level table E(r) = E_hi(r >> L) * E_lo(r & (2^L - 1)) built in SMEM with sincospi,
// so the twiddle matrices never touch HBM ("no full-length arrays").
//
// a3 (FP64): FP64 tensor cores (mma.sync m16n8k16 .f64, SASS DMMA), 64x64 P tile per CTA,
// 8 warps of 16x32, double-buffered slabs of 16 buckets (one k16 MMA step per slab).
// Accumulation is hierarchical: a fresh register accumulator per chunk of <= kChunk buckets
// is added into a running total, bounding the rounding error by about
// (kRowBucketCapFp64 + kChunk + R/kChunk) u B instead of K u B.
#include "common.cuh"

namespace fcfs {

static constexpr int kBK = 32;        // row buckets per slab (two k16 DMMA steps per barrier)
static constexpr int kChunk = 2048;   // buckets per register accumulator (<= kRowBucketCapFp64 corners each)
static constexpr int kThreads = 256;  // 16 x 16 threads, 4x4 outputs each

__device__ __forceinline__ void build_tables(const TwiddleGeom &g, double2 *thi, double2 *tlo) {
    const int L = 1 << g.lbits;
    for (int i = threadIdx.x; i < g.nhi + L; i += blockDim.x) {
        double s, c;
        if (i < g.nhi) {
            sincospi(2.0 * (double)((int64_t)i << g.lbits) / (double)g.T, &s, &c);
            thi[i] = make_double2(c, s);
        } else {
            int b = i - g.nhi;
            sincospi(2.0 * (double)b / (double)g.T, &s, &c);
            tlo[b] = make_double2(c, s);
        }
    }
}

// (cos, sin) of 2 pi r / T via the two-level table
__device__ __forceinline__ double2 twiddle(uint32_t r, const TwiddleGeom &g, const double2 *thi,
                                           const double2 *tlo) {
    double2 a = thi[r >> g.lbits];
    double2 b = tlo[r & ((1u << g.lbits) - 1)];
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.y, b.x, a.x * b.y));
}

// (row 2p, row 2p+1) values of one side for corner coordinate v and weight wt
__device__ __forceinline__ double2 side_pair(int p_global, const SidePlan &sp, int32_t v, double wt,
                                             const TwiddleGeom &g, const double2 *thi, const double2 *tlo) {
    if (p_global < sp.nf) {
        uint32_t r = phase_mod((uint32_t)(sp.f0 + p_global), (uint32_t)v, g);
        double2 cs = twiddle(r, g, thi, tlo);
        return make_double2(wt * cs.x, wt * cs.y);
    }
    if (p_global == sp.nf && sp.axis) return make_double2(wt * (double)v, 0.0);
    return make_double2(0.0, 0.0);
}

// x-side pair of one row bucket: sum over its corners [cb, ce) of w_k (cos, sin)(2 pi f x_k / T)
// (G of the row-bucketed Step 4, buckets.cu), or sum w_k x_k for the axis row.  The warp (32 pairs
// of one bucket) runs the corner loop uniformly; x / w come through L1 (one line per warp).
__device__ __forceinline__ double2 bucket_pair(int p_global, const SidePlan &sp, const int32_t *__restrict__ xs,
                                               const int32_t *__restrict__ ws, int cb, int ce, const TwiddleGeom &g,
                                               const double2 *thi, const double2 *tlo) {
    double re = 0.0, im = 0.0;
    if (p_global < sp.nf) {
        const uint32_t f = (uint32_t)(sp.f0 + p_global);
        int c = cb;
        for (; c + 1 < ce; c += 2) {
            const int32_t x0 = __ldg(xs + c), x1 = __ldg(xs + c + 1);
            const double w0 = (double)__ldg(ws + c), w1 = (double)__ldg(ws + c + 1);
            const double2 e0 = twiddle(phase_mod(f, (uint32_t)x0, g), g, thi, tlo);
            const double2 e1 = twiddle(phase_mod(f, (uint32_t)x1, g), g, thi, tlo);
            re = fma(w0, e0.x, re); im = fma(w0, e0.y, im);
            re = fma(w1, e1.x, re); im = fma(w1, e1.y, im);
        }
        if (c < ce) {
            const int32_t x0 = __ldg(xs + c);
            const double w0 = (double)__ldg(ws + c);
            const double2 e0 = twiddle(phase_mod(f, (uint32_t)x0, g), g, thi, tlo);
            re = fma(w0, e0.x, re); im = fma(w0, e0.y, im);
        }
    } else if (p_global == sp.nf && sp.axis) {
        long long a = 0;
        for (int c = cb; c < ce; ++c) a += (long long)__ldg(ws + c) * (long long)__ldg(xs + c);
        re = (double)a;
    }
    return make_double2(re, im);
}

// FP64 tensor-core MMA (DMMA): D[16x8] += A[16x16] B[16x8], fragments per the sm_90+/sm_100
// mma.sync.m16n8k16.f64 layout (g = lane / 4, t = lane % 4):
//   a[j] = A[g + 8 (j & 1)][t + 4 (j >> 1)],  b[v] = B[t + 4 v][g],  c[v] = C[g + 8 (v >> 1)][2 t + (v & 1)]
__device__ __forceinline__ void dmma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
        "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
          "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

static constexpr int kLd = kTile + 4;   // padded smem row (doubles): conflict-free fragment loads

// 16-byte asynchronous global -> shared copy (LDGSTS); src_size 0 zero-fills the destination
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc, bool valid) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gsrc), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// kLoadA = false: A (x-side bucket sums) generated per slab; one launch covers the whole bucket range.
// kLoadA = true: A read from G (k_gsum_fp64: the sums of one chunk of ch.cb buckets, computed once
// instead of once per column tile); the items cover that chunk and ADD into P_ws (zeroed before
// the first chunk), so successive chunk launches accumulate the full sum in a fixed order.
template <bool kLoadA>
__global__ void __launch_bounds__(kThreads, 2)
k_gemm_fp64(CornerSrc src, GemmPlan plan, TwiddleGeom g, double *__restrict__ P_ws, FpChunk ch) {
    if (kLoadA && src.clip_bptr[0] + ch.chunk * ch.cb >= src.clip_bptr[1]) return;   // chunk past the buckets
    extern __shared__ __align__(16) double smem_d[];
    double2 *thi = (double2 *)smem_d;
    double2 *tlo = thi + g.nhi;
    double *As = (double *)(tlo + (1 << g.lbits));   // [2][kBK][kLd]
    double *Bs = As + 2 * kBK * kLd;                 // [2][kBK][kLd]

    build_tables(g, thi, tlo);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int wm = (warp & 3) * 16, wn = (warp >> 2) * 32;   // warp tile 16 x 32 (4 MMAs of n8)
    const int lg = lane >> 2, lt = lane & 3;
    const int gp = tid & 31, gk = tid >> 5;                  // generation: pair gp, corner gk (+8)
    const int64_t per_clip = (int64_t)plan.tiles_x * plan.tiles_y * plan.splits;

    for (int64_t item = blockIdx.x; item < plan.items; item += gridDim.x) {
        const int64_t clip = item / per_clip;
        int64_t rem = item - clip * per_clip;
        const int tix = (int)(rem / ((int64_t)plan.tiles_y * plan.splits));
        rem -= (int64_t)tix * plan.tiles_y * plan.splits;
        const int tiy = (int)(rem / plan.splits);
        const int split = (int)(rem - (int64_t)tiy * plan.splits);
        // bucket range of the item (the split partitions the clip's row buckets, or the chunk's)
        int64_t kb = src.clip_bptr[clip], ke = src.clip_bptr[clip + 1];
        const int64_t chunk0 = kb + ch.chunk * ch.cb;   // kLoadA: first bucket of the chunk
        if (kLoadA) {
            kb = chunk0;
            if (ke > chunk0 + ch.cb) ke = chunk0 + ch.cb;
            if (kb >= ke) continue;                     // past the clip's buckets: adds nothing
        }
        const int64_t span = ke - kb;
        const int64_t k0 = kb + span * split / plan.splits;
        const int64_t k1 = kb + span * (split + 1) / plan.splits;

        double tot[4][4], acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) tot[i][j] = 0.0;

        __syncthreads();   // tables ready / previous item's smem reads done
        // slab of kBK buckets [ks, ks + kBK) (zeros past kend): A = bucket sums, B = row twiddles
        auto generate = [&](int buf, int64_t ks, int64_t kend) {
#pragma unroll
            for (int h = 0; h < kBK / 8; ++h) {
                const int kk = gk + 8 * h;
                const int64_t b = ks + kk;
                double2 a = make_double2(0.0, 0.0), bv = make_double2(0.0, 0.0);
                if (kLoadA) {   // x side: asynchronous copy of the precomputed sums (overlaps the DMMAs)
                    const bool ok = b < kend;
                    const double *gs = ok ? ch.G + ((int64_t)tix * ch.cb + (b - chunk0)) * kTile + 2 * gp : ch.G;
                    cp_async16(&As[(buf * kBK + kk) * kLd + 2 * gp], gs, ok);
                }
                if (kLoadA) {   // y side: the precomputed row twiddles, likewise
                    const bool ok = b < kend;
                    const double *hs = ok ? ch.H + ((int64_t)tiy * ch.cb + (b - chunk0)) * kTile + 2 * gp : ch.H;
                    cp_async16(&Bs[(buf * kBK + kk) * kLd + 2 * gp], hs, ok);
                } else {
                    if (b < kend) {
                        const int cb = __ldg(src.bptr + b), ce = __ldg(src.bptr + b + 1);
                        a = bucket_pair(tix * (kTile / 2) + gp, plan.X, src.x, src.w, cb, ce, g, thi, tlo);
                        bv = side_pair(tiy * (kTile / 2) + gp, plan.Y, __ldg(src.by + b), 1.0, g, thi, tlo);
                    }
                    *(double2 *)&As[(buf * kBK + kk) * kLd + 2 * gp] = a;
                    *(double2 *)&Bs[(buf * kBK + kk) * kLd + 2 * gp] = bv;
                }
            }
        };

        for (int64_t c0 = k0; c0 < k1; c0 += kChunk) {
            const int64_t c1 = c0 + kChunk < k1 ? c0 + kChunk : k1;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
            int buf = 0;
            generate(0, c0, c1);
            if (kLoadA) cp_async_wait_all();
            __syncthreads();
            for (int64_t ks = c0; ks < c1; ks += kBK) {
                if (ks + kBK < c1) generate(buf ^ 1, ks + kBK, c1);
#pragma unroll
                for (int k16 = 0; k16 < kBK; k16 += 16) {
                    const double *Ab = As + (buf * kBK + k16) * kLd;
                    const double *Bb = Bs + (buf * kBK + k16) * kLd;
                    double a[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) a[j] = Ab[(lt + 4 * (j >> 1)) * kLd + wm + lg + 8 * (j & 1)];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        double bf[4];
#pragma unroll
                        for (int v = 0; v < 4; ++v) bf[v] = Bb[(lt + 4 * v) * kLd + wn + 8 * t + lg];
                        dmma16816(acc[t], a, bf);
                    }
                }
                if (kLoadA) cp_async_wait_all();   // the next slab's x-side copy has landed
                __syncthreads();
                buf ^= 1;
            }
            // corners k >= c1 of the last slab were generated as zeros (A = B = 0)
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) tot[i][j] += acc[i][j];
        }
        double *out = P_ws + item * (int64_t)(kTile * kTile);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int col = wn + 8 * t + 2 * lt;
            double2 *o0 = (double2 *)(out + (wm + lg) * kTile + col), *o1 = (double2 *)(out + (wm + lg + 8) * kTile + col);
            if (kLoadA) {   // this CTA owns the tile within the launch: plain read-modify-write
                const double2 p0 = *o0, p1 = *o1;
                *o0 = make_double2(p0.x + tot[t][0], p0.y + tot[t][1]);
                *o1 = make_double2(p1.x + tot[t][2], p1.y + tot[t][3]);
            } else {
                *o0 = make_double2(tot[t][0], tot[t][1]);
                *o1 = make_double2(tot[t][2], tot[t][3]);
            }
        }
    }
}

// x-side bucket sums of one chunk of ch.cb buckets of a single clip, for every x tile:
// G[(tix * cb + b) * 64 + 2p + t] = sum_{k in bucket} w_k (cos, sin)(2 pi f_p x_k / T) (t = 0, 1), with the
// axis pair (f = nf) carrying sum w_k x_k.  Persistent blocks over (64 buckets, x tile) units; thread =
// (bucket, block of 8 pairs): per corner two table lookups (E(f0 x) and the step E(x)) and the FP64
// angle-addition recurrence over the 8 pairs (<= 7 steps, ~1 ulp each), i.e. a quarter of the
// shared-memory lookups of one lookup per (corner, pair).
static constexpr int kGsumBuckets = kThreads / 4;   // 64 buckets per unit
__global__ void __launch_bounds__(kThreads)
k_gsum_fp64(CornerSrc src, GemmPlan plan, TwiddleGeom g, FpChunk ch, double *__restrict__ G) {
    if (src.clip_bptr[0] + ch.chunk * ch.cb >= src.clip_bptr[1]) return;   // chunk past the buckets
    extern __shared__ __align__(16) double smem_d[];
    double2 *thi = (double2 *)smem_d;
    double2 *tlo = thi + g.nhi;
    build_tables(g, thi, tlo);
    __syncthreads();
    const int kk = threadIdx.x >> 2, pb = threadIdx.x & 3;   // bucket in the unit, 8-pair block
    const int64_t cb0 = src.clip_bptr[0], cb1 = src.clip_bptr[1];
    const int64_t chunk0 = cb0 + ch.chunk * ch.cb;
    const int64_t chunk1 = chunk0 + ch.cb < cb1 ? chunk0 + ch.cb : cb1;
    if (chunk0 >= chunk1) return;
    const int64_t nunit_b = (chunk1 - chunk0 + kGsumBuckets - 1) / kGsumBuckets;
    const int64_t units = nunit_b * plan.tiles_x;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int tix = (int)(u % plan.tiles_x);
        const int64_t b = chunk0 + (u / plan.tiles_x) * kGsumBuckets + kk;
        if (b >= chunk1) continue;
        const int p0 = tix * (kTile / 2) + 8 * pb;           // first pair (global) of the block
        double re[8], im[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { re[i] = 0.0; im[i] = 0.0; }
        long long ax = 0;
        const int cb = __ldg(src.bptr + b), ce = __ldg(src.bptr + b + 1);
        const uint32_t f0 = (uint32_t)(plan.X.f0 + p0);
        for (int c = cb; c < ce; ++c) {
            const int32_t x = __ldg(src.x + c);
            const int32_t wi = __ldg(src.w + c);
            const double w = (double)wi;
            ax += (long long)wi * (long long)x;
            const double2 e0 = twiddle(phase_mod(f0, (uint32_t)x, g), g, thi, tlo);
            const double2 e1 = twiddle(phase_mod(1u, (uint32_t)x, g), g, thi, tlo);
            double cr = w * e0.x, ci = w * e0.y;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                re[i] += cr;
                im[i] += ci;
                if (i < 7) {
                    const double nr = fma(cr, e1.x, -ci * e1.y);
                    const double ni = fma(ci, e1.x, cr * e1.y);
                    cr = nr;
                    ci = ni;
                }
            }
        }
        double *out = G + ((int64_t)tix * ch.cb + (b - chunk0)) * kTile + 2 * 8 * pb;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int p = p0 + i;
            double2 v = make_double2(0.0, 0.0);
            if (p < plan.X.nf) v = make_double2(re[i], im[i]);
            else if (p == plan.X.nf && plan.X.axis) v = make_double2((double)ax, 0.0);
            *(double2 *)(out + 2 * i) = v;
        }
    }
}

// y-side row twiddles of one chunk for every y tile: H[(tiy * cb + b) * 64 + 2p + t] = (cos, sin)(2 pi n_p y_b / T),
// the axis pair carrying y_b.  Same unit / thread mapping and recurrence as k_gsum_fp64, one row y per bucket.
__global__ void __launch_bounds__(kThreads)
k_hsum_fp64(CornerSrc src, GemmPlan plan, TwiddleGeom g, FpChunk ch, double *__restrict__ H) {
    if (src.clip_bptr[0] + ch.chunk * ch.cb >= src.clip_bptr[1]) return;   // chunk past the buckets
    extern __shared__ __align__(16) double smem_d[];
    double2 *thi = (double2 *)smem_d;
    double2 *tlo = thi + g.nhi;
    build_tables(g, thi, tlo);
    __syncthreads();
    const int kk = threadIdx.x >> 2, pb = threadIdx.x & 3;
    const int64_t cb0 = src.clip_bptr[0], cb1 = src.clip_bptr[1];
    const int64_t chunk0 = cb0 + ch.chunk * ch.cb;
    const int64_t chunk1 = chunk0 + ch.cb < cb1 ? chunk0 + ch.cb : cb1;
    if (chunk0 >= chunk1) return;
    const int64_t nunit_b = (chunk1 - chunk0 + kGsumBuckets - 1) / kGsumBuckets;
    const int64_t units = nunit_b * plan.tiles_y;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int tiy = (int)(u % plan.tiles_y);
        const int64_t b = chunk0 + (u / plan.tiles_y) * kGsumBuckets + kk;
        if (b >= chunk1) continue;
        const int p0 = tiy * (kTile / 2) + 8 * pb;
        const int32_t y = __ldg(src.by + b);
        const double2 e0 = twiddle(phase_mod((uint32_t)(plan.Y.f0 + p0), (uint32_t)y, g), g, thi, tlo);
        const double2 e1 = twiddle(phase_mod(1u, (uint32_t)y, g), g, thi, tlo);
        double cr = e0.x, ci = e0.y;
        double *out = H + ((int64_t)tiy * ch.cb + (b - chunk0)) * kTile + 2 * 8 * pb;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int p = p0 + i;
            double2 v = make_double2(0.0, 0.0);
            if (p < plan.Y.nf) v = make_double2(cr, ci);
            else if (p == plan.Y.nf && plan.Y.axis) v = make_double2((double)y, 0.0);
            *(double2 *)(out + 2 * i) = v;
            const double nr = fma(cr, e1.x, -ci * e1.y);
            const double ni = fma(ci, e1.x, cr * e1.y);
            cr = nr;
            ci = ni;
        }
    }
}

static size_t fp64_smem(const TwiddleGeom &g) {
    return sizeof(double2) * (size_t)(g.nhi + (1 << g.lbits)) + sizeof(double) * 4 * kBK * kLd;
}

fcfs_status launch_gemm_fp64(const CornerSrc &src, const GemmPlan &plan, int32_t T, double *P_ws,
                             cudaStream_t s) {
    if (plan.items <= 0) return FCFS_OK;
    TwiddleGeom g = make_twiddle_geom(T);
    FCFS_TRY(ensure_smem((const void *)k_gemm_fp64<false>, 100 * 1024));
    int64_t grid = plan.items < 148 * 16 ? plan.items : 148 * 16;
    k_gemm_fp64<false><<<(unsigned)grid, kThreads, fp64_smem(g), s>>>(src, plan, g, P_ws, FpChunk{nullptr, 0, 0, nullptr});
    FCFS_CHECK_LAUNCH("k_gemm_fp64");
    return FCFS_OK;
}

int64_t fp64_chunk_buckets(int64_t K) {
    int64_t cb = K < kFpChunkBuckets ? K : kFpChunkBuckets;
    cb = (cb + kBK - 1) / kBK * kBK;
    return cb < kBK ? kBK : cb;
}

// single clip, chunked: G of each chunk once (k_gsum_fp64), then the DMMA GEMM reading it (P_ws +=)
fcfs_status launch_gemm_fp64_chunked(const CornerSrc &src, const GemmPlan &plan, int32_t T, int64_t K, double *G,
                                     double *H, double *P_ws, cudaStream_t s) {
    if (plan.items <= 0) return FCFS_OK;
    TwiddleGeom g = make_twiddle_geom(T);
    FCFS_TRY(ensure_smem((const void *)k_gemm_fp64<true>, 100 * 1024));
    FCFS_TRY(ensure_smem((const void *)k_gsum_fp64, 100 * 1024));
    FCFS_TRY(ensure_smem((const void *)k_hsum_fp64, 100 * 1024));
    FCFS_TRY_CUDA(cudaMemsetAsync(P_ws, 0, sizeof(double) * (size_t)plan.items * kTile * kTile, s));
    const int64_t cb = chunk_buckets(K, plan.tiles_x, plan.tiles_y);
    const int64_t nchunk = K > 0 ? (K + cb - 1) / cb : 0;   // K = the clip's bucket count here
    const size_t tsm = sizeof(double2) * (size_t)(g.nhi + (1 << g.lbits));
    int64_t grid = plan.items < 148 * 16 ? plan.items : 148 * 16;
    for (int64_t c = 0; c < nchunk; ++c) {
        const FpChunk ch{G, c, cb, H};
        k_gsum_fp64<<<148 * 4, kThreads, tsm, s>>>(src, plan, g, ch, G);
        FCFS_CHECK_LAUNCH("k_gsum_fp64");
        k_hsum_fp64<<<148 * 4, kThreads, tsm, s>>>(src, plan, g, ch, H);
        FCFS_CHECK_LAUNCH("k_hsum_fp64");
        k_gemm_fp64<true><<<(unsigned)grid, kThreads, fp64_smem(g), s>>>(src, plan, g, P_ws, ch);
        FCFS_CHECK_LAUNCH("k_gemm_fp64");
    }
    return FCFS_OK;
}

// sum_k w_k x_k y_k over [k_lo, k_hi) (vertex-block DC), exact int64
__global__ void k_block_area(const int32_t *x, const int32_t *y, const int32_t *w, int64_t k_lo, int64_t k_hi,
                             int64_t *area) {
    long long s = 0;
    for (int64_t k = k_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < k_hi;
         k += (int64_t)gridDim.x * blockDim.x)
        s += (long long)w[k] * (long long)x[k] * (long long)y[k];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s != 0) atomicAdd((unsigned long long *)area, (unsigned long long)s);
}

fcfs_status launch_block_area(const CornerSrc &src, int64_t *area_dev, cudaStream_t s) {
    FCFS_TRY_CUDA(cudaMemsetAsync(area_dev, 0, sizeof(int64_t), s));
    int64_t n = src.k_hi - src.k_lo;
    if (n <= 0) return FCFS_OK;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 4) blocks = 148 * 4;
    k_block_area<<<(unsigned)blocks, 256, 0, s>>>(src.x, src.y, src.w, src.k_lo, src.k_hi, area_dev);
    FCFS_CHECK_LAUNCH("k_block_area");
    return FCFS_OK;
}

}  // namespace fcfs

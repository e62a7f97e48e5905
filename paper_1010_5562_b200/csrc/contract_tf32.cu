// contract_tf32.cu — a2 + a3 (split-TF32 / split-FP16): the quadrant GEMM P = A diag(w) B^T on
// the 5th-generation tensor cores (tcgen05.mma kind::tf32 or kind::f16, accumulators in TMEM).
// kF16 = 0: operands tf32 hi/lo (4 B per value, 32 corners per stage);
// kF16 = 1: operands fp16 hi/lo (2 B per value, 64 corners per stage, twice the MMA rate and half
//           the shared-memory bytes per corner; same FP32-accurate tolerance 1e-5 B).
//
// Same product as contract_fp64.cu (Eq. Fkl P:843-846 / Steps 2-4 P:870-904, evaluated
// directly as in P:917-920), FP32-accurate:
//   * every generated operand value v (w*cos, w*sin, axis weight) is split v = hi + lo with
//     hi = tf32(v), lo = tf32(v - hi); the operand tile stacks [hi rows; lo rows] (128 rows),
//     so ONE M=128 x N=128 x K=8 MMA yields hi*hi, hi*lo, lo*hi (and lo*lo) for a 64x64 tile;
//   * FP32 TMEM partials are flushed into FP64 registers every kChunk corners (hierarchical
//     accumulation), double-buffered in TMEM so the flush overlaps the MMAs.
//
// a2 is fused: producer warps reduce the phase (f * v) mod T exactly in integers (lattice
// vertices), look up e^{i 2 pi r/T} in an SMEM table and write the split operand
// tiles straight into the canonical SWIZZLE_128B K-major UMMA layout; the twiddle matrices
// never exist in HBM ("no full-length arrays").
//
// Warp roles (416 threads, 1 CTA per SM, persistent over work items):
//   warps 0-3   epilogue: tcgen05.ld TMEM -> registers, combine 4 quadrant blocks, FP64 flush,
//               write the item's 64x64 FP64 P tile (phys layout 1: c0..c31, s0..s31)
//   warps 4-11  producers: twiddle generation into a 5-stage SMEM ring (mbarrier full/empty);
//               4 groups of 2 warps (side A, side B), group g fills every 4th stage, so a group
//               never waits for the consumption of the stage it produced last (ring > groups)
//   warp 12     TMEM allocator + single-thread MMA issuer (tcgen05.mma / tcgen05.commit)
#include <cuda_fp16.h>

#include "coeff.cuh"
#include "umma.cuh"

namespace fcfs {
namespace tc {

// Ablation switches (experiments only): compiled in only with -DFCFS_ABLATE (tools/ablate_build.sh builds
// that variant as a separate libfcfs_ablate.so); in the shipped library every ABL(bit) is the constant 0.
#ifdef FCFS_ABLATE
#define ABL(bit) (plan.dbg & (bit))
#else
#define ABL(bit) 0
#endif

constexpr int kBK = 32;                         // corners per stage (K of 4 MMAs)
constexpr int kStages = 5;                      // ring depth (> kGroups: no self-wait)
constexpr int kGroups = 4;                      // producer groups (2 warps each)
constexpr int kRows = 128;                      // operand rows: 64 hi + 64 lo
constexpr int kRowBytes = kBK * 4;              // one operand row of a stage = one SW128 atom row (128 B)
constexpr int kOpBytes = kRows * kRowBytes;     // 16 KB per operand per stage
constexpr int kStageBytes = 2 * kOpBytes;       // A + B
constexpr int kChunk = 1024;                    // corners per TMEM accumulation (FP64 flush)
constexpr int kEpiWarps = 4, kProdWarps = 8;
constexpr int kThreads = (kEpiWarps + kProdWarps + 1) * 32;
constexpr int kMmaWarp = kEpiWarps + kProdWarps;
constexpr int kTmemCols = 256;                  // 2 accumulators x 128 fp32 columns
constexpr int kXStride = 33;                    // exchange buffer row stride (floats)
constexpr int kSingleTableMax = 2048;           // T <= this: one-level table of T entries (smem budget)
constexpr int kMaxFuseRows = 64;                // fused epilogue: at most 63 output rows (M <= 31)
constexpr int kMaxFuseOut = 63 * 63;            // fused epilogue: output (m, n) table entries
// instruction descriptor: D=F32, A=B=TF32, K-major both, N=128, M=128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(128 >> 3) << 17) |
                            ((uint32_t)(128 >> 4) << 24);

struct Smem {
    // offsets from the 1024-aligned dynamic smem base
    uint32_t stage0, table, xbuf, bars;
    uint32_t total;
};

constexpr int kStagesLoadA = 6;                 // load-A mode: no fused-epilogue tables, one more stage
constexpr int kStagesEdge = 5;                  // edge mode (SFU twiddles, no table): 6 fits but measured no faster
constexpr int kBarBytes = 192;                  // mbarriers (<= 2 x 6 + 4) + the TMEM address slot

// stages: operand ring depth; fused: room for the fused epilogue's output tables
__host__ __device__ inline Smem smem_layout(int table_entries, int stages = kStages, bool fused = true) {
    Smem s;
    s.stage0 = 0;
    s.table = stages * kStageBytes;
    s.xbuf = s.table + ((table_entries * 8 + 1023) & ~1023);
    s.bars = s.xbuf + 2 * 64 * kXStride * 4;       // xbuf also holds the fused epilogue's fp32 P tile (64 x 65)
    s.total = s.bars + kBarBytes + (fused ? 4 * (kMaxFuseRows + 2) + 8 * 3 * kMaxFuseRows + 4 * kMaxFuseOut : 0);
    return s;
}

// ---- debug event trace (FCFS_DEBUG bit 256; CTA 0 only): clock64 << 24 | event << 16 | stage
constexpr int kTraceMax = 1 << 16;
__device__ unsigned long long g_trace[kTraceMax];
__device__ unsigned int g_trace_n;
__device__ __forceinline__ void trace(int on, int ev, uint32_t sc) {
#ifndef FCFS_TRACE
    return;   // compiled in only with -DFCFS_TRACE (tools/trace_*.py)
#endif
    if (!on || blockIdx.x != 0) return;
    const unsigned int i = atomicAdd(&g_trace_n, 1u);
    if (i < kTraceMax) g_trace[i] = ((unsigned long long)clock64() << 24) | ((unsigned long long)ev << 16) | (sc & 0xFFFFu);
}

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate)
        : "memory");
}
// instruction descriptor for kind::f16 with fp16 A/B (format 0), D=F32, K-major, N=128, M=128
constexpr uint32_t kIdescF16 = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(128 >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(kIdescF16), "r"(accumulate)
        : "memory");
}
template <int kF16>
__device__ __forceinline__ void umma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    if (kF16) umma_f16(d_tmem, adesc, bdesc, accumulate);
    else umma_tf32(d_tmem, adesc, bdesc, accumulate);
}

struct ItemInfo {
    int64_t k0, k1;
    int tix, tiy;
};

// chunked row-bucket mode (single clip): the x-side operand of every stage comes from G, the
// pre-split bucket sums of chunk `chunk` (k_gsum_tc), [tiles_x][stages of the chunk][16 KB]
struct TcChunk {
    const uint8_t *G;     // x side: pre-split bucket sums, [tiles_x][stages of the chunk][16 KB]
    int64_t chunk, cb;    // chunk index, buckets per chunk (a multiple of 2 kBK)
    const uint8_t *H;     // y side: pre-split row twiddles E_y[n, y_b], [tiles_y][stages][16 KB]
};

// item -> bucket range of the chunk, split at stage (kBK-bucket) boundaries
template <int kBKp>
__device__ __forceinline__ ItemInfo item_info_chunk(const CornerSrc &src, const GemmPlan &plan, const TcChunk &ch,
                                                    int64_t item, int64_t &chunk0) {
    const int64_t per_clip = (int64_t)plan.tiles_x * plan.tiles_y * plan.splits;
    int64_t rem = item % per_clip;
    ItemInfo it;
    it.tix = (int)(rem / ((int64_t)plan.tiles_y * plan.splits));
    rem -= (int64_t)it.tix * plan.tiles_y * plan.splits;
    it.tiy = (int)(rem / plan.splits);
    const int split = (int)(rem - (int64_t)it.tiy * plan.splits);
    chunk0 = src.clip_bptr[0] + ch.chunk * ch.cb;
    int64_t ke = src.clip_bptr[1];
    if (ke > chunk0 + ch.cb) ke = chunk0 + ch.cb;
    const int64_t nst = ke > chunk0 ? (ke - chunk0 + kBKp - 1) / kBKp : 0;
    it.k0 = chunk0 + kBKp * (nst * split / plan.splits);
    it.k1 = chunk0 + kBKp * (nst * (split + 1) / plan.splits);
    if (it.k1 > ke) it.k1 = ke;
    if (it.k0 > it.k1) it.k0 = it.k1;
    return it;
}

__device__ __forceinline__ ItemInfo item_info(const CornerSrc &src, const GemmPlan &plan, int64_t item) {
    const int64_t per_clip = (int64_t)plan.tiles_x * plan.tiles_y * plan.splits;
    const int64_t clip = item / per_clip;
    int64_t rem = item - clip * per_clip;
    ItemInfo it;
    it.tix = (int)(rem / ((int64_t)plan.tiles_y * plan.splits));
    rem -= (int64_t)it.tix * plan.tiles_y * plan.splits;
    it.tiy = (int)(rem / plan.splits);
    const int split = (int)(rem - (int64_t)it.tiy * plan.splits);
    int64_t kb, ke;
    if (src.corner_ptr) {
        kb = src.corner_ptr[clip];
        ke = src.ecnt ? kb + src.ecnt[clip] : src.corner_ptr[clip + 1];   // edge form: the clip's edges
    } else {
        kb = src.k_lo; ke = src.k_hi;
    }
    const int64_t span = ke - kb;
    it.k0 = kb + span * split / plan.splits;
    it.k1 = kb + span * (split + 1) / plan.splits;
    return it;
}

struct TabGeom {
    int32_t T, single, lbits, nhi, pow2;
};

// (cos, sin)(2 pi r / T) in fp32.  kFast: one-level table and power-of-two T (compile time).
template <bool kFast>
__device__ __forceinline__ float2 twiddle(uint32_t r, const TabGeom &g, const float2 *tab) {
    if (kFast || g.single) return tab[r];
    float2 a = tab[r >> g.lbits];
    float2 b = tab[g.nhi + (r & ((1u << g.lbits) - 1))];
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.y, b.x, a.x * b.y));
}

template <bool kFast>
__device__ __forceinline__ uint32_t phase(uint32_t f, uint32_t v, const TabGeom &g) {
    if (kFast || g.pow2) return (f * v) & (uint32_t)(g.T - 1);
    return (uint32_t)(((uint64_t)f * v) % (uint64_t)g.T);
}

// hi/lo split for the tensor core: hi keeps the top 10 mantissa bits (exact bit mask), lo = v - hi
// is exact in fp32 and is read by the MMA as tf32 (|lo| <= 2^-10 |v|: relative error <= 2^-20).
__device__ __forceinline__ void split(float v, float &hi, float &lo) {
    hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    lo = v - hi;
}

// ---- packed FP32x2 arithmetic (SASS FFMA2 / FMUL2): two independent lanes of work per instruction
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n mov.b64 rc, {%6, %7};\n"
        " fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;\n}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    float2 d;
    asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
        " mul.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    float2 d;
    asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
        " sub.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
// lo part of the hi/lo split for two values: v - (v with the low 13 mantissa bits cleared), exact
__device__ __forceinline__ float2 lo2(float2 v) {
    return sub2(v, make_float2(__uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u),
                               __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u)));
}
// (re, im) <- (re, im) (c + i s) for two independent values, one per FP32x2 lane:
// re' = re c - im s, im' = im c + re s (the same rounding sequence as the scalar fmaf form)
__device__ __forceinline__ void rot2(float2 &re, float2 &im, float2 c, float2 sn) {
    const float2 t = mul2(im, sn);
    const float2 u = mul2(re, sn);
    re = fma2(re, c, make_float2(-t.x, -t.y));
    im = fma2(im, c, u);
}

// (cos, sin)(2 pi r / T) on the SFU (MUFU.SIN/COS, |err| <~ 2^-21 on [-pi, pi]) instead of a table load
__device__ __forceinline__ float2 twiddle_sfu(uint32_t r, int32_t T, float w2pi) {
    int32_t rr = (int32_t)r;
    if (rr > (T >> 1)) rr -= T;
    float sn, cs;
    __sincosf((float)rr * w2pi, &sn, &cs);
    return make_float2(cs, sn);
}

// One producer task: 4 consecutive corners (16-byte chunk `quad` of the stage) x 8 consecutive
// pair slots (p0 .. p0+7) of one side.  (cos, sin)(f v) comes from an exact-phase table lookup
// for the first frequency, pre-multiplied by the corner weight, and the angle-addition
// recurrence E(f+1) = E(f) E(1) for the other 7.  The split values go straight into the SW128
// K-major operand tile: rows j0+i (cos hi), 32+j0+i (sin hi), 64+j0+i (cos lo), 96+j0+i (sin lo).
// The hi rows store v itself (the tf32 MMA reads only its top 19 bits, hi = v & 0xFFFFE000);
// the lo rows store the exact v - hi.  Padding slots (p > nf) keep recurrence values: they only
// feed P entries nobody reads.  The axis slot (p == nf) is overwritten with the coordinate weight.
// Bank use: a warp (one side) = 8 quads x 4 slot blocks; every STS.128 covers 4 full 128 B rows.
template <bool kFast, int kSlots = 8, bool kSfu = false>
__device__ __forceinline__ void produce(uint8_t *op, int quad, int j0, int p0, const SidePlan &sp,
                                        const int32_t v[4], const float wt[4], const TabGeom &g,
                                        const float2 *tab) {
    const uint32_t f0 = (uint32_t)(sp.f0 + p0);
    float4 re, im, c1, s1;
    {
        float2 a[4], e[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if constexpr (kSfu) {
                const float w2pi = 6.28318530717958647692f / (float)g.T;
                a[q] = twiddle_sfu(phase<kFast>(f0, (uint32_t)v[q], g), g.T, w2pi);
                e[q] = twiddle_sfu(phase<kFast>(1u, (uint32_t)v[q], g), g.T, w2pi);
            } else {
                a[q] = twiddle<kFast>(phase<kFast>(f0, (uint32_t)v[q], g), g, tab);
                e[q] = twiddle<kFast>(phase<kFast>(1u, (uint32_t)v[q], g), g, tab);
            }
        }
        re = make_float4(wt[0] * a[0].x, wt[1] * a[1].x, wt[2] * a[2].x, wt[3] * a[3].x);
        im = make_float4(wt[0] * a[0].y, wt[1] * a[1].y, wt[2] * a[2].y, wt[3] * a[3].y);
        c1 = make_float4(e[0].x, e[1].x, e[2].x, e[3].x);
        s1 = make_float4(e[0].y, e[1].y, e[2].y, e[3].y);
    }
    const uint32_t M13 = 0xFFFFE000u;
#pragma unroll
    for (int i = 0; i < kSlots; ++i) {
        const float2 rl01 = lo2(make_float2(re.x, re.y)), rl23 = lo2(make_float2(re.z, re.w));
        const float2 il01 = lo2(make_float2(im.x, im.y)), il23 = lo2(make_float2(im.z, im.w));
        const float4 rl = make_float4(rl01.x, rl01.y, rl23.x, rl23.y), il = make_float4(il01.x, il01.y, il23.x, il23.y);
        // row j0 + i; 8-slot blocks start on an 8-row atom (j0 % 8 == 0): r % 8 == i
        const int r7 = kSlots == 8 ? i : ((j0 + i) & 7);
        uint8_t *base = op + (kSlots == 8 ? (j0 >> 3) : ((j0 + i) >> 3)) * 1024 + r7 * kRowBytes + ((quad ^ r7) << 4);
        *(float4 *)(base) = re;                    // row r
        *(float4 *)(base + 4 * 1024) = im;         // row 32 + r
        *(float4 *)(base + 8 * 1024) = rl;         // row 64 + r
        *(float4 *)(base + 12 * 1024) = il;        // row 96 + r
        if (i < kSlots - 1) {   // packed: corners (0, 1) and (2, 3) per instruction
            float2 r01 = make_float2(re.x, re.y), r23 = make_float2(re.z, re.w);
            float2 i01 = make_float2(im.x, im.y), i23 = make_float2(im.z, im.w);
            rot2(r01, i01, make_float2(c1.x, c1.y), make_float2(s1.x, s1.y));
            rot2(r23, i23, make_float2(c1.z, c1.w), make_float2(s1.z, s1.w));
            re = make_float4(r01.x, r01.y, r23.x, r23.y);
            im = make_float4(i01.x, i01.y, i23.x, i23.y);
        }
    }
    const int ia = sp.nf - p0;
    if (sp.axis && ia >= 0 && ia < kSlots) {
        float4 c, cl;
        c = make_float4(wt[0] * (float)v[0], wt[1] * (float)v[1], wt[2] * (float)v[2], wt[3] * (float)v[3]);
        cl.x = c.x - __uint_as_float(__float_as_uint(c.x) & M13);
        cl.y = c.y - __uint_as_float(__float_as_uint(c.y) & M13);
        cl.z = c.z - __uint_as_float(__float_as_uint(c.z) & M13);
        cl.w = c.w - __uint_as_float(__float_as_uint(c.w) & M13);
        const int r7 = (j0 + ia) & 7;
        uint8_t *base = op + ((j0 + ia) >> 3) * 1024 + r7 * kRowBytes + ((quad ^ r7) << 4);
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        *(float4 *)(base) = c;
        *(float4 *)(base + 4 * 1024) = z;
        *(float4 *)(base + 8 * 1024) = cl;
        *(float4 *)(base + 12 * 1024) = z;
    }
}

// Edge-form producer task (kEdge, edges.cu): 4 consecutive edges x kSlots pair slots of the x side.
// Edge (x_a, x_b, c) contributes c (E(f x_a) - E(f x_b)); both ends run their own angle-addition
// recurrence and the difference is split and stored exactly like a corner's value (x_b < 0: one
// end).  The axis slot carries c (x_a - x_b) (an exact integer, |.| < 2^24).
template <bool kFast, int kSlots, bool kSfu = false>
__device__ __forceinline__ void produce_edge(uint8_t *op, int quad, int j0, int p0, const SidePlan &sp,
                                             const int32_t xa[4], const int32_t xb[4], const int32_t c[4],
                                             const TabGeom &g, const float2 *tab) {
    const uint32_t f0 = (uint32_t)(sp.f0 + p0);
    float2 ra01, ra23, ia01, ia23, rb01, rb23, ib01, ib23;   // end a / end b, edges (0,1) and (2,3)
    float2 ca01, ca23, sa01, sa23, cb01, cb23, sb01, sb23;
    {
        float2 a[4], e[4], bb[4], eb[4];
        float wa[4], wb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t vb = xb[q] >= 0 ? (uint32_t)xb[q] : 0u;
            if constexpr (kSfu) {
                const float w2pi = 6.28318530717958647692f / (float)g.T;
                a[q] = twiddle_sfu(phase<kFast>(f0, (uint32_t)xa[q], g), g.T, w2pi);
                bb[q] = twiddle_sfu(phase<kFast>(f0, vb, g), g.T, w2pi);
                e[q] = twiddle_sfu(phase<kFast>(1u, (uint32_t)xa[q], g), g.T, w2pi);
                eb[q] = twiddle_sfu(phase<kFast>(1u, vb, g), g.T, w2pi);
            } else {
                a[q] = twiddle<kFast>(phase<kFast>(f0, (uint32_t)xa[q], g), g, tab);
                bb[q] = twiddle<kFast>(phase<kFast>(f0, vb, g), g, tab);
                e[q] = twiddle<kFast>(phase<kFast>(1u, (uint32_t)xa[q], g), g, tab);
                eb[q] = twiddle<kFast>(phase<kFast>(1u, vb, g), g, tab);
            }
            wa[q] = (float)c[q];
            wb[q] = xb[q] >= 0 ? (float)c[q] : 0.f;
        }
        ra01 = make_float2(wa[0] * a[0].x, wa[1] * a[1].x); ra23 = make_float2(wa[2] * a[2].x, wa[3] * a[3].x);
        ia01 = make_float2(wa[0] * a[0].y, wa[1] * a[1].y); ia23 = make_float2(wa[2] * a[2].y, wa[3] * a[3].y);
        rb01 = make_float2(wb[0] * bb[0].x, wb[1] * bb[1].x); rb23 = make_float2(wb[2] * bb[2].x, wb[3] * bb[3].x);
        ib01 = make_float2(wb[0] * bb[0].y, wb[1] * bb[1].y); ib23 = make_float2(wb[2] * bb[2].y, wb[3] * bb[3].y);
        ca01 = make_float2(e[0].x, e[1].x); ca23 = make_float2(e[2].x, e[3].x);
        sa01 = make_float2(e[0].y, e[1].y); sa23 = make_float2(e[2].y, e[3].y);
        cb01 = make_float2(eb[0].x, eb[1].x); cb23 = make_float2(eb[2].x, eb[3].x);
        sb01 = make_float2(eb[0].y, eb[1].y); sb23 = make_float2(eb[2].y, eb[3].y);
    }
    const uint32_t M13 = 0xFFFFE000u;
#pragma unroll
    for (int i = 0; i < kSlots; ++i) {
        const float4 re = make_float4(ra01.x - rb01.x, ra01.y - rb01.y, ra23.x - rb23.x, ra23.y - rb23.y);
        const float4 im = make_float4(ia01.x - ib01.x, ia01.y - ib01.y, ia23.x - ib23.x, ia23.y - ib23.y);
        float4 rl, il;
        rl.x = re.x - __uint_as_float(__float_as_uint(re.x) & M13);
        rl.y = re.y - __uint_as_float(__float_as_uint(re.y) & M13);
        rl.z = re.z - __uint_as_float(__float_as_uint(re.z) & M13);
        rl.w = re.w - __uint_as_float(__float_as_uint(re.w) & M13);
        il.x = im.x - __uint_as_float(__float_as_uint(im.x) & M13);
        il.y = im.y - __uint_as_float(__float_as_uint(im.y) & M13);
        il.z = im.z - __uint_as_float(__float_as_uint(im.z) & M13);
        il.w = im.w - __uint_as_float(__float_as_uint(im.w) & M13);
        const int r7 = (j0 + i) & 7;
        uint8_t *base = op + ((j0 + i) >> 3) * 1024 + r7 * kRowBytes + ((quad ^ r7) << 4);
        *(float4 *)(base) = re;
        *(float4 *)(base + 4 * 1024) = im;
        *(float4 *)(base + 8 * 1024) = rl;
        *(float4 *)(base + 12 * 1024) = il;
        if (i < kSlots - 1) {
            rot2(ra01, ia01, ca01, sa01);
            rot2(ra23, ia23, ca23, sa23);
            rot2(rb01, ib01, cb01, sb01);
            rot2(rb23, ib23, cb23, sb23);
        }
    }
    const int ia = sp.nf - p0;
    if (sp.axis && ia >= 0 && ia < kSlots) {
        float4 v, vl;
        v.x = (float)(c[0] * (xa[0] - (xb[0] >= 0 ? xb[0] : 0)));
        v.y = (float)(c[1] * (xa[1] - (xb[1] >= 0 ? xb[1] : 0)));
        v.z = (float)(c[2] * (xa[2] - (xb[2] >= 0 ? xb[2] : 0)));
        v.w = (float)(c[3] * (xa[3] - (xb[3] >= 0 ? xb[3] : 0)));
        vl.x = v.x - __uint_as_float(__float_as_uint(v.x) & M13);
        vl.y = v.y - __uint_as_float(__float_as_uint(v.y) & M13);
        vl.z = v.z - __uint_as_float(__float_as_uint(v.z) & M13);
        vl.w = v.w - __uint_as_float(__float_as_uint(v.w) & M13);
        const int r7 = (j0 + ia) & 7;
        uint8_t *base = op + ((j0 + ia) >> 3) * 1024 + r7 * kRowBytes + ((quad ^ r7) << 4);
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        *(float4 *)(base) = v;
        *(float4 *)(base + 4 * 1024) = z;
        *(float4 *)(base + 8 * 1024) = vl;
        *(float4 *)(base + 12 * 1024) = z;
    }
}

__device__ __forceinline__ uint32_t pack_h2(float lo_elem, float hi_elem) {
    __half2 h = __floats2half2_rn(lo_elem, hi_elem);   // .x (low 16 bits) = the lower K index
    return *(uint32_t *)&h;
}

// FP16 producer task: 8 consecutive corners (16-byte chunk `oct` of the 64-corner stage) x 8
// consecutive pair slots of one side.  hi = v with the mantissa cut to 10 bits (exact in fp16 for
// normal values), lo = fp16(v - hi): |v - (hi + lo)| <= 2^-22 |v| + 2^-25 (fp16 subnormal step).
// The axis slot carries the coordinate weight scaled by axs = 2^-s (exact) to stay in fp16
// range; the epilogue multiplies the axis row / column of P back by 2^s.
template <bool kFast, int kSlots = 8>
__device__ __forceinline__ void produce_f16(uint8_t *op, int oct, int j0, int p0, const SidePlan &sp,
                                            const int32_t v[8], const float wt[8], float axs, const TabGeom &g,
                                            const float2 *tab) {
    const uint32_t f0 = (uint32_t)(sp.f0 + p0);
    float re[8], im[8], c1[8], s1[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const float2 a = twiddle<kFast>(phase<kFast>(f0, (uint32_t)v[q], g), g, tab);
        const float2 e = twiddle<kFast>(phase<kFast>(1u, (uint32_t)v[q], g), g, tab);
        re[q] = wt[q] * a.x;
        im[q] = wt[q] * a.y;
        c1[q] = e.x;
        s1[q] = e.y;
    }
    const uint32_t M13 = 0xFFFFE000u;
#pragma unroll
    for (int i = 0; i < kSlots; ++i) {
        uint32_t hc[4], hs[4], lc[4], ls[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const float r0 = re[2 * h], r1 = re[2 * h + 1], i0 = im[2 * h], i1 = im[2 * h + 1];
            const float mr0 = __uint_as_float(__float_as_uint(r0) & M13), mr1 = __uint_as_float(__float_as_uint(r1) & M13);
            const float mi0 = __uint_as_float(__float_as_uint(i0) & M13), mi1 = __uint_as_float(__float_as_uint(i1) & M13);
            hc[h] = pack_h2(mr0, mr1);
            hs[h] = pack_h2(mi0, mi1);
            lc[h] = pack_h2(r0 - mr0, r1 - mr1);
            ls[h] = pack_h2(i0 - mi0, i1 - mi1);
        }
        const int r7 = kSlots == 8 ? i : ((j0 + i) & 7);
        uint8_t *base = op + (kSlots == 8 ? (j0 >> 3) : ((j0 + i) >> 3)) * 1024 + r7 * kRowBytes + ((oct ^ r7) << 4);
        *(uint4 *)(base) = make_uint4(hc[0], hc[1], hc[2], hc[3]);
        *(uint4 *)(base + 4 * 1024) = make_uint4(hs[0], hs[1], hs[2], hs[3]);
        *(uint4 *)(base + 8 * 1024) = make_uint4(lc[0], lc[1], lc[2], lc[3]);
        *(uint4 *)(base + 12 * 1024) = make_uint4(ls[0], ls[1], ls[2], ls[3]);
        if (i < kSlots - 1) {   // scalar here: the packed form spills at this register budget
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const float nr = fmaf(re[q], c1[q], -im[q] * s1[q]);
                const float ni = fmaf(im[q], c1[q], re[q] * s1[q]);
                re[q] = nr;
                im[q] = ni;
            }
        }
    }
    const int ia = sp.nf - p0;
    if (sp.axis && ia >= 0 && ia < kSlots) {
        uint32_t hc[4], lc[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const float c0 = wt[2 * h] * (float)v[2 * h] * axs, cc1 = wt[2 * h + 1] * (float)v[2 * h + 1] * axs;
            const float m0 = __uint_as_float(__float_as_uint(c0) & M13), m1 = __uint_as_float(__float_as_uint(cc1) & M13);
            hc[h] = pack_h2(m0, m1);
            lc[h] = pack_h2(c0 - m0, cc1 - m1);
        }
        const int r7 = (j0 + ia) & 7;
        uint8_t *base = op + ((j0 + ia) >> 3) * 1024 + r7 * kRowBytes + ((oct ^ r7) << 4);
        const uint4 z = make_uint4(0u, 0u, 0u, 0u);
        *(uint4 *)(base) = make_uint4(hc[0], hc[1], hc[2], hc[3]);
        *(uint4 *)(base + 4 * 1024) = z;
        *(uint4 *)(base + 8 * 1024) = make_uint4(lc[0], lc[1], lc[2], lc[3]);
        *(uint4 *)(base + 12 * 1024) = z;
    }
}

// kLoadA (tf32 only, single clip, row buckets): the x-side stage tile is a 16 KB bulk copy from the
// chunk's pre-split bucket sums (k_gsum_tc) issued by the group's x-side warp; the y-side warp
// generates one twiddle set per bucket (the bucket's row y); P tiles are ADDED into P_ws.
// kEdge (tf32, batched, edges.cu): stages of 32 edges; both warps of a group make both sides
// (16 slots each, 4 per lane): the x side evaluates both ends of each edge, the y side one twiddle.
template <bool kFast, int kF16, bool kLoadA = false, bool kEdge = false>
__global__ void __launch_bounds__(kThreads, 1)
k_gemm_tf32(CornerSrc src, GemmPlan plan, TabGeom g, double *__restrict__ P_ws, EpiArgs ea, void *F, int fuse,
            int axis_shift, TcChunk ch) {
    if (kLoadA && src.clip_bptr[0] + ch.chunk * ch.cb >= src.clip_bptr[1]) return;   // chunk past the buckets
    constexpr int kBKp = kF16 ? 2 * kBK : kBK;          // corners per stage (one 128 B row of K)
    constexpr int kCq = kF16 ? 8 : 4;                    // corners per 16-byte chunk (per producer task)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-align by offset arithmetic on the __shared__ array (keeps the shared address space, so
    // loads / stores compile to LDS / STS rather than generic LD / ST)
    uint8_t *smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    const int tab_entries = kEdge ? 0 : (g.single ? g.T : g.nhi + (1 << g.lbits));   // edge: SFU twiddles
    constexpr int kS = kLoadA ? kStagesLoadA : (kEdge ? kStagesEdge : kStages);   // operand ring depth
    const Smem L = smem_layout(tab_entries, kS, !kLoadA);
    float2 *tab = (float2 *)(smem + L.table);
    float *xbuf = (float *)(smem + L.xbuf);
    uint64_t *bars = (uint64_t *)(smem + L.bars);
    // barrier indices: full[0..S), empty[S..2S), tfull[2S..2S+2), tempty[2S+2..2S+4)
    uint32_t *tmem_slot = (uint32_t *)(bars + 2 * kS + 4);
    int32_t *rowoff = (int32_t *)(smem + L.bars + kBarBytes);   // fused pupil layout: output offset per row
    // fused output tables: scale factors per |m| / |n| and the packed (m, n) of every output
    double *f_rows = (double *)(smem + L.bars + kBarBytes + 4 * (kMaxFuseRows + 2));   // -1/(4 pi^2 a)
    double *f_invn = f_rows + kMaxFuseRows;                                      // 1/b
    double *f_axm = f_invn + kMaxFuseRows;                                       // 1/(2 pi a T)
    uint32_t *f_mn = (uint32_t *)(f_axm + kMaxFuseRows);                        // (m+M) << 16 | (n+N), bit 31: masked
    const uint32_t bar0 = su32(bars);
    auto FULL = [&](int s) { return bar0 + 8u * s; };
    auto EMPTY = [&](int s) { return bar0 + 8u * (kS + s); };
    auto TFULL = [&](int b) { return bar0 + 8u * (2 * kS + b); };
    auto TEMPTY = [&](int b) { return bar0 + 8u * (2 * kS + 2 + b); };

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int tr = ABL(256);

    // twiddle table (all threads), barriers (thread 0), TMEM (MMA warp)
    for (int i = tid; i < tab_entries; i += kThreads) {
        double sn, cs;
        if (g.single) sincospi(2.0 * (double)i / (double)g.T, &sn, &cs);
        else if (i < g.nhi) sincospi(2.0 * (double)((int64_t)i << g.lbits) / (double)g.T, &sn, &cs);
        else sincospi(2.0 * (double)(i - g.nhi) / (double)g.T, &sn, &cs);
        tab[i] = make_float2((float)cs, (float)sn);
    }
    if (tid == 0 && fuse) {
        // output offset of each row m = -M..M (pupil: 2 nmax(m) + 1 entries, dense: 2N + 1)
        int32_t off = 0;
        for (int i = 0; i <= 2 * ea.M; ++i) {
            rowoff[i] = off;
            const int c = ea.layout == FCFS_LAYOUT_PUPIL ? pupil_nmax(i - ea.M, ea.r2, ea.N) : ea.N;
            off += c < 0 ? 0 : 2 * c + 1;
        }
        rowoff[2 * ea.M + 1] = off;
    }
    if (tid == 0) {
        // FULL: one arrive per producer warp (after every lane's proxy fence + __syncwarp)
        // FULL: one arrive per producer warp of the group (+ the x-side bulk copy's expect_tx in kLoadA)
        for (int s = 0; s < kS; ++s) { mbar_init(FULL(s), kLoadA ? 1 : kProdWarps / kGroups); mbar_init(EMPTY(s), 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(TFULL(b), 1); mbar_init(TEMPTY(b), kEpiWarps * 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async();
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (fuse) {
        const double pi = 3.141592653589793238462643383279502884;
        for (int a = tid; a < kMaxFuseRows; a += kThreads) {
            f_rows[a] = a ? -1.0 / (4.0 * pi * pi * (double)a) : 0.0;
            f_invn[a] = a ? 1.0 / (double)a : 0.0;
            f_axm[a] = a ? 1.0 / (2.0 * pi * (double)a * (double)ea.T) : 0.0;
        }
        // packed (m, n) of every output, row by row (rows in the layout's order)
        for (int i = 0; i <= 2 * ea.M; ++i) {
            const int cnt = rowoff[i + 1] - rowoff[i];
            const int h = (cnt - 1) / 2;
            for (int j = tid; j < cnt; j += kThreads) {
                const int m = i - ea.M, n = j - h;
                uint32_t pk = ((uint32_t)(m + ea.M) << 16) | (uint32_t)(n + ea.N);
                if (ea.layout == FCFS_LAYOUT_DENSE && ea.r2 >= 0.0 &&
                    (double)m * (double)m + (double)n * (double)n > ea.r2)
                    pk |= 0x80000000u;
                f_mn[rowoff[i] + j] = pk;
            }
        }
        __syncthreads();
    }

    if (warp >= kEpiWarps && warp < kMmaWarp) {
        // ============================== producers ==============================
        // group gq = warps (4 + 2 gq, 5 + 2 gq) fills stages sc = gq (mod 4) into ring slot sc % 5.
        // Warp = one side (A: x-side weighted, B: y-side); lane -> (corner quad, 8-slot block).
        const int pt = tid - kEpiWarps * 32;
        const int gq = pt >> 6;
        const int sideB = (pt >> 5) & 1;
        const int l = pt & 31;
        // kLoadA: both warps of a group make the y side (16 slots each, 4 per lane); lane 0 of warp 0
        // also issues the x-side bulk copy
        const int quad = l & 7;                           // quad: 16-byte chunk of the stage
        const int j0 = (kLoadA || kEdge) ? 16 * sideB + 4 * (l >> 3) : (l >> 3) << 3;
        const float axs = ldexpf(1.0f, -axis_shift);
        const bool yside = kLoadA || sideB;
        const SidePlan sp = yside ? plan.Y : plan.X;
        const int32_t *vsrc = kLoadA ? src.by : (sideB ? src.y : src.x);
        const int64_t nst_chunk = kLoadA ? ch.cb / kBKp : 0;
        uint32_t sc = 0;                                  // global stage counter
        int slot = 0;                                     // sc % kStages
        uint32_t ph = 0;                                  // (sc / kStages) & 1
        for (int64_t item = blockIdx.x; item < plan.items; item += gridDim.x) {
            int64_t chunk0 = 0;
            const ItemInfo it = kLoadA ? item_info_chunk<kBKp>(src, plan, ch, item, chunk0) : item_info(src, plan, item);
            const int p0 = (yside ? it.tiy : it.tix) * 32 + j0;
            const int p0x = it.tix * 32 + j0, p0y = it.tiy * 32 + j0;   // kEdge: both sides
            for (int64_t c0 = it.k0; c0 < it.k1; c0 += kChunk) {
                const int64_t c1 = c0 + kChunk < it.k1 ? c0 + kChunk : it.k1;
                // 32-bit corner offsets relative to the chunk base; one-own-stage-ahead prefetch
                const int n = (int)(c1 - c0);
                const int32_t *vp = vsrc + c0;
                const int32_t *wp = src.w + c0;
                const int first = (gq - (int)(sc & 3)) & 3;
                int32_t vn[kCq], wn[kCq];
                int32_t an[kEdge ? 4 : 1], bn[kEdge ? 4 : 1];   // kEdge: x_a, x_b (vn = y, wn = c)
                auto fetch = [&](int kr0) {
#pragma unroll
                    for (int q = 0; q < kCq; ++q) {
                        const int kr = kr0 + q;
                        const bool ok = kr < n;
                        if constexpr (kEdge) {
                            an[q] = ok ? __ldg(src.exa + c0 + kr) : 0;
                            bn[q] = ok ? __ldg(src.exb + c0 + kr) : -1;
                            vn[q] = ok ? __ldg(src.ey + c0 + kr) : 0;
                            wn[q] = ok ? __ldg(src.ec + c0 + kr) : 0;
                        } else {
                            vn[q] = ok ? __ldg(vp + kr) : 0;
                            wn[q] = ok ? (yside ? 1 : __ldg(wp + kr)) : 0;
                        }
                    }
                };
                int kr0 = first * kBKp + kCq * quad;
                fetch(kr0);
                for (int64_t ks = c0; ks < c1; ks += kBKp, ++sc) {
                    const int my_slot = slot;
                    FCFS_DCHECK(my_slot >= 0 && my_slot < kS && n >= 1 && n <= kChunk);
                    const uint32_t my_ph = ph;
                    if (++slot == kS) { slot = 0; ph ^= 1; }
                    if ((int)(sc & 3) != gq) continue;
                    // corner data 16 stages ahead -> L2 (the register prefetch below is only one own
                    // stage = 4 stages ahead, about one HBM latency): one line per lane, per array
                    // edge form: no L2 prefetch — the edges were just written by k_edges and the
                    // prefetch instructions cost more issue slots than they saved (0.997 vs 1.027 ms)
                    if (!kEdge && !kLoadA && !(ABL(128))) {
                        constexpr int kLines = kBKp * 4 / 128;          // 128-byte lines per array per stage
                        const int64_t kp = ks + 16 * kBKp + (int64_t)(l % kLines) * 32;
                        if (l < (yside ? 1 : 2) * kLines && kp < it.k1) {
                            const int32_t *pa = (yside || l < kLines) ? vsrc : src.w;
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(pa + kp));
                        }
                    }
                    int32_t v[kCq];
                    float wt[kCq];
                    int32_t xa[kEdge ? 4 : 1], xb[kEdge ? 4 : 1], ci[kEdge ? 4 : 1];
#pragma unroll
                    for (int q = 0; q < kCq; ++q) {
                        v[q] = vn[q];
                        wt[q] = kEdge ? 1.f : (float)wn[q];
                        if constexpr (kEdge) { xa[q] = an[q]; xb[q] = bn[q]; ci[q] = wn[q]; }
                    }
                    kr0 += kGroups * kBKp;
                    if (!(ABL(16))) fetch(kr0);
                    if (l == 0) trace(tr, 10 + gq * 2 + sideB, sc);
                    mbar_wait(EMPTY(my_slot), my_ph ^ 1, ABL(32));
                    if (l == 0) trace(tr, 20 + gq * 2 + sideB, sc);
                    uint8_t *op = smem + L.stage0 + my_slot * kStageBytes + (yside ? kOpBytes : 0);
                    if (kLoadA) {
                        // both operand tiles of the stage are precomputed (k_gsum_tc / k_hsum_tc): one
                        // lane issues the two 16 KB bulk copies; its expect_tx is the only arrival on
                        // FULL and the copies' bytes complete the phase.  The tiles 16 stages ahead are
                        // prefetched into L2, so the copies that must wait for the slot find them on chip.
                        if (!sideB && l == 0) {
                            const int64_t sti = (ks - chunk0) / kBKp;
                            const uint8_t *gsrc = ch.G + ((int64_t)it.tix * nst_chunk + sti) * kOpBytes;
                            const uint8_t *hsrc = ch.H + ((int64_t)it.tiy * nst_chunk + sti) * kOpBytes;
                            mbar_expect_tx(FULL(my_slot), 2 * kOpBytes);
                            bulk_g2s(su32(op - kOpBytes), gsrc, kOpBytes, FULL(my_slot));
                            bulk_g2s(su32(op), hsrc, kOpBytes, FULL(my_slot));
                            if (ks + 16 * kBKp < it.k1) {
                                prefetch_l2(gsrc + 16 * kOpBytes, kOpBytes);
                                prefetch_l2(hsrc + 16 * kOpBytes, kOpBytes);
                            }
                        }
                        __syncwarp();
                        continue;
                    }
                    if (!(ABL(1))) {
                        constexpr int kSl = (kLoadA || kEdge) ? 4 : 8;
                        if constexpr (kEdge) {
                            uint8_t *opx = smem + L.stage0 + my_slot * kStageBytes;
                            produce_edge<kFast, 4, true>(opx, quad, j0, p0x, plan.X, xa, xb, ci, g, tab);
                            produce<kFast, 4, true>(opx + kOpBytes, quad, j0, p0y, plan.Y, (const int32_t *)v,
                                              (const float *)wt, g, tab);
                        } else if constexpr (kF16) {
                            produce_f16<kFast, kSl>(op, quad, j0, p0, sp, v, wt, axs, g, tab);
                        } else {
                            produce<kFast, kSl>(op, quad, j0, p0, sp, (const int32_t *)v, (const float *)wt, g, tab);
                        }
                    }
                    if (!(ABL(8))) fence_proxy_async();
                    __syncwarp();
                    if (l == 0) { trace(tr, 30 + gq * 2 + sideB, sc); mbar_arrive(FULL(my_slot)); }
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ============================== MMA issuer ==============================
        // The whole warp runs the (warp-uniform) loop and waits; one elected lane issues the
        // MMAs and commits.  Descriptors are built once; a stage only adds its address offset.
        {
            int stage = 0;
            uint32_t phase_bit = 0;
            uint32_t chunk_ctr = 0;
            uint32_t msc = 0;
            const uint32_t smem_base = su32(smem + L.stage0);
            const uint64_t adesc0 = umma_desc(smem_base), bdesc0 = umma_desc(smem_base + kOpBytes);
            const bool no_mma = (ABL(2)) != 0;
            for (int64_t item = blockIdx.x; item < plan.items; item += gridDim.x) {
                int64_t chunk0 = 0;
            const ItemInfo it = kLoadA ? item_info_chunk<kBKp>(src, plan, ch, item, chunk0) : item_info(src, plan, item);
                for (int64_t c0 = it.k0; c0 < it.k1; c0 += kChunk, ++chunk_ctr) {
                    const int64_t c1 = c0 + kChunk < it.k1 ? c0 + kChunk : it.k1;
                    const uint32_t b = chunk_ctr & 1;
                    mbar_wait(TEMPTY(b), ((chunk_ctr >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + b * 128;
                    const int nst = (int)((c1 - c0 + kBKp - 1) / kBKp);   // stages in this chunk
                    // two stages per iteration: the barrier waits, fences and the elect are paid once
                    // per 8 MMAs, so the single issuing warp stays ahead of the tensor pipe
                    // kLoadA: one stage at a time (a slot is released as soon as its own MMAs complete:
                    // the bulk copies that refill it start earlier).  Per-corner mode: two stages per
                    // iteration, so the waits, fences and the elect are paid once per 8 MMAs.
                    constexpr int kPer = kLoadA ? 1 : 2;
                    for (int st = 0; st < nst; st += kPer) {
                        const int two = (kPer == 2 && st + 1 < nst) ? 1 : 0;
                        const int s1 = (stage + 1 == kS) ? 0 : stage + 1;
                        const uint32_t p1 = (stage + 1 == kS) ? phase_bit ^ 1 : phase_bit;
                        FCFS_DCHECK(stage >= 0 && stage < kS && s1 >= 0 && s1 < kS && nst >= 1);
                        mbar_wait(FULL(stage), phase_bit, ABL(64));
                        if (two) mbar_wait(FULL(s1), p1, ABL(64));
                        if (lane == 0) trace(tr, 50, msc);
                        tc_fence_after();
                        const uint64_t off0 = (uint64_t)((stage * kStageBytes) >> 4);
                        const uint64_t off1 = (uint64_t)((s1 * kStageBytes) >> 4);
                        if (elect_one()) {
                            if (!no_mma) {
#pragma unroll
                                for (int u = 0; u < 4; ++u)   // 4 MMAs of 32 B of K (8 tf32 / 16 fp16)
                                    umma<kF16>(d_tmem, adesc0 + off0 + 2 * u, bdesc0 + off0 + 2 * u,
                                               (st > 0 || u > 0) ? 1u : 0u);
                            }
                            umma_commit(EMPTY(stage));
                            if (two) {
                                if (!no_mma) {
#pragma unroll
                                    for (int u = 0; u < 4; ++u)
                                        umma<kF16>(d_tmem, adesc0 + off1 + 2 * u, bdesc0 + off1 + 2 * u, 1u);
                                }
                                umma_commit(EMPTY(s1));
                            }
                        }
                        __syncwarp();
                        msc += 1 + two;
                        stage = two ? s1 : stage;
                        phase_bit = two ? p1 : phase_bit;
                        if (++stage == kS) { stage = 0; phase_bit ^= 1; }
                    }
                    if (elect_one()) umma_commit(TFULL(b));
                    __syncwarp();
                }
            }
        }
    } else {
        // ============================== epilogue ==============================
        const int L_ = tid;                          // TMEM lane = D row
        const int hi_row = L_ < 64;
        const int r = hi_row ? L_ : L_ - 64;         // physical P row in the 64-row tile
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        uint32_t chunk_ctr = 0;
        for (int64_t item = blockIdx.x; item < plan.items; item += gridDim.x) {
            int64_t chunk0 = 0;
            const ItemInfo it = kLoadA ? item_info_chunk<kBKp>(src, plan, ch, item, chunk0) : item_info(src, plan, item);
            double acc[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = 0.0;
            for (int64_t c0 = it.k0; c0 < it.k1; c0 += kChunk, ++chunk_ctr) {
                const uint32_t b = chunk_ctr & 1;
                mbar_wait_sleep(TFULL(b), (chunk_ctr >> 1) & 1);
                tc_fence_after();
                if (ABL(4)) {
                    tc_fence_before();
                    mbar_arrive(TEMPTY(b));
                    continue;
                }
                const uint32_t tb = tmem_base + lane_base + b * 128;
                // D[L][c] + D[L][64+c] for the 32 columns this row keeps and the 32 it sends
                float *XH = xbuf, *XL = xbuf + 64 * kXStride;   // single buffer: barriers on both sides
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int col = 16 * q;          // columns col..col+15 (send half for q >= 2 if hi row)
                    uint32_t ra[16], rb[16];
                    TMEM_LD16(tb + col, ra);
                    TMEM_LD16(tb + 64 + col, rb);
                    tmem_wait_ld();
                    const bool keep = hi_row ? (q < 2) : (q >= 2);
                    float *xdst = hi_row ? XH : XL;
                    const int o = (q & 1) * 16;
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const float v = __uint_as_float(ra[i]) + __uint_as_float(rb[i]);
                        if (keep) acc[o + i] += (double)v;
                        else xdst[r * kXStride + o + i] = v;
                    }
                }
                tc_fence_before();
                mbar_arrive(TEMPTY(b));
                named_bar(1, kEpiWarps * 32);
                {
                    const float *xsrc = hi_row ? XL : XH;
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[i] += (double)xsrc[r * kXStride + i];
                }
                named_bar(1, kEpiWarps * 32);   // exchange buffer free for the next chunk / the P tile
            }
            if (kF16 && axis_shift) {   // undo the fp16 range scaling of the axis row / column
                const double up = ldexp(1.0, axis_shift);
                const int ax_l = (plan.X.axis && plan.X.nf / 32 == it.tix) ? plan.X.nf % 32 : -1;
                const int ay_l = (plan.Y.axis && plan.Y.nf / 32 == it.tiy) ? plan.Y.nf % 32 : -1;
                if (r == ax_l) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[i] *= up;
                }
                const int cb = hi_row ? 0 : 32;
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (cb + i == ay_l) acc[i] *= up;
            }
            if (ABL(4)) continue;
            if (!fuse) {
                double *out = P_ws + item * (int64_t)(kTile * kTile) + r * kTile + (hi_row ? 0 : 32);
                if (kLoadA) {   // chunk partials add up in P_ws (zeroed before the first chunk)
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        const double2 p = *(const double2 *)(out + i);
                        *(double2 *)(out + i) = make_double2(p.x + acc[i], p.y + acc[i + 1]);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 32; i += 2) *(double2 *)(out + i) = make_double2(acc[i], acc[i + 1]);
                }
                continue;
            }
            // ---- fused a4 + a5: P tile (fp32; |dP| <= 2^-24 of the per-term bound B) -> SMEM ->
            // this clip's outputs.  Same arithmetic as coeff_from_P (coeff.cuh) with the 1/(4 pi^2 m n)
            // and 1/(2 pi m T) factors taken from tables instead of divisions.
            float *Ps = xbuf;              // [64][65]
#pragma unroll
            for (int i = 0; i < 32; ++i) Ps[r * 65 + (hi_row ? 0 : 32) + i] = (float)acc[i];
            named_bar(1, kEpiWarps * 32);
            {
                const int64_t clip = item;
                const double dc = (double)(ea.area_dev ? ea.area_dev[clip] : ea.area_host) / ((double)ea.T * (double)ea.T);
                const int W = rowoff[2 * ea.M + 1];
                const int ax = plan.X.nf, ay = plan.Y.nf;          // axis pair slots (f0 == 1 here)
                void *Fc = ea.out_f32 ? (void *)((float2 *)F + clip * ea.out_per_clip)
                                      : (void *)((double2 *)F + clip * ea.out_per_clip);
                for (int o = tid; o < W; o += kEpiWarps * 32) {
                    const uint32_t pk = f_mn[o];
                    int m = (int)((pk >> 16) & 0x7FFF) - ea.M, n = (int)(pk & 0xFFFF) - ea.N;
                    double2 v = make_double2(0.0, 0.0);
                    if (!(pk & 0x80000000u)) {
                        if (m == 0 && n == 0) {
                            v = make_double2(dc, 0.0);
                        } else {
                            const bool neg = (m < 0) || (m == 0 && n < 0);
                            if (neg) { m = -m; n = -n; }
                            double re, im;
                            if (n == 0) {            // row c_m / s_m x axis column y (pair ay, t 0)
                                const int pm = m - 1;
                                const double sre = Ps[pm * 65 + ay], sim = -(double)Ps[(32 + pm) * 65 + ay];
                                re = -sim * f_axm[m]; im = sre * f_axm[m];
                            } else if (m == 0) {     // axis row x (pair ax) x columns c_n / s_n
                                const int pn = n - 1;
                                const double sre = Ps[ax * 65 + pn], sim = -(double)Ps[ax * 65 + 32 + pn];
                                re = -sim * f_axm[n]; im = sre * f_axm[n];   // 1/(2 pi n T)
                            } else {
                                const int an = n < 0 ? -n : n;
                                const int pm = m - 1, pn = an - 1;
                                const double pcc = Ps[pm * 65 + pn], pcs = Ps[pm * 65 + 32 + pn];
                                const double psc = Ps[(32 + pm) * 65 + pn], pss = Ps[(32 + pm) * 65 + 32 + pn];
                                double sre, sim;
                                if (n > 0) { sre = pcc - pss; sim = -(psc + pcs); }
                                else { sre = pcc + pss; sim = -(psc - pcs); }
                                const double sc = f_rows[m] * (n > 0 ? f_invn[an] : -f_invn[an]);
                                re = sre * sc; im = sim * sc;
                            }
                            v = make_double2(re, neg ? -im : im);
                        }
                    }
                    store_out(Fc, o, v, ea.out_f32);
                }
            }
            named_bar(1, kEpiWarps * 32);  // P tile consumed before the next item's chunk flush
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols)
                     : "memory");
    }
}

// x-side bucket sums of one chunk for every x tile, split hi/lo and stored in the exact SW128
// K-major stage layout of k_gemm_tf32<., kF16, true> (16 KB per (x tile, stage of 32 / 64 buckets)):
// G[f, b] = sum_{k in bucket b} w_k E(f x_k); the axis pair carries sum_k w_k x_k (x axs for fp16).
// A block builds the tiles of 64 buckets of one x tile in shared memory and writes them out
// coalesced; thread = (bucket, block of 8 pairs): per corner two exact-phase table lookups (E(f0 x),
// step E(x)) and the angle-addition recurrence over the 8 pairs, FP32 sums of <= 32 terms.
template <bool kFast, int kF16>
__global__ void __launch_bounds__(256)
k_gsum_tc(CornerSrc src, GemmPlan plan, TabGeom g, TcChunk ch, uint8_t *__restrict__ G, float axs) {
    if (src.clip_bptr[0] + ch.chunk * ch.cb >= src.clip_bptr[1]) return;   // chunk past the buckets
    constexpr int kBKp = kF16 ? 2 * kBK : kBK;   // buckets per stage tile
    constexpr int kTiles = 64 / kBKp;            // stage tiles per 64-bucket unit (tf32: 2, fp16: 1)
    extern __shared__ __align__(1024) uint8_t gsm_raw[];
    uint8_t *sm = gsm_raw + ((1024u - (su32(gsm_raw) & 1023u)) & 1023u);
    uint8_t *tile = sm;                                       // kTiles x 16 KB
    float2 *tab = (float2 *)(sm + 2 * kOpBytes);
    const int tab_entries = g.single ? g.T : g.nhi + (1 << g.lbits);
    for (int i = threadIdx.x; i < tab_entries; i += blockDim.x) {
        double sn, cs;
        if (g.single) sincospi(2.0 * (double)i / (double)g.T, &sn, &cs);
        else if (i < g.nhi) sincospi(2.0 * (double)((int64_t)i << g.lbits) / (double)g.T, &sn, &cs);
        else sincospi(2.0 * (double)(i - g.nhi) / (double)g.T, &sn, &cs);
        tab[i] = make_float2((float)cs, (float)sn);
    }
    __syncthreads();
    const int kk = threadIdx.x >> 2, pb = threadIdx.x & 3;   // bucket of the unit, 8-pair block
    const int64_t chunk0 = src.clip_bptr[0] + ch.chunk * ch.cb;
    int64_t ke = src.clip_bptr[1];
    if (ke > chunk0 + ch.cb) ke = chunk0 + ch.cb;
    if (chunk0 >= ke) return;
    const int64_t nunit = (ke - chunk0 + 63) / 64, nst_chunk = ch.cb / kBKp;
    const uint32_t M13 = 0xFFFFE000u;
    for (int64_t u = blockIdx.x; u < nunit * plan.tiles_x; u += gridDim.x) {
        const int tix = (int)(u % plan.tiles_x);
        const int64_t unit = u / plan.tiles_x;
        const int64_t b = chunk0 + unit * 64 + kk;
        const int p0 = tix * 32 + 8 * pb;                     // first pair (global) of the block
        const uint32_t f0 = (uint32_t)(plan.X.f0 + p0);
        float re[8], im[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { re[i] = 0.f; im[i] = 0.f; }
        float ax = 0.f;
        if (b < ke) {
            const int cb = __ldg(src.bptr + b), ce = __ldg(src.bptr + b + 1);
            for (int c = cb; c < ce; ++c) {
                const int32_t x = __ldg(src.x + c);
                const float wt = (float)__ldg(src.w + c);
                ax = fmaf(wt, (float)x, ax);
                const float2 a = twiddle<kFast>(phase<kFast>(f0, (uint32_t)x, g), g, tab);
                const float2 e = twiddle<kFast>(phase<kFast>(1u, (uint32_t)x, g), g, tab);
                float cr = wt * a.x, ci = wt * a.y;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    re[i] += cr;
                    im[i] += ci;
                    if (i < 7) {
                        const float nr = fmaf(cr, e.x, -ci * e.y);
                        const float ni = fmaf(ci, e.x, cr * e.y);
                        cr = nr;
                        ci = ni;
                    }
                }
            }
        }
        uint8_t *tl = tile + (kk / kBKp) * kOpBytes;          // stage tile of this bucket
        const int kq = kk % kBKp;                             // K position inside the tile
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int p = p0 + i, r = 8 * pb + i, r7 = r & 7;
            float vr = 0.f, vi = 0.f;
            if (p < plan.X.nf) { vr = re[i]; vi = im[i]; }
            else if (plan.X.axis && p == plan.X.nf) vr = ax * (kF16 ? axs : 1.f);
            const float hr = __uint_as_float(__float_as_uint(vr) & M13), hs = __uint_as_float(__float_as_uint(vi) & M13);
            if constexpr (!kF16) {
                uint8_t *base = tl + (r >> 3) * 1024 + r7 * kRowBytes + ((((kq >> 2) ^ r7)) << 4) + ((kq & 3) << 2);
                *(float *)(base) = vr;                        // cos hi row (the MMA reads the top 19 bits)
                *(float *)(base + 4 * 1024) = vi;             // sin hi
                *(float *)(base + 8 * 1024) = vr - hr;        // cos lo
                *(float *)(base + 12 * 1024) = vi - hs;       // sin lo
            } else {                                          // hi: 11 significant bits, exact in fp16
                uint8_t *base = tl + (r >> 3) * 1024 + r7 * kRowBytes + ((((kq >> 3) ^ r7)) << 4) + ((kq & 7) << 1);
                *(__half *)(base) = __float2half_rn(hr);
                *(__half *)(base + 4 * 1024) = __float2half_rn(hs);
                *(__half *)(base + 8 * 1024) = __float2half_rn(vr - hr);
                *(__half *)(base + 12 * 1024) = __float2half_rn(vi - hs);
            }
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < kTiles; ++t) {
            const int64_t st = unit * kTiles + t;             // stage index within the chunk
            if (st * kBKp >= ke - chunk0) break;
            uint4 *dst = (uint4 *)(G + ((int64_t)tix * nst_chunk + st) * kOpBytes);
            const uint4 *srct = (const uint4 *)(tile + t * kOpBytes);
            for (int i = threadIdx.x; i < kOpBytes / 16; i += blockDim.x) dst[i] = srct[i];
        }
        __syncthreads();
    }
}

// y-side row twiddles of one chunk for every y tile, split hi/lo, in the same stage layout:
// H[n, b] = E(n y_b) (one exact-phase table lookup per (bucket, pair)); the axis pair carries y_b.
template <bool kFast, int kF16>
__global__ void __launch_bounds__(256)
k_hsum_tc(CornerSrc src, GemmPlan plan, TabGeom g, TcChunk ch, uint8_t *__restrict__ H, float axs) {
    if (src.clip_bptr[0] + ch.chunk * ch.cb >= src.clip_bptr[1]) return;   // chunk past the buckets
    constexpr int kBKp = kF16 ? 2 * kBK : kBK;
    constexpr int kPerWarp = kBKp / 8;
    extern __shared__ __align__(1024) uint8_t hsm_raw[];
    uint8_t *sm = hsm_raw + ((1024u - (su32(hsm_raw) & 1023u)) & 1023u);
    uint8_t *tile = sm;
    float2 *tab = (float2 *)(sm + kOpBytes);
    const int tab_entries = g.single ? g.T : g.nhi + (1 << g.lbits);
    for (int i = threadIdx.x; i < tab_entries; i += blockDim.x) {
        double sn, cs;
        if (g.single) sincospi(2.0 * (double)i / (double)g.T, &sn, &cs);
        else if (i < g.nhi) sincospi(2.0 * (double)((int64_t)i << g.lbits) / (double)g.T, &sn, &cs);
        else sincospi(2.0 * (double)(i - g.nhi) / (double)g.T, &sn, &cs);
        tab[i] = make_float2((float)cs, (float)sn);
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t chunk0 = src.clip_bptr[0] + ch.chunk * ch.cb;
    int64_t ke = src.clip_bptr[1];
    if (ke > chunk0 + ch.cb) ke = chunk0 + ch.cb;
    const int64_t nst = (ke - chunk0 + kBKp - 1) / kBKp, nst_chunk = ch.cb / kBKp;
    const uint32_t M13 = 0xFFFFE000u;
    for (int64_t u = blockIdx.x; u < nst * plan.tiles_y; u += gridDim.x) {
        const int tiy = (int)(u % plan.tiles_y);
        const int64_t st = u / plan.tiles_y;
        const int pg = tiy * 32 + lane;
        const uint32_t f = (uint32_t)(plan.Y.f0 + pg);
        const bool tw = pg < plan.Y.nf, axis = plan.Y.axis && pg == plan.Y.nf;
#pragma unroll
        for (int q = 0; q < kPerWarp; ++q) {
            const int kk = kPerWarp * warp + q;
            const int64_t b = chunk0 + st * kBKp + kk;
            float re = 0.f, im = 0.f;
            if (b < ke) {
                const int32_t y = __ldg(src.by + b);
                if (tw) {
                    const float2 e = twiddle<kFast>(phase<kFast>(f, (uint32_t)y, g), g, tab);
                    re = e.x;
                    im = e.y;
                } else if (axis) {
                    re = (float)y * (kF16 ? axs : 1.f);
                }
            }
            const float hr = __uint_as_float(__float_as_uint(re) & M13), hs = __uint_as_float(__float_as_uint(im) & M13);
            const int r7 = lane & 7;
            if constexpr (!kF16) {
                uint8_t *base = tile + (lane >> 3) * 1024 + r7 * kRowBytes + ((((kk >> 2) ^ r7)) << 4) + ((kk & 3) << 2);
                *(float *)(base) = re;
                *(float *)(base + 4 * 1024) = im;
                *(float *)(base + 8 * 1024) = re - hr;
                *(float *)(base + 12 * 1024) = im - hs;
            } else {
                uint8_t *base = tile + (lane >> 3) * 1024 + r7 * kRowBytes + ((((kk >> 3) ^ r7)) << 4) + ((kk & 7) << 1);
                *(__half *)(base) = __float2half_rn(hr);
                *(__half *)(base + 4 * 1024) = __float2half_rn(hs);
                *(__half *)(base + 8 * 1024) = __float2half_rn(re - hr);
                *(__half *)(base + 12 * 1024) = __float2half_rn(im - hs);
            }
        }
        __syncthreads();
        uint4 *dst = (uint4 *)(H + ((int64_t)tiy * nst_chunk + st) * kOpBytes);
        const uint4 *srct = (const uint4 *)tile;
        for (int i = threadIdx.x; i < kOpBytes / 16; i += blockDim.x) dst[i] = srct[i];
        __syncthreads();
    }
}

}  // namespace tc

static tc::TabGeom make_tab(int32_t T) {
    tc::TabGeom g;
    g.T = T;
    g.pow2 = (T & (T - 1)) == 0;
    g.single = T <= tc::kSingleTableMax ? 1 : 0;
    int tb = ilog2_ceil(T);
    g.lbits = (tb + 1) / 2;
    g.nhi = (int32_t)((T + (1 << g.lbits) - 1) >> g.lbits);
    return g;
}

fcfs_status tf32_supported(const GemmPlan &plan, int32_t T) {
    (void)plan;
    if (T > (1 << 20)) {
        set_error("TF32X3: T=%d too large", T);
        return FCFS_E_UNSUPPORTED;
    }
    return FCFS_OK;
}

bool tf32_can_fuse(const GemmPlan &plan, const EpiArgs &ea) {
    return plan.tiles_x == 1 && plan.tiles_y == 1 && plan.splits == 1 && ea.m_lo == -ea.M && ea.m_hi == ea.M &&
           2 * ea.M + 1 < tc::kMaxFuseRows && 2 * ea.N + 1 < tc::kMaxFuseRows && plan.X.f0 == 1 &&
           plan.Y.f0 == 1;
}

fcfs_status launch_gemm_tf32(const CornerSrc &src, const GemmPlan &plan, int32_t T, double *P_ws, const EpiArgs *ea,
                             void *F, bool f16, cudaStream_t s) {
    if (plan.items <= 0) return FCFS_OK;
    const int fuse = (ea && F && tf32_can_fuse(plan, *ea)) ? 1 : 0;
    EpiArgs e{};
    if (ea) e = *ea;
    tc::TabGeom g = make_tab(T);
    const int entries = g.single ? g.T : g.nhi + (1 << g.lbits);
    const bool edge = src.ecnt != nullptr && !f16;
    const tc::Smem L = edge ? tc::smem_layout(0, tc::kStagesEdge) : tc::smem_layout(entries);
    const size_t smem = L.total + 1024;
    const bool fast = g.single && g.pow2;
    auto kern = f16 ? (fast ? tc::k_gemm_tf32<true, 1> : tc::k_gemm_tf32<false, 1>)
                    : edge ? (fast ? tc::k_gemm_tf32<true, 0, false, true> : tc::k_gemm_tf32<false, 0, false, true>)
                           : (fast ? tc::k_gemm_tf32<true, 0> : tc::k_gemm_tf32<false, 0>);
    FCFS_TRY(ensure_smem((const void *)kern, smem));
    // fp16 range: coordinate weights (<= T) of the axis slot are scaled by 2^-shift, T 2^-shift <= 256
    int shift = 0;
    if (f16) {
        const int tb = ilog2_ceil((int64_t)T + 1);
        shift = tb > 8 ? tb - 8 : 0;
    }
    int sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = plan.items < sms ? plan.items : sms;
    kern<<<(unsigned)grid, tc::kThreads, smem, s>>>(src, plan, g, P_ws, e, F, fuse, shift, tc::TcChunk{nullptr, 0, 0, nullptr});
    FCFS_CHECK_LAUNCH("k_gemm_tf32");
    return FCFS_OK;
}

int64_t tc_chunk_buckets(int64_t K) {   // a multiple of both stage sizes (32 tf32 / 64 fp16 buckets)
    int64_t cb = K < kFpChunkBuckets ? K : kFpChunkBuckets;
    cb = (cb + 2 * tc::kBK - 1) / (2 * tc::kBK) * (2 * tc::kBK);
    return cb < 2 * tc::kBK ? 2 * tc::kBK : cb;
}

// one clip over row buckets, split-TF32: per chunk of buckets, the x-side tiles once (k_gsum_tc),
// then the tcgen05 GEMM streaming them by bulk copy and adding into P_ws
fcfs_status launch_gemm_tf32_chunked(const CornerSrc &src, const GemmPlan &plan, int32_t T, int64_t K, uint8_t *G,
                                     uint8_t *H, double *P_ws, bool f16, cudaStream_t s) {
    if (plan.items <= 0) return FCFS_OK;
    FCFS_TRY_CUDA(cudaMemsetAsync(P_ws, 0, sizeof(double) * (size_t)plan.items * kTile * kTile, s));
    if (K <= 0) return FCFS_OK;
    tc::TabGeom g = make_tab(T);
    const int entries = g.single ? g.T : g.nhi + (1 << g.lbits);
    const tc::Smem L = tc::smem_layout(entries, tc::kStagesLoadA, false);
    const size_t smem = L.total + 1024;
    const size_t gsmem = 2 * tc::kOpBytes + 1024 + (size_t)entries * 8;
    const bool fast = g.single && g.pow2;
    auto kern = f16 ? (fast ? tc::k_gemm_tf32<true, 1, true> : tc::k_gemm_tf32<false, 1, true>)
                    : (fast ? tc::k_gemm_tf32<true, 0, true> : tc::k_gemm_tf32<false, 0, true>);
    auto gk = f16 ? (fast ? tc::k_gsum_tc<true, 1> : tc::k_gsum_tc<false, 1>)
                  : (fast ? tc::k_gsum_tc<true, 0> : tc::k_gsum_tc<false, 0>);
    auto hk = f16 ? (fast ? tc::k_hsum_tc<true, 1> : tc::k_hsum_tc<false, 1>)
                  : (fast ? tc::k_hsum_tc<true, 0> : tc::k_hsum_tc<false, 0>);
    // (the GEMM's and the operand kernels' shared memory grow differently with the table size)
    FCFS_TRY(ensure_smem((const void *)kern, smem));
    FCFS_TRY(ensure_smem((const void *)gk, gsmem));
    FCFS_TRY(ensure_smem((const void *)hk, gsmem));
    int sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = plan.items < sms ? plan.items : sms;
    const int64_t cb = chunk_buckets(K, plan.tiles_x, plan.tiles_y);
    const int64_t nchunk = (K + cb - 1) / cb;   // K = the clip's bucket count here
    EpiArgs e{};
    // fp16 range: the axis slots carry sums of <= kRowBucketCapFp64 coordinate weights (<= T |w|),
    // scaled by 2^-shift so that 32 (T + 1) 2^-shift <= 2048
    int shift = 0;
    if (f16) {
        const int tb = ilog2_ceil((int64_t)kRowBucketCapFp64 * ((int64_t)T + 1));
        shift = tb > 11 ? tb - 11 : 0;
    }
    const float axs = ldexpf(1.0f, -shift);
    for (int64_t c = 0; c < nchunk; ++c) {
        const tc::TcChunk ch{G, c, cb, H};
        gk<<<(unsigned)(2 * sms), 256, gsmem, s>>>(src, plan, g, ch, G, axs);
        FCFS_CHECK_LAUNCH("k_gsum_tc");
        hk<<<(unsigned)(2 * sms), 256, gsmem, s>>>(src, plan, g, ch, H, axs);
        FCFS_CHECK_LAUNCH("k_hsum_tc");
        kern<<<(unsigned)grid, tc::kThreads, smem, s>>>(src, plan, g, P_ws, e, nullptr, 0, shift, ch);
        FCFS_CHECK_LAUNCH("k_gemm_tf32");
    }
    return FCFS_OK;
}

}  // namespace fcfs

// debug only (not in fcfs.h): copy the CTA-0 event trace of the last FCFS_DEBUG&256 run to the host
extern "C" int64_t fcfs_debug_trace(unsigned long long *host, int64_t cap) {
    unsigned int n = 0;
    if (cudaMemcpyFromSymbol(&n, fcfs::tc::g_trace_n, sizeof(n)) != cudaSuccess) return -1;
    int64_t m = n < (unsigned)fcfs::tc::kTraceMax ? n : fcfs::tc::kTraceMax;
    if (m > cap) m = cap;
    if (m > 0 && cudaMemcpyFromSymbol(host, fcfs::tc::g_trace, sizeof(unsigned long long) * m) != cudaSuccess) return -1;
    const unsigned int z = 0;
    cudaMemcpyToSymbol(fcfs::tc::g_trace_n, &z, sizeof(z));
    return m;
}

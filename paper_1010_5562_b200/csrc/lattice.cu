// lattice.cu — the batched split-TF32 contraction over LATTICE ROWS (DESIGN.md §7,
// "lattice-row form").  Step 4 of the paper evaluates the interior coefficients as row DFTs of the sparse
// corner image f~_xy followed by DFTs along y over the lattice rows:
//
//     S[m,n] = sum_k w_k E(m x_k) E(n y_k) = sum_{y=0..T} G[m,y] E(n y),
//     G[m,y] = sum_{k: y_k = y} w_k E(m x_k)                     (the row DFT of row y)
//
// With T <= 2048 the second factor is a FIXED table over the T+1 lattice rows, the same for every clip, so
// the contraction becomes a dense GEMM whose B operand (E(n y) split hi/lo, 16 KB per 32 rows) streams
// from L2 by bulk copies and is shared by all clips, and whose A operand G is generated on the fly:
//
//   * A lives in TENSOR MEMORY (tcgen05.mma with A from TMEM, "TS" form): TMEM sub-partition q holds clip
//     q of a 4-clip work item, lane l = frequency m = l+1 (lane M: the x-weighted axis row of Eq. F0l).
//     The producer warp of sub-partition q gathers E(m x_k) for its 32 lanes from a quarter-wave SMEM table
//     (one conflict-free LDS.64 of (cos, sin) per corner), accumulates the row sums in registers and
//     writes each finished row's hi/lo split into the stage's TMEM columns (tcgen05.st).  G never exists
//     in HBM or SMEM ("no full-length arrays").
//   * The MMA warp issues per 32-row chunk and 4-clip item: D_c += A_c^hi B^hi + A_c^lo B^hi + A_c^hi B^lo
//     and the same for D_s (sin rows): 24 MMAs of M=128, N=64, K=8 (tf32), A from TMEM, B from SMEM.
//   * FP32 TMEM accumulation in blocks of 8 chunks (96 MMA roundings); the epilogue warps add
//     every block into FP32 registers and, per item, write the window / pupil coefficients (a4 + a5).
//
// Phases are exact integers (lattice vertices): the table row is u = x, T/2 - x, x - T/2 or
// T - x (quarter-wave symmetry), with the sign (-1)^m applied by a sign-bit flip on odd m and the sin sign
// folded into the corner weight.  Requires: T % 4 == 0, (T/4 + 1) * 8 M bytes of table in SMEM, M <= 31,
// N <= 31, the full signed window rows, and corners sorted by y within each clip (checked on the device).
#include "coeff.cuh"
#include "umma.cuh"

namespace fcfs {
namespace lat {
using namespace fcfs::tc;

constexpr int kYC = 32;                     // lattice rows per chunk (the K of 4 MMAs per product)
constexpr int kClips = 4;                   // clips per work item: clip q on TMEM lanes 32q .. 32q+31
constexpr int kAS = 3;                      // A stages in TMEM (128 columns each)
constexpr int kBS = 4;                      // B chunk ring in SMEM
constexpr int kProd = 8;                    // producer warps: sub-partition q = w & 3, chunk parity w >> 2
constexpr int kEpi = 8;                     // epilogue warps: sub-partition q = e & 3, cos (e < 4) / sin
constexpr int kMma = kProd + kEpi;          // MMA + B-loader warp
constexpr int kThreads = (kMma + 1) * 32;   // 544
constexpr int kBTile = 64 * kYC * 4;        // 8 KB: 64 B rows x 32 lattice rows, tf32, SW128 K-major
constexpr int kBChunk = 2 * kBTile;         // hi + lo
constexpr int kFlush = 8;                   // chunks per FP32 TMEM accumulation block
constexpr int kXS = 65;                     // exchange row stride (floats)
constexpr int kStageBytesPerWarp = 32 * 12; // decoded corner records {a, wcs} + x-weight prefixes
constexpr int kMaxRows = 64;                // output rows |m| <= 31 -> 63 rows (+1)
// instruction descriptor: D = F32, A = B = TF32, K-major, N = 64, M = 128
constexpr uint32_t kIdesc =
    (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
constexpr uint32_t kLastBit = 1u << 23, kFlipBit = 1u << 31;

struct Layout {
    uint32_t bring, table, zero, stage, xchg, tabs, bars, total;
};

__host__ __device__ inline Layout layout(int T, int M) {
    Layout L;
    L.bring = 0;
    L.table = kBS * kBChunk;
    const uint32_t tab_bytes = (uint32_t)(T / 4 + 1) * 8u * (uint32_t)(M > 0 ? M : 1);
    L.zero = (L.table + tab_bytes + 15u) & ~15u;
    L.stage = L.zero + 16;
    L.xchg = L.stage + kProd * kStageBytesPerWarp;
    L.tabs = (L.xchg + kClips * 32 * kXS * 4 + 15u) & ~15u;
    // rowoff int32[kMaxRows + 1], nmax int32[kMaxRows], then doubles f_rows, f_invn, f_axm [kMaxRows each]
    L.bars = L.tabs + 4 * (2 * kMaxRows + 2) + 8 * 3 * kMaxRows;
    L.bars = (L.bars + 7u) & ~7u;
    L.total = L.bars + 8 * (2 * kAS + 2 * kBS + 4) + 16;
    return L;
}

__device__ __forceinline__ float2 lds64(uint32_t addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint2 lds64u(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ int32_t lds32i(uint32_t addr) {
    int32_t v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts64u(uint32_t addr, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void sts32i(uint32_t addr, int32_t a) {
    asm volatile("st.shared.s32 [%0], %1;" ::"r"(addr), "r"(a) : "memory");
}
__device__ __forceinline__ void tmem_st1(uint32_t taddr, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_st_zero32(uint32_t taddr) {
    const uint32_t z = 0;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(z)
        : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// TS-form MMA: D[tmem] (+)= A[tmem] * B[smem desc]^T
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(accumulate), "r"(kIdesc)
        : "memory");
}

// split for the tensor core: hi = the top 10 mantissa bits (exact tf32), lo = tf32(v - hi) (rna)
__device__ __forceinline__ void split_hl(float v, uint32_t &hi, uint32_t &lo) {
    hi = __float_as_uint(v) & 0xFFFFE000u;
    lo = tf32_rna(v - __uint_as_float(hi));
}

__device__ __forceinline__ uint32_t bf16_bits(float v) {   // exact for the small integer weights
    return __float_as_uint(v) >> 16;
}

// chunk block bookkeeping (identical in the MMA and epilogue warps)
__host__ __device__ inline int blocks_c(int nch) { return (nch + kFlush - 1) / kFlush; }
__host__ __device__ inline int blocks_s(int nch) { return nch <= kFlush / 2 ? 1 : 1 + (nch - kFlush / 2 + kFlush - 1) / kFlush; }
__device__ __forceinline__ bool c_start(int j) { return j % kFlush == 0; }
__device__ __forceinline__ bool s_start(int j) { return j == 0 || j % kFlush == kFlush / 2; }
__device__ __forceinline__ bool c_end(int j, int nch) { return j % kFlush == kFlush - 1 || j == nch - 1; }
__device__ __forceinline__ bool s_end(int j, int nch) { return j % kFlush == kFlush / 2 - 1 || j == nch - 1; }

struct Args {
    const int64_t *corner_ptr;
    int64_t B;
    const int32_t *x, *y, *w;
    const int32_t *cptr;        // [B][nch + 1] chunk starts (relative to the clip's first corner)
    const uint8_t *btab;        // [nch][hi 8 KB | lo 8 KB]
    int32_t T, M, N, nch;
    int64_t items;
    EpiArgs ea;
    void *F;
};

__global__ void __launch_bounds__(kThreads, 1) k_lattice(Args A) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = su32(smem);
    const int T = A.T, M = A.M, nch = A.nch;
    const Layout L = layout(T, M);
    uint64_t *bars = (uint64_t *)(smem + L.bars);
    uint32_t *tmem_slot = (uint32_t *)(bars + 2 * kAS + 2 * kBS + 4);
    const uint32_t bar0 = su32(bars);
    auto AFULL = [&](int s) { return bar0 + 8u * s; };
    auto AEMPTY = [&](int s) { return bar0 + 8u * (kAS + s); };
    auto BFULL = [&](int s) { return bar0 + 8u * (2 * kAS + s); };
    auto BEMPTY = [&](int s) { return bar0 + 8u * (2 * kAS + kBS + s); };
    auto DFULL = [&](int d) { return bar0 + 8u * (2 * kAS + 2 * kBS + d); };
    auto DEMPTY = [&](int d) { return bar0 + 8u * (2 * kAS + 2 * kBS + 2 + d); };
    int32_t *rowoff = (int32_t *)(smem + L.tabs);          // [2M + 2]
    int32_t *nmaxr = rowoff + (kMaxRows + 1);               // [2M + 1] entries per output row (half count)
    double *f_rows = (double *)(smem + L.tabs + 4 * (2 * kMaxRows + 2));
    double *f_invn = f_rows + kMaxRows;
    double *f_axm = f_invn + kMaxRows;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const EpiArgs &ea = A.ea;

    // ---- setup: quarter-wave table, output tables, barriers, TMEM
    {
        const int rows = T / 4 + 1;
        float2 *tab = (float2 *)(smem + L.table);
        for (int i = tid; i < rows * M; i += kThreads) {
            const int u = i / M, m = i % M + 1;
            double sn, cs;
            sincospi(2.0 * (double)(((int64_t)m * u) % T) / (double)T, &sn, &cs);
            tab[i] = make_float2((float)cs, (float)sn);
        }
        if (tid < 4) ((uint32_t *)(smem + L.zero))[tid] = 0u;
        const double pi = 3.141592653589793238462643383279502884;
        for (int a = tid; a < kMaxRows; a += kThreads) {
            f_rows[a] = a ? -1.0 / (4.0 * pi * pi * (double)a) : 0.0;
            f_invn[a] = a ? 1.0 / (double)a : 0.0;
            f_axm[a] = a ? 1.0 / (2.0 * pi * (double)a * (double)T) : 0.0;
        }
        if (tid == 0) {
            int32_t off = 0;
            for (int i = 0; i <= 2 * ea.M; ++i) {
                rowoff[i] = off;
                const int c = ea.layout == FCFS_LAYOUT_PUPIL ? pupil_nmax(i - ea.M, ea.r2, ea.N) : ea.N;
                nmaxr[i] = c;
                off += c < 0 ? 0 : 2 * c + 1;
            }
            rowoff[2 * ea.M + 1] = off;
            for (int s = 0; s < kAS; ++s) { mbar_init(AFULL(s), 4); mbar_init(AEMPTY(s), 1); }
            for (int s = 0; s < kBS; ++s) { mbar_init(BFULL(s), 1); mbar_init(BEMPTY(s), 1); }
            for (int d = 0; d < 2; ++d) { mbar_init(DFULL(d), 1); mbar_init(DEMPTY(d), 4); }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        fence_proxy_async();
        if (warp == kMma) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tmem_slot))
                         : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        __syncthreads();
        tc_fence_after();
    }
    const uint32_t tmem = *tmem_slot;

    if (warp < kProd) {
        // ================================ producers ================================
        const int q = warp & 3, par = warp >> 2;
        const uint32_t lrow = (uint32_t)(32 * q) << 16;                  // TMEM lane base of sub-partition q
        const bool tl = lane < M;                                         // table lane: m = lane + 1
        const bool axis = lane == M;                                      // x-weighted axis row (Eq. F0l)
        const uint32_t lmask = tl ? 0x3FFFFu : 0u;
        const uint32_t lbase = tl ? (uint32_t)(8 * lane) : sbase + L.zero;
        const uint32_t oddm = (tl && !(lane & 1)) ? kFlipBit : 0u;       // (-1)^m flip for odd m
        const uint32_t stg = sbase + L.stage + warp * kStageBytesPerWarp; // {a, wcs} x 32, then prefixes x 32
        const uint32_t tabaddr = sbase + L.table;
        const int T2 = T / 2, T4 = T / 4, T34 = 3 * (T / 4);
        uint32_t gc = 0;
        for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x) {
            const int64_t clip = item * kClips + q;
            const bool real = clip < A.B;
            const int64_t k0 = real ? A.corner_ptr[clip] : 0;
            const int32_t *cp = A.cptr + (real ? clip : 0) * (int64_t)(nch + 1);
            for (int j = 0; j < nch; ++j, ++gc) {
                if ((j & 1) != par) continue;
                const int s = (int)(gc % kAS);
                const uint32_t ph = (gc / kAS) & 1u;
                mbar_wait(AEMPTY(s), ph ^ 1u);
                tc_fence_after();
                const uint32_t tcol = tmem + lrow + 128u + 128u * (uint32_t)s;
                tmem_st_zero32(tcol);
                tmem_st_zero32(tcol + 32);
                tmem_st_zero32(tcol + 64);
                tmem_st_zero32(tcol + 96);
                tmem_wait_st();
                const int32_t ca = real ? __ldg(cp + j) : 0, cb = real ? __ldg(cp + j + 1) : 0;
                const int32_t y0 = j * kYC;
                float ac = 0.f, as = 0.f;
                int32_t carry = 0, pbase = 0;
                for (int32_t kb = ca; kb < cb; kb += 32) {
                    const int n = cb - kb < 32 ? cb - kb : 32;
                    // ---- decode (lane i = corner kb + i): record {a, wcs} + inclusive prefix of w x
                    {
                        const bool ok = lane < n;
                        const int64_t k = k0 + kb + lane;
                        const int32_t x = ok ? __ldg(A.x + k) : 0;
                        const int32_t yy = ok ? __ldg(A.y + k) : 0;
                        const int32_t w = ok ? __ldg(A.w + k) : 0;
                        int32_t ynext = __shfl_down_sync(0xffffffffu, yy, 1);
                        if (lane == n - 1) ynext = (kb + n < cb) ? __ldg(A.y + k + 1) : -1;
                        const bool last = ynext != yy;
                        int32_t u;
                        uint32_t flip = 0u;
                        float ss = 1.f;
                        if (x <= T4) { u = x; }
                        else if (x <= T2) { u = T2 - x; flip = kFlipBit; ss = -1.f; }
                        else if (x <= T34) { u = x - T2; flip = kFlipBit; }
                        else { u = T - x; ss = -1.f; }
                        const uint32_t a = (tabaddr + (uint32_t)u * 8u * (uint32_t)M) | ((uint32_t)(yy - y0) << 18) |
                                           (last ? kLastBit : 0u) | flip;
                        const float wf = (float)w;
                        const uint32_t wcs = bf16_bits(wf) | (bf16_bits(wf * ss) << 16);
                        int32_t p = w * x;
#pragma unroll
                        for (int d = 1; d < 32; d <<= 1) {
                            const int32_t t = __shfl_up_sync(0xffffffffu, p, d);
                            if (lane >= d) p += t;
                        }
                        p += carry;
                        carry = __shfl_sync(0xffffffffu, p, 31);
                        sts64u(stg + 8u * lane, ok ? a : 0u, ok ? wcs : 0u);
                        sts32i(stg + 256u + 4u * lane, p);
                    }
                    __syncwarp();
                    // ---- gather: corner by corner (uniform loop), one LDS.64 of (cos, sin) per lane
                    for (int i = 0; i < n; ++i) {
                        const uint2 r = lds64u(stg + 8u * i);
                        const float2 v = lds64((r.x & lmask) + lbase);
                        const float vc = __uint_as_float(__float_as_uint(v.x) ^ (r.x & oddm));
                        const float vs = __uint_as_float(__float_as_uint(v.y) ^ (r.x & oddm));
                        ac = fmaf(vc, __uint_as_float(r.y << 16), ac);
                        as = fmaf(vs, __uint_as_float(r.y & 0xFFFF0000u), as);
                        if (__any_sync(0xffffffffu, (r.x & kLastBit) != 0u)) {
                            const uint32_t col = (r.x >> 18) & 31u;
                            const int32_t p = lds32i(stg + 256u + 4u * i);
                            if (axis) ac = (float)(p - pbase);
                            pbase = p;
                            uint32_t h, l;
                            split_hl(ac, h, l);
                            tmem_st1(tcol + col, h);
                            tmem_st1(tcol + 32u + col, l);
                            split_hl(as, h, l);
                            tmem_st1(tcol + 64u + col, h);
                            tmem_st1(tcol + 96u + col, l);
                            ac = 0.f;
                            as = 0.f;
                        }
                    }
                    __syncwarp();
                }
                tmem_wait_st();
                __syncwarp();
                tc_fence_before();
                if (lane == 0) mbar_arrive(AFULL(s));
            }
        }
    } else if (warp == kMma) {
        // ============================ MMA issuer + B loader ============================
        const uint32_t bring = sbase + L.bring;
        int64_t my_items = 0;
        for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x) ++my_items;
        const uint32_t total = (uint32_t)(my_items * nch);
        uint32_t lc = 0;   // B chunks loaded
        auto pump = [&](uint32_t upto) {
            while (lc < upto && lc < total) {
                const int slot = (int)(lc % kBS);
                mbar_wait(BEMPTY(slot), ((lc / kBS) & 1u) ^ 1u);
                if (elect_one()) {
                    mbar_expect_tx(BFULL(slot), kBChunk);
                    bulk_g2s(bring + (uint32_t)slot * kBChunk, A.btab + (size_t)(lc % (uint32_t)nch) * kBChunk, kBChunk,
                             BFULL(slot));
                }
                __syncwarp();
                ++lc;
            }
        };
        pump(kBS - 1);
        uint32_t gc = 0, tc_ = 0, ts_ = 0;   // chunk counter, D_c / D_s block counters
        for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x) {
            for (int j = 0; j < nch; ++j, ++gc) {
                const int s = (int)(gc % kAS);
                const int b = (int)(gc % kBS);
                mbar_wait(BFULL(b), (gc / kBS) & 1u);
                mbar_wait(AFULL(s), (gc / kAS) & 1u);
                tc_fence_after();
                const uint32_t a0 = tmem + 128u + 128u * (uint32_t)s;
                const uint64_t bh = umma_desc(bring + (uint32_t)b * kBChunk), bl = umma_desc(bring + (uint32_t)b * kBChunk + kBTile);
                const bool cs = c_start(j), ss = s_start(j);
                auto issue = [&](int d) {
                    const uint32_t dt = tmem + 64u * (uint32_t)d;
                    const uint32_t ah = a0 + 64u * (uint32_t)d, al = ah + 32u;
                    const uint32_t fresh = d == 0 ? (cs ? 1u : 0u) : (ss ? 1u : 0u);
                    if (elect_one()) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            umma_ts(dt, ah + 8u * u, bh + 2u * u, (u > 0 || !fresh) ? 1u : 0u);
                            umma_ts(dt, al + 8u * u, bh + 2u * u, 1u);
                            umma_ts(dt, ah + 8u * u, bl + 2u * u, 1u);
                        }
                    }
                    __syncwarp();
                };
                auto wait_d = [&](int d) {
                    uint32_t &t = d == 0 ? tc_ : ts_;
                    mbar_wait(DEMPTY(d), (t & 1u) ^ 1u);
                    tc_fence_after();
                };
                // a D whose accumulation block starts here waits for the epilogue to have read its last
                // block; the other D's MMAs are issued first so the tensor pipe stays busy meanwhile
                if (cs && ss) { wait_d(0); wait_d(1); issue(0); issue(1); }
                else if (cs) { issue(1); wait_d(0); issue(0); }
                else if (ss) { issue(0); wait_d(1); issue(1); }
                else { issue(0); issue(1); }
                if (elect_one()) {
                    umma_commit(AEMPTY(s));
                    umma_commit(BEMPTY(b));
                    if (c_end(j, nch)) umma_commit(DFULL(0));
                    if (s_end(j, nch)) umma_commit(DFULL(1));
                }
                __syncwarp();
                if (c_end(j, nch)) ++tc_;
                if (s_end(j, nch)) ++ts_;
                pump(gc + kBS);
            }
        }
    } else {
        // ================================ epilogue ================================
        const int e = warp - kProd, q = e & 3, kind = e >> 2;   // kind 0: D_c (cos rows), 1: D_s (sin rows)
        const uint32_t dt = tmem + ((uint32_t)(32 * q) << 16) + 64u * (uint32_t)kind;
        const int nb = kind == 0 ? blocks_c(nch) : blocks_s(nch);
        float *xc = (float *)(smem + L.xchg) + (size_t)(q * 32 + lane) * kXS;
        uint32_t t = 0;
        for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x) {
            float S[64];
#pragma unroll
            for (int i = 0; i < 64; ++i) S[i] = 0.f;
            for (int bi = 0; bi < nb; ++bi, ++t) {
                mbar_wait_sleep(DFULL(kind), t & 1u);
                tc_fence_after();
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    uint32_t r0[16];
                    TMEM_LD16(dt + 16u * h, r0);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) S[16 * h + i] += __uint_as_float(r0[i]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(DEMPTY(kind));
            }
            // ---- a4 + a5: cos rows combine with the sin rows of the same lane (exchange in SMEM).  D columns:
            // c < 31: n = c + 1 (cos), 31: the y-weighted axis column, 31 + b: n = b (sin) — fixed offsets so
            // that S stays in registers (static indices below)
            if (kind == 1) {
#pragma unroll
                for (int i = 0; i < 64; ++i) xc[i] = S[i];
            }
            named_bar(1, kEpi * 32);
            const int64_t clip = item * kClips + q;
            if (kind == 0 && clip < A.B && lane <= M) {
                void *Fc = ea.out_f32 ? (void *)((float2 *)A.F + clip * ea.out_per_clip)
                                      : (void *)((double2 *)A.F + clip * ea.out_per_clip);
                const bool dmask = ea.layout == FCFS_LAYOUT_DENSE && ea.r2 >= 0.0;
                if (lane < M) {
                    const int m = lane + 1;
                    const int nm = nmaxr[ea.M + m];
                    if (nm >= 0) {
                        const int32_t op = rowoff[ea.M + m] + nm, on = rowoff[ea.M - m] + nm;
                        const double mm = (double)m * (double)m;
                        {   // n = 0: Eq. Fk0, F[m,0] = i (Pc_ax - i Ps_ax) / (2 pi m T)
                            const bool mk = dmask && mm > ea.r2;
                            const double re = mk ? 0.0 : (double)xc[31] * f_axm[m], im = mk ? 0.0 : (double)S[31] * f_axm[m];
                            store_out(Fc, op, make_double2(re, im), ea.out_f32);
                            store_out(Fc, on, make_double2(re, -im), ea.out_f32);
                        }
#pragma unroll
                        for (int b = 1; b <= 31; ++b) {
                            if (b > nm) break;
                            // Eq. Fkl: S(m, +-b) from the quadrant products, F = -S / (4 pi^2 m n)
                            const double pcc = S[b - 1], pcs = S[31 + b], psc = xc[b - 1], pss = xc[31 + b];
                            const bool mk = dmask && mm + (double)b * (double)b > ea.r2;
                            const double sc = f_rows[m] * f_invn[b];
                            double re = mk ? 0.0 : (pcc - pss) * sc, im = mk ? 0.0 : -(psc + pcs) * sc;   // n = +b
                            store_out(Fc, op + b, make_double2(re, im), ea.out_f32);
                            store_out(Fc, on - b, make_double2(re, -im), ea.out_f32);
                            re = mk ? 0.0 : -(pcc + pss) * sc;                                              // n = -b
                            im = mk ? 0.0 : (psc - pcs) * sc;
                            store_out(Fc, op - b, make_double2(re, im), ea.out_f32);
                            store_out(Fc, on + b, make_double2(re, -im), ea.out_f32);
                        }
                    }
                } else {   // lane == M: row m = 0 (the x-weighted axis row, Eq. F0l) and the DC (Eq. Fdc)
                    const int nm = nmaxr[ea.M];
                    if (nm >= 0) {
                        const int32_t o0 = rowoff[ea.M] + nm;
                        const double dc = (double)ea.area_dev[clip] / ((double)T * (double)T);
                        store_out(Fc, o0, make_double2(dc, 0.0), ea.out_f32);
#pragma unroll
                        for (int b = 1; b <= 31; ++b) {
                            if (b > nm) break;
                            const bool mk = dmask && (double)b * (double)b > ea.r2;
                            // F[0,b] = i (P_ax,c - i P_ax,s) / (2 pi b T)
                            const double re = mk ? 0.0 : (double)S[31 + b] * f_axm[b], im = mk ? 0.0 : (double)S[b - 1] * f_axm[b];
                            store_out(Fc, o0 + b, make_double2(re, im), ea.out_f32);
                            store_out(Fc, o0 - b, make_double2(re, -im), ea.out_f32);
                        }
                    }
                }
            }
            named_bar(1, kEpi * 32);   // exchange buffer free for the next item
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == kMma) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// B operand of every chunk (64 rows, fixed offsets): row b - 1 = cos(2 pi b y / T) for b = 1..N, row 31 = y
// (the coordinate weight of Eq. Fk0), row 31 + b = sin(2 pi b y / T); other rows and lattice rows y > T: 0.
// hi = tf32(v), lo = tf32(v - hi), both in the SW128 K-major stage layout (row r, k = y - 32 c).
__global__ void k_lat_btab(int32_t T, int32_t N, int32_t nch, uint8_t *__restrict__ btab) {
    const int64_t total = (int64_t)nch * 64 * kYC;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i / (64 * kYC));
        const int r = (int)((i / kYC) % 64);
        const int k = (int)(i % kYC);
        const int64_t y = (int64_t)c * kYC + k;
        double v = 0.0;
        if (y <= T) {
            if (r < 31 && r < N) v = cospi(2.0 * (double)(((int64_t)(r + 1) * y) % T) / (double)T);
            else if (r == 31) v = (double)y;
            else if (r > 31 && r - 31 <= N) v = sinpi(2.0 * (double)(((int64_t)(r - 31) * y) % T) / (double)T);
        }
        const float hi = __uint_as_float(tc::tf32_rna((float)v));
        const float lo = __uint_as_float(tc::tf32_rna((float)(v - (double)hi)));
        const uint32_t off = (uint32_t)(r / 8) * 1024u + (uint32_t)(r % 8) * 128u + ((uint32_t)((k / 4) ^ (r % 8)) << 4) +
                             (uint32_t)(k % 4) * 4u;
        uint8_t *ch = btab + (size_t)c * kBChunk;
        *(float *)(ch + off) = hi;
        *(float *)(ch + kBTile + off) = lo;
    }
}

// chunk starts of every clip: cptr[b][j] = first corner (relative to the clip's start) with y >= 32 j,
// j = 0 .. nch (cptr[b][nch] = the clip's corner count); flags an unsorted clip in *unsorted.
__global__ void __launch_bounds__(256) k_lat_cptr(const int64_t *__restrict__ corner_ptr, int64_t B,
                                                  const int32_t *__restrict__ y, int32_t nch, int32_t *__restrict__ cptr,
                                                  int32_t *__restrict__ unsorted) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < B; b += nw) {
        const int64_t k0 = corner_ptr[b];
        const int32_t K = (int32_t)(corner_ptr[b + 1] - k0);
        int32_t *out = cptr + b * (int64_t)(nch + 1);
        int bad = 0;
        for (int32_t i = lane; i < K; i += 32) {
            const int32_t yy = __ldg(y + k0 + i);
            const int32_t c = yy >> 5;
            const int32_t cprev = i > 0 ? (__ldg(y + k0 + i - 1) >> 5) : -1;
            if (i > 0 && __ldg(y + k0 + i - 1) > yy) bad = 1;
            for (int32_t jj = cprev + 1; jj <= c && jj <= nch; ++jj) out[jj] = i;
        }
        if (lane == 0) {
            const int32_t clast = K > 0 ? (__ldg(y + k0 + K - 1) >> 5) : -1;
            for (int32_t jj = clast + 1; jj <= nch; ++jj) out[jj] = K;
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) *unsorted = 1;
    }
}

}  // namespace lat

int32_t lattice_chunks(int32_t T) { return (T + 1 + lat::kYC - 1) / lat::kYC; }

size_t lattice_smem_bytes(int32_t T, int32_t M) { return (size_t)lat::layout(T, M).total + 1024; }

// the lattice-row form applies (T and window limits, SMEM budget); the caller adds the sortedness condition
bool lattice_eligible(int32_t T, const EpiArgs &ea) {
    if (T < 4 || (T % 4) != 0 || T > 4096) return false;
    if (ea.M < 0 || ea.N < 0 || ea.M > 31 || ea.N > 31) return false;
    if (ea.m_lo != -ea.M || ea.m_hi != ea.M || !ea.out_f32) return false;
    return lattice_smem_bytes(T, ea.M) <= 227 * 1024;
}

size_t lattice_ws_bytes(int64_t B, int32_t T) {
    const int32_t nch = lattice_chunks(T);
    return (size_t)nch * lat::kBChunk + 256 + (size_t)B * (nch + 1) * 4 + 256 + 256;
}

fcfs_status launch_lattice_prepare(const int64_t *corner_ptr, int64_t B, const int32_t *y, int32_t T, int32_t N,
                                   void *ws, int32_t *unsorted_dev, cudaStream_t s) {
    const int32_t nch = lattice_chunks(T);
    uint8_t *btab = (uint8_t *)ws;
    int32_t *cptr = (int32_t *)(btab + (((size_t)nch * lat::kBChunk + 255) & ~(size_t)255));
    lat::k_lat_btab<<<148, 256, 0, s>>>(T, N, nch, btab);
    FCFS_CHECK_LAUNCH("k_lat_btab");
    const int64_t blocks = (B + 7) / 8;
    lat::k_lat_cptr<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, s>>>(corner_ptr, B, y, nch, cptr, unsorted_dev);
    FCFS_CHECK_LAUNCH("k_lat_cptr");
    return FCFS_OK;
}

fcfs_status launch_lattice(const int64_t *corner_ptr, int64_t B, const int32_t *x, const int32_t *y, const int32_t *w,
                           int32_t T, const EpiArgs &ea, void *F, void *ws, cudaStream_t s) {
    const int32_t nch = lattice_chunks(T);
    lat::Args a{};
    a.corner_ptr = corner_ptr;
    a.B = B;
    a.x = x; a.y = y; a.w = w;
    a.btab = (const uint8_t *)ws;
    a.cptr = (const int32_t *)((const uint8_t *)ws + (((size_t)nch * lat::kBChunk + 255) & ~(size_t)255));
    a.T = T; a.M = ea.M; a.N = ea.N; a.nch = nch;
    a.items = (B + lat::kClips - 1) / lat::kClips;
    a.ea = ea;
    a.F = F;
    const size_t smem = lattice_smem_bytes(T, ea.M);
    FCFS_TRY(ensure_smem((const void *)lat::k_lattice, smem, true));
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = a.items < sms ? a.items : sms;
    lat::k_lattice<<<(unsigned)grid, lat::kThreads, smem, s>>>(a);
    FCFS_CHECK_LAUNCH("k_lattice");
    return FCFS_OK;
}

}  // namespace fcfs

// lattice.cu — the batched split-TF32 contraction over LATTICE ROWS (DESIGN.md §7,
// "lattice-row form").  Step 4 of the paper evaluates the interior coefficients as row DFTs of the sparse
// corner image f~_xy followed by DFTs along y over the lattice rows:
//
//     S[m,n] = sum_k w_k E(m x_k) E(n y_k) = sum_{y=0..T} G[m,y] E(n y),
//     G[m,y] = sum_{k: y_k = y} w_k E(m x_k)                     (the row DFT of row y)
//
// With T <= 2496 the second factor is a FIXED table over the T+1 lattice rows, the same for every clip, so
// the contraction becomes a dense GEMM whose B operand (E(n y) split hi/lo) streams from L2 by bulk copies
// and is shared by all clips, and whose A operand G is generated on the fly:
//
//   * A lives in TENSOR MEMORY (tcgen05.mma with A from TMEM, "TS" form): TMEM sub-partition q holds clip
//     q of a 4-clip work item, lane l = frequency m = l+1 (lane M: the x-weighted axis row of Eq. F0l).
//     Four producer warps per sub-partition gather E(m x_k) for their 32 lanes from a quarter-wave SMEM
//     table (one conflict-free LDS.64 of (cos, sin) per corner), accumulate the row sums in registers (one
//     FFMA2 per corner) and store each finished row's hi/lo split into its TMEM stage (tcgen05.st).  G never
//     exists in HBM or SMEM ("no full-length arrays").
//   * A stage holds 12 lattice rows with hi and lo interleaved along K, (hi_0, lo_0, hi_1, lo_1, ...), so
//     one MMA stream against B' = (B^hi_0, B^hi_0, B^hi_1, B^hi_1, ...) gives (A^hi + A^lo) B^hi and one
//     against B'' = (B^lo_0, 0, B^lo_1, 0, ...) gives A^hi B^lo: the three products of the split, 12 MMAs
//     of M=128, N=64, K=8 per chunk and 4 clips (cos and sin rows).  Eight 48-column stages (two per
//     producer warp: it fills one while the MMAs of the other run); one MMA-issuer warp per accumulator
//     (D_c, D_s) and a B-loader warp streaming the 16 KB chunks of the shared table from L2.
//   * FP32 TMEM accumulation in blocks of 21 chunks (252 rows, 126 MMA roundings); the
//     epilogue warps copy every block out of TMEM (releasing D at once), add it into FP32 sums in an
//     L2-resident global scratch and, per item, write the window / pupil coefficients (a4 + a5).
//
// Phases are exact integers (lattice vertices): the table row is u = x, T/2 - x, x - T/2 or
// T - x (quarter-wave symmetry), with the sign (-1)^m of odd m folded into per-lane-parity weights and the
// sin sign into the sin weight.  Requires: T % 4 == 0, T <= 2496, M, N <= 31, the full signed window rows,
// and corners sorted by y within each clip (checked on the device unless the caller guarantees it).
#include "coeff.cuh"
#include "umma.cuh"

namespace fcfs {
namespace lat {
#ifndef KBS_
#define KBS_ 6
#endif
using namespace fcfs::tc;

constexpr int kYC = 12;                     // lattice rows per chunk (K = 24 of the 32-wide B tiles)
constexpr int kClips = 4;                   // clips per work item: clip q on TMEM lanes 32q .. 32q+31
constexpr int kAS = 8;                      // A stages in TMEM (48 columns each): the CTA's g-th chunk (counted
                                            // over its items) uses stage g % 8
constexpr int kBS = KBS_;                   // B chunk ring in SMEM (12 KB slots)
constexpr int kPW = 4;                      // producer warps per sub-partition (chunk j of an item: warp j % kPW;
                                            // 5 measured 3% slower: spills and shared-memory pipe contention)
constexpr int kProd = 4 * kPW;              // producer warps: sub-partition q = w & 3, chunks j = w >> 2 (mod kPW)
constexpr int kEpi = 4;                     // epilogue warps: sub-partition q = e
constexpr int kMma = kProd + kEpi;          // MMA issuer warp
constexpr int kLoad = kMma + 2;             // B-loader warp; kMma and kMma + 1 issue the D_c and D_s MMAs
constexpr int kThreads = (kLoad + 1) * 32;
constexpr int kBTile = 64 * 2 * kYC * 4;    // 6 KB: 64 B rows x 24 K (12 lattice rows hi/lo interleaved), no swizzle
constexpr int kBChunk = 2 * kBTile;         // B' + B''
constexpr int kFlush = 21;                  // chunks per FP32 TMEM accumulation block (252 rows, 126 MMA roundings)
constexpr int kRec = 24;                    // decoded corner record: 3 lane-halves {row address, weights}
constexpr int kStageBytesPerWarp = 32 * kRec + 32 * 4;   // 32 records + 32 flush columns
constexpr int kMaxRows = 64;                // output rows |m| <= 31 -> 63 rows (+1)
constexpr int kMaxChunks = 209;             // chunks per clip: (T + 1) / 12 rounded up, T <= 2496
constexpr int kStageCols = 4 * kYC;         // TMEM columns per A stage: cos (hi, lo) x 12 rows | sin (hi, lo) x 12
// TMEM columns: D_c [0,64), D_s [64,128), A stage s at 128 + 48 s: cos (hi, lo) x 12 rows | sin (hi, lo) x 12.
// The epilogue's FP32 block sums S live in an L2-resident global scratch ([CTA][clip q][col / 4][lane]
// float4: 64 KB per CTA), which frees TMEM for the eight A stages (two per producer warp).
constexpr uint32_t kColA = 128;
// named barriers: 2 + d: D block d finished (MMA -> epilogue); 4 + s: stage s full (producers -> MMA).
// Stage s free (MMA completion -> producers) is the commit's mbarrier alone (a sleeping poll).
constexpr int kBarD = 2, kBarFull = 4;
static_assert(kBarFull + kAS <= 16, "named barriers");
constexpr int kFullCount = 32 * kClips + 64;   // stage full: one producer warp per clip + both MMA warps
static_assert(kPW <= kAS, "a producer's previous chunk proves the stage's older use complete");
// instruction descriptor: D = F32, A = B = TF32, K-major, N = 64, M = 128
constexpr uint32_t kIdesc =
    (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

struct Layout {
    uint32_t bring, table, stage, tabs, bars, total;
};

__host__ __device__ inline Layout layout(int T, int M) {
    Layout L;
    L.bring = 0;
    L.table = kBS * kBChunk;
    // row u: lanes 0 .. M (M table lanes + the axis lane), stride 8 (M + 1) B; lanes above M read into the
    // next row (finite values into A rows nobody reads); one zero row of padding at the end
    const uint32_t tab_bytes = (uint32_t)(T / 4 + 2) * 8u * (uint32_t)(M + 1) + 256u;
    L.stage = (L.table + tab_bytes + 15u) & ~15u;
    L.tabs = L.stage + kProd * kStageBytesPerWarp;
    // rowoff int32[kMaxRows + 1], nmax int32[kMaxRows], then doubles f_rows, f_invn, f_axm [kMaxRows each]
    L.bars = (L.tabs + 4 * (2 * kMaxRows + 2) + 8 * 3 * kMaxRows + 7u) & ~7u;
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
__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t a) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(a) : "memory");
}
__device__ __forceinline__ void sts64u(uint32_t addr, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, uint32_t a, uint32_t b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void tmem_st_zero32(uint32_t taddr) {
    const uint32_t z = 0;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(z)
        : "memory");
}
__device__ __forceinline__ void tmem_st_zero16(uint32_t taddr) {
    const uint32_t z = 0;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(z)
        : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_ld1(uint32_t taddr, uint32_t (&r)[1]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// packed FP32x2 FMA (SASS FFMA2): (ac, as) += (v.x, v.y) * (wc, ws)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n mov.b64 rc, {%6, %7};\n"
        " fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;\n}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

// TS-form MMA: D[tmem] (+)= A[tmem] * B[smem desc]^T
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %3, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(accumulate), "r"(kIdesc)
        : "memory");
}

// split for the tensor core: hi = the top 10 mantissa bits (exact tf32), lo = v - hi (exact in fp32; the
// MMA reads its top 19 bits: |lo - tf32(lo)| < 2^-10 |lo| < 2^-20 |v|)
__device__ __forceinline__ void split_hl(float v, uint32_t &hi, uint32_t &lo) {
    hi = __float_as_uint(v) & 0xFFFFE000u;
    lo = __float_as_uint(v - __uint_as_float(hi));
}

__device__ __forceinline__ uint32_t bf16_bits(float v) {   // exact for the small integer weights
    return __float_as_uint(v) >> 16;
}

// accumulation blocks (identical in the MMA and epilogue warps): D_c blocks start at chunks j % kFlush == 0,
// D_s blocks at j % kFlush == kFlush / 2 (and j == 0), so the two flushes never coincide inside an item
__host__ __device__ inline bool c_start(int j) { return j % kFlush == 0; }
__host__ __device__ inline bool s_start(int j) { return j == 0 || j % kFlush == kFlush / 2; }
__host__ __device__ inline bool c_end(int j, int nch) { return j % kFlush == kFlush - 1 || j == nch - 1; }
__host__ __device__ inline bool s_end(int j, int nch) { return j % kFlush == kFlush / 2 - 1 || j == nch - 1; }


struct Args {
    const int64_t *corner_ptr;
    int64_t B;
    const int32_t *x, *y, *w;
    const int32_t *cptr;        // [B][nch + 1] chunk starts (relative to the clip's first corner)
    const uint8_t *btab;        // [nch][B' 8 KB | B'' 8 KB]
    const float2 *qtab;         // the quarter-wave table, built once per call (k_lat_qtab)
    int32_t T, M, N, nch;
    int64_t items;
    EpiArgs ea;
    void *F;
    float4 *S;                  // [gridDim][kClips][32 col quads][32 lanes] FP32 block sums
};

#ifdef LAT_TRACE
// diagnostic build only (tools/lat_trace.py): clock64 stamps of CTA 0's chunks
constexpr int kTrMax = 8192;
__device__ long long g_tr[kTrMax][12];   // per chunk g: [q] wait start, [4+q] fill start, [8+q] full
__device__ long long g_trm[kTrMax][4];   // per chunk g: MMA warp d after FULL [d], before BFULL [2 + d]
#define TR(stmt) do { if (blockIdx.x == 0) { stmt; } } while (0)
#else
#define TR(stmt) do { } while (0)
#endif

__global__ void __launch_bounds__(kThreads, 1) k_lattice(Args A) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = su32(smem);
    const int T = A.T, M = A.M, N = A.N, nch = A.nch;
    const Layout L = layout(T, M);
    uint64_t *bars = (uint64_t *)(smem + L.bars);
    uint32_t *tmem_slot = (uint32_t *)(bars + 2 * kAS + 2 * kBS + 4);
    const uint32_t bar0 = su32(bars);
    auto AEMPTY = [&](int s) { return bar0 + 8u * (kAS + s); };
    auto BFULL = [&](int s) { return bar0 + 8u * (2 * kAS + s); };
    auto BEMPTY = [&](int s) { return bar0 + 8u * (2 * kAS + kBS + s); };
    auto DFULL = [&](int d) { return bar0 + 8u * (2 * kAS + 2 * kBS + d); };
    auto DEMPTY = [&](int d) { return bar0 + 8u * (2 * kAS + 2 * kBS + 2 + d); };
    int32_t *rowoff = (int32_t *)(smem + L.tabs);          // [2M + 2]
    int32_t *nmaxr = rowoff + (kMaxRows + 1);               // [2M + 1] half-width of each output row
    double *f_rows = (double *)(smem + L.tabs + 4 * (2 * kMaxRows + 2));
    double *f_invn = f_rows + kMaxRows;
    double *f_axm = f_invn + kMaxRows;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const EpiArgs &ea = A.ea;

    // ---- setup: quarter-wave table, output tables, barriers, TMEM
    {
        // row u, lane l < M: (cos, sin)(2 pi (l+1) u / T); lane M: (T/2, u) (the x-weighted axis row:
        // x = c_q T/2 + s_q u, see the decode)
        const int rows = T / 4 + 2, lanes = M + 1;
        float2 *tab = (float2 *)(smem + L.table);
        for (int i = tid; i < rows * lanes + 32; i += kThreads) tab[i] = __ldg(A.qtab + i);   // from L2
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
            for (int st = 0; st < kAS; ++st) mbar_init(AEMPTY(st), 2);   // one commit per MMA warp
            for (int st = 0; st < kBS; ++st) { mbar_init(BFULL(st), 1); mbar_init(BEMPTY(st), 2); }
            for (int d = 0; d < 2; ++d) { mbar_init(DFULL(d), 1); mbar_init(DEMPTY(d), kEpi); }
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
    int64_t my_items = 0;
    for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x) ++my_items;

    if (warp < kProd) {
        // ================================ producers ================================
        // Warp (q, p) gathers clip q of every item for the chunks j = p (mod kPW) into TMEM stage g % kAS (g:
        // the CTA's chunk counter over its items).  Per batch of <= 32 corners a lane-parallel decode writes one
        // 24-byte record per corner: three lane-halves {row address, bf16 weight pair}, for even lanes (odd m:
        // the (-1)^m quarter-wave flip folded into the weights), odd lanes, and the axis lane (weights (w c_q,
        // w s_q) against the table's (T/2, u): x = c_q T/2 + s_q u).  The gather walks the corners with
        // uniform control: one LDS.64 of the lane's record half, one LDS.64 of (cos, sin) from the table row,
        // one FFMA2; at a row end (bit mask) the two sums are split hi/lo into the row's TMEM columns.
        const int q = warp & 3, p = warp >> 2;
        const uint32_t lrow = (uint32_t)(32 * q) << 16;                  // TMEM lane base of sub-partition q
        const bool axis = lane == M;
        const uint32_t lane8 = 8u * (uint32_t)lane;
        const uint32_t rowb = 8u * (uint32_t)(M + 1);                     // table row stride
        const uint32_t stg = sbase + L.stage + warp * kStageBytesPerWarp;
        const uint32_t recl = stg + (axis ? 16u : ((lane & 1) ? 8u : 0u));   // this lane's half of each record
        const uint32_t fcl = stg + 32u * kRec;                              // flush columns [32]
        const uint32_t tabaddr = sbase + L.table;
        const int T2 = T / 2, T4 = T / 4, T34 = 3 * (T / 4);
        uint32_t gbase = 0;                                                 // the CTA's chunks before this item
        for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x) {
            const int64_t clip = item * kClips + q;
            const bool real = clip < A.B;
            const int64_t k0 = real ? A.corner_ptr[clip] : 0;
            // this warp's chunk bounds in registers: lane l holds the bounds of chunks p + kPW (l + 32 h)
            constexpr int kNB = (kMaxChunks / kPW + 31) / 32;
            const int32_t *cp = A.cptr + (real ? clip : 0) * (int64_t)(nch + 1);
            int32_t cs[kNB], ce[kNB];
#pragma unroll
            for (int h = 0; h < kNB; ++h) {
                const int jj = p + kPW * (32 * h + lane);
                cs[h] = ce[h] = 0;
                if (real && jj < nch) { cs[h] = __ldg(cp + jj); ce[h] = __ldg(cp + jj + 1); }
            }
            const int nt = nch > p ? (nch - p + kPW - 1) / kPW : 0;       // chunks of this warp in the item
            auto bound = [&](int t, bool end) -> uint32_t {   // uniform
                int32_t v = 0;
#pragma unroll
                for (int h = 0; h < kNB; ++h) {
                    const int32_t a = __shfl_sync(0xffffffffu, end ? ce[h] : cs[h], t & 31);
                    if ((t >> 5) == h) v = a;
                }
                return (uint32_t)v;
            };
            // software prefetch of the next batch's corners (x, y, w of corner kb + lane) and of the y after it
            int ptc = 0;
            uint32_t pkb = 0, pce = 0;
            int32_t px = 0, py = 0, pw = 0, pyn = -1;
            auto advance = [&](int t, uint32_t kb_next) {
                uint32_t ce = t < nt ? bound(t, true) : 0u;
                while (t < nt && kb_next >= ce) {
                    ++t;
                    if (t >= nt) break;
                    kb_next = bound(t, false);
                    ce = bound(t, true);
                }
                ptc = t < nt ? t : nt;
                pkb = kb_next;
                pce = ce;
                if (ptc < nt) {
                    const bool ok = pkb + (uint32_t)lane < pce;
                    const int64_t k = k0 + pkb + lane;
                    px = ok ? __ldg(A.x + k) : 0;
                    py = ok ? __ldg(A.y + k) : 0;
                    pw = ok ? __ldg(A.w + k) : 0;
                    pyn = (pkb + 32u < pce) ? __ldg(A.y + k0 + pkb + 32) : -1;
                }
            };
            advance(0, nt > 0 ? bound(0, false) : 0u);
            for (int t = 0; t < nt; ++t) {
                const int j = p + kPW * t;
                const uint32_t g = gbase + (uint32_t)j;
                const int s = (int)(g % kAS);     // the stage's (g / kAS)-th use
                const uint32_t ca = bound(t, false), cb = bound(t, true);
                FCFS_DCHECK(ca <= cb && (!real || (int64_t)cb <= A.corner_ptr[clip + 1] - k0));
                // stage s is free once the MMAs of its previous use (chunk g - kAS) completed; an older use
                // cannot be pending: this warp's previous chunk g - kPW >= g - kAS waited for chunk g - kPW - kAS
                // (a sleeping poll: try_wait's own suspend wakes on every barrier event of the CTA, so a parked
                // warp would keep taking issue slots from the working producers of its sub-partition)
                TR(if (lane == 0 && g < kTrMax) g_tr[g][q] = clock64());
                mbar_wait_backoff(AEMPTY(s), ((g / kAS) & 1u) ^ 1u, 128);
                TR(if (lane == 0 && g < kTrMax) g_tr[g][4 + q] = clock64());
                tc_fence_after();
                const uint32_t tcol = tmem + lrow + kColA + (uint32_t)kStageCols * (uint32_t)s;
                tmem_st_zero32(tcol);
                tmem_st_zero16(tcol + 32);
                tmem_wait_st();
                const int32_t y0 = j * kYC;
                float2 acc = make_float2(0.f, 0.f);     // (cos, sin) sums of the current row
                for (uint32_t kb = ca; kb < cb; kb += 32) {
                    const uint32_t n = cb - kb < 32u ? cb - kb : 32u;
                    uint32_t lastmask;
                    // ---- decode (lane i = corner kb + i), from the prefetched registers
                    {
                        const bool ok = (uint32_t)lane < n;
                        const int32_t x = px, yy = py, w = pw, yafter = pyn;
                        advance(t, kb + 32);                      // next batch's loads in flight
                        int32_t ynext = __shfl_down_sync(0xffffffffu, yy, 1);
                        if ((uint32_t)lane == n - 1) ynext = yafter;   // -1 at the chunk's end
                        const bool last = ok && ynext != yy;
                        // quarter-wave row: x = c_q T/2 + s_q u; cos(m x) = f_q cos(m u), sin(m x) = f_q s_q sin(m u)
                        // with f_q = (-1)^m for q = 1, 2
                        int32_t u;
                        float fs = 1.f, ss = 1.f, cq = 0.f;
                        if (x <= T4) { u = x; }
                        else if (x <= T2) { u = T2 - x; fs = -1.f; ss = -1.f; cq = 1.f; }
                        else if (x <= T34) { u = x - T2; fs = -1.f; cq = 1.f; }
                        else { u = T - x; ss = -1.f; cq = 2.f; }
                        const uint32_t a = tabaddr + (uint32_t)u * rowb;
                        FCFS_DCHECK(!ok || (u >= 0 && u <= T4 && yy >= y0 && yy < y0 + kYC));
                        const float wf = (float)w;
                        const uint32_t wodd = bf16_bits(wf) | (bf16_bits(wf * ss) << 16);            // even m
                        const uint32_t wevn = bf16_bits(wf * fs) | (bf16_bits(wf * ss * fs) << 16);   // odd m
                        const uint32_t wax = bf16_bits(wf * cq) | (bf16_bits(wf * ss) << 16);         // axis lane
                        sts64u(stg + kRec * lane, a, wevn);          // lane l even <-> m = l + 1 odd
                        sts64u(stg + kRec * lane + 8u, a, wodd);
                        sts64u(stg + kRec * lane + 16u, a, wax);
                        lastmask = __reduce_or_sync(0xffffffffu, last ? (1u << lane) : 0u);
                        FCFS_DCHECK(n >= 1 && n <= 32);
                        sts32(fcl + 4u * lane, 2u * (uint32_t)(yy - y0));   // the row's (hi, lo) column pair
                    }
                    __syncwarp();
                    // ---- gather (uniform control)
                    for (uint32_t i = 0; i < n; ++i) {
                        const uint2 r = lds64u(recl + kRec * i);
                        const float2 v = lds64(r.x + lane8);
                        acc = ffma2(v, make_float2(__uint_as_float(r.y << 16), __uint_as_float(r.y & 0xFFFF0000u)), acc);
                        FCFS_DCHECK(r.x >= tabaddr && r.x + lane8 + 8u <= sbase + L.stage);
                        if ((lastmask >> i) & 1u) {   // row end: its (hi, lo) pairs into the row's columns
                            const uint32_t col = lds32(fcl + 4u * i);
                            FCFS_DCHECK(col < 2u * kYC);
                            uint32_t h, l, h2, l2;
                            split_hl(acc.x, h, l);
                            split_hl(acc.y, h2, l2);
                            tmem_st2(tcol + col, h, l);
                            tmem_st2(tcol + 2u * kYC + col, h2, l2);
                            acc = make_float2(0.f, 0.f);
                        }
                    }
                    __syncwarp();
                }
                tmem_wait_st();
                __syncwarp();
                tc_fence_before();
                TR(if (lane == 0 && g < kTrMax) g_tr[g][8 + q] = clock64());
                named_arrive(kBarFull + s, kFullCount);     // stage full: the MMA warps wait on this
            }
            gbase += (uint32_t)nch;
        }
    } else if (warp == kMma || warp == kMma + 1) {
        // ============================ MMA issuers: D_c (kMma), D_s (kMma + 1) ============================
        // Two warps, one per accumulator: each waits for the chunk, issues its 6 MMAs and commits (the
        // stage and B slot barriers expect both commits), so neither loop is on the other's critical path.
        const int d = warp - kMma;
        const uint32_t bring = sbase + L.bring;
        const uint64_t bdesc0 = umma_desc_kmajor_noswz(bring, 64 * 16, 128);   // K core columns 1 KB apart
        const uint32_t dt = tmem + 64u * (uint32_t)d;
        uint32_t td = 0;   // D blocks issued
        uint32_t gc = 0;
        // incremental stage / slot / phase / block counters (no division in the issue loop)
        uint32_t s = 0, b = 0, bph = 0;
        for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x) {
            // (j - first block start) mod kFlush: D_c blocks start at j % kFlush == 0, D_s at kFlush / 2
            int jf = d == 0 ? 0 : kFlush - kFlush / 2;
            for (int j = 0; j < nch; ++j, ++gc) {
                FCFS_DCHECK(s == gc % kAS && b == gc % kBS && bph == ((gc / kBS) & 1u));
                TR(if (lane == 0 && gc < kTrMax) g_trm[gc][2 + d] = clock64());
                mbar_wait_park(BFULL(b), bph);
                named_bar(kBarFull + (int)s, kFullCount);   // the 4 producer warps of the chunk have filled it
                TR(if (lane == 0 && gc < kTrMax) g_trm[gc][d] = clock64());
                const bool fresh = j == 0 || jf == 0;
                FCFS_DCHECK(fresh == (d == 0 ? c_start(j) : s_start(j)));
                if (fresh) mbar_wait_park(DEMPTY(d), (td & 1u) ^ 1u);   // the epilogue took the last block
                tc_fence_after();
                const uint32_t ad = tmem + kColA + (uint32_t)kStageCols * s + 2u * kYC * (uint32_t)d;
                const uint64_t b1 = bdesc0 + (uint64_t)(b * (uint32_t)(kBChunk >> 4));
                const uint64_t b2 = b1 + (uint64_t)(kBTile >> 4);
                const bool end = jf == kFlush - 1 || j == nch - 1;
                FCFS_DCHECK(end == (d == 0 ? c_end(j, nch) : s_end(j, nch)));
                const uint32_t sc = s, bc = b;
                static_assert((kAS & (kAS - 1)) == 0, "stage counter wraps by mask");
                s = (s + 1u) & (kAS - 1u);
                if (++b == (uint32_t)kBS) { b = 0; bph ^= 1u; }
                if (++jf == kFlush) jf = 0;
                if (elect_one()) {
#pragma unroll
                    for (int u = 0; u < kYC / 4; ++u)   // (A^hi + A^lo) B^hi over the interleaved K
                        umma_ts(dt, ad + 8u * u, b1 + 128u * u, (u > 0 || !fresh) ? 1u : 0u);
#pragma unroll
                    for (int u = 0; u < kYC / 4; ++u)   // A^hi B^lo
                        umma_ts(dt, ad + 8u * u, b2 + 128u * u, 1u);
                    umma_commit(AEMPTY(sc));
                    umma_commit(BEMPTY(bc));
                    if (end) umma_commit(DFULL(d));
                }
                __syncwarp();
                if (end) { named_arrive(kBarD + d, 32 + kEpi * 32); ++td; }
            }
        }
    } else if (warp == kLoad) {
        // ================================ B loader ================================
        // streams the B chunks (16 KB each, L2-resident: the table is shared by every clip) into the ring
        const uint32_t bring = sbase + L.bring;
        uint32_t lc = 0;
        for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x) {
            for (int j = 0; j < nch; ++j, ++lc) {
                const int slot = (int)(lc % kBS);
                // a sleeping poll: the loader runs kBS chunks ahead, and a spinning wait would take issue
                // slots from the producers of its sub-partition
                mbar_wait_backoff(BEMPTY(slot), ((lc / kBS) & 1u) ^ 1u, 256);
                if (elect_one()) {
                    mbar_expect_tx(BFULL(slot), kBChunk);
                    bulk_g2s(bring + (uint32_t)slot * kBChunk, A.btab + (size_t)j * kBChunk, kBChunk, BFULL(slot));
                }
                __syncwarp();
            }
        }
    } else {
        // ================================ epilogue ================================
        // Warp q owns TMEM lanes 32q..32q+31 = clip q of each item.  Per finished accumulation block of D_c
        // or D_s it copies the block to registers, releases D at once, then adds it into the FP32 sums S
        // in the CTA's global scratch (its own lane's row: float4 loads / stores coalesced over the warp);
        // per item it then writes the clip's window / pupil coefficients from S.
        const int q = warp - kProd;   // warps kProd .. kProd + 3: warp % 4 == q (TMEM lane quadrant)
        const uint32_t lrow = (uint32_t)(32 * q) << 16;
        float4 *Sq = A.S + ((size_t)blockIdx.x * kClips + q) * 32 * 32;   // [col quad][lane]
        uint32_t t_[2] = {0u, 0u};
        for (int64_t item = blockIdx.x; item < A.items; item += gridDim.x) {
            bool first[2] = {true, true};
            for (int j = 0; j < nch; ++j) {
                const bool ev[2] = {c_end(j, nch), s_end(j, nch)};
#pragma unroll
                for (int d = 0; d < 2; ++d) {   // at a shared j (j == nch-1) the MMA warp arrives for c first
                    if (!ev[d]) continue;
                    named_bar(kBarD + d, 32 + kEpi * 32);
                    mbar_wait(DFULL(d), t_[d] & 1u);
                    tc_fence_after();
                    const uint32_t dsrc = tmem + lrow + 64u * (uint32_t)d;
                    uint32_t rd[64];
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        uint32_t r16[16];
                        TMEM_LD16(dsrc + 16u * h, r16);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; ++i) rd[16 * h + i] = r16[i];
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(DEMPTY(d));   // D is free for the next block's MMAs
                    float4 *Sd = Sq + (size_t)(16 * d) * 32 + lane;
#pragma unroll
                    for (int c4 = 0; c4 < 16; ++c4) {
                        float4 v = make_float4(__uint_as_float(rd[4 * c4]), __uint_as_float(rd[4 * c4 + 1]),
                                               __uint_as_float(rd[4 * c4 + 2]), __uint_as_float(rd[4 * c4 + 3]));
                        if (!first[d]) {
                            const float4 o = Sd[c4 * 32];
                            v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
                        }
                        Sd[c4 * 32] = v;
                    }
                    first[d] = false;
                    ++t_[d];
                }
            }
            // ---- a4 + a5.  S columns: c < 31: n = c + 1 (cos), 31: the y-weighted axis column, 31 + b: n = b (sin).
            // The TMEM loads are warp-wide (tcgen05.ld is .sync.aligned); each lane then writes its own row.
            const int64_t clip = item * kClips + q;
            if (clip < A.B) {
                void *Fc = ea.out_f32 ? (void *)((float2 *)A.F + clip * ea.out_per_clip)
                                      : (void *)((double2 *)A.F + clip * ea.out_per_clip);
                const bool dmask = ea.layout == FCFS_LAYOUT_DENSE && ea.r2 >= 0.0;
                auto Sv = [&](int c) -> float {   // S column c of this lane (c < 64: D_c, c >= 64: D_s)
                    const float4 v = Sq[(size_t)(c >> 2) * 32 + lane];
                    return (c & 3) == 0 ? v.x : ((c & 3) == 1 ? v.y : ((c & 3) == 2 ? v.z : v.w));
                };
                const bool row = lane < M, ax = lane == M;
                const int m = lane + 1;
                const int nm = row ? nmaxr[ea.M + m] : (ax ? nmaxr[ea.M] : -1);
                const int32_t op = row ? rowoff[ea.M + m] + nm : (ax ? rowoff[ea.M] + nm : 0);
                const int32_t on = row ? rowoff[ea.M - m] + nm : 0;
                const double mm = (double)m * (double)m;
                FCFS_DCHECK(nm < 0 || (op - nm >= 0 && op + nm < ea.out_per_clip &&
                                       (!row || (on - nm >= 0 && on + nm < ea.out_per_clip))));
                {
                    const float a1 = Sv(31), a2 = Sv(64 + 31);
                    if (row && nm >= 0) {   // n = 0: Eq. Fk0, F[m,0] = i (Pc_ax - i Ps_ax) / (2 pi m T)
                        const bool mk = dmask && mm > ea.r2;
                        const double re = mk ? 0.0 : (double)a2 * f_axm[m];
                        const double im = mk ? 0.0 : (double)a1 * f_axm[m];
                        store_out(Fc, op, make_double2(re, im), ea.out_f32);
                        store_out(Fc, on, make_double2(re, -im), ea.out_f32);
                    } else if (ax && nm >= 0) {   // DC (Eq. Fdc)
                        const double dc = (double)ea.area_dev[clip] / ((double)T * (double)T);
                        store_out(Fc, op, make_double2(dc, 0.0), ea.out_f32);
                    }
                }
#pragma unroll
                for (int g = 0; g < 4; ++g) {   // b = 8 g + 1 .. 8 g + 8
                    if (8 * g + 1 > N) break;   // uniform
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int b = 8 * g + i + 1;
                        if (b > nm) break;
                        // S_c[b - 1], S_c[31 + b], S_s[b - 1], S_s[31 + b]
                        const double c_c = Sv(b - 1), c_s = Sv(31 + b);
                        const double s_c = Sv(64 + b - 1), s_s = Sv(64 + 31 + b);
                        if (row) {
                            // Eq. Fkl: S(m, +-b) from the quadrant products, F = -S / (4 pi^2 m n)
                            const bool mk = dmask && mm + (double)b * (double)b > ea.r2;
                            const double sc = f_rows[m] * f_invn[b];
                            double re = mk ? 0.0 : (c_c - s_s) * sc, im = mk ? 0.0 : -(s_c + c_s) * sc;   // n = +b
                            store_out(Fc, op + b, make_double2(re, im), ea.out_f32);
                            store_out(Fc, on - b, make_double2(re, -im), ea.out_f32);
                            re = mk ? 0.0 : -(c_c + s_s) * sc;                                              // n = -b
                            im = mk ? 0.0 : (s_c - c_s) * sc;
                            store_out(Fc, op - b, make_double2(re, im), ea.out_f32);
                            store_out(Fc, on + b, make_double2(re, -im), ea.out_f32);
                        } else {   // lane M: F[0,b] = i (P_ax,c - i P_ax,s) / (2 pi b T), P_ax = D_c + D_s of lane M
                            const bool mk = dmask && (double)b * (double)b > ea.r2;
                            const double re = mk ? 0.0 : (c_s + s_s) * f_axm[b];
                            const double im = mk ? 0.0 : (c_c + s_c) * f_axm[b];
                            store_out(Fc, op + b, make_double2(re, im), ea.out_f32);
                            store_out(Fc, op - b, make_double2(re, -im), ea.out_f32);
                        }
                    }
                }
            }
            __syncwarp();
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == kMma) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

// B operand of chunk c (kYC lattice rows y = kYC c + i), N-rows: b - 1 = cos(2 pi b y / T) for b = 1..N, 31 = y
// (the coordinate weight of Eq. Fk0), 31 + b = sin(2 pi b y / T); other rows and y > T: 0.  Split v = hi + lo
// (hi = tf32(v), lo = tf32(v - hi)); B' holds (hi, hi) at K = (2i, 2i+1), B'' holds (lo, 0); both in the
// K-major no-swizzle layout (row r, k).
__global__ void k_lat_btab(int32_t T, int32_t N, int32_t nch, uint8_t *__restrict__ btab) {
    constexpr int kKP = kYC;   // K pairs (hi, hi) / (lo, 0): one per lattice row
    const int64_t total = (int64_t)nch * 64 * kKP;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i / (64 * kKP));
        const int r = (int)((i / kKP) % 64);
        const int yi = (int)(i % kKP);
        const int64_t y = (int64_t)c * kYC + yi;
        double v = 0.0;
        if (yi < kYC && y <= T) {
            if (r < 31 && r < N) v = cospi(2.0 * (double)(((int64_t)(r + 1) * y) % T) / (double)T);
            else if (r == 31) v = (double)y;
            else if (r > 31 && r - 31 <= N) v = sinpi(2.0 * (double)(((int64_t)(r - 31) * y) % T) / (double)T);
        }
        const float hi = __uint_as_float(tc::tf32_rna((float)v));
        const float lo = __uint_as_float(tc::tf32_rna((float)(v - (double)hi)));
        uint8_t *ch = btab + (size_t)c * kBChunk;
        for (int h = 0; h < 2; ++h) {
            const int k = 2 * yi + h;
            // K-major, no swizzle: 8-row x 16-byte core matrices, 128 B apart along N, 1 KB apart along K
            const uint32_t off = (uint32_t)(k / 4) * 1024u + (uint32_t)(r / 8) * 128u + (uint32_t)(r % 8) * 16u +
                                 (uint32_t)(k % 4) * 4u;
            *(float *)(ch + off) = hi;
            *(float *)(ch + kBTile + off) = h == 0 ? lo : 0.f;
        }
    }
}

// the quarter-wave table of k_lattice, once per call (every CTA copies it from L2 instead of evaluating
// (T/4 + 2)(M + 1) FP64 sincospi): row u, lane l < M: (cos, sin)(2 pi (l+1) u / T); lane M: (T/2, u) (the
// x-weighted axis row); rows past T/4: 0
__global__ void k_lat_qtab(int32_t T, int32_t M, float2 *__restrict__ qtab) {
    const int rows = T / 4 + 2, lanes = M + 1;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows * lanes + 32; i += gridDim.x * blockDim.x) {
        const int u = i / lanes, l = i % lanes;
        double sn = 0.0, cs = 0.0;
        if (u <= T / 4) {
            if (l < M) sincospi(2.0 * (double)(((int64_t)(l + 1) * u) % T) / (double)T, &sn, &cs);
            else { cs = 0.5 * (double)T; sn = (double)u; }
        }
        qtab[i] = make_float2((float)cs, (float)sn);
    }
}

// chunk starts of every clip: cptr[b][j] = first corner (relative to the clip's start) with y >= 16 j,
// j = 0 .. nch (cptr[b][nch] = the clip's corner count): one thread per (clip, j), a binary search over the
// clip's y-sorted corners (latency hidden by the thread count)
__global__ void __launch_bounds__(256) k_lat_cptr(const int64_t *__restrict__ corner_ptr, int64_t B,
                                                  const int32_t *__restrict__ y, int32_t nch, int32_t *__restrict__ cptr) {
    const int64_t total = B * (int64_t)(nch + 1);
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / (nch + 1);
        const int32_t j = (int32_t)(t - b * (nch + 1));
        const int64_t k0 = corner_ptr[b];
        int32_t lo = 0, hi = (int32_t)(corner_ptr[b + 1] - k0);
        const int32_t yv = j * kYC;
        while (lo < hi) {
            const int32_t mid = (lo + hi) >> 1;
            if (__ldg(y + k0 + mid) < yv) lo = mid + 1;
            else hi = mid;
        }
        cptr[t] = lo;
    }
}

// y-sortedness of every clip: a decrease y[k-1] > y[k] is allowed only where k starts a clip
__global__ void __launch_bounds__(256) k_lat_sorted(const int64_t *__restrict__ corner_ptr, int64_t B,
                                                    const int32_t *__restrict__ y, int64_t K, int32_t *__restrict__ unsorted) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; k < K; k += (int64_t)gridDim.x * blockDim.x) {
        if (__ldg(y + k - 1) <= __ldg(y + k)) continue;
        int64_t lo = 0, hi = B;   // is k a clip start?  (rare: a decrease)
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (corner_ptr[mid] < k) lo = mid + 1;
            else hi = mid;
        }
        if (lo > B || corner_ptr[lo] != k) *unsorted = 1;
    }
}

}  // namespace lat

int32_t lattice_chunks(int32_t T) { return (T + 1 + lat::kYC - 1) / lat::kYC; }

size_t lattice_smem_bytes(int32_t T, int32_t M) { return (size_t)lat::layout(T, M).total + 1024; }

// the lattice-row form applies (T and window limits, SMEM budget); the caller adds the sortedness condition
bool lattice_eligible(int32_t T, const EpiArgs &ea) {
    if (T < 4 || (T % 4) != 0 || T > 2496) return false;   // quarter-wave table rows in SMEM; chunk registers
    if (ea.M < 0 || ea.N < 0 || ea.M > 31 || ea.N > 31) return false;
    if (ea.m_lo != -ea.M || ea.m_hi != ea.M || !ea.out_f32) return false;
    if (lattice_chunks(T) > lat::kMaxChunks) return false;   // the producers' register-cached chunk bounds
    return lattice_smem_bytes(T, ea.M) <= 227 * 1024;
}

static size_t btab_bytes(int32_t T) { return ((size_t)lattice_chunks(T) * lat::kBChunk + 255) & ~(size_t)255; }

static int lattice_grid(int64_t B) {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t items = (B + lat::kClips - 1) / lat::kClips;
    return (int)(items < sms ? items : sms);
}

static size_t cptr_bytes(int64_t B, int32_t T) { return ((size_t)B * (lattice_chunks(T) + 1) * 4 + 255) & ~(size_t)255; }
static constexpr size_t kSBytesPerCta = (size_t)lat::kClips * 32 * 32 * sizeof(float4);   // 64 KB

static size_t qtab_bytes(int32_t T) { return ((size_t)(T / 4 + 2) * (lat::kMaxRows / 2) * 8 + 32 * 8 + 255) & ~(size_t)255; }

size_t lattice_ws_bytes(int64_t B, int32_t T) {
    return btab_bytes(T) + cptr_bytes(B, T) + (size_t)lattice_grid(B) * kSBytesPerCta + qtab_bytes(T) + 256;
}

fcfs_status launch_lattice_prepare(const int64_t *corner_ptr, int64_t B, const int32_t *y, int64_t K, int32_t T,
                                   int32_t M, int32_t N, void *ws, int32_t *unsorted_dev, bool check, cudaStream_t s) {
    const int32_t nch = lattice_chunks(T);
    uint8_t *btab = (uint8_t *)ws;
    int32_t *cptr = (int32_t *)(btab + btab_bytes(T));
    lat::k_lat_btab<<<148, 256, 0, s>>>(T, N, nch, btab);
    FCFS_CHECK_LAUNCH("k_lat_btab");
    float2 *qtab = (float2 *)(btab + btab_bytes(T) + cptr_bytes(B, T) + (size_t)lattice_grid(B) * kSBytesPerCta);
    lat::k_lat_qtab<<<148, 256, 0, s>>>(T, M, qtab);
    FCFS_CHECK_LAUNCH("k_lat_qtab");
    const int64_t threads = B * (int64_t)(nch + 1);
    const int64_t blocks = (threads + 255) / 256;
    lat::k_lat_cptr<<<(unsigned)(blocks < 65536 ? blocks : 65536), 256, 0, s>>>(corner_ptr, B, y, nch, cptr);
    FCFS_CHECK_LAUNCH("k_lat_cptr");
    if (check && K > 1) {
        const int64_t kb = (K + 255) / 256;
        lat::k_lat_sorted<<<(unsigned)(kb < 65536 ? kb : 65536), 256, 0, s>>>(corner_ptr, B, y, K, unsorted_dev);
        FCFS_CHECK_LAUNCH("k_lat_sorted");
    }
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
    a.cptr = (const int32_t *)((const uint8_t *)ws + btab_bytes(T));
    a.S = (float4 *)((uint8_t *)ws + btab_bytes(T) + cptr_bytes(B, T));
    a.qtab = (const float2 *)((const uint8_t *)ws + btab_bytes(T) + cptr_bytes(B, T) +
                              (size_t)lattice_grid(B) * kSBytesPerCta);
    a.T = T; a.M = ea.M; a.N = ea.N; a.nch = nch;
    a.items = (B + lat::kClips - 1) / lat::kClips;
    a.ea = ea;
    a.F = F;
    const size_t smem = lattice_smem_bytes(T, ea.M);
    FCFS_TRY(ensure_smem((const void *)lat::k_lattice, smem, true));
    const int grid = lattice_grid(B);
    lat::k_lattice<<<(unsigned)grid, lat::kThreads, smem, s>>>(a);
    FCFS_CHECK_LAUNCH("k_lattice");
    return FCFS_OK;
}

}  // namespace fcfs

#ifdef LAT_TRACE
extern "C" int fcfs_lat_trace_read(void *tr, void *trm) {
    if (cudaMemcpyFromSymbol(tr, fcfs::lat::g_tr, sizeof(fcfs::lat::g_tr)) != cudaSuccess) return -1;
    if (cudaMemcpyFromSymbol(trm, fcfs::lat::g_trm, sizeof(fcfs::lat::g_trm)) != cudaSuccess) return -1;
    return 0;
}
#endif

// edges.cu — the K/2-term form of Eq. Fkl (SURVEY §8(f) NEXT-1 "edge pairing") for the
// batched split-TF32 contraction.  Two consecutive corners of the list that lie on one row (same y)
// with opposite weights, w_{k+1} = -w_k, are one horizontal edge:
//
//     w_k E(m x_k) E(n y) + w_{k+1} E(m x_{k+1}) E(n y) = w_k (E(m x_k) - E(m x_{k+1})) E(n y),
//
// so the contraction runs over edges (x_a, x_b, y, c) instead of corners: the y-side operand, the
// operand bytes, the MMAs and the pipeline stages halve (the x side evaluates both ends).  Pairs are
// taken along each maximal chain of such links at chain positions (0,1), (2,3), ...; an unpaired
// corner is a one-ended edge (x_b = -1: no second term).  The identity is term-by-term, so it is
// exact for ANY corner list (any order, any weights), and sum over edges of 2 |c| = sum_k |w_k|: the
// error budget of the 1e-5 B contract is unchanged.  Canonical lists (rows y-sorted, weights
// alternating +-1 along x, as fcfs_vertices_from_* emit them) give about K/2 edges.
//
// Layout: the edges of clip b occupy [corner_ptr[b], corner_ptr[b] + ecnt[b]) of four int32 arrays
// (a clip never has more edges than corners), so no global compaction and no host sync.  The edges
// keep the corner order (each edge sits at its head corner's rank among the emitted corners).
#include "common.cuh"

namespace fcfs {

// warp per clip, kCpl consecutive corners per lane (32 kCpl per step).  The next step's corners are loaded
// while this one is processed; inside a lane the links, chain starts and emits are local; across
// lanes one ballot finds the last chain start before each lane and one warp scan places the edges.
constexpr int kCpl = 2;   // corners per lane per step (measured: 1: 0.160 ms, 2: 0.118, 4: 0.141, 8: 0.165 on c3)

__global__ void __launch_bounds__(256)
k_edges(const int32_t *__restrict__ x, const int32_t *__restrict__ y, const int32_t *__restrict__ w,
        const int64_t *__restrict__ corner_ptr, int64_t B, int32_t *exa, int32_t *exb, int32_t *ey, int32_t *ec,
        int32_t *ecnt) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < B; b += nw) {
        const int64_t kb = corner_ptr[b], ke = corner_ptr[b + 1];
        int64_t cstart = kb;            // last chain start before the current step
        int32_t py = 0, pw = 0;         // the corner before the current step (valid if g0 > kb)
        int32_t cnt = 0;
        int32_t X[kCpl], Y[kCpl], W[kCpl], NX = 0, NY = 0, NW = 0;   // a step + the corner after it
        auto load = [&](int64_t g0) {
#pragma unroll
            for (int i = 0; i < kCpl; ++i) {
                const int64_t k = g0 + kCpl * lane + i;
                const bool ok = k < ke;
                X[i] = ok ? __ldg(x + k) : 0;
                Y[i] = ok ? __ldg(y + k) : 0;
                W[i] = ok ? __ldg(w + k) : 0;
            }
            const int64_t kn = g0 + 32 * kCpl;
            if (lane == 31 && kn < ke) { NX = __ldg(x + kn); NY = __ldg(y + kn); NW = __ldg(w + kn); }
        };
        load(kb);
        for (int64_t g0 = kb; g0 < ke; g0 += 32 * kCpl) {
            int32_t cx[kCpl], cy[kCpl], cw[kCpl];
#pragma unroll
            for (int i = 0; i < kCpl; ++i) { cx[i] = X[i]; cy[i] = Y[i]; cw[i] = W[i]; }
            const int32_t cnx = NX, cny = NY, cnw = NW;
            const int64_t gn = g0 + 32 * kCpl;
            if (gn < ke) load(gn);      // in flight while this step is processed
            const int64_t k0 = g0 + kCpl * lane;
            // neighbours across lanes
            int32_t ly = __shfl_up_sync(0xffffffffu, cy[kCpl - 1], 1), lw = __shfl_up_sync(0xffffffffu, cw[kCpl - 1], 1);
            if (lane == 0) { ly = py; lw = pw; }
            int32_t nx = __shfl_down_sync(0xffffffffu, cx[0], 1), ny = __shfl_down_sync(0xffffffffu, cy[0], 1),
                    nw_ = __shfl_down_sync(0xffffffffu, cw[0], 1);
            if (lane == 31) { nx = cnx; ny = cny; nw_ = cnw; }   // the corner after the step (or unused)
            bool lin[kCpl], lout[kCpl];
#pragma unroll
            for (int i = 0; i < kCpl; ++i) {
                const int64_t k = k0 + i;
                const bool valid = k < ke;
                const int32_t yp = i ? cy[i - 1] : ly, wp = i ? cw[i - 1] : lw;
                lin[i] = valid && k > kb && yp == cy[i] && wp == -cw[i];
                const int32_t yn = i + 1 < kCpl ? cy[i + 1 < kCpl ? i + 1 : 0] : ny;
                const int32_t wn = i + 1 < kCpl ? cw[i + 1 < kCpl ? i + 1 : 0] : nw_;
                lout[i] = valid && k + 1 < ke && yn == cy[i] && wn == -cw[i];
            }
            // last chain start in this lane (-1: none), then the last one before this lane
            int lst = -1;
#pragma unroll
            for (int i = 0; i < kCpl; ++i)
                if (k0 + i < ke && !lin[i]) lst = i;
            const unsigned has = __ballot_sync(0xffffffffu, lst >= 0);
            const unsigned before = has & ((1u << lane) - 1u);
            const int src = before ? 31 - __clz(before) : 0;
            const int lst_src = __shfl_sync(0xffffffffu, lst, src);
            int64_t st = before ? g0 + kCpl * src + lst_src : cstart;
            int n_emit = 0;
            bool em[kCpl];
#pragma unroll
            for (int i = 0; i < kCpl; ++i) {
                const int64_t k = k0 + i;
                if (k < ke && !lin[i]) st = k;
                em[i] = k < ke && ((k - st) & 1) == 0;
                n_emit += em[i];
            }
            int inc = n_emit;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += v;
            }
            int64_t p = kb + cnt + (inc - n_emit);
#pragma unroll
            for (int i = 0; i < kCpl; ++i) {
                if (em[i]) {
                    const int32_t xn = i + 1 < kCpl ? cx[i + 1 < kCpl ? i + 1 : 0] : nx;
                    exa[p] = cx[i];
                    exb[p] = lout[i] ? xn : -1;
                    ey[p] = cy[i];
                    ec[p] = cw[i];
                    ++p;
                }
            }
            cnt += __shfl_sync(0xffffffffu, inc, 31);
            if (has) {
                const int ls = 31 - __clz(has);
                cstart = g0 + kCpl * ls + __shfl_sync(0xffffffffu, lst, ls);
            } else {
                (void)__shfl_sync(0xffffffffu, lst, 0);
            }
            py = __shfl_sync(0xffffffffu, cy[kCpl - 1], 31);
            pw = __shfl_sync(0xffffffffu, cw[kCpl - 1], 31);
        }
        if (lane == 0) ecnt[b] = cnt;
    }
}

void carve_edges(Carver &cv, int64_t K, int64_t B, EdgeWs &e) {
    const size_t k1 = (size_t)(K > 0 ? K : 1);
    e.xa = cv.take<int32_t>(k1);
    e.xb = cv.take<int32_t>(k1);
    e.y = cv.take<int32_t>(k1);
    e.c = cv.take<int32_t>(k1);
    e.cnt = cv.take<int32_t>((size_t)(B > 0 ? B : 1));
}

fcfs_status run_edges(const int32_t *x, const int32_t *y, const int32_t *w, const int64_t *corner_ptr, int64_t B,
                      const EdgeWs &e, cudaStream_t s) {
    int64_t blocks = (B * 32 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    k_edges<<<(unsigned)blocks, 256, 0, s>>>(x, y, w, corner_ptr, B, e.xa, e.xb, e.y, e.c, e.cnt);
    FCFS_CHECK_LAUNCH("k_edges");
    return FCFS_OK;
}

}  // namespace fcfs

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
// (a clip never has more edges than corners), so no global compaction and no host sync.
#include "common.cuh"

namespace fcfs {

// warp per clip; groups of kG chunks of 32 corners whose loads are all issued together (the loop is
// otherwise one dependent HBM round trip per chunk); the chain start is carried across chunks
constexpr int kG = 8;

__global__ void k_edges(const int32_t *__restrict__ x, const int32_t *__restrict__ y, const int32_t *__restrict__ w,
                        const int64_t *__restrict__ corner_ptr, int64_t B, int32_t *exa, int32_t *exb, int32_t *ey,
                        int32_t *ec, int32_t *ecnt) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < B; b += nw) {
        const int64_t kb = corner_ptr[b], ke = corner_ptr[b + 1];
        int64_t cstart = kb;   // start of the chain the next chunk's first corner may continue
        int32_t cnt = 0;
        for (int64_t g0 = kb; g0 < ke; g0 += 32 * kG) {
            int32_t X[kG], Y[kG], W[kG];
#pragma unroll
            for (int j = 0; j < kG; ++j) {
                const int64_t k = g0 + 32 * j + lane;
                const bool ok = k < ke;
                X[j] = ok ? __ldg(x + k) : 0;
                Y[j] = ok ? __ldg(y + k) : 0;
                W[j] = ok ? __ldg(w + k) : 0;
            }
            const int64_t gn = g0 + 32 * kG;
            const int32_t yprev = g0 > kb ? __ldg(y + g0 - 1) : 0, wprev = g0 > kb ? __ldg(w + g0 - 1) : 0;
            const int32_t xnext = gn < ke ? __ldg(x + gn) : 0, ynext = gn < ke ? __ldg(y + gn) : 0,
                          wnext = gn < ke ? __ldg(w + gn) : 0;
#pragma unroll
            for (int j = 0; j < kG; ++j) {
                const int64_t k0 = g0 + 32 * j;
                if (k0 >= ke) break;   // warp-uniform
                const int64_t k = k0 + lane;
                const bool valid = k < ke;
                const int32_t xk = X[j], yk = Y[j], wk = W[j];
                // neighbours: inside the chunk by shuffles, across chunks from the adjacent registers
                const int32_t pl_y = j > 0 ? __shfl_sync(0xffffffffu, Y[j > 0 ? j - 1 : 0], 31) : yprev;
                const int32_t pl_w = j > 0 ? __shfl_sync(0xffffffffu, W[j > 0 ? j - 1 : 0], 31) : wprev;
                const int32_t nf_x = j + 1 < kG ? __shfl_sync(0xffffffffu, X[j + 1 < kG ? j + 1 : 0], 0) : xnext;
                const int32_t nf_y = j + 1 < kG ? __shfl_sync(0xffffffffu, Y[j + 1 < kG ? j + 1 : 0], 0) : ynext;
                const int32_t nf_w = j + 1 < kG ? __shfl_sync(0xffffffffu, W[j + 1 < kG ? j + 1 : 0], 0) : wnext;
                int32_t yp = __shfl_up_sync(0xffffffffu, yk, 1), wp = __shfl_up_sync(0xffffffffu, wk, 1);
                if (lane == 0) { yp = pl_y; wp = pl_w; }
                int32_t xn = __shfl_down_sync(0xffffffffu, xk, 1), yn = __shfl_down_sync(0xffffffffu, yk, 1),
                        wn = __shfl_down_sync(0xffffffffu, wk, 1);
                if (lane == 31) { xn = nf_x; yn = nf_y; wn = nf_w; }
                const bool link_in = valid && k > kb && yp == yk && wp == -wk;        // (k-1, k) may pair
                const bool link_out = valid && k + 1 < ke && yn == yk && wn == -wk;   // (k, k+1) may pair
                const unsigned starts = __ballot_sync(0xffffffffu, !link_in);
                const unsigned upto = starts & (0xffffffffu >> (31 - lane));
                const int64_t st = upto ? k0 + (31 - __clz(upto)) : cstart;
                const bool emit = valid && ((k - st) & 1) == 0;   // a pair's head, or an unpaired corner
                const unsigned em = __ballot_sync(0xffffffffu, emit);
                if (emit) {
                    const int64_t p = kb + cnt + __popc(em & ((1u << lane) - 1u));
                    exa[p] = xk;
                    exb[p] = link_out ? xn : -1;
                    ey[p] = yk;
                    ec[p] = wk;
                }
                cnt += __popc(em);
                if (starts) cstart = k0 + (31 - __clz(starts));
            }
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

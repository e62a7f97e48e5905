// common.cuh — internal helpers of libfcfs.so (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdio>
#include <stdint.h>

#include "../../include/fcfs.h"

namespace fcfs {

// ---- error plumbing -------------------------------------------------------------------
void set_error(const char *fmt, ...);
fcfs_status cuda_status(cudaError_t e, const char *where);
void count_launch(int n = 1);
// raise a kernel's dynamic shared-memory limit (and optionally its carveout to the maximum) on the
// current device, once per (device, kernel, size): thread-safe
fcfs_status ensure_smem(const void *fn, size_t bytes, bool max_carveout = false);

// stage timing (fcfs_profile_*): RAII pair of events around a stage on stream s
enum Stage { kStageExtract = 0, kStageContract = 1, kStageEpilogue = 2, kStagePair = 3, kNumStages = 4 };
void profile_mark(int stage, int begin, cudaStream_t s);
struct StageScope {
    int stage;
    cudaStream_t s;
    StageScope(int st, cudaStream_t ss) : stage(st), s(ss) { profile_mark(stage, 1, s); }
    ~StageScope() { profile_mark(stage, 0, s); }
};

#define FCFS_TRY(expr)                                            \
    do {                                                          \
        fcfs_status _st = (expr);                                 \
        if (_st != FCFS_OK) return _st;                           \
    } while (0)
#define FCFS_TRY_CUDA(expr)                                      \
    do {                                                         \
        cudaError_t _e = (expr);                                 \
        if (_e != cudaSuccess) return fcfs::cuda_status(_e, #expr); \
    } while (0)

#define FCFS_CHECK_LAUNCH(name)                                  \
    do {                                                         \
        fcfs::count_launch();                                    \
        cudaError_t _e = cudaGetLastError();                     \
        if (_e != cudaSuccess) return fcfs::cuda_status(_e, name); \
    } while (0)

// ---- device-side invariant checks of the checked build (libfcfs_checked.so, -DFCFS_CHECKED):
// index / address / protocol invariants of the hand-written kernels; a violation prints the site and
// traps (the launch then fails with cudaErrorLaunchFailure -> FCFS_E_CUDA).  Compiled out of
// libfcfs.so.  compute-sanitizer is closed on this GPU pool; this build is the bounds check instead.
#ifdef FCFS_CHECKED
#define FCFS_DCHECK(cond)                                                                              \
    do {                                                                                               \
        if (!(cond)) {                                                                                 \
            printf("FCFS_DCHECK failed: %s at %s:%d block %d thread %d\n", #cond, __FILE__, __LINE__,  \
                   (int)blockIdx.x, (int)threadIdx.x);                                                 \
            __trap();                                                                                  \
        }                                                                                              \
    } while (0)
#else
#define FCFS_DCHECK(cond) ((void)0)
#endif

// ---- workspace carving (256-byte aligned bump allocator) ---------------------------------
struct Carver {
    char *base;
    size_t off, cap;
    explicit Carver(void *b, size_t c) : base((char *)b), off(0), cap(c) {}
    template <typename T>
    T *take(size_t n) {
        size_t a = (off + 255) & ~size_t(255);
        off = a + n * sizeof(T);
        return base ? (T *)(base + a) : nullptr;
    }
    size_t used() const { return (off + 255) & ~size_t(255); }
    bool fits() const { return used() <= cap; }
};

// ---- plan of the real quadrant GEMM P = A diag(w) B^T -------------------
// Side X rows: row 2j = w*cos(2 pi (m0+j) x / T), row 2j+1 = w*sin(...), j < nm;
//              row 2*nm = w*x (axis row) if has_axis.
// Side Y rows: row 2j = cos(2 pi (n0+j) y / T), row 2j+1 = sin(...), j < nn; row 2*nn = y.
// P[ix][iy] = sum_k A[ix,k] B[iy,k].  The epilogue combines quadrant entries into F.
struct SidePlan {
    int32_t f0;      // first positive frequency (>= 1)
    int32_t nf;      // number of positive frequencies
    int32_t axis;    // 1 if the axis row (coordinate weight) is present
    int32_t rows;    // 2*nf + axis
};

// Tiling of P over (clips x tiles_x x tiles_y x splits) work items; P_ws holds one
// kTile x kTile FP64 block per item, row-major [ix][iy].
static constexpr int kTile = 64;

struct GemmPlan {
    SidePlan X, Y;
    int32_t tiles_x, tiles_y, splits;
    int64_t B;                // clips
    int64_t items;            // B * tiles_x * tiles_y * splits
    int32_t dbg;              // ablation build only (-DFCFS_ABLATE, env FCFS_DEBUG); 0 in the shipped library
    int32_t phys;             // P_ws row order inside a 64-row tile: 0 = (c0,s0,c1,s1,...) [FP64 kernel],
                              // 1 = (c0..c31, s0..s31) [tcgen05 kernel]
};

// physical row of logical quadrant row (pair p, t = 0 cos / 1 sin) inside P_ws
__host__ __device__ inline int phys_row(int p, int t, int phys) {
    const int tile = p / (kTile / 2), pp = p - tile * (kTile / 2);
    return tile * kTile + (phys ? pp + (kTile / 2) * t : 2 * pp + t);
}

// Corner source of one contraction: either one clip [k_lo, k_hi) or B clips by CSR, plus its
// row buckets (buckets.cu): the contraction runs over buckets, bucket b = corners
// [bptr[b], bptr[b+1]) sharing the row by[b]; clip c owns buckets [clip_bptr[c], clip_bptr[c+1]).
struct CornerSrc {
    const int32_t *x, *y, *w;
    const int64_t *corner_ptr;   // device CSR [B+1] or nullptr
    int64_t k_lo, k_hi;          // used when corner_ptr == nullptr
    const int32_t *bptr, *by;    // [nb+1], [nb] (workspace, padded for 16-byte bulk copies)
    const int64_t *clip_bptr;    // [B+1] (B = 1 for a single range)
    int64_t kend;                // length of the x / w arrays (bulk copies stay below kend & ~3)
    // edge form (edges.cu; batched split-TF32): clip b's edges are [corner_ptr[b], + ecnt[b]) of
    // (exa, exb, ey, ec); ecnt == nullptr: corner form
    const int32_t *exa, *exb, *ey, *ec, *ecnt;
};

// edge pairing pre-pass (edges.cu)
struct EdgeWs {
    int32_t *xa, *xb, *y, *c, *cnt;
};
void carve_edges(Carver &cv, int64_t K, int64_t B, EdgeWs &e);
fcfs_status run_edges(const int32_t *x, const int32_t *y, const int32_t *w, const int64_t *corner_ptr, int64_t B,
                      const EdgeWs &e, cudaStream_t s);

// row-bucket workspace and pass (buckets.cu)
struct BucketWs {
    int32_t *bptr, *by;
    int64_t *clip_bptr;
    int32_t *counts, *offs;
    void *cub_tmp;
    size_t cub_bytes;
};
void carve_buckets(Carver &cv, int64_t K, int64_t B, BucketWs &w);
size_t buckets_workspace_bytes(int64_t K, int64_t B);
fcfs_status run_buckets(const int32_t *y, const int64_t *corner_ptr, int64_t B, int64_t k_lo, int64_t k_hi,
                        int32_t cap, const BucketWs &w, cudaStream_t s);
static constexpr int kRowBucketCapFp64 = 32;   // max corners per bucket (the FP64 kernel walks a bucket
                                               // warp-uniformly: 32 pairs of one bucket per warp)

struct EpiArgs {
    int32_t M, N, layout;
    double r2;
    int32_t m_lo, m_hi;          // output rows (signed)
    int64_t out_per_clip;
    int32_t T;
    const int64_t *area_dev;     // per-clip area (device) or nullptr
    int64_t area_host;
    int32_t out_f32;             // 1: complex64, 0: complex128
    // ROWS shard written straight into full-window buffers (fcfs_coeffs_rows_to_peers): every output of
    // this rank's rows goes to peer[0 .. peer_n) at its full DENSE-window position; 0 = write F as usual
    int32_t peer_n = 0;
    void *peer[8] = {};
};
constexpr int kMaxPeers = 8;

__host__ __device__ inline int32_t ilog2_ceil(int64_t v) {
    int32_t b = 0;
    while ((int64_t(1) << b) < v) ++b;
    return b;
}

// Two-level twiddle table: r = hi*L + lo, e^{-i th(r)} = E_hi[hi] * E_lo[lo], th(r) = 2 pi r / T.
// Tables hold (cos, sin) of +th; the sign of the imaginary part is applied by the caller.
struct TwiddleGeom {
    int32_t T;
    int32_t lbits;   // L = 2^lbits
    int32_t nhi;     // ceil(T / L)
    int32_t pow2;    // T is a power of two
};

inline TwiddleGeom make_twiddle_geom(int32_t T) {
    TwiddleGeom g;
    g.T = T;
    int32_t tb = ilog2_ceil(T);
    g.lbits = (tb + 1) / 2;
    g.nhi = (int32_t)((T + (1 << g.lbits) - 1) >> g.lbits);
    g.pow2 = ((T & (T - 1)) == 0) ? 1 : 0;
    return g;
}

// exact (m * v) mod T for m >= 0, 0 <= v <= T
__device__ __forceinline__ uint32_t phase_mod(uint32_t m, uint32_t v, const TwiddleGeom &g) {
    if (g.pow2) return (m * v) & (uint32_t)(g.T - 1);   // T | 2^32: wrap-around is harmless
    return (uint32_t)(((uint64_t)m * v) % (uint64_t)g.T);
}

// launchers (contract_fp64.cu, epilogue.cu)
struct FpChunk {
    const double *G;   // x-side bucket sums of the chunk, [tiles_x][cb][64]
    int64_t chunk;     // chunk index
    int64_t cb;        // buckets per chunk
    const double *H;   // y-side row twiddles of the chunk, [tiles_y][cb][64]
};
static constexpr int64_t kFpChunkBuckets = 131072;
// Buckets per chunk of the single-clip paths (the chunk's x- and y-side tiles live in the workspace,
// 512 B per bucket per tile): large chunks, since every chunk re-reads and re-writes the P partials
// (measured: L2-sized chunks of ~4K buckets were slower on configs[3] / [4]); a multiple of 64.
inline int64_t chunk_buckets(int64_t K, int tiles_x, int tiles_y) {
    (void)tiles_x; (void)tiles_y;
    int64_t cb = (K + 63) / 64 * 64;
    if (cb > kFpChunkBuckets) cb = kFpChunkBuckets;
    return cb < 64 ? 64 : cb;
}
int64_t fp64_chunk_buckets(int64_t K);
fcfs_status launch_gemm_fp64(const CornerSrc &src, const GemmPlan &plan, int32_t T, double *P_ws,
                             cudaStream_t s);
fcfs_status launch_gemm_fp64_chunked(const CornerSrc &src, const GemmPlan &plan, int32_t T, int64_t K, double *G,
                                     double *H, double *P_ws, cudaStream_t s);
int64_t tc_chunk_buckets(int64_t K);
fcfs_status launch_gemm_tf32_chunked(const CornerSrc &src, const GemmPlan &plan, int32_t T, int64_t K, uint8_t *G,
                                     uint8_t *H, double *P_ws, bool f16, cudaStream_t s);
fcfs_status launch_epilogue(const GemmPlan &plan, const double *P_ws, const EpiArgs &ea, void *F,
                            cudaStream_t s);
fcfs_status launch_block_area(const CornerSrc &src, int64_t *area_dev, cudaStream_t s);

// the lattice-FFT route of one FP64 clip (fft_route.cu)
struct FftPlan {
    int32_t T, T2, N;
    int32_t f32;       // 1: FP32 arithmetic (split-precision contract), 0: FP64
    int32_t row0;      // the x-weighted row (m = 0) is needed
    int32_t mA, nm;    // rows |m| = mA .. mA + nm - 1
    int32_t nr;        // row0 + nm
    int64_t rc;        // rows per chunk of the G workspace
    int32_t sp;        // sub-row ranges per row in k_fr_fft2 (partial X sums, added in fixed order)
};
bool fft_route_plan(int32_t T, int32_t M, int32_t N, int32_t m_lo, int32_t m_hi, int64_t K, bool f32, FftPlan &p,
                    int32_t route = FCFS_ROUTE_AUTO);
size_t fft_route_ws_bytes(const FftPlan &p);
fcfs_status fft_route_prepare_dev(const int32_t *y, const int64_t *K_dev, int64_t K_cap, const FftPlan &p, void *ws,
                                  size_t ws_bytes, int32_t *status_dev, cudaStream_t s);
fcfs_status fft_route_prepare(const int32_t *y, int64_t k_lo, int64_t K, const FftPlan &p, void *ws, size_t ws_bytes,
                              bool &sorted, cudaStream_t s);
fcfs_status fft_route_run(const int32_t *x, const int32_t *w, int64_t k_lo, const FftPlan &p, void *ws,
                          size_t ws_bytes, const EpiArgs &ea, void *F, cudaStream_t s);

}  // namespace fcfs

// fcfs_abi.cu — the extern "C" boundary of libfcfs.so (include/fcfs.h): argument
// validation, planning, workspace carving and kernel launches on the caller's stream.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"

namespace fcfs {

static thread_local char g_err[1024] = "";
static thread_local int g_launches = 0;

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

fcfs_status cuda_status(cudaError_t e, const char *where) {
    set_error("%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
    return FCFS_E_CUDA;
}

void count_launch(int n) { g_launches += n; }

fcfs_status ensure_smem(const void *fn, size_t bytes, bool max_carveout) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> done;
    int dev = 0;
    FCFS_TRY_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_pair(dev, fn);
    const auto it = done.find(key);
    if (it != done.end() && it->second >= bytes) return FCFS_OK;
    FCFS_TRY_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    if (max_carveout) FCFS_TRY_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    done[key] = bytes;
    return FCFS_OK;
}

struct ProfRec {
    cudaEvent_t a, b;
    int stage;
};
static thread_local bool g_prof_on = false;
static thread_local std::vector<ProfRec> g_prof;        // recorded pairs
static thread_local std::vector<cudaEvent_t> g_pool;    // free events
static thread_local cudaEvent_t g_open[kNumStages] = {};

static cudaEvent_t pool_get() {
    if (!g_pool.empty()) { cudaEvent_t e = g_pool.back(); g_pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

void profile_mark(int stage, int begin, cudaStream_t s) {
    if (!g_prof_on) return;
    cudaEvent_t e = pool_get();
    cudaEventRecord(e, s);
    if (begin) { g_open[stage] = e; return; }
    g_prof.push_back(ProfRec{g_open[stage], e, stage});
    g_open[stage] = nullptr;
}

// extract.cu
size_t extract_workspace_bytes(int64_t R, int64_t G, int64_t B, int64_t max_group, bool singleton);
fcfs_status extract_clips_async(const int32_t *rects, int64_t R, const int64_t *clip_ptr, int64_t B, int32_t T,
                                int64_t max_clip_rects, int32_t *x, int32_t *y, int32_t *w, int64_t cap,
                                int64_t *corner_ptr, int64_t *area, int64_t *K_dev, int32_t *status_dev, void *ws,
                                size_t ws_bytes, cudaStream_t s);
fcfs_status extract(const int32_t *rects, int64_t R, const int64_t *group_ptr, int64_t G,
                    const int64_t *clip_ptr, int64_t B, int32_t T, int64_t max_group, int32_t *x,
                    int32_t *y, int32_t *w, int64_t cap, int64_t *corner_ptr, int64_t *area,
                    int64_t *K_host, void *ws, size_t ws_bytes, cudaStream_t s, int32_t y_lo = 0,
                    int32_t y_hi = 0x7fffffff, int64_t *K_dev = nullptr, int32_t *status_dev = nullptr);
size_t small_clip_smem_bytes(int32_t T, int64_t max_group);
bool small_clip_eligible(int64_t R, int64_t G, int32_t T, int64_t max_group, int32_t M, int32_t N, bool grouped);
fcfs_status launch_small_clip(const int32_t *rects, int64_t R, const int64_t *group_ptr, int64_t G, int32_t T,
                              int64_t max_group, const fcfs_window &win, int32_t out_f32, void *F, int64_t *K_dev,
                              int32_t *status_dev, cudaStream_t s);
size_t extract_polygons_workspace_bytes(int64_t V, int64_t B);
fcfs_status extract_polygons(const int32_t *vx, const int32_t *vy, int64_t V, const int64_t *poly_ptr, int64_t P,
                             const int64_t *clip_ptr, int64_t B, int32_t T, int32_t *x, int32_t *y, int32_t *w,
                             int64_t cap, int64_t *corner_ptr, int64_t *area, int64_t *K_host, void *ws,
                             size_t ws_bytes, cudaStream_t s);
// haar.cu
size_t haar_workspace_bytes(int64_t B, int32_t T);
fcfs_status haar_clips(const int32_t *x, const int32_t *y, const int32_t *w, const int64_t *corner_ptr, int64_t B,
                       int64_t K, const int64_t *area, int32_t T, double *out, void *ws, size_t ws_bytes,
                       cudaStream_t s);
// chop.cu
size_t chop_workspace_bytes(int64_t R, int64_t cap, int64_t tiles);
fcfs_status chop_rects(const int32_t *rects, int64_t R, int32_t T, int32_t tiles_x, int32_t tiles_y,
                       int32_t *out, int64_t cap, int64_t *tile_ptr, int64_t *n_host, void *ws, size_t ws_bytes,
                       cudaStream_t s);
// contract_tf32.cu
fcfs_status tf32_supported(const GemmPlan &plan, int32_t T);
fcfs_status launch_gemm_tf32(const CornerSrc &src, const GemmPlan &plan, int32_t T, double *P_ws,
                             const EpiArgs *ea, void *F, bool f16, cudaStream_t s);
bool tf32_can_fuse(const GemmPlan &plan, const EpiArgs &ea);

// lattice.cu
bool lattice_eligible(int32_t T, const EpiArgs &ea);
size_t lattice_ws_bytes(int64_t B, int32_t T);
fcfs_status launch_lattice_prepare(const int64_t *corner_ptr, int64_t B, const int32_t *y, int64_t K, int32_t T,
                                   int32_t M, int32_t N, void *ws, int32_t *unsorted_dev, bool check, cudaStream_t s);
fcfs_status launch_lattice(const int64_t *corner_ptr, int64_t B, const int32_t *x, const int32_t *y, const int32_t *w,
                           int32_t T, const EpiArgs &ea, void *F, void *ws, cudaStream_t s);

// sm_100 check, cached per device (atomics: several host threads call this concurrently)
static fcfs_status device_ok() {
    static std::atomic<int> cached[64];   // 0 = unknown, 1 = sm_100, 2 = other
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_status(e, "device query");
    int c = (dev >= 0 && dev < 64) ? cached[dev].load(std::memory_order_relaxed) : 0;
    int major = 0, minor = 0;
    if (c == 0) {
        e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
        if (e != cudaSuccess) return cuda_status(e, "device query");
        c = (major == 10 && minor == 0) ? 1 : 2;
        if (dev >= 0 && dev < 64) cached[dev].store(c, std::memory_order_relaxed);
    }
    if (c != 1) {
        set_error("device %d is not sm_100; libfcfs.so is built for sm_100a only", dev);
        return FCFS_E_UNSUPPORTED;
    }
    return FCFS_OK;
}

static bool valid_T(int32_t T) { return T >= 1 && T <= (1 << 20); }

static fcfs_status check_window(const fcfs_window *win) {
    if (!win) { set_error("win is NULL"); return FCFS_E_INVALID; }
    if (win->M < 0 || win->N < 0 || win->M > 65535 || win->N > 65535) {
        set_error("window M=%d N=%d out of range", win->M, win->N);
        return FCFS_E_INVALID;
    }
    if (win->layout != FCFS_LAYOUT_DENSE && win->layout != FCFS_LAYOUT_PUPIL) {
        set_error("bad layout %d", win->layout);
        return FCFS_E_INVALID;
    }
    if (win->layout == FCFS_LAYOUT_PUPIL && !(win->pupil_r2 >= 0.0)) {
        set_error("PUPIL layout needs pupil_r2 >= 0");
        return FCFS_E_INVALID;
    }
    return FCFS_OK;
}

static int64_t pupil_count(int32_t M, int32_t N, double r2, int32_t *mo, int32_t *no, int64_t cap) {
    int64_t c = 0;
    for (int64_t m = -M; m <= M; ++m)
        for (int64_t n = -N; n <= N; ++n) {
            if ((double)m * (double)m + (double)n * (double)n > r2) continue;
            if (mo && no && c < cap) { mo[c] = (int32_t)m; no[c] = (int32_t)n; }
            ++c;
        }
    return c;
}

static SidePlan side_for_rows(int32_t m_lo, int32_t m_hi) {
    SidePlan sp;
    sp.axis = (m_lo <= 0 && 0 <= m_hi) ? 1 : 0;
    int32_t a, b;
    if (m_lo >= 1) { a = m_lo; b = m_hi; }
    else if (m_hi <= -1) { a = -m_hi; b = -m_lo; }
    else { a = 1; b = (-m_lo > m_hi) ? -m_lo : m_hi; }
    sp.f0 = a;
    sp.nf = b >= a ? b - a + 1 : 0;
    if (sp.nf == 0) sp.f0 = 1;
    sp.rows = 2 * sp.nf + sp.axis;
    return sp;
}

static GemmPlan make_plan(int32_t M, int32_t N, int32_t m_lo, int32_t m_hi, int64_t B, int64_t K, bool batched) {
    GemmPlan p;
    p.X = side_for_rows(m_lo, m_hi);
    p.Y = side_for_rows(-N, N);
    p.tiles_x = (p.X.rows + kTile - 1) / kTile;
    p.tiles_y = (p.Y.rows + kTile - 1) / kTile;
    if (p.tiles_x < 1) p.tiles_x = 1;
    if (p.tiles_y < 1) p.tiles_y = 1;
    int64_t tiles = (int64_t)p.tiles_x * p.tiles_y;
    int64_t splits = 1;
    if (!batched) {
        const int64_t target = 2 * 2 * 148;   // two waves of 2 CTAs/SM
        splits = (target + tiles - 1) / tiles;
        int64_t kcap = (K + 511) / 512;
        if (splits > kcap) splits = kcap;
        if (splits < 1) splits = 1;
        if (splits > 4096) splits = 4096;
    }
    p.splits = (int32_t)splits;
    p.B = B;
    p.items = B * tiles * splits;
    p.phys = 0;
#ifdef FCFS_ABLATE
    const char *dbg = getenv("FCFS_DEBUG");   // ablation build only (libfcfs_ablate.so), never shipped
    p.dbg = dbg ? atoi(dbg) : 0;
#else
    p.dbg = 0;
#endif
    return p;
}

struct CoeffWs {
    double *P;
    int64_t *area;
    BucketWs bk;
    double *G;   // single clip: x-side bucket sums of one chunk, [tiles_x][cb][64 doubles or 128 tf32 rows]
    double *H;   // single clip, split precisions: y-side row twiddles of the chunk, [tiles_y][cb][128 rows]
    void *fft;   // single FP64 clip: the lattice-FFT route's workspace (overlaps bk / G / H: one or the other)
    size_t fft_bytes;
    EdgeWs edges;   // batched split-TF32: the edge form of the corner lists (edges.cu)
    void *lat;      // batched split-TF32, lattice-row form: B chunk table + chunk pointers (lattice.cu)
    int32_t *flag;  // device flag (unsorted corner list)
};

static const fcfs_options kDefaultOptions = {FCFS_ROUTE_AUTO, FCFS_FORM_AUTO, 0, {0, 0, 0, 0, 0}};

static fcfs_status check_options(const fcfs_options *&opt) {
    if (!opt) { opt = &kDefaultOptions; return FCFS_OK; }
    if (opt->route < FCFS_ROUTE_AUTO || opt->route > FCFS_ROUTE_FFT || opt->form < FCFS_FORM_AUTO ||
        opt->form > FCFS_FORM_LATTICE || opt->sorted_y < 0 || opt->sorted_y > 1) {
        set_error("bad options: route %d form %d sorted_y %d", opt->route, opt->form, opt->sorted_y);
        return FCFS_E_INVALID;
    }
    for (int i = 0; i < 5; ++i)
        if (opt->reserved[i]) { set_error("fcfs_options.reserved[%d] != 0", i); return FCFS_E_INVALID; }
    return FCFS_OK;
}

// the batched split-TF32 contraction form (assuming y-sorted lists): the lattice-row form where it applies
// (and, under AUTO, where the clips are dense enough in corners for its T+1 rows), else the edge form
// (the K/2-term form) unless the caller asks for corners
static int32_t batched_form(fcfs_precision prec, const fcfs_options *opt, int64_t B, int64_t K_total, int32_t T,
                            const fcfs_window *win) {
    if (prec == FCFS_FP64) return 0;
    if (prec == FCFS_F16X3) return FCFS_FORM_CORNER;   // split-FP16 keeps the corner form
    if (opt->form == FCFS_FORM_CORNER) return FCFS_FORM_CORNER;
    if (opt->form == FCFS_FORM_EDGE) return FCFS_FORM_EDGE;
    EpiArgs ea{};
    ea.M = win->M; ea.N = win->N; ea.m_lo = -win->M; ea.m_hi = win->M; ea.out_f32 = 1;
    if (lattice_eligible(T, ea) &&
        (opt->form == FCFS_FORM_LATTICE || (B > 0 && 4 * K_total >= B * ((int64_t)T + 1))))
        return FCFS_FORM_LATTICE;
    return FCFS_FORM_EDGE;
}

// P_ws is not needed when the tcgen05 kernel fuses the epilogue (batched: whole clip = one 64x64
// tile).  A single clip always takes the chunked row-bucket path, which writes P.
static bool fusable(const GemmPlan &p, fcfs_precision prec, int32_t M, int32_t m_lo, int32_t m_hi, bool single = false) {
    if (single) return false;   // one clip: the chunked row-bucket path, which writes P
    EpiArgs ea{};
    ea.M = M; ea.m_lo = m_lo; ea.m_hi = m_hi;
    return (prec == FCFS_TF32X3 || prec == FCFS_F16X3) && tf32_can_fuse(p, ea);
}

// number of row buckets of a single range (the chunk loop of the single-clip paths runs on the
// host): one stream synchronisation
static fcfs_status bucket_count_host(const BucketWs &bk, int64_t &nb, cudaStream_t s) {
    int64_t h[2] = {0, 0};
    FCFS_TRY_CUDA(cudaMemcpyAsync(h, bk.clip_bptr, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    FCFS_TRY_CUDA(cudaStreamSynchronize(s));
    nb = h[1] - h[0];
    return FCFS_OK;
}

// the row buckets (buckets.cu) feed the FP64 contraction; the tcgen05 kernels walk corners
static void carve_coeff(Carver &cv, const GemmPlan &p, CoeffWs &w, bool need_P, int64_t K, int64_t B,
                        fcfs_precision prec, bool single = false, const FftPlan *fp = nullptr, int32_t lat_T = 0) {
    w.P = cv.take<double>(need_P ? (size_t)p.items * kTile * kTile : 1);
    w.area = cv.take<int64_t>(1);
    w.bk = BucketWs{};
    w.G = nullptr;
    w.H = nullptr;
    w.fft = nullptr;
    w.fft_bytes = 0;
    const size_t mark = cv.off;
    if (fp) {   // the FFT route's region, overlapping the row-bucket path's (never both in one call)
        w.fft_bytes = fft_route_ws_bytes(*fp);
        w.fft = cv.take<char>(w.fft_bytes);
    }
    const size_t fft_end = cv.off;
    cv.off = mark;
    const bool bucketed = prec == FCFS_FP64 || single;
    if (bucketed) carve_buckets(cv, K, B, w.bk);
    w.edges = EdgeWs{};
    w.lat = nullptr;
    w.flag = nullptr;
    if (!single && prec == FCFS_TF32X3) {
        carve_edges(cv, K, B, w.edges);
        w.flag = cv.take<int32_t>(64);
        if (lat_T > 0) w.lat = cv.take<char>(lattice_ws_bytes(B, lat_T));
    }
    if (bucketed && single) {
        // x-side bucket sums of one chunk: 64 doubles (FP64) or 128 tf32 rows x 4 B (split-TF32) per bucket
        const int64_t cb = chunk_buckets(K, p.tiles_x, p.tiles_y);
        w.G = cv.take<double>((size_t)p.tiles_x * cb * kTile);
        // the y-side row twiddles of the chunk as well (64 doubles or 128 tf32 rows x 4 B per bucket)
        w.H = cv.take<double>((size_t)p.tiles_y * cb * kTile);
    }
    if (cv.off < fft_end) cv.off = fft_end;
}

static fcfs_status resolve_rows(const fcfs_window *win, const fcfs_shard *shard, int32_t &m_lo, int32_t &m_hi) {
    m_lo = -win->M;
    m_hi = win->M;
    if (shard && shard->kind == FCFS_SHARD_ROWS) {
        if (win->layout != FCFS_LAYOUT_DENSE) { set_error("ROWS shard needs the DENSE layout"); return FCFS_E_INVALID; }
        if (shard->m_lo < -win->M || shard->m_hi > win->M || shard->m_lo > shard->m_hi) {
            set_error("ROWS shard [%d, %d] outside [-M, M]", shard->m_lo, shard->m_hi);
            return FCFS_E_INVALID;
        }
        m_lo = shard->m_lo;
        m_hi = shard->m_hi;
    } else if (shard && shard->kind != FCFS_SHARD_NONE && shard->kind != FCFS_SHARD_VERTEX_BLOCK) {
        set_error("bad shard kind %d", shard->kind);
        return FCFS_E_INVALID;
    }
    return FCFS_OK;
}

// a2 + a3 (+ a4/a5 when the tcgen05 kernel can fuse its epilogue); *fused tells the caller
// whether the stand-alone epilogue kernel is still needed.
static fcfs_status run_gemm(const CornerSrc &src, const GemmPlan &plan, int32_t T, fcfs_precision prec,
                            double *P, const EpiArgs &ea, void *F, cudaStream_t s, bool *fused) {
    *fused = false;
    if (prec == FCFS_FP64) return launch_gemm_fp64(src, plan, T, P, s);
    if (prec == FCFS_TF32X3 || prec == FCFS_F16X3) {
        fcfs_status st = tf32_supported(plan, T);
        if (st != FCFS_OK) return st;
        *fused = tf32_can_fuse(plan, ea);
        // P in phys layout 1 when not fused
        return launch_gemm_tf32(src, plan, T, P, &ea, F, prec == FCFS_F16X3, s);
    }
    set_error("bad precision %d", prec);
    return FCFS_E_INVALID;
}

}  // namespace fcfs

using namespace fcfs;

extern "C" {

const char *fcfs_status_string(fcfs_status s) {
    switch (s) {
        case FCFS_OK: return "FCFS_OK";
        case FCFS_E_INVALID: return "FCFS_E_INVALID";
        case FCFS_E_RANGE: return "FCFS_E_RANGE";
        case FCFS_E_CAPACITY: return "FCFS_E_CAPACITY";
        case FCFS_E_WORKSPACE: return "FCFS_E_WORKSPACE";
        case FCFS_E_UNSUPPORTED: return "FCFS_E_UNSUPPORTED";
        case FCFS_E_CUDA: return "FCFS_E_CUDA";
        default: return "FCFS_E_UNKNOWN";
    }
}

const char *fcfs_last_error(void) { return g_err; }

int32_t fcfs_kernel_launches(void) { return g_launches; }

fcfs_status fcfs_device_check(void) { return device_ok(); }

fcfs_status fcfs_profile_enable(int32_t on) {
    g_prof_on = on != 0;
    return FCFS_OK;
}

fcfs_status fcfs_profile_read(double *ms_host, int64_t *count_host, int32_t n_stages) {
    if (n_stages < 0 || n_stages > kNumStages || (n_stages > 0 && (!ms_host || !count_host))) {
        set_error("fcfs_profile_read: bad arguments");
        return FCFS_E_INVALID;
    }
    for (int i = 0; i < n_stages; ++i) { ms_host[i] = 0.0; count_host[i] = 0; }
    fcfs_status st = FCFS_OK;
    for (auto &r : g_prof) {
        float ms = 0.f;
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
        if (e != cudaSuccess) st = cuda_status(e, "fcfs_profile_read");
        if (r.stage < n_stages) { ms_host[r.stage] += ms; count_host[r.stage] += 1; }
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_prof.clear();
    return st;
}

int64_t fcfs_window_size(const fcfs_window *win) {
    if (check_window(win) != FCFS_OK) return -1;
    if (win->layout == FCFS_LAYOUT_PUPIL) return pupil_count(win->M, win->N, win->pupil_r2, nullptr, nullptr, 0);
    return (int64_t)(2 * win->M + 1) * (2 * win->N + 1);
}

int64_t fcfs_pupil_indices(int32_t M, int32_t N, double r2, int32_t *m_out_host, int32_t *n_out_host, int64_t cap) {
    if (M < 0 || N < 0) return -1;
    return pupil_count(M, N, r2, m_out_host, n_out_host, cap);
}

size_t fcfs_vertices_workspace_bytes(int64_t R, int64_t G, int64_t B, int64_t max_group) {
    // the singleton path is chosen by group_ptr == NULL at call time; size for the larger
    size_t a = extract_workspace_bytes(R, G, B, max_group, true);
    size_t b = extract_workspace_bytes(R, G, B, max_group, false);
    return a > b ? a : b;
}

}  // extern "C"

// a1 for rects; eo != NULL also writes the edge pairing of the output corners (k_edges after the
// extraction; pairing inside the per-clip bucket kernel measured slower: DESIGN.md §7)
static fcfs_status vertices_impl(const int32_t *rects, int64_t R, const int64_t *group_ptr, int64_t G,
                                 const int64_t *clip_ptr, int64_t B, int32_t T, int64_t max_group, int32_t *x,
                                 int32_t *y, int32_t *w, int64_t cap, int64_t *corner_ptr, int64_t *area,
                                 int64_t *K_total_host, void *ws, size_t ws_bytes, void *stream, const EdgeWs *eo,
                                 int32_t y_lo = 0, int32_t y_hi = 0x7fffffff, int64_t *K_dev = nullptr,
                                 int32_t *status_dev = nullptr) {
    if (!valid_T(T)) { set_error("T=%d outside [1, 2^20]", T); return FCFS_E_INVALID; }
    if (R < 0 || B < 1 || B >= (int64_t(1) << 22) || (R > 0 && (!rects || ((uintptr_t)rects & 15u))) || !corner_ptr || !area ||
        (!K_total_host && !(K_dev && status_dev))) {
        set_error("fcfs_vertices_from_rects: invalid sizes or null pointers");
        return FCFS_E_INVALID;
    }
    if (cap > 0 && (!x || !y || !w)) { set_error("null corner output with cap > 0"); return FCFS_E_INVALID; }
    if (group_ptr == nullptr && G != R) { set_error("group_ptr NULL requires G == R"); return FCFS_E_INVALID; }
    if (clip_ptr == nullptr && B != 1) { set_error("clip_ptr NULL requires B == 1"); return FCFS_E_INVALID; }
    if (ws == nullptr || ((uintptr_t)ws & 255)) { set_error("ws NULL or not 256-byte aligned"); return FCFS_E_WORKSPACE; }
    fcfs_status st = device_ok();
    if (st != FCFS_OK) return st;
    StageScope scope(kStageExtract, (cudaStream_t)stream);
    st = extract(rects, R, group_ptr, G, clip_ptr, B, T, max_group, x, y, w, cap, corner_ptr, area, K_total_host,
                 ws, ws_bytes, (cudaStream_t)stream, y_lo, y_hi, K_dev, status_dev);
    if (K_dev) return st;   // sync-free: no host K, no edge pass
    if (st != FCFS_OK || !eo) return st;
    if (*K_total_host > 0) return run_edges(x, y, w, corner_ptr, B, *eo, (cudaStream_t)stream);
    FCFS_TRY_CUDA(cudaMemsetAsync(eo->cnt, 0, sizeof(int32_t) * (size_t)B, (cudaStream_t)stream));
    return FCFS_OK;
}

extern "C" {

fcfs_status fcfs_vertices_from_rects(const int32_t *rects, int64_t R, const int64_t *group_ptr, int64_t G,
                                     const int64_t *clip_ptr, int64_t B, int32_t T, int64_t max_group,
                                     int32_t *x, int32_t *y, int32_t *w, int64_t cap, int64_t *corner_ptr,
                                     int64_t *area, int64_t *K_total_host, void *ws, size_t ws_bytes,
                                     void *stream) {
    return vertices_impl(rects, R, group_ptr, G, clip_ptr, B, T, max_group, x, y, w, cap, corner_ptr, area,
                         K_total_host, ws, ws_bytes, stream, nullptr);
}

fcfs_status fcfs_vertices_from_rects_edges(const int32_t *rects, int64_t R, const int64_t *group_ptr, int64_t G,
                                           const int64_t *clip_ptr, int64_t B, int32_t T, int64_t max_group,
                                           int32_t *x, int32_t *y, int32_t *w, int64_t cap, int64_t *corner_ptr,
                                           int64_t *area, int64_t *K_total_host, int32_t *xa, int32_t *xb,
                                           int32_t *ye, int32_t *c, int32_t *ecnt, void *ws, size_t ws_bytes,
                                           void *stream) {
    if ((cap > 0 && (!xa || !xb || !ye || !c)) || !ecnt) {
        set_error("fcfs_vertices_from_rects_edges: null edge output");
        return FCFS_E_INVALID;
    }
    EdgeWs e;
    e.xa = xa; e.xb = xb; e.y = ye; e.c = c; e.cnt = ecnt;
    return vertices_impl(rects, R, group_ptr, G, clip_ptr, B, T, max_group, x, y, w, cap, corner_ptr, area,
                         K_total_host, ws, ws_bytes, stream, &e);
}

fcfs_status fcfs_vertices_from_rects_async(const int32_t *rects, int64_t R, const int64_t *group_ptr, int64_t G,
                                           const int64_t *clip_ptr, int64_t B, int32_t T, int64_t max_group, int32_t *x,
                                           int32_t *y, int32_t *w, int64_t cap, int64_t *corner_ptr, int64_t *area,
                                           int64_t *K_dev, int32_t *status_dev, void *ws, size_t ws_bytes, void *stream) {
    if (!K_dev || !status_dev) { set_error("fcfs_vertices_from_rects_async: K_dev / status_dev NULL"); return FCFS_E_INVALID; }
    return vertices_impl(rects, R, group_ptr, G, clip_ptr, B, T, max_group, x, y, w, cap, corner_ptr, area, nullptr, ws,
                         ws_bytes, stream, nullptr, 0, 0x7fffffff, K_dev, status_dev);
}

fcfs_status fcfs_vertices_from_clips_async(const int32_t *rects, int64_t R, const int64_t *clip_ptr, int64_t B,
                                           int32_t T, int64_t max_clip_rects, int32_t *x, int32_t *y, int32_t *w,
                                           int64_t cap, int64_t *corner_ptr, int64_t *area, int64_t *K_dev,
                                           int32_t *status_dev, void *ws, size_t ws_bytes, void *stream) {
    if (!valid_T(T)) { set_error("T=%d outside [1, 2^20]", T); return FCFS_E_INVALID; }
    if (R < 0 || B < 1 || B >= (int64_t(1) << 22) || !clip_ptr || (R > 0 && (!rects || ((uintptr_t)rects & 15u))) ||
        !corner_ptr || !area || !K_dev || !status_dev || (cap > 0 && (!x || !y || !w))) {
        set_error("fcfs_vertices_from_clips_async: invalid sizes or null pointers");
        return FCFS_E_INVALID;
    }
    if (ws == nullptr || ((uintptr_t)ws & 255)) { set_error("ws NULL or not 256-byte aligned"); return FCFS_E_WORKSPACE; }
    fcfs_status st = device_ok();
    if (st != FCFS_OK) return st;
    StageScope scope(kStageExtract, (cudaStream_t)stream);
    return extract_clips_async(rects, R, clip_ptr, B, T, max_clip_rects, x, y, w, cap, corner_ptr, area, K_dev,
                               status_dev, ws, ws_bytes, (cudaStream_t)stream);
}

fcfs_status fcfs_vertices_from_rects_band(const int32_t *rects, int64_t R, const int64_t *group_ptr, int64_t G,
                                          int32_t T, int64_t max_group, int32_t y_lo, int32_t y_hi, int32_t *x,
                                          int32_t *y, int32_t *w, int64_t cap, int64_t *corner_ptr, int64_t *area,
                                          int64_t *K_host, void *ws, size_t ws_bytes, void *stream) {
    if (y_lo < 0 || y_hi < y_lo) {
        set_error("fcfs_vertices_from_rects_band: band [%d, %d) invalid", y_lo, y_hi);
        return FCFS_E_INVALID;
    }
    return vertices_impl(rects, R, group_ptr, G, nullptr, 1, T, max_group, x, y, w, cap, corner_ptr, area, K_host, ws,
                         ws_bytes, stream, nullptr, y_lo, y_hi);
}

size_t fcfs_haar_workspace_bytes(int64_t B, int32_t T) { return haar_workspace_bytes(B, T); }

fcfs_status fcfs_haar(const int64_t *corner_ptr, int64_t B, int64_t K, const int32_t *x, const int32_t *y,
                      const int32_t *w, const int64_t *area, int32_t T, double *out, void *ws, size_t ws_bytes,
                      void *stream) {
    if (T < 2 || T > 4096 || (T & (T - 1)) != 0) { set_error("fcfs_haar: T=%d not a power of two in [2, 4096]", T); return FCFS_E_INVALID; }
    if (B < 1 || K < 0 || (K > 0 && (!x || !y || !w)) || !area || !out || (corner_ptr == nullptr && B != 1) ||
        K >= (int64_t(1) << 31)) {
        set_error("fcfs_haar: invalid sizes or null pointers");
        return FCFS_E_INVALID;
    }
    if (ws == nullptr || ((uintptr_t)ws & 255)) { set_error("ws NULL or not 256-byte aligned"); return FCFS_E_WORKSPACE; }
    fcfs_status st = device_ok();
    if (st != FCFS_OK) return st;
    StageScope scope(kStageContract, (cudaStream_t)stream);
    return haar_clips(x, y, w, corner_ptr, B, K, area, T, out, ws, ws_bytes, (cudaStream_t)stream);
}

size_t fcfs_chop_workspace_bytes(int64_t R, int64_t cap, int32_t tiles_x, int32_t tiles_y) {
    if (R < 0 || cap < 0 || tiles_x < 1 || tiles_y < 1) return 0;
    return chop_workspace_bytes(R, cap, (int64_t)tiles_x * tiles_y);
}

fcfs_status fcfs_chop_rects(const int32_t *rects, int64_t R, int32_t T, int32_t tiles_x, int32_t tiles_y,
                            int32_t *out_rects, int64_t cap, int64_t *tile_ptr, int64_t *n_host, void *ws,
                            size_t ws_bytes, void *stream) {
    if (!valid_T(T)) { set_error("T=%d outside [1, 2^20]", T); return FCFS_E_INVALID; }
    if (R < 0 || (R > 0 && (!rects || ((uintptr_t)rects & 15u))) || tiles_x < 1 || tiles_y < 1 || !tile_ptr || !n_host || cap < 0 ||
        (cap > 0 && !out_rects) || (int64_t)tiles_x * tiles_y >= (int64_t(1) << 31) ||
        (int64_t)tiles_x * T >= (int64_t(1) << 31) || (int64_t)tiles_y * T >= (int64_t(1) << 31) ||
        cap >= (int64_t(1) << 31)) {
        set_error("fcfs_chop_rects: invalid sizes or null pointers");
        return FCFS_E_INVALID;
    }
    if (ws == nullptr || ((uintptr_t)ws & 255)) { set_error("ws NULL or not 256-byte aligned"); return FCFS_E_WORKSPACE; }
    fcfs_status st = device_ok();
    if (st != FCFS_OK) return st;
    StageScope scope(kStageExtract, (cudaStream_t)stream);
    return chop_rects(rects, R, T, tiles_x, tiles_y, out_rects, cap, tile_ptr, n_host, ws, ws_bytes,
                      (cudaStream_t)stream);
}

size_t fcfs_polygons_workspace_bytes(int64_t V, int64_t P, int64_t B) {
    (void)P;
    return extract_polygons_workspace_bytes(V, B);
}

fcfs_status fcfs_vertices_from_polygons(const int32_t *vx, const int32_t *vy, int64_t V, const int64_t *poly_ptr,
                                        int64_t P, const int64_t *clip_ptr, int64_t B, int32_t T, int32_t *x,
                                        int32_t *y, int32_t *w, int64_t cap, int64_t *corner_ptr, int64_t *area,
                                        int64_t *K_total_host, void *ws, size_t ws_bytes, void *stream) {
    if (!valid_T(T)) { set_error("T=%d outside [1, 2^20]", T); return FCFS_E_INVALID; }
    if (V < 0 || P < 0 || B < 1 || B >= (int64_t(1) << 22) || (V > 0 && (!vx || !vy)) || !poly_ptr || !corner_ptr ||
        !area || !K_total_host) {
        set_error("fcfs_vertices_from_polygons: invalid sizes or null pointers");
        return FCFS_E_INVALID;
    }
    if (cap > 0 && (!x || !y || !w)) { set_error("null corner output with cap > 0"); return FCFS_E_INVALID; }
    if (clip_ptr == nullptr && B != 1) { set_error("clip_ptr NULL requires B == 1"); return FCFS_E_INVALID; }
    if (ws == nullptr || ((uintptr_t)ws & 255)) { set_error("ws NULL or not 256-byte aligned"); return FCFS_E_WORKSPACE; }
    fcfs_status st = device_ok();
    if (st != FCFS_OK) return st;
    StageScope scope(kStageExtract, (cudaStream_t)stream);
    return extract_polygons(vx, vy, V, poly_ptr, P, clip_ptr, B, T, x, y, w, cap, corner_ptr, area, K_total_host,
                            ws, ws_bytes, (cudaStream_t)stream);
}

size_t fcfs_coeffs_workspace_bytes(int64_t K, int32_t T, const fcfs_window *win, fcfs_precision prec,
                                   const fcfs_shard *shard, const fcfs_options *opt) {
    if (check_window(win) != FCFS_OK || check_options(opt) != FCFS_OK) return 0;
    int32_t m_lo, m_hi;
    if (resolve_rows(win, shard, m_lo, m_hi) != FCFS_OK) return 0;
    int64_t k = K;
    if (shard && shard->kind == FCFS_SHARD_VERTEX_BLOCK) k = shard->k_hi - shard->k_lo;
    GemmPlan p = make_plan(win->M, win->N, m_lo, m_hi, 1, k, false);
    FftPlan fp;
    const bool fft = valid_T(T) && (prec == FCFS_FP64 || prec == FCFS_TF32X3 || prec == FCFS_F16X3) &&
                     fft_route_plan(T, win->M, win->N, m_lo, m_hi, k, prec != FCFS_FP64, fp, opt->route);
    Carver cv(nullptr, 0);
    CoeffWs w;
    carve_coeff(cv, p, w, !fusable(p, prec, win->M, m_lo, m_hi, true), k, 1, prec, true, fft ? &fp : nullptr);
    return cv.used();
}

int32_t fcfs_coeffs_route(int64_t K, int32_t T, const fcfs_window *win, fcfs_precision prec,
                          const fcfs_shard *shard, const fcfs_options *opt) {
    if (!valid_T(T) || check_window(win) != FCFS_OK || check_options(opt) != FCFS_OK) return 0;
    if (prec != FCFS_FP64 && prec != FCFS_TF32X3 && prec != FCFS_F16X3) return 0;
    int32_t m_lo, m_hi;
    if (resolve_rows(win, shard, m_lo, m_hi) != FCFS_OK) return 0;
    int64_t k = K;
    if (shard && shard->kind == FCFS_SHARD_VERTEX_BLOCK) k = shard->k_hi - shard->k_lo;
    FftPlan fp;
    return fft_route_plan(T, win->M, win->N, m_lo, m_hi, k, prec != FCFS_FP64, fp, opt->route) ? 1 : 0;
}

int32_t fcfs_small_clip_supported(int64_t R, int64_t G, int32_t T, int64_t max_group, const fcfs_window *win) {
    if (!valid_T(T) || R < 0 || !win || check_window(win) != FCFS_OK) return 0;
    return small_clip_eligible(R, G, T, max_group, win->M, win->N, G != R || max_group > 1) ? 1 : 0;
}

fcfs_status fcfs_small_clip(const int32_t *rects, int64_t R, const int64_t *group_ptr, int64_t G, int32_t T,
                            int64_t max_group, const fcfs_window *win, fcfs_precision prec, void *F, int64_t *K_dev,
                            int32_t *status_dev, void *stream) {
    if (!valid_T(T)) { set_error("T=%d outside [1, 2^20]", T); return FCFS_E_INVALID; }
    fcfs_status st = check_window(win);
    if (st != FCFS_OK) return st;
    if (R < 0 || (R > 0 && (!rects || ((uintptr_t)rects & 15u))) || !F || !status_dev || (group_ptr == nullptr && G != R) || G < 0) {
        set_error("fcfs_small_clip: invalid sizes or null pointers");
        return FCFS_E_INVALID;
    }
    if (prec != FCFS_FP64 && prec != FCFS_TF32X3 && prec != FCFS_F16X3) { set_error("bad precision %d", prec); return FCFS_E_INVALID; }
    const int64_t mg = group_ptr == nullptr ? 1 : max_group;
    if (!small_clip_eligible(R, G, T, mg, win->M, win->N, group_ptr != nullptr)) {
        set_error("fcfs_small_clip: outside the small-clip limits (T <= 8192, M <= 63, N <= 4096, groups <= 100 rects, "
                  "<= 2048 raw corners)");
        return FCFS_E_UNSUPPORTED;
    }
    st = device_ok();
    if (st != FCFS_OK) return st;
    StageScope scope(kStageContract, (cudaStream_t)stream);
    return launch_small_clip(rects, R, group_ptr, G, T, mg, *win, prec != FCFS_FP64, F, K_dev, status_dev,
                             (cudaStream_t)stream);
}

static fcfs_status coeffs_one(const int32_t *x, const int32_t *y, const int32_t *w, int64_t K, int64_t area, int32_t T,
                              const fcfs_window *win, fcfs_precision prec, const fcfs_shard *shard,
                              const fcfs_options *opt, void *F, void *ws, size_t ws_bytes, void *stream,
                              void *const *peers, int32_t n_peers) {
    if (!valid_T(T)) { set_error("T=%d outside [1, 2^20]", T); return FCFS_E_INVALID; }
    fcfs_status st = check_window(win);
    if (st == FCFS_OK) st = check_options(opt);
    if (st != FCFS_OK) return st;
    if (K < 0 || (K > 0 && (!x || !y || !w)) || !F) { set_error("fcfs_coeffs: null pointer or K < 0"); return FCFS_E_INVALID; }
    if (prec != FCFS_FP64 && prec != FCFS_TF32X3 && prec != FCFS_F16X3) {
        set_error("bad precision %d", prec);
        return FCFS_E_INVALID;
    }
    int32_t m_lo, m_hi;
    st = resolve_rows(win, shard, m_lo, m_hi);
    if (st != FCFS_OK) return st;
    CornerSrc src{};
    src.x = x; src.y = y; src.w = w; src.corner_ptr = nullptr; src.k_lo = 0; src.k_hi = K;
    bool vblock = shard && shard->kind == FCFS_SHARD_VERTEX_BLOCK;
    if (vblock) {
        if (shard->k_lo < 0 || shard->k_hi > K || shard->k_lo > shard->k_hi) {
            set_error("VERTEX_BLOCK [%lld, %lld) outside [0, K)", (long long)shard->k_lo, (long long)shard->k_hi);
            return FCFS_E_INVALID;
        }
        src.k_lo = shard->k_lo; src.k_hi = shard->k_hi;
    }
    if (ws == nullptr || ((uintptr_t)ws & 255)) { set_error("ws NULL or not 256-byte aligned"); return FCFS_E_WORKSPACE; }
    st = device_ok();
    if (st != FCFS_OK) return st;
    GemmPlan plan = make_plan(win->M, win->N, m_lo, m_hi, 1, src.k_hi - src.k_lo, false);
    plan.phys = prec == FCFS_FP64 ? 0 : 1;
    FftPlan fp;
    const bool fft = fft_route_plan(T, win->M, win->N, m_lo, m_hi, src.k_hi - src.k_lo, prec != FCFS_FP64, fp,
                                    opt->route);
    Carver cv(ws, ws_bytes);
    CoeffWs W;
    carve_coeff(cv, plan, W, !fusable(plan, prec, win->M, m_lo, m_hi, true), src.k_hi - src.k_lo, 1, prec, true,
                fft ? &fp : nullptr);
    if (!cv.fits()) { set_error("fcfs_coeffs: workspace %zu < %zu", ws_bytes, cv.used()); return FCFS_E_WORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    EpiArgs ea;
    ea.M = win->M; ea.N = win->N; ea.layout = win->layout; ea.r2 = win->pupil_r2;
    ea.m_lo = m_lo; ea.m_hi = m_hi; ea.T = T; ea.area_dev = nullptr; ea.area_host = area;
    ea.out_f32 = prec == FCFS_FP64 ? 0 : 1;
    ea.out_per_clip = 0;
    ea.peer_n = n_peers;
    for (int32_t i = 0; i < n_peers; ++i) ea.peer[i] = peers[i];
    if (vblock) {
        st = launch_block_area(src, W.area, s);
        if (st != FCFS_OK) return st;
        ea.area_dev = W.area;
    }
    src.bptr = W.bk.bptr; src.by = W.bk.by; src.clip_bptr = W.bk.clip_bptr; src.kend = K;
    if (fft) {
        // the lattice-FFT route (y-sorted corner lists; otherwise the row-bucket GEMM below)
        StageScope scope(kStageContract, s);
        bool sorted = false;
        st = fft_route_prepare(y, src.k_lo, src.k_hi - src.k_lo, fp, W.fft, W.fft_bytes, sorted, s);
        if (st != FCFS_OK) return st;
        if (sorted) return fft_route_run(x, w, src.k_lo, fp, W.fft, W.fft_bytes, ea, F, s);
    }
    bool fused = false;
    {
        StageScope scope(kStageContract, s);
        if (prec == FCFS_FP64) {
            // one clip: x-side bucket sums once per chunk, then the DMMA GEMM over them
            st = run_buckets(y, nullptr, 1, src.k_lo, src.k_hi, kRowBucketCapFp64, W.bk, s);
            int64_t nb = 0;
            if (st == FCFS_OK) st = bucket_count_host(W.bk, nb, s);
            if (st == FCFS_OK) st = launch_gemm_fp64_chunked(src, plan, T, nb, W.G, W.H, W.P, s);
        } else if (prec == FCFS_TF32X3 || prec == FCFS_F16X3) {
            // the same chunked row-bucket scheme on the tcgen05 tensor cores
            st = tf32_supported(plan, T);
            if (st == FCFS_OK) st = run_buckets(y, nullptr, 1, src.k_lo, src.k_hi, kRowBucketCapFp64, W.bk, s);
            int64_t nb = 0;
            if (st == FCFS_OK) st = bucket_count_host(W.bk, nb, s);
            if (st == FCFS_OK)
                st = launch_gemm_tf32_chunked(src, plan, T, nb, (uint8_t *)W.G, (uint8_t *)W.H, W.P, prec == FCFS_F16X3,
                                              s);
        } else {
            st = run_gemm(src, plan, T, prec, W.P, ea, F, s, &fused);
        }
    }
    if (st != FCFS_OK || fused) return st;
    StageScope scope(kStageEpilogue, s);
    return launch_epilogue(plan, W.P, ea, F, s);
}

fcfs_status fcfs_coeffs(const int32_t *x, const int32_t *y, const int32_t *w, int64_t K, int64_t area, int32_t T,
                        const fcfs_window *win, fcfs_precision prec, const fcfs_shard *shard,
                        const fcfs_options *opt, void *F, void *ws, size_t ws_bytes, void *stream) {
    return coeffs_one(x, y, w, K, area, T, win, prec, shard, opt, F, ws, ws_bytes, stream, nullptr, 0);
}

fcfs_status fcfs_coeffs_rows_to_peers(const int32_t *x, const int32_t *y, const int32_t *w, int64_t K, int64_t area,
                                      int32_t T, const fcfs_window *win, fcfs_precision prec, const fcfs_shard *shard,
                                      const fcfs_options *opt, void *const *peers, int32_t n_peers, void *ws,
                                      size_t ws_bytes, void *stream) {
    if (!shard || shard->kind != FCFS_SHARD_ROWS) {
        set_error("fcfs_coeffs_rows_to_peers: needs a ROWS shard");
        return FCFS_E_INVALID;
    }
    if (!win || win->layout != FCFS_LAYOUT_DENSE) {
        set_error("fcfs_coeffs_rows_to_peers: ROWS shards use the DENSE layout");
        return FCFS_E_INVALID;
    }
    if (!peers || n_peers < 1 || n_peers > kMaxPeers) {
        set_error("fcfs_coeffs_rows_to_peers: n_peers=%d outside [1, %d]", n_peers, kMaxPeers);
        return FCFS_E_INVALID;
    }
    for (int32_t i = 0; i < n_peers; ++i)
        if (!peers[i]) { set_error("fcfs_coeffs_rows_to_peers: peer %d is NULL", i); return FCFS_E_INVALID; }
    return coeffs_one(x, y, w, K, area, T, win, prec, shard, opt, peers[0], ws, ws_bytes, stream, peers, n_peers);
}

fcfs_status fcfs_coeffs_async(const int32_t *x, const int32_t *y, const int32_t *w, const int64_t *K_dev, int64_t K_cap,
                              const int64_t *area_dev, int32_t T, const fcfs_window *win, fcfs_precision prec, void *F,
                              int32_t *status_dev, void *ws, size_t ws_bytes, void *stream) {
    if (!valid_T(T)) { set_error("T=%d outside [1, 2^20]", T); return FCFS_E_INVALID; }
    fcfs_status st = check_window(win);
    if (st != FCFS_OK) return st;
    if (K_cap < 1 || !x || !y || !w || !K_dev || !area_dev || !F || !status_dev) {
        set_error("fcfs_coeffs_async: null pointer or K_cap < 1");
        return FCFS_E_INVALID;
    }
    if (prec != FCFS_FP64 && prec != FCFS_TF32X3 && prec != FCFS_F16X3) { set_error("bad precision %d", prec); return FCFS_E_INVALID; }
    if (ws == nullptr || ((uintptr_t)ws & 255)) { set_error("ws NULL or not 256-byte aligned"); return FCFS_E_WORKSPACE; }
    st = device_ok();
    if (st != FCFS_OK) return st;
    GemmPlan plan = make_plan(win->M, win->N, -win->M, win->M, 1, K_cap, false);
    plan.phys = prec == FCFS_FP64 ? 0 : 1;
    FftPlan fp;
    if (!fft_route_plan(T, win->M, win->N, -win->M, win->M, K_cap, prec != FCFS_FP64, fp, FCFS_ROUTE_FFT)) {
        set_error("fcfs_coeffs_async: the lattice-FFT route does not apply to T=%d, N=%d", T, win->N);
        return FCFS_E_UNSUPPORTED;
    }
    Carver cv(ws, ws_bytes);
    CoeffWs W;
    carve_coeff(cv, plan, W, !fusable(plan, prec, win->M, -win->M, win->M, true), K_cap, 1, prec, true, &fp);
    if (!cv.fits()) { set_error("fcfs_coeffs_async: workspace %zu < %zu", ws_bytes, cv.used()); return FCFS_E_WORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    EpiArgs ea;
    ea.M = win->M; ea.N = win->N; ea.layout = win->layout; ea.r2 = win->pupil_r2;
    ea.m_lo = -win->M; ea.m_hi = win->M; ea.T = T; ea.area_dev = area_dev; ea.area_host = 0;
    ea.out_f32 = prec == FCFS_FP64 ? 0 : 1;
    ea.out_per_clip = 0;
    StageScope scope(kStageContract, s);
    FCFS_TRY(fft_route_prepare_dev(y, K_dev, K_cap, fp, W.fft, W.fft_bytes, status_dev, s));
    return fft_route_run(x, w, 0, fp, W.fft, W.fft_bytes, ea, F, s);
}

size_t fcfs_batched_workspace_bytes(int64_t B, int64_t K_total, int64_t K_max, int32_t T, const fcfs_window *win,
                                    fcfs_precision prec, const fcfs_options *opt) {
    (void)T;
    if (check_window(win) != FCFS_OK || check_options(opt) != FCFS_OK || B < 1) return 0;
    GemmPlan p = make_plan(win->M, win->N, -win->M, win->M, B, K_max, true);
    Carver cv(nullptr, 0);
    CoeffWs w;
    const bool lat = valid_T(T) && batched_form(prec, opt, B, K_total, T, win) == FCFS_FORM_LATTICE;
    carve_coeff(cv, p, w, !fusable(p, prec, win->M, -win->M, win->M), K_total, B, prec, false, nullptr, lat ? T : 0);
    return cv.used();
}

int32_t fcfs_coeffs_batched_form(int64_t B, int64_t K_total, int64_t K_max, int32_t T, const fcfs_window *win,
                                 fcfs_precision prec, const fcfs_options *opt) {
    (void)K_max;
    if (!valid_T(T) || check_window(win) != FCFS_OK || check_options(opt) != FCFS_OK) return 0;
    if (prec != FCFS_FP64 && prec != FCFS_TF32X3 && prec != FCFS_F16X3) return 0;
    return batched_form(prec, opt, B, K_total, T, win);
}

}  // extern "C"

static fcfs_status batched_impl(const int64_t *corner_ptr, int64_t B, int64_t K_total, int64_t K_max,
                                const int32_t *x, const int32_t *y, const int32_t *w, const int64_t *area,
                                int32_t T, const fcfs_window *win, fcfs_precision prec, const fcfs_options *opt,
                                void *F, void *ws, size_t ws_bytes, void *stream, const EdgeWs *given) {
    if (!valid_T(T)) { set_error("T=%d outside [1, 2^20]", T); return FCFS_E_INVALID; }
    fcfs_status st = check_window(win);
    if (st == FCFS_OK) st = check_options(opt);
    if (st != FCFS_OK) return st;
    if (B < 1 || !corner_ptr || !area || !F || K_total < 0 || K_max < 0 || (K_total > 0 && (!x || !y || !w))) {
        set_error("fcfs_coeffs_batched: invalid sizes or null pointers");
        return FCFS_E_INVALID;
    }
    if (prec != FCFS_FP64 && prec != FCFS_TF32X3 && prec != FCFS_F16X3) {
        set_error("bad precision %d", prec);
        return FCFS_E_INVALID;
    }
    if (ws == nullptr || ((uintptr_t)ws & 255)) { set_error("ws NULL or not 256-byte aligned"); return FCFS_E_WORKSPACE; }
    st = device_ok();
    if (st != FCFS_OK) return st;
    GemmPlan plan = make_plan(win->M, win->N, -win->M, win->M, B, K_max, true);
    plan.phys = prec == FCFS_FP64 ? 0 : 1;
    Carver cv(ws, ws_bytes);
    CoeffWs W;
    int32_t form = batched_form(prec, opt, B, K_total, T, win);
    if (given && form == FCFS_FORM_LATTICE && opt->form != FCFS_FORM_LATTICE) form = FCFS_FORM_EDGE;
    carve_coeff(cv, plan, W, !fusable(plan, prec, win->M, -win->M, win->M), K_total, B, prec, false, nullptr,
                form == FCFS_FORM_LATTICE ? T : 0);
    if (!cv.fits()) { set_error("fcfs_coeffs_batched: workspace %zu < %zu", ws_bytes, cv.used()); return FCFS_E_WORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    CornerSrc src{};
    src.x = x; src.y = y; src.w = w; src.corner_ptr = corner_ptr; src.k_lo = 0; src.k_hi = K_total;
    src.bptr = W.bk.bptr; src.by = W.bk.by; src.clip_bptr = W.bk.clip_bptr; src.kend = K_total;
    EpiArgs ea;
    ea.M = win->M; ea.N = win->N; ea.layout = win->layout; ea.r2 = win->pupil_r2;
    ea.m_lo = -win->M; ea.m_hi = win->M; ea.T = T; ea.area_dev = area; ea.area_host = 0;
    ea.out_f32 = prec == FCFS_FP64 ? 0 : 1;
    ea.out_per_clip = fcfs_window_size(win);
    bool fused = false;
    if (form == FCFS_FORM_LATTICE) {
        // the lattice-row form (lattice.cu): B chunk table + chunk pointers, then one kernel with the fused
        // epilogue.  Unless the caller guarantees y-sorted lists, the chunk pass's flag is read back (one
        // stream sync) and an unsorted batch takes the edge form instead
        StageScope scope(kStageContract, s);
        FCFS_TRY_CUDA(cudaMemsetAsync(W.flag, 0, sizeof(int32_t), s));
        st = launch_lattice_prepare(corner_ptr, B, y, K_total, T, win->M, win->N, W.lat, W.flag, !opt->sorted_y, s);
        if (st != FCFS_OK) return st;
        int32_t unsorted = 0;
        if (!opt->sorted_y) {
            FCFS_TRY_CUDA(cudaMemcpyAsync(&unsorted, W.flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
            FCFS_TRY_CUDA(cudaStreamSynchronize(s));
        }
        if (!unsorted) return launch_lattice(corner_ptr, B, x, y, w, T, ea, F, W.lat, s);
        form = FCFS_FORM_EDGE;
    }
    if (prec == FCFS_TF32X3 && K_total > 0 && (given || form == FCFS_FORM_EDGE)) {   // K/2-term form
        const EdgeWs *e = given ? given : &W.edges;
        if (!given) {
            StageScope scope(kStagePair, s);
            st = run_edges(x, y, w, corner_ptr, B, W.edges, s);
        }
        src.exa = e->xa; src.exb = e->xb; src.ey = e->y; src.ec = e->c;
        src.ecnt = e->cnt;
    }
    if (st == FCFS_OK) {
        StageScope scope(kStageContract, s);
        if (prec == FCFS_FP64) st = run_buckets(y, corner_ptr, B, 0, K_total, kRowBucketCapFp64, W.bk, s);
        if (st == FCFS_OK) st = run_gemm(src, plan, T, prec, W.P, ea, F, s, &fused);
    }
    if (st != FCFS_OK || fused) return st;
    StageScope scope(kStageEpilogue, s);
    return launch_epilogue(plan, W.P, ea, F, s);
}

fcfs_status fcfs_edges(const int32_t *x, const int32_t *y, const int32_t *w, const int64_t *corner_ptr,
                       int64_t B, int32_t *xa, int32_t *xb, int32_t *ye, int32_t *c, int32_t *ecnt,
                       void *stream) {
    if (B < 1 || !corner_ptr || !x || !y || !w || !xa || !xb || !ye || !c || !ecnt) {
        set_error("fcfs_edges: invalid sizes or null pointers");
        return FCFS_E_INVALID;
    }
    fcfs_status st = device_ok();
    if (st != FCFS_OK) return st;
    EdgeWs e;
    e.xa = xa; e.xb = xb; e.y = ye; e.c = c; e.cnt = ecnt;
    return run_edges(x, y, w, corner_ptr, B, e, (cudaStream_t)stream);
}

extern "C" {

fcfs_status fcfs_coeffs_batched(const int64_t *corner_ptr, int64_t B, int64_t K_total, int64_t K_max,
                                const int32_t *x, const int32_t *y, const int32_t *w, const int64_t *area,
                                int32_t T, const fcfs_window *win, fcfs_precision prec, const fcfs_options *opt,
                                void *F, void *ws, size_t ws_bytes, void *stream) {
    return batched_impl(corner_ptr, B, K_total, K_max, x, y, w, area, T, win, prec, opt, F, ws, ws_bytes, stream,
                        nullptr);
}

fcfs_status fcfs_coeffs_batched_edges(const int64_t *corner_ptr, int64_t B, int64_t K_total, int64_t K_max,
                                      const int32_t *x, const int32_t *y, const int32_t *w, const int64_t *area,
                                      const int32_t *xa, const int32_t *xb, const int32_t *ye, const int32_t *c,
                                      const int32_t *ecnt, int32_t T, const fcfs_window *win, fcfs_precision prec,
                                      const fcfs_options *opt, void *F, void *ws, size_t ws_bytes, void *stream) {
    if (K_total > 0 && (!xa || !xb || !ye || !c || !ecnt)) {
        set_error("fcfs_coeffs_batched_edges: null edge input");
        return FCFS_E_INVALID;
    }
    EdgeWs e;
    e.xa = const_cast<int32_t *>(xa); e.xb = const_cast<int32_t *>(xb); e.y = const_cast<int32_t *>(ye);
    e.c = const_cast<int32_t *>(c); e.cnt = const_cast<int32_t *>(ecnt);
    return batched_impl(corner_ptr, B, K_total, K_max, x, y, w, area, T, win, prec, opt, F, ws, ws_bytes, stream, &e);
}

size_t fcfs_row_buckets_workspace_bytes(int64_t K, int64_t B) {
    if (K < 0 || B < 1) return 0;
    return buckets_workspace_bytes(K, B);
}

fcfs_status fcfs_row_buckets(const int32_t *y, const int64_t *corner_ptr, int64_t B, int64_t K, int32_t cap,
                             int32_t *bptr, int32_t *by, int64_t *clip_bptr, int64_t *nb_host, void *ws,
                             size_t ws_bytes, void *stream) {
    if (K < 0 || B < 1 || (K > 0 && !y) || !bptr || !by || !clip_bptr || !nb_host || cap < 1 || cap > 32 ||
        (corner_ptr == nullptr && B != 1)) {
        set_error("fcfs_row_buckets: invalid sizes or null pointers");
        return FCFS_E_INVALID;
    }
    if (ws == nullptr || ((uintptr_t)ws & 255)) { set_error("ws NULL or not 256-byte aligned"); return FCFS_E_WORKSPACE; }
    fcfs_status st = device_ok();
    if (st != FCFS_OK) return st;
    Carver cv(ws, ws_bytes);
    BucketWs W;
    carve_buckets(cv, K, B, W);
    if (!cv.fits()) { set_error("fcfs_row_buckets: workspace %zu < %zu", ws_bytes, cv.used()); return FCFS_E_WORKSPACE; }
    cudaStream_t s = (cudaStream_t)stream;
    st = run_buckets(y, corner_ptr, B, 0, K, cap, W, s);
    if (st != FCFS_OK) return st;
    // the pass writes into the workspace; copy the caller-visible arrays out
    int64_t nb = 0;
    FCFS_TRY_CUDA(cudaMemcpyAsync(&nb, W.clip_bptr + B, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    FCFS_TRY_CUDA(cudaStreamSynchronize(s));
    FCFS_TRY_CUDA(cudaMemcpyAsync(bptr, W.bptr, sizeof(int32_t) * (nb + 1), cudaMemcpyDeviceToDevice, s));
    if (nb > 0) FCFS_TRY_CUDA(cudaMemcpyAsync(by, W.by, sizeof(int32_t) * nb, cudaMemcpyDeviceToDevice, s));
    FCFS_TRY_CUDA(cudaMemcpyAsync(clip_bptr, W.clip_bptr, sizeof(int64_t) * (B + 1), cudaMemcpyDeviceToDevice, s));
    *nb_host = nb;
    return FCFS_OK;
}

}  // extern "C"

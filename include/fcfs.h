/*
 * fcfs.h — C-ABI of libfcfs.so: the B200 (sm_100a) hot path of the fast continuous
 * Fourier series (FCFS) of rectilinear polygons, arXiv 1010.5562.
 *
 * Citations are PAPER.md line numbers ("P:n") with the section / equation they fall in.
 *
 * Problem (readings A1-A7).  A clip of period T holds the mask
 *     f(x,y) = sum over polygon groups g of 1[ union of the rects of g ]      (P:589-595 Eq. signal_model)
 * and the library returns its continuous-Fourier-series coefficients
 *     F[m,n] = (1/T^2) * integral_[0,T)^2 f(x,y) e^{-2 pi i (m x + n y)/T} dx dy
 * (the paper's orthonormal F^_{k,l} equals T*F[k,l]), from the signed corner list of f:
 *     F[0,0] = area/T^2                                  Eq. Fdc P:831-834 (Step 1)
 *     F[m,0] = i/(2 pi m T) sum_k w_k y_k E_x[m,k]        Eq. Fk0 P:835-838 (Step 2)
 *     F[0,n] = i/(2 pi n T) sum_k w_k x_k E_y[n,k]        Eq. F0l P:839-842 (Step 3)
 *     F[m,n] = -1/(4 pi^2 m n) sum_k w_k E_x[m,k] E_y[n,k] Eq. Fkl P:843-846 (Step 4)
 * with E_x[m,k] = e^{-2 pi i ((m x_k) mod T)/T}; phases are reduced exactly in integers
 * because the vertices lie on the integer lattice.  The contraction is the
 * paper's "Goertzel-like" direct evaluation restricted to a low-pass window
 * or pupil disk (future work P:1247-1255), run in parallel (future work P:1257-1259); for
 * one large clip the library may instead take the paper's Step 4 as row DFTs followed by
 * an output-pruned FFT along y (fcfs_coeffs_route).
 *
 * Entry points:
 *   a1   fcfs_vertices_from_rects[_edges], fcfs_vertices_from_polygons, fcfs_chop_rects (layout -> tiles)
 *   a2-5 fcfs_coeffs (one clip, optional ROWS / VERTEX_BLOCK shard), fcfs_coeffs_batched[_edges],
 *        fcfs_coeffs_route, fcfs_row_buckets, fcfs_edges
 *   CHT  fcfs_haar (the paper's continuous Haar transform of the same corners)
 *   misc *_workspace_bytes, fcfs_window_size, fcfs_pupil_indices, fcfs_status_string,
 *        fcfs_last_error, fcfs_device_check, fcfs_kernel_launches, fcfs_profile_enable/read
 *
 * Conventions for every entry point:
 *  - All array pointers are DEVICE pointers owned by the caller unless the name ends in
 *    _host or the argument is a struct pointer (fcfs_window, fcfs_shard: host structs).
 *    The library never allocates or frees device memory; scratch comes from `ws`,
 *    sized by the matching *_workspace_bytes query.  `ws` must be 256-byte aligned.
 *  - `stream` is a cudaStream_t (0 = legacy default stream).  All device work is
 *    enqueued on it; outputs are valid once that stream's work completes.
 *  - Return value: FCFS_OK or an error code; no exception crosses the ABI.  A
 *    human-readable detail for the last error of the calling thread is available from
 *    fcfs_last_error().  On error nothing useful has been written to the outputs.
 *  - Coordinates: rects are half-open [x0,x1) x [y0,y1) with
 *    0 <= x0 < x1 <= T, 0 <= y0 < y1 <= T, T in [1, 2^20].  Corners with x = T or
 *    y = T are kept with their raw coordinate (reading A7): only phases wrap mod T.
 */
#ifndef FCFS_H_
#define FCFS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t fcfs_status;
#define FCFS_OK 0
#define FCFS_E_INVALID 1     /* null pointer, T out of range, M or N < 0, bad enum, bad CSR   */
#define FCFS_E_RANGE 2       /* a rect outside [0,T]^2 or with x0 >= x1 / y0 >= y1 (device-checked) */
#define FCFS_E_CAPACITY 3    /* more corners than `cap`; *K_total_host still holds the count   */
#define FCFS_E_WORKSPACE 4   /* ws too small (or unaligned) for this call                       */
#define FCFS_E_UNSUPPORTED 5 /* device is not sm_100, or a size limit of this build is exceeded */
#define FCFS_E_CUDA 6        /* a CUDA runtime error (detail in fcfs_last_error())              */

/* Arithmetic of the contraction (BASELINE.json north_star (3)). */
typedef int32_t fcfs_precision;
#define FCFS_FP64 0    /* FP64 throughout; output complex128 (double re, double im); |err| <= 1e-12 B */
#define FCFS_TF32X3 1  /* split-TF32 tcgen05 tensor-core contraction, FP64 flush of FP32 TMEM partials;
                          output complex64 (float re, float im); |err| <= 1e-5 B                      */
#define FCFS_F16X3 2   /* split-FP16 tcgen05 contraction (hi/lo fp16 operands, kind::f16, FP32 TMEM
                          accumulation, FP64 flush): the same FP32-accurate contract as FCFS_TF32X3
                          at half the operand bytes; output complex64; |err| <= 1e-5 B              */

/* Output layout. */
#define FCFS_LAYOUT_DENSE 0  /* (2M+1) x (2N+1) row-major, entry (m,n) at (m+M)*(2N+1) + (n+N);
                                if pupil_r2 >= 0, entries with m^2+n^2 > pupil_r2 are written as 0 */
#define FCFS_LAYOUT_PUPIL 1  /* packed: only |m|<=M, |n|<=N, m^2+n^2 <= pupil_r2, m-major then n
                                (fcfs_pupil_indices gives the order); requires pupil_r2 >= 0    */

/* Frequency window (reading A3: signed window, alpha at the signed index) and pupil disk
 * (BASELINE.json cut-off NA(1+sigma)/lambda, inclusive, reading A11). */
typedef struct {
    int32_t M;          /* |m| <= M */
    int32_t N;          /* |n| <= N */
    double pupil_r2;    /* < 0: rectangular window; else keep m^2+n^2 <= pupil_r2 */
    int32_t layout;     /* FCFS_LAYOUT_DENSE or FCFS_LAYOUT_PUPIL */
} fcfs_window;

/* Explicit kernel-route options (the library reads no environment variables: what it computes is fixed
 * by its arguments).  Pass NULL for the defaults (every field AUTO).  Every route and form meets the same
 * accuracy contract of `prec`; the options exist for A/B measurement and for the tests that force each
 * route on the same inputs. */
#define FCFS_ROUTE_AUTO 0   /* fcfs_coeffs: the cost model picks (fcfs_coeffs_route)                      */
#define FCFS_ROUTE_GEMM 1   /* fcfs_coeffs: the row-bucket GEMM on the tensor cores                      */
#define FCFS_ROUTE_FFT 2    /* fcfs_coeffs: the lattice-FFT route wherever it applies (power-of-two T >= 64,
                               2N+1 <= min(T, 4096), y-sorted corners); elsewhere the row-bucket GEMM   */
#define FCFS_FORM_AUTO 0    /* fcfs_coeffs_batched (split precisions): the library's choice               */
#define FCFS_FORM_EDGE 1    /* FCFS_TF32X3: contract over edges (fcfs_edges; the K/2-term form of Eq. Fkl) */
#define FCFS_FORM_CORNER 2  /* contract over corners (the K-term form of Eq. Fkl)                         */
#define FCFS_FORM_LATTICE 3 /* FCFS_TF32X3: contract over the T+1 lattice rows (Step 4 as row DFTs, then the
                               DFT along y as a tensor-core GEMM against a fixed table).  Needs
                               T % 4 == 0, T <= 4096, M, N <= 31 and y-sorted corner lists; where a condition
                               fails the library takes the edge form instead                               */
typedef struct {
    int32_t route;      /* FCFS_ROUTE_*  */
    int32_t form;       /* FCFS_FORM_*   */
    int32_t sorted_y;   /* 1: the caller guarantees every clip's corners are sorted by y (fcfs_vertices_from_*
                           output is); 0: the lattice-row form checks it on the device (one stream sync)   */
    int32_t reserved[5];/* must be 0     */
} fcfs_options;

/* Work partition of one clip (BASELINE.json north_star (6); linearity Prop. 2). */
#define FCFS_SHARD_NONE 0
#define FCFS_SHARD_ROWS 1          /* rows m in [m_lo, m_hi] (signed, inside [-M, M]) of the DENSE
                                      layout; F holds (m_hi-m_lo+1)*(2N+1) entries                    */
#define FCFS_SHARD_VERTEX_BLOCK 2  /* corners [k_lo, k_hi) only: F = that block's partial window
                                      (full DENSE/PUPIL layout).  Its DC is (sum w x y over the block)/T^2,
                                      so the sum of the P blocks' F equals the unsharded F (`area` unused) */
typedef struct {
    int32_t kind;
    int32_t m_lo, m_hi;
    int64_t k_lo, k_hi;
} fcfs_shard;

/* ------------------------------------------------------------------------------------------
 * a1 — vertex extraction (Alg. 2 lines 1-14; Prop. 1; Step 1 P:866-868).
 *
 * rects      int32 [R][4] (x0, y0, x1, y1), device, 16-byte aligned (one int4 load per rect; else
 *            FCFS_E_INVALID).  Corner arrays (x, y, w) of every entry point need only 4-byte alignment.
 * group_ptr  int64 [G+1] CSR over rects, device; NULL => every rect is its own group (G == R).
 *            Within a group the rects are UNIONED; groups are SUMMED (reading A5).
 * clip_ptr   int64 [B+1] CSR over groups, device; NULL => one clip (B == 1).
 * x, y, w    int32 [cap] out: canonical signed corners w(x,y) = f(x,y)-f(x-1,y)-f(x,y-1)+f(x-1,y-1)
 *            of every clip, zero weights dropped, sorted by (clip, y, x).  Bit-exact.
 * corner_ptr int64 [B+1] out: CSR of corners per clip.
 * area       int64 [B] out: sum_k w_k x_k y_k = area of f per clip (exact).
 * K_total_host  out (host): total corner count.  This call synchronises `stream` once.
 * max_group  the largest number of rects in one group (host-known; sizes the workspace).
 * Limits: T <= 2^20, B < 2^22, groups of at most 100 rects (else FCFS_E_UNSUPPORTED).
 * ------------------------------------------------------------------------------------------ */
size_t fcfs_vertices_workspace_bytes(int64_t R, int64_t G, int64_t B, int64_t max_group);
fcfs_status fcfs_vertices_from_rects(const int32_t *rects, int64_t R, const int64_t *group_ptr,
                                     int64_t G, const int64_t *clip_ptr, int64_t B, int32_t T,
                                     int64_t max_group, int32_t *x, int32_t *y, int32_t *w,
                                     int64_t cap, int64_t *corner_ptr, int64_t *area,
                                     int64_t *K_total_host, void *ws, size_t ws_bytes,
                                     void *stream);

/* The same, also writing the edge pairing of the output corners (fcfs_edges' rule and layout:
 * xa, xb, ye, c int32 [cap], ecnt int32 [B]; fcfs_edges' pass runs after the extraction), for
 * fcfs_coeffs_batched_edges: pair once, contract several windows. */
fcfs_status fcfs_vertices_from_rects_edges(const int32_t *rects, int64_t R, const int64_t *group_ptr,
                                           int64_t G, const int64_t *clip_ptr, int64_t B, int32_t T,
                                           int64_t max_group, int32_t *x, int32_t *y, int32_t *w,
                                           int64_t cap, int64_t *corner_ptr, int64_t *area,
                                           int64_t *K_total_host, int32_t *xa, int32_t *xb,
                                           int32_t *ye, int32_t *c, int32_t *ecnt, void *ws,
                                           size_t ws_bytes, void *stream);

/* One clip's canonical corners restricted to the lattice rows y_lo <= y < y_hi — the y-band
 * shard of a1 for multi-GPU single-clip runs (Prop. 2 linearity).  A
 * canonical corner is the sum of the raw corners of one (x, y) key (Prop. 1), so the
 * band's list is exactly the unbanded list's rows in [y_lo, y_hi): rank r of P extracting the band
 * [y_r, y_{r+1}) and the bands concatenated in order give the canonical list bit for bit.
 * Arguments as fcfs_vertices_from_rects with clip_ptr = NULL, B = 1 (same workspace query with
 * B = 1); corner_ptr int64 [2]; area = sum over the band's corners of w x y (the bands' areas sum
 * to the clip's).  0 <= y_lo <= y_hi (y_hi > T: no upper cut), else FCFS_E_INVALID.  One sync. */
fcfs_status fcfs_vertices_from_rects_band(const int32_t *rects, int64_t R, const int64_t *group_ptr,
                                          int64_t G, int32_t T, int64_t max_group, int32_t y_lo,
                                          int32_t y_hi, int32_t *x, int32_t *y, int32_t *w, int64_t cap,
                                          int64_t *corner_ptr, int64_t *area, int64_t *K_host, void *ws,
                                          size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------------------------
 * a1 from polygon vertex lists (the paper's own input: Alg. 2 REQUIRE "clockwise vertex lists",
 * P:930-935; lines 9-10 "+1 at the end, -1 at the start of each horizontal edge").
 *
 * vx, vy     int32 [V] vertices, device.  Polygon p is vertices [poly_ptr[p], poly_ptr[p+1]),
 *            closed (edge i runs from vertex i to vertex i+1 mod n).  Any start vertex, either
 *            orientation (reading A16: a list whose area sum_h y_a (x_b - x_a) is negative is
 *            taken reversed), collinear vertices allowed; every edge must be horizontal or
 *            vertical with non-zero length.  Self-intersection is not checked.
 * poly_ptr   int64 [P+1] CSR over vertices, device (poly_ptr[0] == 0, poly_ptr[P] == V).
 * clip_ptr   int64 [B+1] CSR over polygons, device; NULL => one clip (B == 1).
 *            The polygons of a clip are SUMMED (signal model).
 * x, y, w, corner_ptr, area, K_total_host: as fcfs_vertices_from_rects (bit-exact canonical
 *            corners sorted by (clip, y, x); one stream sync).
 * Errors: FCFS_E_INVALID for a diagonal or zero-length edge (device-checked), FCFS_E_RANGE for a
 * vertex outside [0,T]^2, FCFS_E_CAPACITY if K > cap (K_total_host still written).
 * Limits: T <= 2^20, B < 2^22, V < 2^31.
 * ------------------------------------------------------------------------------------------ */
size_t fcfs_polygons_workspace_bytes(int64_t V, int64_t P, int64_t B);
fcfs_status fcfs_vertices_from_polygons(const int32_t *vx, const int32_t *vy, int64_t V,
                                        const int64_t *poly_ptr, int64_t P, const int64_t *clip_ptr,
                                        int64_t B, int32_t T, int32_t *x, int32_t *y, int32_t *w,
                                        int64_t cap, int64_t *corner_ptr, int64_t *area,
                                        int64_t *K_total_host, void *ws, size_t ws_bytes,
                                        void *stream);

/* ------------------------------------------------------------------------------------------
 * The continuous Haar transform of B clips (the paper's CHT / PCHT; reading
 * A18): the dyadic nonstandard 2D Haar basis over [0,T)^2, T = 2^J (2 <= T <= 4096), J = log2 T
 * levels, h = (1,-1)/sqrt2 (first half positive), psi^(hg) = h along x.
 *
 * corner_ptr int64 [B+1] CSR over corners (device), or NULL for B == 1;  x, y, w  int32 [K] corners
 *            as produced by fcfs_vertices_from_* (any order);  area  int64 [B] (device).
 * out        double [B][T][T] (device): out[b][r][c], r = y index: (0,0) = X_{0,0,0} = area/T; level j:
 *            hg at (ky, 2^j + kx), gh at (2^j + ky, kx), hh at (2^j + ky, 2^j + kx).  Every value is
 *            exact (an integer times 2^j / T).  Clips whose corners are sorted by y (the order
 *            fcfs_vertices_from_* emit) take a band sweep that reads only the corners; any other order
 *            takes a scatter of the corners into a per-clip scratch (a device flag picks the path: no
 *            host sync).  Workspace (fcfs_haar_workspace_bytes): the scatter scratch, 5 (T^2 - 1) / 3
 *            int64 per clip, which must be zero-initialised before its first use and which every
 *            successful call leaves zero (the kernels clear the entries they used instead of an O(T^2)
 *            memset per call), then B (T + 1) + 1 int32 of per-call scratch (row pointers, the flag).
 * ------------------------------------------------------------------------------------------ */
size_t fcfs_haar_workspace_bytes(int64_t B, int32_t T);
fcfs_status fcfs_haar(const int64_t *corner_ptr, int64_t B, int64_t K, const int32_t *x, const int32_t *y,
                      const int32_t *w, const int64_t *area, int32_t T, double *out, void *ws,
                      size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------------------------
 * Layout -> tiles (the paper's flow: "chops polygons and places them in their corresponding tiles.
 * Each tile is then transformed individually"; reading A17).
 *
 * rects      int32 [R][4] (x0, y0, x1, y1) half-open in layout coordinates, device,
 *            0 <= x0 < x1 <= tiles_x T, 0 <= y0 < y1 <= tiles_y T (else FCFS_E_RANGE).
 * Tile (tx, ty) = [tx T, (tx+1) T) x [ty T, (ty+1) T), index ty * tiles_x + tx.
 * out_rects  int32 [cap][4] out: every rect cut at the tile edges into non-empty pieces in tile-local
 *            coordinates (0 <= x0 < x1 <= T), ordered by tile, then by rect (deterministic).
 * tile_ptr   int64 [tiles_x tiles_y + 1] out: CSR of pieces per tile — pass it as clip_ptr (with
 *            group_ptr NULL) to fcfs_vertices_from_rects to get every tile's corners as one batch.
 * n_host     out (host): the number of pieces (written also when it exceeds cap: FCFS_E_CAPACITY).
 * The call synchronises `stream` once.  Limits: tiles and pieces < 2^31, tiles_x T and tiles_y T < 2^31.
 * ------------------------------------------------------------------------------------------ */
size_t fcfs_chop_workspace_bytes(int64_t R, int64_t cap, int32_t tiles_x, int32_t tiles_y);
fcfs_status fcfs_chop_rects(const int32_t *rects, int64_t R, int32_t T, int32_t tiles_x, int32_t tiles_y,
                            int32_t *out_rects, int64_t cap, int64_t *tile_ptr, int64_t *n_host,
                            void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------------------------
 * a2-a5 — coefficients of ONE clip: phase reduction + twiddles (a2), the separable
 * contraction P = A diag(w) B^T over cos/sin quadrant rows (a3), axes + DC (a4) and the
 * window / pupil epilogue with exact conj mirroring F[-m,-n] = conj F[m,n] (a5).
 *
 * x, y, w  int32 [K] corners (device) as produced by fcfs_vertices_from_rects (any order
 *          is accepted; results are order-independent up to rounding).
 * area     sum_k w_k x_k y_k (host value), used for F[0,0] = area/T^2.
 * win      host struct, see fcfs_window.   prec  FCFS_FP64, FCFS_TF32X3 or FCFS_F16X3.
 * shard    host struct or NULL (= FCFS_SHARD_NONE).
 * F        out (device): complex128 (FP64) or complex64 (TF32X3 / F16X3) in the window layout.
 * Two routes (fcfs_coeffs_route): the lattice-FFT route (Step 4 as row DFTs, then an output-pruned
 * FFT along y) when it is cheaper and the corners are y-sorted, else the
 * row-bucket GEMM: the corners contracted over their row buckets (fcfs_row_buckets, cap 32) in
 * chunks of <= 128K buckets.  Either way the call synchronises `stream` once (sortedness flag or
 * bucket count).
 * ------------------------------------------------------------------------------------------ */
size_t fcfs_coeffs_workspace_bytes(int64_t K, int32_t T, const fcfs_window *win,
                                   fcfs_precision prec, const fcfs_shard *shard,
                                   const fcfs_options *opt);
/* Which single-clip route fcfs_coeffs takes for these sizes (planning / reporting; no device work):
 * 1 = the lattice-FFT route (power-of-two T >= 64, 2N+1 <= min(T, 4096), chosen by a cost model over
 * the row-bucket GEMM; taken only if the corner list is y-sorted, as fcfs_vertices_from_* produce it
 * — fcfs_coeffs checks on the device and otherwise falls back).  FCFS_FP64 runs it in FP64;
 * FCFS_TF32X3 / FCFS_F16X3 run it in FP32 on the CUDA cores (FP64 outer and axis sums) under their
 * 1e-5 B contract and complex64 output.  0 = the row-bucket GEMM on the tensor cores (DMMA, or the
 * split tcgen05 kernels).  opt->route (FCFS_ROUTE_GEMM / FCFS_ROUTE_FFT) overrides the cost model;
 * opt NULL = FCFS_ROUTE_AUTO.  Both routes meet the same tolerance. */
int32_t fcfs_coeffs_route(int64_t K, int32_t T, const fcfs_window *win, fcfs_precision prec,
                          const fcfs_shard *shard, const fcfs_options *opt);
fcfs_status fcfs_coeffs(const int32_t *x, const int32_t *y, const int32_t *w, int64_t K,
                        int64_t area, int32_t T, const fcfs_window *win, fcfs_precision prec,
                        const fcfs_shard *shard, const fcfs_options *opt, void *F, void *ws,
                        size_t ws_bytes, void *stream);
/* The ROWS shard of one clip with its all_gather fused into the epilogue (multi-GPU single clips,
 * BASELINE.json north_star (6); linearity Prop. 2): as fcfs_coeffs with a FCFS_SHARD_ROWS
 * shard and the DENSE layout, but instead of writing the shard's rows to F, the epilogue stores every
 * output (m, n) of rows [m_lo, m_hi] at its FULL-window position (m + M)(2N + 1) + (n + N) into each of
 * peers[0 .. n_peers) — full-window buffers of all ranks (this rank's own and the peers' mapped into
 * this process, e.g. by CUDA IPC over NVLink).  1 <= n_peers <= 8.  The kernel ends with a system-scope
 * fence; the caller orders the ranks (a barrier or any collective after this call on every rank)
 * before reading a buffer.  Workspace: fcfs_coeffs_workspace_bytes with the same shard. */
fcfs_status fcfs_coeffs_rows_to_peers(const int32_t *x, const int32_t *y, const int32_t *w, int64_t K,
                                      int64_t area, int32_t T, const fcfs_window *win,
                                      fcfs_precision prec, const fcfs_shard *shard,
                                      const fcfs_options *opt, void *const *peers, int32_t n_peers,
                                      void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------------------------
 * a3-a5 batched — B independent clips (the paper's tiles) in one launch sequence.
 * corner_ptr int64 [B+1] (device) CSR into x, y, w; area int64 [B] (device).
 * K_total = corner_ptr[B] and K_max = max_b (corner_ptr[b+1]-corner_ptr[b]) are passed from
 * the host (fcfs_vertices_from_rects returns K_total; K_max sizes the per-clip plan).
 * F out: B consecutive output blocks of fcfs_window_size(win) entries each.
 * ------------------------------------------------------------------------------------------ */
size_t fcfs_batched_workspace_bytes(int64_t B, int64_t K_total, int64_t K_max, int32_t T,
                                    const fcfs_window *win, fcfs_precision prec,
                                    const fcfs_options *opt);
/* Which contraction form fcfs_coeffs_batched runs for these sizes (FCFS_FORM_LATTICE / FCFS_FORM_EDGE /
 * FCFS_FORM_CORNER; 0 for FCFS_FP64, which contracts over row buckets), assuming y-sorted corner lists:
 * planning / reporting, no device work.  FCFS_FORM_AUTO takes the lattice-row form where it applies and the
 * clips hold at least (T+1)/4 corners on average, else the edge form (FCFS_TF32X3). */
int32_t fcfs_coeffs_batched_form(int64_t B, int64_t K_total, int64_t K_max, int32_t T,
                                 const fcfs_window *win, fcfs_precision prec, const fcfs_options *opt);
fcfs_status fcfs_coeffs_batched(const int64_t *corner_ptr, int64_t B, int64_t K_total,
                                int64_t K_max, const int32_t *x, const int32_t *y,
                                const int32_t *w, const int64_t *area, int32_t T,
                                const fcfs_window *win, fcfs_precision prec,
                                const fcfs_options *opt, void *F, void *ws, size_t ws_bytes,
                                void *stream);

/* The same with the edge pairing of the corner lists given (the output of fcfs_edges or of
 * fcfs_vertices_from_rects_edges for these corners; arrays as fcfs_edges documents): FCFS_TF32X3
 * contracts over them instead of pairing again (the edge form unless opt->form is FCFS_FORM_LATTICE); other precisions
 * ignore them.  Same workspace. */
fcfs_status fcfs_coeffs_batched_edges(const int64_t *corner_ptr, int64_t B, int64_t K_total,
                                      int64_t K_max, const int32_t *x, const int32_t *y,
                                      const int32_t *w, const int64_t *area, const int32_t *xa,
                                      const int32_t *xb, const int32_t *ye, const int32_t *c,
                                      const int32_t *ecnt, int32_t T, const fcfs_window *win,
                                      fcfs_precision prec, const fcfs_options *opt, void *F, void *ws,
                                      size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------------------------
 * Sync-free single-clip pipeline (capturable in a CUDA graph; SURVEY §8(b) "device-side K"):
 *
 * fcfs_vertices_from_rects_async — a1 exactly as fcfs_vertices_from_rects (same workspace query, same
 *   bit-exact canonical output) but with no host synchronisation: the corner count goes to K_dev
 *   (int64 [1], device) and the outcome to status_dev (int32 [1], device: FCFS_OK, FCFS_E_RANGE,
 *   FCFS_E_UNSUPPORTED, FCFS_E_WORKSPACE or FCFS_E_CAPACITY when K > cap), to be read after the stream's
 *   work completes.  Always the general (sort) path; no edge output.
 * fcfs_coeffs_async — a2-a5 of one clip on the lattice-FFT route for a corner
 *   list whose count K is in device memory (K_dev, K <= K_cap) and whose area is area_dev (int64 [1]);
 *   corners must be y-sorted (fcfs_vertices_from_rects_async output is).  Workspace:
 *   fcfs_coeffs_workspace_bytes(K_cap, T, win, prec, NULL, &opt) with opt.route = FCFS_ROUTE_FFT.
 *   status_dev (device) becomes FCFS_E_INVALID if the corners are not y-sorted, FCFS_E_CAPACITY if
 *   K > K_cap; it is only written when it holds FCFS_OK, so the extraction's status carries through
 *   when both calls share one word.  FCFS_E_UNSUPPORTED (host) when the FFT route does not apply. */
fcfs_status fcfs_vertices_from_rects_async(const int32_t *rects, int64_t R, const int64_t *group_ptr,
                                           int64_t G, const int64_t *clip_ptr, int64_t B, int32_t T,
                                           int64_t max_group, int32_t *x, int32_t *y, int32_t *w,
                                           int64_t cap, int64_t *corner_ptr, int64_t *area,
                                           int64_t *K_dev, int32_t *status_dev, void *ws,
                                           size_t ws_bytes, void *stream);
/* fcfs_vertices_from_clips_async — a1 of B clips of singleton groups (group_ptr NULL: every rect its own
 *   group, clip_ptr required) with no host synchronisation, on the per-clip shared-memory bucket path of
 *   fcfs_vertices_from_rects (bit-exact, the same canonical output): the caller bounds the rects per clip,
 *   max_clip_rects <= 2048 (T <= 65534), which selects the kernel variant up front instead of a read-back.
 *   K_dev / status_dev as fcfs_vertices_from_rects_async (FCFS_E_UNSUPPORTED in status_dev if a clip holds
 *   more than the launched variant's capacity).  Workspace: fcfs_vertices_workspace_bytes(R, R, B, 1).
 *   With fcfs_coeffs_batched on the lattice-row form (opt.sorted_y = 1: no host sync either; K_total and
 *   K_max then serve only planning, so upper bounds are valid) a whole batched step is capturable. */
fcfs_status fcfs_vertices_from_clips_async(const int32_t *rects, int64_t R, const int64_t *clip_ptr, int64_t B,
                                           int32_t T, int64_t max_clip_rects, int32_t *x, int32_t *y, int32_t *w,
                                           int64_t cap, int64_t *corner_ptr, int64_t *area, int64_t *K_dev,
                                           int32_t *status_dev, void *ws, size_t ws_bytes, void *stream);
fcfs_status fcfs_coeffs_async(const int32_t *x, const int32_t *y, const int32_t *w,
                              const int64_t *K_dev, int64_t K_cap, const int64_t *area_dev, int32_t T,
                              const fcfs_window *win, fcfs_precision prec, void *F, int32_t *status_dev,
                              void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------------------------
 * Latency path for ONE SMALL CLIP: a1-a5 in a single kernel launch with NO host synchronisation
 * (capturable in a CUDA graph) — the paper's "only a few CFS coefficients" regime, evaluated term
 * by term (Goertzel-like) with the exact integer phase.  Every CTA extracts
 * the clip's canonical corners in shared memory (as fcfs_vertices_from_rects: unions within groups,
 * groups summed) and computes its rows of the half window (Eqs. Fkl / Fk0 / F0l / Fdc),
 * mirrored by conjugation.  Arithmetic is FP64 for every `prec` (the split precisions only select
 * complex64 output), so the result meets the FP64 contract (1e-12 B).
 *
 * rects, R, group_ptr, G, T, max_group: as fcfs_vertices_from_rects with clip_ptr = NULL (B = 1).
 * win        window / pupil, output layout as fcfs_coeffs (F: complex128 for FCFS_FP64, else complex64).
 * K_dev      int64 [1] device out (canonical corner count) or NULL.
 * status_dev int32 [1] device out: FCFS_OK, FCFS_E_RANGE (a bad rect) or FCFS_E_UNSUPPORTED (a group
 *            above max_group / more than 2048 raw corners), written by the kernel — the call itself
 *            does not synchronise, so read it after the stream's work completes.
 * Limits (host-checked, FCFS_E_UNSUPPORTED): T <= 8192, M <= 63, N <= 4096, max_group <= 100, 4 R <= 2048 for
 * singleton groups.  fcfs_small_clip_supported() answers the same question (1 / 0). */
int32_t fcfs_small_clip_supported(int64_t R, int64_t G, int32_t T, int64_t max_group, const fcfs_window *win);
fcfs_status fcfs_small_clip(const int32_t *rects, int64_t R, const int64_t *group_ptr, int64_t G,
                            int32_t T, int64_t max_group, const fcfs_window *win, fcfs_precision prec,
                            void *F, int64_t *K_dev, int32_t *status_dev, void *stream);

/* ------------------------------------------------------------------------------------------
 * Row buckets of a corner list — the row structure of Step 4: corners on one row
 * y share E_y[n, y], so sum_k w_k E_x[m,k] E_y[n,k] = sum_b E_y[n, y_b] sum_{k in b} w_k E_x[m,k]
 * and the FP64 contraction runs over buckets instead of corners.  fcfs_coeffs[_batched] compute
 * them internally; this entry point exposes the same pass (for tests and planning).
 *
 * A bucket is a maximal run of CONSECUTIVE corners with equal y, cut at every clip start
 * (corner_ptr[b]), at every corner index k with k % 4096 == 0 (the pass's segment size) and every
 * `cap` corners inside a run (counted from the run start).  Any corner order is valid.
 * y          int32 [K] (device), K = corner_ptr[B] (or the K argument when corner_ptr is NULL).
 * corner_ptr int64 [B+1] (device) or NULL (one range [0, K), B must be 1).
 * cap        1 .. 32.
 * bptr       int32 [K + 1] out (device): global corner index of each bucket start; bptr[nb] = K.
 * by         int32 [K] out (device): the bucket's y.
 * clip_bptr  int64 [B+1] out (device): CSR of buckets per clip.
 * nb_host    out (host): bucket count (this call synchronises `stream` once).
 * ------------------------------------------------------------------------------------------ */
/* ------------------------------------------------------------------------------------------
 * Edge pairing of a corner list — the K/2-term form of Eq. Fkl: two consecutive
 * corners k, k+1 of one clip with equal y and w_{k+1} = -w_k are one horizontal edge,
 *     w_k E_x[m,k] E_y[n,k] + w_{k+1} E_x[m,k+1] E_y[n,k+1] = w_k (E_x[m,k] - E_x[m,k+1]) E_y[n,k].
 * fcfs_coeffs_batched (FCFS_TF32X3) runs its contraction over these edges; this entry point
 * exposes the same pass (for tests and planning).
 *
 * Rule: a link joins k-1 and k when both lie in one clip, y[k-1] == y[k] and w[k-1] == -w[k];
 * along each maximal chain of links the corners at even chain positions (0, 2, ...) each emit
 * one edge: a pair's head (x_a = x[k], x_b = x[k+1], y[k], c = w[k]) when k+1 continues the
 * chain, else a one-ended edge (x_b = -1).  Exact for any corner list (order, weights).
 * x, y, w    int32 [K] (device), K = corner_ptr[B].
 * corner_ptr int64 [B+1] (device).
 * xa, xb, ye, c  int32 [K] out (device): clip b's edges, in corner order, at
 *            [corner_ptr[b], corner_ptr[b] + ecnt[b]); the rest of [corner_ptr[b], corner_ptr[b+1])
 *            is left unwritten.
 * ecnt       int32 [B] out (device): edges per clip.
 * Asynchronous on `stream`; no workspace, no host synchronisation.
 * ------------------------------------------------------------------------------------------ */
fcfs_status fcfs_edges(const int32_t *x, const int32_t *y, const int32_t *w, const int64_t *corner_ptr,
                       int64_t B, int32_t *xa, int32_t *xb, int32_t *ye, int32_t *c, int32_t *ecnt,
                       void *stream);

size_t fcfs_row_buckets_workspace_bytes(int64_t K, int64_t B);
fcfs_status fcfs_row_buckets(const int32_t *y, const int64_t *corner_ptr, int64_t B, int64_t K,
                             int32_t cap, int32_t *bptr, int32_t *by, int64_t *clip_bptr,
                             int64_t *nb_host, void *ws, size_t ws_bytes, void *stream);

/* Host helpers. */
int64_t fcfs_window_size(const fcfs_window *win);        /* outputs per clip; -1 if invalid */
int64_t fcfs_pupil_indices(int32_t M, int32_t N, double r2, int32_t *m_out_host,
                           int32_t *n_out_host, int64_t cap); /* packed order; returns count */
const char *fcfs_status_string(fcfs_status s);
const char *fcfs_last_error(void);                        /* thread-local detail string */
fcfs_status fcfs_device_check(void);                      /* FCFS_OK iff current device is sm_100 */
int32_t fcfs_kernel_launches(void);                       /* kernels launched by this thread so far */

/* Stage timing for the bench (CUDA events recorded on the caller's stream around each stage
 * while enabled).  Stages: 0 = a1 extraction, 1 = a2+a3 contraction, 2 = a4+a5 epilogue,
 * 3 = the edge pairing pre-pass of the batched split-TF32 contraction.
 * fcfs_profile_read synchronises the recorded events, writes the summed milliseconds and the
 * number of recorded launches per stage (n_stages <= 4; stages >= n_stages are dropped), and
 * clears the record. */
fcfs_status fcfs_profile_enable(int32_t on);
fcfs_status fcfs_profile_read(double *ms_host, int64_t *count_host, int32_t n_stages);

#ifdef __cplusplus
}
#endif
#endif /* FCFS_H_ */

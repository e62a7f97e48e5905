/*
 * fcfs_oracle.c — plain, slow, obviously-correct CPU oracle for the FCFS hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_1010_5562_b200/,
 * include/, csrc) may include, link or call this file.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * use it.  It shares no code, header, table or constant with the CUDA path.
 *
 * What it computes (citations are PAPER.md line numbers, "P:n"):
 *
 *   f(x,y) = sum over polygon groups g of 1[ union of the rects in g ]        (Eq. signal_model;
 *                                                                              reading A5 of DESIGN.md)
 *   F[m,n] = (1/T^2) * integral_[0,T)^2 f(x,y) exp(-2 pi i (m x + n y)/T)     (Eq. fourier_basis;
 *                                                                              normalisation reading A1)
 *
 *   evaluated with the closed forms of Proposition 3, written
 *   over the signed corner list (x_k, y_k, w_k) of f (Alg. 2 lines 9-10):
 *
 *     F[0,0] = area / T^2,  area = sum_k w_k x_k y_k                          (Eq. Fdc; Step 1 P:866-868)
 *     F[m,0] = i/(2 pi m T) * sum_k w_k y_k e^{-2 pi i m x_k / T}             (Eq. Fk0, alpha case 2)
 *     F[0,n] = i/(2 pi n T) * sum_k w_k x_k e^{-2 pi i n y_k / T}             (Eq. F0l, alpha case 3)
 *     F[m,n] = -1/(4 pi^2 m n) * sum_k w_k e^{-2 pi i (m x_k + n y_k) / T}    (Eq. Fkl, alpha case 4)
 *
 *   The exponent is reduced exactly in integers, (m x + n y) mod T, because the
 *   vertices lie on the integer lattice, and looked up in a
 *   long-double table of e^{-2 pi i r / T}.  Each sum is a Neumaier-compensated
 *   long-double sum in corner order, directly at the requested signed (m, n):
 *   no symmetry, no blocking, no FFT (this is the paper's "Goertzel-like" direct
 *   evaluation).
 *
 *   The per-coefficient L1 bound B[m,n] = sum_k |term_k| (BASELINE.json north_star)
 *   is returned alongside.  For F[0,0] B = 0: the DC must be exact.
 *
 * Vertex extraction (Alg. 2 lines 1-14; Prop. 1; half-open
 * convention P:398-402): per group, coordinate-compress the group's
 * rect edges, mark covered compressed cells, take the mixed difference
 *   w(x,y) = c(x,y) - c(x-1,y) - c(x,y-1) + c(x-1,y-1)
 * of the cell indicator c, then sum over groups, sort by (clip, y, x), merge
 * equal keys and drop zeros.  The area is computed twice (sum w x y and sum of
 * covered compressed-cell areas) and the two must agree.
 *
 * Haar (oracle_haar): the continuous Haar transform from child-cell areas of the corner form.
 * Chopping (oracle_chop_rects): every rect intersected with every T x T tile it overlaps, pieces in
 * tile-local coordinates, ordered by tile then rect.
 * Polygon vertex lists (oracle_extract_polygons): Alg. 2 lines 9-10 on every horizontal edge of
 * the clockwise list (+1 end, -1 start), counter-clockwise lists reversed, polygons summed.
 *
 * Parity is pinned in tests/test_oracle_pins.py (P1..P12, E1..E10 and H1..H4 of DESIGN.md).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_E_INVALID 1
#define OR_E_RANGE 2
#define OR_E_CAPACITY 3
#define OR_E_SELFCHECK 7
#define OR_E_NOMEM 8

typedef struct {
    int64_t clip;
    int64_t y;
    int64_t x;
    int64_t w;
} or_corner;

static int cmp_i64(const void *a, const void *b) {
    int64_t u = *(const int64_t *)a, v = *(const int64_t *)b;
    return (u > v) - (u < v);
}

static int cmp_corner(const void *a, const void *b) {
    const or_corner *p = (const or_corner *)a, *q = (const or_corner *)b;
    if (p->clip != q->clip) return (p->clip > q->clip) - (p->clip < q->clip);
    if (p->y != q->y) return (p->y > q->y) - (p->y < q->y);
    return (p->x > q->x) - (p->x < q->x);
}

/* sort + unique, returns the new length */
static int64_t sort_unique(int64_t *v, int64_t n) {
    qsort(v, (size_t)n, sizeof(int64_t), cmp_i64);
    int64_t u = 0;
    for (int64_t i = 0; i < n; ++i)
        if (u == 0 || v[u - 1] != v[i]) v[u++] = v[i];
    return u;
}

static int64_t find_idx(const int64_t *v, int64_t n, int64_t key) {
    int64_t lo = 0, hi = n - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (v[mid] == key) return mid;
        if (v[mid] < key) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/*
 * Extraction.  rects: int32[R][4] = (x0, y0, x1, y1), half-open, 0<=x0<x1<=T, 0<=y0<y1<=T.
 * group_ptr: int64[G+1] CSR over rects, or NULL => every rect is its own group (G == R).
 * clip_ptr:  int64[B+1] CSR over groups, or NULL => one clip (B == 1).
 * Outputs: x, y, w (capacity cap), corner_ptr int64[B+1], area int64[B], *K_out.
 */
int oracle_extract(const int32_t *rects, int64_t R, const int64_t *group_ptr, int64_t G,
                   const int64_t *clip_ptr, int64_t B, int32_t T,
                   int32_t *x, int32_t *y, int32_t *w, int64_t cap,
                   int64_t *corner_ptr, int64_t *area, int64_t *K_out) {
    if (T <= 0 || R < 0 || B < 1 || K_out == NULL || corner_ptr == NULL || area == NULL) return OR_E_INVALID;
    if (group_ptr == NULL && G != R) return OR_E_INVALID;
    if (clip_ptr == NULL && B != 1) return OR_E_INVALID;
    for (int64_t r = 0; r < R; ++r) {
        const int32_t *q = rects + 4 * r;
        if (q[0] < 0 || q[1] < 0 || q[2] > T || q[3] > T || q[0] >= q[2] || q[1] >= q[3]) return OR_E_RANGE;
    }
    /* pass 1: count candidate corners to size the buffer */
    int64_t ncand = 0;
    for (int64_t g = 0; g < G; ++g) {
        int64_t r0 = group_ptr ? group_ptr[g] : g, r1 = group_ptr ? group_ptr[g + 1] : g + 1;
        if (r0 < 0 || r1 < r0 || r1 > R) return OR_E_INVALID;
        int64_t n = 2 * (r1 - r0);
        ncand += n * n;
    }
    or_corner *cand = (or_corner *)malloc(sizeof(or_corner) * (size_t)(ncand > 0 ? ncand : 1));
    __int128 *area_cells = (__int128 *)calloc((size_t)B, sizeof(__int128));
    if (!cand || !area_cells) { free(cand); free(area_cells); return OR_E_NOMEM; }
    int64_t nc = 0;
    for (int64_t b = 0; b < B; ++b) {
        int64_t g0 = clip_ptr ? clip_ptr[b] : 0, g1 = clip_ptr ? clip_ptr[b + 1] : G;
        if (g0 < 0 || g1 < g0 || g1 > G) { free(cand); free(area_cells); return OR_E_INVALID; }
        for (int64_t g = g0; g < g1; ++g) {
            int64_t r0 = group_ptr ? group_ptr[g] : g, r1 = group_ptr ? group_ptr[g + 1] : g + 1;
            int64_t n = r1 - r0;
            if (n == 0) continue;
            int64_t *xs = (int64_t *)malloc(sizeof(int64_t) * 2 * n);
            int64_t *ys = (int64_t *)malloc(sizeof(int64_t) * 2 * n);
            for (int64_t i = 0; i < n; ++i) {
                const int32_t *q = rects + 4 * (r0 + i);
                xs[2 * i] = q[0]; xs[2 * i + 1] = q[2];
                ys[2 * i] = q[1]; ys[2 * i + 1] = q[3];
            }
            int64_t nx = sort_unique(xs, 2 * n), ny = sort_unique(ys, 2 * n);
            /* cell (i,j) = [xs[i],xs[i+1]) x [ys[j],ys[j+1]),  i < nx-1, j < ny-1 */
            unsigned char *cov = (unsigned char *)calloc((size_t)(nx * ny), 1);
            for (int64_t t = 0; t < n; ++t) {
                const int32_t *q = rects + 4 * (r0 + t);
                int64_t i0 = find_idx(xs, nx, q[0]), i1 = find_idx(xs, nx, q[2]);
                int64_t j0 = find_idx(ys, ny, q[1]), j1 = find_idx(ys, ny, q[3]);
                for (int64_t i = i0; i < i1; ++i)
                    for (int64_t j = j0; j < j1; ++j) cov[i * ny + j] = 1;
            }
            for (int64_t i = 0; i + 1 < nx; ++i)
                for (int64_t j = 0; j + 1 < ny; ++j)
                    if (cov[i * ny + j]) area_cells[b] += (__int128)(xs[i + 1] - xs[i]) * (ys[j + 1] - ys[j]);
            /* mixed difference at every grid point (i, j), 0<=i<nx, 0<=j<ny */
            for (int64_t i = 0; i < nx; ++i)
                for (int64_t j = 0; j < ny; ++j) {
                    int c00 = (i < nx - 1 && j < ny - 1) ? cov[i * ny + j] : 0;
                    int cm0 = (i > 0 && j < ny - 1) ? cov[(i - 1) * ny + j] : 0;
                    int c0m = (i < nx - 1 && j > 0) ? cov[i * ny + j - 1] : 0;
                    int cmm = (i > 0 && j > 0) ? cov[(i - 1) * ny + j - 1] : 0;
                    int wv = c00 - cm0 - c0m + cmm;
                    if (wv != 0) {
                        cand[nc].clip = b; cand[nc].y = ys[j]; cand[nc].x = xs[i]; cand[nc].w = wv;
                        ++nc;
                    }
                }
            free(cov); free(xs); free(ys);
        }
    }
    qsort(cand, (size_t)nc, sizeof(or_corner), cmp_corner);
    /* merge equal keys (sum across groups), drop zeros */
    int64_t K = 0;
    for (int64_t b = 0; b <= B; ++b) corner_ptr[b] = 0;
    for (int64_t b = 0; b < B; ++b) area[b] = 0;
    __int128 *area_w = (__int128 *)calloc((size_t)B, sizeof(__int128));
    int64_t i = 0;
    while (i < nc) {
        int64_t j = i, s = 0;
        while (j < nc && cand[j].clip == cand[i].clip && cand[j].y == cand[i].y && cand[j].x == cand[i].x) s += cand[j++].w;
        if (s != 0) {
            if (K < cap && x && y && w) {
                x[K] = (int32_t)cand[i].x; y[K] = (int32_t)cand[i].y; w[K] = (int32_t)s;
            }
            corner_ptr[cand[i].clip + 1] += 1;
            area_w[cand[i].clip] += (__int128)s * cand[i].x * cand[i].y;
            ++K;
        }
        i = j;
    }
    for (int64_t b = 0; b < B; ++b) corner_ptr[b + 1] += corner_ptr[b];
    int rc = OR_OK;
    for (int64_t b = 0; b < B; ++b) {
        if (area_w[b] != area_cells[b]) rc = OR_E_SELFCHECK; /* the two area computations must agree */
        area[b] = (int64_t)area_w[b];
    }
    *K_out = K;
    free(cand); free(area_cells); free(area_w);
    if (rc != OR_OK) return rc;
    return K > cap ? OR_E_CAPACITY : OR_OK;
}

/*
 * Extraction from polygon vertex lists (the paper's own input, Alg. 2 REQUIRE and lines 1-14,
 * P:930-950).  vx, vy: int32[V] vertices; poly_ptr: int64[P+1] CSR over vertices; every polygon is
 * closed (edge i runs from vertex i to vertex (i+1) mod n); clip_ptr: int64[B+1] CSR over polygons
 * or NULL (one clip).  Every edge is horizontal or vertical with non-zero length (else
 * OR_E_INVALID) and every vertex lies in [0,T]^2 (else OR_E_RANGE).
 *
 * Step by step, per polygon:
 *   1. orientation: A = sum over horizontal edges a->b of y_a (x_b - x_a) (the vertex form of
 *      Eq. Fdc) is the area, > 0 for a clockwise (y up) list ("which we
 *      arbitrarily choose to be clockwise").  A list with A < 0 is the counter-clockwise list of
 *      the same polygon: it is REVERSED first (reading A17 of DESIGN.md);
 *   2. Alg. 2 lines 9-10 / Step 4: every horizontal edge a->b of the
 *      clockwise list puts +1 at its end (x_b, y_a) and -1 at its start (x_a, y_a).  The loop runs
 *      over EVERY edge and tests it, so lists need not start with a horizontal edge and may hold
 *      collinear vertices (their +1 / -1 cancel);
 * then the entries of all polygons of a clip are SUMMED (the signal model f = sum of indicator
 * functions), sorted by (clip, y, x), equal keys merged, zeros dropped.
 * Self-check: sum_k w_k x_k y_k == sum over the clip's polygons of |A| (exact, __int128).
 */
int oracle_extract_polygons(const int32_t *vx, const int32_t *vy, const int64_t *poly_ptr, int64_t P,
                            const int64_t *clip_ptr, int64_t B, int32_t T,
                            int32_t *x, int32_t *y, int32_t *w, int64_t cap,
                            int64_t *corner_ptr, int64_t *area, int64_t *K_out) {
    if (T <= 0 || P < 0 || B < 1 || poly_ptr == NULL || K_out == NULL || corner_ptr == NULL || area == NULL)
        return OR_E_INVALID;
    if (clip_ptr == NULL && B != 1) return OR_E_INVALID;
    const int64_t V = poly_ptr[P];
    if (poly_ptr[0] != 0) return OR_E_INVALID;
    for (int64_t p = 0; p < P; ++p)
        if (poly_ptr[p + 1] < poly_ptr[p]) return OR_E_INVALID;
    for (int64_t v = 0; v < V; ++v)
        if (vx[v] < 0 || vy[v] < 0 || vx[v] > T || vy[v] > T) return OR_E_RANGE;
    or_corner *cand = (or_corner *)malloc(sizeof(or_corner) * (size_t)(2 * V > 0 ? 2 * V : 1));
    __int128 *area_poly = (__int128 *)calloc((size_t)B, sizeof(__int128));
    int64_t *px = (int64_t *)malloc(sizeof(int64_t) * (size_t)(V > 0 ? V : 1));
    int64_t *py = (int64_t *)malloc(sizeof(int64_t) * (size_t)(V > 0 ? V : 1));
    if (!cand || !area_poly || !px || !py) { free(cand); free(area_poly); free(px); free(py); return OR_E_NOMEM; }
    int64_t nc = 0;
    int rc = OR_OK;
    for (int64_t b = 0; b < B && rc == OR_OK; ++b) {
        int64_t p0 = clip_ptr ? clip_ptr[b] : 0, p1 = clip_ptr ? clip_ptr[b + 1] : P;
        if (p0 < 0 || p1 < p0 || p1 > P) { rc = OR_E_INVALID; break; }
        for (int64_t p = p0; p < p1; ++p) {
            const int64_t v0 = poly_ptr[p], n = poly_ptr[p + 1] - v0;
            if (n == 0) continue;
            for (int64_t i = 0; i < n; ++i) { px[i] = vx[v0 + i]; py[i] = vy[v0 + i]; }
            /* edges: horizontal or vertical, non-zero */
            for (int64_t i = 0; i < n; ++i) {
                const int64_t j = (i + 1) % n;
                const int hor = py[i] == py[j] && px[i] != px[j];
                const int ver = px[i] == px[j] && py[i] != py[j];
                if (!hor && !ver) rc = OR_E_INVALID;
            }
            if (rc != OR_OK) break;
            /* 1. orientation */
            __int128 A = 0;
            for (int64_t i = 0; i < n; ++i) {
                const int64_t j = (i + 1) % n;
                if (py[i] == py[j]) A += (__int128)py[i] * (px[j] - px[i]);
            }
            if (A < 0) {   /* counter-clockwise: reverse the list */
                for (int64_t i = 0, j = n - 1; i < j; ++i, --j) {
                    int64_t t = px[i]; px[i] = px[j]; px[j] = t;
                    t = py[i]; py[i] = py[j]; py[j] = t;
                }
                A = -A;
            }
            area_poly[b] += A;
            /* 2. +1 at the end, -1 at the start of every horizontal edge */
            for (int64_t i = 0; i < n; ++i) {
                const int64_t j = (i + 1) % n;
                if (py[i] != py[j]) continue;
                cand[nc].clip = b; cand[nc].y = py[i]; cand[nc].x = px[j]; cand[nc].w = +1; ++nc;
                cand[nc].clip = b; cand[nc].y = py[i]; cand[nc].x = px[i]; cand[nc].w = -1; ++nc;
            }
        }
    }
    free(px); free(py);
    if (rc != OR_OK) { free(cand); free(area_poly); return rc; }
    qsort(cand, (size_t)nc, sizeof(or_corner), cmp_corner);
    int64_t K = 0;
    for (int64_t b = 0; b <= B; ++b) corner_ptr[b] = 0;
    __int128 *area_w = (__int128 *)calloc((size_t)B, sizeof(__int128));
    int64_t i = 0;
    while (i < nc) {
        int64_t j = i, s = 0;
        while (j < nc && cand[j].clip == cand[i].clip && cand[j].y == cand[i].y && cand[j].x == cand[i].x) s += cand[j++].w;
        if (s != 0) {
            if (K < cap && x && y && w) {
                x[K] = (int32_t)cand[i].x; y[K] = (int32_t)cand[i].y; w[K] = (int32_t)s;
            }
            corner_ptr[cand[i].clip + 1] += 1;
            area_w[cand[i].clip] += (__int128)s * cand[i].x * cand[i].y;
            ++K;
        }
        i = j;
    }
    for (int64_t b = 0; b < B; ++b) corner_ptr[b + 1] += corner_ptr[b];
    for (int64_t b = 0; b < B; ++b) {
        if (area_w[b] != area_poly[b]) rc = OR_E_SELFCHECK;
        area[b] = (int64_t)area_w[b];
    }
    *K_out = K;
    free(cand); free(area_poly); free(area_w);
    if (rc != OR_OK) return rc;
    return K > cap ? OR_E_CAPACITY : OR_OK;
}

/*
 * Chopping a layout into tiles (the paper's flow: "chops polygons and places them in their
 * corresponding tiles. Each tile is then transformed individually").  rects: int32[R][4]
 * (x0, y0, x1, y1) half-open in layout coordinates, 0 <= x0 < x1 <= tiles_x T, 0 <= y0 < y1 <= tiles_y T.
 * Tile (tx, ty) = [tx T, (tx+1) T) x [ty T, (ty+1) T), index ty * tiles_x + tx (row-major).  Every
 * rect is intersected with every tile it overlaps; each non-empty piece is emitted in the tile's
 * local coordinates (0 <= x0 < x1 <= T).  Pieces are ordered by tile, and by rect index within a
 * tile.  out: int32[cap][4]; tile_ptr: int64[tiles+1]; *n_out = number of pieces.
 */
int oracle_chop_rects(const int32_t *rects, int64_t R, int32_t T, int32_t tiles_x, int32_t tiles_y,
                      int32_t *out, int64_t cap, int64_t *tile_ptr, int64_t *n_out) {
    if (T <= 0 || tiles_x <= 0 || tiles_y <= 0 || R < 0 || tile_ptr == NULL || n_out == NULL) return OR_E_INVALID;
    const int64_t W = (int64_t)tiles_x * T, H = (int64_t)tiles_y * T, nt = (int64_t)tiles_x * tiles_y;
    for (int64_t r = 0; r < R; ++r) {
        const int32_t *q = rects + 4 * r;
        if (q[0] < 0 || q[1] < 0 || q[2] > W || q[3] > H || q[0] >= q[2] || q[1] >= q[3]) return OR_E_RANGE;
    }
    for (int64_t t = 0; t <= nt; ++t) tile_ptr[t] = 0;
    /* pass 1: pieces per tile */
    for (int64_t r = 0; r < R; ++r) {
        const int32_t *q = rects + 4 * r;
        for (int64_t ty = q[1] / T; ty * T < q[3]; ++ty)
            for (int64_t tx = q[0] / T; tx * T < q[2]; ++tx) tile_ptr[ty * tiles_x + tx + 1] += 1;
    }
    for (int64_t t = 0; t < nt; ++t) tile_ptr[t + 1] += tile_ptr[t];
    *n_out = tile_ptr[nt];
    if (out == NULL || cap < tile_ptr[nt]) return tile_ptr[nt] > cap ? OR_E_CAPACITY : OR_OK;
    /* pass 2: emit in rect order into each tile's slots */
    int64_t *fill = (int64_t *)calloc((size_t)nt, sizeof(int64_t));
    if (!fill) return OR_E_NOMEM;
    for (int64_t r = 0; r < R; ++r) {
        const int32_t *q = rects + 4 * r;
        for (int64_t ty = q[1] / T; ty * T < q[3]; ++ty)
            for (int64_t tx = q[0] / T; tx * T < q[2]; ++tx) {
                const int64_t t = ty * tiles_x + tx, o = tile_ptr[t] + fill[t]++;
                const int64_t ax = tx * T, ay = ty * T;
                out[4 * o + 0] = (int32_t)((q[0] > ax ? q[0] : ax) - ax);
                out[4 * o + 1] = (int32_t)((q[1] > ay ? q[1] : ay) - ay);
                out[4 * o + 2] = (int32_t)((q[2] < ax + T ? q[2] : ax + T) - ax);
                out[4 * o + 3] = (int32_t)((q[3] < ay + T ? q[3] : ay + T) - ay);
            }
    }
    free(fill);
    return OR_OK;
}

/*
 * Continuous Haar transform of one clip (NEXT-4; the paper's CHT, Lemma polyip P:633-642,
 * IntersectionArea Alg. 1): the dyadic 2D (nonstandard) Haar basis over [0,T)^2, T = 2^J,
 *   phi_{j,kx,ky} = (2^j / T) 1[cell_{j,kx,ky}],  cell side T / 2^j,
 *   psi^{(ab)}_{j,kx,ky} = sum_{n,m} a_n b_m phi_{j+1, 2kx+n, 2ky+m},  g = (1, 1)/sqrt2, h = (1, -1)/sqrt2,
 * (n indexes x, m indexes y).  Coefficients are inner products with f = sum_k w_k H(x - x_k) H(y - y_k):
 *   X_{0,0,0} = area(f) / T,
 *   C^{(ab)}_{j,kx,ky} = (2^j / T) sum_{n,m} s^a_n s^b_m A_{j+1, 2kx+n, 2ky+m},  s^g = (1, 1), s^h = (1, -1),
 * with A = the integral of f over a child cell, computed from the corners (the corner form of the
 * intersection area of Alg. 1): A([a1,a2) x [b1,b2)) = sum_k w_k clamp(a2 - max(a1, x_k)) clamp(b2 - max(b1, y_k)).
 * Areas are exact integers (int64 / __int128); each coefficient is an integer times a power of two.
 * Output layout (reading A18): out[r * T + c], r = y-index, c = x-index: (0,0) = X_{0,0,0}; level j:
 * hg at (ky, 2^j + kx), gh at (2^j + ky, kx), hh at (2^j + ky, 2^j + kx).
 */
static __int128 or_area(const int32_t *x, const int32_t *y, const int32_t *w, int64_t K,
                        int64_t a1, int64_t a2, int64_t b1, int64_t b2) {
    __int128 s = 0;
    for (int64_t k = 0; k < K; ++k) {
        int64_t lx = a2 - (x[k] > a1 ? x[k] : a1), ly = b2 - (y[k] > b1 ? y[k] : b1);
        if (lx <= 0 || ly <= 0) continue;
        s += (__int128)w[k] * lx * ly;
    }
    return s;
}

int oracle_haar(const int32_t *x, const int32_t *y, const int32_t *w, int64_t K, int32_t T, double *out) {
    if (T < 2 || (T & (T - 1)) != 0 || out == NULL) return OR_E_INVALID;
    int J = 0;
    while ((1 << J) < T) ++J;
    out[0] = (double)or_area(x, y, w, K, 0, T, 0, T) / (double)T;
    for (int j = 0; j < J; ++j) {
        const int64_t n = (int64_t)1 << j, s = T >> j, h = s / 2;
        const double scale = (double)n / (double)T;
        for (int64_t ky = 0; ky < n; ++ky)
            for (int64_t kx = 0; kx < n; ++kx) {
                const int64_t a1 = kx * s, b1 = ky * s;
                __int128 A[2][2];   /* A[n][m]: child 2kx+n (x), 2ky+m (y) */
                for (int i = 0; i < 2; ++i)
                    for (int l = 0; l < 2; ++l)
                        A[i][l] = or_area(x, y, w, K, a1 + i * h, a1 + (i + 1) * h, b1 + l * h, b1 + (l + 1) * h);
                const __int128 hg = A[0][0] + A[0][1] - A[1][0] - A[1][1];
                const __int128 gh = A[0][0] - A[0][1] + A[1][0] - A[1][1];
                const __int128 hh = A[0][0] - A[0][1] - A[1][0] + A[1][1];
                out[ky * T + (n + kx)] = (double)hg * scale;
                out[(n + ky) * T + kx] = (double)gh * scale;
                out[(n + ky) * T + (n + kx)] = (double)hh * scale;
            }
    }
    return OR_OK;
}

/* Neumaier compensated accumulator */
typedef struct { long double s, c; } or_acc;
static inline void acc_add(or_acc *a, long double v) {
    long double t = a->s + v;
    if (fabsl(a->s) >= fabsl(v)) a->c += (a->s - t) + v; else a->c += (v - t) + a->s;
    a->s = t;
}
static inline long double acc_get(const or_acc *a) { return a->s + a->c; }

static inline int64_t pmod(int64_t a, int64_t T) { int64_t r = a % T; return r < 0 ? r + T : r; }

/*
 * Coefficients at an explicit list of signed (m, n).  Corners (x, y, w) of ONE clip.
 * F_re/F_im/Bnd: double[n_out].  nthreads <= 0 => OpenMP default.
 */
int oracle_coeffs(const int32_t *x, const int32_t *y, const int32_t *w, int64_t K, int64_t area,
                  int32_t T, const int32_t *ms, const int32_t *ns, int64_t n_out,
                  double *F_re, double *F_im, double *Bnd, int nthreads) {
    if (T <= 0 || K < 0 || n_out < 0) return OR_E_INVALID;
    if (n_out == 0) return OR_OK;
    if (!ms || !ns || !F_re || !F_im || !Bnd || (K > 0 && (!x || !y || !w))) return OR_E_INVALID;
    /* e^{-2 pi i r / T} for r in [0, T) */
    long double *tc = (long double *)malloc(sizeof(long double) * (size_t)T);
    long double *ts = (long double *)malloc(sizeof(long double) * (size_t)T);
    if (!tc || !ts) { free(tc); free(ts); return OR_E_NOMEM; }
    const long double two_pi = 2.0L * 3.141592653589793238462643383279502884L;
    for (int64_t r = 0; r < T; ++r) {
        long double th = two_pi * (long double)r / (long double)T;
        tc[r] = cosl(th);
        ts[r] = -sinl(th);
    }
    const long double pi = 3.141592653589793238462643383279502884L;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 4)
#endif
    for (int64_t o = 0; o < n_out; ++o) {
        int64_t m = ms[o], n = ns[o];
        or_acc re = {0, 0}, im = {0, 0};
        long double l1 = 0;
        if (m == 0 && n == 0) {
            F_re[o] = (double)area / ((double)T * (double)T);
            F_im[o] = 0.0;
            Bnd[o] = 0.0;
            continue;
        } else if (n == 0) {
            for (int64_t k = 0; k < K; ++k) {
                int64_t r = pmod(m * (int64_t)x[k], T);
                long double a = (long double)w[k] * (long double)y[k];
                acc_add(&re, a * tc[r]);
                acc_add(&im, a * ts[r]);
                l1 += fabsl(a);
            }
            /* i/(2 pi m T) * (re + i im) = (-im + i re) / (2 pi m T) */
            long double d = 2.0L * pi * (long double)m * (long double)T;
            F_re[o] = (double)(-acc_get(&im) / d);
            F_im[o] = (double)(acc_get(&re) / d);
            Bnd[o] = (double)(l1 / fabsl(d));
        } else if (m == 0) {
            for (int64_t k = 0; k < K; ++k) {
                int64_t r = pmod(n * (int64_t)y[k], T);
                long double a = (long double)w[k] * (long double)x[k];
                acc_add(&re, a * tc[r]);
                acc_add(&im, a * ts[r]);
                l1 += fabsl(a);
            }
            long double d = 2.0L * pi * (long double)n * (long double)T;
            F_re[o] = (double)(-acc_get(&im) / d);
            F_im[o] = (double)(acc_get(&re) / d);
            Bnd[o] = (double)(l1 / fabsl(d));
        } else {
            for (int64_t k = 0; k < K; ++k) {
                int64_t r = pmod(m * (int64_t)x[k] + n * (int64_t)y[k], T);
                long double a = (long double)w[k];
                acc_add(&re, a * tc[r]);
                acc_add(&im, a * ts[r]);
                l1 += fabsl(a);
            }
            long double d = -4.0L * pi * pi * (long double)m * (long double)n;
            F_re[o] = (double)(acc_get(&re) / d);
            F_im[o] = (double)(acc_get(&im) / d);
            Bnd[o] = (double)(l1 / fabsl(d));
        }
    }
    free(tc); free(ts);
    return OR_OK;
}

/*
 * Output index sets.  Dense centred window: (m, n) for m = -M..M (outer), n = -N..N (inner),
 * i.e. index (m+M)*(2N+1) + (n+N).  Pupil: the same order restricted to m^2 + n^2 <= r2
 * (inclusive; reading A11).  Returns the count; writes at most cap entries.
 */
int64_t oracle_window(int32_t M, int32_t N, double r2, int32_t *ms, int32_t *ns, int64_t cap) {
    int64_t c = 0;
    for (int64_t m = -M; m <= M; ++m)
        for (int64_t n = -N; n <= N; ++n) {
            if (r2 >= 0 && (double)(m * m + n * n) > r2) continue;
            if (c < cap && ms && ns) { ms[c] = (int32_t)m; ns[c] = (int32_t)n; }
            ++c;
        }
    return c;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

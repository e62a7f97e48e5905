/* fcfs_c_demo.c — the C-ABI used from plain C (no Python, no torch): one clip of rects in, its FP64
 * coefficient window out.
 *
 *   fcfs_c_demo <rects.bin> <R> <T> <M> <out.bin>
 *
 * rects.bin: R x 4 int32 (x0, y0, x1, y1), one union group (the c1 shape, BASELINE configs[0]);
 * out.bin:   (2M+1)^2 complex128 (re, im) in the DENSE layout, then int64 K and int64 area.
 * Build: gcc -O2 fcfs_c_demo.c -I include -L paper_1010_5562_b200 -lfcfs -L /usr/local/cuda/lib64 -lcudart
 *        -Wl,-rpath,<dirs>.  Exit code 0 on success; on a library error the status string and detail
 * are printed (fcfs_status_string / fcfs_last_error) and the exit code is 1. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "fcfs.h"

#define CK(call)                                                                                    \
    do {                                                                                            \
        fcfs_status st_ = (call);                                                                   \
        if (st_ != FCFS_OK) {                                                                       \
            fprintf(stderr, "%s: %s: %s\n", #call, fcfs_status_string(st_), fcfs_last_error());      \
            return 1;                                                                               \
        }                                                                                           \
    } while (0)
#define CU(call)                                                                                    \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess) {                                                                    \
            fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));                             \
            return 1;                                                                               \
        }                                                                                           \
    } while (0)

int main(int argc, char **argv) {
    if (argc != 6) {
        fprintf(stderr, "usage: %s rects.bin R T M out.bin\n", argv[0]);
        return 2;
    }
    const int64_t R = atoll(argv[2]);
    const int32_t T = atoi(argv[3]), M = atoi(argv[4]);
    int32_t *rects_h = (int32_t *)malloc((size_t)R * 16);
    FILE *f = fopen(argv[1], "rb");
    if (!f || fread(rects_h, 16, (size_t)R, f) != (size_t)R) { fprintf(stderr, "cannot read rects\n"); return 2; }
    fclose(f);
    CK(fcfs_device_check());

    /* a1: one union group of all R rects */
    int64_t gp_h[2] = {0, R};
    int32_t *rects, *x, *y, *w;
    int64_t *gp, *corner_ptr, *area;
    const int64_t cap = 16 * R + 16;
    CU(cudaMalloc((void **)&rects, (size_t)R * 16));
    CU(cudaMalloc((void **)&gp, sizeof gp_h));
    CU(cudaMalloc((void **)&x, (size_t)cap * 4));
    CU(cudaMalloc((void **)&y, (size_t)cap * 4));
    CU(cudaMalloc((void **)&w, (size_t)cap * 4));
    CU(cudaMalloc((void **)&corner_ptr, 2 * sizeof(int64_t)));
    CU(cudaMalloc((void **)&area, sizeof(int64_t)));
    CU(cudaMemcpy(rects, rects_h, (size_t)R * 16, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(gp, gp_h, sizeof gp_h, cudaMemcpyHostToDevice));
    size_t ws_bytes = fcfs_vertices_workspace_bytes(R, 1, 1, R);
    void *ws = NULL;
    CU(cudaMalloc(&ws, ws_bytes));
    int64_t K = 0;
    CK(fcfs_vertices_from_rects(rects, R, gp, 1, NULL, 1, T, R, x, y, w, cap, corner_ptr, area, &K, ws,
                                ws_bytes, NULL));
    int64_t area_h = 0;
    CU(cudaMemcpy(&area_h, area, sizeof area_h, cudaMemcpyDeviceToHost));

    /* a2-a5: the dense FP64 window |m|, |n| <= M */
    fcfs_window win = {M, M, -1.0, FCFS_LAYOUT_DENSE};
    fcfs_options opt = {FCFS_ROUTE_AUTO, FCFS_FORM_AUTO, 1, {0, 0, 0, 0, 0}};
    const int64_t nout = fcfs_window_size(&win);
    size_t cws = fcfs_coeffs_workspace_bytes(K, T, &win, FCFS_FP64, NULL, &opt);
    void *cw = NULL, *F = NULL;
    CU(cudaMalloc(&cw, cws));
    CU(cudaMalloc(&F, (size_t)nout * 16));
    CK(fcfs_coeffs(x, y, w, K, area_h, T, &win, FCFS_FP64, NULL, &opt, F, cw, cws, NULL));
    double *F_h = (double *)malloc((size_t)nout * 16);
    CU(cudaMemcpy(F_h, F, (size_t)nout * 16, cudaMemcpyDeviceToHost));

    FILE *o = fopen(argv[5], "wb");
    if (!o) { fprintf(stderr, "cannot write %s\n", argv[5]); return 2; }
    fwrite(F_h, 16, (size_t)nout, o);
    fwrite(&K, sizeof K, 1, o);
    fwrite(&area_h, sizeof area_h, 1, o);
    fclose(o);
    printf("K=%lld area=%lld F[0,0]=%.17g window=%lld kernels=%d\n", (long long)K, (long long)area_h,
           F_h[2 * ((int64_t)M * (2 * M + 1) + M)], (long long)nout, fcfs_kernel_launches());
    cudaFree(rects); cudaFree(gp); cudaFree(x); cudaFree(y); cudaFree(w); cudaFree(corner_ptr); cudaFree(area);
    cudaFree(ws); cudaFree(cw); cudaFree(F);
    free(rects_h); free(F_h);
    return 0;
}

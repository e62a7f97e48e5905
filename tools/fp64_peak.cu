// fp64_peak.cu — measure FP64 DFMA vs DMMA (mma.sync f64) throughput on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double *out, int iters) {
    double a[8], b = 1.0000001, c = 0.9999999;
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.0) out[0] = s;
}

__global__ void dmma884_loop(double *out, int iters) {
    double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
    double d[4][2];
    for (int i = 0; i < 4; ++i) { d[i][0] = 0; d[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void dmma16816_loop(double *out, int iters) {
    double a[8], b[4];
    for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-6 + i;
    for (int i = 0; i < 4; ++i) b[i] = 0.999 - i * 1e-3;
    double d[2][4];
    for (int i = 0; i < 2; ++i) for (int j = 0; j < 4; ++j) d[i][j] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 2; ++i)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                         : "+d"(d[i][0]), "+d"(d[i][1]), "+d"(d[i][2]), "+d"(d[i][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                           "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double s = 0;
    for (int i = 0; i < 2; ++i) for (int j = 0; j < 4; ++j) s += d[i][j];
    if (s == 12345.0) out[0] = s;
}

int main() {
    double *out;
    cudaMalloc(&out, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        // DFMA: blocks x threads x iters x 8 FMA x 2 flop
        int blocks = sms * 4, threads = 256;
        cudaEventRecord(a);
        dfma_loop<<<blocks, threads>>>(out, iters);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        double fl = (double)blocks * threads * iters * 8 * 2;
        printf("DFMA            %.2f TFLOP/s\n", fl / ms / 1e9);
        cudaEventRecord(a);
        dmma884_loop<<<blocks, threads>>>(out, iters);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        fl = (double)blocks * (threads / 32) * iters * 4 * (8 * 8 * 4) * 2;
        printf("DMMA m8n8k4     %.2f TFLOP/s\n", fl / ms / 1e9);
        cudaEventRecord(a);
        dmma16816_loop<<<blocks, threads>>>(out, iters);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        fl = (double)blocks * (threads / 32) * iters * 2 * (16 * 8 * 16) * 2;
        printf("DMMA m16n8k16   %.2f TFLOP/s  (err=%s)\n", fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

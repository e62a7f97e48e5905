// mio_probe.cu — throughput of the shared-memory / shuffle (MIO) instructions the lattice-row gather
// loop is built from (tools only).  One CTA of W warps per SM on all SMs; each warp runs a long unrolled
// stream of one instruction kind; reported: warp-instructions per clock per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mio_probe tools/mio_probe.cu
#include <cstdint>
#include <cstdio>

template <int KIND>
__global__ void __launch_bounds__(512, 1) probe(int iters, float *sink, long long *cyc) {
    extern __shared__ __align__(16) float sm[];
    const int t = threadIdx.x, lane = t & 31;
    for (int i = t; i < 16384; i += blockDim.x) sm[i] = (float)(i & 15);
    __syncthreads();
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    uint32_t r = lane;
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (KIND == 0) {          // LDS.32, conflict-free (lane-contiguous)
                a0 += sm[((it * 16 + j) * 32 + lane) & 16383];
            } else if (KIND == 1) {   // LDS.32 broadcast (uniform address)
                a0 += sm[(it * 16 + j) & 16383];
            } else if (KIND == 2) {   // LDS.128 broadcast
                const float4 v = ((const float4 *)sm)[(it * 16 + j) & 4095];
                a0 += v.x; a1 += v.y; a2 += v.z; a3 += v.w;
            } else if (KIND == 3) {   // SHFL.IDX with a uniform source lane
                r = __shfl_sync(0xffffffffu, r, j) + 1u;
            } else if (KIND == 4) {   // LDS.32 conflict-free + SHFL (the two together)
                a0 += sm[((it * 16 + j) * 32 + lane) & 16383];
                r = __shfl_sync(0xffffffffu, r, j) + 1u;
            } else if (KIND == 5) {   // LDS.32 conflict-free + LDS.128 broadcast
                a0 += sm[((it * 16 + j) * 32 + lane) & 16383];
                const float4 v = ((const float4 *)sm)[(it * 16 + j) & 4095];
                a1 += v.x + v.y;
            } else if (KIND == 6) {   // LDS.64 broadcast
                const float2 v = ((const float2 *)sm)[(it * 16 + j) & 8191];
                a0 += v.x; a1 += v.y;
            }
        }
    }
    const long long c1 = clock64();
    sink[blockIdx.x * blockDim.x + t] = a0 + a1 + a2 + a3 + (float)r;
    if (t == 0) cyc[blockIdx.x] = c1 - c0;
}

template <int KIND>
void run(const char *name, int warps, float *dS, long long *dC) {
    const int iters = 4096;
    cudaFuncSetAttribute(probe<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    probe<KIND><<<148, warps * 32, 65536>>>(iters, dS, dC);
    cudaDeviceSynchronize();
    long long c[148];
    cudaMemcpy(c, dC, sizeof(c), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    const double instr = (double)warps * iters * 16;
    printf("%-40s warps=%2d: %.3f warp-instr/clk/SM  (%.1f clk per instr per SMSP)\n", name, warps, instr / mx,
           mx / (instr / 4));
}

int main() {
    float *dS;
    long long *dC;
    cudaMalloc(&dS, 148 * 512 * 4);
    cudaMalloc(&dC, 148 * 8);
    for (int w : {8, 16}) {
        run<0>("LDS.32 conflict-free", w, dS, dC);
        run<1>("LDS.32 broadcast", w, dS, dC);
        run<2>("LDS.128 broadcast", w, dS, dC);
        run<6>("LDS.64 broadcast", w, dS, dC);
        run<3>("SHFL.IDX uniform lane", w, dS, dC);
        run<4>("LDS.32 + SHFL (pairs)", w, dS, dC);
        run<5>("LDS.32 + LDS.128 bcast (pairs)", w, dS, dC);
    }
    return 0;
}

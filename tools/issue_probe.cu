// issue_probe.cu — how fast can one warp issue tcgen05.mma (tools only)?  Cycles per MMA (tf32, K = 8)
// for M = 128 and N = 64 / 128 / 256, SS (both operands in SMEM) and TS (A in TMEM), with the issue
// loop in the form the kernels use: the whole warp runs a warp-uniform loop, one elected lane issues
// U MMAs per election, into NACC accumulators (compile-time round robin).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/issue_probe tools/issue_probe.cu
#include <cstdint>
#include <cstdio>

__device__ inline uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ inline uint64_t desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
           ((uint64_t)2 << 61);
}
__device__ inline bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n .reg .b32 rx;\n .reg .pred px;\n elect.sync rx|px, %1;\n @px mov.s32 %0, 1;\n}" : "+r"(pred) : "r"(0xffffffffu));
    return pred != 0;
}
template <int kTS>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint32_t at, uint64_t b, uint32_t id) {
    if constexpr (kTS)
        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(d), "r"(at), "l"(b), "r"(id));
    else
        asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b), "r"(id));
}

template <int kTS, int N, int U, int NACC>
__global__ void __launch_bounds__(128, 1) probe(int NIT, long long *cyc) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t *sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < (16384 + 32768) / 4; i += blockDim.x) ((float *)sm)[i] = 0.f;
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = desc_sw128(su32(sm)), db = desc_sw128(su32(sm + 16384));
    if (warp == 0) {
        const long long c0 = clock64();
        for (int it = 0; it < NIT; ++it) {
            if (elect_one()) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t d = tmem + 256 + (uint32_t)((u % NACC) * (256 / NACC));
                    mma<kTS>(d, da + 2 * (u & 3), tmem + 8 * (u & 3), db + 2 * (u & 3), id);
                }
            }
            __syncwarp();
        }
        if (elect_one())
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        __syncwarp();
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0,1,0,p;\n}"
                         : "=r"(ok) : "r"(su32(&bar)) : "memory");
        if (t == 0) cyc[0] = clock64() - c0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int kTS, int N, int U, int NACC>
void run(long long *dC) {
    auto k = probe<kTS, N, U, NACC>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
    const int NIT = 16384 / U;
    k<<<1, 128, 50 * 1024>>>(NIT, dC);
    cudaError_t e = cudaDeviceSynchronize();
    long long c = 0;
    cudaMemcpy(&c, dC, 8, cudaMemcpyDeviceToHost);
    printf("%s N=%3d U=%d NACC=%d: %s cyc/MMA %.2f (floor %.1f)\n", kTS ? "TS" : "SS", N, U, NACC,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e), (double)c / (NIT * U), 128.0 * N / 256.0);
}

int main() {
    long long *dC;
    cudaMalloc(&dC, 64);
    run<0, 128, 4, 1>(dC);
    run<0, 128, 8, 1>(dC);
    run<0, 128, 8, 2>(dC);
    run<0, 256, 8, 1>(dC);
    run<0, 64, 8, 1>(dC);
    run<0, 64, 8, 4>(dC);
    run<1, 64, 4, 1>(dC);
    run<1, 64, 8, 1>(dC);
    run<1, 64, 16, 1>(dC);
    run<1, 64, 16, 2>(dC);
    run<1, 64, 16, 4>(dC);
    run<1, 128, 16, 1>(dC);
    run<1, 128, 16, 2>(dC);
    run<1, 256, 16, 1>(dC);
    return 0;
}

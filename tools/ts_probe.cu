// ts_probe.cu — bring-up + rate probe for the lattice-row kernel's MMA shape (tools only).
//  (1) correctness: tcgen05.mma kind::tf32 with A in TMEM (TS form: A written by tcgen05.st.32x32b,
//      lane = row, column = K element), B in SMEM (SW128 K-major), M = 128, N = 64 / 128, vs the host.
//  (2) rate: cycles per MMA (K = 8 tf32) for SS and TS forms at N = 64 / 128, alone and while 4 other
//      warps stream conflict-free LDS.32 from shared memory (the gather's traffic), and the LDS rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ts_probe tools/ts_probe.cu
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <vector>

__device__ inline uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ inline uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__device__ inline uint32_t sw128_off(int r, int kbyte) {
    const int c = kbyte / 16, in = kbyte % 16;
    return (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) * 16) + in;
}
__device__ inline uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ inline void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                 ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ inline void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}"
                 ::"r"(d), "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ inline void commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ inline void wait_bar(uint32_t bar, uint32_t ph) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
                     : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
}

// KT = 32 tf32 (one SW128 row of K).  A: 128 x 32, B: N x 32.  mode 0: SS, 1: TS.
// Rate part: NIT repetitions of the 4 MMAs (accumulate), lds: warps 4..7 stream LDS.32 meanwhile.
__global__ void __launch_bounds__(256, 1) probe(const float *A, const float *B, float *D, int N, int mode, int NIT,
                                                int lds, long long *cyc, float *sink, int nacc) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t *sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
    uint8_t *sA = sm, *sB = sm + 16384, *sL = sm + 49152;   // sB: up to 256 rows; sL: 64 KB for the LDS stream
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    if (t < 128)
        for (int k = 0; k < 32; ++k) *(float *)(sA + sw128_off(t, k * 4)) = A[t * 32 + k];
    if (t < N)
        for (int k = 0; k < 32; ++k) *(float *)(sB + sw128_off(t, k * 4)) = B[t * 32 + k];
    for (int i = t; i < 65536 / 4; i += blockDim.x) ((float *)sL)[i] = (float)(i & 7);
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
    // A into TMEM columns [0, 32): warp w (w < 4) writes lanes 32 w .. 32 w + 31, thread = row
    if (warp < 4) {
        uint32_t r[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) r[k] = __float_as_uint(A[t * 32 + k]);
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                     "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
                     "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
                     "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
                     "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
                     "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t dcol = tmem + 256;
    const uint32_t id = idesc_tf32(128, N);
    const uint64_t da = desc_sw128(su32(sA)), db = desc_sw128(su32(sB));
    // correctness: one pass of 4 MMAs
    if (t == 0) {
        for (int u = 0; u < 4; ++u) {
            if (mode == 0) mma_ss(dcol, da + 2 * u, db + 2 * u, id, u > 0);
            else mma_ts(dcol, tmem + 8 * u, db + 2 * u, id, u > 0);
        }
        commit(su32(&bar));
    }
    wait_bar(su32(&bar), 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {
        for (int c = 0; c < N; ++c) {
            uint32_t r;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(dcol + ((uint32_t)(warp * 32) << 16) + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            D[t * 256 + c] = __uint_as_float(r);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // rate
    if (t == 0) {
        const long long c0 = clock64();
        // nacc independent accumulators (round robin per MMA) at columns 256 + (j % nacc) * (256 / nacc)
        const uint32_t step = 256u / (uint32_t)nacc;
        uint32_t j = 0;
        for (int it = 0; it < NIT; ++it)
            for (int u = 0; u < 4; ++u) {
                const uint32_t d = dcol + (j % (uint32_t)nacc) * step;
                ++j;
                if (mode == 0) mma_ss(d, da + 2 * u, db + 2 * u, id, 1);
                else mma_ts(d, tmem + 8 * u, db + 2 * u, id, 1);
            }
        commit(su32(&bar));
        wait_bar(su32(&bar), 1);
        cyc[0] = clock64() - c0;
    } else if (lds && warp >= 4) {
        const long long c0 = clock64();
        float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const float *p = (const float *)sL + lane;
        const int n = lds;   // LDS.32 per thread
        for (int i = 0; i < n; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) s[j] += p[((i + j) * 32 + warp * 96) & 16383];
        }
        sink[t] = s[0] + s[1] + s[2] + s[3] + s[4] + s[5] + s[6] + s[7];
        if (lane == 0) cyc[1 + warp - 4] = clock64() - c0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    std::vector<float> A(128 * 32), B(256 * 32);
    for (int r = 0; r < 256; ++r)
        for (int k = 0; k < 32; ++k) {
            if (r < 128) A[r * 32 + k] = (float)(((r * 8 + k * 5) * 7) % 13 - 6);
            B[r * 32 + k] = (float)(((r * 5 + k * 3) * 11) % 9 - 4);
        }
    float *dA, *dB, *dD, *dS;
    long long *dC;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, 128 * 256 * 4);
    cudaMalloc(&dC, 8 * 8); cudaMalloc(&dS, 256 * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    int fails = 0;
    for (int mode = 0; mode < 2; ++mode)
        for (int N : {64, 128, 256})
            for (int nacc : {1, 2, 4})
            for (int lds : {0, 65536}) {
                if (N * nacc > 256) continue;
                const int NIT = 4096;
                cudaMemset(dD, 0, 128 * 256 * 4);
                probe<<<1, 256, 120 * 1024>>>(dA, dB, dD, N, mode, NIT, lds, dC, dS, nacc);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("mode %d N %d: CUDA error %s\n", mode, N, cudaGetErrorString(e)); return 1; }
                std::vector<float> D(128 * 256);
                long long cyc[8];
                cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
                cudaMemcpy(cyc, dC, sizeof(cyc), cudaMemcpyDeviceToHost);
                int bad = 0;
                for (int i = 0; i < 128; ++i)
                    for (int j = 0; j < N; ++j) {
                        float s = 0;
                        for (int k = 0; k < 32; ++k) s += A[i * 32 + k] * B[j * 32 + k];
                        if (fabsf(D[i * 256 + j] - s) > 1e-3f) ++bad;
                    }
                fails += bad != 0;
                const double per = (double)cyc[0] / (4.0 * NIT);
                printf("%s N=%3d nacc=%d lds=%d: %s bad=%d  cyc/MMA(K=8) %.2f (floor 128*N/256 = %.1f)", mode ? "TS" : "SS",
                       N, nacc, lds ? 1 : 0, bad ? "FAIL" : "PASS", bad, per, 128.0 * N / 256.0);
                if (lds) printf("  LDS warp cycles %lld (%.2f B/clk/SM from 4 warps)", cyc[1],
                                4.0 * 32 * 4 * (double)lds / (double)cyc[1]);
                printf("\n");
            }
    return fails;
}

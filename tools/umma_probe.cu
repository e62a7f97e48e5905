// umma_probe.cu — bring-up harness for hand-written tcgen05 operand layouts.
// One CTA fills A (128 x KT) and B (128 x KT) with small integers in a candidate smem layout,
// issues KT/Kmma tcgen05.mma (M=128, N=128) with accumulation, reads D from TMEM and compares
// with A B^T on the host.  Variants: tf32 / f16, K-major no-swizzle / K-major SWIZZLE_128B.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tools/umma_probe tools/umma_probe.cu
#include <cuda_fp16.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

struct Variant {
    const char *name;
    int f16;        // 0: tf32 (4 B), 1: f16 (2 B)
    int swz128;     // 0: no swizzle (core matrices 8 rows x 16 B; chunks 2 KB apart), 1: SW128 K-major
};

constexpr int KT_BYTES = 128;   // bytes of K per row in the tile (one SW128 atom row)

__device__ __host__ inline uint32_t offset_of(const Variant &v, int r, int kbyte) {
    const int c = kbyte / 16, in = kbyte % 16;
    if (!v.swz128) return c * (16 * 128) + (r / 8) * 128 + (r % 8) * 16 + in;
    return (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) * 16) + in;
}

__device__ inline uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(Variant v, const float *A, const float *B, float *D) {
    __shared__ __align__(1024) uint8_t sA[128 * KT_BYTES];
    __shared__ __align__(1024) uint8_t sB[128 * KT_BYTES];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x;
    const int esz = v.f16 ? 2 : 4, KT = KT_BYTES / esz;
    for (int k = 0; k < KT; ++k) {
        uint32_t oa = offset_of(v, t, k * esz);
        if (v.f16) {
            *(__half *)(sA + oa) = __float2half(A[t * KT + k]);
            *(__half *)(sB + oa) = __float2half(B[t * KT + k]);
        } else {
            *(float *)(sA + oa) = A[t * KT + k];
            *(float *)(sB + oa) = B[t * KT + k];
        }
    }
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tmem = tslot;
    if (t == 0) {
        auto desc = [&](uint32_t saddr) {
            uint64_t d = 0;
            d |= (uint64_t)((saddr >> 4) & 0x3FFF);
            if (v.swz128) {
                d |= (uint64_t)1 << 16;                          // LBO unused for swizzled K-major
                d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;     // SBO: 8-row group stride
                d |= (uint64_t)2 << 61;                          // SWIZZLE_128B
            } else {
                d |= (uint64_t)(((16 * 128) >> 4) & 0x3FFF) << 16;
                d |= (uint64_t)((128 >> 4) & 0x3FFF) << 32;
            }
            d |= (uint64_t)1 << 46;
            return d;
        };
        const uint32_t fmt = v.f16 ? 0u : 2u;
        const uint32_t kind_k_bytes = 32;   // one MMA consumes 32 bytes of K
        uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
        for (int u = 0; u < KT_BYTES / 32; ++u) {
            uint32_t adv = v.swz128 ? u * kind_k_bytes : u * 2 * (16 * 128);
            uint64_t da = desc(su32(sA) + adv), db = desc(su32(sB) + adv);
            uint32_t acc = u > 0;
            if (v.f16)
                asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                             ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
            else
                asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                             ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    }
    {
        uint32_t ok = 0;
        while (!ok) {
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0,1,0,p;\n}"
                         : "=r"(ok) : "r"(su32(&bar)));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c = 0; c < 128; ++c) {
        uint32_t r;
        uint32_t addr = tmem + ((uint32_t)((t / 32) * 32) << 16) + c;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        D[t * 128 + c] = __uint_as_float(r);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
    Variant vs[] = {
        {"tf32 K-major no-swizzle", 0, 0},
        {"tf32 K-major SWIZZLE_128B", 0, 1},
        {"f16  K-major no-swizzle", 1, 0},
        {"f16  K-major SWIZZLE_128B", 1, 1},
    };
    int fails = 0;
    for (auto &v : vs) {
        const int KT = KT_BYTES / (v.f16 ? 2 : 4);
        std::vector<float> A(128 * KT), B(128 * KT), D(128 * 128), R(128 * 128);
        for (int r = 0; r < 128; ++r)
            for (int k = 0; k < KT; ++k) {
                A[r * KT + k] = (float)(((r * 8 + k * 5) * 7) % 13 - 6);
                B[r * KT + k] = (float)(((r * 5 + k * 3) * 11) % 9 - 4);
            }
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < 128; ++j) {
                float s = 0;
                for (int k = 0; k < KT; ++k) s += A[i * KT + k] * B[j * KT + k];
                R[i * 128 + j] = s;
            }
        float *dA, *dB, *dD;
        cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
        cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 128>>>(v, dA, dB, dD);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%-32s CUDA error %s\n", v.name, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double maxerr = 0;
        int bad = 0;
        for (int i = 0; i < 128 * 128; ++i) {
            double d = fabs(D[i] - R[i]);
            if (d > 1e-3) ++bad;
            maxerr = d > maxerr ? d : maxerr;
        }
        fails += bad != 0;
        printf("%-32s %s  bad=%d maxerr=%g  D[0..2]=%g %g %g ref=%g %g %g\n", v.name, bad ? "FAIL" : "PASS", bad,
               maxerr, D[0], D[1], D[2], R[0], R[1], R[2]);
        cudaFree(dA); cudaFree(dB); cudaFree(dD);
    }
    return fails;
}

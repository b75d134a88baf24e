// tcgen05 kind::i8 probe: one CTA computes C (128 x N, int32) = A (128 x K) * B (N x K)^T
// with int8 operands loaded by TMA (128-byte swizzle, K-major) and the accumulator in
// TMEM, then checks against a CPU product and times a persistent loop of MMAs.
// Validates the UMMA smem/instruction descriptor encodings used by csrc/gemm_i8.cu.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__);                   \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

constexpr int M = 128, N = 64, KTOT = 256, KB = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3fff);          // start address
    d |= (uint64_t)1 << 16;                           // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;                 // SBO: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                           // version (Blackwell)
    d |= (uint64_t)2 << 61;                           // SWIZZLE_128B
    return d;
}

__global__ void probe_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                             int* C, int reps) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = smem;                 // KTOT/KB stages of 128 x 128 B
    uint8_t* sB = smem + (KTOT / KB) * M * KB;
    __shared__ uint64_t bar_load, bar_mma;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_load)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_mma)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;

    if (threadIdx.x == 0) {
        const uint32_t bar = smem_u32(&bar_load);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((M + N) * KTOT));
        for (int s = 0; s < KTOT / KB; ++s) {
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(smem_u32(sA + s * M * KB)), "l"((uint64_t)&ma), "r"(s * KB), "r"(0), "r"(bar) : "memory");
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(smem_u32(sB + s * N * KB)), "l"((uint64_t)&mb), "r"(s * KB), "r"(0), "r"(bar) : "memory");
        }
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                         : "=r"(ok) : "r"(bar) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;");
        // idesc: c S32 (2 << 4), a s8 (1 << 7), b s8 (1 << 10), K-major both, N>>3 << 17, M>>4 << 24
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        for (int r = 0; r < reps; ++r) {
            for (int s = 0; s < KTOT / KB; ++s)
                for (int k = 0; k < KB / 32; ++k) {
                    const uint64_t da = sw128_kmajor_desc(smem_u32(sA + s * M * KB) + k * 32);
                    const uint64_t db = sw128_kmajor_desc(smem_u32(sB + s * N * KB) + k * 32);
                    const uint32_t acc = (r | s | k) ? 1u : 0u;
                    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar_mma)) : "memory");
    }
    __syncwarp();
    // all 4 warps wait for the MMAs, then read their 32 TMEM lanes
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                         : "=r"(ok) : "r"(smem_u32(&bar_mma)) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int row = warp * 32 + (threadIdx.x & 31);
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) C[row * N + c0 + j] = (int)v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main(int argc, char** argv) {
    // argv[1]: timed repetitions (default 20000); argv[2]: digit magnitude bound
    // (default 128 = full-entropy int8; smaller values probe data-dependent power)
    const int reps_arg = argc > 1 ? atoi(argv[1]) : 20000;
    const int mag = argc > 2 ? atoi(argv[2]) : 128;
    std::vector<int8_t> A(M * KTOT), B(N * KTOT);
    srand(1);
    for (auto& x : A) x = (int8_t)(rand() % (2 * mag) - mag);
    for (auto& x : B) x = (int8_t)(rand() % (2 * mag) - mag);
    int8_t *dA, *dB;
    int* dC;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, B.size()));
    CK(cudaMalloc(&dC, M * N * 4));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    CUtensorMap ma, mb;
    cuuint64_t dimsA[2] = {KTOT, M}, dimsB[2] = {KTOT, N}, str[1] = {KTOT};
    cuuint32_t boxA[2] = {KB, M}, boxB[2] = {KB, N}, es[2] = {1, 1};
    if (encode(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dA, dimsA, str, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
        encode(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, dB, dimsB, str, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
        printf("encode failed\n");
        return 1;
    }
    const int smem = (M + N) * KTOT + 1024;
    CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    probe_kernel<<<1, 128, smem>>>(ma, mb, dC, 1);
    CK(cudaDeviceSynchronize());
    std::vector<int> C(M * N);
    CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            long s = 0;
            for (int k = 0; k < KTOT; ++k) s += (long)A[i * KTOT + k] * B[j * KTOT + k];
            if (s != C[i * N + j]) {
                if (bad < 5) printf("mismatch (%d,%d): got %d want %ld\n", i, j, C[i * N + j], s);
                ++bad;
            }
        }
    printf("{\"probe\": \"tcgen05.mma.kind::i8 M=128 N=64 K=256\", \"mismatches\": %ld}\n", bad);
    // throughput: one CTA per SM, reps x 8 MMAs of 128x64x32
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = reps_arg;
    probe_kernel<<<sms, 128, smem>>>(ma, mb, dC, 10);
    cudaEventRecord(e0);
    probe_kernel<<<sms, 128, smem>>>(ma, mb, dC, reps);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * M * N * KTOT * (double)reps * sms;
    printf("{\"tcgen05_i8_tops_single_cta_N64\": %.1f}\n", ops / ms / 1e9);
    return bad != 0;
}

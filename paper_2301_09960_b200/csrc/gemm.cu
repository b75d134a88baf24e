// gemm.cu -- K2 + K3: slice-pair FP64 GEMMs on the DMMA tensor pipe with the
// K-word accumulation fused into the epilogue.
//
// Reference: the product loop and accumulation of ozaki_gemm<K>
// (proj/include/mpmat/ozaki.hpp:223-244) over the GemmBackend plugin
// (backend.hpp:12-13, reference_backend_gemm in proj/src/backend.cpp:55-103).
//
// Why the result is bit-identical to the reference: every slice product
// C_ab = A_a * B_b is exact in binary64 in ANY summation order (the split
// bounds slice significands by the inner dimension, ozaki.hpp:15-29), so the
// DMMA tree order is irrelevant; the epilogue then adds C_ab into the K-word
// accumulator with the reference's own MultiFloat<K> + double sequence
// (kword.cuh) in the reference's alpha-major pair order.
//
// B200 mapping
//  * FP64 tensor cores are reachable only through mma.sync (tcgen05 has no
//    kind::f64); m8n8k4.f64 lowers 1:1 to SASS DMMA.8x8x4.
//  * Persistent CTAs, one per SM: 8 warps (2 per SM sub-partition, so each
//    thread may hold up to 255 registers) own a 128x128 C tile as 2x4 warp
//    tiles of 64x32 (64 FP64 accumulators per thread).  128x16 A and B^T
//    tiles arrive by TMA (cp.async.bulk.tensor, 128-byte swizzle) in a
//    5-stage mbarrier ring; thread 0 re-arms a slot as soon as all eight
//    warps have released it (a dedicated 9th producer warp would put three
//    warps on one sub-partition and cap registers at 168, forcing spills).
//  * Each CTA walks tile -> pair -> k-block; the TMA issue runs ahead across
//    pair and tile boundaries, so the only DMMA bubble is the K-word
//    epilogue (a global read-modify-write of the C tile, ~0.2 % of a pair's
//    mainloop at l = 8192).
//  * k is permuted inside a 16-wide k-block: lane t feeds k = 4t..4t+3 to
//    the four k-steps, so every operand fetch is one conflict-free LDS.128
//    (16-byte chunk (2t+h) ^ (row & 7) of a swizzled 128-byte row).  A and B
//    use the same permutation, so the contraction is unchanged.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "kword.cuh"
#include "ozk_internal.cuh"

namespace ozk {
namespace {

constexpr int BM = 128, BN = 128, BK = 16;
constexpr int kStages = 5;
constexpr int kConsumerWarps = 8;
constexpr int kThreads = kConsumerWarps * 32;
constexpr int kTileBytes = BM * BK * 8;          // 16 KiB per operand tile
constexpr int kStageBytes = 2 * kTileBytes;      // A + B
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
constexpr int kGroupM = 8;                       // tile raster group (L2 reuse)

struct TmaMaps {
    CUtensorMap a;  // 3D: (k, row, slice)
    CUtensorMap b;  // 4D: (k, col-in-block, slice, block)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!ok);
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

__device__ __forceinline__ double2 lds128(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

struct TileCoord {
    int tm, blk, jt;
};

__device__ __forceinline__ TileCoord tile_of(int id, int tiles_m, int tiles_n_blk, int nblk) {
    const int tiles_n = tiles_n_blk * nblk;
    const int group = kGroupM * tiles_n;
    const int first_m = (id / group) * kGroupM;
    const int gm = min(kGroupM, tiles_m - first_m);
    const int in_group = id % group;
    TileCoord t;
    t.tm = first_m + in_group % gm;
    const int tn = in_group / gm;
    t.blk = tn / tiles_n_blk;
    t.jt = tn % tiles_n_blk;
    return t;
}

// Producer-side iterator over the flat (tile, pair, k-block) sequence.
struct ProdIter {
    int tile, p, kb;
};

template <int K, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
pair_gemm_kernel(const __grid_constant__ TmaMaps maps, const __grid_constant__ PairList pairs,
                 GemmProblem prob, int tiles_m, int tiles_n_blk) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    const uint32_t smem_base = smem_u32(smem);
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kStages);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_tiles = tiles_m * tiles_n_blk * prob.nblk;
    const int num_kb = (int)((prob.l + BK - 1) / BK);
    const int npairs = pairs.count;

    // TMA issue for one ring slot: A_alpha rows of the tile, B_beta^T rows of
    // the tile's column block, both the k-block kb.
    auto issue = [&](const ProdIter& it, int stage) {
        const TileCoord tc = tile_of(it.tile, tiles_m, tiles_n_blk, prob.nblk);
        const uint32_t full = full0 + 8 * stage;
        mbar_expect_tx(full, kStageBytes);
        const uint32_t sa = smem_base + stage * kStageBytes;
        tma_load_3d(sa, &maps.a, full, it.kb * BK, tc.tm * BM, pairs.alpha[it.p]);
        tma_load_4d(sa + kTileBytes, &maps.b, full, it.kb * BK, tc.jt * BN, pairs.beta[it.p],
                    tc.blk);
    };
    auto advance = [&](ProdIter& it) {
        if (++it.kb == num_kb) {
            it.kb = 0;
            if (++it.p == npairs) {
                it.p = 0;
                it.tile += gridDim.x;
            }
        }
    };

    ProdIter pit{(int)blockIdx.x, 0, 0};
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.b)));
        for (int s = 0; s < kStages && pit.tile < num_tiles; ++s) {
            issue(pit, s);
            advance(pit);
        }
    }
    __syncthreads();

    const int wm = warp >> 2;  // 0..1 : 64-row half of the tile
    const int wn = warp & 3;   // 0..3 : 32-col quarter
    const int g = lane >> 2, t = lane & 3;
    // byte offsets of this lane's 16-byte chunk for k-half h = 0/1 (swizzled)
    const uint32_t chunk0 = (uint32_t)(((2 * t + 0) ^ g) << 4);
    const uint32_t chunk1 = (uint32_t)(((2 * t + 1) ^ g) << 4);
    const uint32_t a_row = (uint32_t)((wm * 64 + g) * 128);
    const uint32_t b_row = (uint32_t)(kTileBytes + (wn * 32 + g) * 128);

    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    int stage = 0;
    uint32_t phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const TileCoord tc = tile_of(tile, tiles_m, tiles_n_blk, prob.nblk);
        for (int p = 0; p < npairs; ++p) {
            for (int kb = 0; kb < num_kb; ++kb) {
                mbar_wait(full0 + 8 * stage, phase);
                const uint32_t sbase = smem_base + stage * kStageBytes;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t ch = h ? chunk1 : chunk0;
                    double2 af[8], bf[4];
#pragma unroll
                    for (int mf = 0; mf < 8; ++mf) af[mf] = lds128(sbase + a_row + mf * 1024 + ch);
#pragma unroll
                    for (int nf = 0; nf < 4; ++nf) bf[nf] = lds128(sbase + b_row + nf * 1024 + ch);
#pragma unroll
                    for (int u = 0; u < 2; ++u)
#pragma unroll
                        for (int mf = 0; mf < 8; ++mf)
#pragma unroll
                            for (int nf = 0; nf < 4; ++nf)
                                dmma(acc[mf][nf][0], acc[mf][nf][1], u ? af[mf].y : af[mf].x,
                                     u ? bf[nf].y : bf[nf].x);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty0 + 8 * stage);
                // Thread 0 refills this slot once every warp has released it.
                if (threadIdx.x == 0 && pit.tile < num_tiles) {
                    mbar_wait(empty0 + 8 * stage, phase);
                    issue(pit, stage);
                    advance(pit);
                }
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }

            // ---------------- epilogue for pair p of this tile ----------------
            const size_t row0 = (size_t)tc.tm * BM + wm * 64 + g;
            const int jj0 = tc.jt * BN + wn * 32 + 2 * t;
#pragma unroll
            for (int mf = 0; mf < 8; ++mf) {
                const size_t row = row0 + mf * 8;
#pragma unroll
                for (int nf = 0; nf < 4; ++nf) {
#pragma unroll
                    for (int v = 0; v < 2; ++v) {
                        const int jj = jj0 + nf * 8 + v;
                        const size_t col = (size_t)tc.blk * prob.ncb + jj;
                        const double y = acc[mf][nf][v];
                        acc[mf][nf][v] = 0.0;
                        if (row >= prob.m || jj >= prob.ncb || col >= prob.n) continue;
                        if constexpr (MODE == kAccumulate) {
                            double* cp = prob.c + (row * prob.ldc + col) * K;
                            double w[K];
                            if (p == 0) {
#pragma unroll
                                for (int k = 0; k < K; ++k) w[k] = 0.0;
                            } else {
#pragma unroll
                                for (int k = 0; k < K; ++k) w[k] = cp[k];
                            }
                            kw_add<K>(w, y);
#pragma unroll
                            for (int k = 0; k < K; ++k) cp[k] = w[k];
                        } else if constexpr (MODE == kStorePlain) {
                            prob.c[row * prob.ldc + col] = y;
                        } else {
                            prob.c[(size_t)p * prob.c_pair_stride + row * prob.ldc + col] = y;
                        }
                    }
                }
            }
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

template <int K, int MODE>
cudaError_t launch_typed(const GemmProblem& prob, const PairList& pairs, cudaStream_t st,
                         int num_sms) {
    auto encode = get_encode();
    if (!encode) return cudaErrorNotSupported;
    TmaMaps maps;
    {
        cuuint64_t dims[3] = {prob.l, prob.m, (cuuint64_t)prob.a_slices};
        cuuint64_t strides[2] = {prob.lda * 8, prob.a_slice_stride * 8};
        cuuint32_t box[3] = {BK, BM, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = encode(&maps.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                            const_cast<double*>(prob.a), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    {
        cuuint64_t dims[4] = {prob.l, (cuuint64_t)prob.ncb, (cuuint64_t)prob.b_slices,
                              (cuuint64_t)prob.nblk};
        cuuint64_t strides[3] = {prob.ldb * 8, prob.b_slice_stride * 8, prob.b_blk_stride * 8};
        cuuint32_t box[4] = {BK, BN, 1, 1};
        cuuint32_t estr[4] = {1, 1, 1, 1};
        CUresult r = encode(&maps.b, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                            const_cast<double*>(prob.b), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
    const int tiles_m = (int)((prob.m + BM - 1) / BM);
    const int tiles_n_blk = (prob.ncb + BN - 1) / BN;
    const long num_tiles = (long)tiles_m * tiles_n_blk * prob.nblk;
    if (num_tiles == 0 || pairs.count == 0) return cudaSuccess;
    auto kern = pair_gemm_kernel<K, MODE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmemBytes);
    if (e != cudaSuccess) return e;
    const int grid = (int)(num_tiles < num_sms ? num_tiles : num_sms);
    kern<<<grid, kThreads, kSmemBytes, st>>>(maps, pairs, prob, tiles_m, tiles_n_blk);
    return cudaGetLastError();
}

} // namespace

cudaError_t launch_pair_gemm(int K, GemmMode mode, const GemmProblem& prob, const PairList& pairs,
                             cudaStream_t st, int num_sms) {
    if (mode == kStorePlain) return launch_typed<1, kStorePlain>(prob, pairs, st, num_sms);
    if (mode == kStoreProducts) return launch_typed<1, kStoreProducts>(prob, pairs, st, num_sms);
    switch (K) {
    case 2: return launch_typed<2, kAccumulate>(prob, pairs, st, num_sms);
    case 3: return launch_typed<3, kAccumulate>(prob, pairs, st, num_sms);
    case 4: return launch_typed<4, kAccumulate>(prob, pairs, st, num_sms);
    default: return cudaErrorInvalidValue;
    }
}

} // namespace ozk

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
//  * Persistent CTAs, one per SM: 8 consumer warps in two ping-pong groups
//    of 4 (one warp of each group per SM sub-partition) plus a producer
//    warpgroup.  A group owns a 64x128 C tile (four 64x32 warp tiles, 64 FP64
//    accumulators per thread) and its own 4-stage ring of 64x16 A and 128x16
//    B^T tiles filled by TMA (cp.async.bulk.tensor, 128-byte swizzle) under
//    mbarriers; one producer lane per group keeps its ring full.
//    setmaxnreg moves registers from the producer warpgroup (40) to the
//    consumers (232): two consumers + one producer per sub-partition fit its
//    16K-register file.
//  * A group walks tile -> pair -> k-block; its loads run ahead across pair
//    and tile boundaries.  The K-word epilogue (a read-modify-write of the C
//    tile after every pair) stalls only its own group: the other group's
//    warp on the same sub-partition keeps the DMMA pipe busy.  The C rows of
//    the coming epilogue are prefetched into L2 a few k-blocks ahead and
//    read in batches of eight elements.
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

// Ping-pong layout: two independent 4-warp consumer groups per CTA, one warp
// of each on every SM sub-partition, plus a producer warpgroup.  A group owns
// a BM x BN C tile (its 4 warps each own 64 x 32) and its own TMA ring, so
// while one group runs its K-word epilogue the other keeps the
// sub-partition's DMMA pipe busy (one warp with 32 independent accumulators
// saturates it).
constexpr int BM = 64, BN = 128, BK = 16;
constexpr int kStages = 4;                       // per group
constexpr int kGroups = 2;
constexpr int kWarpsPerGroup = 4;
constexpr int kConsumerWarps = kGroups * kWarpsPerGroup;
constexpr int kThreads = (kConsumerWarps + 4) * 32;   // + producer warpgroup
constexpr int kConsumerRegs = 232;               // setmaxnreg budget: 2*232 + 40 per SMSP
constexpr int kProducerRegs = 40;
constexpr int kATileBytes = BM * BK * 8;         // 8 KiB
constexpr int kBTileBytes = BN * BK * 8;         // 16 KiB
constexpr int kStageBytes = kATileBytes + kBTileBytes;
constexpr int kGroupSmem = kStages * kStageBytes;
constexpr int kSmemBytes = kGroups * kGroupSmem + 1024 /*align*/ + 256 /*barriers*/;
constexpr int kGroupM = 16;                      // tile raster group (L2 reuse)
constexpr int kPrefetchKb = 6;                   // k-blocks before the epilogue: L2 prefetch of C

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

// W: word type of the K-word C in kAccumulate mode (double: DD/TD/QD, float:
// TS -- an exact binary64 slice product of binary32 slices is exactly
// representable in binary32, so the cast before the TS epilogue is exact).
template <int K, int MODE, typename W>
__global__ void __launch_bounds__(kThreads, 1)
pair_gemm_kernel(const __grid_constant__ TmaMaps maps, const __grid_constant__ PairChunk pairs,
                 GemmProblem prob, int tiles_m, int tiles_n_blk) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* bars_all = reinterpret_cast<uint64_t*>(smem + kGroups * kGroupSmem);
    const uint32_t start_bar = smem_u32(bars_all + kGroups * 2 * kStages);

    const int num_tiles = tiles_m * tiles_n_blk * prob.nblk;
    const int num_kb = (int)((prob.l + BK - 1) / BK);
    const int npairs = pairs.count;
    constexpr bool kAcc = MODE == kAccumulate || MODE == kAccumulateLU;
    const int nworkers = gridDim.x * kGroups;

    if (threadIdx.x == 0) {
        for (int b = 0; b < kGroups * 2 * kStages; ++b)
            mbar_init(smem_u32(bars_all + b), (b % (2 * kStages)) < kStages ? 1 : kWarpsPerGroup);
        mbar_init(start_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp >= kConsumerWarps) {
        // ---------------- producer warpgroup: one lane per consumer group ----------------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProducerRegs));
        const int grp = warp - kConsumerWarps;
        if (grp >= kGroups || lane != 0) return;
        const uint32_t ring = smem_u32(smem) + grp * kGroupSmem;
        const uint32_t full0 = smem_u32(bars_all + grp * 2 * kStages);
        const uint32_t empty0 = full0 + 8 * kStages;
        if (grp == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a)));
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.b)));
        }
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = blockIdx.x * kGroups + grp; tile < num_tiles; tile += nworkers) {
            const TileCoord tc = tile_of(tile, tiles_m, tiles_n_blk, prob.nblk);
            for (int p = 0; p < npairs; ++p) {
                const int al = pairs.alpha[p], be = pairs.beta[p];
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(empty0 + 8 * stage, phase ^ 1);
                    const uint32_t full = full0 + 8 * stage;
                    mbar_expect_tx(full, kStageBytes);
                    const uint32_t sa = ring + stage * kStageBytes;
                    tma_load_3d(sa, &maps.a, full, kb * BK, tc.tm * BM, al);
                    tma_load_4d(sa + kATileBytes, &maps.b, full, kb * BK, tc.jt * BN, be, tc.blk);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        return;
    }

    // ---------------- DMMA consumers ----------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsumerRegs));
    const int grp = warp / kWarpsPerGroup;   // ping-pong group
    const int wn = warp % kWarpsPerGroup;    // 32-column quarter of the group tile
    const uint32_t ring = smem_u32(smem) + grp * kGroupSmem;
    const uint32_t full0 = smem_u32(bars_all + grp * 2 * kStages);
    const uint32_t empty0 = full0 + 8 * kStages;
    const int worker = blockIdx.x * kGroups + grp;
    // Group 0 releases group 1 half-way through its first pair, so the two
    // groups' epilogues start out of phase (their drift afterwards is neutral).
    const int kick_kb = num_kb / 2;
    if (grp == 0 && wn == 0 && lane == 0 && worker >= num_tiles) mbar_arrive(start_bar);
    if (grp == 1) mbar_wait(start_bar, 0);

    const int g = lane >> 2, t = lane & 3;
    // byte offsets of this lane's 16-byte chunk for k-half h = 0/1 (swizzled)
    const uint32_t chunk0 = (uint32_t)(((2 * t + 0) ^ g) << 4);
    const uint32_t chunk1 = (uint32_t)(((2 * t + 1) ^ g) << 4);
    const uint32_t a_row = (uint32_t)(g * 128);
    const uint32_t b_row = (uint32_t)(kATileBytes + (wn * 32 + g) * 128);

    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    int stage = 0;
    uint32_t phase = 0;
    bool kicked = false;
    for (int tile = worker; tile < num_tiles; tile += nworkers) {
        const TileCoord tc = tile_of(tile, tiles_m, tiles_n_blk, prob.nblk);
        const size_t row0 = (size_t)tc.tm * BM + g;
        const int jj0 = tc.jt * BN + wn * 32 + 2 * t;
        // element validity masks (rows by mf, columns by nf*2+v)
        uint32_t rmask = 0, cmask = 0;
#pragma unroll
        for (int mf = 0; mf < 8; ++mf) rmask |= (row0 + mf * 8 < prob.m) ? (1u << mf) : 0u;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int jj = jj0 + (q >> 1) * 8 + (q & 1);
            const size_t col = (size_t)tc.blk * prob.ncb + jj;
            cmask |= (jj < prob.ncb && col < prob.n) ? (1u << q) : 0u;
        }
        const size_t col0 = (size_t)tc.blk * prob.ncb + jj0;

        for (int p = 0; p < npairs; ++p) {
            for (int kb = 0; kb < num_kb; ++kb) {
                if (grp == 0 && !kicked && kb == kick_kb) {
                    kicked = true;
                    if (wn == 0 && lane == 0) mbar_arrive(start_bar);
                }
                mbar_wait(full0 + 8 * stage, phase);
                const uint32_t sbase = ring + stage * kStageBytes;
                // dep: XOR of every fragment this warp reads from the stage.
                // Feeding it (masked by a runtime zero) into the release
                // address makes the arrive wait, through the register
                // scoreboard, for all of the stage's LDS to have returned; a
                // bare arrive can issue while the last LDS is in flight and
                // let TMA overwrite the slot under it.
                uint32_t dep = 0;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t ch = h ? chunk1 : chunk0;
                    double2 af[8], bf[4];
#pragma unroll
                    for (int mf = 0; mf < 8; ++mf) {
                        af[mf] = lds128(sbase + a_row + mf * 1024 + ch);
                        dep ^= (uint32_t)__double2loint(af[mf].x);
                    }
#pragma unroll
                    for (int nf = 0; nf < 4; ++nf) {
                        bf[nf] = lds128(sbase + b_row + nf * 1024 + ch);
                        dep ^= (uint32_t)__double2loint(bf[nf].x);
                    }
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
                if (lane == 0) mbar_arrive(empty0 + 8 * stage + (dep & prob.zero));
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
                if constexpr (kAcc) {
                    if (kb == num_kb - kPrefetchKb && (p > 0 || prob.c_continue)) {
                        // pull this pair's C rows into L2 ahead of the read-modify-write
#pragma unroll
                        for (int mf = 0; mf < 8; ++mf)
#pragma unroll
                            for (int nf = 0; nf < 4; ++nf)
                                if ((rmask >> mf) & (cmask >> (2 * nf)) & 1u)
                                    asm volatile("prefetch.global.L2 [%0];" ::"l"(
                                        static_cast<W*>(prob.c) +
                                        ((row0 + mf * 8) * prob.ldc + col0 + nf * 8) * K));
                    }
                }
            }

            // ---------------- epilogue for pair p of this tile ----------------
            // Two code shapes, chosen per format from B200 measurements
            // (tools/exp_epilogue.py, profiles/r01_ncu_summary.md):
            //  * fully unrolled over the 8 fragment rows: all C addresses are
            //    compile-time offsets of one base, so the compiler batches the
            //    loads of every row ahead of the K-word math (shortest epilogue
            //    latency).  Best for DD: 95.0 % of the DMMA ceiling vs 90.3 %.
            //  * runtime loop over the rows, the row's 8 accumulators picked out
            //    with predicated selects: 5-8x less code; the unrolled K >= 3
            //    epilogues (13.5K-18K SASS instructions) thrash the instruction
            //    cache.  Best for TD (87.3 % vs 84.5-87.7 %), QD (85.0 % vs
            //    80.1 %) and TS.
            constexpr bool kLoopRows = K >= 3;
#pragma unroll(kLoopRows ? 1 : 8)
            for (int mf = 0; mf < 8; ++mf) {
                if (!((rmask >> mf) & 1u)) continue;
                double y[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    double v = acc[0][q >> 1][q & 1];
#pragma unroll
                    for (int r = 1; r < 8; ++r) v = (mf == r) ? acc[r][q >> 1][q & 1] : v;
                    y[q] = v;
                }
                const size_t row = row0 + mf * 8;
                if constexpr (kAcc) {
                    // batch: load the 8 K-word elements of this row first
                    W w[8][K];
                    W* cp = static_cast<W*>(prob.c) + (row * prob.ldc + col0) * K;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const bool ok = (cmask >> q) & 1u;
                        const int off = ((q >> 1) * 8 + (q & 1)) * K;
#pragma unroll
                        for (int k = 0; k < K; ++k)
                            w[q][k] = (ok && (p > 0 || prob.c_continue)) ? cp[off + k] : W(0);
                    }
#ifdef OZK_EXPERIMENT_TRIVIAL_EPILOGUE
#pragma unroll
                    for (int q = 0; q < 8; ++q) w[q][0] = w[q][0] + (W)y[q];
#else
#pragma unroll
                    for (int q = 0; q < 8; ++q) kw_add<K, W, true, true>(w[q], (W)y[q]);
#endif
                    if constexpr (MODE == kAccumulateLU) {
                        if (prob.lu_final && p == npairs - 1) {
                            // the list's last pair: A22 -= sum (lu.hpp:121-124,
                            // MultiFloat -= MultiFloat = x + (-y), multifloat.hpp:
                            // 300,178-199) in place of the C store
                            double* ap = prob.lu_a22 + (row * prob.lu_lda + col0) * K;
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                if (!((cmask >> q) & 1u)) continue;
                                const int off = ((q >> 1) * 8 + (q & 1)) * K;
                                double x[K], ny[K];
#pragma unroll
                                for (int k = 0; k < K; ++k) x[k] = ap[off + k];
                                kw_neg<K>(w[q], ny);
                                kw_add_kw<K>(x, ny);
#pragma unroll
                                for (int k = 0; k < K; ++k) ap[off + k] = x[k];
                            }
                            continue;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int off = ((q >> 1) * 8 + (q & 1)) * K;
                        if ((cmask >> q) & 1u) {
#pragma unroll
                            for (int k = 0; k < K; ++k) cp[off + k] = w[q][k];
                        }
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (!((cmask >> q) & 1u)) continue;
                        const size_t col = col0 + (q >> 1) * 8 + (q & 1);
                        double* cd = static_cast<double*>(prob.c);
                        if constexpr (MODE == kStorePlain)
                            cd[row * prob.ldc + col] = y[q];
                        else
                            cd[(size_t)p * prob.c_pair_stride + row * prob.ldc + col] = y[q];
                    }
                }
            }
#pragma unroll
            for (int mf = 0; mf < 8; ++mf)
#pragma unroll
                for (int nf = 0; nf < 4; ++nf) acc[mf][nf][0] = acc[mf][nf][1] = 0.0;
        }
    }
    // group 0 with fewer k-blocks than the kick point still has to release group 1
    if (grp == 0 && !kicked && worker < num_tiles && wn == 0 && lane == 0) mbar_arrive(start_bar);
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

template <int K, int MODE, typename W = double>
cudaError_t launch_typed(const GemmProblem& prob, const PairChunk& pairs, cudaStream_t st,
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
    auto kern = pair_gemm_kernel<K, MODE, W>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmemBytes);
    if (e != cudaSuccess) return e;
    const long ctas = (num_tiles + kGroups - 1) / kGroups;
    const int grid = (int)(ctas < num_sms ? ctas : num_sms);
    kern<<<grid, kThreads, kSmemBytes, st>>>(maps, pairs, prob, tiles_m, tiles_n_blk);
    return cudaGetLastError();
}

} // namespace

namespace {
cudaError_t launch_chunk(int K, GemmMode mode, const GemmProblem& prob, const PairChunk& pairs,
                         cudaStream_t st, int num_sms, int word_bytes) {
    if (mode == kStorePlain) return launch_typed<1, kStorePlain>(prob, pairs, st, num_sms);
    if (mode == kAccumulate && word_bytes == 4) {
        if (K != 3) return cudaErrorInvalidValue;
        return launch_typed<3, kAccumulate, float>(prob, pairs, st, num_sms);
    }
    if (mode == kStoreProducts) return launch_typed<1, kStoreProducts>(prob, pairs, st, num_sms);
    if (mode == kAccumulateLU) {
        if (word_bytes != 8) return cudaErrorInvalidValue;
        switch (K) {
        case 2: return launch_typed<2, kAccumulateLU>(prob, pairs, st, num_sms);
        case 3: return launch_typed<3, kAccumulateLU>(prob, pairs, st, num_sms);
        case 4: return launch_typed<4, kAccumulateLU>(prob, pairs, st, num_sms);
        default: return cudaErrorInvalidValue;
        }
    }
    switch (K) {
    case 2: return launch_typed<2, kAccumulate>(prob, pairs, st, num_sms);
    case 3: return launch_typed<3, kAccumulate>(prob, pairs, st, num_sms);
    case 4: return launch_typed<4, kAccumulate>(prob, pairs, st, num_sms);
    default: return cudaErrorInvalidValue;
    }
}
}  // namespace

// Pair lists longer than one launch's parameter block run as consecutive
// launches: each later chunk continues the K-word sum already in C (same
// per-element pair order), or writes its products further along.
cudaError_t launch_pair_gemm(int K, GemmMode mode, const GemmProblem& prob, const PairList& pairs,
                             cudaStream_t st, int num_sms, int word_bytes) {
    for (int q0 = 0; q0 < pairs.count; q0 += kPairsPerLaunch) {
        GemmProblem pb = prob;
        if (mode == kAccumulate || mode == kAccumulateLU)
            pb.c_continue = prob.c_continue || q0 > 0;
        pb.lu_final = q0 + kPairsPerLaunch >= pairs.count;
        if (mode == kStoreProducts) pb.c = static_cast<double*>(prob.c) + q0 * prob.c_pair_stride;
        const cudaError_t e = launch_chunk(K, mode, pb, pair_chunk(pairs, q0), st, num_sms,
                                           word_bytes);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

} // namespace ozk

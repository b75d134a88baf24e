// gemm_i8.cu -- exact slice products on the INT8 tensor cores (tcgen05.mma
// kind::i8), with the same fused K-word epilogue as the DMMA kernel.
//
// Why it is bit-identical to the reference.  Slice a of row i is an integer
// multiple of 2^g(a,i), g = e + sigma - 54, with |piece / 2^g| <= 2^(54-sigma)
// (the split's grid, ozaki.hpp:15-29; test_ozaki.cpp:61-92).  For inner
// dimension l > 512 (sigma >= 32) that integer M fits 3 signed base-256 digits
// d0 + 256 d1 + 65536 d2 (split.cu writes them next to the FP64 slice).  Then
//   C_ab(i,j) = 2^(gA(i) + gB(j)) * sum_{s,t} 256^(s+t) * sum_k dA_s(i,k) dB_t(j,k)
// where every int8 x int8 -> int32 digit GEMM is exact (|level| < 3 l 2^14 <
// 2^31 for l < 43690) and the int64 recombination equals the exact integer
// slice product, which is < 2^53 (the split's exactness bound) -- so the
// binary64 value is exactly the C_ab any FP64 backend (reference_backend_gemm,
// DMMA) computes.  The K-word accumulation that follows is the same
// kw_add<K> sequence in the same pair order.
//
// B200 mapping (one persistent CTA per SM, 12 warps):
//   warp 0      TMA producer: per 128-deep k-block, the 3 A-digit tiles (128x128
//               int8) and 3 B-digit tiles (64x128 int8), 128-byte swizzle,
//               3-stage mbarrier ring (72 KiB per stage).
//   warp 1      TMEM allocator + single-thread MMA issuer: 9 digit pairs x 4
//               k-chunks = 36 tcgen05.mma (M=128, N=64, K=32) per k-block into
//               5 TMEM level accumulators (levels s+t = 0..4, 64 columns each);
//               tcgen05.commit releases the smem stage and, after a pair's last
//               k-block, hands TMEM to the epilogue.
//   warps 4-11  two epilogue warpgroups, one per 32-column half of the tile (one
//               TMEM lane = one C row per thread): tcgen05.ld the 5 levels,
//               recombine in int64, scale by 2^(gA + gB), release TMEM (the MMAs
//               of the next pair start), then the K-word read-modify-write of the
//               thread's 32 contiguous C elements.  setmaxnreg moves registers
//               from the producer/MMA warpgroup (40) to the epilogue (232).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "kword.cuh"
#include "ozk_internal.cuh"

namespace ozk {
namespace {

constexpr int BM = 128, BKB = 128;            // tile M, k bytes per stage
constexpr int kEpiGroups = 2;                 // epilogue warpgroups (column halves)
constexpr int kThreads = (4 + 4 * kEpiGroups) * 32;
constexpr int kGroupM = 8;
constexpr int kSmemBudget = 200 * 1024;       // operand ring

// Compile-time shape of one engine instance.
//   W   word type of C (double: DD/TD/QD, float: TS)
//   ND  int8 digits per slice integer (3 for binary64 slices at l > 512; 1 for
//       TS slices at l > 4096, where |M| <= 2^(25 - sigma) <= 64; 2 below)
//   BN  tile width; 2*ND-1 level accumulators of BN TMEM columns each
template <int K, typename W, int ND, int BN>
struct I8Cfg {
    static constexpr int kLevels = 2 * ND - 1;
    static constexpr int kATile = BM * BKB;
    static constexpr int kBTile = BN * BKB;
    static constexpr int kStageBytes = ND * (kATile + kBTile);
    static constexpr int kStages = kSmemBudget / kStageBytes < 8 ? kSmemBudget / kStageBytes : 8;
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
    static constexpr int kTmemCols = kLevels * BN <= 32 ? 32 : kLevels * BN <= 64 ? 64
                                   : kLevels * BN <= 128 ? 128 : kLevels * BN <= 256 ? 256 : 512;
    static constexpr int kEpiCols = BN / kEpiGroups;  // columns per epilogue thread
    // K-word adds unrolled per epilogue step (B200 A/B at n = 8192,
    // tools/variants_bench.py): DD 8 (104.6 ms; 2: 109.1), TD 2 (316 ms; 8: 349),
    // QD 2 (582 ms; 8: 664) -- the K >= 3 bodies are large enough that more
    // unrolling costs instruction-cache misses and registers instead of latency.
    static constexpr int kChunk = (K == 2 && sizeof(W) == 8) ? 8 : 2;
    static_assert(kStages >= 2, "operand ring too small");
    static_assert(kLevels * BN <= 512, "TMEM");
};

struct MapsI8 {
    CUtensorMap a;  // 4D: (k, row, digit, slice)
    CUtensorMap b;
};

struct I8Problem {
    size_t m, n, l;
    const int* gA;     // [d][m] grid exponents
    const int* gB;     // [d][n]
    size_t gA_stride, gB_stride;
    void* c;           // K-word AoS C, row stride ldc elements
    size_t ldc;
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
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
// UMMA shared-memory descriptor: K-major operand, 128-byte swizzle, 8-row groups
// 1024 B apart (CuTe mma_sm100_desc.hpp SmemDescriptor, version 1 = Blackwell).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)1 << 16) |
           ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

// Exact int64 -> binary64 for |s| < 2^53 on the FP64 pipe (I2F.F64.S64 runs on
// the slow XU pipe, which bound the epilogue at 76 % XU utilisation):
// s = hi * 2^26 + lo with the two halves converted by exponent-bias tricks.
__device__ __forceinline__ double i64_to_f64_exact(long long s) {
    const long long hi = s >> 26;                      // |hi| < 2^27
    const long long lo = s & ((1ll << 26) - 1);        // 0 <= lo < 2^26
    const double dh = __dsub_rn(__longlong_as_double(0x4338000000000000ll + hi),
                                6755399441055744.0);   // 2^52 + 2^51
    const double dl = __dsub_rn(__longlong_as_double(0x4330000000000000ll | lo),
                                4503599627370496.0);   // 2^52
    return __fma_rn(dh, 67108864.0, dl);               // exact: the result is s
}

// y * 2^e with one correct rounding (= scalbn): for normal 2^e a single
// multiply by the bit-built power of two, off the XU pipe; scalbn only for the
// rare exponents outside the normal range.
__device__ __forceinline__ double ldexp_fast(double y, int e) {
    if (e >= -1022 && e <= 1023)
        return __dmul_rn(y, __longlong_as_double((long long)(e + 1023) << 52));
    return scalbn(y, e);
}

struct TileCoord {
    int tm, tn;
};
__device__ __forceinline__ TileCoord tile_of(int id, int tiles_m, int tiles_n) {
    const int group = kGroupM * tiles_n;
    const int first_m = (id / group) * kGroupM;
    const int gm = min(kGroupM, tiles_m - first_m);
    const int in_group = id % group;
    return TileCoord{first_m + in_group % gm, in_group / gm};
}

template <int K, typename W, int ND, int BN>
__global__ void __launch_bounds__(kThreads, 1)
pair_gemm_i8_kernel(const __grid_constant__ MapsI8 maps, const __grid_constant__ PairList pairs,
                    I8Problem prob, int tiles_m, int tiles_n) {
    using Cfg = I8Cfg<K, W, ND, BN>;
    constexpr int kStages = Cfg::kStages, kStageBytes = Cfg::kStageBytes;
    constexpr int kATile = Cfg::kATile, kBTile = Cfg::kBTile, kEpiCols = Cfg::kEpiCols;
    constexpr int kTmemCols = Cfg::kTmemCols, kLevels = Cfg::kLevels;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    // bars: full[S], empty[S], tmem_full, tmem_empty ; then the TMEM base word
    const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * kStages;
    const uint32_t tmem_full = empty0 + 8 * kStages, tmem_empty = tmem_full + 8;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2);
    const uint32_t ring = smem_u32(smem);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_tiles = tiles_m * tiles_n;
    const int num_kb = (int)((prob.l + BKB - 1) / BKB);
    const int npairs = pairs.count;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 4 * kEpiGroups);  // one arrive per epilogue warp
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
      if (warp == 0 && lane == 0) {
        // ---------------- TMA producer ----------------
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.b)));
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const TileCoord tc = tile_of(tile, tiles_m, tiles_n);
            for (int p = 0; p < npairs; ++p) {
                const int al = pairs.alpha[p], be = pairs.beta[p];
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(empty0 + 8 * stage, phase ^ 1);
                    const uint32_t full = full0 + 8 * stage;
                    mbar_expect_tx(full, kStageBytes);
                    const uint32_t sa = ring + stage * kStageBytes;
#pragma unroll
                    for (int dgt = 0; dgt < ND; ++dgt) {
                        tma_load_4d(sa + dgt * kATile, &maps.a, full, kb * BKB, tc.tm * BM, dgt, al);
                        tma_load_4d(sa + ND * kATile + dgt * kBTile, &maps.b, full, kb * BKB,
                                    tc.tn * BN, dgt, be);
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
      } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer ----------------
        // kind::i8 instruction descriptor: D s32, A/B signed 8-bit, K-major,
        // N = 64, M = 128 (CuTe mma_sm100_desc.hpp InstrDescriptor)
        constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                   ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
        int stage = 0;
        uint32_t phase = 0, tphase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            for (int p = 0; p < npairs; ++p) {
                mbar_wait(tmem_empty, tphase ^ 1);  // epilogue drained the levels
                tphase ^= 1;
                asm volatile("tcgen05.fence::after_thread_sync;");
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(full0 + 8 * stage, phase);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa = ring + stage * kStageBytes;
#pragma unroll
                    for (int kc = 0; kc < BKB / 32; ++kc) {
                        // digit pairs level by level; the first MMA of each
                        // level in a pair's first chunk overwrites the accumulator
#pragma unroll
                        for (int lvl = 0; lvl < kLevels; ++lvl) {
#pragma unroll
                            for (int ds = 0; ds < ND; ++ds) {
                                const int dt = lvl - ds;
                                if (dt < 0 || dt >= ND) continue;
                                const bool first = ds == (lvl - ND + 1 > 0 ? lvl - ND + 1 : 0);
                                const uint64_t da = sw128_desc(sa + ds * kATile + kc * 32);
                                const uint64_t db =
                                    sw128_desc(sa + ND * kATile + dt * kBTile + kc * 32);
                                const uint32_t acc = (kb | kc) ? 1u : (first ? 0u : 1u);
                                umma_i8(tmem + lvl * BN, da, db, idesc, acc);
                            }
                        }
                    }
                    umma_commit(empty0 + 8 * stage);  // frees the stage when the MMAs retire
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(tmem_full);
            }
        }
      }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
        // ---------------- epilogue warpgroups ----------------
        // warpgroup eg owns columns [eg*32, eg*32+32) of every tile for every
        // pair (so no two threads ever touch the same C element); warp % 4
        // selects the 32 TMEM lanes (C rows) it may access.
        const int eg = (warp - 4) / 4;
        const int wq = warp % 4;
        const uint32_t tlane = tmem + ((uint32_t)(wq * 32) << 16) + eg * kEpiCols;
        uint32_t tphase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const TileCoord tc = tile_of(tile, tiles_m, tiles_n);
            const size_t row = (size_t)tc.tm * BM + wq * 32 + lane;
            const size_t col0 = (size_t)tc.tn * BN + eg * kEpiCols;
            const bool row_ok = row < prob.m;
            for (int p = 0; p < npairs; ++p) {
                const int al = pairs.alpha[p], be = pairs.beta[p];
                const int ga = row_ok ? prob.gA[(size_t)al * prob.gA_stride + row] : 0;
                mbar_wait(tmem_full, tphase);
                tphase ^= 1;
                asm volatile("tcgen05.fence::after_thread_sync;");
                double y[kEpiCols];
#pragma unroll
                for (int c = 0; c < kEpiCols; c += 16) {
                    int32_t lv[kLevels][16];
#pragma unroll
                    for (int u = 0; u < kLevels; ++u) tmem_ld16(tlane + u * BN + c, lv[u]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        long long s = lv[0][j];
#pragma unroll
                        for (int u = 1; u < kLevels; ++u) s += (long long)lv[u][j] << (8 * u);
                        y[c + j] = i64_to_f64_exact(s);  // exact: |s| < 2^53
                    }
                }
                // levels are in registers: hand TMEM back to the MMA issuer
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive(tmem_empty);
                if (!row_ok) continue;
                W* cp = static_cast<W*>(prob.c) + (row * prob.ldc + col0) * K;
                const int* gbp = prob.gB + (size_t)be * prob.gB_stride + col0;
#pragma unroll 1
                constexpr int kChunk = Cfg::kChunk;
                for (int c = 0; c < kEpiCols; c += kChunk) {
                    // y[0..kChunk) are this chunk's products; the array is
                    // shifted down after each chunk so every index stays static
                    W w[kChunk][K];
#pragma unroll
                    for (int j = 0; j < kChunk; ++j) {
                        const bool ok = col0 + c + j < prob.n;
#pragma unroll
                        for (int k = 0; k < K; ++k)
                            w[j][k] = (ok && p > 0) ? cp[(c + j) * K + k] : W(0);
                    }
#pragma unroll
                    for (int j = 0; j < kChunk; ++j) {
                        const bool ok = col0 + c + j < prob.n;
                        const int gb = ok ? __ldg(gbp + c + j) : 0;
                        // exact scaled slice product (a TS product is exact in binary32)
                        kw_add<K>(w[j], (W)ldexp_fast(y[j], ga + gb));
                    }
#pragma unroll
                    for (int j = 0; j < kChunk; ++j) {
                        if (col0 + c + j < prob.n) {
#pragma unroll
                            for (int k = 0; k < K; ++k) cp[(c + j) * K + k] = w[j][k];
                        }
                    }
#pragma unroll
                    for (int j = 0; j < kEpiCols - kChunk; ++j) y[j] = y[j + kChunk];
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kTmemCols));
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_i8() {
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

template <int K, typename W, int ND, int BN>
cudaError_t launch_i8_typed(const I8Operands& op, const PairList& pairs, cudaStream_t st,
                            int num_sms) {
    using Cfg = I8Cfg<K, W, ND, BN>;
    auto encode = get_encode_i8();
    if (!encode) return cudaErrorNotSupported;
    MapsI8 maps;
    {
        cuuint64_t dims[4] = {op.l, op.m, (cuuint64_t)ND, (cuuint64_t)op.d};
        cuuint64_t strides[3] = {op.a_ld, op.a_digit_stride, op.a_slice_stride};
        cuuint32_t box[4] = {BKB, BM, 1, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (encode(&maps.a, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(op.a), dims,
                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    {
        cuuint64_t dims[4] = {op.l, op.n, (cuuint64_t)ND, (cuuint64_t)op.d};
        cuuint64_t strides[3] = {op.b_ld, op.b_digit_stride, op.b_slice_stride};
        cuuint32_t box[4] = {BKB, BN, 1, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (encode(&maps.b, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(op.b), dims,
                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    I8Problem prob;
    prob.m = op.m;
    prob.n = op.n;
    prob.l = op.l;
    prob.gA = op.gA;
    prob.gB = op.gB;
    prob.gA_stride = op.m;
    prob.gB_stride = op.n;
    prob.c = op.c;
    prob.ldc = op.ldc;
    const int tiles_m = (int)((op.m + BM - 1) / BM), tiles_n = (int)((op.n + BN - 1) / BN);
    const int num_tiles = tiles_m * tiles_n;
    if (num_tiles == 0 || pairs.count == 0) return cudaSuccess;
    auto kern = pair_gemm_i8_kernel<K, W, ND, BN>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    const int grid = num_tiles < num_sms ? num_tiles : num_sms;
    kern<<<grid, kThreads, Cfg::kSmemBytes, st>>>(maps, pairs, prob, tiles_m, tiles_n);
    return cudaGetLastError();
}

} // namespace

cudaError_t launch_pair_gemm_i8(int K, int word_bytes, const I8Operands& op,
                                const PairList& pairs, cudaStream_t st, int num_sms) {
    if (word_bytes == 4) {  // TS: binary32 words, 1 or 2 digits
        if (K != 3) return cudaErrorInvalidValue;
        if (op.nd == 1) return launch_i8_typed<3, float, 1, 128>(op, pairs, st, num_sms);
        if (op.nd == 2) return launch_i8_typed<3, float, 2, 64>(op, pairs, st, num_sms);
        return cudaErrorInvalidValue;
    }
    if (op.nd != 3) return cudaErrorInvalidValue;
    switch (K) {
    case 2: return launch_i8_typed<2, double, 3, 64>(op, pairs, st, num_sms);
    case 3: return launch_i8_typed<3, double, 3, 64>(op, pairs, st, num_sms);
    case 4: return launch_i8_typed<4, double, 3, 64>(op, pairs, st, num_sms);
    default: return cudaErrorInvalidValue;
    }
}

} // namespace ozk

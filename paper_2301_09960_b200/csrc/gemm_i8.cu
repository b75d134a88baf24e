// gemm_i8.cu -- exact slice products on the INT8 tensor cores (tcgen05.mma
// kind::i8), with the same fused K-word epilogue as the DMMA kernel.
//
// Why it is bit-identical to the reference.  Slice a of row i is an integer
// multiple of 2^g(a,i), g = e + sigma - 53, with |piece / 2^g| <= 2^(53-sigma)
// (the split's grid, ozaki.hpp:15-29; test_ozaki.cpp:61-92).  For inner
// dimension l > 128 (sigma >= 31) that integer M fits 3 signed base-256 digits
// d0 + 256 d1 + 65536 d2 (split.cu writes them next to the FP64 slice).  Then
//   C_ab(i,j) = 2^(gA(i) + gB(j)) * sum_{s,t} 256^(s+t) * sum_k dA_s(i,k) dB_t(j,k)
// where every int8 x int8 -> int32 digit GEMM is exact (|level| < 3 l 2^14 <
// 2^31 for l < 43690) and the int64 recombination equals the exact integer
// slice product, which is < 2^53 (the split's exactness bound) -- so the
// binary64 value is exactly the C_ab any FP64 backend (reference_backend_gemm,
// DMMA) computes.  The K-word accumulation that follows is the same
// kw_add<K> sequence in the same pair order.
//
// B200 mapping: one persistent CTA per SM, 4 + 4*EG warps (EG epilogue
// warpgroups: DD 4, TD/QD 6, TS 7), 2-CTA clusters.  The tile is transposed with respect
// to C: the MMA's M side (128 TMEM lanes) runs over 128 C COLUMNS (B-slice
// digits) and its N side over TR (DD 64, TD/QD 48, TS 112) C rows per A-slice
// digit, so every epilogue thread owns one C column and a warp's C accesses
// are a contiguous K-word row segment instead of 32 rows apart.
//   warp 0      TMA producer: per 128-deep k-block, the ND B-digit tiles (128 x
//               128 int8) and the ND A-digit tiles (TR x 128, adjacent in shared
//               memory), 128-byte swizzle, 3-stage mbarrier ring.  The two CTAs
//               of a cluster own vertically adjacent tiles and share the B-digit
//               tile: each loads half and multicasts it (.multicast::cluster).
//               Wave pacing: a cluster starts (wave, pair) step s only after
//               every cluster has started s-1 (global arrival counters, bounded
//               spin), so all clusters stream the same slices and L2 holds them.
//   warp 1      TMEM allocator + MMA issuer (whole warp, elect.sync issue,
//               warp-uniform descriptors).  The ND A-digit tiles form ONE
//               N = ND*TR operand, so MMA(Bdigit t, [A_0;...;A_ND-1]) with its
//               accumulator based at level block t lands digit product (t, u) in
//               block t + u = its level: ND MMAs per 32-deep k-chunk instead of
//               ND^2.  The first k-chunk of a pair issues the ND^2 single-digit
//               products instead, each level's first one overwriting.  A stage's
//               commit arrives on the empty barriers of every CTA that
//               multicasts into it.
//   warps 4..   EG epilogue warpgroups, TR/EG rows each (one TMEM lane = one C
//               column per thread): NB = 1 (DD) drains the 2ND-1 levels to
//               registers, recombines them exactly (int64 -> binary64, scale by
//               2^(gA + gB)) and releases TMEM at once; NB = 2 (TD/QD/TS) reads
//               them in place from double-buffered accumulators; TS keeps 4
//               buffers and updates C once per two pairs.
//               Then the K-word read-modify-write of the thread's column
//               segment, ping-pong C prefetch, 16-byte accesses.  setmaxnreg
//               moves registers from the producer/MMA warpgroup (40) to the
//               epilogue.
// Diagnostic builds: -DOZK_I8_TRACE (cycle stamps, tools/i8_trace.py) and
// -DOZK_I8_EPI_MODE=1..6 (timing-only variants with parts of the work removed;
// wrong results by design).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <atomic>

#include "kword.cuh"
#include "ozk_internal.cuh"

namespace ozk {
namespace {

// k bytes per operand stage: 128 (128-byte swizzle) or 64 (64-byte swizzle:
// half-depth stages, twice as many in the same shared memory).  64 measured
// bit-identical but slower (TD slice GEMM 180 -> 217 ms, DD 74 -> 80, TS 94 ->
// 130): twice the barrier/commit/TMA traffic per k outweighs the deeper ring.
#ifndef OZK_I8_BKB
#define OZK_I8_BKB 128
#endif
constexpr int TC = 128, BKB = OZK_I8_BKB;     // tile C columns (MMA M), k bytes per stage
static_assert(BKB == 128 || BKB == 64, "operand stage depth");
#ifndef OZK_I8_GROUPM
#define OZK_I8_GROUPM 8
#endif
constexpr int kGroupM = OZK_I8_GROUPM;  // tile rows per rasterization group
// binary64 TD/QD: 6 epilogue warpgroups over 48-row tiles, levels read in place
// from 2 TMEM buffers (TD/QD slice GEMM 178-180 / 339 ms vs 188 / 361 with the
// DD shape below; their epilogue is FP64-bound, more warps hide more latency)
#ifndef OZK_I8_EG
#define OZK_I8_EG 6
#endif
#ifndef OZK_I8_CM
#define OZK_I8_CM 2
#endif
#ifndef OZK_I8_TR
#define OZK_I8_TR 48
#endif
#ifndef OZK_I8_NB
#define OZK_I8_NB 2
#endif
// DD: 4 warpgroups over 64-row tiles in drain mode (73.6 ms vs 78.1 with the
// TD/QD shape: DD is operand-traffic bound, the larger tile wins; TR 80 = 64)
#ifndef OZK_I8_DD_EG
#define OZK_I8_DD_EG 4
#endif
#ifndef OZK_I8_DD_TR
#define OZK_I8_DD_TR 64
#endif
#ifndef OZK_I8_DD_NB
#define OZK_I8_DD_NB 1
#endif
#ifndef OZK_I8_EPI_UNROLL
#define OZK_I8_EPI_UNROLL 1
#endif
// trips of the K-word ping-pong loop unrolled (2: DD/TD/QD/TS 76.0/191.1/370.5/102.7
// ms vs 73.2/189.8/362.2/101.0 with 1 -- more code, no more overlap)
constexpr int kEpiUnroll = OZK_I8_EPI_UNROLL;
#ifndef OZK_I8_TS_EG
#define OZK_I8_TS_EG 7
#endif
#ifndef OZK_I8_TS_TR
#define OZK_I8_TS_TR 112
#endif
// TS (one level per pair): TMEM accumulator buffers; 4 = two pairs share each
// C read-modify-write while the MMAs fill the other two (TS slice GEMM 92.5 ->
// 90.0 ms vs 2 buffers, bit-identical; binary64 formats need 240-320 columns
// per buffer, so 4 do not fit).  8 buffers (4 pairs per pass) need 64-row
// tiles: 112 ms with 4 epilogue warpgroups, 129 with 2 -- worse.
// TS epilogue K-word compares on the integer bits (1) or as FP32 compares (0):
// same results; 1 measured faster (90.1 vs 91.7 ms) although the TS epilogue
// is issue-bound and integer ops dominate its samples
#ifndef OZK_I8_TS_INTCMP
#define OZK_I8_TS_INTCMP 1
#endif
#ifndef OZK_I8_TS_NB
#define OZK_I8_TS_NB 4
#endif
#ifndef OZK_I8_PACE
#define OZK_I8_PACE 1
#endif
#ifndef OZK_I8_CN
#define OZK_I8_CN 1
#endif
constexpr int kSmemBudget = 221 * 1024;       // operand ring

// Compile-time shape of one engine instance.
//   W   word type of C (double: DD/TD/QD, float: TS)
//   ND  int8 digits per slice integer (3 for binary64 slices at l > 128; 1 for
//       TS slices at l > 1024, where |M| <= 2^(24 - sigma) <= 64; 2 below)
//   TR  tile C rows per digit (MMA N); 2*ND-1 level accumulators of TR TMEM
//       columns each, stacked MMA width ND*TR <= 256, two accumulator buffers
//   EG  epilogue warpgroups; each owns TR/EG rows of the tile
//   NB  accumulator buffers in TMEM: 2 = the epilogue reads the levels in place
//       while the next pair's MMAs fill the other buffer; 1 = the epilogue
//       drains the levels to registers first and releases TMEM at once (taller
//       tiles fit: 5 levels x TR <= 512)
template <int K, typename W, int ND, int TR, int EG, int NB = 2>
struct I8Cfg {
    static constexpr int kLevels = 2 * ND - 1;
    static constexpr int kBTile = TC * BKB;   // one B digit (C columns), MMA operand A
    static constexpr int kATile = TR * BKB;   // one A digit (C rows), MMA operand B
    static constexpr int kStageBytes = ND * (kATile + kBTile);
    static constexpr int kStages = kSmemBudget / kStageBytes < 8 ? kSmemBudget / kStageBytes : 8;
    // + 1024 alignment slack + barriers (2 per stage, 2 per TMEM buffer) and the TMEM word
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 512;
    static constexpr int kBufCols = kLevels * TR;  // one accumulator buffer
    static constexpr int kTmemCols = NB * kBufCols <= 32 ? 32 : NB * kBufCols <= 64 ? 64
                                   : NB * kBufCols <= 128 ? 128 : NB * kBufCols <= 256 ? 256 : 512;
    static constexpr int kThreads = (4 + 4 * EG) * 32;
    static constexpr int kEpiRows = TR / EG;  // C rows per epilogue thread
    // rows per K-word update step; two steps (ping-pong C buffers) per loop trip
#ifdef OZK_I8_CHUNK
    static constexpr int kChunk = OZK_I8_CHUNK;
#else
    static constexpr int kChunk = (K == 2 && sizeof(W) == 8 && EG == 2) ? 4 : 2;
#endif
    // register split between the producer/MMA warpgroup and the epilogue:
    // setmaxnreg.inc blocks until the registers released by the .dec are
    // available, so the epilogue may grow only by what the first warpgroup
    // gives back from the launch allocation (65536 / threads, rounded to 8)
    static constexpr int kLaunchRegs = (65536 / ((4 + 4 * EG) * 32)) / 8 * 8;
    static constexpr int kEpiRegs =
        (kLaunchRegs + (kLaunchRegs - 40) / EG) / 8 * 8 > 232
            ? 232 : (kLaunchRegs + (kLaunchRegs - 40) / EG) / 8 * 8;
    static_assert(kStages >= 2, "operand ring too small");
    static_assert((2 * kStages + 2 * NB) * 8 + 4 <= 512, "barrier area");
    static_assert(NB * kBufCols <= 512 && (NB == 1 || NB == 2 || NB == 4 || NB == 8),
                  "TMEM accumulator buffers");
    static_assert(NB == 2 || kEpiRows % 4 == 0, "drain width");
    static_assert(ND * TR <= 256 && TR % 16 == 0, "stacked MMA width");
    static_assert(kATile % (8 * BKB) == 0, "A-digit tiles must stack in 8-row swizzle groups");
    static_assert(kEpiRows % (2 * kChunk) == 0, "epilogue rows per ping-pong trip");
    static_assert(40 * 128 + kEpiRegs * 128 * EG <= kLaunchRegs * (4 + 4 * EG) * 32,
                  "setmaxnreg pool");
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
    void* c;           // K-word AoS C, row stride ldc elements (PR: binary64 products)
    size_t ldc;
    size_t pair_stride;  // PR: doubles between consecutive pair products
    int c_init;          // 1: the first pair of the list starts C from zero; 0: C holds a
                         //    running sum (a later chunk of a long pair list)
    // wave pacing (see the producer): pace[s] counts the clusters that have
    // started global step s = wave * npairs + pair; null disables pacing
    unsigned int* pace;
    int pace_slack;
    // LU: after the list's last pair, A22 -= sum (row stride lu_lda) instead of
    // the C store (lu_final: this launch holds the last pair)
    double* lu_a22;
    size_t lu_lda;
    int lu_final;
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
// UMMA shared-memory descriptor: K-major operand, BKB-byte swizzle (layout type
// 2 = 128B, 4 = 64B), 8-row groups 8*BKB bytes apart (CuTe mma_sm100_desc.hpp
// SmemDescriptor, version 1 = Blackwell).
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr) {
    constexpr uint64_t kLayout = BKB == 128 ? 2 : 4;
    return (uint64_t)((saddr >> 4) & 0x3fff) | ((uint64_t)1 << 16) |
           ((uint64_t)((8 * BKB) >> 4) << 32) | ((uint64_t)1 << 46) | (kLayout << 61);
}
// L2 sector promotion of the operand TMA loads (OZK_I8_L2PROMO: 0 none, 1 64B,
// 2 128B, 3 256B)
#ifndef OZK_I8_L2PROMO
#define OZK_I8_L2PROMO 3
#endif
constexpr CUtensorMapL2promotion kL2Promo =
    OZK_I8_L2PROMO == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
    : OZK_I8_L2PROMO == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
    : OZK_I8_L2PROMO == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                          : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
constexpr CUtensorMapSwizzle kTmaSwizzle =
    BKB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
// Multicast variants for thread-block clusters: the tile lands at the same
// shared-memory offset in every CTA of ctaMask and signals each one's barrier
// at the same offset; the commit arrives on the barrier of every CTA in the mask.
__device__ __forceinline__ void tma_load_4d_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                               int c0, int c1, int c2, int c3, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "h"(mask)
        : "memory");
}
[[maybe_unused]] __device__ __forceinline__ void tma_load_4d_h(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                              int c0, int c1, int c2, int c3, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(pol)
        : "memory");
}
[[maybe_unused]] __device__ __forceinline__ void tma_load_4d_mc_h(uint32_t dst, const CUtensorMap* map,
                                                 uint32_t bar, int c0, int c1, int c2, int c3,
                                                 uint16_t mask, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster.L2::cache_hint [%0], [%1, {%3, %4, %5, %6}], [%2], %7, %8;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "h"(mask), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void umma_commit_mc(uint32_t bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
        : "memory");
}

template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, int32_t* v) {
    static_assert(N == 2 || N == 4 || N == 8 || N == 16, "tmem_ld width");
    if constexpr (N == 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
            "%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
    } else if constexpr (N == 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                       "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr));
    } else if constexpr (N == 2) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];"
                     : "=r"(v[0]), "=r"(v[1]) : "r"(taddr));
    } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(taddr));
    }
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

// The exact slice product s * 2^e (s: the recombined int64 level sum, exact in
// W: |s| < 2^53 for binary64, < 2^24 for the TS products) built with integer
// operations only: leading-one position, mantissa shift, exponent field.  The
// FP64 pipe is the one the epilogue contends on with the tensor cores, and this
// replaces the two-DADD + FMA conversion and the scaling multiply.  Results
// that would be subnormal or overflow (and any |s| too wide) take the
// floating-point path, so the value is identical either way.
// Off: same-box A/B (profiles/r02_variants_intconv.log) measured it no faster
// for TD/QD/DD and 3 % slower for TS -- the extra integer instructions cost more
// issue slots than the four FP64 operations they replace save.
#ifndef OZK_I8_INTCONV
#define OZK_I8_INTCONV 0
#endif
template <typename W>
__device__ __forceinline__ W scaled_int_to(long long s, int e) {
    constexpr int M = sizeof(W) == 8 ? 52 : 23;
    constexpr int B = sizeof(W) == 8 ? 1023 : 127;
    if (s == 0) return W(0);
    const unsigned long long a = s < 0 ? 0ull - (unsigned long long)s : (unsigned long long)s;
    const int msb = 63 - __clzll((long long)a);
    const int be = msb + e + B;
    if (msb > M || be <= 0 || be >= 2 * B + 1) return (W)ldexp_fast(i64_to_f64_exact(s), e);
    const unsigned long long m = (a << (M - msb)) & ((1ull << M) - 1);
    if constexpr (sizeof(W) == 8) {
        const unsigned long long bits =
            (s < 0 ? (1ull << 63) : 0ull) | ((unsigned long long)be << 52) | m;
        return __longlong_as_double((long long)bits);
    } else {
        const unsigned bits = (s < 0 ? 0x80000000u : 0u) | ((unsigned)be << 23) | (unsigned)m;
        return __uint_as_float(bits);
    }
}
using ProdT = long long;  // the exact integer slice product as read from TMEM
// TS (binary32 words): the product fits 24 bits (it is exact in binary32), so
// it converts exactly with one I2F and scales exactly with one FMUL by a
// bit-built power of two whenever the result is a normal float -- no FP64 in
// the TS epilogue.  Subnormal results, exponents outside the binary32 range and
// wider integers take the binary64 path, so the value is identical either way.
// Off: neutral on the B200 (TS D=15 -0.8 %, D=12 +1.3 %, profiles/r02_variants_tsconv.log).
#ifndef OZK_I8_TS_F32CONV
#define OZK_I8_TS_F32CONV 0
#endif
template <typename W>
__device__ __forceinline__ W scale_prod(ProdT s, int e) {
    if constexpr (sizeof(W) == 4 && OZK_I8_TS_F32CONV) {
        if (s > -(1ll << 24) && s < (1ll << 24) && e >= -126 && e <= 127) {
            const float p = __fmul_rn(__ll2float_rn(s), __uint_as_float((unsigned)(e + 127) << 23));
            const unsigned bits = __float_as_uint(p);
            if ((bits & 0x7f800000u) != 0u || (bits & 0x7fffffffu) == 0u) return p;  // normal or 0
        }
        return (W)ldexp_fast(i64_to_f64_exact(s), e);
    } else if constexpr (OZK_I8_INTCONV) {
        return scaled_int_to<W>(s, e);
    } else {
        return (W)ldexp_fast(i64_to_f64_exact(s), e);
    }
}

// C accesses with an L2 eviction-priority hint (OZK_I8_CHINT >= 1: C loads and
// stores evict_last; 2: also the operand TMA loads evict_first).  Off: with
// wave pacing both measured within noise / worse (n=8192 DD/TD/QD: evict_last
// 72.2/191.4/353.4 ms vs 73.8/187.3/359.7; +evict_first 79.9/201.5/363.2).
#ifndef OZK_I8_CHINT
#define OZK_I8_CHINT 0
#endif
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
[[maybe_unused]] __device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double2 ld2h(const double* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld1h(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st2h(double* p, double a, double b, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(a), "d"(b),
                 "l"(pol) : "memory");
}
__device__ __forceinline__ void st1h(double* p, double a, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(a), "l"(pol)
                 : "memory");
}

// One K-word C element as few, wide memory operations.  kVec (16-byte aligned
// C base, binary64 words): DD one 16-byte access, QD two; TD one 16-byte and
// one 8-byte access whose order follows the parity q of the element's word
// offset, so every lane issues the same instruction shape.  Otherwise (TS, or
// a C base that is only 8-byte aligned) one access per word.
template <int K, typename W>
__device__ __forceinline__ void ld_kword(const W* p, int q, bool vec, W (&w)[K],
                                         uint64_t pol = 0) {
    if constexpr (sizeof(W) == 8 && (K == 2 || K == 4)) {
        if (vec) {
#pragma unroll
            for (int h = 0; h < K / 2; ++h) {
                const double2 v = OZK_I8_CHINT ? ld2h(p + 2 * h, pol)
                                               : *reinterpret_cast<const double2*>(p + 2 * h);
                w[2 * h] = v.x;
                w[2 * h + 1] = v.y;
            }
            return;
        }
    } else if constexpr (sizeof(W) == 8 && K == 3) {
        if (vec) {
            const double2 v = OZK_I8_CHINT ? ld2h(p + q, pol)
                                           : *reinterpret_cast<const double2*>(p + q);
            const double t = OZK_I8_CHINT ? ld1h(p + (q ? 0 : 2), pol) : p[q ? 0 : 2];
            w[0] = q ? t : v.x;
            w[1] = q ? v.x : v.y;
            w[2] = q ? v.y : t;
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) w[k] = p[k];
}
template <int K, typename W>
__device__ __forceinline__ void st_kword(W* p, int q, bool vec, const W (&w)[K],
                                         uint64_t pol = 0) {
    if constexpr (sizeof(W) == 8 && (K == 2 || K == 4)) {
        if (vec) {
#pragma unroll
            for (int h = 0; h < K / 2; ++h) {
                if (OZK_I8_CHINT)
                    st2h(p + 2 * h, w[2 * h], w[2 * h + 1], pol);
                else
                    *reinterpret_cast<double2*>(p + 2 * h) = make_double2(w[2 * h], w[2 * h + 1]);
            }
            return;
        }
    } else if constexpr (sizeof(W) == 8 && K == 3) {
        if (vec) {
            const double2 v = q ? make_double2(w[1], w[2]) : make_double2(w[0], w[1]);
            const double t = q ? w[0] : w[2];
            if (OZK_I8_CHINT) {
                st2h(p + q, v.x, v.y, pol);
                st1h(p + (q ? 0 : 2), t, pol);
            } else {
                *reinterpret_cast<double2*>(p + q) = v;
                p[q ? 0 : 2] = t;
            }
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) p[k] = w[k];
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

// Diagnostic timeline (build with -DOZK_I8_TRACE, tools/i8_trace.py): SM clock
// stamps of CTA 0's first kTracePairs (tile, pair) steps -- MMA issuer: wait for
// TMEM, TMEM granted, last MMA issued; epilogue warp 4: wait start, levels
// ready, TMEM released, K-word update done.
#ifdef OZK_I8_TRACE
constexpr int kTracePairs = 512;
__device__ unsigned long long g_i8_trace[kTracePairs][8];
__device__ __forceinline__ void trace_stamp(int step, int slot, bool on) {
    if (on && blockIdx.x == 0 && step < kTracePairs) g_i8_trace[step][slot] = clock64();
}
#else
__device__ __forceinline__ void trace_stamp(int, int, bool) {}
#endif

// CM x CN thread-block cluster: CTAs (cm, cn) own tile (gm*CM + cm, gn*CN + cn)
// of tile group (gm, gn).  The CM CTAs of a cluster column share the B-digit
// tile (same C columns): each loads TC/CM of its rows and multicasts them; the
// CN CTAs of a cluster row share the A-digit tile the same way.  A stage of CTA
// x is written by x's cluster row and column, so its empty barrier counts
// CM + CN - 1 MMA completions, each CTA's commit arriving on all of them.
// PR (parity hook, ozk_pair_products_digits_device): instead of the K-word
// accumulation, every exact slice product C_ab is stored as binary64 into its
// own plane (products[p][row][col]).
// LU (blocked-LU trailing update, ozk_lu_trailing_update): the list's last
// pair subtracts the finished K-word sum from A22 in place of the C store.
template <int K, typename W, int ND, int TR, int EG, bool kVec, int CM, int CN, int NB,
          bool PR = false, bool LU = false>
__global__ void __launch_bounds__(I8Cfg<K, W, ND, TR, EG, NB>::kThreads, 1)
pair_gemm_i8_kernel(const __grid_constant__ MapsI8 maps, const __grid_constant__ PairChunk pairs,
                    I8Problem prob, int tiles_m, int tiles_n) {
    constexpr int kCluster = CM * CN;
    static_assert((TC / CM) % 8 == 0 && (TR / CN) % 8 == 0, "multicast slices of 8-row atoms");
    using Cfg = I8Cfg<K, W, ND, TR, EG, NB>;
    constexpr int kStages = Cfg::kStages, kStageBytes = Cfg::kStageBytes;
    constexpr int kATile = Cfg::kATile, kBTile = Cfg::kBTile, kEpiRows = Cfg::kEpiRows;
    constexpr int kTmemCols = Cfg::kTmemCols, kLevels = Cfg::kLevels, kBufCols = Cfg::kBufCols;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    // bars: full[S], empty[S], tmem_full[NB], tmem_empty[NB] ; then the TMEM base word
    const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * kStages;
    const uint32_t tfull0 = empty0 + 8 * kStages, tempty0 = tfull0 + 8 * NB;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 2 * NB);
    const uint32_t ring = smem_u32(smem);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_kb = (int)((prob.l + BKB - 1) / BKB);
    const int npairs = pairs.count;
    // cluster coordinates and the persistent loop over tile groups
    const int crank = kCluster > 1 ? (int)cluster_ctarank() : 0;
    const int cm = crank % CM, cn = crank / CM;
    const int groups_m = (tiles_m + CM - 1) / CM, groups_n = (tiles_n + CN - 1) / CN;
    const int num_groups = groups_m * groups_n;
    const int cluster_id = blockIdx.x / kCluster, num_clusters = gridDim.x / kCluster;
    auto tile_of_group = [&](int g) {
        const TileCoord gc = tile_of(g, groups_m, groups_n);
        return TileCoord{gc.tm * CM + cm, gc.tn * CN + cn};
    };
    // CTAs sharing this CTA's B tile (same cn) and A tile (same cm)
    uint16_t col_mask = 0, row_mask = 0;
#pragma unroll
    for (int i = 0; i < CM; ++i) col_mask |= (uint16_t)(1u << (i + cn * CM));
#pragma unroll
    for (int j = 0; j < CN; ++j) row_mask |= (uint16_t)(1u << (cm + j * CM));

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, CM + CN - 1);
        }
        for (int b = 0; b < NB; ++b) {
            mbar_init(tfull0 + 8 * b, 1);
            mbar_init(tempty0 + 8 * b, 4 * EG);  // one arrive per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "n"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    if constexpr (kCluster > 1)
        cluster_sync();  // peers' barriers initialised before any multicast
    else
        __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
      if (warp == 0 && lane == 0) {
        // ---------------- TMA producer ----------------
        // stage layout: ND B-digit tiles (TC x BKB), then ND A-digit tiles
        // (TR x BKB) back to back = the stacked MMA N operand
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.b)));
        int stage = 0;
        uint32_t phase = 0;
        int wave = 0;
        bool pace = prob.pace != nullptr;
#if OZK_I8_CHINT >= 2
        const uint64_t opol = l2_policy_evict_first();
#endif
        for (int g = cluster_id; g < num_groups; g += num_clusters, ++wave) {
            const TileCoord tc = tile_of_group(g);
            for (int p = 0; p < npairs; ++p) {
                const int al = pairs.alpha[p], be = pairs.beta[p];
                if (pace) {
                    // Wave pacing: all clusters stream the same slice pair of
                    // neighbouring tiles, but persistent clusters drift apart and
                    // the live panels then span many slices and thrash L2 (1 TB of
                    // DRAM reads for one TD n=8192 GEMM).  Start step s only after
                    // every cluster has started step s - slack.  Pacing is only a
                    // hint: a wait that exceeds ~5 ms (a cluster not co-resident,
                    // e.g. the GPU shared with other work) turns it off.
                    const int st = wave * npairs + p, wait = st - prob.pace_slack;
                    if (wait >= 0) {
                        const int w2 = wait / npairs;
                        const int left = num_groups - w2 * num_clusters;
                        const unsigned target = (unsigned)(left < num_clusters ? left : num_clusters);
                        const volatile unsigned* slot = prob.pace + wait;
                        for (int spin = 0; *slot < target; ++spin) {
                            if (spin > 20000) {
                                pace = false;
                                break;
                            }
                            __nanosleep(256);
                        }
                    }
                    if (crank == 0 && pace) atomicAdd(prob.pace + st, 1u);
                }
                for (int kb = 0; kb < num_kb; ++kb) {
                    mbar_wait(empty0 + 8 * stage, phase ^ 1);
                    const uint32_t full = full0 + 8 * stage;
#if defined(OZK_I8_EPI_MODE) && OZK_I8_EPI_MODE == 5
                    mbar_arrive(full);  // diagnostic: no operand traffic (stale tiles)
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                    continue;
#endif
                    mbar_expect_tx(full, kStageBytes);
                    const uint32_t sa = ring + stage * kStageBytes;
#pragma unroll
                    for (int dgt = 0; dgt < ND; ++dgt) {
                        // this CTA's slice of the shared tiles (whole tiles when unshared)
                        const uint32_t db = sa + dgt * kBTile + cm * (TC / CM) * BKB;
                        const uint32_t da = sa + ND * kBTile + dgt * kATile + cn * (TR / CN) * BKB;
                        const int rb = tc.tn * TC + cm * (TC / CM), ra = tc.tm * TR + cn * (TR / CN);
#if OZK_I8_CHINT >= 2
                        if constexpr (CM > 1)
                            tma_load_4d_mc_h(db, &maps.b, full, kb * BKB, rb, dgt, be, col_mask, opol);
                        else
                            tma_load_4d_h(db, &maps.b, full, kb * BKB, rb, dgt, be, opol);
                        if constexpr (CN > 1)
                            tma_load_4d_mc_h(da, &maps.a, full, kb * BKB, ra, dgt, al, row_mask, opol);
                        else
                            tma_load_4d_h(da, &maps.a, full, kb * BKB, ra, dgt, al, opol);
#else
                        if constexpr (CM > 1)
                            tma_load_4d_mc(db, &maps.b, full, kb * BKB, rb, dgt, be, col_mask);
                        else
                            tma_load_4d(db, &maps.b, full, kb * BKB, rb, dgt, be);
                        if constexpr (CN > 1)
                            tma_load_4d_mc(da, &maps.a, full, kb * BKB, ra, dgt, al, row_mask);
                        else
                            tma_load_4d(da, &maps.a, full, kb * BKB, ra, dgt, al);
#endif
                    }
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
      } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        // The whole warp runs the loop so every descriptor is warp-uniform (kept
        // in uniform registers) and one elected lane issues; descriptors of a
        // stage are its base plus compile-time offsets.
        // kind::i8 instruction descriptors: D s32, A/B signed 8-bit, K-major,
        // M = 128, N = TR (one digit) or ND*TR (stacked digits)
        // (CuTe mma_sm100_desc.hpp InstrDescriptor)
        constexpr uint32_t idesc1 = (2u << 4) | (1u << 7) | (1u << 10) |
                                    ((uint32_t)(TR >> 3) << 17) | ((uint32_t)(TC >> 4) << 24);
        constexpr uint32_t idescN = (2u << 4) | (1u << 7) | (1u << 10) |
                                    ((uint32_t)((ND * TR) >> 3) << 17) | ((uint32_t)(TC >> 4) << 24);
        int stage = 0;
        uint32_t phase = 0;
        int step = 0;
        for (int g = cluster_id; g < num_groups; g += num_clusters) {
            for (int p = 0; p < npairs; ++p, ++step) {
                // accumulator buffer step % NB, free once the epilogue of step - NB is done
                const int buf = step % NB;
                trace_stamp(step, 0, lane == 0);
                mbar_wait(tempty0 + 8 * buf, ((step / NB) & 1) ^ 1);
                trace_stamp(step, 1, lane == 0);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t acc0 = tmem + buf * kBufCols;
#ifdef OZK_I8_TRACE
                unsigned long long full_wait = 0;
#endif
                for (int kb = 0; kb < num_kb; ++kb) {
#ifdef OZK_I8_TRACE
                    const unsigned long long w0 = clock64();
                    mbar_wait(full0 + 8 * stage, phase);
                    full_wait += clock64() - w0;
#else
                    mbar_wait(full0 + 8 * stage, phase);
#endif
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sb = ring + stage * kStageBytes;  // B digits (M side)
                    const uint64_t db = sw_desc(sb);              // B digit 0, k-chunk 0
                    const uint64_t da = sw_desc(sb + ND * kBTile);  // A digits (N side)
                    if (elect_one()) {
#pragma unroll
                        for (int kc = 0; kc < BKB / 32; ++kc) {
#if defined(OZK_I8_EPI_MODE) && OZK_I8_EPI_MODE == 6
                            if (kc > 0) break;  // diagnostic: only the first chunk's MMAs
#endif
                            if (kc == 0 && kb == 0) {
                                // first chunk: single-digit products level by level, the
                                // first of each level overwriting its accumulator block
#pragma unroll
                                for (int lvl = 0; lvl < kLevels; ++lvl) {
#pragma unroll
                                    for (int t = 0; t < ND; ++t) {
                                        const int u = lvl - t;
                                        if (u < 0 || u >= ND) continue;
                                        const bool first =
                                            t == (lvl - ND + 1 > 0 ? lvl - ND + 1 : 0);
                                        umma_i8(acc0 + lvl * TR, db + (t * kBTile >> 4),
                                                da + (u * kATile >> 4), idesc1, first ? 0u : 1u);
                                    }
                                }
                            } else {
#pragma unroll
                                for (int t = 0; t < ND; ++t)
                                    umma_i8(acc0 + t * TR, db + ((t * kBTile + kc * 32) >> 4),
                                            da + (kc * 32 >> 4), idescN, 1u);
                            }
                        }
                        // frees the stage (here and in every CTA that multicasts into
                        // it) when the MMAs retire; commits track this lane's MMAs
                        if constexpr (kCluster > 1)
                            umma_commit_mc(empty0 + 8 * stage, (uint16_t)(col_mask | row_mask));
                        else
                            umma_commit(empty0 + 8 * stage);
                    }
                    __syncwarp();
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (elect_one()) umma_commit(tfull0 + 8 * buf);
                __syncwarp();
                trace_stamp(step, 2, lane == 0);
#ifdef OZK_I8_TRACE
                if (lane == 0 && blockIdx.x == 0 && step < kTracePairs)
                    g_i8_trace[step][7] = full_wait;
#endif
            }
        }
      }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(Cfg::kEpiRegs));
        // ---------------- epilogue warpgroups ----------------
        // warpgroup eg owns rows [eg*kEpiRows, (eg+1)*kEpiRows) of every tile for
        // every pair (no two threads ever touch the same C element); warp % 4
        // selects the 32 TMEM lanes = C columns it may access, one per thread.
        // The levels are read from TMEM chunk by chunk (no register copy of
        // the tile), and the buffer is released after the last chunk: the
        // MMAs of the next pair run meanwhile in the other buffer.
        constexpr int kChunk = Cfg::kChunk;
        constexpr int PG = NB >= 4 ? NB / 2 : 1;  // slice pairs per C read-modify-write
        // K-word compares on integer halves where FP64 is the contended pipe
        // (binary64 words); binary32 (TS) words: see OZK_I8_TS_INTCMP
        constexpr bool kEpiIntCmp = sizeof(W) == 8 ? true : (OZK_I8_TS_INTCMP != 0);
        const int eg = (warp - 4) / 4;
        const int wq = warp % 4;
        const uint32_t tlane = tmem + ((uint32_t)(wq * 32) << 16) + eg * kEpiRows;
        int step = 0;
        const bool tracer = warp == 4 && lane == 0;
        const uint64_t cpol = OZK_I8_CHINT ? l2_policy_evict_last() : 0;
        for (int g = cluster_id; g < num_groups; g += num_clusters) {
            const TileCoord tc = tile_of_group(g);
            const size_t col = (size_t)tc.tn * TC + wq * 32 + lane;
            const size_t row0 = (size_t)tc.tm * TR + eg * kEpiRows;
            const bool col_ok = col < prob.n;
            // out-of-range lanes and rows read a valid element and never store
            const size_t col_c = col_ok ? col : prob.n - 1;
            for (int p = 0; p < npairs;) {
                // PG = NB / 2 (>= 4 TMEM buffers): consecutive pairs p .. p+np-1
                // share one C read-modify-write, their K-word adds in the
                // reference order, while the MMAs fill the other NB / 2 buffers
                const int np = npairs - p < PG ? npairs - p : PG;
                int gbq[PG];
                const int* gapq[PG];
                uint32_t tbufq[PG];
#pragma unroll
                for (int q = 0; q < PG; ++q) {
                    const int pq = q < np ? p + q : p;
                    const int al = pairs.alpha[pq], be = pairs.beta[pq];
                    gbq[q] = prob.gB[(size_t)be * prob.gB_stride + col_c];
                    gapq[q] = prob.gA + (size_t)al * prob.gA_stride;
                    tbufq[q] = tlane + ((step + q) % NB) * kBufCols;
                }
                const bool first = p == 0 && prob.c_init;  // C starts from zero
                const bool lu_last = LU && prob.lu_final && p + np == npairs;
                trace_stamp(step, 3, tracer);
                for (int q = 0; q < np; ++q)
                    mbar_wait(tfull0 + 8 * ((step + q) % NB), ((step + q) / NB) & 1);
                trace_stamp(step, 4, tracer);
                asm volatile("tcgen05.fence::after_thread_sync;");
                W* const cbase = static_cast<W*>(prob.c);
                auto row_of = [&](int r) -> size_t {
                    const size_t rr = row0 + r;
                    return rr < prob.m ? rr : prob.m - 1;
                };
                auto load_chunk = [&](int r, W (&w)[kChunk][K]) {
#pragma unroll
                    for (int j = 0; j < (PR ? 0 : kChunk); ++j) {
                        const size_t e = row_of(r + j) * prob.ldc + col_c;
#if defined(OZK_I8_EPI_MODE) && OZK_I8_EPI_MODE == 1
                        if (true) {  // diagnostic: no C reads
#else
                        if (first) {
#endif
#pragma unroll
                            for (int k = 0; k < K; ++k) w[j][k] = W(0);
                        } else {
                            ld_kword<K>(cbase + e * K, (int)(e & 1), kVec, w[j], cpol);
                        }
                    }
                };
                // levels of rows [r, r + N) recombined to the exact binary64 products
                auto read_levels = [&](int r, auto& y, uint32_t tbuf) {
                    constexpr int N = sizeof(y) / sizeof(ProdT);
                    int32_t lv[kLevels][N];
#pragma unroll
                    for (int u = 0; u < kLevels; ++u) tmem_ld<N>(tbuf + u * TR + r, lv[u]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int j = 0; j < N; ++j) {
                        long long sum = lv[0][j];
#pragma unroll
                        for (int u = 1; u < kLevels; ++u) sum += (long long)lv[u][j] << (8 * u);
                        y[j] = sum;  // the exact integer slice product (|sum| < 2^53)
                    }
                };
                // NB == 1: drain every level of this thread's rows, then release TMEM
                // so the next pair's MMAs start while the K-word updates run
                ProdT yall[NB == 1 ? kEpiRows : 1];
                if constexpr (NB == 1) {
#pragma unroll
                    for (int r = 0; r < kEpiRows; r += (kEpiRows % 16 == 0 ? 16 : 4)) {
                        ProdT (&ys)[kEpiRows % 16 == 0 ? 16 : 4] =
                            *reinterpret_cast<ProdT (*)[kEpiRows % 16 == 0 ? 16 : 4]>(yall + r);
                        read_levels(r, ys, tbufq[0]);
                    }
#if !(defined(OZK_I8_EPI_MODE) && OZK_I8_EPI_MODE == 3)
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty0 + 8 * (step % NB));
#endif
                }
                auto update_chunk = [&](int r, W (&w)[kChunk][K]) {
                    ProdT yc[PG][kChunk];
                    if constexpr (NB == 1) {
                        // this chunk's products are yall[0..kChunk); shift the rest
                        // down so every register index stays static
#pragma unroll
                        for (int j = 0; j < kChunk; ++j) yc[0][j] = yall[j];
#pragma unroll
                        for (int j = 0; j < kEpiRows - kChunk; ++j) yall[j] = yall[j + kChunk];
                    } else {
#pragma unroll
                        for (int q = 0; q < PG; ++q)
                            if (q < np) read_levels(r, yc[q], tbufq[q]);
                    }
#pragma unroll
                    for (int j = 0; j < kChunk; ++j) {
#pragma unroll
                        for (int q = 0; q < PG; ++q) {
                            if (q >= np) break;
                            const ProdT y = yc[q][j];
                            const int ga = __ldg(gapq[q] + row_of(r + j));
                            if constexpr (PR) {
                                const size_t rr = row0 + r + j;
                                if (col_ok && rr < prob.m)
                                    static_cast<double*>(prob.c)[(size_t)(p + q) * prob.pair_stride +
                                                                 rr * prob.ldc + col] =
                                        scale_prod<double>(y, ga + gbq[q]);
                                continue;
                            }
                            // exact scaled slice product (a TS product is exact in binary32)
#if defined(OZK_I8_EPI_MODE) && OZK_I8_EPI_MODE == 2
                            w[j][0] += scale_prod<W>(y, ga + gbq[q]);  // diagnostic: no K-word add
#else
                            kw_add<K, W, kEpiIntCmp, true>(w[j], scale_prod<W>(y, ga + gbq[q]));
#endif
                        }
                    }
#pragma unroll
                    for (int j = 0; j < (PR ? 0 : kChunk); ++j) {
                        const size_t rr = row0 + r + j;
                        if (col_ok && rr < prob.m) {
                            if constexpr (LU) {
                                if (lu_last) {
                                    // A22 -= sum (lu.hpp:121-124; MultiFloat -=
                                    // MultiFloat = x + (-y), multifloat.hpp:300,178-199)
                                    double* ap = prob.lu_a22 + (rr * prob.lu_lda + col) * K;
                                    double x[K], ny[K];
#pragma unroll
                                    for (int k = 0; k < K; ++k) x[k] = ap[k];
                                    kw_neg<K>(w[j], ny);
                                    kw_add_kw<K>(x, ny);
#pragma unroll
                                    for (int k = 0; k < K; ++k) ap[k] = x[k];
                                    continue;
                                }
                            }
                            const size_t e = rr * prob.ldc + col;
                            st_kword<K>(cbase + e * K, (int)(e & 1), kVec, w[j], cpol);
                        }
                    }
                };
                W ca[kChunk][K], cb[kChunk][K];
                load_chunk(0, ca);
#pragma unroll kEpiUnroll
                for (int r = 0; r < kEpiRows; r += 2 * kChunk) {
                    load_chunk(r + kChunk, cb);  // in flight during the update of ca
                    update_chunk(r, ca);
                    if (r + 2 * kChunk < kEpiRows) load_chunk(r + 2 * kChunk, ca);
                    update_chunk(r + kChunk, cb);
                }
#if defined(OZK_I8_EPI_MODE) && OZK_I8_EPI_MODE == 3
                if (true) {  // diagnostic: the next pair's MMAs wait for the whole epilogue
#else
                if constexpr (NB >= 2) {
#endif
                    // all levels read: hand the buffers back to the MMA issuer
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    __syncwarp();
                    if (lane == 0)
                        for (int q = 0; q < np; ++q) mbar_arrive(tempty0 + 8 * ((step + q) % NB));
                }
                trace_stamp(step, 5, tracer);
                trace_stamp(step, 6, tracer);
                p += np;
                step += np;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    // no CTA leaves while a peer may still multicast into it or arrive on it
    if constexpr (kCluster > 1)
        cluster_sync();
    else
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

// Persistent clusters: as many as can be co-resident (GPC packing can leave
// SMs idle for clusters > 1); the occupancy query is made once per instance.
template <int K, typename W, int ND, int TR, int EG, int CM, int CN, int NB>
int resident_clusters(int num_sms) {
    using Cfg = I8Cfg<K, W, ND, TR, EG, NB>;
    constexpr int kCluster = CM * CN;
    static std::atomic<int> cached{0};  // per instance; one GPU model per process
    if (const int c = cached.load(std::memory_order_relaxed); c > 0) return c;
    int clusters = num_sms / kCluster;
    if constexpr (kCluster > 1) {
        // the vectorised-C instance has the same resources as the scalar one
        auto kern = pair_gemm_i8_kernel<K, W, ND, TR, EG, false, CM, CN, NB>;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg::kSmemBytes) != cudaSuccess)
            return 0;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kCluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(Cfg::kThreads);
        cfg.dynamicSmemBytes = Cfg::kSmemBytes;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(clusters * kCluster);
        int active = 0;
        if (cudaOccupancyMaxActiveClusters(&active, kern, &cfg) == cudaSuccess && active > 0 &&
            active < clusters)
            clusters = active;
    }
    cached.store(clusters, std::memory_order_relaxed);
    return clusters;
}

template <int K, typename W, int ND, int TR, int EG, int CM, int CN, int NB>
I8Geometry geometry_typed(int num_sms) {
    I8Geometry g;
    g.group_rows = CM * TR;
    g.group_cols = CN * TC;
    g.clusters = resident_clusters<K, W, ND, TR, EG, CM, CN, NB>(num_sms);
    g.cluster_sms = CM * CN;
    return g;
}

template <int K, typename W, int ND, int TR, int EG = 2, int CM = 1, int CN = 1, int NB = 2,
          bool PR = false>
cudaError_t launch_i8_chunk(const I8Operands& op, const PairChunk& pairs, cudaStream_t st,
                            int num_sms, bool lu_final) {
    using Cfg = I8Cfg<K, W, ND, TR, EG, NB>;
    auto encode = get_encode_i8();
    if (!encode) return cudaErrorNotSupported;
    MapsI8 maps;
    {
        cuuint64_t dims[4] = {op.l, op.m, (cuuint64_t)ND, (cuuint64_t)op.d};
        cuuint64_t strides[3] = {op.a_ld, op.a_digit_stride, op.a_slice_stride};
        cuuint32_t box[4] = {BKB, TR / CN, 1, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (encode(&maps.a, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(op.a), dims,
                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, kTmaSwizzle,
                   kL2Promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    {
        cuuint64_t dims[4] = {op.l, op.n, (cuuint64_t)ND, (cuuint64_t)op.d};
        cuuint64_t strides[3] = {op.b_ld, op.b_digit_stride, op.b_slice_stride};
        cuuint32_t box[4] = {BKB, TC / CM, 1, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (encode(&maps.b, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(op.b), dims,
                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, kTmaSwizzle,
                   kL2Promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    I8Problem prob;
    prob.m = op.m;
    prob.n = op.n;
    prob.l = op.l;
    prob.gA = op.gA;
    prob.gB = op.gB;
    prob.gA_stride = op.gA_stride ? op.gA_stride : op.m;
    prob.gB_stride = op.gB_stride ? op.gB_stride : op.n;
    prob.c = op.c;
    prob.ldc = op.ldc;
    prob.pair_stride = op.pair_stride;
    prob.c_init = op.c_init ? 1 : 0;
    prob.pace = nullptr;
    prob.pace_slack = OZK_I8_PACE;
    prob.lu_a22 = op.lu_a22;
    prob.lu_lda = op.lu_lda;
    prob.lu_final = lu_final ? 1 : 0;
    const bool vec = !PR && sizeof(W) == 8 && (reinterpret_cast<uintptr_t>(op.c) & 15) == 0;
    const int tiles_m = (int)((op.m + TR - 1) / TR), tiles_n = (int)((op.n + TC - 1) / TC);
    const int num_tiles = tiles_m * tiles_n;
    if (num_tiles == 0 || pairs.count == 0) return cudaSuccess;
    auto kern = pair_gemm_i8_kernel<K, W, ND, TR, EG, false, CM, CN, NB, PR>;
    if constexpr (sizeof(W) == 8 && !PR) {
        if (op.lu_a22)
            kern = vec ? pair_gemm_i8_kernel<K, W, ND, TR, EG, true, CM, CN, NB, false, true>
                       : pair_gemm_i8_kernel<K, W, ND, TR, EG, false, CM, CN, NB, false, true>;
        else if (vec)
            kern = pair_gemm_i8_kernel<K, W, ND, TR, EG, true, CM, CN, NB>;
    } else if (op.lu_a22) {
        return cudaErrorInvalidValue;  // binary64 formats only
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    constexpr int kCluster = CM * CN;
    const int groups = ((tiles_m + CM - 1) / CM) * ((tiles_n + CN - 1) / CN);
    int clusters = resident_clusters<K, W, ND, TR, EG, CM, CN, NB>(num_sms);
    if (clusters <= 0) return cudaErrorInvalidConfiguration;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(Cfg::kThreads);
    cfg.dynamicSmemBytes = Cfg::kSmemBytes;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (groups < clusters) clusters = groups;
    cfg.gridDim = dim3(clusters * kCluster);
    // pacing counters: one per (wave, pair) step, stream-ordered scratch
    const size_t steps = (size_t)((groups + clusters - 1) / clusters) * pairs.count;
    if (OZK_I8_PACE > 0 && clusters > 1) {
        e = cudaMallocAsync(reinterpret_cast<void**>(&prob.pace), steps * sizeof(unsigned), st);
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(prob.pace, 0, steps * sizeof(unsigned), st);
        if (e != cudaSuccess) return e;
    }
    e = cudaLaunchKernelEx(&cfg, kern, maps, pairs, prob, tiles_m, tiles_n);
    if (prob.pace) {
        const cudaError_t f = cudaFreeAsync(prob.pace, st);
        if (e == cudaSuccess) e = f;
    }
    return e;
}

// Pair lists longer than one launch's parameter block: consecutive launches,
// each later chunk continuing the K-word sum in C (PR: writing further along).
template <int K, typename W, int ND, int TR, int EG = 2, int CM = 1, int CN = 1, int NB = 2,
          bool PR = false>
cudaError_t launch_i8_typed(const I8Operands& op, const PairList& pairs, cudaStream_t st,
                            int num_sms) {
    for (int q0 = 0; q0 < pairs.count; q0 += kPairsPerLaunch) {
        I8Operands o = op;
        o.c_init = op.c_init && q0 == 0;
        if (PR) o.c = static_cast<double*>(op.c) + q0 * op.pair_stride;
        const cudaError_t e = launch_i8_chunk<K, W, ND, TR, EG, CM, CN, NB, PR>(
            o, pair_chunk(pairs, q0), st, num_sms, q0 + kPairsPerLaunch >= pairs.count);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

} // namespace

cudaError_t launch_pair_products_i8(int word_bytes, const I8Operands& op, const PairList& pairs,
                                    cudaStream_t st, int num_sms) {
    // the binary64 engine shape (TD/QD); TS with its own digit counts
    if (word_bytes == 4) {
        if (op.nd == 1)
            return launch_i8_typed<3, float, 1, OZK_I8_TS_TR, OZK_I8_TS_EG, OZK_I8_CM, OZK_I8_CN,
                                   OZK_I8_TS_NB, true>(op, pairs, st, num_sms);
        if (op.nd == 2)
            return launch_i8_typed<3, float, 2, 64, 4, OZK_I8_CM, OZK_I8_CN, 2, true>(op, pairs, st,
                                                                                      num_sms);
        return cudaErrorInvalidValue;
    }
    if (op.nd != 3) return cudaErrorInvalidValue;
    return launch_i8_typed<3, double, 3, OZK_I8_TR, OZK_I8_EG, OZK_I8_CM, OZK_I8_CN, OZK_I8_NB,
                           true>(op, pairs, st, num_sms);
}

I8Geometry pair_gemm_i8_geometry(int K, int word_bytes, int nd, int num_sms) {
    if (word_bytes == 4) {
        if (K == 3 && nd == 1)
            return geometry_typed<3, float, 1, OZK_I8_TS_TR, OZK_I8_TS_EG, OZK_I8_CM, OZK_I8_CN, OZK_I8_TS_NB>(num_sms);
        if (K == 3 && nd == 2)
            return geometry_typed<3, float, 2, 64, 4, OZK_I8_CM, OZK_I8_CN, 2>(num_sms);
        return I8Geometry{};
    }
    if (nd != 3) return I8Geometry{};
    switch (K) {
    case 2: return geometry_typed<2, double, 3, OZK_I8_DD_TR, OZK_I8_DD_EG, OZK_I8_CM, OZK_I8_CN, OZK_I8_DD_NB>(num_sms);
    case 3: return geometry_typed<3, double, 3, OZK_I8_TR, OZK_I8_EG, OZK_I8_CM, OZK_I8_CN, OZK_I8_NB>(num_sms);
    case 4: return geometry_typed<4, double, 3, OZK_I8_TR, OZK_I8_EG, OZK_I8_CM, OZK_I8_CN, OZK_I8_NB>(num_sms);
    default: return I8Geometry{};
    }
}

cudaError_t launch_pair_gemm_i8(int K, int word_bytes, const I8Operands& op,
                                const PairList& pairs, cudaStream_t st, int num_sms) {
    if (word_bytes == 4) {  // TS: binary32 words, 1 or 2 digits
        if (K != 3) return cudaErrorInvalidValue;
        if (op.nd == 1)
            return launch_i8_typed<3, float, 1, OZK_I8_TS_TR, OZK_I8_TS_EG, OZK_I8_CM, OZK_I8_CN, OZK_I8_TS_NB>(op, pairs, st, num_sms);
        if (op.nd == 2)
            return launch_i8_typed<3, float, 2, 64, 4, OZK_I8_CM, OZK_I8_CN>(op, pairs, st, num_sms);
        return cudaErrorInvalidValue;
    }
    if (op.nd != 3) return cudaErrorInvalidValue;
    switch (K) {
    case 2: return launch_i8_typed<2, double, 3, OZK_I8_DD_TR, OZK_I8_DD_EG, OZK_I8_CM, OZK_I8_CN, OZK_I8_DD_NB>(op, pairs, st, num_sms);
    case 3: return launch_i8_typed<3, double, 3, OZK_I8_TR, OZK_I8_EG, OZK_I8_CM, OZK_I8_CN, OZK_I8_NB>(op, pairs, st, num_sms);
    case 4: return launch_i8_typed<4, double, 3, OZK_I8_TR, OZK_I8_EG, OZK_I8_CM, OZK_I8_CN, OZK_I8_NB>(op, pairs, st, num_sms);
    default: return cudaErrorInvalidValue;
    }
}

} // namespace ozk

#ifdef OZK_I8_TRACE
// diagnostic builds only (tools/i8_trace.py): copy CTA 0's timeline to the host
extern "C" int ozk_i8_trace_read(unsigned long long* out, int max_steps) {
    const int n = max_steps < ozk::kTracePairs ? max_steps : ozk::kTracePairs;
    return (int)cudaMemcpyFromSymbol(out, ozk::g_i8_trace, sizeof(unsigned long long) * 8 * n);
}
#endif

// api.cu -- host runtime behind the C-ABI (include/ozk.h): argument checks in
// the reference's order, device buffers from the stream-ordered pool, split
// planning, pair lists, and the launches of K1 (split.cu) and K2+K3 (gemm.cu).
//
// Reference call stack being replaced: ozaki_gemm<K> (ozaki.hpp:180-249) ->
// split_matrix (:74-147) x2 -> backend (backend.hpp:12-13) x P -> accumulate.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <functional>
#include <memory>
#include <algorithm>
#include <vector>
#include <condition_variable>
#include <thread>
#include <cstdint>
#include <tuple>
#include <initializer_list>
#include <map>

#include <sched.h>

#include "../../include/ozk.h"
#include "ozk_internal.cuh"

using namespace ozk;

namespace {

thread_local std::string g_last_error;

int word_bytes_of_fmt(int fmt) { return fmt == OZK_TS ? 4 : 8; }

// Slice-product engine: OZK_ENGINE_AUTO picks the exact INT8-digit tcgen05
// engine whenever it applies (binary64 words, D >= 2, 128 < l < 43690), else
// the FP64 DMMA engine.  Initialised from $OZK_ENGINE (auto|dmma|int8).
std::atomic<int> g_engine{-1};

int engine_setting() {
    int e = g_engine.load();
    if (e < 0) {
        e = OZK_ENGINE_AUTO;
        if (const char* v = std::getenv("OZK_ENGINE")) {
            if (!std::strcmp(v, "dmma")) e = OZK_ENGINE_DMMA;
            if (!std::strcmp(v, "int8")) e = OZK_ENGINE_INT8;
        }
        g_engine.store(e);
    }
    return e;
}

// Digits per slice integer for the INT8 engine, 0 = not applicable.  The
// slice integer on the split's grid 2^(e + sigma - S) is bounded by
// 2^(S - sigma) (S = 53 / 24, split.cu); signed
// base-256 digits hold |M| <= 127 (1), 32639 (2), 8355711 (3).  Every digit
// level (at most 3 digit products per output) stays below 2^31 for l < 43690.
int int8_digits(int fmt, size_t l, int d) {
    if (d < 2 || l >= 43690) return 0;
    int cl = 0;
    while ((size_t(1) << cl) < l) ++cl;
    const int S = word_bytes_of_fmt(fmt) == 4 ? 24 : 53;
    const int bits = S - (S + cl + 1) / 2;  // |M| <= 2^bits
    if (bits <= 6) return 1;
    if (bits <= 14) return 2;
    if (bits <= 22) return word_bytes_of_fmt(fmt) == 8 ? 3 : 0;
    return 0;  // binary64 slices at l <= 128 would need 4 digits: DMMA engine
}

bool int8_applicable(int fmt, size_t l, int d) { return int8_digits(fmt, l, d) > 0; }

ozk_status fail(ozk_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

ozk_status cuda_fail(cudaError_t e, const char* where) {
    (void)cudaGetLastError();  // clear sticky-free errors
    if (e == cudaErrorMemoryAllocation) return fail(OZK_ENOMEM, std::string(where) + ": out of device memory");
    return fail(OZK_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define OZK_CUDA(call, where)                                  \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return cuda_fail(e_, where);    \
    } while (0)

int num_sms_cached() {
    static int sms = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // keep freed pool memory: repeated calls reuse it instead of re-mapping
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
    return sms > 0 ? sms : 148;
}

// Stream-ordered device scratch, freed on scope exit.
// $OZK_POISON_SCRATCH=1 fills every scratch allocation with 0xFF bytes (NaN
// words, -1 digits and exponents) before use: a kernel that reads scratch it
// never wrote then corrupts the result, which the parity tests catch
// (tests/test_gpu_parity.py::test_poisoned_scratch_bitexact; compute-sanitizer
// is closed on this GPU pool, so this stands in for its initcheck).
bool poison_scratch() {
    const char* v = std::getenv("OZK_POISON_SCRATCH");
    return v && v[0] == '1';
}

struct DevBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    cudaError_t alloc(size_t bytes, cudaStream_t s) {
        st = s;
        cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 16, s);
        if (e == cudaSuccess && poison_scratch()) e = cudaMemsetAsync(p, 0xFF, bytes ? bytes : 16, s);
        return e;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

// Private stream for host-buffer entry points (reentrancy).
struct OwnStream {
    cudaStream_t s = nullptr;
    cudaError_t create() { return cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); }
    ~OwnStream() {
        if (s) cudaStreamDestroy(s);
    }
};

bool valid_fmt(int fmt) {
    return fmt == OZK_DD || fmt == OZK_TD || fmt == OZK_QD || fmt == OZK_TS;
}
// words per element and bytes per word of a format
int words_of(int fmt) { return fmt == OZK_TS ? 3 : fmt; }
int word_bytes_of(int fmt) { return fmt == OZK_TS ? 4 : 8; }
size_t elem_bytes(int fmt) { return (size_t)words_of(fmt) * word_bytes_of(fmt); }

// split_shift_bits (ozaki.hpp:43-48); short_bits = 53 for binary64 words, 24 for TS
int shift_bits(size_t inner, int short_bits = 53) {
    int cl = 0;
    while ((size_t(1) << cl) < inner) ++cl;
    return (short_bits + cl + 1) / 2;
}

// ozaki.hpp:209-221: alpha-major triangular set, optionally pruned
void triangular_pairs(int d, PairList& pl) {
    pl.clear();
    for (int a = 0; a < d; ++a)
        for (int b = 0; a + b < d; ++b) pl.push(a, b);
}

void pruned_pairs(int d, const double* amax, const double* bmax, double drop, PairList& pl) {
    const double lead = amax[0] * bmax[0];
    pl.clear();
    for (int a = 0; a < d; ++a)
        for (int b = 0; a + b < d; ++b) {
            if (drop > 0.0 && amax[a] * bmax[b] < drop * lead) continue;
            pl.push(a, b);
        }
}

ozk_status check_dev_err(int flag, const char* what) {
    if (flag == kDevNonFinite) return fail(OZK_EPARAM, std::string(what) + ": non-finite entry");
    if (flag == kDevTooLarge)
        return fail(OZK_EPARAM, std::string(what) + ": entries too large to shift");
    return OZK_OK;
}

// Split of a K-word matrix into slices in the operand layout (see ozk.h).
// work must hold outer*inner elements.  Returns a CUDA error code.
cudaError_t split_to_slices(int fmt, size_t rows, size_t cols, size_t ld, const void* mat, int d,
                            int side, double* slices, size_t plane_rows, void* work,
                            unsigned long long* pmax, int* err, cudaStream_t st,
                            const DigitOut& dig = DigitOut{}, bool keep_residual = false) {
    const int K = words_of(fmt), wb = word_bytes_of(fmt);
    const size_t inner = side == OZK_SIDE_ROWS ? cols : rows;
    const size_t ldk = slice_ld(inner);
    const int sigma = shift_bits(inner, wb == 4 ? 24 : 53);
    if (side == OZK_SIDE_ROWS)
        return launch_split_rows(K, wb, mat, ld, work, rows, cols, d, sigma, slices, ldk,
                                 plane_rows * ldk, pmax, err, st, dig, keep_residual);
    // columns: transpose to (cols x rows) so each column is a contiguous row
    cudaError_t e = launch_transpose(K, wb, mat, ld, work, rows, rows, cols, st);
    if (e != cudaSuccess) return e;
    return launch_split_rows(K, wb, work, rows, work, cols, rows, d, sigma, slices, ldk,
                             plane_rows * ldk, pmax, err, st, dig, keep_residual);
}

struct Timer {
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    bool on = false;
    explicit Timer(bool enable) : on(enable) {
        if (on)
            for (auto& e : ev) cudaEventCreate(&e);
    }
    void mark(int i, cudaStream_t st) {
        if (on) cudaEventRecord(ev[i], st);
    }
    double secs(int a, int b) const {
        if (!on) return 0.0;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[a], ev[b]);
        return ms * 1e-3;
    }
    ~Timer() {
        if (on)
            for (auto& e : ev) cudaEventDestroy(e);
    }
};

// Row bands of the host-buffer schedule (ozk_ozaki_gemm), as row starts
// [0, r_1, ..., m].  Each band is one slice-GEMM launch whose persistent
// clusters take one cluster tile per wave, so a band of R cluster rows over T
// cluster columns costs ceil(R*T / clusters) waves: bands whose tile counts sit
// just below a multiple of the cluster count waste nothing, others up to a
// wave each.  Band 0 (about m/8; the GEMM waits for it and for B) is sized for
// the best wave fill of its B column blocks.  The rest is chosen by a DP from
// the end: minimise GEMM waves x t_wave + the last band's C copy, with each
// band's C copy no longer than the next band's GEMM (so copies stay hidden);
// band sizes come from the sizes with >= 90 % wave fill (and 1..4 rows), and
// each band's A rows must cross PCIe during the previous band's GEMM (band 1's
// during band 0's last column block: A follows all of B on the copy stream).
// t_wave: one cluster tile's work at the measured per-SM INT8 rate of the
// format (bench_r01_f2: DD 19, TD 16.5, QD 15, TS 9.5 Tops/s per SM).
struct BandKey {
    size_t m, n, l, block_cols, band0;
    int fmt, d, rows, cols, clusters;
    bool operator<(const BandKey& o) const {
        return std::tie(m, n, l, block_cols, band0, fmt, d, rows, cols, clusters) <
               std::tie(o.m, o.n, o.l, o.block_cols, o.band0, o.fmt, o.d, o.rows, o.cols,
                        o.clusters);
    }
};

// band0_rows > 0 forces band 0's size (in rows, rounded to cluster rows)
std::vector<size_t> plan_bands_uncached(int fmt, size_t m, size_t n, size_t l, int d,
                                        size_t block_cols, const I8Geometry& g,
                                        size_t band0_rows = 0) {
    std::vector<size_t> starts{0};
    const size_t rtot = g.group_rows > 0 ? (m + g.group_rows - 1) / g.group_rows : 0;
    if (m < 2048 || g.clusters <= 0 || rtot < 8) {
        starts.push_back(m);
        return starts;
    }
    if (rtot > 512) {  // quantisation loss per band < 1 %: 8 equal bands
        for (size_t q = 1; q <= 8; ++q) starts.push_back(m * q / 8);
        return starts;
    }
    const size_t C = (size_t)g.clusters;
    const size_t T = (n + g.group_cols - 1) / g.group_cols;
    const size_t Tb = (block_cols + g.group_cols - 1) / g.group_cols;
    auto waves = [&](size_t r, size_t t) { return (r * t + C - 1) / C; };
    auto fill = [&](size_t r, size_t t) { return double(r * t) / double(waves(r, t) * C); };
    // band 0: best fill of its column blocks within [rtot/12, rtot/6]
    size_t r0 = 1;
    {
        const size_t lo = rtot / 12 > 0 ? rtot / 12 : 1, hi = rtot / 6 > lo ? rtot / 6 : lo;
        double best = -1.0;
        for (size_t r = lo; r <= hi; ++r)  // ties go to the larger band
            if (fill(r, Tb) >= best - 1e-9) {
                best = fill(r, Tb) > best ? fill(r, Tb) : best;
                r0 = r;
            }
        if (band0_rows > 0)
            r0 = std::max<size_t>(1, std::min(rtot - 1, band0_rows / g.group_rows));
    }
    const size_t rest = rtot - r0;
    const int K = words_of(fmt), wb = word_bytes_of(fmt);
    const int nd = int8_digits(fmt, l, d);
    const double rate_sm = wb == 4 ? 9.5e12 : (K == 2 ? 19e12 : (K == 3 ? 16.5e12 : 15e12));
    const double pairs = 0.5 * d * (d + 1);
    const double t_wave = pairs * nd * nd * 2.0 * g.group_rows * g.group_cols * (double)l /
                          (rate_sm * g.cluster_sms);
    const double t_row_d2h = (double)g.group_rows * (double)n * elem_bytes(fmt) / 45e9;
    const double t_row_h2d = (double)g.group_rows * (double)l * elem_bytes(fmt) / 45e9;
    std::vector<size_t> cand;
    for (size_t r = 1; r <= rest; ++r)
        if (r <= 4 || fill(r, T) >= 0.9) cand.push_back(r);
    const size_t nc = cand.size();
    constexpr int kMaxBands = 7;  // after band 0
    const double inf = 1e30;
    auto idx = [&](int jj, size_t x, size_t c) { return ((size_t)jj * (rest + 1) + x) * nc + c; };
    std::vector<double> best;
    std::vector<size_t> from;
    double bv = inf;
    int bj = 0;
    size_t bc = 0;
    // the A-arrival constraints are dropped when nothing satisfies them (small
    // GEMMs whose A bands take longer to copy than to multiply)
    for (int pass = 0; pass < 2 && bj == 0; ++pass) {
        const bool arrive = pass == 0;
        // best[j][x][c]: cost of covering the last x cluster rows with j bands
        // whose earliest band has size cand[c]
        best.assign((size_t)(kMaxBands + 1) * (rest + 1) * nc, inf);
        from.assign(best.size(), SIZE_MAX);
        for (size_t c = 0; c < nc; ++c)
            best[idx(1, cand[c], c)] = waves(cand[c], T) * t_wave + cand[c] * t_row_d2h;
        for (int jj = 1; jj < kMaxBands; ++jj)
            for (size_t x = 1; x <= rest; ++x)
                for (size_t c = 0; c < nc && cand[c] <= x; ++c) {
                    const double cur = best[idx(jj, x, c)];
                    if (cur >= inf) continue;
                    const double next_gemm = waves(cand[c], T) * t_wave;
                    for (size_t p = 0; p < nc && x + cand[p] <= rest; ++p) {
                        if (cand[p] * t_row_d2h > next_gemm) continue;  // its C copy must hide
                        // the next band's A rows must land during this band's GEMM
                        if (arrive && cand[c] * t_row_h2d > waves(cand[p], T) * t_wave) continue;
                        const double v = cur + waves(cand[p], T) * t_wave;
                        double& slot = best[idx(jj + 1, x + cand[p], p)];
                        if (v < slot - 1e-12) {
                            slot = v;
                            from[idx(jj + 1, x + cand[p], p)] = c;
                        }
                    }
                }
        // band 1's A rows cross PCIe after all of B, during band 0's last block
        const double band0_tail = waves(r0, Tb) * t_wave;
        for (int jj = 1; jj <= kMaxBands; ++jj)
            for (size_t c = 0; c < nc; ++c)
                if ((!arrive || cand[c] * t_row_h2d <= band0_tail) &&
                    best[idx(jj, rest, c)] < bv - 1e-12) {
                    bv = best[idx(jj, rest, c)];
                    bj = jj;
                    bc = c;
                }
    }
    if (bj == 0) {  // no feasible plan: 8 equal bands
        for (size_t q = 1; q <= 8; ++q) starts.push_back(m * q / 8);
        return starts;
    }
    std::vector<size_t> sizes{r0};
    for (size_t x = rest, c = bc; bj > 0; --bj) {
        sizes.push_back(cand[c]);
        const size_t prev = from[idx(bj, x, c)];
        x -= cand[c];
        c = prev;
    }
    size_t acc = 0;
    for (size_t q = 0; q < sizes.size(); ++q) {
        acc += sizes[q] * (size_t)g.group_rows;
        starts.push_back(acc < m ? acc : m);
    }
    starts.back() = m;
    return starts;
}

// 2-D head schedule (HostOverlap::head_bands): h head bands of one wave per B
// block each (rows = cluster rows x floor(clusters / tiles per block)), then
// the remaining rows planned as above for full-width bands.  Returns the band
// starts; the number of head bands actually used is written to *heads.
std::vector<size_t> plan_head_bands(int fmt, size_t m, size_t n, size_t l, int d,
                                    size_t block_cols, const I8Geometry& g, int h, int* heads) {
    *heads = 0;
    std::vector<size_t> starts{0};
    const size_t tb = (block_cols + g.group_cols - 1) / g.group_cols;
    if (h < 2 || g.clusters <= 0 || tb == 0) return starts;
    const size_t rb = (size_t)g.group_rows * std::max<size_t>(1, (size_t)g.clusters / tb);
    size_t acc = 0;
    for (int q = 0; q < h && acc + rb < m; ++q) {
        acc += rb;
        starts.push_back(acc);
        ++*heads;
    }
    if (*heads < 2) {
        *heads = 0;
        return {0};
    }
    const size_t m_tail = m - acc;
    const std::vector<size_t> tail = plan_bands_uncached(fmt, m_tail, n, l, d, n, g);
    for (size_t q = 1; q < tail.size(); ++q) starts.push_back(acc + tail[q]);
    if (starts.back() != m) starts.push_back(m);
    return starts;
}

std::vector<size_t> plan_bands(int fmt, size_t m, size_t n, size_t l, int d, size_t block_cols,
                               const I8Geometry& g, size_t band0_rows = 0) {
    static std::mutex mu;
    static std::map<BandKey, std::vector<size_t>> cache;
    const BandKey key{m, n, l, block_cols, band0_rows, fmt, d, g.group_rows, g.group_cols,
                      g.clusters};
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    std::vector<size_t> plan = plan_bands_uncached(fmt, m, n, l, d, block_cols, g, band0_rows);
    std::lock_guard<std::mutex> lock(mu);
    if (cache.size() > 256) cache.clear();
    cache[key] = plan;
    return plan;
}

// Host-buffer overlap hooks (ozk_ozaki_gemm): wait on b_ready before the B
// split (whole-B mode), and run the slice GEMM in `bands` row bands
// [band_start[q], band_start[q+1]) (plan_bands), calling on_band(r0, r1) after
// each is enqueued so its D2H copy overlaps the next band (rows are
// independent, so banding does not change a bit).
struct HostOverlap {
    cudaEvent_t b_ready = nullptr;
    int bands = 1;
    std::vector<size_t> band_start;  // bands + 1 row starts (plan_bands)
    std::function<cudaError_t(size_t, size_t)> on_band;
    // optional: A arrives band by band (a_ready[b] = rows of band b on the
    // device); then B is split first and each band's A rows are split right
    // before its GEMM (not with drop_threshold > 0: the pair list needs every
    // slice maximum first)
    const cudaEvent_t* a_ready = nullptr;
    // optional (INT8 engine, with a_ready): B arrives in b_blocks column blocks
    // of b_block_cols columns (b_block_ready[j]); each block is split as it
    // lands and the first A band is multiplied block by block, so the GEMM
    // starts after one A band and one B block instead of all of B.  Columns
    // are split independently (per-column maxima, ozaki.hpp:102-103) and C
    // elements are independent, so this does not change a bit either.
    int b_blocks = 1;
    size_t b_block_cols = 0;
    const cudaEvent_t* b_block_ready = nullptr;
    // optional (with B blocks): bands [0, head_bands) are "head" bands whose A
    // rows arrive interleaved with the B blocks -- A0, B0, B1, A1, B2, A2, ...
    // -- and every (head band, B block) product is multiplied as soon as both
    // are in; the remaining bands follow full width.  0: only band 0 is
    // multiplied block by block.
    int head_bands = 0;
    // optional: called before every wait on one of the events above (pageable
    // buffers: blocks until the staging worker has recorded it)
    std::function<cudaError_t(cudaEvent_t)> before_wait;
    cudaError_t wait(cudaStream_t st, cudaEvent_t ev) const {
        if (before_wait) {
            const cudaError_t e = before_wait(ev);
            if (e != cudaSuccess) return e;
        }
        return cudaStreamWaitEvent(st, ev, 0);
    }
};

// C = A * B via the Ozaki scheme on device buffers; A has row stride lda, B
// row stride ldb (elements), C is dense m x n.
// forced (optional): the pair list to use instead of the one from this call's
// own slice maxima (ozk_ozaki_gemm_multi: one list from the global maxima of
// every device's rows).
// lu (optional, binary64 formats): the blocked-LU trailing update -- the
// finished sum is subtracted from the m x n block lu->a22 (row stride lu->lda
// elements) by the slice-GEMM epilogue of the last pair, and c is only the
// running-sum scratch.
struct LuTarget {
    double* a22;
    size_t lda;
};
ozk_status ozaki_device_impl(int fmt, size_t m, size_t l, size_t n, const void* a, size_t lda,
                             const void* b, size_t ldb, int d, double drop, void* c,
                             cudaStream_t st, ozk_profile* prof,
                             const HostOverlap* ov = nullptr, const PairList* forced = nullptr,
                             const LuTarget* lu = nullptr, int* async_flags = nullptr) {
    const int K = words_of(fmt), wb = word_bytes_of(fmt);
    const int sms = num_sms_cached();
    const size_t ldk = slice_ld(l);
    const int eng = engine_setting();
    const bool use_i8 = eng != OZK_ENGINE_DMMA && int8_applicable(fmt, l, d);
    if (eng == OZK_ENGINE_INT8 && !use_i8)
        return fail(OZK_EPARAM, "ozaki_gemm: INT8 engine needs D >= 2 and 128 < l < 43690 "
                                "(binary64 words) or l < 43690 (TS)");
    const int nd = use_i8 ? int8_digits(fmt, l, d) : 0;
    const size_t ld8 = (l + 15) & ~size_t(15);
    DevBuf sa, sb, work, flags, da8, db8, ga, gb;
    if (use_i8) {
        OZK_CUDA(da8.alloc((size_t)d * nd * m * ld8, st), "ozaki_gemm: digits A");
        OZK_CUDA(db8.alloc((size_t)d * nd * n * ld8, st), "ozaki_gemm: digits B");
        OZK_CUDA(ga.alloc(sizeof(int) * d * m, st), "ozaki_gemm: exponents A");
        OZK_CUDA(gb.alloc(sizeof(int) * d * n, st), "ozaki_gemm: exponents B");
    } else {
        OZK_CUDA(sa.alloc(sizeof(double) * d * m * ldk, st), "ozaki_gemm: slices A");
        OZK_CUDA(sb.alloc(sizeof(double) * d * n * ldk, st), "ozaki_gemm: slices B");
    }
    OZK_CUDA(work.alloc(elem_bytes(fmt) * (m > n ? m : n) * l, st), "ozaki_gemm: work");
    // flags layout: [A err int][B err int][amax d][bmax d]; separate A and B
    // flags so an A error is reported first, as split_matrix(a) runs before
    // split_matrix(b) (ozaki.hpp:194-195)
    OZK_CUDA(flags.alloc(8 + 16 * (size_t)d, st), "ozaki_gemm: flags");
    OZK_CUDA(cudaMemsetAsync(flags.p, 0, 8 + 16 * (size_t)d, st), "ozaki_gemm: memset");
    int* err = flags.as<int>();
    int* errB = err + 1;
    unsigned long long* amax = reinterpret_cast<unsigned long long*>(flags.as<char>() + 8);
    unsigned long long* bmax = amax + d;
    const bool want_max = drop > 0.0 && !forced;
    DigitOut digA, digB;
    if (use_i8) {
        digA.nd = nd;
        digA.digits = da8.as<int8_t>();
        digA.ld = ld8;
        digA.digit_stride = m * ld8;
        digA.slice_stride = (size_t)nd * m * ld8;
        digA.exps = ga.as<int>();
        digA.exp_stride = m;
        digB.nd = nd;
        digB.digits = db8.as<int8_t>();
        digB.ld = ld8;
        digB.digit_stride = n * ld8;
        digB.slice_stride = (size_t)nd * n * ld8;
        digB.exps = gb.as<int>();
        digB.exp_stride = n;
    }

    Timer tm(prof != nullptr);
    tm.mark(0, st);
    const bool banded_a = ov && ov->a_ready && !want_max && ov->bands > 1;
    const bool blocked_b = banded_a && use_i8 && ov->b_block_ready && ov->b_blocks > 1;
    if (!banded_a) {
        if (ov && ov->a_ready)
            for (int q = 0; q < ov->bands; ++q)
                OZK_CUDA(ov->wait(st, ov->a_ready[q]), "ozaki_gemm: wait A");
        OZK_CUDA(split_to_slices(fmt, m, l, lda, a, d, OZK_SIDE_ROWS, sa.as<double>(), m, work.p,
                                 want_max ? amax : nullptr, err, st, digA),
                 "ozaki_gemm: split A");
    }
    if (!blocked_b) {
        if (ov && ov->b_ready) OZK_CUDA(ov->wait(st, ov->b_ready), "ozaki_gemm: wait B");
        OZK_CUDA(split_to_slices(fmt, l, n, ldb, b, d, OZK_SIDE_COLS, sb.as<double>(), n, work.p,
                                 want_max ? bmax : nullptr, errB, st, digB),
                 "ozaki_gemm: split B");
    }
    tm.mark(1, st);

    PairList pl;
    if (forced) {
        pl = *forced;
    } else if (want_max) {
        std::vector<double> host(1 + 2 * (size_t)d);
        OZK_CUDA(cudaMemcpyAsync(host.data(), flags.p, 8 + 16 * (size_t)d, cudaMemcpyDeviceToHost,
                                 st),
                 "ozaki_gemm: maxima");
        OZK_CUDA(cudaStreamSynchronize(st), "ozaki_gemm: split");
        int flag[2];
        std::memcpy(flag, host.data(), sizeof(flag));
        if (ozk_status s = check_dev_err(flag[0], "split_matrix")) return s;
        if (ozk_status s = check_dev_err(flag[1], "split_matrix")) return s;
        pruned_pairs(d, host.data() + 1, host.data() + 1 + d, drop, pl);
    } else {
        triangular_pairs(d, pl);
    }

    GemmProblem prob{};
    prob.a = sa.as<double>();
    prob.lda = ldk;
    prob.a_slice_stride = m * ldk;
    prob.a_slices = d;
    prob.b = sb.as<double>();
    prob.ldb = ldk;
    prob.b_slice_stride = n * ldk;
    prob.b_blk_stride = (size_t)d * n * ldk;
    prob.b_slices = d;
    prob.ncb = (int)n;
    prob.nblk = 1;
    prob.m = m;
    prob.n = n;
    prob.l = l;
    prob.c = c;
    prob.ldc = n;
    const int bands = (ov && ov->bands > 1 && (pl.count > 0 || banded_a)) ? ov->bands : 1;
    const size_t eb = elem_bytes(fmt);
    std::vector<std::unique_ptr<Timer>> split_timers;  // per-band A / per-block B splits (profile)
    int band = 0;
    // C rows [r0, r0 + rows) x columns [c0, c0 + w) on the INT8 engine
    auto gemm_block = [&](size_t r0, size_t rows, size_t c0, size_t w) -> cudaError_t {
        I8Operands op{};
        op.nd = nd;
        op.a = da8.as<int8_t>() + r0 * ld8;
        op.a_ld = ld8;
        op.a_digit_stride = m * ld8;
        op.a_slice_stride = (size_t)nd * m * ld8;
        op.b = db8.as<int8_t>() + c0 * ld8;
        op.b_ld = ld8;
        op.b_digit_stride = n * ld8;
        op.b_slice_stride = (size_t)nd * n * ld8;
        op.gA = ga.as<int>() + r0;
        op.gB = gb.as<int>() + c0;
        op.gA_stride = m;
        op.gB_stride = n;
        op.m = rows;
        op.n = w;
        op.l = l;
        op.d = d;
        op.c = static_cast<char*>(c) + (r0 * n + c0) * eb;
        op.ldc = n;
        if (lu) {
            op.lu_a22 = lu->a22 + (r0 * lu->lda + c0) * K;
            op.lu_lda = lu->lda;
        }
        return launch_pair_gemm_i8(K, wb, op, pl, st, sms);
    };
    auto split_a_band = [&](size_t r0, size_t rows) -> cudaError_t {
        // per-row split, identical to the rows of the whole-matrix split
        // (ozaki.hpp:102-103)
        DigitOut dband = digA;
        if (use_i8) {
            dband.digits += r0 * ld8;
            dband.exps += r0;
        }
        split_timers.push_back(std::make_unique<Timer>(prof != nullptr));
        split_timers.back()->mark(0, st);
        const cudaError_t e =
            split_to_slices(fmt, rows, l, lda, static_cast<const char*>(a) + r0 * lda * eb, d,
                            OZK_SIDE_ROWS, use_i8 ? nullptr : sa.as<double>() + r0 * ldk, m,
                            work.p, nullptr, err, st, dband);
        split_timers.back()->mark(1, st);
        return e;
    };
    auto split_b_block = [&](size_t c0, size_t w) -> cudaError_t {
        // per-column split of B's columns [c0, c0 + w) (ozaki.hpp:102-103)
        DigitOut dblk = digB;
        dblk.digits += c0 * ld8;
        dblk.exps += c0;
        split_timers.push_back(std::make_unique<Timer>(prof != nullptr));
        split_timers.back()->mark(0, st);
        const cudaError_t e =
            split_to_slices(fmt, l, w, ldb, static_cast<const char*>(b) + c0 * eb, d,
                            OZK_SIDE_COLS, nullptr, n, work.p, nullptr, errB, st, dblk);
        split_timers.back()->mark(1, st);
        return e;
    };
    if (blocked_b && pl.count > 0 && ov->head_bands > 1) {
        // 2-D head: A bands and B blocks arrive interleaved (A0, B0, B1, A1,
        // B2, A2, ...); each arrival is split and multiplied against every
        // block / band already in, so the GEMM work available grows with the
        // product of what has crossed PCIe.  C elements are independent:
        // bit-identical to one GEMM.
        const int nb = ov->b_blocks, nh = std::min(ov->head_bands, bands);
        auto blk = [&](int j, size_t& c0, size_t& w) {
            c0 = std::min(n, (size_t)j * ov->b_block_cols);
            w = std::min(ov->b_block_cols, n - c0);
        };
        int a_in = 0, b_in = 0;  // arrived head bands / B blocks
        auto arrive_a = [&](int q) -> cudaError_t {
            const size_t r0 = ov->band_start[q], rows = ov->band_start[q + 1] - r0;
            cudaError_t e = ov->wait(st, ov->a_ready[q]);
            if (e == cudaSuccess && rows) e = split_a_band(r0, rows);
            for (int j = 0; j < b_in && e == cudaSuccess; ++j) {
                size_t c0, w;
                blk(j, c0, w);
                if (rows && w) e = gemm_block(r0, rows, c0, w);
            }
            a_in = q + 1;
            return e;
        };
        auto arrive_b = [&](int j) -> cudaError_t {
            size_t c0, w;
            blk(j, c0, w);
            cudaError_t e = ov->wait(st, ov->b_block_ready[j]);
            if (e == cudaSuccess && w) e = split_b_block(c0, w);
            for (int q = 0; q < a_in && e == cudaSuccess; ++q) {
                const size_t r0 = ov->band_start[q], rows = ov->band_start[q + 1] - r0;
                if (rows && w) e = gemm_block(r0, rows, c0, w);
            }
            b_in = j + 1;
            return e;
        };
        OZK_CUDA(arrive_a(0), "ozaki_gemm: head band");
        OZK_CUDA(arrive_b(0), "ozaki_gemm: head block");
        for (int k = 1; k < std::max(nb, nh); ++k) {
            if (k < nb) OZK_CUDA(arrive_b(k), "ozaki_gemm: head block");
            if (k < nh) OZK_CUDA(arrive_a(k), "ozaki_gemm: head band");
        }
        for (int q = 0; q < nh; ++q)  // head bands complete: their C rows go back
            if (ov->on_band)
                OZK_CUDA(ov->on_band(ov->band_start[q], ov->band_start[q + 1]),
                         "ozaki_gemm: band copy");
        band = nh;
    }
    for (; band < bands; ++band) {
        size_t r0 = 0, r1 = m;
        if (bands > 1) {
            r0 = ov->band_start[band];
            r1 = ov->band_start[band + 1];
        }
        const size_t rows = r1 - r0;
        if (rows == 0) continue;
        char* cb = static_cast<char*>(c) + r0 * n * eb;
        if (banded_a) {
            OZK_CUDA(ov->wait(st, ov->a_ready[band]), "ozaki_gemm: wait A");
            OZK_CUDA(split_a_band(r0, rows), "ozaki_gemm: split A band");
        }
        if (pl.count == 0) {  // every pair pruned (drop_threshold > 1): C = 0
            OZK_CUDA(cudaMemsetAsync(cb, 0, eb * rows * n, st), "ozaki_gemm: zero C");
            if (lu)  // A22 -= 0, through the reference's subtraction
                OZK_CUDA(launch_kw_sub_inplace(K, lu->a22 + r0 * lu->lda * K, lu->lda,
                                               reinterpret_cast<const double*>(cb), rows, n, st),
                         "ozaki_gemm: LU subtract");
            if (blocked_b && band == 0)  // the B blocks still arrive in order (nothing to split)
                for (int j = 0; j < ov->b_blocks; ++j)
                    OZK_CUDA(ov->wait(st, ov->b_block_ready[j]), "ozaki_gemm: wait B");
        } else if (use_i8) {
            if (blocked_b && band == 0) {
                // B column blocks: split each as it lands, then its GEMM block
                for (int j = 0; j < ov->b_blocks; ++j) {
                    const size_t c0 = (size_t)j * ov->b_block_cols;
                    if (c0 >= n) break;
                    const size_t w = n - c0 < ov->b_block_cols ? n - c0 : ov->b_block_cols;
                    OZK_CUDA(ov->wait(st, ov->b_block_ready[j]), "ozaki_gemm: wait B");
                    OZK_CUDA(split_b_block(c0, w), "ozaki_gemm: split B block");
                    OZK_CUDA(gemm_block(r0, rows, c0, w), "ozaki_gemm: INT8 slice GEMM");
                }
            } else {
                OZK_CUDA(gemm_block(r0, rows, 0, n), "ozaki_gemm: INT8 slice GEMM");
            }
        } else {
            GemmProblem pb = prob;
            pb.a = prob.a + r0 * ldk;
            pb.m = rows;
            pb.c = cb;
            if (lu) {
                pb.lu_a22 = lu->a22 + r0 * lu->lda * K;
                pb.lu_lda = lu->lda;
            }
            OZK_CUDA(launch_pair_gemm(K, lu ? kAccumulateLU : kAccumulate, pb, pl, st, sms, wb),
                     "ozaki_gemm: slice GEMM");
        }
        if (ov && ov->on_band) OZK_CUDA(ov->on_band(r0, r0 + rows), "ozaki_gemm: band copy");
    }
    tm.mark(2, st);

    if (async_flags) {
        // asynchronous form: the split's data-error flags (A, then B) go to the
        // caller's device ints, read later with ozk_check_split_flag
        OZK_CUDA(cudaMemcpyAsync(async_flags, err, 2 * sizeof(int), cudaMemcpyDeviceToDevice, st),
                 "ozaki_gemm: flag");
        return OZK_OK;
    }
    int flag[2] = {0, 0};
    OZK_CUDA(cudaMemcpyAsync(flag, err, sizeof(flag), cudaMemcpyDeviceToHost, st),
             "ozaki_gemm: flag");
    OZK_CUDA(cudaStreamSynchronize(st), "ozaki_gemm");
    if (ozk_status s = check_dev_err(flag[0], "split_matrix")) return s;
    if (ozk_status s = check_dev_err(flag[1], "split_matrix")) return s;
    if (prof) {
        double split_banded = 0.0;
        for (const auto& t : split_timers) split_banded += t->secs(0, 1);
        prof->split_seconds = tm.secs(0, 1) + split_banded;
        prof->product_seconds = tm.secs(1, 2) - split_banded;
        prof->accumulate_seconds = 0.0;
        prof->total_seconds = prof->split_seconds + prof->product_seconds;
        prof->split_count = d;
        prof->pairs = pl.count;
        prof->gpus = 1;
        prof->engine = use_i8 ? OZK_ENGINE_INT8 : OZK_ENGINE_DMMA;
    }
    return OZK_OK;
}

ozk_status check_gemm_args(int fmt, size_t m, size_t l, size_t n, int d, double drop) {
    if (!valid_fmt(fmt)) return fail(OZK_EPARAM, "ozaki_gemm: format must be DD, TD, QD or TS");
    if (m == 0 || l == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (d < 1) return fail(OZK_EPARAM, "ozaki_gemm: split count must be >= 1");
    if (drop < 0.0) return fail(OZK_EPARAM, "ozaki_gemm: negative drop threshold");
    if (d > kMaxSplits) return fail(OZK_EPARAM, "ozaki_gemm: split count above 65535 is not supported");
    if (m > 0x7fffffffull || n > 0x7fffffffull || l > 0x7fffffffull)
        return fail(OZK_ESHAPE, "ozaki_gemm: dimension too large");
    return OZK_OK;
}

}  // namespace

namespace ozk {
// thread-local error text for the other host translation units (io.cu)
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace ozk

// Null operands are rejected at the boundary: a null device pointer would
// fault the kernel and leave the CUDA context unusable for the process.
static ozk_status need(std::initializer_list<const void*> ptrs, const char* what) {
    for (const void* p : ptrs)
        if (!p) return fail(OZK_EPARAM, std::string(what) + ": null pointer");
    return OZK_OK;
}

extern "C" {

const char* ozk_last_error(void) { return g_last_error.c_str(); }

ozk_status ozk_set_engine(int engine) {
    if (engine != OZK_ENGINE_AUTO && engine != OZK_ENGINE_DMMA && engine != OZK_ENGINE_INT8)
        return fail(OZK_EPARAM, "set_engine: unknown engine");
    g_engine.store(engine);
    return OZK_OK;
}

int ozk_get_engine(void) { return engine_setting(); }

ozk_status ozk_trim_device_pool(void) {
    int dev = 0;
    OZK_CUDA(cudaGetDevice(&dev), "trim_device_pool");
    cudaMemPool_t pool;
    OZK_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev), "trim_device_pool");
    OZK_CUDA(cudaDeviceSynchronize(), "trim_device_pool");
    OZK_CUDA(cudaMemPoolTrimTo(pool, 0), "trim_device_pool");
    return OZK_OK;
}
int ozk_version(void) { return 1; }

int ozk_split_shift_bits(size_t inner) { return shift_bits(inner ? inner : 1); }

int ozk_exponent_ceil_log2(double x) {
    int e = std::ilogb(x);
    return std::scalbn(1.0, e) == x ? e : e + 1;
}

size_t ozk_slice_ld(size_t inner) { return slice_ld(inner); }

ozk_status ozk_ozaki_gemm_device(ozk_format fmt, size_t m, size_t l, size_t n, const void* a,
                                 const void* b, int d, double drop, void* c, void* stream,
                                 ozk_profile* prof) {
    if (ozk_status s = check_gemm_args(fmt, m, l, n, d, drop)) return s;
    if (ozk_status s = need({a, b, c}, "ozaki_gemm")) return s;
    return ozaki_device_impl((int)fmt, m, l, n, a, l, b, n, d, drop, c, (cudaStream_t)stream,
                             prof);
}

ozk_status ozk_ozaki_gemm_device_async(ozk_format fmt, size_t m, size_t l, size_t n,
                                       const void* a, const void* b, int d, double drop, void* c,
                                       int* dev_flags, void* stream) {
    if (ozk_status s = check_gemm_args(fmt, m, l, n, d, drop)) return s;
    if (ozk_status s = need({a, b, c, dev_flags}, "ozaki_gemm")) return s;
    return ozaki_device_impl((int)fmt, m, l, n, a, l, b, n, d, drop, c, (cudaStream_t)stream,
                             nullptr, nullptr, nullptr, nullptr, dev_flags);
}

ozk_status ozk_ozaki_gemm(ozk_format fmt, size_t m, size_t l, size_t n, const void* a,
                          const void* b, int d, double drop, void* c, ozk_profile* prof) {
    if (ozk_status s = check_gemm_args(fmt, m, l, n, d, drop)) return s;
    if (ozk_status s = need({a, b, c}, "ozaki_gemm")) return s;
    const size_t eb = elem_bytes(fmt);
    auto t0 = std::chrono::steady_clock::now();
    OwnStream os;
    OZK_CUDA(os.create(), "ozaki_gemm: stream");
    num_sms_cached();
    // Transfers overlap compute on two copy streams: A arrives in row bands
    // (plan_bands), B whole or in column blocks split as they land, and C goes
    // back band by band while later bands compute (HostOverlap).
    OwnStream xs, ys;  // H2D copies, D2H copies
    OZK_CUDA(xs.create(), "ozaki_gemm: copy stream");
    OZK_CUDA(ys.create(), "ozaki_gemm: copy stream");
    DevBuf da, db, dc;
    // events are destroyed after the staging workers and copy streams drained
    struct EventGuard {
        std::vector<cudaEvent_t> evs;  // owned handles
        ~EventGuard() {
            for (cudaEvent_t e : evs) cudaEventDestroy(e);
        }
    } guard;
    // Pageable caller buffers (DenseMatrix storage) move through pinned staging
    // slots on worker threads (staging.cu), keeping the same band schedule.
    const bool staging_on = [] {
        const char* v = std::getenv("OZK_PAGEABLE_STAGING");
        return !(v && !std::strcmp(v, "0"));
    }();
    // Buffers below 2 MiB are left to the driver's own pageable copies, which
    // are as fast at that size as starting the two staging workers
    // ($OZK_STAGING_MIN_MB; the copy teams and slots are cached per process).
    const size_t stage_min = [] {
        const char* v = std::getenv("OZK_STAGING_MIN_MB");
        return (size_t)(v ? std::max(0, std::atoi(v)) : 2) << 20;
    }();
    auto staged = [&](const void* p, size_t bytes) {
        return staging_on && bytes >= stage_min && !host_is_pinned(p);
    };
    const bool a_pg = staged(a, eb * m * l), b_pg = staged(b, eb * l * n),
               c_pg = staged(c, eb * m * n);
    std::unique_ptr<HostStaging> hs;
    // on every exit: the staging workers drained and the copy streams idle
    // before the device buffers go back to the pool
    struct Drain {
        std::unique_ptr<HostStaging>* hs;
        cudaStream_t s[3];
        ~Drain() {
            if (*hs) (*hs)->finish();
            for (cudaStream_t x : s) cudaStreamSynchronize(x);
        }
    } drain{&hs, {xs.s, ys.s, os.s}};
    if (a_pg || b_pg || c_pg) {
        // host copy threads: H2D one per usable CPU (at most 16), D2H half as
        // many (the copies are memory-bound, so the two teams may oversubscribe
        // the cores; B200 host, 16 CPUs: 16 + 8 gave 219 ms for TD n=8192 vs
        // 225 (8 + 8), 239 (8 + 4), 205 pinned, 540 unstaged --
        // tools/staging_sweep.py), or $OZK_STAGING_THREADS = "h2d[,d2h]"
        int cpus = (int)std::thread::hardware_concurrency();
        cpu_set_t set;
        if (sched_getaffinity(0, sizeof(set), &set) == 0) cpus = CPU_COUNT(&set);
        int th = std::max(1, std::min(16, cpus)), th2 = std::max(1, std::min(8, cpus / 2));
        if (const char* v = std::getenv("OZK_STAGING_THREADS")) {
            const int x = std::atoi(v);
            const char* comma = std::strchr(v, ',');
            const int y = comma ? std::atoi(comma + 1) : x;
            if (x > 0) th = x;
            if (y > 0) th2 = y;
        }
        hs = std::make_unique<HostStaging>(xs.s, ys.s, th, th2);
    }
    std::map<cudaEvent_t, int> staged_job;  // H2D event -> staging job number
    OZK_CUDA(da.alloc(eb * m * l, os.s), "ozaki_gemm: A");
    OZK_CUDA(db.alloc(eb * l * n, os.s), "ozaki_gemm: B");
    OZK_CUDA(dc.alloc(eb * m * n, os.s), "ozaki_gemm: C");
    cudaEvent_t allocated = nullptr, b_ready = nullptr;
    OZK_CUDA(cudaEventCreateWithFlags(&allocated, cudaEventDisableTiming), "ozaki_gemm: event");
    guard.evs.push_back(allocated);
    OZK_CUDA(cudaEventCreateWithFlags(&b_ready, cudaEventDisableTiming), "ozaki_gemm: event");
    guard.evs.push_back(b_ready);
    // B in column blocks (whole 128-column tiles) when the first band can be
    // multiplied block by block (INT8 engine, no pruning, n >= 4096)
    const bool i8 = engine_setting() != OZK_ENGINE_DMMA && int8_applicable((int)fmt, l, d);
    const bool blockable = m >= 2048 && drop == 0.0 && i8 && n >= 4096;
    // B column blocks: 8 at n >= 8192 (1024-column blocks: the first GEMM
    // starts after 1/8 of B; TD n=8192 203 ms vs 208 with 4 blocks, DD within
    // noise, profiles/r02_host_schedule_sweep_*.log), else 4.  Knobs for A/B
    // sweeps (tools/host_schedule_sweep.py): $OZK_HOST_BBLOCKS, $OZK_HOST_BAND0
    // (band-0 rows)
    int nblk = n >= 8192 ? 8 : 4;
    size_t band0_rows = 0;
    if (const char* v = std::getenv("OZK_HOST_BBLOCKS")) nblk = std::max(1, std::atoi(v));
    if (const char* v = std::getenv("OZK_HOST_BAND0")) band0_rows = (size_t)std::max(0, std::atoi(v));
    const size_t b_block_cols =
        blockable ? (((n + nblk - 1) / nblk + 127) / 128) * 128 : n;
    // row bands from the slice GEMM's tile geometry (DMMA engine: 8 equal bands)
    const I8Geometry geo =
        i8 ? pair_gemm_i8_geometry(words_of((int)fmt), word_bytes_of((int)fmt),
                                   int8_digits((int)fmt, l, d), num_sms_cached())
           : I8Geometry{};
    std::vector<size_t> band_start;
    // $OZK_HOST_HEAD = h >= 2: the 2-D head schedule with h head bands
    int head = 0;
    if (const char* v = std::getenv("OZK_HOST_HEAD")) head = std::max(0, std::atoi(v));
    int heads = 0;
    if (i8 && blockable && head >= 2)
        band_start = plan_head_bands((int)fmt, m, n, l, d, b_block_cols, geo, head, &heads);
    if (heads >= 2) {
        // planned above
    } else if (i8) {
        band_start = plan_bands((int)fmt, m, n, l, d, b_block_cols, geo, band0_rows);
    } else {
        const size_t nb = m >= 2048 ? 8 : 1;
        for (size_t q = 0; q <= nb; ++q) band_start.push_back(m * q / nb);
    }
    const int bands = (int)band_start.size() - 1;
    const int b_blocks = (int)((n + b_block_cols - 1) / b_block_cols);
    std::vector<cudaEvent_t> band_done(bands, nullptr), a_ready(bands, nullptr),
        b_block_ready(b_blocks, nullptr);
    for (auto* vec : {&band_done, &a_ready, &b_block_ready})
        for (auto& e : *vec) {
            OZK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "ozaki_gemm: event");
            guard.evs.push_back(e);
        }
    OZK_CUDA(cudaEventRecord(allocated, os.s), "ozaki_gemm: event");
    OZK_CUDA(cudaStreamWaitEvent(xs.s, allocated, 0), "ozaki_gemm: wait");
    OZK_CUDA(cudaStreamWaitEvent(ys.s, allocated, 0), "ozaki_gemm: wait");
    // one H2D copy of `rows` rows of `width` bytes (pitches dpitch / spitch),
    // followed by `ev` on the H2D stream: staged when the source is pageable
    auto h2d = [&](bool pageable, void* dst, size_t dpitch, const void* src, size_t spitch,
                   size_t width, size_t rows, cudaEvent_t ev) -> cudaError_t {
        if (pageable) {
            StagedCopy sc;
            sc.dev = dst;
            sc.host = const_cast<void*>(src);
            sc.width = width;
            sc.height = rows;
            sc.dev_pitch = dpitch;
            sc.host_pitch = spitch;
            sc.event = ev;
            const int job = hs->push_h2d(sc);
            if (ev) staged_job[ev] = job;
            return cudaSuccess;
        }
        cudaError_t e = cudaSuccess;
        if (width && rows)
            e = rows == 1 ? cudaMemcpyAsync(dst, src, width, cudaMemcpyHostToDevice, xs.s)
                          : cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows,
                                              cudaMemcpyHostToDevice, xs.s);
        if (e == cudaSuccess && ev) e = cudaEventRecord(ev, xs.s);
        return e;
    };
    // Copy order on the H2D stream.  Whole B: B (its split gates every band),
    // then A band by band.  B in column blocks: A band 0, then the B blocks
    // (strided copies of the row-major B), then the other A bands.
    auto copy_a_band = [&](int q) -> cudaError_t {
        const size_t r0 = band_start[q], rows = band_start[q + 1] - r0;
        return h2d(a_pg, static_cast<char*>(da.p) + r0 * l * eb, 0,
                   static_cast<const char*>(a) + r0 * l * eb, 0, rows * l * eb, 1, a_ready[q]);
    };
    auto copy_b_block = [&](int j) -> cudaError_t {
        const size_t c0 = std::min(n, (size_t)j * b_block_cols);
        const size_t w = std::min(b_block_cols, n - c0);
        return h2d(b_pg, static_cast<char*>(db.p) + c0 * eb, n * eb,
                   static_cast<const char*>(b) + c0 * eb, n * eb, w * eb, l, b_block_ready[j]);
    };
    int next_a = 0;  // first A band not yet queued
    if (b_blocks > 1 && heads >= 2) {
        // 2-D head: A0, B0, B1, A1, B2, A2, ... (ozaki_device_impl multiplies
        // each arrival against everything already in, in this order)
        OZK_CUDA(copy_a_band(0), "ozaki_gemm: H2D A");
        OZK_CUDA(copy_b_block(0), "ozaki_gemm: H2D B block");
        for (int k = 1; k < std::max(b_blocks, heads); ++k) {
            if (k < b_blocks) OZK_CUDA(copy_b_block(k), "ozaki_gemm: H2D B block");
            if (k < heads) OZK_CUDA(copy_a_band(k), "ozaki_gemm: H2D A");
        }
        OZK_CUDA(h2d(b_pg, nullptr, 0, nullptr, 0, 0, 0, b_ready), "ozaki_gemm: event");
        next_a = heads;
    } else if (b_blocks > 1) {
        OZK_CUDA(copy_a_band(0), "ozaki_gemm: H2D A");
        for (int j = 0; j < b_blocks; ++j) OZK_CUDA(copy_b_block(j), "ozaki_gemm: H2D B block");
        OZK_CUDA(h2d(b_pg, nullptr, 0, nullptr, 0, 0, 0, b_ready), "ozaki_gemm: event");
        next_a = 1;
    } else {
        OZK_CUDA(h2d(b_pg, db.p, 0, b, 0, eb * l * n, 1, b_ready), "ozaki_gemm: H2D B");
    }
    for (int q = next_a; q < bands; ++q) OZK_CUDA(copy_a_band(q), "ozaki_gemm: H2D A");
    HostOverlap ov;
    ov.b_ready = b_ready;
    ov.bands = bands;
    ov.band_start = band_start;
    ov.a_ready = a_ready.data();
    if (b_blocks > 1) {
        ov.b_blocks = b_blocks;
        ov.b_block_cols = b_block_cols;
        ov.b_block_ready = b_block_ready.data();
        ov.head_bands = heads;
    }
    if (hs)
        ov.before_wait = [&](cudaEvent_t ev) -> cudaError_t {
            auto it = staged_job.find(ev);
            return it == staged_job.end() ? cudaSuccess : hs->wait_recorded(it->second);
        };
    int band = 0;
    ov.on_band = [&](size_t r0, size_t r1) -> cudaError_t {
        cudaEvent_t ev = band_done[band < bands ? band : bands - 1];
        ++band;
        cudaError_t e = cudaEventRecord(ev, os.s);
        if (e != cudaSuccess) return e;
        char* hc = static_cast<char*>(c) + r0 * n * eb;
        char* dcp = static_cast<char*>(dc.p) + r0 * n * eb;
        if (c_pg) {
            StagedCopy sc;
            sc.dev = dcp;
            sc.host = hc;
            sc.width = (r1 - r0) * n * eb;
            sc.event = ev;
            hs->push_d2h(sc);
            return cudaSuccess;
        }
        e = cudaStreamWaitEvent(ys.s, ev, 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(hc, dcp, (r1 - r0) * n * eb, cudaMemcpyDeviceToHost, ys.s);
        return e;
    };
    ozk_profile local{};
    ozk_status s =
        ozaki_device_impl((int)fmt, m, l, n, da.p, l, db.p, n, d, drop, dc.p, os.s, &local, &ov);
    if (s != OZK_OK) return s;  // drain syncs the copy streams first
    if (hs) OZK_CUDA(hs->finish(), "ozaki_gemm: staged copies");
    OZK_CUDA(cudaStreamSynchronize(xs.s), "ozaki_gemm: H2D");
    OZK_CUDA(cudaStreamSynchronize(ys.s), "ozaki_gemm: D2H C");
    OZK_CUDA(cudaStreamSynchronize(os.s), "ozaki_gemm");
    if (prof) {
        *prof = local;
        const double wall =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        prof->transfer_seconds = wall > local.total_seconds ? wall - local.total_seconds : 0.0;
    }
    return OZK_OK;
}

ozk_status ozk_split(ozk_format fmt, size_t rows, size_t cols, const void* mat, int d,
                     ozk_side side, void* pieces, void* residual) {
    if (!valid_fmt(fmt)) return fail(OZK_EPARAM, "split_matrix: format must be DD, TD, QD or TS");
    if (rows == 0 || cols == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (d < 1) return fail(OZK_EPARAM, "split_matrix: split count must be >= 1");
    if (d > kMaxSplits) return fail(OZK_EPARAM, "split_matrix: split count above 65535 is not supported");
    if (side != OZK_SIDE_ROWS && side != OZK_SIDE_COLS)
        return fail(OZK_EPARAM, "split_matrix: bad side");
    if (ozk_status s = need({mat}, "split_matrix")) return s;
    const int K = words_of(fmt), wb = word_bytes_of(fmt);
    const size_t eb = elem_bytes(fmt);
    const size_t N = rows * cols;
    const size_t inner = side == OZK_SIDE_ROWS ? cols : rows;
    const size_t outer = side == OZK_SIDE_ROWS ? rows : cols;
    const size_t ldk = slice_ld(inner);
    OwnStream os;
    OZK_CUDA(os.create(), "split_matrix: stream");
    num_sms_cached();
    DevBuf dm, work, sl, tp, tr, flags;
    OZK_CUDA(dm.alloc(eb * N, os.s), "split_matrix: input");
    OZK_CUDA(work.alloc(eb * N, os.s), "split_matrix: work");
    OZK_CUDA(sl.alloc(sizeof(double) * d * outer * ldk, os.s), "split_matrix: slices");
    OZK_CUDA(tp.alloc(sizeof(double) * d * N, os.s), "split_matrix: pieces");
    OZK_CUDA(flags.alloc(8, os.s), "split_matrix: flags");
    OZK_CUDA(cudaMemsetAsync(flags.p, 0, 8, os.s), "split_matrix: memset");
    OZK_CUDA(cudaMemcpyAsync(dm.p, mat, eb * N, cudaMemcpyHostToDevice, os.s), "split_matrix: H2D");
    OZK_CUDA(split_to_slices(fmt, rows, cols, cols, dm.p, d, side, sl.as<double>(), outer, work.p,
                             nullptr, flags.as<int>(), os.s, DigitOut{}, /*keep_residual=*/true),
             "split_matrix");
    int flag = 0;
    OZK_CUDA(cudaMemcpyAsync(&flag, flags.p, sizeof(int), cudaMemcpyDeviceToHost, os.s),
             "split_matrix: flag");
    OZK_CUDA(cudaStreamSynchronize(os.s), "split_matrix");
    if (ozk_status s = check_dev_err(flag, "split_matrix")) return s;
    // pieces back to the reference layout (rows x cols, row-major) in binary64
    if (side == OZK_SIDE_ROWS) {
        OZK_CUDA(cudaMemcpy2DAsync(tp.p, cols * 8, sl.p, ldk * 8, cols * 8, rows * (size_t)d,
                                   cudaMemcpyDeviceToDevice, os.s),
                 "split_matrix: pack pieces");
    } else {
        for (int a = 0; a < d; ++a)
            OZK_CUDA(launch_transpose(1, 8, sl.as<double>() + (size_t)a * outer * ldk, ldk,
                                      tp.as<double>() + (size_t)a * N, cols, cols, rows, os.s),
                     "split_matrix: transpose pieces");
    }
    // residual back to the reference layout
    const void* res_src = work.p;
    if (side == OZK_SIDE_COLS) {
        OZK_CUDA(tr.alloc(eb * N, os.s), "split_matrix: residual");
        OZK_CUDA(launch_transpose(K, wb, work.p, rows, tr.p, cols, cols, rows, os.s),
                 "split_matrix: transpose residual");
        res_src = tr.p;
    }
    OZK_CUDA(cudaMemcpyAsync(residual, res_src, eb * N, cudaMemcpyDeviceToHost, os.s),
             "split_matrix: D2H residual");
    if (wb == 8) {
        OZK_CUDA(cudaMemcpyAsync(pieces, tp.p, sizeof(double) * d * N, cudaMemcpyDeviceToHost, os.s),
                 "split_matrix: D2H pieces");
        OZK_CUDA(cudaStreamSynchronize(os.s), "split_matrix");
    } else {
        // TS pieces are binary32 values held exactly in binary64 slices
        std::vector<double> host((size_t)d * N);
        OZK_CUDA(cudaMemcpyAsync(host.data(), tp.p, sizeof(double) * d * N, cudaMemcpyDeviceToHost,
                                 os.s),
                 "split_matrix: D2H pieces");
        OZK_CUDA(cudaStreamSynchronize(os.s), "split_matrix");
        float* out = static_cast<float*>(pieces);
        for (size_t i = 0; i < host.size(); ++i) out[i] = (float)host[i];
    }
    return OZK_OK;
}

ozk_status ozk_split_slices_device(ozk_format fmt, size_t rows, size_t cols, size_t ld,
                                   const void* mat, int d, ozk_side side, double* slices,
                                   size_t plane_rows, double* piece_max, void* stream) {
    if (!valid_fmt(fmt)) return fail(OZK_EPARAM, "split_matrix: format must be DD, TD, QD or TS");
    if (rows == 0 || cols == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (d < 1) return fail(OZK_EPARAM, "split_matrix: split count must be >= 1");
    if (d > kMaxSplits) return fail(OZK_EPARAM, "split_matrix: split count above 65535 is not supported");
    if (ld < cols) return fail(OZK_ESHAPE, "split_matrix: ld < cols");
    if (plane_rows < (side == OZK_SIDE_ROWS ? rows : cols))
        return fail(OZK_ESHAPE, "split_matrix: plane_rows < outer dimension");
    if (ozk_status s = need({mat, slices}, "split_matrix")) return s;
    cudaStream_t st = (cudaStream_t)stream;
    num_sms_cached();
    DevBuf work, flags;
    OZK_CUDA(work.alloc(elem_bytes(fmt) * rows * cols, st), "split_matrix: work");
    OZK_CUDA(flags.alloc(8, st), "split_matrix: flags");
    OZK_CUDA(cudaMemsetAsync(flags.p, 0, 8, st), "split_matrix: memset");
    OZK_CUDA(split_to_slices(fmt, rows, cols, ld, mat, d, side, slices, plane_rows, work.p,
                             reinterpret_cast<unsigned long long*>(piece_max), flags.as<int>(), st),
             "split_matrix");
    int flag = 0;
    OZK_CUDA(cudaMemcpyAsync(&flag, flags.p, sizeof(int), cudaMemcpyDeviceToHost, st),
             "split_matrix: flag");
    OZK_CUDA(cudaStreamSynchronize(st), "split_matrix");
    return check_dev_err(flag, "split_matrix");
}

ozk_status ozk_pair_list(int d, const double* amax, const double* bmax, double drop, int* pairs,
                         int* npairs) {
    if (d < 1) return fail(OZK_EPARAM, "pair_list: split count must be >= 1");
    if (d > kMaxSplits) return fail(OZK_EPARAM, "pair_list: split count above 65535 is not supported");
    if (drop < 0.0) return fail(OZK_EPARAM, "pair_list: negative drop threshold");
    PairList pl;
    if (drop > 0.0)
        pruned_pairs(d, amax, bmax, drop, pl);
    else
        triangular_pairs(d, pl);
    for (int p = 0; p < pl.count; ++p) {
        pairs[2 * p] = pl.alpha[p];
        pairs[2 * p + 1] = pl.beta[p];
    }
    *npairs = pl.count;
    return OZK_OK;
}

static ozk_status fill_pairs(int d, const int* pairs, int npairs, PairList& pl) {
    if (npairs < 0 || (npairs > 0 && !pairs)) return fail(OZK_EPARAM, "bad pair list");
    pl.clear();
    for (int p = 0; p < npairs; ++p) {
        if (pairs[2 * p] < 0 || pairs[2 * p] >= d || pairs[2 * p + 1] < 0 ||
            pairs[2 * p + 1] >= d)
            return fail(OZK_EPARAM, "pair index out of range");
        pl.push(pairs[2 * p], pairs[2 * p + 1]);
    }
    return OZK_OK;
}

ozk_status ozk_slices_gemm_device(ozk_format fmt, size_t m, size_t l, size_t n,
                                  const double* a_slices, const double* b_slices, size_t ncb,
                                  size_t nblk, size_t b_blk_stride, int d, const int* pairs,
                                  int npairs, void* c, size_t ldc, void* stream) {
    if (!valid_fmt(fmt)) return fail(OZK_EPARAM, "slices_gemm: format must be DD, TD, QD or TS");
    if (m == 0 || l == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (d < 1 || d > kMaxSplits) return fail(OZK_EPARAM, "slices_gemm: bad split count");
    if (ncb == 0 || nblk == 0 || ncb * nblk < n) return fail(OZK_ESHAPE, "slices_gemm: bad column blocks");
    if (ldc < n) return fail(OZK_ESHAPE, "slices_gemm: ldc < n");
    PairList pl;
    if (ozk_status s = fill_pairs(d, pairs, npairs, pl)) return s;
    if (ozk_status s = need({a_slices, b_slices, c}, "slices_gemm")) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t ldk = slice_ld(l);
    GemmProblem prob{};
    prob.a = a_slices;
    prob.lda = ldk;
    prob.a_slice_stride = m * ldk;
    prob.a_slices = d;
    prob.b = b_slices;
    prob.ldb = ldk;
    prob.b_slice_stride = ncb * ldk;
    prob.b_blk_stride = nblk > 1 ? b_blk_stride : (size_t)d * ncb * ldk;
    prob.b_slices = d;
    prob.ncb = (int)ncb;
    prob.nblk = (int)nblk;
    prob.m = m;
    prob.n = n;
    prob.l = l;
    prob.c = c;
    prob.ldc = ldc;
    if (pl.count == 0) {
        // nothing survives pruning: C = 0
        OZK_CUDA(cudaMemset2DAsync(c, ldc * elem_bytes(fmt), 0, n * elem_bytes(fmt), m, st),
                 "slices_gemm: zero");
    } else {
        OZK_CUDA(launch_pair_gemm(words_of(fmt), kAccumulate, prob, pl, st, num_sms_cached(),
                                  word_bytes_of(fmt)),
                 "slices_gemm");
    }
    OZK_CUDA(cudaStreamSynchronize(st), "slices_gemm");
    return OZK_OK;
}

int ozk_auto_split_count(ozk_format fmt, size_t inner_dim) {
    if (!valid_fmt(fmt) || inner_dim == 0) return 0;
    const int S = word_bytes_of(fmt) == 4 ? 24 : 53;
    const int K = words_of(fmt);
    const int sigma = shift_bits(inner_dim, S);
    const int per = S - sigma;  // significand bits one slice captures
    if (per <= 0) return kMaxSplits;
    const int d = (S * K + per - 1) / per + 2;
    return d < kMaxSplits ? d : kMaxSplits;
}

namespace {
// Host barrier for the per-device threads of ozk_ozaki_gemm_multi.  Every
// thread arrives at every barrier, failed or not, so none can hang.
struct HostBarrier {
    std::mutex mu;
    std::condition_variable cv;
    int n, count = 0, gen = 0;
    explicit HostBarrier(int parties) : n(parties) {}
    void arrive_and_wait() {
        std::unique_lock<std::mutex> lk(mu);
        const int g = gen;
        if (++count == n) {
            count = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};
}  // namespace

ozk_status ozk_ozaki_gemm_multi(ozk_format fmt, int ngpus, const int* devices, size_t m, size_t l,
                                size_t n, const void* a, const void* b, int split_count,
                                double drop, void* c, ozk_profile* prof) {
    if (ozk_status s = check_gemm_args(fmt, m, l, n, split_count, drop)) return s;
    if (ngpus < 1 || ngpus > 64) return fail(OZK_EPARAM, "ozaki_gemm_multi: 1..64 devices");
    if (ozk_status s = need({a, b, c}, "ozaki_gemm_multi")) return s;
    const int d = split_count;
    const size_t eb = elem_bytes(fmt);
    const int nd = engine_setting() != OZK_ENGINE_DMMA ? int8_digits(fmt, l, d) : 0;
    const size_t ld8 = (l + 15) & ~size_t(15);
    const size_t ncb = (n + ngpus - 1) / ngpus;  // B columns per device (ceil partition)
    const size_t n_pad = ncb * (size_t)ngpus;
    auto dev_of = [&](int r) { return devices ? devices[r] : r; };
    auto rows_of = [&](int r, size_t& r0, size_t& r1) {
        r0 = m * (size_t)r / ngpus;
        r1 = m * (size_t)(r + 1) / ngpus;
    };
    HostBarrier bar(ngpus);
    std::vector<ozk_status> st(ngpus, OZK_OK);
    std::vector<std::string> msg(ngpus);
    std::vector<int8_t*> b8_of(ngpus, nullptr);  // each device's gathered B digit planes
    std::vector<int*> gb_of(ngpus, nullptr);
    std::vector<double> maxima((size_t)ngpus * 2 * d, 0.0);
    std::vector<double> secs(ngpus, 0.0);
    std::atomic<bool> failed{false};
    std::atomic<int> pairs_used{-1};
    auto worker = [&](int r) {
        auto t0 = std::chrono::steady_clock::now();
        size_t r0, r1;
        rows_of(r, r0, r1);
        const size_t rows = r1 - r0;
        const size_t c0 = std::min(n, (size_t)r * ncb), c1 = std::min(n, c0 + ncb);
        auto fail_here = [&](ozk_status s) {
            st[r] = s;
            msg[r] = g_last_error;
            failed = true;
        };
        auto cuda_ok = [&](cudaError_t e, const char* what) {
            if (e == cudaSuccess) return true;
            fail_here(fail(OZK_ECUDA, std::string(what) + ": " + cudaGetErrorString(e)));
            return false;
        };
        OwnStream os;
        DevBuf da, db, dc, a8, ga, b8, gb, pmax;
        bool ok = cuda_ok(cudaSetDevice(dev_of(r)), "ozaki_gemm_multi: device") &&
                  cuda_ok(os.create(), "ozaki_gemm_multi: stream");
        if (ok && nd == 0) {
            // DMMA engine or an inner dimension the INT8 engine does not take:
            // this device's rows against the whole B.  With pruning, the pair
            // list comes from the GLOBAL slice maxima (every device's rows, as
            // the reference's piece_max over all of A, ozaki.hpp:194-208), so
            // every device keeps the same pairs as the 1-GPU call.
            DevBuf work, mx;
            ok = cuda_ok(da.alloc(eb * std::max<size_t>(rows, 1) * l, os.s), "alloc A") &&
                 cuda_ok(db.alloc(eb * l * n, os.s), "alloc B") &&
                 cuda_ok(dc.alloc(eb * std::max<size_t>(rows, 1) * n, os.s), "alloc C") &&
                 cuda_ok(work.alloc(eb * l * std::max(std::max<size_t>(rows, 1), n), os.s),
                         "alloc") &&
                 cuda_ok(mx.alloc(8 + 16 * (size_t)d, os.s), "alloc") &&
                 cuda_ok(cudaMemsetAsync(mx.p, 0, 8 + 16 * (size_t)d, os.s), "memset");
            if (ok && rows)
                ok = cuda_ok(cudaMemcpyAsync(da.p, static_cast<const char*>(a) + r0 * l * eb,
                                             rows * l * eb, cudaMemcpyHostToDevice, os.s),
                             "ozaki_gemm_multi: H2D A");
            if (ok)
                ok = cuda_ok(cudaMemcpyAsync(db.p, b, eb * l * n, cudaMemcpyHostToDevice, os.s),
                             "ozaki_gemm_multi: H2D B");
            if (ok && drop > 0.0) {
                // maxima only: the split kernel without slice outputs
                int* ferr = mx.as<int>();
                auto* am = reinterpret_cast<unsigned long long*>(mx.as<char>() + 8);
                if (rows)
                    ok = cuda_ok(split_to_slices(fmt, rows, l, l, da.p, d, OZK_SIDE_ROWS, nullptr,
                                                 rows, work.p, am, ferr, os.s),
                                 "ozaki_gemm_multi: maxima A");
                if (ok)
                    ok = cuda_ok(split_to_slices(fmt, l, n, n, db.p, d, OZK_SIDE_COLS, nullptr, n,
                                                 work.p, am + d, ferr + 1, os.s),
                                 "ozaki_gemm_multi: maxima B");
                std::vector<double> host(1 + 2 * (size_t)d);
                if (ok)
                    ok = cuda_ok(cudaMemcpyAsync(host.data(), mx.p, 8 + 16 * (size_t)d,
                                                 cudaMemcpyDeviceToHost, os.s),
                                 "ozaki_gemm_multi: maxima") &&
                         cuda_ok(cudaStreamSynchronize(os.s), "ozaki_gemm_multi: maxima");
                if (ok) {
                    int flag[2];
                    std::memcpy(flag, host.data(), sizeof(flag));
                    for (int f : flag)
                        if (ok && f) {
                            const ozk_status s2 = check_dev_err(f, "split_matrix");
                            fail_here(s2);
                            ok = false;
                        }
                    std::memcpy(maxima.data() + (size_t)r * 2 * d, host.data() + 1,
                                sizeof(double) * 2 * d);
                }
            }
            bar.arrive_and_wait();  // every device's maxima are in
            if (ok && !failed && rows) {
                PairList pl;
                if (drop > 0.0) {
                    std::vector<double> am(d, 0.0), bm(d, 0.0);
                    for (int q = 0; q < ngpus; ++q)
                        for (int s2 = 0; s2 < d; ++s2) {
                            am[s2] = std::max(am[s2], maxima[(size_t)q * 2 * d + s2]);
                            bm[s2] = std::max(bm[s2], maxima[(size_t)q * 2 * d + d + s2]);
                        }
                    pruned_pairs(d, am.data(), bm.data(), drop, pl);
                } else {
                    triangular_pairs(d, pl);
                }
                pairs_used = pl.count;
                const ozk_status s2 = ozaki_device_impl(fmt, rows, l, n, da.p, l, db.p, n, d, drop,
                                                        dc.p, os.s, nullptr, nullptr, &pl);
                if (s2 != OZK_OK) fail_here(s2), ok = false;
                if (ok)
                    ok = cuda_ok(cudaMemcpyAsync(static_cast<char*>(c) + r0 * n * eb, dc.p,
                                                 rows * n * eb, cudaMemcpyDeviceToHost, os.s),
                                 "ozaki_gemm_multi: D2H C") &&
                         cuda_ok(cudaStreamSynchronize(os.s), "ozaki_gemm_multi");
            }
            bar.arrive_and_wait();
            bar.arrive_and_wait();
            secs[r] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            return;
        }
        // 1. copies in, splits: A rows locally, B column block into its place
        //    in the full-width digit planes
        if (ok) {
            ok = cuda_ok(da.alloc(eb * std::max<size_t>(rows, 1) * l, os.s), "alloc A") &&
                 cuda_ok(db.alloc(eb * l * std::max<size_t>(c1 - c0, 1), os.s), "alloc B") &&
                 cuda_ok(dc.alloc(eb * std::max<size_t>(rows, 1) * n, os.s), "alloc C") &&
                 cuda_ok(a8.alloc((size_t)d * nd * std::max<size_t>(rows, 1) * ld8, os.s), "alloc") &&
                 cuda_ok(ga.alloc(sizeof(int) * d * std::max<size_t>(rows, 1), os.s), "alloc") &&
                 cuda_ok(b8.alloc((size_t)d * nd * n_pad * ld8, os.s), "alloc") &&
                 cuda_ok(gb.alloc(sizeof(int) * d * n_pad, os.s), "alloc") &&
                 cuda_ok(pmax.alloc(sizeof(double) * 2 * d, os.s), "alloc") &&
                 cuda_ok(cudaMemsetAsync(pmax.p, 0, sizeof(double) * 2 * d, os.s), "memset") &&
                 cuda_ok(cudaMemsetAsync(b8.p, 0, (size_t)d * nd * n_pad * ld8, os.s), "memset") &&
                 cuda_ok(cudaMemsetAsync(gb.p, 0, sizeof(int) * d * n_pad, os.s), "memset");
        }
        if (ok && rows)
            ok = cuda_ok(cudaMemcpyAsync(da.p, static_cast<const char*>(a) + r0 * l * eb,
                                         rows * l * eb, cudaMemcpyHostToDevice, os.s),
                         "ozaki_gemm_multi: H2D A");
        if (ok && c1 > c0)
            ok = cuda_ok(cudaMemcpy2DAsync(db.p, (c1 - c0) * eb,
                                           static_cast<const char*>(b) + c0 * eb, n * eb,
                                           (c1 - c0) * eb, l, cudaMemcpyHostToDevice, os.s),
                         "ozaki_gemm_multi: H2D B");
        double* pm = pmax.as<double>();
        if (ok && rows) {
            const ozk_status s2 = ozk_split_digits_device(
                fmt, rows, l, l, da.p, d, OZK_SIDE_ROWS, a8.as<int8_t>(), ld8, rows,
                ga.as<int>(), drop > 0.0 ? pm : nullptr, os.s);
            if (s2 != OZK_OK) fail_here(s2), ok = false;
        }
        if (ok && c1 > c0) {
            const ozk_status s2 = ozk_split_digits_device(
                fmt, l, c1 - c0, c1 - c0, db.p, d, OZK_SIDE_COLS, b8.as<int8_t>() + c0 * ld8, ld8,
                n_pad, gb.as<int>() + c0, drop > 0.0 ? pm + d : nullptr, os.s);
            if (s2 != OZK_OK) fail_here(s2), ok = false;
        }
        if (ok && drop > 0.0)
            ok = cuda_ok(cudaMemcpy(maxima.data() + (size_t)r * 2 * d, pm, sizeof(double) * 2 * d,
                                    cudaMemcpyDeviceToHost),
                         "ozaki_gemm_multi: maxima");
        b8_of[r] = b8.as<int8_t>();
        gb_of[r] = gb.as<int>();
        bar.arrive_and_wait();  // every device has split its block
        // 2. pair list (global slice maxima with pruning: every device's
        // maxima are in after the barrier)
        PairList pl;
        std::vector<int> flat;
        if (ok && !failed) {
            if (drop > 0.0) {
                std::vector<double> am(d, 0.0), bm(d, 0.0);
                for (int q = 0; q < ngpus; ++q)
                    for (int s2 = 0; s2 < d; ++s2) {
                        am[s2] = std::max(am[s2], maxima[(size_t)q * 2 * d + s2]);
                        bm[s2] = std::max(bm[s2], maxima[(size_t)q * 2 * d + d + s2]);
                    }
                pruned_pairs(d, am.data(), bm.data(), drop, pl);
            } else {
                triangular_pairs(d, pl);
            }
            pairs_used = pl.count;
            flat.resize(2 * (size_t)pl.count);
            for (int p = 0; p < pl.count; ++p) {
                flat[2 * p] = pl.alpha[p];
                flat[2 * p + 1] = pl.beta[p];
            }
        }
        // C columns [q0, q1) of this device's rows from the digit planes at
        // plane rows [q0, q1) (the n_pad layout: column j is plane row j)
        auto gemm_cols = [&](size_t q0, size_t q1) -> bool {
            if (!rows || q1 <= q0 || pl.count == 0) return true;
            const ozk_status s2 = ozk_digits_gemm_device_async(
                fmt, rows, l, q1 - q0, a8.as<int8_t>(), ga.as<int>(), rows,
                b8.as<int8_t>() + q0 * ld8, gb.as<int>() + q0, n_pad, ld8, d, flat.data(),
                pl.count, static_cast<char*>(dc.p) + q0 * eb, n, os.s);
            if (s2 != OZK_OK) fail_here(s2);
            return s2 == OZK_OK;
        };
        // 3. the device's own B column block is multiplied while the other
        // blocks arrive: all-gather of the B digit planes and exponents by peer
        // copies on a second stream (C elements are independent: the same bits
        // as one GEMM over all columns)
        OwnStream cs;
        if (ok && !failed) ok = cuda_ok(cs.create(), "ozaki_gemm_multi: stream");
        if (ok && !failed) ok = gemm_cols(c0, c1);
        if (ok && !failed) {
            for (int q = 0; q < ngpus && ok; ++q) {
                if (q == r) continue;
                const size_t q0 = std::min(n, (size_t)q * ncb), q1 = std::min(n, q0 + ncb);
                if (q1 <= q0) continue;
                for (int s2 = 0; s2 < d * nd && ok; ++s2) {
                    const size_t off = ((size_t)s2 * n_pad + q0) * ld8;
                    ok = cuda_ok(cudaMemcpyPeerAsync(b8_of[r] + off, dev_of(r), b8_of[q] + off,
                                                     dev_of(q), (q1 - q0) * ld8, cs.s),
                                 "ozaki_gemm_multi: peer copy");
                }
                for (int s2 = 0; s2 < d && ok; ++s2) {
                    const size_t off = (size_t)s2 * n_pad + q0;
                    ok = cuda_ok(cudaMemcpyPeerAsync(gb_of[r] + off, dev_of(r), gb_of[q] + off,
                                                     dev_of(q), (q1 - q0) * sizeof(int), cs.s),
                                 "ozaki_gemm_multi: peer copy");
                }
            }
        }
        if (cs.s) {
            const bool synced = cuda_ok(cudaStreamSynchronize(cs.s), "ozaki_gemm_multi: gather");
            ok = ok && synced;
        }
        bar.arrive_and_wait();  // no device frees what a peer still reads
        // 4. the gathered columns on either side, C rows back
        if (ok && !failed && rows) {
            if (pl.count == 0)
                ok = cuda_ok(cudaMemsetAsync(dc.p, 0, eb * rows * n, os.s), "memset C");
            else
                ok = gemm_cols(0, c0) && gemm_cols(c1, n);
            if (ok)
                ok = cuda_ok(cudaMemcpyAsync(static_cast<char*>(c) + r0 * n * eb, dc.p,
                                             rows * n * eb, cudaMemcpyDeviceToHost, os.s),
                             "ozaki_gemm_multi: D2H C") &&
                     cuda_ok(cudaStreamSynchronize(os.s), "ozaki_gemm_multi");
        }
        bar.arrive_and_wait();
        secs[r] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    // worker 0 runs on the caller's thread: its current device is restored after
    int caller_dev = 0;
    OZK_CUDA(cudaGetDevice(&caller_dev), "ozaki_gemm_multi: device");
    // Direct peer access between every pair of distinct devices, so the
    // digit-plane all-gather (cudaMemcpyPeerAsync) runs device to device over
    // NVLink / NVSwitch instead of being staged through host memory.
    {
        std::vector<int> ids;
        for (int r = 0; r < ngpus; ++r)
            if (std::find(ids.begin(), ids.end(), dev_of(r)) == ids.end()) ids.push_back(dev_of(r));
        for (int i : ids)
            for (int j : ids) {
                if (i == j) continue;
                int can = 0;
                if (cudaDeviceCanAccessPeer(&can, i, j) != cudaSuccess || !can) {
                    (void)cudaGetLastError();
                    continue;
                }
                OZK_CUDA(cudaSetDevice(i), "ozaki_gemm_multi: device");
                const cudaError_t e = cudaDeviceEnablePeerAccess(j, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                    cudaSetDevice(caller_dev);
                    return cuda_fail(e, "ozaki_gemm_multi: peer access");
                }
                (void)cudaGetLastError();  // clear "already enabled"
            }
        OZK_CUDA(cudaSetDevice(caller_dev), "ozaki_gemm_multi: device");
    }
    std::vector<std::thread> threads;
    for (int r = 1; r < ngpus; ++r) threads.emplace_back(worker, r);
    worker(0);
    for (auto& t : threads) t.join();
    cudaSetDevice(caller_dev);
    for (int r = 0; r < ngpus; ++r)
        if (st[r] != OZK_OK) {
            g_last_error = msg[r];
            return st[r];
        }
    if (prof) {
        *prof = ozk_profile{};
        prof->total_seconds = *std::max_element(secs.begin(), secs.end());
        prof->split_count = d;
        PairList pl;
        triangular_pairs(d, pl);
        prof->pairs = pairs_used.load() >= 0 ? pairs_used.load() : pl.count;
        prof->gpus = ngpus;
        prof->engine = nd > 0 ? OZK_ENGINE_INT8 : OZK_ENGINE_DMMA;
    }
    return OZK_OK;
}

int ozk_plan_row_bands(ozk_format fmt, size_t m, size_t n, size_t l, int split_count,
                       size_t block_cols, int group_rows, int group_cols, int clusters,
                       int cluster_sms, size_t* starts, int max_bands) {
    if (!valid_fmt(fmt) || !starts || max_bands < 1 || split_count < 1 || group_rows <= 0 ||
        group_cols <= 0 || cluster_sms <= 0 || block_cols == 0)
        return -1;
    I8Geometry g;
    g.group_rows = group_rows;
    g.group_cols = group_cols;
    g.clusters = clusters;
    g.cluster_sms = cluster_sms;
    const std::vector<size_t> plan =
        plan_bands_uncached((int)fmt, m, n, l, split_count, block_cols, g);
    const int bands = (int)plan.size() - 1;
    if (bands > max_bands) return -1;
    for (size_t q = 0; q < plan.size(); ++q) starts[q] = plan[q];
    return bands;
}

double ozk_auto_drop_threshold(ozk_format fmt, size_t inner_dim) {
    if (!valid_fmt(fmt) || inner_dim == 0) return 0.0;
    const int S = word_bytes_of(fmt) == 4 ? 24 : 53;
    int cl = 0;
    while ((size_t(1) << cl) < inner_dim) ++cl;
    return std::ldexp(1.0, -(S * words_of(fmt) + cl + 2));
}

int ozk_int8_digits(ozk_format fmt, size_t inner_dim, int d) {
    if (!valid_fmt(fmt)) return 0;
    return int8_digits(fmt, inner_dim, d);
}

ozk_status ozk_split_digits_device_async(ozk_format fmt, size_t rows, size_t cols, size_t ld,
                                         const void* mat, int d, ozk_side side, int8_t* digits,
                                         size_t ld8, size_t plane_rows, int* exps,
                                         double* piece_max, int* dev_flag, void* stream) {
    if (!valid_fmt(fmt)) return fail(OZK_EPARAM, "split_digits: format must be DD, TD, QD or TS");
    if (rows == 0 || cols == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (d < 1) return fail(OZK_EPARAM, "split_matrix: split count must be >= 1");
    if (d > kMaxSplits) return fail(OZK_EPARAM, "split_matrix: split count above 65535 is not supported");
    if (ld < cols) return fail(OZK_ESHAPE, "split_matrix: ld < cols");
    const size_t inner = side == OZK_SIDE_ROWS ? cols : rows;
    const size_t outer = side == OZK_SIDE_ROWS ? rows : cols;
    const int nd = int8_digits(fmt, inner, d);
    if (nd == 0) return fail(OZK_EPARAM, "split_digits: INT8 engine not applicable to this inner dimension");
    if (ld8 < inner || ld8 % 16) return fail(OZK_ESHAPE, "split_digits: ld8 must be >= inner and a multiple of 16");
    if (plane_rows < outer) return fail(OZK_ESHAPE, "split_digits: plane_rows < outer dimension");
    if (!digits || !exps || !dev_flag) return fail(OZK_EPARAM, "split_digits: null output");
    if (ozk_status s = need({mat}, "split_digits")) return s;
    cudaStream_t st = (cudaStream_t)stream;
    num_sms_cached();
    DigitOut dig;
    dig.nd = nd;
    dig.digits = digits;
    dig.ld = ld8;
    dig.digit_stride = plane_rows * ld8;
    dig.slice_stride = (size_t)nd * plane_rows * ld8;
    dig.exps = exps;
    dig.exp_stride = plane_rows;
    DevBuf work;  // stream-ordered: freed after the split on `stream`
    OZK_CUDA(work.alloc(elem_bytes(fmt) * rows * cols, st), "split_digits: work");
    OZK_CUDA(split_to_slices(fmt, rows, cols, ld, mat, d, side, nullptr, plane_rows, work.p,
                             reinterpret_cast<unsigned long long*>(piece_max), dev_flag, st, dig),
             "split_digits");
    return OZK_OK;
}

ozk_status ozk_check_split_flag(const int* dev_flag, void* stream) {
    int flag = 0;
    cudaStream_t st = (cudaStream_t)stream;
    OZK_CUDA(cudaMemcpyAsync(&flag, dev_flag, sizeof(int), cudaMemcpyDeviceToHost, st),
             "split flag");
    OZK_CUDA(cudaStreamSynchronize(st), "split flag");
    return check_dev_err(flag, "split_matrix");
}

ozk_status ozk_split_digits_device(ozk_format fmt, size_t rows, size_t cols, size_t ld,
                                   const void* mat, int d, ozk_side side, int8_t* digits,
                                   size_t ld8, size_t plane_rows, int* exps, double* piece_max,
                                   void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    DevBuf flags;
    OZK_CUDA(flags.alloc(8, st), "split_digits: flags");
    OZK_CUDA(cudaMemsetAsync(flags.p, 0, 8, st), "split_digits: memset");
    if (ozk_status s = ozk_split_digits_device_async(fmt, rows, cols, ld, mat, d, side, digits,
                                                     ld8, plane_rows, exps, piece_max,
                                                     flags.as<int>(), stream))
        return s;
    return ozk_check_split_flag(flags.as<int>(), stream);
}

ozk_status ozk_digits_gemm_device_async(ozk_format fmt, size_t m, size_t l, size_t n,
                                        const int8_t* a_digits, const int* a_exps,
                                        size_t a_plane_rows, const int8_t* b_digits,
                                        const int* b_exps, size_t b_plane_rows, size_t ld8, int d,
                                        const int* pairs, int npairs, void* c, size_t ldc,
                                        void* stream) {
    if (!valid_fmt(fmt)) return fail(OZK_EPARAM, "digits_gemm: format must be DD, TD, QD or TS");
    if (m == 0 || l == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (d < 1 || d > kMaxSplits) return fail(OZK_EPARAM, "digits_gemm: bad split count");
    const int nd = int8_digits(fmt, l, d);
    if (nd == 0) return fail(OZK_EPARAM, "digits_gemm: INT8 engine not applicable to this inner dimension");
    if (ld8 < l || ld8 % 16) return fail(OZK_ESHAPE, "digits_gemm: ld8 must be >= l and a multiple of 16");
    if (a_plane_rows < m || b_plane_rows < n) return fail(OZK_ESHAPE, "digits_gemm: plane_rows too small");
    if (ldc < n) return fail(OZK_ESHAPE, "digits_gemm: ldc < n");
    PairList pl;
    if (ozk_status s = fill_pairs(d, pairs, npairs, pl)) return s;
    if (ozk_status s = need({a_digits, a_exps, b_digits, b_exps, c}, "digits_gemm")) return s;
    cudaStream_t st = (cudaStream_t)stream;
    if (pl.count == 0) {
        OZK_CUDA(cudaMemset2DAsync(c, ldc * elem_bytes(fmt), 0, n * elem_bytes(fmt), m, st),
                 "digits_gemm: zero");
    } else {
        I8Operands op{};
        op.nd = nd;
        op.a = a_digits;
        op.a_ld = ld8;
        op.a_digit_stride = a_plane_rows * ld8;
        op.a_slice_stride = (size_t)nd * a_plane_rows * ld8;
        op.b = b_digits;
        op.b_ld = ld8;
        op.b_digit_stride = b_plane_rows * ld8;
        op.b_slice_stride = (size_t)nd * b_plane_rows * ld8;
        op.gA = a_exps;
        op.gB = b_exps;
        op.gA_stride = a_plane_rows;
        op.gB_stride = b_plane_rows;
        op.m = m;
        op.n = n;
        op.l = l;
        op.d = d;
        op.c = c;
        op.ldc = ldc;
        OZK_CUDA(launch_pair_gemm_i8(words_of(fmt), word_bytes_of(fmt), op, pl, st,
                                     num_sms_cached()),
                 "digits_gemm");
    }
    return OZK_OK;
}

ozk_status ozk_digits_gemm_device(ozk_format fmt, size_t m, size_t l, size_t n,
                                  const int8_t* a_digits, const int* a_exps, size_t a_plane_rows,
                                  const int8_t* b_digits, const int* b_exps, size_t b_plane_rows,
                                  size_t ld8, int d, const int* pairs, int npairs, void* c,
                                  size_t ldc, void* stream) {
    if (ozk_status s = ozk_digits_gemm_device_async(fmt, m, l, n, a_digits, a_exps, a_plane_rows,
                                                    b_digits, b_exps, b_plane_rows, ld8, d, pairs,
                                                    npairs, c, ldc, stream))
        return s;
    OZK_CUDA(cudaStreamSynchronize((cudaStream_t)stream), "digits_gemm");
    return OZK_OK;
}

ozk_status ozk_pair_products_digits_device(ozk_format fmt, size_t m, size_t l, size_t n,
                                           const int8_t* a_digits, const int* a_exps,
                                           size_t a_plane_rows, const int8_t* b_digits,
                                           const int* b_exps, size_t b_plane_rows, size_t ld8,
                                           int d, const int* pairs, int npairs, double* products,
                                           void* stream) {
    if (!valid_fmt(fmt)) return fail(OZK_EPARAM, "pair_products: format must be DD, TD, QD or TS");
    if (m == 0 || l == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (d < 1 || d > kMaxSplits) return fail(OZK_EPARAM, "pair_products: bad split count");
    const int nd = int8_digits(fmt, l, d);
    if (nd == 0) return fail(OZK_EPARAM, "pair_products: INT8 engine not applicable to this inner dimension");
    if (ld8 < l || ld8 % 16) return fail(OZK_ESHAPE, "pair_products: ld8 must be >= l and a multiple of 16");
    if (a_plane_rows < m || b_plane_rows < n) return fail(OZK_ESHAPE, "pair_products: plane_rows too small");
    PairList pl;
    if (ozk_status s = fill_pairs(d, pairs, npairs, pl)) return s;
    if (ozk_status s = need({a_digits, a_exps, b_digits, b_exps, products}, "pair_products"))
        return s;
    cudaStream_t st = (cudaStream_t)stream;
    if (pl.count > 0) {
        I8Operands op{};
        op.nd = nd;
        op.a = a_digits;
        op.a_ld = ld8;
        op.a_digit_stride = a_plane_rows * ld8;
        op.a_slice_stride = (size_t)nd * a_plane_rows * ld8;
        op.b = b_digits;
        op.b_ld = ld8;
        op.b_digit_stride = b_plane_rows * ld8;
        op.b_slice_stride = (size_t)nd * b_plane_rows * ld8;
        op.gA = a_exps;
        op.gB = b_exps;
        op.gA_stride = a_plane_rows;
        op.gB_stride = b_plane_rows;
        op.m = m;
        op.n = n;
        op.l = l;
        op.d = d;
        op.c = products;
        op.ldc = n;
        op.pair_stride = m * n;
        OZK_CUDA(launch_pair_products_i8(word_bytes_of(fmt), op, pl, st, num_sms_cached()),
                 "pair_products");
    }
    OZK_CUDA(cudaStreamSynchronize(st), "pair_products");
    return OZK_OK;
}

ozk_status ozk_pair_products_device(size_t m, size_t l, size_t n, const double* a_slices,
                                    const double* b_slices, int d, const int* pairs, int npairs,
                                    double* products, void* stream) {
    if (m == 0 || l == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (d < 1 || d > kMaxSplits) return fail(OZK_EPARAM, "pair_products: bad split count");
    PairList pl;
    if (ozk_status s = fill_pairs(d, pairs, npairs, pl)) return s;
    if (ozk_status s = need({a_slices, b_slices, products}, "pair_products")) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t ldk = slice_ld(l);
    GemmProblem prob{};
    prob.a = a_slices;
    prob.lda = ldk;
    prob.a_slice_stride = m * ldk;
    prob.a_slices = d;
    prob.b = b_slices;
    prob.ldb = ldk;
    prob.b_slice_stride = n * ldk;
    prob.b_blk_stride = (size_t)d * n * ldk;
    prob.b_slices = d;
    prob.ncb = (int)n;
    prob.nblk = 1;
    prob.m = m;
    prob.n = n;
    prob.l = l;
    prob.c = products;
    prob.ldc = n;
    prob.c_pair_stride = m * n;
    OZK_CUDA(launch_pair_gemm(1, kStoreProducts, prob, pl, st, num_sms_cached()), "pair_products");
    OZK_CUDA(cudaStreamSynchronize(st), "pair_products");
    return OZK_OK;
}

ozk_status ozk_backend_gemm_device(size_t m, size_t l, size_t n, const double* a,
                                   const double* b, double* c, void* stream) {
    if (m == 0 || l == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (m > 0x7fffffffull || n > 0x7fffffffull || l > 0x7fffffffull)
        return fail(OZK_ESHAPE, "backend_gemm: dimension too large");
    if (ozk_status s = need({a, b, c}, "backend_gemm")) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t ldk = slice_ld(l);
    DevBuf ap, bt;
    OZK_CUDA(ap.alloc(sizeof(double) * m * ldk, st), "backend_gemm: A");
    OZK_CUDA(bt.alloc(sizeof(double) * n * ldk, st), "backend_gemm: B^T");
    if (ldk != l) OZK_CUDA(cudaMemsetAsync(ap.p, 0, sizeof(double) * m * ldk, st), "backend_gemm");
    OZK_CUDA(cudaMemsetAsync(bt.p, 0, sizeof(double) * n * ldk, st), "backend_gemm");
    OZK_CUDA(cudaMemcpy2DAsync(ap.p, ldk * 8, a, l * 8, l * 8, m, cudaMemcpyDeviceToDevice, st),
             "backend_gemm: pad A");
    OZK_CUDA(launch_transpose(1, 8, b, n, bt.p, ldk, l, n, st), "backend_gemm: B^T");
    GemmProblem prob{};
    prob.a = ap.as<double>();
    prob.lda = ldk;
    prob.a_slice_stride = m * ldk;
    prob.a_slices = 1;
    prob.b = bt.as<double>();
    prob.ldb = ldk;
    prob.b_slice_stride = n * ldk;
    prob.b_blk_stride = n * ldk;
    prob.b_slices = 1;
    prob.ncb = (int)n;
    prob.nblk = 1;
    prob.m = m;
    prob.n = n;
    prob.l = l;
    prob.c = c;
    prob.ldc = n;
    PairList pl;
    triangular_pairs(1, pl);
    OZK_CUDA(launch_pair_gemm(1, kStorePlain, prob, pl, st, num_sms_cached()), "backend_gemm");
    OZK_CUDA(cudaStreamSynchronize(st), "backend_gemm");
    return OZK_OK;
}

ozk_status ozk_backend_gemm(size_t m, size_t l, size_t n, const double* a, const double* b,
                            double* c) {
    if (m == 0 || l == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (ozk_status s = need({a, b, c}, "backend_gemm")) return s;
    OwnStream os;
    OZK_CUDA(os.create(), "backend_gemm: stream");
    num_sms_cached();
    DevBuf da, db, dc;
    OZK_CUDA(da.alloc(sizeof(double) * m * l, os.s), "backend_gemm: A");
    OZK_CUDA(db.alloc(sizeof(double) * l * n, os.s), "backend_gemm: B");
    OZK_CUDA(dc.alloc(sizeof(double) * m * n, os.s), "backend_gemm: C");
    OZK_CUDA(cudaMemcpyAsync(da.p, a, sizeof(double) * m * l, cudaMemcpyHostToDevice, os.s),
             "backend_gemm: H2D");
    OZK_CUDA(cudaMemcpyAsync(db.p, b, sizeof(double) * l * n, cudaMemcpyHostToDevice, os.s),
             "backend_gemm: H2D");
    if (ozk_status s = ozk_backend_gemm_device(m, l, n, da.as<double>(), db.as<double>(),
                                               dc.as<double>(), os.s))
        return s;
    OZK_CUDA(cudaMemcpyAsync(c, dc.p, sizeof(double) * m * n, cudaMemcpyDeviceToHost, os.s),
             "backend_gemm: D2H");
    OZK_CUDA(cudaStreamSynchronize(os.s), "backend_gemm");
    return OZK_OK;
}

ozk_status ozk_accumulate_products_device(ozk_format fmt, size_t m, size_t n,
                                          const double* products, int nproducts, void* c,
                                          void* stream) {
    if (!valid_fmt(fmt)) return fail(OZK_EPARAM, "accumulate: format must be DD, TD, QD or TS");
    if (m == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (nproducts < 0) return fail(OZK_EPARAM, "accumulate: negative product count");
    if (nproducts > 0 && !products) return fail(OZK_EPARAM, "accumulate: null pointer");
    if (ozk_status s = need({c}, "accumulate")) return s;
    cudaStream_t st = (cudaStream_t)stream;
    if (nproducts == 0) {
        OZK_CUDA(cudaMemsetAsync(c, 0, elem_bytes(fmt) * m * n, st), "accumulate: zero");
    } else {
        OZK_CUDA(launch_accumulate_products(words_of(fmt), word_bytes_of(fmt), products, nproducts,
                                            m * n, c, st),
                 "accumulate");
    }
    OZK_CUDA(cudaStreamSynchronize(st), "accumulate");
    return OZK_OK;
}

ozk_status ozk_accumulate_products(ozk_format fmt, size_t m, size_t n,
                                   const double* const* products, int nproducts, void* c) {
    if (!valid_fmt(fmt)) return fail(OZK_EPARAM, "accumulate: format must be DD, TD, QD or TS");
    if (m == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (nproducts < 0 || (nproducts > 0 && !products))
        return fail(OZK_EPARAM, "accumulate: bad product list");
    if (ozk_status s = need({c}, "accumulate")) return s;
    for (int p = 0; p < nproducts; ++p)
        if (!products[p]) return fail(OZK_EPARAM, "accumulate: null pointer");
    const size_t eb = elem_bytes(fmt);
    OwnStream os;
    OZK_CUDA(os.create(), "accumulate: stream");
    num_sms_cached();
    // row blocks keep the device copy of the products under ~1 GiB
    const size_t per_row = (size_t)(nproducts > 0 ? nproducts : 1) * n * sizeof(double);
    size_t rb = ((size_t)1 << 30) / per_row;
    rb = rb < 1 ? 1 : (rb > m ? m : rb);
    DevBuf dp, dc;
    OZK_CUDA(dp.alloc(per_row * rb, os.s), "accumulate: products");
    OZK_CUDA(dc.alloc(eb * rb * n, os.s), "accumulate: C");
    for (size_t r0 = 0; r0 < m; r0 += rb) {
        const size_t rows = m - r0 < rb ? m - r0 : rb;
        for (int p = 0; p < nproducts; ++p)
            OZK_CUDA(cudaMemcpyAsync(dp.as<double>() + (size_t)p * rows * n, products[p] + r0 * n,
                                     rows * n * sizeof(double), cudaMemcpyHostToDevice, os.s),
                     "accumulate: H2D");
        if (ozk_status s = ozk_accumulate_products_device(fmt, rows, n, dp.as<double>(), nproducts,
                                                          dc.p, os.s))
            return s;
        OZK_CUDA(cudaMemcpyAsync(static_cast<char*>(c) + r0 * n * eb, dc.p, rows * n * eb,
                                 cudaMemcpyDeviceToHost, os.s),
                 "accumulate: D2H");
    }
    OZK_CUDA(cudaStreamSynchronize(os.s), "accumulate");
    return OZK_OK;
}

ozk_status ozk_lu_trailing_update_device(ozk_format fmt, size_t tm, size_t pw, size_t tn,
                                         const void* l21, size_t ldl, const void* u12,
                                         size_t ldu, void* a22, size_t lda, int d,
                                         void* stream) {
    if (fmt != OZK_DD && fmt != OZK_TD && fmt != OZK_QD)
        return fail(OZK_EPARAM, "lu_trailing_update: format must be DD, TD or QD");
    if (ozk_status s = check_gemm_args(fmt, tm, pw, tn, d, 0.0)) return s;
    if (ldl < pw || ldu < tn || lda < tn)
        return fail(OZK_ESHAPE, "lu_trailing_update: leading dimension too small");
    if (ozk_status s = need({l21, u12, a22}, "lu_trailing_update")) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const int K = (int)fmt;
    // the running sum lives in `sum`; the last pair's epilogue subtracts it
    // from A22 in place (no separate update matrix pass)
    DevBuf sum;
    OZK_CUDA(sum.alloc(sizeof(double) * K * tm * tn, st), "lu_trailing_update: sum");
    const LuTarget lt{static_cast<double*>(a22), lda};
    if (ozk_status s = ozaki_device_impl(K, tm, pw, tn, l21, ldl, u12, ldu, d, 0.0, sum.p, st,
                                         nullptr, nullptr, nullptr, &lt))
        return s;
    OZK_CUDA(cudaStreamSynchronize(st), "lu_trailing_update");
    return OZK_OK;
}

ozk_status ozk_lu_trailing_update(ozk_format fmt, size_t tm, size_t pw, size_t tn,
                                  const void* l21, size_t ldl, const void* u12, size_t ldu,
                                  void* a22, size_t lda, int d) {
    if (fmt != OZK_DD && fmt != OZK_TD && fmt != OZK_QD)
        return fail(OZK_EPARAM, "lu_trailing_update: format must be DD, TD or QD");
    if (ozk_status s = check_gemm_args(fmt, tm, pw, tn, d, 0.0)) return s;
    if (ldl < pw || ldu < tn || lda < tn)
        return fail(OZK_ESHAPE, "lu_trailing_update: leading dimension too small");
    if (ozk_status s = need({l21, u12, a22}, "lu_trailing_update")) return s;
    const size_t eb = elem_bytes(fmt);
    OwnStream os;
    OZK_CUDA(os.create(), "lu_trailing_update: stream");
    num_sms_cached();
    DevBuf dl, du, da;
    OZK_CUDA(dl.alloc(eb * tm * pw, os.s), "lu_trailing_update: L21");
    OZK_CUDA(du.alloc(eb * pw * tn, os.s), "lu_trailing_update: U12");
    OZK_CUDA(da.alloc(eb * tm * tn, os.s), "lu_trailing_update: A22");
    OZK_CUDA(cudaMemcpy2DAsync(dl.p, eb * pw, l21, eb * ldl, eb * pw, tm, cudaMemcpyHostToDevice,
                               os.s),
             "lu_trailing_update: H2D");
    OZK_CUDA(cudaMemcpy2DAsync(du.p, eb * tn, u12, eb * ldu, eb * tn, pw, cudaMemcpyHostToDevice,
                               os.s),
             "lu_trailing_update: H2D");
    OZK_CUDA(cudaMemcpy2DAsync(da.p, eb * tn, a22, eb * lda, eb * tn, tm, cudaMemcpyHostToDevice,
                               os.s),
             "lu_trailing_update: H2D");
    if (ozk_status s = ozk_lu_trailing_update_device(fmt, tm, pw, tn, dl.p, pw, du.p, tn, da.p,
                                                     tn, d, os.s))
        return s;
    OZK_CUDA(cudaMemcpy2DAsync(a22, eb * lda, da.p, eb * tn, eb * tn, tm, cudaMemcpyDeviceToHost,
                               os.s),
             "lu_trailing_update: D2H");
    OZK_CUDA(cudaStreamSynchronize(os.s), "lu_trailing_update");
    return OZK_OK;
}

ozk_status ozk_ts_direct_gemm_device(size_t m, size_t l, size_t n, const float* a, const float* b,
                                     float* c, void* stream) {
    if (m == 0 || l == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (m > 0x7fffffffull || n > 0x7fffffffull || l > 0x7fffffffull)
        return fail(OZK_ESHAPE, "ts_direct_gemm: dimension too large");
    if (ozk_status s = need({a, b, c}, "ts_direct_gemm")) return s;
    cudaStream_t st = (cudaStream_t)stream;
    OZK_CUDA(launch_ts_direct(a, b, c, m, l, n, st), "ts_direct_gemm");
    OZK_CUDA(cudaStreamSynchronize(st), "ts_direct_gemm");
    return OZK_OK;
}

ozk_status ozk_ts_direct_gemm(size_t m, size_t l, size_t n, const float* a, const float* b,
                              float* c) {
    if (m == 0 || l == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (ozk_status s = need({a, b, c}, "ts_direct_gemm")) return s;
    OwnStream os;
    OZK_CUDA(os.create(), "ts_direct_gemm: stream");
    DevBuf da, db, dc;
    OZK_CUDA(da.alloc(12 * m * l, os.s), "ts_direct_gemm: A");
    OZK_CUDA(db.alloc(12 * l * n, os.s), "ts_direct_gemm: B");
    OZK_CUDA(dc.alloc(12 * m * n, os.s), "ts_direct_gemm: C");
    OZK_CUDA(cudaMemcpyAsync(da.p, a, 12 * m * l, cudaMemcpyHostToDevice, os.s), "ts_direct: H2D");
    OZK_CUDA(cudaMemcpyAsync(db.p, b, 12 * l * n, cudaMemcpyHostToDevice, os.s), "ts_direct: H2D");
    if (ozk_status s = ozk_ts_direct_gemm_device(m, l, n, da.as<float>(), db.as<float>(),
                                                 dc.as<float>(), os.s))
        return s;
    OZK_CUDA(cudaMemcpyAsync(c, dc.p, 12 * m * n, cudaMemcpyDeviceToHost, os.s), "ts_direct: D2H");
    OZK_CUDA(cudaStreamSynchronize(os.s), "ts_direct_gemm");
    return OZK_OK;
}

ozk_status ozk_direct_gemm_device(ozk_format fmt, size_t m, size_t l, size_t n, const void* a,
                                  const void* b, void* c, void* stream) {
    if (fmt != OZK_DD && fmt != OZK_TD && fmt != OZK_QD)
        return fail(OZK_EPARAM, "direct_gemm: format must be DD, TD or QD (TS: ozk_ts_direct_gemm)");
    if (m == 0 || l == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (m > 0xffff0ull * 16 || n > 0xffff0ull * 16) return fail(OZK_ESHAPE, "direct_gemm: dimension too large");
    if (ozk_status s = need({a, b, c}, "direct_gemm")) return s;
    cudaStream_t st = (cudaStream_t)stream;
    OZK_CUDA(launch_direct_gemm(words_of(fmt), static_cast<const double*>(a),
                                static_cast<const double*>(b), static_cast<double*>(c), m, l, n, st),
             "direct_gemm");
    OZK_CUDA(cudaStreamSynchronize(st), "direct_gemm");
    return OZK_OK;
}

ozk_status ozk_direct_gemm(ozk_format fmt, size_t m, size_t l, size_t n, const void* a,
                           const void* b, void* c) {
    if (fmt != OZK_DD && fmt != OZK_TD && fmt != OZK_QD)
        return fail(OZK_EPARAM, "direct_gemm: format must be DD, TD or QD (TS: ozk_ts_direct_gemm)");
    if (m == 0 || l == 0 || n == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (ozk_status s = need({a, b, c}, "direct_gemm")) return s;
    const size_t eb = elem_bytes(fmt);
    OwnStream os;
    OZK_CUDA(os.create(), "direct_gemm: stream");
    DevBuf da, db, dc;
    OZK_CUDA(da.alloc(eb * m * l, os.s), "direct_gemm: A");
    OZK_CUDA(db.alloc(eb * l * n, os.s), "direct_gemm: B");
    OZK_CUDA(dc.alloc(eb * m * n, os.s), "direct_gemm: C");
    OZK_CUDA(cudaMemcpyAsync(da.p, a, eb * m * l, cudaMemcpyHostToDevice, os.s), "direct: H2D");
    OZK_CUDA(cudaMemcpyAsync(db.p, b, eb * l * n, cudaMemcpyHostToDevice, os.s), "direct: H2D");
    if (ozk_status s = ozk_direct_gemm_device(fmt, m, l, n, da.p, db.p, dc.p, os.s)) return s;
    OZK_CUDA(cudaMemcpyAsync(c, dc.p, eb * m * n, cudaMemcpyDeviceToHost, os.s), "direct: D2H");
    OZK_CUDA(cudaStreamSynchronize(os.s), "direct_gemm");
    return OZK_OK;
}

ozk_status ozk_gen_spread_device(ozk_format fmt, size_t rows, size_t cols, uint64_t seed,
                                 int spread, void* out, void* stream) {
    if (!valid_fmt(fmt)) return fail(OZK_EPARAM, "gen: format must be DD, TD, QD or TS");
    if (rows == 0 || cols == 0) return fail(OZK_ESHAPE, "matrix dimensions must be positive");
    if (spread < 0 || spread > 400) return fail(OZK_EPARAM, "gen: spread must be in [0, 400]");
    if (ozk_status s = need({out}, "gen")) return s;
    cudaStream_t st = (cudaStream_t)stream;
    OZK_CUDA(launch_gen_eq1(words_of(fmt), word_bytes_of(fmt), out, rows * cols, seed, spread, st),
             "gen");
    OZK_CUDA(cudaStreamSynchronize(st), "gen");
    return OZK_OK;
}

ozk_status ozk_gen_eq1_device(ozk_format fmt, size_t rows, size_t cols, uint64_t seed,
                              void* out, void* stream) {
    return ozk_gen_spread_device(fmt, rows, cols, seed, 0, out, stream);
}

}  // extern "C"

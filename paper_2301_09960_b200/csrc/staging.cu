// staging.cu -- host<->device copies of PAGEABLE caller buffers for the
// host-buffer entry points (ozk_ozaki_gemm).
//
// A drop-in caller hands over DenseMatrix storage (a std::vector: pageable
// memory).  cudaMemcpyAsync from pageable memory is synchronous for the host
// and goes through the driver's small bounce buffers, so the band schedule of
// ozk_ozaki_gemm (A arriving band by band, B in column blocks, C leaving band
// by band while later bands compute) would serialise behind it.  Here each
// direction has its own worker thread and a ring of pinned slots: the H2D
// worker copies the next chunk of the caller's buffer into a free slot with a
// team of host threads (parallel memcpy) and queues the slot's DMA on the copy
// stream; the D2H worker queues a band's DMA into slots and copies them out as
// they land.  Slot reuse is ordered by per-slot events.  Pinned slot sets are
// cached process-wide and handed out one per concurrent call (the entry points
// are reentrant).
#include <cuda_runtime.h>
#include <emmintrin.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "ozk_internal.cuh"

namespace ozk {

bool host_is_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

namespace {

constexpr int kSlots = 6;                    // per direction
constexpr size_t kSlotBytes = size_t(32) << 20;

// A set of pinned slots for both directions, reused across calls on the same
// device (the slot events belong to the device current at creation; the
// portable pinned memory itself would serve any device).
struct SlotSet {
    char* mem[2][kSlots] = {};
    cudaEvent_t ev[2][kSlots] = {};
    int device = -1;
    bool ok = false;
    explicit SlotSet(int dev) : device(dev) {
        ok = true;
        for (int d = 0; d < 2 && ok; ++d)
            for (int s = 0; s < kSlots && ok; ++s)
                ok = cudaHostAlloc(reinterpret_cast<void**>(&mem[d][s]), kSlotBytes,
                                   cudaHostAllocPortable) == cudaSuccess &&
                     cudaEventCreateWithFlags(&ev[d][s], cudaEventDisableTiming) == cudaSuccess;
    }
};

std::mutex g_slot_mu;
std::vector<std::unique_ptr<SlotSet>> g_free_slots;

// a cached set of device `dev` (the current device of the calling thread)
std::unique_ptr<SlotSet> acquire_slots(int dev) {
    {
        std::lock_guard<std::mutex> lk(g_slot_mu);
        for (size_t i = g_free_slots.size(); i-- > 0;)
            if (g_free_slots[i]->device == dev) {
                auto s = std::move(g_free_slots[i]);
                g_free_slots.erase(g_free_slots.begin() + (std::ptrdiff_t)i);
                return s;
            }
    }
    auto s = std::make_unique<SlotSet>(dev);
    return s->ok ? std::move(s) : nullptr;
}

void release_slots(std::unique_ptr<SlotSet> s) {
    if (!s) return;
    std::lock_guard<std::mutex> lk(g_slot_mu);
    g_free_slots.push_back(std::move(s));
}

// Copies of staged chunks use non-temporal (streaming) 16-byte stores: the
// destination (a pinned slot, or the caller's C buffer) is not read again by
// this thread, and plain stores would first read every destination line
// (read-for-ownership) -- a third more host-memory traffic on a path that is
// bound by it ($OZK_STAGING_NT=0: plain memcpy, for A/B runs).
bool staging_nt() {  // read per chunk (cheap next to a 2 MB copy): A/B in one process
    const char* v = std::getenv("OZK_STAGING_NT");
    return !(v && !std::strcmp(v, "0"));
}

void stream_copy(char* dst, const char* src, size_t n) {
    if (n < 4096 || !staging_nt()) {
        std::memcpy(dst, src, n);
        return;
    }
    const size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
    std::memcpy(dst, src, head);
    dst += head;
    src += head;
    n -= head;
    const size_t body = n & ~size_t(63);
    for (size_t i = 0; i < body; i += 64) {
        const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
        const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
        const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
    }
    std::memcpy(dst + body, src + body, n - body);
    _mm_sfence();  // the streamed lines are globally visible before the DMA / the caller
}

// A team of host threads for one parallel memcpy at a time (the caller is
// member 0).
class Team {
public:
    explicit Team(int n) : n_(n < 1 ? 1 : n) {
        for (int i = 1; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    ~Team() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            quit_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    // rows x width bytes from src (pitch spitch) to dst (pitch dpitch)
    void copy2d(char* dst, size_t dpitch, const char* src, size_t spitch, size_t width,
                size_t rows) {
        auto part = [=](int i) {
            if (rows == 1) {  // one long row: split the bytes
                const size_t b0 = width * i / n_, b1 = width * (i + 1) / n_;
                stream_copy(dst + b0, src + b0, b1 - b0);
                return;
            }
            const size_t r0 = rows * i / n_, r1 = rows * (i + 1) / n_;
            for (size_t r = r0; r < r1; ++r) stream_copy(dst + r * dpitch, src + r * spitch, width);
        };
        if (n_ == 1) {
            part(0);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            task_ = part;
            pending_ = n_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        part(0);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return pending_ == 0; });
    }

private:
    void loop(int i) {
        uint64_t seen = 0;
        for (;;) {
            std::function<void(int)> f;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return quit_ || gen_ != seen; });
                if (quit_) return;
                seen = gen_;
                f = task_;
            }
            f(i);
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    std::function<void(int)> task_;
    uint64_t gen_ = 0;
    int pending_ = 0;
    bool quit_ = false;

public:
    int size() const { return n_; }
};

// Copy teams are cached process-wide like the slot sets: starting ~24 host
// threads per call cost ~1 ms, which small and mid-size calls felt.
std::mutex g_team_mu;
std::vector<std::unique_ptr<Team>> g_free_teams;

std::unique_ptr<Team> acquire_team(int n) {
    {
        std::lock_guard<std::mutex> lk(g_team_mu);
        for (size_t i = g_free_teams.size(); i-- > 0;)
            if (g_free_teams[i]->size() == (n < 1 ? 1 : n)) {
                auto t = std::move(g_free_teams[i]);
                g_free_teams.erase(g_free_teams.begin() + (std::ptrdiff_t)i);
                return t;
            }
    }
    return std::make_unique<Team>(n);
}

void release_team(std::unique_ptr<Team> t) {
    if (!t) return;
    std::lock_guard<std::mutex> lk(g_team_mu);
    g_free_teams.push_back(std::move(t));
}

}  // namespace

struct HostStaging::Impl {
    int device;  // the caller's current device: the copy streams' device
    cudaStream_t h2d_stream, d2h_stream;
    std::unique_ptr<SlotSet> slots;
    std::unique_ptr<Team> h2d_team, d2h_team;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<StagedCopy> queue[2];
    int recorded = 0;  // H2D jobs whose ready event has been recorded
    bool closing = false;
    std::atomic<cudaError_t> err{cudaSuccess};  // first error; read by the workers' loops
    std::thread worker[2];
    int slot_next[2] = {0, 0};
    bool slot_used[2][kSlots] = {};

    static int current_device() {
        int d = 0;
        if (cudaGetDevice(&d) != cudaSuccess) {
            (void)cudaGetLastError();
            d = 0;
        }
        return d;
    }

    Impl(cudaStream_t h2d, cudaStream_t d2h, int h2d_threads, int d2h_threads)
        : device(current_device()), h2d_stream(h2d), d2h_stream(d2h),
          slots(acquire_slots(device)), h2d_team(acquire_team(h2d_threads)),
          d2h_team(acquire_team(d2h_threads)) {
        if (!slots) err = cudaErrorMemoryAllocation;
        for (int d = 0; d < 2; ++d) worker[d] = std::thread([this, d] { run(d); });
    }

    void fail(cudaError_t e) {
        std::lock_guard<std::mutex> lk(mu);
        cudaError_t ok = cudaSuccess;
        err.compare_exchange_strong(ok, e);
        cv.notify_all();
    }

    // next slot of direction d, once its previous DMA has finished
    int take_slot(int d) {
        const int s = slot_next[d];
        slot_next[d] = (s + 1) % kSlots;
        if (slot_used[d][s]) {
            const cudaError_t e = cudaEventSynchronize(slots->ev[d][s]);
            if (e != cudaSuccess) fail(e);
        }
        slot_used[d][s] = true;
        return s;
    }

    void h2d(const StagedCopy& j) {
        // rows per slot (a row longer than a slot is sent in byte chunks)
        const size_t rows_per = j.width >= kSlotBytes || j.width == 0 ? 1 : kSlotBytes / j.width;
        for (size_t r0 = 0; j.width && r0 < j.height && err == cudaSuccess; r0 += rows_per) {
            const size_t rows = j.height - r0 < rows_per ? j.height - r0 : rows_per;
            for (size_t b0 = 0; b0 < j.width && err == cudaSuccess; b0 += kSlotBytes) {
                const size_t w = j.width - b0 < kSlotBytes ? j.width - b0 : kSlotBytes;
                const int s = take_slot(0);
                char* slot = slots->mem[0][s];
                const char* src = static_cast<const char*>(j.host) + r0 * j.host_pitch + b0;
                h2d_team->copy2d(slot, w, src, j.host_pitch, w, rows);
                char* dst = static_cast<char*>(j.dev) + r0 * j.dev_pitch + b0;
                cudaError_t e = rows == 1
                    ? cudaMemcpyAsync(dst, slot, w, cudaMemcpyHostToDevice, h2d_stream)
                    : cudaMemcpy2DAsync(dst, j.dev_pitch, slot, w, w, rows,
                                        cudaMemcpyHostToDevice, h2d_stream);
                if (e == cudaSuccess) e = cudaEventRecord(slots->ev[0][s], h2d_stream);
                if (e != cudaSuccess) fail(e);
            }
        }
        if (j.event && err == cudaSuccess) {
            const cudaError_t e = cudaEventRecord(j.event, h2d_stream);
            if (e != cudaSuccess) fail(e);
        }
        std::lock_guard<std::mutex> lk(mu);
        ++recorded;
        cv.notify_all();
    }

    void d2h(const StagedCopy& j) {
        if (j.event) {
            const cudaError_t e = cudaStreamWaitEvent(d2h_stream, j.event, 0);
            if (e != cudaSuccess) return fail(e);
        }
        // contiguous rows: byte chunks of one slot each, copied out as they land
        const size_t total = j.width * j.height;
        struct Pending {
            int slot;
            size_t off, bytes;
        };
        std::deque<Pending> inflight;
        auto drain_one = [&] {
            const Pending p = inflight.front();
            inflight.pop_front();
            const cudaError_t e = cudaEventSynchronize(slots->ev[1][p.slot]);
            if (e != cudaSuccess) return fail(e);
            d2h_team->copy2d(static_cast<char*>(j.host) + p.off, p.bytes, slots->mem[1][p.slot],
                            p.bytes, p.bytes, 1);
            slot_used[1][p.slot] = false;
        };
        for (size_t off = 0; off < total && err == cudaSuccess; off += kSlotBytes) {
            const size_t bytes = total - off < kSlotBytes ? total - off : kSlotBytes;
            if ((int)inflight.size() == kSlots) drain_one();
            const int s = take_slot(1);
            cudaError_t e = cudaMemcpyAsync(slots->mem[1][s], static_cast<const char*>(j.dev) + off,
                                            bytes, cudaMemcpyDeviceToHost, d2h_stream);
            if (e == cudaSuccess) e = cudaEventRecord(slots->ev[1][s], d2h_stream);
            if (e != cudaSuccess) return fail(e);
            inflight.push_back({s, off, bytes});
        }
        while (!inflight.empty() && err == cudaSuccess) drain_one();
    }

    void run(int d) {
        // a new thread starts on device 0: make the slot events' and copy
        // streams' device current (ozk_ozaki_gemm called on another device)
        if (const cudaError_t e = cudaSetDevice(device); e != cudaSuccess) fail(e);
        for (;;) {
            StagedCopy j;
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return closing || !queue[d].empty(); });
                if (queue[d].empty()) return;
                j = queue[d].front();
                queue[d].pop_front();
            }
            if (err != cudaSuccess) {
                if (d == 0) {
                    std::lock_guard<std::mutex> lk(mu);
                    ++recorded;
                    cv.notify_all();
                }
                continue;
            }
            if (d == 0)
                h2d(j);
            else
                d2h(j);
        }
    }
};

HostStaging::HostStaging(cudaStream_t h2d, cudaStream_t d2h, int h2d_threads, int d2h_threads)
    : impl_(new Impl(h2d, d2h, h2d_threads, d2h_threads)) {}

HostStaging::~HostStaging() {
    finish();
    release_slots(std::move(impl_->slots));
    release_team(std::move(impl_->h2d_team));
    release_team(std::move(impl_->d2h_team));
    delete impl_;
}

int HostStaging::push_h2d(const StagedCopy& c) {
    std::lock_guard<std::mutex> lk(impl_->mu);
    impl_->queue[0].push_back(c);
    impl_->cv.notify_all();
    return ++pushed_h2d_;
}

void HostStaging::push_d2h(const StagedCopy& c) {
    std::lock_guard<std::mutex> lk(impl_->mu);
    impl_->queue[1].push_back(c);
    impl_->cv.notify_all();
}

cudaError_t HostStaging::wait_recorded(int job) {
    std::unique_lock<std::mutex> lk(impl_->mu);
    impl_->cv.wait(lk, [&] { return impl_->recorded >= job || impl_->err != cudaSuccess; });
    return impl_->err.load();
}

cudaError_t HostStaging::finish() {
    if (impl_->worker[0].joinable()) {
        {
            std::lock_guard<std::mutex> lk(impl_->mu);
            impl_->closing = true;
        }
        impl_->cv.notify_all();
        for (auto& w : impl_->worker) w.join();
    }
    return impl_->err.load();
}

}  // namespace ozk

// Host <-> device staging for pageable user buffers.
//
// The reference's runtime moves host tensors to its offload device with plain
// copies (reference runtime.cpp:314-462, OffloadDevice::upload). Here the
// device sits behind PCIe, and a pageable cudaMemcpy goes through the
// driver's small bounce buffer at a fraction of link rate. Large uploads
// instead use a per-context ring of pinned chunks:
//   * a small persistent thread pool copies chunk i from the user buffer into
//     pinned memory, split across threads;
//   * the DMA of chunk i overlaps the fill of chunk i+1;
//   * a chunk is refilled only after its event shows the previous DMA
//     finished.
// The call returns once every byte has been read from the source, matching
// the synchronous-source contract of nncb_h2d.
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "nncb_internal.cuh"

namespace {

// Fixed-size fork/join pool: run(f, n) calls f(0..n-1) across the workers
// and the caller, returning when all are done.
class CopyPool {
public:
    static CopyPool& get() {
        static CopyPool pool;
        return pool;
    }
    int width() const { return static_cast<int>(workers_.size()) + 1; }

    void run(const std::function<void(int)>& f, int n) {
        if (n <= 1 || workers_.empty()) {
            for (int i = 0; i < n; ++i) f(i);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(m_);
            job_ = &f;
            njobs_ = n;
            next_ = 0;
            done_ = 0;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lk(m_);
        done_cv_.wait(lk, [&] { return done_ == njobs_; });
        job_ = nullptr;
    }

private:
    CopyPool() {
        unsigned hw = std::thread::hardware_concurrency();
        int n = static_cast<int>(std::min(8u, hw > 2 ? hw / 2 : 1u)) - 1;
        if (const char* e = getenv("NNCB_COPY_THREADS")) n = std::max(0, atoi(e) - 1);
        for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    // claim and run job indices until none are left
    void work() {
        for (;;) {
            int i;
            const std::function<void(int)>* f;
            {
                std::lock_guard<std::mutex> lk(m_);
                if (!job_ || next_ >= njobs_) return;
                i = next_++;
                f = job_;
            }
            (*f)(i);
            std::lock_guard<std::mutex> lk(m_);
            if (++done_ == njobs_) done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }

    std::vector<std::thread> workers_;
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* job_ = nullptr;
    int njobs_ = 0, next_ = 0, done_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

constexpr size_t kChunk = 16u << 20;   // pinned chunk
constexpr int kRing = 3;
constexpr size_t kStagedMin = 2u << 20;  // below this the driver path is as good

struct Staging {
    void* pin[kRing] = {};
    cudaEvent_t ev[kRing] = {};
    bool ok = false;
};

void parallel_copy(void* dst, const void* src, size_t bytes) {
    CopyPool& pool = CopyPool::get();
    const size_t min_part = 1u << 20;
    int parts = static_cast<int>(std::min<size_t>(pool.width(), (bytes + min_part - 1) / min_part));
    if (parts <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const size_t per = ((bytes + parts - 1) / parts + 63) & ~size_t(63);
    pool.run(
        [&](int i) {
            const size_t off = per * i;
            if (off < bytes) std::memcpy(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off,
                                         std::min(per, bytes - off));
        },
        parts);
}

}  // namespace

namespace nncb {

Staging* staging_for(nncb_ctx* c) {
    if (!c->staging) {
        auto* s = new Staging;
        s->ok = true;
        for (int i = 0; i < kRing && s->ok; ++i) {
            s->ok = cudaHostAlloc(&s->pin[i], kChunk, cudaHostAllocDefault) == cudaSuccess &&
                    cudaEventCreateWithFlags(&s->ev[i], cudaEventDisableTiming) == cudaSuccess;
        }
        if (!s->ok) cudaGetLastError();
        c->staging = s;
    }
    return static_cast<Staging*>(c->staging);
}

void staging_release(nncb_ctx* c) {
    auto* s = static_cast<Staging*>(c->staging);
    if (!s) return;
    for (int i = 0; i < kRing; ++i) {
        if (s->ev[i]) {
            cudaEventSynchronize(s->ev[i]);
            cudaEventDestroy(s->ev[i]);
        }
        if (s->pin[i]) cudaFreeHost(s->pin[i]);
    }
    delete s;
    c->staging = nullptr;
}

// Pageable upload through the pinned ring on `stream`: the copy threads fill
// chunk i while the DMA of chunk i-1 (and i-2) runs.
int h2d_staged(nncb_ctx* c, void* dst, const void* src, size_t bytes, cudaStream_t stream, bool allow_ring) {
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, src) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    Staging* s = (allow_ring && bytes >= kStagedMin && !pinned) ? staging_for(c) : nullptr;
    if (!s || !s->ok) {
        NNCB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream));
        if (!pinned) NNCB_CUDA(cudaStreamSynchronize(stream));   // pageable: src is reusable on return
        return 0;
    }
    int slot = 0;
    for (size_t off = 0; off < bytes; off += kChunk, slot = (slot + 1) % kRing) {
        const size_t n = std::min(kChunk, bytes - off);
        NNCB_CUDA(cudaEventSynchronize(s->ev[slot]));   // previous DMA out of this chunk has drained
        parallel_copy(s->pin[slot], static_cast<const char*>(src) + off, n);
        NNCB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, s->pin[slot], n, cudaMemcpyHostToDevice, stream));
        NNCB_CUDA(cudaEventRecord(s->ev[slot], stream));
    }
    return 0;
}

}  // namespace nncb

extern "C" {

int nncb_h2d_async(nncb_ctx* c, void* dst, const void* src, size_t bytes) {
    if (!bytes) return 0;
    return nncb::h2d_staged(c, dst, src, bytes, c->copy_stream, true);
}

int nncb_d2h_async(nncb_ctx* c, void* dst, const void* src, size_t bytes) {
    if (!bytes) return 0;
    NNCB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    return 0;
}

int nncb_h2d(nncb_ctx* c, void* dst, const void* src, size_t bytes) {
    if (!bytes) return 0;
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, src) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(c->stream, &cap);
    Staging* s = (bytes >= kStagedMin && !pinned && cap == cudaStreamCaptureStatusNone) ? nncb::staging_for(c) : nullptr;
    if (!s || !s->ok) {
        NNCB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
        return 0;
    }
    int slot = 0;
    for (size_t off = 0; off < bytes; off += kChunk, slot = (slot + 1) % kRing) {
        const size_t n = std::min(kChunk, bytes - off);
        NNCB_CUDA(cudaEventSynchronize(s->ev[slot]));   // previous DMA out of this chunk has drained
        parallel_copy(s->pin[slot], static_cast<const char*>(src) + off, n);
        NNCB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, s->pin[slot], n, cudaMemcpyHostToDevice, c->stream));
        NNCB_CUDA(cudaEventRecord(s->ev[slot], c->stream));
    }
    return 0;
}

// Large downloads into pageable memory: DMA chunk i+1 (and i+2) into the pinned
// ring while the copy threads move chunk i out; returns once dst is filled.
int nncb_d2h(nncb_ctx* c, void* dst, const void* src, size_t bytes) {
    if (!bytes) return 0;
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, dst) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    cudaGetLastError();
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(c->stream, &cap);
    Staging* s = (bytes >= kStagedMin && !pinned && cap == cudaStreamCaptureStatusNone) ? nncb::staging_for(c) : nullptr;
    if (!s || !s->ok) {
        NNCB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
        return 0;
    }
    const size_t nchunks = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t i) -> int {
        const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
        const int slot = static_cast<int>(i % kRing);
        NNCB_CUDA(cudaEventSynchronize(s->ev[slot]));   // the slot's previous user is done
        NNCB_CUDA(cudaMemcpyAsync(s->pin[slot], static_cast<const char*>(src) + off, n, cudaMemcpyDeviceToHost,
                                  c->stream));
        NNCB_CUDA(cudaEventRecord(s->ev[slot], c->stream));
        return 0;
    };
    for (size_t i = 0; i < std::min<size_t>(kRing, nchunks); ++i)
        if (int rc = issue(i)) return rc;
    for (size_t i = 0; i < nchunks; ++i) {
        const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
        const int slot = static_cast<int>(i % kRing);
        NNCB_CUDA(cudaEventSynchronize(s->ev[slot]));
        parallel_copy(static_cast<char*>(dst) + off, s->pin[slot], n);
        if (i + kRing < nchunks)
            if (int rc = issue(i + kRing)) return rc;
    }
    return 0;
}

int nncb_host_copy(void* dst, const void* src, size_t bytes) {
    if (bytes) parallel_copy(dst, src, bytes);
    return 0;
}

}  // extern "C"

// hostio.cu -- upload of the reference's int64 index arrays (in_sources,
// out_targets) as the device's int32 column indices.
//
// The int64 host array has the same values as the int32 one the engines
// keep, so half of every element is zero bytes over PCIe.  The upload is a
// two-lane pipeline:
//   * host lane: each thread of a host pool narrows its own chunks of the
//     head of the array into its page-locked int32 staging slots and queues
//     their copies on copy stream 0 (4 bytes/element over PCIe), double
//     buffered per thread;
//   * copy lane: the tail goes over PCIe as raw int64 on copy stream 1 (no
//     host work) into a device staging buffer and is narrowed by k_narrow.
// Both lanes run at once and meet in the middle: the host threads claim
// chunks from the head of the array, the copy lane claims pieces from its
// tail, until the claims meet.  With host narrowing rate c (GB/s of int64
// input) and PCIe rate b (~55 GB/s) the best share of the host lane is
// f = 2c / (2b + c): its int32 copies use c/2 of the link and the raw lane the
// rest.  c differs from host to host (16 threads with AVX2 streaming stores:
// 30-90 GB/s on the B200 boxes seen), so it is measured while the upload
// runs -- the time each thread spends inside the narrowing loop -- and the
// copy lane only claims a piece while its share stays below 1 - f; whatever
// the estimate, the array is consumed from both ends, so a wrong guess costs
// a late piece, not a stalled lane.  PUSHRANK_UPLOAD_HOSTFRAC pins a static
// split (tests, A/B).  Fast host (c ~ 90): f ~ 0.9, the C5 upload (1.06 G
// in-sources + both offset arrays, 9.56 GB as int64) takes ~121 ms instead of
// 175 ms for the plain copy.  Pageable host memory takes the host lane only
// (a pageable cudaMemcpy stages through the driver anyway).  The values are
// identical to the single-copy path (tests/test_gpu_upload.py).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <immintrin.h>

#include "internal.cuh"

namespace pr {

__global__ void k_narrow(const int64_t *__restrict__ in, int64_t count, int32_t *__restrict__ out);
static unsigned narrow_grid(const Ctx &ctx, int64_t items) {
    int64_t b = (items + 255) / 256, cap = (int64_t)ctx.sm_count * 16;
    return (unsigned)(b > cap ? cap : b < 1 ? 1 : b);
}

// Fixed pool of host threads: run(f) calls f(k, T) for k = 0..T-1 (the
// caller is k = 0) and returns when every call has returned.
class HostPool {
  public:
    explicit HostPool(int n) : n_(n < 1 ? 1 : n) {
        for (int k = 1; k < n_; ++k) th_.emplace_back([this, k] { loop(k); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> l(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto &t : th_) t.join();
    }
    int size() const { return n_; }
    void run(const std::function<void(int, int)> &f) {
        {
            std::lock_guard<std::mutex> l(mu_);
            job_ = &f;
            left_ = n_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        f(0, n_);
        std::unique_lock<std::mutex> l(mu_);
        done_.wait(l, [&] { return left_ == 0; });
        job_ = nullptr;
    }

  private:
    void loop(int k) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int, int)> *f;
            {
                std::unique_lock<std::mutex> l(mu_);
                cv_.wait(l, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                f = job_;
            }
            (*f)(k, n_);
            {
                std::lock_guard<std::mutex> l(mu_);
                if (--left_ == 0) done_.notify_one();
            }
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    const std::function<void(int, int)> *job_ = nullptr;
    uint64_t gen_ = 0;
    int left_ = 0;
    bool stop_ = false;
};

static int64_t env_i64(const char *name, int64_t dflt) {
    const char *e = getenv(name);
    return e && *e ? atoll(e) : dflt;
}

// Per-context state of the host lane, created on the first large upload:
// every pool thread owns SLOTS page-locked int32 staging slots and runs its
// own narrow -> copy pipeline over the chunks k = t, t + T, ...
struct Uploader {
    static constexpr int SLOTS = 2;
    HostPool pool;
    int64_t chunk;
    std::vector<int32_t *> slot;
    std::vector<cudaEvent_t> ev;
    std::vector<char> used;
    cudaStream_t cs[2] = {};
    explicit Uploader(int threads, int64_t chunk_elems) : pool(threads), chunk(chunk_elems) {}
    ~Uploader() {
        for (int k = 0; k < 2; ++k)
            if (cs[k]) {
                cudaStreamSynchronize(cs[k]);
                cudaStreamDestroy(cs[k]);
            }
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        for (auto p : slot)
            if (p) cudaFreeHost(p);
    }
};

void uploader_destroy(Ctx &ctx) {
    delete ctx.up;
    ctx.up = nullptr;
}

static int uploader(Ctx &ctx, Uploader **out) {
    if (!ctx.up) {
        unsigned hw = std::thread::hardware_concurrency();
        int threads = (int)env_i64("PUSHRANK_UPLOAD_THREADS", std::min<unsigned>(hw ? hw : 1, 16));
        int64_t chunk = env_i64("PUSHRANK_UPLOAD_CHUNK", 1ll << 20);
        if (chunk < 1024) chunk = 1024;
        chunk = (chunk + 7) / 8 * 8;
        auto *u = new Uploader(threads, chunk);
        const int ns = Uploader::SLOTS * u->pool.size();
        u->slot.assign(ns, nullptr);
        u->ev.assign(ns, nullptr);
        u->used.assign(ns, 0);
        for (int k = 0; k < ns; ++k) {
            if (cudaHostAlloc((void **)&u->slot[k], 4 * (size_t)chunk, cudaHostAllocDefault) != cudaSuccess ||
                cudaEventCreateWithFlags(&u->ev[k], cudaEventDisableTiming) != cudaSuccess) {
                delete u;
                return fail(PR_ERR_CUDA, "upload: page-locked staging allocation failed");
            }
        }
        for (int k = 0; k < 2; ++k)
            if (cudaStreamCreateWithFlags(&u->cs[k], cudaStreamNonBlocking) != cudaSuccess) {
                delete u;
                return fail(PR_ERR_CUDA, "upload: copy stream creation failed");
            }
        ctx.up = u;
    }
    *out = ctx.up;
    return PR_OK;
}

// int64 -> int32 of len values; dst 32-byte aligned.  Streaming stores: the
// staging slot is written once and read by the copy engine, so the cache
// lines need no read-for-ownership.
__attribute__((target("avx2"))) static void narrow_avx2(const int64_t *src, int32_t *dst, int64_t len) {
    const __m256i even = _mm256_setr_epi32(0, 2, 4, 6, 1, 3, 5, 7);
    int64_t i = 0;
    for (; i + 8 <= len; i += 8) {
        __m256i a = _mm256_permutevar8x32_epi32(_mm256_loadu_si256((const __m256i *)(src + i)), even);
        __m256i b = _mm256_permutevar8x32_epi32(_mm256_loadu_si256((const __m256i *)(src + i + 4)), even);
        _mm256_stream_si256((__m256i *)(dst + i), _mm256_permute2x128_si256(a, b, 0x20));
    }
    for (; i < len; ++i) dst[i] = (int32_t)src[i];
    _mm_sfence();
}

static void narrow_host(const int64_t *src, int32_t *dst, int64_t len) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    if (avx2 && ((uintptr_t)dst & 31) == 0) {
        narrow_avx2(src, dst, len);
        return;
    }
    for (int64_t i = 0; i < len; ++i) dst[i] = (int32_t)src[i];
}

static bool page_locked(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// count int64 values at h -> int32 at d (device, allocated on ctx.stream).
// Ordered after earlier work on ctx.stream; later work on ctx.stream waits
// for it.  *h2d (if given) += the bytes copied over PCIe.
int upload_narrow(Ctx &ctx, const int64_t *h, int64_t count, int32_t *d, int64_t *h2d, const RawCopy *extra,
                  int n_extra) {
    cudaStream_t st = ctx.stream;
    if (count <= 0) {
        for (int k = 0; k < n_extra; ++k)
            PR_CUDA(cudaMemcpyAsync(extra[k].dst, extra[k].src, extra[k].bytes, cudaMemcpyHostToDevice, st));
        return PR_OK;
    }
    const int64_t min_elems = env_i64("PUSHRANK_UPLOAD_MIN", 1ll << 22);
    if (count < min_elems || env_i64("PUSHRANK_UPLOAD_THREADS", 2) < 1) {
        // small arrays: one copy of the int64 values, narrowed on the device
        for (int k = 0; k < n_extra; ++k)
            PR_CUDA(cudaMemcpyAsync(extra[k].dst, extra[k].src, extra[k].bytes, cudaMemcpyHostToDevice, st));
        DevBuf stage;
        PR_TRY(ensure(stage, 8 * count));
        PR_CUDA(cudaMemcpyAsync(stage.ptr, h, 8 * count, cudaMemcpyHostToDevice, st));
        k_narrow<<<narrow_grid(ctx, count), 256, 0, st>>>(stage.as<int64_t>(), count, d);
        PR_CUDA(cudaGetLastError());
        if (h2d) *h2d += 8 * count;
        return PR_OK;
    }
    Uploader *u = nullptr;
    PR_TRY(uploader(ctx, &u));
    const int T = u->pool.size();
    const int64_t CH = u->chunk;
    const int64_t n_chunks = (count + CH - 1) / CH;
    const bool pinned = page_locked(h);
    // static split (tests, A/B): the first `fixed` chunks take the host lane
    int64_t fixed = -1;
    if (const char *e = getenv("PUSHRANK_UPLOAD_HOSTFRAC")) {
        const double f = std::min(1.0, std::max(0.0, atof(e)));
        fixed = f >= 1.0 ? n_chunks : (int64_t)(f * (double)count) / CH;
    } else if (!pinned || T < 2) {
        fixed = n_chunks;   // host lane only
    }
    // copy lane pieces: RAW chunks each, two device staging slots in rotation
    const int64_t RAW = std::max<int64_t>(1, env_i64("PUSHRANK_UPLOAD_RAW_CHUNKS", 8));
    const double b = 55.0;                                   // PCIe, GB/s
    double c0 = std::min(11.0 * T, 90.0);                    // first guess of the narrowing rate
    if (const char *e = getenv("PUSHRANK_UPLOAD_RATE"))
        if (atof(e) > 0) c0 = atof(e);
    const bool raw_lane = fixed < n_chunks;
    // both copy streams start after the allocations queued on ctx.stream
    cudaEvent_t ev_start, ev_done[2], ev_raw[2];
    PR_CUDA(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
    PR_CUDA(cudaEventCreateWithFlags(&ev_done[0], cudaEventDisableTiming));
    PR_CUDA(cudaEventCreateWithFlags(&ev_done[1], cudaEventDisableTiming));
    PR_CUDA(cudaEventCreateWithFlags(&ev_raw[0], cudaEventDisableTiming));
    PR_CUDA(cudaEventCreateWithFlags(&ev_raw[1], cudaEventDisableTiming));
    DevBuf stage;
    int rc = PR_OK;
    const int64_t piece = RAW * CH;
    if (raw_lane) rc = ensure(stage, 2 * 8 * (size_t)piece);
    int64_t host_elems = 0, raw_elems = 0;
    if (rc == PR_OK) {
        cudaError_t e = cudaEventRecord(ev_start, st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(u->cs[0], ev_start, 0);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(u->cs[1], ev_start, 0);
        // copy lane first: the caller's extra raw copies
        for (int k = 0; e == cudaSuccess && k < n_extra; ++k)
            e = cudaMemcpyAsync(extra[k].dst, extra[k].src, extra[k].bytes, cudaMemcpyHostToDevice, u->cs[1]);
        if (e == cudaSuccess) {
            // claims: chunks [0, head) belong to the host lane, [tail, n_chunks) to the copy lane
            std::mutex mu;
            int64_t head = 0, tail = n_chunks;
            std::atomic<int> err{0};
            std::atomic<int64_t> narrowed{0}, narrow_ns{0};
            using clk = std::chrono::steady_clock;
            // one chunk of the host lane on thread t (its j-th); false when none is left
            auto host_one = [&](int t, int j) -> bool {
                int64_t k;
                {
                    std::lock_guard<std::mutex> l(mu);
                    if (head >= (fixed >= 0 ? fixed : tail)) return false;
                    k = head++;
                }
                const int s = Uploader::SLOTS * t + (j % Uploader::SLOTS);
                cudaError_t x = cudaSuccess;
                if (u->used[s]) x = cudaEventSynchronize(u->ev[s]);
                const int64_t off = k * CH, len = std::min(CH, count - off);
                if (x == cudaSuccess) {
                    const auto t0 = clk::now();
                    narrow_host(h + off, u->slot[s], len);
                    narrow_ns.fetch_add(std::chrono::duration_cast<std::chrono::nanoseconds>(clk::now() - t0).count());
                    narrowed.fetch_add(len);
                    x = cudaMemcpyAsync(d + off, u->slot[s], 4 * len, cudaMemcpyHostToDevice, u->cs[0]);
                }
                if (x == cudaSuccess) x = cudaEventRecord(u->ev[s], u->cs[0]);
                u->used[s] = 1;
                if (x != cudaSuccess) err.store((int)x);
                return true;
            };
            auto host_lane = [&](int t, int j) {
                while (!err.load(std::memory_order_relaxed) && host_one(t, j)) ++j;
            };
            // thread 0: the copy lane; while that is ahead of its share, one host chunk at a time
            auto copy_lane = [&]() -> int {
                int64_t claimed = 0;   // chunks this lane has taken
                int hj = 0;            // host chunks thread 0 has narrowed
                for (int j = 0; !err.load(std::memory_order_relaxed);) {
                    int64_t k0 = 0, take = 0;
                    bool done = false;
                    {
                        std::lock_guard<std::mutex> l(mu);
                        const int64_t lo = fixed >= 0 ? std::max(fixed, head) : head;
                        if (lo >= tail) {
                            done = true;
                        } else {
                            take = std::min(RAW, tail - lo);
                            if (fixed < 0) {
                                // share of the host lane from its measured narrowing rate
                                const int64_t ns = narrow_ns.load(), el = narrowed.load();
                                const double c = el >= T * CH && ns > 0 ? 8.0 * (double)el / (double)ns * T : c0;
                                const double f = 2.0 * c / (2.0 * b + c);
                                if ((double)(claimed + take) > (1.0 - f) * (double)n_chunks + 0.5)
                                    take = 0;   // ahead of its share: leave the rest to the host threads for now
                            }
                            if (take > 0) {
                                tail -= take;
                                k0 = tail;
                            }
                        }
                    }
                    if (done) break;
                    if (take == 0) {
                        if (host_one(0, hj)) ++hj;
                        continue;
                    }
                    cudaError_t x = cudaSuccess;
                    if (j >= 2) x = cudaEventSynchronize(ev_raw[j & 1]);   // its staging slot is free again
                    const int64_t off = k0 * CH, len = std::min(count, (k0 + take) * CH) - off;
                    int64_t *slot = stage.as<int64_t>() + (int64_t)(j & 1) * piece;
                    if (x == cudaSuccess) x = cudaMemcpyAsync(slot, h + off, 8 * len, cudaMemcpyHostToDevice, u->cs[1]);
                    if (x == cudaSuccess) {
                        k_narrow<<<narrow_grid(ctx, len), 256, 0, u->cs[1]>>>(slot, len, d + off);
                        x = cudaGetLastError();
                    }
                    if (x == cudaSuccess) x = cudaEventRecord(ev_raw[j & 1], u->cs[1]);
                    if (x != cudaSuccess) err.store((int)x);
                    raw_elems += len;
                    claimed += take;
                    ++j;
                }
                return hj;
            };
            const auto t_begin = clk::now();
            u->pool.run([&](int t, int) {
                // thread 0 drives the copy lane when there is one, then helps narrowing
                host_lane(t, t == 0 && raw_lane ? copy_lane() : 0);
            });
            host_elems = narrowed.load();
            if (err.load()) e = (cudaError_t)err.load();
            if (getenv("PUSHRANK_TIMING")) {
                const double wall = std::chrono::duration<double>(clk::now() - t_begin).count();
                const double ns = (double)narrow_ns.load();
                fprintf(stderr, "[upload] %lld elements: host lane %.1f%% (%d threads, %.1f GB/s per thread of int64 in), "
                        "copy lane %.1f%%, queued in %.1f ms\n", (long long)count, 100.0 * host_elems / count, T,
                        ns > 0 ? 8.0 * host_elems / ns : 0.0, 100.0 * raw_elems / count, 1e3 * wall);
            }
        }
        if (e == cudaSuccess) e = cudaEventRecord(ev_done[0], u->cs[0]);
        if (e == cudaSuccess) e = cudaEventRecord(ev_done[1], u->cs[1]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev_done[0], 0);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev_done[1], 0);
        if (e != cudaSuccess) {
            // leave no copy running into buffers the caller may free
            cudaStreamSynchronize(u->cs[0]);
            cudaStreamSynchronize(u->cs[1]);
            rc = fail(PR_ERR_CUDA, std::string("upload: ") + cudaGetErrorString(e));
        }
    }
    // the staging slots' free is ordered after the copy lane's narrowing (ctx.stream waits on it)
    stage.release();
    cudaEventDestroy(ev_start);
    for (int k = 0; k < 2; ++k) {
        cudaEventDestroy(ev_done[k]);
        cudaEventDestroy(ev_raw[k]);
    }
    if (rc == PR_OK && h2d) *h2d += 4 * host_elems + 8 * raw_elems;
    return rc;
}

}  // namespace pr

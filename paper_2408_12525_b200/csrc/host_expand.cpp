// host_expand.cpp -- bit stream -> float32/uint8 observation expansion on the
// host cores (see host_expand.h). Non-temporal stores: the destination is
// write-once output many times larger than the caches.
#include "host_expand.h"

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <sched.h>
#include <vector>

namespace lg_host {
namespace {

struct Luts {
    alignas(64) float f8[256][8];  // byte -> 8 floats (bit k -> element k)
    alignas(64) float f4[16][4];   // nibble -> 4 floats
    uint64_t b8[256];              // byte -> 8 bytes of 0/1
    Luts() {
        for (int b = 0; b < 256; b++) {
            uint64_t u = 0;
            for (int k = 0; k < 8; k++) {
                f8[b][k] = ((b >> k) & 1) ? 1.0f : 0.0f;
                u |= (uint64_t)((b >> k) & 1) << (8 * k);
            }
            b8[b] = u;
        }
        for (int n = 0; n < 16; n++)
            for (int k = 0; k < 4; k++) f4[n][k] = ((n >> k) & 1) ? 1.0f : 0.0f;
    }
};
const Luts &luts() {
    static const Luts L;
    return L;
}

// bytes [b0, b1) of the stream -> elements [8*b0, 8*b1)
__attribute__((target("avx"))) void f32_avx(const uint8_t *bits, float *dst, size_t b0, size_t b1) {
    const Luts &L = luts();
    for (size_t i = b0; i < b1; i++) _mm256_stream_ps(dst + 8 * i, _mm256_load_ps(L.f8[bits[i]]));
}

void f32_sse(const uint8_t *bits, float *dst, size_t b0, size_t b1) {
    const Luts &L = luts();
    for (size_t i = b0; i < b1; i++) {
        const uint8_t b = bits[i];
        _mm_stream_ps(dst + 8 * i, _mm_load_ps(L.f4[b & 15]));
        _mm_stream_ps(dst + 8 * i + 4, _mm_load_ps(L.f4[b >> 4]));
    }
}

void f32_plain(const uint8_t *bits, float *dst, size_t b0, size_t b1) {
    const Luts &L = luts();
    for (size_t i = b0; i < b1; i++) std::memcpy(dst + 8 * i, L.f8[bits[i]], 32);
}

// b0 even (16-byte pairs)
void u8_sse(const uint8_t *bits, uint8_t *dst, size_t b0, size_t b1) {
    const Luts &L = luts();
    size_t i = b0;
    for (; i + 1 < b1; i += 2)
        _mm_stream_si128(reinterpret_cast<__m128i *>(dst + 8 * i),
                         _mm_set_epi64x((long long)L.b8[bits[i + 1]], (long long)L.b8[bits[i]]));
    for (; i < b1; i++) std::memcpy(dst + 8 * i, &L.b8[bits[i]], 8);
}

void u8_plain(const uint8_t *bits, uint8_t *dst, size_t b0, size_t b1) {
    const Luts &L = luts();
    for (size_t i = b0; i < b1; i++) std::memcpy(dst + 8 * i, &L.b8[bits[i]], 8);
}

class Pool {
  public:
    explicit Pool(int n) : n_(n) {
        for (int i = 1; i < n_; i++) th_.emplace_back([this, i] { loop(i); });
    }
    int size() const { return n_; }
    // run fn(i) for i in [0, n): i = 0 on the caller
    void run(const std::function<void(int)> &fn) {
        std::lock_guard<std::mutex> serial(call_);
        {
            std::lock_guard<std::mutex> g(m_);
            job_ = &fn;
            pending_ = n_ - 1;
            gen_++;
        }
        cv_.notify_all();
        fn(0);
        std::unique_lock<std::mutex> g(m_);
        done_.wait(g, [this] { return pending_ == 0; });
        job_ = nullptr;
    }

  private:
    void loop(int i) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int)> *job;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return gen_ != seen; });
                seen = gen_;
                job = job_;
            }
            (*job)(i);
            {
                std::lock_guard<std::mutex> g(m_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::mutex m_, call_;
    std::condition_variable cv_, done_;
    uint64_t gen_ = 0;
    int pending_ = 0;
    const std::function<void(int)> *job_ = nullptr;
};

Pool &pool() {
    // leaked on purpose: worker threads outlive static destruction at exit
    static Pool *p = [] {
        // one worker per core this process may run on (a multi-GPU launcher
        // gives each rank its own slice of the host's cores), LG_HOST_THREADS overrides
        int n = (int)std::thread::hardware_concurrency();
        cpu_set_t cs;
        CPU_ZERO(&cs);
        if (sched_getaffinity(0, sizeof cs, &cs) == 0 && CPU_COUNT(&cs) > 0) n = CPU_COUNT(&cs);
        if (const char *v = std::getenv("LG_HOST_THREADS")) n = std::atoi(v);
        if (n < 1) n = 1;
        if (n > 256) n = 256;
        return new Pool(n);
    }();
    return *p;
}

}  // namespace

int expand_threads() { return pool().size(); }

void expand_bits(const uint8_t *bits, void *dst, int fmt, size_t n_elems, size_t chunk_bytes,
                 bool (*ready)(void *ctx, size_t chunk), void *ctx) {
    const size_t full_bytes = n_elems / 8, tail = n_elems % 8;
    const size_t nbytes = full_bytes + (tail ? 1 : 0);
    if (chunk_bytes < 64) chunk_bytes = 64;
    chunk_bytes &= ~(size_t)63;
    const size_t nchunks = (nbytes + chunk_bytes - 1) / chunk_bytes;
    const uintptr_t a = reinterpret_cast<uintptr_t>(dst);
    // small outputs: waking the pool costs more than the expansion itself, and
    // the caller reads them right away, so plain (cached) stores on this thread
    const bool small = n_elems * (fmt == 0 ? 4 : 1) < ((size_t)4 << 20);
    const bool avx = !small && fmt == 0 && (a & 31) == 0 && __builtin_cpu_supports("avx");
    const bool sse = !small && (a & 15) == 0;
    std::atomic<size_t> ready_upto{0};
    std::mutex poll;
    const int T = small ? 1 : pool().size();
    auto work = [&](int j) {
        for (size_t c = 0; c < nchunks; c++) {
            while (ready_upto.load(std::memory_order_acquire) <= c) {
                if (poll.try_lock()) {
                    size_t k = ready_upto.load(std::memory_order_relaxed);
                    while (k < nchunks && (!ready || ready(ctx, k))) k++;
                    ready_upto.store(k, std::memory_order_release);
                    poll.unlock();
                    if (k > c) break;
                }
                std::this_thread::yield();
            }
            // thread j's slice of chunk c, in 64-byte units of the stream
            const size_t c0 = c * chunk_bytes, c1 = std::min(nbytes, c0 + chunk_bytes);
            const size_t units = (c1 - c0 + 63) / 64;
            const size_t u0 = units * j / T, u1 = units * (j + 1) / T;
            size_t b0 = c0 + u0 * 64, b1 = std::min(c1, c0 + u1 * 64);
            if (b0 >= b1) continue;
            const size_t bf = std::min(b1, full_bytes);  // whole bytes in this slice
            if (fmt == 0) {
                float *o = static_cast<float *>(dst);
                if (b0 < bf) {
                    if (avx) f32_avx(bits, o, b0, bf);
                    else if (sse) f32_sse(bits, o, b0, bf);
                    else f32_plain(bits, o, b0, bf);
                }
                if (b1 > full_bytes)  // trailing partial byte
                    for (size_t k = 0; k < tail; k++) o[8 * full_bytes + k] = ((bits[full_bytes] >> k) & 1) ? 1.0f : 0.0f;
            } else {
                uint8_t *o = static_cast<uint8_t *>(dst);
                if (b0 < bf) {
                    if (sse) u8_sse(bits, o, b0, bf);
                    else u8_plain(bits, o, b0, bf);
                }
                if (b1 > full_bytes)
                    for (size_t k = 0; k < tail; k++) o[8 * full_bytes + k] = (bits[full_bytes] >> k) & 1;
            }
        }
        _mm_sfence();
    };
    if (small) work(0);
    else pool().run(work);
}

}  // namespace lg_host

// host_simd.cpp -- see host_simd.hpp.  AVX-512 paths are selected at run
// time (__builtin_cpu_supports); the scalar loops are the reference
// semantics and the fallback.
#include "host_simd.hpp"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace nb200 {

namespace {

// Persistent host worker pool for the ABI's conversion loops (a C3 state()
// splits into ~13 pieces of 16 threads each: spawning threads per piece
// cost milliseconds).  Callers post one batch of chunk jobs and help run it;
// several callers (the main thread and a snapshot thread) may post at once.
class HostPool {
 public:
  static HostPool& get() {
    // never destroyed: a snapshot thread may still use it during exit
    static HostPool* pool = new HostPool;
    return *pool;
  }
  unsigned size() const { return static_cast<unsigned>(workers_.size()) + 1; }
  // Runs job(i) for i in [0, count); returns when all are done.  The
  // batch state is shared with the queued helpers, so a helper that starts
  // after the batch finished finds no work and touches nothing else.
  void run(unsigned count, std::function<void(unsigned)> job) {
    struct State {
      std::atomic<unsigned> next{0}, done{0};
      unsigned count = 0;
      std::function<void(unsigned)> job;
    };
    auto st = std::make_shared<State>();
    st->count = count;
    st->job = std::move(job);
    auto drain = [st] {
      for (unsigned i; (i = st->next.fetch_add(1)) < st->count;) {
        st->job(i);
        st->done.fetch_add(1);
      }
    };
    {
      std::lock_guard<std::mutex> lk(m_);
      for (unsigned w = 0; w + 1 < count && w < workers_.size(); ++w) tasks_.push_back(drain);
    }
    cv_.notify_all();
    drain();
    while (st->done.load() < count) std::this_thread::yield();
  }

 private:
  // Workers: NASCH_B200_HOST_THREADS, else the hardware threads shared by
  // the processes of this node (LOCAL_WORLD_SIZE, set by torchrun, so eight
  // ranks of one box do not each spin a thread per core), at most 64.
  HostPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const char* e = std::getenv("NASCH_B200_HOST_THREADS");
    const char* lw = std::getenv("LOCAL_WORLD_SIZE");
    const long local = lw && *lw ? std::max(1l, std::strtol(lw, nullptr, 10)) : 1l;
    const long want = e && *e ? std::strtol(e, nullptr, 10) : std::max(1l, long(hw) / local);
    const unsigned n = static_cast<unsigned>(std::max(1l, std::min(want, 64l)));
    for (unsigned t = 1; t < n; ++t) workers_.emplace_back([this] { loop(); });
  }
  void loop() {
    for (;;) {
      std::function<void()> t;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || !tasks_.empty(); });
        if (stop_ && tasks_.empty()) return;
        t = std::move(tasks_.front());
        tasks_.pop_front();
      }
      t();
    }
  }
  std::vector<std::thread> workers_;
  std::deque<std::function<void()>> tasks_;
  std::mutex m_;
  std::condition_variable cv_;
  bool stop_ = false;  // never set: the pool lives for the process
};


void widen_u32_scalar(const uint32_t* src, uint64_t* dst, size_t n) {
  for (size_t i = 0; i < n; ++i) dst[i] = src[i];
}
void widen_u8_scalar(const uint8_t* src, uint64_t* dst, size_t n) {
  for (size_t i = 0; i < n; ++i) dst[i] = src[i];
}

void widen_u8_u32_scalar(const uint8_t* src, uint32_t* dst, size_t n) {
  for (size_t i = 0; i < n; ++i) dst[i] = src[i];
}

#if defined(__x86_64__)
bool have_avx512() {
  static const bool ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");
  return ok;
}

__attribute__((target("avx512f,avx512bw"))) void widen_u32_avx512(const uint32_t* src, uint64_t* dst, size_t n) {
  size_t i = 0;
  // scalar head until dst is 64-byte aligned (streaming stores need it)
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 63u)) {
    dst[i] = src[i];
    ++i;
  }
  for (; i + 16 <= n; i += 16) {
    const __m512i s = _mm512_loadu_si512(reinterpret_cast<const void*>(src + i));
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i), _mm512_cvtepu32_epi64(_mm512_castsi512_si256(s)));
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i + 8),
                        _mm512_cvtepu32_epi64(_mm512_extracti64x4_epi64(s, 1)));
  }
  for (; i < n; ++i) dst[i] = src[i];
  _mm_sfence();
}

__attribute__((target("avx512f,avx512bw"))) void widen_u8_avx512(const uint8_t* src, uint64_t* dst, size_t n) {
  size_t i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 63u)) {
    dst[i] = src[i];
    ++i;
  }
  for (; i + 16 <= n; i += 16) {
    const __m128i s = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i), _mm512_cvtepu8_epi64(s));
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i + 8), _mm512_cvtepu8_epi64(_mm_srli_si128(s, 8)));
  }
  for (; i < n; ++i) dst[i] = src[i];
  _mm_sfence();
}

__attribute__((target("avx512f,avx512bw"))) void widen_u8_u32_avx512(const uint8_t* src, uint32_t* dst, size_t n) {
  size_t i = 0;
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 63u)) {
    dst[i] = src[i];
    ++i;
  }
  for (; i + 16 <= n; i += 16) {
    const __m128i s = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i), _mm512_cvtepu8_epi32(s));
  }
  for (; i < n; ++i) dst[i] = src[i];
  _mm_sfence();
}

// 8 cars at a time: narrow with vpmovqd / vpmovqb, rules as masks.
__attribute__((target("avx512f,avx512bw"))) int narrow_avx512(const uint64_t* x, const uint64_t* v, size_t lo,
                                                              size_t hi, uint64_t L, uint64_t vmax,
                                                              uint64_t vlim, uint32_t* x32, void* vout,
                                                              int vbytes) {
  const __m512i vL = _mm512_set1_epi64(static_cast<long long>(L));
  const __m512i vVmax = _mm512_set1_epi64(static_cast<long long>(vmax));
  const __m512i vVlim = _mm512_set1_epi64(static_cast<long long>(vlim));
  size_t i = lo;
  // the first car has no predecessor: scalar until x[i-1] exists
  for (; i < hi && i == 0; ++i) {
    const uint64_t xi = x[i], vi = v[i];
    if (xi >= L) return 1;
    if (vi > vmax) return 3;
    if (vi > vlim) return 4;
    x32[i] = static_cast<uint32_t>(xi);
    if (vbytes == 1) static_cast<uint8_t*>(vout)[i] = static_cast<uint8_t>(vi);
    else static_cast<uint32_t*>(vout)[i] = static_cast<uint32_t>(vi);
  }
  // scalar until i is a multiple of 8 (32-byte aligned non-temporal stores
  // into the page-aligned staging)
  for (; i < hi && (i & 7u); ++i) {
    const uint64_t xi = x[i], vi = v[i];
    if (xi >= L) return 1;
    if (x[i - 1] >= xi) return 2;
    if (vi > vmax) return 3;
    if (vi > vlim) return 4;
    x32[i] = static_cast<uint32_t>(xi);
    if (vbytes == 1) static_cast<uint8_t*>(vout)[i] = static_cast<uint8_t>(vi);
    else static_cast<uint32_t*>(vout)[i] = static_cast<uint32_t>(vi);
  }
  for (; i + 8 <= hi; i += 8) {
    const __m512i xs = _mm512_loadu_si512(reinterpret_cast<const void*>(x + i));
    const __m512i vs = _mm512_loadu_si512(reinterpret_cast<const void*>(v + i));
    const __m512i prevs = _mm512_loadu_si512(reinterpret_cast<const void*>(x + i - 1));  // i >= 1
    const __mmask8 bad_l = _mm512_cmpge_epu64_mask(xs, vL);
    const __mmask8 bad_inc = _mm512_cmple_epu64_mask(xs, prevs);
    const __mmask8 bad_vmax = _mm512_cmpgt_epu64_mask(vs, vVmax);
    const __mmask8 bad_vlim = _mm512_cmpgt_epu64_mask(vs, vVlim);
    if (bad_l | bad_inc | bad_vmax | bad_vlim) {
      // first offending car, first rule in the scalar order
      for (size_t k = i; k < i + 8; ++k) {
        if (x[k] >= L) return 1;
        if (k && x[k - 1] >= x[k]) return 2;
        if (v[k] > vmax) return 3;
        if (v[k] > vlim) return 4;
      }
    }
    _mm256_stream_si256(reinterpret_cast<__m256i*>(x32 + i), _mm512_cvtepi64_epi32(xs));
    if (vbytes == 1) {
      _mm_stream_si64(reinterpret_cast<long long*>(static_cast<uint8_t*>(vout) + i),
                      _mm_cvtsi128_si64(_mm512_cvtepi64_epi8(vs)));
    } else {
      _mm256_stream_si256(reinterpret_cast<__m256i*>(static_cast<uint32_t*>(vout) + i), _mm512_cvtepi64_epi32(vs));
    }
  }
  _mm_sfence();
  for (; i < hi; ++i) {
    const uint64_t xi = x[i], vi = v[i];
    if (xi >= L) return 1;
    if (i && x[i - 1] >= xi) return 2;
    if (vi > vmax) return 3;
    if (vi > vlim) return 4;
    x32[i] = static_cast<uint32_t>(xi);
    if (vbytes == 1) static_cast<uint8_t*>(vout)[i] = static_cast<uint8_t>(vi);
    else static_cast<uint32_t*>(vout)[i] = static_cast<uint32_t>(vi);
  }
  return 0;
}
#endif

}  // namespace

void widen_u32(const uint32_t* src, uint64_t* dst, size_t n) {
#if defined(__x86_64__)
  if (have_avx512() && n >= 64) return widen_u32_avx512(src, dst, n);
#endif
  widen_u32_scalar(src, dst, n);
}

void widen_u8_u32(const uint8_t* src, uint32_t* dst, size_t n) {
#if defined(__x86_64__)
  if (have_avx512() && n >= 64) return widen_u8_u32_avx512(src, dst, n);
#endif
  widen_u8_u32_scalar(src, dst, n);
}

void widen_u8(const uint8_t* src, uint64_t* dst, size_t n) {
#if defined(__x86_64__)
  if (have_avx512() && n >= 64) return widen_u8_avx512(src, dst, n);
#endif
  widen_u8_scalar(src, dst, n);
}

#if defined(__x86_64__)
// 16 cars at a time: u32 rules as masks, velocities narrowed with vpmovdb.
__attribute__((target("avx512f,avx512bw"))) int narrow32_avx512(const uint32_t* x, const uint32_t* v, size_t lo,
                                                                size_t hi, uint32_t L, uint32_t vmax, uint32_t vlim,
                                                                uint32_t* x32, void* vout, int vbytes) {
  const __m512i vL = _mm512_set1_epi32(static_cast<int>(L));
  const __m512i vVmax = _mm512_set1_epi32(static_cast<int>(vmax));
  const __m512i vVlim = _mm512_set1_epi32(static_cast<int>(vlim));
  size_t i = lo;
  auto scalar = [&](size_t k) -> int {
    if (x[k] >= L) return 1;
    if (k && x[k - 1] >= x[k]) return 2;
    if (v[k] > vmax) return 3;
    if (v[k] > vlim) return 4;
    if (x32) x32[k] = x[k];
    if (vbytes == 1) static_cast<uint8_t*>(vout)[k] = static_cast<uint8_t>(v[k]);
    else static_cast<uint32_t*>(vout)[k] = v[k];
    return 0;
  };
  // scalar until i > 0 and a multiple of 16 (aligned streaming stores)
  for (; i < hi && (i == 0 || (i & 15u)); ++i)
    if (const int e = scalar(i)) return e;
  for (; i + 16 <= hi; i += 16) {
    const __m512i xs = _mm512_loadu_si512(reinterpret_cast<const void*>(x + i));
    const __m512i vs = _mm512_loadu_si512(reinterpret_cast<const void*>(v + i));
    const __m512i prevs = _mm512_loadu_si512(reinterpret_cast<const void*>(x + i - 1));
    const __mmask16 bad = _mm512_cmpge_epu32_mask(xs, vL) | _mm512_cmple_epu32_mask(xs, prevs) |
                          _mm512_cmpgt_epu32_mask(vs, vVmax) | _mm512_cmpgt_epu32_mask(vs, vVlim);
    if (bad) {
      for (size_t k = i; k < i + 16; ++k)
        if (const int e = scalar(k)) return e;
    }
    if (x32) _mm512_stream_si512(reinterpret_cast<__m512i*>(x32 + i), xs);
    if (vbytes == 1) _mm_stream_si128(reinterpret_cast<__m128i*>(static_cast<uint8_t*>(vout) + i), _mm512_cvtepi32_epi8(vs));
    else _mm512_stream_si512(reinterpret_cast<__m512i*>(static_cast<uint32_t*>(vout) + i), vs);
  }
  _mm_sfence();
  for (; i < hi; ++i)
    if (const int e = scalar(i)) return e;
  return 0;
}
#endif

int narrow_validate32(const uint32_t* x, const uint32_t* v, size_t lo, size_t hi, uint64_t L, uint64_t vmax,
                      uint64_t vlim, uint32_t* x32, void* vout, int vbytes) {
  const uint32_t L32 = static_cast<uint32_t>(L);
  const uint32_t vmax32 = static_cast<uint32_t>(vmax > 0xffffffffull ? 0xffffffffull : vmax);
  const uint32_t vlim32 = static_cast<uint32_t>(vlim > 0xffffffffull ? 0xffffffffull : vlim);
#if defined(__x86_64__)
  if (have_avx512()) return narrow32_avx512(x, v, lo, hi, L32, vmax32, vlim32, x32, vout, vbytes);
#endif
  for (size_t i = lo; i < hi; ++i) {
    const uint32_t xi = x[i], vi = v[i];
    if (xi >= L32) return 1;
    if (i && x[i - 1] >= xi) return 2;
    if (vi > vmax32) return 3;
    if (vi > vlim32) return 4;
    if (x32) x32[i] = xi;
    if (vbytes == 1) static_cast<uint8_t*>(vout)[i] = static_cast<uint8_t>(vi);
    else static_cast<uint32_t*>(vout)[i] = vi;
  }
  return 0;
}

int narrow_validate(const uint64_t* x, const uint64_t* v, size_t lo, size_t hi, uint64_t L, uint64_t vmax,
                    uint64_t vlim, uint32_t* x32, void* vout, int vbytes) {
#if defined(__x86_64__)
  if (have_avx512()) return narrow_avx512(x, v, lo, hi, L, vmax, vlim, x32, vout, vbytes);
#endif
  for (size_t i = lo; i < hi; ++i) {
    const uint64_t xi = x[i], vi = v[i];
    if (xi >= L) return 1;
    if (i && x[i - 1] >= xi) return 2;
    if (vi > vmax) return 3;
    if (vi > vlim) return 4;
    x32[i] = static_cast<uint32_t>(xi);
    if (vbytes == 1) static_cast<uint8_t*>(vout)[i] = static_cast<uint8_t>(vi);
    else static_cast<uint32_t*>(vout)[i] = static_cast<uint32_t>(vi);
  }
  return 0;
}

#if defined(__x86_64__)
__attribute__((target("avx512f,avx512bw"))) uint64_t narrow_v32_avx512(const uint32_t* v, size_t lo, size_t hi,
                                                                      uint32_t vmax, uint32_t vlim, void* vout,
                                                                      int vbytes) {
  const __m512i vVmax = _mm512_set1_epi32(static_cast<int>(vmax));
  const __m512i vVlim = _mm512_set1_epi32(static_cast<int>(vlim));
  auto scalar = [&](size_t k) -> uint64_t {
    if (v[k] > vmax) return 4 * uint64_t(k) + 2;
    if (v[k] > vlim) return 4 * uint64_t(k) + 3;
    if (vbytes == 1) static_cast<uint8_t*>(vout)[k] = static_cast<uint8_t>(v[k]);
    else static_cast<uint32_t*>(vout)[k] = v[k];
    return ~0ull;
  };
  size_t i = lo;
  for (; i < hi && (i & 15u); ++i)
    if (const uint64_t c = scalar(i); c != ~0ull) return c;
  for (; i + 16 <= hi; i += 16) {
    const __m512i vs = _mm512_loadu_si512(reinterpret_cast<const void*>(v + i));
    if (_mm512_cmpgt_epu32_mask(vs, vVmax) | _mm512_cmpgt_epu32_mask(vs, vVlim)) {
      for (size_t k = i; k < i + 16; ++k)
        if (const uint64_t c = scalar(k); c != ~0ull) return c;
    }
    if (vbytes == 1) {
      _mm_stream_si128(reinterpret_cast<__m128i*>(static_cast<uint8_t*>(vout) + i), _mm512_cvtepi32_epi8(vs));
    } else {
      _mm512_storeu_si512(reinterpret_cast<void*>(static_cast<uint32_t*>(vout) + i), vs);
    }
  }
  for (; i < hi; ++i)
    if (const uint64_t c = scalar(i); c != ~0ull) return c;
  _mm_sfence();
  return ~0ull;
}
#endif

uint64_t narrow_v32(const uint32_t* v, size_t lo, size_t hi, uint64_t vmax, uint64_t vlim, void* vout, int vbytes) {
  const uint32_t vmax32 = static_cast<uint32_t>(vmax > 0xffffffffull ? 0xffffffffull : vmax);
  const uint32_t vlim32 = static_cast<uint32_t>(vlim > 0xffffffffull ? 0xffffffffull : vlim);
#if defined(__x86_64__)
  if (have_avx512()) return narrow_v32_avx512(v, lo, hi, vmax32, vlim32, vout, vbytes);
#endif
  for (size_t i = lo; i < hi; ++i) {
    if (v[i] > vmax32) return 4 * uint64_t(i) + 2;
    if (v[i] > vlim32) return 4 * uint64_t(i) + 3;
    if (vbytes == 1) static_cast<uint8_t*>(vout)[i] = static_cast<uint8_t>(v[i]);
    else static_cast<uint32_t*>(vout)[i] = v[i];
  }
  return ~0ull;
}

unsigned host_threads() { return HostPool::get().size(); }

void host_run(unsigned count, std::function<void(unsigned)> job) { HostPool::get().run(count, std::move(job)); }

}  // namespace nb200

// Device context: stream, stream-ordered memory pool, transition tables,
// list allocation and host<->device transfer.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <dlfcn.h>
#include <execinfo.h>
#include <sstream>
#include <vector>

#include "dev.hpp"
#include "util.cuh"

namespace synchro::dev {

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  std::ostringstream os;
  os << "CUDA error " << cudaGetErrorName(e) << " (" << cudaGetErrorString(e) << ") at " << file
     << ":" << line << " in " << what;
  throw DeviceError(os.str());
}

int device_count() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

Context::Context(const Automaton& aut, int device) {
  int ndev = device_count();
  if (ndev == 0) throw DeviceError("no CUDA device available (the B200 data plane has no CPU fallback)");
  if (device < 0) SW_CUDA(cudaGetDevice(&device));
  device_ = device;
  SW_CUDA(cudaSetDevice(device_));
  cudaStream_t s;
  SW_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  stream_ = s;
  // The device's default pool, keeping freed blocks (lists are re-allocated
  // every level, and every solve_exact call creates a context: a pool of its
  // own would start empty each time — measured: +100 ms per n=300 solve; it
  // did not help the threaded batch runner either).
  cudaMemPool_t pool;
  SW_CUDA(cudaDeviceGetDefaultMemPool(&pool, device_));
  u64 thresh = ~u64{0};
  SW_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
  pool_ = pool;
  bind(aut);
}

// (Re)bind to an automaton: upload its tables, reset the counters.  The
// stream and scratch buffers stay, so a worker thread reuses one context
// for a whole batch of solves (experiment.cpp).
void Context::bind(const Automaton& aut) {
  const u32 n = aut.state_count(), k = aut.alphabet_size();
  if (words_for(n) > static_cast<u32>(kMaxW))
    throw std::invalid_argument("n > 1024 states is not supported by the device kernels");
  if (static_cast<u64>(n) * k > 24576)
    throw std::invalid_argument("n*k > 24576 transitions is not supported by the device kernels");
  SW_CUDA(cudaSetDevice(device_));
  if (d_img) free(const_cast<void*>(d_img));
  d_img = nullptr;
  n_ = n;
  k_ = k;
  W_ = words_for(n);
  counters = Counters{};
  timing = false;
  contain_stats = false;

  // Image table u16[k*n] at [a*n+q].
  std::vector<uint16_t> img(static_cast<size_t>(k_) * n_);
  for (u32 a = 0; a < k_; ++a)
    for (u32 q = 0; q < n_; ++q) img[static_cast<size_t>(a) * n_ + q] = static_cast<uint16_t>(aut.next(q, a));
  void* p1 = alloc(img.size() * 2);
  memcpy_h2d(p1, img.data(), img.size() * 2);
  d_img = p1;

  sync();
}

Context::~Context() {
  cudaSetDevice(device_);
  for (auto& s : scratch_)
    if (s.p) cudaFreeAsync(s.p, as_stream(stream_));
  for (auto& v : cache_)
    for (void* p : v) cudaFreeAsync(p, as_stream(stream_));
  if (d_img) cudaFreeAsync(const_cast<void*>(d_img), as_stream(stream_));
  cudaStreamSynchronize(as_stream(stream_));
  cudaStreamDestroy(as_stream(stream_));
}

void* Context::alloc(size_t bytes) {
  if (bytes == 0) bytes = 16;
  int cls = -1;
  if (bytes <= (size_t{256} << (kCacheClasses - 1))) {
    cls = 0;
    while ((size_t{256} << cls) < bytes) ++cls;
    if (!cache_[cls].empty()) {
      void* p = cache_[cls].back();
      cache_[cls].pop_back();
      cached_bytes_ -= size_t{256} << cls;
      cached_live_[p] = cls;
      return p;
    }
    bytes = size_t{256} << cls;
  }
  void* p = nullptr;
  counters.allocs++;
  SW_CUDA(cudaMallocFromPoolAsync(&p, bytes, static_cast<cudaMemPool_t>(pool_), as_stream(stream_)));
  if (cls >= 0) cached_live_[p] = cls;
  return p;
}

void Context::free(void* p) {
  if (!p) return;
  constexpr size_t kMaxCached = size_t{256} << 20;
  if (auto it = cached_live_.find(p); it != cached_live_.end()) {
    const int cls = it->second;
    cached_live_.erase(it);
    if (cached_bytes_ + (size_t{256} << cls) <= kMaxCached) {
      cache_[cls].push_back(p);
      cached_bytes_ += size_t{256} << cls;
      return;
    }
  }
  SW_CUDA(cudaFreeAsync(p, as_stream(stream_)));
}

void Context::memcpy_d2d(void* dst, const void* src, size_t bytes) {
  if (bytes) SW_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, as_stream(stream_)));
}

void Context::sync() {
  counters.syncs++;
  static const bool trace = [] {
    const char* e = std::getenv("SYNCHRO_TRACE_SYNCS");
    return e && *e == '1';
  }();
  if (trace) {  // library offsets of the calling frames (resolve with addr2line)
    void* fr[6];
    const int nf = backtrace(fr, 6);
    std::fprintf(stderr, "SYNC");
    for (int i = 1; i < nf; ++i) {
      Dl_info info{};
      if (dladdr(fr[i], &info) && info.dli_fbase)
        std::fprintf(stderr, " %zx", static_cast<size_t>(static_cast<char*>(fr[i]) -
                                                         static_cast<char*>(info.dli_fbase)));
    }
    std::fprintf(stderr, "\n");
  }
  SW_CUDA(cudaStreamSynchronize(as_stream(stream_)));
}

StreamTimer::StreamTimer(Context& c) : c_(c) {
  cudaEvent_t a, b;
  SW_CUDA(cudaEventCreate(&a));
  SW_CUDA(cudaEventCreate(&b));
  e0_ = a;
  e1_ = b;
}
StreamTimer::~StreamTimer() {
  cudaEventDestroy(static_cast<cudaEvent_t>(e0_));
  cudaEventDestroy(static_cast<cudaEvent_t>(e1_));
}
void StreamTimer::start() { SW_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(e0_), as_stream(c_.stream()))); }
double StreamTimer::stop_ms() {
  SW_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(e1_), as_stream(c_.stream())));
  SW_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(e1_)));
  float ms = 0;
  SW_CUDA(cudaEventElapsedTime(&ms, static_cast<cudaEvent_t>(e0_), static_cast<cudaEvent_t>(e1_)));
  return ms;
}

// Small readbacks (sizes, flags, counters: several per engine step) go
// through a pinned staging buffer: a device-to-pageable copy is staged by the
// driver under a lock that the batch runner's threads contend on.
constexpr size_t kPinnedBytes = 64 * 1024;

void Context::memcpy_d2h(void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  counters.d2h_bytes += bytes;
  if (bytes <= kPinnedBytes) {
    // one buffer per host thread, kept for the thread's lifetime (allocating
    // and freeing pinned memory per context costs milliseconds: cudaFreeHost
    // synchronises the device)
    thread_local void* pinned = nullptr;
    if (!pinned) SW_CUDA(cudaHostAlloc(&pinned, kPinnedBytes, cudaHostAllocPortable));
    SW_CUDA(cudaMemcpyAsync(pinned, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream_)));
    sync();
    std::memcpy(dst, pinned, bytes);
    return;
  }
  SW_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream_)));
  sync();
}

void Context::memcpy_h2d(void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  counters.h2d_bytes += bytes;
  SW_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream_)));
}

void* Context::scratch(int slot, size_t bytes) {
  Scratch& s = scratch_[slot];
  if (s.bytes < bytes) {
    if (s.p) free(s.p);
    s.bytes = bytes + bytes / 4 + 4096;
    s.p = alloc(s.bytes);
  }
  return s.p;
}

// ------------------------------------------------------------------ DList
DList::DList(Context* ctx, size_t cap, bool tagged) : ctx_(ctx), tagged_(tagged) { reserve(cap); }

DList::~DList() { release(); }

DList& DList::operator=(DList&& o) noexcept {
  if (this != &o) {
    release();
    words = o.words;
    cards = o.cards;
    tags = o.tags;
    ctx_ = o.ctx_;
    size_ = o.size_;
    cap_ = o.cap_;
    tagged_ = o.tagged_;
    stats_ok_ = o.stats_ok_;
    known_stats_ = o.known_stats_;
    o.stats_ok_ = false;
    o.words = nullptr;
    o.cards = nullptr;
    o.tags = nullptr;
    o.size_ = o.cap_ = 0;
  }
  return *this;
}

void DList::release() {
  if (ctx_) {
    try {
      ctx_->free(words);
      ctx_->free(cards);
      ctx_->free(tags);
    } catch (...) {
    }
  }
  words = nullptr;
  cards = nullptr;
  tags = nullptr;
  size_ = cap_ = 0;
}

void DList::reserve(size_t cap) {
  if (cap <= cap_ && words) return;
  const size_t W = ctx_->W();
  u64* nw = static_cast<u64*>(ctx_->alloc(cap * W * 8));
  u32* nc = static_cast<u32*>(ctx_->alloc(cap * 4));
  u64* nt = tagged_ ? static_cast<u64*>(ctx_->alloc(cap * 8)) : nullptr;
  cudaStream_t s = as_stream(ctx_->stream());
  if (size_) {
    SW_CUDA(cudaMemcpyAsync(nw, words, size_ * W * 8, cudaMemcpyDeviceToDevice, s));
    SW_CUDA(cudaMemcpyAsync(nc, cards, size_ * 4, cudaMemcpyDeviceToDevice, s));
    if (tagged_) SW_CUDA(cudaMemcpyAsync(nt, tags, size_ * 8, cudaMemcpyDeviceToDevice, s));
  }
  ctx_->free(words);
  ctx_->free(cards);
  ctx_->free(tags);
  words = nw;
  cards = nc;
  tags = nt;
  cap_ = cap;
}

void truncate(DList& l, size_t count) {
  if (count < l.size()) l.set_size(count);
}

// ------------------------------------------------------------ transfers
DList upload(Context& c, const u64* words, const u32* cards, const u64* tags, size_t count) {
  DList l(&c, count, tags != nullptr);
  c.memcpy_h2d(l.words, words, count * c.W() * 8);
  if (cards) {
    c.memcpy_h2d(l.cards, cards, count * 4);
  } else {
    std::vector<u32> cc(count);
    for (size_t i = 0; i < count; ++i) {
      u32 s = 0;
      for (u32 w = 0; w < c.W(); ++w) s += static_cast<u32>(__builtin_popcountll(words[i * c.W() + w]));
      cc[i] = s;
    }
    c.memcpy_h2d(l.cards, cc.data(), count * 4);
    c.sync();
  }
  if (tags) c.memcpy_h2d(l.tags, tags, count * 8);
  l.set_size(count);
  c.sync();
  return l;
}

void download(Context& c, const DList& l, u64* words, u32* cards, u64* tags) {
  if (words) c.memcpy_d2h(words, l.words, l.size() * c.W() * 8);
  if (cards) c.memcpy_d2h(cards, l.cards, l.size() * 4);
  if (tags && l.tagged()) c.memcpy_d2h(tags, l.tags, l.size() * 8);
}

DList make_universe(Context& c, bool tagged) {
  std::vector<u64> u = host_universe(c.n());
  u32 card = c.n();
  u64 tag = 0;
  return upload(c, u.data(), &card, tagged ? &tag : nullptr, 1);
}

DList make_singletons(Context& c, bool tagged) {
  const u32 n = c.n(), W = c.W();
  std::vector<u64> w(static_cast<size_t>(n) * W, 0);
  std::vector<u32> cards(n, 1);
  std::vector<u64> tags(n);
  for (u32 q = 0; q < n; ++q) {
    w[static_cast<size_t>(q) * W + (q >> 6)] = state_bit(q);
    tags[q] = q;
  }
  return upload(c, w.data(), cards.data(), tagged ? tags.data() : nullptr, n);
}

DList copy_list(Context& c, const DList& l, bool tagged) {
  return slice_copy(c, l, 0, l.size(), tagged);
}

DList slice_copy(Context& c, const DList& l, size_t lo, size_t hi, bool tagged) {
  const size_t cnt = hi - lo;
  DList out(&c, cnt, tagged && l.tagged());
  cudaStream_t s = as_stream(c.stream());
  if (cnt) {
    SW_CUDA(cudaMemcpyAsync(out.words, l.words + lo * c.W(), cnt * c.W() * 8, cudaMemcpyDeviceToDevice, s));
    SW_CUDA(cudaMemcpyAsync(out.cards, l.cards + lo, cnt * 4, cudaMemcpyDeviceToDevice, s));
    if (out.tagged()) SW_CUDA(cudaMemcpyAsync(out.tags, l.tags + lo, cnt * 8, cudaMemcpyDeviceToDevice, s));
  }
  out.set_size(cnt);
  return out;
}

DList strided_copy(Context& c, const DList& l, size_t start, size_t stride, bool tagged) {
  const size_t cnt = start < l.size() ? (l.size() - start + stride - 1) / stride : 0;
  DList out(&c, cnt, tagged && l.tagged());
  cudaStream_t s = as_stream(c.stream());
  if (cnt) {  // rows i = start + j*stride: 2D copies with a source pitch of stride rows
    const size_t row = static_cast<size_t>(c.W()) * 8;
    SW_CUDA(cudaMemcpy2DAsync(out.words, row, l.words + start * c.W(), row * stride, row, cnt,
                              cudaMemcpyDeviceToDevice, s));
    SW_CUDA(cudaMemcpy2DAsync(out.cards, 4, l.cards + start, 4 * stride, 4, cnt,
                              cudaMemcpyDeviceToDevice, s));
    if (out.tagged())
      SW_CUDA(cudaMemcpy2DAsync(out.tags, 8, l.tags + start, 8 * stride, 8, cnt,
                                cudaMemcpyDeviceToDevice, s));
  }
  out.set_size(cnt);
  return out;
}

u64 read_tag(Context& c, const DList& l, size_t i) {
  u64 t = 0;
  if (!l.tagged()) throw std::logic_error("read_tag: untagged list");
  c.memcpy_d2h(&t, l.tags + i, 8);
  return t;
}

std::vector<u64> read_tags(Context& c, const DList& l) {
  std::vector<u64> t(l.size());
  if (l.tagged()) c.memcpy_d2h(t.data(), l.tags, l.size() * 8);
  return t;
}

ContainIndex::~ContainIndex() {
  if (ctx) {
    try {
      ctx->free(nodes);
      ctx->free(keysig);
    } catch (...) {
    }
  }
}
ContainIndex::ContainIndex(ContainIndex&& o) noexcept { *this = std::move(o); }
ContainIndex& ContainIndex::operator=(ContainIndex&& o) noexcept {
  if (this != &o) {
    if (ctx) {
      ctx->free(nodes);
      ctx->free(keysig);
    }
    nodes = o.nodes;
    keysig = o.keysig;
    count = o.count;
    ctx = o.ctx;
    o.nodes = nullptr;
    o.keysig = nullptr;
    o.count = 0;
  }
  return *this;
}

}  // namespace synchro::dev

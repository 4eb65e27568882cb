#include "context.h"

#include <chrono>
#include <cstdint>
#include <cstdlib>

#include "tensor_ops.cuh"

namespace pepsb {

Buf::~Buf() {
  if (p && pool) pool->release(p, bytes);
}

void* Pool::alloc(size_t bytes, size_t* reserved) {
  std::lock_guard<std::mutex> lock(mu);
  // size classes: 512 B granules below 1 MiB, 2 MiB granules above
  const size_t g = bytes <= (1u << 20) ? 512 : (2u << 20);
  const size_t want = ((bytes + g - 1) / g) * g;
  auto it = free_blocks.lower_bound(want);
  if (it != free_blocks.end() && it->first <= want + want / 4 + g) {
    void* p = it->second;
    *reserved = it->first;
    cached_bytes -= it->first;
    free_blocks.erase(it);
    return p;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, want);
  if (e != cudaSuccess) {  // release this cache, then the siblings', and retry once
    cudaGetLastError();
    trim_locked();
    trim_siblings(this);
    e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error(kResourceError, "device allocation of " + std::to_string(bytes) + " bytes failed: " +
                                      cudaGetErrorString(e));
    }
  }
  reserved_bytes += want;
  *reserved = want;
  return p;
}

namespace {
std::mutex g_pools_mu;
std::vector<Pool*> g_pools;
}  // namespace

Pool::Pool(int dev) : device(dev) {
  std::lock_guard<std::mutex> g(g_pools_mu);
  g_pools.push_back(this);
}

Pool::~Pool() {
  {
    std::lock_guard<std::mutex> g(g_pools_mu);
    for (auto it = g_pools.begin(); it != g_pools.end(); ++it)
      if (*it == this) {
        g_pools.erase(it);
        break;
      }
  }
  trim();
}

void Pool::trim_siblings(const Pool* self) {
  std::lock_guard<std::mutex> g(g_pools_mu);
  for (Pool* other : g_pools) {
    if (other == self || other->device != self->device) continue;
    // try_lock: two pools failing at once must not wait on each other
    std::unique_lock<std::mutex> l(other->mu, std::try_to_lock);
    if (l.owns_lock()) other->trim_locked();
  }
}

void Pool::release(void* p, size_t bytes) {
  std::lock_guard<std::mutex> g(mu);
  if (defer) {
    parked.emplace_back(bytes, p);
    return;
  }
  free_blocks.emplace(bytes, p);
  cached_bytes += bytes;
}

void Pool::trim() {
  std::lock_guard<std::mutex> g(mu);
  trim_locked();
}

void Pool::trim_locked() {
  if (stream) cudaStreamSynchronize(stream);
  else cudaDeviceSynchronize();
  if (!defer) {
    for (auto& [sz, p] : parked) free_blocks.emplace(sz, p);
    parked.clear();
  }
  for (auto& [sz, p] : free_blocks) {
    cudaFree(p);
    reserved_bytes -= sz;
  }
  free_blocks.clear();
  cached_bytes = 0;
}

int64_t LTensor::extent_of(char c) const {
  auto pos = labels.find(c);
  if (pos == std::string::npos) throw Error(kShapeError, std::string("label '") + c + "' not found");
  return ext[pos];
}

int64_t LTensor::stride_of(char c) const {
  auto pos = labels.find(c);
  if (pos == std::string::npos) throw Error(kShapeError, std::string("label '") + c + "' not found");
  return str[pos];
}

std::vector<int64_t> row_major_strides(const std::vector<int64_t>& ext) {
  std::vector<int64_t> s(ext.size(), 1);
  for (size_t a = ext.size(); a-- > 1;) s[a - 1] = s[a] * ext[a];
  return s;
}

LTensor as_labelled(const DTensor& t, const std::string& labels, bool conj) {
  if (labels.size() != t.shape.size())
    throw Error(kShapeError, "label string '" + labels + "' does not match tensor order " +
                                 std::to_string(t.shape.size()));
  LTensor l;
  l.buf = t.buf;
  l.ptr = t.data();
  l.labels = labels;
  l.ext = t.shape;
  l.str = row_major_strides(t.shape);
  l.conj = conj;
  return l;
}

HostTimer::HostTimer(double* a) : acc(a), t0(0.0) {
  if (acc) t0 = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
HostTimer::~HostTimer() {
  if (acc) *acc += std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count() - t0;
}

Ctx::Ctx(int dev) : device(dev) {
  trace = getenv("PEPSB_TRACE") != nullptr;
  if (const char* e = getenv("PEPSB_OVERLAP")) overlap = e[0] == '0' ? 0 : e[0] == '2' ? 2 : 1;
  if (const char* e = getenv("PEPSB_CONCURRENT_SWEEPS")) concurrent_sweeps = std::atoi(e);
  if (const char* e = getenv("PEPSB_PIPELINE_ROWS")) pipeline_rows = std::atoi(e);
  PEPSB_CUDA(cudaSetDevice(dev));
  PEPSB_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  // The main stream carries the latency chain (Gram -> one-block eigensolver ->
  // small factors) while the side stream runs the overlapped operator
  // applications, whose CTAs fill every SM; with the main stream at the
  // higher priority the eigensolver's block is dispatched to the first SM
  // that drains instead of queueing behind the whole GEMM grid.
  // PEPSB_STREAM_PRIORITY=0 creates both at the default priority.
  int least = 0, greatest = 0;
  const char* pe = getenv("PEPSB_STREAM_PRIORITY");
  if (!(pe && pe[0] == '0')) PEPSB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  PEPSB_CUDA(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, greatest));
  PEPSB_CUDA(cudaStreamCreateWithPriority(&side_stream, cudaStreamNonBlocking, least));
  PEPSB_CUDA(cudaEventCreateWithFlags(&fork_event, cudaEventDisableTiming));
  PEPSB_CUDA(cudaEventCreateWithFlags(&join_event, cudaEventDisableTiming));
  main_stream = stream;
  pool = std::make_shared<Pool>(dev);
  pool->stream = stream;
  PEPSB_CUDA(cudaMalloc(&d_status, 64 * sizeof(int)));
  PEPSB_CUDA(cudaMemset(d_status, 0, 64 * sizeof(int)));
  PEPSB_CUDA(cudaMallocHost(&h_status, 64 * sizeof(int)));
  PEPSB_CUDA(cudaMalloc(&d_degenerate, sizeof(unsigned long long)));
  PEPSB_CUDA(cudaMemset(d_degenerate, 0, sizeof(unsigned long long)));
}

Ctx::~Ctx() {
  helpers.clear();
  if (stream != main_stream) join();
  join_pending();
  prefetched.reset();
  lookahead.reset();
  if (side_stream) cudaStreamSynchronize(side_stream);
  if (stream) cudaStreamSynchronize(stream);
  pool->trim();
  pool->stream = nullptr;  // buffers that outlive the context release into a stream-less pool
  profile_clear();
  for (auto e : event_pool) cudaEventDestroy(e);
  if (d_status) cudaFree(d_status);
  if (d_degenerate) cudaFree(d_degenerate);
  if (h_status) cudaFreeHost(h_status);
  if (stream) cudaStreamDestroy(stream);
  if (side_stream) cudaStreamDestroy(side_stream);
  if (fork_event) cudaEventDestroy(fork_event);
  if (join_event) cudaEventDestroy(join_event);
}

void Ctx::fork() {
  join_pending();
  if (pool->defer) throw Error(kOtherError, "nested stream fork");
  PEPSB_CUDA(cudaEventRecord(fork_event, main_stream));
  std::lock_guard<std::mutex> g(pool->mu);
  pool->defer = true;
}

void Ctx::side() {
  PEPSB_CUDA(cudaStreamWaitEvent(side_stream, fork_event, 0));
  stream = side_stream;
}

void Ctx::back() {
  PEPSB_CUDA(cudaEventRecord(join_event, side_stream));
  stream = main_stream;
  side_pending = true;
}

void Ctx::join_pending() {
  if (!side_pending) return;
  side_pending = false;
  PEPSB_CUDA(cudaStreamWaitEvent(main_stream, join_event, 0));
  std::lock_guard<std::mutex> g(pool->mu);
  pool->defer = false;
  for (auto& [sz, p] : pool->parked) {
    pool->free_blocks.emplace(sz, p);
    pool->cached_bytes += sz;
  }
  pool->parked.clear();
}

void Ctx::join() {
  PEPSB_CUDA(cudaEventRecord(join_event, side_stream));
  stream = main_stream;
  PEPSB_CUDA(cudaStreamWaitEvent(main_stream, join_event, 0));
  std::lock_guard<std::mutex> g(pool->mu);
  pool->defer = false;
  for (auto& [sz, p] : pool->parked) {
    pool->free_blocks.emplace(sz, p);
    pool->cached_bytes += sz;
  }
  pool->parked.clear();
}

BufPtr Ctx::alloc(int64_t n) {
  auto b = std::make_shared<Buf>();
  b->n = n;
  b->pool = pool;
  if (n > 0) {
    HostTimer ht(trace ? &t_alloc : nullptr);
    b->p = static_cast<double2*>(pool->alloc(static_cast<size_t>(n) * sizeof(double2), &b->bytes));
  }
  record_intermediate(static_cast<uint64_t>(n));
  return b;
}

DTensor Ctx::empty(const std::vector<int64_t>& shape) {
  DTensor t;
  t.shape = shape;
  t.buf = alloc(t.size());
  return t;
}

DTensor Ctx::zeros(const std::vector<int64_t>& shape) {
  DTensor t = empty(shape);
  fill_zero(t.data(), t.size(), stream);
  ++launches;
  return t;
}

void Ctx::sync() {
  HostTimer ht(trace ? &t_sync : nullptr);
  if (side_pending) PEPSB_CUDA(cudaStreamSynchronize(side_stream));
  PEPSB_CUDA(cudaStreamSynchronize(stream));
}

void Ctx::sync_main() {
  HostTimer ht(trace ? &t_sync : nullptr);
  PEPSB_CUDA(cudaStreamSynchronize(main_stream));
}

cudaEvent_t Ctx::take_event() {
  if (!event_pool.empty()) {
    cudaEvent_t e = event_pool.back();
    event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  PEPSB_CUDA(cudaEventCreate(&e));
  return e;
}

void Ctx::profile_clear() {
  for (auto& r : prof) {
    event_pool.push_back(r.a);
    event_pool.push_back(r.b);
  }
  prof.clear();
}

void Ctx::profile_report_ex(double* out) {
  sync();
  for (int i = 0; i < 5 * kProfKinds; ++i) out[i] = 0.0;
  for (auto& r : prof) {
    float ms = 0.f;
    PEPSB_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    out[5 * r.kind + 0] += 1.0;
    out[5 * r.kind + 1] += ms;
    out[5 * r.kind + 2] += r.flops;
    out[5 * r.kind + 3] += r.bytes;
    out[5 * r.kind + 4] += r.exec_flops;
  }
}

void Ctx::profile_report(double* out) {
  sync();
  for (int i = 0; i < 4 * kProfKinds; ++i) out[i] = 0.0;
  for (auto& r : prof) {
    float ms = 0.f;
    PEPSB_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    out[4 * r.kind + 0] += 1.0;
    out[4 * r.kind + 1] += ms;
    out[4 * r.kind + 2] += r.flops;
    out[4 * r.kind + 3] += r.bytes;
  }
}

ProfScope::ProfScope(Ctx& c, int kind, double flops, double bytes, double exec_flops) : ctx(c) {
  if (!ctx.profiling) return;
  Ctx::ProfRec r{ctx.take_event(), ctx.take_event(), kind, flops, bytes, exec_flops < 0.0 ? flops : exec_flops,
                 ctx.stream == ctx.side_stream ? 1 : 0};
  PEPSB_CUDA(cudaEventRecord(r.a, ctx.stream));
  ctx.prof.push_back(r);
  idx = static_cast<int>(ctx.prof.size()) - 1;
}

ProfScope::~ProfScope() {
  if (idx >= 0) cudaEventRecord(ctx.prof[idx].b, ctx.stream);
}

}  // namespace pepsb

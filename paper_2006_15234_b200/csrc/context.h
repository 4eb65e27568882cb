// Device context, stream-ordered buffers and labelled tensor views.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace pepsb {

class Ctx;
struct NcclComm;  // sharded.cpp

// Accumulates host wall time into *acc (no-op when acc is null).
struct HostTimer {
  explicit HostTimer(double* acc);
  ~HostTimer();
  double* acc;
  double t0;
};

// Stream-ordered device buffer (cudaMallocAsync from the device pool; freed
// with cudaFreeAsync on the context stream when the last reference drops).
// Caching device allocator.  Every buffer is used on the single context stream,
// so a freed block can be handed to the next allocation immediately (stream
// order protects it); cudaMalloc is only called when no cached block fits.
// Shared by the context and its buffers, so buffers may outlive the context.
struct Pool {
  std::multimap<size_t, void*> free_blocks;
  size_t cached_bytes = 0, reserved_bytes = 0;
  cudaStream_t stream = nullptr;  // cleared when the owning context goes away
  // Two-stream phases (Ctx::fork): blocks released while work runs on two
  // streams are parked until the streams join -- stream order alone no longer
  // protects them from reuse by the other stream.
  bool defer = false;
  std::vector<std::pair<size_t, void*>> parked;
  // Buffers may be released from another host thread (the row pipeline and
  // the concurrent cache sweeps hand tensors between contexts).
  std::mutex mu;
  void* alloc(size_t bytes, size_t* reserved);
  void release(void* p, size_t bytes);
  void trim();  // synchronises, then returns every cached block to the driver
  void trim_locked();
  // Every live pool of a device is registered so that an allocation failing
  // in one pool can reclaim blocks cached by its siblings (the helper contexts
  // of the row pipeline and the concurrent sweeps each own a pool).
  int device = 0;
  explicit Pool(int dev);
  ~Pool();
  static void trim_siblings(const Pool* self);
};

struct Buf {
  double2* p = nullptr;
  int64_t n = 0;
  size_t bytes = 0;  // size class actually reserved
  // Every imaginary part is exactly zero (host data checked on upload; kept by
  // copies and by products of real operands).  GEMMs with a real operand run
  // the complex x real kernel: half the DMMAs of the 4M scheme, bitwise the
  // same sums as complex arithmetic on zero imaginary parts.
  bool real = false;
  std::shared_ptr<Pool> pool;
  ~Buf();
};
using BufPtr = std::shared_ptr<Buf>;

// Contiguous row-major device tensor in the reference's logical axis order.
struct DTensor {
  BufPtr buf;
  std::vector<int64_t> shape;
  int64_t size() const {
    int64_t n = 1;
    for (auto e : shape) n *= e;
    return n;
  }
  double2* data() const { return buf ? buf->p : nullptr; }
};

// Labelled strided view used by the contraction engine.  Axis a carries
// label labels[a], extent ext[a], element stride str[a]; conj is applied
// lazily by the consumer.
struct LTensor {
  BufPtr buf;
  const double2* ptr = nullptr;
  std::string labels;
  std::vector<int64_t> ext, str;
  bool conj = false;
  int64_t size() const {
    int64_t n = 1;
    for (auto e : ext) n *= e;
    return n;
  }
  int64_t extent_of(char c) const;
  int64_t stride_of(char c) const;
};

LTensor as_labelled(const DTensor& t, const std::string& labels, bool conj = false);
std::vector<int64_t> row_major_strides(const std::vector<int64_t>& ext);

class Ctx {
 public:
  explicit Ctx(int device);
  ~Ctx();
  Ctx(const Ctx&) = delete;
  Ctx& operator=(const Ctx&) = delete;

  BufPtr alloc(int64_t n);  // n complex elements (uninitialised)
  std::shared_ptr<struct Pool> pool;
  DTensor empty(const std::vector<int64_t>& shape);
  DTensor zeros(const std::vector<int64_t>& shape);
  void sync();       // every stream of the context
  void sync_main();  // the main stream only (pending side-stream work keeps running)

  // Two-stream phase: fork() marks the fork point on the main stream (blocks
  // released from here on are parked); work enqueued next stays on the main
  // stream; side() switches `stream` to the side stream, which starts after
  // the fork point, i.e. concurrently with the main-stream work enqueued since;
  // join() makes the main stream wait for the side stream, switches back and
  // unparks the blocks.
  void fork();
  void side();
  void join();
  // Leave the side stream without joining (work on it keeps running); a later
  // join_pending() makes the main stream wait for it and unparks the blocks.
  void back();
  void join_pending();
  bool side_pending = false;
  // Row lookahead (decomp.cpp): the next column's operator to start on the
  // side stream during this column's tail, and what was started for this one.
  std::shared_ptr<void> lookahead, prefetched;

  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t main_stream = nullptr, side_stream = nullptr;
  cudaEvent_t fork_event = nullptr, join_event = nullptr;
  // Device status word shared by the small factorization kernels
  // (SmallStatus bits); read back at the einsumsvd sync points.
  int* d_status = nullptr;
  int* h_status = nullptr;  // pinned
  // Simple-update truncations through a degenerate singular pair (device counter).
  unsigned long long* d_degenerate = nullptr;
  // Launch accounting (for the bench's gpu_launches claim).
  int64_t launches = 0;
  // Host-side tracing (PEPSB_TRACE): seconds spent in allocation, free and sync.
  bool trace = false;
  double t_alloc = 0.0, t_free = 0.0, t_sync = 0.0;
  int64_t faithful_redos = 0;  // CholeskyQR breakdowns redone on the Gram-eigh route
  int64_t tsqr_fallbacks = 0;  // projected SVDs that needed the TSQR R factor
  int64_t lookahead_misses = 0;  // row lookaheads discarded (the rank guess was wrong)
  // Cost counters (reference instr::flops definition: 2 per complex MAC,
  // proj/include/peps/instrument.hpp:19-65).
  uint64_t flops = 0;
  uint64_t einsumsvd_flops = 0;
  uint64_t peak_elements = 0;
  void record_intermediate(uint64_t n) {
    if (n > peak_elements) peak_elements = n;
  }
  // Options
  // Power-iteration orthogonalisation: 0 = the reference's Gram-eigh basis
  // (default).  The basis fixes the column phases of U, i.e. the bond gauge of
  // emitted boundary sites, and the NEXT row's sketch Omega is drawn in the
  // reference layout of those bonds -- so multi-row contractions only agree
  // with the reference if the basis does.  1 = CholeskyQR2 (same spans, other
  // basis): identical within one row / one einsumsvd, but across rows it
  // differs from the reference by the sketch-dependent rSVD error.
  int orth_mode = 0;
  // Hide the big-side k x k eigensolver of each power iteration behind the
  // next operator application on a second stream (decomp.cpp
  // apply_orth_speculative): option "overlap" / PEPSB_OVERLAP, 0 off, 1 when
  // the column extent is >= 2^15 (default), 2 always.
  int overlap = 1;
  // build_row_cache: run the bottom sweep on a helper context from a second
  // host thread, concurrently with the top sweep (option "concurrent_sweeps":
  // -1 auto = when max_rank <= 48, where the sweeps are latency-bound; at
  // config 5's m = 64 one sweep already fills the GPU and two contend: 26.0 s
  // concurrent vs 22.3 s sequential; 0 off; 1 on).
  int concurrent_sweeps = -1;
  // contract_two_layer: consecutive rows on two contexts, a few columns apart
  // (option "pipeline_rows").
  int pipeline_rows = -1;  // rows in flight K (< 2: sequential; -1: automatic, peps.cpp pipeline_depth)
  std::vector<std::unique_ptr<Ctx>> helpers;  // lazily created, same device
  // NCCL communicator of the bond-sharded row absorb (pepsb_comm_init; sharded.cpp)
  std::shared_ptr<NcclComm> comm;

  // Optional per-launch device timing (CUDA events on `stream`), used by the
  // bench's roofline pass; off in timed runs.
  enum ProfKind { kProfGemm = 0, kProfSmall = 1, kProfGather = 2, kProfOther = 3, kProfKinds = 4 };
  struct ProfRec {
    cudaEvent_t a, b;
    int kind;
    double flops, bytes;
    double exec_flops;  // flops the hardware executes (3M GEMM: 6 per complex MAC, not 8)
    int side = 0;       // recorded on the side stream
  };
  bool profiling = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t take_event();
  void profile_report(double* out);  // per kind: count, ms, flops, bytes
  void profile_report_ex(double* out);  // per kind: count, ms, flops, bytes, executed flops
  void profile_clear();
};

// RAII device-time scope (no-op unless ctx.profiling).
struct ProfScope {
  ProfScope(Ctx& c, int kind, double flops = 0.0, double bytes = 0.0, double exec_flops = -1.0);
  ~ProfScope();
  Ctx& ctx;
  int idx = -1;
};

}  // namespace pepsb

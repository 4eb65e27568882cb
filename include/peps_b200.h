/*
 * peps_b200.h — C ABI of the B200-native einsumsvd library.
 *
 * The reference (arxiv/paper_2006_15234, /root/reference/proj) has no FFI: its
 * drop-in interface is the public C++ API in the proj/include/peps headers, and
 * proj/include/peps/backend.hpp:7-10 states that another engine "would slot in
 * behind the same kernel signatures".  Each entry point below replaces one of
 * those signatures (cited per function); a reference-side C++ shim that binds
 * them is shown in INTEGRATION.md.
 *
 * Conventions
 *  - Every tensor is complex128, row-major, last index fastest, exactly the
 *    reference's Tensor layout (proj/include/peps/tensor.hpp:13-20); host
 *    buffers are interleaved (re, im) doubles.
 *  - Tensors, states and boundaries live in device memory behind opaque
 *    handles so sweeps never round-trip through the host.
 *  - Every function returns 0 on success or a PEPSB_E_* kind; the message is
 *    in pepsb_last_error() (thread-local).  Kinds mirror the reference
 *    exceptions (proj/include/peps/errors.hpp:10-34).
 *  - There is no CPU fallback: without a usable sm_100a device every call
 *    fails with PEPSB_E_CUDA.
 */
#ifndef PEPS_B200_H
#define PEPS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PEPSB_OK = 0,
  PEPSB_E_SHAPE = 1,      /* peps::ShapeError */
  PEPSB_E_VALIDATION = 2, /* peps::ValidationError */
  PEPSB_E_RESOURCE = 3,   /* peps::ResourceError */
  PEPSB_E_NUMERICAL = 4,  /* peps::NumericalError */
  PEPSB_E_CONFIG = 5,     /* peps::ConfigError */
  PEPSB_E_CUDA = 6,       /* device / driver failure */
  PEPSB_E_OTHER = 9
};

enum { PEPSB_EXACT = 0, PEPSB_IMPLICIT_RSVD = 1 };         /* peps::SvdStrategy (decomposition.hpp:34) */
enum { PEPSB_SPLIT = 0, PEPSB_LEFT = 1, PEPSB_RIGHT = 2 };  /* peps::Absorb (decomposition.hpp:37) */

typedef struct pepsb_ctx pepsb_ctx;
typedef struct pepsb_tensor pepsb_tensor;
typedef struct pepsb_state pepsb_state;
typedef struct pepsb_boundary pepsb_boundary;
typedef struct pepsb_row_cache pepsb_row_cache;
typedef struct pepsb_band_env pepsb_band_env;

/* peps::TruncationPolicy (decomposition.hpp:14-17) */
typedef struct {
  uint64_t max_rank; /* 0: unbounded */
  double rel_cutoff; /* default 1e-14 */
} pepsb_trunc;

/* peps::RsvdConfig (decomposition.hpp:21-25) */
typedef struct {
  int32_t power_iters; /* default 2 */
  int32_t oversample;  /* < 0: max(5, ceil(0.1 * target)) */
  uint64_t seed;
} pepsb_rsvd;

/* peps::ContractOption, two-layer fields (contraction.hpp:18-32) */
typedef struct {
  pepsb_trunc trunc;
  int32_t strategy; /* PEPSB_EXACT / PEPSB_IMPLICIT_RSVD */
  pepsb_rsvd rsvd;
  int32_t canonicalize;
  uint64_t seed;
} pepsb_contract_opt;

/* ---------------------------------------------------------------- context */
const char* pepsb_last_error(void);
int pepsb_last_error_kind(void);
int pepsb_ctx_create(int device, pepsb_ctx** out);
int pepsb_ctx_destroy(pepsb_ctx* ctx);
int pepsb_ctx_sync(pepsb_ctx* ctx);
/* keys: "orth_mode" (0 reference Gram-eigh, 1 CholeskyQR2),
 * "eig_solver" (0 auto, 1 Jacobi, 2 divide and conquer; process-wide),
 * "gemm_algo" (0 4M real embedding, 1 3M, 2 4M complex fragments), "gemm_real",
 * "gemm_small", "gemm_stream", "gemm_ws", "gemm_gram" (process-wide GEMM kernel choices), "overlap" (0..2),
 * "pipeline_rows" (-1 auto, 0..8), "concurrent_sweeps" (-1 auto, 0, 1).
 * Unknown keys fail with ConfigError. */
int pepsb_ctx_set_option(pepsb_ctx* ctx, const char* key, int64_t value);
/* out[0..5] = flops (instr::flops convention, instrument.hpp:19-65),
 * einsumsvd_flops, peak_elements, kernel launches issued by the library,
 * CholeskyQR breakdowns redone on the Gram-eigh route, TSQR fallbacks */
int pepsb_ctx_counters(pepsb_ctx* ctx, uint64_t* out6);
int pepsb_ctx_reset_counters(pepsb_ctx* ctx);
/* Named counter: "flops", "einsumsvd_flops", "peak_elements", "launches",
 * "faithful_redos", "tsqr_fallbacks", "lookahead_misses" (row-absorb
 * lookaheads discarded because the next column's rank guess failed),
 * "degenerate_truncations" (simple-update
 * truncations whose cut falls inside a singular pair equal to 1e-10 relative:
 * the kept subspace there is rounding-dependent). */
int pepsb_ctx_get_counter(pepsb_ctx* ctx, const char* name, uint64_t* value);
/* Per-launch CUDA-event timing of the library's kernels (off by default).
 * Report: 4 kinds (0 GEMM, 1 small factorizations, 2 gathers, 3 other) x
 * {launches, device ms, algorithmic real flops, algorithmic bytes}. */
int pepsb_ctx_profile(pepsb_ctx* ctx, int enable);
int pepsb_ctx_profile_report(pepsb_ctx* ctx, double* out16);
/* Same with a fifth value per kind: the real flops the hardware executes (the
 * 3M GEMM runs 6 real flops per complex MAC where the algorithmic count is 8). */
int pepsb_ctx_profile_report_ex(pepsb_ctx* ctx, double* out20);
/* Per-launch records of the profile (kind, device ms, algorithmic flops) x n; returns n */
int pepsb_ctx_profile_records(pepsb_ctx* ctx, double* out, int cap);
/* Timeline of the profile (streams overlapped as in a timed run): per launch
 * (kind, start ms, end ms, executed flops, stream 0 main / 1 side), times
 * relative to the first record; returns n */
int pepsb_ctx_profile_timeline(pepsb_ctx* ctx, double* out, int cap);
/* Diagnostics: device status word idx (word 7 = cumulative Jacobi sweeps). */
int pepsb_ctx_debug_word(pepsb_ctx* ctx, int idx, int reset);
/* CUDA stream the library enqueues on (cudaStream_t), for event timing */
void* pepsb_ctx_stream(pepsb_ctx* ctx);

/* ---------------------------------------------------------------- tensors (peps::Tensor, tensor.hpp:20-69) */
int pepsb_tensor_from_host(pepsb_ctx* ctx, int ndim, const int64_t* shape, const double* data, pepsb_tensor** out);
int pepsb_tensor_from_device(pepsb_ctx* ctx, int ndim, const int64_t* shape, const void* dptr, pepsb_tensor** out);
int pepsb_tensor_ndim(const pepsb_tensor* t);
int pepsb_tensor_shape(const pepsb_tensor* t, int64_t* shape);
int pepsb_tensor_to_host(pepsb_ctx* ctx, const pepsb_tensor* t, double* out);
/* stream-ordered copy into (pinned) host memory; completes at pepsb_ctx_sync */
int pepsb_tensor_to_host_async(pepsb_ctx* ctx, const pepsb_tensor* t, double* out);
int pepsb_tensor_to_device(pepsb_ctx* ctx, const pepsb_tensor* t, void* dptr);
void pepsb_tensor_free(pepsb_tensor* t);

/* random_tensor / random_tensor_real (tensor.hpp:74-80, tensor.cpp:192-208), bit-identical */
int pepsb_random_tensor(pepsb_ctx* ctx, int ndim, const int64_t* shape, uint64_t seed, int real, pepsb_tensor** out);

/* contract(spec, tensors) (einsum.hpp:27) */
int pepsb_contract(pepsb_ctx* ctx, const char* spec, int n, pepsb_tensor* const* ts, pepsb_tensor** out);

/* ImplicitOperator::apply / adjoint_apply / materialize (implicit.hpp:26-30).
 * labels_csv: comma-separated label strings, one per tensor.
 * mode 0: apply(probe), 1: adjoint_apply(probe), 2: materialize() (probe ignored) */
int pepsb_implicit(pepsb_ctx* ctx, int n, pepsb_tensor* const* ts, const char* labels_csv, const char* rows,
                   const char* cols, const pepsb_tensor* probe, int mode, pepsb_tensor** out);

/* gram_orthogonalize(Tensor, split) (decomposition.hpp:52) */
int pepsb_gram_orthogonalize(pepsb_ctx* ctx, const pepsb_tensor* a, int split, pepsb_tensor** q, pepsb_tensor** r);

/* ---- building blocks of the bond-sharded einsumsvd (paper_2006_15234_b200/sharded.py) */
/* Slice [start, start+count) along `axis` of random_tensor(shape, seed) (tensor.cpp:192-201):
 * bit-identical to the same elements of the full tensor (counter-based stream). */
int pepsb_random_slice(pepsb_ctx* ctx, int ndim, const int64_t* shape, int axis, int64_t start, int64_t count,
                       uint64_t seed, int real, pepsb_tensor** out);
int pepsb_tensor_conj(pepsb_ctx* ctx, const pepsb_tensor* a, pepsb_tensor** out);
/* Copy of [start, start+count) along `axis`. */
int pepsb_tensor_slice(pepsb_ctx* ctx, const pepsb_tensor* a, int axis, int64_t start, int64_t count,
                       pepsb_tensor** out);
/* New handle sharing the buffer with a different shape (same element count). */
int pepsb_tensor_reshape(const pepsb_tensor* a, int ndim, const int64_t* shape, pepsb_tensor** out);
/* Device pointer of the tensor's contiguous row-major complex128 buffer. */
int pepsb_tensor_data_ptr(const pepsb_tensor* a, void** ptr);
/* G = Z^H Z over all leading axes of z (the last axis is the probe axis). */
int pepsb_gram(pepsb_ctx* ctx, const pepsb_tensor* z, pepsb_tensor** g);
/* gram_factors (decomposition.cpp:128-156) of a k x k Gram matrix: P = X l^-1/2,
 * R = l^1/2 X^H, X (phase-fixed eigenvectors), lam (descending), deficient flags. */
int pepsb_gram_factors(pepsb_ctx* ctx, const pepsb_tensor* g, pepsb_tensor** p, pepsb_tensor** r,
                       pepsb_tensor** vecs, double* lam, int* deficient, int64_t cap);
/* Projected SVD of B = Z^H (the rSVD's last stage): k x k left vectors and sigma. */
int pepsb_projected_svd(pepsb_ctx* ctx, const pepsb_tensor* z, int64_t target, pepsb_tensor** ut, double* s,
                        int64_t cap);

/* eigh(Tensor) (linalg.hpp:41, linalg.cpp:256-295): values descending (capacity cap),
 * vectors n x n with column j the phase-fixed eigenvector j.  n <= 256.  The
 * solver is process-wide option "eig_solver" (0 auto: one-warp Jacobi for n <= 6,
 * else divide and conquer; 1 Jacobi; 2 divide and conquer). */
int pepsb_eigh(pepsb_ctx* ctx, const pepsb_tensor* a, double* values, int64_t cap, pepsb_tensor** vectors);

/* svd(Tensor, split) (linalg.hpp:21-22); s has capacity s_cap, *k = min extent */
int pepsb_svd(pepsb_ctx* ctx, const pepsb_tensor* a, int split, pepsb_tensor** u, double* s, int64_t s_cap,
              int64_t* k, pepsb_tensor** v);

/* randomized_svd (decomposition.hpp:43-44) */
int pepsb_randomized_svd(pepsb_ctx* ctx, int n, pepsb_tensor* const* ts, const char* labels_csv, const char* rows,
                         const char* cols, const pepsb_trunc* policy, const pepsb_rsvd* cfg, pepsb_tensor** u,
                         double* s, int64_t s_cap, int64_t* rank, pepsb_tensor** v, int* rank_clamped);

/* einsumsvd (decomposition.hpp:65-67) */
int pepsb_einsumsvd(pepsb_ctx* ctx, int n, pepsb_tensor* const* ts, const char* labels_csv, const char* rows,
                    const char* cols, const pepsb_trunc* policy, int strategy, int absorb, const pepsb_rsvd* cfg,
                    pepsb_tensor** t1, pepsb_tensor** t2, double* s, int64_t s_cap, int64_t* rank,
                    int* rank_clamped);

/* ---------------------------------------------------------------- PEPS (state.hpp:33-61) */
int pepsb_state_create(pepsb_ctx* ctx, int rows, int cols, int d, pepsb_tensor* const* sites, pepsb_state** out);
int pepsb_state_site(const pepsb_state* s, int row, int col, pepsb_tensor** out);
/* grid size and physical dimension of a state */
int pepsb_state_dims(const pepsb_state* s, int* rows, int* cols, int* d);
void pepsb_state_free(pepsb_state* s);

/* TwoLayerBoundary (contraction.hpp:77-80) */
int pepsb_boundary_create(pepsb_ctx* ctx, int n, pepsb_tensor* const* sites, const int64_t* phys_pairs,
                          pepsb_boundary** out);
int pepsb_boundary_length(const pepsb_boundary* b);
int pepsb_boundary_site(const pepsb_boundary* b, int i, pepsb_tensor** out);
int pepsb_boundary_phys(const pepsb_boundary* b, int64_t* pairs);
void pepsb_boundary_free(pepsb_boundary* b);

/* two_layer_first_row / two_layer_apply_row / contract_two_layer (contraction.hpp:82-90) */
int pepsb_two_layer_first_row(pepsb_ctx* ctx, const pepsb_state* bra, const pepsb_state* ket, pepsb_boundary** out);
int pepsb_two_layer_apply_row(pepsb_ctx* ctx, const pepsb_boundary* top, const pepsb_state* bra,
                              const pepsb_state* ket, int row, const pepsb_contract_opt* opt, uint64_t seed_tag,
                              pepsb_boundary** out);
int pepsb_contract_two_layer(pepsb_ctx* ctx, const pepsb_state* bra, const pepsb_state* ket,
                             const pepsb_contract_opt* opt, double* re, double* im);

/* ---- multi-GPU: one process per GPU, an NCCL communicator per
 * context, the bond-sharded row absorb.  NCCL is loaded at run time
 * (libnccl.so.2).  The reference is single-process; these entry
 * points replace contract_two_layer / two_layer_apply_row (contraction.hpp:83-90)
 * for a caller that owns N GPUs.  Collectives run on the library stream. */
/* ncclGetUniqueId: rank 0 calls it and sends the 128 bytes to every rank */
int pepsb_comm_unique_id(unsigned char* id128);
/* ncclCommInitRank on the context's device (collective over the world) */
int pepsb_comm_init(pepsb_ctx* ctx, const unsigned char* id128, int rank, int world);
int pepsb_comm_destroy(pepsb_ctx* ctx);
/* two_layer_apply_row with every column einsumsvd split along the boundary bond
 * across the communicator's ranks; inputs and the emitted boundary replicated */
int pepsb_two_layer_apply_row_sharded(pepsb_ctx* ctx, const pepsb_boundary* top, const pepsb_state* bra,
                                      const pepsb_state* ket, int row, const pepsb_contract_opt* opt,
                                      uint64_t seed_tag, pepsb_boundary** out);
/* contract_two_layer with every row absorb bond-sharded; the scalar on every rank */
int pepsb_contract_two_layer_sharded(pepsb_ctx* ctx, const pepsb_state* bra, const pepsb_state* ket,
                                     const pepsb_contract_opt* opt, double* re, double* im);

/* chain_scalar (mps.hpp:52) */
int pepsb_chain_scalar(pepsb_ctx* ctx, const pepsb_boundary* b, double* re, double* im);

/* build_row_cache (observables.hpp:61) */
int pepsb_build_row_cache(pepsb_ctx* ctx, const pepsb_state* s, const pepsb_contract_opt* opt, pepsb_row_cache** out);
/* flip_vertical (observables.cpp:261-270): rows reversed, up/down swapped */
int pepsb_flip_vertical(pepsb_ctx* ctx, const pepsb_state* s, pepsb_state** out);
/* which 0: tops[k], 1: bots[k] */
int pepsb_row_cache_get(const pepsb_row_cache* c, int which, int k, pepsb_boundary** out);
void pepsb_row_cache_free(pepsb_row_cache* c);

/* band_environment / band_splice / band_value (contraction.hpp:101-125).
 * Insertion pieces (contraction.hpp:95-99): piece i sits at (rc[2i], rc[2i+1]),
 * operator ops[i] (d_out, d_in, bond...), nbonds[i] bond ids taken in order
 * from bond_ids.  top / bottom may be NULL at the lattice edge. */
int pepsb_band_environment(pepsb_ctx* ctx, const pepsb_boundary* top, const pepsb_state* bra, const pepsb_state* ket,
                           int r0, int r1, const pepsb_boundary* bottom, pepsb_band_env** out);
int pepsb_band_splice(pepsb_ctx* ctx, const pepsb_band_env* env, const pepsb_boundary* top, const pepsb_state* bra,
                      const pepsb_state* ket, const pepsb_boundary* bottom, int npieces, const int* rc,
                      pepsb_tensor* const* ops, const int* nbonds, const int* bond_ids, int c0, int c1, double* re,
                      double* im);
int pepsb_band_value(pepsb_ctx* ctx, const pepsb_boundary* top, const pepsb_state* bra, const pepsb_state* ket, int r0,
                     int r1, const pepsb_boundary* bottom, int npieces, const int* rc, pepsb_tensor* const* ops,
                     const int* nbonds, const int* bond_ids, double* re, double* im);
void pepsb_band_env_free(pepsb_band_env* e);

/* PEPS container (save_peps / load_peps, state.hpp, state.cpp:240-299): the
 * reference's binary format ("PEPS2D01", rows, cols, d, axis tag "pudlr", per
 * site order + extents + complex128 data), so the device path reads and
 * writes the reference's own files. */
int pepsb_save_peps(pepsb_ctx* ctx, const pepsb_state* s, const char* path);
int pepsb_load_peps(pepsb_ctx* ctx, const char* path, pepsb_state** out);

/* ---------------------------------------------------------------- one-layer boundary MPS */
/* approx_apply_mpo (mps.hpp / mps.cpp:44-84): zip-up of an MPO (sites (p, d,
 * left, right)) into an MPS (sites (phys, left, right)) of length n with one
 * einsumsvd per site (network {v(adso), s(pst), o(peoq)}, rows "ad", cols
 * "etq", seed derive_seed(seed_base, i)); out_sites receives n new tensors. */
int pepsb_approx_apply_mpo(pepsb_ctx* ctx, int n, pepsb_tensor* const* mps_sites, pepsb_tensor* const* mpo_sites,
                           const pepsb_trunc* policy, int strategy, int absorb, const pepsb_rsvd* rsvd,
                           uint64_t seed_base, pepsb_tensor** out_sites);
/* contract_one_layer (contraction.hpp:67-75, contraction.cpp:178-252) on an
 * order-4 grid (up, left, down, right), row-major sites: family 0 exact
 * (contract_exact with the element budget; ResourceError above it), 1 bmps,
 * 2 ibmps (contract_boundary: seeds derive_seed(seed, 0x10, r)). */
int pepsb_contract_one_layer(pepsb_ctx* ctx, int rows, int cols, pepsb_tensor* const* sites, int family,
                             const pepsb_contract_opt* opt, uint64_t memory_budget, double* re, double* im);

/* expectation (observables.hpp:87-100, observables.cpp:335-422): sum of local
 * terms over <psi|psi>.  Term i: coefficient (coeff[2i], coeff[2i+1]),
 * nsites[i] in {1, 2} at rc[4i .. 4i+3] (row, col[, row, col]), operator
 * ops[i] of shape (d, d) or (d, d, d, d) with outputs first.  Two-site terms are
 * split by SVD (split_two_site, observables.cpp:284-295) and spliced into a
 * band of one or two rows between the cached boundaries.  Errors as the
 * reference: ValidationError for a non-Hermitian observable unless
 * allow_complex, NumericalError for an imaginary part above 1e-8. */
typedef struct {
  pepsb_contract_opt contract;
  int32_t use_cache;           /* default 1 */
  int32_t shared_environments; /* default 0 */
  int32_t allow_complex;       /* default 0 */
} pepsb_expectation_opt;
typedef struct {
  double value, norm_sq;
  double raw_sum[2], complex_value[2];
  uint64_t full_sweeps, band_contractions, flops;
} pepsb_expectation_result;
int pepsb_expectation(pepsb_ctx* ctx, const pepsb_state* s, int nterms, const double* coeff, const int* nsites,
                      const int* rc, pepsb_tensor* const* ops, const pepsb_expectation_opt* opt,
                      pepsb_expectation_result* out);

/* ---------------------------------------------------------------- simple update / ITE (state.hpp:64-76) */
/* hermitian_function(coeff * op, exp(-tau x)) (linalg.hpp:44): the ITE gate rule of drivers.cpp:56-71 */
int pepsb_hermitian_exp(pepsb_ctx* ctx, const pepsb_tensor* op, double coeff, double tau, pepsb_tensor** out);
/* apply_one_site (state.hpp:64-65) on nsites sites (row, col pairs in rc); returns a new state */
int pepsb_apply_one_site(pepsb_ctx* ctx, const pepsb_state* s, const pepsb_tensor* gate, int nsites, const int* rc,
                         pepsb_state** out);
/* apply_two_site (state.hpp:69-70; UpdateStrategy::qr_svd_gram) on nbonds disjoint adjacent bonds
 * (ar, ac, br, bc per bond), batched; policy NULL = {0, 1e-14} (cap d * pre-gate bond) */
int pepsb_apply_two_site(pepsb_ctx* ctx, const pepsb_state* s, const pepsb_tensor* gate, int nbonds,
                         const int* bonds, const pepsb_trunc* policy, pepsb_state** out);
/* TFIM imaginary-time evolution (drivers.cpp:75-98 loop; H = -J sum ZZ - h sum X, colour-ordered terms) */
int pepsb_ite_tfim(pepsb_ctx* ctx, const pepsb_state* s, double J, double h, double tau, int steps, uint64_t rank,
                   pepsb_state** out);

#ifdef __cplusplus
}
#endif

#endif /* PEPS_B200_H */

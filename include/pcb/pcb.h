/* pcop-b200 — C ABI of the B200-native product-convolution apply path.
 *
 * Drop-in boundary for the reference's assembled operator
 * pcop::ProductConvolutionOperator (reference: proj/core/include/pcop/
 * pc_operator.hpp:17-66).  Plain pointers and sizes only; no C++ or torch
 * types.  Each entry point names the reference interface it replaces.
 *
 * Conventions kept from the reference:
 *   - vectors are in domain lexicographic order, last axis fastest
 *     (grid_function.hpp:11-13); batches are vector-major B x N;
 *   - boxes are inclusive int64 [lo, hi] per axis (box.hpp:22-30);
 *   - a grid function reads 0 outside its stored box (grid_function.hpp:41-43);
 *   - shape / domain violations -> PCB_EINVAL, with the reference's
 *     std::invalid_argument message text in pcb_last_error()
 *     (pc_operator.cpp:34-37,46,59-60,86,101);
 *   - the operator is immutable after pcb_create; calls on one handle are
 *     serialized internally, so concurrent callers are safe
 *     (pc_operator.hpp:15-16).
 * There is no CPU fallback: every compute entry point runs sm_100a kernels
 * and fails with PCB_ECUDA when no suitable device is present.
 */
#ifndef PCB_PCB_H
#define PCB_PCB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define PCB_API __attribute__((visibility("default")))
#else
#define PCB_API
#endif

typedef enum pcb_status {
    PCB_OK = 0,
    PCB_EINVAL = 1,    /* std::invalid_argument in the reference */
    PCB_ENOMEM = 2,
    PCB_ECUDA = 3,     /* CUDA runtime / launch failure, or no sm_100 device */
    PCB_ENCCL = 4,
    PCB_EINTERNAL = 5
} pcb_status;

typedef enum pcb_mode {
    PCB_MODE_AUTO = 0,   /* pick by the cost model (pcb_get_info reports the choice) */
    PCB_MODE_GLOBAL = 1, /* common FFT grid over Omega, sum_k Phi_k . FFT(w_k f) accumulated in
                            frequency space, one inverse FFT per vector */
    PCB_MODE_LOCAL = 2   /* per-term FFT grid on the support-trimmed kernel box (the reference's own
                            per-term padding rule, fft.cpp:64-70, on the nonzero box of phi_k^E) */
} pcb_mode;

typedef struct pcb_op pcb_op;

/* Shard-by-k combine: how the ranks' partial outputs are summed when the handle
 * has a communicator (pcb_options.nccl_id). */
typedef enum pcb_reduce {
    PCB_REDUCE_NONE = 0, /* no combine: apply returns this shard's partial sum */
    PCB_REDUCE_ALL = 1,  /* ncclAllReduce: every rank gets the full apply */
    PCB_REDUCE_ROOT = 2  /* ncclReduce: shard 0 gets the full apply (others keep their partial) */
} pcb_reduce;

/* How the active terms are split into contiguous shards. */
typedef enum pcb_partition {
    PCB_PARTITION_COST = 0, /* balanced by the planner's modelled per-term cost (default) */
    PCB_PARTITION_COUNT = 1 /* balanced by term count */
} pcb_partition;

typedef struct pcb_options {
    int32_t device;        /* CUDA device ordinal; -1 = current device */
    int32_t mode;          /* pcb_mode */
    int32_t max_batch;     /* vectors per internal pass; 0 = default (16) */
    int32_t shard_rank;    /* shard-by-k: this process owns terms of shard_rank ... */
    int32_t shard_count;   /* ... out of shard_count (1 = unsharded) */
    int32_t reduce;        /* pcb_reduce: the combine done inside every apply when nccl_id is set */
    int64_t scratch_bytes; /* scratch budget for pipelined passes; 0 = default */
    /* 128-byte ncclUniqueId (pcb_comm_unique_id on one rank, sent to the others by the caller).
     * With it, pcb_create joins an NCCL communicator of shard_count ranks (collective: every shard
     * calls pcb_create with the same id) and every apply / adjoint / estimator call becomes
     * collective, combining the shards' partials as `reduce` says over NVLink, pipelined with the
     * kernels of the next vector chunk.  NULL: no communicator; apply returns the partial. */
    const void* nccl_id;
    int32_t partition;     /* pcb_partition */
    int32_t host_sub_mb;   /* host-buffer calls: MiB per pipelined H2D / kernels / D2H sub-batch; 0 = 16 */
} pcb_options;

typedef struct pcb_info {
    int32_t dim;
    int32_t rank;           /* r, number of terms */
    int32_t rank_active;    /* terms with a nonzero kernel window owned by this shard */
    int32_t mode;           /* resolved pcb_mode */
    int32_t n_groups;       /* distinct FFT shapes */
    int32_t fft_size[3];    /* FFT shape of the largest group */
    int64_t n_points;       /* N */
    int64_t spectra_bytes;  /* device bytes of stored half spectra Phi_k */
    int64_t device_bytes;   /* all device memory held by the handle */
    double bytes_per_vector;  /* algorithmic HBM bytes per applied vector (spectra read once + f,g) */
    double flops_per_vector;  /* nominal fp64 flops per applied vector */
    int32_t launches_per_batch; /* kernels launched by one apply batch call */
    int32_t n_row_families; /* LOCAL apply: shared row-transform families (separable weights), 0: none */
    /* per applied vector, per kernel family {rows_fwd, mid, cols, rows_inv}: the bytes the kernel
     * must read and write once (its inputs and outputs in this pipeline) and nominal fp64 flops
     * (2.5 P log2 P per real line, 5 P log2 P per complex line, 8 per complex MAC) */
    double kernel_bytes[4];
    double kernel_flops[4];
    int32_t n_column_chains; /* 2-D LOCAL apply: column chains (terms sharing one axis-0 inverse) */
    int32_t n_chained_terms; /* terms in chains of two or more */
    int32_t shard_rank, shard_count;
    int32_t comm_nranks;     /* ranks of the handle's NCCL communicator (0: none) */
    int32_t comm_version;    /* NCCL version code of the loaded library (0: none) */
    int32_t term_lo, term_hi; /* this shard owns the active terms with index in [term_lo, term_hi) (reference k) */
    double shard_cost;       /* modelled cost of this shard's terms (s, at the planner's roofs) */
    double total_cost;       /* modelled cost of all active terms */
    double model_ms_local;   /* planner's modelled time per vector of this shard, LOCAL plan */
    double model_ms_global;  /* ... GLOBAL plan */
    int32_t plan_terms;      /* terms the FFT plan runs: the owned terms, with split terms replaced by their pieces */
    int32_t split_terms;     /* owned terms whose linear convolution exceeds one 4096-point line, split into pieces */
} pcb_info;

PCB_API void pcb_default_options(pcb_options* opt);

/* A fresh 128-byte ncclUniqueId for pcb_options.nccl_id (call on one rank; NCCL is dlopen'ed at
 * run time, PCB_ENCCL when it is absent). */
PCB_API pcb_status pcb_comm_unique_id(void* id128);

/* The planner's shard partition, host only (no device needed; the same inputs as pcb_create):
 * owner[k] = the shard that owns term k (-1: inactive -- no footprint in the domain or an all-zero
 * kernel window), cost[k] = its modelled cost (s per vector); either may be NULL.  pcb_create with
 * shard_rank = s keeps exactly the terms with owner[k] == s. */
PCB_API pcb_status pcb_plan_shards(int32_t dim, const int64_t* dom_lo, const int64_t* dom_hi, int32_t r,
                                   const int64_t* w_lo, const int64_t* w_hi, const double* const* w_vals,
                                   const int64_t* phi_lo, const int64_t* phi_hi, const double* const* phi_vals,
                                   int32_t shard_count, int32_t partition, int32_t* owner, double* cost);
PCB_API const char* pcb_last_error(void);

/* Replaces ProductConvolutionOperator(domain, grid, weights, impulses)
 * (pc_operator.hpp:20-22, pc_operator.cpp:26-38).  Term k: weight w_k on box
 * [w_lo+k*dim, w_hi+k*dim] with values w_vals[k] (lexicographic), extended
 * impulse phi_k^E on [phi_lo+k*dim, phi_hi+k*dim] with values phi_vals[k].
 * points (r*dim, may be NULL) are the sample points p_k (informational).
 * All host inputs are copied; the caller may free them on return.  Builds the
 * spectra (K1) before returning. */
PCB_API pcb_status pcb_create(int32_t dim, const int64_t* dom_lo, const int64_t* dom_hi, int32_t r,
                              const int64_t* points, const int64_t* w_lo, const int64_t* w_hi,
                              const double* const* w_vals, const int64_t* phi_lo, const int64_t* phi_hi,
                              const double* const* phi_vals, const pcb_options* opt, pcb_op** out);
/* Single-process multi-GPU (SURVEY 8(e) from one process, as the reference's own callers are):
 * one handle over ndev devices, shard s (the planner's cost-balanced block s of ndev) on
 * devices[s].  Apply / adjoint / estimator calls take buffers on devices[0] (or host buffers); F
 * reaches the other devices by a scatter + all-gather of peer copies, each shard computes its
 * partial on its own device, and the partials are summed by the library's own reduction kernel
 * (slice s summed on devices[s] from peer loads, stored into G over NVLink; shard order,
 * deterministic).  Entries / blocks are served by shard 0 (every shard holds all the terms for
 * them).  devices may repeat (several shards on one GPU).  No nccl_id in opt. */
PCB_API pcb_status pcb_create_multi(int32_t dim, const int64_t* dom_lo, const int64_t* dom_hi, int32_t r,
                                    const int64_t* points, const int64_t* w_lo, const int64_t* w_hi,
                                    const double* const* w_vals, const int64_t* phi_lo, const int64_t* phi_hi,
                                    const double* const* phi_vals, const pcb_options* opt, const int32_t* devices,
                                    int32_t ndev, pcb_op** out);
PCB_API pcb_status pcb_destroy(pcb_op* op);
PCB_API pcb_status pcb_get_info(const pcb_op* op, pcb_info* info);

/* Replaces ProductConvolutionOperator::apply (pc_operator.cpp:45-56), batched
 * (the reference's closest analogue is fft_convolve_batch, fft.cpp:164-181).
 * F, G: host, B x N.  apply = B == 1. */
PCB_API pcb_status pcb_apply_batch(pcb_op* op, int32_t B, const double* F, double* G);
/* Replaces ProductConvolutionOperator::apply_adjoint (pc_operator.cpp:58-69). */
PCB_API pcb_status pcb_apply_adjoint_batch(pcb_op* op, int32_t B, const double* F, double* G);
/* Device-pointer variants: dF, dG on the handle's device, ordered on `stream`
 * (a cudaStream_t; NULL = legacy default stream). */
PCB_API pcb_status pcb_apply_batch_dev(pcb_op* op, int32_t B, const double* dF, double* dG, void* stream);
PCB_API pcb_status pcb_apply_adjoint_batch_dev(pcb_op* op, int32_t B, const double* dF, double* dG,
                                               void* stream);

/* Replaces ProductConvolutionOperator::entry (pc_operator.cpp:84-96) for cnt
 * (y, x) pairs (y, x: cnt*dim host int64).  Bit-identical to the reference's
 * summation. */
PCB_API pcb_status pcb_entries(pcb_op* op, int64_t cnt, const int64_t* y, const int64_t* x, double* out);
/* Dense blocks for H-matrix conversion (reference caller: dense_block,
 * hmatrix.cpp:138-150): block b has rows t_origin[b] + [0, block_shape) and
 * cols s_origin[b] + [0, block_shape) (points lexicographic);
 * out[b][i][j] row-major, nblk * prod(block_shape)^2 doubles. */
PCB_API pcb_status pcb_blocks(pcb_op* op, int32_t nblk, const int64_t* t_origin, const int64_t* s_origin,
                              const int64_t* block_shape, double* out);
PCB_API pcb_status pcb_blocks_dev(pcb_op* op, int32_t nblk, const int64_t* d_t_origin,
                                  const int64_t* d_s_origin, const int64_t* block_shape, double* d_out,
                                  void* stream);

/* Replaces ProductConvolutionOperator::apply_block (pc_operator.cpp:98-130), batched over nblk
 * (T, S) box pairs (each box inclusive, inside the domain): apply g_b = Atilde[T_b, S_b] f_b, or
 * with adjoint != 0, g_b = (Atilde^*)[T_b, S_b] f_b.  f packs each f_b on S_b (lexicographic)
 * back to back, g packs each g_b on T_b.  Small blocks use the exact entry gather fused with the
 * block matvec; blocks with |T||S| > 2^24 use the FFT apply of f_b extended by zero, cropped. */
PCB_API pcb_status pcb_apply_block(pcb_op* op, int32_t nblk, const int64_t* t_lo, const int64_t* t_hi,
                                   const int64_t* s_lo, const int64_t* s_hi, const double* f, double* g,
                                   int32_t adjoint);

/* Randomized a-posteriori estimator (adaptivity.cpp:75-121): Ytilde_i =
 * Atilde^* zeta_i for q probes Z (q x N), eta_abs = sqrt(sum ||Ytilde-Y||^2/q),
 * eta_rel = ||Ytilde-Y||_F / ||Y||_F, eta_cells[c] over leaf box c.  ytilde
 * may be NULL.  Host pointers. */
PCB_API pcb_status pcb_probe_estimate(pcb_op* op, int32_t q, const double* Z, const double* Y, int32_t nleaf,
                                      const int64_t* leaf_lo, const int64_t* leaf_hi, double* ytilde,
                                      double* eta_cells, double* eta_abs, double* eta_rel);
/* Device variant: dZ, dY, dYt (q x N, dYt required) on device; results to host. */
PCB_API pcb_status pcb_probe_estimate_dev(pcb_op* op, int32_t q, const double* dZ, const double* dY, double* dYt,
                                          int32_t nleaf, const int64_t* leaf_lo, const int64_t* leaf_hi,
                                          double* eta_cells, double* eta_abs, double* eta_rel, void* stream);

/* True operator of the benchmark configurations (reference roles:
 * compute_impulse impulse.cpp:5-15 and make_probes' Y = A^* Z adaptivity.cpp:14-28):
 *   A[y,x] = exp(-sum_a (y_a-x_a)^2 / (2 s_a(x)^2)) / Z(x) on sum_a ((y_a-x_a)/s_a(x))^2 <= 16,
 * domain [0, n_a) per axis, per-source widths sigma (N x dim), Z(x) = the full-lattice sum of the
 * truncated kernel (computed on the device at create).  Direct fp64 stencils. */
typedef struct pcb_blur pcb_blur;
PCB_API pcb_status pcb_blur_create(int32_t dim, const int64_t* n, const double* sigma, pcb_blur** out);
PCB_API pcb_status pcb_blur_destroy(pcb_blur* blur);
/* B vectors (B x N); adjoint != 0 applies A^*.  device_ptrs != 0: F, G on the device, ordered on
 * `stream`; otherwise host pointers (synchronous). */
PCB_API pcb_status pcb_blur_apply(pcb_blur* blur, int32_t B, const double* F, double* G, int32_t adjoint,
                                  int32_t device_ptrs, void* stream);
PCB_API const char* pcb_blur_last_error(void);

/* GPU-resident a-posteriori estimator state (adaptivity.hpp:14-56):
 *   pcb_estimator_create    make_probes' Z: q probes of mt19937_64(seed) via std::normal_distribution,
 *                           probe i = draws [iN, (i+1)N) (adaptivity.cpp:14-28); device-resident
 *   pcb_estimator_set_y     Y = A^* Z from the caller (host or device pointer), or
 *   pcb_estimator_set_y_blur   computed on the device by a pcb_blur true operator;
 *                           ||Y||_F as make_estimator_state (adaptivity.cpp:30-37)
 *   pcb_estimator_update    update_samples (adaptivity.cpp:75-112) incl. its changed_ks checks:
 *                           Ytilde = Atilde^* Z, eta_abs = sqrt(||Ytilde - Y||^2 / q), eta_rel
 *   pcb_estimator_cells     eta_for_cells (adaptivity.cpp:114-121) over inclusive leaf boxes
 *   pcb_estimator_probes    the device pointers of Z, Y, Ytilde (q x N each)
 *   pcb_estimator_read      copies Z / Y / Ytilde to the host (any may be NULL) */
typedef struct pcb_estimator pcb_estimator;
PCB_API pcb_status pcb_estimator_create(int32_t dim, const int64_t* dom_lo, const int64_t* dom_hi, int32_t q,
                                        uint64_t seed, int32_t device, pcb_estimator** out);
/* Probe generators: the reference's mt19937_64 + normal_distribution stream (drawn on the host,
 * sequential: ~1 s for c3's 64 probes) or counter-based Philox4x32-10 + Box-Muller drawn on the
 * device (throughput runs; SURVEY 8(d) allows it when Z is read back for a parity check). */
typedef enum pcb_rng { PCB_RNG_MT19937 = 0, PCB_RNG_PHILOX = 1 } pcb_rng;
PCB_API pcb_status pcb_estimator_create_ex(int32_t dim, const int64_t* dom_lo, const int64_t* dom_hi, int32_t q,
                                           uint64_t seed, int32_t device, int32_t generator, pcb_estimator** out);
PCB_API pcb_status pcb_estimator_destroy(pcb_estimator* est);
PCB_API pcb_status pcb_estimator_probes(pcb_estimator* est, double** dZ, double** dY, double** dYtilde);
PCB_API pcb_status pcb_estimator_set_y(pcb_estimator* est, const double* Y, int32_t device_ptr);
PCB_API pcb_status pcb_estimator_set_y_blur(pcb_estimator* est, pcb_blur* blur);
PCB_API pcb_status pcb_estimator_update(pcb_estimator* est, pcb_op* op, int32_t nchanged, const int32_t* changed_ks,
                                        double* eta_abs, double* eta_rel);
PCB_API pcb_status pcb_estimator_cells(pcb_estimator* est, int32_t nleaf, const int64_t* leaf_lo,
                                       const int64_t* leaf_hi, double* eta_cells);
PCB_API pcb_status pcb_estimator_read(pcb_estimator* est, double* Z, double* Y, double* Ytilde);

/* Domain of an operator (inclusive box, dim entries each). */
PCB_API pcb_status pcb_get_domain(const pcb_op* op, int64_t* dom_lo, int64_t* dom_hi);

/* H-matrix assembly over the GPU operator and the PCHM container (reference
 * hmatrix.hpp:13-103, hmatrix.cpp):
 *   pcb_cluster_tree        ClusterTree::build (hmatrix.cpp:40-76) alone (no blocks)
 *   pcb_hmatrix_assemble    assemble_hmatrix (:338-377): tree, admissible partition, dense leaves
 *                           from batched GPU entries, low-rank blocks by the randomized range
 *                           finder over batched GPU apply_block (:152-234) or by adaptive cross
 *                           approximation over batched GPU entries (:236-318)
 *   pcb_hmatrix_compress    compress_block (:320-336) for listed (t, s) node pairs, appended as
 *                           low-rank blocks
 *   pcb_hmatrix_matvec      HMatrix::matvec (:379-400), host; pcb_hmatrix_matvec_batch: on the GPU
 *   pcb_hmatrix_save/_load  the little-endian "PCHM" v1 container, byte-compatible with the
 *                           reference's save_hmatrix / load_hmatrix (:433-526)
 *   pcb_hmatrix_tree / _block / _admissible / _get_info   inspection */
typedef struct pcb_hmatrix pcb_hmatrix;
typedef enum pcb_hm_method { PCB_HM_RANDOMIZED = 0, PCB_HM_CUR = 1 } pcb_hm_method;
typedef struct pcb_hmatrix_info {
    int32_t dim;
    int32_t leaf_cap;
    int64_t n_points;
    int64_t n_nodes;
    int64_t n_blocks;
    int64_t n_low_rank;
    int64_t n_dense;
    int64_t max_rank;
    int64_t stored_doubles;
    int32_t any_rank_capped;
    int32_t method;
    double tol;
    int32_t fixed_rank;
    int32_t reserved;
} pcb_hmatrix_info;
PCB_API pcb_status pcb_cluster_tree(int32_t dim, const int64_t* dom_lo, const int64_t* dom_hi, int32_t leaf_cap,
                                    pcb_hmatrix** out);
PCB_API pcb_status pcb_hmatrix_assemble(pcb_op* op, double tol, int32_t leaf_cap, int32_t method, int32_t fixed_rank,
                                        pcb_hmatrix** out);
PCB_API pcb_status pcb_hmatrix_compress(pcb_op* op, pcb_hmatrix* h, int32_t nblk, const int32_t* t_nodes,
                                        const int32_t* s_nodes, int32_t method, double tol, int32_t fixed_rank);
PCB_API pcb_status pcb_hmatrix_destroy(pcb_hmatrix* h);
PCB_API pcb_status pcb_hmatrix_get_info(pcb_hmatrix* h, pcb_hmatrix_info* info);
/* perm (N), node_range (2 per node: begin, end), node_links (3 per node: split_axis, child_lo,
 * child_hi), node_bbox (2*dim per node: lo..., hi...); any may be NULL */
PCB_API pcb_status pcb_hmatrix_tree(pcb_hmatrix* h, int64_t* perm, int64_t* node_range, int32_t* node_links,
                                    int64_t* node_bbox);
/* block i: t_s_kind = {t_node, s_node, 0 low rank | 1 dense}, rows_cols_rank = {|T|, |S|, rank};
 * B (|T| x rank), C (rank x |S|) or dense (|T| x |S|), row-major; any may be NULL */
PCB_API pcb_status pcb_hmatrix_block(pcb_hmatrix* h, int64_t i, int32_t* t_s_kind, int64_t* rows_cols_rank, double* B,
                                     double* C, double* dense);
PCB_API pcb_status pcb_hmatrix_admissible(pcb_hmatrix* h, int32_t t, int32_t s, int32_t* adm, double* dist,
                                          double* diam_t, double* diam_s);
PCB_API pcb_status pcb_hmatrix_matvec(pcb_hmatrix* h, const double* f, double* g);
/* The same product for B vectors (B x N, vector-major) on GPU `device`: the blocks are copied to the
 * device on the first call; every row's dot product and the sum over the blocks covering a row keep
 * the host loop's order (IEEE mul / add), so each vector equals pcb_hmatrix_matvec bit for bit. */
PCB_API pcb_status pcb_hmatrix_matvec_batch(pcb_hmatrix* h, int32_t device, int32_t B, const double* F, double* G);
PCB_API pcb_status pcb_hmatrix_save(pcb_hmatrix* h, const char* path);
PCB_API pcb_status pcb_hmatrix_load(const char* path, pcb_hmatrix** out);

/* Debug: with PCB_GUARD=1 in the environment every device allocation of the library carries a
 * 64 KiB canary band before and after it.  Synchronizes the device and counts the guarded
 * allocations alive and the canary bytes that were overwritten (out-of-bounds writes); both are 0
 * without PCB_GUARD. */
PCB_API pcb_status pcb_debug_guard_check(int64_t* n_regions, int64_t* n_bad_bytes);

/* Page-locked host memory for the host-buffer calls: F and G in pinned memory go straight to the
 * copy engines (c3: 5.5k vectors/s end to end), pageable buffers are staged through the handle's
 * pinned bounce slots by host threads (~2.8k vectors/s, host-memory-bound).  pcb::pinned_allocator
 * (operator.hpp) wraps these for std::vector. */
PCB_API pcb_status pcb_host_alloc(uint64_t bytes, void** out);
PCB_API pcb_status pcb_host_free(void* p);
/* Page-lock a buffer the caller already owns (a std::vector the reference code passes to apply(),
 * operators.cpp:39-49) so later host-buffer calls on it take the copy-engine path too.  Locking costs
 * about as much as a few applies: register buffers that are reused, and unregister them before they
 * are freed.  PCB_EINVAL if the range is already (or, for unregister, not) registered. */
PCB_API pcb_status pcb_host_register(void* p, uint64_t bytes);
PCB_API pcb_status pcb_host_unregister(void* p);

/* Number of kernels this library has launched in the process (all handles). */
PCB_API long long pcb_launch_count(void);

/* Per-kernel timing: between pcb_profile_begin and pcb_profile_end every
 * kernel launch of this handle is bracketed by CUDA events on its launching
 * stream.  pcb_profile_end returns, per kernel name (names: max_kernels x 32
 * chars), the summed event time in ms and the launch count. */
PCB_API pcb_status pcb_profile_begin(pcb_op* op);
PCB_API pcb_status pcb_profile_end(pcb_op* op, int32_t max_kernels, char* names, double* ms_total,
                                   int32_t* launches, int32_t* n_kernels);

/* Host utilities reproducing the reference's random streams (libstdc++):
 * std::mt19937_64(seed) + std::normal_distribution<double>(0,1)
 * (adaptivity.cpp:19-23, test_pc_operator.cpp:13-18) and
 * std::uniform_int_distribution<int64_t>(lo, hi). */
PCB_API pcb_status pcb_normal_fill(uint64_t seed, int64_t count, double* out);
PCB_API pcb_status pcb_uniform_int_fill(uint64_t seed, int64_t lo, int64_t hi, int64_t count, int64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* PCB_PCB_H */

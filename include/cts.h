/*
 * cts.h -- C ABI of libcts.so, the B200 (sm_100a) batched compressed-LoRA apply.
 *
 * "Compress then Serve" (arXiv 2407.00066).  A collection of LoRA updates B_i A_i is jointly
 * compressed (JD-Full, Eq. 2; clusters Sec. 3.2) into, per
 * module (projection) and per cluster c, two shared bases and, per adapter i, one r x r matrix:
 *     B_i A_i  ~=  U_c Sigma_i V_c^T          (Eq. 1; clustered form P:L164)
 * The serving hot path applies it to a batch of tokens, each naming its adapter ("each user
 * specifies both the input data and the desired LoRA identifier", App D):
 *     y_t  +=  scale * U_c ( Sigma_i ( V_c^T x_t ) )    for token t bound to adapter i in cluster c
 * evaluated right to left as App D prescribes and as the paper's vLLM/Punica wrapper
 * add_lora_slice_with_sigma does in three launches (App F.4).
 *
 * Role names: in_basis = paper V_c (d_in x r), out_basis = paper U_c
 * (d_out x r), sigma[i] = Sigma_i with ROW = out_basis index, COLUMN = in_basis index.
 *
 * Conventions for every entry point:
 *   - Pointers are DEVICE pointers unless the argument says "host".
 *   - Calls taking a cudaStream_t are stream-ordered and asynchronous unless stated otherwise.
 *   - No call throws or aborts; failures return a cts_status_t and enqueue nothing.
 *   - Element types: bf16 = IEEE-like bfloat16 (1-8-7) stored as 16-bit words; int32 little endian.
 *   - All arithmetic on device: bf16 operands, fp32 accumulation, bf16 round-to-nearest-even out.
 *   - Banks are immutable after load (except through cts_bank_write_clusters); several plans/streams
 *     may apply the same bank concurrently.
 */
#ifndef CTS_H_
#define CTS_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CTS_OK = 0,
  CTS_ERR_INVALID_ARGUMENT = 1,   /* null pointer, negative size, aliasing x/y            */
  CTS_ERR_SHAPE = 2,              /* dimension / alignment / leading-dimension violation  */
  CTS_ERR_INDEX_OUT_OF_RANGE = 3, /* token adapter id outside [-1, N) or cluster id >= C  */
  CTS_ERR_UNSUPPORTED = 4,        /* not an sm_100 device, r > 64, C > 1024               */
  CTS_ERR_OUT_OF_MEMORY = 5,
  CTS_ERR_CUDA = 6,               /* a CUDA runtime/driver call failed                    */
  CTS_ERR_NCCL = 7                /* NCCL missing (libnccl.so.2 not loadable) or a call failed */
} cts_status_t;

typedef struct cts_bank_s* cts_bank_t;   /* owns all device copies of a compressed collection */
typedef struct cts_plan_s* cts_plan_t;   /* per-batch segmentation + scratch, reusable        */
typedef struct cts_comm_s* cts_comm_t;   /* NCCL communicator of a tensor-parallel group     */

/* Storage kind of the per-adapter matrices Sigma_i.
 *   CTS_SIGMA_FULL: JD-Full (Eq. 2), Sigma_i an arbitrary r x r matrix.
 *   CTS_SIGMA_DIAG: JD-Diag (Eq. 3), Sigma_i diagonal; only its r diagonal entries are
 *                   stored and applied ("batched matrix multiplications can be completely
 *                   circumvented", App D): t = scale * sigma_i (elementwise) * (V_c^T x). */
typedef enum { CTS_SIGMA_FULL = 0, CTS_SIGMA_DIAG = 1 } cts_sigma_kind_t;

/*
 * A compressed collection for n_modules projections (e.g. 224 = 32 layers x q,k,v,o,gate,up,
 * down of Mistral-7B).  Every module shares N adapters, C clusters and one rank r (one r for all
 * clusters as App F assumes).  The adapter->cluster map is PER
 * MODULE (App F counts "+1" assignment parameter per LoRA per module; reading R9).
 */
typedef struct {
  int32_t n_modules;             /* >= 1                                                       */
  int32_t n_adapters;            /* N >= 1                                                     */
  int32_t n_clusters;            /* C in [1, 1024]                                             */
  int32_t rank;                  /* r in [1, 64]; padded on device to 16/32/64 with zeros      */
  const int32_t* d_in;           /* host [n_modules]; each a positive multiple of 64           */
  const int32_t* d_out;          /* host [n_modules]; each a positive multiple of 64           */
  const void* const* in_basis;   /* host array [n_modules] of -> bf16 [C][d_in][r] row-major   */
  const void* const* out_basis;  /* host array [n_modules] of -> bf16 [C][d_out][r] row-major  */
  const void* const* sigma;      /* host array [n_modules] of -> bf16 [N][r][r], row = out idx;
                                    CTS_SIGMA_DIAG: bf16 [N][r], the diagonals                 */
  const int32_t* const* cluster_of; /* host array [n_modules] of -> int32 [N], values in [0,C) */
  int32_t sources_on_device;     /* 0: the four pointer arrays point to host memory;
                                    1: they point to device memory                             */
  int32_t sigma_kind;            /* cts_sigma_kind_t; 0 (zero-initialised descriptor) = full    */
} cts_bank_desc_t;

/* Copy and re-lay-out a compressed collection into device memory (the resident bank that lets
 * "U and V be pre-loaded onto the GPU").  SYNCHRONOUS: when it returns the sources may be
 * freed.  Layout on device: in_basis [C][r_pad][d_in] (K-major operand of the shrink GEMM),
 * out_basis [C][d_out][r_pad], sigma [N][r_pad][r_pad] (CTS_SIGMA_DIAG: [N][r_pad]), one int32 map
 * per distinct cluster map.
 * Errors: CTS_ERR_INVALID_ARGUMENT (null, unknown sigma_kind), CTS_ERR_SHAPE (dims), CTS_ERR_INDEX_OUT_OF_RANGE
 * (cluster id), CTS_ERR_UNSUPPORTED (device is not sm_100, r > 64, C > 1024), CTS_ERR_OUT_OF_MEMORY.
 * On error *out is set to NULL and nothing stays allocated. */
cts_status_t cts_bank_load(const cts_bank_desc_t* desc, cudaStream_t stream, cts_bank_t* out);

/* Device bytes owned by the bank (bases + Sigma + maps, including the r padding). */
cts_status_t cts_bank_bytes(cts_bank_t bank, size_t* device_bytes);

/* Parameter count of the bank as App F counts it for module m:
 * sum over clusters of (d_in + d_out) * r  +  N * (r^2 + (C > 1 ? 1 : 0)).  Unpadded.
 * CTS_SIGMA_DIAG banks count r instead of r^2 per adapter (JD-Diag, Eq. 3). */
cts_status_t cts_bank_params(cts_bank_t bank, int32_t module, int64_t* params);

/* Overwrite the shared bases of n (<= 64) distinct clusters of module m with new ones -- the
 * page-in of a resident slot pool (the multi-LoRA baseline the paper compares against swaps adapters
 * between host and GPU memory; App F matched-memory slots): with an
 * uncompressed bank (cluster = adapter slot, Sigma = I) this replaces the LoRAs held in those slots.
 * in_basis: DEVICE bf16 [n][d_in][r] and out_basis: DEVICE bf16 [n][d_out][r] (the cts_bank_desc_t
 * layouts, cluster q's slice q); the caller stages host data itself (e.g. one cudaMemcpyAsync from
 * pinned memory).  Stream-ordered and asynchronous: applies enqueued later on `stream` see the new
 * bases; applies on OTHER streams must not read those clusters concurrently.  Sigma and the
 * adapter->cluster maps are unchanged.  Errors: CTS_ERR_INVALID_ARGUMENT (null, repeated cluster),
 * CTS_ERR_SHAPE (module, n outside [0, 64]), CTS_ERR_INDEX_OUT_OF_RANGE (cluster outside [0, C)). */
cts_status_t cts_bank_write_clusters(cts_bank_t bank, int32_t module, int32_t n, const int32_t* clusters,
                                     const void* in_basis, const void* out_basis, cudaStream_t stream);

/* Release all device memory of the bank.  The caller must ensure no apply still uses it. */
cts_status_t cts_bank_free(cts_bank_t bank);

/* Per-batch state for batches of up to T_max tokens: a device copy of the token->adapter map,
 * per distinct cluster map a stable permutation, offsets and a 128-token tile list, an error
 * word, and the per-module rank-r intermediate scratch.  Errors: CTS_ERR_INVALID_ARGUMENT, OUT_OF_MEMORY. */
cts_status_t cts_plan_create(cts_bank_t bank, int32_t T_max, cts_plan_t* out);
cts_status_t cts_plan_free(cts_plan_t plan);

/* Upper bound on the tile count of any module for a batch of T tokens: ceil(T/128) + min(C, T). */
int32_t cts_plan_max_tiles(cts_plan_t plan, int32_t T);

/* Segment a batch by cluster, for every distinct cluster map, in ONE launch.
 * token_adapter: device int32 [T]; -1 = no adapter (row of y left bit-identical), otherwise an
 * adapter id in [0, N).  For each map: tc[t] = cluster_of[token_adapter[t]], perm = bound tokens
 * stably sorted by (cluster, token index), offset = exclusive prefix sum of counts, tiles =
 * (c, start, len <= 128).  Integer work, bit-exact vs oracle.segment_ref; deterministic.
 * The kernel copies token_adapter into the plan, so the caller may reuse its buffer afterwards.
 * Device-side validation: an id outside [-1, N) records {CTS_ERR_INDEX_OUT_OF_RANGE, smallest
 * offending t} in the plan's error word and poisons the plan: every later cts_apply on it leaves y
 * untouched until the next successful cts_segment.  Host errors: CTS_ERR_INVALID_ARGUMENT
 * (null, T < 0), CTS_ERR_SHAPE (T > T_max). */
cts_status_t cts_segment(cts_plan_t plan, const int32_t* token_adapter, int32_t T,
                         cudaStream_t stream);

/* Test hook: copy module m's segmentation to HOST buffers after the segment completed.
 * perm: host int32 [T] (entries past the bound count are unspecified), offsets: host int32
 * [C+1], tiles: host int32 [max_tiles*3] as (cluster, start, len) rows -- the logical 128-token
 * tiles in cluster order (on device they are packed two-per-slot when <= 64 tokens), n_tiles:
 * host int32 count of those tiles.
 * Any output pointer may be NULL.  Synchronizes the stream. */
cts_status_t cts_segment_readback(cts_plan_t plan, int32_t module, int32_t* perm, int32_t* offsets,
                                  int32_t* tiles, int32_t* n_tiles, cudaStream_t stream);

/* The compressed apply for one module on the last segmented batch (T tokens):
 *     y[t, :] = bf16_rne( y[t, :] + scale * U_c (Sigma_i (V_c^T x[t, :])) )  for bound tokens t
 * x: bf16 [T][ld_x] (first d_in columns used), y: bf16 [T][ld_y] read and written IN PLACE (the
 * base projection output, Punica's in-place slice update P:L1118).  scale (fp32) multiplies the
 * rank-r intermediate before the expand.  Rows of unbound tokens are not touched.  An empty batch
 * (T = 0) is a no-op and may pass NULL x / y (also for cts_apply_group and cts_project).
 * One persistent launch (one CTA per SM; apply_fused.cuh): shrink + Sigma (tcgen05 GEMM over
 * 128-token cluster slots, split-K chunks reduced in a fixed order by the last-arriving CTA,
 * per-token Sigma_i matvec in its epilogue), then expand + residual (tcgen05, y rows moved by TMA)
 * as each slot's rank-r intermediate is published (CTS_FUSED=0: the two as separate launches).
 * Progress of the single launch relies on its CTAs (at most one per SM) being co-resident: expand
 * work waits on flags that other CTAs' shrink work publishes.  The launch is therefore COOPERATIVE
 * (the runtime starts it only when every CTA can be resident), so concurrent applies on other
 * streams cannot deadlock it; see cts_set_exclusive_device for the non-cooperative variant.
 * Deterministic (no float atomics; the reduction order does not depend on scheduling).
 * Host validation: CTS_ERR_INVALID_ARGUMENT (null, x/y overlap), CTS_ERR_SHAPE (module index,
 * ld_x < d_in, ld_y < d_out, ld or pointer not 16-byte aligned). */
cts_status_t cts_apply(cts_plan_t plan, int32_t module, const void* x, int64_t ld_x, void* y,
                       int64_t ld_y, float scale, cudaStream_t stream);

/* The two halves of cts_apply, for callers that schedule them separately (e.g. to time each
 * kernel, or to overlap the expand of one module with the shrink of the next):
 *   cts_shrink: kernel 1 -- t = scale * Sigma_i V_c^T x_t for every bound token, into the plan's
 *               per-module rank-r scratch (bf16 hi + lo pair per element).
 *   cts_expand: kernel 2 -- y_t = bf16_rne(y_t + U_c t_t), consuming the scratch that the last
 *               cts_shrink of the SAME module on this plan (after the last cts_segment) produced.
 * Same arguments, validation and errors as cts_apply (minus the x/y overlap check). */
cts_status_t cts_shrink(cts_plan_t plan, int32_t module, const void* x, int64_t ld_x, float scale,
                        cudaStream_t stream);
cts_status_t cts_expand(cts_plan_t plan, int32_t module, void* y, int64_t ld_y, cudaStream_t stream);

/* Grouped forms: ONE launch per kernel covers n (1..16) distinct modules, e.g. the q, k, v
 * projections of a layer (which may share one x) or gate and up.  modules: host int32 [n];
 * xs / ys: host arrays [n] of device pointers; ld_x / ld_y: host int64 [n] (elements).  Each module
 * behaves exactly as its own cts_apply; the work items of all modules are spread over the SMs of
 * one persistent grid.  Errors as cts_apply, plus CTS_ERR_SHAPE for n > 16 and
 * CTS_ERR_INVALID_ARGUMENT for a repeated module or a y overlapping any x or another y. */
cts_status_t cts_apply_group(cts_plan_t plan, int32_t n, const int32_t* modules, const void* const* xs,
                             const int64_t* ld_x, void* const* ys, const int64_t* ld_y, float scale,
                             cudaStream_t stream);
cts_status_t cts_shrink_group(cts_plan_t plan, int32_t n, const int32_t* modules, const void* const* xs,
                              const int64_t* ld_x, float scale, cudaStream_t stream);
cts_status_t cts_expand_group(cts_plan_t plan, int32_t n, const int32_t* modules, void* const* ys,
                              const int64_t* ld_y, cudaStream_t stream);

/*
 * Tensor-parallel d-split (north_star: "an optional tensor-parallel split along
 * d_model whose rank-r intermediate is all-reduced with NCCL over NVLink").  With G ranks, rank g
 * loads a bank whose in_basis holds columns [g*d_in/G, (g+1)*d_in/G) of every V_c and whose
 * out_basis holds rows [g*d_out/G, (g+1)*d_out/G) of every U_c; Sigma and the maps are replicated
 * and every rank segments the SAME token batch.  Because Sigma_i is linear,
 *     t = scale * Sigma_i V_c^T x = sum_g scale * Sigma_i V_c[g]^T x[g]          (Eq. 1)
 * so each rank computes its partial t_g, the caller sums the partials over ranks (all-reduce), and
 * each rank adds U_c[g] t to its d_out slice of y.
 *
 * cts_plan_partial_elems: *elems = fp32 elements of one module's partial buffer, T_max * r_pad:
 *   row t (r_pad floats, zero-padded rank) is token t's partial; rows of unbound tokens and rows
 *   t >= T are neither written nor read, so only the first T * r_pad floats need the all-reduce.
 * cts_shrink_partial_group: like cts_shrink_group (x = this rank's d_in slice, ld_x its row stride)
 *   but writes t_g as fp32 into parts[i] (device, caller-owned, 16-byte aligned, >= elems floats).
 * cts_expand_reduced_group: parts[i] = the summed partials (same layout); splits them into the
 *   bf16 hi+lo pair of R12 (one launch for the group) and runs the expand + residual add on this
 *   rank's d_out slice of y (one launch).
 * Errors as cts_shrink_group / cts_expand_group; CTS_ERR_INVALID_ARGUMENT for a null or misaligned
 * part.  Every rank must pass the same modules in the same order.
 */
cts_status_t cts_plan_partial_elems(cts_plan_t plan, int64_t* elems);
cts_status_t cts_shrink_partial_group(cts_plan_t plan, int32_t n, const int32_t* modules, const void* const* xs,
                                      const int64_t* ld_x, float scale, float* const* parts, cudaStream_t stream);
cts_status_t cts_expand_reduced_group(cts_plan_t plan, int32_t n, const int32_t* modules, const float* const* parts,
                                      void* const* ys, const int64_t* ld_y, cudaStream_t stream);

/*
 * Tensor-parallel apply with the collective inside the library (cts_comm_create,
 * cts_apply_tp; north_star: "the rank-r intermediate is all-reduced with NCCL over NVLink").
 * NCCL is loaded at run time (dlopen of libnccl.so.2 -- the copy torch already loaded, if any), so
 * libcts itself has no link-time NCCL dependency; without NCCL these calls return CTS_ERR_NCCL.
 * cts_comm_unique_id: id_out = 128 host bytes (ncclGetUniqueId); one rank calls it and the caller
 *   distributes the bytes to every rank (e.g. a torch.distributed broadcast).
 * cts_comm_create: every rank of the group, with the same id, nranks >= 1 and its rank in
 *   [0, nranks); binds to the current CUDA device (ncclCommInitRank, blocking until all ranks join).
 *   Errors: CTS_ERR_INVALID_ARGUMENT (null, bad rank), CTS_ERR_NCCL.
 * cts_apply_tp: the TP d-split of cts_apply_group for this rank's shard (bank holding d_in / d_out
 *   slice `rank`, see cts_shrink_partial_group), the same segmented batch on every rank:
 *     1. shrink on the d_in shard -> fp32 partial t_g in plan-owned buffers (one launch)
 *     2. ncclAllReduce(sum, fp32, T * r_pad) of each module's partial, in one NCCL group, on `stream`
 *     3. hi / lo split + expand + residual add into this rank's d_out slice of y (two launches)
 *   Sums the ranks' partials, so the result equals the unsharded apply up to fp32 reassociation
 *   (Sigma linear, Eq. 1).  Stream-ordered and CUDA-graph capturable (NCCL supports
 *   capture).  Errors as cts_apply_group plus CTS_ERR_NCCL; every rank must pass the same modules.
 * cts_comm_free: destroys the communicator (no apply may still use it).
 */
cts_status_t cts_comm_unique_id(void* id_out);
cts_status_t cts_comm_create(const void* nccl_unique_id, int32_t nranks, int32_t rank, cts_comm_t* out);
cts_status_t cts_comm_free(cts_comm_t comm);
cts_status_t cts_apply_tp(cts_plan_t plan, int32_t n, const int32_t* modules, const void* const* xs,
                          const int64_t* ld_x, void* const* ys, const int64_t* ld_y, float scale, cts_comm_t comm,
                          cudaStream_t stream);

/*
 * Fused base + compressed-LoRA projection: for every token t of the batch
 * segmented into `plan` (all T tokens, bound or not),
 *     y[t] = bf16( W0 x[t] + scale * U_c Sigma_i V_c^T x[t] )        (Sec. 3 P:L107-109 with
 *                                                                       Eq. 1)
 * with the LoRA term omitted for tokens whose id is -1.  W0 = w0: device, bf16, [d_out][ld_w] row
 * major (the nn.Linear weight layout: row o is output feature o), ld_w >= d_in.  x: [T][ld_x] bf16.
 * y: [T][ld_y] bf16, OUTPUT ONLY (overwritten; unlike cts_apply it is not read).  Two launches:
 * the shrink + Sigma kernel (t into the plan), then one persistent tcgen05 GEMM whose 128-row
 * tiles are the cluster-sorted slots (and base-only tiles of the unbound tokens) and whose last
 * pipeline stage adds t U_c^T into the same TMEM accumulator.  Requires r_pad == 16 (rank <= 16),
 * d_out % 256 == 0 and d_in % 64 == 0 (else CTS_ERR_UNSUPPORTED); ld/alignment as cts_apply;
 * CTS_ERR_INVALID_ARGUMENT if y overlaps x or w0.  A poisoned plan leaves y untouched.
 * Stream-ordered; x, w0 and y must stay valid until the stream reaches the call.
 */
cts_status_t cts_project(cts_plan_t plan, int32_t module, const void* x, int64_t ld_x, const void* w0, int64_t ld_w,
                         void* y, int64_t ld_y, float scale, cudaStream_t stream);

/*
 * GPU compression: the joint diagonalization of each cluster's LoRAs by the
 * paper's "Additional Eigenvalue Iteration Algorithm" (App A.2), for a batch of
 * independent problems (e.g. every cluster of a module), `iters` iterations of
 *     U0 <- sum_i B_i (A_i V)(V^T A_i^T)(B_i^T U),   V0 <- sum_i A_i^T (B_i^T U)(U^T B_i)(A_i V),
 *     U <- orthogonalize(U0),  V <- orthogonalize(V0)      (reduced QR with diag(R) > 0)
 * then Sigma_i = U^T B_i A_i V (Eq. sigmastar).  All pointers device, fp32, row major:
 *   a_stack  [n*r_i][d_in]   rows r_i*i .. r_i*i + r_i - 1 = A_i          (the LoRA "A" factors)
 *   bt_stack [n*r_i][d_out]  rows r_i*i + j = column j of B_i (B_i^T)      (the LoRA "B" factors)
 *   U [d_out][r], V [d_in][r]: IN the initial bases (orthonormal columns; the paper fixes no
 *                 initialization), OUT the result (U = out_basis, V = in_basis of the bank)
 *   sigma [n][r][r]: OUT, row = out index (the bank's Sigma layout before bf16 rounding)
 * r in {8, 16, 32, 64} (else CTS_ERR_UNSUPPORTED); d_in, d_out >= r and multiples of 4, the
 * factor and basis pointers 16-byte aligned (else CTS_ERR_SHAPE).  workspace: device, >=
 * cts_jd_workspace_bytes(...), 16-byte aligned (CTS_ERR_SHAPE otherwise).  No normalization is
 * applied (do it on the factors beforehand, Sec. 6.1, if wanted).  Stream-ordered, deterministic.
 * Implementation (same iterates, different rounding): when every problem of a batch has
 * 2r <= n*r_i <= 1024 and r is 16 or 32, all iterations but the last run in the stacked-factor
 * space through the Grams A_stack A_stack^T and Bt_stack Bt_stack^T (formed once on the tensor
 * cores); the last iteration is the explicit one above, so U and V are orthonormal to fp32
 * rounding.  Below 2r (a span that can collapse) every iteration is explicit, and a collapsed
 * column is completed deterministically with standard basis vectors (as the oracle does).
 */
typedef struct {
  const float* a_stack;
  const float* bt_stack;
  int32_t n, r_i, d_in, d_out;
  float* U;
  float* V;
  float* sigma;
} cts_jd_problem_t;
cts_status_t cts_jd_workspace_bytes(const cts_jd_problem_t* problems, int32_t count, int32_t r, size_t* bytes);
cts_status_t cts_jd_eigen_iteration(const cts_jd_problem_t* problems, int32_t count, int32_t r, int32_t iters,
                                    void* workspace, size_t ws_bytes, cudaStream_t stream);

/*
 * Cluster-affinity placement across GPUs ("clustering offers opportunities for
 * efficient scheduling"): each rank holds the bases of the clusters it owns only, and
 * tokens travel to the owner of their cluster (an all-to-all of rows, as in expert parallelism).
 * The collective itself is the caller's (NCCL all-to-all through torch.distributed, placement.py);
 * these two kernels build and apply the routing.
 * cts_route: token_adapter [T] (device, -1 = none), owner [N] (device, adapter -> rank in
 *   [0, world)); writes perm [T] (device) = token indices stably partitioned by destination rank
 *   (tokens without an adapter go to `self`) and counts [world] (device).  world <= 64.
 * cts_rows_move: rows of row_bytes bytes (activation rows or int32 ids; a multiple of 4):
 *   scatter == 0: dst[k] = src[idx[k]] (gather), else dst[idx[k]] = src[k]; ld_src / ld_dst are
 *   row strides in BYTES (multiples of 4), idx [n] device int32.  Stream-ordered;
 *   CTS_ERR_INVALID_ARGUMENT / CTS_ERR_SHAPE on bad arguments.
 */
cts_status_t cts_route(const int32_t* token_adapter, int32_t T, const int32_t* owner, int32_t N, int32_t world,
                       int32_t self, int32_t* perm, int32_t* counts, cudaStream_t stream);
cts_status_t cts_rows_move(const void* src, int64_t ld_src, void* dst, int64_t ld_dst, const int32_t* idx, int32_t n,
                           int32_t row_bytes, int32_t scatter, cudaStream_t stream);

/* Read the plan's device error word (call after synchronizing the stream that ran cts_segment).
 * *code = CTS_OK or CTS_ERR_INDEX_OUT_OF_RANGE; *first_bad_token = smallest offending t or -1. */
cts_status_t cts_plan_error(cts_plan_t plan, int32_t* code, int32_t* first_bad_token);

/* Static description of a status code. */
const char* cts_status_string(cts_status_t status);

/* Declare (1) or revoke (0, the default) exclusive use of the current process's device by libcts
 * launches: the caller guarantees that no other kernel (another stream of this process, another
 * process under MPS) runs while a fused apply is in flight -- e.g. a serving process that owns the
 * GPU and issues its applies on one stream.  Fused applies then launch NON-cooperatively, which
 * lets their prologue overlap the previous kernel's tail under programmatic dependent launch
 * (~1.3 us per launch at decode, measured); under sharing that variant can deadlock (its CTAs wait
 * on flags of CTAs that are not resident), so leave the default when unsure.  Process-wide; takes
 * effect for launches enqueued (or captured) afterwards.  Errors: CTS_ERR_INVALID_ARGUMENT. */
cts_status_t cts_set_exclusive_device(int32_t exclusive);

/* Number of kernels this library has enqueued since it was loaded (process-wide, all banks and
 * plans; launches recorded into a CUDA graph under stream capture count once, at capture).  The
 * difference across a call sequence is that sequence's kernel count: cts_segment = 1,
 * cts_apply / cts_apply_group = 1 (fused kernel; 2 with CTS_FUSED=0), cts_shrink* = cts_expand* = 1,
 * cts_expand_reduced_group = 2, cts_project = 2, cts_jd_eigen_iteration per batch of up to 200
 * problems = 5 + 13 per iteration (tensor-core path), 5 + 15 per iteration (CUDA-core path), or
 * 5 + 3 + 5 per stacked-space iteration + 11 for the last one (stacked-space path, iters >= 2),
 * cts_bank_load = 3 per module.  Never fails. */
uint64_t cts_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* CTS_H_ */

/*
 * dlx_b200.h — C-ABI of the B200-native DiLoCoX outer-synchronisation path.
 *
 * Drop-in boundary for the reference's compressor / worker-sync / outer-optimiser API
 * (reference /root/reference/proj/core; citations are include/dilocox/NAME.hpp and src/NAME.cpp
 * file:line). Every entry point is extern "C", takes plain pointers and sizes, never a
 * torch type. Device pointers are caller-owned CUDA global memory; the library owns
 * per-context workspaces. All compute calls are asynchronous on the given cudaStream_t
 * (passed as void*); one host thread per context; not re-entrant per context.
 *
 * Data layout (device):
 *   - A ParamSet (reference params.hpp:12-33) is ONE fp32 "slab"; tensor i starts at
 *     element dlx_layout_offsets()[i] (256-byte aligned), row-major, in table order.
 *   - Factor buffers (warm Q, and P/Q scratch) are column-major per 2-D tensor, column
 *     stride ld = round_up(rows, 32); offsets via dlx_factor_offsets().
 *   - A compressed payload is one byte buffer of dlx_payload_bytes(): per tensor, in
 *     table order, 16-byte aligned segments  [P codes][Q codes][P scales][Q scales]
 *     (2-D) or [codes][scale] (1-D). Codes are q-bit two's complement, LSB-first,
 *     column-major — byte-identical to the code sections of the reference wire format
 *     (compress.cpp:352-367, 395-426). Scales are fp32. D payloads back to back form
 *     the all-gather buffer that dlx_outer_update consumes.
 *
 * Status codes mirror the reference exception taxonomy (errors.hpp:8-34).
 */
#ifndef DLX_B200_H
#define DLX_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum dlx_status {
  DLX_OK = 0,
  DLX_ERR_VALIDATION = 1, /* dilocox::ValidationError */
  DLX_ERR_SHAPE = 2,      /* dilocox::ShapeError */
  DLX_ERR_FORMAT = 3,     /* dilocox::FormatError */
  DLX_ERR_NUMERIC = 4,    /* dilocox::NumericError */
  DLX_ERR_IO = 5,         /* dilocox::IoError */
  DLX_ERR_CUDA = 6,
  DLX_ERR_NCCL = 7
} dlx_status;

enum { DLX_ROUND_STOCHASTIC = 0, DLX_ROUND_NEAREST = 1 }; /* compress.hpp:13 Rounding */
enum { DLX_MODE_OVERLAPPED = 0, DLX_MODE_SYNC = 1 };      /* engine.cpp:423-509 */

typedef struct dlx_ctx dlx_ctx;
typedef struct dlx_layout dlx_layout;

/* Round statistics written by dlx_outer_update (device doubles; see RoundRecord
 * engine.hpp:74-95). */
typedef struct dlx_round_stats {
  double err_num;        /* sum (dec(payload_self) - delta_pending)^2   (measure_error) */
  double err_den;        /* sum delta_pending^2                                           */
  double delta_norm_sq;  /* ||delta_new||^2        (stage_deltas max_delta_norm)          */
  double err_norm_sq;    /* ||e||^2                (RoundRecord.err_buf_norm)             */
  double nonfinite;      /* count of non-finite anchor values produced (NumericError)     */
  double pad[3];
} dlx_round_stats;

/* ---- context / errors --------------------------------------------------------------- */
const char* dlx_version(void);
const char* dlx_last_error(void); /* thread-local message of the last failing call */
dlx_status dlx_ctx_create(int device, dlx_ctx** out);
dlx_status dlx_ctx_destroy(dlx_ctx* ctx);

/* ---- worker sync (one process per GPU = one DiLoCoX worker) ---------------------------
 * Replaces the reference's in-process collective: allreduce_avg (collective.hpp:23,
 * collective.cpp:17-46) is a mean of per-worker reconstructions, so the exchange of a round
 * is an all-gather of every worker's compressed payload (worker order = rank order) plus the
 * broadcast of worker 0's float Q factors as everyone's next warm start (collective_average,
 * engine.cpp:215-263, 241, 498-501). NCCL over NVLink / NVSwitch, resolved at run time
 * (libnccl.so.2; DLX_ERR_NCCL if absent). The collectives run on a library-owned
 * high-priority side stream, joined to the caller's stream by events.
 *
 * Bootstrap: rank 0 calls dlx_comm_unique_id and ships the 128 bytes to the other ranks by
 * any means (file, TCP, MPI, torch.distributed); every rank then calls dlx_comm_init (a
 * collective: blocks until all ranks have joined). dlx_ctx_create_dist does both steps'
 * second half in one call. */
#define DLX_UNIQUE_ID_BYTES 128
enum { DLX_EXCHANGE_BCAST_DEFERRED = 1 }; /* dlx_exchange flags */
dlx_status dlx_comm_unique_id(void* out /* DLX_UNIQUE_ID_BYTES */);
dlx_status dlx_comm_init(dlx_ctx* ctx, int rank, int world, const void* unique_id);
dlx_status dlx_ctx_create_dist(int device, int rank, int world, const void* unique_id,
                               dlx_ctx** out);
dlx_status dlx_comm_info(const dlx_ctx* ctx, int* rank, int* world);
/* All-gather d_payload (payload_bytes, this worker's) into d_gathered (world * payload_bytes,
 * worker w at offset w * payload_bytes) and broadcast worker 0's d_warm_q (warm_elems floats,
 * in place) to every worker. `stream` is ordered after the all-gather; after the broadcast
 * too unless flags has DLX_EXCHANGE_BCAST_DEFERRED, in which case dlx_exchange_wait_warm
 * joins it later (it is only needed by the next round's compress). world == 1: copies the
 * payload into d_gathered (if distinct) and returns. */
dlx_status dlx_exchange(dlx_ctx* ctx, const uint8_t* d_payload, int64_t payload_bytes,
                        uint8_t* d_gathered, float* d_warm_q, int64_t warm_elems, int flags,
                        void* stream);
dlx_status dlx_exchange_wait_warm(dlx_ctx* ctx, void* stream);
/* Generic pieces of the same communicator: byte all-gather (the no-compress ablation's raw
 * slabs, compress_raw compress.cpp:185-199) and an fp64 sum (the per-tensor effective-rank
 * shards: one nonzero term per entry, so the sum is exact on every rank). */
dlx_status dlx_comm_allgather(dlx_ctx* ctx, const void* d_send, int64_t bytes, void* d_recv,
                              void* stream);
dlx_status dlx_comm_allreduce_sum_f64(dlx_ctx* ctx, double* d_buf, int64_t n, void* stream);
/* Poll the communicator for an asynchronous NCCL failure (ncclCommGetAsyncError): DLX_OK or
 * DLX_ERR_NCCL. Cheap; the engine polls once per round. */
dlx_status dlx_comm_check(dlx_ctx* ctx);
dlx_status dlx_comm_destroy(dlx_ctx* ctx);

/* ---- tensor table (ParamSet layout) ---------------------------------------------------
 * ndim[i] in {1,2}; dims[2i], dims[2i+1] = (rows, cols) or (n, 1). Mirrors
 * ParamSet::add / same_layout (params.hpp:12-33). */
dlx_status dlx_layout_create(dlx_ctx* ctx, int nt, const int* ndim, const int64_t* dims,
                             dlx_layout** out);
dlx_status dlx_layout_destroy(dlx_layout* layout);
int64_t dlx_layout_slab_elems(const dlx_layout* layout);
dlx_status dlx_layout_offsets(const dlx_layout* layout, int64_t* offsets /* nt */);
/* Per-2-D-tensor column-major factor offsets (elements) for the given rank (b side for
 * Q / warm Q when side = 1, a side for P when side = 0); entries for 1-D tensors are -1.
 * Returns the total element count of the factor buffer. */
int64_t dlx_factor_offsets(const dlx_layout* layout, int rank, int side, int64_t* offsets);

/* ---- payload geometry (compress.cpp:92-114, 395-426) --------------------------------- */
int64_t dlx_payload_bytes(const dlx_layout* layout, int rank, int qbits);
/* seg[4*i + {0,1,2,3}] = byte offsets of P codes, Q codes, P scales, Q scales
 * (1-D: codes, -1, scale, -1). */
dlx_status dlx_payload_segments(const dlx_layout* layout, int rank, int qbits, int64_t* seg);
uint64_t dlx_payload_bits(const dlx_layout* layout, int rank, int qbits);

/* ---- synthetic inputs -----------------------------------------------------------------
 * out[t] = (base ? base[t] : 0) + scale * g, g = Tensor::gaussian (tensor.cpp:49-53) drawn
 * from RngStream(seed, stream_key({tag, worker, t})) per tensor t, bit-identical to the
 * reference generator; two separate fp32 roundings (mul, add). */
dlx_status dlx_fill_gaussian(dlx_ctx* ctx, const dlx_layout* layout, float* d_out,
                             const float* d_base, float scale, uint64_t seed, uint64_t tag,
                             uint64_t worker, void* stream);

/* ---- compressor (compress.hpp:94-95 compress) -------------------------------------------
 * Low-rank (warm-started power iteration, power_iters >= 1) + per-column q-bit
 * quantisation of every 2-D tensor, quantisation of every 1-D tensor, in table order,
 * consuming the shared splitmix stream whose state is rng_state (RngStream after
 * construction, rng.hpp:13-16). d_warm_q (nullable) is the previous round's Q factors
 * for warm_rank; used iff warm_rank == rank (compress.cpp:161). Writes the payload and
 * the float Q factors (next warm start, compress.hpp:86-90). *d_draws (nullable, device
 * uint64) receives the number of draws consumed (the reference advances its RngStream&
 * by exactly that). Fully asynchronous: a cold start under stochastic rounding verifies its
 * speculative draw offsets on the device (a CUDA-graph WHILE node redoes the compress body
 * from the observed offsets; all-zero chunks draw nothing, compress.cpp:28-30); the
 * (pathological) failure to converge is reported as *d_draws == UINT64_MAX. */
dlx_status dlx_compress(dlx_ctx* ctx, const dlx_layout* layout, const float* d_delta, int rank,
                        int qbits, int rounding, int power_iters, uint64_t rng_state,
                        const float* d_warm_q, int warm_rank, uint8_t* d_payload,
                        float* d_q_out, uint64_t* d_draws, void* stream);

/* Quantise given float factors exactly as compress does after lowrank_approx
 * (quantize_columns compress.cpp:119-131 per 2-D tensor P then Q, quantize :24-49 per
 * 1-D tensor taken from d_delta). cold != 0 inserts the b*r cold-start draws before each
 * 2-D tensor (compress.cpp:64-69). d_p / d_q use dlx_factor_offsets layouts. */
dlx_status dlx_quantize_factors(dlx_ctx* ctx, const dlx_layout* layout, const float* d_p,
                                const float* d_q, const float* d_delta, int rank, int qbits,
                                int rounding, uint64_t rng_state, int cold,
                                uint8_t* d_payload, uint64_t* d_draws, void* stream);

/* decompress (compress.cpp:201-238) of one payload into a dense slab. */
dlx_status dlx_decompress(dlx_ctx* ctx, const dlx_layout* layout, int rank, int qbits,
                          const uint8_t* d_payload, float* d_out, void* stream);

/* allreduce_avg (collective.cpp:17-46): mean of the D payloads' reconstructions, given the
 * all-gather buffer (D payloads back to back). Dense fp32 output. */
dlx_status dlx_allreduce_avg(dlx_ctx* ctx, const dlx_layout* layout, int rank, int qbits,
                             int D, const uint8_t* d_gathered, float* d_out, void* stream);

/* ---- fused outer update (engine.cpp:254-276 + optim.cpp:56-78) ---------------------------
 * Given the all-gather buffer, reconstructs Delta = (1/D) sum_w P_w Q_w^T per tensor in
 * the tile, never materialising it, and in the same pass:
 *   overlapped: e = pending - Delta; pending <- (anchor - local) + e  (pre-update anchor)
 *   sync:       pending <- pending - Delta                           (pending becomes e)
 *   both:       v <- beta v + Delta; anchor <- anchor - gamma (Delta + beta v)
 *               (classical: anchor <- anchor - gamma v)
 * self_index >= 0 also accumulates measure_error (compress.cpp:246-262) for that worker's
 * payload. d_stats (device dlx_round_stats, nullable) receives the reductions. */
dlx_status dlx_outer_update(dlx_ctx* ctx, const dlx_layout* layout, int rank, int qbits, int D,
                            const uint8_t* d_gathered, int self_index, int mode,
                            float* d_pending, float* d_anchor, const float* d_local,
                            float* d_velocity, float gamma, float beta, int classical,
                            dlx_round_stats* d_stats, void* stream);

/* dlx_outer_update restricted to the layout tensors [t_begin, t_end) (all state buffers are
 * still full slabs; only that range is read and written). d_stats is zeroed only when
 * t_begin == 0, so consecutive ranges accumulate one round's statistics — the host pipeline
 * (OuterSync.step_host) updates each range as soon as its H2D copy has landed. */
dlx_status dlx_outer_update_range(dlx_ctx* ctx, const dlx_layout* layout, int rank, int qbits,
                                  int D, const uint8_t* d_gathered, int self_index, int mode,
                                  float* d_pending, float* d_anchor, const float* d_local,
                                  float* d_velocity, float gamma, float beta, int classical,
                                  dlx_round_stats* d_stats, int t_begin, int t_end,
                                  void* stream);

/* ---- inner optimiser (the overlap partner) ----------------------------
 * adamw_step (optim.cpp:15-47) over n contiguous fp32 parameters (16-B aligned buffers):
 * *step is the caller's persistent step counter and is incremented as in the reference; the
 * bias corrections and warm-up LR are computed on the host exactly as optim.cpp does, so the
 * update is bit-exact. A non-finite gradient sets *d_nonfinite (nullable device int) — the
 * caller raises NumericError after synchronising (the reference throws after the update). */
dlx_status dlx_adamw_step(dlx_ctx* ctx, int64_t n, float lr, float beta1, float beta2, float eps,
                          float weight_decay, int64_t warmup_steps, int64_t* step, float* d_p,
                          const float* d_g, float* d_m, float* d_v, int* d_nonfinite,
                          void* stream);

/* dilocox-no-compress ablation (compress_raw compress.cpp:185-199, engine.cpp:231-233): the
 * exchanged payload is each worker's raw fp32 pending slab; d_gathered holds D slabs back to
 * back (worker order). Delta = float(sum_w double(x_w) * (1/D)) exactly as allreduce_avg,
 * then the same fused error feedback / staging / Nesterov as dlx_outer_update. measure_error
 * of a raw payload is 0 (exact reconstruction). */
dlx_status dlx_outer_update_raw(dlx_ctx* ctx, const dlx_layout* layout, int D,
                                const float* d_gathered, int self_index, int mode,
                                float* d_pending, float* d_anchor, const float* d_local,
                                float* d_velocity, float gamma, float beta, int classical,
                                dlx_round_stats* d_stats, void* stream);

/* stage_deltas (engine.cpp:266-276): pending <- (anchor - local) + (d_err ? d_err : 0).
 * d_err may alias d_pending. d_norm_sq (nullable device double) gets ||pending||^2. */
dlx_status dlx_stage_deltas(dlx_ctx* ctx, const dlx_layout* layout, const float* d_anchor,
                            const float* d_local, const float* d_err, float* d_pending,
                            double* d_norm_sq, void* stream);

/* measure_error (compress.cpp:246-262) of one payload against the dense delta it compressed:
 * d_out[0] = sum (decompress(payload) - delta)^2, d_out[1] = sum delta^2 (device doubles;
 * comp_error = d_out[0] / d_out[1], 0 when d_out[1] == 0). */
dlx_status dlx_measure_error(dlx_ctx* ctx, const dlx_layout* layout, int rank, int qbits,
                             const uint8_t* d_payload, const float* d_delta, double* d_out,
                             void* stream);

/* The same reduction for a dense reconstruction already in a slab (RawDense payloads). */
dlx_status dlx_sqdiff_slabs(dlx_ctx* ctx, const dlx_layout* layout, const float* d_rec,
                            const float* d_delta, double* d_out, void* stream);

/* Worker-order mean of D fp32 slabs of n elements stored ld apart (d_in[w * ld + i]):
 * out = float((sum_w double(x_w)) * (1.0 / D)) — allreduce_avg over compress_raw payloads
 * (collective.cpp:17-46, compress.cpp:185-199) and the per-step gradient mean of the
 * all-reduce baseline (engine.cpp:559-570). Bit-exact. */
dlx_status dlx_mean_slabs(dlx_ctx* ctx, int64_t n, int64_t ld, int D, const float* d_in,
                          float* d_out, void* stream);

/* nesterov_outer_step (optim.cpp:56-78) on a dense averaged delta. */
dlx_status dlx_nesterov(dlx_ctx* ctx, int64_t n, float gamma, float beta, int classical,
                        float* d_anchor, float* d_velocity, const float* d_delta, void* stream);

/* ---- adaptive rank (compress.cpp:306-344, engine.cpp:294-308) ----------------------------
 * effective_rank of the averaged delta, computed in factor space from the all-gather
 * buffer: the nonzero singular values of (1/D) [P_1..P_D][Q_1..Q_D]^T are those of the
 * (D r) x (D r) matrix L^T (P^T P) L with L L^T = Q^T Q, so no dense SVD is needed.
 * d_per_tensor (device int, one per 2-D tensor) and d_energy (device double, per 2-D
 * tensor) are written; dlx_effective_rank_reduce aggregates on the host exactly as the
 * reference (size-weighted mean, ceil, clamp to [1, r_max]). */
dlx_status dlx_effective_rank(dlx_ctx* ctx, const dlx_layout* layout, int rank, int qbits,
                              int D, const uint8_t* d_gathered, double tau, int* d_per_tensor,
                              double* d_energy, void* stream);
/* dlx_effective_rank restricted to the 2-D tensors with (index among 2-D tensors) % nshards
 * == shard; the entries of the other tensors are set to 0. Every rank of a D-worker group
 * holds the same all-gather buffer, so the group splits the eigenproblems (shard = rank,
 * nshards = world) and sums the per-tensor arrays (exact: one nonzero term each). */
dlx_status dlx_effective_rank_shard(dlx_ctx* ctx, const dlx_layout* layout, int rank,
                                    int qbits, int D, const uint8_t* d_gathered, double tau,
                                    int shard, int nshards, int* d_per_tensor, double* d_energy,
                                    void* stream);
dlx_status dlx_effective_rank_reduce(const dlx_layout* layout, const int* per_tensor,
                                     const double* energy, int r_max, int* aggregate,
                                     int* all_zero);
dlx_status dlx_adapt_compression(const int* window, int len, int r1, int H1, int c, int h_min,
                                 int* r_out, int* h_out);
double dlx_omega_bound(int r, int d, int q);

/* ---- wire format (compress.cpp:395-482) -------------------------------------------------
 * Host-side conversion between a device payload (copied to host) and DLXC v1 bytes.
 * Tensor names are caller-provided (names[i]); rank is CompressedDelta::rank. */
int64_t dlx_serialize(const dlx_layout* layout, int rank, int qbits, const char* const* names,
                      const uint8_t* h_payload, uint8_t* out, int64_t cap);
dlx_status dlx_parse(const dlx_layout* layout, int rank, int qbits, const uint8_t* bytes,
                     int64_t size, uint8_t* h_payload);

/* Runtime options (A/B testing). "tensor_cores" (default 1): 0 routes the power-iteration
 * sweeps through the SIMT kernels instead of the tcgen05 ones (env DLX_TENSOR_CORES=0).
 * "outer_tensor_cores" (default 1): 0 runs the fused outer update with the SIMT factor GEMM
 * instead of the tcgen05/TMA kernel (env DLX_OUTER_TC=0). "kernel_events" (default 0): 1
 * brackets each launch of the dominant kernels (k_o5, k_tc_sweep K1/K2) with CUDA events on
 * the launching stream, for dlx_kernel_time. "effrank_big_from" (default 96): effective-rank
 * eigenproblems with K = D * r above this size run the blocked large-K kernel.
 * "cholqr_blocked" (default 1): 0 factors 32 < r <= 128 CholQR Grams with the unblocked
 * shared-memory kernel instead of the blocked DMMA one. */
dlx_status dlx_set_option(const char* key, int value);

/* Device time (ms, from the CUDA events), algorithmic HBM bytes and launch count of every
 * recorded launch of kernel `name` ("k_o5", "k_tc_sweep_k1", "k_tc_sweep_k2") since the last
 * call; synchronises on those events and clears them. Needs "kernel_events" = 1. */
dlx_status dlx_kernel_time(const char* name, double* ms_total, double* bytes_total,
                           int64_t* launches);

/* Test hook: one power-iteration sweep — which = 0: out = delta * in (K1, in = Q factors),
 * which = 1: out = delta^T * in (K2, in = P factors) — on the tcgen05 (use_tc = 1) or SIMT
 * path. Factor buffers use the dlx_factor_offsets layouts. */
dlx_status dlx_debug_sweep(dlx_ctx* ctx, const dlx_layout* layout, int rank, int which,
                           const float* d_slab, const float* d_in, float* d_out, int use_tc,
                           void* stream);

/* Number of kernels this library launched on the calling thread since the last call
 * (launch accounting for benchmarks). */
uint64_t dlx_take_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* DLX_B200_H */

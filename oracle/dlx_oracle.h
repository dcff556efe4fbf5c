/*
 * dlx_oracle.h — C interface shared by the two CPU checkers of this repo.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product path (paper_2506_21263_b200/,
 * include/) may include, link or call this. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs use it, and only as the
 * checker or the timed CPU baseline.
 *
 * Two libraries export exactly these symbols:
 *   oracle/liboracle.so          — dlx_oracle.c, a plain-C restatement of the
 *                                   reference algorithm (file:line cited per function)
 *   oracle/_ref/libdlxref.so     — ref_shim.cpp linked against the reference's own
 *                                   proj/core sources, compiled from /root/reference
 *                                   by oracle/Makefile (never copied into this repo)
 *
 * Conventions (both libraries):
 *   - Tensor table: nt tensors, ndim[i] in {1,2}; dims[2i], dims[2i+1] are (rows, cols)
 *     for 2-D and (n, 1) for 1-D. Dense data is the concatenation of the tensors in
 *     table order, row-major, no padding (the reference ParamSet order).
 *   - RNG streams are passed as the raw splitmix64 state (uint64_t*), advanced in place
 *     by exactly the number of draws consumed (reference rng.hpp:11-59).
 *   - Unpacked payload: codes int8 concatenated per tensor — 2-D: P codes (a*r,
 *     column-major) then Q codes (b*r, column-major); 1-D: n codes. Scales fp32
 *     concatenated — 2-D: r P scales then r Q scales; 1-D: one scale. ranks[i] is r_eff
 *     for 2-D tensors, 0 for 1-D. (Same content as reference TensorPayload,
 *     compress.hpp:83-96.)
 *   - Q factors: per 2-D tensor b*r_eff row-major (reference Tensor layout).
 *   - Return codes: 0 ok, 1 ValidationError, 2 ShapeError, 3 FormatError,
 *     4 NumericError, 5 IoError, 9 other; orc_last_error() holds the message.
 */
#ifndef DLX_ORACLE_H
#define DLX_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
const char* orc_backend(void); /* "restatement" or "reference" */

uint64_t orc_stream_key(const uint64_t* parts, int n);
uint64_t orc_stream_init(uint64_t seed, uint64_t stream_id);
uint64_t orc_next_u64(uint64_t* state);
void orc_gaussian(uint64_t* state, int64_t n, float* out);
void orc_uniform(uint64_t* state, int64_t n, float lo, float hi, float* out);

int orc_matmul(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c);
int orc_matmul_tn(int64_t k, int64_t m, int64_t n, const float* a, const float* b, float* c);
int orc_matmul_nt(int64_t m, int64_t k, int64_t n, const float* a, const float* b, float* c);
int orc_orthonormalize(int64_t n, int64_t r, const float* in, float* out, int* replaced);
int orc_singular_values(int64_t a, int64_t b, const float* m, double* sv_out);

int orc_lowrank_approx(int64_t a, int64_t b, const float* m, int r, const float* warm_q,
                       int iters, uint64_t* state, float* p_out, float* q_out);
int orc_quantize(const float* x, int64_t n, int qbits, int rounding, uint64_t* state,
                 int8_t* codes, float* scale);

int64_t orc_codes_count(int nt, const int* ndim, const int64_t* dims, const int* ranks);
int64_t orc_scales_count(int nt, const int* ndim, const int64_t* dims, const int* ranks);
int64_t orc_qfactor_count(int nt, const int* ndim, const int64_t* dims, const int* ranks);

int orc_compress(int nt, const int* ndim, const int64_t* dims, const float* data, int rank,
                 int qbits, int rounding, int iters, int warm_rank, const float* warm_q,
                 uint64_t* state, int8_t* codes, float* scales, float* q_out, int* ranks,
                 uint64_t* payload_bits);
int orc_decompress(int nt, const int* ndim, const int64_t* dims, const int* ranks,
                   const int8_t* codes, const float* scales, float* out);
int orc_allreduce_avg(int D, int nt, const int* ndim, const int64_t* dims, const int* ranks,
                      const int8_t* const* codes, const float* const* scales, float* out);
int orc_measure_error(int nt, const int* ndim, const int64_t* dims, const float* delta,
                      const int* ranks, const int8_t* codes, const float* scales, double* err);
/* adamw_step (optim.cpp:15-47) on one flat tensor; *step is the persistent step counter
 * (incremented). Returns 4 (NumericError) on a non-finite gradient, like the reference. */
int orc_adamw_step(int64_t n, float lr, float beta1, float beta2, float eps, float weight_decay,
                   int64_t warmup_steps, int64_t* step, float* p, const float* g, float* m,
                   float* v);
int orc_nesterov(int64_t n, float gamma, float beta, int classical, float* anchor, float* v,
                 const float* delta);
int orc_effective_rank(int nt, const int* ndim, const int64_t* dims, const float* data,
                       double tau, int r_max, int* per_tensor, int* aggregate, int* all_zero);
int orc_adapt_compression(const int* window, int len, int r1, int H1, int c, int h_min,
                          int* r_out, int* h_out);
double orc_omega_bound(int r, int d, int q);
uint64_t orc_payload_bits(int nt, const int* ndim, const int64_t* dims, const int* ranks,
                          int qbits);
/* DLXC v1 wire bytes (reference compress.cpp:395-426). Tensor names are "t<i>".
 * Returns the byte count; writes only if out != NULL and cap is large enough. */
int64_t orc_serialize(int nt, const int* ndim, const int64_t* dims, const int* ranks, int rank,
                      int qbits, const int8_t* codes, const float* scales, uint8_t* out,
                      int64_t cap);

/* One overlapped outer-sync round for D workers, as run_round_overlapped steps (2),(4),(5)
 * (reference engine.cpp:458-509 with collective_average :215-263 and stage_deltas
 * :266-276), has_pending assumed true. pending/local are D*n concatenated.
 * In/out: anchor, velocity, pending (old delta in, new delta out), warm (warm_rank,
 * warm_q; pass warm_rank = 0 for none). Out: r_prime (0 if !adaptive), comp_error,
 * payload_bits, err_norm0 (||e_0||), max_delta_norm. threads: compress fan-out over
 * workers as parallel_over (engine.cpp:135-156). */
int orc_outer_round(int D, int nt, const int* ndim, const int64_t* dims, uint64_t seed,
                    int64_t round_index, int rank, int qbits, int rounding, int iters,
                    int adaptive, double tau, int r1, float gamma, float beta, int classical,
                    int threads, float* anchor, float* velocity, float* pending,
                    const float* local, int* warm_rank, float* warm_q, int* r_prime,
                    double* comp_error, uint64_t* payload_bits, double* err_norm0,
                    double* max_delta_norm);

#ifdef __cplusplus
}
#endif
#endif

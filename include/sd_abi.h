/*
 * sd_abi.h — C ABI of the B200-native FastDecode decode hot path.
 *
 * Drop-in boundary for the reference `splitdecode` (FastDecode, arXiv
 * 2403.11421) decode path. Plain pointers and sizes only; no C++ or torch
 * types cross this boundary. Each entry point names the reference interface
 * it replaces (file:line under the reference's proj/).
 *
 * Conventions
 *   - Every function returns an int status (SD_OK == 0). On failure
 *     sd_last_error() returns a thread-local message. Status numbering
 *     follows the reference's wire error codes (transport.hpp:39-44):
 *     3 malformed/ProtocolError, 4 CapacityError, 5 UnknownSequenceError,
 *     6 internal; plus 7 std::logic_error, 8 ConfigError, 9 CUDA, 10 NCCL,
 *     11 AdmissionError (scheduler.hpp:20-23).
 *   - Activations are row-major float32 [rows][width]. Weights are passed in
 *     the reference's storage: Eigen column-major (out x in), element w(j,k)
 *     at w[k*out + j] (core.hpp:79-90).
 *   - Functions without a `_dev` suffix take HOST pointers and are
 *     synchronous (the reference's blocking semantics). `_dev` variants take
 *     DEVICE pointers and enqueue on `stream` (a cudaStream_t; NULL = the
 *     legacy default stream) without synchronizing.
 *   - Validation (positions, capacity, unknown sequences, atomicity) runs on
 *     the host against a mirror of per-(sequence, layer) stored lengths
 *     before anything is launched, so error behaviour is the reference's.
 *   - One handle is used from one host thread (the reference's ownership
 *     model).
 */
#ifndef SD_ABI_H_
#define SD_ABI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define SD_ABI_VERSION 1

enum sd_status {
  SD_OK = 0,
  SD_ERR_PROTOCOL = 3,
  SD_ERR_CAPACITY = 4,
  SD_ERR_UNKNOWN_SEQ = 5,
  SD_ERR_INTERNAL = 6,
  SD_ERR_LOGIC = 7,
  SD_ERR_CONFIG = 8,
  SD_ERR_CUDA = 9,
  SD_ERR_NCCL = 10,
  SD_ERR_ADMISSION = 11,
  SD_ERR_INFEASIBLE = 12 /* InfeasiblePlanError (planner.hpp:18-23) */
};

/* KvFormat (attention.hpp:24). SD_KV_INT4 is an extension: the paper's 4-bit
 * quantization hook with quantize_int8's rules at +-7
 * (per-(position, head) fp32 scale max|x| / 7, round half to even), two
 * values per byte, element 2i in the low nibble; needs an even head_dim. */
enum sd_kv_format { SD_KV_SINGLE = 0, SD_KV_HALF = 1, SD_KV_INT8 = 2, SD_KV_INT4 = 3 };

/* S-Part arithmetic (dense.hpp:16-20 fixes fp32, k-ascending). */
enum sd_dense_mode {
  SD_DENSE_EXACT_F32 = 0, /* CUDA-core fp32, the reference's per-element op order (bitwise) */
  SD_DENSE_BF16 = 1,      /* tcgen05 kind::f16, bf16 operands, fp32 accumulate in TMEM */
  SD_DENSE_TF32 = 2,      /* tcgen05 kind::tf32, fp32 operands (read truncated to tf32), fp32 accumulate */
  SD_DENSE_F16 = 3        /* tcgen05 kind::f16, fp16 operands (RNE, 11-bit significand), fp32 accumulate:
                             tf32-level operand precision at the bf16 rate; operands must stay within
                             fp16 range (|x| < 65504) */
};

/* ShardMode (transport.hpp:150-170) */
enum sd_shard_mode { SD_SHARD_BY_SEQUENCE = 0, SD_SHARD_BY_HEAD = 1, SD_SHARD_HYBRID = 2 };
/* Home (S-Part) placement of a sequence when s_ranks == world, ORed into a
 * shard_mode argument. Default under by-sequence sharding: shard-affine and
 * balanced, each rank is home to floor/ceil(B / world) rows of the step,
 * preferring the rows whose KV it holds (mix64(seq) % world), so only the
 * overflow rows cross NVLink. SD_HOME_MODULO: home = seq % s_ranks, every
 * row crosses when its shard is elsewhere (other shard modes always use it). */
#define SD_HOME_MODULO 0x100

/* ModelSpec (core.hpp:43-50); num_kv_heads is a GQA extension (0 = num_heads). */
typedef struct sd_model_spec {
  int32_t num_layers, model_dim, num_heads, head_dim, mlp_dim, vocab_size, num_kv_heads;
} sd_model_spec;

/* Physical KV store sizing (no reference counterpart: the reference grows
 * std::vectors). All zero = defaults documented in DESIGN.md. The default
 * pool (ceil(capacity / page_positions) + max_sequences page groups, each
 * spanning every layer) always suffices for lockstep decode, where every
 * layer of a sequence advances together. A caller appending layers unevenly
 * (the reference accepts up to capacity * num_layers positions in any
 * spread, attention.cpp:148) can run out of page groups first and gets
 * SD_ERR_CAPACITY ("physical KV pool exhausted"); size pool_pages for its
 * spread (up to capacity * num_layers / page_positions) in that case. */
typedef struct sd_kv_options {
  int32_t max_sequences;  /* live sequences (slots); 0 = min(capacity, 4096) */
  int32_t max_seq_len;    /* positions per sequence; 0 = min(capacity, 32768) */
  int32_t page_positions; /* positions per page group, power of two; 0 = 16 */
  int32_t pool_pages;     /* page groups in the pool; 0 = ceil(cap/P) + max_sequences */
} sd_kv_options;

typedef struct sd_kv sd_kv;
typedef struct sd_weights sd_weights;
typedef struct sd_engine sd_engine;

const char* sd_last_error(void);
int sd_abi_version(void);
/* make_model_spec (core.cpp:11-30) */
int sd_make_model_spec(int num_layers, int model_dim, int num_heads, int mlp_dim,
                       int vocab_size, int num_kv_heads, sd_model_spec* out);
/* mix64 (core.cpp:161-166), prompt_token (core.cpp:168-171) */
uint64_t sd_mix64(uint64_t x);
int sd_prompt_token(uint64_t seed, uint64_t seq, int vocab_size);

/* ---------------------------------------------------------------- R-Part
 * KvShard (attention.hpp:68-140). head_start/head_count index kv heads. */
/* KvShard::KvShard (attention.hpp:70-71) */
int sd_kv_create(const sd_model_spec* spec, int head_start, int head_count,
                 int64_t capacity_tokens, int kv_format, int device,
                 const sd_kv_options* options, sd_kv** out);
int sd_kv_destroy(sd_kv* kv);
/* KvShard::append (attention.hpp:91-92): one (seq, layer) K/V row pair. */
int sd_kv_append(sd_kv* kv, uint64_t seq, int layer, uint32_t position, const float* k,
                 const float* v);
/* KvShard::append_request (attention.hpp:96): all-or-nothing batch append.
 * k, v: [n][width]. */
int sd_kv_append_request(sd_kv* kv, int layer, int32_t n, const uint64_t* seqs,
                         const uint32_t* positions, const float* k, const float* v);
/* KvShard::attend (attention.hpp:102): q, o: [n][q_width], outputs in item order. */
int sd_kv_attend(sd_kv* kv, int layer, int32_t n, const uint64_t* seqs, const float* q,
                 float* o);
/* Fused append_request + attend, the R-worker's QKV handler
 * (workers.cpp:110-111; dense.cpp:111-112). */
int sd_kv_append_attend(sd_kv* kv, int layer, int32_t n, const uint64_t* seqs,
                        const uint32_t* positions, const float* q, const float* k,
                        const float* v, float* o);
/* Device-pointer, stream-ordered variants of the three calls above. */
int sd_kv_append_request_dev(sd_kv* kv, int layer, int32_t n, const uint64_t* seqs,
                             const uint32_t* positions, const float* k_dev,
                             const float* v_dev, void* stream);
int sd_kv_attend_dev(sd_kv* kv, int layer, int32_t n, const uint64_t* seqs,
                     const float* q_dev, float* o_dev, void* stream);
int sd_kv_append_attend_dev(sd_kv* kv, int layer, int32_t n, const uint64_t* seqs,
                            const uint32_t* positions, const float* q_dev,
                            const float* k_dev, const float* v_dev, float* o_dev,
                            void* stream);
/* KvShard::drop_sequence (attention.hpp:106); unknown ids count a warning. */
int sd_kv_drop(sd_kv* kv, int32_t n, const uint64_t* seqs);
/* Queries (attention.hpp:73-111). */
int sd_kv_stored_length(const sd_kv* kv, uint64_t seq, int layer, int32_t* out);
int sd_kv_has_sequence(const sd_kv* kv, uint64_t seq, int32_t* out);
int sd_kv_token_count(const sd_kv* kv, int64_t* out);
int sd_kv_warning_count(const sd_kv* kv, int32_t* out);
int sd_kv_bytes_per_token(const sd_kv* kv, int64_t* out);
int sd_kv_width(const sd_kv* kv, int32_t* width, int32_t* q_width);
/* Stored bytes of one lane (which: 0 = K, 1 = V) in the reference's
 * [pos][head][d] order (attention.cpp:117-118) and, for int8 / int4, the per
 * (pos, head) scales (attention.cpp:129-130); quantized codes come back as
 * the reference's two's-complement bytes (int4: two per byte, element 2i in
 * the low nibble). Returns the byte count (or a negative status); copies
 * when host/scales are large enough. */
int64_t sd_kv_export_lane(const sd_kv* kv, uint64_t seq, int layer, int which, void* host,
                          size_t host_bytes, float* scales, size_t scales_count);
/* Fills every (slot, layer, position < length) of the listed sequences
 * with the counter-based synthetic values of SURVEY §8d (bench prefill).
 * Registers the sequences with stored length `length` in every layer. */
int sd_kv_prefill_synthetic(sd_kv* kv, int32_t n, const uint64_t* seqs, int32_t length,
                            uint64_t salt);
/* Per-launch timing of the attention kernel (CUDA events on the launching
 * stream). enable != 0 starts recording; read returns the summed kernel
 * milliseconds, launches and algorithmic bytes since the last reset. */
/* enable: 0 off, 1 every attention launch, k > 1 the launches of every k-th layer */
int sd_kv_timing(sd_kv* kv, int enable);
int sd_kv_timing_read(sd_kv* kv, double* ms, int64_t* launches, double* bytes, int reset);

/* ---------------------------------------------------------------- S-Part
 * WeightSet (core.hpp:85-90) uploaded once. tensors[] in reference order:
 * embedding (D x V), then per layer w_q, w_k, w_v, w_o, w_mlp_in, w_mlp_out,
 * then head (V x D); each Eigen column-major. */
int sd_weights_upload(const sd_model_spec* spec, const float* const* tensors, int dense_mode,
                      int device, sd_weights** out);
/* seed_random_weights (core.cpp:97-127, WeightSet core.hpp:85-90): the
 * reference's deterministic weights (mt19937 seeded uint32(seed ^ seed>>32),
 * uniform +-1/sqrt(fan_in), embedding +-1, memory-order fill), bit-identical
 * to the reference's, generated on the host (~1 ns per value; the stream is
 * sequential) and uploaded into `dense_mode`'s layout. */
int sd_weights_seed_random(const sd_model_spec* spec, uint64_t seed, int dense_mode, int device,
                           sd_weights** out);
int sd_weights_destroy(sd_weights* w);
/* The embedding as stored (fp32, D x V column-major: token t's column is
 * host[t * D .. t * D + D)), for callers that build TokenBatch.features on
 * the host (workers.cpp:629-638). count >= D * V. */
int sd_weights_export_embedding(const sd_weights* w, float* host, size_t count);
/* project_qkv (dense.hpp:26-27): x [B][D] -> q [B][D], k, v [B][Hkv*hd]. */
int sd_s_project_qkv(sd_weights* w, int layer, int32_t B, const float* x, float* q, float* k,
                     float* v);
/* finish_block (dense.hpp:31-32): x_out = y + silu(y W_in^T) W_out^T, y = o W_o^T + res. */
int sd_s_finish_block(sd_weights* w, int layer, int32_t B, const float* o, const float* res,
                      float* x_out);
/* output_logits + argmax_token (dense.hpp:35-38); logits may be NULL. */
int sd_s_logits_argmax(sd_weights* w, int32_t B, const float* x, float* logits,
                       int32_t* tokens);
/* apply_linear (dense.hpp:20) over an uploaded tensor (index as in
 * sd_weights_upload, 1..6 per layer, 7 = head). */
int sd_s_apply_linear(sd_weights* w, int layer, int which, int32_t B, const float* x, float* y);

/* The tcgen05 GEMM behind the S-Part on device pointers:
 * C[M][N] = A[M][K] . B[N][K]^T, row-major, both operands K-major;
 * kind SD_DENSE_BF16 (bf16 operands) or SD_DENSE_TF32 (fp32 operands); fused
 * epilogue epi: 0 none, 1 + res (dense.cpp:60), 2 SiLU (dense.cpp:47-49).
 * Writes fp32 C and/or bf16 Cb (either may be NULL). */
int sd_gemm_dev(int kind, int M, int N, int K, const void* A, int64_t lda, const void* B,
                int64_t ldb, float* C, int64_t ldc, void* Cb, int64_t ldcb, int epi,
                const float* res, int64_t ldr, void* stream);

/* -------------------------------------------------------------- runtime
 * The GPU StepComputation (workers.hpp:151-158): decode_step_monolithic
 * (dense.cpp:90-129) with the KV store, S-Part and head on one device. */
int sd_engine_create(sd_weights* w, sd_kv* kv, sd_engine** out);
int sd_engine_destroy(sd_engine* e);
/* StepComputation::compute: features = embedding columns of `tokens`
 * (workers.cpp:629-638) for the batch rows `seqs`; writes next tokens and,
 * when non-NULL, the final pre-head activations [B][D]. Host buffers,
 * synchronous. */
int sd_engine_step(sd_engine* e, int32_t B, const uint64_t* seqs, const int32_t* tokens,
                   int32_t* next_tokens, float* final_x);
/* Same with explicit features x [B][D] (TokenBatch.features). */
int sd_engine_step_features(sd_engine* e, int32_t B, const uint64_t* seqs, const float* x,
                            int32_t* next_tokens, float* final_x, float* logits);
/* StepComputation::retire (workers.hpp:157). */
int sd_engine_retire(sd_engine* e, int32_t n, const uint64_t* seqs);
/* Device-timed step loop for the bench: runs `steps` decode steps over the
 * resident batch (tokens fed back on device), returns device milliseconds. */
int sd_engine_bench(sd_engine* e, int32_t B, const uint64_t* seqs, const int32_t* tokens,
                    int32_t steps, int32_t* next_tokens, double* device_ms);
/* CUDA-event timing of the engine's S-Part GEMM launches (sum of kernel
 * milliseconds and algorithmic flops since the last reset). */
/* enable: 0 off, 1 every GEMM, k > 1 the GEMMs of every k-th layer (and the head) */
int sd_engine_timing(sd_engine* e, int enable);
int sd_engine_timing_read(sd_engine* e, double* ms, double* flops, int64_t* launches, int reset);
/* Two-mini-batch pipeline (workers.cpp:405-452): rows split by seq % 2; the
 * R-Part of one mini-batch runs on r_sms SMs (its own stream) beside the
 * S-Part of the other on the remaining SMs. enable = 0: one batch, one
 * stream (default). */
int sd_engine_pipeline(sd_engine* e, int enable, int r_sms);
/* Process-wide tuning switches, for A/B measurements and the
 * variant-equivalence tests (the defaults are the measured-best paths):
 * "gemm_bn" (force the CTA-pair tile width, 64..256, multiple of 16; 0 = the
 * wave cost model), "gemm_pair" (0: single-CTA tiles), "fused_append" (0:
 * separate KV append kernel), "fused_argmax" (0: logits + argmax kernel),
 * "dist_fuse" (0: scatter kernel for the peer exchange), "attn_mma" (0:
 * CUDA-core attention), "pdl" (0: no programmatic dependent launch),
 * "dist_phases" (1: per-phase DistEngine timing on stderr), "attn_i8_quad"
 * (0: int8 stages copy two positions at a time instead of four),
 * "attn_l2_prefetch", "attn_max_stages" (attention prefetch / ring depth
 * variants), "attn_imma" (0: int8 / int4 scores on fp16 tensor cores
 * instead of integer ones), "attn_rps8" (0: shards of 1-2 kv heads copy
 * four positions at a time instead of eight), "attn_ivalue" (0: int8 /
 * int4 KV with G <= 4 runs the value product on fp16 tensor cores over a dequantized
 * V tile instead of integer ones with p as fixed-point byte limbs; a value
 * > 1 also forces the integer path's int32 -> fp32 flush every that many
 * stages, a test hook). Switches that shape a store's
 * shared-memory layout (attn_max_stages, attn_i8_quad, attn_rps8) take effect
 * for stores created afterwards. Unknown names return SD_ERR_CONFIG. */
int sd_tune(const char* name, int value);
/* Kernel launches issued by this library in this process (all devices). */
int64_t sd_launch_count(void);
/* Synthetic device-generated weights (uniform +-1/sqrt(fan_in), counter
 * hash of `seed`) in the requested dense mode: the full-size bench. */
int sd_weights_synthetic(const sd_model_spec* spec, int dense_mode, uint64_t seed, int device,
                         sd_weights** out);

/* drive_schedule (workers.cpp:547-684) over the GPU engine. cold_start: 0
 * fixed-interval, 1 ramped-limit (scheduler.hpp:99). steps <= 0 runs to
 * completion. The transcript (step, seq, token) is returned through a
 * result handle. */
typedef struct sd_drive_config {
  int32_t batch, target_len, interval, cold_start;
  int64_t steps, load_limit;
  uint64_t seed;
  int32_t record_activations;
} sd_drive_config;
typedef struct sd_drive_result sd_drive_result;
int sd_drive(sd_engine* e, const sd_drive_config* cfg, sd_drive_result** out);
int64_t sd_drive_count(const sd_drive_result* r);
int sd_drive_record(const sd_drive_result* r, int64_t i, int64_t* step, uint64_t* seq,
                    int32_t* token);
const float* sd_drive_activations(const sd_drive_result* r);
double sd_drive_wall_seconds(const sd_drive_result* r);
int sd_drive_destroy(sd_drive_result* r);

/* ---------------------------------------------------------- multi-GPU
 * DistributedComputation (workers.cpp:264-501) on NVLink: every rank is an
 * R-shard holding the sequences ShardMap by-sequence assigns it
 * (mix64(seq) % world, transport.cpp:352-353); S-ranks (rank 0 when
 * s_ranks == 1, the paper's topology; every rank when s_ranks == world)
 * run the S-Part for their home rows (SD_HOME_MODULO above: balanced and
 * shard-affine by default, else seq % s_ranks). Per layer Q/K/V rows go to
 * the owning shard and O rows come back (send_layer / receive_layer,
 * workers.cpp:324-391) as NCCL grouped send/recv or peer stores. Every rank
 * passes the full step batch and reads the tokens of its home rows; the
 * next tokens of the whole batch come back on every rank (final activations
 * for the home rows only). */
typedef struct sd_dist sd_dist;
/* ncclGetUniqueId into `out` (NCCL_UNIQUE_ID_BYTES = 128 bytes) on one rank. */
int sd_nccl_unique_id(void* out, size_t bytes);
/* shard_mode (enum sd_shard_mode, over kv heads): BY_SEQUENCE (default,
 * NCCL or peer exchange), BY_HEAD or HYBRID (peer exchange only); `kv` must
 * hold this rank's head range (sd_shardmap_head_range). nccl_id may be NULL:
 * no NCCL communicator is created and the rank must connect the peer
 * exchange (sd_dist_p2p_*) before its first step; the per-layer exchange and
 * the per-step next-token gather then run as peer stores only (this also
 * lets several ranks share one device). */
int sd_dist_create(sd_weights* weights_or_null, sd_kv* kv, int rank, int world,
                   const void* nccl_id, int s_ranks, int shard_mode, sd_dist** out);
int sd_dist_destroy(sd_dist* d);
/* The reference's two interleaved mini-batches (DistributedComputation with
 * pipelined_ = true, workers.cpp:405-452): rows split by seq % 2 (merged
 * when one side is empty); per layer and mini-batch every rank runs its
 * shard's attention, then the S-Part of that mini-batch's home rows and its
 * next QKV, so one mini-batch's R-Part overlaps the other's S-Part across
 * ranks. With world > 1 it needs the peer exchange (connected first). */
int sd_dist_pipeline(sd_dist* d, int enable);
int sd_dist_step(sd_dist* d, int32_t B, const uint64_t* seqs, const int32_t* tokens,
                 int32_t* next_tokens, float* final_x);
int sd_dist_retire(sd_dist* d, int32_t n, const uint64_t* seqs);
int sd_dist_bench(sd_dist* d, int32_t B, const uint64_t* seqs, const int32_t* tokens,
                  int32_t steps, double* device_ms);
/* drive_schedule over the distributed computation; the result holds the
 * transcript rows this rank produced (its home rows). */
int sd_dist_drive(sd_dist* d, const sd_drive_config* cfg, sd_drive_result** out);
int sd_dist_timing(sd_dist* d, int enable);
int sd_dist_timing_read(sd_dist* d, double* exchange_ms, double* exchange_bytes, int reset);
/* Peer-memory exchange over NVLink in place of NCCL send/recv (same rows,
 * same order): each rank allocates receive buffers for up to `max_rows`
 * rows per mini-batch and writes SD_DIST_IPC_BYTES of CUDA IPC handles; after every rank's
 * handles are gathered (rank order, world * SD_DIST_IPC_BYTES), connect maps
 * the peers' buffers. Every later step scatters rows with direct NVLink
 * stores and an epoch flag per (exchange, source). */
#define SD_DIST_IPC_BYTES 384
int sd_dist_p2p_setup(sd_dist* d, int32_t max_rows, void* handles_out);
int sd_dist_p2p_connect(sd_dist* d, const void* all_handles);
/* Host-only row plan of a step (CPU-testable): home rows grouped by shard,
 * shard rows grouped by source, per-peer counts. Arrays sized B / world. */
int sd_dist_plan(int world, int rank, int s_ranks, int shard_mode, int heads, int32_t B, const uint64_t* seqs,
                 int32_t* home_rows, int32_t* n_home, int32_t* shard_rows, int32_t* n_shard,
                 int32_t* send_counts, int32_t* recv_counts);

/* ------------------------------------------------ SDWP attention worker
 * A B200 R-worker speaking the reference's wire protocol (SDWP frames:
 * "SDWP" | version u8 | type u8 | payload_len u32 | payload, little-endian;
 * transport.hpp / transport.cpp:105-301), as AttentionWorkerSession
 * (workers.cpp:40-160): HELLO, CONFIG (JSON: model, head_start, head_count,
 * wire_precision single|half) -> ack, QKV_BATCH -> append_request + attend
 * on a KvShard in HBM -> O_BATCH, DROP_SEQ (no reply), SHUTDOWN -> stats,
 * typed ERROR replies (codes = the status numbering). The reference's
 * DistributedComputation can use it as a remote R-worker. */
typedef struct sd_rworker sd_rworker;
/* AttentionWorkerConfig: capacity_tokens, storage format (enum sd_kv_format) */
int sd_rworker_create(int64_t capacity_tokens, int kv_format, int device, sd_rworker** out);
int sd_rworker_destroy(sd_rworker* w);
/* Feed stream bytes (any split); every complete frame is handled and the
 * reply frames are returned in *replies (valid until the next call). A bad
 * magic or oversized frame is fatal for the stream: SD_ERR_PROTOCOL. */
int sd_rworker_feed(sd_rworker* w, const uint8_t* bytes, size_t n, const uint8_t** replies, size_t* replies_len);
int sd_rworker_shutdown_requested(const sd_rworker* w, int32_t* out);
/* serve_attention_worker (workers.cpp:162-214): blocking TCP loop on
 * "host:port" (port 0 = any; the bound port is written to port_file when
 * non-NULL); once != 0 returns after the first connection ends; a connection
 * idle for recv_timeout_seconds (> 0) ends its session. The `sd_rworker
 * serve` binary is the reference CLI's `serve` subcommand over this. */
int sd_rworker_serve(const char* listen_addr, const char* port_file, int64_t capacity_tokens, int kv_format,
                     int device, int once, double recv_timeout_seconds);

/* ------------------------------------------- planner inputs and planner
 * The planner's measured inputs on the B200, with the reference bench
 * definitions: T(B) = seconds of one block's S-Part (project_qkv +
 * finish_block of layer 0) at batch B (bench_dense_block, dense.cpp:145-196);
 * R = seconds of attend per token-position per layer for a shard holding all
 * kv heads (bench_attention_per_token, attention.cpp:307-354). Device-timed
 * medians of >= 2 ms samples. */
int sd_bench_dense_block(sd_weights* w, const int32_t* batches, int32_t n, int32_t reps, double* seconds_out);
int sd_bench_attention_per_token(const sd_model_spec* spec, int kv_format, int32_t batch, int32_t seq_len,
                                 int32_t reps, int device, double* r_out);
/* C: token positions of full-depth KV (all layers and kv heads) that fit in
 * the device's free memory minus `reserve_bytes`. */
int sd_kv_capacity_tokens(const sd_model_spec* spec, int kv_format, int device, double reserve_bytes,
                          int64_t* tokens_out);

/* The planner (Eq. 7-11; planner.hpp:25-109, planner.cpp:48-222). Host only. */
typedef struct sd_perf_profile {
  const int32_t* batch;   /* ascending */
  const double* seconds;  /* T(batch) per block */
  int32_t n;
  double r_per_token;
  int64_t capacity_c;
} sd_perf_profile;
typedef struct sd_plan_request {
  int32_t num_layers, target_len;
  int32_t has_latency_budget; /* 0: knee rule; 1: budget (must be > 0) */
  double latency_budget;      /* seconds per full sequence */
  const int32_t* candidates;  /* NULL/0: the profile's batches */
  int32_t n_candidates;
  double knee_threshold;     /* 0.10 in the reference */
  double balance_tolerance;  /* 0.15 */
} sd_plan_request;
enum sd_plan_binding { SD_BIND_LATENCY = 0, SD_BIND_KNEE = 1, SD_BIND_MEMORY = 2 };
typedef struct sd_hardware_plan {
  int32_t batch_size, worker_count;
  double worker_estimate, predicted_seq_seconds, efficiency, balance_residual;
  int32_t balanced, binding_constraint;
  int32_t tightest_batch; /* set with SD_ERR_INFEASIBLE */
} sd_hardware_plan;
int sd_plan(const sd_perf_profile* profile, const sd_plan_request* request, sd_hardware_plan* out);
int sd_plan_batch_size(const sd_perf_profile* profile, const sd_plan_request* request, int32_t* batch_out,
                       int32_t* tightest_out);
int sd_plan_block_seconds(const sd_perf_profile* profile, int32_t batch, double* seconds_out);
int sd_plan_worker_count(const sd_perf_profile* profile, int32_t batch, int32_t target_len, int32_t* workers,
                         double* estimate);
int sd_plan_check_memory(int64_t batch, int64_t target_len, int64_t capacity, int64_t workers,
                         int32_t* feasible, int32_t* min_workers);
int sd_plan_check_balance(const sd_perf_profile* profile, int32_t batch, int32_t target_len, int32_t workers,
                          double tolerance, double* stage_seconds, double* residual, int32_t* accepted);

/* ------------------------------------------------------- ShardMap, load
 * ShardMap (transport.cpp:319-380). */
int sd_shardmap_worker_for(int mode, int num_heads, int workers, uint64_t seq, int head,
                           int32_t* out);
int sd_shardmap_head_range(int mode, int num_heads, int workers, int worker, int32_t* start,
                           int32_t* count);
/* micro_batch_size / cold_start_schedule (scheduler.cpp:10-214):
 * admissions as (step, size, target) triples. */
int sd_micro_batch_size(int batch, int interval, int target_len, int32_t* out);
int sd_cold_start_schedule(int batch, int target_len, int interval, int mode, int64_t horizon,
                           int64_t* triples, int64_t capacity, int64_t* count);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* SD_ABI_H_ */

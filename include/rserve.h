/* rserve-b200 — C-ABI drop-in boundary for RServe's intra-request pipeline
 * (chunked multimodal encode -> embedding tracker -> chunked prefill) on
 * NVIDIA B200 (sm_100a).
 *
 * The reference (arxiv 2509.24381, /root/reference/proj, "lmmsim") exposes
 * this path only as a header-only C++ API with an analytic cost seam; it has
 * no FFI. Each entry point below names the reference interface it replaces
 * (file:line under proj/include/lmmsim/). The C++ API itself is kept
 * verbatim in include/lmmsim/ (our implementation), which the
 * reference's own unit suites compile against unchanged.
 *
 * Conventions
 *   - every function returns rs_status; RS_OK == 0. On error the thread-local
 *     message (rs_last_error) holds the exact what() text the reference
 *     would throw, and the status names the exception class
 *     (reference errors.hpp:23-80).
 *   - token indices / counts are uint64 (request.hpp:28-31), times are double
 *     milliseconds.
 *   - strings returned through char** are malloc'd; release with rs_free.
 *   - device pointers are plain CUDA device addresses; no torch types.
 *   - the product path has no CPU fallback: without a usable sm_100 device,
 *     device entry points fail with RS_ERR_CUDA.
 */
#ifndef RSERVE_H_
#define RSERVE_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define RS_API __attribute__((visibility("default")))
#else
#define RS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per reference exception class ------------------ */
typedef enum rs_status {
  RS_OK = 0,
  RS_ERR_CONFIG = 1,               /* ConfigError            errors.hpp:29 */
  RS_ERR_REGISTRY = 2,             /* RegistryError          errors.hpp:35 */
  RS_ERR_DOUBLE_ENCODE = 3,        /* DoubleEncodeError      errors.hpp:41 */
  RS_ERR_ALIGNMENT = 4,            /* AlignmentError         errors.hpp:47 */
  RS_ERR_DEPENDENCY_VIOLATION = 5, /* DependencyViolation    errors.hpp:54 */
  RS_ERR_INPUT = 6,                /* InputError             errors.hpp:60 */
  RS_ERR_DATA = 7,                 /* DataError              errors.hpp:66 */
  RS_ERR_IO = 8,                   /* IoError                errors.hpp:71 */
  RS_ERR_INTERNAL = 9,             /* InternalError          errors.hpp:77 */
  RS_ERR_SIM = 10,                 /* other SimError                        */
  RS_ERR_CUDA = 20,                /* CUDA runtime / driver / no device     */
  RS_ERR_NCCL = 21,                /* NCCL failure                          */
  RS_ERR_UNKNOWN = 99
} rs_status;

RS_API const char* rs_last_error(void);
RS_API void rs_free(void* p);
/* Build identification, e.g. "rserve-b200 sm_100a tcgen05". */
RS_API const char* rs_version(void);

/* ---- host-side config PODs --------------------------------------------- */
enum { RS_POLICY_VANILLA_PP = 0, RS_POLICY_EPD_BASELINE = 1,
       RS_POLICY_INTRA_ONLY = 2, RS_POLICY_RSERVE = 3 };
enum { RS_PIPELINE_DEFAULT = -1, RS_PIPELINE_CPP = 0, RS_PIPELINE_VANILLA = 1 };
enum { RS_RELEASE_FIRST_STAGE = 0, RS_RELEASE_LAST_STAGE = 1 };
#define RS_WHOLE_REQUEST UINT64_MAX /* encoder_sched.hpp:32-33 kWholeRequest */

typedef struct rs_cost_model { /* cost_model.hpp:37-45 */
  double alpha_enc_ms, beta_enc_ms_per_token;
  double eps_tx_ms, zeta_tx_ms_per_token;
  double gamma_stage_ms, delta_stage_ms_per_token, kappa_attn_ms;
  double tp_speedup;
} rs_cost_model;

typedef struct rs_sim_config { /* simengine.hpp:48-75 SimConfig */
  int32_t policy;          /* RS_POLICY_* */
  int32_t pipeline_mode;   /* RS_PIPELINE_* */
  int32_t stages;
  int32_t encoder_workers;
  uint64_t token_budget;           /* B */
  uint64_t embedding_batch_tokens; /* C, or RS_WHOLE_REQUEST */
  int32_t release_at;      /* RS_RELEASE_* */
  uint32_t hidden_size;
  rs_cost_model cost;
} rs_sim_config;

enum { RS_LAYOUT_ALTERNATING = 0, RS_LAYOUT_CONSECUTIVE_MM = 1,
       RS_LAYOUT_TEXT_FIRST = 2 };
typedef struct rs_int_dist { int32_t uniform; uint64_t lo, hi; } rs_int_dist;
typedef struct rs_template { /* workload.hpp:71-107 RequestTemplate */
  int32_t pattern;
  rs_int_dist num_mm_items, mm_item_tokens, text_segment_tokens;
  double probability;
} rs_template;
typedef struct rs_workload_config { /* workload.hpp:109-136 */
  double arrival_rate, duration_s;
  uint64_t seed;
  const rs_template* templates;
  int32_t n_templates;
  int32_t has_slo;
  double slo_ttft_ms;
} rs_workload_config;

/* ---- host scheduling core (no device needed) ---------------------------
 * Workloads travel as the reference's workload-file text
 * (`id,arrival_ms,slo|-,layout` lines; workload.hpp:217-265).            */

/* generate_workload (workload.hpp:139-172) -> workload text */
RS_API rs_status rs_generate_workload(const rs_workload_config* cfg, char** out_text);

/* run_simulation (simengine.hpp:522-526) on the analytic cost model.
 * out_result: canonical decision log (see DESIGN.md §"Decision log"):
 * per-request records, slices, trace, release order; doubles in shortest
 * round-trip form so equal text == bit-identical results.              */
RS_API rs_status rs_simulate(const char* workload_text, const rs_sim_config* cfg,
                      char** out_result, char** out_journal);

/* One report row (experiment.hpp:72-101 run_cell + metrics.hpp:173-194):
 * generate -> run -> compute_report -> CSV row. slo_ttft_ms < 0: none.   */
RS_API rs_status rs_experiment_cell(const rs_workload_config* wcfg,
                             const rs_sim_config* cfg, double slo_ttft_ms,
                             char** out_csv_row);

/* Algorithm 1 (encoder_sched.hpp:48-74): batches as text lines
 * "request item_idx:start-end,... total". C == RS_WHOLE_REQUEST allowed. */
RS_API rs_status rs_plan_batches(const char* layout, uint64_t request_id,
                          uint64_t c_tokens, char** out_text);

/* ---- device pipeline context -------------------------------------------- */
typedef struct rs_ctx rs_ctx;

enum { RS_MODEL_TINY = 0, RS_MODEL_QWEN25VL_7B = 1, RS_MODEL_QWEN25VL_72B_LLM = 2 };

typedef struct rs_model_config {
  /* vision encoder (ViT + 2x2 patch merger) */
  int32_t vit_dim, vit_layers, vit_heads, vit_ff, vit_window; /* window: merged units/side */
  int32_t vit_fullatt_every;  /* full attention at layers l % every == every-1 */
  int32_t patch_dim;          /* 3*2*14*14 = 1176 */
  /* LLM decoder */
  int32_t llm_dim, llm_layers, llm_q_heads, llm_kv_heads, llm_head_dim, llm_ff;
  int32_t vocab;
  float rope_theta_llm, rope_theta_vit, rms_eps;
  uint64_t weight_seed;
} rs_model_config;

/* Fills the preset shapes: TINY (cfg1), QWEN25VL_7B (cfg2-4), 72B-LLM (cfg5). */
RS_API rs_status rs_model_preset(int32_t preset, rs_model_config* out);

typedef struct rs_ctx_options {
  int32_t device;              /* CUDA ordinal for this process            */
  uint64_t max_prompt_tokens;  /* per-request cap, sizes staging buffers   */
  uint64_t slot_tokens;        /* embedding-slot pool capacity (tokens)     */
  uint64_t kv_tokens;          /* paged-KV pool capacity (tokens)           */
  uint64_t max_chunk_tokens;   /* B upper bound (prefill M)                 */
  uint64_t max_encode_tokens;  /* C upper bound incl. largest item (LLM tokens) */
  int32_t layer_begin, layer_end; /* LLM layers owned here ([0,L) = all)    */
  int32_t with_vit;            /* allocate the vision encoder here           */
  int32_t with_lm_head;        /* allocate final norm + LM head here         */
  int32_t tp_size;             /* tensor-parallel LLM shards (0/1 = none); all on `device` (loopback) */
  int32_t tp_rank;             /* tp_group: this context's rank in [0, tp_size)          */
  int32_t tp_group;            /* 1: one rank of a tp_size-rank TP group (one shard here,
                                  peers in other processes / GPUs, rs_tp_connect)         */
} rs_ctx_options;

RS_API rs_status rs_ctx_create(const rs_model_config* model, const rs_ctx_options* opt,
                        rs_ctx** out);
RS_API rs_status rs_ctx_destroy(rs_ctx* ctx);

/* ---- tracker data plane (device) ----------------------------------------
 * Replaces EmbeddingTracker ctor (tracker.hpp:44-59) + create_tracker
 * (193-198): reserves slot pages for the request, uploads text token ids,
 * gathers text embeddings into the slots (K8), initialises the readiness
 * bitmap with text = 1 and keeps the host tracker mirror.               */
RS_API rs_status rs_request_create(rs_ctx* ctx, uint64_t id, const char* layout,
                            const int32_t* text_token_ids /* may be NULL */);
/* mark_encoded / on_embeddings_ready (tracker.hpp:83-105,
 * token_sched.hpp:184-187): scatter [tokens, d_llm] bf16 rows (device
 * pointer, row-major, in item order) into the item's slots and set its
 * bitmap bits (K6); host mirror is updated and errors mirror the
 * reference (AlignmentError / DoubleEncodeError).                       */
RS_API rs_status rs_mark_encoded(rs_ctx* ctx, uint64_t id, uint64_t start, uint64_t end,
                          const void* embeddings_dev);
/* schedulable_tokens (tracker.hpp:79) from the host mirror, plus the
 * device ready-prefix (K7, warp ballot over the bitmap) for cross-check. */
RS_API rs_status rs_schedulable(rs_ctx* ctx, uint64_t id, uint64_t* host_count,
                         uint64_t* device_count);
/* advance_prefill (tracker.hpp:109-122). */
RS_API rs_status rs_advance_prefill(rs_ctx* ctx, uint64_t id, uint64_t n,
                             uint64_t* out_start, uint64_t* out_end);
/* release (tracker.hpp:126-135) + slot-page free once fully released. */
RS_API rs_status rs_release(rs_ctx* ctx, uint64_t id, uint64_t start, uint64_t end);
RS_API rs_status rs_request_erase(rs_ctx* ctx, uint64_t id);
/* Device bitmap words (ceil(T/32) u32) and slot rows (bf16) read back. */
RS_API rs_status rs_read_bitmap(rs_ctx* ctx, uint64_t id, uint32_t* out_words, uint64_t n_words);
RS_API rs_status rs_read_slots(rs_ctx* ctx, uint64_t id, uint64_t start, uint64_t end,
                        void* out_host_bf16);
/* live / peak / released token accounting of the host mirror. */
RS_API rs_status rs_tracker_stats(rs_ctx* ctx, uint64_t id, uint64_t out[6]);

/* ---- compute entry points ------------------------------------------------
 * encode_time_ms seam (cost_model.hpp:68-71): ViT forward of one
 * Algorithm-1 batch. `items` = (start,end) prompt ranges of the batch's
 * items; patches: host or device bf16 [4*tokens, patch_dim] in item
 * order (window-major patch order within an item).
 * Output: merged embeddings [tokens, d_llm] bf16 in LLM row-major token
 * order, written to *out_embeddings_dev when non-NULL on entry (caller
 * device memory), else to ctx staging (valid until the next encode).      */
RS_API rs_status rs_encode(rs_ctx* ctx, const uint64_t* items, int32_t n_items,
                    const void* patches, int32_t patches_on_host,
                    void** out_embeddings_dev);
/* stage_time_ms seam (cost_model.hpp:76-82): one chunk through this
 * context's layers. slices: n x (request id, start, end). Reads the chunk
 * rows from the request slots (first stage) and appends to the paged KV.
 * When the context owns the LM head, requests whose slice ends at their
 * prompt end get first-token logits (rs_logits).                        */
RS_API rs_status rs_prefill_chunk(rs_ctx* ctx, const uint64_t* slices, int32_t n_slices);
RS_API rs_status rs_logits(rs_ctx* ctx, uint64_t id, float* out_host, int32_t* out_argmax);

/* ---- caller-owned event loop (asynchronous seam) -------------------------
 * For a host scheduler that owns its event loop — the reference's
 * Simulation handlers (simengine.hpp:275-441) calling the cost seam
 * (encode_time_ms / stage_time_ms, cost_model.hpp:68-82) — the launches below
 * return at once (work queued on the context's encode / stage streams, or on
 * `stream` when non-NULL: a cudaStream_t of the context's device) and their
 * completions come back from rs_poll, tagged with the caller's `tag`, in the
 * reference's event classes (simengine.hpp:211-248: encode before stage at
 * equal times, then issue order). Times are device milliseconds since the
 * context's first asynchronous launch. On one GPU the encoder -> prefill
 * link is the reference's zero-cost transfer: the caller's TransferDone is
 * its EncodeDone, at which it calls rs_embeddings_ready.                  */
typedef struct rs_segment {   /* request.hpp:47-52 SegmentSpec */
  int32_t kind;               /* RS_SEG_TEXT / RS_SEG_MULTIMODAL */
  uint64_t tokens;
} rs_segment;
enum { RS_SEG_TEXT = 0, RS_SEG_MULTIMODAL = 1 };
/* = rs_request_create with a POD segment array (request.hpp:94-102 validate
 * errors: RS_ERR_INPUT with the reference's text).                        */
RS_API rs_status rs_request_create_segments(rs_ctx* ctx, uint64_t id, const rs_segment* segs,
                                            int32_t n_segs, const int32_t* text_token_ids);
/* completion classes (PipelineEngine::EventKind numbering) */
enum { RS_EV_ENCODE_DONE = 1, RS_EV_TRANSFER_DONE = 2, RS_EV_STAGE_DONE = 3, RS_EV_CHUNK_COMPLETE = 4 };
typedef struct rs_event {
  int32_t kind;     /* RS_EV_* */
  int32_t stage;    /* pipeline stage (0 on a one-stage context) */
  uint64_t tag;     /* the launch's tag */
  double time_ms;   /* device completion time */
} rs_event;
/* encode_time_ms seam, non-blocking: ViT forward of one Algorithm-1 batch of
 * request `id` (items = (start,end) pairs; patches as for rs_encode; host
 * patches must stay valid until the ENCODE_DONE of `tag`). The embeddings
 * wait in a staging buffer owned by `tag`.                                */
RS_API rs_status rs_encode_batch_async(rs_ctx* ctx, uint64_t id, const uint64_t* items, int32_t n_items,
                                       const void* patches, int32_t patches_on_host, void* stream,
                                       uint64_t tag);
/* on_embeddings_ready (token_sched.hpp:184-187) for every item of encode
 * `tag`, at the caller's TransferDone: host tracker mirror updated at once
 * (reference errors), K6 scatter + bitmap queued after the encode.         */
RS_API rs_status rs_embeddings_ready(rs_ctx* ctx, uint64_t tag);
/* stage_time_ms seam, non-blocking: one chunk (n x (id, start, end)); the
 * slices are validated against the trackers before any is advanced. Its
 * completion is STAGE_DONE and, on a context with the LM head, a
 * CHUNK_COMPLETE at the same time, after which rs_logits serves the
 * requests whose prompt ended in the chunk.                               */
RS_API rs_status rs_prefill_chunk_async(rs_ctx* ctx, const uint64_t* slices, int32_t n_slices,
                                        void* stream, uint64_t tag);
/* release (tracker.hpp:126-135) of [start, end): the slot pages return to the
 * pool once chunk `after_tag` (the last reader) has completed.             */
RS_API rs_status rs_release_async(rs_ctx* ctx, uint64_t id, uint64_t start, uint64_t end,
                                  uint64_t after_tag);
RS_API rs_status rs_request_erase_async(rs_ctx* ctx, uint64_t id, uint64_t after_tag);
/* Completed launches since the last call (<= cap events), in completion
 * order. wait != 0: block until at least one completes (if any pending).  */
RS_API rs_status rs_poll(rs_ctx* ctx, rs_event* out, int32_t cap, int32_t wait, int32_t* n_out);
RS_API rs_status rs_synchronize(rs_ctx* ctx);

/* ---- the engine on the device ------------------------------------------
 * run_simulation (simengine.hpp:522-526) with the B200 backend.
 * clock: 0 = lock-step (event order from the cost model — bit-exact vs the
 * reference; work executed for real), 1 = real clock (GPU timestamps).
 * Payloads (pixels, token ids) are generated from per-request hashes.
 * e2e: inputs staged from pinned host memory inside the run, logits read
 * back to host at completion.                                          */
typedef struct rs_run_options {
  int32_t clock;        /* 0 lock-step, 1 real clock */
  int32_t e2e;          /* 1: H2D inputs / D2H logits inside the run */
  int32_t serialize;    /* 1: encoders share the prefill stream (profiling) */
  uint64_t payload_seed;
  const char* payload_text; /* optional payload file (see below); co-located runs */
  int32_t keep_kv;      /* 1: completed requests keep KV pages + slot for rs_decode */
} rs_run_options;

/* ---- decode after the first token ------------------------
 * The reference fixes the output length to 1: TTFT ends the
 * request. With keep_kv, requests completed by rs_engine_run stay on the
 * device (paged KV, logits slot); rs_decode then runs `n_steps` greedy
 * decode steps batched over the given requests — each step embeds the
 * previous argmax (the first from the prefill logits), runs every layer on
 * one row per request against its paged KV (appending the new K/V), and the
 * LM head + argmax. out_tokens [n_steps][n_requests]; out_logits optional
 * [n_steps][n_requests][vocab]; out_ms = device time of the loop.
 * rs_decode_release frees a kept request.                                 */
RS_API rs_status rs_decode(rs_ctx* ctx, const uint64_t* request_ids, int32_t n_requests,
                           int32_t n_steps, int32_t* out_tokens, float* out_logits,
                           double* out_ms);
RS_API rs_status rs_decode_release(rs_ctx* ctx, uint64_t request_id);

/* ---- tensor parallelism across GPUs ------------------------
 * The reference models TP only as stage_time_ms / tp_speedup
 * (cost_model.hpp:35-36,76-82). A TP group is tp_size contexts created with
 * tp_group = 1, one per GPU (one process each, or several in one process):
 * rank r holds q / kv heads [r H/T, (r+1) H/T) and SwiGLU width slice r, O /
 * down by input columns. Each layer's O and down partials go to the rank's
 * exchange buffer; a reduction kernel signals every rank through flags in
 * peer memory (release / acquire, system scope) and sums the T partials in
 * rank order straight over NVLink — the same bf16 residual on every rank, no
 * NCCL. Setup: every rank exports its buffer (rs_tp_buffer: device pointer +
 * CUDA IPC handle), the caller exchanges them (e.g. torch.distributed
 * all_gather), and every rank calls rs_tp_connect(ptrs, handles) — ptrs[r]
 * for ranks of this process, the IPC handle otherwise. Requests on a rank are
 * KV-only (rs_kv_request_create); rs_tp_prefill runs one chunk whose input
 * rows [M, d] (bf16, device, the chunk's embeddings — the tracker lives on
 * the engine's rank) are updated in place to the last layer's residual; the
 * rank(s) created with_lm_head produce first-token logits (rs_tp_logits).
 * rs_tp_prefill only enqueues (on `stream`, NULL = the context's aux stream):
 * every rank must issue the same chunk sequence.                          */
RS_API rs_status rs_tp_buffer(rs_ctx* ctx, void** out_dev_ptr, void* out_ipc_handle /* 64 B */);
RS_API rs_status rs_tp_connect(rs_ctx* ctx, const void* const* peer_ptrs, const void* ipc_handles);
RS_API rs_status rs_kv_request_create(rs_ctx* ctx, uint64_t id, const char* layout);
RS_API rs_status rs_tp_prefill(rs_ctx* ctx, const uint64_t* slices, int32_t n_slices, void* x_dev,
                               void* stream);
RS_API rs_status rs_tp_logits(rs_ctx* ctx, uint64_t id, float* out_host, int32_t* out_argmax);

/* ---- PD (prefill -> decode) KV transfer -------------------
 * The paper serves EPD-disaggregated (§5.1: encode, prefill and
 * decode on separate nodes); the reference stops at the first token. A
 * request kept after its prefill (keep_kv) is exported as one contiguous
 * device image — a 64-byte header (first token, next M-RoPE id) followed by
 * its paged KV, [tp shard][layer][page][K page | V^T page] — which the
 * caller moves to the decode GPU (NCCL send/recv, CUDA IPC, cudaMemcpyPeer),
 * and imported there as a kept request that rs_decode continues. Both
 * contexts must hold the same LLM layers / kv heads / TP; the importer needs
 * the whole LLM and its head. Export leaves the source request kept (free it
 * with rs_decode_release). Both calls enqueue on `stream` (NULL: the
 * context's aux stream) and return without synchronising.              */
typedef struct rs_kv_meta {
  uint64_t tokens;       /* KV length (prompt tokens)                        */
  uint64_t image_bytes;  /* header + KV pages                               */
  int32_t next_rope;     /* M-RoPE id of the next generated token            */
  int32_t layer_begin, layer_end, kv_heads, head_dim, page_tokens, tp_size;
} rs_kv_meta;
RS_API rs_status rs_kv_image_bytes(rs_ctx* ctx, uint64_t tokens, uint64_t* out_bytes);
RS_API rs_status rs_kv_export(rs_ctx* ctx, uint64_t request_id, void* dst_dev, uint64_t cap_bytes,
                              rs_kv_meta* out_meta, void* stream);
RS_API rs_status rs_kv_import(rs_ctx* ctx, uint64_t request_id, const rs_kv_meta* meta,
                              const void* src_dev, void* stream);

/* ---- payload files ---------------------------------------
 * The reference's workload file (workload.hpp:217-265) carries layouts only.
 * A payload file beside it pins per-segment inputs: image grids and pixel
 * seeds, text token-id seeds or explicit ids:
 *   # rserve payload v1
 *   <req_id>,<segment_index>,M,grid=<gh>x<gw>[;seed=<u64>]
 *   <req_id>,<segment_index>,T,seed=<u64> | ids=<id> <id> ...
 * Errors: RS_ERR_INPUT with "payload line N: ..." / "payload: request ...". */
RS_API rs_status rs_payload_generate(const char* workload_text, uint64_t seed, char** out_text);
RS_API rs_status rs_payload_validate(const char* workload_text, const char* payload_text,
                                     int32_t vocab, char** out_normalized);
typedef struct rs_run_stats {
  double wall_ms;            /* host wall time of the run                 */
  double gpu_ms;             /* first launch -> last completion (events)  */
  uint64_t h2d_bytes, d2h_bytes;
  uint64_t kernel_launches;  /* our kernels launched during the run       */
  double encode_gpu_ms, prefill_gpu_ms; /* summed per-op device time      */
  double host_max_gap_ms;    /* longest host stretch between engine polls  */
  double host_last_seen_ms;  /* host clock when the last completion was seen */
  double host_max_call_ms;   /* longest backend call (launch / scatter)    */
  int32_t host_max_call_kind; /* 0 encode, 1 stage, 2 scatter, 3 transfer  */
  int32_t reserved0;
  double host_max_launch_ms; /* longest single kernel-launch API call     */
  double host_finish_sync_ms; /* final device synchronise of the run       */
} rs_run_stats;
RS_API rs_status rs_engine_run(rs_ctx* ctx, const char* workload_text,
                        const rs_sim_config* cfg, const rs_run_options* opt,
                        char** out_result, char** out_journal,
                        rs_run_stats* out_stats);

/* ---- EP disaggregation: encoders and prefill stages on separate GPUs ----
 * The paper's EP deployment (RServe §4; the reference models it only as the
 * eps/zeta transfer cost, cost_model.hpp:84-88, and stages > 1,
 * simengine.hpp:494-515). Ranks: P_s = s (s < stages), E_w = stages + w.
 * Rank 0 (P0) runs the engine, the device tracker and prefill stage 0;
 * encoder ranks run the ViT; ranks 1..stages-1 run later LLM layers (the
 * last one holds the LM head). Messages go over one directed link per rank
 * pair: NCCL (one process per GPU) or loopback (all ranks are threads of
 * this process, each with its own rs_ctx, on any devices).              */
typedef struct rs_ep rs_ep;
typedef struct rs_ep_options {
  int32_t stages;      /* prefill ranks (>= 1)                               */
  int32_t encoders;    /* encoder ranks (>= 1)                               */
  int32_t transport;   /* 0 loopback, 1 NCCL, 2 CUDA-IPC peer memory         */
  int32_t rank;        /* NCCL / IPC: this process's rank; loopback: ignored */
  int32_t device;      /* CUDA device of this rank (loopback: of all ranks)  */
  const void* nccl_ids;/* NCCL: n_links x 128-byte ncclUniqueId, links order */
  uint64_t slot_bytes; /* IPC: mailbox slot size (>= the largest message)    */
  const char* shm_name;/* IPC: POSIX shm name shared by the group's ranks    */
} rs_ep_options;
/* Directed links (src, dst) of a topology, in creation order: pairs must
 * hold 2 * n entries (NULL: only *n_links is written).                    */
RS_API rs_status rs_ep_links(int32_t stages, int32_t encoders, int32_t* n_links, int32_t* pairs);
RS_API rs_status rs_nccl_unique_id(void* out128);
RS_API rs_status rs_ep_create(const rs_ep_options* opt, rs_ep** out);
RS_API rs_status rs_ep_destroy(rs_ep* ep);
/* IPC only, after rs_ep_create on every rank: this rank's receive handles
 * (mailboxes, events) -> blob; then connect with all ranks' blobs (rank
 * order, exchanged by the caller's plumbing, e.g. torch.distributed).      */
RS_API rs_status rs_ep_ipc_export(rs_ep* ep, void* out, uint64_t capacity, uint64_t* size);
RS_API rs_status rs_ep_ipc_connect(rs_ep* ep, const void* blobs, const uint64_t* sizes, int32_t n);
/* Worker ranks (NCCL): payloads of the run (encoders), then serve until P0
 * sends STOP at the end of its rs_ep_engine_run.                          */
RS_API rs_status rs_ep_worker_prepare(rs_ep* ep, rs_ctx* ctx, const char* workload_text,
                                      uint64_t payload_seed, int32_t e2e);
RS_API rs_status rs_ep_worker_run(rs_ep* ep, rs_ctx* ctx);
/* P0: one engine run. Loopback: `workers` holds the contexts of ranks
 * 1..world-1 (run on threads of this call); NCCL: workers = NULL.         */
RS_API rs_status rs_ep_engine_run(rs_ep* ep, rs_ctx* p0, rs_ctx* const* workers,
                                  const char* workload_text, const rs_sim_config* cfg,
                                  const rs_run_options* opt, char** out_result,
                                  char** out_journal, rs_run_stats* out_stats);
/* Engine-backed experiment cell (the device counterpart of
 * rs_experiment_cell / experiment.hpp run_cell): generates the workload of
 * `wcfg`, runs it through the device engine — co-located on `ctx` (ep NULL)
 * or EP with `ctx` as P0 — and returns the report CSV row (metrics.hpp
 * report_csv_row) plus the Chrome trace (trace_to_json_text) whose spans
 * are the engine's op launches and their CUDA-event completions.       */
RS_API rs_status rs_engine_cell(rs_ctx* ctx, rs_ep* ep, rs_ctx* const* workers,
                                const rs_workload_config* wcfg, const rs_sim_config* cfg,
                                double slo_ttft_ms, const rs_run_options* opt,
                                char** out_csv_row, char** out_trace_json, rs_run_stats* out_stats);
/* Control-message codec (host only): text form <-> the 32 KB wire message. */
RS_API rs_status rs_ep_ctrl_pack(const char* text, void* out_msg, uint64_t msg_bytes);
RS_API rs_status rs_ep_ctrl_unpack(const void* msg, uint64_t msg_bytes, char** out_text);

#ifdef __cplusplus
}  /* extern "C" */
#endif
#endif  /* RSERVE_H_ */

/*
 * tcb.h — C ABI of tc-b200, the B200-native execution path for the Tensor
 * Comprehensions benchmark operators (arXiv 1802.04730).
 *
 * This is the drop-in boundary. It mirrors the paper's framework-agnostic
 * ExecutionEngine (define / inferOutputTensorInfo /
 * compile(name, inputs, outputs, options) -> handle / run(name, inputs,
 * outputs, handle, profile) -> Duration) and replaces, on the reference
 * side (proj/, C++ only, no C ABI of its own):
 *
 *   tcb_define          lang::parse + pipeline::check
 *                       (proj/include/tc/lang/parser.h:20, proj/src/pipeline.cc:36-43)
 *   tcb_infer_outputs   sem::inferRanges shapes of the returns
 *                       (proj/src/sem/ranges.cc:599-601)
 *   tcb_compile         pipeline::specialize + pipeline::compile
 *                       (proj/src/pipeline.cc:45-101; proj/include/tc/pipeline.h:64-66)
 *                       + the compile-time cache replay the spec gives the CLI
 *
 *   tcb_run             backend::emulate, the executor
 *                       (proj/src/backend/emulator.cc:448-559; emulator.h:60)
 *                       — with host tensors it is also the TensorMap-in /
 *                       TensorMap-out call of backend::interpretReference
 *                       (proj/src/backend/interpreter.cc:301-349)
 *   tcb_tune            tuner::tune (proj/src/tuner/genetic.cc:383-481)
 *   tcb_cache_*         cache::Cache lookup/update/save/load/purge/setHistoryPath
 *                       (proj/include/tc/cache/cache.h:91-125)
 *   tcb_session_inputs  tuner::makeSessionInputs (proj/src/tuner/genetic.cc:255-291)
 *   tcb_options_*       tuner::MappingOptions validate/toJson/fromJson/digest,
 *                       baselineOptions (proj/src/tuner/options.cc:57-208)
 *   tcb_canonical       cache::canonicalize + CacheKey::lookupKey
 *                       (proj/src/cache/cache.cc:233-281)
 *
 * Conventions
 *   - Every function returns 0 on success, otherwise (ErrorKind + 1) with the
 *     reference's ErrorKind numbering (proj/include/tc/support/diagnostics.h:
 *     36-68), extended by TCB_ERR_NOKERNEL and TCB_ERR_CUDA. The message of
 *     the last failure on the calling thread is tcb_last_error().
 *   - Tensors are dense row-major; the library never owns tensor memory.
 *     `location` says whether `data` is a device pointer (TCB_DEVICE) or a
 *     host pointer (TCB_HOST; tcb_run then copies in and out itself).
 *   - Returns that the definition reads before writing (C3's `+=` target,
 *     MLP3's pass-through O1) are in/out: their incoming contents are used.
 *   - Handles are owned by the engine. tcb_run is safe to call concurrently
 *     on distinct streams; define/compile/tune serialise on the engine lock,
 *     cache operations on the cache lock.
 */
#ifndef TCB_H
#define TCB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCB_F32 0
#define TCB_I32 1
#define TCB_DEVICE 0
#define TCB_HOST 1
#define TCB_MAX_RANK 8

/* error codes: ErrorKind + 1 (diagnostics.h:36-68) */
#define TCB_OK 0
#define TCB_ERR_PARSE 1
#define TCB_ERR_NAME 2
#define TCB_ERR_UNSUPPORTED_CALL 3
#define TCB_ERR_UNDER_CONSTRAINED 4
#define TCB_ERR_AMBIGUOUS 5
#define TCB_ERR_EMPTY_RANGE 6
#define TCB_ERR_LIVENESS 7
#define TCB_ERR_OUT_OF_BOUNDS 8
#define TCB_ERR_UNINITIALIZED_READ 9
#define TCB_ERR_MAPPING_INVALID 13
#define TCB_ERR_INDEX_OUT_OF_RANGE 16
#define TCB_ERR_DEGENERATE_POPULATION 19
#define TCB_ERR_NO_VIABLE_CANDIDATE 20
#define TCB_ERR_CORRUPT_STORE 21
#define TCB_ERR_MISSING_BINDING 22
#define TCB_ERR_SHAPE_MISMATCH 23
#define TCB_ERR_IO 24
#define TCB_ERR_INTERNAL 25
#define TCB_ERR_NOKERNEL 26
#define TCB_ERR_CUDA 27

/* arithmetic of a compiled handle (tcb_compile_ex) */
#define TCB_MATH_FFMA 0   /* default: FFMA-exact kernels, bit-identical to the reference interpreter */
#define TCB_MATH_TF32 1   /* tcgen05 .kind::tf32 tensor cores (GEMM-NT, FC chains, gconv, 3KRU); tolerance DESIGN.md §2 */
#define TCB_MATH_3XTF32 3 /* tcgen05 TF32 with hi/lo operand split (3 MMAs): near-fp32 accuracy */

/* run flags */
#define TCB_RUN_PROFILE 1  /* time the launch with CUDA events (synchronises) */
#define TCB_RUN_NOCHECK 2  /* skip the post-launch device error check (graph capture) */
#define TCB_RUN_ASYNC 4    /* host tensors: return once the H2D copies, the launch and the D2H copies
                            * are enqueued on `stream`; the caller synchronises the stream before
                            * reading outputs or reusing inputs (pinned buffers make the copies
                            * asynchronous). Two async host runs of one handle must share a stream. */

typedef struct tcb_tensor {
  void* data;
  int32_t dtype;    /* TCB_F32 | TCB_I32 */
  int32_t rank;     /* 0..TCB_MAX_RANK; rank 0 in compile() = "shape not given" */
  int64_t shape[TCB_MAX_RANK];
  int32_t location; /* TCB_DEVICE | TCB_HOST */
  int32_t reserved;
} tcb_tensor;

typedef struct tcb_engine tcb_engine;

const char* tcb_version(void);
const char* tcb_last_error(void);
/* "B200 sm_100 148 SMs ..." for device `dev`; fails without a GPU */
int tcb_device_info(int dev, char* buf, int len);
/* measured device peaks not in MEASURED_PEAKS.json, as JSON:
 * {"ffma_tflops": fp32 fma.rn throughput, ...}; fails without a GPU */
int tcb_measure_peaks(int dev, char* buf, int len);

int tcb_engine_create(tcb_engine** out);
void tcb_engine_destroy(tcb_engine* e);

/* ExecutionEngine::define — parse and check every def of `tc_source`. */
int tcb_define(tcb_engine* e, const char* tc_source);
/* the built-in operator corpus (tc/ops.tc) as TC source */
const char* tcb_builtin_ops(void);

/* number of parameters / returns of a defined def, and their names */
int tcb_def_signature(tcb_engine* e, const char* name, int* n_params, int* n_returns, char* names,
                      int names_len /* "p0,p1,...;r0,r1,..." */);

/* ExecutionEngine::inferOutputTensorInfo. `outputs` may carry the shapes of
 * returns that are read but never written (rank>0), others rank 0. Fills
 * rank/shape/dtype of every return. */
int tcb_infer_outputs(tcb_engine* e, const char* name, const tcb_tensor* inputs, int n_inputs,
                      tcb_tensor* outputs, int n_outputs);

/* ExecutionEngine::compile. options_json NULL ⇒ use the cache's best entry
 * for (canonical TC, shapes, target) when present, else the family default.
 * Writes the handle. */
int tcb_compile(tcb_engine* e, const char* name, const tcb_tensor* inputs, int n_inputs,
                const tcb_tensor* outputs, int n_outputs, const char* options_json, uint64_t* handle);

/* compile with an explicit arithmetic (TCB_MATH_*). Tensor-core modes exist
 * for tmm, tbmm, C3, MLP1, 2FCRelu, MLP3, gconv and 3KRU; other defs fail with
 * TCB_ERR_MAPPING_INVALID. Their cache entries carry the target suffix
 * " math=<mode>" and never mix with the exact ones. */
int tcb_compile_ex(tcb_engine* e, const char* name, const tcb_tensor* inputs, int n_inputs,
                   const tcb_tensor* outputs, int n_outputs, const char* options_json, int math,
                   uint64_t* handle);

/* ExecutionEngine::run. stream: a cudaStream_t (NULL = legacy default).
 * With TCB_RUN_PROFILE, *duration_ns receives the device time of the call. */
int tcb_run(tcb_engine* e, uint64_t handle, const tcb_tensor* inputs, int n_inputs,
            const tcb_tensor* outputs, int n_outputs, void* stream, int flags, int64_t* duration_ns);

/* Batch sharding, one process per GPU (the reference has
 * no distributed code — the paper used several GPUs only to tune,
 * PAPER.md:1512-1521). Every registered form has one independent outer
 * dimension (TMM/C3 rows, TBMM batches, FC-chain rows, 3-KRU M, gconv N,
 * LUT rows) and no reduction across it. tcb_shard_range gives rank `rank`'s
 * balanced contiguous slice [lo, hi) of that dimension (the first
 * extent % world ranks get one extra: TBMM 500 over 8 = 63 x 4, 62 x 4).
 * tcb_run_shard runs only that slice of a handle compiled for the FULL
 * shapes, reading and writing the full device tensors in place (weights
 * replicated on every rank). The caller then all-gathers the output slices
 * (ncclAllGather / torch.distributed; shard.py does it). No host tensors. */
int tcb_shard_range(tcb_engine* e, uint64_t handle, int rank, int world, int64_t* lo, int64_t* hi,
                    int64_t* extent);
int tcb_run_shard(tcb_engine* e, uint64_t handle, const tcb_tensor* inputs, int n_inputs,
                  const tcb_tensor* outputs, int n_outputs, int rank, int world, void* stream, int flags);

/* releases a compiled handle: its device staging buffers and error flag are
 * freed after its last stream drains; the handle id is not reused and any
 * later use of it fails with TCB_ERR_NAME. The caller must not release a
 * handle another thread is running. */
int tcb_release(tcb_engine* e, uint64_t handle);

/* synchronises the handle's last stream and reports a device-side error
 * (IndexOutOfRange from a data-dependent subscript) raised since the last check */
int tcb_check(tcb_engine* e, uint64_t handle);

/* JSON description of a compiled handle: form, family, kernel variant,
 * options, options source ("explicit" | "cache" | "default"), algorithmic
 * flops/bytes, canonical TC, cache lookup key. */
int tcb_describe(tcb_engine* e, uint64_t handle, char* buf, int len);

/* tuner::tune on the GPU. tune_options_json keys (all optional):
 * population (100), generations (25), mutation_rate (0.05), seed (0),
 * timing_iters (10), cold_l2 (true: a 2x-L2 buffer is rewritten before each
 * timed launch), session_log (path), use_baselines (true),
 * math ("ffma" | "tf32" | "3xtf32": tune the tcgen05 tile/split genes; a
 * candidate must then agree with the mode's default plan within the stated
 * tolerance instead of bit-for-bit). Writes the best MappingOptions JSON.
 * Every evaluated candidate updates the process cache (min-update; the
 * tensor-core modes under the " math=<mode>" target). */
int tcb_tune(tcb_engine* e, const char* name, const tcb_tensor* inputs, int n_inputs,
             const tcb_tensor* outputs, int n_outputs, const char* tune_options_json, char* best_json,
             int best_len);

/* process-wide compilation cache (TCCACHE 1 format) */
int tcb_cache_load(const char* path);
int tcb_cache_save(const char* path);
int tcb_cache_size(void);
int tcb_cache_purge(void);
int tcb_cache_set_history(const char* path);
int tcb_cache_serialize(char* buf, int len);
int tcb_cache_deserialize(const char* text);
/* best cached options for (def, shapes); TCB_ERR_IO-free miss: returns 0 and *hit = 0 */
int tcb_cache_lookup(tcb_engine* e, const char* name, const tcb_tensor* inputs, int n_inputs,
                     const tcb_tensor* outputs, int n_outputs, int* hit, char* options_json, int len);
/* inject an entry (origin "injected") */
int tcb_cache_inject(tcb_engine* e, const char* name, const tcb_tensor* inputs, int n_inputs,
                     const tcb_tensor* outputs, int n_outputs, const char* options_json, int64_t cost);

/* canonical TC text and cache lookup key for (def, shapes) */
int tcb_canonical(tcb_engine* e, const char* name, const tcb_tensor* inputs, int n_inputs,
                  const tcb_tensor* outputs, int n_outputs, char* canon, int canon_len, char* key,
                  int key_len);

/* tuner::makeSessionInputs into caller-owned HOST tensors (parameters in
 * declaration order; data must hold the inferred shape) */
int tcb_session_inputs(tcb_engine* e, const char* name, const tcb_tensor* inputs, int n_inputs,
                       const tcb_tensor* outputs, int n_outputs, uint64_t seed);
/* fill n floats (or int32s) from mt19937_64(seed): U[lo,hi) / integers [lo,hi) */
int tcb_fill_uniform(void* host, int64_t n, int32_t dtype, uint64_t seed, double lo, double hi);

/* MappingOptions helpers */
int tcb_options_validate(const char* options_json);
int tcb_options_normalize(const char* options_json, char* out, int len); /* fromJson→toJson */
int tcb_options_digest(const char* options_json, char* out, int len);
int tcb_options_baseline(int i, char* out, int len); /* reference presets 0..2 */
int tcb_options_default(tcb_engine* e, const char* name, const tcb_tensor* inputs, int n_inputs,
                        const tcb_tensor* outputs, int n_outputs, char* out, int len);

/* TCTN1 tensor files, byte-compatible with the reference's
 * writeTensorFile / readTensorFile (proj/src/support/tensor_data.cc:122-189).
 * read: fills a TCB_HOST tensor whose data the caller releases with
 * tcb_tensor_file_free. Malformed / truncated files fail with TCB_ERR_IO. */
int tcb_tensor_file_write(const char* path, const tcb_tensor* host_tensor);
int tcb_tensor_file_read(const char* path, tcb_tensor* out_host_tensor);
void tcb_tensor_file_free(void* data);

/* declared parameters of a defined def, as JSON:
 * {"params": [{"name", "elem": "float"|"int", "dims": [symbol or literal...]}],
 *  "returns": [...], "inout_returns": [...]}  (binds CLI --sizes to shapes) */
int tcb_def_params(tcb_engine* e, const char* name, char* buf, int len);
/* every cache entry as a JSON array (cache list / inspect) */
int tcb_cache_entries(char* buf, int len);

/* dst[r][:] = [src_0[r][:] | src_1[r][:] | ...] on the device (row-major,
 * `rows` rows, widths[i] columns each, 1..8 sources). The production
 * model's concat between 2LUT/C3 and MLP1, which TC
 * itself cannot express. */
int tcb_concat_cols(const float* const* srcs, const int64_t* widths, int n, int64_t rows, float* dst,
                    void* stream);

/* pinned host memory for TCB_HOST tensors (cudaMallocHost) */
int tcb_host_alloc(void** p, int64_t bytes);
int tcb_host_free(void* p);
/* device memory and synchronisation for hosts that do not link the CUDA
 * runtime themselves (the `tcb` CLI's latency verb): cudaMalloc / cudaFree,
 * cudaMemcpy (kind inferred from the pointers), cudaStreamSynchronize */
int tcb_device_alloc(void** p, int64_t bytes);
int tcb_device_free(void* p);
int tcb_copy(void* dst, const void* src, int64_t bytes);
int tcb_stream_sync(void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TCB_H */

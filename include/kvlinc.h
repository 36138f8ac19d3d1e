/*
 * kvlinc.h — C ABI of the B200-native KVLinC decode hot path.
 *
 * The reference (`quantkv`, /root/reference/pkg/src/quantkv) is a pure NumPy
 * package; its "FFI" for this path is its public Python API.  Every entry point
 * below replaces one reference function (cited file:line) and is what a
 * ctypes / cffi binding of that API binds.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers, caller-allocated, C-contiguous.
 *   - `stream` is a cudaStream_t passed as void*; every call is stream-ordered
 *     and asynchronous; nothing here synchronises the device.
 *   - Every call returns 0 on success or a KVLC_E* code; kvlc_last_error()
 *     returns a thread-local message carrying the reference's ValueError text
 *     ("query shape", "block_tokens", "empty cache", "power of two", ...).
 *   - There is no CPU fallback: a host without an sm_100 device gets
 *     KVLC_ENODEV from every compute entry point.
 *
 * Two families:
 *   kvlc_ref_*   reference-semantics kernels in float64 for any (d, G, bits,
 *                rank): the per-head drop-in `KVCacheState` / `quantize_tensor`
 *                / `decode_step_blocked` shim is built on these.
 *   kvlc_*       the serving path: batched [B, Hkv] 2-bit cache at d = G = 128,
 *                R = 128, D = 256, bf16 activations, fp16 metadata, fp32 S/P;
 *                fused flush (quantize+FWHT+state update) and the fused
 *                split-KV GQA decode + LSE combine.
 */
#ifndef KVLINC_H
#define KVLINC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVLC_OK 0
#define KVLC_EINVAL 1    /* bad argument: message mirrors the reference ValueError */
#define KVLC_ECUDA 2     /* CUDA runtime error */
#define KVLC_ENODEV 3    /* no sm_100 device */
#define KVLC_ENOSPC 4    /* workspace / capacity too small */

#define KVLC_AXIS_TOKEN 0
#define KVLC_AXIS_CHANNEL 1
#define KVLC_PLACE_PRE 0
#define KVLC_PLACE_POST 1

/* ------------------------------------------------------------------------ */
/* library                                                                  */
/* ------------------------------------------------------------------------ */
int kvlc_version(void);
const char* kvlc_last_error(void);
/* 1 when a CUDA device of compute capability 10.x is visible. */
int kvlc_device_ok(void);

/* ------------------------------------------------------------------------ */
/* reference-semantics kernels (float64)                                    */
/* ------------------------------------------------------------------------ */

/* pack_codes (quantize.py:71-94): codes u8 [rows][n] -> words u32
 * [rows][ceil(n/L)], little-endian lanes, L = 16/8/8/4 for bits 2/3/4/8. */
int kvlc_ref_pack(const uint8_t* codes, int64_t rows, int64_t n, int bits,
                  uint32_t* words, void* stream);

/* unpack_codes (quantize.py:97-114): words [rows][nwords] -> codes [rows][count]. */
int kvlc_ref_unpack(const uint32_t* words, int64_t rows, int64_t nwords,
                    int64_t count, int bits, uint8_t* codes, void* stream);

/* quantize_tensor (quantize.py:220-239) with _quantize_rows (quantize.py:189-209):
 * x [rows][cols] float64.  token axis: words [rows][ceil(cols/L)], scales/zeros
 * [rows][ceil(cols/G)].  channel axis: words [ceil(rows/L)][cols], scales/zeros
 * [ceil(rows/G)][cols].  codes_scratch: rows*cols bytes.  Bit-exact codes and
 * float64 scales (IEEE division, half-to-even rounding, scale-0 groups). */
int kvlc_ref_quantize(const double* x, int64_t rows, int64_t cols, int bits,
                      int group, int axis, uint32_t* words, double* scales,
                      double* zeros, uint8_t* codes_scratch, void* stream);

/* QuantizedTensor.dequantize (quantize.py:174-180, 212-217): float64 out [rows][cols]. */
int kvlc_ref_dequantize(const uint32_t* words, const double* scales,
                        const double* zeros, int64_t rows, int64_t cols,
                        int bits, int group, int axis, double* out, void* stream);

/* rotate (hadamard.py:45-57) in float64 as the reference computes it: a dense
 * product with the Sylvester matrix H (sequential FMA over the inner index, the
 * reference's x @ H order; bit-identical to numpy/OpenBLAS on the golden
 * vectors).  post: out = x @ H (x [rows][dim]);  pre: out = H @ x (x [dim][cols]).
 * dim must be a power of two <= 4096.  (The serving flush uses a warp-shuffle
 * FWHT with an exact fallback near rounding ties.) */
int kvlc_ref_rotate(const double* x, int64_t rows, int64_t cols, int placement,
                    double* out, void* stream);

/* feature_map (adapter.py:80-88): out [n][2h] = [softmax(x W1), softmax(x W2)],
 * x [n][d], W1/W2 [d][h], float64. */
int kvlc_ref_feature_map(const double* x, int64_t n, int d, const double* w1,
                         const double* w2, int h, double* out, void* stream);

/* Causal attention over one head, float64 (attention.py:50-57, 99-155): q, k, v
 * [n][d].  shifted != 0: attention_reference (max-shifted softmax; `weights`,
 * optional, receives the [n][n] softmax rows).  shifted == 0: the corrected
 * forms, raw exponentials plus phi_q(q_t) . phi_k(k_err_i) from phq / phk
 * [n][rank] (NULL: no adapter): out_t = sum (e + f) v / sum (e + f). */
int kvlc_ref_attention(const double* q, const double* k, const double* v, int64_t n,
                       int d, const double* phq, const double* phk, int rank,
                       int shifted, double* weights, double* out, void* stream);

/* Corrected causal prefill attention, fast path (attention.py:99-155: the quadratic and
 * recurrent forms give the same outputs): for every head and query t,
 *   out_t = sum_{i<=t} (e^{q_t.k_i/sqrt(128)} + phq_t . phk_i) v_i / sum_{i<=t} (...)
 * q, k (the dequantized keys), v (dequantized values), out: fp32 [heads][n][128];
 * phq = phi_q(q), phk = phi_k(k_err): fp32 [heads][n][256] (rank 256), or rank 0 and NULL
 * (no adapter).  Tensor cores (mma.sync, fp16 hi / lo operands, fp32 accumulation); the
 * exponentials are shifted by max(0, running max) with the correction scaled alike.
 * Workspace: kvlc_corrected_attention_workspace(n, heads, rank) bytes. */
size_t kvlc_corrected_attention_workspace(int64_t n, int heads, int rank);
int kvlc_corrected_attention(const float* q, const float* k, const float* v, const float* phq,
                             const float* phk, int64_t n, int heads, int rank, float* out,
                             void* ws, size_t ws_bytes, void* stream);

/* Adapter calibration, the trainer's inner loop (adapter.py:180-251), float64 device
 * arrays: for query positions pos[b] (int32) sharing keys 0..n-1 with the causal mask,
 * the batched corrected-row cross-entropy (loss, one double) and its gradients
 * g1q/g2q/g1k/g2k [d][rank/2] for the weights w1q/w2q/w1k/w2k [d][rank/2]
 * (_batched_loss_and_grads).  a_full [n][n] full-precision attention rows, q / khat /
 * kerr [n][d].  Workspace: kvlc_adapter_grads_workspace(n, b, d, rank) bytes. */
size_t kvlc_adapter_grads_workspace(int64_t n, int b, int d, int rank);
int kvlc_adapter_grads(const double* a_full, const double* q, const double* khat,
                       const double* kerr, int64_t n, int d, const int32_t* pos, int b,
                       const double* w1q, const double* w2q, const double* w1k,
                       const double* w2k, int rank, double* g1q, double* g2q, double* g1k,
                       double* g2k, double* loss, void* ws, size_t ws_bytes, void* stream);
/* AdamState.step (adapter.py:230-251) on one weight tensor in place: moments m, v, step
 * count `step` (>= 1) for the bias correction. */
int kvlc_adam_step(double* w, double* m, double* v, const double* g, int64_t count, double lr,
                   double beta1, double beta2, double eps, int64_t step, void* stream);

/* One flush of a per-head cache (cache.py:132-158): the oldest `group`
 * residual tokens k_blk/v_blk [group][d] are quantized (keys channel-wise,
 * values optionally post-rotated then token-wise) and, when w1k != NULL, the
 * adapter states are updated token by token in append order:
 *     S[d][rank] += outer(v_q[i], phi_k(k_err[i])),  P[rank] += phi_k(k_err[i]).
 * Outputs: kwords [ceil(group/L)][d], kscales/kzeros [1][d]; vwords
 * [group][ceil(d/L)], vscales/vzeros [group][ceil(d/group)].
 * scratch: kvlc_ref_flush_scratch() bytes. */
size_t kvlc_ref_flush_scratch(int d, int group, int rank);
int kvlc_ref_flush(const double* k_blk, const double* v_blk, int d, int group,
                   int bits, int rotate, const double* w1k, const double* w2k,
                   int rank, uint32_t* kwords, double* kscales, double* kzeros,
                   uint32_t* vwords, double* vscales, double* vzeros,
                   double* s_state, double* p_state, void* scratch, void* stream);

/* decode_step_blocked (attention.py:197-276) on one per-head cache.
 *   q [d] float64; keys: n_chunks chunks of kwords [ceil(G/L)][d] with
 *   kscales/kzeros [n_chunks][d]; values: vwords [nq][ceil(d/L)],
 *   vscales/vzeros [nq][ceil(d/G)]; residual rk/rv [nr][d] float64.
 *   Correction (w1q != NULL and s_state != NULL): phi_q(q) from W1q/W2q
 *   [d][rank/2], corr_num = S phi, corr_den = P . phi.
 *   block_tokens >= 1; literal != 0 selects literal_correction.
 *   out [d] float64.  Partials (optional, may be NULL): y [nb+1][d], m, l
 *   float32, nb = ceil(nq/block) (+1 row when nr > 0) — DecodePartial
 *   (attention.py:41-47).  scratch: kvlc_ref_decode_scratch() bytes. */
size_t kvlc_ref_decode_scratch(int d, int64_t nq, int64_t nr, int block, int rank);
int kvlc_ref_decode(const double* q, int d, int group, int bits, int rotated,
                    int64_t n_chunks, const uint32_t* kwords,
                    const double* kscales, const double* kzeros,
                    const uint32_t* vwords, const double* vscales,
                    const double* vzeros, int64_t nr, const double* rk,
                    const double* rv, const double* w1q, const double* w2q,
                    const double* s_state, const double* p_state, int rank,
                    int block_tokens, int literal, double* out, float* part_y,
                    float* part_m, float* part_l, void* scratch, void* stream);

/* ------------------------------------------------------------------------ */
/* serving path: batched 2-bit cache, d = G = 128, R = 128, D = 256          */
/* ------------------------------------------------------------------------ */

#define KVLC_D 128
#define KVLC_G 128
#define KVLC_R 128
#define KVLC_RANK 256
#define KVLC_SLOTS 256 /* residual ring capacity R + G */

/* Device cache descriptor (POD; every pointer is device memory).
 * One (b, kv-head) pair is a "unit".  Layouts (u = b*Hkv + kvh):
 *   kcodes [u][max_chunks][1024] u32, vcodes [u][max_chunks][1024] u32: the
 *          2-bit codes of a chunk (G = 128 tokens x 128 channels) in the
 *          decode kernels' fragment-native word order (NOT the reference's
 *          word order; kvlc_export_chunk() / kvlc_serialize_unit() return the
 *          reference layout, kvlc_deserialize_unit() writes this one).  Word
 *          wi = (w*32 + lane)*8 + i, lane = 4*g + t0 (w, g, i in 0..3 / 0..7 /
 *          0..7, t0 in 0..3) holds 16 codes, code (byte q, pair j) at bit
 *          (8*q + 2*j + 2) mod 32 (the unrotated word rotated left by 2):
 *            K word: byte q = channel 16*i + 2*t0 + {0,8,1,9}[q],
 *                    pair j = token 32*w + 4*g + j;
 *            V word: byte q = token 32*w + 8*t0 + 2*(i>>2) + {0,1,4,5}[q],
 *                    pair j = channel 32*(i&3) + 8*j + g.
 *          (tests/test_gpu_batched.py::test_documented_code_word_layout checks
 *          this formula against kvlc_export_chunk.)
 *   kscale/kzero [u][max_chunks][128] f16 (per channel), vscale/vzero
 *          [u][max_chunks][128] f16 (per token, natural order).
 *   kres [u][256][128] bf16 (ring slot-major), vres [u][128][256] bf16
 *          (channel-major); live slots [res_start, res_start+res_len) mod 256.
 *   S [u][128][256] f32, P [u][256] f32 (zero until the first adapter flush).
 *   n_chunks / res_start / res_len: [B] int32 per sequence. */
typedef struct kvlc_cache {
  int32_t B, Hkv, Hq, max_chunks;
  uint32_t* kcodes;
  uint32_t* vcodes;
  uint16_t* kscale;
  uint16_t* kzero;
  uint16_t* vscale;
  uint16_t* vzero;
  uint16_t* kres;
  uint16_t* vres;
  float* S;
  float* P;
  int32_t* n_chunks;
  int32_t* res_start;
  int32_t* res_len;
} kvlc_cache;

/* One CorrectionAdapter per kv head, float32 [Hkv][128][128]
 * each; all NULL (or enabled == 0) = no adapter. */
typedef struct kvlc_adapter {
  const float* w1q;
  const float* w2q;
  const float* w1k;
  const float* w2k;
  int32_t enabled;
} kvlc_adapter;

/* Bulk prefill (N streaming appends, cache.py:120-130, in one pass):
 * k, v bf16 [B][Hkv][n_tok][128]; sequence b takes its first lens[b]
 * (host array) tokens.  keep_window != 0: flushes floor((len-R)/G) chunks
 * (K1+K2+K3 fused) and loads the rest into the residual ring, exactly as the
 * streaming rule; keep_window == 0: flushes floor(len/G) chunks (a non-tail
 * shard of a sequence-parallel cache).  Cache must be empty. */
int kvlc_prefill(const kvlc_cache* cache, const kvlc_adapter* ad,
                 const uint16_t* k, const uint16_t* v, int64_t n_tok,
                 const int32_t* lens_host, int32_t keep_window, void* ws,
                 size_t ws_bytes, void* stream);
size_t kvlc_prefill_workspace(const kvlc_cache* cache, int64_t n_tok);

/* Workspace for kvlc_append / kvlc_flush_due to run their flushes on the tensor-core path
 * (with an adapter); without it (ws NULL or smaller) they use the SIMT flush kernel. */
size_t kvlc_append_workspace(const kvlc_cache* cache);

/* Append one token per sequence (cache.py:120-130): k_t, v_t bf16
 * [B][Hkv][128].  active_host[b] != 0 selects the sequences that append;
 * flush_host[b] != 0 flushes sequence b's oldest G tokens afterwards (the
 * host mirrors the lengths, so it knows which sequences hit R+G). */
int kvlc_append(const kvlc_cache* cache, const kvlc_adapter* ad,
                const uint16_t* k_t, const uint16_t* v_t,
                const int32_t* active_host, const int32_t* flush_host,
                void* ws, size_t ws_bytes, void* stream);

/* Decode options.  chunks_per_split: quantized chunks per warp task (0 = auto).
 * literal: literal_correction (attention.py:188-189). */
typedef struct kvlc_decode_opts {
  int32_t chunks_per_split;
  int32_t literal;
  int32_t max_chunks_hint; /* max n_chunks over the batch (host mirror) */
  int32_t out_fp32;        /* 1: `out` is float32 [B][Hq][128] instead of bf16 */
  void* ev_begin;          /* optional cudaEvent_t recorded right before / after */
  void* ev_end;            /* the split-KV kernel (measurement hook, may be NULL) */
} kvlc_decode_opts;

/* Fused GQA decode (Algorithm 1 / decode_step_blocked, attention.py:197-276)
 * for every (b, q-head): q bf16 [B][Hq][128] -> out bf16 [B][Hq][128].
 * Launches the split-KV kernel (correction, quantized splits, residual
 * window) and the LSE combine kernel, PDL-chained; plans with more than 64
 * records per unit (explicit small chunks_per_split) fuse the combine into the
 * last CTA of each (b, kv-head) unit instead.  The launch may overlap the
 * previous kernel on `stream` (programmatic dependent launch): q may be
 * produced by any kernel; its first code copies are issued before the
 * predecessor completes, so cache state must be written through this library
 * (prefill / a flushing append / flush_due / deserialize_unit mark the CACHE,
 * independent of host thread and stream, and the next decode of that cache
 * waits fully) or the writer must call kvlc_note_cache_write().  The workspace must be
 * zero-filled before its first use (its head holds per-unit arrival counters
 * that every launch leaves at zero). */
size_t kvlc_decode_workspace(const kvlc_cache* cache, const kvlc_decode_opts* o);
int kvlc_decode(const kvlc_cache* cache, const kvlc_adapter* ad,
                const uint16_t* q, void* out, const kvlc_decode_opts* o,
                void* ws, size_t ws_bytes, void* stream);

/* decode_step_blocked(..., return_partials=True) at block_tokens = G on the serving cache
 * (attention.py:41-47, 197-276): the fused decode (out as kvlc_decode) plus, per (b, q-head),
 * its per-block partials in blocks [B][Hq][max_blocks][2 + 128] fp32 = (block max m in natural
 * logit units, block sum l = sum exp(s - m), y = sum exp(s - m) v in the stored basis): the
 * ceil(n_chunks[b] / c) quantized blocks of block_tokens = c G (c = o->chunks_per_split, 1 when
 * 0: block_tokens = G), then the residual window as one block; rows past a sequence's blocks are
 * zero.  max_blocks >= ceil(max n_chunks / c) + 1.  Workspace: kvlc_decode_workspace() with
 * chunks_per_split = c. */
int kvlc_decode_blocks(const kvlc_cache* cache, const kvlc_adapter* ad, const uint16_t* q,
                       void* out, float* blocks, int32_t max_blocks, const kvlc_decode_opts* o,
                       void* ws, size_t ws_bytes, void* stream);

/* Marks `cache` as written outside this library (codes, metadata or chunk counts):
 * its next decode launches without overlapping the preceding kernel. */
void kvlc_note_cache_write(const kvlc_cache* cache);

/* Split-KV across devices.  kvlc_decode_partial computes, for the chunk range
 * [chunk_lo, chunk_hi) of every sequence, one merged record per (b, q-head):
 *   rec [B][Hq][4 + 2*128] f32 = (m_log2, l, 0, 0, y_rot[128], y_raw[128])
 * include_tail != 0 adds the residual window (raw basis) to the record and
 * writes the correction record corr [B][Hq][1 + 128] = (C_d, C_n[128]).
 * kvlc_merge_records LSE-merges n_rec such records (e.g. all-gathered over
 * NCCL) plus the correction into out [B][Hq][128] (bf16, or f32 when out_fp32)
 * (_reduce_blocks, attention.py:158-194, then H^T and the divide, :262-267). */
int kvlc_decode_partial(const kvlc_cache* cache, const kvlc_adapter* ad,
                        const uint16_t* q, int32_t chunk_lo, int32_t chunk_hi,
                        int32_t include_tail, float* rec, float* corr,
                        const kvlc_decode_opts* o, void* ws, size_t ws_bytes,
                        void* stream);
/* Copies a step's input (e.g. q, bf16 [B][Hq][128]) from pinned host memory
 * `src` to device `dst` in a kernel that lets the following kvlc_decode start
 * early (programmatic dependent launch): the decode streams its codes while q
 * arrives and reads q only after the copy completes.  16-byte aligned, bytes a
 * multiple of 16.  For a host-to-host decode step in one CUDA graph. */
int kvlc_stage_input(const void* src, void* dst, size_t bytes, void* stream);

int kvlc_merge_records(const float* recs, int32_t n_rec, int64_t rec_stride,
                       const float* corr, int32_t B, int32_t Hq, int32_t literal,
                       int32_t out_fp32, void* out, void* stream);

/* Export one quantized chunk of unit u in the reference layout:
 * kwords [8][128], vwords [128][8] (value_rows order, cache.py:146-147),
 * scales/zeros as stored (f16).  For parity checks and .kvlc export. */
int kvlc_export_chunk(const kvlc_cache* cache, int32_t unit, int32_t chunk,
                      uint32_t* kwords, uint32_t* vwords, uint16_t* kscale,
                      uint16_t* kzero, uint16_t* vscale, uint16_t* vzero,
                      void* stream);

/* .kvlc image of one (b, kv-head) unit (serialize_cache / deserialize_cache,
 * cache.py:197-307): the reference's little-endian per-head format — header
 * "KVLC" + 9 u32, key / value code words in the reference layouts, f16
 * metadata, f16 residual (oldest first) and f16 S / P (rank 0 = no states).
 * `image` is a device buffer of kvlc_unit_image_bytes() bytes (0 = invalid
 * arguments).  The host mirrors the sequence counters and passes them.
 * Deserialization loads the residual at ring slot 0 (rounded f16 -> bf16) and
 * sets the counters of sequence unit / Hkv (all its units must agree). */
size_t kvlc_unit_image_bytes(int32_t n_chunks, int32_t res_len, int32_t rank);
int kvlc_serialize_unit(const kvlc_cache* cache, int32_t unit, int32_t n_chunks,
                        int32_t res_start, int32_t res_len, int32_t rank,
                        uint8_t* image, void* stream);
int kvlc_deserialize_unit(const kvlc_cache* cache, int32_t unit,
                          const uint8_t* image, int32_t n_chunks,
                          int32_t res_len, int32_t rank, void* stream);

/* ------------------------------------------------------------------------ */
/* standalone blocks (bf16 in, serving formats out) for callers with their   */
/* own K / V storage; codes are bit-identical to quantize_tensor on the same  */
/* bf16 values, fp16 scale / zero = float16(reference float64 value).         */
/* ------------------------------------------------------------------------ */

/* quantize_tensor (quantize.py:220-239) on x bf16 [rows][ld] (first `cols`
 * columns): token axis -> words [rows][ceil(cols/L)], scale/zero
 * [rows][ceil(cols/G)]; channel axis (a key chunk, cache.py:141) -> words
 * [ceil(rows/L)][cols], scale/zero [ceil(rows/G)][cols] (f16).  err_opt
 * (may be NULL): float [rows][cols] = x - dequantize (k_err, cache.py:153). */
int kvlc_quantize_pack(const uint16_t* x, int64_t rows, int64_t cols, int64_t ld,
                       int axis, int bits, int group, uint32_t* words,
                       uint16_t* scale, uint16_t* zero, float* err_opt,
                       void* stream);

/* Value path of flush_group (cache.py:143-145): rotate(x, H, "post")
 * (hadamard.py:45-57) of bf16 rows [rows][ld] (dim a power of two), then
 * token-wise quantization: words [rows][ceil(dim/L)], scale/zero
 * [rows][ceil(dim/G)] f16; vq_opt (may be NULL): float [rows][dim] = the
 * dequantized rotated values (v_q, cache.py:154). */
size_t kvlc_fwht_quantize_workspace(int64_t rows, int dim);
int kvlc_fwht_quantize_pack(const uint16_t* x, int64_t rows, int dim, int64_t ld,
                            int bits, int group, uint32_t* words,
                            uint16_t* scale, uint16_t* zero, float* vq_opt,
                            void* ws, size_t ws_bytes, void* stream);

/* Adapter-state update of flush_group (cache.py:155-158) for n tokens:
 * S [d][rank] += sum_i outer(vq_rot[i], phi_k(k_err[i])), P [rank] +=
 * sum_i phi_k(k_err[i]); k_err, vq_rot float [n][d], W1k / W2k float
 * [d][rank/2] (adapter.py:80-96); float64 arithmetic, fp32 state. */
size_t kvlc_state_update_workspace(int64_t n, int rank);
int kvlc_state_update(const float* k_err, const float* vq_rot, int64_t n, int d,
                      int rank, const float* w1k, const float* w2k, float* S,
                      float* P, void* ws, size_t ws_bytes, void* stream);

/* flush_group (cache.py:132-158) on every sequence b with flush_host[b] != 0
 * (residual length >= R + G), without appending: the fused K1+K2+K3 kernel. */
int kvlc_flush_due(const kvlc_cache* cache, const kvlc_adapter* ad,
                   const int32_t* flush_host, void* ws, size_t ws_bytes,
                   void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KVLINC_H */

/*
 * gs_capi.h -- C ABI of the B200-native GhostServe shadow-checkpointing byte
 * path (libghostserve_b200.so). Plain pointers and sizes only: no C++ or
 * torch types cross this boundary, no exceptions escape it.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/proj/include/ghostserve/...). The reference API itself is
 * mirrored on top of this ABI by include/ghostserve_gpu/coding.hpp (C++) and
 * paper_2605_00831_b200/coding.py (Python); see INTEGRATION.md.
 *
 * Conventions
 *  - Return value: gs_status. GS_OK = 0. The message for the last failure on
 *    the calling thread is gs_last_error().
 *  - Status <-> reference exception: GS_INVALID_ARGUMENT = std::invalid_argument,
 *    GS_UNRECOVERABLE = ghostserve::UnrecoverableError, GS_DOMAIN_ERROR =
 *    std::domain_error, GS_CUDA_ERROR / GS_UNSUPPORTED have no reference twin.
 *  - Shard numbering is the reference's: data shards 0..n-1, parity shards
 *    n..n+k-1 (coding.hpp:126-137, recovery.hpp:117-121).
 *  - "stream" arguments are cudaStream_t passed as void* (NULL = legacy
 *    default stream); they are caller-owned.
 *  - Device pointers may point into a peer GPU's memory (cudaIpcOpenMemHandle
 *    or peer access enabled): kernels then load/store over NVLink directly.
 *  - There is no CPU fallback: every byte of parity or rebuilt KV comes out of
 *    a CUDA kernel. Without a CUDA device the compute calls return
 *    GS_CUDA_ERROR.
 */
#ifndef GS_CAPI_H
#define GS_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GS_OK = 0,
  GS_INVALID_ARGUMENT = 1,
  GS_UNRECOVERABLE = 2,
  GS_DOMAIN_ERROR = 3,
  GS_CUDA_ERROR = 4,
  GS_UNSUPPORTED = 5,
  GS_LOGIC_ERROR = 6,   /* std::logic_error (duplicate store entry) */
  GS_RUNTIME_ERROR = 7  /* std::runtime_error (parity file format / integrity) */
} gs_status;

/* CodeKind (coding.hpp:19). All three run on the GPU (RDP: gs_rdp.cuh,
 * position-dependent -- byte-range striping across ranks refuses it). */
typedef enum { GS_XOR = 0, GS_RDP = 1, GS_RS = 2 } gs_code_kind;

typedef struct gs_codec gs_codec;       /* immutable coefficient plan + kernel choice */
typedef struct gs_pipeline gs_pipeline; /* per-device staging ring + events for host-link overlap */
typedef struct gs_store gs_store;       /* host tier: ParityStore on pinned slabs */
typedef struct gs_verify gs_verify;     /* an in-flight split parity verification (recovery) */

/* ---- diagnostics ------------------------------------------------------- */
const char* gs_status_string(int status);
const char* gs_last_error(void);
int gs_abi_version(void);
/* Drop queued runtime-specialisation builds and wait for the one in flight
 * (tests that want a quiet library). NOT needed before exit: NVRTC runs in a
 * helper process (gs_jit_helper), so a process may exit mid-build. */
int gs_jit_quiesce(void);
/* Number of kernels this library launched in this process (all devices). */
uint64_t gs_kernel_launches(void);
/* Number of offload calls that took the zero-copy epilogue (the kernel stores
 * the parity straight into pinned host memory; calls with <= 2 MiB of parity,
 * GS_ZC_BYTES overrides, 0 = off). */
uint64_t gs_zero_copy_offloads(void);
/* Set that threshold (bytes of parity per call; 0 disables the epilogue). */
int gs_set_zero_copy_bytes(uint64_t bytes);
/* 1 if a CUDA device is usable from this process. */
int gs_cuda_available(void);

/* ---- GF(2^8) and scheme (host) ----------------------------------------- */
/* gf256.hpp:42-61 */
uint8_t gs_gf_mul(uint8_t a, uint8_t b);
int gs_gf_inv(uint8_t a, uint8_t* out);            /* GS_DOMAIN_ERROR for 0 */
int gs_gf_div(uint8_t a, uint8_t b, uint8_t* out); /* GS_DOMAIN_ERROR for b == 0 */
/* CodingScheme::validate (coding.hpp:44-60) */
int gs_scheme_validate(int kind, int n, int k);
/* max_tolerance (coding.hpp:69-76); -1 for an unknown kind */
int gs_max_tolerance(int kind, int n, int k);
/* build_encoding_matrix (coding.hpp:96-118): k*n row-major into coef */
int gs_encoding_matrix(int kind, int n, int k, uint8_t* coef);

/* ---- codecs ---------------------------------------------------------------
 * Encoder for a scheme: replaces the matrix build + dispatch of encode()
 * (coding.hpp:313-336, 269-275). Outputs = k parity shards. */
int gs_encoder_create(int kind, int n, int k, gs_codec** out);
/* Decoder for (scheme, erasure pattern): replaces the per-call planning in
 * reconstruct() (coding.hpp:458-571): validation, tolerance, row choice
 * (:540-544), e x e Gauss-Jordan inverse on the HOST (:545-551, 187-223)
 * and coefficient folding (:554-566). `lost` is deduplicated like
 * ErasurePattern (:131-134). Outputs = the lost DATA shards, ascending. */
int gs_decoder_create(int kind, int n, int k, const int* lost, int n_lost, gs_codec** out);
/* Same, with flags: GS_FLAG_DECODER selects gs_decoder_create semantics,
 * GS_FLAG_GENERIC forces the runtime-coefficient kernel (used by the tests
 * to cross-check the two kernel back ends). */
#define GS_FLAG_GENERIC 1
#define GS_FLAG_DECODER 2
int gs_codec_create_ex(int kind, int n, int k, const int* lost, int n_lost, int flags, gs_codec** out);
int gs_codec_destroy(gs_codec* c);
/* Shape of a codec: number of outputs and, per output, the shard index it
 * produces; number of shard slots it reads (n for encoders, n+k for
 * decoders); 1 in *specialised when a compile-time kernel serves it. */
int gs_codec_info(const gs_codec* c, int* n_out, int* out_index, int* n_slots,
                  int* specialised);
/* Coefficients as applied: n_out x n_slots row-major (0 = slot unused). */
int gs_codec_coefficients(const gs_codec* c, uint8_t* coef);

/* ---- device path (K1 / K2), asynchronous on `stream` ----------------------
 * Applies the codec to n_stripes independent stripes of `len` bytes each.
 *  slots[s * n_slots + j] : device pointer of shard slot j of stripe s
 *                           (encoder: data 0..n-1; decoder: shard index
 *                           0..n+k-1, NULL allowed for lost / unused slots)
 *  outs[s * n_out + i]    : device pointer receiving output i of stripe s
 * Replaces encode() (coding.hpp:313) / reconstruct() (:458) byte loops. */
int gs_apply_device(const gs_codec* c, int n_stripes, const void* const* slots,
                    void* const* outs, size_t len, void* stream);

/* ---- paged KV cache ------------------------------------------
 * A slice in the reference byte order [K,V][layer][token][H*D/tp]
 * (kv_layout.hpp:59-68) read straight out of a paged KV cache. The slice is
 * 2*layers segments of page_bytes = chunk tokens * token_bytes; segment
 * (t, l) lives at  base + l*layer_stride + t*kv_stride  plus the block:
 *  - block_table == NULL: the chunk is one cache block and each per-stripe
 *    base pointer already includes the block's offset;
 *  - block_table != NULL (device int32 [stripes][table_stride]): the chunk
 *    spans page_bytes / block_bytes blocks; block i of stripe s is
 *    block_table[s*table_stride + i] at offset block * block_bytes (the same
 *    ids for every layer and for K and V, as in vLLM-style caches), and the
 *    per-stripe base pointers are the worker's cache base.
 * Tokens >= valid_tokens of a segment read as zero (pad_partial,
 * kv_layout.hpp:73-84) and are never written. Sizes and strides are
 * multiples of 16. */
typedef struct {
  uint32_t page_bytes;
  uint32_t layers;
  uint32_t token_bytes;
  uint32_t valid_tokens;
  uint64_t layer_stride;
  uint64_t kv_stride;
  const int32_t* block_table;
  uint32_t block_bytes;
  uint32_t table_stride;
} gs_page_map;
/* gs_apply_device with slots whose bit is set in paged_slot_mask read through
 * src_map and (dst_map != NULL) outputs scattered through dst_map. */
int gs_apply_device_paged(const gs_codec* c, int n_stripes, const void* const* slots, void* const* outs,
                          size_t len, const gs_page_map* src_map, uint32_t paged_slot_mask,
                          const gs_page_map* dst_map, void* stream);

/* ---- host-link pipelines ----------------------------------------------------
 * A pipeline owns device staging (`staging_bytes`, split into a ring) and
 * events on `device`. Not thread-safe; one per (device, caller thread). */
int gs_pipeline_create(int device, size_t staging_bytes, gs_pipeline** out);
/* Resolve every kernel of the library on `device` (CUDA loads modules
 * lazily at first launch); gs_pipeline_create calls it, so recovery never
 * pays module loading on its critical path. */
int gs_prewarm(int device);
/* Variant of the specialised kernels for aligned bodies (process-wide):
 * 0 = register-streaming LDG.128 kernel, 1 = bulk-copy (cp.async.bulk)
 * shared-memory pipeline with producer/consumer warps, 2 = auto (default:
 * bulk for encodes with shards >= 48 MiB, register kernel otherwise). All are
 * bit-identical; exposed for benchmarking and cross-checking. */
int gs_set_kernel_variant(int variant);
/* Runtime-specialised kernels: a codec with no compiled specialisation
 * (e.g. RS(10,4) decode, RS(9,2)) starts on the runtime-coefficient kernel
 * and, on its first GPU launch, queues an NVRTC build of the specialised
 * Horner kernel for its matrix (background thread, cubin cached on disk in
 * _lib/jit or $GS_JIT_CACHE); later launches use it. Bytes are identical.
 * gs_set_jit(0) / GS_JIT=0 disables. jit_status: -2 not applicable
 * (compiled kernel, RDP, disabled, matrix too large), 0 building, 1 ready,
 * -1 failed (GS_RUNTIME_ERROR with the compiler log); wait != 0 blocks
 * until the build is done (and requests it if not yet requested). */
int gs_set_jit(int on);
int gs_codec_jit_status(const gs_codec* c, int wait, int* status);
int gs_pipeline_destroy(gs_pipeline* p);
/* Live kernel timing of the pipelined calls (encode_offload /
 * reconstruct_upload): while on, each codec launch group is measured two
 * ways inside the caller's real schedule: (1) timing events on the compute
 * stream around the group, after the slot waits; (2) kernel-internal
 * %globaltimer stamps (first CTA start, last warp's stores performed),
 * which unlike (1) carry no front-end latency when copy engines are busy on
 * other streams. kernel_time synchronises and returns both summed times
 * (device_ms may be NULL), the number of launch groups and of kernel
 * launches since set_timing / the previous kernel_time, then resets.
 * Ignored under stream capture. */
int gs_pipeline_set_timing(gs_pipeline* p, int on);
int gs_pipeline_kernel_time(gs_pipeline* p, double* event_ms, double* device_ms, int* groups, uint64_t* launches);

/* Checkpoint offload (PAPER Alg.1 / checkpoint.hpp:143-146 + the host tier of
 * parity_store.hpp:77-90): encode device-resident data into staging on
 * `compute`, D2H each finished piece to `h_parity` (pinned host; k per
 * stripe) on `copy`, pieces overlapped. Returns once work is ENQUEUED;
 * completion = `copy` stream.
 * CUDA graphs: both pipeline calls may be stream-captured (capture on
 * `compute`; `copy` is forked off it inside the call). Completion rules are
 * unchanged, so an offload's capturer joins `copy` back into its origin
 * stream before ending the capture. A graph bakes in the staging ring:
 * order its launches against eager calls on the same pipeline. */
int gs_encode_offload(gs_pipeline* p, const gs_codec* enc, int n_stripes,
                      const void* const* d_data, void* const* h_parity, size_t len,
                      void* compute, void* copy);

/* Same, data slices gathered from a paged KV cache (no staging copy). */
int gs_encode_offload_paged(gs_pipeline* p, const gs_codec* enc, int n_stripes, const void* const* d_data,
                            void* const* h_parity, size_t len, const gs_page_map* src_map, void* compute,
                            void* copy);

/* Recovery upload (recovery.hpp:100-133 byte path): parity slots of `slots`
 * are HOST pointers (pinned), data slots DEVICE pointers (local or peer).
 * Used parity rows are H2D'd piecewise on `copy` into staging; the rebuild
 * kernel runs per piece on `compute` and writes `outs` (device, may be a
 * peer's KV buffer). Returns once enqueued; completion = `compute`. */
int gs_reconstruct_upload(gs_pipeline* p, const gs_codec* dec, int n_stripes,
                          const void* const* slots, void* const* outs, size_t len,
                          void* compute, void* copy);

/* Same with the surviving data slots read from paged caches (src_map) and
 * the rebuilt slices scattered into the replacement's paged cache (dst_map);
 * either map may be NULL (contiguous). */
int gs_reconstruct_upload_paged(gs_pipeline* p, const gs_codec* dec, int n_stripes, const void* const* slots,
                                void* const* outs, size_t len, const gs_page_map* src_map,
                                const gs_page_map* dst_map, void* compute, void* copy);

/* Drop-in host-buffer calls (synchronous): the byte semantics of
 * ghostserve::encode (coding.hpp:313) and ghostserve::reconstruct (:458) with
 * host inputs and outputs; H2D, kernel and D2H overlapped through `p`.
 * For reconstruct, slots are host pointers (n+k, NULL for lost). */
int gs_encode_host(gs_pipeline* p, const gs_codec* enc, const void* const* h_data,
                   void* const* h_parity, size_t len);
int gs_reconstruct_host(gs_pipeline* p, const gs_codec* dec, const void* const* h_slots,
                        void* const* h_out, size_t len);
/* Stream-ordered forms for callers that keep several calls in flight (a
 * serving loop checkpointing block after block from host buffers): return
 * once enqueued on the pipeline's own streams; host buffers must stay valid
 * and unmodified until gs_pipeline_sync(p) returns. Successive calls on one
 * pipeline overlap (the H2D of call i+1 runs under the D2H of call i). */
int gs_encode_host_async(gs_pipeline* p, const gs_codec* enc, const void* const* h_data,
                         void* const* h_parity, size_t len);
int gs_reconstruct_host_async(gs_pipeline* p, const gs_codec* dec, const void* const* h_slots,
                              void* const* h_out, size_t len);
/* Wait for everything enqueued on the pipeline. */
int gs_pipeline_sync(gs_pipeline* p);

/* ---- one-call forms (the boundary as SURVEY §8b words it) ----------------
 * Same kernels and pipelines as above, with the staging pipeline implicit: a
 * per-(calling thread, device) default pipeline (256 MiB staging) is created
 * on first use and reused.
 *  gs_codec_create      = gs_encoder_create (coding.hpp:96-118 + :44-60).
 *  gs_encode_async      : one stripe, n device shards (local or peer-mapped)
 *                         -> k pinned host parity buffers (checkpoint.hpp:
 *                         143-146); K1 on `compute`, D2H on `copy`.
 *  gs_reconstruct_async : lost shard indices (coding.hpp:458-571), index-
 *                         aligned DEVICE data shards (NULL for lost), the k
 *                         pinned HOST parity rows (NULL for lost), outputs =
 *                         the lost data shards ascending (device). The
 *                         decoder (host Gauss-Jordan) is cached per pattern.
 *                         Only the parity rows the decode uses are H2D'd.
 *  gs_sync              : wait for `stream` (NULL = the legacy default stream)
 *                         and the calling thread's default pipelines. */
int gs_codec_create(int kind, int n, int k, gs_codec** out);
int gs_encode_async(const gs_codec* enc, const void* const* d_shards, size_t len, void* const* h_parity,
                    void* compute, void* copy);
int gs_reconstruct_async(const gs_codec* enc, const int* lost, int n_lost, const void* const* d_survivors,
                         const void* const* h_parity, void* const* d_out, size_t len, void* stream);
int gs_sync(void* stream);
/* The calling thread's default pipeline for its CURRENT device
 * (cudaGetDevice), created on first use and owned by the library: what the
 * C++ drop-in (ghostserve_gpu/coding.hpp) runs its host-buffer calls on, so
 * concurrent callers never share a staging ring and each uses its own GPU. */
int gs_thread_pipeline(gs_pipeline** out);
/* The device a pipeline was created on. */
int gs_pipeline_device(gs_pipeline* p, int* device);
/* Background checkpoints: cap the CTAs of the pipeline's encode launches
 * (0 = the whole GPU, the default). A decode-block checkpoint next to the
 * serving engine's decode kernels then occupies a few SMs for a little longer
 * instead of every SM for a moment (bench decode_overhead). */
int gs_pipeline_set_max_ctas(gs_pipeline* p, int max_ctas);

/* ---- KV data model (kv_layout.hpp) ------------------------------------- */
/* slice_bytes (kv_layout.hpp:40-45), validate (:21-28) */
int gs_slice_bytes(int layers, int kv_heads, int head_dim, int tp, uint32_t chunk_size,
                   uint64_t* out);
/* make_ground_truth_slice (kv_layout.hpp:110-134) generated on the device,
 * bit-identical to the reference stream, pad_partial included. */
int gs_ground_truth_slice_device(uint64_t kv_seed, uint64_t request_id, uint32_t chunk,
                                 int worker, int layers, int kv_heads, int head_dim, int tp,
                                 uint32_t chunk_size, uint32_t valid_tokens, void* d_out,
                                 void* stream);
/* The same into host memory (device generation + copy back; synchronous). */
int gs_ground_truth_slice(uint64_t kv_seed, uint64_t request_id, uint32_t chunk, int worker, int layers,
                          int kv_heads, int head_dim, int tp, uint32_t chunk_size, uint32_t valid_tokens,
                          void* h_out);
/* pad_partial (kv_layout.hpp:73-84) on a device slice */
int gs_pad_partial_device(void* d_slice, int layers, int kv_heads, int head_dim, int tp,
                          uint32_t chunk_size, uint32_t valid_tokens, void* stream);

/* ---- parity seal (parity_store.hpp:19-53), host ------------------------ */
uint64_t gs_fnv1a64(const void* bytes, size_t len, uint64_t h);
/* 1 when the host FNV-1a (gs_fnv1a64, the checksums, the store's seal and the
 * recovery verification) runs the bit-sliced AVX-512 chain of gs_fnv_simd.cpp
 * (~6 GB/s per chain and core), 0 when it runs the scalar chain. */
int gs_fnv_host_simd(void);
/* Switch the bit-sliced chain off (0) or back on (1, when the CPU has it) for
 * A/B runs; returns gs_fnv_host_simd() afterwards. */
int gs_fnv_host_set_simd(int on);
/* ParityChunk::compute_checksum: FNV-1a chained over k buffers in order */
uint64_t gs_parity_checksum(const void* const* parity, int k, size_t len);
/* Seal many chunks concurrently on up to `threads` host threads:
 * out[c] = checksum of parity[c*k .. c*k+k-1]. */
int gs_parity_checksum_batch(const void* const* parity, int n_chunks, int k, size_t len,
                             int threads, uint64_t* out);
/* Continue m independent FNV-1a chains, one segment each, on up to `threads`
 * host threads: h_out[q] = fnv1a64(bufs[q][0..lens[q]), h_in[q]) (h_out may
 * alias h_in; a zero length passes the state through). One round of the
 * striped verification relay (peer.py chain_striped): at N>1 every rank holds
 * a byte range of each parity row, and a chunk's checksum (ParityChunk::seal,
 * parity_store.hpp:19-53) is one chain through the ranks' ranges in order. */
int gs_fnv1a64_continue_batch(const void* const* bufs, const uint64_t* lens, const uint64_t* h_in,
                              uint64_t* h_out, int m, int threads);
/* The same relay without rounds, for the ranks of ONE node: `board` is host
 * memory shared by the ranks' processes (gs_relay_board_bytes(n_chunks, k,
 * world) bytes, zeroed once), holding one tagged chain state per (chunk,
 * chain position). Every rank calls gs_fnv_relay with the same `epoch` (> 0,
 * a new one per call, calls on one board separated by a barrier) and rows[c*k
 * + i] = its range of parity row i of chunk c (`len` bytes); its `threads`
 * continue its segments as their predecessors' states appear and sums[c]
 * receives chunk c's checksum on every rank. A peer that does not deliver
 * within `timeout_s` seconds (<= 0: 60) makes the call fail with
 * GS_RUNTIME_ERROR. */
uint64_t gs_relay_board_bytes(int n_chunks, int k, int world);
int gs_fnv_relay(void* board, uint64_t epoch, int rank, int world, const void* const* rows, uint64_t len,
                 int n_chunks, int k, uint64_t h0, int threads, double timeout_s, uint64_t* sums);
/* gs_fnv_relay with the first k_dev rows of every chunk hashed on this rank's
 * GPU (the seeded window kernel, gs_fnv1a64_device_seeded, in batches of
 * `batch` chunks on `stream`; the calling thread drives it and relays the
 * states through the board): d_rows[c*k_dev + i] = device address of this
 * rank's range of row i of chunk c (16-B aligned; len % 16 == 0), ready[c]
 * (cudaEvent_t, or NULL / a NULL entry) = recorded once chunk c's device rows
 * are complete (e.g. their H2D); rows k_dev..k-1 come from the host rows
 * h_rows[c*k + i] on `threads` host threads. Same board, epoch and result
 * contract as gs_fnv_relay; ranks may mix k_dev values only if all use the
 * same k. */
int gs_fnv_relay_device(void* board, uint64_t epoch, int rank, int world, const void* const* d_rows, int k_dev,
                        void* const* ready, const void* const* h_rows, uint64_t len, int n_chunks, int k,
                        uint64_t h0, int threads, int batch, void* stream, double timeout_s, uint64_t* sums);
/* The same FNV-1a on the GPU, bit-exact (gs_fnv_gpu.cu): chain c is the k
 * device buffers bufs[c*k .. c*k+k-1] of `len` bytes each, concatenated in
 * order and hashed from h0 (0xcbf29ce484222325 = ParityChunk checksum);
 * d_out[c] (device memory) receives the hash, stream-ordered on `stream`.
 * len % 16 == 0 and 16-B aligned buffers (GS_INVALID_ARGUMENT otherwise).
 * Replaces the serial parity_store.hpp:19-25 loop for parity that is already
 * in HBM: bit-sliced low-byte recovery + a linear reduction, no serial chain. */
int gs_fnv1a64_device(const void* const* bufs, int n_chains, int k, uint64_t len, uint64_t h0,
                      uint64_t* d_out, void* stream);
/* Upload chunks' pinned host parity rows (h_parity[c*k + i]) into device rows
 * (d_parity[c*k + i]) on `copy` and checksum them on the GPU on `compute` as
 * groups land: d_sums[c] = ParityChunk::compute_checksum of chunk c as it sits
 * in HBM (the verification of reconstruct_chunk, recovery.hpp:108-113, moved
 * off the host; the uploaded rows then feed K2 directly). */
int gs_parity_upload_checksum(const void* const* h_parity, int n_chunks, int k, uint64_t len,
                              void* const* d_parity, uint64_t* d_sums, void* compute, void* copy);
/* The checkpoint-side mirror: K1's parity rows in HBM (written on `compute`)
 * are copied to pinned host rows on `copy` while the GPU computes their chunk
 * checksums; h_sums[c] (pinned host or device memory) receives them behind
 * the rows, on `copy`. Pair with gs_store_commit_sealed_batch on `copy`. */
int gs_parity_offload_sealed(const void* const* d_parity, int n_chunks, int k, uint64_t len,
                             void* const* h_parity, uint64_t* h_sums, void* compute, void* copy);
/* Recovery's parity verification split between the GPU and host threads.
 * enqueue: chunks [0, n_full) upload all k rows (h_parity[c*k+i] -> d_parity[c*k+i])
 * and are checksummed on the GPU; chunks [n_full, n_chunks) upload only rows
 * 0..u-1 (the rows the decode uses), the GPU hashes them and host threads
 * continue the serial FNV chain over rows u..k-1 from the host copy. Uploads
 * on `copy`, hashing on `compute`; rows not uploaded may be NULL in d_parity.
 * finish: blocks, sums[c] = ParityChunk::compute_checksum of chunk c (bit-exact),
 * frees the handle. */
int gs_verify_enqueue(const void* const* h_parity, int n_chunks, int k, uint64_t len, int n_full, int u,
                      void* const* d_parity, void* compute, void* copy, gs_verify** out);
int gs_verify_finish(gs_verify* v, int threads, uint64_t* sums);
/* n_full < 0: DYNAMIC split -- rows 0..u-1 of every chunk are uploaded and
 * hashed on the GPU (d_parity rows >= u may be NULL); the rest of each chain
 * is claimed at run time by host threads (from the front, as the GPU states
 * land) or by a GPU feeder (from the back: remaining rows uploaded into an
 * internal ring behind the row-0 uploads, chain continued on the GPU from
 * the device state), so the split adapts to this host's speed.
 * *gpu_chunks = chunks whose whole chain was hashed on the GPU. */
int gs_verify_finish_ex(gs_verify* v, int threads, uint64_t* sums, int* gpu_chunks);
/* Dynamic split pacing (optional, before finish): the host link's rate and
 * one host thread's serial FNV rate (GB/s); host threads then stop claiming
 * chunks the GPU would finish sooner (the host rate is refined online). */
int gs_verify_set_rates(gs_verify* v, double link_gbs, double host_chain_gbs);
/* Make `stream` wait until chunk `chunk`'s uploaded rows are in HBM (and hashed
 * there): the decode can then run K2 group by group under the remaining
 * uploads instead of after all of them. Valid after enqueue and before finish,
 * or while a hold is taken: gs_verify_hold keeps a concurrently running
 * gs_verify_finish from releasing the handle (it waits for the matching
 * gs_verify_release before destroying the upload events), so a caller can
 * start finish on another thread first and queue its K2 launches behind. */
int gs_verify_stream_wait(gs_verify* v, int chunk, void* stream);
int gs_verify_hold(gs_verify* v);
int gs_verify_release(gs_verify* v);
/* Chains (process total) a host thread handed over to the GPU mid-chain in a
 * dynamic split, because it had fallen behind the GPU (diagnostics). */
uint64_t gs_verify_handoffs(void);
/* The last dynamic split: {host threads done, feeder done, hash stream
 * drained} in s after gs_verify_finish started, and the chunks verified by
 * host threads / entirely on the GPU / handed over mid-chain. */
int gs_verify_last_stats(double* out6);
/* gs_fnv1a64_device with a per-chain seed in device memory (d_h0[c], must
 * not alias d_out): continues chains hashed earlier. */
int gs_fnv1a64_device_seeded(const void* const* bufs, int n_chains, int k, uint64_t len, const uint64_t* d_h0,
                             uint64_t* d_out, void* stream);

/* ---- host tier: ParityStore on pinned slabs (parity_store.hpp:31-263) ----
 * Entries are keyed (request, chunk). Reserve -> the D2H of K1 writes the k
 * parity buffers straight into the returned pinned pointers (no try_put
 * copy, checkpoint.hpp:207) -> commit: the FNV-1a seal runs on host threads
 * once `stream` reaches that point (an event waited on by the store's landing
 * thread; the stream never blocks on the host), off the GPU path. Commits
 * cannot be captured into CUDA graphs (GS_INVALID_ARGUMENT). */
int gs_store_create(uint64_t capacity_bytes /* ~0 = unlimited */, int seal_threads, gs_store** out);
int gs_store_destroy(gs_store* s);
/* Place the store's future pinned slabs on `device`'s NUMA node (the socket
 * of the GPU whose D2H fills them); -1 = unbound (cudaHostAlloc). */
int gs_store_bind_device(gs_store* s, int device);
/* try_put accounting (parity_store.hpp:77-90): *accepted = 0 is back-pressure
 * (store unchanged); a duplicate key is GS_LOGIC_ERROR. parity_out[k]. */
int gs_store_reserve(gs_store* s, uint64_t request_id, uint32_t chunk, int kind, int n, int k,
                     uint32_t valid_tokens, uint64_t slice_len, int* accepted, void** parity_out);
int gs_store_commit(gs_store* s, uint64_t request_id, uint32_t chunk, void* stream);
/* Batched forms for a decode block's S requests: one host callback seals
 * the whole batch; reserve_batch stops at the first back-pressure refusal
 * (*accepted = entries reserved). parity_out[i*k + j]. */
int gs_store_reserve_batch(gs_store* s, int count, const uint64_t* request_ids, const uint32_t* chunks, int kind,
                           int n, int k, uint32_t valid_tokens, uint64_t slice_len, int* accepted,
                           void** parity_out);
int gs_store_commit_batch(gs_store* s, int count, const uint64_t* request_ids, const uint32_t* chunks,
                          void* stream);
/* Commit entries whose checksums were computed on the GPU (gs_parity_offload_
 * sealed): the entries are sealed with checksums[i] -- no host FNV pass.
 * `checksums` may be device or host memory; the store copies it on `stream`
 * (at this point of the stream) into pinned memory it owns, so the caller's
 * buffer only has to stay valid until `stream` passes this call, like the
 * source of any cudaMemcpyAsync. */
int gs_store_commit_sealed_batch(gs_store* s, int count, const uint64_t* request_ids, const uint32_t* chunks,
                                 const uint64_t* checksums, void* stream);
int gs_store_wait_sealed(gs_store* s);
/* Copying put (reference try_put): sealed != 0 keeps `checksum` as given.
 * parity == NULL: a cost-only entry (no payload; accounted, get() -> kOk). */
int gs_store_put(gs_store* s, uint64_t request_id, uint32_t chunk, int kind, int n, int k,
                 uint32_t valid_tokens, uint64_t slice_len, const void* const* parity, uint64_t checksum,
                 int sealed, int* accepted);
/* get (parity_store.hpp:92-101): *status 0 = kOk, 1 = kMissing, 2 = kCorrupt
 * (FNV re-verified when verify != 0). kind_n_k[3] optional. */
int gs_store_get(gs_store* s, uint64_t request_id, uint32_t chunk, int verify, int* status, void** parity_out,
                 uint64_t* slice_len, uint32_t* valid_tokens, uint64_t* checksum, int* kind_n_k);
int gs_store_contains(gs_store* s, uint64_t request_id, uint32_t chunk);
int gs_store_erase_request(gs_store* s, uint64_t request_id);
/* out5 = {used_bytes, capacity_bytes, payload_bytes, peak_payload_bytes, entry_count} */
int gs_store_stats(gs_store* s, uint64_t* out5);
int gs_store_audit(gs_store* s);
int gs_store_corrupt_entry(gs_store* s, uint64_t request_id, uint32_t chunk);
int gs_store_keys(gs_store* s, uint64_t* keys, uint64_t max_entries, uint64_t* count);
/* GSRV file image (parity_store.hpp:145-263); out == NULL queries *size. */
int gs_store_serialize(gs_store* s, void* out, uint64_t cap, uint64_t* size);
int gs_store_deserialize(const void* bytes, uint64_t size, uint64_t capacity, int seal_threads, gs_store** out);

/* ---- peer memory over NVLink (multi-GPU striping) ---------------------- */
#define GS_IPC_HANDLE_BYTES 64
/* Export the allocation holding d_ptr: handle (64 B) + byte offset of d_ptr
 * inside it. The importer maps the allocation with gs_ipc_open and adds the
 * offset. Replaces the paper's NCCL gather: peers' KV shards
 * are read in place by K1/K2 over NVLink instead of being copied first. */
int gs_ipc_handle(const void* d_ptr, void* handle_out, uint64_t* offset_out);
int gs_ipc_open(const void* handle, int device, void** d_base);
int gs_ipc_close(void* d_ptr);
int gs_peer_enable(int device, int peer);
/* Byte range [*off, *off + *len) of a shard of `total` bytes owned by rank
 * `rank` of `world` when the range is striped 4 KiB-aligned. */
int gs_stripe_range(uint64_t total, int rank, int world, uint64_t* off, uint64_t* len);

/* ---- pinned host memory for the parity host tier ----------------------- */
int gs_host_alloc(size_t bytes, void** out);
/* Pinned host memory on `device`'s NUMA node (its host link's socket):
 * mmap + mbind + first touch + cudaHostRegister; plain cudaHostAlloc on
 * single-node hosts. Free either kind with gs_host_free. */
int gs_host_alloc_near(int device, size_t bytes, void** out);
int gs_host_free(void* p);
/* NUMA node of the GPU's PCI device (-1 if unknown) and its local CPU list
 * (sysfs local_cpulist, e.g. "0-47,96-143"; "" if unknown). */
int gs_device_numa_node(int device, int* node);
int gs_device_local_cpus(int device, char* buf, size_t cap);

#ifdef __cplusplus
}
#endif
#endif /* GS_CAPI_H */

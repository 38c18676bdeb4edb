/*
 * gs_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the GhostServe shadow-checkpointing byte path
 * (reference: /root/reference/proj/include/ghostserve/{gf256,coding,kv_layout,
 * parity_store}.hpp). It exists to CHECK the CUDA path: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it. The product library (paper_2605_00831_b200/csrc) never links it.
 *
 * Parity pinning: the restatement is checked against (a) the reference's own
 * known-answer tests (gf256_test.cpp:26-57, coding_test.cpp:151-159,
 * kv_model_test.cpp:49-64) and (b) golden vectors produced by the reference
 * itself, compiled from its headers in place (oracle/ref_shim.cpp ->
 * oracle/_ref/libghostserve_ref.so; fixtures in tests/golden/ made by
 * tests/golden/make_golden.py).
 *
 * Status codes are shared with include/gs_capi.h.
 */
#ifndef GS_ORACLE_H
#define GS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same numbering as gs_capi.h's gs_status / gs_code_kind. */
enum { GSO_OK = 0, GSO_INVALID_ARGUMENT = 1, GSO_UNRECOVERABLE = 2, GSO_DOMAIN_ERROR = 3 };
enum { GSO_XOR = 0, GSO_RDP = 1, GSO_RS = 2 };

/* GF(2^8), poly 0x11D (gf256.hpp:14-61). */
uint8_t gso_gf_mul(uint8_t a, uint8_t b);
int gso_gf_inv(uint8_t a, uint8_t* out);           /* GSO_DOMAIN_ERROR for a == 0 */
int gso_gf_div(uint8_t a, uint8_t b, uint8_t* out); /* GSO_DOMAIN_ERROR for b == 0 */
uint8_t gso_gf_exp2(unsigned e);
void gso_gf_tables(uint8_t exp_out[512], uint8_t log_out[256]);

/* CodingScheme::validate / max_tolerance / build_encoding_matrix (coding.hpp:44-118). */
int gso_validate(int kind, int n, int k);
int gso_max_tolerance(int kind, int k);
int gso_encoding_matrix(int kind, int n, int k, uint8_t* coef /* k*n row-major */);

/* encode (coding.hpp:313-336): n data buffers of len bytes -> k parity buffers
 * (XOR, RS and the shortened RDP of coding.hpp:225-307). */
int gso_encode(int kind, int n, int k, const uint8_t* const* data, size_t len,
               uint8_t* const* parity);

/* reconstruct (coding.hpp:458-571). shards[n+k] index-aligned, NULL for lost
 * entries; lost[] any order (deduplicated like ErasurePattern); out[] receives
 * one buffer per lost DATA shard in ascending index order. *n_out is set to
 * the number of data shards rebuilt. */
int gso_reconstruct(int kind, int n, int k, const uint8_t* const* shards, const int* lost,
                    int n_lost, size_t len, uint8_t* const* out, int* n_out);

/* Decode coefficients exactly as coding.hpp:535-566 picks them: for each lost
 * data shard b (ascending), coef_data[b*n + j] for data column j (0 for lost
 * columns) and coef_par[b*k + i] for parity row i (0 for unused rows). */
int gso_decode_matrix(int kind, int n, int k, const int* lost, int n_lost, uint8_t* coef_data,
                      uint8_t* coef_par, int* n_lost_data);

/* kv_layout.hpp:14-134 */
int gso_slice_bytes(int layers, int kv_heads, int head_dim, int tp, uint32_t chunk_size,
                    uint64_t* out);
int gso_pad_partial(uint8_t* bytes, int layers, int kv_heads, int head_dim, int tp,
                    uint32_t chunk_size, uint32_t valid_tokens);
int gso_make_ground_truth_slice(uint64_t kv_seed, uint64_t request_id, uint32_t chunk,
                                int worker, int layers, int kv_heads, int head_dim, int tp,
                                uint32_t chunk_size, uint32_t valid_tokens, uint8_t* out);

/* parity_store.hpp:19-53 */
uint64_t gso_fnv1a64(const uint8_t* bytes, size_t len, uint64_t h);
uint64_t gso_parity_checksum(const uint8_t* const* parity, int k, size_t len);

#ifdef __cplusplus
}
#endif
#endif

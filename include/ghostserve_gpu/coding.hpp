// ghostserve_gpu/coding.hpp -- drop-in C++ facade over gs_capi.h with the
// reference's signatures (/root/reference/proj/include/ghostserve/coding.hpp):
//
//   ghostserve_gpu::encode(const CodingScheme&, std::span<const ConstShardSpan>)
//       -> std::vector<std::vector<uint8_t>>                       (coding.hpp:313)
//   ghostserve_gpu::encode(const CodingScheme&, const std::vector<std::vector<uint8_t>>&)  (:332)
//   ghostserve_gpu::reconstruct(const CodingScheme&, const std::map<int, ConstShardSpan>&,
//                               const ErasurePattern&) -> std::map<int, std::vector<uint8_t>> (:458)
//   build_encoding_matrix / max_tolerance / memory_overhead_ratio / CodingScheme /
//   ErasurePattern / EncodingMatrix / UnrecoverableError                (:17-137)
//
// Status codes map back to the reference exception types:
//   GS_INVALID_ARGUMENT -> std::invalid_argument, GS_UNRECOVERABLE ->
//   UnrecoverableError, GS_DOMAIN_ERROR -> std::domain_error, GS_LOGIC_ERROR ->
//   std::logic_error, others ->
//   std::runtime_error. A consumer switches by changing the namespace (or a
//   `namespace ghostserve = ghostserve_gpu;` alias) and linking
//   libghostserve_b200.so; every byte is computed by the sm_100a kernels.
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../gs_capi.h"

namespace ghostserve_gpu {

enum class CodeKind { kXor = GS_XOR, kRdp = GS_RDP, kReedSolomon = GS_RS };

inline const char* to_string(CodeKind k) {
  switch (k) {
    case CodeKind::kXor: return "xor";
    case CodeKind::kRdp: return "rdp";
    case CodeKind::kReedSolomon: return "rs";
  }
  return "?";
}

class UnrecoverableError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int status, const char* what) {
  if (status == GS_OK) return;
  std::string msg = std::string(what) + ": " + gs_last_error();
  switch (status) {
    case GS_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case GS_UNRECOVERABLE: throw UnrecoverableError(msg);
    case GS_DOMAIN_ERROR: throw std::domain_error(msg);
    case GS_LOGIC_ERROR: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}
}  // namespace detail

struct CodingScheme {
  CodeKind kind = CodeKind::kXor;
  int n = 1;
  int k = 1;

  void validate() const { detail::check(gs_scheme_validate(static_cast<int>(kind), n, k), "coding"); }
  static CodingScheme xor_code(int n) { return {CodeKind::kXor, n, 1}; }
  static CodingScheme rdp(int n) { return {CodeKind::kRdp, n, 2}; }
  static CodingScheme reed_solomon(int n, int k) { return {CodeKind::kReedSolomon, n, k}; }
  bool operator==(const CodingScheme&) const = default;
};

inline int max_tolerance(const CodingScheme& s) { return gs_max_tolerance(static_cast<int>(s.kind), s.n, s.k); }

inline double memory_overhead_ratio(const CodingScheme& s) {
  return static_cast<double>(s.k) / static_cast<double>(s.n);
}

struct EncodingMatrix {
  int rows = 0;
  int cols = 0;
  std::vector<std::uint8_t> coef;
  std::uint8_t at(int r, int c) const { return coef[static_cast<std::size_t>(r) * cols + c]; }
};

inline EncodingMatrix build_encoding_matrix(const CodingScheme& s) {
  EncodingMatrix m;
  s.validate();
  m.rows = s.k;
  m.cols = s.n;
  m.coef.assign(static_cast<std::size_t>(s.k) * s.n, 0);
  detail::check(gs_encoding_matrix(static_cast<int>(s.kind), s.n, s.k, m.coef.data()), "coding");
  return m;
}

struct ErasurePattern {
  std::vector<int> lost;
  explicit ErasurePattern(std::vector<int> indices = {}) : lost(std::move(indices)) {
    std::sort(lost.begin(), lost.end());
    lost.erase(std::unique(lost.begin(), lost.end()), lost.end());
  }
  bool contains(int idx) const { return std::binary_search(lost.begin(), lost.end(), idx); }
};

using ConstShardSpan = std::span<const std::uint8_t>;

namespace detail {

// Codecs are immutable after creation and shareable across threads and
// devices (the reference codec is safe to call from many
// threads): one per (scheme, lost set), created once under a short lock that
// is NOT held across the GPU round trip. Never destroyed (process lifetime),
// so no static destructor races a call still in flight on another thread.
struct Codecs {
  std::mutex mu;
  std::map<std::tuple<int, int, int, std::vector<int>, bool>, gs_codec*> by_key;
};

inline Codecs& codecs() {
  static Codecs* c = new Codecs;
  return *c;
}

inline gs_codec* codec(const CodingScheme& s, const std::vector<int>* lost) {
  auto& h = codecs();
  auto key = std::make_tuple(static_cast<int>(s.kind), s.n, s.k, lost ? *lost : std::vector<int>{}, lost != nullptr);
  std::lock_guard<std::mutex> lk(h.mu);
  auto it = h.by_key.find(key);
  if (it != h.by_key.end()) return it->second;
  gs_codec* c = nullptr;
  if (lost)
    check(gs_decoder_create(static_cast<int>(s.kind), s.n, s.k, lost->data(), static_cast<int>(lost->size()), &c),
          "reconstruct");
  else
    check(gs_encoder_create(static_cast<int>(s.kind), s.n, s.k, &c), "encode");
  h.by_key.emplace(key, c);
  return c;
}

// The calling thread's staging pipeline on its current device (cudaGetDevice):
// concurrent callers each get their own, on their own GPU.
inline gs_pipeline* pipeline() {
  gs_pipeline* p = nullptr;
  check(gs_thread_pipeline(&p), "pipeline");
  return p;
}

}  // namespace detail

// coding.hpp:313-330
inline std::vector<std::vector<std::uint8_t>> encode(const CodingScheme& scheme,
                                                     std::span<const ConstShardSpan> data) {
  scheme.validate();
  if (static_cast<int>(data.size()) != scheme.n)
    throw std::invalid_argument("coding: expected " + std::to_string(scheme.n) + " data shards, got " +
                                std::to_string(data.size()));
  for (std::size_t i = 1; i < data.size(); ++i)
    if (data[i].size() != data[0].size())
      throw std::invalid_argument("coding: shard buffers must all have the same length");
  const std::size_t len = data.empty() ? 0 : data[0].size();
  std::vector<std::vector<std::uint8_t>> parity(static_cast<std::size_t>(scheme.k));
  for (auto& p : parity) p.assign(len, 0);
  if (len == 0) return parity;
  gs_codec* c = detail::codec(scheme, nullptr);
  std::vector<const void*> in;
  std::vector<void*> out;
  for (const auto& d : data) in.push_back(d.data());
  for (auto& p : parity) out.push_back(p.data());
  detail::check(gs_encode_host(detail::pipeline(), c, in.data(), out.data(), len), "encode");
  return parity;
}

// coding.hpp:332-336
inline std::vector<std::vector<std::uint8_t>> encode(const CodingScheme& scheme,
                                                     const std::vector<std::vector<std::uint8_t>>& data) {
  std::vector<ConstShardSpan> spans(data.begin(), data.end());
  return encode(scheme, spans);
}

// coding.hpp:458-571
inline std::map<int, std::vector<std::uint8_t>> reconstruct(const CodingScheme& scheme,
                                                            const std::map<int, ConstShardSpan>& surviving,
                                                            const ErasurePattern& lost) {
  scheme.validate();
  const int total = scheme.n + scheme.k;
  for (int idx : lost.lost)
    if (idx < 0 || idx >= total) throw std::invalid_argument("coding: lost shard index out of range");
  if (static_cast<int>(lost.lost.size()) > max_tolerance(scheme))
    throw UnrecoverableError("coding: " + std::to_string(lost.lost.size()) + " erasures exceed tolerance " +
                             std::to_string(max_tolerance(scheme)) + " for scheme " + to_string(scheme.kind));
  std::size_t len = 0;
  bool have = false;
  std::vector<const void*> slots(static_cast<std::size_t>(total), nullptr);
  for (int idx = 0; idx < total; ++idx) {
    if (lost.contains(idx)) continue;
    auto it = surviving.find(idx);
    if (it == surviving.end())
      throw std::invalid_argument("coding: surviving shard " + std::to_string(idx) + " missing from input");
    if (!have) {
      len = it->second.size();
      have = true;
    } else if (it->second.size() != len) {
      throw std::invalid_argument("coding: shard buffers must all have the same length");
    }
    slots[static_cast<std::size_t>(idx)] = it->second.data();
  }
  std::map<int, std::vector<std::uint8_t>> out;
  gs_codec* c = detail::codec(scheme, &lost.lost);
  int n_out = 0;
  std::vector<int> idx(256);
  detail::check(gs_codec_info(c, &n_out, idx.data(), nullptr, nullptr), "reconstruct");
  if (n_out == 0) return out;
  std::vector<void*> dst;
  for (int i = 0; i < n_out; ++i) {
    auto& v = out[idx[static_cast<std::size_t>(i)]];
    v.assign(len, 0);
  }
  for (int i = 0; i < n_out; ++i) dst.push_back(out[idx[static_cast<std::size_t>(i)]].data());
  if (len) detail::check(gs_reconstruct_host(detail::pipeline(), c, slots.data(), dst.data(), len), "reconstruct");
  return out;
}

// ---- device-pointer overloads (the serving engine's calls) -----------------
// KV already lives in HBM: K1 over n device shards (local or peer-mapped over
// NVLink), parity D2H'd into k PINNED host buffers (the host tier) on the
// caller's streams; returns once enqueued (completion = `copy`). The byte
// work of checkpoint_chunk (checkpoint.hpp:143-146). Streams are
// cudaStream_t passed as void*.
inline void encode_device(const CodingScheme& scheme, std::span<const void* const> d_shards, std::size_t len,
                          std::span<void* const> h_parity, void* compute, void* copy) {
  scheme.validate();
  if (static_cast<int>(d_shards.size()) != scheme.n)
    throw std::invalid_argument("coding: expected " + std::to_string(scheme.n) + " data shards, got " +
                                std::to_string(d_shards.size()));
  if (static_cast<int>(h_parity.size()) != scheme.k)
    throw std::invalid_argument("coding: expected " + std::to_string(scheme.k) + " parity buffers");
  if (len == 0) return;
  gs_codec* c = detail::codec(scheme, nullptr);
  detail::check(gs_encode_async(c, d_shards.data(), len, h_parity.data(), compute, copy), "encode");
}

// Rebuild the lost DATA shards into d_out (ascending shard index) from the
// index-aligned device survivors (NULL for lost) and the k pinned host parity
// rows (NULL for lost): decode matrix inverted on the host (coding.hpp:
// 540-566), only the used parity rows H2D'd, K2 on `stream`; returns once
// enqueued. reconstruct()'s errors: invalid_argument, UnrecoverableError.
inline void reconstruct_device(const CodingScheme& scheme, const ErasurePattern& lost,
                               std::span<const void* const> d_survivors, std::span<const void* const> h_parity,
                               std::span<void* const> d_out, std::size_t len, void* stream) {
  scheme.validate();
  const int total = scheme.n + scheme.k;
  for (int idx : lost.lost)
    if (idx < 0 || idx >= total) throw std::invalid_argument("coding: lost shard index out of range");
  if (static_cast<int>(lost.lost.size()) > max_tolerance(scheme))
    throw UnrecoverableError("coding: " + std::to_string(lost.lost.size()) + " erasures exceed tolerance " +
                             std::to_string(max_tolerance(scheme)) + " for scheme " + to_string(scheme.kind));
  if (static_cast<int>(d_survivors.size()) != scheme.n || static_cast<int>(h_parity.size()) != scheme.k)
    throw std::invalid_argument("coding: expected n device shards and k parity buffers");
  int data_lost = 0;
  for (int idx : lost.lost) data_lost += idx < scheme.n;
  if (static_cast<int>(d_out.size()) < data_lost) throw std::invalid_argument("coding: too few output buffers");
  if (len == 0 || data_lost == 0) return;
  gs_codec* c = detail::codec(scheme, nullptr);
  detail::check(gs_reconstruct_async(c, lost.lost.data(), static_cast<int>(lost.lost.size()), d_survivors.data(),
                                     h_parity.data(), d_out.data(), len, stream),
                "reconstruct");
}

// Wait for `stream` and the calling thread's implicit staging pipelines.
inline void sync(void* stream) { detail::check(gs_sync(stream), "sync"); }

}  // namespace ghostserve_gpu

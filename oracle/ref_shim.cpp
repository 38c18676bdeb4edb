// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the UNMODIFIED reference headers in place
// (-I/root/reference/proj/include; nothing is copied into this repo) and
// exposes their byte path through a C ABI so tests/ can generate golden
// vectors and bench.py can time the reference CPU codec (--impl reference,
// cpu_baseline.kind = "reference"). Built by oracle/Makefile into
// oracle/_ref/libghostserve_ref.so (git-ignored, travels with gpurun).
//
// Timing follows the reference bench convention (tools/ghostserve.cpp:262-283):
// steady_clock around the encode / reconstruct call only.
//
// The *_striped entry points are OUR wrapper, not the reference's: they call
// ghostserve::encode / reconstruct on disjoint byte stripes from T threads,
// which is valid because XOR and RS are position-wise (coding.hpp:143-172).
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

// kv_layout.hpp must precede parity_store.hpp (parity_store.hpp:15 vs :33).
#include "ghostserve/kv_layout.hpp"
#include "ghostserve/coding.hpp"
#include "ghostserve/gf256.hpp"
#include "ghostserve/parity_store.hpp"
#include "ghostserve/checkpoint.hpp"
#include "ghostserve/recovery.hpp"

using namespace ghostserve;

namespace {

int map_exception() {
  try {
    throw;
  } catch (const UnrecoverableError&) {
    return 2;
  } catch (const std::domain_error&) {
    return 3;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::logic_error&) {
    return 1;
  } catch (...) {
    return 2;
  }
}

CodingScheme scheme_of(int kind, int n, int k) {
  CodingScheme s;
  s.kind = kind == 0 ? CodeKind::kXor : kind == 1 ? CodeKind::kRdp : CodeKind::kReedSolomon;
  s.n = n;
  s.k = k;
  return s;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int encode_range(const CodingScheme& s, const uint8_t* const* data, size_t off, size_t len,
                 uint8_t* const* parity) {
  std::vector<ConstShardSpan> spans;
  for (int j = 0; j < s.n; ++j) spans.emplace_back(data[j] + off, len);
  auto out = encode(s, spans);
  for (int i = 0; i < s.k; ++i)
    if (len) std::memcpy(parity[i] + off, out[static_cast<size_t>(i)].data(), len);
  return 0;
}

int reconstruct_range(const CodingScheme& s, const uint8_t* const* shards, const int* lost,
                      int n_lost, size_t off, size_t len, uint8_t* const* out, int* n_out) {
  ErasurePattern pattern(std::vector<int>(lost, lost + n_lost));
  std::map<int, ConstShardSpan> surviving;
  for (int idx = 0; idx < s.n + s.k; ++idx)
    if (shards[idx] != nullptr) surviving[idx] = ConstShardSpan(shards[idx] + off, len);
  auto rebuilt = reconstruct(s, surviving, pattern);
  int b = 0;
  for (auto& [idx, bytes] : rebuilt) {
    (void)idx;
    if (len) std::memcpy(out[b] + off, bytes.data(), len);
    ++b;
  }
  *n_out = b;
  return 0;
}

}  // namespace

extern "C" {

uint8_t ghs_gf_mul(uint8_t a, uint8_t b) { return gf256::mul(a, b); }

int ghs_gf_inv(uint8_t a, uint8_t* out) {
  try {
    *out = gf256::inv(a);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

void ghs_gf_tables(uint8_t* exp_out, uint8_t* log_out) {
  std::memcpy(exp_out, gf256::kTables.exp.data(), 512);
  std::memcpy(log_out, gf256::kTables.log.data(), 256);
}

void ghs_mul_table(uint8_t* out /* 65536 */) {
  for (unsigned c = 0; c < 256; ++c) std::memcpy(out + c * 256, gf256::mul_row(static_cast<uint8_t>(c)), 256);
}

int ghs_validate(int kind, int n, int k) {
  try {
    scheme_of(kind, n, k).validate();
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ghs_max_tolerance(int kind, int n, int k) { return max_tolerance(scheme_of(kind, n, k)); }

int ghs_encoding_matrix(int kind, int n, int k, uint8_t* coef) {
  try {
    auto m = build_encoding_matrix(scheme_of(kind, n, k));
    std::memcpy(coef, m.coef.data(), m.coef.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ghs_encode(int kind, int n, int k, const uint8_t* const* data, size_t len,
               uint8_t* const* parity, double* secs) {
  try {
    const auto s = scheme_of(kind, n, k);
    std::vector<ConstShardSpan> spans;
    for (int j = 0; j < n; ++j) spans.emplace_back(data[j], len);
    const auto t0 = std::chrono::steady_clock::now();
    auto out = encode(s, spans);
    if (secs) *secs = seconds_since(t0);
    for (int i = 0; i < k; ++i)
      if (len) std::memcpy(parity[i], out[static_cast<size_t>(i)].data(), len);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ghs_reconstruct(int kind, int n, int k, const uint8_t* const* shards, const int* lost,
                    int n_lost, size_t len, uint8_t* const* out, int* n_out, double* secs) {
  try {
    const auto s = scheme_of(kind, n, k);
    ErasurePattern pattern(std::vector<int>(lost, lost + n_lost));
    std::map<int, ConstShardSpan> surviving;
    for (int idx = 0; idx < n + k; ++idx)
      if (shards[idx] != nullptr) surviving[idx] = ConstShardSpan(shards[idx], len);
    const auto t0 = std::chrono::steady_clock::now();
    auto rebuilt = reconstruct(s, surviving, pattern);
    if (secs) *secs = seconds_since(t0);
    int b = 0;
    for (auto& [idx, bytes] : rebuilt) {
      (void)idx;
      if (len) std::memcpy(out[b], bytes.data(), len);
      ++b;
    }
    *n_out = b;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Striped multi-thread wrappers (ours): T threads over disjoint 64-B aligned
// byte ranges, each calling the reference codec on its sub-spans.
int ghs_encode_striped(int kind, int n, int k, const uint8_t* const* data, size_t len,
                       uint8_t* const* parity, int threads, double* secs) {
  try {
    const auto s = scheme_of(kind, n, k);
    s.validate();
    if (threads < 1) threads = 1;
    size_t per = (len + threads - 1) / threads;
    per = (per + 63) & ~size_t{63};
    std::vector<std::thread> pool;
    std::vector<int> status(static_cast<size_t>(threads), 0);
    const auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < threads; ++t) {
      const size_t off = std::min(len, per * t), end = std::min(len, per * (t + 1));
      pool.emplace_back([&, t, off, end] {
        try {
          encode_range(s, data, off, end - off, parity);
        } catch (...) {
          status[static_cast<size_t>(t)] = map_exception();
        }
      });
    }
    for (auto& th : pool) th.join();
    if (secs) *secs = seconds_since(t0);
    for (int st : status)
      if (st) return st;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ghs_reconstruct_striped(int kind, int n, int k, const uint8_t* const* shards,
                            const int* lost, int n_lost, size_t len, uint8_t* const* out,
                            int* n_out, int threads, double* secs) {
  try {
    const auto s = scheme_of(kind, n, k);
    if (threads < 1) threads = 1;
    size_t per = (len + threads - 1) / threads;
    per = (per + 63) & ~size_t{63};
    std::vector<std::thread> pool;
    std::vector<int> status(static_cast<size_t>(threads), 0), counts(static_cast<size_t>(threads), 0);
    const auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < threads; ++t) {
      const size_t off = std::min(len, per * t), end = std::min(len, per * (t + 1));
      pool.emplace_back([&, t, off, end] {
        try {
          reconstruct_range(s, shards, lost, n_lost, off, end - off, out,
                            &counts[static_cast<size_t>(t)]);
        } catch (...) {
          status[static_cast<size_t>(t)] = map_exception();
        }
      });
    }
    for (auto& th : pool) th.join();
    if (secs) *secs = seconds_since(t0);
    for (int st : status)
      if (st) return st;
    *n_out = counts[0];
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Batch of independent stripes (e.g. the 32 requests of a decode block) on
// T threads, each thread taking whole stripes: the natural all-cores way to
// drive the reference codec (ours, not the reference's). Pointers are
// stripe-major: data[s*n + j], parity[s*k + i].
int ghs_encode_batch(int kind, int n, int k, int n_stripes, const uint8_t* const* data, size_t len,
                     uint8_t* const* parity, int threads, double* secs) {
  try {
    const auto s = scheme_of(kind, n, k);
    s.validate();
    if (threads < 1) threads = 1;
    std::atomic<int> next{0};
    std::vector<int> status(static_cast<size_t>(threads), 0);
    const auto t0 = std::chrono::steady_clock::now();
    auto work = [&](int t) {
      try {
        for (int st = next.fetch_add(1); st < n_stripes; st = next.fetch_add(1))
          encode_range(s, data + static_cast<size_t>(st) * n, 0, len, parity + static_cast<size_t>(st) * k);
      } catch (...) {
        status[static_cast<size_t>(t)] = map_exception();
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    if (secs) *secs = seconds_since(t0);
    for (int st : status)
      if (st) return st;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ghs_slice_bytes(int layers, int kv_heads, int head_dim, int tp, uint32_t chunk_size,
                    uint64_t* out) {
  try {
    ModelConfig m;
    m.layers = layers;
    m.kv_heads = kv_heads;
    m.head_dim = head_dim;
    m.tp_degree = tp;
    *out = slice_bytes(m, chunk_size);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ghs_make_ground_truth_slice(uint64_t seed, uint64_t req, uint32_t chunk, int worker,
                                int layers, int kv_heads, int head_dim, int tp,
                                uint32_t chunk_size, uint32_t valid, uint8_t* out) {
  try {
    ModelConfig m;
    m.layers = layers;
    m.kv_heads = kv_heads;
    m.head_dim = head_dim;
    m.tp_degree = tp;
    auto s = make_ground_truth_slice(seed, req, ChunkId{chunk}, worker, m, chunk_size, valid);
    std::memcpy(out, s.bytes.data(), s.bytes.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

uint64_t ghs_fnv1a64(const uint8_t* bytes, size_t len, uint64_t h) {
  return fnv1a64(std::span<const uint8_t>(bytes, len), h);
}

// checkpoint_chunk's byte work (checkpoint.hpp:143-147): encode + seal.
// Returns the sealed checksum; *secs covers encode + seal.
int ghs_encode_and_seal(int kind, int n, int k, const uint8_t* const* data, size_t len,
                        uint8_t* const* parity, uint64_t* checksum, double* secs) {
  try {
    const auto s = scheme_of(kind, n, k);
    std::vector<ConstShardSpan> spans;
    for (int j = 0; j < n; ++j) spans.emplace_back(data[j], len);
    const auto t0 = std::chrono::steady_clock::now();
    ParityChunk pc;
    pc.scheme = s;
    pc.slice_len = len;
    pc.parity = encode(s, spans);
    pc.seal();
    if (secs) *secs = seconds_since(t0);
    *checksum = pc.checksum;
    for (int i = 0; i < k; ++i)
      if (len) std::memcpy(parity[i], pc.parity[static_cast<size_t>(i)].data(), len);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

}  // extern "C"

// GSRV image of a ParityStore built by the reference (parity_store.hpp:145-263)
// from `count` entries: keys req[i]/chunk[i]/valid[i], parity[i*k + j] of
// slice_len bytes each, sealed with the reference's own seal().
extern "C" int ghs_gsrv_image(int kind, int n, int k, int count, const uint64_t* req, const uint32_t* chunk,
                              const uint32_t* valid, uint64_t slice_len, const uint8_t* const* parity,
                              uint8_t* out, uint64_t cap, uint64_t* size) {
  try {
    ParityStore store;
    for (int i = 0; i < count; ++i) {
      ParityChunk c;
      c.request_id = req[i];
      c.chunk_id = ChunkId{chunk[i]};
      c.scheme = scheme_of(kind, n, k);
      c.valid_tokens = valid[i];
      c.slice_len = slice_len;
      c.parity.resize(static_cast<size_t>(k));
      for (int j = 0; j < k; ++j)
        c.parity[static_cast<size_t>(j)].assign(parity[i * k + j], parity[i * k + j] + slice_len);
      c.seal();
      store.try_put(std::move(c));
    }
    auto bytes = serialize_parity_store(store);
    *size = bytes.size();
    if (out && cap >= bytes.size()) std::memcpy(out, bytes.data(), bytes.size());
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// The reference's own per-chunk entry points, timed as the reference bench
// does (steady_clock around the call): checkpoint_chunk (checkpoint.hpp:123-149:
// validate, encode, seal) and reconstruct_chunk (recovery.hpp:100-133: FNV
// verify, reconstruct, wrap). Slices are materialised as KvChunkSlice copies
// and the ParityChunk is sealed OUTSIDE the timed region.
namespace {
ModelConfig model_of(int layers, int kv_heads, int head_dim, int tp) {
  ModelConfig m;
  m.layers = layers;
  m.kv_heads = kv_heads;
  m.head_dim = head_dim;
  m.tp_degree = tp;
  return m;
}
}  // namespace

extern "C" int ghs_checkpoint_chunk_timed(int kind, int n, int k, int layers, int kv_heads, int head_dim,
                                          uint32_t chunk_size, uint64_t req, uint32_t chunk, uint32_t valid,
                                          const uint8_t* const* data, uint8_t* const* parity,
                                          uint64_t* checksum, double* secs) {
  try {
    CheckpointConfig cfg;
    cfg.scheme = scheme_of(kind, n, k);
    cfg.chunk_size = chunk_size;
    cfg.model = model_of(layers, kv_heads, head_dim, n);
    const uint64_t len = slice_bytes(cfg.model, chunk_size);
    std::vector<KvChunkSlice> slices(static_cast<size_t>(n));
    for (int w = 0; w < n; ++w) {
      auto& sl = slices[static_cast<size_t>(w)];
      sl.request_id = req;
      sl.chunk_id = ChunkId{chunk};
      sl.worker = w;
      sl.valid_tokens = valid;
      sl.bytes.assign(data[w], data[w] + len);
    }
    AssignmentState state;
    const auto t0 = std::chrono::steady_clock::now();
    auto out = checkpoint_chunk(slices, cfg, state, ChunkTiming{});
    if (secs) *secs = seconds_since(t0);
    *checksum = out.parity.checksum;
    for (int i = 0; i < k; ++i)
      if (len) std::memcpy(parity[i], out.parity.parity[static_cast<size_t>(i)].data(), len);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// slots[0..n+k): data workers then parity rows; NULL = lost. Rebuilt data
// workers (ascending) -> out. `sealed` = the checksum stored at checkpoint
// time (0: seal the given parity here). Returns 4 for kBadParity.
extern "C" int ghs_reconstruct_chunk_timed(int kind, int n, int k, uint64_t len, const uint8_t* const* slots,
                                           uint64_t sealed, uint8_t* const* out, int* n_out, double* secs) {
  try {
    ParityChunk pc;
    pc.scheme = scheme_of(kind, n, k);
    pc.slice_len = len;
    pc.parity.resize(static_cast<size_t>(k));
    for (int i = 0; i < k; ++i)
      if (slots[n + i]) pc.parity[static_cast<size_t>(i)].assign(slots[n + i], slots[n + i] + len);
    pc.seal();
    if (sealed) pc.checksum = sealed;
    std::vector<KvChunkSlice> surviving;
    std::set<int> failed;
    for (int w = 0; w < n; ++w) {
      if (!slots[w]) {
        failed.insert(w);
        continue;
      }
      KvChunkSlice sl;
      sl.worker = w;
      sl.bytes.assign(slots[w], slots[w] + len);
      surviving.push_back(std::move(sl));
    }
    const auto t0 = std::chrono::steady_clock::now();
    auto res = reconstruct_chunk(ChunkId{0}, surviving, pc, failed);
    if (secs) *secs = seconds_since(t0);
    if (res.status != ChunkRepairStatus::kOk) return 4;
    int b = 0;
    for (auto& [w, sl] : res.recovered) {
      (void)w;
      if (len) std::memcpy(out[b], sl.bytes.data(), len);
      ++b;
    }
    *n_out = b;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// The reference's hybrid recovery planner (recovery.hpp:58-88) on a given
// cost model (cost_model.hpp:18-24); the orchestration mirror is checked
// against it.
extern "C" int ghs_get_recompute_units(uint32_t n, uint32_t chunk_size, int kind, int sn, int sk, uint64_t slice,
                                       double compute_per_token, double intra_bw, double host_bw,
                                       double encode_rate, double reconstruct_rate, double fixed_latency,
                                       double restart, uint32_t* out) {
  try {
    CostModel c;
    c.compute_per_token = compute_per_token;
    c.intra_bw = intra_bw;
    c.host_bw = host_bw;
    c.encode_rate = encode_rate;
    c.reconstruct_rate = reconstruct_rate;
    c.fixed_collective_latency = fixed_latency;
    c.restart_overhead = restart;
    *out = get_recompute_units(n, chunk_size, scheme_of(kind, sn, sk), slice, c);
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// A reference ParityStore driven op by op (parity_store.hpp:62-143), so the
// host-tier mirror can be checked against it on random operation sequences.
extern "C" void* ghs_store_new(uint64_t capacity) { return new ParityStore(capacity); }
extern "C" void ghs_store_free(void* s) { delete static_cast<ParityStore*>(s); }
extern "C" int ghs_store_try_put(void* s, uint64_t req, uint32_t chunk, int kind, int n, int k, uint32_t valid,
                                 uint64_t slice_len, const uint8_t* const* parity, int* accepted) {
  try {
    ParityChunk c;
    c.request_id = req;
    c.chunk_id = ChunkId{chunk};
    c.scheme = scheme_of(kind, n, k);
    c.valid_tokens = valid;
    c.slice_len = slice_len;
    if (parity) {
      c.parity.resize(static_cast<size_t>(k));
      for (int i = 0; i < k; ++i) c.parity[static_cast<size_t>(i)].assign(parity[i], parity[i] + slice_len);
    }
    c.seal();
    *accepted = static_cast<ParityStore*>(s)->try_put(std::move(c)) ? 1 : 0;
    return 0;
  } catch (...) {
    return map_exception();
  }
}
extern "C" int ghs_store_get(void* s, uint64_t req, uint32_t chunk) {
  return static_cast<int>(static_cast<ParityStore*>(s)->get(req, chunk, nullptr));
}
extern "C" int ghs_store_contains(void* s, uint64_t req, uint32_t chunk) {
  return static_cast<ParityStore*>(s)->contains(req, chunk) ? 1 : 0;
}
extern "C" void ghs_store_erase(void* s, uint64_t req) { static_cast<ParityStore*>(s)->erase_request(req); }
extern "C" void ghs_store_corrupt(void* s, uint64_t req, uint32_t chunk) {
  static_cast<ParityStore*>(s)->corrupt_entry(req, chunk);
}
extern "C" void ghs_store_stats(void* s, uint64_t* out5) {
  auto* st = static_cast<ParityStore*>(s);
  out5[0] = st->used_bytes();
  out5[1] = st->payload_bytes();
  out5[2] = st->peak_payload_bytes();
  out5[3] = st->entry_count();
  out5[4] = st->audit() ? 1 : 0;
}

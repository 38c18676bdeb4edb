// ghostserve_gpu/parity_store.hpp -- drop-in facade for the reference's host
// tier (/root/reference/proj/include/ghostserve/parity_store.hpp:19-263) over
// the library's pinned-slab store (gs_store_*, csrc/gs_store.cu): same
// types, statuses, accounting, exceptions and GSRV image. try_put copies
// into pinned slabs (the reference's copying put); get re-verifies FNV-1a
// and hands out a pointer to a host copy owned by the facade, valid until the
// next get / erase of that entry or the store's destruction.
#pragma once

#include <cstdint>
#include <limits>
#include <map>
#include <span>
#include <stdexcept>
#include <utility>
#include <vector>

#include "kv_layout.hpp"

namespace ghostserve_gpu {

inline std::uint64_t fnv1a64(std::span<const std::uint8_t> bytes, std::uint64_t h = 0xcbf29ce484222325ull) {
  return gs_fnv1a64(bytes.data(), bytes.size(), h);
}

struct ParityChunk {  // :28-53
  std::uint64_t request_id = 0;
  ChunkId chunk_id;
  CodingScheme scheme;
  std::vector<std::vector<std::uint8_t>> parity;
  std::uint32_t valid_tokens = 0;
  std::uint64_t slice_len = 0;
  std::uint64_t checksum = 0;

  bool payload_present() const { return !parity.empty(); }
  std::uint64_t payload_bytes() const { return static_cast<std::uint64_t>(scheme.k) * slice_len; }
  std::uint64_t compute_checksum() const {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (const auto& buf : parity) h = fnv1a64(buf, h);
    return h;
  }
  void seal() { checksum = compute_checksum(); }
};

enum class ParityGetStatus { kOk, kMissing, kCorrupt };

class ParityStore {  // :62-143
 public:
  static constexpr std::uint64_t kPerEntryMetadataBytes = 64;
  static constexpr std::uint64_t kUnlimited = std::numeric_limits<std::uint64_t>::max();

  explicit ParityStore(std::uint64_t capacity_bytes = kUnlimited) {
    detail::check(gs_store_create(capacity_bytes, 2, &s_), "parity store");
  }
  explicit ParityStore(gs_store* adopted) : s_(adopted) {}
  ParityStore(ParityStore&& o) noexcept
      : s_(std::exchange(o.s_, nullptr)), view_(std::move(o.view_)), all_(std::move(o.all_)) {}
  ParityStore& operator=(ParityStore&& o) noexcept {
    if (this != &o) {
      if (s_) gs_store_destroy(s_);
      s_ = std::exchange(o.s_, nullptr);
      view_ = std::move(o.view_);
      all_ = std::move(o.all_);
    }
    return *this;
  }
  ParityStore(const ParityStore&) = delete;
  ParityStore& operator=(const ParityStore&) = delete;
  ~ParityStore() {
    if (s_) gs_store_destroy(s_);
  }

  std::uint64_t used_bytes() const { return stat(0); }
  std::uint64_t capacity_bytes() const { return stat(1); }
  std::uint64_t payload_bytes() const { return stat(2); }
  std::uint64_t peak_payload_bytes() const { return stat(3); }
  std::size_t entry_count() const { return static_cast<std::size_t>(stat(4)); }

  // :77-90 -- duplicate -> std::logic_error; over capacity -> false (no eviction).
  bool try_put(ParityChunk chunk) {
    std::vector<const void*> ptrs;
    for (const auto& b : chunk.parity) ptrs.push_back(b.data());
    if (chunk.payload_present() && static_cast<int>(ptrs.size()) != chunk.scheme.k)
      throw std::invalid_argument("parity store: entries carry k parity buffers");
    int accepted = 0;
    // no payload: a cost-only entry (KvPolicy::materialize = false)
    detail::check(gs_store_put(s_, chunk.request_id, chunk.chunk_id.index, static_cast<int>(chunk.scheme.kind),
                               chunk.scheme.n, chunk.scheme.k, chunk.valid_tokens, chunk.slice_len,
                               chunk.payload_present() ? ptrs.data() : nullptr, chunk.checksum, 1, &accepted),
                  "parity store");
    return accepted != 0;
  }

  // :92-101 -- kMissing / kCorrupt (FNV re-verified) / kOk with *out.
  ParityGetStatus get(std::uint64_t request_id, std::uint32_t chunk_index, const ParityChunk** out) const {
    ParityChunk c;
    const int status = materialize(request_id, chunk_index, /*verify=*/1, c);
    if (status == 1) return ParityGetStatus::kMissing;
    if (status == 2) return ParityGetStatus::kCorrupt;
    if (out) {
      ParityChunk& slot = view_[{request_id, chunk_index}];
      slot = std::move(c);
      *out = &slot;
    }
    return ParityGetStatus::kOk;
  }

  bool contains(std::uint64_t request_id, std::uint32_t chunk_index) const {
    return gs_store_contains(s_, request_id, chunk_index) != 0;
  }
  void erase_request(std::uint64_t request_id) {
    detail::check(gs_store_erase_request(s_, request_id), "parity store");
    view_.erase(view_.lower_bound({request_id, 0}), view_.upper_bound({request_id, ~std::uint32_t{0}}));
  }
  bool audit() const { return gs_store_audit(s_) != 0; }
  void corrupt_entry(std::uint64_t request_id, std::uint32_t chunk_index) {  // test hook (:126-131)
    gs_store_corrupt_entry(s_, request_id, chunk_index);
  }
  gs_store* handle() const { return s_; }

  // :133-135 -- every entry as stored (no verification: a corrupted entry's
  // bytes and recorded checksum), rebuilt from the store on each call; the
  // map stays valid until the next entries() call.
  const std::map<std::pair<std::uint64_t, std::uint32_t>, ParityChunk>& entries() const {
    std::uint64_t cnt = 0;
    detail::check(gs_store_keys(s_, nullptr, 0, &cnt), "parity store");
    std::vector<std::uint64_t> keys(2 * cnt + 2);
    detail::check(gs_store_keys(s_, keys.data(), cnt, &cnt), "parity store");
    all_.clear();
    for (std::uint64_t e = 0; e < cnt; ++e) {
      const auto req = keys[2 * e];
      const auto idx = static_cast<std::uint32_t>(keys[2 * e + 1]);
      materialize(req, idx, /*verify=*/0, all_[{req, idx}]);
    }
    return all_;
  }

 private:
  // copy of entry (req, idx) into c; returns the store status (0 ok, 1 missing, 2 corrupt)
  int materialize(std::uint64_t request_id, std::uint32_t chunk_index, int verify, ParityChunk& c) const {
    int status = 0, knk[3] = {0, 0, 0};
    void* rows[256];
    std::uint64_t slice_len = 0, checksum = 0;
    std::uint32_t valid = 0;
    detail::check(gs_store_get(s_, request_id, chunk_index, verify, &status, rows, &slice_len, &valid, &checksum,
                               knk),
                  "parity store");
    if (status != 0) return status;
    c = ParityChunk{};
    c.request_id = request_id;
    c.chunk_id = ChunkId{chunk_index};
    c.scheme = CodingScheme{static_cast<CodeKind>(knk[0]), knk[1], knk[2]};
    c.valid_tokens = valid;
    c.slice_len = slice_len;
    c.checksum = checksum;
    for (int i = 0; i < knk[2] && rows[0]; ++i) {  // rows NULL: cost-only entry, no payload
      const auto* p = static_cast<const std::uint8_t*>(rows[i]);
      c.parity.emplace_back(p, p + slice_len);
    }
    return 0;
  }

  std::uint64_t stat(int i) const {
    std::uint64_t v[5] = {0, 0, 0, 0, 0};
    detail::check(gs_store_stats(s_, v), "parity store");
    return v[i];
  }
  gs_store* s_ = nullptr;
  mutable std::map<std::pair<std::uint64_t, std::uint32_t>, ParityChunk> view_;
  mutable std::map<std::pair<std::uint64_t, std::uint32_t>, ParityChunk> all_;
};

// :201-263 -- the GSRV image, byte-identical to the reference's writer.
inline std::vector<std::uint8_t> serialize_parity_store(const ParityStore& store) {
  std::uint64_t size = 0;
  detail::check(gs_store_serialize(store.handle(), nullptr, 0, &size), "parity store");
  std::vector<std::uint8_t> out(size);
  detail::check(gs_store_serialize(store.handle(), out.data(), size, &size), "parity store");
  out.resize(size);
  return out;
}

inline ParityStore deserialize_parity_store(std::span<const std::uint8_t> bytes,
                                            std::uint64_t capacity_bytes = ParityStore::kUnlimited) {
  gs_store* s = nullptr;
  detail::check(gs_store_deserialize(bytes.data(), bytes.size(), capacity_bytes, 2, &s), "parity file");
  return ParityStore(s);
}

}  // namespace ghostserve_gpu

// gs_store.cu -- the host tier of the checkpoint: a ParityStore on pinned
// slabs (parity_store.hpp:31-143, 145-263 restated B200-side).
//
// Differences from the reference, all on the byte path's behalf:
//  * entries are RESERVED first and the encode kernel's D2H lands directly in
//    the entry's pinned slab (the reference encodes into fresh vectors and
//    copies them again in try_put, checkpoint.hpp:207);
//  * the FNV-1a seal (serial per chunk, ~1 GB/s per core) runs on a pool of
//    host threads once the parity bytes have landed (an event on the copy
//    stream, waited on by a landing thread: the stream never blocks on the
//    host), or arrives precomputed by the GPU (gs_store_commit_sealed_batch);
//  * pinned memory comes from a slab pool (cudaHostAlloc costs ~ms per call);
//    freed entries are reused lowest-address first, so a batch's entries stay
//    ascending and its D2H rows constant-pitch (one 2-D copy per row).
// Accounting, back-pressure, duplicate handling, get() verification and the
// GSRV file format are the reference's.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "../../include/gs_capi.h"
#include "gs_fnv.hpp"
#include "gs_host.hpp"

namespace gsb {
void set_last_error(const char* msg);  // gs_capi.cu: shared gs_last_error() slot
}

namespace {

int sfail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  gsb::set_last_error(buf);
  return status;
}

constexpr uint64_t kMetaBytes = 64;  // parity_store.hpp:67 kPerEntryMetadataBytes
constexpr uint64_t kUnlimited = ~0ull;

// Pinned slabs carved by exact size class; blocks are recycled, slabs are
// returned when the store dies.
class SlabPool {
 public:
  explicit SlabPool(size_t slab) : slab_(slab) {}
  ~SlabPool() {
    for (void* s : slabs_)
      if (!gsb::pinned_free_near(s)) cudaFreeHost(s);
  }
  int device = -1;  // >= 0: slabs placed on this GPU's NUMA node
  cudaError_t host_alloc(void** p, size_t bytes) {
    if (device >= 0) return gsb::pinned_alloc_near(device, bytes, p) == GS_OK ? cudaSuccess : cudaErrorMemoryAllocation;
    return cudaHostAlloc(p, bytes, cudaHostAllocPortable);
  }
  int alloc(size_t bytes, uint8_t** out) {
    bytes = std::max<size_t>(4096, (bytes + 4095) / 4096 * 4096);
    auto& fl = free_[bytes];
    if (!fl.empty()) {  // lowest address first: a batch's entries come back ascending,
      *out = *fl.begin();  // so its D2H rows stay constant-pitch runs (one 2-D copy per row)
      fl.erase(fl.begin());
      return GS_OK;
    }
    if (bytes > slab_ / 4) {  // large entries get their own allocation
      void* p = nullptr;
      cudaError_t e = host_alloc(&p, bytes);
      if (e != cudaSuccess) return sfail(GS_CUDA_ERROR, "store: pinned alloc of %zu B: %s", bytes, cudaGetErrorString(e));
      slabs_.push_back(p);
      *out = static_cast<uint8_t*>(p);
      return GS_OK;
    }
    if (!cur_ || used_ + bytes > slab_) {
      void* p = nullptr;
      cudaError_t e = host_alloc(&p, slab_);
      if (e != cudaSuccess) return sfail(GS_CUDA_ERROR, "store: pinned slab alloc: %s", cudaGetErrorString(e));
      slabs_.push_back(p);
      cur_ = static_cast<uint8_t*>(p);
      used_ = 0;
    }
    *out = cur_ + used_;
    used_ += bytes;
    return GS_OK;
  }
  void release(uint8_t* p, size_t bytes) {
    bytes = std::max<size_t>(4096, (bytes + 4095) / 4096 * 4096);
    free_[bytes].insert(p);
  }

 private:
  size_t slab_;
  std::vector<void*> slabs_;
  uint8_t* cur_ = nullptr;
  size_t used_ = 0;
  std::map<size_t, std::set<uint8_t*>> free_;
};

uint64_t fnv_chain(const uint8_t* p, size_t n, uint64_t h) { return gs_fnv1a64(p, n, h); }

}  // namespace

struct gs_store {
  struct Entry {
    int kind = 0, n = 0, k = 0;
    uint32_t valid = 0;
    uint64_t slice_len = 0;
    uint8_t* buf = nullptr;  // k * slice_len, parity i at buf + i * slice_len
    uint64_t checksum = 0;
    bool sealed = false;
    bool owned = true;
    uint64_t payload() const { return static_cast<uint64_t>(k) * slice_len; }
  };
  using Key = std::pair<uint64_t, uint32_t>;

  uint64_t capacity = kUnlimited;
  uint64_t used = 0, payload = 0, peak = 0;
  std::map<Key, Entry> entries;
  SlabPool pool{size_t{256} << 20};
  SlabPool sums_pool{size_t{1} << 20};  // 4 KiB pinned blocks for GPU-seal checksums
  std::mutex mu;
  std::condition_variable sealed_cv;

  // seal workers
  std::deque<Key> jobs;
  std::condition_variable job_cv;
  std::vector<std::thread> workers;
  bool stop = false;
  std::atomic<uint64_t> pending{0};

  // Seal workers hash pending entries: FNV-1a chained over the k buffers in
  // order == FNV over the entry's contiguous k * slice_len bytes
  // (parity_store.hpp:46-50). With the bit-sliced chain a worker takes ONE
  // entry at a time (the workers share a block's entries); the scalar chain
  // takes up to four of equal size and hashes them in lockstep (gs_fnv.hpp).
  void worker() {
    for (;;) {
      Key keys[4];
      const uint8_t* bufs[4];
      uint64_t len = 0;
      int m = 0, dropped = 0;
      const int claim = gsb::fnv_simd_available() ? 1 : 4;
      {
        std::unique_lock<std::mutex> lk(mu);
        job_cv.wait(lk, [&] { return stop || !jobs.empty(); });
        if (stop && jobs.empty()) return;
        while (!jobs.empty() && m < claim) {
          const Key key = jobs.front();
          auto it = entries.find(key);
          if (it == entries.end()) {
            jobs.pop_front();
            ++dropped;
            continue;
          }
          if (m > 0 && it->second.payload() != len) break;
          jobs.pop_front();
          len = it->second.payload();
          keys[m] = key;
          bufs[m] = it->second.buf;
          ++m;
        }
        pending -= static_cast<uint64_t>(dropped);
      }
      if (m == 0) {
        sealed_cv.notify_all();
        continue;
      }
      uint64_t h[4] = {gsb::kFnvOffset, gsb::kFnvOffset, gsb::kFnvOffset, gsb::kFnvOffset};
      if (len) gsb::fnv1a64_chains(bufs, m, len, h);
      {
        std::lock_guard<std::mutex> lk(mu);
        for (int q = 0; q < m; ++q) {
          auto it = entries.find(keys[q]);
          if (it != entries.end()) {
            it->second.checksum = h[q];
            it->second.sealed = true;
          }
        }
        pending -= static_cast<uint64_t>(m);
      }
      sealed_cv.notify_all();
    }
  }

  struct HostJob {
    gs_store* s;
    std::vector<Key> keys;
    // GPU seal: the checksums, copied on the commit's stream into pinned memory
    // the STORE owns (a pool block), so the caller's buffer only has to outlive
    // that stream position -- never the landing thread's wake-up.
    uint64_t* sums = nullptr;
    size_t sums_bytes = 0;
  };
  static void CUDART_CB on_stream(void* p) {
    auto* j = static_cast<HostJob*>(p);
    if (j->sums) {  // sealed on the device: record the checksums, no host FNV
      {
        std::lock_guard<std::mutex> lk(j->s->mu);
        for (size_t i = 0; i < j->keys.size(); ++i) {
          auto it = j->s->entries.find(j->keys[i]);
          if (it != j->s->entries.end()) {
            it->second.checksum = j->sums[i];
            it->second.sealed = true;
          }
        }
        j->s->sums_pool.release(reinterpret_cast<uint8_t*>(j->sums), j->sums_bytes);
        j->s->pending -= static_cast<uint64_t>(j->keys.size());
      }
      j->s->sealed_cv.notify_all();
      delete j;
      return;
    }
    {
      std::lock_guard<std::mutex> lk(j->s->mu);
      for (const auto& k : j->keys) j->s->jobs.push_back(k);
    }
    j->s->job_cv.notify_all();
    delete j;
  }

  // Landing queue: commit records an event on the D2H stream and this thread
  // waits for it, so the stream itself never blocks on a host callback (a
  // cudaLaunchHostFunc per block stalled the copy engine until the callback
  // thread ran: 207 -> 131 GB/s of KV on C2 blocks).
  struct Landing {
    cudaEvent_t ev;
    HostJob* job;
  };
  std::deque<Landing> landing;
  std::condition_variable land_cv;
  std::thread waiter;
  bool waiter_stop = false;

  void wait_loop() {
    for (;;) {
      Landing l{};
      {
        std::unique_lock<std::mutex> lk(mu);
        land_cv.wait(lk, [&] { return waiter_stop || !landing.empty(); });
        if (landing.empty()) return;  // stop requested and drained
        l = landing.front();
        landing.pop_front();
      }
      cudaEventSynchronize(l.ev);
      cudaEventDestroy(l.ev);
      on_stream(l.job);
    }
  }

  ~gs_store() {
    {
      std::lock_guard<std::mutex> lk(mu);
      waiter_stop = true;
    }
    land_cv.notify_all();
    if (waiter.joinable()) waiter.join();
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    job_cv.notify_all();
    for (auto& t : workers) t.join();
  }
};

extern "C" {

int gs_store_create(uint64_t capacity_bytes, int seal_threads, gs_store** out) {
  if (!out) return sfail(GS_INVALID_ARGUMENT, "store_create: out is NULL");
  auto* s = new gs_store;
  s->capacity = capacity_bytes;
  const int t = std::max(1, seal_threads);
  for (int i = 0; i < t; ++i) s->workers.emplace_back([s] { s->worker(); });
  s->waiter = std::thread([s] { s->wait_loop(); });
  *out = s;
  return GS_OK;
}

int gs_store_bind_device(gs_store* s, int device) {
  if (!s) return sfail(GS_INVALID_ARGUMENT, "store_bind_device: NULL store");
  std::lock_guard<std::mutex> lk(s->mu);
  s->pool.device = device;
  return GS_OK;
}

int gs_store_destroy(gs_store* s) {
  if (!s) return GS_OK;
  gs_store_wait_sealed(s);
  delete s;
  return GS_OK;
}

int gs_store_reserve(gs_store* s, uint64_t request_id, uint32_t chunk, int kind, int n, int k,
                     uint32_t valid_tokens, uint64_t slice_len, int* accepted, void** parity_out) {
  if (!s || !accepted) return sfail(GS_INVALID_ARGUMENT, "store_reserve: NULL argument");
  if (int st = gs_scheme_validate(kind, n, k)) return sfail(st, "%s", gs_last_error());
  *accepted = 0;
  std::lock_guard<std::mutex> lk(s->mu);
  const gs_store::Key key{request_id, chunk};
  if (s->entries.count(key))  // parity_store.hpp:78-82
    return sfail(GS_LOGIC_ERROR, "parity store: duplicate entry for request %llu chunk %u",
                 static_cast<unsigned long long>(request_id), chunk);
  const uint64_t pay = static_cast<uint64_t>(k) * slice_len;
  const uint64_t cost = pay + kMetaBytes;
  if (s->capacity != kUnlimited && s->used + cost > s->capacity) return GS_OK;  // back-pressure (:83)
  gs_store::Entry e;
  e.kind = kind;
  e.n = n;
  e.k = k;
  e.valid = valid_tokens;
  e.slice_len = slice_len;
  if (pay) {
    if (int st = s->pool.alloc(pay, &e.buf)) return st;
  }
  s->used += cost;
  s->payload += pay;
  s->peak = std::max(s->peak, s->payload);
  if (parity_out)
    for (int i = 0; i < k; ++i) parity_out[i] = e.buf ? e.buf + static_cast<uint64_t>(i) * slice_len : nullptr;
  s->entries.emplace(key, e);
  *accepted = 1;
  return GS_OK;
}

static int commit_batch(gs_store* s, int count, const uint64_t* request_ids, const uint32_t* chunks,
                        const uint64_t* sums, void* stream) {
  if (!s || count < 0 || (count > 0 && (!request_ids || !chunks)))
    return sfail(GS_INVALID_ARGUMENT, "store_commit: bad arguments");
  if (count == 0) return GS_OK;
  auto* job = new gs_store::HostJob{s, {}, nullptr, 0};
  job->keys.reserve(static_cast<size_t>(count));
  {
    std::lock_guard<std::mutex> lk(s->mu);
    for (int i = 0; i < count; ++i) {
      if (!s->entries.count({request_ids[i], chunks[i]})) {
        delete job;
        return sfail(GS_INVALID_ARGUMENT, "store_commit: no reserved entry for request %llu chunk %u",
                     static_cast<unsigned long long>(request_ids[i]), chunks[i]);
      }
      job->keys.push_back({request_ids[i], chunks[i]});
    }
    if (sums) {
      job->sums_bytes = sizeof(uint64_t) * static_cast<size_t>(count);
      uint8_t* blk = nullptr;
      if (int st = s->sums_pool.alloc(job->sums_bytes, &blk)) {
        delete job;
        return st;
      }
      job->sums = reinterpret_cast<uint64_t*>(blk);
    }
    s->pending += static_cast<uint64_t>(count);
  }
  auto undo = [&](int st) {
    std::lock_guard<std::mutex> lk(s->mu);
    if (job->sums) s->sums_pool.release(reinterpret_cast<uint8_t*>(job->sums), job->sums_bytes);
    s->pending -= static_cast<uint64_t>(count);
    delete job;
    s->sealed_cv.notify_all();
    return st;
  };
  cudaStream_t cst = static_cast<cudaStream_t>(stream);
  if (stream) {  // seal once the D2H on `stream` has landed: an event, waited on by the landing thread
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(cst, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
      return undo(sfail(GS_INVALID_ARGUMENT, "store_commit: cannot be captured into a CUDA graph (commit each replay)"));
    cudaError_t e = cudaSuccess;
    // checksums (device or host memory) -> the store's pinned block, ordered on the stream
    if (job->sums) e = cudaMemcpyAsync(job->sums, sums, job->sums_bytes, cudaMemcpyDefault, cst);
    cudaEvent_t ev = nullptr;
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventBlockingSync);
    if (e == cudaSuccess) e = cudaEventRecord(ev, cst);
    if (e != cudaSuccess) {
      if (ev) cudaEventDestroy(ev);
      return undo(sfail(GS_CUDA_ERROR, "store_commit: %s", cudaGetErrorString(e)));
    }
    {
      std::lock_guard<std::mutex> lk(s->mu);
      s->landing.push_back({ev, job});
    }
    s->land_cv.notify_one();
    return GS_OK;
  }
  if (job->sums) {  // no stream: the checksums are final now
    cudaError_t e = cudaMemcpy(job->sums, sums, job->sums_bytes, cudaMemcpyDefault);
    if (e != cudaSuccess) return undo(sfail(GS_CUDA_ERROR, "store_commit: %s", cudaGetErrorString(e)));
  }
  gs_store::on_stream(job);
  return GS_OK;
}

int gs_store_commit_batch(gs_store* s, int count, const uint64_t* request_ids, const uint32_t* chunks,
                          void* stream) {
  return commit_batch(s, count, request_ids, chunks, nullptr, stream);
}

int gs_store_commit_sealed_batch(gs_store* s, int count, const uint64_t* request_ids, const uint32_t* chunks,
                                 const uint64_t* checksums, void* stream) {
  if (count > 0 && !checksums) return sfail(GS_INVALID_ARGUMENT, "store_commit_sealed: NULL checksums");
  return commit_batch(s, count, request_ids, chunks, checksums, stream);
}

int gs_store_commit(gs_store* s, uint64_t request_id, uint32_t chunk, void* stream) {
  return gs_store_commit_batch(s, 1, &request_id, &chunk, stream);
}

// Reserve `count` entries of one scheme / length at once (all-or-nothing on
// back-pressure: *accepted = number reserved before the first refusal).
int gs_store_reserve_batch(gs_store* s, int count, const uint64_t* request_ids, const uint32_t* chunks, int kind,
                           int n, int k, uint32_t valid_tokens, uint64_t slice_len, int* accepted,
                           void** parity_out) {
  if (!s || !accepted || count < 0) return sfail(GS_INVALID_ARGUMENT, "store_reserve: bad arguments");
  *accepted = 0;
  for (int i = 0; i < count; ++i) {
    int acc = 0;
    if (int st = gs_store_reserve(s, request_ids[i], chunks[i], kind, n, k, valid_tokens, slice_len, &acc,
                                  parity_out ? parity_out + static_cast<size_t>(i) * k : nullptr))
      return st;
    if (!acc) return GS_OK;
    ++*accepted;
  }
  return GS_OK;
}

int gs_store_wait_sealed(gs_store* s) {
  if (!s) return GS_OK;
  std::unique_lock<std::mutex> lk(s->mu);
  s->sealed_cv.wait(lk, [&] { return s->pending.load() == 0; });
  return GS_OK;
}

// Copying put with the reference's try_put semantics (parity_store.hpp:77-90):
// parity[k] host buffers are copied into the store and sealed synchronously.
int gs_store_put(gs_store* s, uint64_t request_id, uint32_t chunk, int kind, int n, int k,
                 uint32_t valid_tokens, uint64_t slice_len, const void* const* parity, uint64_t checksum,
                 int sealed, int* accepted) {
  void* dst[256];
  if (k > 256) return sfail(GS_INVALID_ARGUMENT, "store_put: k too large");
  if (!parity) {  // cost-only entry (the reference's KvPolicy::materialize = false, checkpoint.hpp:51-54):
                  // accounted like a full one, no bytes held, get() -> kOk without a payload
    if (!s || !accepted) return sfail(GS_INVALID_ARGUMENT, "store_put: NULL argument");
    if (int st = gs_scheme_validate(kind, n, k)) return sfail(st, "%s", gs_last_error());
    *accepted = 0;
    std::lock_guard<std::mutex> lk(s->mu);
    const gs_store::Key key{request_id, chunk};
    if (s->entries.count(key))
      return sfail(GS_LOGIC_ERROR, "parity store: duplicate entry for request %llu chunk %u",
                   static_cast<unsigned long long>(request_id), chunk);
    const uint64_t pay = static_cast<uint64_t>(k) * slice_len, cost = pay + kMetaBytes;
    if (s->capacity != kUnlimited && s->used + cost > s->capacity) return GS_OK;
    gs_store::Entry e;
    e.kind = kind;
    e.n = n;
    e.k = k;
    e.valid = valid_tokens;
    e.slice_len = slice_len;
    e.owned = false;
    e.checksum = sealed ? checksum : 0xcbf29ce484222325ull;
    e.sealed = true;
    s->used += cost;
    s->payload += pay;
    s->peak = std::max(s->peak, s->payload);
    s->entries.emplace(key, e);
    *accepted = 1;
    return GS_OK;
  }
  if (int st = gs_store_reserve(s, request_id, chunk, kind, n, k, valid_tokens, slice_len, accepted, dst)) return st;
  if (!*accepted) return GS_OK;
  for (int i = 0; i < k; ++i)
    if (slice_len) std::memcpy(dst[i], parity[i], slice_len);
  std::lock_guard<std::mutex> lk(s->mu);
  auto& e = s->entries.at({request_id, chunk});
  e.checksum = sealed ? checksum : (e.buf ? fnv_chain(e.buf, e.payload(), 0xcbf29ce484222325ull)
                                          : 0xcbf29ce484222325ull);
  e.sealed = true;
  return GS_OK;
}

// parity_store.hpp:92-101: kOk / kMissing / kCorrupt (status out: 0/1/2).
int gs_store_get(gs_store* s, uint64_t request_id, uint32_t chunk, int verify, int* status, void** parity_out,
                 uint64_t* slice_len, uint32_t* valid_tokens, uint64_t* checksum, int* kind_n_k) {
  if (!s || !status) return sfail(GS_INVALID_ARGUMENT, "store_get: NULL argument");
  std::unique_lock<std::mutex> lk(s->mu);
  auto it = s->entries.find({request_id, chunk});
  if (it == s->entries.end()) {
    *status = 1;
    return GS_OK;
  }
  s->sealed_cv.wait(lk, [&] {
    auto jt = s->entries.find({request_id, chunk});
    return jt == s->entries.end() || jt->second.sealed;
  });
  it = s->entries.find({request_id, chunk});
  if (it == s->entries.end()) {
    *status = 1;
    return GS_OK;
  }
  const gs_store::Entry e = it->second;
  lk.unlock();
  if (verify && e.buf && fnv_chain(e.buf, e.payload(), 0xcbf29ce484222325ull) != e.checksum) {
    *status = 2;
    return GS_OK;
  }
  *status = 0;
  if (parity_out)
    for (int i = 0; i < e.k; ++i) parity_out[i] = e.buf ? e.buf + static_cast<uint64_t>(i) * e.slice_len : nullptr;
  if (slice_len) *slice_len = e.slice_len;
  if (valid_tokens) *valid_tokens = e.valid;
  if (checksum) *checksum = e.checksum;
  if (kind_n_k) {
    kind_n_k[0] = e.kind;
    kind_n_k[1] = e.n;
    kind_n_k[2] = e.k;
  }
  return GS_OK;
}

int gs_store_contains(gs_store* s, uint64_t request_id, uint32_t chunk) {
  if (!s) return 0;
  std::lock_guard<std::mutex> lk(s->mu);
  return s->entries.count({request_id, chunk}) ? 1 : 0;
}

// parity_store.hpp:105-112
int gs_store_erase_request(gs_store* s, uint64_t request_id) {
  if (!s) return sfail(GS_INVALID_ARGUMENT, "store_erase: NULL store");
  gs_store_wait_sealed(s);
  std::lock_guard<std::mutex> lk(s->mu);
  auto it = s->entries.lower_bound({request_id, 0u});
  while (it != s->entries.end() && it->first.first == request_id) {
    s->used -= it->second.payload() + kMetaBytes;
    s->payload -= it->second.payload();
    if (it->second.buf && it->second.owned) s->pool.release(it->second.buf, it->second.payload());
    it = s->entries.erase(it);
  }
  return GS_OK;
}

// used, capacity, payload, peak_payload, entry_count
int gs_store_stats(gs_store* s, uint64_t* out5) {
  if (!s || !out5) return sfail(GS_INVALID_ARGUMENT, "store_stats: NULL argument");
  std::lock_guard<std::mutex> lk(s->mu);
  out5[0] = s->used;
  out5[1] = s->capacity;
  out5[2] = s->payload;
  out5[3] = s->peak;
  out5[4] = s->entries.size();
  return GS_OK;
}

// parity_store.hpp:115-123
int gs_store_audit(gs_store* s) {
  if (!s) return 0;
  std::lock_guard<std::mutex> lk(s->mu);
  uint64_t sum = 0;
  for (const auto& kv : s->entries) sum += kv.second.payload() + kMetaBytes;
  return sum == s->used ? 1 : 0;
}

// Test hook (parity_store.hpp:126-131): flip parity[0][0].
int gs_store_corrupt_entry(gs_store* s, uint64_t request_id, uint32_t chunk) {
  if (!s) return GS_OK;
  gs_store_wait_sealed(s);
  std::lock_guard<std::mutex> lk(s->mu);
  auto it = s->entries.find({request_id, chunk});
  if (it == s->entries.end() || !it->second.buf || !it->second.payload()) return GS_OK;
  it->second.buf[0] ^= 0xFF;
  return GS_OK;
}

// Keys in (request, chunk) order: keys[2*i] = request, keys[2*i+1] = chunk.
int gs_store_keys(gs_store* s, uint64_t* keys, uint64_t max_entries, uint64_t* count) {
  if (!s || !count) return sfail(GS_INVALID_ARGUMENT, "store_keys: NULL argument");
  std::lock_guard<std::mutex> lk(s->mu);
  uint64_t i = 0;
  for (const auto& kv : s->entries) {
    if (keys && i < max_entries) {
      keys[2 * i] = kv.first.first;
      keys[2 * i + 1] = kv.first.second;
    }
    ++i;
  }
  *count = i;
  return GS_OK;
}

// ---- GSRV persistence (parity_store.hpp:145-263) --------------------------
// magic "GSRV", u16 version=1, u8 kind, u8 n, u8 k; per entry (key order):
// u64 request, u32 chunk, u32 valid_tokens, u64 slice_len, k * slice_len
// parity bytes, u64 checksum. All little-endian.
int gs_store_serialize(gs_store* s, void* out, uint64_t cap, uint64_t* size) {
  if (!s || !size) return sfail(GS_INVALID_ARGUMENT, "store_serialize: NULL argument");
  gs_store_wait_sealed(s);
  std::lock_guard<std::mutex> lk(s->mu);
  if (s->entries.empty()) return sfail(GS_INVALID_ARGUMENT, "parity store: nothing to serialize");
  const auto& first = s->entries.begin()->second;
  uint64_t need = 4 + 2 + 3;
  for (const auto& kv : s->entries) {
    const auto& e = kv.second;
    if (e.kind != first.kind || e.n != first.n || e.k != first.k)
      return sfail(GS_INVALID_ARGUMENT, "parity store: mixed schemes cannot be serialized");
    if (!e.buf && e.payload())
      return sfail(GS_INVALID_ARGUMENT, "parity store: cannot serialize entries without payloads");
    need += 8 + 4 + 4 + 8 + e.payload() + 8;
  }
  *size = need;
  if (!out) return GS_OK;
  if (cap < need) return sfail(GS_INVALID_ARGUMENT, "store_serialize: buffer too small (%llu < %llu)",
                               static_cast<unsigned long long>(cap), static_cast<unsigned long long>(need));
  uint8_t* p = static_cast<uint8_t*>(out);
  auto put = [&](uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) *p++ = static_cast<uint8_t>(v >> (8 * i));
  };
  *p++ = 'G';
  *p++ = 'S';
  *p++ = 'R';
  *p++ = 'V';
  put(1, 2);
  put(static_cast<uint64_t>(first.kind), 1);
  put(static_cast<uint64_t>(first.n), 1);
  put(static_cast<uint64_t>(first.k), 1);
  for (const auto& kv : s->entries) {
    const auto& e = kv.second;
    put(kv.first.first, 8);
    put(kv.first.second, 4);
    put(e.valid, 4);
    put(e.slice_len, 8);
    if (e.payload()) std::memcpy(p, e.buf, e.payload());
    p += e.payload();
    put(e.checksum, 8);
  }
  return GS_OK;
}

int gs_store_deserialize(const void* bytes, uint64_t size, uint64_t capacity, int seal_threads, gs_store** out) {
  if (!bytes || !out) return sfail(GS_INVALID_ARGUMENT, "store_deserialize: NULL argument");
  *out = nullptr;
  const uint8_t* p = static_cast<const uint8_t*>(bytes);
  uint64_t pos = 0;
  auto take = [&](uint64_t n, const uint8_t** q) -> bool {
    if (pos + n > size) return false;
    *q = p + pos;
    pos += n;
    return true;
  };
  auto get = [&](int nbytes, uint64_t* v) -> bool {
    const uint8_t* q;
    if (!take(static_cast<uint64_t>(nbytes), &q)) return false;
    *v = 0;
    for (int i = 0; i < nbytes; ++i) *v |= static_cast<uint64_t>(q[i]) << (8 * i);
    return true;
  };
  const uint8_t* magic;
  if (!take(4, &magic)) return sfail(GS_RUNTIME_ERROR, "parity file: truncated");
  if (std::memcmp(magic, "GSRV", 4) != 0) return sfail(GS_RUNTIME_ERROR, "parity file: bad magic");
  uint64_t version, kind, n, k;
  if (!get(2, &version)) return sfail(GS_RUNTIME_ERROR, "parity file: truncated");
  if (version != 1) return sfail(GS_RUNTIME_ERROR, "parity file: unsupported version");
  if (!get(1, &kind) || !get(1, &n) || !get(1, &k)) return sfail(GS_RUNTIME_ERROR, "parity file: truncated");
  if (int st = gs_scheme_validate(static_cast<int>(kind), static_cast<int>(n), static_cast<int>(k)))
    return sfail(st, "%s", gs_last_error());
  gs_store* s = nullptr;
  gs_store_create(capacity, seal_threads, &s);
  while (pos < size) {
    uint64_t req, chunk, valid, slice;
    if (!get(8, &req) || !get(4, &chunk) || !get(4, &valid) || !get(8, &slice)) {
      gs_store_destroy(s);
      return sfail(GS_RUNTIME_ERROR, "parity file: truncated");
    }
    const uint8_t* payload;
    if (slice > size || !take(k * slice, &payload)) {
      gs_store_destroy(s);
      return sfail(GS_RUNTIME_ERROR, "parity file: truncated");
    }
    uint64_t checksum;
    if (!get(8, &checksum)) {
      gs_store_destroy(s);
      return sfail(GS_RUNTIME_ERROR, "parity file: truncated");
    }
    if (fnv_chain(payload, k * slice, 0xcbf29ce484222325ull) != checksum) {
      gs_store_destroy(s);
      return sfail(GS_RUNTIME_ERROR, "parity file: checksum mismatch for request %llu chunk %llu",
                   static_cast<unsigned long long>(req), static_cast<unsigned long long>(chunk));
    }
    const void* par[256];
    for (uint64_t i = 0; i < k; ++i) par[i] = payload + i * slice;
    int accepted = 0;
    int st = gs_store_put(s, req, static_cast<uint32_t>(chunk), static_cast<int>(kind), static_cast<int>(n),
                          static_cast<int>(k), static_cast<uint32_t>(valid), slice, par, checksum, 1, &accepted);
    if (st) {
      gs_store_destroy(s);
      return st;
    }
    if (!accepted) {
      gs_store_destroy(s);
      return sfail(GS_RUNTIME_ERROR, "parity file: contents exceed store capacity");
    }
  }
  *out = s;
  return GS_OK;
}

}  // extern "C"

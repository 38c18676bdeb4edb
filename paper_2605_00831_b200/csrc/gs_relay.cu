// gs_relay.cu -- host side of the striped seal at N>1 (peer.py chain_striped /
// RelayBoard): a ParityChunk checksum (parity_store.hpp:19-53) is one FNV-1a
// chain over a chunk's whole parity rows, and with byte-range striping each
// rank holds one range of every row, so the chain is continued range by range
// through the ranks: on host threads (the bit-sliced chain of gs_fnv_simd.cpp)
// and, for rows already in HBM, on this rank's GPU (the seeded window kernel
// of gs_fnv_gpu.cu, gs_fnv_relay_device).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/gs_capi.h"
#include "gs_fnv.hpp"

namespace gsb {
void set_last_error(const char* msg);  // gs_capi.cu: shared gs_last_error() slot
}

using namespace gsb;

namespace {

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  gsb::set_last_error(buf);
  return status;
}

}  // namespace

int gs_fnv1a64_continue_batch(const void* const* bufs, const uint64_t* lens, const uint64_t* h_in,
                              uint64_t* h_out, int m, int threads) {
  if (m < 0 || (m > 0 && (!bufs || !lens || !h_in || !h_out)))
    return fail(GS_INVALID_ARGUMENT, "fnv1a64_continue_batch: bad arguments");
  for (int q = 0; q < m; ++q)
    if (lens[q] && !bufs[q]) return fail(GS_INVALID_ARGUMENT, "fnv1a64_continue_batch: NULL segment");
  // segments are claimed longest first so a round's tail is one short chain
  std::vector<int> order(static_cast<size_t>(m));
  for (int q = 0; q < m; ++q) order[q] = q;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return lens[a] > lens[b]; });
  threads = std::max(1, std::min(threads, m));
  std::atomic<int> next{0};
  auto work = [&] {
    for (int i = next.fetch_add(1); i < m; i = next.fetch_add(1)) {
      const int q = order[i];
      const uint8_t* p = static_cast<const uint8_t*>(bufs[q]);
      uint64_t h = h_in[q];
      fnv1a64_chains(&p, 1, lens[q], &h);
      h_out[q] = h;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  return GS_OK;
}

// Striped checksum relay through a board in host memory shared by the ranks of
// one node. Chain position p = i*world + r is (row i, rank r's range); slot
// (c, p) receives the chain state after that segment, tagged with the call's
// epoch (release store; the next position's owner acquires it). Each rank's
// threads claim its segments in (row, chunk) order, the order the states
// arrive in, so no barrier separates rows or ranks: rank r runs one segment
// behind rank r-1, and rank 0's row i+1 finds rank W-1's row i long done.
namespace {

struct RelaySlot {
  uint64_t h, tag;
};

// One call's view of the board: the slots of [n_chunks][k * world], this
// call's epoch, a deadline, and an abort flag every waiter checks.
class Board {
 public:
  Board(void* mem, uint64_t epoch, int npos, double timeout_s)
      : slots_(static_cast<RelaySlot*>(mem)),
        epoch_(epoch),
        npos_(npos),
        deadline_(std::chrono::steady_clock::now() +
                  std::chrono::microseconds(static_cast<int64_t>((timeout_s > 0 ? timeout_s : 60.0) * 1e6))) {}

  // The state after position p of chunk c, once published in this epoch. A
  // segment takes milliseconds, so a waiter backs off to short sleeps after a
  // brief spin: the ranks' relays share the node's cores, and a spinning
  // waiter would take cycles from the threads it is waiting for.
  bool await(int c, int p, uint64_t* h) {
    RelaySlot& s = slot(c, p);
    for (uint32_t spin = 0;; ++spin) {
      if (__atomic_load_n(&s.tag, __ATOMIC_ACQUIRE) == epoch_) {
        *h = s.h;
        return true;
      }
      if (failed_.load(std::memory_order_relaxed)) return false;
      if (spin < 512) {
        __builtin_ia32_pause();
        continue;
      }
      if ((spin & 63) == 0 && std::chrono::steady_clock::now() > deadline_) {
        failed_.store(1);
        return false;
      }
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }
  void publish(int c, int p, uint64_t h) {
    RelaySlot& s = slot(c, p);
    s.h = h;
    __atomic_store_n(&s.tag, epoch_, __ATOMIC_RELEASE);
  }
  void abort() { failed_.store(1); }
  bool failed() const { return failed_.load() != 0; }

 private:
  RelaySlot& slot(int c, int p) { return slots_[static_cast<size_t>(c) * npos_ + p]; }
  RelaySlot* slots_;
  uint64_t epoch_;
  int npos_;
  std::chrono::steady_clock::time_point deadline_;
  std::atomic<int> failed_{0};
};

// Small pinned seed/state arrays of the GPU worker, recycled across calls:
// cudaFreeHost would synchronise the whole device at the end of every relay
// (an unrelated decode included).
std::mutex g_io_mu;
std::vector<std::pair<size_t, void*>> g_io_free;

void* io_take(size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_io_mu);
    for (size_t i = 0; i < g_io_free.size(); ++i)
      if (g_io_free[i].first >= bytes) {
        void* p = g_io_free[i].second;
        g_io_free.erase(g_io_free.begin() + static_cast<long>(i));
        return p;
      }
  }
  void* p = nullptr;
  return cudaHostAlloc(&p, std::max<size_t>(bytes, 4096), cudaHostAllocDefault) == cudaSuccess ? p : nullptr;
}

void io_give(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_io_mu);
  g_io_free.push_back({std::max<size_t>(bytes, 4096), p});
}

// The GPU worker (rows 0..k_dev-1 on this rank's GPU), run by the calling
// thread: for each device row, in batches of `batch` chunks in chunk order,
// wait for the batch's predecessor states, upload them as seeds, run the
// seeded window kernel over this rank's ranges (after the chunks' `ready`
// events), read the states back and publish them.
int gpu_worker(Board& bd, int rank, int world, const void* const* d_rows, int k_dev, void* const* ready,
               uint64_t len, int n_chunks, uint64_t h0, int batch, cudaStream_t st) {
  const size_t io_bytes = sizeof(uint64_t) * 2 * batch;  // [seeds | states] x batch
  uint64_t* h_io = static_cast<uint64_t*>(io_take(io_bytes));
  uint64_t* d_io = nullptr;
  cudaError_t e = h_io ? cudaSuccess : cudaErrorMemoryAllocation;
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&d_io), io_bytes, st);
  int status = e == cudaSuccess ? GS_OK : fail(GS_CUDA_ERROR, "fnv_relay_device: buffers: %s", cudaGetErrorString(e));
  std::vector<const void*> bufs(static_cast<size_t>(batch));
  for (int i = 0; i < k_dev && status == GS_OK; ++i) {
    const int p = i * world + rank;
    for (int c0 = 0; c0 < n_chunks && status == GS_OK; c0 += batch) {
      const int cnt = std::min(batch, n_chunks - c0);
      for (int q = 0; q < cnt && status == GS_OK; ++q) {
        h_io[q] = h0;
        if (p > 0 && !bd.await(c0 + q, p - 1, &h_io[q]))
          status = fail(GS_RUNTIME_ERROR, "fnv_relay_device: timed out waiting for a peer rank's chain state");
        bufs[q] = d_rows[static_cast<size_t>(c0 + q) * k_dev + i];
      }
      if (status != GS_OK) break;
      if (len) {
        if (i == 0 && ready)  // the chunks' device rows are complete (later rows follow in stream order)
          for (int q = 0; q < cnt && e == cudaSuccess; ++q)
            if (ready[c0 + q]) e = cudaStreamWaitEvent(st, static_cast<cudaEvent_t>(ready[c0 + q]), 0);
        if (e == cudaSuccess) e = cudaMemcpyAsync(d_io, h_io, sizeof(uint64_t) * cnt, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) {
          status = fail(GS_CUDA_ERROR, "fnv_relay_device: %s", cudaGetErrorString(e));
          break;
        }
        if ((status = gs_fnv1a64_device_seeded(bufs.data(), cnt, 1, len, d_io, d_io + batch, st)) != GS_OK) break;
        e = cudaMemcpyAsync(h_io + batch, d_io + batch, sizeof(uint64_t) * cnt, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
          status = fail(GS_CUDA_ERROR, "fnv_relay_device: %s", cudaGetErrorString(e));
          break;
        }
      } else {
        for (int q = 0; q < cnt; ++q) h_io[batch + q] = h_io[q];  // an empty range passes the state on
      }
      for (int q = 0; q < cnt; ++q) bd.publish(c0 + q, p, h_io[batch + q]);
    }
  }
  if (d_io) cudaFreeAsync(d_io, st);
  cudaStreamSynchronize(st);  // h_io's last D2H has landed before it is recycled
  io_give(h_io, io_bytes);
  return status;
}

// Rows k_dev..k-1 of every chunk on host threads (the calling thread joins in
// when there is no GPU work), then every chunk's checksum from the last
// position. `d_rows` / `st` are used only when k_dev > 0.
int relay(void* board, uint64_t epoch, int rank, int world, const void* const* d_rows, int k_dev, void* const* ready,
          const void* const* h_rows, uint64_t len, int n_chunks, int k, uint64_t h0, int threads, int batch,
          cudaStream_t st, double timeout_s, uint64_t* sums) {
  const int npos = k * world;
  Board bd(board, epoch, npos, timeout_s);
  const int segs = n_chunks * (k - k_dev);
  std::atomic<int> next{0};
  auto host_work = [&] {
    for (int q = next.fetch_add(1); q < segs; q = next.fetch_add(1)) {
      const int i = k_dev + q / n_chunks, c = q % n_chunks, p = i * world + rank;
      uint64_t h = h0;
      if (p > 0 && !bd.await(c, p - 1, &h)) return;
      const uint8_t* b = static_cast<const uint8_t*>(len ? h_rows[static_cast<size_t>(c) * k + i] : nullptr);
      fnv1a64_chains(&b, 1, len, &h);
      bd.publish(c, p, h);
    }
  };
  const bool gpu = k_dev > 0 && n_chunks > 0;
  const int spawn = segs > 0 ? std::max(1, std::min(threads, segs)) - (gpu ? 0 : 1) : 0;
  std::vector<std::thread> pool;
  for (int t = 0; t < spawn; ++t) pool.emplace_back(host_work);
  int status = GS_OK;
  if (gpu) {
    status = gpu_worker(bd, rank, world, d_rows, k_dev, ready, len, n_chunks, h0, batch, st);
    if (status != GS_OK) bd.abort();  // release the host threads
  } else if (segs > 0) {
    host_work();
  }
  for (auto& t : pool) t.join();
  if (status != GS_OK) return status;
  for (int c = 0; c < n_chunks && !bd.failed(); ++c)
    if (!bd.await(c, npos - 1, &sums[c])) break;
  if (bd.failed()) return fail(GS_RUNTIME_ERROR, "fnv_relay: timed out waiting for a peer rank's chain state");
  return GS_OK;
}

}  // namespace

uint64_t gs_relay_board_bytes(int n_chunks, int k, int world) {
  if (n_chunks < 0 || k < 1 || world < 1) return 0;
  return static_cast<uint64_t>(n_chunks) * k * world * sizeof(RelaySlot);
}

int gs_fnv_relay(void* board, uint64_t epoch, int rank, int world, const void* const* rows, uint64_t len,
                 int n_chunks, int k, uint64_t h0, int threads, double timeout_s, uint64_t* sums) {
  if (!board || epoch == 0 || world < 1 || rank < 0 || rank >= world || n_chunks < 0 || k < 1 || !sums ||
      (n_chunks > 0 && len && !rows))
    return fail(GS_INVALID_ARGUMENT, "fnv_relay: bad arguments");
  if (len)
    for (int q = 0; q < n_chunks * k; ++q)
      if (!rows[q]) return fail(GS_INVALID_ARGUMENT, "fnv_relay: NULL row");
  return relay(board, epoch, rank, world, nullptr, 0, nullptr, rows, len, n_chunks, k, h0, threads, 1, nullptr,
               timeout_s, sums);
}

// gs_fnv_relay with the leading k_dev rows of every chunk hashed on this
// rank's GPU (gpu_worker). Host threads depend on GPU-published states only,
// and the GPU workers of the ranks only on each other, so the two relays
// cannot wait on one another in a cycle.
int gs_fnv_relay_device(void* board, uint64_t epoch, int rank, int world, const void* const* d_rows, int k_dev,
                        void* const* ready, const void* const* h_rows, uint64_t len, int n_chunks, int k,
                        uint64_t h0, int threads, int batch, void* stream, double timeout_s, uint64_t* sums) {
  if (!board || epoch == 0 || world < 1 || rank < 0 || rank >= world || n_chunks < 0 || k < 1 || k_dev < 0 ||
      k_dev > k || batch < 1 || !sums || (n_chunks > 0 && k_dev > 0 && len && !d_rows) ||
      (n_chunks > 0 && k_dev < k && len && !h_rows))
    return fail(GS_INVALID_ARGUMENT, "fnv_relay_device: bad arguments");
  if (k_dev > 0 && len % 16) return fail(GS_INVALID_ARGUMENT, "fnv_relay_device: range length must be a multiple of 16");
  if (len)
    for (int c = 0; c < n_chunks; ++c) {
      for (int i = 0; i < k_dev; ++i)
        if (!d_rows[static_cast<size_t>(c) * k_dev + i]) return fail(GS_INVALID_ARGUMENT, "fnv_relay_device: NULL device row");
      for (int i = k_dev; i < k; ++i)
        if (!h_rows[static_cast<size_t>(c) * k + i]) return fail(GS_INVALID_ARGUMENT, "fnv_relay_device: NULL host row");
    }
  return relay(board, epoch, rank, world, d_rows, k_dev, ready, h_rows, len, n_chunks, k, h0, threads, batch,
               static_cast<cudaStream_t>(stream), timeout_s, sums);
}

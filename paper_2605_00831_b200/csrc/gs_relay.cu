// gs_relay.cu -- host side of the striped seal at N>1 (peer.py chain_striped /
// RelayBoard): a ParityChunk checksum (parity_store.hpp:19-53) is one FNV-1a
// chain over a chunk's whole parity rows, and with byte-range striping each
// rank holds one range of every row, so the chain is continued range by range
// through the ranks. Host code only (the bit-sliced chain of gs_fnv_simd.cpp).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
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
  RelaySlot* slots = static_cast<RelaySlot*>(board);
  const int npos = k * world, segs = n_chunks * k;
  auto slot = [&](int c, int p) -> RelaySlot& { return slots[static_cast<size_t>(c) * npos + p]; };
  const auto deadline = std::chrono::steady_clock::now() +
                        std::chrono::microseconds(static_cast<int64_t>((timeout_s > 0 ? timeout_s : 60.0) * 1e6));
  std::atomic<int> next{0}, failed{0};
  // A segment takes milliseconds, so a waiting thread backs off to short
  // sleeps after a brief spin: the ranks' relays share the node's cores, and a
  // spinning waiter would take cycles from the threads it is waiting for.
  auto await = [&](RelaySlot& s) -> bool {
    for (uint32_t spin = 0;; ++spin) {
      if (__atomic_load_n(&s.tag, __ATOMIC_ACQUIRE) == epoch) return true;
      if (failed.load(std::memory_order_relaxed)) return false;
      if (spin < 512) {
        __builtin_ia32_pause();
        continue;
      }
      if ((spin & 63) == 0 && std::chrono::steady_clock::now() > deadline) {
        failed.store(1);
        return false;
      }
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  };
  auto work = [&] {
    for (int q = next.fetch_add(1); q < segs; q = next.fetch_add(1)) {
      const int i = q / n_chunks, c = q % n_chunks, p = i * world + rank;
      uint64_t h = h0;
      if (p > 0) {
        RelaySlot& prev = slot(c, p - 1);
        if (!await(prev)) return;
        h = prev.h;
      }
      const uint8_t* b = static_cast<const uint8_t*>(len ? rows[static_cast<size_t>(c) * k + i] : nullptr);
      fnv1a64_chains(&b, 1, len, &h);
      RelaySlot& mine = slot(c, p);
      mine.h = h;
      __atomic_store_n(&mine.tag, epoch, __ATOMIC_RELEASE);
    }
  };
  threads = std::max(1, std::min(threads, std::max(segs, 1)));
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  for (int c = 0; c < n_chunks && !failed.load(); ++c) {
    RelaySlot& last = slot(c, npos - 1);
    if (!await(last)) break;
    sums[c] = last.h;
  }
  if (failed.load()) return fail(GS_RUNTIME_ERROR, "fnv_relay: timed out waiting for a peer rank's chain state");
  return GS_OK;
}


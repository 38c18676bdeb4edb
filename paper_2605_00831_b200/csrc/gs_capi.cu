// gs_capi.cu -- host side of libghostserve_b200.so: the C ABI of
// include/gs_capi.h. Coefficient planning (Cauchy matrix, decode-matrix
// inversion) happens here on the host; every byte of parity / rebuilt KV is
// produced by the kernels of gs_kernels.cuh / gs_special.cuh.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/gs_capi.h"
#include "gs_field.hpp"
#include "gs_fnv.hpp"
#include "gs_host.hpp"
#include "gs_jit.hpp"
#include "gs_kernels.cuh"
#include "gs_kv.cuh"
#include "gs_rdp.cuh"
#include "gs_rdp_pairs.cuh"
#include "gs_special.cuh"

namespace gsb {
int special_encoders(SpecialEntry* out);
int special_decoders_kxor_2_1(SpecialEntry* out);
int special_decoders_kxor_4_1(SpecialEntry* out);
int special_decoders_kxor_8_1(SpecialEntry* out);
int special_decoders_kreedsolomon_4_1(SpecialEntry* out);
int special_decoders_kreedsolomon_4_2(SpecialEntry* out);
int special_decoders_kreedsolomon_6_2_e1(SpecialEntry* out);
int special_decoders_kreedsolomon_6_2_e2(SpecialEntry* out);
int special_decoders_kreedsolomon_8_2_e1(SpecialEntry* out);
int special_decoders_kreedsolomon_8_2_e2(SpecialEntry* out);
int batch_copies(void* const* dst, const void* const* src, int n, size_t bytes, int kind_d2h, cudaStream_t st);
}  // namespace gsb

using namespace gsb;

namespace gsb {
void set_last_error(const char* msg);
}

// ============================================================================
// errors
// ============================================================================
namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
std::atomic<uint64_t> g_zero_copy_calls{0};  // offloads that took the zero-copy epilogue
// Zero-copy epilogue of the offload: parity bytes per call at or below this
// go straight from the kernel into pinned host memory (GS_ZC_BYTES /
// gs_set_zero_copy_bytes, 0 = off).
std::atomic<uint64_t> g_zero_copy_max{[] {
  const char* e = std::getenv("GS_ZC_BYTES");
  return e ? std::strtoull(e, nullptr, 0) : (2ull << 20);
}()};

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return status;
}

#define GS_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(GS_CUDA_ERROR, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                  \
  } while (0)

int validate_scheme(int kind, int n, int k) {
  // coding.hpp:44-60, same order of checks and the same outcome classes.
  if (n < 1) return fail(GS_INVALID_ARGUMENT, "coding: data shard count must be positive");
  if (k < 1) return fail(GS_INVALID_ARGUMENT, "coding: parity shard count must be positive");
  if (n + k > 255)
    return fail(GS_INVALID_ARGUMENT, "coding: n + k exceeds the GF(2^8) bound of 255");
  switch (kind) {
    case GS_XOR:
      if (k != 1) return fail(GS_INVALID_ARGUMENT, "coding: xor requires exactly one parity shard");
      return GS_OK;
    case GS_RDP:
      if (k != 2) return fail(GS_INVALID_ARGUMENT, "coding: rdp requires exactly two parity shards");
      return GS_OK;
    case GS_RS:
      if (k > n) return fail(GS_INVALID_ARGUMENT, "coding: reed-solomon requires k <= n");
      return GS_OK;
    default:
      return fail(GS_INVALID_ARGUMENT, "coding: unknown code kind %d", kind);
  }
}

int tolerance(int kind, int k) { return kind == GS_XOR ? 1 : kind == GS_RDP ? 2 : k; }

// Per-device properties cached once.
struct DeviceInfo {
  int sms = 0;
};
std::mutex g_dev_mu;
std::map<int, DeviceInfo> g_dev;
std::map<std::tuple<int, const void*, size_t>, int> g_occ;  // (device, kernel, smem) -> blocks per SM

int device_sms(int dev) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto it = g_dev.find(dev);
  if (it != g_dev.end()) return it->second.sms;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  g_dev[dev].sms = sms > 0 ? sms : 148;
  return g_dev[dev].sms;
}

int blocks_per_sm(int dev, const void* kernel, size_t smem, int threads = kThreads) {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto key = std::make_tuple(dev, kernel, smem);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) return it->second;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem) != cudaSuccess || b < 1)
    b = 1;
  g_occ[key] = b;
  return b;
}

// Which specialised kernel variant serves aligned bodies: 0 = register
// (LDG.128) streaming, 1 = bulk-copy smem pipeline, 2 = auto (measured on
// B200, tools/kernel_sweep.py: the bulk pipeline wins for encoders once a
// launch moves >= 128 MB; the register kernel everywhere else).
std::atomic<int> g_variant{[] {
  const char* e = std::getenv("GS_KERNEL_VARIANT");  // 0 / 1 / 2 as gs_set_kernel_variant (A/B runs)
  const int v = e ? std::atoi(e) : 2;
  return v >= 0 && v <= 2 ? v : 2;
}()};
// Tuning override for the register kernel's resident CTAs per SM (0 = max).
int g_ctas_per_sm = [] {
  const char* e = std::getenv("GS_CTAS_PER_SM");
  return e ? std::atoi(e) : 0;
}();
// Tuning override: grid = every tile (non-persistent) when set.
int g_full_grid = [] {
  const char* e = std::getenv("GS_FULL_GRID");
  return e ? std::atoi(e) : 0;
}();
// Auto variant: the bulk TMA ring for encodes whose shards are long enough
// (per-shard length, not launch bytes): from ~64 MiB shards the register
// kernel can lose half its rate (allocation-dependent, tools/k1_layout_probe.py)
// while the bulk ring holds 6 TB/s; up to 32 MiB the register kernel is as
// fast in isolation and faster next to the pipeline's D2H (C3 pieces of
// 32 MiB: 46 vs 48 us per launch in the timed steps).
constexpr uint64_t kBulkAutoShardBytes = 48ull << 20;
// Paged K1/K2 walk tiles page-major (GS_PAGE_MAJOR=0: stripe-major, for A/B).
const bool g_page_major = [] {
  const char* e = std::getenv("GS_PAGE_MAJOR");
  return !(e && std::atoi(e) == 0);
}();
// Paged K1 page-per-tile addressing (GS_TILE_PAGES=0: the general paged walk, for A/B).
const bool g_tile_pages = [] {
  const char* e = std::getenv("GS_TILE_PAGES");
  return !(e && std::atoi(e) == 0);
}();
// RDP whole-dstripe body on the pipelined kernels (GS_RDP_FAST=0: tile kernels only, for A/B).
const bool g_rdp_fast = [] {
  const char* e = std::getenv("GS_RDP_FAST");
  return !(e && std::atoi(e) == 0);
}();

int bulk_stages(const SpecialEntry* e) {
  const size_t per = static_cast<size_t>(e->used_cols) * e->tile_bulk;
  return per ? static_cast<int>(std::min<size_t>(bulk::kMaxStages, (kBulkSmemMax - kBulkSmemHeader) / per)) : 0;
}

// Registry of compile-time kernels, built once.
struct Registry {
  std::vector<SpecialEntry> entries;
  Registry() {
    std::vector<SpecialEntry> buf(4096);
    int c = 0;
    c += special_encoders(buf.data() + c);
    c += special_decoders_kxor_2_1(buf.data() + c);
    c += special_decoders_kxor_4_1(buf.data() + c);
    c += special_decoders_kxor_8_1(buf.data() + c);
    c += special_decoders_kreedsolomon_4_1(buf.data() + c);
    c += special_decoders_kreedsolomon_4_2(buf.data() + c);
    c += special_decoders_kreedsolomon_6_2_e1(buf.data() + c);
    c += special_decoders_kreedsolomon_6_2_e2(buf.data() + c);
    c += special_decoders_kreedsolomon_8_2_e1(buf.data() + c);
    c += special_decoders_kreedsolomon_8_2_e2(buf.data() + c);
    entries.assign(buf.begin(), buf.begin() + c);
  }
  const SpecialEntry* find(bool decoder, int kind, int n, int k, uint64_t mask) const {
    for (const auto& e : entries)
      if (e.decoder == decoder && e.kind == kind && e.n == n && e.k == k && e.mask == mask) return &e;
    return nullptr;
  }
};

const Registry& registry() {
  static const Registry r;
  return r;
}

}  // namespace

void gsb::set_last_error(const char* msg) { g_err = msg; }

// ============================================================================
// codec
// ============================================================================
struct gs_codec {
  bool decoder = false;
  int kind = 0, n = 0, k = 0;
  int n_out = 0;                 // outputs produced
  int n_slots = 0;               // shard slots read (n or n+k)
  std::vector<int> out_index;    // shard index per output
  std::vector<uint8_t> coef;     // n_out x n_slots
  std::vector<int> used;         // slots with a nonzero coefficient (generic path)
  const SpecialEntry* special = nullptr;
  std::vector<CoefWords> words;  // n_out x used.size(), generic path table
  // RDP (position-dependent): p of the array, the two lost array columns of
  // a chain recovery, or an XOR decoder for single-column recoveries.
  int rdp_p = 0;
  int rdp_li = -1, rdp_lj = -1;
  gs_codec* xor_helper = nullptr;
  mutable std::mutex mu;
  mutable std::map<int, CoefWords*> dev_words;  // device -> uploaded table
  // runtime-specialised kernel (gs_jit.hpp), requested on the first GPU run
  // when no compiled specialisation exists
  mutable JitKernel* jit = nullptr;
  mutable bool jit_tried = false;

  ~gs_codec() {
    delete xor_helper;
    for (auto& kv : dev_words) {
      int prev = 0;
      cudaGetDevice(&prev);
      cudaSetDevice(kv.first);
      cudaFree(kv.second);
      cudaSetDevice(prev);
    }
  }
};

namespace {

void finish_codec(gs_codec* c) {
  for (int j = 0; j < c->n_slots; ++j) {
    bool any = false;
    for (int i = 0; i < c->n_out; ++i) any |= c->coef[static_cast<size_t>(i) * c->n_slots + j] != 0;
    if (any) c->used.push_back(j);
  }
  c->words.resize(static_cast<size_t>(c->n_out) * c->used.size());
  for (int i = 0; i < c->n_out; ++i)
    for (size_t u = 0; u < c->used.size(); ++u)
      c->words[static_cast<size_t>(i) * c->used.size() + u] =
          make_coef_words(c->coef[static_cast<size_t>(i) * c->n_slots + c->used[u]]);
}

// coding.hpp:187-223 (Gauss-Jordan over GF(2^8)); false if singular.
bool invert(std::vector<uint8_t> m, int dim, std::vector<uint8_t>& out) {
  out.assign(static_cast<size_t>(dim) * dim, 0);
  for (int i = 0; i < dim; ++i) out[static_cast<size_t>(i) * dim + i] = 1;
  auto at = [dim](std::vector<uint8_t>& v, int r, int c) -> uint8_t& {
    return v[static_cast<size_t>(r) * dim + c];
  };
  for (int col = 0; col < dim; ++col) {
    int piv = -1;
    for (int r = col; r < dim && piv < 0; ++r)
      if (at(m, r, col)) piv = r;
    if (piv < 0) return false;
    if (piv != col)
      for (int c = 0; c < dim; ++c) {
        std::swap(at(m, piv, c), at(m, col, c));
        std::swap(at(out, piv, c), at(out, col, c));
      }
    const uint8_t pi = gf_inv(at(m, col, col));
    for (int c = 0; c < dim; ++c) {
      at(m, col, c) = gf_mul(at(m, col, c), pi);
      at(out, col, c) = gf_mul(at(out, col, c), pi);
    }
    for (int r = 0; r < dim; ++r) {
      if (r == col) continue;
      const uint8_t f = at(m, r, col);
      if (!f) continue;
      for (int c = 0; c < dim; ++c) {
        at(m, r, c) ^= gf_mul(f, at(m, col, c));
        at(out, r, c) ^= gf_mul(f, at(out, col, c));
      }
    }
  }
  return true;
}

int current_device(int* dev) {
  GS_CUDA(cudaGetDevice(dev));
  return GS_OK;
}

int upload_words(const gs_codec* c, int dev, const CoefWords** out) {
  std::lock_guard<std::mutex> lk(c->mu);
  auto it = c->dev_words.find(dev);
  if (it != c->dev_words.end()) {
    *out = it->second;
    return GS_OK;
  }
  CoefWords* d = nullptr;
  const size_t bytes = std::max<size_t>(c->words.size(), 1) * sizeof(CoefWords);
  GS_CUDA(cudaMalloc(&d, bytes));
  GS_CUDA(cudaMemcpy(d, c->words.data(), c->words.size() * sizeof(CoefWords), cudaMemcpyHostToDevice));
  c->dev_words[dev] = d;
  *out = d;
  return GS_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <int KB>
cudaError_t launch_generic_kb(const void* const* ptrs, int count, const TileGeom& g, int grid,
                              cudaStream_t st, const CoefWords* coef, int ns) {
  PtrTable<kPtrCap> tab;
  for (int i = 0; i < count; ++i) tab.p[i] = static_cast<const uint8_t*>(ptrs[i]);
  const size_t smem = static_cast<size_t>(KB) * ns * sizeof(CoefWords);
  k_apply_generic<KB, kPtrCap><<<grid, kThreads, smem, st>>>(tab, g, coef, ns);
  return cudaGetLastError();
}

const void* generic_kernel(int kb) {
  switch (kb) {
    case 1: return reinterpret_cast<const void*>(&k_apply_generic<1, kPtrCap>);
    case 2: return reinterpret_cast<const void*>(&k_apply_generic<2, kPtrCap>);
    case 3: return reinterpret_cast<const void*>(&k_apply_generic<3, kPtrCap>);
    default: return reinterpret_cast<const void*>(&k_apply_generic<4, kPtrCap>);
  }
}

JitKernel* codec_jit(const gs_codec* c) {
  std::lock_guard<std::mutex> lk(c->mu);
  if (!c->jit_tried) {
    c->jit_tried = true;
    c->jit = jit_request(c->n_out, c->n_slots, c->coef.data());
  }
  return c->jit;
}

// Launch the codec over stripes. slot_ptr(s, j) / out_ptr(s, i) give the
// (already offset) pointers; every stripe has `len` bytes.
// Paging (optional): slots whose bit is set in pg.paged_slots are paged-cache
// bases mapped with pg.src (NOT pre-offset: the kernel maps logical0 + off);
// outputs are mapped with pg.dst when pg.dst.page_bytes != 0.
struct Paging {
  uint32_t paged_slots = 0;
  uint64_t logical0 = 0;
  uint64_t total_len = 0;  // RDP: absolute column length (0 = this launch's len)
  uint64_t stripe0 = 0;    // absolute index of stripe 0 of this call (block-table rows)
  PageMap src{};
  PageMap dst{};
  unsigned long long* tstamp = nullptr;  // kernel-internal timing slot (gs_pipeline_set_timing)
  int max_grid = 0;                       // cap on the launch's CTAs (gs_pipeline_set_max_ctas; 0 = none)
  bool any() const { return paged_slots != 0 || dst.page_bytes != 0; }
};

PageMap to_map(const gs_page_map* m) {
  PageMap r{};
  if (m) {
    r.page_bytes = m->page_bytes;
    r.layers = m->layers;
    r.token_bytes = m->token_bytes;
    r.valid_tokens = m->valid_tokens;
    r.layer_stride = m->layer_stride;
    r.kv_stride = m->kv_stride;
    r.table = m->block_table;
    r.block_bytes = m->block_table ? m->block_bytes : m->page_bytes;
    r.table_stride = m->table_stride;
    r.page_m = fastdiv_magic(r.page_bytes);
    r.layers_m = fastdiv_magic(r.layers);
    r.block_m = fastdiv_magic(r.block_bytes);
  }
  return r;
}

int check_page_map(const PageMap& m, const char* what) {
  if (m.page_bytes == 0) return GS_OK;
  if (m.page_bytes % kVec || m.token_bytes == 0 || m.token_bytes % kVec || m.layers == 0 ||
      m.layer_stride % kVec || m.kv_stride % kVec || m.page_bytes % m.token_bytes)
    return fail(GS_INVALID_ARGUMENT, "%s page map: page/token bytes and strides must be multiples of 16", what);
  if (static_cast<uint64_t>(m.valid_tokens) * m.token_bytes > m.page_bytes)
    return fail(GS_INVALID_ARGUMENT, "kv: valid_tokens exceeds chunk size");
  if (m.table && (m.block_bytes == 0 || m.block_bytes % kVec || m.page_bytes % m.block_bytes ||
                  m.block_bytes % m.token_bytes || m.table_stride < m.page_bytes / m.block_bytes))
    return fail(GS_INVALID_ARGUMENT, "%s page map: block_bytes must divide the segment and the table must cover it", what);
  return GS_OK;
}

template <class SlotFn, class OutFn>
int run_rdp(const gs_codec* c, int n_stripes, SlotFn slot_ptr, OutFn out_ptr, uint64_t len, cudaStream_t st,
            const Paging& pg);

template <class SlotFn, class OutFn>
int run_codec(const gs_codec* c, int n_stripes, SlotFn slot_ptr, OutFn out_ptr, uint64_t len,
              cudaStream_t st, const Paging& pg = Paging{}) {
  if (len == 0 || n_stripes == 0 || c->n_out == 0) return GS_OK;
  if (c->kind == GS_RDP) return run_rdp(c, n_stripes, slot_ptr, out_ptr, len, st, pg);
  int dev = 0;
  if (int s = current_device(&dev)) return s;
  const int sms = device_sms(dev);
  if (pg.any()) {
    if (c->n_slots > 32) return fail(GS_INVALID_ARGUMENT, "paged apply: at most 32 shard slots");
    if (len % kVec) return fail(GS_INVALID_ARGUMENT, "paged apply: slice length must be a multiple of 16");
    if (pg.paged_slots && pg.src.page_bytes == 0)
      return fail(GS_INVALID_ARGUMENT, "paged apply: paged slots need a source page map");
    if (int s = check_page_map(pg.src, "source")) return s;
    if (int s = check_page_map(pg.dst, "output")) return s;
  }

  bool aligned = true;
  for (int s = 0; s < n_stripes; ++s) {
    for (int j : c->used) {
      const void* p = slot_ptr(s, j);
      if (p == nullptr)
        return fail(GS_INVALID_ARGUMENT, "apply: shard slot %d of stripe %d is NULL but required", j, s);
      aligned &= aligned16(p);
    }
    for (int i = 0; i < c->n_out; ++i) {
      const void* p = out_ptr(s, i);
      if (p == nullptr) return fail(GS_INVALID_ARGUMENT, "apply: output %d of stripe %d is NULL", i, s);
      aligned &= aligned16(p);
    }
  }
  // The generic table is uploaded up front (the specialised path still needs
  // it for ragged tails), so later calls never synchronise -- graph-safe.
  const CoefWords* dw = nullptr;
  if (int s = upload_words(c, dev, &dw)) return s;
  std::vector<const void*> ptrs;

  // Specialised kernel over the 16-byte-aligned body: compiled registry, or
  // a runtime-specialised (JIT) build of this codec's matrix once it is ready.
  uint64_t done = 0;
  if (pg.any() && !aligned) return fail(GS_INVALID_ARGUMENT, "paged apply: pointers must be 16-B aligned");
  JitKernel* jit = nullptr;
  if (!c->special && aligned && len >= kVec && !pg.any()) {
    jit = codec_jit(c);
    if (jit && jit_status(jit, false) != 1) jit = nullptr;
    if (jit && jit_occupancy(jit) < 1) jit = nullptr;
  }
  if ((c->special || jit) && aligned && len >= kVec) {
    const uint64_t body = len / kVec * kVec;
    const int stages = c->special ? bulk_stages(c->special) : 0;
    const int variant = g_variant.load(std::memory_order_relaxed);
    const bool use_bulk = c->special && !pg.any() && stages >= 2 &&
                          (variant == 1 || (variant == 2 && !c->decoder && body >= kBulkAutoShardBytes));
    const uint64_t tile = static_cast<uint64_t>(use_bulk ? c->special->tile_bulk : c->special ? c->special->tile : kTile);
    const uint64_t tps64 = (body + tile - 1) / tile;
    const int stride = c->n_slots + c->n_out;
    const int per = kPtrCap / stride;
    const size_t smem = use_bulk ? kBulkSmemHeader + static_cast<size_t>(stages) * c->special->used_cols *
                                                         c->special->tile_bulk
                                 : 0;
    const bool paged = pg.any();
    int occ = jit        ? jit_occupancy(jit)
              : use_bulk ? blocks_per_sm(dev, c->special->kernel_bulk, smem, kBulkThreads)
                         : blocks_per_sm(dev, paged ? c->special->kernel_paged : c->special->kernel, 0);
    if (!use_bulk && g_ctas_per_sm > 0) occ = std::min(occ, g_ctas_per_sm);
    for (int s0 = 0; s0 < n_stripes; s0 += per) {
      const int cnt = std::min(per, n_stripes - s0);
      ptrs.assign(static_cast<size_t>(cnt) * stride, nullptr);
      for (int s = 0; s < cnt; ++s) {
        for (int j = 0; j < c->n_slots; ++j) ptrs[s * stride + j] = slot_ptr(s0 + s, j);
        for (int i = 0; i < c->n_out; ++i) ptrs[s * stride + c->n_slots + i] = out_ptr(s0 + s, i);
      }
      const uint64_t total = tps64 * cnt;
      if (total > 0xFFFFFFFFull) return fail(GS_INVALID_ARGUMENT, "apply: too many tiles in one launch");
      TileGeom g{body, static_cast<uint32_t>(tps64), static_cast<uint32_t>(total), stride, c->n_slots, 1,
                 pg.paged_slots, pg.logical0, pg.src, pg.dst};
      g.tps_m = fastdiv_magic(g.tps);
      g.tstamp = pg.tstamp;
      if (paged && !jit && !use_bulk && g_page_major) {  // page-major walk (gs_kernels.cuh TileGeom)
        g.nstripes = static_cast<uint32_t>(cnt);
        g.nstripes_m = fastdiv_magic(g.nstripes);
        uint32_t used = 0;
        for (int j : c->used) used |= 1u << j;
        g.tile_pages = g_tile_pages && (pg.paged_slots & used) == used && pg.dst.page_bytes == 0 &&
                       pg.src.page_bytes % kTile == 0 && pg.logical0 % kTile == 0 &&
                       (!pg.src.table || pg.src.block_bytes % kTile == 0) &&
                       static_cast<uint64_t>(pg.src.valid_tokens) * pg.src.token_bytes == pg.src.page_bytes &&
                       pg.logical0 + body <= 0xFFFFFFFFull;
      }
      if (g.src.table) g.src.table += (pg.stripe0 + s0) * g.src.table_stride;
      if (g.dst.table) g.dst.table += (pg.stripe0 + s0) * g.dst.table_stride;
      // Decoders (K2) run one CTA per tile up to 8 waves (C2 rebuild: 14.4 ->
      // 13.5 us; the extra sources per tile hide less latency in a
      // grid-stride loop); encoders stay persistent (C2 K1: 15.3 vs 20.4 us).
      const uint64_t persistent = static_cast<uint64_t>(occ) * sms;
      const bool full = !use_bulk && (g_full_grid || (c->decoder && total <= 8 * persistent));
      int grid = static_cast<int>(std::min<uint64_t>(total, full ? total : persistent));
      if (pg.max_grid > 0 && !jit) grid = std::min(grid, pg.max_grid);  // grid-stride: any grid covers every tile
      cudaError_t e = jit        ? jit_launch(jit, ptrs.data(), cnt * stride, g, sms, st)
                      : use_bulk ? c->special->launch_bulk(ptrs.data(), cnt * stride, g, grid, st, stages, smem)
                      : paged    ? c->special->launch_paged(ptrs.data(), cnt * stride, g, grid, st)
                                 : c->special->launch(ptrs.data(), cnt * stride, g, grid, st);
      if (e != cudaSuccess) return fail(GS_CUDA_ERROR, "special kernel launch: %s", cudaGetErrorString(e));
      g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    done = body;
    if (done == len) return GS_OK;
  }

  // Generic kernel: everything, or the ragged tail [done, len).
  const uint64_t glen = len - done;
  const uint64_t tps64 = (glen + kTile - 1) / kTile;
  const bool galigned = aligned && (done % kVec == 0);
  const int ns = static_cast<int>(c->used.size());
  const int stride = ns + c->n_out;
  const int per = kPtrCap / stride;
  if (per < 1) return fail(GS_INVALID_ARGUMENT, "apply: stripe needs %d pointers (> %d)", stride, kPtrCap);
  uint32_t gpaged = 0;  // paged bits in compacted (used-slot) order
  for (int u = 0; u < ns; ++u)
    if ((pg.paged_slots >> c->used[u]) & 1u) gpaged |= 1u << u;
  for (int s0 = 0; s0 < n_stripes; s0 += per) {
    const int cnt = std::min(per, n_stripes - s0);
    ptrs.assign(static_cast<size_t>(cnt) * stride, nullptr);
    for (int s = 0; s < cnt; ++s) {
      for (int u = 0; u < ns; ++u)
        ptrs[s * stride + u] = static_cast<const uint8_t*>(slot_ptr(s0 + s, c->used[u])) +
                               (((gpaged >> u) & 1u) ? 0 : done);
      for (int i = 0; i < c->n_out; ++i)
        ptrs[s * stride + ns + i] = static_cast<const uint8_t*>(out_ptr(s0 + s, i)) +
                                    (pg.dst.page_bytes ? 0 : done);
    }
    const uint64_t total = tps64 * cnt;
    if (total > 0xFFFFFFFFull) return fail(GS_INVALID_ARGUMENT, "apply: too many tiles in one launch");
    for (int r0 = 0; r0 < c->n_out; r0 += kMaxGenericRows) {
      const int kb = std::min(kMaxGenericRows, c->n_out - r0);
      TileGeom g{glen, static_cast<uint32_t>(tps64), static_cast<uint32_t>(total), stride, ns + r0,
                 galigned ? 1 : 0, gpaged, pg.logical0 + done, pg.src, pg.dst};
      g.tps_m = fastdiv_magic(g.tps);
      g.tstamp = pg.tstamp;
      if (g.src.table) g.src.table += (pg.stripe0 + s0) * g.src.table_stride;
      if (g.dst.table) g.dst.table += (pg.stripe0 + s0) * g.dst.table_stride;
      const size_t smem = static_cast<size_t>(kb) * ns * sizeof(CoefWords);
      const int occ = blocks_per_sm(dev, generic_kernel(kb), smem);
      int grid = static_cast<int>(std::min<uint64_t>(total, static_cast<uint64_t>(occ) * sms));
      if (pg.max_grid > 0) grid = std::min(grid, pg.max_grid);
      const CoefWords* cw = dw + static_cast<size_t>(r0) * ns;
      cudaError_t e;
      switch (kb) {
        case 1: e = launch_generic_kb<1>(ptrs.data(), cnt * stride, g, grid, st, cw, ns); break;
        case 2: e = launch_generic_kb<2>(ptrs.data(), cnt * stride, g, grid, st, cw, ns); break;
        case 3: e = launch_generic_kb<3>(ptrs.data(), cnt * stride, g, grid, st, cw, ns); break;
        default: e = launch_generic_kb<4>(ptrs.data(), cnt * stride, g, grid, st, cw, ns); break;
      }
      if (e != cudaSuccess) return fail(GS_CUDA_ERROR, "generic kernel launch: %s", cudaGetErrorString(e));
      g_launches.fetch_add(1, std::memory_order_relaxed);
    }
  }
  return GS_OK;
}

// RDP (position-dependent, coding.hpp:225-534): tile kernels of gs_rdp.cuh
// for encode and two-column recovery; single-column recovery through the
// XOR helper codec. `pg.logical0` / `pg.total_len` place this launch's range
// inside the column (pipelines split on dstripe boundaries).
// Compiled lost-pair RDP recovery kernels (gs_rdp_pairs.cuh); nullptr when
// the prime has none or GS_RDP_PAIRS=0.
const RdpPair* rdp_pair(int p, int li, int lj) {
  static const bool on = [] {
    const char* e = std::getenv("GS_RDP_PAIRS");
    return !(e && std::atoi(e) == 0);
  }();
  static const std::vector<RdpPair> table = [] {
    std::vector<RdpPair> t(kRdpPairP * kRdpPairP);
    rdp_pairs_p11_i0(t.data());
    rdp_pairs_p11_i1(t.data());
    rdp_pairs_p11_i2(t.data());
    rdp_pairs_p11_i3(t.data());
    rdp_pairs_p11_i4(t.data());
    rdp_pairs_p11_i5(t.data());
    rdp_pairs_p11_i6(t.data());
    rdp_pairs_p11_i7(t.data());
    rdp_pairs_p11_i8(t.data());
    rdp_pairs_p11_i9(t.data());
    return t;
  }();
  if (!on || p != kRdpPairP || li < 0 || lj <= li || lj >= p) return nullptr;
  const RdpPair& r = table[static_cast<size_t>(li) * p + lj];
  return r.kernel ? &r : nullptr;
}

template <class SlotFn, class OutFn>
int run_rdp(const gs_codec* c, int n_stripes, SlotFn slot_ptr, OutFn out_ptr, uint64_t len, cudaStream_t st,
            const Paging& pg) {
  if (pg.paged_slots || pg.dst.page_bytes) return fail(GS_UNSUPPORTED, "rdp: paged KV caches are not supported");
  if (c->xor_helper) return run_codec(c->xor_helper, n_stripes, slot_ptr, out_ptr, len, st);
  const int n = c->n, p = c->rdp_p, rows = p - 1;
  const uint64_t total = pg.total_len ? pg.total_len : len;
  if (pg.logical0 % static_cast<uint64_t>(rows))
    return fail(GS_INVALID_ARGUMENT, "rdp: range must start on a dstripe boundary");
  int dev = 0;
  if (int s = current_device(&dev)) return s;
  const int sms = device_sms(dev);
  bool aligned = true;
  const bool encode = !c->decoder;
  for (int s = 0; s < n_stripes; ++s) {
    for (int j = 0; j < c->n_slots; ++j) {
      const void* q = slot_ptr(s, j);
      const bool needed = encode || std::find(c->used.begin(), c->used.end(), j) != c->used.end();
      if (needed && !q) return fail(GS_INVALID_ARGUMENT, "apply: shard slot %d of stripe %d is NULL but required", j, s);
      if (q) aligned &= aligned16(q);
    }
    for (int i = 0; i < c->n_out; ++i) {
      const void* q = out_ptr(s, i);
      if (!q) return fail(GS_INVALID_ARGUMENT, "apply: output %d of stripe %d is NULL", i, s);
      aligned &= aligned16(q);
    }
  }
  const int in_slots = encode ? n : n + 2;
  const int stride = in_slots + c->n_out;
  const int per = kPtrCap / stride;
  if (per < 1) return fail(GS_INVALID_ARGUMENT, "rdp: stripe needs %d pointers (> %d)", stride, kPtrCap);
  // Pipelined kernels take the whole range when the columns are 16-B aligned
  // and it holds at least one whole dstripe: every whole dstripe (the last
  // tile may be partial) plus the P/Q tail past the last one. Otherwise the
  // shared-memory tile kernels run the lot.
  const uint64_t full_abs = total / rows * rows;
  const uint32_t TB = rdpb::tile_bytes(p);
  // two-column recovery with a compiled pair kernel: chains in registers, no chain scratch
  const RdpPair* pair = !encode && c->rdp_li >= 0 ? rdp_pair(p, c->rdp_li, c->rdp_lj) : nullptr;
  const size_t fixed = rdpb::kHeader + rdpb::out_bytes(p) + (encode || pair ? 0 : rdpb::chain_bytes(p));
  const int fast_stages = fixed < rdpb::kSmemBudget
                              ? static_cast<int>(std::min<size_t>(rdpb::kMaxStages, (rdpb::kSmemBudget - fixed) / TB))
                              : 0;
  uint64_t body = 0;  // whole-dstripe bytes handled by the pipelined kernel
  if (aligned && fast_stages >= 2 && g_rdp_fast && full_abs > pg.logical0)
    body = std::min<uint64_t>(len, full_abs - pg.logical0);
  const void* kfast = nullptr;
#define GS_RDP_PICK_FAST(P_)                                                                  \
  if (p == P_)                                                                                \
    kfast = encode ? reinterpret_cast<const void*>(&k_rdp_encode_bulk<kPtrCap, P_>)           \
                   : reinterpret_cast<const void*>(&k_rdp_recover_bulk<kPtrCap, P_>);
  GS_RDP_PRIMES(GS_RDP_PICK_FAST)
#undef GS_RDP_PICK_FAST
  if (pair) kfast = pair->kernel;
  const size_t fast_smem = fixed + static_cast<size_t>(fast_stages) * TB;
  if (body && kfast) {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (cudaFuncSetAttribute(kfast, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(fast_smem)) !=
        cudaSuccess) {
      cudaGetLastError();
      body = 0;
    }
  } else {
    body = 0;
  }
  const uint32_t fast_tail = body ? static_cast<uint32_t>(len - body) : 0;  // < rows bytes
  if (body) body = len;  // the pipelined kernel covers the tail too
  // tail coefficients of the two-column recovery (coding.hpp:415-448)
  uint8_t tail_gj = 0, tail_inv = 0;
  if (!encode && c->rdp_li >= 0) {
    const uint8_t gi = exp2_of(c->rdp_li);
    if (c->rdp_lj == p - 1) {
      tail_inv = gf_inv(gi);
    } else {
      tail_gj = exp2_of(c->rdp_lj);
      tail_inv = gf_inv(static_cast<uint8_t>(gi ^ tail_gj));
    }
  }
  const uint64_t rest = len - body;
  const uint32_t T = static_cast<uint32_t>(rows) * kRdpThreads;
  const uint64_t tps64 = (rest + T - 1) / T;
  const size_t smem = static_cast<size_t>(encode ? rows + 2 : p + 1) * T;
  const void* kern = nullptr;
#define GS_RDP_PICK(P_)                                                                        \
  if (p == P_)                                                                                 \
    kern = encode ? reinterpret_cast<const void*>(&k_rdp_encode<kPtrCap, P_>)                  \
                  : reinterpret_cast<const void*>(&k_rdp_recover<kPtrCap, P_>);
  GS_RDP_PRIMES(GS_RDP_PICK)
#undef GS_RDP_PICK
  if (!kern) return fail(GS_UNSUPPORTED, "rdp: no kernel for p = %d", p);
  const int occ = rest ? blocks_per_sm(dev, kern, smem, kRdpThreads) : 1;
  std::vector<const void*> ptrs;
  for (int s0 = 0; s0 < n_stripes; s0 += per) {
    const int cnt = std::min(per, n_stripes - s0);
    ptrs.assign(static_cast<size_t>(cnt) * stride, nullptr);
    for (int s = 0; s < cnt; ++s) {
      for (int j = 0; j < in_slots; ++j) ptrs[s * stride + j] = slot_ptr(s0 + s, j);
      for (int i = 0; i < c->n_out; ++i) ptrs[s * stride + in_slots + i] = out_ptr(s0 + s, i);
    }
    PtrTable<kPtrCap> tab;
    if (body) {
      const uint64_t whole = len - fast_tail;
      const uint64_t ftps = (whole + TB - 1) / TB, fntiles = ftps * cnt;
      for (int i = 0; i < cnt * stride; ++i) tab.p[i] = static_cast<const uint8_t*>(ptrs[i]);
      RdpGeom g{n, p, rows, whole, pg.logical0, full_abs, total, static_cast<uint32_t>(ftps),
                static_cast<uint32_t>(fntiles), stride, 1, c->rdp_li, c->rdp_lj, tail_gj, tail_inv, fast_tail};
      const int grid = static_cast<int>(std::min<uint64_t>(fntiles, static_cast<uint64_t>(sms)));
      const int threads = (rdpb::kCW + 1) * 32;
#define GS_RDP_LAUNCH_FAST(P_)                                                                               \
  if (p == P_) {                                                                                             \
    if (encode)                                                                                              \
      k_rdp_encode_bulk<kPtrCap, P_><<<grid, threads, fast_smem, st>>>(tab, g, fast_stages);                 \
    else                                                                                                     \
      k_rdp_recover_bulk<kPtrCap, P_><<<grid, threads, fast_smem, st>>>(tab, g, fast_stages, c->n_out,       \
                                                                        in_slots);                           \
  }
      cudaError_t e = cudaSuccess;
      if (pair) {
        e = pair->launch(grid, threads, fast_smem, st, tab, g, fast_stages, c->n_out, in_slots);
      } else {
        GS_RDP_PRIMES(GS_RDP_LAUNCH_FAST)
        e = cudaGetLastError();
      }
#undef GS_RDP_LAUNCH_FAST
      if (e != cudaSuccess) return fail(GS_CUDA_ERROR, "rdp kernel launch: %s", cudaGetErrorString(e));
      g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    if (!rest) continue;
    const uint64_t ntiles = tps64 * cnt;
    RdpGeom g{n, p, rows, rest, pg.logical0 + body, full_abs, total, static_cast<uint32_t>(tps64),
              static_cast<uint32_t>(ntiles), stride, aligned ? 1 : 0, c->rdp_li, c->rdp_lj, tail_gj, tail_inv, 0};
    for (int i = 0; i < cnt * stride; ++i)
      tab.p[i] = ptrs[i] ? static_cast<const uint8_t*>(ptrs[i]) + body : nullptr;
    const int grid = static_cast<int>(std::min<uint64_t>(ntiles, static_cast<uint64_t>(occ) * sms));
#define GS_RDP_LAUNCH(P_)                                                                      \
  if (p == P_) {                                                                               \
    if (encode)                                                                                \
      k_rdp_encode<kPtrCap, P_><<<grid, kRdpThreads, smem, st>>>(tab, g);                      \
    else                                                                                       \
      k_rdp_recover<kPtrCap, P_><<<grid, kRdpThreads, smem, st>>>(tab, g, c->n_out, in_slots); \
  }
    GS_RDP_PRIMES(GS_RDP_LAUNCH)
#undef GS_RDP_LAUNCH
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(GS_CUDA_ERROR, "rdp kernel launch: %s", cudaGetErrorString(e));
    g_launches.fetch_add(1, std::memory_order_relaxed);
  }
  return GS_OK;
}

}  // namespace

// ============================================================================
// pipeline (staging ring for host-link overlap)
// ============================================================================
struct gs_pipeline {
  int device = 0;
  size_t bytes = 0;
  uint8_t* staging = nullptr;
  static constexpr int kSlots = 4;
  cudaEvent_t ready[kSlots]{}, done[kSlots]{}, drained[kSlots]{};
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaStream_t s_h2d = nullptr, s_comp = nullptr, s_d2h = nullptr;  // for the *_host calls
  int next = 0;
  size_t slot_bytes() const { return bytes / kSlots / 4096 * 4096; }

  // Optional live kernel timing (gs_pipeline_set_timing): a pair of timing
  // events on the compute stream brackets each codec launch group of the
  // pipelined calls -- recorded after the slot waits, so a pair measures the
  // kernels alone, inside the caller's real schedule. Not under capture.
  bool timing = false;
  int max_ctas = 0;              // gs_pipeline_set_max_ctas: background checkpoints (0 = whole GPU)
  std::vector<cudaEvent_t> tev;  // 2 per timed launch group
  size_t tused = 0;
  uint64_t tlaunch0 = 0;
  // and a {start, end} %globaltimer pair per group written by the kernels
  static constexpr size_t kStampSlots = 4096;
  unsigned long long* d_stamps = nullptr;
  cudaError_t reset_stamps() {
    if (!d_stamps) {
      if (cudaError_t e = cudaMalloc(&d_stamps, kStampSlots * 2 * sizeof(unsigned long long))) return e;
    }
    std::vector<unsigned long long> init(kStampSlots * 2);
    for (size_t i = 0; i < kStampSlots; ++i) {
      init[2 * i] = ~0ull;
      init[2 * i + 1] = 0;
    }
    return cudaMemcpy(d_stamps, init.data(), init.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice);
  }
  unsigned long long* stamp_slot() const {
    const size_t g = tused / 2;  // group index after timed_begin
    return (timing && d_stamps && g >= 1 && g <= kStampSlots) ? d_stamps + 2 * (g - 1) : nullptr;
  }
  cudaError_t timed_begin(cudaStream_t st, cudaEvent_t* e0, cudaEvent_t* e1) {
    *e0 = *e1 = nullptr;
    if (!timing || capturing) return cudaSuccess;
    if (tused + 2 > tev.size()) {
      for (int i = 0; i < 512; ++i) {
        cudaEvent_t e;
        if (cudaError_t err = cudaEventCreate(&e)) return err;
        tev.push_back(e);
      }
    }
    *e0 = tev[tused];
    *e1 = tev[tused + 1];
    tused += 2;
    return cudaEventRecord(*e0, st);
  }

  // CUDA-graph capture: while `compute` is being captured,
  // only events recorded inside the same capture may be waited on; slot
  // hazards across replays are ordered by the graph launches themselves.
  unsigned long long capture_id = 0;
  bool capturing = false;
  bool captured = false;            // a capture used the events since the last eager call
  bool in_capture[3][kSlots] = {};  // ready / done / drained recorded in this capture

  // Called with the compute and copy streams of a call; under capture the
  // copy stream is forked from the compute stream so it joins the graph.
  cudaError_t begin(cudaStream_t st, cudaStream_t copy) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    unsigned long long id = 0;
    cudaStreamGetCaptureInfo(st, &cs, &id);
    capturing = cs == cudaStreamCaptureStatusActive;
    if (capturing && id != capture_id) {
      capture_id = id;
      for (auto& row : in_capture)
        for (bool& b : row) b = false;
    }
    if (capturing) {
      captured = true;
    } else if (captured) {
      // Events last recorded inside a capture cannot be waited on eagerly:
      // re-arm them on this stream (ordered after any graph launched on it).
      captured = false;
      for (int i = 0; i < kSlots; ++i)
        for (cudaEvent_t e : {ready[i], done[i], drained[i]})
          if (cudaError_t err = cudaEventRecord(e, st)) return err;
    }
    if (capturing && copy != st) {
      if (cudaError_t e = cudaEventRecord(fork, st)) return e;
      return cudaStreamWaitEvent(copy, fork, 0);
    }
    return cudaSuccess;
  }
  // Under capture, join the copy stream back into the compute stream. The
  // offload does not call it: its completion is the copy stream, in a graph
  // as eagerly, so the next block's kernels overlap this block's D2H; the
  // capturer joins `copy` into its origin stream before ending the capture.
  cudaError_t end(cudaStream_t st, cudaStream_t copy) {
    if (!capturing || copy == st) return cudaSuccess;
    if (cudaError_t e = cudaEventRecord(join, copy)) return e;
    return cudaStreamWaitEvent(st, join, 0);
  }
  cudaError_t wait(cudaStream_t st, int kind, int slot) {
    cudaEvent_t* evs = kind == 0 ? ready : kind == 1 ? done : drained;
    if (capturing && !in_capture[kind][slot]) return cudaSuccess;
    return cudaStreamWaitEvent(st, evs[slot], 0);
  }
  cudaError_t record(cudaStream_t st, int kind, int slot) {
    cudaEvent_t* evs = kind == 0 ? ready : kind == 1 ? done : drained;
    if (capturing) in_capture[kind][slot] = true;
    return cudaEventRecord(evs[slot], st);
  }
};

namespace {

// Host-buffer pipelines: bytes per shard per piece (GS_HOST_PIECE overrides).
const uint64_t kHostPiece = [] {
  const char* e = std::getenv("GS_HOST_PIECE");
  const uint64_t v = e ? std::strtoull(e, nullptr, 0) : 0;
  return v >= 4096 ? v / 4096 * 4096 : (1ull << 20);
}();

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Piece geometry of the pipelines. Every piece start stays 16-B aligned (the
// vector kernels' requirement) and, for RDP, on a dstripe boundary (p-1
// bytes); pieces are 4 KiB multiples whenever that fits in the staging slot.
uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) {
    const uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

uint64_t piece_unit(const gs_codec* c, uint64_t base) {
  if (c->kind != GS_RDP || c->xor_helper) return base;
  const uint64_t rows = static_cast<uint64_t>(c->rdp_p - 1);
  return base / gcd_u64(base, rows) * rows;  // lcm(base, rows)
}

uint64_t align_down_piece(const gs_codec* c, uint64_t x) {
  const uint64_t big = piece_unit(c, 4096);
  if (x >= big) return x / big * big;
  const uint64_t u = piece_unit(c, 16);
  return x / u * u;
}

// Bytes per shard per piece: as large as the slot (and `cap`) allows.
// 0 = the slot cannot hold one aligned piece (the caller reports it).
uint64_t piece_len(const gs_codec* c, uint64_t len, size_t slot, int per_byte, uint64_t cap = ~0ull) {
  const uint64_t room = std::min<uint64_t>(slot / static_cast<uint64_t>(std::max(per_byte, 1)), cap);
  const uint64_t r = align_down_piece(c, room);
  return r ? std::min<uint64_t>(r, len) : 0;
}

// Tapered piece schedule of the host-buffer pipelines: full pieces, then the
// last full piece's worth split into quarters, so the drain after the final
// H2D (last kernel + last D2H) is a quarter piece instead of a whole one.
uint64_t taper(uint64_t r0, uint64_t len, uint64_t rl_max, uint64_t quarter) {
  const uint64_t left = len - r0;
  if (left > rl_max || quarter == 0) return std::min<uint64_t>(rl_max, left);
  return std::min<uint64_t>(quarter, left);
}

// Host-link copies of one piece. Adjacent (dst, src) runs are merged into
// one 1-D copy; what remains is grouped by `key` (e.g. parity row) into
// constant-pitch runs issued as single 2-D copies, so a batch of 32 request
// slices costs one DMA command per parity row instead of 32.
struct CopyOp {
  uint8_t* dst;
  const uint8_t* src;
  size_t bytes;
  int key;
};

int issue_copies(std::vector<CopyOp>& ops, cudaMemcpyKind kind, cudaStream_t st) {
  std::vector<CopyOp> merged;
  for (size_t i = 0; i < ops.size();) {
    CopyOp cur = ops[i];
    size_t j = i + 1;
    while (j < ops.size() && ops[j].dst == cur.dst + cur.bytes && ops[j].src == cur.src + cur.bytes) {
      cur.bytes += ops[j].bytes;
      ++j;
    }
    if (cur.bytes) merged.push_back(cur);
    i = j;
  }
  ops.clear();
  std::stable_sort(merged.begin(), merged.end(), [](const CopyOp& a, const CopyOp& b) { return a.key < b.key; });
  for (size_t i = 0; i < merged.size();) {
    const CopyOp& a = merged[i];
    size_t j = i + 1;
    if (j < merged.size() && merged[j].key == a.key && merged[j].bytes == a.bytes && merged[j].dst > a.dst &&
        merged[j].src > a.src) {
      const size_t dp = static_cast<size_t>(merged[j].dst - a.dst), sp = static_cast<size_t>(merged[j].src - a.src);
      constexpr size_t kMaxPitch = (size_t{1} << 31) - 1;
      if (dp >= a.bytes && sp >= a.bytes && dp <= kMaxPitch && sp <= kMaxPitch) {
        while (j < merged.size() && merged[j].key == a.key && merged[j].bytes == a.bytes &&
               merged[j].dst == merged[j - 1].dst + dp && merged[j].src == merged[j - 1].src + sp)
          ++j;
        // A constant-pitch run can still straddle two allocations (e.g. pinned
        // slabs that happen to be adjacent in VA space); the driver rejects
        // that up front, and the rows then go as 1-D copies.
        cudaError_t e2 = cudaMemcpy2DAsync(a.dst, dp, a.src, sp, a.bytes, j - i, kind, st);
        if (e2 == cudaErrorInvalidValue) {
          cudaGetLastError();
          for (size_t r = i; r < j; ++r)
            GS_CUDA(cudaMemcpyAsync(merged[r].dst, merged[r].src, merged[r].bytes, kind, st));
        } else {
          GS_CUDA(e2);
        }
        i = j;
        continue;
      }
    }
    GS_CUDA(cudaMemcpyAsync(a.dst, a.src, a.bytes, kind, st));
    i = i + 1;
  }
  return GS_OK;
}

}  // namespace

// Batched host-link copies for other translation units (gs_fnv_gpu.cu):
// same merging into 1-D runs / constant-pitch 2-D copies as the pipelines.
int gsb::batch_copies(void* const* dst, const void* const* src, int n, size_t bytes, int kind_d2h, cudaStream_t st) {
  std::vector<CopyOp> ops;
  ops.reserve(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i)
    ops.push_back({static_cast<uint8_t*>(dst[i]), static_cast<const uint8_t*>(src[i]), bytes, 0});
  return issue_copies(ops, kind_d2h ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, st);
}

extern "C" {

// ============================================================================
// diagnostics
// ============================================================================
const char* gs_status_string(int status) {
  switch (status) {
    case GS_OK: return "ok";
    case GS_INVALID_ARGUMENT: return "invalid argument";
    case GS_UNRECOVERABLE: return "unrecoverable";
    case GS_DOMAIN_ERROR: return "domain error";
    case GS_CUDA_ERROR: return "cuda error";
    case GS_UNSUPPORTED: return "unsupported";
    case GS_LOGIC_ERROR: return "logic error";
    case GS_RUNTIME_ERROR: return "runtime error";
    default: return "unknown status";
  }
}
const char* gs_last_error(void) { return g_err.c_str(); }
int gs_abi_version(void) { return 1; }

int gs_jit_quiesce(void) {
  gsb::jit_quiesce();
  return GS_OK;
}
uint64_t gs_kernel_launches(void) { return g_launches.load(); }
uint64_t gs_zero_copy_offloads(void) { return g_zero_copy_calls.load(); }
int gs_set_zero_copy_bytes(uint64_t bytes) {
  g_zero_copy_max.store(bytes);
  return GS_OK;
}
int gs_cuda_available(void) {
  int n = 0;
  return cudaGetDeviceCount(&n) == cudaSuccess && n > 0 ? 1 : 0;
}

// ============================================================================
// field + scheme
// ============================================================================
uint8_t gs_gf_mul(uint8_t a, uint8_t b) { return gf_mul(a, b); }

int gs_gf_inv(uint8_t a, uint8_t* out) {
  if (a == 0) return fail(GS_DOMAIN_ERROR, "gf256: zero has no multiplicative inverse");
  *out = gf_inv(a);
  return GS_OK;
}

int gs_gf_div(uint8_t a, uint8_t b, uint8_t* out) {
  if (b == 0) return fail(GS_DOMAIN_ERROR, "gf256: division by zero");
  *out = a == 0 ? 0 : gf_mul(a, gf_inv(b));
  return GS_OK;
}

int gs_scheme_validate(int kind, int n, int k) { return validate_scheme(kind, n, k); }

int gs_max_tolerance(int kind, int n, int k) {
  (void)n;
  if (kind < GS_XOR || kind > GS_RS) return -1;
  return tolerance(kind, k);
}

int gs_encoding_matrix(int kind, int n, int k, uint8_t* coef) {
  if (int s = validate_scheme(kind, n, k)) return s;
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < n; ++j)
      coef[static_cast<size_t>(i) * n + j] = kind == GS_RS ? cauchy(k, i, j) : 1;
  return GS_OK;
}

// ============================================================================
// codecs
// ============================================================================
static int encoder_create(int kind, int n, int k, bool generic, gs_codec** out) {
  if (!out) return fail(GS_INVALID_ARGUMENT, "encoder_create: out is NULL");
  *out = nullptr;
  if (int s = validate_scheme(kind, n, k)) return s;
  if (kind == GS_RDP && smallest_prime_ge(n + 1) > kRdpMaxCols)
    return fail(GS_UNSUPPORTED, "coding: rdp on the GPU path supports n <= %d", kRdpMaxCols - 2);
  auto* c = new gs_codec;
  c->kind = kind;
  c->n = n;
  c->k = k;
  c->n_out = k;
  c->n_slots = n;
  if (kind == GS_RDP) c->rdp_p = smallest_prime_ge(n + 1);
  c->coef.resize(static_cast<size_t>(k) * n);
  gs_encoding_matrix(kind, n, k, c->coef.data());
  for (int i = 0; i < k; ++i) c->out_index.push_back(n + i);
  c->special = (generic || kind == GS_RDP) ? nullptr : registry().find(false, kind, n, k, 0);
  finish_codec(c);
  *out = c;
  return GS_OK;
}

static int decoder_create(int kind, int n, int k, const int* lost_in, int n_lost, bool generic,
                          gs_codec** out) {
  if (!out) return fail(GS_INVALID_ARGUMENT, "decoder_create: out is NULL");
  *out = nullptr;
  if (int s = validate_scheme(kind, n, k)) return s;
  if (kind == GS_RDP && smallest_prime_ge(n + 1) > kRdpMaxCols)
    return fail(GS_UNSUPPORTED, "coding: rdp on the GPU path supports n <= %d", kRdpMaxCols - 2);
  if (n_lost < 0 || (n_lost > 0 && lost_in == nullptr))
    return fail(GS_INVALID_ARGUMENT, "decoder_create: bad lost list");
  // ErasurePattern: sort + dedup (coding.hpp:131-134)
  std::vector<int> lost(lost_in, lost_in + n_lost);
  std::sort(lost.begin(), lost.end());
  lost.erase(std::unique(lost.begin(), lost.end()), lost.end());
  const int total = n + k;
  for (int idx : lost)  // coding.hpp:463-465
    if (idx < 0 || idx >= total) return fail(GS_INVALID_ARGUMENT, "coding: lost shard index out of range");
  if (static_cast<int>(lost.size()) > tolerance(kind, k))  // :466-470
    return fail(GS_UNRECOVERABLE, "coding: %zu erasures exceed tolerance %d for scheme %s", lost.size(),
                tolerance(kind, k), kind == GS_XOR ? "xor" : kind == GS_RDP ? "rdp" : "rs");
  auto is_lost = [&](int idx) { return std::binary_search(lost.begin(), lost.end(), idx); };
  std::vector<int> ld;
  for (int idx : lost)
    if (idx < n) ld.push_back(idx);
  const int e = static_cast<int>(ld.size());

  auto* c = new gs_codec;
  c->decoder = true;
  c->kind = kind;
  c->n = n;
  c->k = k;
  c->n_out = e;
  c->n_slots = total;
  c->out_index = ld;
  c->coef.assign(static_cast<size_t>(e) * total, 0);
  if (e > 0 && kind == GS_RDP) {  // coding.hpp:503-534
    const int p = smallest_prime_ge(n + 1);
    c->rdp_p = p;
    const bool row_lost = is_lost(n), diag_lost = is_lost(n + 1);
    if (e == 1 && !row_lost) {
      // single data column, row parity present: XOR of every present column
      // (diagonal parity unused) -- served by the XOR(n) decoder, whose
      // slots 0..n coincide with RDP's data + row parity.
      const int lo = ld[0];
      if (int st = decoder_create(GS_XOR, n, 1, &lo, 1, generic, &c->xor_helper)) {
        delete c;
        return st;
      }
      for (int s2 = 0; s2 <= n; ++s2)
        if (s2 != lo) c->coef[s2] = 1;
    } else {
      (void)diag_lost;  // two lost columns imply a surviving diagonal parity
      c->rdp_li = ld[0];
      c->rdp_lj = e == 2 ? ld[1] : p - 1;
      for (int b = 0; b < e; ++b)
        for (int s2 = 0; s2 < total; ++s2)
          if (!is_lost(s2)) c->coef[static_cast<size_t>(b) * total + s2] = 1;
    }
    c->out_index = ld;
    finish_codec(c);
    *out = c;
    return GS_OK;
  }
  if (e > 0) {
    if (kind == GS_XOR) {  // coding.hpp:496-502
      for (int s = 0; s < total; ++s)
        if (!is_lost(s)) c->coef[s] = 1;
    } else {  // coding.hpp:535-566
      std::vector<int> rows;
      for (int i = 0; i < k && static_cast<int>(rows.size()) < e; ++i)
        if (!is_lost(n + i)) rows.push_back(i);
      if (static_cast<int>(rows.size()) < e) {
        delete c;
        return fail(GS_UNRECOVERABLE, "coding: not enough surviving parity shards");
      }
      std::vector<uint8_t> sys(static_cast<size_t>(e) * e), inv;
      for (int a = 0; a < e; ++a)
        for (int b = 0; b < e; ++b) sys[static_cast<size_t>(a) * e + b] = cauchy(k, rows[a], ld[b]);
      if (!invert(sys, e, inv)) {
        delete c;
        return fail(GS_UNRECOVERABLE, "coding: singular decode system");
      }
      for (int b = 0; b < e; ++b) {
        for (int j = 0; j < n; ++j) {
          if (is_lost(j)) continue;
          uint8_t v = 0;
          for (int a = 0; a < e; ++a) v ^= gf_mul(inv[static_cast<size_t>(b) * e + a], cauchy(k, rows[a], j));
          c->coef[static_cast<size_t>(b) * total + j] = v;
        }
        for (int a = 0; a < e; ++a)
          c->coef[static_cast<size_t>(b) * total + n + rows[a]] = inv[static_cast<size_t>(b) * e + a];
      }
    }
    if (total <= 64 && !generic) {
      uint64_t mask = 0;
      for (int idx : lost) mask |= 1ull << idx;
      c->special = registry().find(true, kind, n, k, canonical_mask(kind, n, k, mask));
    }
  }
  finish_codec(c);
  *out = c;
  return GS_OK;
}

int gs_encoder_create(int kind, int n, int k, gs_codec** out) {
  return encoder_create(kind, n, k, false, out);
}

int gs_decoder_create(int kind, int n, int k, const int* lost, int n_lost, gs_codec** out) {
  return decoder_create(kind, n, k, lost, n_lost, false, out);
}

int gs_codec_create_ex(int kind, int n, int k, const int* lost, int n_lost, int flags, gs_codec** out) {
  const bool generic = (flags & GS_FLAG_GENERIC) != 0;
  const int st = (flags & GS_FLAG_DECODER) ? decoder_create(kind, n, k, lost, n_lost, generic, out)
                                           : encoder_create(kind, n, k, generic, out);
  // a forced-generic codec stays on the runtime-coefficient kernel (no JIT):
  // it is how the tests cross-check the two back ends
  if (st == GS_OK && generic) (*out)->jit_tried = true;
  return st;
}

int gs_codec_destroy(gs_codec* c) {
  delete c;
  return GS_OK;
}

int gs_codec_info(const gs_codec* c, int* n_out, int* out_index, int* n_slots, int* specialised) {
  if (!c) return fail(GS_INVALID_ARGUMENT, "codec_info: NULL codec");
  if (n_out) *n_out = c->n_out;
  if (out_index)
    for (int i = 0; i < c->n_out; ++i) out_index[i] = c->out_index[i];
  if (n_slots) *n_slots = c->n_slots;
  if (specialised) *specialised = c->special ? 1 : 0;
  return GS_OK;
}

int gs_codec_coefficients(const gs_codec* c, uint8_t* coef) {
  if (!c || !coef) return fail(GS_INVALID_ARGUMENT, "codec_coefficients: NULL argument");
  std::memcpy(coef, c->coef.data(), c->coef.size());
  return GS_OK;
}

// ============================================================================
// device path
// ============================================================================
int gs_apply_device(const gs_codec* c, int n_stripes, const void* const* slots, void* const* outs,
                    size_t len, void* stream) {
  if (!c) return fail(GS_INVALID_ARGUMENT, "apply: NULL codec");
  if (n_stripes < 0) return fail(GS_INVALID_ARGUMENT, "apply: negative stripe count");
  if (len == 0 || n_stripes == 0 || c->n_out == 0) return GS_OK;
  if (!slots || !outs) return fail(GS_INVALID_ARGUMENT, "apply: NULL pointer array");
  auto slot = [&](int s, int j) -> const void* { return slots[static_cast<size_t>(s) * c->n_slots + j]; };
  auto out = [&](int s, int i) -> const void* { return outs[static_cast<size_t>(s) * c->n_out + i]; };
  return run_codec(c, n_stripes, slot, out, len, static_cast<cudaStream_t>(stream));
}

int gs_apply_device_paged(const gs_codec* c, int n_stripes, const void* const* slots, void* const* outs,
                          size_t len, const gs_page_map* src_map, uint32_t paged_slot_mask,
                          const gs_page_map* dst_map, void* stream) {
  if (!c) return fail(GS_INVALID_ARGUMENT, "apply: NULL codec");
  if (n_stripes < 0) return fail(GS_INVALID_ARGUMENT, "apply: negative stripe count");
  if (len == 0 || n_stripes == 0 || c->n_out == 0) return GS_OK;
  if (!slots || !outs) return fail(GS_INVALID_ARGUMENT, "apply: NULL pointer array");
  Paging pg;
  pg.src = to_map(src_map);
  pg.dst = to_map(dst_map);
  pg.paged_slots = src_map ? paged_slot_mask : 0;
  auto slot = [&](int s, int j) -> const void* { return slots[static_cast<size_t>(s) * c->n_slots + j]; };
  auto out = [&](int s, int i) -> const void* { return outs[static_cast<size_t>(s) * c->n_out + i]; };
  return run_codec(c, n_stripes, slot, out, len, static_cast<cudaStream_t>(stream), pg);
}

// ============================================================================
// pipelines
// ============================================================================
int gs_set_jit(int on) {
  jit_set_enabled(on != 0);
  return GS_OK;
}

int gs_codec_jit_status(const gs_codec* c, int wait, int* status) {
  if (!c || !status) return fail(GS_INVALID_ARGUMENT, "codec_jit_status: NULL argument");
  *status = -2;  // compiled registry kernel, RDP, disabled or not eligible
  if (c->special || c->kind == GS_RDP) return GS_OK;
  JitKernel* k = codec_jit(c);
  if (!k) return GS_OK;
  *status = jit_status(k, wait != 0);
  if (*status == -1) return fail(GS_RUNTIME_ERROR, "jit: %s", jit_last_log(k));
  return GS_OK;
}

int gs_set_kernel_variant(int variant) {
  if (variant < 0 || variant > 2) return fail(GS_INVALID_ARGUMENT, "kernel variant must be 0, 1 or 2");
  g_variant.store(variant);
  return GS_OK;
}

int gs_prewarm(int device) {
  // CUDA loads kernels lazily on first launch; a recovery must not pay that
  // on its critical path, so resolve every kernel (and its occupancy) now.
  DeviceGuard g(device);
  const int sms = device_sms(device);
  (void)sms;
  for (const auto& e : registry().entries) {
    cudaFuncAttributes a;
    GS_CUDA(cudaFuncGetAttributes(&a, e.kernel));
    blocks_per_sm(device, e.kernel, 0);
    GS_CUDA(cudaFuncGetAttributes(&a, e.kernel_paged));
    blocks_per_sm(device, e.kernel_paged, 0);
    GS_CUDA(cudaFuncGetAttributes(&a, e.kernel_bulk));
    const int stages = bulk_stages(&e);
    if (stages >= 2)
      blocks_per_sm(device, e.kernel_bulk,
                    kBulkSmemHeader + static_cast<size_t>(stages) * e.used_cols * e.tile_bulk, kBulkThreads);
  }
  for (int kb = 1; kb <= kMaxGenericRows; ++kb) {
    cudaFuncAttributes a;
    GS_CUDA(cudaFuncGetAttributes(&a, generic_kernel(kb)));
  }
  cudaFuncAttributes a;
  GS_CUDA(cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(&k_ground_truth)));
  GS_CUDA(cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(&k_pad_partial)));
  return GS_OK;
}

int gs_pipeline_create(int device, size_t staging_bytes, gs_pipeline** out) {
  if (!out) return fail(GS_INVALID_ARGUMENT, "pipeline_create: out is NULL");
  *out = nullptr;
  if (staging_bytes < gs_pipeline::kSlots * 4096ull)
    return fail(GS_INVALID_ARGUMENT, "pipeline_create: staging must hold at least %d x 4 KiB",
                gs_pipeline::kSlots);
  DeviceGuard g(device);
  auto* p = new gs_pipeline;
  p->device = device;
  p->bytes = staging_bytes;
  cudaError_t e = cudaMalloc(&p->staging, staging_bytes);
  if (e != cudaSuccess) {
    delete p;
    return fail(GS_CUDA_ERROR, "pipeline staging alloc (%zu B): %s", staging_bytes, cudaGetErrorString(e));
  }
  for (int i = 0; i < gs_pipeline::kSlots; ++i) {
    cudaEventCreateWithFlags(&p->ready[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&p->done[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&p->drained[i], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&p->join, cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&p->s_comp, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking);
  if (int st = gs_prewarm(device)) {
    gs_pipeline_destroy(p);
    return st;
  }
  *out = p;
  return GS_OK;
}

int gs_pipeline_set_timing(gs_pipeline* p, int on) {
  if (!p) return fail(GS_INVALID_ARGUMENT, "pipeline_set_timing: NULL pipeline");
  DeviceGuard g(p->device);
  p->timing = on != 0;
  p->tused = 0;
  p->tlaunch0 = g_launches.load();
  if (p->timing) GS_CUDA(p->reset_stamps());
  return GS_OK;
}

int gs_pipeline_kernel_time(gs_pipeline* p, double* event_ms, double* device_ms, int* groups, uint64_t* launches) {
  if (!p || !event_ms || !groups) return fail(GS_INVALID_ARGUMENT, "pipeline_kernel_time: NULL argument");
  DeviceGuard g(p->device);
  double sum = 0;
  for (size_t i = 0; i + 1 < p->tused; i += 2) {
    GS_CUDA(cudaEventSynchronize(p->tev[i + 1]));
    float ms = 0;
    GS_CUDA(cudaEventElapsedTime(&ms, p->tev[i], p->tev[i + 1]));
    sum += ms;
  }
  const size_t n = std::min(p->tused / 2, gs_pipeline::kStampSlots);
  if (device_ms) {
    double dsum = 0;
    if (n && p->d_stamps) {
      std::vector<unsigned long long> h(2 * n);
      GS_CUDA(cudaMemcpy(h.data(), p->d_stamps, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < n; ++i)
        if (h[2 * i + 1] > h[2 * i] && h[2 * i] != ~0ull) dsum += static_cast<double>(h[2 * i + 1] - h[2 * i]) * 1e-6;
    }
    *device_ms = dsum;
  }
  *event_ms = sum;
  *groups = static_cast<int>(p->tused / 2);
  if (launches) *launches = g_launches.load() - p->tlaunch0;
  p->tused = 0;
  p->tlaunch0 = g_launches.load();
  if (p->timing) GS_CUDA(p->reset_stamps());
  return GS_OK;
}

int gs_pipeline_destroy(gs_pipeline* p) {
  if (!p) return GS_OK;
  DeviceGuard g(p->device);
  cudaDeviceSynchronize();
  for (cudaEvent_t e : p->tev) cudaEventDestroy(e);
  cudaFree(p->d_stamps);
  for (int i = 0; i < gs_pipeline::kSlots; ++i) {
    cudaEventDestroy(p->ready[i]);
    cudaEventDestroy(p->done[i]);
    cudaEventDestroy(p->drained[i]);
  }
  cudaEventDestroy(p->fork);
  cudaEventDestroy(p->join);
  cudaStreamDestroy(p->s_h2d);
  cudaStreamDestroy(p->s_comp);
  cudaStreamDestroy(p->s_d2h);
  cudaFree(p->staging);
  delete p;
  return GS_OK;
}

static int encode_offload(gs_pipeline* p, const gs_codec* c, int n_stripes, const void* const* d_data,
                          void* const* h_parity, size_t len, void* compute, void* copy, const gs_page_map* src_map);

// Encode device data, stage parity, D2H it piecewise (checkpoint offload).
int gs_encode_offload(gs_pipeline* p, const gs_codec* c, int n_stripes, const void* const* d_data,
                      void* const* h_parity, size_t len, void* compute, void* copy) {
  return encode_offload(p, c, n_stripes, d_data, h_parity, len, compute, copy, nullptr);
}

int gs_encode_offload_paged(gs_pipeline* p, const gs_codec* c, int n_stripes, const void* const* d_data,
                            void* const* h_parity, size_t len, const gs_page_map* src_map, void* compute,
                            void* copy) {
  return encode_offload(p, c, n_stripes, d_data, h_parity, len, compute, copy, src_map);
}

// Zero-copy epilogue of the offload: parity bytes per call at or below this
// go straight from the kernel into pinned host memory (GS_ZC_BYTES, 0 = off).


// Every destination is page-locked host memory the device addresses at the
// same pointer (UVA), 16-B aligned: the kernel can store into it directly.
static bool zero_copy_eligible(void* const* h, int count, uint64_t bytes) {
  if (bytes == 0 || bytes > g_zero_copy_max.load(std::memory_order_relaxed) || count > 64) return false;
  for (int i = 0; i < count; ++i) {
    cudaPointerAttributes a{};
    if (!h[i] || !aligned16(h[i]) || cudaPointerGetAttributes(&a, h[i]) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (a.type != cudaMemoryTypeHost || a.devicePointer != h[i]) return false;
  }
  return true;
}

static int encode_offload(gs_pipeline* p, const gs_codec* c, int n_stripes, const void* const* d_data,
                          void* const* h_parity, size_t len, void* compute, void* copy, const gs_page_map* src_map) {
  if (!p || !c) return fail(GS_INVALID_ARGUMENT, "encode_offload: NULL pipeline/codec");
  if (c->decoder) return fail(GS_INVALID_ARGUMENT, "encode_offload: codec is a decoder");
  if (len == 0 || n_stripes == 0) return GS_OK;
  if (!d_data || !h_parity) return fail(GS_INVALID_ARGUMENT, "encode_offload: NULL pointer array");
  DeviceGuard g(p->device);
  auto cs = static_cast<cudaStream_t>(compute);
  auto ks = static_cast<cudaStream_t>(copy);
  GS_CUDA(p->begin(cs, ks));
  const int K = c->n_out, N = c->n_slots;
  if (zero_copy_eligible(h_parity, n_stripes * K, static_cast<uint64_t>(n_stripes) * K * len)) {
    // Small calls: the codec kernel stores the parity rows straight into the
    // pinned host buffers (device-mapped under UVA) -- one kernel, no staging
    // and no DMA descriptor, whose fixed cost dominates a short D2H
    // (tools/small_l_probe.py: 64 KiB shards 6.3 -> 2.6 us per step in a
    // graph). Completion is still signalled on the copy stream.
    auto src = [&](int s, int j) -> const void* { return d_data[static_cast<size_t>(s) * N + j]; };
    auto dst = [&](int s, int i) -> const void* { return h_parity[static_cast<size_t>(s) * K + i]; };
    Paging pg;
    pg.logical0 = 0;
    pg.total_len = len;
    pg.max_grid = p->max_ctas;
    if (src_map) {
      pg.src = to_map(src_map);
      pg.paged_slots = N >= 32 ? ~0u : (1u << N) - 1;
    }
    cudaEvent_t t0, t1;
    GS_CUDA(p->timed_begin(cs, &t0, &t1));
    if (t0) pg.tstamp = p->stamp_slot();
    if (int st = run_codec(c, n_stripes, src, dst, len, cs, pg)) return st;
    if (t1) GS_CUDA(cudaEventRecord(t1, cs));
    if (ks != cs) {
      const int sl = p->next;
      p->next = (p->next + 1) % gs_pipeline::kSlots;
      GS_CUDA(p->record(cs, 1, sl));
      GS_CUDA(p->wait(ks, 1, sl));
    }
    g_zero_copy_calls.fetch_add(1, std::memory_order_relaxed);
    return GS_OK;
  }
  const size_t slot = p->slot_bytes();
  const uint64_t rl_max = piece_len(c, len, slot, K);
  if (!rl_max) return fail(GS_INVALID_ARGUMENT, "encode_offload: staging slot of %zu B cannot hold one piece", slot);
  std::vector<CopyOp> ops;
  for (uint64_t r0 = 0; r0 < len; r0 += rl_max) {
    const uint64_t rl = std::min<uint64_t>(rl_max, len - r0);
    const int spp = static_cast<int>(std::max<uint64_t>(1, slot / (K * rl)));
    for (int s0 = 0; s0 < n_stripes; s0 += spp) {
      const int cnt = std::min(spp, n_stripes - s0);
      const int sl = p->next;
      p->next = (p->next + 1) % gs_pipeline::kSlots;
      uint8_t* base = p->staging + static_cast<size_t>(sl) * slot;
      GS_CUDA(p->wait(cs, 2, sl));  // slot's previous D2H finished
      auto src = [&](int s, int j) -> const void* {
        return static_cast<const uint8_t*>(d_data[static_cast<size_t>(s0 + s) * N + j]) + (src_map ? 0 : r0);
      };
      auto dst = [&](int s, int i) -> const void* { return base + (static_cast<size_t>(s) * K + i) * rl; };
      Paging pg;
      pg.logical0 = r0;
      pg.total_len = len;
      pg.stripe0 = static_cast<uint64_t>(s0);
      pg.max_grid = p->max_ctas;
      if (src_map) {
        pg.src = to_map(src_map);
        pg.paged_slots = N >= 32 ? ~0u : (1u << N) - 1;
      }
      cudaEvent_t t0, t1;
      GS_CUDA(p->timed_begin(cs, &t0, &t1));
      if (t0) pg.tstamp = p->stamp_slot();
      if (int st = run_codec(c, cnt, src, dst, rl, cs, pg)) return st;
      if (t1) GS_CUDA(cudaEventRecord(t1, cs));
      GS_CUDA(p->record(cs, 1, sl));
      GS_CUDA(p->wait(ks, 1, sl));
      for (int s = 0; s < cnt; ++s)
        for (int i = 0; i < K; ++i)
          ops.push_back({static_cast<uint8_t*>(h_parity[static_cast<size_t>(s0 + s) * K + i]) + r0,
                         base + (static_cast<size_t>(s) * K + i) * rl, rl, i});
      if (int st = issue_copies(ops, cudaMemcpyDeviceToHost, ks)) return st;
      GS_CUDA(p->record(ks, 2, sl));
    }
  }
  return GS_OK;
}

static int reconstruct_upload(gs_pipeline* p, const gs_codec* c, int n_stripes, const void* const* slots,
                              void* const* outs, size_t len, void* compute, void* copy, const gs_page_map* src_map,
                              const gs_page_map* dst_map);

// Rebuild lost shards: H2D used parity rows piecewise, rebuild per piece.
int gs_reconstruct_upload(gs_pipeline* p, const gs_codec* c, int n_stripes, const void* const* slots,
                          void* const* outs, size_t len, void* compute, void* copy) {
  return reconstruct_upload(p, c, n_stripes, slots, outs, len, compute, copy, nullptr, nullptr);
}

int gs_reconstruct_upload_paged(gs_pipeline* p, const gs_codec* c, int n_stripes, const void* const* slots,
                                void* const* outs, size_t len, const gs_page_map* src_map,
                                const gs_page_map* dst_map, void* compute, void* copy) {
  return reconstruct_upload(p, c, n_stripes, slots, outs, len, compute, copy, src_map, dst_map);
}

static int reconstruct_upload(gs_pipeline* p, const gs_codec* c, int n_stripes, const void* const* slots,
                              void* const* outs, size_t len, void* compute, void* copy, const gs_page_map* src_map,
                              const gs_page_map* dst_map) {
  if (!p || !c) return fail(GS_INVALID_ARGUMENT, "reconstruct_upload: NULL pipeline/codec");
  if (!c->decoder) return fail(GS_INVALID_ARGUMENT, "reconstruct_upload: codec is an encoder");
  if (len == 0 || n_stripes == 0 || c->n_out == 0) return GS_OK;
  if (!slots || !outs) return fail(GS_INVALID_ARGUMENT, "reconstruct_upload: NULL pointer array");
  DeviceGuard g(p->device);
  auto cs = static_cast<cudaStream_t>(compute);
  auto ks = static_cast<cudaStream_t>(copy);
  GS_CUDA(p->begin(cs, ks));
  const int NS = c->n_slots, NO = c->n_out, n = c->n;
  std::vector<int> host_slots;  // parity slots actually used
  for (int j : c->used)
    if (j >= n) host_slots.push_back(j);
  const int H = std::max<int>(1, static_cast<int>(host_slots.size()));
  const size_t slot = p->slot_bytes();
  // Recovery is latency-bound on the H2D: cut the upload into >= 4 pieces
  // (>= 1 MiB each) so the rebuild of piece i runs under the H2D of piece
  // i+1 instead of after the whole upload.
  const uint64_t total_h2d = static_cast<uint64_t>(n_stripes) * H * len;
  static const uint64_t min_pieces = [] {
    const char* e = std::getenv("GS_UPLOAD_PIECES");
    return static_cast<uint64_t>(e && std::atoi(e) > 0 ? std::atoi(e) : 4);
  }();
  const uint64_t piece_cap = std::max<uint64_t>(1ull << 20, total_h2d / min_pieces);
  const uint64_t rl_max = piece_len(c, len, slot, H, std::max<uint64_t>(4096, piece_cap / H));
  if (!rl_max) return fail(GS_INVALID_ARGUMENT, "reconstruct_upload: staging slot of %zu B cannot hold one piece", slot);
  std::vector<CopyOp> ops;
  for (uint64_t r0 = 0; r0 < len; r0 += rl_max) {
    const uint64_t rl = std::min<uint64_t>(rl_max, len - r0);
    const int spp = static_cast<int>(
        std::max<uint64_t>(1, std::min<uint64_t>(slot / (H * rl), piece_cap / (H * rl))));
    for (int s0 = 0; s0 < n_stripes; s0 += spp) {
      const int cnt = std::min(spp, n_stripes - s0);
      const int sl = p->next;
      p->next = (p->next + 1) % gs_pipeline::kSlots;
      uint8_t* base = p->staging + static_cast<size_t>(sl) * slot;
      GS_CUDA(p->wait(ks, 1, sl));  // slot's previous kernel consumed it
      for (int s = 0; s < cnt; ++s)
        for (size_t h = 0; h < host_slots.size(); ++h) {
          const void* hp = slots[static_cast<size_t>(s0 + s) * NS + host_slots[h]];
          if (!hp) return fail(GS_INVALID_ARGUMENT, "reconstruct_upload: parity slot %d is NULL", host_slots[h]);
          ops.push_back({base + (static_cast<size_t>(s) * H + h) * rl, static_cast<const uint8_t*>(hp) + r0, rl,
                         static_cast<int>(h)});
        }
      if (int st = issue_copies(ops, cudaMemcpyHostToDevice, ks)) return st;
      GS_CUDA(p->record(ks, 0, sl));
      GS_CUDA(p->wait(cs, 0, sl));
      auto src = [&](int s, int j) -> const void* {
        if (j >= n) {
          const auto it = std::find(host_slots.begin(), host_slots.end(), j);
          if (it == host_slots.end()) return nullptr;
          return base + (static_cast<size_t>(s) * H + (it - host_slots.begin())) * rl;
        }
        const void* d = slots[static_cast<size_t>(s0 + s) * NS + j];
        return d ? static_cast<const uint8_t*>(d) + (src_map ? 0 : r0) : nullptr;
      };
      auto dst = [&](int s, int i) -> const void* {
        return static_cast<const uint8_t*>(outs[static_cast<size_t>(s0 + s) * NO + i]) + (dst_map ? 0 : r0);
      };
      Paging pg;
      pg.logical0 = r0;
      pg.total_len = len;
      pg.stripe0 = static_cast<uint64_t>(s0);
      if (src_map) {
        pg.src = to_map(src_map);
        pg.paged_slots = n >= 32 ? ~0u : (1u << n) - 1;  // data slots; parity comes from staging
      }
      if (dst_map) pg.dst = to_map(dst_map);
      cudaEvent_t t0, t1;
      GS_CUDA(p->timed_begin(cs, &t0, &t1));
      if (t0) pg.tstamp = p->stamp_slot();
      if (int st = run_codec(c, cnt, src, dst, rl, cs, pg)) return st;
      if (t1) GS_CUDA(cudaEventRecord(t1, cs));
      GS_CUDA(p->record(cs, 1, sl));
    }
  }
  GS_CUDA(p->end(cs, ks));
  return GS_OK;
}

// ---- one-call forms ------------------------------------------
namespace {
// Default pipelines live until process exit: they are not destroyed from
// thread-exit destructors, which may run after the CUDA runtime unloads.
struct DefaultPipelines {
  std::map<int, gs_pipeline*> by_dev;
};
thread_local DefaultPipelines t_pipes;

int default_pipeline(gs_pipeline** out) {
  int dev = 0;
  GS_CUDA(cudaGetDevice(&dev));
  auto it = t_pipes.by_dev.find(dev);
  if (it != t_pipes.by_dev.end()) {
    *out = it->second;
    return GS_OK;
  }
  gs_pipeline* p = nullptr;
  if (int st = gs_pipeline_create(dev, 256ull << 20, &p)) return st;
  t_pipes.by_dev[dev] = p;
  *out = p;
  return GS_OK;
}

// decoders cached per (encoder scheme, canonical lost set); process-wide
std::mutex g_dec_mu;
std::map<std::tuple<int, int, int, std::vector<int>>, gs_codec*> g_dec_cache;
}  // namespace

int gs_codec_create(int kind, int n, int k, gs_codec** out) { return gs_encoder_create(kind, n, k, out); }

int gs_pipeline_set_max_ctas(gs_pipeline* p, int max_ctas) {
  if (!p || max_ctas < 0) return fail(GS_INVALID_ARGUMENT, "pipeline_set_max_ctas: bad arguments");
  p->max_ctas = max_ctas;
  return GS_OK;
}

int gs_pipeline_device(gs_pipeline* p, int* device) {
  if (!p || !device) return fail(GS_INVALID_ARGUMENT, "pipeline_device: NULL argument");
  *device = p->device;
  return GS_OK;
}

int gs_thread_pipeline(gs_pipeline** out) {
  if (!out) return fail(GS_INVALID_ARGUMENT, "thread_pipeline: NULL out");
  return default_pipeline(out);
}

int gs_encode_async(const gs_codec* enc, const void* const* d_shards, size_t len, void* const* h_parity,
                    void* compute, void* copy) {
  if (!enc) return fail(GS_INVALID_ARGUMENT, "encode_async: NULL codec");
  gs_pipeline* p = nullptr;
  if (int st = default_pipeline(&p)) return st;
  return gs_encode_offload(p, enc, 1, d_shards, h_parity, len, compute, copy);
}

int gs_reconstruct_async(const gs_codec* enc, const int* lost, int n_lost, const void* const* d_survivors,
                         const void* const* h_parity, void* const* d_out, size_t len, void* stream) {
  if (!enc) return fail(GS_INVALID_ARGUMENT, "reconstruct_async: NULL codec");
  if (enc->decoder) return fail(GS_INVALID_ARGUMENT, "reconstruct_async: pass the scheme's encoder codec");
  if (n_lost < 0 || (n_lost > 0 && !lost)) return fail(GS_INVALID_ARGUMENT, "reconstruct_async: bad lost list");
  std::vector<int> key_lost(lost, lost + n_lost);
  std::sort(key_lost.begin(), key_lost.end());
  key_lost.erase(std::unique(key_lost.begin(), key_lost.end()), key_lost.end());
  gs_codec* dec = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_dec_mu);
    auto key = std::make_tuple(enc->kind, enc->n, enc->k, key_lost);
    auto it = g_dec_cache.find(key);
    if (it != g_dec_cache.end()) {
      dec = it->second;
    } else {
      if (int st = gs_decoder_create(enc->kind, enc->n, enc->k, key_lost.data(),
                                     static_cast<int>(key_lost.size()), &dec))
        return st;
      g_dec_cache[key] = dec;
    }
  }
  if (dec->n_out == 0) return GS_OK;
  if (!d_survivors || !h_parity || !d_out) return fail(GS_INVALID_ARGUMENT, "reconstruct_async: NULL pointer array");
  std::vector<const void*> slots(static_cast<size_t>(enc->n + enc->k), nullptr);
  for (int j = 0; j < enc->n; ++j) slots[j] = d_survivors[j];
  for (int i = 0; i < enc->k; ++i) slots[enc->n + i] = h_parity[i];
  for (int idx : key_lost)
    if (idx >= 0 && idx < enc->n + enc->k) slots[idx] = nullptr;
  gs_pipeline* p = nullptr;
  if (int st = default_pipeline(&p)) return st;
  return gs_reconstruct_upload(p, dec, 1, slots.data(), d_out, len, stream, stream);
}

int gs_sync(void* stream) {
  // NULL is the legacy default stream -- work enqueued there (gs_encode_async
  // with compute = copy = NULL) must be waited for like any other stream's
  GS_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  for (auto& kv : t_pipes.by_dev)
    if (int st = gs_pipeline_sync(kv.second)) return st;
  return GS_OK;
}

// Host buffers in, host buffers out: H2D data -> kernel -> D2H parity, per
// piece, three streams so both copy directions and the kernel overlap.
int gs_encode_host_async(gs_pipeline* p, const gs_codec* c, const void* const* h_data, void* const* h_parity,
                         size_t len) {
  if (!p || !c) return fail(GS_INVALID_ARGUMENT, "encode_host: NULL pipeline/codec");
  if (c->decoder) return fail(GS_INVALID_ARGUMENT, "encode_host: codec is a decoder");
  if (len == 0) return GS_OK;
  if (!h_data || !h_parity) return fail(GS_INVALID_ARGUMENT, "encode_host: NULL pointer array");
  for (int j = 0; j < c->n_slots; ++j)
    if (!h_data[j]) return fail(GS_INVALID_ARGUMENT, "encode_host: data shard %d is NULL", j);
  DeviceGuard g(p->device);
  GS_CUDA(p->begin(p->s_h2d, p->s_h2d));
  const int N = c->n_slots, K = c->n_out;
  const size_t slot = p->slot_bytes();
  // ~2 MiB per shard per piece: deep enough pipelining that the H2D of piece
  // i+1, the kernel of piece i and the D2H of piece i-1 overlap.
  const uint64_t rl_max = piece_len(c, len, slot, N + K, kHostPiece);
  if (!rl_max) return fail(GS_INVALID_ARGUMENT, "encode_host: staging slot of %zu B cannot hold one piece", slot);
  std::vector<CopyOp> ops;
  const uint64_t quarter = rl_max >= 4 * 4096 ? std::min<uint64_t>(align_down_piece(c, rl_max / 4), len) : 0;
  for (uint64_t r0 = 0, rl = 0; r0 < len; r0 += rl) {
    rl = taper(r0, len, rl_max, quarter);
    const int sl = p->next;
    p->next = (p->next + 1) % gs_pipeline::kSlots;
    uint8_t* in = p->staging + static_cast<size_t>(sl) * slot;
    uint8_t* outb = in + static_cast<size_t>(N) * rl;
    GS_CUDA(cudaStreamWaitEvent(p->s_h2d, p->drained[sl], 0));
    for (int j = 0; j < N; ++j)
      ops.push_back({in + static_cast<size_t>(j) * rl, static_cast<const uint8_t*>(h_data[j]) + r0, rl, 0});
    if (int st = issue_copies(ops, cudaMemcpyHostToDevice, p->s_h2d)) return st;
    GS_CUDA(cudaEventRecord(p->ready[sl], p->s_h2d));
    GS_CUDA(cudaStreamWaitEvent(p->s_comp, p->ready[sl], 0));
    auto src = [&](int, int j) -> const void* { return in + static_cast<size_t>(j) * rl; };
    auto dst = [&](int, int i) -> const void* { return outb + static_cast<size_t>(i) * rl; };
    Paging pg;
    pg.logical0 = r0;
    pg.total_len = len;
    if (int st = run_codec(c, 1, src, dst, rl, p->s_comp, pg)) return st;
    GS_CUDA(cudaEventRecord(p->done[sl], p->s_comp));
    GS_CUDA(cudaStreamWaitEvent(p->s_d2h, p->done[sl], 0));
    for (int i = 0; i < K; ++i)
      ops.push_back({static_cast<uint8_t*>(h_parity[i]) + r0, outb + static_cast<size_t>(i) * rl, rl, 0});
    if (int st = issue_copies(ops, cudaMemcpyDeviceToHost, p->s_d2h)) return st;
    GS_CUDA(cudaEventRecord(p->drained[sl], p->s_d2h));
  }
  return GS_OK;
}

int gs_pipeline_sync(gs_pipeline* p) {
  if (!p) return fail(GS_INVALID_ARGUMENT, "pipeline_sync: NULL pipeline");
  DeviceGuard g(p->device);
  GS_CUDA(cudaStreamSynchronize(p->s_h2d));
  GS_CUDA(cudaStreamSynchronize(p->s_comp));
  GS_CUDA(cudaStreamSynchronize(p->s_d2h));
  return GS_OK;
}

int gs_encode_host(gs_pipeline* p, const gs_codec* c, const void* const* h_data, void* const* h_parity,
                   size_t len) {
  if (int st = gs_encode_host_async(p, c, h_data, h_parity, len)) return st;
  return p ? gs_pipeline_sync(p) : GS_OK;
}

int gs_reconstruct_host_async(gs_pipeline* p, const gs_codec* c, const void* const* h_slots,
                              void* const* h_out, size_t len) {
  if (!p || !c) return fail(GS_INVALID_ARGUMENT, "reconstruct_host: NULL pipeline/codec");
  if (!c->decoder) return fail(GS_INVALID_ARGUMENT, "reconstruct_host: codec is an encoder");
  if (len == 0 || c->n_out == 0) return GS_OK;
  if (!h_slots || !h_out) return fail(GS_INVALID_ARGUMENT, "reconstruct_host: NULL pointer array");
  for (int j : c->used)
    if (!h_slots[j]) return fail(GS_INVALID_ARGUMENT, "coding: surviving shard %d missing from input", j);
  DeviceGuard g(p->device);
  GS_CUDA(p->begin(p->s_h2d, p->s_h2d));
  const int U = static_cast<int>(c->used.size()), E = c->n_out;
  const size_t slot = p->slot_bytes();
  const uint64_t rl_max = piece_len(c, len, slot, U + E, kHostPiece);
  if (!rl_max) return fail(GS_INVALID_ARGUMENT, "reconstruct_host: staging slot of %zu B cannot hold one piece", slot);
  std::vector<CopyOp> ops;
  const uint64_t quarter = rl_max >= 4 * 4096 ? std::min<uint64_t>(align_down_piece(c, rl_max / 4), len) : 0;
  for (uint64_t r0 = 0, rl = 0; r0 < len; r0 += rl) {
    rl = taper(r0, len, rl_max, quarter);
    const int sl = p->next;
    p->next = (p->next + 1) % gs_pipeline::kSlots;
    uint8_t* in = p->staging + static_cast<size_t>(sl) * slot;
    uint8_t* outb = in + static_cast<size_t>(U) * rl;
    GS_CUDA(cudaStreamWaitEvent(p->s_h2d, p->drained[sl], 0));
    for (int u = 0; u < U; ++u)
      ops.push_back({in + static_cast<size_t>(u) * rl, static_cast<const uint8_t*>(h_slots[c->used[u]]) + r0, rl, 0});
    if (int st = issue_copies(ops, cudaMemcpyHostToDevice, p->s_h2d)) return st;
    GS_CUDA(cudaEventRecord(p->ready[sl], p->s_h2d));
    GS_CUDA(cudaStreamWaitEvent(p->s_comp, p->ready[sl], 0));
    auto src = [&](int, int j) -> const void* {
      const auto it = std::find(c->used.begin(), c->used.end(), j);
      return it == c->used.end() ? nullptr : in + static_cast<size_t>(it - c->used.begin()) * rl;
    };
    auto dst = [&](int, int i) -> const void* { return outb + static_cast<size_t>(i) * rl; };
    Paging pg;
    pg.logical0 = r0;
    pg.total_len = len;
    if (int st = run_codec(c, 1, src, dst, rl, p->s_comp, pg)) return st;
    GS_CUDA(cudaEventRecord(p->done[sl], p->s_comp));
    GS_CUDA(cudaStreamWaitEvent(p->s_d2h, p->done[sl], 0));
    for (int i = 0; i < E; ++i)
      ops.push_back({static_cast<uint8_t*>(h_out[i]) + r0, outb + static_cast<size_t>(i) * rl, rl, 0});
    if (int st = issue_copies(ops, cudaMemcpyDeviceToHost, p->s_d2h)) return st;
    GS_CUDA(cudaEventRecord(p->drained[sl], p->s_d2h));
  }
  return GS_OK;
}

int gs_reconstruct_host(gs_pipeline* p, const gs_codec* c, const void* const* h_slots, void* const* h_out,
                        size_t len) {
  if (int st = gs_reconstruct_host_async(p, c, h_slots, h_out, len)) return st;
  return p ? gs_pipeline_sync(p) : GS_OK;
}

// ============================================================================
// KV data model
// ============================================================================
int gs_slice_bytes(int layers, int kv_heads, int head_dim, int tp, uint32_t chunk_size, uint64_t* out) {
  if (layers < 1 || kv_heads < 1 || head_dim < 1 || tp < 1)
    return fail(GS_INVALID_ARGUMENT, "model: all dimensions must be positive");
  if ((static_cast<int64_t>(kv_heads) * head_dim) % tp != 0)
    return fail(GS_INVALID_ARGUMENT, "model: kv_heads * head_dim must divide evenly across workers");
  const uint64_t elems = static_cast<uint64_t>(kv_heads) * head_dim / tp;
  *out = 2ull * layers * chunk_size * elems * 2ull;
  return GS_OK;
}

static uint64_t splitmix_step(uint64_t& s) {
  s += 0x9E3779B97F4A7C15ull;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int gs_ground_truth_slice_device(uint64_t kv_seed, uint64_t request_id, uint32_t chunk, int worker,
                                 int layers, int kv_heads, int head_dim, int tp, uint32_t chunk_size,
                                 uint32_t valid_tokens, void* d_out, void* stream) {
  uint64_t len = 0;
  if (int s = gs_slice_bytes(layers, kv_heads, head_dim, tp, chunk_size, &len)) return s;
  if (valid_tokens > chunk_size) return fail(GS_INVALID_ARGUMENT, "kv: valid_tokens exceeds chunk size");
  if (len == 0) return GS_OK;
  if (!d_out) return fail(GS_INVALID_ARGUMENT, "ground_truth: NULL output");
  // mix_key (kv_layout.hpp:96-103)
  uint64_t a = request_id + 0x9E3779B97F4A7C15ull, b = chunk + 0xC2B2AE3D27D4EB4Full,
           c = static_cast<uint64_t>(static_cast<int64_t>(worker)) + 0x165667B19E3779F9ull;
  uint64_t state = kv_seed;
  state ^= splitmix_step(a);
  state ^= splitmix_step(b);
  state ^= splitmix_step(c);
  const uint64_t stride = static_cast<uint64_t>(kv_heads) * head_dim / tp * 2;
  const uint64_t block = stride * chunk_size, keep = stride * valid_tokens;
  int dev = 0;
  if (int s = current_device(&dev)) return s;
  const uint64_t words = (len + 7) / 8;
  const int grid = static_cast<int>(std::min<uint64_t>((words + 255) / 256, device_sms(dev) * 8ull));
  k_ground_truth<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<uint8_t*>(d_out), len, state,
                                                                      block, keep);
  GS_CUDA(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return GS_OK;
}

// Host-buffer form (the reference's make_ground_truth_slice returns host
// bytes): generated by k_ground_truth into a temporary device buffer, copied
// back; synchronous.
int gs_ground_truth_slice(uint64_t kv_seed, uint64_t request_id, uint32_t chunk, int worker, int layers,
                          int kv_heads, int head_dim, int tp, uint32_t chunk_size, uint32_t valid_tokens,
                          void* h_out) {
  uint64_t len = 0;
  if (int s = gs_slice_bytes(layers, kv_heads, head_dim, tp, chunk_size, &len)) return s;
  if (valid_tokens > chunk_size) return fail(GS_INVALID_ARGUMENT, "kv: valid_tokens exceeds chunk size");
  if (len == 0) return GS_OK;
  if (!h_out) return fail(GS_INVALID_ARGUMENT, "ground_truth: NULL output");
  void* d = nullptr;
  GS_CUDA(cudaMalloc(&d, len));
  int st = gs_ground_truth_slice_device(kv_seed, request_id, chunk, worker, layers, kv_heads, head_dim, tp,
                                        chunk_size, valid_tokens, d, nullptr);
  if (st == GS_OK) {
    const cudaError_t e = cudaMemcpy(h_out, d, len, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) st = fail(GS_CUDA_ERROR, "ground_truth copy: %s", cudaGetErrorString(e));
  }
  cudaFree(d);
  return st;
}

int gs_pad_partial_device(void* d_slice, int layers, int kv_heads, int head_dim, int tp, uint32_t chunk_size,
                          uint32_t valid_tokens, void* stream) {
  uint64_t len = 0;
  if (int s = gs_slice_bytes(layers, kv_heads, head_dim, tp, chunk_size, &len)) return s;
  if (valid_tokens > chunk_size) return fail(GS_INVALID_ARGUMENT, "kv: valid_tokens exceeds chunk size");
  if (len == 0 || valid_tokens == chunk_size) return GS_OK;
  const uint64_t stride = static_cast<uint64_t>(kv_heads) * head_dim / tp * 2;
  int dev = 0;
  if (int s = current_device(&dev)) return s;
  const int grid = static_cast<int>(std::min<uint64_t>((len + 255) / 256, device_sms(dev) * 8ull));
  k_pad_partial<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<uint8_t*>(d_slice), len,
                                                                     stride * chunk_size, stride * valid_tokens);
  GS_CUDA(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return GS_OK;
}

// ============================================================================
// parity seal
// ============================================================================
uint64_t gs_fnv1a64(const void* bytes, size_t len, uint64_t h) {
  const uint8_t* p = static_cast<const uint8_t*>(bytes);
  if (len >= kFnvSimdMin && fnv_simd_available()) return fnv1a64_fast(p, len, h);
  return fnv1a64_one(p, len, h);
}

int gs_fnv_host_simd(void) { return fnv_simd_available() ? 1 : 0; }

int gs_fnv_host_set_simd(int on) { return fnv_simd_set(on != 0) ? 1 : 0; }

uint64_t gs_parity_checksum(const void* const* parity, int k, size_t len) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (int i = 0; i < k; ++i) h = gs_fnv1a64(parity[i], len, h);
  return h;
}

int gs_parity_checksum_batch(const void* const* parity, int n_chunks, int k, size_t len, int threads,
                             uint64_t* out) {
  if (n_chunks < 0 || k < 1 || !out || (n_chunks > 0 && !parity))
    return fail(GS_INVALID_ARGUMENT, "checksum_batch: bad arguments");
  if (threads < 1) threads = 1;
  // Every chain is serial (one multiply per byte), so the wall time is the
  // number of chains one thread advances one after another times a chain's
  // length: give each thread ONE lockstep group of ceil(chunks / threads)
  // chains (4..8) rather than several groups of four.
  // With the SIMD chain (several GB/s per chain) one chain per claim spreads
  // the chunks over every thread.
  const int per = fnv_simd_available() ? 1 : std::max(4, std::min(8, (n_chunks + threads - 1) / std::max(threads, 1)));
  const int groups = (n_chunks + per - 1) / per;
  threads = std::min(threads, std::max(1, groups));
  std::atomic<int> next{0};
  auto work = [&] {
    for (int g = next.fetch_add(1); g < groups; g = next.fetch_add(1)) {
      const int c0 = per * g, m = std::min(per, n_chunks - c0);
      uint64_t h[8];
      for (int q = 0; q < 8; ++q) h[q] = kFnvOffset;
      for (int i = 0; i < k; ++i) {  // chained over the k buffers in order
        const uint8_t* ps[8];
        for (int q = 0; q < m; ++q) ps[q] = static_cast<const uint8_t*>(parity[static_cast<size_t>(c0 + q) * k + i]);
        fnv1a64_chains(ps, m, len, h);
      }
      for (int q = 0; q < m; ++q) out[c0 + q] = h[q];
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  return GS_OK;
}

// ============================================================================
// peer memory
// ============================================================================
int gs_ipc_handle(const void* d_ptr, void* handle_out, uint64_t* offset_out) {
  if (!d_ptr || !handle_out || !offset_out) return fail(GS_INVALID_ARGUMENT, "ipc_handle: NULL argument");
  // IPC handles name whole allocations; find the base of the allocation that
  // holds d_ptr (e.g. inside a caching-allocator block) through the driver.
  using AddrRangeFn = int (*)(unsigned long long*, size_t*, unsigned long long);
  static AddrRangeFn range_fn = nullptr;
  if (!range_fn) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    GS_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (!fn) return fail(GS_CUDA_ERROR, "ipc_handle: cuMemGetAddressRange unavailable");
    range_fn = reinterpret_cast<AddrRangeFn>(fn);
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, reinterpret_cast<unsigned long long>(d_ptr)) != 0)
    return fail(GS_CUDA_ERROR, "ipc_handle: cuMemGetAddressRange failed for %p", d_ptr);
  cudaIpcMemHandle_t h;
  GS_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  static_assert(sizeof(h) == GS_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle_out, &h, sizeof h);
  *offset_out = reinterpret_cast<unsigned long long>(d_ptr) - base;
  return GS_OK;
}

int gs_ipc_open(const void* handle, int device, void** d_base) {
  if (!handle || !d_base) return fail(GS_INVALID_ARGUMENT, "ipc_open: NULL argument");
  DeviceGuard g(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  GS_CUDA(cudaIpcOpenMemHandle(d_base, h, cudaIpcMemLazyEnablePeerAccess));
  return GS_OK;
}

int gs_ipc_close(void* d_ptr) {
  GS_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return GS_OK;
}

int gs_peer_enable(int device, int peer) {
  if (device == peer) return GS_OK;
  int can = 0;
  GS_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) return fail(GS_UNSUPPORTED, "peer access %d -> %d not supported", device, peer);
  DeviceGuard g(device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return GS_OK;
  }
  GS_CUDA(e);
  return GS_OK;
}

int gs_stripe_range(uint64_t total, int rank, int world, uint64_t* off, uint64_t* len) {
  if (world < 1 || rank < 0 || rank >= world || !off || !len)
    return fail(GS_INVALID_ARGUMENT, "stripe_range: bad rank/world");
  uint64_t per = (total + world - 1) / world;
  per = (per + 4095) / 4096 * 4096;
  const uint64_t o = std::min<uint64_t>(total, per * rank);
  const uint64_t e = std::min<uint64_t>(total, o + per);
  *off = o;
  *len = e - o;
  return GS_OK;
}

// ============================================================================
// pinned host memory
// ============================================================================
int gs_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(GS_INVALID_ARGUMENT, "host_alloc: out is NULL");
  GS_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocPortable));
  return GS_OK;
}

int gs_host_free(void* p) {
  if (gsb::pinned_free_near(p)) return GS_OK;
  GS_CUDA(cudaFreeHost(p));
  return GS_OK;
}

}  // extern "C"

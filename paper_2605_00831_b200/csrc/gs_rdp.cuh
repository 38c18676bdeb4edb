// gs_rdp.cuh -- shortened RDP (row-diagonal parity) on sm_100a.
//
// Reference: coding.hpp:225-251 (layout), :277-307 (encode), :343-449
// (two-column recovery), :503-534 (dispatch). The array is (p-1) rows x
// (p+1) columns for the smallest prime p >= n+1; a "dstripe" is p-1
// consecutive bytes of every column. Data columns 0..n-1 (n..p-2 virtual
// zero), row parity = column p-1 (= byte-wise XOR of the data), diagonal
// d = (r + c) mod p stored at row d of the diagonal buffer for d <= p-2.
// Bytes past the last whole dstripe are protected by P (row parity) and
// Q = sum_c 2^c * data_c over GF(2^8).
//
// RDP is position-dependent, so unlike XOR/RS it cannot stream 16-byte
// groups straight through registers: each CTA stages a tile of 256
// dstripes of every column in shared memory with coalesced loads, one
// thread per dstripe evaluates the diagonals (or walks the two recovery
// chains) out of shared memory, and the results leave through shared memory
// with coalesced stores. Single-column recoveries are plain XORs and run on
// the XOR kernels instead.
#pragma once

#include <cstdint>

#include "gs_kernels.cuh"

namespace gsb {

constexpr int kRdpThreads = 256;  // one dstripe per thread per tile
constexpr int kRdpMaxCols = 24;   // p <= 23 -> n <= 22 on this path

// Primes with kernels (p = smallest prime >= n+1 for n = 1..22).
#define GS_RDP_PRIMES(X) X(2) X(3) X(5) X(7) X(11) X(13) X(17) X(19) X(23)

struct RdpGeom {
  int n, p, rows;
  uint64_t len;       // bytes of this launch's range (per column)
  uint64_t logical0;  // absolute offset of byte 0 of the range (multiple of rows)
  uint64_t full;      // absolute end of the whole dstripes
  uint64_t total;     // absolute column length
  uint32_t tps, ntiles;
  int stride;         // pointers per codec stripe in the table
  int aligned;
  // recovery: the two lost array columns (i < j; j == p-1 => row parity lost)
  int li, lj;
};

__device__ __forceinline__ uint8_t gf_mul_dev(uint8_t a, uint8_t b) { return gf_mul(a, b); }

// (a mod p) for a in (-p, 2p): one compare-and-add instead of an integer
// division (all the array index arithmetic stays in that range).
__device__ __forceinline__ int pmod(int a, int p) {
  a = a < 0 ? a + p : a;
  return a >= p ? a - p : a;
}

// Cooperative tile load of `bytes` bytes at src into smem (16-B vectors when
// aligned, bytes otherwise; zero-fill to `span`).
__device__ __forceinline__ void rdp_load(uint8_t* dst, const uint8_t* src, uint32_t bytes, uint32_t span,
                                         bool aligned) {
  if (aligned) {
    const uint32_t vec = bytes / 16;
    for (uint32_t v = threadIdx.x; v < vec; v += blockDim.x)
      reinterpret_cast<uint4*>(dst)[v] = ld_stream(src + v * 16);
    for (uint32_t b = vec * 16 + threadIdx.x; b < span; b += blockDim.x) dst[b] = b < bytes ? src[b] : 0;
  } else {
    for (uint32_t b = threadIdx.x; b < span; b += blockDim.x) dst[b] = b < bytes ? src[b] : 0;
  }
}

__device__ __forceinline__ void rdp_store(uint8_t* dst, const uint8_t* src, uint32_t bytes, bool aligned) {
  if (aligned) {
    const uint32_t vec = bytes / 16;
    for (uint32_t v = threadIdx.x; v < vec; v += blockDim.x)
      st_stream(dst + v * 16, reinterpret_cast<const uint4*>(src)[v]);
    for (uint32_t b = vec * 16 + threadIdx.x; b < bytes; b += blockDim.x) dst[b] = src[b];
  } else {
    for (uint32_t b = threadIdx.x; b < bytes; b += blockDim.x) dst[b] = src[b];
  }
}

// Encode: out0 = row parity (whole range), out1 = diagonal parity (whole
// dstripes) + Q (tail). smem: p-1 column tiles (virtual columns n..p-2 are
// zero, so the diagonal loop is the same for every n) + row + diag tiles.
// P is a template parameter: every index in the diagonal loop is a
// compile-time constant and the 90-odd byte XORs per dstripe fully unroll.
template <int CAP, int P>
__global__ void __launch_bounds__(kRdpThreads) k_rdp_encode(const PtrTable<CAP> tab, const RdpGeom g) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int R = P - 1;
  constexpr uint32_t T = static_cast<uint32_t>(R) * kRdpThreads;
  const int n = g.n;
  uint8_t* data = sm;
  uint8_t* rowp = sm + static_cast<size_t>(R) * T;
  uint8_t* diag = rowp + T;
  for (uint32_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
    const uint32_t s = t / g.tps;
    const uint64_t off = static_cast<uint64_t>(t - s * g.tps) * T;
    const uint32_t bytes = static_cast<uint32_t>(g.len - off < T ? g.len - off : T);
    const int base = static_cast<int>(s) * g.stride;
    __syncthreads();  // previous tile's smem fully consumed
    for (int c = 0; c < n; ++c) rdp_load(data + static_cast<size_t>(c) * T, tab.p[base + c] + off, bytes, T, g.aligned);
    for (int c = n; c < R; ++c)
      for (uint32_t v = threadIdx.x; v < T / 16; v += blockDim.x)
        reinterpret_cast<uint4*>(data + static_cast<size_t>(c) * T)[v] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    for (uint32_t v16 = threadIdx.x; v16 < T / 16; v16 += blockDim.x) {  // T = rows * 256: 16-B multiple
      uint4 v = make_uint4(0, 0, 0, 0);
      for (int c = 0; c < n; ++c) {
        const uint4 x = reinterpret_cast<const uint4*>(data + static_cast<size_t>(c) * T)[v16];
        v.x ^= x.x;
        v.y ^= x.y;
        v.z ^= x.z;
        v.w ^= x.w;
      }
      reinterpret_cast<uint4*>(rowp)[v16] = v;
    }
    __syncthreads();
    // one dstripe per thread
    const uint64_t abs0 = g.logical0 + off;
    const uint32_t sb = threadIdx.x * R;
    if (sb < bytes) {
      if (abs0 + sb + R <= g.full) {
        uint8_t dv[R];
#pragma unroll
        for (int d = 0; d < R; ++d) {
          uint8_t v = 0;
#pragma unroll
          for (int c = 0; c < R; ++c) {
            const int r = (d - c + P) % P;
            if (r != P - 1) v ^= data[static_cast<size_t>(c) * T + sb + r];
          }
          const int r = (d + 1) % P;  // row-parity column p-1
          if (r != P - 1) v ^= rowp[sb + r];
          dv[d] = v;
        }
#pragma unroll
        for (int d = 0; d < R; ++d) diag[sb + d] = dv[d];
      } else {  // tail bytes (only in the range's last tile): Q parity
        for (uint32_t x = sb; x < bytes && x < sb + R; ++x) {
          uint8_t v = 0;
          for (int c = 0; c < n; ++c) v ^= gf_mul_dev(exp2_of(c), data[static_cast<size_t>(c) * T + x]);
          diag[x] = v;
        }
      }
    }
    __syncthreads();
    rdp_store(const_cast<uint8_t*>(tab.p[base + n]) + off, rowp, bytes, g.aligned);
    rdp_store(const_cast<uint8_t*>(tab.p[base + n + 1]) + off, diag, bytes, g.aligned);
  }
}

// Two-column recovery with the diagonal parity present. Slots per codec
// stripe: data 0..n-1 (NULL if lost), row parity (NULL if lost), diagonal;
// outputs: the lost data columns (ascending). smem: p column tiles (array
// order, lost ones are the outputs being built, virtual ones zero) + diag.
template <int CAP, int P>
__global__ void __launch_bounds__(kRdpThreads) k_rdp_recover(const PtrTable<CAP> tab, const RdpGeom g, int n_out,
                                                             int out0) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int p = P, rows = P - 1;
  constexpr uint32_t T = static_cast<uint32_t>(rows) * kRdpThreads;
  const int n = g.n;
  uint8_t* col = sm;                                   // p tiles
  uint8_t* diag = sm + static_cast<size_t>(p) * T;
  const int i = g.li, j = g.lj;
  for (uint32_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
    const uint32_t s = t / g.tps;
    const uint64_t off = static_cast<uint64_t>(t - s * g.tps) * T;
    const uint32_t bytes = static_cast<uint32_t>(g.len - off < T ? g.len - off : T);
    const int base = static_cast<int>(s) * g.stride;
    __syncthreads();
    for (int c = 0; c < p; ++c) {
      uint8_t* dst = col + static_cast<size_t>(c) * T;
      const uint8_t* src = c < n ? tab.p[base + c] : (c == p - 1 ? tab.p[base + n] : nullptr);
      if (c == i || c == j || src == nullptr) {
        for (uint32_t v = threadIdx.x; v < T / 16; v += blockDim.x)
          reinterpret_cast<uint4*>(dst)[v] = make_uint4(0, 0, 0, 0);
      } else {
        rdp_load(dst, src + off, bytes, T, g.aligned);
      }
    }
    rdp_load(diag, tab.p[base + n + 1] + off, bytes, T, g.aligned);
    __syncthreads();
    const uint64_t abs0 = g.logical0 + off;
    const uint32_t sb = threadIdx.x * rows;
    if (sb < bytes) {
      uint8_t* ci = col + static_cast<size_t>(i) * T + sb;
      uint8_t* cj = col + static_cast<size_t>(j) * T + sb;
      if (abs0 + sb + rows <= g.full) {
        // coding.hpp:384-413: chain (primary i, partner j) then (j, i).
        for (int pass = 0; pass < 2; ++pass) {
          const int prim = pass == 0 ? i : j, part = pass == 0 ? j : i;
          uint8_t* po = pass == 0 ? ci : cj;
          uint8_t* qo = pass == 0 ? cj : ci;
          int d = pmod(part - 1, p);
          const int step = pmod(part - prim, p);
          while (d != p - 1) {
            const int r = pmod(d - prim, p);
            uint8_t v = diag[sb + d];
#pragma unroll
            for (int c = 0; c < p; ++c) {
              if (c == prim) continue;
              const int rc = pmod(d - c, p);
              if (rc != p - 1) v ^= col[static_cast<size_t>(c) * T + sb + rc];
            }
            po[r] = v;
            uint8_t w = 0;
#pragma unroll
            for (int c = 0; c < p; ++c)
              if (c != part) w ^= col[static_cast<size_t>(c) * T + sb + r];
            qo[r] = w;
            d = pmod(d + step, p);
          }
        }
      } else {
        // coding.hpp:415-448: P/Q algebra on the tail bytes.
        for (uint32_t x = sb; x < bytes && x < sb + rows; ++x) {
          uint8_t ps = 0, qs = diag[x];
          for (int c = 0; c < n; ++c) {
            if (c == i || c == j) continue;
            const uint8_t v = col[static_cast<size_t>(c) * T + x];
            ps ^= v;
            qs ^= gf_mul_dev(exp2_of(c), v);
          }
          if (j == p - 1) {
            const uint8_t di = gf_mul_dev(qs, gf_inv(exp2_of(i)));
            ci[x - sb] = di;
            cj[x - sb] = static_cast<uint8_t>(ps ^ di);
          } else {
            ps ^= col[static_cast<size_t>(p - 1) * T + x];
            const uint8_t gi = exp2_of(i), gj = exp2_of(j);
            const uint8_t di = gf_mul_dev(static_cast<uint8_t>(qs ^ gf_mul_dev(gj, ps)), gf_inv(gi ^ gj));
            ci[x - sb] = di;
            cj[x - sb] = static_cast<uint8_t>(ps ^ di);
          }
        }
      }
    }
    __syncthreads();
    int o = 0;
    if (i < n) rdp_store(const_cast<uint8_t*>(tab.p[base + out0 + o++]) + off, col + static_cast<size_t>(i) * T, bytes,
                         g.aligned);
    if (j < n && o < n_out)
      rdp_store(const_cast<uint8_t*>(tab.p[base + out0 + o]) + off, col + static_cast<size_t>(j) * T, bytes,
                g.aligned);
  }
}

}  // namespace gsb

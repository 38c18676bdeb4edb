/*
 * gs_oracle.c -- TEST INFRASTRUCTURE ONLY (see gs_oracle.h).
 *
 * Plain-C restatement of the reference byte path. Every function cites the
 * reference file:line it follows (paths relative to
 * /root/reference/proj/include/ghostserve/). Deliberately scalar and simple:
 * it is the checker, never the thing measured or shipped.
 */
#include "gs_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---- GF(2^8) ------------------------------------------------------------ */

static uint8_t g_exp[512];
static uint8_t g_log[256];
static int g_ready = 0;

/* gf256.hpp:21-34: generator 2, poly 0x11D, exp doubled to 510 (+2 spare). */
static void tables_init(void) {
  if (g_ready) return;
  unsigned x = 1;
  for (unsigned i = 0; i < 255; ++i) {
    g_exp[i] = (uint8_t)x;
    g_exp[i + 255] = (uint8_t)x;
    g_log[x] = (uint8_t)i;
    x <<= 1;
    if (x & 0x100u) x ^= 0x11Du;
  }
  g_exp[510] = g_exp[0];
  g_exp[511] = g_exp[1];
  g_log[0] = 0; /* unused, as in the reference */
  g_ready = 1;
}

void gso_gf_tables(uint8_t exp_out[512], uint8_t log_out[256]) {
  tables_init();
  memcpy(exp_out, g_exp, 512);
  memcpy(log_out, g_log, 256);
}

/* gf256.hpp:42-45 */
uint8_t gso_gf_mul(uint8_t a, uint8_t b) {
  tables_init();
  if (a == 0 || b == 0) return 0;
  return g_exp[(unsigned)g_log[a] + g_log[b]];
}

/* gf256.hpp:47-50 (throws std::domain_error on zero) */
int gso_gf_inv(uint8_t a, uint8_t* out) {
  tables_init();
  if (a == 0) return GSO_DOMAIN_ERROR;
  *out = g_exp[255u - g_log[a]];
  return GSO_OK;
}

/* gf256.hpp:52-56 */
int gso_gf_div(uint8_t a, uint8_t b, uint8_t* out) {
  tables_init();
  if (b == 0) return GSO_DOMAIN_ERROR;
  *out = a == 0 ? 0 : g_exp[(unsigned)g_log[a] + 255u - g_log[b]];
  return GSO_OK;
}

/* gf256.hpp:59-61 */
uint8_t gso_gf_exp2(unsigned e) {
  tables_init();
  return g_exp[e % 255u];
}

/* ---- scheme ------------------------------------------------------------- */

/* coding.hpp:44-60 */
int gso_validate(int kind, int n, int k) {
  if (n < 1 || k < 1 || n + k > 255) return GSO_INVALID_ARGUMENT;
  switch (kind) {
    case GSO_XOR: return k == 1 ? GSO_OK : GSO_INVALID_ARGUMENT;
    case GSO_RDP: return k == 2 ? GSO_OK : GSO_INVALID_ARGUMENT;
    case GSO_RS: return k <= n ? GSO_OK : GSO_INVALID_ARGUMENT;
    default: return GSO_INVALID_ARGUMENT;
  }
}

/* coding.hpp:69-76 */
int gso_max_tolerance(int kind, int k) {
  switch (kind) {
    case GSO_XOR: return 1;
    case GSO_RDP: return 2;
    case GSO_RS: return k;
    default: return 0;
  }
}

/* coding.hpp:96-118: XOR/RDP all ones; RS systematic Cauchy
 * C[i][j] = inv(i ^ (k + j)). */
int gso_encoding_matrix(int kind, int n, int k, uint8_t* coef) {
  int st = gso_validate(kind, n, k);
  if (st) return st;
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < n; ++j) {
      if (kind == GSO_RS) {
        st = gso_gf_inv((uint8_t)(i ^ (k + j)), &coef[i * n + j]);
        if (st) return st;
      } else {
        coef[i * n + j] = 1;
      }
    }
  return GSO_OK;
}

/* coding.hpp:156-172: dst ^= c * src, byte by byte through the product row
 * c * x (gf256.hpp:66-77 keeps the 256x256 table; one row suffices here). */
static void mul_xor(uint8_t* dst, const uint8_t* src, size_t len, uint8_t c) {
  if (c == 0) return;
  uint8_t row[256];
  for (unsigned x = 0; x < 256; ++x) row[x] = gso_gf_mul(c, (uint8_t)x);
  for (size_t b = 0; b < len; ++b) dst[b] ^= row[src[b]];
}

/* ---- RDP (coding.hpp:225-251 layout, :277-307 encode, :343-449 recover) -- */

/* coding.hpp:174-184 */
static int smallest_prime_ge(int x) {
  int v = x < 2 ? 2 : x;
  for (;; ++v) {
    int prime = v >= 2;
    for (int d = 2; d * d <= v; ++d)
      if (v % d == 0) prime = 0;
    if (prime) return v;
  }
}

static int pmod(int a, int p) { return ((a % p) + p) % p; }

/* Array of (p-1) rows x (p+1) columns over the smallest prime p >= n+1:
 * data columns 0..n-1 (n..p-2 virtual zeros), row parity = column p-1,
 * diagonal d = (r + c) mod p stored at row d of the diagonal buffer for
 * d <= p-2. Bytes past the last whole stripe are protected by P (row parity)
 * and Q = sum_c 2^c * data_c. */
static int rdp_encode(int n, const uint8_t* const* data, size_t len, uint8_t* const* parity) {
  const int p = smallest_prime_ge(n + 1), rows = p - 1;
  const size_t full = len / (size_t)rows * (size_t)rows;
  uint8_t* rp = parity[0];
  uint8_t* dp = parity[1];
  memset(rp, 0, len);
  memset(dp, 0, len);
  for (int c = 0; c < n; ++c)
    for (size_t b = 0; b < len; ++b) rp[b] ^= data[c][b];
  for (size_t base = 0; base < full; base += (size_t)rows) {
    for (int c = 0; c < n; ++c)
      for (int r = 0; r < rows; ++r) {
        const int d = (r + c) % p;
        if (d != p - 1) dp[base + (size_t)d] ^= data[c][base + (size_t)r];
      }
    for (int r = 0; r < rows; ++r) {
      const int d = (r + p - 1) % p;
      if (d != p - 1) dp[base + (size_t)d] ^= rp[base + (size_t)r];
    }
  }
  for (int c = 0; c < n; ++c) mul_xor(dp + full, data[c] + full, len - full, gso_gf_exp2((unsigned)c));
  return GSO_OK;
}

/* coding.hpp:343-449: lost_cols are array columns (data c, row parity p-1);
 * col[] holds present columns (NULL otherwise); outputs into outc[c]. */
static void rdp_recover(int n, int p, size_t len, const uint8_t* const* col, const int* lost_cols, int nl,
                        const uint8_t* diag, uint8_t** outc) {
  const int rows = p - 1;
  const size_t full = len / (size_t)rows * (size_t)rows;
  for (int a = 0; a < nl; ++a) memset(outc[lost_cols[a]], 0, len);
  if (nl == 1) { /* :356-371 single column: XOR of the present columns */
    uint8_t* dst = outc[lost_cols[0]];
    for (int c = 0; c < p; ++c)
      if (col[c] && (lost_cols[0] != p - 1 || c != p - 1))
        for (size_t b = 0; b < len; ++b) dst[b] ^= col[c][b];
    return;
  }
  const int i = lost_cols[0] < lost_cols[1] ? lost_cols[0] : lost_cols[1];
  const int j = lost_cols[0] < lost_cols[1] ? lost_cols[1] : lost_cols[0];
  uint8_t* oi = outc[i];
  uint8_t* oj = outc[j];
  for (size_t base = 0; base < full; base += (size_t)rows) {
    /* :384-413: two diagonal-walk chains, each solving its primary column from
     * a stored diagonal, then the partner's cell in that row from the row sum. */
    for (int pass = 0; pass < 2; ++pass) {
      const int prim = pass == 0 ? i : j, part = pass == 0 ? j : i;
      uint8_t* po = pass == 0 ? oi : oj;
      uint8_t* qo = pass == 0 ? oj : oi;
      int d = pmod(part - 1, p);
      const int step = pmod(part - prim, p);
      while (d != p - 1) {
        const int r = pmod(d - prim, p);
        uint8_t v = diag[base + (size_t)d];
        for (int c = 0; c < p; ++c) {
          if (c == prim) continue;
          const int rc = pmod(d - c, p);
          if (rc == p - 1) continue;
          v ^= c == i ? oi[base + (size_t)rc] : c == j ? oj[base + (size_t)rc] : col[c] ? col[c][base + (size_t)rc] : 0;
        }
        po[base + (size_t)r] = v;
        uint8_t w = 0;
        for (int c = 0; c < p; ++c) {
          if (c == part) continue;
          w ^= c == i ? oi[base + (size_t)r] : c == j ? oj[base + (size_t)r] : col[c] ? col[c][base + (size_t)r] : 0;
        }
        qo[base + (size_t)r] = w;
        d = (d + step) % p;
      }
    }
  }
  const size_t tail = len - full; /* :415-448 P/Q algebra on the tail */
  if (!tail) return;
  uint8_t* ps = (uint8_t*)calloc(tail, 1);
  uint8_t* qs = (uint8_t*)calloc(tail, 1);
  for (int c = 0; c < n; ++c) {
    if (c == i || c == j || !col[c]) continue;
    for (size_t b = 0; b < tail; ++b) ps[b] ^= col[c][full + b];
    mul_xor(qs, col[c] + full, tail, gso_gf_exp2((unsigned)c));
  }
  for (size_t b = 0; b < tail; ++b) qs[b] ^= diag[full + b];
  if (j == p - 1) {
    uint8_t ci;
    gso_gf_inv(gso_gf_exp2((unsigned)i), &ci);
    for (size_t b = 0; b < tail; ++b) {
      oi[full + b] = gso_gf_mul(qs[b], ci);
      oj[full + b] = (uint8_t)(ps[b] ^ oi[full + b]);
    }
  } else {
    for (size_t b = 0; b < tail; ++b) ps[b] ^= col[p - 1][full + b];
    const uint8_t gi = gso_gf_exp2((unsigned)i), gj = gso_gf_exp2((unsigned)j);
    uint8_t den;
    gso_gf_inv((uint8_t)(gi ^ gj), &den);
    for (size_t b = 0; b < tail; ++b) {
      const uint8_t di = gso_gf_mul((uint8_t)(qs[b] ^ gso_gf_mul(gj, ps[b])), den);
      oi[full + b] = di;
      oj[full + b] = (uint8_t)(ps[b] ^ di);
    }
  }
  free(ps);
  free(qs);
}

/* coding.hpp:313-336 (+ encode_xor :263-267, encode_rs :269-275, encode_rdp
 * :277-307). */
int gso_encode(int kind, int n, int k, const uint8_t* const* data, size_t len,
               uint8_t* const* parity) {
  int st = gso_validate(kind, n, k);
  if (st) return st;
  if (kind == GSO_RDP) return rdp_encode(n, data, len, parity);
  uint8_t* coef = (uint8_t*)malloc((size_t)k * (size_t)n);
  st = gso_encoding_matrix(kind, n, k, coef);
  if (st) {
    free(coef);
    return st;
  }
  for (int i = 0; i < k; ++i) {
    memset(parity[i], 0, len);
    for (int j = 0; j < n; ++j) mul_xor(parity[i], data[j], len, coef[i * n + j]);
  }
  free(coef);
  return GSO_OK;
}

/* coding.hpp:187-223: Gauss-Jordan over GF(2^8); 0 if singular. */
static int invert(uint8_t* m, int dim, uint8_t* out) {
  memset(out, 0, (size_t)dim * (size_t)dim);
  for (int i = 0; i < dim; ++i) out[i * dim + i] = 1;
  for (int col = 0; col < dim; ++col) {
    int piv = -1;
    for (int r = col; r < dim; ++r)
      if (m[r * dim + col]) {
        piv = r;
        break;
      }
    if (piv < 0) return 0;
    if (piv != col)
      for (int c = 0; c < dim; ++c) {
        uint8_t t = m[piv * dim + c];
        m[piv * dim + c] = m[col * dim + c];
        m[col * dim + c] = t;
        t = out[piv * dim + c];
        out[piv * dim + c] = out[col * dim + c];
        out[col * dim + c] = t;
      }
    uint8_t pinv;
    gso_gf_inv(m[col * dim + col], &pinv);
    for (int c = 0; c < dim; ++c) {
      m[col * dim + c] = gso_gf_mul(m[col * dim + c], pinv);
      out[col * dim + c] = gso_gf_mul(out[col * dim + c], pinv);
    }
    for (int r = 0; r < dim; ++r) {
      if (r == col) continue;
      uint8_t f = m[r * dim + col];
      if (!f) continue;
      for (int c = 0; c < dim; ++c) {
        m[r * dim + c] ^= gso_gf_mul(f, m[col * dim + c]);
        out[r * dim + c] ^= gso_gf_mul(f, out[col * dim + c]);
      }
    }
  }
  return 1;
}

/* ErasurePattern (coding.hpp:131-134): sorted, deduplicated. Returns count. */
static int normalise_lost(const int* lost, int n_lost, int* sorted) {
  int m = 0;
  for (int a = 0; a < n_lost; ++a) {
    int v = lost[a], dup = 0;
    for (int b = 0; b < m; ++b)
      if (sorted[b] == v) dup = 1;
    if (!dup) sorted[m++] = v;
  }
  for (int a = 1; a < m; ++a)
    for (int b = a; b > 0 && sorted[b - 1] > sorted[b]; --b) {
      int t = sorted[b];
      sorted[b] = sorted[b - 1];
      sorted[b - 1] = t;
    }
  return m;
}

static int contains(const int* s, int m, int v) {
  for (int a = 0; a < m; ++a)
    if (s[a] == v) return 1;
  return 0;
}

/* coding.hpp:535-566: rows = first e surviving parity rows; sys[a][b] =
 * C[rows[a]][lost_b]; fold inv(sys) into per-source coefficients. */
int gso_decode_matrix(int kind, int n, int k, const int* lost_in, int n_lost_in,
                      uint8_t* coef_data, uint8_t* coef_par, int* n_lost_data) {
  int st = gso_validate(kind, n, k);
  if (st) return st;
  if (kind == GSO_RDP) return GSO_INVALID_ARGUMENT;
  int* lost = (int*)malloc(sizeof(int) * (size_t)(n_lost_in > 0 ? n_lost_in : 1));
  int m = normalise_lost(lost_in, n_lost_in, lost);
  for (int a = 0; a < m; ++a)
    if (lost[a] < 0 || lost[a] >= n + k) {
      free(lost);
      return GSO_INVALID_ARGUMENT;
    }
  if (m > gso_max_tolerance(kind, k)) {
    free(lost);
    return GSO_UNRECOVERABLE;
  }
  int e = 0;
  int ld[255];
  for (int a = 0; a < m; ++a)
    if (lost[a] < n) ld[e++] = lost[a];
  *n_lost_data = e;
  if (e == 0) {
    free(lost);
    return GSO_OK;
  }
  memset(coef_data, 0, (size_t)e * (size_t)n);
  memset(coef_par, 0, (size_t)e * (size_t)k);
  if (kind == GSO_XOR) { /* coding.hpp:496-502: XOR of every survivor */
    for (int j = 0; j < n; ++j)
      if (!contains(lost, m, j)) coef_data[j] = 1;
    if (!contains(lost, m, n)) coef_par[0] = 1;
    free(lost);
    return GSO_OK;
  }
  uint8_t* C = (uint8_t*)malloc((size_t)k * (size_t)n);
  gso_encoding_matrix(kind, n, k, C);
  int rows[255], nr = 0;
  for (int i = 0; i < k && nr < e; ++i)
    if (!contains(lost, m, n + i)) rows[nr++] = i;
  if (nr < e) {
    free(C);
    free(lost);
    return GSO_UNRECOVERABLE;
  }
  uint8_t* sys = (uint8_t*)malloc((size_t)e * (size_t)e);
  uint8_t* inv = (uint8_t*)malloc((size_t)e * (size_t)e);
  for (int a = 0; a < e; ++a)
    for (int b = 0; b < e; ++b) sys[a * e + b] = C[rows[a] * n + ld[b]];
  if (!invert(sys, e, inv)) {
    free(sys), free(inv), free(C), free(lost);
    return GSO_UNRECOVERABLE;
  }
  for (int b = 0; b < e; ++b) {
    for (int j = 0; j < n; ++j) {
      if (contains(lost, m, j)) continue;
      uint8_t c = 0;
      for (int a = 0; a < e; ++a) c ^= gso_gf_mul(inv[b * e + a], C[rows[a] * n + j]);
      coef_data[b * n + j] = c;
    }
    for (int a = 0; a < e; ++a) coef_par[b * k + rows[a]] = inv[b * e + a];
  }
  free(sys), free(inv), free(C), free(lost);
  return GSO_OK;
}

/* coding.hpp:458-571 (XOR, RDP and RS branches). */
int gso_reconstruct(int kind, int n, int k, const uint8_t* const* shards, const int* lost_in,
                    int n_lost, size_t len, uint8_t* const* out, int* n_out) {
  int st = gso_validate(kind, n, k);
  if (st) return st;
  int lost[255];
  if (n_lost > 255) return GSO_INVALID_ARGUMENT;
  int m = normalise_lost(lost_in, n_lost, lost);
  for (int a = 0; a < m; ++a)
    if (lost[a] < 0 || lost[a] >= n + k) return GSO_INVALID_ARGUMENT; /* :463-465 */
  if (m > gso_max_tolerance(kind, k)) return GSO_UNRECOVERABLE;       /* :466-470 */
  for (int idx = 0; idx < n + k; ++idx)                               /* :474-486 */
    if (!contains(lost, m, idx) && shards[idx] == NULL) return GSO_INVALID_ARGUMENT;
  if (kind == GSO_RDP) { /* coding.hpp:503-534 */
    int ld[2], e = 0;
    for (int a = 0; a < m; ++a)
      if (lost[a] < n) ld[e++] = lost[a];
    *n_out = e;
    if (e == 0) return GSO_OK;
    const int p = smallest_prime_ge(n + 1);
    const uint8_t** col = (const uint8_t**)calloc((size_t)p, sizeof(uint8_t*));
    uint8_t** outc = (uint8_t**)calloc((size_t)p, sizeof(uint8_t*));
    for (int c = 0; c < n; ++c)
      if (!contains(lost, m, c)) col[c] = shards[c];
    if (!contains(lost, m, n)) col[p - 1] = shards[n];
    int lc[3], nl = 0;
    for (int a = 0; a < e; ++a) lc[nl++] = ld[a];
    if (contains(lost, m, n)) lc[nl++] = p - 1;
    uint8_t* scratch = NULL;
    for (int a = 0; a < e; ++a) outc[ld[a]] = out[a];
    if (contains(lost, m, n)) outc[p - 1] = scratch = (uint8_t*)malloc(len ? len : 1);
    rdp_recover(n, p, len, col, lc, nl, contains(lost, m, n + 1) ? NULL : shards[n + 1], outc);
    free(scratch);
    free(col);
    free(outc);
    return GSO_OK;
  }
  uint8_t* cd = (uint8_t*)malloc((size_t)255 * (size_t)n);
  uint8_t* cp = (uint8_t*)malloc((size_t)255 * (size_t)k);
  int e = 0;
  st = gso_decode_matrix(kind, n, k, lost, m, cd, cp, &e);
  if (st) {
    free(cd), free(cp);
    return st;
  }
  *n_out = e;
  for (int b = 0; b < e; ++b) {
    memset(out[b], 0, len);
    for (int j = 0; j < n; ++j) mul_xor(out[b], shards[j], len, cd[b * n + j]);
    for (int i = 0; i < k; ++i) mul_xor(out[b], shards[n + i], len, cp[b * k + i]);
  }
  free(cd), free(cp);
  return GSO_OK;
}

/* ---- KV layout ---------------------------------------------------------- */

/* kv_layout.hpp:21-28 + :40-45 (bytes_per_elem fixed at 2) */
int gso_slice_bytes(int layers, int kv_heads, int head_dim, int tp, uint32_t chunk_size,
                    uint64_t* out) {
  if (layers < 1 || kv_heads < 1 || head_dim < 1 || tp < 1) return GSO_INVALID_ARGUMENT;
  if (((int64_t)kv_heads * head_dim) % tp != 0) return GSO_INVALID_ARGUMENT;
  uint64_t elems = (uint64_t)kv_heads * (uint64_t)head_dim / (uint64_t)tp;
  *out = 2ull * (uint64_t)layers * chunk_size * elems * 2ull;
  return GSO_OK;
}

/* kv_layout.hpp:73-84 */
int gso_pad_partial(uint8_t* bytes, int layers, int kv_heads, int head_dim, int tp,
                    uint32_t chunk_size, uint32_t valid_tokens) {
  if (valid_tokens > chunk_size) return GSO_INVALID_ARGUMENT;
  uint64_t total;
  int st = gso_slice_bytes(layers, kv_heads, head_dim, tp, chunk_size, &total);
  if (st) return st;
  uint64_t stride = (uint64_t)kv_heads * (uint64_t)head_dim / (uint64_t)tp * 2ull;
  uint64_t block = stride * chunk_size, keep = stride * valid_tokens;
  for (uint64_t b = 0; b < 2ull * (uint64_t)layers; ++b)
    memset(bytes + b * block + keep, 0, (size_t)(block - keep));
  return GSO_OK;
}

/* kv_layout.hpp:88-94 */
static uint64_t splitmix_next(uint64_t* s) {
  *s += 0x9E3779B97F4A7C15ull;
  uint64_t z = *s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* kv_layout.hpp:96-103: each argument is bumped by its constant and then fed
 * through one splitmix step (which bumps it again by the golden gamma). */
static uint64_t seed_state(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t s = seed;
  a += 0x9E3779B97F4A7C15ull;
  s ^= splitmix_next(&a);
  b += 0xC2B2AE3D27D4EB4Full;
  s ^= splitmix_next(&b);
  c += 0x165667B19E3779F9ull;
  s ^= splitmix_next(&c);
  return s;
}

/* kv_layout.hpp:110-134: little-endian splitmix words, then pad_partial. */
int gso_make_ground_truth_slice(uint64_t kv_seed, uint64_t request_id, uint32_t chunk,
                                int worker, int layers, int kv_heads, int head_dim, int tp,
                                uint32_t chunk_size, uint32_t valid_tokens, uint8_t* out) {
  uint64_t len;
  int st = gso_slice_bytes(layers, kv_heads, head_dim, tp, chunk_size, &len);
  if (st) return st;
  if (valid_tokens > chunk_size) return GSO_INVALID_ARGUMENT;
  uint64_t s = seed_state(kv_seed, request_id, chunk, (uint64_t)(int64_t)worker);
  uint64_t i = 0;
  for (; i + 8 <= len; i += 8) {
    uint64_t w = splitmix_next(&s);
    for (int b = 0; b < 8; ++b) out[i + b] = (uint8_t)(w >> (8 * b));
  }
  if (i < len) {
    uint64_t w = splitmix_next(&s);
    for (int b = 0; i + b < len; ++b) out[i + b] = (uint8_t)(w >> (8 * b));
  }
  return gso_pad_partial(out, layers, kv_heads, head_dim, tp, chunk_size, valid_tokens);
}

/* ---- parity seal -------------------------------------------------------- */

/* parity_store.hpp:19-25 */
uint64_t gso_fnv1a64(const uint8_t* bytes, size_t len, uint64_t h) {
  for (size_t i = 0; i < len; ++i) {
    h ^= bytes[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* parity_store.hpp:46-50: FNV chained across the k buffers in order. */
uint64_t gso_parity_checksum(const uint8_t* const* parity, int k, size_t len) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (int i = 0; i < k; ++i) h = gso_fnv1a64(parity[i], len, h);
  return h;
}

/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the B200 GCN hot path.
 *
 * A plain-C restatement of the reference algorithms (plexuskit, paths below
 * relative to /root/reference/proj/include/plexuskit/). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg load it, and only
 * as a checker. The product library never links or calls it.
 *
 * Numeric contract: every float op is one IEEE
 * round-to-nearest op in the same order as the reference; the file is built
 * without -march so there is no FMA contraction (the reference is built the
 * same way). Pinned against the reference itself (oracle/_ref) and against
 * tests/golden/ by tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint8_t u8;
typedef uint32_t u32;
typedef uint64_t u64;

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (rng.hpp:17-104)                                            */

typedef struct {
  u32 key[2];
  u32 ctr[4];
  u32 block[4];
  int pos;
} ora_philox;

static void philox_block(const u32 in[4], const u32 key_in[2], u32 out[4]) {
  /* rng.hpp:80-92: 10 rounds, multipliers D2511F53/CD9E8D57, Weyl keys */
  u32 c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
  u32 k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    u64 p0 = (u64)0xD2511F53u * c0;
    u64 p1 = (u64)0xCD9E8D57u * c2;
    u32 hi0 = (u32)(p0 >> 32), lo0 = (u32)p0;
    u32 hi1 = (u32)(p1 >> 32), lo1 = (u32)p1;
    u32 n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0, c1 = n1, c2 = n2, c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0, out[1] = c1, out[2] = c2, out[3] = c3;
}

void ora_philox_init(ora_philox* p, u64 seed, u64 stream) {
  /* rng.hpp:21-23: key = seed halves, counter = (0, 0, stream lo, stream hi) */
  p->key[0] = (u32)seed;
  p->key[1] = (u32)(seed >> 32);
  p->ctr[0] = 0, p->ctr[1] = 0;
  p->ctr[2] = (u32)stream, p->ctr[3] = (u32)(stream >> 32);
  p->pos = 4;
}

static u32 philox_u32(ora_philox* p) {
  /* rng.hpp:25-32, advance_counter 94-98 */
  if (p->pos == 4) {
    philox_block(p->ctr, p->key, p->block);
    for (int i = 0; i < 4; ++i)
      if (++p->ctr[i] != 0) break;
    p->pos = 0;
  }
  return p->block[p->pos++];
}

static u64 philox_u64(ora_philox* p) {
  u64 lo = philox_u32(p);
  u64 hi = philox_u32(p);
  return (hi << 32) | lo;
}

static double philox_double(ora_philox* p) {
  return (double)(philox_u64(p) >> 11) * 0x1.0p-53; /* rng.hpp:41-43 */
}

static u64 philox_randint(ora_philox* p, u64 bound) {
  u64 threshold = (~bound + 1) % bound; /* rng.hpp:47-55 */
  for (;;) {
    u64 r = philox_u64(p);
    if (r >= threshold) return r % bound;
  }
}

void ora_philox_u64(u64 seed, u64 stream, u64 count, u64* out) {
  ora_philox p;
  ora_philox_init(&p, seed, stream);
  for (u64 i = 0; i < count; ++i) out[i] = philox_u64(&p);
}

/* Fisher-Yates (rng.hpp:57-66) */
void ora_permutation(u64 seed, u64 stream, u64 n, u32* out) {
  ora_philox p;
  ora_philox_init(&p, seed, stream);
  for (u64 i = 0; i < n; ++i) out[i] = (u32)i;
  for (u64 i = n; i > 1; --i) {
    u64 j = philox_randint(&p, i);
    u32 t = out[i - 1];
    out[i - 1] = out[j];
    out[j] = t;
  }
}

/* generate_permutation_pair (graph.hpp:84-93): streams 1 and 2 */
void ora_permutation_pair(u64 n, u64 seed, u32* row_perm, u32* col_perm) {
  ora_permutation(seed, 1, n, row_perm);
  ora_permutation(seed, 2, n, col_perm);
}

/* ------------------------------------------------------------------------ */
/* sorting helpers                                                           */

static void radix_sort_u64(u64* keys, u64 n) {
  if (n < 2) return;
  u64* tmp = (u64*)malloc(n * sizeof(u64));
  u64* src = keys;
  u64* dst = tmp;
  for (int shift = 0; shift < 64; shift += 16) {
    u64* cnt = (u64*)calloc(65536 + 1, sizeof(u64));
    for (u64 i = 0; i < n; ++i) cnt[((src[i] >> shift) & 0xFFFF) + 1]++;
    for (int b = 0; b < 65536; ++b) cnt[b + 1] += cnt[b];
    for (u64 i = 0; i < n; ++i) dst[cnt[(src[i] >> shift) & 0xFFFF]++] = src[i];
    free(cnt);
    u64* t = src;
    src = dst;
    dst = t;
  }
  /* 4 passes: result back in `keys` */
  free(tmp);
}

static u64 unique_u64(u64* keys, u64 n) {
  if (n == 0) return 0;
  u64 w = 1;
  for (u64 i = 1; i < n; ++i)
    if (keys[i] != keys[w - 1]) keys[w++] = keys[i];
  return w;
}

/* ------------------------------------------------------------------------ */
/* synthetic RMAT (graph.hpp:291-322) and dataset assembly (197-249)         */

/* Returns the kept edge count; `uv` must hold 2*edges u32. */
u64 ora_rmat_edges(int scale, u64 edges, double a, double b, double c, u64 seed,
                   u32* uv) {
  ora_philox p;
  ora_philox_init(&p, seed, 5);
  u64 kept = 0;
  for (u64 e = 0; e < edges; ++e) {
    u32 u = 0, v = 0;
    for (int bit = 0; bit < scale; ++bit) {
      const double r = philox_double(&p);
      u <<= 1;
      v <<= 1;
      if (r < a) {
      } else if (r < a + b) {
        v |= 1;
      } else if (r < a + b + c) {
        u |= 1;
      } else {
        u |= 1;
        v |= 1;
      }
    }
    if (u != v) {
      uv[2 * kept] = u;
      uv[2 * kept + 1] = v;
      ++kept;
    }
  }
  return kept;
}

/* features: (T)next_double() from stream 3, row-major (graph.hpp:233-236) */
void ora_features_f32(u64 seed, u64 count, float* out) {
  ora_philox p;
  ora_philox_init(&p, seed, 3);
  for (u64 i = 0; i < count; ++i) out[i] = (float)philox_double(&p);
}

/* mask: stream 4 when train_fraction < 1 (graph.hpp:238-246) */
void ora_train_mask(u64 seed, u64 n, double train_fraction, u8* mask) {
  for (u64 i = 0; i < n; ++i) mask[i] = 1;
  if (train_fraction >= 1.0) return;
  ora_philox p;
  ora_philox_init(&p, seed, 4);
  int any = 0;
  for (u64 i = 0; i < n; ++i) {
    mask[i] = philox_double(&p) < train_fraction ? 1 : 0;
    any |= mask[i];
  }
  if (!any) mask[0] = 1;
}

static const u64* g_sort_degree;
static int cmp_deg(const void* x, const void* y) {
  u32 a = *(const u32*)x, b = *(const u32*)y;
  if (g_sort_degree[a] != g_sort_degree[b])
    return g_sort_degree[a] < g_sort_degree[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}

/* degree_quantile_labels (graph.hpp:197-222) */
void ora_degree_quantile_labels(const u32* uv, u64 num_edges, u64 n, u32 classes,
                                u32* labels) {
  u64* keys = (u64*)malloc((2 * num_edges + 1) * sizeof(u64));
  u64 k = 0;
  for (u64 e = 0; e < num_edges; ++e) {
    u32 u = uv[2 * e], v = uv[2 * e + 1];
    if (u == v) continue;
    keys[k++] = ((u64)u << 32) | v;
    keys[k++] = ((u64)v << 32) | u;
  }
  radix_sort_u64(keys, k);
  k = unique_u64(keys, k);
  u64* degree = (u64*)calloc(n, sizeof(u64));
  for (u64 i = 0; i < k; ++i) degree[keys[i] >> 32]++;
  free(keys);
  u32* order = (u32*)malloc(n * sizeof(u32));
  for (u64 i = 0; i < n; ++i) order[i] = (u32)i;
  g_sort_degree = degree;
  qsort(order, n, sizeof(u32), cmp_deg);
  for (u64 pos = 0; pos < n; ++pos) labels[order[pos]] = (u32)(pos * classes / n);
  free(order);
  free(degree);
}

/* ------------------------------------------------------------------------ */
/* normalize_adjacency (graph.hpp:40-76)                                     */

/* Pass 1: returns nnz (call with outputs NULL); pass 2 fills row_ptr (n+1),
 * col_idx and values. Degrees are counted after dedup and self loops; value
 * = (float)(1.0 / sqrt((double)d_u * d_v)). */
u64 ora_normalize_f32(u64 n, const u32* uv, u64 num_edges, int undirected,
                      u64* row_ptr, u32* col_idx, float* values) {
  u64 cap = num_edges * (undirected ? 2 : 1) + n;
  u64* keys = (u64*)malloc(cap * sizeof(u64));
  u64 k = 0;
  for (u64 e = 0; e < num_edges; ++e) {
    u32 u = uv[2 * e], v = uv[2 * e + 1];
    keys[k++] = ((u64)u << 32) | v;
    if (undirected) keys[k++] = ((u64)v << 32) | u;
  }
  for (u64 u = 0; u < n; ++u) keys[k++] = (u << 32) | u;
  radix_sort_u64(keys, k);
  k = unique_u64(keys, k);
  if (row_ptr) {
    u64* degree = (u64*)calloc(n, sizeof(u64));
    for (u64 i = 0; i < k; ++i) degree[keys[i] >> 32]++;
    memset(row_ptr, 0, (n + 1) * sizeof(u64));
    for (u64 i = 0; i < k; ++i) row_ptr[(keys[i] >> 32) + 1]++;
    for (u64 i = 0; i < n; ++i) row_ptr[i + 1] += row_ptr[i];
    for (u64 i = 0; i < k; ++i) {
      u32 u = (u32)(keys[i] >> 32), v = (u32)keys[i];
      col_idx[i] = v;
      values[i] = (float)(1.0 / sqrt((double)degree[u] * (double)degree[v]));
    }
    free(degree);
  }
  free(keys);
  return k;
}

/* ------------------------------------------------------------------------ */
/* CSR ops (csr.hpp:78-120, graph.hpp:101-131)                               */

/* counting-sort transpose (csr.hpp:78-95); out_row_ptr has cols+1 entries */
void ora_csr_transpose_f32(u64 rows, u64 cols, const u64* rp, const u32* ci,
                           const float* v, u64* orp, u32* oci, float* ov) {
  memset(orp, 0, (cols + 1) * sizeof(u64));
  for (u64 k = 0; k < rp[rows]; ++k) orp[ci[k] + 1]++;
  for (u64 i = 0; i < cols; ++i) orp[i + 1] += orp[i];
  u64* fill = (u64*)malloc((cols + 1) * sizeof(u64));
  memcpy(fill, orp, (cols + 1) * sizeof(u64));
  for (u64 i = 0; i < rows; ++i)
    for (u64 k = rp[i]; k < rp[i + 1]; ++k) {
      u64 pos = fill[ci[k]]++;
      oci[pos] = (u32)i;
      ov[pos] = v[k];
    }
  free(fill);
}

/* block extraction (csr.hpp:97-120). Pass 1 (oci NULL) fills orp and returns
 * nnz; pass 2 fills oci/ov. */
u64 ora_csr_block_f32(const u64* rp, const u32* ci, const float* v, u64 r0,
                      u64 r1, u64 c0, u64 c1, u64* orp, u32* oci, float* ov) {
  u64 w = 0;
  orp[0] = 0;
  for (u64 i = r0; i < r1; ++i) {
    for (u64 k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] >= c0 && ci[k] < c1) {
        if (oci) {
          oci[w] = (u32)(ci[k] - c0);
          ov[w] = v[k];
        }
        ++w;
      }
    orp[i - r0 + 1] = w;
  }
  return w;
}

/* permute_csr (graph.hpp:101-131): result[i,j] = a[row_perm[i], col_perm[j]].
 * Keys (inv_r<<32 | inv_c) are unique, so sorting them reproduces the
 * reference's (r,c) order exactly. */
void ora_permute_csr_f32(u64 n, const u64* rp, const u32* ci, const float* v,
                         const u32* row_perm, const u32* col_perm, u64* orp,
                         u32* oci, float* ov) {
  u32* inv_r = (u32*)malloc(n * sizeof(u32));
  u32* inv_c = (u32*)malloc(n * sizeof(u32));
  for (u64 i = 0; i < n; ++i) inv_r[row_perm[i]] = (u32)i, inv_c[col_perm[i]] = (u32)i;
  const u64 nnz = rp[n];
  /* sort (key, value-index) pairs: pack key and original position */
  u64* keys = (u64*)malloc(nnz * sizeof(u64));
  u64* pos = (u64*)malloc(nnz * sizeof(u64));
  u64* tk = (u64*)malloc(nnz * sizeof(u64));
  u64* tp = (u64*)malloc(nnz * sizeof(u64));
  for (u64 i = 0; i < n; ++i)
    for (u64 k = rp[i]; k < rp[i + 1]; ++k) {
      keys[k] = ((u64)inv_r[i] << 32) | inv_c[ci[k]];
      pos[k] = k;
    }
  for (int shift = 0; shift < 64; shift += 16) {
    u64* cnt = (u64*)calloc(65536 + 1, sizeof(u64));
    for (u64 i = 0; i < nnz; ++i) cnt[((keys[i] >> shift) & 0xFFFF) + 1]++;
    for (int b = 0; b < 65536; ++b) cnt[b + 1] += cnt[b];
    for (u64 i = 0; i < nnz; ++i) {
      u64 d = cnt[(keys[i] >> shift) & 0xFFFF]++;
      tk[d] = keys[i];
      tp[d] = pos[i];
    }
    free(cnt);
    u64* t = keys; keys = tk; tk = t;
    t = pos; pos = tp; tp = t;
  }
  memset(orp, 0, (n + 1) * sizeof(u64));
  for (u64 k = 0; k < nnz; ++k) orp[(keys[k] >> 32) + 1]++;
  for (u64 i = 0; i < n; ++i) orp[i + 1] += orp[i];
  for (u64 k = 0; k < nnz; ++k) {
    oci[k] = (u32)keys[k];
    ov[k] = v[pos[k]];
  }
  free(keys), free(pos), free(tk), free(tp), free(inv_r), free(inv_c);
}

/* ------------------------------------------------------------------------ */
/* kernels (kernels.hpp)                                                     */

/* spmm_rows (kernels.hpp:39-62); out is (r1-r0) x d, zero-initialized here */
void ora_spmm_rows_f32(const u64* rp, const u32* ci, const float* v,
                       const float* x, u64 d, u64 r0, u64 r1, float* out) {
  memset(out, 0, (r1 - r0) * d * sizeof(float));
  for (u64 i = r0; i < r1; ++i) {
    float* dst = out + (i - r0) * d;
    for (u64 k = rp[i]; k < rp[i + 1]; ++k) {
      const float a = v[k];
      const float* src = x + (u64)ci[k] * d;
      for (u64 j = 0; j < d; ++j) dst[j] += a * src[j];
    }
  }
}

/* gemm (kernels.hpp:64-92): C(m x n) = op(A) op(B), acc from 0, k ascending.
 * Loop nest reordered for the cache; every C element still accumulates its
 * k terms in ascending order starting from +0 with separate mul and add. */
void ora_gemm_f32(const float* a, u64 ar, u64 ac, const float* b, u64 br, u64 bc,
                  int ta, int tb, float* c) {
  const u64 m = ta ? ac : ar, ka = ta ? ar : ac, n = tb ? br : bc;
  (void)br;
  memset(c, 0, m * n * sizeof(float));
  if (ta && !tb) {
    for (u64 k = 0; k < ka; ++k) {
      const float* arow = a + k * ac;
      const float* brow = b + k * bc;
      for (u64 i = 0; i < m; ++i) {
        const float av = arow[i];
        float* crow = c + i * n;
        for (u64 j = 0; j < n; ++j) crow[j] += av * brow[j];
      }
    }
  } else if (!tb) {
    for (u64 i = 0; i < m; ++i) {
      float* crow = c + i * n;
      for (u64 k = 0; k < ka; ++k) {
        const float av = ta ? a[k * ac + i] : a[i * ac + k];
        const float* brow = b + k * bc;
        for (u64 j = 0; j < n; ++j) crow[j] += av * brow[j];
      }
    }
  } else {
    for (u64 i = 0; i < m; ++i)
      for (u64 j = 0; j < n; ++j) {
        float acc = 0;
        for (u64 k = 0; k < ka; ++k) {
          const float av = ta ? a[k * ac + i] : a[i * ac + k];
          acc += av * b[j * bc + k];
        }
        c[i * n + j] = acc;
      }
  }
}

/* relu (kernels.hpp:94-111) */
void ora_relu_forward_f32(const float* q, u64 n, float* out) {
  for (u64 i = 0; i < n; ++i) out[i] = q[i] > 0.0f ? q[i] : 0.0f;
}
void ora_relu_backward_f32(const float* q, const float* df, u64 n, float* out) {
  for (u64 i = 0; i < n; ++i) out[i] = q[i] > 0.0f ? df[i] : 0.0f;
}

/* softmax_cross_entropy_sums (kernels.hpp:117-158). Returns 0 on success,
 * 1 if a masked-in label is out of range. */
int ora_ce_sums_f32(const float* logits, u64 rows, u64 c, const u32* labels,
                    const u8* mask, double* loss_sum, u64* count, u64* correct,
                    float* dlogits) {
  double ls = 0;
  u64 cnt = 0, cor = 0;
  memset(dlogits, 0, rows * c * sizeof(float));
  for (u64 i = 0; i < rows; ++i) {
    if (!mask[i]) continue;
    if (labels[i] >= c) return 1;
    const float* row = logits + i * c;
    float mx = row[0];
    u64 argmax = 0;
    for (u64 j = 1; j < c; ++j)
      if (row[j] > mx) mx = row[j], argmax = j;
    float denom = 0;
    for (u64 j = 0; j < c; ++j) denom += expf(row[j] - mx);
    ls += (double)(logf(denom) - (row[labels[i]] - mx));
    cnt++;
    if (argmax == labels[i]) cor++;
    float* d = dlogits + i * c;
    for (u64 j = 0; j < c; ++j) d[j] = expf(row[j] - mx) / denom;
    d[labels[i]] -= 1.0f;
  }
  *loss_sum = ls;
  *count = cnt;
  *correct = cor;
  return 0;
}

/* finalize_loss scaling (trainer.hpp:84-87): d *= (T)1/(T)count */
void ora_scale_dlogits_f32(float* d, u64 n, u64 global_count) {
  const float s = 1.0f / (float)global_count;
  for (u64 i = 0; i < n; ++i) d[i] *= s;
}

/* adam_step (model.hpp:88-111); `step` is the count AFTER increment */
void ora_adam_f32(float* p, const float* g, float* m, float* v, u64 n, u64 step,
                  double lr_d, double b1_d, double b2_d, double eps_d) {
  const float b1 = (float)b1_d, b2 = (float)b2_d;
  const float bias1 = (float)(1.0 - pow(b1_d, (double)step));
  const float bias2 = (float)(1.0 - pow(b2_d, (double)step));
  const float lr = (float)lr_d, eps = (float)eps_d;
  for (u64 i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + (1.0f - b1) * g[i];
    v[i] = b2 * v[i] + (1.0f - b2) * g[i] * g[i];
    const float mh = m[i] / bias1;
    const float vh = v[i] / bias2;
    p[i] -= lr * mh / (sqrtf(vh) + eps);
  }
}

/* init_weights (model.hpp:17-33): Philox(seed, 100+l).uniform(-b, b) */
void ora_init_weights_f32(const u64* dims, int ndims, u64 seed, float* out) {
  u64 off = 0;
  for (int l = 0; l + 1 < ndims; ++l) {
    const double bound = sqrt(6.0 / (double)(dims[l] + dims[l + 1]));
    ora_philox p;
    ora_philox_init(&p, seed, 100 + (u64)l);
    const u64 sz = dims[l] * dims[l + 1];
    for (u64 i = 0; i < sz; ++i) {
      const double u = philox_double(&p);
      out[off + i] = (float)(-bound + (bound - -bound) * u);
    }
    off += sz;
  }
}

/* ------------------------------------------------------------------------ */
/* serial forward+backward (trainer.hpp:137-169) on full permuted matrices.  */
/* dims has L+1 entries. a_even/a_odd and their transposes are passed in.   */
/* Outputs: logits n x C, dw concatenated, df0 n x D0; returns 0 or 1 (empty */
/* mask) / 2 (non-finite loss).                                             */
int ora_serial_forward_backward_f32(
    u64 n, const u64* dims, int ndims, const u64* erp, const u32* eci,
    const float* ev, const u64* orp, const u32* oci, const float* ov,
    const u64* etrp, const u32* etci, const float* etv, const u64* otrp,
    const u32* otci, const float* otv, const float* features, const float* w_cat,
    const u32* labels, const u8* mask, double* loss, double* acc, float* logits,
    float* dw_cat, float* df0) {
  const int L = ndims - 1;
  float** h = (float**)calloc(L, sizeof(float*));
  float** q = (float**)calloc(L, sizeof(float*));
  const float** w = (const float**)calloc(L, sizeof(float*));
  u64 off = 0;
  for (int l = 0; l < L; ++l) w[l] = w_cat + off, off += dims[l] * dims[l + 1];
  const float* f = features;
  float* fbuf = NULL;
  for (int l = 0; l < L; ++l) {
    const int odd = l % 2;
    h[l] = (float*)malloc(n * dims[l] * sizeof(float));
    ora_spmm_rows_f32(odd ? orp : erp, odd ? oci : eci, odd ? ov : ev, f, dims[l],
                      0, n, h[l]);
    q[l] = (float*)malloc(n * dims[l + 1] * sizeof(float));
    ora_gemm_f32(h[l], n, dims[l], w[l], dims[l], dims[l + 1], 0, 0, q[l]);
    float* nf = (float*)malloc(n * dims[l + 1] * sizeof(float));
    if (l == L - 1)
      memcpy(nf, q[l], n * dims[l + 1] * sizeof(float));
    else
      ora_relu_forward_f32(q[l], n * dims[l + 1], nf);
    free(fbuf);
    fbuf = nf;
    f = nf;
  }
  const u64 C = dims[L];
  memcpy(logits, f, n * C * sizeof(float));
  double ls;
  u64 cnt, cor;
  float* df = (float*)malloc(n * C * sizeof(float));
  int rc = ora_ce_sums_f32(logits, n, C, labels, mask, &ls, &cnt, &cor, df);
  if (rc == 0 && cnt == 0) rc = 1;
  if (rc == 0) {
    *loss = ls / (double)cnt;
    *acc = (double)cor / (double)cnt;
    if (!isfinite(*loss)) rc = 2;
    ora_scale_dlogits_f32(df, n * C, cnt);
  }
  off = 0;
  u64* dw_off = (u64*)calloc(L, sizeof(u64));
  for (int l = 0; l < L; ++l) dw_off[l] = off, off += dims[l] * dims[l + 1];
  for (int l = L - 1; l >= 0 && rc == 0; --l) {
    const int odd = l % 2;
    float* dq = (float*)malloc(n * dims[l + 1] * sizeof(float));
    if (l == L - 1)
      memcpy(dq, df, n * dims[l + 1] * sizeof(float));
    else
      ora_relu_backward_f32(q[l], df, n * dims[l + 1], dq);
    ora_gemm_f32(h[l], n, dims[l], dq, n, dims[l + 1], 1, 0, dw_cat + dw_off[l]);
    float* dh = (float*)malloc(n * dims[l] * sizeof(float));
    ora_gemm_f32(dq, n, dims[l + 1], w[l], dims[l], dims[l + 1], 0, 1, dh);
    free(df);
    df = (float*)malloc(n * dims[l] * sizeof(float));
    ora_spmm_rows_f32(odd ? otrp : etrp, odd ? otci : etci, odd ? otv : etv, dh,
                      dims[l], 0, n, df);
    free(dq);
    free(dh);
  }
  if (rc == 0) memcpy(df0, df, n * dims[0] * sizeof(float));
  free(df);
  free(fbuf);
  for (int l = 0; l < L; ++l) free(h[l]), free(q[l]);
  free(h), free(q), free(w), free(dw_off);
  return rc;
}

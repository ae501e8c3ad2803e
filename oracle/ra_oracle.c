/* CPU restatement of the RetrievalAttention decode hot path — see ra_oracle.h.
 *
 * TEST INFRASTRUCTURE ONLY (parity checker). Compiled with
 * -ffp-contract=off so every a*b+c below rounds exactly as written; fma()
 * appears exactly where the reference (through Eigen's product/redux
 * kernels, shimmed in oracle/shim/Eigen/Dense) accumulates with FMA.
 * Citations are /root/reference/proj file:line.
 */
#include "ra_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static _Thread_local char g_err[256];
static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return -1;
}
const char* ora_last_error(void) { return g_err; }

/* ---- util.hpp:13-66 ----------------------------------------------------- */
uint64_t ora_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t ora_mix_seed(uint64_t seed, uint64_t a, uint64_t b) {
  uint64_t s = seed;
  uint64_t h = ora_splitmix64(&s);
  s = h ^ (a * 0xD6E8FEB86659FD93ull);
  h = ora_splitmix64(&s);
  s = h ^ (b * 0xCA5A826395121157ull);
  return ora_splitmix64(&s);
}

typedef struct {
  uint64_t state;
  double spare;
  int have_spare;
} rng_t;

static rng_t rng_make(uint64_t seed) {
  rng_t r = {seed, 0.0, 0};
  return r;
}
static double rng_uniform(rng_t* r) {
  return (double)(ora_splitmix64(&r->state) >> 11) * 0x1.0p-53;
}
static uint64_t rng_uniform_index(rng_t* r, uint64_t n) {
  return (uint64_t)(rng_uniform(r) * (double)n) % n;
}
static double rng_normal(rng_t* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = 0.0;
  while (u1 == 0.0) u1 = rng_uniform(r);
  double u2 = rng_uniform(r);
  double rad = sqrt(-2.0 * log(u1));
  double theta = 2.0 * M_PI * u2;
  r->spare = rad * sin(theta);
  r->have_spare = 1;
  return rad * cos(theta);
}

/* ---- ordered (score, id) pairs: index.hpp:95-99 -------------------------- */
typedef struct {
  double s;
  uint32_t id;
} sid_t;

static inline int better(sid_t a, sid_t b) {
  if (a.s != b.s) return a.s > b.s;
  return a.id < b.id;
}
static int cmp_best_first(const void* pa, const void* pb) {
  sid_t a = *(const sid_t*)pa, b = *(const sid_t*)pb;
  if (better(a, b)) return -1;
  if (better(b, a)) return 1;
  return 0;
}

/* binary heap over sid_t; top_is_worst selects TopKCollector (worst on top,
 * index.hpp:58-101) vs. the search frontier (best on top, :367-375) */
typedef struct {
  sid_t* a;
  size_t n, cap;
  int top_is_worst;
} heap_t;

static inline int heap_above(const heap_t* h, sid_t x, sid_t y) {
  return h->top_is_worst ? better(y, x) : better(x, y);
}
static void heap_init(heap_t* h, size_t cap, int top_is_worst) {
  h->cap = cap ? cap : 1;
  h->a = (sid_t*)malloc(h->cap * sizeof(sid_t));
  h->n = 0;
  h->top_is_worst = top_is_worst;
}
static void heap_free(heap_t* h) { free(h->a); }
static void heap_sift_up(heap_t* h, size_t i) {
  while (i > 0) {
    size_t p = (i - 1) / 2;
    if (!heap_above(h, h->a[i], h->a[p])) break;
    sid_t t = h->a[i];
    h->a[i] = h->a[p];
    h->a[p] = t;
    i = p;
  }
}
static void heap_sift_down(heap_t* h, size_t i) {
  for (;;) {
    size_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < h->n && heap_above(h, h->a[l], h->a[m])) m = l;
    if (r < h->n && heap_above(h, h->a[r], h->a[m])) m = r;
    if (m == i) break;
    sid_t t = h->a[i];
    h->a[i] = h->a[m];
    h->a[m] = t;
    i = m;
  }
}
static void heap_push(heap_t* h, sid_t x) {
  if (h->n == h->cap) {
    h->cap *= 2;
    h->a = (sid_t*)realloc(h->a, h->cap * sizeof(sid_t));
  }
  h->a[h->n++] = x;
  heap_sift_up(h, h->n - 1);
}
static sid_t heap_pop(heap_t* h) {
  sid_t top = h->a[0];
  h->a[0] = h->a[--h->n];
  if (h->n) heap_sift_down(h, 0);
  return top;
}

/* TopKCollector::offer (index.hpp:63-77) */
static void topk_offer(heap_t* h, size_t k, uint32_t id, double s) {
  sid_t x = {s, id};
  if (h->n >= k) {
    if (k == 0 || !better(x, h->a[0])) return;
    h->a[0] = x;
    heap_sift_down(h, 0);
    return;
  }
  heap_push(h, x);
}
/* TopKCollector::finish (index.hpp:80-88): best-first */
static void topk_finish(heap_t* h) { qsort(h->a, h->n, sizeof(sid_t), cmp_best_first); }

/* dot_f64 (index_oodgraph.cpp:40-44): exact f32 products, in-order sum */
static inline double dot_f64(const float* a, const float* b, uint32_t d) {
  double acc = 0.0;
  for (uint32_t i = 0; i < d; ++i) acc += (double)a[i] * (double)b[i];
  return acc;
}

/* Mask::contains (index.hpp:22-24) */
static int mask_contains(const uint32_t* m, uint64_t n, uint32_t id) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (m[mid] < id)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < n && m[lo] == id;
}

/* ---- workload.cpp:102-203 (Eigen ops as shimmed: fma chains in order) --- */
/* C[r][N] = A[r][K] * B[K][N], accumulator per output from 0.0 over k */
static void gemm_fma(const double* A, const double* B, double* C, size_t r, size_t K,
                     size_t N) {
  for (size_t i = 0; i < r; ++i) {
    double* c = C + i * N;
    for (size_t j = 0; j < N; ++j) c[j] = 0.0;
    for (size_t k = 0; k < K; ++k) {
      const double aik = A[i * K + k];
      const double* b = B + k * N;
      for (size_t j = 0; j < N; ++j) c[j] = fma(aik, b[j], c[j]);
    }
  }
}

int ora_generate_workload(uint64_t n_ctx, uint32_t d_model, uint32_t d_head,
                          uint32_t n_heads, uint32_t n_kv_groups, uint64_t seed,
                          double ood_strength, double concentration, uint64_t n_decode,
                          float* prefill_q, float* decode_q, float* keys_out,
                          float* values_out) {
  /* WorkloadSpec::validate (workload.cpp:29-44) */
  if (d_model < 1) return fail("WorkloadSpec.d_model must be >= 1");
  if (d_head < 1) return fail("WorkloadSpec.d_head must be >= 1");
  if (d_head > d_model) return fail("WorkloadSpec.d_head must be <= d_model");
  if (n_heads < 1) return fail("WorkloadSpec.n_heads must be >= 1");
  if (n_kv_groups < 1) return fail("WorkloadSpec.n_kv_groups must be >= 1");
  if (n_heads % n_kv_groups != 0)
    return fail("WorkloadSpec.n_heads must be divisible by n_kv_groups");
  if (ood_strength < 0) return fail("WorkloadSpec.ood_strength must be >= 0");
  if (!(concentration > 0)) return fail("WorkloadSpec.concentration must be > 0");

  enum { kMuDir = 1, kHidden = 2, kPerturb = 3, kDecHidden = 4, kDecPerturb = 5,
         kProjBase = 6, kProjKey = 7, kProjValue = 8, kCalib = 9, kProjQuery = 100 };
  const double kMuScale = 2.5, kQueryPerturb = 0.25;
  const uint32_t hpg = n_heads / n_kv_groups;
  const size_t N = (size_t)n_ctx, DM = d_model, DH = d_head, ND = (size_t)n_decode;

  double* scale = malloc(DM * sizeof(double));
  double* mu = malloc(DM * sizeof(double));
  double* h = malloc(N * DM * sizeof(double));
  double* hq = malloc(N * DM * sizeof(double));
  double* hdec = malloc((ND ? ND : 1) * DM * sizeof(double));
  double* w0 = malloc(DM * DH * sizeof(double));
  double* wk = malloc(DM * DH * sizeof(double));
  double* wv = malloc(DM * DH * sizeof(double));
  double* wq = malloc(DM * DH * sizeof(double));
  double* kk = malloc((N ? N : 1) * DH * sizeof(double));
  double* vv = malloc((N ? N : 1) * DH * sizeof(double));
  double* qp = malloc((size_t)hpg * (N ? N : 1) * DH * sizeof(double));
  double* qd = malloc((size_t)hpg * (ND ? ND : 1) * DH * sizeof(double));

  for (uint32_t g = 0; g < n_kv_groups; ++g) {
#define GROUP_RNG(tag) rng_make(ora_mix_seed(seed, (uint64_t)g + 1, (tag)))
    for (size_t j = 0; j < DM; ++j) scale[j] = sqrt(1.0 / (double)(j + 1));
    rng_t r = GROUP_RNG(kMuDir);
    for (size_t j = 0; j < DM; ++j) mu[j] = rng_normal(&r);
    double nn = 0.0;
    for (size_t j = 0; j < DM; ++j) nn = fma(mu[j], mu[j], nn);
    nn = sqrt(nn);
    if (nn > 0)
      for (size_t j = 0; j < DM; ++j) mu[j] /= nn;
    double sn = 0.0;
    for (size_t j = 0; j < DM; ++j) sn = fma(scale[j], scale[j], sn);
    const double mus = kMuScale * sqrt(sn);
    for (size_t j = 0; j < DM; ++j) mu[j] *= mus;

    r = GROUP_RNG(kHidden);
    for (size_t i = 0; i < N; ++i)
      for (size_t j = 0; j < DM; ++j) h[i * DM + j] = mu[j] + rng_normal(&r) * scale[j];
    memcpy(hq, h, N * DM * sizeof(double));
    r = GROUP_RNG(kPerturb);
    for (size_t i = 0; i < N; ++i)
      for (size_t j = 0; j < DM; ++j)
        hq[i * DM + j] += kQueryPerturb * rng_normal(&r) * scale[j];
    r = GROUP_RNG(kDecHidden);
    for (size_t i = 0; i < ND; ++i)
      for (size_t j = 0; j < DM; ++j) hdec[i * DM + j] = mu[j] + rng_normal(&r) * scale[j];
    r = GROUP_RNG(kDecPerturb);
    for (size_t i = 0; i < ND; ++i)
      for (size_t j = 0; j < DM; ++j)
        hdec[i * DM + j] += kQueryPerturb * rng_normal(&r) * scale[j];

    const double proj_scale = 1.0 / sqrt((double)d_model);
    const double s = ood_strength;
    const double mixn = 1.0 / sqrt(1.0 + s * s);
    r = GROUP_RNG(kProjBase);
    for (size_t i = 0; i < DM * DH; ++i) w0[i] = rng_normal(&r) * proj_scale;
    r = GROUP_RNG(kProjKey);
    for (size_t i = 0; i < DM * DH; ++i)
      wk[i] = (w0[i] + s * (rng_normal(&r) * proj_scale)) * mixn;
    r = GROUP_RNG(kProjValue);
    for (size_t i = 0; i < DM * DH; ++i) wv[i] = rng_normal(&r) * proj_scale;
    gemm_fma(h, wk, kk, N, DM, DH);
    gemm_fma(h, wv, vv, N, DM, DH);
    for (uint32_t m = 0; m < hpg; ++m) {
      const uint64_t head = (uint64_t)g * hpg + m;
      rng_t rq = rng_make(ora_mix_seed(seed, n_kv_groups + head + 1, kProjQuery));
      for (size_t i = 0; i < DM * DH; ++i)
        wq[i] = (w0[i] + s * (rng_normal(&rq) * proj_scale)) * mixn;
      gemm_fma(hq, wq, qp + (size_t)m * N * DH, N, DM, DH);
      gemm_fma(hdec, wq, qd + (size_t)m * ND * DH, ND, DM, DH);
    }

    /* joint concentration scaling (workload.cpp:161-185) */
    double c = 1.0;
    if (n_ctx > 0 && n_heads > 0) {
      rng_t cr = GROUP_RNG(kCalib);
      const size_t nqs = N < 256 ? N : 256, nks = N < 8192 ? N : 8192;
      double* qs = malloc(nqs * DH * sizeof(double));
      double* ksT = malloc(DH * nks * sizeof(double));
      double* z = malloc(nqs * nks * sizeof(double));
      for (size_t i = 0; i < nqs; ++i) {
        uint32_t m = (uint32_t)rng_uniform_index(&cr, hpg);
        uint64_t row = rng_uniform_index(&cr, n_ctx);
        memcpy(qs + i * DH, qp + ((size_t)m * N + row) * DH, DH * sizeof(double));
      }
      for (size_t i = 0; i < nks; ++i) {
        uint64_t row = rng_uniform_index(&cr, n_ctx);
        for (size_t j = 0; j < DH; ++j) ksT[j * nks + i] = kk[row * DH + j];
      }
      gemm_fma(qs, ksT, z, nqs, DH, nks);
      const double sq = sqrt((double)d_head);
      double sigma_sum = 0.0;
      for (size_t i = 0; i < nqs; ++i) {
        double* zr = z + i * nks;
        for (size_t j = 0; j < nks; ++j) zr[j] /= sq;
        double sum = 0.0;
        for (size_t j = 0; j < nks; ++j) sum += zr[j];
        const double mean = sum / (double)nks;
        double vs = 0.0;
        for (size_t j = 0; j < nks; ++j) {
          const double t = zr[j] - mean;
          vs += t * t;
        }
        sigma_sum += sqrt(vs / (double)nks);
      }
      const double sigma_raw = sigma_sum / (double)nqs;
      if (sigma_raw > 0) c = sqrt(concentration / sigma_raw);
      free(qs);
      free(ksT);
      free(z);
    }

    for (size_t i = 0; i < N * DH; ++i) {
      keys_out[(size_t)g * N * DH + i] = (float)(kk[i] * c);
      values_out[(size_t)g * N * DH + i] = (float)vv[i];
    }
    for (uint32_t m = 0; m < hpg; ++m) {
      const size_t head = (size_t)g * hpg + m;
      for (size_t i = 0; i < N * DH; ++i)
        prefill_q[head * N * DH + i] = (float)(qp[(size_t)m * N * DH + i] * c);
      for (size_t i = 0; i < ND * DH; ++i)
        decode_q[head * ND * DH + i] = (float)(qd[(size_t)m * ND * DH + i] * c);
    }
#undef GROUP_RNG
  }
  free(scale); free(mu); free(h); free(hq); free(hdec); free(w0); free(wk);
  free(wv); free(wq); free(kk); free(vv); free(qp); free(qd);
  return 0;
}

/* ---- graph build (index_oodgraph.cpp:89-355) ---------------------------- */
void ora_training_knn(const float* keys, uint64_t n, uint32_t d, const float* tq,
                      uint64_t nq, uint32_t kt_req, uint32_t* knn) {
  const uint32_t kt = (uint32_t)(kt_req < n ? kt_req : n);
  heap_t top;
  heap_init(&top, kt + 1, 1);
  for (uint64_t i = 0; i < nq; ++i) {
    top.n = 0;
    const float* q = tq + i * d;
    for (uint64_t id = 0; id < n; ++id) topk_offer(&top, kt, (uint32_t)id, dot_f64(q, keys + id * d, d));
    topk_finish(&top);
    for (uint32_t j = 0; j < top.n; ++j) knn[i * kt + j] = top.a[j].id;
  }
  heap_free(&top);
}

static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}
static size_t unique_u64(uint64_t* v, size_t n) {
  if (!n) return 0;
  size_t w = 1;
  for (size_t i = 1; i < n; ++i)
    if (v[i] != v[w - 1]) v[w++] = v[i];
  return w;
}
static int cmp_pair_asc(const void* pa, const void* pb) {
  /* std::pair<double,uint32_t> operator< */
  sid_t a = *(const sid_t*)pa, b = *(const sid_t*)pb;
  if (a.s < b.s) return -1;
  if (b.s < a.s) return 1;
  return a.id < b.id ? -1 : a.id > b.id;
}

typedef struct {
  uint32_t* v;
  uint32_t n, cap;
} vec32;
static void v32_push(vec32* a, uint32_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? a->cap * 2 : 8;
    a->v = (uint32_t*)realloc(a->v, a->cap * sizeof(uint32_t));
  }
  a->v[a->n++] = x;
}

int ora_graph_build(const float* keys, uint64_t n64, uint32_t d, const float* tq,
                    uint64_t nq, const ora_build_params* p, ora_graph* out) {
  /* ctor validation (index_oodgraph.cpp:71-79) */
  if (n64 == 0) return fail("empty keys");
  if (n64 > 0xFFFFFFFFull) return fail("too many keys");
  if (p->k_train < 1) return fail("k_train must be >= 1");
  if (p->max_degree < 1) return fail("max_degree must be >= 1");
  if (p->ef_construction < 1) return fail("ef_construction must be >= 1");
  const uint32_t n = (uint32_t)n64, M = p->max_degree;
  const int euclid = !p->prune_inner_product;

  double* norms = malloc((size_t)n * sizeof(double));
  for (uint32_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (uint32_t j = 0; j < d; ++j) {
      const double x = keys[(size_t)i * d + j];
      acc = fma(x, x, acc);
    }
    norms[i] = acc;
  }

  /* phase 1 */
  const uint32_t kt = p->k_train < n ? p->k_train : n;
  uint32_t* knn = malloc((nq ? nq : 1) * (size_t)kt * sizeof(uint32_t));
  ora_training_knn(keys, n, d, tq, nq, kt, knn);

  /* phase 2 (:130-156): per 1024-query chunk sort+unique, then global */
  size_t cap = 1024, ne = 0;
  uint64_t* edges = malloc(cap * sizeof(uint64_t));
  for (uint64_t q0 = 0; q0 < nq; q0 += 1024) {
    const uint64_t q1 = nq < q0 + 1024 ? nq : q0 + 1024;
    for (uint64_t qi = q0; qi < q1; ++qi) {
      const uint32_t* row = knn + qi * kt;
      for (uint32_t b = 1; b < kt; ++b) {
        const uint64_t u = row[b];
        const uint32_t lo = (p->edge_window > 0 && b > p->edge_window) ? b - p->edge_window : 0;
        if (ne + b + 2 > cap) {
          cap = cap * 2 + b + 2;
          edges = realloc(edges, cap * sizeof(uint64_t));
        }
        if (lo > 0) edges[ne++] = u << 32 | row[0];
        for (uint32_t a = lo; a < b; ++a) edges[ne++] = u << 32 | row[a];
      }
    }
  }
  qsort(edges, ne, sizeof(uint64_t), cmp_u64);
  ne = unique_u64(edges, ne);
  free(knn);

  size_t* cand_off = calloc((size_t)n + 1, sizeof(size_t));
  for (size_t e = 0; e < ne; ++e) ++cand_off[(edges[e] >> 32) + 1];
  for (uint32_t u = 0; u < n; ++u) cand_off[u + 1] += cand_off[u];

  /* phase 3 (:162-202) */
  vec32* adj = calloc(n, sizeof(vec32));
  sid_t* ordered = NULL;
  size_t ord_cap = 0;
  for (uint32_t u = 0; u < n; ++u) {
    const size_t c0 = cand_off[u], c1 = cand_off[u + 1];
    if (c0 == c1) continue;
    if (c1 - c0 > ord_cap) {
      ord_cap = c1 - c0;
      ordered = realloc(ordered, ord_cap * sizeof(sid_t));
    }
    size_t no = 0;
    for (size_t e = c0; e < c1; ++e) {
      const uint32_t v = (uint32_t)edges[e];
      const double ip = dot_f64(keys + (size_t)u * d, keys + (size_t)v * d, d);
      ordered[no].s = euclid ? norms[u] + norms[v] - 2.0 * ip : -ip;
      ordered[no].id = v;
      ++no;
    }
    qsort(ordered, no, sizeof(sid_t), cmp_pair_asc);
    if (no > p->ef_construction) no = p->ef_construction;
    vec32* kept = &adj[u];
    for (size_t i = 0; i < no; ++i) {
      const double m_uv = ordered[i].s;
      const uint32_t v = ordered[i].id;
      int occluded = 0;
      for (uint32_t j = 0; j < kept->n; ++j) {
        const uint32_t w = kept->v[j];
        const double ip_vw = dot_f64(keys + (size_t)v * d, keys + (size_t)w * d, d);
        const double m_vw = euclid ? norms[v] + norms[w] - 2.0 * ip_vw : -ip_vw;
        if (m_vw < m_uv) {
          occluded = 1;
          break;
        }
      }
      if (!occluded) {
        v32_push(kept, v);
        if (kept->n == M) break;
      }
    }
    if (kept->n < M) {
      for (size_t i = 0; i < no; ++i) {
        if (kept->n == M) break;
        int found = 0;
        for (uint32_t j = 0; j < kept->n; ++j)
          if (kept->v[j] == ordered[i].id) found = 1;
        if (!found) v32_push(kept, ordered[i].id);
      }
    }
  }
  free(ordered);
  free(edges);
  free(cand_off);

  /* entry point (:207-233) */
  uint64_t entry;
  {
    uint32_t* pool = malloc((size_t)n * sizeof(uint32_t));
    uint32_t np = 0;
    for (uint32_t u = 0; u < n; ++u)
      if (adj[u].n) pool[np++] = u;
    if (np == 0) {
      for (uint32_t u = 0; u < n; ++u) pool[u] = u;
      np = n;
    }
    uint32_t best = pool[0];
    if (p->entry_maxnorm) {
      for (uint32_t i = 0; i < np; ++i)
        if (norms[pool[i]] > norms[best]) best = pool[i];
    } else {
      double* mean = calloc(d, sizeof(double));
      for (uint32_t j = 0; j < d; ++j) {
        double acc = 0.0;
        for (uint32_t i = 0; i < n; ++i) acc += (double)keys[(size_t)i * d + j];
        mean[j] = acc / (double)n;
      }
      double best_d = INFINITY;
      for (uint32_t i = 0; i < np; ++i) {
        const uint32_t u = pool[i];
        double acc = 0.0;
        for (uint32_t j = 0; j < d; ++j) {
          const double t = (double)keys[(size_t)u * d + j] - mean[j];
          acc = fma(t, t, acc);
        }
        if (acc < best_d) {
          best_d = acc;
          best = u;
        }
      }
      free(mean);
    }
    entry = best;
    free(pool);
  }

  /* phase 4 repair (:235-348) */
  uint8_t* reached = malloc(n);
  uint32_t* stack = malloc((size_t)n * sizeof(uint32_t));
  uint32_t* pending = malloc((size_t)n * sizeof(uint32_t));
  uint32_t* anchors = malloc(((size_t)n + 1) * sizeof(uint32_t));
  for (;;) {
    memset(reached, 0, n);
    size_t sp = 0;
    stack[sp++] = (uint32_t)entry;
    reached[entry] = 1;
    while (sp) {
      const uint32_t u = stack[--sp];
      for (uint32_t j = 0; j < adj[u].n; ++j) {
        const uint32_t v = adj[u].v[j];
        if (!reached[v]) {
          reached[v] = 1;
          stack[sp++] = v;
        }
      }
    }
    size_t npend = 0, na = 0;
    for (uint32_t u = 0; u < n; ++u)
      if (!reached[u]) pending[npend++] = u;
    if (!npend) break;
    for (uint32_t v = 0; v < n; ++v)
      if (reached[v] && adj[v].n < M) anchors[na++] = v;
    if (!na) {
      /* deepest BFS node, depth ties -> lower id; drop its last edge */
      uint32_t* depth = malloc((size_t)n * sizeof(uint32_t));
      for (uint32_t i = 0; i < n; ++i) depth[i] = 0xFFFFFFFFu;
      size_t qh = 0, qt = 0;
      stack[qt++] = (uint32_t)entry;
      depth[entry] = 0;
      uint32_t deepest = (uint32_t)entry;
      for (; qh < qt; ++qh) {
        const uint32_t u = stack[qh];
        if (depth[u] > depth[deepest] || (depth[u] == depth[deepest] && u < deepest))
          deepest = u;
        for (uint32_t j = 0; j < adj[u].n; ++j) {
          const uint32_t v = adj[u].v[j];
          if (depth[v] == 0xFFFFFFFFu) {
            depth[v] = depth[u] + 1;
            stack[qt++] = v;
          }
        }
      }
      free(depth);
      adj[deepest].n--;
      anchors[na++] = deepest;
    }
    /* nearest anchor: argmin a_norm - 2 u.a, ties -> first (lower) anchor */
    uint64_t* by_anchor = malloc(npend * sizeof(uint64_t));
    for (size_t i = 0; i < npend; ++i) {
      const float* uk = keys + (size_t)pending[i] * d;
      size_t best = 0;
      double best_d = norms[anchors[0]] - 2.0 * dot_f64(uk, keys + (size_t)anchors[0] * d, d);
      for (size_t j = 1; j < na; ++j) {
        const double dist =
            norms[anchors[j]] - 2.0 * dot_f64(uk, keys + (size_t)anchors[j] * d, d);
        if (dist < best_d) {
          best_d = dist;
          best = j;
        }
      }
      by_anchor[i] = (uint64_t)anchors[best] << 32 | pending[i];
    }
    qsort(by_anchor, npend, sizeof(uint64_t), cmp_u64);
    uint32_t* attached = malloc(npend * sizeof(uint32_t));
    size_t g0 = 0;
    while (g0 < npend) {
      size_t g1 = g0;
      while (g1 < npend && (by_anchor[g1] >> 32) == (by_anchor[g0] >> 32)) ++g1;
      uint32_t t = (uint32_t)(by_anchor[g0] >> 32);
      size_t na_t = 0, next_t = 0;
      int deferred = 0;
      for (size_t i = g0; i < g1; ++i) {
        const uint32_t u = (uint32_t)by_anchor[i];
        while (adj[t].n >= M) {
          if (next_t >= na_t) {
            deferred = 1;
            break;
          }
          t = attached[next_t++];
        }
        if (deferred) break;
        v32_push(&adj[t], u);
        attached[na_t++] = u;
        if (adj[u].n < M) t = u;
      }
      g0 = g1;
    }
    free(attached);
    free(by_anchor);
  }
  free(reached);
  free(stack);
  free(pending);
  free(anchors);

  /* CSR (:350-354) */
  out->n = n;
  out->d = d;
  out->max_degree = M;
  out->default_ef = p->default_ef;
  out->entry = entry;
  out->offsets = malloc(((size_t)n + 1) * sizeof(uint64_t));
  out->offsets[0] = 0;
  for (uint32_t u = 0; u < n; ++u) out->offsets[u + 1] = out->offsets[u] + adj[u].n;
  out->adjacency = malloc((out->offsets[n] ? out->offsets[n] : 1) * sizeof(uint32_t));
  for (uint32_t u = 0; u < n; ++u) {
    if (adj[u].n) memcpy(out->adjacency + out->offsets[u], adj[u].v, adj[u].n * sizeof(uint32_t));
    free(adj[u].v);
  }
  free(adj);
  free(norms);
  return 0;
}

void ora_graph_free(ora_graph* g) {
  free(g->offsets);
  free(g->adjacency);
  g->offsets = NULL;
  g->adjacency = NULL;
}

uint64_t ora_graph_serialize(const ora_graph* g, char* buf, uint64_t cap) {
  const uint64_t size = 28 + 4 * g->n + 8 * g->offsets[g->n];
  if (!buf || cap < size) return size;
  char* p = buf;
  const uint32_t ver = 1;
  memcpy(p, "OODG", 4); p += 4;
  memcpy(p, &ver, 4); p += 4;
  memcpy(p, &g->n, 8); p += 8;
  memcpy(p, &g->max_degree, 4); p += 4;
  memcpy(p, &g->entry, 8); p += 8;
  for (uint64_t u = 0; u < g->n; ++u) {
    const uint32_t deg = (uint32_t)(g->offsets[u + 1] - g->offsets[u]);
    memcpy(p, &deg, 4); p += 4;
    for (uint64_t j = g->offsets[u]; j < g->offsets[u + 1]; ++j) {
      const uint64_t v = g->adjacency[j];
      memcpy(p, &v, 8); p += 8;
    }
  }
  return size;
}

int ora_graph_from_blob(uint64_t n_keys, uint32_t d, const char* blob, uint64_t size,
                        ora_graph* out) {
  if (n_keys == 0) return fail("empty keys");
  if (size < 4 || memcmp(blob, "OODG", 4) != 0) return fail("bad graph magic");
  uint64_t pos = 4;
#define READ(T, dst)                                              \
  do {                                                            \
    if (pos + sizeof(T) > size) { ora_graph_free(out); return fail("truncated graph blob"); } \
    memcpy(&(dst), blob + pos, sizeof(T));                        \
    pos += sizeof(T);                                             \
  } while (0)
  out->offsets = NULL;
  out->adjacency = NULL;
  uint32_t ver;
  READ(uint32_t, ver);
  if (ver != 1) return fail("unsupported graph version");
  uint64_t n;
  READ(uint64_t, n);
  if (n != n_keys) return fail("graph/key count mismatch");
  uint32_t M;
  READ(uint32_t, M);
  if (M < 1) return fail("bad degree bound");
  uint64_t entry;
  READ(uint64_t, entry);
  if (entry >= n) return fail("entry point out of range");
  out->n = n;
  out->d = d;
  out->max_degree = M;
  out->default_ef = 128;
  out->entry = entry;
  out->offsets = calloc(n + 1, sizeof(uint64_t));
  size_t cap = 1024;
  out->adjacency = malloc(cap * sizeof(uint32_t));
  for (uint64_t u = 0; u < n; ++u) {
    uint32_t deg;
    READ(uint32_t, deg);
    if (deg > M) { ora_graph_free(out); return fail("degree exceeds bound"); }
    out->offsets[u + 1] = out->offsets[u] + deg;
    if (out->offsets[u + 1] > cap) {
      cap = 2 * out->offsets[u + 1];
      out->adjacency = realloc(out->adjacency, cap * sizeof(uint32_t));
    }
    for (uint32_t j = 0; j < deg; ++j) {
      uint64_t v;
      READ(uint64_t, v);
      if (v >= n) { ora_graph_free(out); return fail("neighbor id out of range"); }
      if (v == u) { ora_graph_free(out); return fail("self loop"); }
      out->adjacency[out->offsets[u] + j] = (uint32_t)v;
    }
  }
#undef READ
  if (pos != size) { ora_graph_free(out); return fail("trailing bytes in graph blob"); }
  return 0;
}

/* ---- OODGraph::search (index_oodgraph.cpp:357-411) ----------------------- */
int ora_graph_search(const ora_graph* g, const float* keys, const float* q, uint64_t k,
                     const uint32_t* mask, uint64_t mask_n, int64_t ef_opt, uint32_t* ids,
                     float* scores, uint64_t* n_out, uint64_t* scanned_out,
                     uint8_t* truncated, uint64_t* expanded) {
  if (k < 1) return fail("k must be >= 1");
  const uint64_t ef = ef_opt >= 0 ? (uint64_t)ef_opt : g->default_ef;
  if (ef < k) return fail("ef must be >= k");
  const uint32_t d = g->d;
  uint8_t* visited = calloc(g->n, 1);
  heap_t frontier, pool;
  heap_init(&frontier, 256, 0);
  heap_init(&pool, ef + 1, 1);
  uint64_t scanned = 0, pops = 0;
  const uint32_t entry = (uint32_t)g->entry;
  visited[entry] = 1;
  const double s0 = dot_f64(q, keys + (size_t)entry * d, d);
  ++scanned;
  sid_t e0 = {s0, entry};
  heap_push(&frontier, e0);
  if (!mask_contains(mask, mask_n, entry)) topk_offer(&pool, ef, entry, s0);
  while (frontier.n) {
    const sid_t top = frontier.a[0];
    if (pool.n >= ef && top.s < pool.a[0].s) break;
    heap_pop(&frontier);
    ++pops;
    for (uint64_t j = g->offsets[top.id]; j < g->offsets[top.id + 1]; ++j) {
      const uint32_t v = g->adjacency[j];
      if (visited[v]) continue;
      visited[v] = 1;
      const double sv = dot_f64(q, keys + (size_t)v * d, d);
      ++scanned;
      sid_t ev = {sv, v};
      heap_push(&frontier, ev);
      if (!mask_contains(mask, mask_n, v)) topk_offer(&pool, ef, v, sv);
    }
  }
  topk_finish(&pool);
  const uint64_t take = k < pool.n ? k : pool.n;
  for (uint64_t i = 0; i < take; ++i) {
    ids[i] = pool.a[i].id;
    scores[i] = (float)pool.a[i].s;
  }
  *n_out = take;
  *scanned_out = scanned;
  *truncated = take < k;
  if (expanded) *expanded = pops;
  heap_free(&frontier);
  heap_free(&pool);
  free(visited);
  return 0;
}

/* ---- FlatIndex::search (index_flat.cpp:22-43) ----------------------------- */
int ora_flat_search(const float* keys, uint64_t n, uint32_t d, const float* q, uint64_t k,
                    const uint32_t* mask, uint64_t mask_n, uint32_t* ids, float* scores,
                    uint64_t* n_out, uint64_t* scanned_out) {
  if (n == 0) return fail("empty keys");
  if (n < mask_n || k < 1 || k > n - mask_n) return fail("k out of range after masking");
  heap_t top;
  heap_init(&top, k + 1, 1);
  uint64_t mp = 0, scanned = 0;
  for (uint64_t id = 0; id < n; ++id) {
    if (mp < mask_n && mask[mp] == id) {
      ++mp;
      continue;
    }
    topk_offer(&top, k, (uint32_t)id, dot_f64(q, keys + id * d, d));
    ++scanned;
  }
  topk_finish(&top);
  for (size_t i = 0; i < top.n; ++i) {
    ids[i] = top.a[i].id;
    scores[i] = (float)top.a[i].s;
  }
  *n_out = top.n;
  *scanned_out = scanned;
  heap_free(&top);
  return 0;
}

/* ---- attention.cpp ------------------------------------------------------- */
int ora_partial_attention(const float* q, const float* keys, const float* values,
                          uint64_t n, uint32_t d, const uint32_t* idx, uint64_t m,
                          double* out, double* zmax_out, double* expsum_out) {
  (void)n;
  if (m == 0) return fail("empty index set");
  const double inv_sqrt_d = 1.0 / sqrt((double)d);
  double* z = malloc(m * sizeof(double));
  double zmax = -INFINITY;
  for (uint64_t i = 0; i < m; ++i) {
    z[i] = dot_f64(q, keys + (size_t)idx[i] * d, d) * inv_sqrt_d;
    if (z[i] > zmax) zmax = z[i];
  }
  for (uint32_t j = 0; j < d; ++j) out[j] = 0.0;
  double expsum = 0.0;
  for (uint64_t i = 0; i < m; ++i) {
    const double e = exp(z[i] - zmax);
    expsum += e;
    const float* v = values + (size_t)idx[i] * d;
    for (uint32_t j = 0; j < d; ++j) out[j] += e * (double)v[j];
  }
  for (uint32_t j = 0; j < d; ++j) out[j] /= expsum;
  *zmax_out = zmax;
  *expsum_out = expsum;
  free(z);
  return 0;
}

int ora_merge(uint32_t d, const double* ow, double zw, double sw, int w_empty,
              const double* oo, double zo, double so, int o_empty, double* out,
              double* gw, double* go) {
  if (w_empty && o_empty) return fail("empty attention support");
  if (w_empty) {
    *gw = 0.0;
    *go = 1.0;
    memcpy(out, oo, d * sizeof(double));
    return 0;
  }
  if (o_empty) {
    *gw = 1.0;
    *go = 0.0;
    memcpy(out, ow, d * sizeof(double));
    return 0;
  }
  const double zref = zw > zo ? zw : zo;
  const double ew = exp(zw - zref) * sw;
  const double eo = exp(zo - zref) * so;
  const double denom = ew + eo;
  *gw = ew / denom;
  *go = eo / denom;
  for (uint32_t j = 0; j < d; ++j) out[j] = *gw * ow[j] + *go * oo[j];
  return 0;
}

int ora_static_partition(uint64_t t, uint64_t s_init, uint64_t s_local,
                         uint32_t* static_ids, uint64_t* n_static, uint32_t* pool_ids,
                         uint64_t* n_pool) {
  if (t > 0xFFFFFFFFull) return fail("context length exceeds id width");
  const uint64_t head_end = s_init < t ? s_init : t;
  uint64_t tail_begin = head_end;
  if (t > s_local) tail_begin = (t - s_local) > head_end ? t - s_local : head_end;
  uint64_t ns = 0, np = 0;
  for (uint64_t i = 0; i < head_end; ++i) {
    if (static_ids) static_ids[ns] = (uint32_t)i;
    ++ns;
  }
  for (uint64_t i = tail_begin; i < t; ++i) {
    if (static_ids) static_ids[ns] = (uint32_t)i;
    ++ns;
  }
  for (uint64_t i = head_end; i < tail_begin; ++i) {
    if (pool_ids) pool_ids[np] = (uint32_t)i;
    ++np;
  }
  *n_static = ns;
  *n_pool = np;
  return 0;
}

int ora_run_head(const ora_graph* g, const float* keys, const float* values, uint64_t t,
                 uint32_t d, const float* q, uint64_t s_init, uint64_t s_local,
                 uint32_t top_k, int64_t ef, double* out, uint32_t* omega,
                 uint64_t* scanned) {
  uint64_t ns, np;
  if (ora_static_partition(t, s_init, s_local, NULL, &ns, NULL, &np)) return -1;
  uint32_t* w = malloc((ns ? ns : 1) * sizeof(uint32_t));
  ora_static_partition(t, s_init, s_local, w, &ns, NULL, &np);
  uint32_t* ids = malloc(((size_t)top_k + 1) * sizeof(uint32_t));
  float* sc = malloc(((size_t)top_k + 1) * sizeof(float));
  uint64_t nr = 0, scn = 0;
  uint8_t tr = 0;
  int rc = 0;
  if (np > 0) {
    const uint64_t k = top_k < np ? top_k : np;
    rc = ora_graph_search(g, keys, q, k, w, ns, ef, ids, sc, &nr, &scn, &tr, NULL);
  }
  double* ow = calloc(d, sizeof(double));
  double* oo = calloc(d, sizeof(double));
  double zw = 0, sw = 0, zo = 0, so = 0;
  if (!rc && ns) rc = ora_partial_attention(q, keys, values, t, d, w, ns, ow, &zw, &sw);
  if (!rc && nr) rc = ora_partial_attention(q, keys, values, t, d, ids, nr, oo, &zo, &so);
  double gw, go;
  if (!rc) rc = ora_merge(d, ow, zw, sw, ns == 0, oo, zo, so, nr == 0, out, &gw, &go);
  for (uint32_t i = 0; i < top_k; ++i) omega[i] = i < nr ? ids[i] : 0xFFFFFFFFu;
  *scanned = scn;
  free(w); free(ids); free(sc); free(ow); free(oo);
  return rc;
}

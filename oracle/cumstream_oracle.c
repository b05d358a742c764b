/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.  Never linked into the product.
 *
 * A plain-C restatement of the reference algorithm for the
 * hot path (sliding-window moment update -> moments-to-cumulants -> norms),
 * written from the reference's behaviour, not copied from it.  Each function
 * cites the reference file:line it restates (paths under
 * /root/reference/proj/).  Floating-point evaluation order is reproduced
 * exactly, including the multiply-adds that GCC contracts into FMA in the
 * reference build (-O3 -std=gnu++20, FMA-capable -march): this file is
 * compiled with -ffp-contract=off and spells every such FMA out with fma(),
 * so its results are bit-identical to the reference and independent of the
 * compiler's own contraction choices.  tests/test_oracle.py pins this port
 * against the reference itself (oracle/_ref) and the committed golden
 * vectors under tests/golden/.
 *
 * Threads (OpenMP) only split work by output element -- the pyramid by
 * leading index like the reference's workers, moms2cums by block -- so
 * every element's arithmetic is the single-threaded sequence.
 *
 * Parity pinned: yes (bitwise against oracle/_ref and tests/golden).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OC_MAX_ORDER 20

static uint64_t binom_u64(int n, int k) {
  if (k < 0 || k > n) return 0;
  if (k > n - k) k = n - k;
  uint64_t r = 1;
  for (int i = 1; i <= k; ++i) r = r * (uint64_t)(n - k + i) / (uint64_t)i;
  return r;
}

/* multiset count C(a+r-1, r): symten.cpp:21 */
static uint64_t multiset_count(int a, int r) { return binom_u64(a + r - 1, r); }

/* ---------------------------------------------------------------------- */
/* Lexicographic multiset ranker: symten.hpp:19-59, symten.cpp:31-75       */

typedef struct {
  int alphabet, order;
  uint64_t count;
  uint64_t* prefix; /* order x (alphabet+1) */
} oc_ranker;

static void ranker_init(oc_ranker* r, int alphabet, int order) {
  r->alphabet = alphabet;
  r->order = order;
  r->count = multiset_count(alphabet, order);
  r->prefix = (uint64_t*)calloc((size_t)order * (alphabet + 1), sizeof(uint64_t));
  for (int rem = 0; rem < order; ++rem) {
    uint64_t acc = 0;
    for (int v = 0; v <= alphabet; ++v) {
      r->prefix[(size_t)rem * (alphabet + 1) + v] = acc;
      if (v < alphabet) acc += multiset_count(alphabet - v, rem);
    }
  }
}

static void ranker_free(oc_ranker* r) { free(r->prefix); }

static uint64_t ranker_rank(const oc_ranker* r, const int* t) {
  uint64_t acc = 0;
  int lo = 0;
  for (int i = 0; i < r->order; ++i) {
    const int rem = r->order - 1 - i;
    acc += r->prefix[(size_t)rem * (r->alphabet + 1) + t[i]] -
           r->prefix[(size_t)rem * (r->alphabet + 1) + lo];
    lo = t[i];
  }
  return acc;
}

/* ---------------------------------------------------------------------- */
/* Block layout: SymTensor ctor, symten.cpp:105-140                         */

typedef struct {
  int order, dim, block, grid;
  size_t nblocks, stored;
  int* index;      /* nblocks x order */
  int* ext;        /* nblocks x order */
  size_t* offset;  /* nblocks */
  size_t* volume;  /* nblocks */
  oc_ranker ranker;
} oc_layout;

static int layout_init(oc_layout* L, int order, int dim, int block) {
  if (order < 1 || order > OC_MAX_ORDER || dim < 1 || block < 1 || block > dim) return 1;
  L->order = order;
  L->dim = dim;
  L->block = block;
  L->grid = (dim + block - 1) / block;
  ranker_init(&L->ranker, L->grid, order);
  L->nblocks = (size_t)L->ranker.count;
  L->index = (int*)malloc(L->nblocks * order * sizeof(int));
  L->ext = (int*)malloc(L->nblocks * order * sizeof(int));
  L->offset = (size_t*)malloc(L->nblocks * sizeof(size_t));
  L->volume = (size_t*)malloc(L->nblocks * sizeof(size_t));
  int j[OC_MAX_ORDER] = {0};
  size_t off = 0;
  for (size_t r = 0;; ++r) {
    size_t vol = 1;
    for (int k = 0; k < order; ++k) {
      const int base = j[k] * block;
      const int e = block < dim - base ? block : dim - base;
      L->index[r * order + k] = j[k];
      L->ext[r * order + k] = e;
      vol *= (size_t)e;
    }
    L->offset[r] = off;
    L->volume[r] = vol;
    off += vol;
    int k = order - 1;
    while (k >= 0 && j[k] == L->grid - 1) --k;
    if (k < 0) break;
    const int v = j[k] + 1;
    for (int l = k; l < order; ++l) j[l] = v;
  }
  L->stored = off;
  return 0;
}

static void layout_free(oc_layout* L) {
  free(L->index);
  free(L->ext);
  free(L->offset);
  free(L->volume);
  ranker_free(&L->ranker);
}

/* SymTensor::at_sorted_unchecked, symten.cpp:171-181 */
static double at_sorted(const oc_layout* L, const double* data, const int* idx) {
  int j[OC_MAX_ORDER];
  for (int k = 0; k < L->order; ++k) j[k] = idx[k] / L->block;
  const size_t r = (size_t)ranker_rank(&L->ranker, j);
  const int* e = L->ext + r * L->order;
  size_t off = 0;
  for (int k = 0; k < L->order; ++k) off = off * (size_t)e[k] + (size_t)(idx[k] - j[k] * L->block);
  return data[L->offset[r] + off];
}

/* block_multiplicity, symten.cpp:227-241 */
static uint64_t block_multiplicity(const int* j, int d) {
  uint64_t num = 1;
  for (int i = 2; i <= d; ++i) num *= (uint64_t)i;
  for (int s = 0; s < d;) {
    int e = s + 1;
    while (e < d && j[e] == j[s]) ++e;
    for (int i = 2; i <= e - s; ++i) num /= (uint64_t)i;
    s = e;
  }
  return num;
}

/* ---------------------------------------------------------------------- */
/* Moment pyramid: moments.cpp:32-151.  One flat canonical array per order,
 * lexicographic.  The descent shares prefix products; the two deepest levels
 * are a contiguous multiply-add (contracted to FMA in the reference). */

static void descend(const double* row, int n, int d, int level, int lo, int hi, double p,
                    double** acc, size_t* pos, int write_all) {
  if (level == d - 2) {
    double* a1 = acc[d - 2];
    double* a2 = acc[d - 1];
    size_t p1 = pos[d - 2], p2 = pos[d - 1];
    for (int i = lo; i < hi; ++i) {
      const double q = p * row[i];
      if (write_all) a1[p1] += q;
      ++p1;
      double* out = a2 + p2;
      const double* src = row + i;
      const int len = n - i;
      for (int k = 0; k < len; ++k) out[k] = fma(q, src[k], out[k]); /* moments.cpp:47 */
      p2 += (size_t)len;
    }
    pos[d - 2] = p1;
    pos[d - 1] = p2;
    return;
  }
  for (int i = lo; i < hi; ++i) {
    const double q = p * row[i];
    if (write_all) acc[level][pos[level]] += q;
    ++pos[level];
    descend(row, n, d, level + 1, i, n, q, acc, pos, write_all);
  }
}

/* accumulate<WriteAll>, moments.cpp:122-151.  Workers split the pyramid by
 * leading index (split_leading, moments.cpp:76-101): each owns every
 * element whose first index is i0 and walks all rows in order, so every
 * element sees exactly the single-worker arithmetic (the split never
 * changes a bit, README.md:69-71). */
static void accumulate(double** acc, int n, int d, const double* x, size_t rows, int write_all) {
  if (d == 1) {
    for (size_t r = 0; r < rows; ++r)
      for (int i = 0; i < n; ++i) acc[0][i] += x[r * (size_t)n + i];
  } else {
#pragma omp parallel for schedule(dynamic, 1)
    for (int i0 = 0; i0 < n; ++i0) {
      size_t start[OC_MAX_ORDER], pos[OC_MAX_ORDER];
      /* tuples of order k+1 with first index < i0 precede i0's */
      for (int k = 0; k < d; ++k)
        start[k] = (size_t)(multiset_count(n, k + 1) - multiset_count(n - i0, k + 1));
      for (size_t r = 0; r < rows; ++r) {
        memcpy(pos, start, sizeof(size_t) * (size_t)d);
        descend(x + r * (size_t)n, n, d, 0, i0, i0 + 1, 1.0, acc, pos, write_all);
      }
    }
  }
  const double inv = 1.0 / (double)rows;
  for (int k = 0; k < d; ++k) {
    if (!acc[k]) continue;
    const size_t cnt = (size_t)multiset_count(n, k + 1);
    for (size_t i = 0; i < cnt; ++i) acc[k][i] *= inv;
  }
}

static double** pyramid_alloc(int n, int d, int all_levels) {
  double** acc = (double**)calloc((size_t)d, sizeof(double*));
  for (int k = 0; k < d; ++k)
    if (all_levels || k >= d - 2) acc[k] = (double*)calloc((size_t)multiset_count(n, k + 1), sizeof(double));
  return acc;
}

static void pyramid_free(double** acc, int d) {
  for (int k = 0; k < d; ++k) free(acc[k]);
  free(acc);
}

/* for_each_entry, moments.cpp:156-191: calls f(off, canonical rank) */
static void sort_small(int* v, int m) {
  for (int k = 1; k < m; ++k) {
    const int x = v[k];
    int j = k - 1;
    while (j >= 0 && v[j] > x) {
      v[j + 1] = v[j];
      --j;
    }
    v[j + 1] = x;
  }
}

static void entry_ranks(const oc_layout* L, const oc_ranker* rk, uint64_t* rank_of_entry) {
  const int d = L->order;
  int o[OC_MAX_ORDER], idx[OC_MAX_ORDER];
  for (size_t r = 0; r < L->nblocks; ++r) {
    const int* j = L->index + r * d;
    const int* e = L->ext + r * d;
    memset(o, 0, sizeof(o));
    for (size_t pos = 0;; ++pos) {
      for (int k = 0; k < d; ++k) idx[k] = j[k] * L->block + o[k];
      sort_small(idx, d);
      rank_of_entry[L->offset[r] + pos] = ranker_rank(rk, idx);
      int k = d - 1;
      while (k >= 0 && o[k] == e[k] - 1) o[k--] = 0;
      if (k < 0) break;
      ++o[k];
    }
  }
}

/* ---------------------------------------------------------------------- */
/* Set partitions: restricted growth strings in lex order, cumulants.cpp:16-59 */

typedef struct {
  int* stream; /* per partition: parts, then per part: len, members */
  size_t len, cap, count;
} oc_packed;

static void packed_push(oc_packed* p, int v) {
  if (p->len == p->cap) {
    p->cap = p->cap ? 2 * p->cap : 256;
    p->stream = (int*)realloc(p->stream, p->cap * sizeof(int));
  }
  p->stream[p->len++] = v;
}

static void rgs_emit(const int* a, int s, int parts, oc_packed* out, int min_parts, int exact) {
  if (exact ? parts != exact : parts < min_parts) return;
  ++out->count;
  if (!exact) packed_push(out, parts);
  for (int q = 0; q < parts; ++q) {
    int len = 0;
    for (int i = 0; i < s; ++i) len += a[i] == q;
    packed_push(out, len);
    for (int i = 0; i < s; ++i)
      if (a[i] == q) packed_push(out, i);
  }
}

static void rgs_walk(int i, int s, int max_label, int* a, oc_packed* out, int min_parts,
                     int exact) {
  if (i == s) {
    rgs_emit(a, s, max_label + 1, out, min_parts, exact);
    return;
  }
  for (int v = 0; v <= max_label + 1 && v < s; ++v) {
    a[i] = v;
    rgs_walk(i + 1, s, v > max_label ? v : max_label, a, out, min_parts, exact);
  }
}

static oc_packed pack_corrections(int s) {
  oc_packed p = {0};
  int a[16] = {0};
  rgs_walk(1, s, 0, a, &p, 2, 0);
  return p;
}

/* correction_sorted, cumulants.cpp:64-82 (no FMA: product then sum) */
static double correction_sorted(const int* index, const oc_packed* pk, oc_layout* const* lay,
                                const double* const* lower) {
  double acc = 0.0;
  const int* p = pk->stream;
  const int* end = p + pk->len;
  int sub[OC_MAX_ORDER];
  while (p < end) {
    const int parts = *p++;
    double prod = 1.0;
    for (int q = 0; q < parts; ++q) {
      const int len = *p++;
      for (int k = 0; k < len; ++k) sub[k] = index[p[k]];
      p += len;
      prod *= at_sorted(lay[len - 1], lower[len - 1], sub);
    }
    acc += prod;
  }
  return acc;
}

/* ====================================================================== */
/* Public oracle API (flat block-storage arrays, one per order)            */

int oc_layout_size(int order, int dim, int block, uint64_t* stored, uint64_t* blocks) {
  oc_layout L;
  if (layout_init(&L, order, dim, block)) return 1;
  *stored = L.stored;
  *blocks = L.nblocks;
  layout_free(&L);
  return 0;
}

/* scatter, moments.cpp:200-212 */
static void scatter(const oc_layout* L, const double* src, double* dst) {
  oc_ranker rk;
  ranker_init(&rk, L->dim, L->order);
  uint64_t* ranks = (uint64_t*)malloc(L->stored * sizeof(uint64_t));
  entry_ranks(L, &rk, ranks);
  for (size_t i = 0; i < L->stored; ++i) dst[i] = src[ranks[i]];
  free(ranks);
  ranker_free(&rk);
}

/* moment_series, moments.cpp:229-243 */
int oc_moment_series(const double* x, size_t rows, size_t cols, int d, int b, double* const* out) {
  if (rows < 1 || cols < 1 || d < 1 || d > OC_MAX_ORDER) return 1;
  const int n = (int)cols;
  double** acc = pyramid_alloc(n, d, 1);
  accumulate(acc, n, d, x, rows, 1);
  for (int s = 1; s <= d; ++s) {
    oc_layout L;
    if (layout_init(&L, s, n, b)) {
      pyramid_free(acc, d);
      return 1;
    }
    scatter(&L, acc[s - 1], out[s - 1]);
    layout_free(&L);
  }
  pyramid_free(acc, d);
  return 0;
}

/* moment_tensor, moments.cpp:218-227 */
int oc_moment_tensor(const double* x, size_t rows, size_t cols, int order, int b, double* out) {
  if (rows < 1 || cols < 1 || order < 1 || order > OC_MAX_ORDER) return 1;
  const int n = (int)cols;
  double** acc = pyramid_alloc(n, order, 0);
  accumulate(acc, n, order, x, rows, 0);
  oc_layout L;
  if (layout_init(&L, order, n, b)) {
    pyramid_free(acc, order);
    return 1;
  }
  scatter(&L, acc[order - 1], out);
  layout_free(&L);
  pyramid_free(acc, order);
  return 0;
}

/* moments_update, moments.cpp:268-301 */
int oc_moments_update(double* const* m, size_t window_len, const double* in, const double* outg,
                      size_t rows, size_t cols, int d, int b) {
  if (rows < 1 || cols < 1 || rows > window_len) return 1;
  const int n = (int)cols;
  double** pin = pyramid_alloc(n, d, 1);
  double** pout = pyramid_alloc(n, d, 1);
  accumulate(pin, n, d, in, rows, 1);
  accumulate(pout, n, d, outg, rows, 1);
  const double c = (double)rows / (double)window_len;
  for (int s = 1; s <= d; ++s) {
    oc_layout L;
    layout_init(&L, s, n, b);
    oc_ranker rk;
    ranker_init(&rk, n, s);
    uint64_t* ranks = (uint64_t*)malloc(L.stored * sizeof(uint64_t));
    entry_ranks(&L, &rk, ranks);
    const double* a = pin[s - 1];
    const double* bb = pout[s - 1];
    double* dst = m[s - 1];
    for (size_t i = 0; i < L.stored; ++i) dst[i] = fma(c, a[ranks[i]] - bb[ranks[i]], dst[i]);
    free(ranks);
    ranker_free(&rk);
    layout_free(&L);
  }
  pyramid_free(pin, d);
  pyramid_free(pout, d);
  return 0;
}

/* moms2cums, cumulants.cpp:128-196 */
int oc_moms2cums(const double* const* m, double* const* c, int n, int d, int b) {
  if (d < 1) return 1;
  oc_layout* lay[OC_MAX_ORDER];
  for (int s = 1; s <= d; ++s) {
    lay[s - 1] = (oc_layout*)malloc(sizeof(oc_layout));
    if (layout_init(lay[s - 1], s, n, b)) return 1;
  }
  memcpy(c[0], m[0], lay[0]->stored * sizeof(double));
  for (int s = 2; s <= d; ++s) {
    const oc_layout* L = lay[s - 1];
    double* data = c[s - 1];
    memcpy(data, m[s - 1], L->stored * sizeof(double));
    oc_packed pk = pack_corrections(s);
#pragma omp parallel for schedule(dynamic, 16)
    for (size_t r = 0; r < L->nblocks; ++r) {
      int o[OC_MAX_ORDER], idx[OC_MAX_ORDER], so[OC_MAX_ORDER];
      const int* jx = L->index + r * s;
      const int* e = L->ext + r * s;
      double* blk = data + L->offset[r];
      memset(o, 0, sizeof(o));
      for (size_t pos = 0;; ++pos) {
        int canonical = 1;
        for (int k = 1; k < s; ++k)
          if (jx[k] == jx[k - 1] && o[k] < o[k - 1]) {
            canonical = 0;
            break;
          }
        if (canonical) {
          for (int k = 0; k < s; ++k) idx[k] = jx[k] * b + o[k];
          blk[pos] -= correction_sorted(idx, &pk, lay, (const double* const*)c);
        } else {
          memcpy(so, o, sizeof(int) * (size_t)s);
          for (int a = 0; a < s;) {
            int bb = a + 1;
            while (bb < s && jx[bb] == jx[a]) ++bb;
            sort_small(so + a, bb - a);
            a = bb;
          }
          size_t src = 0;
          for (int k = 0; k < s; ++k) src = src * (size_t)e[k] + (size_t)so[k];
          blk[pos] = blk[src];
        }
        int k = s - 1;
        while (k >= 0 && o[k] == e[k] - 1) o[k--] = 0;
        if (k < 0) break;
        ++o[k];
      }
    }
    free(pk.stream);
  }
  for (int s = 1; s <= d; ++s) {
    layout_free(lay[s - 1]);
    free(lay[s - 1]);
  }
  return 0;
}

/* knorm, symten.cpp:257-276 */
int oc_knorm(const double* t, int order, int n, int b, double k, double* out) {
  if (!(k >= 1.0)) return 1;
  oc_layout L;
  if (layout_init(&L, order, n, b)) return 1;
  double acc = 0.0;
  for (size_t r = 0; r < L.nblocks; ++r) {
    const double mult = (double)block_multiplicity(L.index + r * order, order);
    const double* v = t + L.offset[r];
    double s = 0.0;
    if (k == 2.0) {
      /* The reference build vectorises this fold in order: 4-wide rounded
       * squares added one by one, then an FMA tail (x86-64-v3 codegen of
       * symten.cpp:266).  AVX-512 builds use 8-wide chunks, so the
       * reference's own last bits depend on -march; tests pin knorm to the
       * v3 build bitwise and to the v4 build within 1e-14. */
      const size_t vol = L.volume[r];
      const size_t nvec = vol >= 4 ? (vol & ~(size_t)3) : 0;
      size_t i = 0;
      for (; i < nvec; ++i) s = s + v[i] * v[i];
      for (; i < vol; ++i) s = fma(v[i], v[i], s);
    } else if (k == 1.0) {
      for (size_t i = 0; i < L.volume[r]; ++i) s += fabs(v[i]);
    } else {
      for (size_t i = 0; i < L.volume[r]; ++i) s += pow(fabs(v[i]), k);
    }
    acc = acc + mult * s; /* not contracted in the reference build */
  }
  layout_free(&L);
  if (k == 2.0) *out = sqrt(acc);
  else if (k == 1.0) *out = acc;
  else *out = pow(acc, 1.0 / k);
  return 0;
}

/* nu, gauge.cpp:35-41 */
int oc_nu(const double* const* c, int n, int d, int b, int order, double* out) {
  if (order < 3 || order > d) return 1;
  double n2, nd;
  oc_knorm(c[1], 2, n, b, 2.0, &n2);
  if (n2 <= 0.0) return 3;
  oc_knorm(c[order - 1], order, n, b, 2.0, &nd);
  *out = nd / pow(n2, 0.5 * (double)order);
  return 0;
}

/* make_window_report, gauge.cpp:142-154, with max_abs_diag_* gauge.cpp:64-94.
 * out: [window, rows, norm_c1, norm_c2, skew|nan, kurt|nan, nu3..nu_d] */
int oc_report(const double* const* c, size_t window_len, int n, int d, int b, uint64_t window,
              double* out) {
  if (d < 2) return 1;
  out[0] = (double)window;
  out[1] = (double)window_len;
  oc_knorm(c[0], 1, n, b, 2.0, &out[2]);
  oc_knorm(c[1], 2, n, b, 2.0, &out[3]);
  out[4] = NAN;
  out[5] = NAN;
  for (int o = 3; o <= d; ++o) {
    const int rc = oc_nu(c, n, d, b, o, &out[6 + o - 3]);
    if (rc) return rc;
  }
  if (d >= 3) {
    oc_layout L2, L3;
    layout_init(&L2, 2, n, b);
    layout_init(&L3, 3, n, b);
    double best = 0.0;
    for (int i = 0; i < n; ++i) {
      const int i2[2] = {i, i}, i3[3] = {i, i, i};
      const double v2 = at_sorted(&L2, c[1], i2);
      if (v2 <= 0.0) return 3;
      const double v = fabs(at_sorted(&L3, c[2], i3)) / pow(v2, 1.5);
      best = v > best ? v : best;
    }
    out[4] = best;
    layout_free(&L3);
    if (d >= 4) {
      oc_layout L4;
      layout_init(&L4, 4, n, b);
      best = 0.0;
      for (int i = 0; i < n; ++i) {
        const int i2[2] = {i, i}, i4[4] = {i, i, i, i};
        const double v2 = at_sorted(&L2, c[1], i2);
        if (v2 <= 0.0) return 3;
        const double v = fabs(at_sorted(&L4, c[3], i4)) / (v2 * v2);
        best = v > best ? v : best;
      }
      out[5] = best;
      layout_free(&L4);
    }
    layout_free(&L2);
  }
  return 0;
}

/* Partitions into exactly sigma parts, packed [len, members...] per part:
 * cumulants.cpp:86-96 */
int oc_partitions(int s, int sigma, int* out, size_t cap, size_t* used, size_t* count) {
  if (s < 1 || s > 16 || sigma < 1 || sigma > s) return 1;
  oc_packed p = {0};
  int a[16] = {0};
  rgs_walk(1, s, 0, a, &p, 0, sigma);
  if (p.len > cap) {
    free(p.stream);
    return 4;
  }
  if (p.len) memcpy(out, p.stream, p.len * sizeof(int));
  *used = p.len;
  *count = p.count;
  free(p.stream);
  return 0;
}

/* Sampled-element oracle: one canonical raw moment element of
 * the window, summed in long double, for configs too large to densify. */
double oc_sample_moment(const double* x, size_t rows, size_t cols, const int* idx, int s) {
  long double acc = 0.0L;
  for (size_t r = 0; r < rows; ++r) {
    long double p = 1.0L;
    for (int k = 0; k < s; ++k) p *= (long double)x[r * cols + idx[k]];
    acc += p;
  }
  return (double)(acc / (long double)rows);
}

/* ---------------------------------------------------------------------- */
/* Exact sampled-element oracle (for configs too large to run
 * the full CPU pipeline).  Unlike oc_sample_moment these reproduce the
 * reference's per-element arithmetic bit for bit, so the GPU's stored values
 * can be checked exactly at full size on a sample of elements. */

/* Means of a tile of canonical elements over rows [r0, r0 + rows): for each
 * element the descent of moments.cpp:40-57 -- prefix product from 1.0 left
 * to right, then at the top order of the pyramid the contracted multiply-add
 * out = fma(q, x[i_s], out) (moments.cpp:47), at every lower order the plain
 * add of the full product (moments.cpp:44,55-57) -- in row order, then the
 * reciprocal scaling of moments.cpp:148-150.  Rows are the outer loop so a
 * tile of elements shares each row's reads. */
#define OC_TILE 256
static void sample_means_exact(const double* x, size_t r0, size_t rows, int n, const int* idx, int s, int top,
                               size_t ne, double* out) {
  double acc[OC_TILE];
  for (size_t e = 0; e < ne; ++e) acc[e] = 0.0;
  for (size_t r = r0; r < r0 + rows; ++r) {
    const double* row = x + r * (size_t)n;
    for (size_t e = 0; e < ne; ++e) {
      const int* ix = idx + e * (size_t)s;
      double q = 1.0;
      if (top && s >= 2) {
        for (int k = 0; k < s - 1; ++k) q = q * row[ix[k]];
        acc[e] = fma(q, row[ix[s - 1]], acc[e]);
      } else {
        for (int k = 0; k < s; ++k) q = q * row[ix[k]];
        acc[e] += q;
      }
    }
  }
  const double inv = 1.0 / (double)rows;
  for (size_t e = 0; e < ne; ++e) out[e] = acc[e] * inv;
}

/* Value of canonical elements idx[count][s] of M_s after prime over rows
 * [0, T) of x (rows in arrival order) and `steps` window updates of p rows
 * (step k: incoming rows [T + k p, T + (k+1) p), outgoing [k p, (k+1) p);
 * stream.cpp:85-108 with resync disabled): moment_series, then
 * M = fma(p/T, a - b, M) per update (moments.cpp:287,297).  top != 0 when
 * s is the series' max_order d. */
int oc_sample_stream_moments(const double* x, int n, size_t T, size_t p, int steps, int s, int top,
                             const int* idx, size_t count, double* out) {
  if (s < 1 || s > OC_MAX_ORDER || p < 1 || p > T) return 1;
  const double c = (double)p / (double)T;
  const long ntiles = (long)((count + OC_TILE - 1) / OC_TILE);
#pragma omp parallel for schedule(dynamic, 1)
  for (long t = 0; t < ntiles; ++t) {
    const size_t e0 = (size_t)t * OC_TILE;
    const size_t ne = count - e0 < OC_TILE ? count - e0 : OC_TILE;
    const int* ix = idx + e0 * (size_t)s;
    double m[OC_TILE], a[OC_TILE], b[OC_TILE];
    sample_means_exact(x, 0, T, n, ix, s, top, ne, m);
    for (int k = 0; k < steps; ++k) {
      sample_means_exact(x, T + (size_t)k * p, p, n, ix, s, top, ne, a);
      sample_means_exact(x, (size_t)k * p, p, n, ix, s, top, ne, b);
      for (size_t e = 0; e < ne; ++e) m[e] = fma(c, a[e] - b[e], m[e]);
    }
    for (size_t e = 0; e < ne; ++e) out[e0 + e] = m[e];
  }
  return 0;
}

/* Stored offsets of sorted element indices idx[count][order] in the block
 * layout (at_sorted_unchecked addressing, symten.cpp:171-181). */
int oc_element_offsets(int order, int n, int b, const int* idx, size_t count, uint64_t* out) {
  oc_layout L;
  if (layout_init(&L, order, n, b)) return 1;
  for (size_t e = 0; e < count; ++e) {
    const int* ix = idx + e * (size_t)order;
    int j[OC_MAX_ORDER];
    for (int k = 0; k < order; ++k) j[k] = ix[k] / b;
    const size_t r = (size_t)ranker_rank(&L.ranker, j);
    const int* ex = L.ext + r * order;
    size_t off = 0;
    for (int k = 0; k < order; ++k) off = off * (size_t)ex[k] + (size_t)(ix[k] - j[k] * b);
    out[e] = (uint64_t)(L.offset[r] + off);
  }
  layout_free(&L);
  return 0;
}

/* C_s at sorted element indices from M_s's values there and the complete
 * lower cumulants C_1..C_{s-1} (block storage): C = M - correction_sorted
 * (cumulants.cpp:64-82,171). */
int oc_sample_cumulants(const double* const* c_lower, int n, int b, int s, const int* idx, const double* m_val,
                        size_t count, double* out) {
  if (s < 2 || s > 16) return 1;
  oc_layout* lay[OC_MAX_ORDER];
  for (int k = 1; k < s; ++k) {
    lay[k - 1] = (oc_layout*)malloc(sizeof(oc_layout));
    if (layout_init(lay[k - 1], k, n, b)) return 1;
  }
  oc_packed pk = pack_corrections(s);
#pragma omp parallel for schedule(static)
  for (size_t e = 0; e < count; ++e)
    out[e] = m_val[e] - correction_sorted(idx + e * (size_t)s, &pk, lay, c_lower);
  free(pk.stream);
  for (int k = 1; k < s; ++k) {
    layout_free(lay[k - 1]);
    free(lay[k - 1]);
  }
  return 0;
}

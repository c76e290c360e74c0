/*
 * TEST INFRASTRUCTURE ONLY — C restatement of the reference CER/CSER path.
 *
 * Not linked into the product library.  Used by tests/ (as the checker for
 * configs too big for the numpy port) and by bench.py's CPU baseline.
 *
 * Encoder: restates lemt formats.py:193-295 —
 *   alphabet  = distinct values ordered by (count desc, value asc), the
 *               background (default: head of that order) moved to / prepended
 *               at position 0                               (formats.py:193-209)
 *   layout    = non-background entries sorted by (row, rank, col)
 *                                                           (formats.py:212-224)
 *   CER       = segments for ranks 1..last present rank per row, empty
 *               padding kept                                (formats.py:227-256)
 *   CSER      = present ranks only, frequency order, omegaI = value position
 *                                                           (formats.py:259-295)
 * Dot: restates the reference's literal loop oracle (tests/reference_kernels.py
 *   144-203): per row, per segment, sequential float64 inner sum, one
 *   multiply by (omega - background), sequential outer sum; then
 *   + background * (sequential sum of x) when the background is non-zero.
 *
 * Values are keyed by their float64 value: -0.0 and +0.0 are one element
 * (np.unique compares, it does not hash bits), every NaN is one element that
 * orders after +inf (np.unique equal_nan / np.sort semantics).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ---- tiny dynamic parallel-for over rows (no OpenMP in this toolchain) ---- */
typedef void (*row_fn)(void *ctx, int64_t r, void *scratch);
typedef struct {
  row_fn fn;
  void *ctx;
  int64_t m, chunk;
  int64_t next;
  size_t scratch_bytes;
} pfor_t;

static void *pfor_worker(void *arg) {
  pfor_t *p = (pfor_t *)arg;
  void *scratch = p->scratch_bytes ? malloc(p->scratch_bytes) : NULL;
  for (;;) {
    int64_t r0 = __atomic_fetch_add(&p->next, p->chunk, __ATOMIC_RELAXED);
    if (r0 >= p->m) break;
    int64_t r1 = r0 + p->chunk < p->m ? r0 + p->chunk : p->m;
    for (int64_t r = r0; r < r1; ++r) p->fn(p->ctx, r, scratch);
  }
  free(scratch);
  return NULL;
}

static int g_threads = 0;
void oracle_set_threads(int t) { g_threads = t; }

static void parallel_rows(int64_t m, int64_t chunk, size_t scratch_bytes, row_fn fn, void *ctx) {
  int t = g_threads > 0 ? g_threads : (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (t < 1) t = 1;
  if (t > 256) t = 256;
  pfor_t p = {fn, ctx, m, chunk > 0 ? chunk : 1, 0, scratch_bytes};
  if (t == 1 || m <= chunk) { pfor_worker(&p); return; }
  pthread_t th[256];
  int i;
  for (i = 0; i < t; ++i) pthread_create(&th[i], NULL, pfor_worker, &p);
  for (i = 0; i < t; ++i) pthread_join(th[i], NULL);
}

typedef struct {
  double value;
  int64_t count;
  int64_t slot;
  int has_pos_zero;
} entry_t;

typedef struct {
  int64_t m, n, k, nnz, seg_cer, seg_cser;
  double *omega_freq;     /* k, frequency order, background first */
  int64_t *to_value_pos;  /* k */
  uint32_t *ranks;        /* m*n */
  int32_t *row_counts;    /* m*k */
} oracle_state;

static uint64_t canon_bits(double v) {
  uint64_t b;
  if (v != v) return 0x7ff8000000000000ull;
  if (v == 0.0) v = 0.0;
  memcpy(&b, &v, 8);
  return b;
}

static uint64_t mix64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

/* total order used by np.sort on float64: NaN last, -0 == +0 */
static int value_cmp(double a, double b) {
  int an = a != a, bn = b != b;
  if (an || bn) return an - bn;
  return (a > b) - (a < b);
}

static int freq_cmp(const void *pa, const void *pb) {
  const entry_t *a = (const entry_t *)pa, *b = (const entry_t *)pb;
  if (a->count != b->count) return a->count > b->count ? -1 : 1;
  return value_cmp(a->value, b->value);
}

static const double *g_sort_vals;
static int idx_value_cmp(const void *pa, const void *pb) {
  int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
  return value_cmp(g_sort_vals[a], g_sort_vals[b]);
}

static double load(const void *w, int is_f32, int64_t i) {
  return is_f32 ? (double)((const float *)w)[i] : ((const double *)w)[i];
}

typedef struct {
  oracle_state *st;
  const void *w;
  int is_f32;
  const uint64_t *keys;
  const int64_t *rank_of_slot;
  int64_t cap;
} rank_ctx;

static void rank_row(void *vctx, int64_t r, void *scratch) {
  rank_ctx *c = (rank_ctx *)vctx;
  oracle_state *st = c->st;
  int64_t n = st->n, k = st->k, j;
  for (j = 0; j < n; ++j) {
    uint64_t key = canon_bits(load(c->w, c->is_f32, r * n + j));
    uint64_t h = mix64(key) & (c->cap - 1);
    while (c->keys[h] != key) h = (h + 1) & (c->cap - 1);
    uint32_t rk = (uint32_t)c->rank_of_slot[h];
    st->ranks[r * n + j] = rk;
    st->row_counts[r * k + rk]++;
  }
}

/* returns NULL on allocation failure; *err = 1 for an empty matrix */
void *oracle_encode_begin(const void *w, int is_f32, int64_t m, int64_t n, int bg_mode,
                          double bg_value, int *err) {
  *err = 0;
  if (m <= 0 || n <= 0) { *err = 1; return NULL; }
  int64_t total = m * n;
  /* hash histogram */
  int64_t cap = 64;
  while (cap < 4 * 1024 && cap < 2 * total) cap <<= 1;
  uint64_t *keys = NULL;
  entry_t *vals = NULL;
  int64_t used = 0;
  int64_t i;
  for (;;) {
    keys = (uint64_t *)malloc(cap * sizeof(uint64_t));
    vals = (entry_t *)calloc(cap, sizeof(entry_t));
    if (!keys || !vals) { free(keys); free(vals); return NULL; }
    memset(keys, 0xff, cap * sizeof(uint64_t)); /* 0xff.. is a NaN pattern canon_bits never returns */
    used = 0;
    int grow = 0;
    for (i = 0; i < total; ++i) {
      double v = load(w, is_f32, i);
      uint64_t key = canon_bits(v);
      uint64_t h = mix64(key) & (cap - 1);
      while (keys[h] != key && keys[h] != ~0ull) h = (h + 1) & (cap - 1);
      if (keys[h] == ~0ull) {
        keys[h] = key;
        memcpy(&vals[h].value, &key, 8);
        if (++used * 2 > cap) { grow = 1; break; }
      }
      vals[h].count++;
      if (v == 0.0 && !signbit(v)) vals[h].has_pos_zero = 1;
    }
    if (!grow) break;
    free(keys); free(vals);
    cap <<= 2;
  }
  entry_t *dist = (entry_t *)malloc((used + 1) * sizeof(entry_t));
  int64_t k0 = 0;
  for (i = 0; i < cap; ++i)
    if (keys[i] != ~0ull) {
      dist[k0] = vals[i];
      dist[k0].slot = i;
      if (dist[k0].value == 0.0) dist[k0].value = dist[k0].has_pos_zero ? 0.0 : -0.0;
      ++k0;
    }
  qsort(dist, k0, sizeof(entry_t), freq_cmp);
  double bg = bg_mode ? bg_value : dist[0].value;
  int64_t pos = -1;
  for (i = 0; i < k0; ++i)
    if (dist[i].value == bg) { pos = i; break; }
  int64_t k = pos >= 0 ? k0 : k0 + 1;
  oracle_state *st = (oracle_state *)calloc(1, sizeof(oracle_state));
  st->m = m; st->n = n; st->k = k;
  st->omega_freq = (double *)malloc(k * sizeof(double));
  st->to_value_pos = (int64_t *)malloc(k * sizeof(int64_t));
  st->omega_freq[0] = bg;
  {
    int64_t o = 1;
    for (i = 0; i < k0; ++i)
      if (i != pos) st->omega_freq[o++] = dist[i].value;
  }
  /* rank of every stored hash key */
  int64_t *rank_of_slot = (int64_t *)malloc(cap * sizeof(int64_t));
  for (i = 0; i < k0; ++i)
    rank_of_slot[dist[i].slot] = pos < 0 ? i + 1 : (i == pos ? 0 : (i < pos ? i + 1 : i));
  /* value-ascending positions for CSER */
  {
    int64_t *idx = (int64_t *)malloc(k * sizeof(int64_t));
    for (i = 0; i < k; ++i) idx[i] = i;
    g_sort_vals = st->omega_freq;
    qsort(idx, k, sizeof(int64_t), idx_value_cmp);
    for (i = 0; i < k; ++i) st->to_value_pos[idx[i]] = i;
    free(idx);
  }
  st->ranks = (uint32_t *)malloc(total * sizeof(uint32_t));
  st->row_counts = (int32_t *)calloc(m * k, sizeof(int32_t));
  int64_t r;
  {
    rank_ctx rc = {st, w, is_f32, keys, rank_of_slot, cap};
    parallel_rows(m, 16, 0, rank_row, &rc);
  }
  int64_t nnz = 0, sc = 0, ss = 0;
  for (r = 0; r < m; ++r) {
    int64_t q, last = 0;
    for (q = 1; q < k; ++q) {
      int32_t cnt = st->row_counts[r * k + q];
      if (cnt) { nnz += cnt; ++ss; last = q; }
    }
    sc += last;
  }
  st->nnz = nnz; st->seg_cer = sc; st->seg_cser = ss;
  free(rank_of_slot); free(dist); free(keys); free(vals);
  return st;
}

void oracle_encode_sizes(void *h, int64_t *out /* k, nnz, seg_cer, seg_cser */) {
  oracle_state *st = (oracle_state *)h;
  out[0] = st->k; out[1] = st->nnz; out[2] = st->seg_cer; out[3] = st->seg_cser;
}

typedef struct {
  oracle_state *st;
  int kind;
  const int64_t *entry_off, *row_ptr;
  int64_t *omega_ptr, *col, *omega_index;
} fill_ctx;

static void fill_row(void *vctx, int64_t r, void *scratch) {
  fill_ctx *f = (fill_ctx *)vctx;
  oracle_state *st = f->st;
  int64_t k = st->k, n = st->n, qq, c;
  int64_t *cursor = (int64_t *)scratch;
  const int32_t *cnt = st->row_counts + r * k;
  int64_t e = f->entry_off[r], s = f->row_ptr[r];
  int64_t last = 0;
  for (qq = 1; qq < k; ++qq) if (cnt[qq]) last = qq;
  for (qq = 1; qq < k; ++qq) {
    cursor[qq] = e;
    e += cnt[qq];
    if (f->kind == 0) {
      if (qq <= last) f->omega_ptr[++s] = e;
    } else if (cnt[qq]) {
      f->omega_index[s] = st->to_value_pos[qq];
      f->omega_ptr[++s] = e;
    }
  }
  const uint32_t *rk = st->ranks + r * n;
  for (c = 0; c < n; ++c)
    if (rk[c]) f->col[cursor[rk[c]]++] = c;
}

/* kind 0 = CER, 1 = CSER.  Outputs are int64 / double; the caller narrows the widths.
   omega: k; col: nnz; omega_ptr: S+1; row_ptr: m+1; omega_index (CSER): S.
   returns mode_index for CSER, 0 for CER. */
int64_t oracle_encode_fill(void *h, int kind, double *omega, int64_t *col, int64_t *omega_ptr,
                           int64_t *row_ptr, int64_t *omega_index) {
  oracle_state *st = (oracle_state *)h;
  int64_t m = st->m, k = st->k, r, q;
  if (kind == 0) {
    for (q = 0; q < k; ++q) omega[q] = st->omega_freq[q];
  } else {
    for (q = 0; q < k; ++q) omega[st->to_value_pos[q]] = st->omega_freq[q];
  }
  /* row offsets */
  int64_t *entry_off = (int64_t *)malloc((m + 1) * sizeof(int64_t));
  entry_off[0] = 0; row_ptr[0] = 0;
  for (r = 0; r < m; ++r) {
    int64_t e = 0, segs = 0, last = 0;
    for (q = 1; q < k; ++q) {
      int32_t cnt = st->row_counts[r * k + q];
      e += cnt;
      if (cnt) { ++segs; last = q; }
    }
    entry_off[r + 1] = entry_off[r] + e;
    row_ptr[r + 1] = row_ptr[r] + (kind == 0 ? last : segs);
  }
  omega_ptr[0] = 0;
  {
    fill_ctx fc = {st, kind, entry_off, row_ptr, omega_ptr, col, omega_index};
    parallel_rows(m, 16, k * sizeof(int64_t), fill_row, &fc);
  }
  free(entry_off);
  return kind == 0 ? 0 : st->to_value_pos[0];
}

void oracle_encode_free(void *h) {
  oracle_state *st = (oracle_state *)h;
  if (!st) return;
  free(st->omega_freq); free(st->to_value_pos); free(st->ranks); free(st->row_counts);
  free(st);
}

/* y (m x B) = A.x (n x B, row-major), float64, the reference loop order.
   seg_value[s] is the shared value of segment s (omega[rank] or omega[omegaI]). */
typedef struct {
  int64_t B;
  const int64_t *row_ptr, *omega_ptr, *col;
  const double *seg_value, *x;
  double background, *y;
} dot_ctx;

static void dot_row(void *vctx, int64_t r, void *scratch) {
  dot_ctx *d = (dot_ctx *)vctx;
  int64_t B = d->B, s, i, b;
  double *inner = (double *)scratch, *acc = inner + B;
  int first_outer = 1;
  for (b = 0; b < B; ++b) acc[b] = 0.0;
  for (s = d->row_ptr[r]; s < d->row_ptr[r + 1]; ++s) {
    int64_t e0 = d->omega_ptr[s], e1 = d->omega_ptr[s + 1];
    if (e1 <= e0) continue;
    const double *x0 = d->x + d->col[e0] * B;
    for (b = 0; b < B; ++b) inner[b] = x0[b];
    for (i = e0 + 1; i < e1; ++i) {
      const double *xr = d->x + d->col[i] * B;
      for (b = 0; b < B; ++b) inner[b] += xr[b];
    }
    double v = d->seg_value[s];
    if (d->background != 0.0) v = v - d->background;
    for (b = 0; b < B; ++b) {
      double t = v * inner[b];
      acc[b] = first_outer ? t : acc[b] + t;
    }
    first_outer = 0;
  }
  for (b = 0; b < B; ++b) d->y[r * B + b] = acc[b];
}

/* y (m x B) = A.x (n x B, row-major), float64, the reference loop order.
   seg_value[s] is the shared value of segment s (omega[rank] or omega[omegaI]). */
void oracle_dot(int64_t m, int64_t n, int64_t B, const int64_t *row_ptr, const int64_t *omega_ptr,
                const int64_t *col, const double *seg_value, double background, const double *x,
                double *y) {
  dot_ctx d = {B, row_ptr, omega_ptr, col, seg_value, x, background, y};
  parallel_rows(m, 4, 2 * B * sizeof(double), dot_row, &d);
  if (background != 0.0) {
    int64_t b, j, r;
    for (b = 0; b < B; ++b) {
      double shared = x[b];
      for (j = 1; j < n; ++j) shared += x[j * B + b];
      double corr = background * shared;
      for (r = 0; r < m; ++r) y[r * B + b] += corr;
    }
  }
}

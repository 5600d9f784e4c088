/*
 * actmap_oracle.c -- CPU restatement of the oMAP reference (TEST INFRASTRUCTURE).
 *
 * See actmap_oracle.h for the pinning story.  Every function cites the
 * reference declaration / SPEC clause it restates.  This file is the parity
 * checker and the CPU baseline; the product never links it.
 */
#include "actmap_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* randomness                                                               */
/* ------------------------------------------------------------------------ */

/* splitmix64 (pin P2). */
uint64_t or_splitmix64(uint64_t *state) {
  uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t or_bounded(uint64_t u, uint64_t n) {
  return (uint64_t)(((unsigned __int128)u * (unsigned __int128)n) >> 64);
}

static int dims_ok(uint32_t w, uint32_t h) {
  return w >= 1 && h >= 1 && w <= OR_MAX_DIM && h <= OR_MAX_DIM;
}

/* ------------------------------------------------------------------------ */
/* generators                                                               */
/* ------------------------------------------------------------------------ */

/* grid.hpp:72-76: exactly round(density*cells) obstacles placed by a seeded
 * shuffle.  Pin: selection sampling (Knuth Algorithm S) driven by splitmix64
 * -- a uniformly random m-subset, one sequential pass. */
int or_random_maze(uint32_t w, uint32_t h, double density, uint64_t seed, uint8_t *occ) {
  if (!dims_ok(w, h)) return OR_EINVAL;
  if (!(density >= 0.0) || !(density < 1.0)) return OR_EINVAL;
  const uint64_t n = (uint64_t)w * h;
  uint64_t m = (uint64_t)llround(density * (double)n);
  if (m > n) m = n;
  uint64_t st = seed, chosen = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t remaining = n - i;
    const uint64_t need = m - chosen;
    uint8_t ob = 0;
    if (need) {
      if (need == remaining) {
        ob = 1;
      } else if (or_bounded(or_splitmix64(&st), remaining) < need) {
        ob = 1;
      }
    }
    occ[i] = ob;
    chosen += ob;
  }
  return OR_OK;
}

/* grid.hpp:65-70: serpentine along the longer axis. */
int or_comb_maze(uint32_t w, uint32_t h, uint8_t *occ) {
  if (w < 2 || h < 2 || w > OR_MAX_DIM || h > OR_MAX_DIM) return OR_EINVAL;
  memset(occ, 0, (size_t)w * h);
  if (w >= h) {
    uint32_t k = 0;
    for (uint32_t r = 1; r < h; r += 2, ++k) {
      memset(occ + (size_t)r * w, 1, w);
      const uint32_t gap = (k % 2 == 0) ? 0 : w - 1;
      occ[(size_t)r * w + gap] = 0;
    }
  } else {
    uint32_t k = 0;
    for (uint32_t c = 1; c < w; c += 2, ++k) {
      for (uint32_t r = 0; r < h; ++r) occ[(size_t)r * w + c] = 1;
      const uint32_t gap = (k % 2 == 0) ? 0 : h - 1;
      occ[(size_t)gap * w + c] = 0;
    }
  }
  return OR_OK;
}

static uint32_t uf_find(uint32_t *p, uint32_t x) {
  while (p[x] != x) {
    p[x] = p[p[x]];
    x = p[x];
  }
  return x;
}

/* C2 generator: randomised Kruskal perfect maze, corridor
 * cells at odd (r,c), one-cell walls; harness only. */
int or_kruskal_maze(uint32_t w, uint32_t h, uint64_t seed, uint8_t *occ) {
  if (!dims_ok(w, h) || w < 3 || h < 3) return OR_EINVAL;
  memset(occ, 1, (size_t)w * h);
  const uint32_t cw = (w - 1) / 2, ch = (h - 1) / 2; /* corridor lattice */
  const uint64_t nc = (uint64_t)cw * ch;
  for (uint32_t i = 0; i < ch; ++i)
    for (uint32_t j = 0; j < cw; ++j) occ[(size_t)(2 * i + 1) * w + (2 * j + 1)] = 0;
  /* edges: id = 2*cell + dir (0 = right, 1 = down) */
  uint64_t ne = 0;
  uint64_t *edges = (uint64_t *)malloc(sizeof(uint64_t) * 2 * nc);
  uint32_t *par = (uint32_t *)malloc(sizeof(uint32_t) * nc);
  if (!edges || !par) {
    free(edges);
    free(par);
    return OR_EINVAL;
  }
  for (uint64_t c = 0; c < nc; ++c) {
    par[c] = (uint32_t)c;
    const uint32_t j = (uint32_t)(c % cw), i = (uint32_t)(c / cw);
    if (j + 1 < cw) edges[ne++] = 2 * c;
    if (i + 1 < ch) edges[ne++] = 2 * c + 1;
  }
  uint64_t st = seed;
  for (uint64_t i = ne; i > 1; --i) { /* Fisher-Yates */
    const uint64_t k = or_bounded(or_splitmix64(&st), i);
    const uint64_t t = edges[i - 1];
    edges[i - 1] = edges[k];
    edges[k] = t;
  }
  for (uint64_t e = 0; e < ne; ++e) {
    const uint64_t c = edges[e] >> 1;
    const int dir = (int)(edges[e] & 1);
    const uint64_t d = dir ? c + cw : c + 1;
    const uint32_t a = uf_find(par, (uint32_t)c), b = uf_find(par, (uint32_t)d);
    if (a == b) continue;
    par[a] = b;
    const uint32_t j = (uint32_t)(c % cw), i = (uint32_t)(c / cw);
    const uint32_t r = 2 * i + 1 + (dir ? 1 : 0), col = 2 * j + 1 + (dir ? 0 : 1);
    occ[(size_t)r * w + col] = 0;
  }
  free(edges);
  free(par);
  return OR_OK;
}

/* C3 generator: city blocks of side U[32,96] separated by
 * streets of width U[3,8]; 10% of blocks are free plazas; 1% single-cell
 * clutter on free cells.  Harness only. */
int or_city_grid(uint32_t w, uint32_t h, uint64_t seed, uint8_t *occ) {
  if (!dims_ok(w, h)) return OR_EINVAL;
  uint64_t st = seed;
  /* 1 = inside a block band along that axis */
  uint8_t *rowb = (uint8_t *)calloc(h, 1), *colb = (uint8_t *)calloc(w, 1);
  uint32_t *rowid = (uint32_t *)calloc(h, sizeof(uint32_t));
  uint32_t *colid = (uint32_t *)calloc(w, sizeof(uint32_t));
  if (!rowb || !colb || !rowid || !colid) {
    free(rowb); free(colb); free(rowid); free(colid);
    return OR_EINVAL;
  }
  uint32_t pos = 0, id = 0;
  pos = (uint32_t)(3 + or_bounded(or_splitmix64(&st), 6));
  while (pos < h) {
    uint32_t b = (uint32_t)(32 + or_bounded(or_splitmix64(&st), 65));
    for (uint32_t r = pos; r < pos + b && r < h; ++r) { rowb[r] = 1; rowid[r] = id; }
    ++id;
    pos += b + (uint32_t)(3 + or_bounded(or_splitmix64(&st), 6));
  }
  const uint32_t nrowblocks = id;
  pos = (uint32_t)(3 + or_bounded(or_splitmix64(&st), 6));
  id = 0;
  while (pos < w) {
    uint32_t b = (uint32_t)(32 + or_bounded(or_splitmix64(&st), 65));
    for (uint32_t c = pos; c < pos + b && c < w; ++c) { colb[c] = 1; colid[c] = id; }
    ++id;
    pos += b + (uint32_t)(3 + or_bounded(or_splitmix64(&st), 6));
  }
  const uint32_t ncolblocks = id;
  const uint64_t plaza_seed = or_splitmix64(&st), clutter_seed = or_splitmix64(&st);
  (void)nrowblocks;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < (int64_t)h; ++r) {
    for (uint32_t c = 0; c < w; ++c) {
      const uint64_t idx = (uint64_t)r * w + c;
      uint8_t ob = 0;
      if (rowb[r] && colb[c]) {
        uint64_t s = plaza_seed ^ ((uint64_t)rowid[r] * ncolblocks + colid[c]) * 0xD1B54A32D192ED03ull;
        ob = or_bounded(or_splitmix64(&s), 100) >= 10; /* 10% plazas */
      }
      if (!ob) {
        uint64_t s = clutter_seed ^ idx * 0x9E3779B97F4A7C15ull;
        ob = or_bounded(or_splitmix64(&s), 100) < 1; /* 1% clutter */
      }
      occ[idx] = ob;
    }
  }
  free(rowb); free(colb); free(rowid); free(colid);
  return OR_OK;
}

int or_sample_free_cells(uint32_t w, uint32_t h, const uint8_t *occ, uint64_t n,
                         uint64_t seed, const uint8_t *exclude, uint32_t *rc_out) {
  if (!dims_ok(w, h)) return OR_EINVAL;
  uint64_t nfree = 0;
  const uint64_t cells = (uint64_t)w * h;
  for (uint64_t i = 0; i < cells; ++i) nfree += (occ[i] == 0 && !(exclude && exclude[i]));
  if (n > nfree) return OR_EINVAL;
  uint64_t st = seed, got = 0, tries = 0;
  while (got < n) {
    const uint32_t r = (uint32_t)or_bounded(or_splitmix64(&st), h);
    const uint32_t c = (uint32_t)or_bounded(or_splitmix64(&st), w);
    const uint64_t i = (uint64_t)r * w + c;
    if (++tries > 1000ull * (n + 16) + cells) return OR_EINVAL;
    if (occ[i] || (exclude && exclude[i])) continue;
    int dup = 0;
    for (uint64_t k = 0; k < got && !dup; ++k) dup = rc_out[2 * k] == r && rc_out[2 * k + 1] == c;
    if (dup) continue;
    rc_out[2 * got] = r;
    rc_out[2 * got + 1] = c;
    ++got;
  }
  return OR_OK;
}

/* grid.hpp:78-90: nonempty, in bounds, free; duplicates collapse (pin P10). */
int or_source_mask(uint32_t w, uint32_t h, const uint8_t *occ, const uint32_t *src_rc,
                   uint64_t n_src, uint8_t *srcmask) {
  if (!dims_ok(w, h) || n_src == 0) return OR_EINVAL;
  memset(srcmask, 0, (size_t)w * h);
  for (uint64_t k = 0; k < n_src; ++k) {
    const uint32_t r = src_rc[2 * k], c = src_rc[2 * k + 1];
    if (r >= h || c >= w) return OR_EINVAL;
    const uint64_t i = (uint64_t)r * w + c;
    if (occ[i]) return OR_EINVAL;
    srcmask[i] = 1;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* propagation                                                              */
/* ------------------------------------------------------------------------ */

/* activity.hpp:20-21: 1 at each source, 0 elsewhere. */
int or_initial(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask, uint32_t *out) {
  (void)occ;
  const uint64_t n = (uint64_t)w * h;
  for (uint64_t i = 0; i < n; ++i) out[i] = srcmask[i] ? 1u : 0u;
  return OR_OK;
}

static inline uint32_t max3u(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t m = a > b ? a : b;
  return m > c ? m : c;
}

/* propagate.hpp:34-38: out(c) = 0 at obstacles, else the
 * 3x3 max (out-of-bounds = 0) plus 1 at sources.  uint32
 * arithmetic.  Rows are independent given the input (double buffer,
 * SPEC.md:164), so any thread count gives the same result. */
int or_propagate_layer(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                       const uint32_t *in, uint32_t *out, int threads) {
  if (!dims_ok(w, h)) return OR_EINVAL;
  if (threads < 1) threads = 1;
#pragma omp parallel num_threads(threads)
  {
    uint32_t *v = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)w + 2));
#pragma omp for schedule(static)
    for (int64_t r = 0; r < (int64_t)h; ++r) {
      const uint32_t *mid = in + (size_t)r * w;
      const uint32_t *up = r > 0 ? mid - w : NULL;
      const uint32_t *dn = r + 1 < (int64_t)h ? mid + w : NULL;
      v[0] = 0;
      v[w + 1] = 0;
      if (up && dn) {
        for (uint32_t c = 0; c < w; ++c) v[c + 1] = max3u(up[c], mid[c], dn[c]);
      } else {
        for (uint32_t c = 0; c < w; ++c) {
          uint32_t m = mid[c];
          if (up && up[c] > m) m = up[c];
          if (dn && dn[c] > m) m = dn[c];
          v[c + 1] = m;
        }
      }
      const uint8_t *o = occ + (size_t)r * w;
      const uint8_t *s = srcmask + (size_t)r * w;
      uint32_t *dst = out + (size_t)r * w;
      for (uint32_t c = 0; c < w; ++c) {
        const uint32_t m = max3u(v[c], v[c + 1], v[c + 2]) + (uint32_t)(s[c] != 0);
        dst[c] = o[c] ? 0u : m;
      }
    }
    free(v);
  }
  return OR_OK;
}

/* propagate.hpp:40-43: L >= 1 applications from initial().
 * Batched runs an internal buffer pair; iterative hands a fresh buffer to
 * each layer call.  Outputs are identical by construction. */
int or_propagate(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                 uint32_t layers, int mode, int threads, uint32_t *out) {
  if (!dims_ok(w, h) || layers == 0 || layers > OR_MAX_LAYERS) return OR_EINVAL;
  const size_t n = (size_t)w * h;
  if (mode == OR_MODE_ITERATIVE) {
    uint32_t *cur = (uint32_t *)malloc(n * 4);
    or_initial(w, h, occ, srcmask, cur);
    for (uint32_t l = 0; l < layers; ++l) {
      uint32_t *fresh = (uint32_t *)malloc(n * 4);
      or_propagate_layer(w, h, occ, srcmask, cur, fresh, threads);
      free(cur);
      cur = fresh;
    }
    memcpy(out, cur, n * 4);
    free(cur);
    return OR_OK;
  }
  uint32_t *tmp = (uint32_t *)malloc(n * 4);
  uint32_t *a = (layers % 2 == 0) ? out : tmp; /* final write lands in out */
  uint32_t *b = (layers % 2 == 0) ? tmp : out;
  or_initial(w, h, occ, srcmask, a);
  for (uint32_t l = 0; l < layers; ++l) {
    or_propagate_layer(w, h, occ, srcmask, a, b, threads);
    uint32_t *t = a;
    a = b;
    b = t;
  }
  free(tmp);
  return OR_OK;
}

uint64_t or_zero_free_cells(uint32_t w, uint32_t h, const uint8_t *occ, const uint32_t *vals) {
  const int64_t n = (int64_t)w * h;
  uint64_t z = 0;
#pragma omp parallel for reduction(+ : z) schedule(static)
  for (int64_t i = 0; i < n; ++i) z += (occ[i] == 0 && vals[i] == 0);
  return z;
}

/* propagate.hpp:45-61, pin P3: apply >= 1 layer; after
 * layer l: z_l == 0 -> Filled(l); z_l == z_{l-1} -> Stalled(l); l == cap ->
 * CapReached.  Literal per-layer zero-set count (the GPU path uses a
 * different, cheaper signal; the tests compare the two). */
int or_propagate_auto(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                      uint32_t auto_cap, int threads, uint32_t *out,
                      uint32_t *layers_used, int *cause) {
  if (!dims_ok(w, h) || auto_cap == 0 || auto_cap > OR_MAX_LAYERS) return OR_EINVAL;
  const size_t n = (size_t)w * h;
  uint32_t *a = (uint32_t *)malloc(n * 4), *b = (uint32_t *)malloc(n * 4);
  or_initial(w, h, occ, srcmask, a);
  uint64_t z_prev = or_zero_free_cells(w, h, occ, a);
  uint32_t l = 1;
  int why = OR_STOP_CAP;
  for (; l <= auto_cap; ++l) {
    or_propagate_layer(w, h, occ, srcmask, a, b, threads);
    uint32_t *t = a;
    a = b;
    b = t;
    const uint64_t z = or_zero_free_cells(w, h, occ, a);
    if (z == 0) { why = OR_STOP_FILLED; break; }
    if (z == z_prev) { why = OR_STOP_STALLED; break; }
    z_prev = z;
  }
  if (why == OR_STOP_CAP) l = auto_cap;
  memcpy(out, a, n * 4);
  free(a);
  free(b);
  *layers_used = l;
  *cause = why;
  return OR_OK;
}

/* propagate.hpp:63-68: signed int32 map,
 * obstacles carry INT32_MIN (I_e), sources +1 (I_s), ReLU after the add. */
int or_propagate_reference(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                           uint32_t layers, uint32_t *out) {
  if (!dims_ok(w, h) || layers == 0 || layers > OR_MAX_LAYERS) return OR_EINVAL;
  const size_t n = (size_t)w * h;
  int32_t *a = (int32_t *)malloc(n * 4), *b = (int32_t *)malloc(n * 4);
  for (size_t i = 0; i < n; ++i) a[i] = srcmask[i] ? 1 : 0; /* A_0 = I_s */
  for (uint32_t l = 0; l < layers; ++l) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < (int64_t)h; ++r) {
      for (int64_t c = 0; c < (int64_t)w; ++c) {
        int32_t m = 0; /* zero padding */
        for (int dr = -1; dr <= 1; ++dr) {
          const int64_t rr = r + dr;
          if (rr < 0 || rr >= (int64_t)h) continue;
          for (int dc = -1; dc <= 1; ++dc) {
            const int64_t cc = c + dc;
            if (cc < 0 || cc >= (int64_t)w) continue;
            const int32_t v = a[rr * w + cc];
            if (v > m) m = v;
          }
        }
        const size_t i = (size_t)r * w + (size_t)c;
        const int32_t ie = occ[i] ? INT32_MIN : 0;
        const int32_t is = srcmask[i] ? 1 : 0;
        const int64_t t = (int64_t)m + ie + is;
        b[i] = t > 0 ? (int32_t)t : 0; /* ReLU */
      }
    }
    int32_t *t = a;
    a = b;
    b = t;
  }
  for (size_t i = 0; i < n; ++i) out[i] = (uint32_t)a[i];
  free(a);
  free(b);
  return OR_OK;
}

/* propagate.hpp:70-79, SPEC.md:142-150 (n = height, m = width). */
void or_layer_bound(uint32_t w, uint32_t h, uint64_t *worst, uint32_t *lo, uint32_t *hi) {
  const uint64_t mx = w > h ? w : h, mn = w > h ? h : w;
  *worst = mx * ((mn + 1) / 2) + mn / 2;
  *lo = (uint32_t)((3 * mx + 1) / 2);
  *hi = (uint32_t)(2 * mx);
}

/* ------------------------------------------------------------------------ */
/* oracles                                                                  */
/* ------------------------------------------------------------------------ */

static const int DR8[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
static const int DC8[8] = {-1, 0, 1, -1, 1, -1, 0, 1};

static int bfs_core(uint32_t w, uint32_t h, const uint8_t *occ, uint32_t *hops,
                    uint64_t *queue, uint64_t qn) {
  uint64_t head = 0, tail = qn;
  while (head < tail) {
    const uint64_t i = queue[head++];
    const uint32_t r = (uint32_t)(i / w), c = (uint32_t)(i % w);
    const uint32_t d = hops[i] + 1;
    for (int k = 0; k < 8; ++k) {
      const int64_t rr = (int64_t)r + DR8[k], cc = (int64_t)c + DC8[k];
      if (rr < 0 || cc < 0 || rr >= h || cc >= w) continue;
      const uint64_t j = (uint64_t)rr * w + (uint64_t)cc;
      if (occ[j] || hops[j] != OR_UNREACH) continue;
      hops[j] = d;
      queue[tail++] = j;
    }
  }
  return OR_OK;
}

/* oracle.hpp:73-76: exact 8-connected hop distances (diagonals always
 * allowed between free cells). */
int or_bfs_multi_source(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                        uint32_t *hops) {
  const uint64_t n = (uint64_t)w * h;
  uint64_t *q = (uint64_t *)malloc(sizeof(uint64_t) * (n ? n : 1));
  uint64_t qn = 0;
  for (uint64_t i = 0; i < n; ++i) {
    hops[i] = OR_UNREACH;
    if (srcmask[i] && !occ[i]) {
      hops[i] = 0;
      q[qn++] = i;
    }
  }
  bfs_core(w, h, occ, hops, q, qn);
  free(q);
  return OR_OK;
}

/* oracle.hpp:78-79. */
int or_bfs_from(uint32_t w, uint32_t h, const uint8_t *occ, uint32_t row, uint32_t col,
                uint32_t *hops) {
  if (row >= h || col >= w) return OR_EINVAL;
  const uint64_t n = (uint64_t)w * h;
  for (uint64_t i = 0; i < n; ++i) hops[i] = OR_UNREACH;
  const uint64_t s = (uint64_t)row * w + col;
  if (occ[s]) return OR_EINVAL;
  uint64_t *q = (uint64_t *)malloc(sizeof(uint64_t) * n);
  hops[s] = 0;
  q[0] = s;
  bfs_core(w, h, occ, hops, q, 1);
  free(q);
  return OR_OK;
}

/* oracle.hpp:17-40: sign of (a1 + b1*sqrt2) - (a2 + b2*sqrt2), exact. */
static int octile_cmp(int64_t a1, int64_t b1, int64_t a2, int64_t b2) {
  const __int128 da = (__int128)a1 - a2, db = (__int128)b1 - b2;
  if (da >= 0 && db >= 0) return (da || db) ? 1 : 0;
  if (da <= 0 && db <= 0) return -1;
  const __int128 lhs = da * da, rhs = 2 * db * db;
  if (da > 0) return lhs > rhs ? 1 : (lhs < rhs ? -1 : 0);
  return rhs > lhs ? 1 : (rhs < lhs ? -1 : 0);
}

typedef struct { int64_t a, b; uint64_t cell; } heap_item;

static int heap_less(const heap_item *x, const heap_item *y) {
  return octile_cmp(x->a, x->b, y->a, y->b) < 0;
}

/* oracle.hpp:81-85: exact octile Dijkstra; diagonal moves obey `rule`
 * (strict forbids squeezing between two diagonally adjacent obstacles). */
int or_dijkstra_octile(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                       int rule, int64_t *axis, int64_t *diag) {
  const uint64_t n = (uint64_t)w * h;
  heap_item *hp = (heap_item *)malloc(sizeof(heap_item) * (8 * n + 16));
  uint64_t hn = 0;
  uint8_t *done = (uint8_t *)calloc(n, 1);
  for (uint64_t i = 0; i < n; ++i) {
    axis[i] = -1;
    diag[i] = -1;
  }
#define HPUSH(A, B, C)                                                   \
  do {                                                                   \
    heap_item it = {(A), (B), (C)};                                      \
    uint64_t k = hn++;                                                   \
    hp[k] = it;                                                          \
    while (k > 0 && heap_less(&hp[k], &hp[(k - 1) / 2])) {               \
      heap_item t = hp[k]; hp[k] = hp[(k - 1) / 2]; hp[(k - 1) / 2] = t; \
      k = (k - 1) / 2;                                                   \
    }                                                                    \
  } while (0)
  for (uint64_t i = 0; i < n; ++i)
    if (srcmask[i] && !occ[i]) {
      axis[i] = 0;
      diag[i] = 0;
      HPUSH(0, 0, i);
    }
  while (hn) {
    heap_item top = hp[0];
    hp[0] = hp[--hn];
    uint64_t k = 0;
    for (;;) {
      uint64_t l = 2 * k + 1, r = l + 1, m = k;
      if (l < hn && heap_less(&hp[l], &hp[m])) m = l;
      if (r < hn && heap_less(&hp[r], &hp[m])) m = r;
      if (m == k) break;
      heap_item t = hp[k]; hp[k] = hp[m]; hp[m] = t;
      k = m;
    }
    const uint64_t i = top.cell;
    if (done[i]) continue;
    if (axis[i] != top.a || diag[i] != top.b) continue;
    done[i] = 1;
    const int64_t r0 = (int64_t)(i / w), c0 = (int64_t)(i % w);
    for (int d = 0; d < 8; ++d) {
      const int64_t rr = r0 + DR8[d], cc = c0 + DC8[d];
      if (rr < 0 || cc < 0 || rr >= h || cc >= w) continue;
      const uint64_t j = (uint64_t)rr * w + (uint64_t)cc;
      if (occ[j] || done[j]) continue;
      const int is_diag = DR8[d] != 0 && DC8[d] != 0;
      if (is_diag && rule == OR_CORNER_STRICT) {
        if (occ[(uint64_t)r0 * w + (uint64_t)cc] && occ[(uint64_t)rr * w + (uint64_t)c0]) continue;
      }
      const int64_t na = top.a + (is_diag ? 0 : 1), nb = top.b + (is_diag ? 1 : 0);
      if (axis[j] < 0 || octile_cmp(na, nb, axis[j], diag[j]) < 0) {
        axis[j] = na;
        diag[j] = nb;
        HPUSH(na, nb, j);
      }
    }
  }
#undef HPUSH
  free(hp);
  free(done);
  return OR_OK;
}

/* oracle.hpp:87-98: value(c) == max(0, L+1-d(c)) on free
 * cells; obstacle cells must be 0. */
uint64_t or_check_activity(uint32_t w, uint32_t h, const uint8_t *occ, const uint32_t *vals,
                           const uint32_t *hops, uint32_t layers, uint32_t *samples_rc,
                           uint32_t max_samples) {
  const uint64_t n = (uint64_t)w * h;
  uint64_t bad = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t expect = 0;
    if (!occ[i] && hops[i] != OR_UNREACH) {
      const int64_t e = (int64_t)layers + 1 - (int64_t)hops[i];
      expect = e > 0 ? (uint64_t)e : 0;
    }
    if ((uint64_t)vals[i] != expect) {
      if (samples_rc && bad < max_samples) {
        samples_rc[2 * bad] = (uint32_t)(i / w);
        samples_rc[2 * bad + 1] = (uint32_t)(i % w);
      }
      ++bad;
    }
  }
  return bad;
}

/* ------------------------------------------------------------------------ */
/* path extraction                                                          */
/* ------------------------------------------------------------------------ */

static int check_target(uint32_t w, uint32_t h, const uint8_t *occ, const uint32_t *vals,
                        uint32_t tr, uint32_t tc) {
  if (tr >= h || tc >= w) return OR_EINVAL;                 /* pin P8 */
  if (occ[(uint64_t)tr * w + tc]) return OR_EINVAL;         /* reconstruct.hpp:36 */
  if (vals[(uint64_t)tr * w + tc] == 0) return OR_EUNCOVERED; /* reconstruct.hpp:37 */
  return OR_OK;
}

#define PUSH_PT(R, C)                        \
  do {                                       \
    if (n >= cap) return OR_EINVAL;          \
    pts_rc[2 * n] = (R);                     \
    pts_rc[2 * n + 1] = (C);                 \
    ++n;                                     \
  } while (0)

/* reconstruct.hpp:34-40, pins P2/P5: greedy 8-neighbour
 * ascent; candidates = in-bounds neighbours with the maximal value in
 * row-major order; one splitmix64 draw only when >= 2 candidates tie, index
 * = (u * count) >> 64; stop on SourceSet membership. */
int or_reconstruct_simple(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                          const uint32_t *vals, uint32_t trow, uint32_t tcol, uint64_t seed,
                          uint32_t *pts_rc, uint64_t cap, uint64_t *npts) {
  *npts = 0;
  int st = check_target(w, h, occ, vals, trow, tcol);
  if (st) return st;
  uint64_t rng = seed, n = 0;
  uint32_t r = trow, c = tcol;
  PUSH_PT(r, c);
  while (!srcmask[(uint64_t)r * w + c]) {
    const uint32_t cur = vals[(uint64_t)r * w + c];
    uint32_t best = 0;
    int have = 0;
    for (int k = 0; k < 8; ++k) {
      const int64_t rr = (int64_t)r + DR8[k], cc = (int64_t)c + DC8[k];
      if (rr < 0 || cc < 0 || rr >= h || cc >= w) continue;
      const uint32_t v = vals[(uint64_t)rr * w + (uint64_t)cc];
      if (!have || v > best) { best = v; have = 1; }
    }
    if (!have || best <= cur) return OR_EINTERNAL;
    int cand[8], nc = 0;
    for (int k = 0; k < 8; ++k) {
      const int64_t rr = (int64_t)r + DR8[k], cc = (int64_t)c + DC8[k];
      if (rr < 0 || cc < 0 || rr >= h || cc >= w) continue;
      if (vals[(uint64_t)rr * w + (uint64_t)cc] == best) cand[nc++] = k;
    }
    int pick = 0;
    if (nc >= 2) pick = (int)or_bounded(or_splitmix64(&rng), (uint64_t)nc);
    r = (uint32_t)((int64_t)r + DR8[cand[pick]]);
    c = (uint32_t)((int64_t)c + DC8[cand[pick]]);
    PUSH_PT(r, c);
  }
  *npts = n;
  return OR_OK;
}

/* reconstruct.hpp:42-47, pin P1: first-listed
 * maximal axis neighbour in order (i,j-1),(i,j+1),(i-1,j),(i+1,j) if it
 * strictly increases; otherwise first-listed maximal diagonal in order
 * (-1,-1),(-1,+1),(+1,-1),(+1,+1) if it strictly increases; then
 * straighten(path, grid, rule) (pin P4). */
int or_reconstruct_euclidean(uint32_t w, uint32_t h, const uint8_t *occ, const uint8_t *srcmask,
                             const uint32_t *vals, uint32_t trow, uint32_t tcol, int rule,
                             uint32_t *pts_rc, uint64_t cap, uint64_t *npts) {
  static const int AR[4] = {0, 0, -1, 1}, AC[4] = {-1, 1, 0, 0};
  static const int GR[4] = {-1, -1, 1, 1}, GC[4] = {-1, 1, -1, 1};
  *npts = 0;
  int st = check_target(w, h, occ, vals, trow, tcol);
  if (st) return st;
  uint64_t n = 0;
  uint32_t r = trow, c = tcol;
  PUSH_PT(r, c);
  while (!srcmask[(uint64_t)r * w + c]) {
    const uint32_t cur = vals[(uint64_t)r * w + c];
    int best = -1;
    uint32_t bv = 0;
    for (int k = 0; k < 4; ++k) {
      const int64_t rr = (int64_t)r + AR[k], cc = (int64_t)c + AC[k];
      if (rr < 0 || cc < 0 || rr >= h || cc >= w) continue;
      const uint32_t v = vals[(uint64_t)rr * w + (uint64_t)cc];
      if (best < 0 || v > bv) { best = k; bv = v; }
    }
    int dr, dc;
    if (best >= 0 && bv > cur) {
      dr = AR[best];
      dc = AC[best];
    } else {
      best = -1;
      for (int k = 0; k < 4; ++k) {
        const int64_t rr = (int64_t)r + GR[k], cc = (int64_t)c + GC[k];
        if (rr < 0 || cc < 0 || rr >= h || cc >= w) continue;
        const uint32_t v = vals[(uint64_t)rr * w + (uint64_t)cc];
        if (best < 0 || v > bv) { best = k; bv = v; }
      }
      if (best < 0 || bv <= cur) return OR_EINTERNAL;
      dr = GR[best];
      dc = GC[best];
    }
    r = (uint32_t)((int64_t)r + dr);
    c = (uint32_t)((int64_t)c + dc);
    PUSH_PT(r, c);
  }
  uint64_t m = 0;
  or_straighten(pts_rc, n, occ, w, h, rule, pts_rc, &m);
  *npts = m;
  return OR_OK;
}

/* reconstruct.hpp:49-58, pin P4: remove the first
 * qualifying interior point scanning target->source, restart, until no
 * change.  Implemented as the equivalent single stack pass (a removal at t
 * can only make t-1 newly qualify). */
int or_straighten(const uint32_t *pts_rc, uint64_t n, const uint8_t *occ, uint32_t w,
                  uint32_t h, int rule, uint32_t *out_rc, uint64_t *nout) {
  (void)h;
  if (n < 3) {
    if (out_rc != pts_rc) memmove(out_rc, pts_rc, sizeof(uint32_t) * 2 * n);
    *nout = n;
    return OR_OK;
  }
  uint32_t *tmp = (uint32_t *)malloc(sizeof(uint32_t) * 2 * n);
  uint64_t m = 0;
  for (uint64_t i = 0; i < n; ++i) {
    tmp[2 * m] = pts_rc[2 * i];
    tmp[2 * m + 1] = pts_rc[2 * i + 1];
    ++m;
    while (m >= 3) {
      const int64_t ar = tmp[2 * (m - 3)], ac = tmp[2 * (m - 3) + 1];
      const int64_t br = tmp[2 * (m - 1)], bc = tmp[2 * (m - 1) + 1];
      const int64_t dr = ar - br, dc = ac - bc;
      if (dr * dr + dc * dc != 2) break;
      if (occ && rule == OR_CORNER_STRICT) {
        if (occ[(uint64_t)ar * w + (uint64_t)bc] && occ[(uint64_t)br * w + (uint64_t)ac]) break;
      }
      tmp[2 * (m - 2)] = tmp[2 * (m - 1)];
      tmp[2 * (m - 2) + 1] = tmp[2 * (m - 1) + 1];
      --m;
    }
  }
  memcpy(out_rc, tmp, sizeof(uint32_t) * 2 * m);
  free(tmp);
  *nout = m;
  return OR_OK;
}

/* reconstruct.hpp:26-32: steps = points-1; length =
 * (#axis moves) + (#diagonal moves)*sqrt(2) (+ exact norm of any longer
 * move). */
void or_path_metrics(const uint32_t *pts_rc, uint64_t n, uint64_t *steps, double *length) {
  *steps = n ? n - 1 : 0;
  uint64_t ax = 0, dg = 0;
  double other = 0.0;
  for (uint64_t i = 1; i < n; ++i) {
    const int64_t dr = (int64_t)pts_rc[2 * i] - pts_rc[2 * i - 2];
    const int64_t dc = (int64_t)pts_rc[2 * i + 1] - pts_rc[2 * i - 1];
    const int64_t q = dr * dr + dc * dc;
    if (q == 1) ++ax;
    else if (q == 2) ++dg;
    else other += sqrt((double)q);
  }
  *length = (double)ax + (double)dg * 1.4142135623730951 + other;
}

/* ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference tilejoin self-join with its scalar
 * (direct-form) refinement, used as the parity checker for the CUDA path and as
 * the CPU baseline in bench.py.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it; the product
 * path (paper_2209_11287_b200) never does.
 *
 * Followed reference lines (/root/reference/pkg/src/tilejoin):
 *   grid.py:81       coords = floor(x[:, :k] / eps)  (IEEE divide, then floor)
 *   grid.py:83-94    stable lexicographic order of points by cell, dim 0 primary
 *   grid.py:104-133  candidates = members of the occupied cells at Chebyshev
 *                    distance <= 1, lexicographic cell order, ids ascending
 *   join.py:310-318  per query: acc = 0; for dim: diff = q - c; acc += diff*diff;
 *                    keep acc <= eps*eps  (oracle.py:75-84 is the same sum order)
 *   join.py:203-204  pairs sorted by (query id, neighbour id)
 * Compile with -ffp-contract=off so acc + diff*diff is never fused (numpy
 * evaluates the product and the sum as two correctly rounded operations).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXK 16

typedef struct {
  const int64_t* cc; /* n * k cell coordinates */
  int k;
} sort_ctx;

static sort_ctx g_sort; /* qsort has no context argument; sorting is single-threaded */

static int cmp_point(const void* a, const void* b) {
  const uint32_t i = *(const uint32_t*)a, j = *(const uint32_t*)b;
  const int64_t* x = g_sort.cc + (int64_t)i * g_sort.k;
  const int64_t* y = g_sort.cc + (int64_t)j * g_sort.k;
  for (int t = 0; t < g_sort.k; ++t) {
    if (x[t] < y[t]) return -1;
    if (x[t] > y[t]) return 1;
  }
  return (i > j) - (i < j); /* stable: ids ascending inside a cell */
}

static int cmp_coord(const int64_t* x, const int64_t* y, int k) {
  for (int t = 0; t < k; ++t) {
    if (x[t] < y[t]) return -1;
    if (x[t] > y[t]) return 1;
  }
  return 0;
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

typedef struct {
  int64_t n, n_cells;
  int k;
  uint32_t* order;   /* n: point ids in cell order */
  int64_t* cstart;   /* n_cells + 1 */
  int64_t* ccoord;   /* n_cells * k */
} grid_t;

static int build_grid(const double* x, int64_t n, int d, int64_t ld, int k, double eps,
                      grid_t* g) {
  (void)d;
  int64_t* cc = (int64_t*)malloc(sizeof(int64_t) * n * k);
  g->order = (uint32_t*)malloc(sizeof(uint32_t) * n);
  if (!cc || !g->order) return -1;
  for (int64_t i = 0; i < n; ++i) {
    for (int t = 0; t < k; ++t) cc[i * k + t] = (int64_t)floor(x[i * ld + t] / eps);
    g->order[i] = (uint32_t)i;
  }
  /* stable lexicographic order (grid.py:83): when the k coordinate spans pack
   * into 64 bits, an LSD radix sort of (packed key, id) -- ids ascending inside
   * a cell because LSD passes are stable; otherwise qsort with the id tie-break. */
  int64_t lo[MAXK], hi[MAXK];
  int bits[MAXK], total_bits = 0;
  for (int t = 0; t < k; ++t) {
    lo[t] = INT64_MAX;
    hi[t] = INT64_MIN;
  }
  for (int64_t i = 0; i < n; ++i)
    for (int t = 0; t < k; ++t) {
      const int64_t c = cc[i * k + t];
      if (c < lo[t]) lo[t] = c;
      if (c > hi[t]) hi[t] = c;
    }
  for (int t = 0; t < k; ++t) {
    const uint64_t span = (uint64_t)(hi[t] - lo[t]);
    bits[t] = 0;
    while (bits[t] < 64 && (span >> bits[t]) != 0) ++bits[t];
    total_bits += bits[t];
  }
  if (n > 1 && total_bits <= 64 && hi[0] - lo[0] >= 0) {
    uint64_t* key = (uint64_t*)malloc(sizeof(uint64_t) * n);
    uint64_t* key2 = (uint64_t*)malloc(sizeof(uint64_t) * n);
    uint32_t* ord2 = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (int64_t i = 0; i < n; ++i) {
      uint64_t kk = 0;
      for (int t = 0; t < k; ++t)
        kk = (bits[t] ? (kk << bits[t]) : kk) | (uint64_t)(cc[i * k + t] - lo[t]);
      key[i] = kk;
    }
    for (int shift = 0; shift < total_bits; shift += 11) {
      int64_t cnt[2049];
      memset(cnt, 0, sizeof(cnt));
      for (int64_t i = 0; i < n; ++i) ++cnt[((key[i] >> shift) & 2047) + 1];
      for (int b = 0; b < 2048; ++b) cnt[b + 1] += cnt[b];
      for (int64_t i = 0; i < n; ++i) {
        const int64_t at = cnt[(key[i] >> shift) & 2047]++;
        key2[at] = key[i];
        ord2[at] = g->order[i];
      }
      uint64_t* tk = key; key = key2; key2 = tk;
      uint32_t* to = g->order; g->order = ord2; ord2 = to;
    }
    free(key);
    free(key2);
    free(ord2);
  } else {
    g_sort.cc = cc;
    g_sort.k = k;
    qsort(g->order, (size_t)n, sizeof(uint32_t), cmp_point);
  }
  g->cstart = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  g->ccoord = (int64_t*)malloc(sizeof(int64_t) * n * k);
  int64_t nc = 0;
  for (int64_t p = 0; p < n; ++p) {
    const int64_t* c = cc + (int64_t)g->order[p] * k;
    if (p == 0 || cmp_coord(c, g->ccoord + (nc - 1) * k, k) != 0) {
      memcpy(g->ccoord + nc * k, c, sizeof(int64_t) * k);
      g->cstart[nc++] = p;
    }
  }
  g->cstart[nc] = n;
  g->n = n;
  g->n_cells = nc;
  g->k = k;
  free(cc);
  return 0;
}

static void free_grid(grid_t* g) {
  free(g->order);
  free(g->cstart);
  free(g->ccoord);
}

static int64_t find_cell(const grid_t* g, const int64_t* c) {
  int64_t lo = 0, hi = g->n_cells;
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    int r = cmp_coord(g->ccoord + mid * g->k, c, g->k);
    if (r == 0) return mid;
    if (r < 0) lo = mid + 1;
    else hi = mid;
  }
  return -1;
}

/* Occupied neighbour cells of cell `ci`, lexicographic (itertools.product order). */
static int neighbours(const grid_t* g, int64_t ci, int64_t* out) {
  const int k = g->k;
  int64_t nb[MAXK];
  int cnt = 0;
  int total = 1;
  for (int t = 0; t < k; ++t) total *= 3;
  for (int r = 0; r < total; ++r) {
    int rr = r;
    for (int t = k - 1; t >= 0; --t) {
      nb[t] = g->ccoord[ci * k + t] + (rr % 3) - 1;
      rr /= 3;
    }
    int64_t f = find_cell(g, nb);
    if (f >= 0) out[cnt++] = f;
  }
  return cnt;
}

static inline int direct_le(const double* x, int64_t ld, int d, uint32_t q, uint32_t c,
                            double eps_sq) {
  const double* a = x + (int64_t)q * ld;
  const double* b = x + (int64_t)c * ld;
  double acc = 0.0;
  for (int t = 0; t < d; ++t) {
    double diff = a[t] - b[t];
    acc = acc + diff * diff;
  }
  return acc <= eps_sq;
}

/* Squared distance in the reference order (exported for boundary classification). */
double oracle_sqdist(const double* x, int64_t ld, int d, int64_t q, int64_t c) {
  const double* a = x + q * ld;
  const double* b = x + c * ld;
  double acc = 0.0;
  for (int t = 0; t < d; ++t) {
    double diff = a[t] - b[t];
    acc = acc + diff * diff;
  }
  return acc;
}

/* Refine the query cells listed in `cells` (or all cells when cells == NULL).
 * Pass 1 (nbrs == NULL): counts[q] = |R(q)| for every query in those cells.
 * Pass 2: writes each row at nbrs[offsets[q]...] ascending. */
static void refine_cells(const grid_t* g, const double* x, int64_t ld, int d, double eps_sq,
                         const int64_t* cells, int64_t n_sel, int64_t* counts,
                         const int64_t* offsets, uint32_t* nbrs, int threads) {
  int max_nb = 1;
  for (int t = 0; t < g->k; ++t) max_nb *= 3;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
  {
    int64_t* nb = (int64_t*)malloc(sizeof(int64_t) * max_nb);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
    for (int64_t s = 0; s < n_sel; ++s) {
      const int64_t ci = cells ? cells[s] : s;
      const int nn = neighbours(g, ci, nb);
      for (int64_t qp = g->cstart[ci]; qp < g->cstart[ci + 1]; ++qp) {
        const uint32_t q = g->order[qp];
        int64_t cnt = 0;
        uint32_t* row = nbrs ? nbrs + offsets[q] : NULL;
        for (int m = 0; m < nn; ++m) {
          for (int64_t cp = g->cstart[nb[m]]; cp < g->cstart[nb[m] + 1]; ++cp) {
            const uint32_t c = g->order[cp];
            if (direct_le(x, ld, d, q, c, eps_sq)) {
              if (row) row[cnt] = c;
              ++cnt;
            }
          }
        }
        if (row) qsort(row, (size_t)cnt, sizeof(uint32_t), cmp_u32);
        else counts[q] = cnt;
      }
    }
    free(nb);
  }
}

/* Grid summary for parity of the device index (grid.py semantics).
 * Returns n_cells; fills point_order (n), cell_start (n_cells+1, caller sized n+1),
 * cell_coords (n_cells*k, caller sized n*k) when non-NULL, and per-cell candidate
 * counts (n_cells) when cand != NULL. */
int64_t oracle_grid(const double* x, int64_t n, int d, int64_t ld, int k, double eps,
                    uint32_t* point_order, int64_t* cell_start, int64_t* cell_coords,
                    int64_t* cand) {
  grid_t g;
  if (k < 1 || k > MAXK || build_grid(x, n, d, ld, k, eps, &g) != 0) return -1;
  if (point_order) memcpy(point_order, g.order, sizeof(uint32_t) * n);
  if (cell_start) memcpy(cell_start, g.cstart, sizeof(int64_t) * (g.n_cells + 1));
  if (cell_coords) memcpy(cell_coords, g.ccoord, sizeof(int64_t) * g.n_cells * k);
  if (cand) {
    int max_nb = 1;
    for (int t = 0; t < k; ++t) max_nb *= 3;
    int64_t* nb = (int64_t*)malloc(sizeof(int64_t) * max_nb);
    for (int64_t c = 0; c < g.n_cells; ++c) {
      int nn = neighbours(&g, c, nb);
      int64_t s = 0;
      for (int m = 0; m < nn; ++m) s += g.cstart[nb[m] + 1] - g.cstart[nb[m]];
      cand[c] = s;
    }
    free(nb);
  }
  int64_t nc = g.n_cells;
  free_grid(&g);
  return nc;
}

/* Full (or cell-sampled) self-join.  Output CSR by original id: offsets[n+1]
 * (rows of unselected queries are empty), neighbours ascending.  Two calls:
 * first with nbrs == NULL to get *total, then with a buffer of *total ids.
 * sel_cells: indices into the lexicographic cell list (NULL = all cells). */
int oracle_self_join(const double* x, int64_t n, int d, int64_t ld, int k, double eps,
                     const int64_t* sel_cells, int64_t n_sel, int64_t* offsets,
                     uint32_t* nbrs, int64_t* total, int threads) {
  grid_t g;
  if (k < 1 || k > MAXK || build_grid(x, n, d, ld, k, eps, &g) != 0) return -1;
  const double eps_sq = eps * eps;
  const int64_t m = sel_cells ? n_sel : g.n_cells;
  if (sel_cells) {
    for (int64_t s = 0; s < n_sel; ++s)
      if (sel_cells[s] < 0 || sel_cells[s] >= g.n_cells) {
        free_grid(&g);
        return -2;
      }
  }
  if (!nbrs) {
    int64_t* counts = (int64_t*)calloc((size_t)n, sizeof(int64_t));
    refine_cells(&g, x, ld, d, eps_sq, sel_cells, m, counts, NULL, NULL, threads);
    int64_t acc = 0;
    for (int64_t i = 0; i < n; ++i) {
      offsets[i] = acc;
      acc += counts[i];
    }
    offsets[n] = acc;
    *total = acc;
    free(counts);
  } else {
    refine_cells(&g, x, ld, d, eps_sq, sel_cells, m, NULL, offsets, nbrs, threads);
  }
  free_grid(&g);
  return 0;
}

/* Rows of selected queries only (for sampled parity on large inputs).
 * counts[i] = |R(qids[i])|; with nbrs != NULL the rows are written back to back
 * in qids order (each ascending), nbrs sized sum(counts). */
int oracle_rows(const double* x, int64_t n, int d, int64_t ld, int k, double eps,
                const int64_t* qids, int64_t nq, int64_t* counts, uint32_t* nbrs, int threads) {
  grid_t g;
  if (k < 1 || k > MAXK || build_grid(x, n, d, ld, k, eps, &g) != 0) return -1;
  const double eps_sq = eps * eps;
  int64_t* pos_of = (int64_t*)malloc(sizeof(int64_t) * n);
  for (int64_t p = 0; p < n; ++p) pos_of[g.order[p]] = p;
  int64_t* base = NULL;
  if (nbrs) {
    base = (int64_t*)malloc(sizeof(int64_t) * (nq + 1));
    base[0] = 0;
    for (int64_t i = 0; i < nq; ++i) base[i + 1] = base[i] + counts[i];
  }
  int max_nb = 1;
  for (int t = 0; t < k; ++t) max_nb *= 3;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
  {
    int64_t* nb = (int64_t*)malloc(sizeof(int64_t) * max_nb);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
    for (int64_t i = 0; i < nq; ++i) {
      const uint32_t q = (uint32_t)qids[i];
      const int64_t p = pos_of[q];
      int64_t lo = 0, hi = g.n_cells; /* cell containing position p */
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) / 2;
        if (g.cstart[mid] <= p) lo = mid;
        else hi = mid;
      }
      const int nn = neighbours(&g, lo, nb);
      int64_t cnt = 0;
      uint32_t* row = nbrs ? nbrs + base[i] : NULL;
      for (int m = 0; m < nn; ++m)
        for (int64_t cp = g.cstart[nb[m]]; cp < g.cstart[nb[m] + 1]; ++cp) {
          const uint32_t c = g.order[cp];
          if (direct_le(x, ld, d, q, c, eps_sq)) {
            if (row) row[cnt] = c;
            ++cnt;
          }
        }
      if (row) qsort(row, (size_t)cnt, sizeof(uint32_t), cmp_u32);
      else counts[i] = cnt;
    }
    free(nb);
  }
  free(base);
  free(pos_of);
  free_grid(&g);
  return 0;
}

/* CPU-baseline timing (bench.py cpu_baseline / --impl reference): the grid is
 * built once (timed: *grid_s), then the selected query cells are refined in ONE
 * pass that emits every pair into per-thread buffers and sorts each row
 * (timed: *refine_s) -- the reference's per-batch work (join.py:184-204)
 * without the count pass oracle_self_join needs to size its output.
 * Returns the number of pairs emitted, < 0 on failure. */
#include <time.h>
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int64_t oracle_time_join(const double* x, int64_t n, int d, int64_t ld, int k, double eps,
                         const int64_t* sel_cells, int64_t n_sel, int threads, double* grid_s,
                         double* refine_s) {
  grid_t g;
  double t0 = now_s();
  if (k < 1 || k > MAXK || build_grid(x, n, d, ld, k, eps, &g) != 0) return -1;
  *grid_s = now_s() - t0;
  const double eps_sq = eps * eps;
  const int64_t m = sel_cells ? n_sel : g.n_cells;
  int max_nb = 1;
  for (int t = 0; t < k; ++t) max_nb *= 3;
  int64_t total = 0;
  t0 = now_s();
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel reduction(+ : total)
#endif
  {
    int64_t* nb = (int64_t*)malloc(sizeof(int64_t) * max_nb);
    size_t cap = 1 << 16, len = 0;
    uint32_t* buf = (uint32_t*)malloc(sizeof(uint32_t) * cap);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
    for (int64_t s = 0; s < m; ++s) {
      const int64_t ci = sel_cells ? sel_cells[s] : s;
      const int nn = neighbours(&g, ci, nb);
      for (int64_t qp = g.cstart[ci]; qp < g.cstart[ci + 1]; ++qp) {
        const uint32_t q = g.order[qp];
        const size_t row0 = len;
        for (int mm = 0; mm < nn; ++mm)
          for (int64_t cp = g.cstart[nb[mm]]; cp < g.cstart[nb[mm] + 1]; ++cp) {
            const uint32_t c = g.order[cp];
            if (direct_le(x, ld, d, q, c, eps_sq)) {
              if (len == cap) {
                cap *= 2;
                buf = (uint32_t*)realloc(buf, sizeof(uint32_t) * cap);
              }
              buf[len++] = c;
            }
          }
        qsort(buf + row0, len - row0, sizeof(uint32_t), cmp_u32);
        total += (int64_t)(len - row0);
        if (len > (1u << 24)) len = 0; /* rows are consumed; keep the buffer bounded */
      }
    }
    free(buf);
    free(nb);
  }
  *refine_s = now_s() - t0;
  free_grid(&g);
  return total;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---- full-set digest (parity of the large configs without materialising 10+ GB) ----
 * An order-independent digest of the pair set R = {(q, c)}: with
 * key = (uint64)q << 32 | c, s1 = sum splitmix64(key), s2 = sum splitmix64(key + K2)
 * (mod 2^64), plus |R|.  tests/test_gpu_parity.py computes the same digest from the
 * device CSR (tests/digest.py; the two are pinned against each other on CPU).
 * The direct form is the reference's (join.py:310-318); the running sum stops once
 * it exceeds eps^2 -- exact, because fl(acc + t) >= acc for t >= 0, so a partial sum
 * above eps^2 stays above it. */
static inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}
#define DIGEST_K2 0x632be59bd9b4e019ull

static inline int direct_le_exit(const double* a, const double* b, int d, double eps_sq) {
  double acc = 0.0;
  int t = 0;
  for (; t + 4 <= d; t += 4) {
    double d0 = a[t] - b[t], d1 = a[t + 1] - b[t + 1], d2 = a[t + 2] - b[t + 2],
           d3 = a[t + 3] - b[t + 3];
    acc = acc + d0 * d0;
    acc = acc + d1 * d1;
    acc = acc + d2 * d2;
    acc = acc + d3 * d3;
    if (acc > eps_sq) return 0;
  }
  for (; t < d; ++t) {
    double df = a[t] - b[t];
    acc = acc + df * df;
  }
  return acc <= eps_sq;
}

void oracle_digest_keys(const uint64_t* keys, int64_t m, uint64_t* out) {
  uint64_t s1 = 0, s2 = 0;
  for (int64_t i = 0; i < m; ++i) {
    s1 += mix64(keys[i]);
    s2 += mix64(keys[i] + DIGEST_K2);
  }
  out[0] = (uint64_t)m;
  out[1] = s1;
  out[2] = s2;
}

/* out[0] = |R|, out[1] = s1, out[2] = s2, out[3] = largest row. */
int oracle_digest(const double* x, int64_t n, int d, int64_t ld, int k, double eps, int threads,
                  uint64_t* out) {
  grid_t g;
  if (k < 1 || k > MAXK || build_grid(x, n, d, ld, k, eps, &g) != 0) return -1;
  const double eps_sq = eps * eps;
  int max_nb = 1;
  for (int t = 0; t < k; ++t) max_nb *= 3;
  uint64_t cnt = 0, s1 = 0, s2 = 0, mx = 0;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel reduction(+ : cnt, s1, s2) reduction(max : mx)
#endif
  {
    int64_t* nb = (int64_t*)malloc(sizeof(int64_t) * max_nb);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
    for (int64_t ci = 0; ci < g.n_cells; ++ci) {
      const int nn = neighbours(&g, ci, nb);
      for (int64_t qp = g.cstart[ci]; qp < g.cstart[ci + 1]; ++qp) {
        const uint32_t q = g.order[qp];
        const double* a = x + (int64_t)q * ld;
        uint64_t row = 0;
        for (int m = 0; m < nn; ++m)
          for (int64_t cp = g.cstart[nb[m]]; cp < g.cstart[nb[m] + 1]; ++cp) {
            const uint32_t c = g.order[cp];
            if (direct_le_exit(a, x + (int64_t)c * ld, d, eps_sq)) {
              const uint64_t key = ((uint64_t)q << 32) | c;
              s1 += mix64(key);
              s2 += mix64(key + DIGEST_K2);
              ++row;
            }
          }
        cnt += row;
        if (row > mx) mx = row;
      }
    }
    free(nb);
  }
  out[0] = cnt;
  out[1] = s1;
  out[2] = s2;
  out[3] = mx;
  free_grid(&g);
  return 0;
}

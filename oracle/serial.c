/*
 * CPU ORACLE (plain C) -- test infrastructure only; never linked into the
 * product.  Sequential restatements of the reference's independent oracles
 * (reference pkg/tests/_oracles.py) and of the primitives' definitions, used
 * by tests/ to check the CUDA path at sizes where the numpy port
 * (oracle/graphfx_port.py) is too slow.  Built by oracle/Makefile into
 * oracle/liboracle.so.
 *
 * Graph arguments: row int64[n+1], col int32[m] (sorted neighbour lists).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define UNV INT64_MAX

/* _oracles.py:17-28 serial_bfs (FIFO queue) */
int64_t ora_bfs(int64_t n, const int64_t* row, const int32_t* col, int64_t src, int64_t* labels) {
  for (int64_t i = 0; i < n; ++i) labels[i] = UNV;
  int32_t* q = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  if (!q) return -1;
  int64_t head = 0, tail = 0;
  labels[src] = 0;
  q[tail++] = (int32_t)src;
  while (head < tail) {
    int32_t v = q[head++];
    for (int64_t e = row[v]; e < row[v + 1]; ++e) {
      int32_t w = col[e];
      if (labels[w] == UNV) {
        labels[w] = labels[v] + 1;
        q[tail++] = w;
      }
    }
  }
  free(q);
  return tail;
}

/* _oracles.py:31-48 dijkstra with a binary heap of (dist, vertex) */
typedef struct { int64_t d; int32_t v; } HeapItem;

static void heap_push(HeapItem* h, int64_t* sz, HeapItem x) {
  int64_t i = (*sz)++;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (h[p].d < x.d || (h[p].d == x.d && h[p].v <= x.v)) break;
    h[i] = h[p];
    i = p;
  }
  h[i] = x;
}

static HeapItem heap_pop(HeapItem* h, int64_t* sz) {
  HeapItem top = h[0];
  HeapItem x = h[--(*sz)];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, s = i;
    HeapItem best = x;
    if (l < *sz && (h[l].d < best.d || (h[l].d == best.d && h[l].v < best.v))) { s = l; best = h[l]; }
    if (r < *sz && (h[r].d < best.d || (h[r].d == best.d && h[r].v < best.v))) { s = r; best = h[r]; }
    if (s == i) break;
    h[i] = h[s];
    i = s;
  }
  h[i] = x;
  return top;
}

int64_t ora_dijkstra(int64_t n, const int64_t* row, const int32_t* col, const int64_t* w,
                     int64_t src, int64_t* labels) {
  int64_t m = row[n];
  for (int64_t i = 0; i < n; ++i) labels[i] = UNV;
  HeapItem* h = (HeapItem*)malloc(sizeof(HeapItem) * (size_t)(m + 2));
  char* done = (char*)calloc((size_t)(n > 0 ? n : 1), 1);
  if (!h || !done) return -1;
  int64_t sz = 0, settled = 0;
  labels[src] = 0;
  HeapItem s0 = {0, (int32_t)src};
  heap_push(h, &sz, s0);
  while (sz) {
    HeapItem it = heap_pop(h, &sz);
    if (done[it.v]) continue;
    done[it.v] = 1;
    ++settled;
    for (int64_t e = row[it.v]; e < row[it.v + 1]; ++e) {
      int32_t u = col[e];
      int64_t nd = it.d + w[e];
      if (nd < labels[u]) {
        labels[u] = nd;
        HeapItem x = {nd, u};
        heap_push(h, &sz, x);
      }
    }
  }
  free(h);
  free(done);
  return settled;
}

/* _oracles.py:82-105 union-find (union by min root) -> canonical min-id */
static int64_t uf_find(int64_t* p, int64_t x) {
  int64_t r = x;
  while (p[r] != r) r = p[r];
  while (p[x] != r) {
    int64_t nx = p[x];
    p[x] = r;
    x = nx;
  }
  return r;
}

int64_t ora_cc(int64_t n, const int64_t* row, const int32_t* col, int64_t* comp) {
  for (int64_t i = 0; i < n; ++i) comp[i] = i;
  for (int64_t v = 0; v < n; ++v)
    for (int64_t e = row[v]; e < row[v + 1]; ++e) {
      int64_t a = uf_find(comp, v), b = uf_find(comp, col[e]);
      if (a != b) {
        if (a < b) comp[b] = a; else comp[a] = b;
      }
    }
  int64_t ncomp = 0;
  for (int64_t v = 0; v < n; ++v) {
    comp[v] = uf_find(comp, v);
    if (comp[v] == v) ++ncomp;
  }
  return ncomp;
}

/* tc.py:53-76: orient deg[s] > deg[d] or (== and s < d); per oriented edge
 * |N+(u) ∩ N+(v)| by sorted merge; counts in oriented CSR order. */
int64_t ora_tc(int64_t n, const int64_t* row, const int32_t* col, int64_t* orow_out,
               int32_t* ocol_out, int64_t* counts) {
  int64_t k = 0;
  orow_out[0] = 0;
  for (int64_t s = 0; s < n; ++s) {
    int64_t ds = row[s + 1] - row[s];
    for (int64_t e = row[s]; e < row[s + 1]; ++e) {
      int32_t d = col[e];
      int64_t dd = row[d + 1] - row[d];
      if (ds > dd || (ds == dd && s < d)) ocol_out[k++] = d;
    }
    orow_out[s + 1] = k;
  }
  int64_t total = 0;
  for (int64_t u = 0; u < n; ++u)
    for (int64_t e = orow_out[u]; e < orow_out[u + 1]; ++e) {
      int32_t v = ocol_out[e];
      int64_t i = orow_out[u], ie = orow_out[u + 1], j = orow_out[v], je = orow_out[v + 1], c = 0;
      while (i < ie && j < je) {
        if (ocol_out[i] < ocol_out[j]) ++i;
        else if (ocol_out[i] > ocol_out[j]) ++j;
        else { ++c; ++i; ++j; }
      }
      counts[e] = c;
      total += c;
    }
  return total;
}

/* pagerank.py:30-91 with epsilon = 0: synchronous power iteration; pulls
 * contributions in ascending in-neighbour order (rrow/rcol = reverse CSR). */
void ora_pagerank(int64_t n, const int64_t* row, const int64_t* rrow, const int32_t* rcol,
                  double damping, int64_t iters, double* rank) {
  double* nxt = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double* contrib = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (int64_t v = 0; v < n; ++v) rank[v] = 1.0 / (double)n;
  for (int64_t it = 0; it < iters; ++it) {
    double dangling = 0.0;
    for (int64_t v = 0; v < n; ++v) {
      int64_t d = row[v + 1] - row[v];
      if (d == 0) { dangling += rank[v]; contrib[v] = 0.0; }
      else contrib[v] = damping * rank[v] / (double)d;
    }
    double base = (1.0 - damping) / (double)n + damping * dangling / (double)n;
    for (int64_t v = 0; v < n; ++v) {
      double s = base;
      for (int64_t e = rrow[v]; e < rrow[v + 1]; ++e) s += contrib[rcol[e]];
      nxt[v] = s;
    }
    memcpy(rank, nxt, sizeof(double) * (size_t)n);
  }
  free(nxt);
  free(contrib);
}

/* _oracles.py:51-79 brandes_dependencies (unweighted, single source) */
void ora_bc(int64_t n, const int64_t* row, const int32_t* col, const int64_t* rrow,
            const int32_t* rcol, int64_t src, double* delta_out) {
  double* sigma = (double*)calloc((size_t)n, sizeof(double));
  int64_t* dist = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) { dist[i] = -1; delta_out[i] = 0.0; }
  int64_t head = 0, tail = 0;
  sigma[src] = 1.0;
  dist[src] = 0;
  order[tail++] = (int32_t)src;
  while (head < tail) {
    int32_t v = order[head++];
    for (int64_t e = row[v]; e < row[v + 1]; ++e) {
      int32_t w = col[e];
      if (dist[w] < 0) { dist[w] = dist[v] + 1; order[tail++] = w; }
      if (dist[w] == dist[v] + 1) sigma[w] += sigma[v];
    }
  }
  for (int64_t i = tail - 1; i >= 0; --i) {
    int32_t w = order[i];
    for (int64_t e = rrow[w]; e < rrow[w + 1]; ++e) {
      int32_t v = rcol[e];
      /* v (an in-neighbour of w) is a predecessor iff dist[v] == dist[w]-1 */
      if (dist[v] >= 0 && dist[v] == dist[w] - 1)
        delta_out[v] += sigma[v] / sigma[w] * (1.0 + delta_out[w]);
    }
  }
  delta_out[src] = 0.0;
  free(sigma);
  free(dist);
  free(order);
}

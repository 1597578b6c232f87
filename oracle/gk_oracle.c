/*
 * gk_oracle.c -- CPU restatement of the reference BFS path (TEST
 * INFRASTRUCTURE ONLY; see gk_oracle.h).  Plain C99, serial, no OpenMP:
 * every result here is a pure function of its inputs.
 *
 * Reference = /root/reference/proj/include/gapkit (header-only C++20).
 */
#include "gk_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng.hpp:12-17 ---------------------------------------------------- */
uint64_t gko_mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* rng.hpp:26-27: state = Mix64(seed) ^ Mix64(~stream) */
void gko_rng_init(gko_rng* r, uint64_t seed, uint64_t stream) {
  r->state = gko_mix64(seed) ^ gko_mix64(~stream);
}

/* rng.hpp:29-35 */
uint64_t gko_rng_next(gko_rng* r) {
  r->state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = r->state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* rng.hpp:38-50: masked rejection on the high 32 bits */
uint32_t gko_rng_bounded(gko_rng* r, uint32_t bound) {
  uint32_t mask = bound - 1;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  for (;;) {
    uint32_t v = (uint32_t)(gko_rng_next(r) >> 32) & mask;
    if (v < bound) return v;
  }
}

/* rng.hpp:53 */
double gko_rng_unit(gko_rng* r) {
  return (double)(gko_rng_next(r) >> 11) * 0x1.0p-53;
}

/* ---- generator.hpp:56-77 (GenerateUniform) ----------------------------- */
int64_t gko_gen_urand(int scale, int degree, uint64_t seed, uint32_t* edges) {
  const int64_t n = (int64_t)1 << scale;
  const int64_t m = (int64_t)degree * n;
  const uint32_t bound = (uint32_t)n;
  const int64_t blocks = (m + GKO_GEN_BLOCK - 1) / GKO_GEN_BLOCK;
  for (int64_t b = 0; b < blocks; b++) {
    gko_rng r;
    gko_rng_init(&r, seed, GKO_EDGE_STREAM | (uint64_t)b);
    int64_t end = (b + 1) * GKO_GEN_BLOCK;
    if (end > m) end = m;
    for (int64_t i = b * GKO_GEN_BLOCK; i < end; i++) {
      uint32_t s = gko_rng_bounded(&r, bound);
      uint32_t d = gko_rng_bounded(&r, bound);
      edges[2 * i] = s;
      edges[2 * i + 1] = d;
    }
  }
  return m;
}

/* ---- generator.hpp:79-112 (GenerateKronecker; A=.57 B=.19 C=.19) ------- */
int64_t gko_gen_kron(int scale, int degree, uint64_t seed, uint32_t* edges) {
  const double kA = 0.57, kB = 0.19, kC = 0.19;
  const double ab = kA + kB;       /* generator.hpp:99 */
  const double abc = kA + kB + kC; /* generator.hpp:103 */
  const int64_t n = (int64_t)1 << scale;
  const int64_t m = (int64_t)degree * n;
  const int64_t blocks = (m + GKO_GEN_BLOCK - 1) / GKO_GEN_BLOCK;
  for (int64_t b = 0; b < blocks; b++) {
    gko_rng r;
    gko_rng_init(&r, seed, GKO_EDGE_STREAM | (uint64_t)b);
    int64_t end = (b + 1) * GKO_GEN_BLOCK;
    if (end > m) end = m;
    for (int64_t i = b * GKO_GEN_BLOCK; i < end; i++) {
      uint32_t s = 0, d = 0;
      for (int depth = 0; depth < scale; depth++) {
        double p = gko_rng_unit(&r);
        s <<= 1;
        d <<= 1;
        if (p < ab) {
          if (p > kA) d |= 1;
        } else {
          s |= 1;
          if (p > abc) d |= 1;
        }
      }
      edges[2 * i] = s;
      edges[2 * i + 1] = d;
    }
  }
  return m;
}

/* ---- seeded ID permutation (new) -------
 * Four rounds of {multiply by an odd key, add a key, xorshift} modulo
 * 2^scale.  Each step is a bijection on scale-bit integers, so the
 * composition is one.  Keys come from Rng(seed, GKO_PERM_STREAM). */
void gko_perm_keys(uint64_t seed, int scale, uint64_t keys[8]) {
  gko_rng r;
  gko_rng_init(&r, seed, GKO_PERM_STREAM | (uint64_t)scale);
  for (int i = 0; i < 8; i++) keys[i] = gko_rng_next(&r);
  for (int i = 0; i < 4; i++) keys[2 * i] |= 1ULL; /* odd multipliers */
}

uint32_t gko_permute(uint32_t v, int scale, const uint64_t keys[8]) {
  if (scale <= 0) return v;
  const uint64_t mask = (scale >= 64) ? ~0ULL : ((1ULL << scale) - 1);
  const int sh = (scale + 1) / 2;
  uint64_t x = v;
  for (int i = 0; i < 4; i++) {
    x = (x * keys[2 * i]) & mask;
    x = (x + keys[2 * i + 1]) & mask;
    x ^= x >> sh;
  }
  return (uint32_t)x;
}

void gko_permute_edges(uint32_t* edges, int64_t m, int scale, uint64_t seed) {
  uint64_t keys[8];
  gko_perm_keys(seed, scale, keys);
  for (int64_t i = 0; i < 2 * m; i++) edges[i] = gko_permute(edges[i], scale, keys);
}

/* ---- road-like grid (new; BASELINE config 4) ----------------------------
 * rows x cols cells, vertex (r,c) = r*cols + c.  Base 4-neighbour edges are
 * indexed horizontals first (r*(cols-1)+c), then verticals (H + r*cols+c);
 * edge i is deleted when the i-th draw of its 1024-edge block stream
 * Rng(seed, GRID_DEL|block) has NextUnit() < p_delete.  Every cell with a
 * row below owns one diagonal slot: its block stream Rng(seed,
 * GRID_DIAG|block) draws NextUnit(); if < p_diag a second draw's top bit
 * picks (r+1,c+1) or (r+1,c-1) (reflected at the border). */
int64_t gko_grid_max_edges(int64_t rows, int64_t cols) {
  int64_t h = rows * (cols - 1), v = (rows - 1) * cols;
  if (h < 0) h = 0;
  if (v < 0) v = 0;
  return h + v + (rows > 1 ? (rows - 1) * cols : 0);
}

int64_t gko_gen_grid(int64_t rows, int64_t cols, double p_delete,
                     double p_diag, uint64_t seed, uint32_t* edges) {
  const int64_t H = rows * (cols - 1) > 0 ? rows * (cols - 1) : 0;
  const int64_t V = (rows - 1) * cols > 0 ? (rows - 1) * cols : 0;
  const int64_t B = H + V;
  int64_t out = 0;
  for (int64_t b = 0; b * GKO_GEN_BLOCK < B; b++) {
    gko_rng r;
    gko_rng_init(&r, seed, GKO_GRID_DEL_STREAM | (uint64_t)b);
    int64_t end = (b + 1) * GKO_GEN_BLOCK;
    if (end > B) end = B;
    for (int64_t i = b * GKO_GEN_BLOCK; i < end; i++) {
      double u = gko_rng_unit(&r);
      if (u < p_delete) continue;
      int64_t a, c2;
      if (i < H) {
        int64_t rr = i / (cols - 1), cc = i % (cols - 1);
        a = rr * cols + cc;
        c2 = a + 1;
      } else {
        int64_t j = i - H;
        a = j;
        c2 = j + cols;
      }
      edges[2 * out] = (uint32_t)a;
      edges[2 * out + 1] = (uint32_t)c2;
      out++;
    }
  }
  const int64_t D = V; /* cells with a row below */
  if (cols > 1) {
    for (int64_t b = 0; b * GKO_GEN_BLOCK < D; b++) {
      gko_rng r;
      gko_rng_init(&r, seed, GKO_GRID_DIAG_STREAM | (uint64_t)b);
      int64_t end = (b + 1) * GKO_GEN_BLOCK;
      if (end > D) end = D;
      for (int64_t j = b * GKO_GEN_BLOCK; j < end; j++) {
        double u = gko_rng_unit(&r);
        if (!(u < p_diag)) continue;
        int64_t d = (gko_rng_next(&r) >> 63) ? 1 : -1;
        int64_t cc = j % cols;
        if (cc + d < 0 || cc + d >= cols) d = -d;
        edges[2 * out] = (uint32_t)j;
        edges[2 * out + 1] = (uint32_t)(j + cols + d);
        out++;
      }
    }
  }
  return out;
}

/* ---- builder.hpp:54-186 (BuildCsr, unweighted) --------------------------
 * Self-loops dropped; neighbours sorted ascending; duplicates collapsed.
 * The reference sorts (neighbour, origin) pairs; for unweighted graphs the
 * origin only breaks ties between equal neighbours, which dedup removes, so
 * sorting bare neighbour ids yields the same arrays. */
static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

int64_t gko_build_csr(int64_t n, const uint32_t* edges, int64_t m,
                      int symmetrize, int64_t* offsets, uint32_t* neighbors) {
  for (int64_t i = 0; i < 2 * m; i++)
    if ((int64_t)edges[i] >= n) return -1; /* builder.hpp:66-67 */
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t i = 0; i < m; i++) { /* builder.hpp:76-82 */
    uint32_t s = edges[2 * i], d = edges[2 * i + 1];
    if (s == d) continue;
    cnt[(int64_t)s + 1]++;
    if (symmetrize) cnt[(int64_t)d + 1]++;
  }
  for (int64_t v = 0; v < n; v++) cnt[v + 1] += cnt[v];
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
  memcpy(cur, cnt, sizeof(int64_t) * ((size_t)n + 1));
  for (int64_t i = 0; i < m; i++) { /* builder.hpp:86-98 */
    uint32_t s = edges[2 * i], d = edges[2 * i + 1];
    if (s == d) continue;
    neighbors[cur[s]++] = d;
    if (symmetrize) neighbors[cur[d]++] = s;
  }
  free(cur);
  /* builder.hpp:101-116: sort + dedup in place, then compact. */
  int64_t w = 0;
  offsets[0] = 0;
  for (int64_t v = 0; v < n; v++) {
    int64_t b = cnt[v], e = cnt[v + 1];
    qsort(neighbors + b, (size_t)(e - b), sizeof(uint32_t), cmp_u32);
    for (int64_t j = b; j < e; j++) {
      if (j > b && neighbors[j] == neighbors[j - 1]) continue;
      neighbors[w++] = neighbors[j];
    }
    offsets[v + 1] = w;
  }
  free(cnt);
  return w;
}

/* builder.hpp:139-173: transpose of the deduped out-edges, sorted. */
void gko_transpose(int64_t n, const int64_t* off, const uint32_t* nb,
                   int64_t* in_off, uint32_t* in_nb) {
  memset(in_off, 0, sizeof(int64_t) * ((size_t)n + 1));
  const int64_t m = off[n];
  for (int64_t j = 0; j < m; j++) in_off[(int64_t)nb[j] + 1]++;
  for (int64_t v = 0; v < n; v++) in_off[v + 1] += in_off[v];
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
  memcpy(cur, in_off, sizeof(int64_t) * ((size_t)n + 1));
  /* u ascending, so each in-list comes out sorted without a sort. */
  for (int64_t u = 0; u < n; u++)
    for (int64_t j = off[u]; j < off[u + 1]; j++) in_nb[cur[nb[j]]++] = (uint32_t)u;
  free(cur);
}

/* ---- source_picker.hpp:22-54 ------------------------------------------- */
int gko_pick_sources(int64_t n, const int64_t* off, int64_t count,
                     uint64_t seed, uint32_t* out) {
  if (off[n] == 0) return -1; /* "cannot pick sources: graph has no edges" */
  gko_rng r;
  gko_rng_init(&r, seed, 0); /* Rng(seed) : stream defaults to 0 */
  for (int64_t i = 0; i < count; i++) {
    uint32_t c;
    do {
      c = gko_rng_bounded(&r, (uint32_t)n);
    } while (off[c + 1] - off[c] == 0);
    out[i] = c;
  }
  return 0;
}

/* ---- verify.hpp:42-58 (detail::BfsDepths) ------------------------------ */
void gko_bfs_depths(int64_t n, const int64_t* off, const uint32_t* nb,
                    uint32_t src, int32_t* depth) {
  uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t v = 0; v < n; v++) depth[v] = -1;
  int64_t head = 0, tail = 0;
  depth[src] = 0;
  q[tail++] = src;
  while (head < tail) {
    uint32_t u = q[head++];
    for (int64_t j = off[u]; j < off[u + 1]; j++) {
      uint32_t v = nb[j];
      if (depth[v] == -1) {
        depth[v] = depth[u] + 1;
        q[tail++] = v;
      }
    }
  }
  free(q);
}

/* graph.hpp:82-85 */
static int has_edge(const int64_t* off, const uint32_t* nb, uint32_t u, uint32_t v) {
  int64_t lo = off[u], hi = off[u + 1];
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (nb[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo < off[u + 1] && nb[lo] == v;
}

/* ---- verify.hpp:62-98 (VerifyBfs); messages follow the reference ------- */
int gko_verify_bfs(int64_t n, const int64_t* off, const uint32_t* nb,
                   uint32_t src, const int32_t* parent, char* msg, int msglen) {
  if (msg && msglen > 0) msg[0] = 0;
  if (parent[src] != (int32_t)src) {
    if (msg) snprintf(msg, (size_t)msglen, "parent[source] != source at vertex %u", src);
    return 0;
  }
  int32_t* depth = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  gko_bfs_depths(n, off, nb, src, depth);
  int ok = 1;
  for (int64_t v = 0; v < n && ok; v++) {
    if (depth[v] == -1) {
      if (parent[v] != -1) {
        if (msg) snprintf(msg, (size_t)msglen, "unreachable vertex %lld has parent %d", (long long)v, parent[v]);
        ok = 0;
      }
      continue;
    }
    if (v == (int64_t)src) continue;
    int32_t p = parent[v];
    if (p < 0) {
      if (msg) snprintf(msg, (size_t)msglen, "reachable vertex %lld marked unreached", (long long)v);
      ok = 0;
    } else if ((int64_t)p >= n) {
      if (msg) snprintf(msg, (size_t)msglen, "parent id out of range at vertex %lld", (long long)v);
      ok = 0;
    } else if (!has_edge(off, nb, (uint32_t)p, (uint32_t)v)) {
      if (msg) snprintf(msg, (size_t)msglen, "no edge (%d,%lld) for claimed parent", p, (long long)v);
      ok = 0;
    } else if (depth[p] != depth[v] - 1) {
      if (msg) snprintf(msg, (size_t)msglen, "parent of vertex %lld has depth %d, expected %d", (long long)v, depth[p], depth[v] - 1);
      ok = 0;
    }
  }
  free(depth);
  return ok;
}

/* ---- bfs.hpp:117-177 (Bfs), serial restatement --------------------------
 * The claimed set, scout/awake counts and the direction sequence are pure
 * functions of (graph, source, alpha, beta, strategy); top-down parents are
 * the serial (first-claimer) choice, bottom-up parents are exactly the
 * reference's (first in-neighbour in ascending order with its front bit). */
int64_t gko_bfs_replay(int64_t n, int64_t m_arcs, const int64_t* out_off,
                       const uint32_t* out_nb, const int64_t* in_off,
                       const uint32_t* in_nb, uint32_t src, int64_t alpha,
                       int64_t beta, int strategy, int32_t* parent,
                       gko_step* steps, int64_t max_steps) {
  if ((int64_t)src >= n) return -1; /* bfs.hpp:120-121 */
  if (alpha <= 0 || beta <= 0) return -1; /* bfs.hpp:122-123 */
  const int encode = strategy != GKO_TD_RESCAN; /* bfs.hpp:125 */
  for (int64_t v = 0; v < n; v++) { /* bfs.hpp:126-131 */
    int64_t deg = encode ? out_off[v + 1] - out_off[v] : 0;
    parent[v] = deg != 0 ? (int32_t)(-deg) : -1;
  }
  parent[src] = (int32_t)src; /* bfs.hpp:132 */
  uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n + 1));
  uint8_t* front = (uint8_t*)calloc((size_t)n + 1, 1);
  uint8_t* next = (uint8_t*)calloc((size_t)n + 1, 1);
  int64_t tail = 0, qs = 0, qe = 0;
  q[tail++] = src;
  qs = qe; qe = tail; /* SlideWindow */
  int64_t edges_to_check = m_arcs;                    /* bfs.hpp:139 */
  int64_t scout = out_off[src + 1] - out_off[src];    /* bfs.hpp:140 */
  int64_t ns = 0;
  while (qe > qs) {
    if (strategy == GKO_DO && scout > edges_to_check / alpha) { /* :143-144 */
      memset(front, 0, (size_t)n);
      for (int64_t i = qs; i < qe; i++) front[q[i]] = 1; /* QueueToBitmap */
      int64_t awake = qe - qs;
      qs = qe; qe = tail;
      int64_t old_awake;
      do { /* bfs.hpp:149-154 */
        old_awake = awake;
        memset(next, 0, (size_t)n);
        awake = 0;
        for (int64_t v = 0; v < n; v++) { /* BfsBottomUpStep bfs.hpp:47-66 */
          if (parent[v] < 0) {
            for (int64_t j = in_off[v]; j < in_off[v + 1]; j++) {
              uint32_t u = in_nb[j];
              if (front[u]) {
                parent[v] = (int32_t)u;
                awake++;
                next[v] = 1;
                break;
              }
            }
          }
        }
        uint8_t* t = front; front = next; next = t;
        if (ns < max_steps && steps) {
          steps[ns].dir = 'B'; steps[ns].pad = 0;
          steps[ns].frontier = old_awake; steps[ns].result = awake;
          steps[ns].edges_to_check = edges_to_check;
        }
        ns++;
      } while (awake >= old_awake || awake > n / beta);
      for (int64_t v = 0; v < n; v++) /* BitmapToQueue bfs.hpp:99-113 */
        if (front[v]) q[tail++] = (uint32_t)v;
      qs = qe; qe = tail;
      scout = 1; /* bfs.hpp:156 */
    } else {
      edges_to_check -= scout; /* bfs.hpp:158 */
      int64_t fsize = qe - qs;
      scout = 0;
      for (int64_t i = qs; i < qe; i++) { /* BfsTopDownStep bfs.hpp:68-91 */
        uint32_t u = q[i];
        for (int64_t j = out_off[u]; j < out_off[u + 1]; j++) {
          uint32_t v = out_nb[j];
          int32_t cur = parent[v];
          if (cur < 0) {
            parent[v] = (int32_t)u;
            q[tail++] = v;
            scout += -(int64_t)cur;
          }
        }
      }
      qs = qe; qe = tail;
      if (strategy == GKO_TD_RESCAN) { /* bfs.hpp:161-167 */
        int64_t tot = 0;
        for (int64_t i = qs; i < qe; i++) tot += out_off[q[i] + 1] - out_off[q[i]];
        scout = tot;
      }
      if (ns < max_steps && steps) {
        steps[ns].dir = 'T'; steps[ns].pad = 0;
        steps[ns].frontier = fsize; steps[ns].result = scout;
        steps[ns].edges_to_check = edges_to_check;
      }
      ns++;
    }
  }
  for (int64_t v = 0; v < n; v++) /* bfs.hpp:171-175 */
    if (parent[v] < 0) parent[v] = -1;
  free(q); free(front); free(next);
  return ns;
}

/* ---- byte model ---------------------------------------
 * Step i works on the level-i frontier {depth == i}:
 *  TD: sum_{u in F} (4 + 32 + sec(deg u)) + 36*|C|      (use: 4+8+4deg, 4|C|)
 *  BU: 3W + sum_{v in U} (8 + sec(s_v))                 (use: 8 + 4 s_v)
 *      U = unvisited vertices with in-degree > 0; s_v = in-arcs scanned up
 *      to and including the first with depth == i (all, when none).
 *  switch (TD->BU before a BU run, BU->TD after it): W + 4|F|.
 *  plus 4n for the parent array. */
static double sec_bytes(int64_t k) { return 32.0 * (double)((4 * k + 31) / 32); }

void gko_byte_model(int64_t n, const int64_t* out_off, const uint32_t* out_nb,
                    const int64_t* in_off, const uint32_t* in_nb,
                    const int32_t* depth, const char* dirs, int64_t n_steps,
                    double* b_sec, double* b_use) {
  (void)out_nb;
  const double W = (double)((n + 7) / 8);
  int32_t maxd = -1;
  for (int64_t v = 0; v < n; v++) if (depth[v] > maxd) maxd = depth[v];
  int64_t L = (int64_t)maxd + 2;
  if (L < n_steps + 1) L = n_steps + 1;
  int64_t* cnt = (int64_t*)calloc((size_t)L + 1, sizeof(int64_t));
  double* td_sec = (double*)calloc((size_t)L + 1, sizeof(double));
  double* td_use = (double*)calloc((size_t)L + 1, sizeof(double));
  for (int64_t v = 0; v < n; v++) {
    int32_t d = depth[v];
    if (d < 0) continue;
    int64_t deg = out_off[v + 1] - out_off[v];
    cnt[d]++;
    td_sec[d] += 4.0 + 32.0 + sec_bytes(deg);
    td_use[d] += 4.0 + 8.0 + 4.0 * (double)deg;
  }
  double bs = 4.0 * (double)n, bu = 4.0 * (double)n;
  for (int64_t i = 0; i < n_steps; i++) {
    if (dirs[i] == 'T') {
      bs += td_sec[i] + 36.0 * (double)cnt[i + 1];
      bu += td_use[i] + 4.0 * (double)cnt[i + 1];
    } else {
      if (i == 0 || dirs[i - 1] != 'B') { bs += W + 4.0 * cnt[i]; bu += W + 4.0 * cnt[i]; }
      bs += 3.0 * W; bu += 3.0 * W;
      for (int64_t v = 0; v < n; v++) {
        int32_t d = depth[v];
        if (d >= 0 && d <= i) continue; /* visited before this step */
        int64_t b = in_off[v], e = in_off[v + 1];
        if (e == b) continue; /* isolated */
        int64_t s = e - b;
        for (int64_t j = b; j < e; j++)
          if (depth[in_nb[j]] == (int32_t)i) { s = j - b + 1; break; }
        bs += 8.0 + sec_bytes(s);
        bu += 8.0 + 4.0 * (double)s;
      }
      if (i + 1 == n_steps || dirs[i + 1] != 'B') { bs += W + 4.0 * cnt[i + 1]; bu += W + 4.0 * cnt[i + 1]; }
    }
  }
  free(cnt); free(td_sec); free(td_use);
  *b_sec = bs;
  *b_use = bu;
}

int64_t gko_component_edges(int64_t n, const int64_t* off,
                            const int32_t* depth_or_parent, int directed) {
  int64_t s = 0;
  for (int64_t v = 0; v < n; v++)
    if (depth_or_parent[v] >= 0) s += off[v + 1] - off[v];
  return directed ? s : s / 2;
}

/* benchmark.hpp:127-135 */
uint64_t gko_fnv1a(const void* data, int64_t len) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 14695981039346656037ULL;
  for (int64_t i = 0; i < len; i++) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}


/* ---- Brandes betweenness (betweenness.hpp:38-145), serial restatement ----
 * Test infrastructure only.  Forward: level-synchronous BFS over out-edges
 * counting shortest paths (sigma) and flagging successor edges (one flag per
 * stored arc), betweenness.hpp:38-80 run serially.  Backward: levels deepest
 * first, delta(u) = sum over flagged arcs (u,v), in arc order, of
 * sigma(u)/sigma(v) * (1 + delta(v)); scores(u) += (float)delta(u) for u !=
 * source (betweenness.hpp:104-122).  Then max normalisation (:129-143).
 * Returns 0, or -1 for no sources, -2 out of range, -3 zero out-degree. */
int gko_brandes(int64_t n, const int64_t* off, const uint32_t* nb, const uint32_t* sources,
                int64_t count, float* scores) {
  if (count <= 0) return -1;
  for (int64_t i = 0; i < count; i++) {
    if ((int64_t)sources[i] >= n) return -2;
    if (off[sources[i] + 1] == off[sources[i]]) return -3;
  }
  const int64_t m = off[n];
  double* sigma = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double* delta = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  int32_t* depth = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  uint32_t* q = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(n > 0 ? n : 1));
  int64_t* bounds = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 2));
  uint8_t* succ = (uint8_t*)malloc((size_t)(m > 0 ? m : 1));
  for (int64_t v = 0; v < n; v++) scores[v] = 0.0f;
  for (int64_t si = 0; si < count; si++) {
    const uint32_t src = sources[si];
    for (int64_t v = 0; v < n; v++) {
      sigma[v] = 0.0;
      depth[v] = -1;
    }
    memset(succ, 0, (size_t)(m > 0 ? m : 1));
    depth[src] = 0;
    sigma[src] = 1.0;
    int64_t tail = 0, nb_levels = 0;
    q[tail++] = src;
    bounds[nb_levels++] = 0;
    int64_t qs = 0, qe = 1;
    int32_t d = 0;
    while (qs < qe) {
      d++;
      for (int64_t i = qs; i < qe; i++) {
        const uint32_t u = q[i];
        for (int64_t j = off[u]; j < off[u + 1]; j++) {
          const uint32_t v = nb[j];
          if (depth[v] == -1) {
            depth[v] = d;
            q[tail++] = v;
          }
          if (depth[v] == d) {
            succ[j] = 1;
            sigma[v] += sigma[u];
          }
        }
      }
      bounds[nb_levels++] = qe;
      qs = qe;
      qe = tail;
    }
    /* bounds[] = level starts, ending with the empty window */
    for (int64_t v = 0; v < n; v++) delta[v] = 0.0;
    for (int64_t l = nb_levels - 2; l >= 0; l--) {
      for (int64_t i = bounds[l]; i < bounds[l + 1]; i++) {
        const uint32_t u = q[i];
        double du = 0.0;
        for (int64_t j = off[u]; j < off[u + 1]; j++)
          if (succ[j]) du += (sigma[u] / sigma[nb[j]]) * (1.0 + delta[nb[j]]);
        delta[u] = du;
        if (u != src) scores[u] += (float)du;
      }
    }
  }
  float mx = 0.0f;
  for (int64_t v = 0; v < n; v++)
    if (scores[v] > mx) mx = scores[v];
  if (mx > 0.0f)
    for (int64_t v = 0; v < n; v++) scores[v] /= mx;
  free(sigma);
  free(delta);
  free(depth);
  free(q);
  free(bounds);
  free(succ);
  return 0;
}

/*
 * fw_oracle.c — CPU oracle for blocked Floyd–Warshall APSP (arxiv 1811.01201).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_1811_01201_b200/, include/fw.h) shares no code, header, table or helper
 * with this file, and never calls it.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * SURVEY §8(c) = /root/repo/SURVEY.md "Oracle" section; DESIGN.md "Readings".
 *
 * Contents
 *  - oracle_fw_f32 / oracle_fw_i32: the naive triple-loop Floyd–Warshall of the
 *    paper's Fig. 1, reconstructed from the prose ("at k-th iteration it
 *    evaluates all the possible paths between each pair of vertices from i to j
 *    through the intermediate vertex k"; P:125 loop body "one addition, one
 *    comparison and (may be) two assign operations"). Strict '<' (reading R2),
 *    ties keep the old value. P is the next-hop matrix (reading R1) or, in
 *    LAST_K mode, the paper's "most recently added intermediate node".
 *    Plain C float / int32 arithmetic, compiled without fast-math or FP
 *    contraction: every sum is one IEEE round-to-nearest add.
 *  - oracle_dijkstra_*: Dijkstra from a list of sources (dense O(n^2) per source),
 *    sums in double / int64 (exact for these inputs). Independent algorithm used to
 *    pin the FW oracle and to check sizes the triple loop cannot finish (BJ:5).
 *  - oracle_bruteforce_f64: exhaustive simple-path enumeration, n <= 8.
 *  - oracle_minplus_closure_f64: repeated min-plus squaring, n <= 64.
 *  - oracle_check_next / oracle_check_lastk: path validity by walking / expanding P
 *    and summing the original edge weights (BJ:5 "P is validated by reconstructing
 *    every checked path and summing its edge weights to D").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_INF_I32 0x3FFFFFFF /* BJ:9 INT32_MAX/2 */

/* ---- Floyd–Warshall, FP32 --------------------------------------------------
 * D: in = adjacency W (n x n row-major, +inf = no edge), out = distances.
 * P: NULL, or out: mode 0 = next hop, mode 1 = last intermediate k (-1 = none).
 * The diagonal is forced to 0 first (reading R4). Returns 0. */
int oracle_fw_f32(float *D, int32_t *P, int64_t n, int mode) {
  for (int64_t i = 0; i < n; ++i) D[i * n + i] = 0.0f;
  if (P) {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) {
        int32_t v;
        if (mode == 1) v = -1;                       /* S:35-41 NO_INTERMEDIATE */
        else if (i == j) v = (int32_t)i;             /* next hop of (i,i) is i */
        else v = isinf(D[i * n + j]) ? -1 : (int32_t)j;  /* direct edge or none */
        P[i * n + j] = v;
      }
  }
  for (int64_t k = 0; k < n; ++k) {
    const float *Dk = D + k * n;
    /* Row k and column k do not change during step k because D[k][k] = 0, so the
       i-iterations are independent (parallelising over i does not change results). */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      float *Di = D + i * n;
      const float dik = Di[k];
      if (isinf(dik)) continue;   /* every sum would be +inf: no strict improvement */
      int32_t *Pi = P ? P + i * n : NULL;
      const int32_t pik = P ? Pi[k] : 0;
      for (int64_t j = 0; j < n; ++j) {
        const float s = dik + Dk[j];
        if (s < Di[j]) {
          Di[j] = s;
          if (Pi) Pi[j] = (mode == 1) ? (int32_t)k : pik;
        }
      }
    }
  }
  return 0;
}

/* ---- bounded sample: outer iterations k in [k0, k1) of the same FP32 triple loop ----------
 * Used only by bench.py's cpu_baseline / --impl reference legs to time the oracle on a
 * bounded slice of the benchmark workload (each k-step is n^2 relaxations). D must
 * already hold W with a zero diagonal; P (next-hop) may be NULL. */
int oracle_fw_f32_steps(float *D, int32_t *P, int64_t n, int64_t k0, int64_t k1) {
  for (int64_t k = k0; k < k1 && k < n; ++k) {
    const float *Dk = D + k * n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      float *Di = D + i * n;
      const float dik = Di[k];
      if (isinf(dik)) continue;
      int32_t *Pi = P ? P + i * n : NULL;
      const int32_t pik = P ? Pi[k] : 0;
      for (int64_t j = 0; j < n; ++j) {
        const float s = dik + Dk[j];
        if (s < Di[j]) {
          Di[j] = s;
          if (Pi) Pi[j] = pik;
        }
      }
    }
  }
  return 0;
}

/* ---- Floyd–Warshall, INT32 (INF = 0x3FFFFFFF, sums of two values <= 2^31-2) ---- */
int oracle_fw_i32(int32_t *D, int32_t *P, int64_t n, int mode) {
  for (int64_t i = 0; i < n; ++i) D[i * n + i] = 0;
  if (P) {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) {
        int32_t v;
        if (mode == 1) v = -1;
        else if (i == j) v = (int32_t)i;
        else v = (D[i * n + j] >= ORACLE_INF_I32) ? -1 : (int32_t)j;
        P[i * n + j] = v;
      }
  }
  for (int64_t k = 0; k < n; ++k) {
    const int32_t *Dk = D + k * n;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      int32_t *Di = D + i * n;
      const int32_t dik = Di[k];
      if (dik >= ORACLE_INF_I32) continue;
      int32_t *Pi = P ? P + i * n : NULL;
      const int32_t pik = P ? Pi[k] : 0;
      for (int64_t j = 0; j < n; ++j) {
        const int32_t s = dik + Dk[j];   /* <= 2*(2^30-1): no overflow */
        if (s < Di[j]) {
          Di[j] = s;
          if (Pi) Pi[j] = (mode == 1) ? (int32_t)k : pik;
        }
      }
    }
  }
  return 0;
}

/* ---- Dijkstra (dense, O(n^2) per source) ---------------------------------------
 * out[s*n + v] = exact shortest distance src[s] -> v as double (FP32 weights summed
 * in double: exact for <= 2^29 terms of 24-bit mantissas within range), +inf if
 * unreachable. Weights: +inf = no edge. The diagonal of W is ignored. */
int oracle_dijkstra_f32(const float *W, int64_t n, const int64_t *src, int64_t nsrc, double *out) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (int64_t s = 0; s < nsrc; ++s) {
    double *dist = out + s * n;
    unsigned char *done = (unsigned char *)calloc((size_t)n, 1);
    if (!done) { bad = 1; continue; }
    for (int64_t v = 0; v < n; ++v) dist[v] = INFINITY;
    dist[src[s]] = 0.0;
    for (int64_t it = 0; it < n; ++it) {
      int64_t u = -1; double best = INFINITY;
      for (int64_t v = 0; v < n; ++v)
        if (!done[v] && dist[v] < best) { best = dist[v]; u = v; }
      if (u < 0) break;
      done[u] = 1;
      const float *Wu = W + u * n;
      for (int64_t v = 0; v < n; ++v) {
        if (v == u || done[v] || isinf(Wu[v])) continue;
        const double c = best + (double)Wu[v];
        if (c < dist[v]) dist[v] = c;
      }
    }
    free(done);
  }
  return bad ? 2 : 0;
}

/* INT32 weights (INF_I32 = no edge); out in int64, unreachable = INT64_MAX. */
int oracle_dijkstra_i32(const int32_t *W, int64_t n, const int64_t *src, int64_t nsrc, int64_t *out) {
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : bad)
  for (int64_t s = 0; s < nsrc; ++s) {
    int64_t *dist = out + s * n;
    unsigned char *done = (unsigned char *)calloc((size_t)n, 1);
    if (!done) { bad = 1; continue; }
    for (int64_t v = 0; v < n; ++v) dist[v] = INT64_MAX;
    dist[src[s]] = 0;
    for (int64_t it = 0; it < n; ++it) {
      int64_t u = -1, best = INT64_MAX;
      for (int64_t v = 0; v < n; ++v)
        if (!done[v] && dist[v] < best) { best = dist[v]; u = v; }
      if (u < 0) break;
      done[u] = 1;
      const int32_t *Wu = W + u * n;
      for (int64_t v = 0; v < n; ++v) {
        if (v == u || done[v] || Wu[v] >= ORACLE_INF_I32) continue;
        const int64_t c = best + (int64_t)Wu[v];
        if (c < dist[v]) dist[v] = c;
      }
    }
    free(done);
  }
  return bad ? 2 : 0;
}

/* ---- brute force: minimum over all simple paths (DFS), n <= 8 -------------------- */
static void bf_dfs(const double *W, int64_t n, int64_t src, int64_t u, double len,
                   unsigned visited, double *row) {
  if (len < row[u]) row[u] = len;
  for (int64_t v = 0; v < n; ++v) {
    if ((visited >> v) & 1u) continue;
    if (isinf(W[u * n + v])) continue;
    bf_dfs(W, n, src, v, len + W[u * n + v], visited | (1u << v), row);
  }
}

int oracle_bruteforce_f64(const double *W, int64_t n, double *out) {
  if (n > 10) return 1;
  for (int64_t i = 0; i < n; ++i) {
    double *row = out + i * n;
    for (int64_t j = 0; j < n; ++j) row[j] = INFINITY;
    bf_dfs(W, n, i, i, 0.0, 1u << i, row);   /* the empty path gives row[i] = 0 */
  }
  return 0;
}

/* ---- min-plus closure by repeated squaring, n <= 64 -----------------------
 * M_0 = W with zero diagonal; M_{t+1}[i][j] = min_k M_t[i][k] + M_t[k][j];
 * ceil(log2(n)) squarings cover every simple path (<= n-1 edges). */
int oracle_minplus_closure_f64(const double *W, int64_t n, double *out) {
  if (n > 4096) return 1;
  double *M = (double *)malloc(sizeof(double) * n * n);
  double *T = (double *)malloc(sizeof(double) * n * n);
  if (!M || !T) { free(M); free(T); return 2; }
  memcpy(M, W, sizeof(double) * n * n);
  for (int64_t i = 0; i < n; ++i) M[i * n + i] = 0.0;
  int64_t reach = 1;
  while (reach < n - 1) {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) {
        double best = INFINITY;
        for (int64_t k = 0; k < n; ++k) {
          const double c = M[i * n + k] + M[k * n + j];
          if (c < best) best = c;
        }
        T[i * n + j] = best;
      }
    memcpy(M, T, sizeof(double) * n * n);
    reach *= 2;
  }
  memcpy(out, M, sizeof(double) * n * n);
  free(M); free(T);
  return 0;
}

/* ---- path validity --------------------------------------------------------------
 * Wd: original weights as double (+inf = no edge), Dd: the distances under test as
 * double (+inf = unreachable), P: int32 path matrix, rows: the source rows to check.
 * For every checked (i,j):
 *   i == j        : next-hop mode requires P == i; LAST_K mode requires P == -1;
 *   D == inf      : P must be -1;
 *   otherwise     : reconstruct the path and require (a) every hop is an edge,
 *                   (b) at most n-1 hops, (c) |sum - D| <= rtol * max(1, |D|)
 *                   (rtol = 0 demands exact equality; used for integer data).
 * Returns the number of failing pairs (0 = all valid); *first_bad = i*n+j of the first. */
int64_t oracle_check_next(const double *Wd, const double *Dd, const int32_t *P, int64_t n,
                          const int64_t *rows, int64_t nrows, double rtol, int64_t *first_bad) {
  int64_t bad = 0, first = -1;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : bad)
  for (int64_t r = 0; r < nrows; ++r) {
    const int64_t i = rows[r];
    for (int64_t j = 0; j < n; ++j) {
      const int32_t p = P[i * n + j];
      const double d = Dd[i * n + j];
      int ok = 1;
      if (i == j) ok = (p == (int32_t)i) && d == 0.0;
      else if (isinf(d)) ok = (p == -1);
      else {
        int64_t cur = i, hops = 0;
        double sum = 0.0;
        while (cur != j) {
          const int32_t h = P[cur * n + j];
          if (h < 0 || h >= n || isinf(Wd[cur * n + h]) || h == cur || ++hops > n - 1) { ok = 0; break; }
          sum += Wd[cur * n + h];
          cur = h;
        }
        if (ok) ok = fabs(sum - d) <= rtol * fmax(1.0, fabs(d));
      }
      if (!ok) {
        ++bad;
#pragma omp critical
        { if (first < 0 || i * n + j < first) first = i * n + j; }
      }
    }
  }
  if (first_bad) *first_bad = first;
  return bad;
}

/* LAST_K mode: path(i,j) = path(i,k) ++ path(k,j) with k = P[i][j]; P = -1 means the
 * direct edge. Iterative expansion with an explicit stack. */
int64_t oracle_check_lastk(const double *Wd, const double *Dd, const int32_t *P, int64_t n,
                           const int64_t *rows, int64_t nrows, double rtol, int64_t *first_bad) {
  int64_t bad = 0, first = -1;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : bad)
  for (int64_t r = 0; r < nrows; ++r) {
    const int64_t i = rows[r];
    int64_t *stk = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)(n + 2));
    for (int64_t j = 0; j < n; ++j) {
      const int32_t p = P[i * n + j];
      const double d = Dd[i * n + j];
      int ok = 1;
      if (i == j) ok = (p == -1) && d == 0.0;
      else if (isinf(d)) ok = (p == -1);
      else if (!stk) ok = 0;
      else {
        int64_t top = 0, edges = 0;
        double sum = 0.0;
        stk[top++] = i; stk[top++] = j;
        while (top > 0 && ok) {
          const int64_t b = stk[--top], a = stk[--top];
          const int32_t k = P[a * n + b];
          if (k < 0) {
            if (isinf(Wd[a * n + b]) || a == b || ++edges > n - 1) ok = 0;
            else sum += Wd[a * n + b];
          } else {
            if (k >= n || k == a || k == b || top + 4 > 2 * (n + 2)) { ok = 0; break; }
            stk[top++] = k; stk[top++] = b;   /* second half, expanded after the first */
            stk[top++] = a; stk[top++] = k;
          }
        }
        if (ok) ok = fabs(sum - d) <= rtol * fmax(1.0, fabs(d));
      }
      if (!ok) {
        ++bad;
#pragma omp critical
        { if (first < 0 || i * n + j < first) first = i * n + j; }
      }
    }
    free(stk);
  }
  if (first_bad) *first_bad = first;
  return bad;
}

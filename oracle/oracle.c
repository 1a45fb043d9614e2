/*
 * oracle.c — the CPU ORACLE for the linear-chain CRF hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2002_00876_b200/) never includes, links or calls anything here, and
 * nothing here includes anything from the product path.  The only shared code
 * is the input generator tsgen/tsgen.h (integer index -> dyadic value), which
 * holds none of the method's arithmetic.
 *
 * Plain, slow, obviously correct: float64 everywhere, IEEE exp()/log() from
 * libm (no fast-math), single thread per sequence, threads only across the
 * batch.  Each function cites the passage it follows (P:n = /root/reference/PAPER.md
 * line n; S:n = SPEC.md line n; readings R1..R12 = DESIGN.md §2).
 *
 * What is computed ("the definition"):
 *   Score(z) = sum_{t < E_b} l[b,t,z_t,z_{t+1}]
 *   A_b      = log sum_z exp Score(z)
 *   mu[b,t,i,j] = sum_{z: z_t=i, z_{t+1}=j} exp(Score(z) - A_b) = dA/dl
 *   A*_b     = max_z Score(z);  z*_b canonical (R5)
 * via the classical two-pass algorithm the paper says it replaces, with
 * the stabilised log-semiring product of §6(c): q = max per output cell.
 *
 * Parity status: every exported function is pinned by tests/test_oracle_*.py
 * (brute-force enumeration, closed forms, finite differences, invariants).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../tsgen/tsgen.h"

/* Per-sequence flags: the documented contract values (DESIGN.md §2 R10/R11),
 * restated here independently of include/ts_b200.h. */
#define OR_F_EMPTY 1u
#define OR_F_NONFINITE 2u
#define OR_F_BADLEN 4u

#define OR_SEMI_LOG 0
#define OR_SEMI_MAX 1

/* ---------------------------------------------------------------------------
 * Semiring primitives (Table 2): Log = (LSE, +), Max = (max, +).
 * ------------------------------------------------------------------------- */

/* V[m,o] = (+)_n T[m,n] (x) U[n,o].  Log: V = log sum_n exp(T+U-q) + q with
 * q = max_n(T+U) per output cell (§6(c); reading R4); V = -inf if q = -inf.
 * Max: V = max_n (T+U). */
int oracle_semiring_matmul(int semiring, const double* T, const double* U, int64_t n, int64_t m,
                           int64_t o, double* V) {
  if (!T || !U || !V || n < 1 || m < 1 || o < 1) return 1;
  for (int64_t r = 0; r < n; ++r) {
    for (int64_t c = 0; c < o; ++c) {
      double q = -INFINITY;
      for (int64_t k = 0; k < m; ++k) {
        double v = T[r * m + k] + U[k * o + c];
        if (v > q) q = v;
      }
      if (semiring == OR_SEMI_MAX || q == -INFINITY) {
        V[r * o + c] = q;
        continue;
      }
      double s = 0.0;
      for (int64_t k = 0; k < m; ++k) s += exp(T[r * m + k] + U[k * o + c] - q);
      V[r * o + c] = log(s) + q;
    }
  }
  return 0;
}

/* ---------------------------------------------------------------------------
 * One sequence: forward-backward + marginals (P:187 two-pass; P:252-256 forward).
 * l is accessed through a getter so the same code serves a resident buffer and
 * the on-the-fly generator (huge configs).
 * ------------------------------------------------------------------------- */

typedef struct {
  const float* pot; /* [E][C][C] for this sequence, or NULL => generator */
  uint64_t seed;
  int s;
  int64_t b, E_global, C;
} pot_src;

static inline double pot_get(const pot_src* p, int64_t t, int64_t i, int64_t j) {
  if (p->pot) return (double)p->pot[(t * p->C + i) * p->C + j];
  return (double)tsgen_value(p->seed, p->s, tsgen_index(p->b, t, i, j, p->E_global, p->C));
}

/* Widen edge t's C x C tile into w[i*C+j] (fp32 -> fp64 is exact). */
static void load_tile(const pot_src* p, int64_t t, double* w) {
  for (int64_t i = 0; i < p->C; ++i)
    for (int64_t j = 0; j < p->C; ++j) w[i * p->C + j] = pot_get(p, t, i, j);
}

/* Returns flags; writes logz, and (if marg) mu for t < len-1, zero elsewhere.
 * If edges/n_edges given (sampled mode), marg is [n_edges][C][C] for those edges. */
static uint32_t seq_marginals(const pot_src* p, int64_t N, int32_t len, double* logz, double* marg,
                              const int64_t* edges, int64_t n_edges) {
  const int64_t C = p->C, E = N - 1;
  const int64_t CC = C * C;
  int64_t nout = edges ? n_edges : E;
  if (marg) memset(marg, 0, sizeof(double) * (size_t)(nout * CC));
  if (len < 1 || len > N) {
    *logz = NAN;
    return OR_F_BADLEN;
  }
  const int64_t Eb = (int64_t)len - 1; /* edges used (reading R10) */
  /* NONFINITE: NaN or +inf on a used edge (reading R11); -inf is a legal mask. */
  double* w = (double*)malloc(sizeof(double) * (size_t)CC); /* edge t's tile, fp64 */
  for (int64_t t = 0; t < Eb; ++t) {
    load_tile(p, t, w);
    for (int64_t k = 0; k < CC; ++k)
      if (isnan(w[k]) || w[k] == INFINITY) {
        free(w);
        *logz = NAN;
        return OR_F_NONFINITE;
      }
  }
  /* alpha_0 = log-one (0) for every label: no start/unary parts (reading R3). */
  double* alpha = (double*)malloc(sizeof(double) * (size_t)((Eb + 1) * C));
  double* beta = (double*)malloc(sizeof(double) * (size_t)(2 * C));
  for (int64_t i = 0; i < C; ++i) alpha[i] = 0.0;
  /* forward: alpha_{t+1}[j] = q + log sum_i exp(alpha_t[i] + l_t[i,j] - q) */
  for (int64_t t = 0; t < Eb; ++t) {
    const double* a = alpha + t * C;
    double* an = alpha + (t + 1) * C;
    load_tile(p, t, w);
    for (int64_t j = 0; j < C; ++j) {
      double q = -INFINITY;
      for (int64_t i = 0; i < C; ++i) {
        double v = a[i] + w[i * C + j];
        if (v > q) q = v;
      }
      if (q == -INFINITY) {
        an[j] = -INFINITY;
        continue;
      }
      double s = 0.0;
      for (int64_t i = 0; i < C; ++i) s += exp(a[i] + w[i * C + j] - q);
      an[j] = q + log(s);
    }
  }
  /* A = LSE_j alpha_E[j] */
  double q = -INFINITY;
  for (int64_t j = 0; j < C; ++j)
    if (alpha[Eb * C + j] > q) q = alpha[Eb * C + j];
  double A;
  if (q == -INFINITY) {
    A = -INFINITY;
  } else {
    double s = 0.0;
    for (int64_t j = 0; j < C; ++j) s += exp(alpha[Eb * C + j] - q);
    A = q + log(s);
  }
  *logz = A;
  uint32_t flags = 0;
  if (A == -INFINITY) flags |= OR_F_EMPTY; /* mu stays 0 (reading R11) */
  if (marg && A != -INFINITY) {
    /* backward: beta_E = 0; beta_t[i] = LSE_j(l_t[i,j] + beta_{t+1}[j]);
     * mu_t[i,j] = exp(alpha_t[i] + l_t[i,j] + beta_{t+1}[j] - A) */
    double* bn = beta;     /* beta_{t+1} */
    double* bc = beta + C; /* beta_t */
    for (int64_t j = 0; j < C; ++j) bn[j] = 0.0;
    int64_t ei = n_edges - 1; /* sampled mode: edges sorted ascending, walk backwards */
    for (int64_t t = Eb - 1; t >= 0; --t) {
      double* mt = NULL;
      if (!edges) {
        mt = marg + t * CC;
      } else {
        while (ei >= 0 && edges[ei] > t) --ei;
        if (ei >= 0 && edges[ei] == t) mt = marg + ei * CC;
      }
      load_tile(p, t, w);
      if (mt) {
        for (int64_t i = 0; i < C; ++i)
          for (int64_t j = 0; j < C; ++j)
            mt[i * C + j] = exp(alpha[t * C + i] + w[i * C + j] + bn[j] - A);
      }
      for (int64_t i = 0; i < C; ++i) {
        double qq = -INFINITY;
        for (int64_t j = 0; j < C; ++j) {
          double v = w[i * C + j] + bn[j];
          if (v > qq) qq = v;
        }
        if (qq == -INFINITY) {
          bc[i] = -INFINITY;
          continue;
        }
        double s = 0.0;
        for (int64_t j = 0; j < C; ++j) s += exp(w[i * C + j] + bn[j] - qq);
        bc[i] = qq + log(s);
      }
      double* tmp = bn;
      bn = bc;
      bc = tmp;
    }
  }
  free(alpha);
  free(beta);
  free(w);
  return flags;
}

/* Viterbi (reading R5): delta_0 = 0; delta_{t+1}[j] = max_i(delta_t[i] + l_t[i,j]);
 * bp_t[j] = first i (scanning upward, strict '>') attaining the max; z_E = first argmax of
 * delta_E; z_t = bp_t[z_{t+1}]; score = delta_E[z_E].  path[n] = -1 for n >= len. */
static uint32_t seq_viterbi(const pot_src* p, int64_t N, int32_t len, int32_t* path,
                            double* score) {
  const int64_t C = p->C;
  for (int64_t n = 0; n < N; ++n) path[n] = -1;
  if (len < 1 || len > N) {
    *score = NAN;
    return OR_F_BADLEN;
  }
  const int64_t Eb = (int64_t)len - 1;
  double* w = (double*)malloc(sizeof(double) * (size_t)(C * C));
  for (int64_t t = 0; t < Eb; ++t) {
    load_tile(p, t, w);
    for (int64_t k = 0; k < C * C; ++k)
      if (isnan(w[k]) || w[k] == INFINITY) {
        free(w);
        *score = NAN;
        return OR_F_NONFINITE;
      }
  }
  double* d = (double*)malloc(sizeof(double) * (size_t)C);
  double* dn = (double*)malloc(sizeof(double) * (size_t)C);
  int32_t* bp = (int32_t*)malloc(sizeof(int32_t) * (size_t)((Eb > 0 ? Eb : 1) * C));
  for (int64_t i = 0; i < C; ++i) d[i] = 0.0;
  for (int64_t t = 0; t < Eb; ++t) {
    load_tile(p, t, w);
    for (int64_t j = 0; j < C; ++j) {
      double best = d[0] + w[j];
      int32_t arg = 0;
      for (int64_t i = 1; i < C; ++i) {
        double v = d[i] + w[i * C + j];
        if (v > best) {
          best = v;
          arg = (int32_t)i;
        }
      }
      dn[j] = best;
      bp[t * C + j] = arg;
    }
    double* tmp = d;
    d = dn;
    dn = tmp;
  }
  double best = d[0];
  int32_t z = 0;
  for (int64_t j = 1; j < C; ++j)
    if (d[j] > best) {
      best = d[j];
      z = (int32_t)j;
    }
  uint32_t flags = 0;
  if (best == -INFINITY) {
    *score = -INFINITY;
    flags = OR_F_EMPTY; /* path stays -1 */
  } else {
    *score = best;
    path[Eb] = z;
    for (int64_t t = Eb - 1; t >= 0; --t) {
      z = bp[t * C + z];
      path[t] = z;
    }
  }
  free(d);
  free(dn);
  free(bp);
  free(w);
  return flags;
}

/* ---------------------------------------------------------------------------
 * Batched entry points (threads across b only).
 * ------------------------------------------------------------------------- */

typedef struct {
  int op; /* 0 = marginals/logz, 1 = viterbi */
  const float* pot;
  const int32_t* lengths;
  int64_t B, N, C;
  double* logz;
  double* marg;
  int32_t* path;
  double* score;
  uint32_t* flags;
  int64_t b0, b1;
} job_t;

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  const int64_t E = j->N - 1, CC = j->C * j->C;
  for (int64_t b = j->b0; b < j->b1; ++b) {
    pot_src p = {j->pot + b * (E > 0 ? E : 0) * CC, 0, 0, b, E, j->C};
    int32_t len = j->lengths ? j->lengths[b] : (int32_t)j->N;
    uint32_t f;
    if (j->op == 0) {
      f = seq_marginals(&p, j->N, len, &j->logz[b], j->marg ? j->marg + b * E * CC : NULL, NULL,
                        0);
    } else {
      f = seq_viterbi(&p, j->N, len, j->path + b * j->N, &j->score[b]);
    }
    if (j->flags) j->flags[b] = f;
  }
  return NULL;
}

static int run_batched(job_t proto, int threads) {
  if (threads < 1) threads = 1;
  if (threads > proto.B) threads = (int)proto.B;
  if (threads <= 1) {
    proto.b0 = 0;
    proto.b1 = proto.B;
    run_job(&proto);
    return 0;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)threads);
  for (int k = 0; k < threads; ++k) {
    jobs[k] = proto;
    jobs[k].b0 = proto.B * k / threads;
    jobs[k].b1 = proto.B * (k + 1) / threads;
    pthread_create(&th[k], NULL, run_job, &jobs[k]);
  }
  for (int k = 0; k < threads; ++k) pthread_join(th[k], NULL);
  free(th);
  free(jobs);
  return 0;
}

/* logZ (+ marginals if marg != NULL).  pot [B][N-1][C][C] fp32 (widened exactly);
 * lengths [B] or NULL (= N).  logz [B], marg [B][N-1][C][C] fp64, flags [B]. */
int oracle_chain_marginals(const float* pot, const int32_t* lengths, int64_t B, int64_t N,
                           int64_t C, double* logz, double* marg, uint32_t* flags, int threads) {
  if (B < 1 || N < 1 || C < 1 || !logz || (!pot && N > 1)) return 1;
  job_t j = {0, pot, lengths, B, N, C, logz, marg, NULL, NULL, flags, 0, 0};
  return run_batched(j, threads);
}

/* Viterbi: path [B][N] int32 (-1 beyond len), score [B] fp64, flags [B]. */
int oracle_chain_viterbi(const float* pot, const int32_t* lengths, int64_t B, int64_t N, int64_t C,
                         int32_t* path, double* score, uint32_t* flags, int threads) {
  if (B < 1 || N < 1 || C < 1 || !path || !score || (!pot && N > 1)) return 1;
  job_t j = {1, pot, lengths, B, N, C, NULL, NULL, path, score, flags, 0, 0};
  return run_batched(j, threads);
}

/* On-the-fly generator mode for full-size configs (tsgen recipe; no l buffer):
 * sequence b of a (seed, s) chain with N positions, full length.  Writes logz and
 * mu for the requested edges (ascending) into marg [n_edges][C][C]. */
int oracle_gen_marginals(uint64_t seed, int s, int64_t b, int64_t N, int64_t C,
                         const int64_t* edges, int64_t n_edges, double* logz, double* marg,
                         uint32_t* flags) {
  if (N < 1 || C < 1 || !logz) return 1;
  pot_src p = {NULL, seed, s, b, N - 1, C};
  uint32_t f = seq_marginals(&p, N, (int32_t)N, logz, n_edges > 0 ? marg : NULL, edges, n_edges);
  if (flags) *flags = f;
  return 0;
}

int oracle_gen_viterbi(uint64_t seed, int s, int64_t b, int64_t N, int64_t C, int32_t* path,
                       double* score, uint32_t* flags) {
  if (N < 1 || C < 1 || !path || !score) return 1;
  pot_src p = {NULL, seed, s, b, N - 1, C};
  uint32_t f = seq_viterbi(&p, N, (int32_t)N, path, score);
  if (flags) *flags = f;
  return 0;
}

/* Segment transfer matrix (the chain product of §6(a)): S = l_0 (x) l_1 (x) ... (x) l_{E-1},
 * S[i,j] = (+) over label paths from i at the segment start to j at its end.  fp64 [C][C].
 * E = 0 gives the identity I (0 on the diagonal, -inf off it). */
int oracle_chain_summary(int semiring, const float* pot, int64_t E, int64_t C, double* S) {
  if (C < 1 || E < 0 || !S || (E > 0 && !pot)) return 1;
  const int64_t CC = C * C;
  double* tile = (double*)malloc(sizeof(double) * (size_t)CC);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)CC);
  for (int64_t i = 0; i < C; ++i)
    for (int64_t j = 0; j < C; ++j) S[i * C + j] = (i == j) ? 0.0 : -INFINITY;
  for (int64_t t = 0; t < E; ++t) {
    for (int64_t k = 0; k < CC; ++k) tile[k] = (double)pot[t * CC + k];
    oracle_semiring_matmul(semiring, S, tile, C, C, C, tmp);
    memcpy(S, tmp, sizeof(double) * (size_t)CC);
  }
  free(tile);
  free(tmp);
  return 0;
}

/* The paper's parallel-scan ordering (§6(a), Fig. 4): pad the T edge
 * matrices to the next power of two with I, combine pairwise in a balanced tree of
 * semiring matmuls, then (+) over all root entries.  Returns the root value; *layers is
 * the number of sequential matmul layers (= ceil(log2 T)). */
int oracle_scan_partition(int semiring, const float* pot, int64_t T, int64_t C, double* root,
                          int* layers) {
  if (T < 1 || C < 1 || !pot || !root) return 1;
  const int64_t CC = C * C;
  int64_t P = 1;
  int nl = 0;
  while (P < T) {
    P <<= 1;
    ++nl;
  }
  double* nodes = (double*)malloc(sizeof(double) * (size_t)(P * CC));
  for (int64_t k = 0; k < P; ++k)
    for (int64_t i = 0; i < C; ++i)
      for (int64_t j = 0; j < C; ++j)
        nodes[k * CC + i * C + j] =
            (k < T) ? (double)pot[k * CC + i * C + j] : ((i == j) ? 0.0 : -INFINITY);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)CC);
  for (int64_t w = P; w > 1; w >>= 1) {
    for (int64_t k = 0; k < w / 2; ++k) {
      oracle_semiring_matmul(semiring, nodes + (2 * k) * CC, nodes + (2 * k + 1) * CC, C, C, C,
                             tmp);
      memcpy(nodes + k * CC, tmp, sizeof(double) * (size_t)CC);
    }
  }
  /* (+) over the root's entries */
  double q = -INFINITY;
  for (int64_t k = 0; k < CC; ++k)
    if (nodes[k] > q) q = nodes[k];
  if (semiring == OR_SEMI_MAX || q == -INFINITY) {
    *root = q;
  } else {
    double s = 0.0;
    for (int64_t k = 0; k < CC; ++k) s += exp(nodes[k] - q);
    *root = q + log(s);
  }
  if (layers) *layers = nl;
  free(nodes);
  free(tmp);
  return 0;
}

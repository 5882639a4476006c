/* oracle/gpref.c -- TEST INFRASTRUCTURE ONLY (not product code).
 *
 * The plain, slow, obviously-correct CPU oracle for the hot path of arXiv
 * 2105.10312.  Read oracle/gpref.h for the citation convention and the
 * import rule (only tests/, __graft_entry__.smoke() and bench.py's CPU
 * baseline may use this file).  Shares nothing with the CUDA path.
 *
 * Style rule for this file: every function follows the paper's definition or
 * algorithm step by step, in the paper's order and notation (with the readings
 * of SURVEY.md §8(c) / DESIGN.md where the paper is silent).  No blocking, no
 * fusion, no algebraic shortcuts: the EDF test evaluates dbf at EVERY deadline
 * up to the hyperperiod, the merge scan of Alg. 2 is linear, every candidate
 * is evaluated directly.  Wide sums use __int128 so that overflow cannot hide.
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * against the paper's worked example, SPEC's worked values, closed forms,
 * textbook reductions or brute force -- except the tie-breaking details of
 * the heuristics and the generator's distributional choices, which are
 * "parity unpinned" against the paper (no paper data exists).
 */
#include "gpref.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

/* ======================================================================= */
/* Integer helpers                                                          */
/* ======================================================================= */

static int64_t ceil_div(int64_t a, int64_t b) { /* a >= 0, b > 0 */
  return (a + b - 1) / b;
}

static int64_t gcd64(int64_t a, int64_t b) {
  while (b != 0) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

uint64_t gpref_splitmix64(uint64_t x) {
  /* Steele/Lea/Flood SplitMix64 finaliser applied to x + golden gamma. */
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* ======================================================================= */
/* A1: Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), used as the       */
/* counter-based generator of §8(c) C.1.10.                                 */
/* ======================================================================= */

void gpref_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t x0 = ctr[0], x1 = ctr[1], x2 = ctr[2], x3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { /* key schedule: Weyl sequence */
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)x0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)x2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t y0 = hi1 ^ x1 ^ k0;
    uint32_t y1 = lo1;
    uint32_t y2 = hi0 ^ x3 ^ k1;
    uint32_t y3 = lo0;
    x0 = y0; x1 = y1; x2 = y2; x3 = y3;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* ======================================================================= */
/* A3: WCET model                                                           */
/* ======================================================================= */

/* §8(c) C.1.3: W(m) = ceil(B/m) * c + f.
 * Block form of the worked example: B blocks dealt round-robin to m
 * SMs give ceil(B/m) waves (tail effect), each wave
 * costing the co-runner-dependent block cost c; f is the non-parallel floor
 * b of the §3.3 curves C(m) = a/m + b.                          */
int64_t gpref_wcet(int64_t B, int64_t c, int64_t f, int64_t m) {
  if (m <= 0 || B < 0) return -1;
  return ceil_div(B, m) * c + f;
}

/* §8(c) C.1.4: per-SM form used only to check the worked example (P:4-25 and
 * figure).  Blocks go round-robin starting at SM 0 (reading A-5):
 * blocks_on(j) = floor(B/m) + [j < B mod m];  W_j = blocks_on(j)*cost_j + f;
 * task WCET = max_j W_j.                                                     */
int gpref_wcet_per_sm(int64_t B, int32_t m, const int64_t *cost_per_sm, int64_t f,
                      int64_t *per_sm_out, int64_t *task_wcet) {
  if (m <= 0 || B < 0) return 1;
  int64_t worst = 0;
  for (int32_t j = 0; j < m; ++j) {
    int64_t blocks_on = B / m + ((j < B % m) ? 1 : 0);
    int64_t w = blocks_on * cost_per_sm[j] + f;
    if (per_sm_out) per_sm_out[j] = w;
    if (w > worst) worst = w;
  }
  *task_wcet = worst;
  return 0;
}

/* §8(c) C.1.5 / P:462: task i of the block is in conflict iff ANOTHER task of
 * the same type is allocated to the same partition.  Alone => no conflict
 * (P:576).  Returns 1 (conflict, use C^c) or 0 (use C^n).                     */
int gpref_conflict(int32_t n, const uint8_t *type, uint32_t block_mask, int32_t i) {
  for (int32_t j = 0; j < n; ++j) {
    if (j == i) continue;
    if (((block_mask >> j) & 1u) && type[j] == type[i]) return 1;
  }
  return 0;
}

/* C_i(T(P), |P|) of the case equation P:479-486 in the integer W form. */
static int64_t task_wcet_in_block(const gpref_sets *s, int32_t set, int32_t i, uint32_t mask,
                                  int32_t m) {
  int32_t n = s->n_tasks;
  const uint8_t *type = s->type + (int64_t)set * n;
  int64_t base = (int64_t)set * n + i;
  if (gpref_conflict(n, type, mask, i))
    return gpref_wcet(s->B[base], s->cc[base], s->fc[base], m);
  return gpref_wcet(s->B[base], s->cn[base], s->fn[base], m);
}

int gpref_wcet_batch(const gpref_sets *s, const int32_t *set_of_cand,
                     const int8_t *block_of_task, const int16_t *block_size, int64_t n_cand,
                     int32_t *wcet, uint8_t *conflict) {
  int32_t n = s->n_tasks;
  for (int64_t c = 0; c < n_cand; ++c) {
    int32_t set = set_of_cand[c];
    if (set < 0 || set >= s->n_sets) return 1;
    for (int32_t i = 0; i < n; ++i) {
      int32_t b = block_of_task[c * n + i];
      if (b < 0 || b >= n) return 1;
      int32_t m = block_size[c * n + b];
      if (m <= 0) return 1; /* m = 0 is invalid */
      uint32_t mask = 0;
      for (int32_t j = 0; j < n; ++j)
        if (block_of_task[c * n + j] == b) mask |= 1u << j;
      const uint8_t *type = s->type + (int64_t)set * n;
      conflict[c * n + i] = (uint8_t)gpref_conflict(n, type, mask, i);
      int64_t w = task_wcet_in_block(s, set, i, mask, m);
      if (w > INT32_MAX) return 2;
      wcet[c * n + i] = (int32_t)w;
    }
  }
  return 0;
}

/* ======================================================================= */
/* A4: EDF processor-demand criterion (policy fixed per P:816-817 reading  */
/* A-6; definition, §8(c) C.1.7).                                     */
/* ======================================================================= */

int gpref_hyperperiod(int32_t n, const int64_t *T, int64_t *H) {
  int64_t h = 1; /* empty set: 1 */
  for (int32_t i = 0; i < n; ++i) {
    if (T[i] <= 0) return 1;
    int64_t g = gcd64(h, T[i]);
    i128 l = (i128)(h / g) * (i128)T[i];
    if (l > (i128)INT64_MAX) return 2; /* never a silent wrap */
    h = (int64_t)l;
  }
  *H = h;
  return 0;
}

static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

/* Schedulable iff for every absolute deadline t = D_i + q*T_i <= H:
 *   dbf(t) = sum_i [t >= D_i] * (floor((t - D_i)/T_i) + 1) * C_i  <=  t.
 * Returns 1 schedulable, 0 not (witness = smallest violating t), <0 error.
 * n_points (optional) receives the number of distinct deadlines examined.  */
int gpref_edf_pdc(int32_t n, const int64_t *C, const int64_t *D, const int64_t *T,
                  int64_t *witness, int64_t *n_points) {
  if (n_points) *n_points = 0;
  if (n == 0) return 1; /* empty block: schedulable */
  for (int32_t i = 0; i < n; ++i)
    if (T[i] <= 0 || D[i] <= 0 || D[i] > T[i] || C[i] < 0) return -1;
  int64_t H;
  int rc = gpref_hyperperiod(n, T, &H);
  if (rc) return -rc - 1;
  /* every absolute deadline <= H */
  int64_t count = 0;
  for (int32_t i = 0; i < n; ++i) count += (H - D[i]) / T[i] + 1;
  int64_t *pts = (int64_t *)malloc(sizeof(int64_t) * (size_t)count);
  if (!pts) return -3;
  int64_t k = 0;
  for (int32_t i = 0; i < n; ++i)
    for (int64_t t = D[i]; t <= H; t += T[i]) pts[k++] = t;
  qsort(pts, (size_t)count, sizeof(int64_t), cmp_i64);
  int verdict = 1;
  int64_t examined = 0;
  for (int64_t p = 0; p < count; ++p) {
    if (p > 0 && pts[p] == pts[p - 1]) continue; /* distinct deadlines */
    int64_t t = pts[p];
    ++examined;
    i128 dbf = 0;
    for (int32_t i = 0; i < n; ++i)
      if (t >= D[i]) dbf += (i128)((t - D[i]) / T[i] + 1) * (i128)C[i];
    if (dbf > (i128)t) {
      if (witness) *witness = t;
      verdict = 0;
      break;
    }
  }
  free(pts);
  if (n_points) *n_points = examined;
  return verdict;
}

/* Oracle of the oracle: unit-tick discrete-event preemptive EDF
 * on one resource, synchronous release at 0, over [0, horizon).  Ties between
 * equal absolute deadlines go to the lower task index (any tie rule gives the
 * same miss/no-miss answer for EDF).  Returns 1 iff no job misses.           */
int gpref_simulate_edf(int32_t n, const int64_t *C, const int64_t *D, const int64_t *T,
                       int64_t horizon) {
  int64_t *rem = (int64_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  int64_t *dl = (int64_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
  int ok = 1;
  for (int64_t t = 0; t < horizon && ok; ++t) {
    for (int32_t i = 0; i < n; ++i) {
      if (t % T[i] == 0) {           /* release of a new job */
        if (rem[i] > 0) { ok = 0; break; } /* previous job unfinished (D<=T) */
        rem[i] = C[i];
        dl[i] = t + D[i];
      }
    }
    if (!ok) break;
    int32_t pick = -1;
    for (int32_t i = 0; i < n; ++i)
      if (rem[i] > 0 && (pick < 0 || dl[i] < dl[pick])) pick = i;
    if (pick >= 0) rem[pick] -= 1; /* execute one tick in [t, t+1) */
    for (int32_t i = 0; i < n; ++i)
      if (rem[i] > 0 && dl[i] <= t + 1) { ok = 0; break; } /* deadline passed */
  }
  free(rem);
  free(dl);
  return ok;
}

/* ======================================================================= */
/* A2: candidate space (§8(c) C.1.6).                                       */
/* A candidate is (k, pi, s): pi a restricted growth string (RGS) over the  */
/* n tasks with exactly k labels, s in Z>=1^k with sum(s) <= M.  Rank order: */
/* k ascending, pi lexicographic, s lexicographic.                           */
/* ======================================================================= */

static i128 stirling2(int n, int k) { /* S(n,k), textbook recurrence */
  if (n == 0 && k == 0) return 1;
  if (n == 0 || k == 0) return 0;
  return (i128)k * stirling2(n - 1, k) + stirling2(n - 1, k - 1);
}

static i128 binom(int64_t a, int64_t b) {
  if (b < 0 || a < 0 || b > a) return 0;
  i128 r = 1;
  for (int64_t i = 1; i <= b; ++i) {
    r = r * (a - b + i) / i;
    if (r > ((i128)1 << 100)) return ((i128)1 << 100); /* saturate: >> 2^63 */
  }
  return r;
}

int gpref_count_candidates(int32_t M, int32_t n, uint64_t *count) {
  if (M < 1 || n < 1 || n > 32) return 1;
  i128 total = 0;
  for (int32_t k = 1; k <= n && k <= M; ++k) {
    total += stirling2(n, k) * binom(M, k);
    if (total >= ((i128)1 << 63)) return 2;
  }
  *count = (uint64_t)total;
  return 0;
}

/* Next RGS in lexicographic order over ALL label counts; returns 0 at end. */
static int rgs_next(int32_t n, int8_t *a) {
  for (int32_t i = n - 1; i >= 1; --i) {
    int8_t mx = 0;
    for (int32_t j = 0; j < i; ++j)
      if (a[j] > mx) mx = a[j];
    if (a[i] <= mx) { /* a[i] may grow up to 1 + max(prefix) */
      a[i] += 1;
      for (int32_t j = i + 1; j < n; ++j) a[j] = 0;
      return 1;
    }
  }
  return 0;
}

static int rgs_labels(int32_t n, const int8_t *a) {
  int mx = -1;
  for (int32_t i = 0; i < n; ++i)
    if (a[i] > mx) mx = a[i];
  return mx + 1;
}

/* Visitor over every candidate in rank order (plain nested loops). */
typedef int (*cand_fn)(void *ctx, uint64_t rank, int32_t k, const int8_t *rgs,
                       const int16_t *sizes);

typedef struct {
  int32_t M, k;
  int16_t s[33];
  uint64_t *rank;
  const int8_t *rgs;
  int32_t n;
  cand_fn fn;
  void *ctx;
  int stop;
} srec_t;

static void sizes_rec(srec_t *r, int32_t pos, int32_t remaining) {
  if (r->stop) return;
  if (pos == r->k) {
    if (r->fn(r->ctx, *r->rank, r->k, r->rgs, r->s)) r->stop = 1;
    *r->rank += 1;
    return;
  }
  /* leave at least one SM for each later block */
  for (int32_t v = 1; v <= remaining - (r->k - pos - 1); ++v) {
    r->s[pos] = (int16_t)v;
    sizes_rec(r, pos + 1, remaining - v);
    if (r->stop) return;
  }
}

static void for_each_candidate(int32_t M, int32_t n, cand_fn fn, void *ctx) {
  uint64_t rank = 0;
  int8_t a[32];
  for (int32_t k = 1; k <= n && k <= M; ++k) {
    memset(a, 0, sizeof(a));
    do {
      if (rgs_labels(n, a) != k) continue;
      srec_t r;
      memset(&r, 0, sizeof(r));
      r.M = M; r.k = k; r.rank = &rank; r.rgs = a; r.n = n; r.fn = fn; r.ctx = ctx;
      sizes_rec(&r, 0, M);
      if (r.stop) return;
    } while (rgs_next(n, a));
  }
}

typedef struct {
  uint64_t first;
  int64_t count;
  int32_t n;
  int8_t *bot;
  int16_t *bs;
} enum_ctx;

static int enum_visit(void *vctx, uint64_t rank, int32_t k, const int8_t *rgs,
                      const int16_t *sizes) {
  enum_ctx *c = (enum_ctx *)vctx;
  if (rank < c->first) return 0;
  if (rank >= c->first + (uint64_t)c->count) return 1;
  int64_t row = (int64_t)(rank - c->first);
  for (int32_t i = 0; i < c->n; ++i) c->bot[row * c->n + i] = rgs[i];
  for (int32_t j = 0; j < c->n; ++j) c->bs[row * c->n + j] = (int16_t)(j < k ? sizes[j] : 0);
  return 0;
}

int gpref_enumerate(int32_t M, int32_t n, uint64_t first_rank, int64_t count,
                    int8_t *block_of_task, int16_t *block_size) {
  uint64_t total;
  int rc = gpref_count_candidates(M, n, &total);
  if (rc) return rc;
  if (count < 0 || first_rank + (uint64_t)count > total) return 1;
  enum_ctx c = {first_rank, count, n, block_of_task, block_size};
  if (count > 0) for_each_candidate(M, n, enum_visit, &c);
  return 0;
}

/* Number of ways to finish an RGS whose positions 0..i-1 are fixed and use j
 * labels, so that exactly k labels are used in total (plain recursion).     */
static i128 rgs_completions(int32_t n, int32_t i, int32_t j, int32_t k) {
  if (j > k) return 0;
  if (i == n) return j == k ? 1 : 0;
  return (i128)j * rgs_completions(n, i + 1, j, k) + rgs_completions(n, i + 1, j + 1, k);
}

int gpref_unrank(int32_t M, int32_t n, uint64_t rank, int8_t *block_of_task,
                 int16_t *block_size) {
  uint64_t total;
  int rc = gpref_count_candidates(M, n, &total);
  if (rc) return rc;
  if (rank >= total) return 1;
  i128 r = rank;
  int32_t k = 1;
  for (; k <= n && k <= M; ++k) {
    i128 cnt = stirling2(n, k) * binom(M, k);
    if (r < cnt) break;
    r -= cnt;
  }
  i128 per_pi = binom(M, k);
  i128 pi_idx = r / per_pi, s_idx = r % per_pi;
  /* unrank pi: lexicographic among RGS with exactly k labels */
  int32_t used = 0;
  for (int32_t i = 0; i < n; ++i) {
    int32_t lim = (i == 0) ? 0 : used; /* candidate labels 0..used (new = used) */
    for (int32_t lab = 0; lab <= lim; ++lab) {
      int32_t used2 = (lab == used) ? used + 1 : used;
      i128 c = rgs_completions(n, i + 1, used2, k);
      if (pi_idx < c) {
        block_of_task[i] = (int8_t)lab;
        used = used2;
        break;
      }
      pi_idx -= c;
    }
  }
  /* unrank s: lexicographic, s_j >= 1, sum <= M */
  int32_t remaining = M;
  for (int32_t j = 0; j < k; ++j) {
    for (int32_t v = 1;; ++v) {
      /* completions with s_j = v: later k-j-1 parts >=1 with sum <= remaining-v */
      i128 c = binom(remaining - v, k - j - 1);
      if (s_idx < c) {
        block_size[j] = (int16_t)v;
        remaining -= v;
        break;
      }
      s_idx -= c;
    }
  }
  for (int32_t j = k; j < n; ++j) block_size[j] = 0;
  return 0;
}

/* ======================================================================= */
/* A2-A4: exhaustive verdicts (§8(c) C.1.8)                                  */
/* ======================================================================= */

/* EDF-PDC of block `mask` at size m with the conflict-resolved WCETs. */
static int block_schedulable(const gpref_sets *s, int32_t set, uint32_t mask, int32_t m) {
  int32_t n = s->n_tasks;
  int64_t C[32], D[32], T[32];
  int32_t q = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (!((mask >> i) & 1u)) continue;
    int64_t base = (int64_t)set * n + i;
    C[q] = task_wcet_in_block(s, set, i, mask, m);
    D[q] = s->D[base];
    T[q] = s->T[base];
    ++q;
  }
  int v = gpref_edf_pdc(q, C, D, T, NULL, NULL);
  return v == 1;
}

typedef struct {
  const gpref_sets *s;
  int32_t set;
  uint64_t lo, hi;
  int64_t n_sched, pi_star, first_rank;
  uint64_t hash;
  uint32_t *bits;
  const uint8_t *admissible; /* [M+1] or NULL (f4, reading B-9) */
} exh_ctx;

static int exh_visit(void *vctx, uint64_t rank, int32_t k, const int8_t *rgs,
                     const int16_t *sizes) {
  exh_ctx *c = (exh_ctx *)vctx;
  if (rank < c->lo) return 0;
  if (rank >= c->hi) return 1;
  int32_t n = c->s->n_tasks;
  int ok = 1;
  int64_t sum_s = 0;
  for (int32_t j = 0; j < k; ++j) { /* candidate verdict = AND over blocks */
    uint32_t mask = 0;
    for (int32_t i = 0; i < n; ++i)
      if (rgs[i] == j) mask |= 1u << i;
    sum_s += sizes[j];
    /* f4 (reading B-9): a block on an inadmissible size is not deployable */
    if (c->admissible && !c->admissible[sizes[j]]) ok = 0;
    if (ok && !block_schedulable(c->s, c->set, mask, sizes[j])) ok = 0;
  }
  if (ok) {
    c->n_sched += 1;
    if (c->pi_star == 0 || sum_s < c->pi_star) c->pi_star = sum_s;
    if (c->first_rank < 0) c->first_rank = (int64_t)rank;
    c->hash += gpref_splitmix64(rank);
    if (c->bits) {
      uint64_t off = rank - c->lo;
      c->bits[off / 32] |= 1u << (off % 32);
    }
  }
  return 0;
}

typedef struct {
  const gpref_sets *s;
  uint64_t lo, hi;
  int64_t *per_set;
  uint32_t *bits;
  int64_t words;
  const uint8_t *admissible;
  int32_t next; /* shared work counter */
  pthread_mutex_t mu;
} exh_job;

static void exhaustive_one(exh_job *j, int32_t set) {
  exh_ctx c;
  memset(&c, 0, sizeof(c));
  c.s = j->s; c.set = set; c.lo = j->lo; c.hi = j->hi; c.first_rank = -1;
  c.admissible = j->admissible;
  c.bits = j->bits ? j->bits + (int64_t)set * j->words : NULL;
  if (c.bits) memset(c.bits, 0, sizeof(uint32_t) * (size_t)j->words);
  for_each_candidate(j->s->M, j->s->n_tasks, exh_visit, &c);
  j->per_set[set * 4 + 0] = c.n_sched;
  j->per_set[set * 4 + 1] = c.pi_star;
  j->per_set[set * 4 + 2] = c.first_rank;
  j->per_set[set * 4 + 3] = (int64_t)c.hash;
}

static void *exh_worker(void *arg) {
  exh_job *j = (exh_job *)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    int32_t set = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (set >= j->s->n_sets) return NULL;
    exhaustive_one(j, set);
  }
}

int gpref_exhaustive(const gpref_sets *s, uint64_t rank_lo, uint64_t rank_hi,
                     int64_t *per_set, uint32_t *verdict_bits, int64_t words_per_set,
                     int32_t n_threads) {
  return gpref_exhaustive_ex(s, rank_lo, rank_hi, NULL, per_set, verdict_bits, words_per_set,
                             n_threads);
}

int gpref_exhaustive_ex(const gpref_sets *s, uint64_t rank_lo, uint64_t rank_hi,
                        const uint8_t *admissible, int64_t *per_set, uint32_t *verdict_bits,
                        int64_t words_per_set, int32_t n_threads) {
  uint64_t total;
  int rc = gpref_count_candidates(s->M, s->n_tasks, &total);
  if (rc) return rc;
  if (rank_hi > total) rank_hi = total;
  if (rank_lo > rank_hi) return 1;
  if (verdict_bits && (uint64_t)words_per_set * 32 < rank_hi - rank_lo) return 1;
  exh_job j;
  memset(&j, 0, sizeof(j));
  j.s = s; j.lo = rank_lo; j.hi = rank_hi; j.per_set = per_set; j.bits = verdict_bits;
  j.words = words_per_set;
  j.admissible = admissible;
  pthread_mutex_init(&j.mu, NULL);
  if (n_threads < 1) n_threads = 1;
  pthread_t th[256];
  if (n_threads > 256) n_threads = 256;
  for (int32_t t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, exh_worker, &j);
  for (int32_t t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&j.mu);
  return 0;
}

/* ======================================================================= */
/* A5: heuristics -- Algorithm 1, Lemma 1, Lemma 2   */
/* (P:580-598), Pi and Lemma 3, Def. 3 and Algorithm 2           */
/* (P:654-694), Def. 4 / Def. 5 orders, forbidden list           */
/* (P:775-781), Algorithm 3; tie-breaks per §8(c) C.1.9.          */
/* ======================================================================= */

/* Task sets up to GPREF_MAX_TASKS tasks: partition task-sets are bitsets. */
#define GPREF_MAX_TASKS 256
#define GPREF_W (GPREF_MAX_TASKS / 64)

typedef struct {
  uint64_t w[GPREF_W];
} tmask;

static int tm_has(const tmask *m, int32_t i) { return (int)((m->w[i >> 6] >> (i & 63)) & 1u); }
static void tm_set(tmask *m, int32_t i) { m->w[i >> 6] |= 1ull << (i & 63); }
static tmask tm_or(tmask a, tmask b) {
  for (int x = 0; x < GPREF_W; ++x) a.w[x] |= b.w[x];
  return a;
}
static int tm_eq(const tmask *a, const tmask *b) {
  for (int x = 0; x < GPREF_W; ++x)
    if (a->w[x] != b->w[x]) return 0;
  return 1;
}
static tmask tm_single(int32_t i) {
  tmask m;
  memset(&m, 0, sizeof(m));
  tm_set(&m, i);
  return m;
}

/* P:462 on a bitset block: another task of the same type in the block */
static int conflict_bs(int32_t n, const uint8_t *type, const tmask *mask, int32_t i) {
  for (int32_t j = 0; j < n; ++j)
    if (j != i && tm_has(mask, j) && type[j] == type[i]) return 1;
  return 0;
}

static int64_t task_wcet_bs(const gpref_sets *s, int32_t set, int32_t i, const tmask *mask,
                            int32_t m) {
  int32_t n = s->n_tasks;
  const uint8_t *type = s->type + (int64_t)set * n;
  int64_t base = (int64_t)set * n + i;
  if (conflict_bs(n, type, mask, i)) return gpref_wcet(s->B[base], s->cc[base], s->fc[base], m);
  return gpref_wcet(s->B[base], s->cn[base], s->fn[base], m);
}

/* EDF-PDC of a bitset block at size m with the conflict-resolved WCETs. */
static int block_schedulable_bs(const gpref_sets *s, int32_t set, const tmask *mask, int32_t m) {
  int32_t n = s->n_tasks;
  int64_t C[GPREF_MAX_TASKS], D[GPREF_MAX_TASKS], T[GPREF_MAX_TASKS];
  int32_t q = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (!tm_has(mask, i)) continue;
    int64_t base = (int64_t)set * n + i;
    C[q] = task_wcet_bs(s, set, i, mask, m);
    D[q] = s->D[base];
    T[q] = s->T[base];
    ++q;
  }
  return gpref_edf_pdc(q, C, D, T, NULL, NULL) == 1;
}

typedef struct {
  tmask mask;
  int32_t size;
  int64_t uh; /* U(P) * H, Def. 5 with /T_i (reading A-19) scaled by H */
} part_t;

typedef struct {
  tmask a, b; /* unordered pair of partition task-sets (snapshot) */
} snap_t;

typedef struct {
  const gpref_sets *s;
  int32_t set, n, M;
  int64_t H;
  int64_t n_tests;
  part_t list[GPREF_MAX_TASKS]; /* par_list, kept sorted */
  int32_t len;
  snap_t *snaps;
  int32_t n_snaps, cap_snaps;
  uint8_t *forb; /* ACT task pairs, n x n */
  int act;
  /* f4 variants (gpref_alloc_opts) */
  int binary;                /* Algorithm 2 by binary search      */
  int increasing;            /* par_list in increasing utilisation */
  const uint8_t *admissible; /* [M+1]: admissible partition sizes, or NULL */
} heur_t;

static int32_t min_task(const tmask *mask) {
  for (int32_t i = 0; i < GPREF_MAX_TASKS; ++i)
    if (tm_has(mask, i)) return i;
  return GPREF_MAX_TASKS;
}

/* U(P) * H = sum_{i in P} C_i(T^P - {tau_i}, |P|) * (H / T_i) (A-19) */
static int64_t part_uh(const heur_t *h, const tmask *mask, int32_t m) {
  i128 u = 0;
  for (int32_t i = 0; i < h->n; ++i) {
    if (!tm_has(mask, i)) continue;
    int64_t base = (int64_t)h->set * h->n + i;
    u += (i128)task_wcet_bs(h->s, h->set, i, mask, m) * (h->H / h->s->T[base]);
  }
  return (int64_t)u;
}

/* Best-fit order (A-21): decreasing utilisation, ties by lower min task id.
 * It is also the par_list order (A-17) unless the f4 increasing variant is on. */
static int part_before(const part_t *x, const part_t *y) {
  if (x->uh != y->uh) return x->uh > y->uh;
  return min_task(&x->mask) < min_task(&y->mask);
}

/* par_list order: decreasing utilisation (A-17), or increasing
 * (f4: "decreasing/increasing utilization order"); ties by lower min task id. */
static int list_before(const heur_t *h, const part_t *x, const part_t *y) {
  if (x->uh != y->uh) return h->increasing ? x->uh < y->uh : x->uh > y->uh;
  return min_task(&x->mask) < min_task(&y->mask);
}

/* Is m an admissible partition size?  Without a mask every m >= 1 is (the
 * paper's Algorithm 2 may even exceed M); with a mask (f4, MIG-style slices,
 * P:1139) only the listed sizes 1..M are.                                    */
static int size_ok(const heur_t *h, int32_t m) {
  if (!h->admissible) return m >= 1;
  return m >= 1 && m <= h->M && h->admissible[m];
}

static void list_insert(heur_t *h, part_t p) {
  int32_t pos = h->len;
  for (int32_t q = 0; q < h->len; ++q)
    if (list_before(h, &p, &h->list[q])) { pos = q; break; }
  for (int32_t q = h->len; q > pos; --q) h->list[q] = h->list[q - 1];
  h->list[pos] = p;
  h->len += 1;
}

static void list_remove(heur_t *h, const tmask *mask) {
  int32_t q = 0;
  while (q < h->len && !tm_eq(&h->list[q].mask, mask)) ++q;
  for (; q + 1 < h->len; ++q) h->list[q] = h->list[q + 1];
  h->len -= 1;
}

static int test_schedulability(heur_t *h, const tmask *mask, int32_t m) {
  h->n_tests += 1; /* every EDF-PDC call counts (C.1.9 step 7) */
  return block_schedulable_bs(h->s, h->set, mask, m);
}

/* Algorithm 2: try m = max(|P1|,|P2|), ..., |P1|+|P2|-1 in order;
 * the strict upper bound is Def. 3's m3 < m1 + m2.  Returns m or 0.
 * f4 variants: only admissible sizes are tried, and the binary search
 * "between max{|P1|,|P2|} and |P1|+|P2|" replaces the scan: over
 * the ascending list L of candidate sizes, lo = 0, hi = |L|; while lo < hi:
 * mid = floor((lo+hi)/2), schedulable at L[mid] ? hi = mid : lo = mid + 1;
 * the answer is L[lo] if lo < |L|.  Schedulability is monotone in m (W_i is
 * non-increasing in m, C.1.3; the demand test is monotone in the C_i), so both
 * searches return the same m; only the number of tests differs.            */
static int32_t merge(heur_t *h, const part_t *p1, const part_t *p2) {
  tmask t3 = tm_or(p1->mask, p2->mask);
  int32_t first = p1->size > p2->size ? p1->size : p2->size;
  int32_t *L = (int32_t *)malloc(sizeof(int32_t) * (size_t)(p1->size + p2->size));
  int32_t len = 0;
  for (int32_t m = first; m < p1->size + p2->size; ++m)
    if (size_ok(h, m)) L[len++] = m;
  int32_t found = 0;
  if (!h->binary) {
    for (int32_t x = 0; x < len && !found; ++x)
      if (test_schedulability(h, &t3, L[x])) found = L[x];
  } else {
    int32_t lo = 0, hi = len;
    while (lo < hi) {
      int32_t mid = (lo + hi) / 2;
      if (test_schedulability(h, &t3, L[mid])) hi = mid;
      else lo = mid + 1;
    }
    if (lo < len) found = L[lo];
  }
  free(L);
  return found;
}

static void add_to_forbidden_moves(heur_t *h, const tmask *a, const tmask *b) {
  if (h->n_snaps == h->cap_snaps) {
    h->cap_snaps = h->cap_snaps ? 2 * h->cap_snaps : 64;
    h->snaps = (snap_t *)realloc(h->snaps, sizeof(snap_t) * (size_t)h->cap_snaps);
  }
  h->snaps[h->n_snaps].a = *a;
  h->snaps[h->n_snaps].b = *b;
  h->n_snaps += 1;
}

/* Is P' in forbidden(P) (Alg. 3 line 7)?  Snapshots in both modes; in ACT
 * mode also any task pair of the prefilled list ("at least one task is
 * implied in a forbidden merge with a task of P").                          */
static int forbidden(const heur_t *h, const tmask *p, const tmask *q) {
  for (int32_t x = 0; x < h->n_snaps; ++x)
    if ((tm_eq(&h->snaps[x].a, p) && tm_eq(&h->snaps[x].b, q)) ||
        (tm_eq(&h->snaps[x].a, q) && tm_eq(&h->snaps[x].b, p)))
      return 1;
  if (h->act)
    for (int32_t a = 0; a < h->n; ++a)
      if (tm_has(p, a))
        for (int32_t b = 0; b < h->n; ++b)
          if (tm_has(q, b) && h->forb[a * h->n + b]) return 1;
  return 0;
}

/* init_partitions, Lemma 2: one singleton partition per task with
 * |P| = min{m in 1..M : C^n(m) <= D} (f4: m admissible), inserted into
 * par_list in order.  Returns Pi = sum of the sizes, or -1 if some task has
 * no feasible size.                                                          */
static int32_t init_partitions(heur_t *h) {
  const gpref_sets *s = h->s;
  int32_t n = h->n, set = h->set, Pi = 0;
  for (int32_t i = 0; i < n; ++i) {
    int64_t b = (int64_t)set * n + i;
    int32_t size = 0;
    for (int32_t m = 1; m <= h->M; ++m) {
      if (size_ok(h, m) && gpref_wcet(s->B[b], s->cn[b], s->fn[b], m) - s->D[b] <= 0) {
        size = m;
        break;
      }
    }
    if (size == 0) return -1;
    part_t p = {tm_single(i), size, 0};
    p.uh = part_uh(h, &p.mask, size);
    list_insert(h, p);
    Pi += size;
  }
  return Pi;
}

/* Def. 5 order > as best fit (A-21): insertion sort of the eligible partners
 * by their U*H descending, ties lower min task id.                          */
static void sort_best_fit(part_t *cand, int32_t n_elig) {
  for (int32_t x = 1; x < n_elig; ++x)
    for (int32_t y = x; y > 0 && part_before(&cand[y], &cand[y - 1]); --y) {
      part_t t = cand[y]; cand[y] = cand[y - 1]; cand[y - 1] = t;
    }
}

/* §5.3 fill_forbidden_list (ACT, Alg. 1 line 3): "every couple of
 * tasks is tested to check if they are mergeable" -- the Lemma-2 singleton
 * partitions of every pair i < j (in task-id order) go through Algorithm 2;
 * a failing pair is recorded as a forbidden TASK pair.  The
 * singletons are the entries of par_list (one per task before any merge). */
static void fill_forbidden_list(heur_t *h) {
  int32_t n = h->n;
  h->forb = (uint8_t *)calloc((size_t)n * n, 1);
  part_t *single = (part_t *)calloc((size_t)n, sizeof(part_t));
  for (int32_t q = 0; q < h->len; ++q) single[min_task(&h->list[q].mask)] = h->list[q];
  for (int32_t i = 0; i < n; ++i)
    for (int32_t j = i + 1; j < n; ++j)
      if (merge(h, &single[i], &single[j]) == 0) h->forb[i * n + j] = h->forb[j * n + i] = 1;
  free(single);
}

/* Algorithm 3 select_partitions: candidates in par_list order,
 * choose_from = the head (A-18); forbidden(P) per Alg. 3 line 7 (snapshots,
 * plus ACT's task pairs); elig = par_list minus P (A-26) minus
 * forbidden(P), in par_list order (SMS evaluates every merge, so its order
 * does not matter; BF sorts it afterwards, A-21).  Returns the index of P in
 * par_list, or -1 when every candidate has an empty elig list.              */
static int32_t select_partitions(const heur_t *h, part_t *cand, int32_t *n_elig) {
  for (int32_t c = 0; c < h->len; ++c) {
    *n_elig = 0;
    for (int32_t q = 0; q < h->len; ++q) {
      if (q == c) continue; /* P itself is not eligible (A-26) */
      if (forbidden(h, &h->list[c].mask, &h->list[q].mask)) continue;
      cand[(*n_elig)++] = h->list[q];
    }
    if (*n_elig > 0) return c;
  }
  *n_elig = 0;
  return -1;
}

static void write_solution(const heur_t *h, int ok, uint8_t *okp, int16_t *bot, int16_t *bs,
                           int32_t *pi, int32_t *k, int64_t *nt, int with_parts) {
  int32_t n = h->n, set = h->set;
  okp[set] = (uint8_t)ok;
  nt[set] = h->n_tests;
  for (int32_t i = 0; i < n; ++i) {
    bot[(int64_t)set * n + i] = -1;
    bs[(int64_t)set * n + i] = 0;
  }
  if (!with_parts) {
    pi[set] = 0;
    k[set] = 0;
    return;
  }
  /* canonical labels: partitions numbered by increasing min task id */
  int32_t label = 0, total = 0;
  for (int32_t i = 0; i < n; ++i) {
    for (int32_t q = 0; q < h->len; ++q) {
      if (min_task(&h->list[q].mask) != i) continue;
      for (int32_t t = 0; t < n; ++t)
        if (tm_has(&h->list[q].mask, t)) bot[(int64_t)set * n + t] = (int16_t)label;
      bs[(int64_t)set * n + label] = (int16_t)h->list[q].size;
      total += h->list[q].size;
      label += 1;
    }
  }
  pi[set] = total;
  k[set] = label;
}

static void allocate_one(const gpref_sets *s, int32_t set, int32_t variant,
                         const gpref_alloc_opts *opts, uint8_t *okp, int16_t *bot, int16_t *bs,
                         int32_t *pi, int32_t *kk, int64_t *nt) {
  heur_t *h = (heur_t *)calloc(1, sizeof(heur_t));

  h->s = s; h->set = set; h->n = s->n_tasks; h->M = s->M;
  if (opts) {
    h->binary = (opts->flags & GPREF_AL_BINARY_MERGE) != 0;
    h->increasing = (opts->flags & GPREF_AL_INCREASING) != 0;
    h->admissible = opts->admissible;
  }
  int32_t n = h->n, M = h->M;
  int64_t Tv[GPREF_MAX_TASKS];
  for (int32_t i = 0; i < n; ++i) Tv[i] = s->T[(int64_t)set * n + i];
  if (gpref_hyperperiod(n, Tv, &h->H) != 0) h->H = 0;
  tmask empty;
  memset(&empty, 0, sizeof(empty));

  if (variant == GPREF_1G) {
    /* 1G: the whole GPU as one partition of M SMs; with a
     * size mask, the largest admissible size (f4)                           */
    int32_t size = M;
    while (!size_ok(h, size)) size -= 1;
    part_t all = {empty, size, 0};
    for (int32_t i = 0; i < n; ++i) tm_set(&all.mask, i);
    int ok = test_schedulability(h, &all.mask, size);
    h->list[0] = all;
    h->len = 1;
    write_solution(h, ok, okp, bot, bs, pi, kk, nt, 1);
    free(h);
    return;
  }
  h->act = (variant == GPREF_SMS_ACT || variant == GPREF_BF_ACT);
  int sms = (variant == GPREF_SMS_ACT || variant == GPREF_SMS_INA);

  /* Lemma 1: reject if sum_i C_i^n(1)/T_i > M, i.e. in integers
   * sum_i W_i(1,n) * (H/T_i) > M * H (reading A-16).                       */
  i128 lhs = 0;
  for (int32_t i = 0; i < n; ++i) {
    int64_t b = (int64_t)set * n + i;
    lhs += (i128)gpref_wcet(s->B[b], s->cn[b], s->fn[b], 1) * (h->H / s->T[b]);
  }
  if (lhs > (i128)M * h->H) {
    write_solution(h, 0, okp, bot, bs, pi, kk, nt, 0);
    free(h);
    return;
  }
  int32_t Pi = init_partitions(h);
  if (Pi < 0) { /* no feasible size: fail */
    write_solution(h, 0, okp, bot, bs, pi, kk, nt, 0);
    free(h);
    return;
  }
  /* Lemma 3: exit on success at any time -- before the ACT
   * prefill (reading A-24).                                                  */
  if (Pi <= M) {
    write_solution(h, 1, okp, bot, bs, pi, kk, nt, 1);
    free(h);
    return;
  }
  /* Alg. 1 line 3 / §5.3: ACT tests every couple of tasks. */
  if (h->act) fill_forbidden_list(h);
  /* Alg. 1 lines 4-18 */
  while (Pi > M) {
    int32_t n_elig = 0;
    part_t cand[GPREF_MAX_TASKS];
    int32_t sel = select_partitions(h, cand, &n_elig);
    if (sel < 0) { /* Alg. 1 line 6-7: return false */
      write_solution(h, 0, okp, bot, bs, pi, kk, nt, 1);
      free(h->snaps);
      free(h->forb);
      free(h);
      return;
    }
    part_t P = h->list[sel];
    if (sms) {
      /* Def. 4 order >>: evaluate every eligible merge, record the
       * failures, keep the best: smallest merged size, then smaller merged
       * U*H, then lower min task id of the partner (A-20, A-22).            */
      int32_t best = -1, best_m = 0;
      int64_t best_uh = 0;
      for (int32_t e = 0; e < n_elig; ++e) {
        int32_t m = merge(h, &P, &cand[e]);
        if (m == 0) {
          add_to_forbidden_moves(h, &P.mask, &cand[e].mask);
          continue;
        }
        tmask u3 = tm_or(P.mask, cand[e].mask);
        int64_t uh = part_uh(h, &u3, m);
        int better = 0;
        if (best < 0) better = 1;
        else if (m != best_m) better = m < best_m;
        else if (uh != best_uh) better = uh < best_uh;
        else better = min_task(&cand[e].mask) < min_task(&cand[best].mask);
        if (better) { best = e; best_m = m; best_uh = uh; }
      }
      if (best >= 0) {
        part_t merged = {tm_or(P.mask, cand[best].mask), best_m, best_uh};
        list_remove(h, &P.mask);
        list_remove(h, &cand[best].mask);
        list_insert(h, merged);
        Pi = Pi - P.size - cand[best].size + best_m;
      }
    } else {
      /* Def. 5 order > as best fit (A-21): sort the eligible partners by
       * their U*H descending, ties lower min task id; Alg. 1 repeat-loop:
       * try in order, record failures, commit the first success.           */
      sort_best_fit(cand, n_elig);
      for (int32_t e = 0; e < n_elig; ++e) {
        int32_t m = merge(h, &P, &cand[e]);
        if (m == 0) {
          add_to_forbidden_moves(h, &P.mask, &cand[e].mask);
          continue;
        }
        tmask u3 = tm_or(P.mask, cand[e].mask);
        part_t merged = {u3, m, part_uh(h, &u3, m)};
        list_remove(h, &P.mask);
        list_remove(h, &cand[e].mask);
        list_insert(h, merged);
        Pi = Pi - P.size - cand[e].size + m;
        break;
      }
    }
  }
  write_solution(h, 1, okp, bot, bs, pi, kk, nt, 1);
  free(h->snaps);
  free(h->forb);
  free(h);
}

typedef struct {
  const gpref_sets *s;
  int32_t variant;
  const gpref_alloc_opts *opts;
  uint8_t *ok;
  int16_t *bot;
  int16_t *bs;
  int32_t *pi, *k;
  int64_t *nt;
  int32_t next;
  pthread_mutex_t mu;
} alloc_job;

static void *alloc_worker(void *arg) {
  alloc_job *j = (alloc_job *)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    int32_t set = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (set >= j->s->n_sets) return NULL;
    allocate_one(j->s, set, j->variant, j->opts, j->ok, j->bot, j->bs, j->pi, j->k, j->nt);
  }
}

int gpref_allocate(const gpref_sets *s, int32_t variant, uint8_t *ok, int16_t *block_of_task,
                   int16_t *block_size, int32_t *pi, int32_t *k, int64_t *n_tests,
                   int32_t n_threads) {
  return gpref_allocate_ex(s, variant, NULL, ok, block_of_task, block_size, pi, k, n_tests,
                           n_threads);
}

int gpref_allocate_ex(const gpref_sets *s, int32_t variant, const gpref_alloc_opts *opts,
                      uint8_t *ok, int16_t *block_of_task, int16_t *block_size, int32_t *pi,
                      int32_t *k, int64_t *n_tests, int32_t n_threads) {
  if (variant < 0 || variant > 4 || s->n_tasks < 1 || s->n_tasks > GPREF_MAX_TASKS || s->M < 1)
    return 1;
  if (opts && opts->admissible) { /* at least one admissible size in 1..M */
    int any = 0;
    for (int32_t m = 1; m <= s->M; ++m) any |= opts->admissible[m] != 0;
    if (!any) return 1;
  }
  alloc_job j;
  memset(&j, 0, sizeof(j));
  j.s = s; j.variant = variant; j.opts = opts; j.ok = ok; j.bot = block_of_task; j.bs = block_size;
  j.pi = pi; j.k = k; j.nt = n_tests;
  pthread_mutex_init(&j.mu, NULL);
  if (n_threads < 1) n_threads = 1;
  if (n_threads > 256) n_threads = 256;
  pthread_t th[256];
  for (int32_t t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, alloc_worker, &j);
  for (int32_t t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&j.mu);
  return 0;
}

/* Test entry points of two steps of Algorithm 1 in isolation (SPEC's
 * select_partitions and fill_forbidden_list examples).  Both run
 * the same static functions as gpref_allocate_ex.  Tasks < 64 (masks are
 * one uint64 word).                                                         */
static int heur_setup(heur_t *h, const gpref_sets *s, int32_t set) {
  if (set < 0 || set >= s->n_sets || s->n_tasks < 1 || s->n_tasks > 64) return 1;
  h->s = s; h->set = set; h->n = s->n_tasks; h->M = s->M;
  int64_t Tv[64];
  for (int32_t i = 0; i < h->n; ++i) Tv[i] = s->T[(int64_t)set * h->n + i];
  return gpref_hyperperiod(h->n, Tv, &h->H) != 0 ? 2 : 0;
}

static tmask tm_from64(uint64_t w) {
  tmask m;
  memset(&m, 0, sizeof(m));
  m.w[0] = w;
  return m;
}

/* fill_forbidden_list: forb[i*n + j] = 1 iff the Lemma-2
 * singletons of tasks i and j fail Algorithm 2; *n_tests = EDF tests run.
 * Returns 3 if some task has no Lemma-2 size.                               */
int gpref_fill_forbidden_list(const gpref_sets *s, int32_t set, uint8_t *forb,
                              int64_t *n_tests) {
  heur_t *h = (heur_t *)calloc(1, sizeof(heur_t));
  int rc = heur_setup(h, s, set);
  if (!rc && init_partitions(h) < 0) rc = 3;
  if (!rc) {
    fill_forbidden_list(h);
    memcpy(forb, h->forb, (size_t)h->n * h->n);
    *n_tests = h->n_tests;
  }
  free(h->forb);
  free(h);
  return rc;
}

/* select_partitions (Algorithm 3) on a given state: par_list =
 * the n_parts partitions (task masks, sizes; inserted in par_list order by
 * their U*H, so the input order does not matter), the INA snapshot pairs
 * (snap_a[x], snap_b[x]) and, if forb != NULL, ACT's forbidden task pairs
 * (n x n).  best_fit != 0 sorts elig as BF does (A-21).  Outputs the mask of
 * the selected P (0 = none) and the elig masks in order.                    */
int gpref_select_partitions(const gpref_sets *s, int32_t set, int32_t n_parts,
                            const uint64_t *masks, const int32_t *sizes, int32_t n_snaps,
                            const uint64_t *snap_a, const uint64_t *snap_b,
                            const uint8_t *forb, int32_t best_fit, uint64_t *sel_mask,
                            uint64_t *elig_masks, int32_t *n_elig) {
  heur_t *h = (heur_t *)calloc(1, sizeof(heur_t));
  int rc = heur_setup(h, s, set);
  if (!rc && (n_parts < 1 || n_parts > 64)) rc = 1;
  if (!rc) {
    for (int32_t q = 0; q < n_parts; ++q) {
      part_t p = {tm_from64(masks[q]), sizes[q], 0};
      p.uh = part_uh(h, &p.mask, sizes[q]);
      list_insert(h, p);
    }
    for (int32_t x = 0; x < n_snaps; ++x) {
      tmask a = tm_from64(snap_a[x]), b = tm_from64(snap_b[x]);
      add_to_forbidden_moves(h, &a, &b);
    }
    if (forb) {
      h->act = 1;
      h->forb = (uint8_t *)malloc((size_t)h->n * h->n);
      memcpy(h->forb, forb, (size_t)h->n * h->n);
    }
    part_t cand[64];
    int32_t ne = 0;
    int32_t sel = select_partitions(h, cand, &ne);
    if (best_fit) sort_best_fit(cand, ne);
    *sel_mask = sel < 0 ? 0 : h->list[sel].mask.w[0];
    for (int32_t e = 0; e < ne; ++e) elig_masks[e] = cand[e].mask.w[0];
    *n_elig = ne;
  }
  free(h->snaps);
  free(h->forb);
  free(h);
  return rc;
}

/* §8(f) f2: scheduled workload ("efficiency") of an allocation (P:965-966,
 * P:1009-1014), in the integer W form: the work of task i is
 * its blocks times its per-block cost, c_i^x * B_i (the a of C = k(a/m + b),
 * reading A-1/A-14), as a utilisation scaled by the set's hyperperiod H:
 *   lower    = sum_i cn_i * B_i * (H/T_i)      (no task in conflict)
 *   upper    = sum_i cc_i * B_i * (H/T_i)      (every task in conflict)
 *   achieved = sum_i c_i^{x_i} * B_i * (H/T_i) (x_i from the allocation)
 * eff[set] = {lower, upper, achieved (0 without an allocation), H}.        */
int gpref_efficiency(const gpref_sets *s, const int16_t *block_of_task, int64_t *eff) {
  int32_t n = s->n_tasks;
  if (n < 1 || n > GPREF_MAX_TASKS) return 1;
  for (int32_t set = 0; set < s->n_sets; ++set) {
    int64_t T[GPREF_MAX_TASKS], H;
    for (int32_t i = 0; i < n; ++i) T[i] = s->T[(int64_t)set * n + i];
    if (gpref_hyperperiod(n, T, &H) != 0) return 2;
    const int16_t *lab = block_of_task + (int64_t)set * n;
    const uint8_t *type = s->type + (int64_t)set * n;
    int has_alloc = lab[0] >= 0;
    i128 lo = 0, up = 0, ach = 0;
    for (int32_t i = 0; i < n; ++i) {
      int64_t b = (int64_t)set * n + i;
      int64_t q = H / T[i];
      lo += (i128)s->cn[b] * s->B[b] * q;
      up += (i128)s->cc[b] * s->B[b] * q;
      if (has_alloc) {
        tmask mask;
        memset(&mask, 0, sizeof(mask));
        for (int32_t j = 0; j < n; ++j)
          if (lab[j] == lab[i]) tm_set(&mask, j);
        int x = conflict_bs(n, type, &mask, i);
        ach += (i128)(x ? s->cc[b] : s->cn[b]) * s->B[b] * q;
      }
    }
    eff[set * 4 + 0] = (int64_t)lo;
    eff[set * 4 + 1] = (int64_t)up;
    eff[set * 4 + 2] = (int64_t)ach;
    eff[set * 4 + 3] = H;
  }
  return 0;
}

/* ======================================================================= */
/* A1: generator (§7.1; §8(c) C.1.10, readings A-9..A-15)          */
/* ======================================================================= */

/* UUniFast-Discard as sorted uniform spacings (reading A-12): the
 * n-1 points are sorted and the n gaps of 0 <= p_(1) <= ... <= p_(n-1) <= Uq
 * are the utilisations, so sum(u) = Uq exactly.                             */
int gpref_uunisort(int32_t n, int64_t Uq, const int64_t *points, int64_t *u) {
  if (n < 1 || n > GPREF_MAX_TASKS) return 1;
  int64_t pts[GPREF_MAX_TASKS];
  for (int32_t j = 0; j < n - 1; ++j) {
    if (points[j] < 0 || points[j] > Uq) return 1;
    pts[j] = points[j];
  }
  for (int32_t x = 1; x < n - 1; ++x) /* insertion sort */
    for (int32_t y = x; y > 0 && pts[y] < pts[y - 1]; --y) {
      int64_t t = pts[y]; pts[y] = pts[y - 1]; pts[y - 1] = t;
    }
  for (int32_t i = 0; i < n; ++i) {
    int64_t hi = (i == n - 1) ? Uq : pts[i];
    int64_t lo = (i == 0) ? 0 : pts[i - 1];
    u[i] = hi - lo;
  }
  return 0;
}

/* One task of §7.1 from its utilisation u (Q20), menu index,
 * block count and type.  out = {T, D, cn, fn, cc, fc, a, feasible_alone}.   */
int gpref_task_fields(const gpref_gen_params *p, int64_t u, int32_t period_idx, int64_t B,
                      int32_t type, int64_t out[9]) {
  int32_t Q = p->ticks_per_unit;
  if (period_idx < 0 || period_idx >= p->n_periods || B < 1) return 1;
  int curve = p->curve_gran > 0;
  /* period from the menu, bumped while the execution time is not
   * "reasonable" (reading A-10): a < max(Q, B), up to the largest period.
   * Curve mode (f1, reading A-1): B is derived from a, so the rule is a < Q. */
  int64_t pi_ = period_idx;
  int64_t T = (int64_t)p->period_menu[pi_] * Q;
  int64_t a = (u * T) >> 20; /* baseline execution time = T * u */
  int64_t need = (curve || B <= Q) ? Q : B;
  while (a < need && pi_ < p->n_periods - 1) {
    pi_ += 1;
    T = (int64_t)p->period_menu[pi_] * Q;
    a = (u * T) >> 20;
  }
  int64_t D = 3 * T / 4;                                /* D = 0.75 T */
  int64_t beta = type ? p->beta_m_num : p->beta_c_num;  /* b = 0.02a / 0.1a */
  int64_t fn = ceil_div(a * beta, p->beta_den);
  int64_t kf = type ? p->km_num : p->kc_num;            /* k = 1.2 / 2.3, A-14 */
  int64_t cn, cc;
  if (curve) {
    /* the §7.1 curve C = k(a/|P| + b) in the W form: a split into granules of
     * g ticks, W(m) = ceil(B/m) * g * k + ceil(k b) with B = ceil(a/g)       */
    int64_t g = p->curve_gran;
    B = ceil_div(a, g);
    if (B < 1) B = 1;
    cn = g;
    cc = ceil_div(g * kf, p->k_den);
  } else {
    cn = ceil_div(a, B); /* per-wave block cost */
    if (cn < 1) cn = 1;
    cc = ceil_div(cn * kf, p->k_den);
  }
  int64_t fc = ceil_div(fn * kf, p->k_den);
  out[0] = T; out[1] = D; out[2] = cn; out[3] = fn; out[4] = cc; out[5] = fc; out[6] = a;
  /* feasible alone on all M SMs without conflict (discard rule, A-9) */
  out[7] = gpref_wcet(B, cn, fn, p->M) <= D;
  out[8] = B;
  return 0;
}

static void generate_one(const gpref_gen_params *p, uint64_t seed, uint64_t g, int32_t bin,
                         int32_t prm_idx, gpref_sets *out, int64_t l) {
  int32_t n = p->n_tasks, M = p->M;
  int64_t Uq = ((int64_t)(bin + 1) * (int64_t)M << 20) / p->n_bins; /* Q20 total (A-31) */
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  int64_t f[GPREF_MAX_TASKS][9], Bv[GPREF_MAX_TASKS];
  uint8_t type[GPREF_MAX_TASKS];
  int valid = 0;
  for (int32_t attempt = 0; attempt < p->max_attempts; ++attempt) {
    int64_t pts[GPREF_MAX_TASKS] = {0}, u[GPREF_MAX_TASKS];
    int32_t pidx[GPREF_MAX_TASKS];
    for (int32_t j = 0; j < n; ++j) {
      uint32_t ctr[4] = {(uint32_t)g, (uint32_t)(g >> 32), (uint32_t)attempt, (uint32_t)j};
      uint32_t w[4];
      gpref_philox4x32_10(ctr, key, w);
      /* alpha > prm => compute, else memory (reading A-15) */
      type[j] = ((uint64_t)w[0] < p->prm_q[prm_idx]) ? 1 : 0;
      pidx[j] = (int32_t)(((uint64_t)w[1] * (uint64_t)p->n_periods) >> 32); /* A-11 */
      Bv[j] = 1 + (int64_t)(((uint64_t)w[2] * (uint64_t)p->b_max) >> 32);  /* A-13 */
      if (j < n - 1) pts[j] = (int64_t)(((uint64_t)w[3] * (uint64_t)(Uq + 1)) >> 32);
    }
    gpref_uunisort(n, Uq, pts, u);
    int discard = 0;
    for (int32_t i = 0; i < n; ++i) {
      gpref_task_fields(p, u[i], pidx[i], Bv[i], type[i], f[i]);
      if (!f[i][7]) discard = 1; /* discard the whole vector (A-9) */
    }
    if (!discard) {
      valid = 1;
      break;
    }
  }
  (void)M;
  for (int32_t i = 0; i < n; ++i) {
    int64_t o = l * n + i;
    out->T[o] = (int32_t)f[i][0];
    out->D[o] = (int32_t)f[i][1];
    out->B[o] = (int32_t)f[i][8];
    out->cn[o] = (int32_t)f[i][2];
    out->fn[o] = (int32_t)f[i][3];
    out->cc[o] = (int32_t)f[i][4];
    out->fc[o] = (int32_t)f[i][5];
    out->type[o] = type[i];
  }
  out->valid[l] = (uint8_t)valid;
}

int gpref_generate(const gpref_gen_params *p, uint64_t seed, uint64_t rep_begin,
                   int32_t rep_count, gpref_sets *out) {
  if (p->n_tasks < 1 || p->n_tasks > GPREF_MAX_TASKS || p->M < 1 || p->n_bins < 1 || p->n_prm < 1 ||
      p->n_periods < 1 || p->max_attempts < 1 || p->b_max < 1 || p->beta_den < 1 ||
      p->k_den < 1 || rep_count < 0 || rep_begin + (uint64_t)rep_count > (uint64_t)p->sets_per_group)
    return 1;
  int32_t n_groups = p->n_prm * p->n_bins;
  if (out->n_sets != n_groups * rep_count || out->n_tasks != p->n_tasks) return 1;
  out->M = p->M;
  out->n_groups = n_groups;
  for (int32_t grp = 0; grp < n_groups; ++grp) {
    int32_t prm_idx = grp / p->n_bins, bin = grp % p->n_bins;
    for (int32_t r = 0; r < rep_count; ++r) {
      uint64_t rep = rep_begin + (uint64_t)r;
      uint64_t g = (uint64_t)grp * (uint64_t)p->sets_per_group + rep; /* global index */
      int64_t l = (int64_t)grp * rep_count + r;
      generate_one(p, seed, g, bin, prm_idx, out, l);
      out->group[l] = grp;
    }
  }
  return 0;
}

/* ======================================================================= */
/* A6: reduction (§7.2; §8(c) C.1.11)                              */
/* counts[setting][group][slot][3] += (ok*valid, 1, !valid)                   */
/* ======================================================================= */

int gpref_sched_ratio(const gpref_sets *s, const uint8_t *verdicts, int32_t n_rows,
                      int32_t slot0, int32_t n_slots, int32_t setting, int64_t *counts) {
  if (slot0 < 0 || slot0 + n_rows > n_slots) return 1;
  for (int32_t row = 0; row < n_rows; ++row)
    for (int32_t set = 0; set < s->n_sets; ++set) {
      int32_t grp = s->group[set];
      if (grp < 0 || grp >= s->n_groups) return 1;
      int64_t *c = counts + (((int64_t)setting * s->n_groups + grp) * n_slots + slot0 + row) * 3;
      int ok = verdicts[(int64_t)row * s->n_sets + set] != 0;
      int valid = s->valid[set] != 0;
      c[0] += ok && valid;
      c[1] += 1;
      c[2] += !valid;
    }
  return 0;
}

/* oracle/gpref.h -- TEST INFRASTRUCTURE ONLY (not product code).
 *
 * Plain, slow, obviously-correct CPU oracle of the hot path of
 *   Zahaf et al., "Contention-Aware GPU Partitioning and Task-to-Partition
 *   Allocation for Real-Time Workloads" (arXiv 2105.10312).
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / equation /
 * algorithm named alongside); "S:n" = SPEC.md line n; "§8(c) C.x" = the
 * binding reading in SURVEY.md §8(c) / DESIGN.md "Readings".
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg (and
 * `bench.py --impl reference`) may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2105_10312_b200/csrc);
 * neither side includes or links the other.
 *
 * Task sets have up to 256 tasks (heuristics, generator, efficiency; the
 * exhaustive enumeration is limited by N_c < 2^63 instead).
 * Everything is integer.  Time is in integer ticks (§8(c) C.1.1).  Host
 * arrays only; layout of every per-task field is [n_sets][n_tasks]
 * (set-major, task-minor) -- the same layout the C ABI documents.
 *
 * Return codes: 0 ok, 1 invalid argument, 2 overflow.
 */
#ifndef GPREF_H
#define GPREF_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t n_sets, n_tasks, M, n_groups;
  int32_t *T, *D, *B, *cn, *cc, *fn, *fc; /* [n_sets][n_tasks] ticks / blocks */
  uint8_t *type;                          /* 0 compute, 1 memory      */
  uint8_t *valid;                         /* [n_sets]                          */
  int32_t *group;                         /* [n_sets]                          */
} gpref_sets;

typedef struct {
  int32_t M, n_tasks, n_bins, n_prm, sets_per_group;
  const uint64_t *prm_q;                  /* [n_prm] memory iff w0 < prm_q     */
  int32_t ticks_per_unit;                 /* Q                                 */
  int32_t n_periods;
  const int32_t *period_menu;             /* paper units, ascending            */
  int32_t b_max;
  int32_t beta_c_num, beta_m_num, beta_den;
  int32_t kc_num, km_num, k_den;
  int32_t max_attempts;
  int32_t curve_gran;                     /* 0: block mode; g > 0: curve mode (f1), granule g ticks */
} gpref_gen_params;

/* ---- A1: counter-based generator (§7.1; §8(c) C.1.10) ---- */
void gpref_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
int gpref_generate(const gpref_gen_params *p, uint64_t seed, uint64_t rep_begin,
                   int32_t rep_count, gpref_sets *out);
int gpref_uunisort(int32_t n, int64_t Uq, const int64_t *points, int64_t *u);
int gpref_task_fields(const gpref_gen_params *p, int64_t u_q20, int32_t period_idx, int64_t B,
                      int32_t type, int64_t out[9]);

/* ---- A3: WCET model (P:4-25 example; §3.3; §4.2) ---- */
int64_t gpref_wcet(int64_t B, int64_t c, int64_t f, int64_t m);              /* C.1.3 */
int gpref_wcet_per_sm(int64_t B, int32_t m, const int64_t *cost_per_sm, int64_t f,
                      int64_t *per_sm_out, int64_t *task_wcet);              /* C.1.4 */
int gpref_conflict(int32_t n, const uint8_t *type, uint32_t block_mask, int32_t i); /* C.1.5 */
int gpref_wcet_batch(const gpref_sets *s, const int32_t *set_of_cand,
                     const int8_t *block_of_task, const int16_t *block_size, int64_t n_cand,
                     int32_t *wcet, uint8_t *conflict);

/* ---- A4: per-partition EDF processor-demand test (§5.5) ---- */
int gpref_hyperperiod(int32_t n, const int64_t *T, int64_t *H);
int gpref_edf_pdc(int32_t n, const int64_t *C, const int64_t *D, const int64_t *T,
                  int64_t *witness, int64_t *n_points);
int gpref_simulate_edf(int32_t n, const int64_t *C, const int64_t *D, const int64_t *T,
                       int64_t horizon);

/* ---- A2: candidate space (§5 intro; §8(c) C.1.6) ---- */
int gpref_count_candidates(int32_t M, int32_t n, uint64_t *count);
int gpref_enumerate(int32_t M, int32_t n, uint64_t first_rank, int64_t count,
                    int8_t *block_of_task, int16_t *block_size);
int gpref_unrank(int32_t M, int32_t n, uint64_t rank, int8_t *block_of_task,
                 int16_t *block_size);

/* ---- A2-A4 exhaustive verdicts (§8(c) C.1.8) ---- */
int gpref_exhaustive(const gpref_sets *s, uint64_t rank_lo, uint64_t rank_hi,
                     int64_t *per_set /*[n_sets][4]*/, uint32_t *verdict_bits,
                     int64_t words_per_set, int32_t n_threads);
/* f4 on the exhaustive path (SURVEY §8(f) f4, P:1136-1140 MIG-style slices;
 * reading B-9 of DESIGN.md): admissible = [M+1] flags (admissible[m] != 0 ->
 * partitions of m SMs may be formed) or NULL (every size).  A candidate that
 * uses an inadmissible size is not a deployable configuration and is counted
 * unschedulable; the rank space, N_c and the ranks are unchanged.          */
int gpref_exhaustive_ex(const gpref_sets *s, uint64_t rank_lo, uint64_t rank_hi,
                        const uint8_t *admissible, int64_t *per_set, uint32_t *verdict_bits,
                        int64_t words_per_set, int32_t n_threads);

/* ---- A5: heuristics, Alg. 1-3 + 1G ---- */
enum { GPREF_1G = 0, GPREF_SMS_ACT = 1, GPREF_SMS_INA = 2, GPREF_BF_ACT = 3, GPREF_BF_INA = 4 };
int gpref_allocate(const gpref_sets *s, int32_t variant, uint8_t *ok, int16_t *block_of_task,
                   int16_t *block_size, int32_t *pi, int32_t *k, int64_t *n_tests,
                   int32_t n_threads);

/* Two steps of Algorithm 1 in isolation (tests of SPEC S:280-296; tasks < 64) */
int gpref_fill_forbidden_list(const gpref_sets *s, int32_t set, uint8_t *forb /*[n][n]*/,
                              int64_t *n_tests);
int gpref_select_partitions(const gpref_sets *s, int32_t set, int32_t n_parts,
                            const uint64_t *masks, const int32_t *sizes, int32_t n_snaps,
                            const uint64_t *snap_a, const uint64_t *snap_b,
                            const uint8_t *forb /*[n][n] or NULL (INA)*/, int32_t best_fit,
                            uint64_t *sel_mask, uint64_t *elig_masks, int32_t *n_elig);

/* ---- f4: the variants the paper names ---- */
enum { GPREF_AL_BINARY_MERGE = 1, /* Algorithm 2 by binary search */
       GPREF_AL_INCREASING = 2 }; /* par_list in increasing utilisation */
typedef struct {
  uint32_t flags;
  const uint8_t *admissible; /* [M+1]; admissible[m] != 0: partitions of m SMs allowed
                                (MIG-style slices); NULL: every size */
} gpref_alloc_opts;
int gpref_allocate_ex(const gpref_sets *s, int32_t variant, const gpref_alloc_opts *opts,
                      uint8_t *ok, int16_t *block_of_task, int16_t *block_size, int32_t *pi,
                      int32_t *k, int64_t *n_tests, int32_t n_threads);

/* ---- f2: scheduled workload of an allocation ---- */
int gpref_efficiency(const gpref_sets *s, const int16_t *block_of_task, int64_t *eff);

/* ---- A6: segmented ratio reduction (§7.2; §8(c) C.1.11) ---- */
int gpref_sched_ratio(const gpref_sets *s, const uint8_t *verdicts, int32_t n_rows,
                      int32_t slot0, int32_t n_slots, int32_t setting, int64_t *counts);

uint64_t gpref_splitmix64(uint64_t x);

#ifdef __cplusplus
}
#endif
#endif

/* include/gpart.h -- C ABI of the B200-native batched, contention-aware
 * schedulability evaluator for arXiv 2105.10312 (Zahaf et al., "Contention-
 * Aware GPU Partitioning and Task-to-Partition Allocation for Real-Time
 * Workloads").  Library: paper_2105_10312_b200/libgpart.so (sm_100a).
 *
 * Citations: "P:n" = line n of the paper text with its section /
 * equation / algorithm; "S:n" = SPEC.md line n; readings "A-n" and the
 * definitions "C.1.x" are listed in DESIGN.md ("Readings", "Definitions").
 *
 * Conventions (all calls):
 *  - Every call returns gp_status.  Nothing throws, aborts, exits or prints.
 *    On error gp_last_error() (thread-local, valid until the next gp_* call
 *    on the same thread) describes the first failing check.
 *  - Ownership: the CALLER allocates and frees every buffer.  Buffers marked
 *    "device" must be device (or managed) memory; "host" buffers are read
 *    during the call only.  The library makes no persistent allocations and
 *    changes no device or memory-pool attribute.  Scratch the caller does not
 *    provide (gp_allocate's 8-byte set counter; gp_sched_ratio(EXHAUSTIVE)'s
 *    workspace when gp_exhaustive_opts.workspace is NULL) is a stream-ordered
 *    temporary: cudaMallocAsync on `stream` from the device's current memory
 *    pool, cudaFreeAsync on `stream` after the call's last kernel.
 *  - Reentrancy: no host-side mutable state (no static caches); calls may run
 *    concurrently from several host threads on different streams / devices.
 *    Kernel attributes (dynamic shared memory limits) are set per call.
 *  - Configuration: there are no environment-variable switches.  Behaviour is
 *    selected by arguments only (flags below); performance A/B variants are
 *    compile-time macros of the build (-DGP_ALLOC_TAB_KB, -DGP_ALLOC_MIN_G,
 *    -DGP_BP_MINB, -DGP_MEMO_MINB, -DGP_BP_CORNER, -DGP_BP_FULLCORNER; defaults are
 *    the product).
 *  - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy
 *    default stream).  Every device call only ENQUEUES work on that stream
 *    and returns; none synchronises.  Outputs are valid once the stream has
 *    progressed past the call.  gp_count_candidates is host-only.
 *  - Task sets hold 1..256 tasks (gp_generate, gp_allocate); the enumeration
 *    calls are limited to n_tasks <= 12 (the candidate count must stay < 2^63).
 *  - Layout of every per-task field is [n_sets][n_tasks]: the tasks of one
 *    set are contiguous (set-major, task-minor), so one warp reads one set's
 *    field with one coalesced 128-byte access at n_tasks = 32.
 *  - Time is integer ticks (C.1.1).  All arithmetic is integer.
 *  - Device-side input contract (checked per set inside the kernels, since
 *    the data are on the device): 1 <= T, 0 < D <= T, B >= 1, 1 <= cn <= cc,
 *    0 <= fn <= fc, and H * (n_tasks + 1) < 2^31 where H = lcm of the set's
 *    periods.  A set that violates it is reported, never silently wrapped:
 *    gp_sched_ratio(EXHAUSTIVE) writes per_set n_sched = -1 and counts it as
 *    invalid; gp_allocate writes ok = 0 and n_tests = -1.  Sets produced by
 *    gp_generate always satisfy it (gp_generate refuses parameters that could
 *    break it with GP_EOVERFLOW).
 *  - Determinism: identical inputs give identical outputs, byte for byte,
 *    whatever the grid, stream or number of GPUs (integer sums only).
 */
#ifndef GPART_H
#define GPART_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GP_OK = 0,
  GP_EINVAL = 1,    /* malformed argument (S:62 m = 0, S:82 task outside block, ...) */
  GP_EOVERFLOW = 2, /* a count, hyperperiod or field would not fit */
  GP_ECUDA = 3      /* a CUDA launch failed; see gp_last_error() */
} gp_status;

/* Thread-local message for the last failing call on this thread ("" if none). */
const char *gp_last_error(void);

/* A batch of task sets (§4.2 task model P:449-471; D3 of DESIGN.md).
 * Device pointers owned by the caller.  n_tasks in 1..256, M in 1..1024.   */
typedef struct {
  int32_t n_sets, n_tasks, M, n_groups;
  int32_t *T;    /* period T_i, ticks                         [n_sets][n_tasks] */
  int32_t *D;    /* relative deadline D_i, 0 < D <= T         [n_sets][n_tasks] */
  int32_t *B;    /* thread blocks of the kernel (P:7, example)         [n_sets][n_tasks] */
  int32_t *cn;   /* per-wave block cost without conflict (C^n)  [n_sets][n_tasks] */
  int32_t *cc;   /* per-wave block cost in conflict (C^c)   [n_sets][n_tasks] */
  int32_t *fn;   /* non-parallel floor without conflict (b^n)   [n_sets][n_tasks] */
  int32_t *fc;   /* non-parallel floor in conflict (b^c)        [n_sets][n_tasks] */
  uint8_t *type; /* M_i: 0 = compute-, 1 = memory-intensive     [n_sets][n_tasks] */
  uint8_t *valid;/* 0 = generator discard budget exhausted (counted unschedulable) [n_sets] */
  int32_t *group;/* segment of the ratio reduction: prm_idx * n_bins + bin  [n_sets] */
} gp_tasksets;

/* Generator parameters (§7.1; C.1.10).  Host memory. */
typedef struct {
  int32_t M, n_tasks, n_bins, n_prm, sets_per_group;
  const uint64_t *prm_q;          /* [n_prm]; task is memory-intensive iff Philox w0 < prm_q
                                     (prm_q = floor(prm * 2^32) <= 2^32, A-15)   */
  int32_t ticks_per_unit;         /* Q: ticks per paper time unit (C.1.1), Q*menu % 4 == 0    */
  int32_t n_periods;              /* 1..16                                                     */
  const int32_t *period_menu;     /* [n_periods] paper units, strictly ascending, > 0 (A-11)  */
  int32_t b_max;                  /* blocks ~ U{1..b_max} (A-13)                               */
  int32_t beta_c_num, beta_m_num, beta_den; /* b = beta * a: 2/100, 10/100          */
  int32_t kc_num, km_num, k_den;  /* conflict factor k: 12/10, 23/10, k >= 1         */
  int32_t max_attempts;           /* UUniFast-Discard budget per set (A-9)                     */
  int32_t curve_gran;             /* 0: block mode (B ~ U{1..b_max}, cn = ceil(a/B)).  g > 0:
                                     curve mode (reading A-1): the §7.1 curve
                                     C = k(a/|P| + b) in the W form with B = ceil(a/g) granules
                                     of g ticks, cn = g, cc = ceil(k g)                       */
} gp_gen_params;

typedef enum { GP_1G = 0, GP_SMS_ACT = 1, GP_SMS_INA = 2, GP_BF_ACT = 3, GP_BF_INA = 4 } gp_variant;
typedef enum {
  GP_FROM_VERDICTS = 0, GP_EXHAUSTIVE = 1, GP_THRESHOLD = 2, GP_FROM_PER_SET = 3
} gp_ratio_mode;

/* ---------------------------------------------------------------------------
 * A1. gp_generate -- counter-based synthetic task sets (§7.1; C.1.10).
 * For every group (prm_idx, bin) (n_prm * n_bins groups) it produces the
 * repetitions rep_begin .. rep_begin + rep_count - 1 (rep_begin + rep_count <=
 * sets_per_group).  Local set l = group * rep_count + (rep - rep_begin); the
 * global index g = group * sets_per_group + rep keys Philox4x32-10 with
 * counter (g, attempt, task) and key = seed, so any GPU can produce any set
 * and a range split across calls / GPUs is byte-identical to one call.
 * Per set: types by prm, utilisations by UUniFast-Discard realised
 * as sorted integer spacings summing exactly to U_q = (bin+1) M 2^20 / n_bins
 * (A-12, A-31), periods from the menu with the "reasonable execution
 * time" bump (A-10), D = 3T/4, per-wave cost
 * cn = max(1, ceil(a/B)), floor fn = ceil(beta a), conflict costs
 * cc = ceil(k cn), fc = ceil(k fn) (A-14); whole-vector discard if
 * any task is infeasible alone on M SMs (A-9); valid = 0 after max_attempts.
 * out: device buffers with out->n_sets == n_prm * n_bins * rep_count and
 * out->n_tasks == p->n_tasks; out->M / n_groups are set by the call (host).
 * Errors: GP_EINVAL (bad parameters), GP_EOVERFLOW (a field could exceed
 * int32 or H*(n+1) could reach 2^31), GP_ECUDA.
 * ------------------------------------------------------------------------- */
gp_status gp_generate(const gp_gen_params *p, uint64_t seed, uint64_t rep_begin,
                      int32_t rep_count, gp_tasksets *out, void *stream);

/* ---------------------------------------------------------------------------
 * A2. Candidate space (§5 intro; C.1.6).  A candidate is (k, pi, s):
 * pi a restricted growth string over the n tasks with exactly k labels (the
 * task-to-partition allocation), s in Z>=1^k with sum(s) <= M (the SM
 * partitioning; leftover SMs idle).  Rank order: k ascending, pi
 * lexicographic, s lexicographic.  Count N_c(M,n) = sum_k S(n,k) C(M,k).
 * gp_count_candidates (HOST ONLY, no CUDA): GP_EOVERFLOW if N_c >= 2^63.
 * ------------------------------------------------------------------------- */
gp_status gp_count_candidates(int32_t M, int32_t n, uint64_t *count /*host*/);

/* gp_enumerate: ranks first_rank .. first_rank+count-1 -> block_of_task
 * (device int8 [count][n], the RGS: block label of task i) and block_size
 * (device int16 [count][n], s_0..s_{k-1} then zeros).  Errors: GP_EINVAL
 * (n not in 1..12, M not in 1..256, count < 0, range beyond N_c, or
 * C(M,k) >= 2^32 for some k <= n), GP_EOVERFLOW (N_c >= 2^63).           */
gp_status gp_enumerate(int32_t M, int32_t n, uint64_t first_rank, int64_t count,
                       int8_t *block_of_task, int16_t *block_size, void *stream);

/* ---------------------------------------------------------------------------
 * A3. gp_wcet -- interference-aware WCET of every task of every candidate
 * (case equation; conflict definition; W form C.1.3):
 *   x_i = [another task of the same type shares i's block]     (A-4)
 *   W_i = ceil(B_i / s_b) * c_i^x + f_i^x  (b = block_of_task[i], s_b = size)
 * set_of_cand: device int32 [n_cand] set index per candidate;
 * block_of_task / block_size: device [n_cand][n_tasks] as gp_enumerate.
 * Outputs (device): wcet int32 [n_cand][n_tasks], conflict uint8 [n_cand][n_tasks].
 * A malformed candidate (set out of range, label out of range, size <= 0 for
 * a used block) gets wcet = -1 and conflict = 255 for the affected tasks
 * (the data are on the device, so this is reported in-band).  W values that
 * exceed int32 saturate at INT32_MAX.
 * ------------------------------------------------------------------------- */
gp_status gp_wcet(const gp_tasksets *ts, const int32_t *set_of_cand,
                  const int8_t *block_of_task, const int16_t *block_size, int64_t n_cand,
                  int32_t *wcet, uint8_t *conflict, void *stream);

/* Per-SM form of the worked example only (figure; C.1.4):
 * B blocks dealt round-robin from SM 0 over m SMs (A-5); SM j
 * costs cost_per_sm[j] per block; per_sm[j] = blocks_on(j)*cost_per_sm[j] + f;
 * task_wcet[0] = max_j per_sm[j].  Device buffers: cost_per_sm, per_sm [m],
 * task_wcet [1].  GP_EINVAL if m < 1 or m > 1024 or B < 0.                */
gp_status gp_wcet_per_sm(int32_t B, int32_t m, const int32_t *cost_per_sm, int32_t f,
                         int32_t *per_sm, int32_t *task_wcet, void *stream);

/* ---------------------------------------------------------------------------
 * A5. gp_allocate -- the paper's heuristics, one warp per task set.
 * GP_1G: all tasks in one partition of M SMs.
 * GP_{SMS,BF}_{ACT,INA}: Lemma 1 -> Lemma 2 sizes ->
 * par_list sorted by U*H descending (Def. 5 U with /T_i, A-17,
 * A-19) -> Lemma 3 exit (A-24) -> [ACT: every task pair tried,
 * failures forbidden, P:781] -> Algorithm 1 loop with Algorithm 3
 * select (A-18, A-23, A-26), Algorithm 2 merge with the linear
 * m scan (Def. 3, A-25), SMS = order >> (Def. 4 P:729,
 * A-20, A-22), BF = order > (Def. 5, A-21).  Per-partition test: EDF
 * processor-demand criterion (A-6; C.1.7).
 * Outputs (device, [n_sets] unless noted): ok (1 = schedulable), block_of_task
 * int16 [n_sets][n_tasks] canonical labels (blocks numbered by their lowest
 * task; -1 when rejected by Lemma 1/2), block_size int16 [n_sets][n_tasks]
 * (0-padded), pi (= sum of sizes, 0 when rejected by Lemma 1/2), k (number
 * of partitions, 0 when rejected by Lemma 1/2), n_tests (EDF-PDC calls; the
 * heuristic-mode "candidate eval" unit).  On a failed Algorithm 1 run the
 * partitions at the moment of failure are reported with ok = 0.
 * efficiency: device int64 [n_sets][4] or NULL (P:965-966,
 * P:1009-1014): the scheduled workload as work per period scaled by
 * the set's hyperperiod H -- {lower = sum cn_i B_i H/T_i (no conflict),
 * upper = sum cc_i B_i H/T_i (all in conflict), achieved = sum c_i^x B_i H/T_i
 * for the reported partitions (0 when rejected by Lemma 1/2), H}.
 * Algorithm 2's size search (paper default): the first schedulable m of
 * max(|P1|,|P2|) .. |P1|+|P2|-1 is found by one test at the top size and a
 * binary search below it -- exact, since EDF-PDC(P, m) is monotone in m (C.1.3)
 * -- while n_tests counts the tests of the paper's linear scan (first success -
 * lo + 1, or the whole range), so every output equals the sequential algorithm's.
 * stats: device uint64 [4] (or [8] with GP_AL_STATS_EXT) or NULL; += {EDF-PDC
 * tests as n_tests counts them, tasks in the tests actually run, distinct
 * deadlines examined by their demand walks, sets} (the per-launch work figures
 * of the roofline).
 * opts: NULL or the f4 variants below.
 * Errors: GP_EINVAL (bad struct / variant / options), GP_ECUDA.
 * ------------------------------------------------------------------------- */
typedef enum {
  GP_AL_BINARY_MERGE = 1, /* Algorithm 2 by binary search "between max{|P1|,|P2|} and
                             |P1|+|P2|": lower-bound search over the ascending
                             candidate sizes (lo = 0, hi = |L|, mid = (lo+hi)/2).  Same
                             partitions as the linear scan (schedulability is monotone in m),
                             fewer EDF tests; only n_tests changes.                         */
  GP_AL_INCREASING = 2,   /* par_list in increasing utilisation order; ties by
                             lower min task id.  Best-fit partner order stays U*H desc (A-21). */
  GP_AL_STATS_EXT = 4     /* not a variant: `stats` has 8 slots; [4..7] += {EDF tests actually
                             run, Algorithm 3 selections, partitions those selections scanned,
                             Algorithm 2 partner searches} (the roofline's executed work)      */
} gp_alloc_flag;

/* f4 options of gp_allocate.  Host memory; NULL = the paper's
 * defaults (linear scan, decreasing order, every partition size).
 * size_mask: NULL, or ceil(M/32) host words; bit (m-1) % 32 of word (m-1) / 32
 *   set = partitions of m SMs are admissible (MIG-style slices).  Bits
 *   above M are ignored; at least one size in 1..M must be admissible
 *   (GP_EINVAL).  With a mask, Lemma 2 sizes round up to the next admissible
 *   size, Algorithm 2 tries admissible sizes only (all <= M), and 1G uses the
 *   largest admissible size.  Without a mask merged sizes follow the paper
 *   (Algorithm 2 may try sizes above M).  Placement of slices on the GPU (GPC
 *   boundaries) is not modelled: only the sizes are restricted.              */
typedef struct {
  uint32_t flags;            /* gp_alloc_flag bits; unknown bits -> GP_EINVAL */
  const uint32_t *size_mask; /* see above */
  const uint32_t *memo;      /* NULL, or DEVICE block verdict words of the SAME task sets,
                                subset-major: word S of set s at memo[S * memo_stride + s]
                                (bit m-1 = task subset S passes EDF-PDC on m SMs, C.1.7): the
                                first 2^n_tasks * N words of the caller-owned workspace of a
                                gp_sched_ratio(GP_EXHAUSTIVE) call on N sets that ran the
                                bit-sliced evaluator without a size_mask (n_tasks <= 8, M <=
                                32, not GP_EX_PER_CANDIDATE), earlier on the stream (memo_stride
                                = N; sets [h, h + n_sets) of that call: memo + h).  Row S = 0
                                holds the set's hyperperiod H (0: input contract violated),
                                which the heuristics then take instead of recomputing it.
                                Every EDF test the heuristics run at a size m <= M becomes a
                                lookup (U*H is still computed for the partition orders); outputs
                                are identical.  n_tasks > 8 or M > 32 -> GP_EINVAL; a memo of
                                other sets or of a masked call gives wrong verdicts (the library
                                cannot check it).                                           */
  int64_t memo_stride;       /* words between the subsets' rows of memo; 0 = n_sets; < n_sets
                                -> GP_EINVAL                                                    */
} gp_alloc_opts;

gp_status gp_allocate(const gp_tasksets *ts, gp_variant v, const gp_alloc_opts *opts,
                      uint8_t *ok, int16_t *block_of_task, int16_t *block_size, int32_t *pi,
                      int32_t *k, int64_t *n_tests, int64_t *efficiency,
                      unsigned long long *stats, void *stream);

/* ---------------------------------------------------------------------------
 * A6 (and A2-A4 fused). gp_sched_ratio -- segmented reduction to the
 * schedulability-rate counts (§7.2; C.1.11):
 *   counts[setting][group][slot][0] += ok * valid   (schedulable)
 *   counts[setting][group][slot][1] += 1            (total)
 *   counts[setting][group][slot][2] += !valid       (generator discards)
 * counts: device int64 [n_settings][n_groups][n_slots][3], ACCUMULATED (+=);
 * the caller zeroes it once.  The rate is sched / total.
 *
 * mode GP_FROM_VERDICTS: verdicts is device uint8 [n_rows][n_sets] (e.g. the
 *   ok outputs of gp_allocate, one row per variant); row r goes to slot
 *   slot0 + r.  `ex` must be NULL.
 * mode GP_EXHAUSTIVE: evaluates every candidate of every set directly --
 *   rank -> (k, pi, s) unranking, conflict flags and W per task (A3), and
 *   the EDF processor-demand test of every block (A4); candidate verdict =
 *   AND over its blocks (C.1.8).  For n_tasks <= 8 and M <= 32 the block
 *   verdicts are memoised per (task subset, size) -- 2^n - 1 subsets x M
 *   sizes, each tested unless a subset S - {i} already fails at that size (S
 *   then fails too: fewer tasks, no more conflicts) -- and each candidate's verdict is the AND of its
 *   blocks' memoised verdicts, evaluated 32 candidates per word along runs of
 *   the last part (workspace: gp_exhaustive_opts.workspace, or a stream-ordered
 *   temporary, see gp_exhaustive_workspace_size); GP_EX_PER_CANDIDATE forces the
 *   per-candidate EDF tests.  Both give identical outputs.  Per set it writes ex->per_set[set][4] =
 *   {n_sched, pi_star = min sum(s) over schedulable candidates (0 if none),
 *   first_rank (-1 if none), hash = sum of splitmix64(rank) mod 2^64 over
 *   schedulable ranks}, optional per-candidate verdict bits, and adds the
 *   set verdict "exists = n_sched > 0" to counts slot slot0 (n_rows must be
 *   1, verdicts NULL).  With a partial rank window, counts must be NULL (the
 *   per-window per_set rows merge by sum / min / min / sum).
 *   Limits: n_tasks <= 12, M <= 256, C(M,k) < 2^32; else GP_EINVAL; N_c >=
 *   2^63 -> GP_EOVERFLOW.
 * mode GP_FROM_PER_SET: the EXHAUSTIVE counting from per-set outputs computed
 *   elsewhere (ex->per_set, READ-ONLY [n_sets][4] in the EXHAUSTIVE convention, e.g.
 *   the per-set merge of candidate-rank shards over several GPUs):
 *   exists = n_sched > 0, a set with n_sched < 0 (contract violated) or valid = 0 is
 *   counted invalid -- the counts equal those of one full-window EXHAUSTIVE call.
 *   verdicts NULL, n_rows 1; only ex->per_set is read.
 * mode GP_THRESHOLD (a different work unit, reported
 *   separately): the same per_set outputs and counts as GP_EXHAUSTIVE, exact by
 *   resource monotonicity: per set, m*(S) = min{s : EDF-PDC(S,s)}
 *   for each of the 2^n - 1 task subsets (binary search), then per allocation
 *   pi the schedulable size vectors are exactly s >= m* (componentwise), so
 *   n_sched = sum_pi C(M - sum(m* - 1), k), pi_star = min sum(m*), first_rank =
 *   rank(pi, m*); the hash enumerates the schedulable vectors only (skipped with
 *   GP_EX_NO_HASH).  Full rank window only; verdict_bits must be NULL;
 *   work_counter optional (when given: the sets' work queue).
 * ------------------------------------------------------------------------- */
typedef struct {
  uint64_t rank_lo, rank_hi;  /* window [lo, hi) of candidate ranks; hi = UINT64_MAX -> N_c  */
  int64_t *per_set;           /* device int64 [n_sets][4], required                           */
  uint32_t *verdict_bits;     /* device [n_sets][words_per_set] or NULL; bit (r - lo) of set  */
  int64_t words_per_set;      /* >= ceil((hi - lo) / 32) when verdict_bits != NULL            */
  unsigned long long *work_counter; /* device scratch, >= 1 u64 (work queue), required     */
  unsigned long long *stats;  /* device [4] or NULL: += {candidates, block tests,
                                 deadline points examined, tasks in tested blocks}
                                 (THRESHOLD: {sets, threshold tests, deadline points,
                                 schedulable candidates enumerated for the hash});
                                 [12] with GP_EX_STATS_EXT: [4] += (set, run) pairs the
                                 bit-sliced evaluator walked one by one, [5] += those with a
                                 non-zero verdict word (a run = the candidates of one
                                 allocation that differ in the last part only), [6] += (set,
                                 sweep) pairs it resolved in closed form (a sweep = the runs
                                 that differ in the second-to-last part only), [7] += the
                                 live runs inside them, [8] += (set, block) pairs whose hash
                                 was one corner-table read (a block = the candidates of one
                                 allocation that differ in the last three parts only), [9] +=
                                 the sweeps inside them (also counted in [6]), [10] +=
                                 (set, allocation) pairs resolved as one full corner (every
                                 block word one bit range; closed form, one table read),
                                 [11] += their blocks; 0 for the other evaluators           */
  uint32_t flags;             /* GP_EX_NO_HASH: skip the verdict hash (per_set[3] = 0);
                                 GP_EX_PER_CANDIDATE (EXHAUSTIVE): force the per-candidate
                                 evaluator; GP_EX_STATS_EXT: stats has 12 slots (above);
                                 test hooks (same outputs, other code paths):
                                 GP_EX_FORCE_RANGES: the bit-sliced evaluator walks every
                                 verdict word range by range (no contiguous fast path);
                                 GP_EX_NATURAL_ORDER: accepted, no effect (the bit-sliced
                                 evaluator's lanes always take sets in index order now);
                                 GP_EX_NO_FULL_CORNER: the bit-sliced evaluator resolves no
                                 (set, allocation) pair as one full corner (its corner-table
                                 blocks, closed-form sweeps and run walks do all the work);
                                 GP_EX_GENERIC: the per-candidate evaluator with runtime
                                 block structure (no shape specialisation), implies
                                 GP_EX_PER_CANDIDATE; unknown bits -> GP_EINVAL              */
  void *workspace;            /* device scratch, 256-byte aligned, of at least
                                 gp_exhaustive_workspace_size() bytes for this call's shapes
                                 and flags, owned by the caller; NULL: a stream-ordered
                                 temporary of that size is allocated and released on `stream` */
  uint64_t workspace_bytes;   /* size of `workspace` (GP_EINVAL if too small)                  */
  const uint32_t *size_mask;  /* EXHAUSTIVE / THRESHOLD: NULL, or
                                 ceil(M/32) HOST words in gp_alloc_opts' layout -- bit (m-1) % 32
                                 of word (m-1) / 32 set = partitions of m SMs are admissible
                                 (MIG-style slices).  Reading B-9: a candidate that
                                 uses an inadmissible size is not deployable and counts as
                                 unschedulable; the rank space, N_c and the ranks are unchanged,
                                 so per_set, verdict bits and windows keep their meaning.  No
                                 admissible size in 1..M -> GP_EINVAL.  THRESHOLD: the count and
                                 hash walk the schedulable runs (cost grows with n_sched)      */
  uint64_t *tables_key;       /* HOST, caller-owned, or NULL (bit-sliced evaluator with a caller
                                 workspace only).  The workspace also holds tables that depend
                                 on (n_tasks, M) only -- RGS labels, the verdict-hash prefix
                                 tables and the corner tables -- like an FFT plan's twiddles.
                                 The call rebuilds them unless *tables_key equals the key of
                                 this call's layout (shapes, flags, workspace address and size),
                                 then stores that key (0 on error).  The caller zeroes it
                                 whenever the workspace is written by anything else, and orders
                                 a call on another stream after the call that built them.
                                 NULL: rebuilt every call                                       */
} gp_exhaustive_opts;
#define GP_EX_NO_HASH 1u
#define GP_EX_PER_CANDIDATE 2u
#define GP_EX_STATS_EXT 4u
#define GP_EX_FORCE_RANGES 8u
#define GP_EX_NATURAL_ORDER 16u
#define GP_EX_GENERIC 32u
#define GP_EX_NO_FULL_CORNER 64u

/* HOST ONLY (no CUDA call): device workspace bytes gp_sched_ratio(mode, flags) needs
 * for n_sets sets of n_tasks tasks on M SMs in n_groups groups -- the bit-sliced
 * evaluator's memo words (n_sets * 2^n * 4 B) and its input-independent tables (RGS
 * labels; when N_c < 2^24 and the hash is wanted: the verdict-hash prefix table and the
 * full corner table, 8 B per rank each, the corner table of the last three parts, 8 B
 * per rank, and the run-prefix table, 8 B per (run, size)); 0 for the per-candidate and
 * threshold evaluators and for FROM_VERDICTS.  C3 with 10^5 sets: about 66 MB.  Errors: GP_EINVAL (shapes outside the EXHAUSTIVE limits). */
gp_status gp_exhaustive_workspace_size(int32_t n_sets, int32_t n_tasks, int32_t M,
                                       int32_t n_groups, gp_ratio_mode mode, uint32_t flags,
                                       uint64_t *bytes /*host*/);

gp_status gp_sched_ratio(const gp_tasksets *ts, gp_ratio_mode mode, const uint8_t *verdicts,
                         int32_t n_rows, int32_t slot0, int32_t n_slots, int32_t setting,
                         int64_t *counts, const gp_exhaustive_opts *ex, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GPART_H */

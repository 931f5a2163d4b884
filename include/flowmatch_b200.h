/*
 * flowmatch_b200.h -- C ABI of the B200-native grid max-flow / dense assignment
 * hot path (libfm_b200.so).  Plain pointers and sizes only; no torch types.
 *
 * Each entry point replaces one reference interface (reference package
 * `flowmatch`, /root/reference/pkg/src/flowmatch):
 *
 *   fm_grid_solve / fm_grid_solve_host
 *       replaces hybrid_solve(net, worker_count, cycle_budget, observer=None)
 *       (maxflow_par.py:157-238) on 4-connected grid networks, which runs
 *       hybrid_init (maxflow_par.py:44-62), init_preflow (maxflow_seq.py:47-64),
 *       lockfree_round (maxflow_par.py:65-129), cancel_violations
 *       (maxflow_par.py:132-154, opt-in flag), global_relabel + gap_relabel
 *       (maxflow_seq.py:119-160) and the marking / ExcessTotal test
 *       (maxflow_par.py:195,223-226).  Adds the minimal source-side cut the
 *       reference does not expose.
 *   fm_grid_begin / fm_grid_round / fm_grid_export
 *       the same solve one coordinator round at a time, so the Python mirror
 *       can honour hybrid_solve's observer(net, hybrid, scanned) hook
 *       (maxflow_par.py:165-166,228-229).
 *   fm_assign_solve / fm_assign_solve_host
 *       replaces solve_assignment(inst, mode="par", ...) (assign_scaling.py:470-497)
 *       = make_scaling_state (:127-142) + min_cost_loop (:400-467) with
 *       begin_refine (:145-182), refine_par / lockfree_refine_round
 *       (assign_par.py:45-237), arc_fix (:185-205), extract_matching (:380-397).
 *
 * Grid layout (all int32, H x W row-major, pixel p = r * W + c):
 *   capR[p]  capacity p -> p+1   (last column must be 0)
 *   capL[p]  capacity p -> p-1   (first column must be 0)
 *   capD[p]  capacity p -> p+W   (last row must be 0)
 *   capU[p]  capacity p -> p-W   (first row must be 0)
 *   capS[p]  capacity s -> p,    capT[p] capacity p -> t;   all >= 0.
 * This is the reference network built by the SURVEY.md 8d adapter (s = H*W,
 * t = H*W + 1) with antiparallel pairs merged; value and minimal cut are equal.
 *
 * Status codes (Python mirror maps 1 -> InfeasibleInstanceError, 2 -> ValueError,
 * 3/4 -> RuntimeError, 5 -> AssertionError, as the reference raises at
 * assign_scaling.py:44-45, maxflow_par.py:168-173, maxflow_par.py:213-214,
 * assign_par.py:101-106,200-214).
 */
#ifndef FLOWMATCH_B200_H
#define FLOWMATCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FM_OK 0
#define FM_INFEASIBLE 1
#define FM_INVALID_ARG 2
#define FM_CUDA_ERROR 3
#define FM_NO_DEVICE 4
#define FM_VALIDATION 5   /* validate=True invariant violated (the reference raises AssertionError) */

/* grid solve flags */
#define FM_GRID_CANCEL_VIOLATIONS 0x1 /* run the maxflow_par.py:132-154 pass each round */
#define FM_GRID_NO_PRECANCEL 0x2      /* do not pre-route min(capS, capT) straight to t */
#define FM_GRID_NO_CUT 0x4            /* skip the min-cut reach */
#define FM_GRID_GLOBAL_SWEEP 0x8      /* A/B: one-thread-per-pixel global-memory sweeps (K1 v1)
                                         instead of the tile-resident kernel (K1 v2) */

/* assignment flags (match solve_assignment keyword arguments) */
#define FM_ASSIGN_PRICE_UPDATE 0x1 /* use_price_update (assign_scaling.py:208-276) */
#define FM_ASSIGN_ARC_FIX 0x2      /* use_arc_fix (assign_scaling.py:185-205) */
#define FM_ASSIGN_VALIDATE 0x4     /* validate=True: device-side invariant checks */

/* dense weight marking an absent arc (sparse instance, complete=False) */
#define FM_ABSENT_WEIGHT INT32_MIN

typedef struct fm_stats {
    int64_t pushes;        /* SolveReport.pushes */
    int64_t relabels;      /* SolveReport.relabels */
    int64_t rounds;        /* SolveReport.rounds: coordinator passes */
    int64_t launches;      /* kernels launched by this solve */
    int64_t pr_sweeps;     /* push-relabel sweeps (grid) / refine phases (assign) */
    int64_t bfs_sweeps;    /* global-relabel tile sweeps (grid) */
    int64_t bfs_levels;    /* deepest residual distance seen by a global relabel */
    int64_t cut_sweeps;    /* min-cut reach tile sweeps */
    int64_t refines;       /* assignment: epsilon phases */
    int64_t bytes_push;    /* algorithmic bytes moved by the push-relabel kernels */
    int64_t bytes_bfs;     /* algorithmic bytes moved by global relabel + cut */
    int64_t pr_tiles;      /* tile visits by the push-relabel kernel */
    double ms_total;       /* device time of the whole solve (CUDA events) */
    double ms_push;        /* push-relabel kernels */
    double ms_bfs;         /* global relabel + gap + mark */
    double ms_cut;         /* min-cut reach */
    double ms_h2d;         /* *_host variants only */
    double ms_d2h;         /* *_host variants only */
    double ms_pr_kern;     /* push-relabel kernels alone (events around launch batches) */
    double ms_bfs_kern;    /* global-relabel tile kernels alone */
    int64_t pr_launches;   /* push-relabel kernel launches */
    int64_t bfs_launches;  /* global-relabel tile kernel launches */
    int64_t reserved[4];
} fm_stats;

/* ----------------------------------------------------------------- common */
const char *fm_last_error(void);  /* thread-local message for the last failure */
int fm_device_count(void);
const char *fm_version(void);

/* ------------------------------------------------------------------- grid */
typedef struct fm_grid fm_grid;

int fm_grid_create(int32_t H, int32_t W, int32_t device, fm_grid **out);
void fm_grid_destroy(fm_grid *g);
/* Kernel-variant and tuning options (DESIGN.md section 4 switch table, lower-case
 * names, e.g. "pr_kernel", "bfs_bits", "packed").  The library reads no environment
 * variables; options apply from the next solve.  Unknown name -> FM_INVALID_ARG. */
int fm_grid_set_option(fm_grid *g, const char *name, int64_t value);

/* Whole solve on device.  cap* are DEVICE pointers (borrowed for the call).
 * cycle_budget = max lock-free sweeps per coordinator round (reference
 * DEFAULT_CYCLE_BUDGET 7000, maxflow_par.py:28).  bfs_interval = sweeps between
 * global relabels inside a round (0 = library default).  flow_out: host int64.
 * cut_out: DEVICE uint8[H*W] (1 = source side) or NULL.  stream: cudaStream_t
 * or NULL for the library's own stream. */
int fm_grid_solve(fm_grid *g, const int32_t *capR, const int32_t *capL,
                  const int32_t *capD, const int32_t *capU, const int32_t *capS,
                  const int32_t *capT, int32_t cycle_budget, int32_t bfs_interval,
                  int32_t flags, int64_t *flow_out, uint8_t *cut_out,
                  fm_stats *stats, void *stream);

/* Same, HOST pointers (copies in and out are part of the call; cut_out host). */
int fm_grid_solve_host(fm_grid *g, const int32_t *capR, const int32_t *capL,
                       const int32_t *capD, const int32_t *capU, const int32_t *capS,
                       const int32_t *capT, int32_t cycle_budget, int32_t bfs_interval,
                       int32_t flags, int64_t *flow_out, uint8_t *cut_out,
                       fm_stats *stats);

/* A batch of `count` independent H x W instances from HOST planes (caps[6 k + p] =
 * plane p of instance k, in the order capR, capL, capD, capU, capS, capT; elements of
 * elem_bytes = 4 (int32), 2 (uint16) or 1 (uint8): narrow planes cross PCIe narrow and
 * are widened on the device), pipelined:
 * the H2D of instance k+1 and the D2H of instance k-1's cut overlap the solve of
 * instance k.  flows_out[count]; cuts_out[count] host arrays (NULL, or an entry NULL:
 * no cut for it); stats: NULL or count entries.  Each result equals
 * fm_grid_solve_host's.  No reference counterpart: the reference solves one network
 * per hybrid_solve call (maxflow_par.py:157-238); a caller's loop over images maps to
 * one call. */
int fm_grid_solve_host_batch(fm_grid *g, int32_t count, const void *const *caps, int32_t elem_bytes,
                             int32_t cycle_budget, int32_t bfs_interval, int32_t flags,
                             int64_t *flows_out, uint8_t *const *cuts_out, fm_stats *stats);

/* Stepwise solve (observer support).  begin copies HOST capacities in and runs
 * the preflow init + first global relabel; round runs one coordinator round
 * (lock-free sweeps, then cancel (opt), global relabel, gap, mark) and sets
 * *done when no unmarked pixel holds excess. */
int fm_grid_begin(fm_grid *g, const int32_t *capR, const int32_t *capL,
                  const int32_t *capD, const int32_t *capU, const int32_t *capS,
                  const int32_t *capT, int32_t flags);
int fm_grid_round(fm_grid *g, int32_t cycle_budget, int32_t bfs_interval,
                  int32_t *done, fm_stats *stats);
/* Copy the current state to HOST buffers (any may be NULL).  rS = flow on s->p.
 * marked = pixels written off by the gap step (maxflow_par.py:223-226). */
int fm_grid_export(fm_grid *g, int32_t *rR, int32_t *rL, int32_t *rD, int32_t *rU,
                   int32_t *rT, int32_t *rS, int32_t *e, int32_t *h, uint8_t *marked,
                   int64_t *flow, int64_t *excess_total);
/* Minimal source-side cut of the current state into a HOST buffer. */
int fm_grid_cut_host(fm_grid *g, uint8_t *cut_out, fm_stats *stats);

/* Copy the current cut plane without recomputing it (dst host or device). */
int fm_grid_cut_plane(fm_grid *g, uint8_t *dst, int32_t dst_on_host);
/* Counters of the last / current solve. */
int fm_grid_stats(fm_grid *g, fm_stats *stats);

/* ------------------------------------------------------------ row bands
 * Multi-GPU grid path -- the reference's coordinator loop
 * (maxflow_par.py:195-229) run by every band of a grid cut into horizontal bands on
 * 32-row tile boundaries.  A band's kernels read the neighbour bands' boundary rows
 * (heights, BFS distances, cut bits) and push flow into their inboxes directly
 * through peer memory (one process: peer access; one process per GPU: CUDA IPC);
 * the bands' global-relabel and min-cut ring launches end on one shared pending
 * counter.  Host-level agreement (idle / budget / active counts) goes through an
 * fm_coll: a shared-memory barrier + all-gather of a few int64 per push batch.
 * hybrid_solve(net, devices=N) (maxflow_par.py:157-162 plus `devices`) uses an
 * in-process fm_group; torchrun ranks use fm_grid_band_* + fm_coll_create(name). */
typedef struct fm_coll fm_coll;
/* name == NULL: process-local (threads); else a POSIX shared-memory segment that rank
 * 0 creates and the other ranks open (after the caller's own barrier). */
int fm_coll_create(const char *name, int32_t nranks, int32_t rank, fm_coll **out);
void fm_coll_destroy(fm_coll *c);
/* every rank passes n <= 8 values; out[r * n + i] = rank r's value i */
int fm_coll_allgather(fm_coll *c, const int64_t *vals, int32_t n, int64_t *out);
/* band borders: edges[0..nbands] (edges[0] = 0, edges[nbands] = H) */
int fm_band_split(int32_t H, int32_t nbands, int32_t *edges);

/* The handle (fm_grid_create(rows of the band, W, device)) becomes band `band` of
 * `nbands` of an H_total-row grid; `colocated` = bands sharing this device. */
int fm_grid_band_setup(fm_grid *g, int32_t band, int32_t nbands, int32_t H_total, int32_t colocated);
#define FM_BAND_EXPORT_BYTES 1024
/* IPC handles of the buffers neighbours need, for fm_grid_band_link in other processes */
int fm_grid_band_export(fm_grid *g, void *blob);
int fm_grid_band_link(fm_grid *g, const void *up_blob, const void *dn_blob, const void *band0_blob);
/* same-process neighbours (any devices with peer access) */
int fm_grid_band_link_local(fm_grid *g, fm_grid *up, fm_grid *dn, fm_grid *band0);
/* This band's share of the solve; every band calls it at once.  Inputs host or device
 * (UVA): the six planes of the band's rows, capD of the row above the band and capU of
 * the row below it (W each, NULL for the first / last band).  flow_out = the whole
 * grid's flow; cut_out (host or device, band rows) = its rows of the minimal cut. */
int fm_grid_band_solve(fm_grid *g, fm_coll *c, const int32_t *capR, const int32_t *capL,
                       const int32_t *capD, const int32_t *capU, const int32_t *capS,
                       const int32_t *capT, const int32_t *capD_above, const int32_t *capU_below,
                       int32_t cycle_budget, int32_t flags, int64_t *flow_out, uint8_t *cut_out,
                       fm_stats *stats);

/* In-process group: nbands bands of an H x W grid, band k on devices[k] (bands may
 * share a device).  fm_group_solve takes whole-grid planes (host or device) and runs
 * one host thread per band; stats = counters summed over bands, times of the slowest. */
typedef struct fm_group fm_group;
int fm_group_create(int32_t H, int32_t W, int32_t nbands, const int32_t *devices, fm_group **out);
void fm_group_destroy(fm_group *grp);
int fm_group_band(fm_group *grp, int32_t k, fm_grid **band, int32_t *row0, int32_t *rows);
int fm_group_solve(fm_group *grp, const int32_t *capR, const int32_t *capL, const int32_t *capD,
                   const int32_t *capU, const int32_t *capS, const int32_t *capT, int32_t cycle_budget,
                   int32_t flags, int64_t *flow_out, uint8_t *cut_out, fm_stats *stats);
int fm_group_band_stats(fm_group *grp, int32_t k, fm_stats *stats);

/* ---------------------------------------------------------- generic (CSR)
 * hybrid_solve on an arbitrary FlowNetwork (maxflow_par.py:157-238): the arc-pair
 * forward star of graph.py:43-84 as CSR (HOST arrays, copied in): ostart[n+1],
 * oarc[m2] = out-arc slot ids per node in input order, head[m2], cap[m2] (reverse
 * slots 0).  Outputs (HOST, any may be NULL): flow, cut[n] (1 = source side of the
 * minimal min cut), final residuals res[m2] and excesses ex[n]. */
int fm_csr_solve(int32_t n, int32_t s, int32_t t, int64_t m2, const int64_t *ostart,
                 const int32_t *oarc, const int32_t *head, const int32_t *cap,
                 int32_t cycle_budget, int32_t flags, int64_t *flow_out, uint8_t *cut_out,
                 int32_t *res_out, int64_t *ex_out, fm_stats *stats);
/* The same with int64 capacities and residuals, for networks whose capacities leave
 * the int32 range (the reference's capacities are unbounded Python ints, graph.py:87-125):
 * every capacity in [0, 2^62) and the source's total out-capacity below 2^63, so no
 * residual or excess can overflow; FM_INVALID_ARG otherwise.  Grid networks too wide for
 * fm_grid's int32 state are solved through this entry point. */
int fm_csr_solve64(int32_t n, int32_t s, int32_t t, int64_t m2, const int64_t *ostart,
                   const int32_t *oarc, const int32_t *head, const int64_t *cap,
                   int32_t cycle_budget, int32_t flags, int64_t *flow_out, uint8_t *cut_out,
                   int64_t *res_out, int64_t *ex_out, fm_stats *stats);

/* ------------------------------------------------------------- assignment */
typedef struct fm_assign fm_assign;

int fm_assign_create(int32_t n, int32_t device, fm_assign **out);
void fm_assign_destroy(fm_assign *a);
/* Options: "heuristic_every_k" (a price update every k refine rounds,
 * assign_par.py:228-234; 0 = off), and tuning switches "ybatch_min", "pu_ring",
 * "pu_threshold", "tail_threshold", "pu_cap". */
int fm_assign_set_option(fm_assign *a, const char *name, int64_t value);

/* Dense max-weight perfect matching.  weights: DEVICE int32[n*n] row-major,
 * weights[x*n+y] = w(x, y) or FM_ABSENT_WEIGHT.  alpha >= 2 (DEFAULT_ALPHA 10,
 * assign_scaling.py:33).  objective_out: host int64.  match_out: HOST int32[n]
 * (match_out[x] = y).  prices_out: HOST int64[2n] (X then Y) or NULL. */
int fm_assign_solve(fm_assign *a, const int32_t *weights, int64_t alpha, int32_t flags,
                    int64_t *objective_out, int32_t *match_out, int64_t *prices_out,
                    fm_stats *stats, void *stream);
/* Same with a HOST weight matrix (copy in is part of the call). */
int fm_assign_solve_host(fm_assign *a, const int32_t *weights, int64_t alpha,
                         int32_t flags, int64_t *objective_out, int32_t *match_out,
                         int64_t *prices_out, fm_stats *stats);

/* Sparse instances (complete=False) in compressed form: the same cost-scaling solve with
 * O(n + m) memory and O(degree) work per operation (CSR rows in edge order + a column
 * index; assign_scaling.py:61-76,470-497).  HOST arcs (xs, ys, ws) in the
 * instance's edge order, int32 weights, no duplicates; outputs HOST (match_out[x] = y,
 * prices_out 2n or NULL).  1 = no perfect matching. */
int fm_assign_sparse_solve(int32_t n, int64_t m, const int32_t *xs, const int32_t *ys, const int32_t *ws,
                           int64_t alpha, int32_t flags, int32_t device, int64_t *objective_out,
                           int32_t *match_out, int64_t *prices_out, fm_stats *stats);

/* ------------------------------------------------------------------ DIMACS
 * Ingest of the reference's file formats (dimacs.py:123-248) with the same
 * validation and line-numbered messages (fm_last_error).  Call once with null
 * arrays to get the counts, then with arrays of at least that many entries.
 * max: out_nst = {node_count, source, sink} (0-based), arcs in file order, capacities
 *      int64 (any non-negative value the file's integers can hold).
 * asn: *out_n = nodes per side, edges (x, y, w) with sides mapped to 0..n-1. */
int fm_dimacs_parse_max(const char *text, int64_t len, int32_t *out_nst, int64_t *out_m,
                        int32_t *tails, int32_t *heads, int64_t *caps, int64_t cap_arcs);
int fm_dimacs_parse_asn(const char *text, int64_t len, int32_t *out_n, int64_t *out_m,
                        int32_t *xs, int32_t *ys, int64_t *ws, int64_t cap_edges);

/* Stepwise solve, one refine at a time (solve_assignment's on_refine_end hook,
 * assign_scaling.py:419-420,451-452).  begin copies HOST weights; refine runs one
 * epsilon phase and reports the new epsilon and whether it was the last (eps == 1);
 * state copies prices (2n), match (n) and the arc-fix bitmask (n * ceil(n/32)
 * words, bit y of row x) to HOST buffers (any may be NULL). */
int fm_assign_begin(fm_assign *a, const int32_t *weights, int64_t alpha, int32_t flags);
int fm_assign_refine(fm_assign *a, int64_t *eps_out, int32_t *done_out);
int fm_assign_state(fm_assign *a, int64_t *prices, int32_t *match, uint32_t *fixed,
                    int64_t *objective_out, fm_stats *stats);

/* Stateful refine on a caller's ScalingState (assign_scaling.py:102-142), one
 * coordinator step per call, so refine_par (assign_par.py:115-237) and min_cost_loop
 * (assign_scaling.py:400-467) keep their observer / on_refine_end hooks and their
 * in-place state semantics.  All buffers HOST.
 *   load: weights n*n (NULL = keep the loaded matrix), epsilon, scale (arc cost
 *         c(x,y) = -scale * w(x,y); <= 0 means n + 1, the reduce_to_mincost scale),
 *         bound (scaled_cost_bound, < 0 = max |c|), prices 2n (X then Y),
 *         match n (match[x] = y carrying x's unit or -1), fixed n*ceil(n/32) words
 *         (bit y of row x = pair (x, y) fixed).  Y excesses follow from match.
 *   begin_refine: assign_scaling.py:145-182 (epsilon shrink, unfrozen flow dropped,
 *         X prices reset), no push.
 *   round: one coordinator round: every active X gets an op, then up to cycle_budget
 *         Y/X phase pairs; out = {pushes, relabels, phase pairs, active nodes left}.
 *   price_update: assign_scaling.py:208-276 (no-op without active nodes).
 *   arc_fix: assign_scaling.py:185-205; *fixed_pairs = pairs newly fixed.
 *   export: current prices / match / fixed / Y excess / epsilon (any NULL). */
int fm_assign_load(fm_assign *a, const int32_t *weights, int64_t alpha, int32_t flags, int64_t epsilon,
                   int64_t scale, int64_t bound, const int64_t *prices, const int32_t *match,
                   const uint32_t *fixed);
int fm_assign_begin_refine(fm_assign *a, int64_t *eps_out);
int fm_assign_round(fm_assign *a, int32_t cycle_budget, int64_t *out);
int fm_assign_price_update(fm_assign *a);
int fm_assign_arc_fix(fm_assign *a, int64_t *fixed_pairs);
int fm_assign_export(fm_assign *a, int64_t *prices, int32_t *match, uint32_t *fixed, int32_t *y_excess,
                     int64_t *eps_out);

/* Exact optimality certificate of a matching, independent of the solver (CLI
 * verify; replaces the reference's brute-force oracle check, cli.py:157-188, for any
 * n): *certified = 1 when match (HOST, n) is a perfect matching over present pairs
 * whose residual graph has no negative cycle (Bellman-Ford from a virtual source,
 * <= 2n + 2 passes; prices HOST 2n potentials at cost scale `scale` speed it up, or
 * NULL), 0 when a negative cycle proves it suboptimal, -1 when it is not a perfect
 * matching.  weights HOST, or DEVICE when weights_on_device.  Overwrites the handle's
 * solve state. */
int fm_assign_certify(fm_assign *a, const int32_t *weights, int32_t weights_on_device, const int32_t *match,
                      const int64_t *prices, int64_t scale, int32_t *certified, int64_t *objective_out,
                      int32_t *passes_out);

#ifdef __cplusplus
}
#endif
#endif /* FLOWMATCH_B200_H */

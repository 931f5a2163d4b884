// fm_assign.cu -- B200-native cost-scaling assignment (max-weight perfect matching)
// on dense integer weight matrices.
//
// Replaces solve_assignment(mode="par") (assign_scaling.py:470-497): the reduction
// to min-cost flow with costs -(n+1) w (assign_scaling.py:85-99), the integral
// epsilon schedule eps <- max(1, ceil(eps/alpha)) down to 1 (:145-182, :400-467),
// the refine run as push-relabel (assign_par.py:45-237), arc fixing (:185-205) and
// matching extraction (:380-397).
//
// Device representation of the unit-capacity network: X nodes
// hold excess 0/1, so an X node's flow is one int match[x] (-1 = unmatched, excess
// 1); a Y node's excess is (#X matched to it) - 1.  Arc costs are never stored:
// c(x,y) = -(n+1) w(x,y) is formed in registers from the int32 weight row.
//
// Refine schedule: bulk-synchronous alternation of an X phase (every active X
// relabels if needed and pushes one unit to its cheapest arc; warp-per-row scan +
// warp min-reduction) and a Y phase (every Y holding excess pushes units back to
// its cheapest incoming X, relabelling when none is admissible).  Inside a phase
// the ops are lock-free (atomic excess updates, owner-only price writes); because
// an X phase only reads Y prices and a Y phase only reads prices of matched X
// (neither changes during that phase), every op sees exact prices, so each phase
// equals some sequential order of reference ops and epsilon-optimality is kept
// exactly -- the stale-price window of the reference's free-running threads
// (assign_par.py:6-8) cannot open.  Phases run inside one cooperative kernel with
// grid-wide barriers; the long single-digit tail drops to one CTA with CTA barriers.
#include <stdio.h>
#include <cooperative_groups.h>
#include <algorithm>
#include <climits>
#include <vector>
#include <string.h>
#include <stdlib.h>

#include "fm_common.cuh"

namespace cg = cooperative_groups;

namespace {

#ifndef FM_ATHREADS
#define FM_ATHREADS 512
#endif
constexpr int ATHREADS = FM_ATHREADS;    // threads per CTA of the refine kernels
constexpr int AWARPS = ATHREADS / 32;
constexpr long long I64_MAX = 0x7fffffffffffffffLL;
constexpr int LINF = 0x3fffffff;         // "unlabelled" in the price update

// cnt[] slots
constexpr int C_X0 = 0, C_Y0 = 2;        // X / Y list counts (double-buffered)
constexpr int C_INFEASIBLE = 4;          // 1 no residual arc, 2 inconsistent, 3 budget, 4/5/6 validation
constexpr int C_EXIT = 5;                // rounds kernel exit: 0 done, 1 price update due, 2 round cap
constexpr int C_ROUND = 6;               // next round index (persists across launches)
constexpr int C_RELABELS = 7;            // relabels since the last price update
constexpr int C_PU_CHG = 8;              // price update: changed flags [8], [9]
constexpr int C_PU_LAST = 10;            // price update: max label over active nodes
constexpr int C_GATE = 11;               // enqueued-ahead launches: 0 rounds run, 1 price update runs, 2 refine over
constexpr int C_PUN = 12;                // price updates run in this refine (gated launches)
constexpr int C_COUNT = 13;
// ops[] slots
constexpr int O_PUSH = 0, O_RELABEL = 1, O_ROUNDS = 2, O_TAIL_ROUNDS = 3, O_FIXED = 4,
              O_PU = 5, O_PU_ITERS = 6, O_TAIL_OPS = 7, O_TAIL_NS = 8, O_MULTI_NS = 9,
              O_PH_Y = 10, O_PH_SYNC1 = 11, O_PH_X = 12, O_PH_SYNC2 = 13,  // multi-round phase ns (CTA 0)
              O_PU_YS = 14, O_PU_ITNS = 15,  // price update: frontier Y visits, ns in BF iterations (CTA 0)
              O_PU_LASTSUM = 16, O_PU_YFIN = 17, O_PU_YLAB = 18,  // price update: sum of last, Y with l <= last, Y labelled
              O_PU_SCANNS = 19,                                    // price update: ns in Y scans (summed over groups)
              O_HIST = 20,   // [20..24]: grid-wide rounds by max(|Y list|, |X list|): <= 8, 32, 148, 592, more
              O_HIST_NS = 25,   // [25..29]: CTA 0's ns in those rounds
              O_COUNT = 40;   // [30..37]: diagnostics of the rounds with long lists (trace)

// validate=True failures (assign_par.py:101-106,200-214; assign_scaling.py:274-275,333-336)
constexpr int V_RELABEL = 4;             // a relabel failed to lower a price
constexpr int V_OWNER = 5;               // a price word written by two ops in one phase
constexpr int V_RAISE = 6;               // the price update would raise a price

// release/acquire fence without the sequentially-consistent one's cost (__threadfence is
// fence.sc.gpu); used where only release ordering of earlier writes is needed
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

struct AssignDev {
    const int32_t *w;      // n x n weights (row x), FM_ABSENT_WEIGHT = no arc
    int64_t *px, *py;      // prices of X and Y
    int32_t *match;        // match[x] = y carrying x's unit, -1 if x holds its excess
    int32_t *ey;           // excess of y
    uint32_t *fixed;       // arc-fix bitmask, row-major n x nw words
    uint32_t *fixed_t;     // its transpose (row y, bit x): the price update scans columns
    uint8_t *frozen;       // frozen[x]: x's matched arc is fixed (its flow never changes)
    int32_t *frozen_in;    // frozen_in[y]: number of frozen matches into y
    int32_t *lx, *ly;      // price-update labels
    int32_t *ybcnt, *ybuf; // per-Y buckets of incoming X (YCAP slots each) for long Y lists
    int32_t *xlist[2], *ylist[2];
    int32_t *cnt;
    unsigned long long *ops;
    int32_t n, nw;
    int64_t scale;         // n + 1
    int64_t eps;
    int64_t max_bucket;    // scaled_cost_bound / eps + 2 (assign_scaling.py:232)
    int32_t pu_cap0;       // first label cap of the price update (0 = 8)
    int use_fix;
    int ybatch_min;         // gathered Y op: rank-batch the push-back from this many units (option ybatch_min)
    int validate;          // validate=True: device-side invariant checks (codes V_*)
    int32_t *pw;           // validate: last phase tag that wrote each price word (X then Y)
    int32_t vbase;         // validate: tag base of this launch (phase tag = vbase + 2 r + 1|2)
    int32_t cta_x, cta_y;  // a phase list up to cta_* x the grid runs one CTA-wide op per node
    int32_t *mw;           // price update: w(x, match[x]) (0 when x holds its unit)
    int64_t *pmx;          // price update: p(match[x]) (prices are constant during an update)
};

// validate=True: a price write must lower the price and be the only write of its word
// in this phase (owner-only writes, assign_par.py:101-106,200-214)
__device__ __forceinline__ void check_price_write(const AssignDev &a, int node, long long oldp, long long newp,
                                                  int tag) {
    if (!a.validate) return;
    if (newp >= oldp) atomicExch(a.cnt + C_INFEASIBLE, V_RELABEL);
    if (tag && atomicExch(a.pw + node, tag) == tag) atomicExch(a.cnt + C_INFEASIBLE, V_OWNER);
}


// (value, index) min with the lower index winning ties (first arc in the
// reference's out-arc order wins, assign_par.py:84-90)
__device__ __forceinline__ void argmin_merge(long long &v, int &i, long long ov, int oi) {
    if (ov < v || (ov == v && oi < i)) { v = ov; i = oi; }
}
__device__ __forceinline__ void warp_argmin(long long &v, int &i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i, o);
        argmin_merge(v, i, ov, oi);
    }
}
// CTA-wide argmin; result in every thread
__device__ __forceinline__ void cta_argmin(long long &v, int &i) {
    __shared__ long long s_v[AWARPS];
    __shared__ int s_i[AWARPS];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    warp_argmin(v, i);
    __syncthreads();
    if (lane == 0) { s_v[wid] = v; s_i[wid] = i; }
    __syncthreads();
    v = s_v[0]; i = s_i[0];
#pragma unroll
    for (int k = 1; k < AWARPS; k++) argmin_merge(v, i, s_v[k], s_i[k]);
}

// Partial scan of row x by thread t of a group of T threads: min over present,
// non-fixed arcs of the part-reduced cost c(x,y) - p(y) (assign_scaling.py:170-182,
// assign_par.py:82-90).  int4 weight loads and longlong2 price loads, four chunks
// in flight per thread.
#ifndef FM_RP_CHUNKS
#define FM_RP_CHUNKS 2
#endif
constexpr int RP_CHUNKS = FM_RP_CHUNKS;

// a weight row chunk: read once per op, kept out of L1 (the Y prices live there)
__device__ __forceinline__ int4 ld_row_na(const int4 *p) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// The Y prices (n x 8 B) are constant during an X phase and read by every X op of
// the phase: L1-cached loads (a grid barrier's acquire drops stale lines), so an SM's
// later X ops of the phase find them in L1 instead of L2.
__device__ __forceinline__ void row_partial(const AssignDev &a, int x, int t, int T,
                                            long long &bv, int &bi) {
    const int n = a.n;
    const int32_t *row = a.w + (size_t)x * n;
    const uint32_t *frow = a.fixed + (size_t)x * a.nw;
    if ((n & 3) == 0) {
        const int n4 = n >> 2;
        const int4 *row4 = reinterpret_cast<const int4 *>(row);
        const longlong2 *py2 = reinterpret_cast<const longlong2 *>(a.py);
        // RP_CHUNKS int4 chunks in flight per thread (2: the cooperative kernel's
        // 128-register cap spilled the 4-chunk version to local memory)
        for (int j0 = t; j0 < n4; j0 += RP_CHUNKS * T) {
            int4 w[RP_CHUNKS];
            longlong2 pa[RP_CHUNKS], pb[RP_CHUNKS];
            uint32_t fw[RP_CHUNKS];
#pragma unroll
            for (int u = 0; u < RP_CHUNKS; u++) {
                const int j = j0 + u * T;
                if (j < n4) {
                    w[u] = ld_row_na(row4 + j);
                    pa[u] = __ldca(py2 + 2 * j);
                    pb[u] = __ldca(py2 + 2 * j + 1);
                    fw[u] = a.use_fix ? (__ldg(frow + (j >> 3)) >> ((4 * j) & 31)) : 0u;
                }
            }
#pragma unroll
            for (int u = 0; u < RP_CHUNKS; u++) {
                const int j = j0 + u * T;
                if (j >= n4) continue;
                const int wv[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
                const long long pv[4] = {pa[u].x, pa[u].y, pb[u].x, pb[u].y};
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    if (wv[k] == FM_ABSENT_WEIGHT || ((fw[u] >> k) & 1u)) continue;
                    const long long v = -(long long)wv[k] * a.scale - pv[k];
                    if (v < bv) { bv = v; bi = 4 * j + k; }
                }
            }
        }
    } else {
        for (int y = t; y < n; y += T) {
            const int wv = __ldg(row + y);
            if (wv == FM_ABSENT_WEIGHT) continue;
            if (a.use_fix && ((__ldg(frow + (y >> 5)) >> (y & 31)) & 1u)) continue;
            const long long v = -(long long)wv * a.scale - __ldcg((const long long *)a.py + y);
            if (v < bv) { bv = v; bi = y; }
        }
    }
}

// Partial scan for Y op: over x matched to y (non-frozen) of the reverse arc's
// part-reduced cost +(n+1) w(x,y) - p(x).
__device__ __forceinline__ void ycand_partial(const AssignDev &a, int y, int t, int T,
                                              long long &bv, int &bi) {
    const int n = a.n;
    if ((n & 3) == 0) {
        const int n4 = n >> 2;
        const int4 *m4 = reinterpret_cast<const int4 *>(a.match);
        for (int j0 = t; j0 < n4; j0 += 4 * T) {
            int4 mm[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int j = j0 + u * T;
                mm[u] = j < n4 ? __ldcg(m4 + j) : make_int4(-1, -1, -1, -1);
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int j = j0 + u * T;
                const int mv[4] = {mm[u].x, mm[u].y, mm[u].z, mm[u].w};
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    if (mv[k] != y) continue;
                    const int x = 4 * j + k;
                    if (__ldcg(a.frozen + x)) continue;
                    const long long v = (long long)__ldg(a.w + (size_t)x * n + y) * a.scale -
                                        __ldcg((const long long *)a.px + x);
                    if (v < bv) { bv = v; bi = x; }
                }
            }
        }
    } else {
        for (int x = t; x < n; x += T) {
            if (__ldcg(a.match + x) != y || __ldcg(a.frozen + x)) continue;
            const long long v = (long long)__ldg(a.w + (size_t)x * n + y) * a.scale -
                                __ldcg((const long long *)a.px + x);
            if (v < bv) { bv = v; bi = x; }
        }
    }
}

// Where an op appends the nodes it activates.  Grid-wide rounds: a global list and its
// global counter.  The single-CTA tail also keeps the counter (and the first TL_CAP
// entries) in shared memory, plus shared copies of the relabel count and the
// infeasibility word: its rounds then need no L2 round trip for list bookkeeping
// (the global list is still written, fire-and-forget, so a later launch resumes
// from it).
constexpr int TL_CAP = 32;   // (static shared memory is nearly full: s_sorted takes 32 KB)
struct Lists {
    int32_t *glist;       // global list
    int32_t *gcnt;        // its global counter (grid-wide rounds)
    int *scnt = nullptr;  // tail: shared counter (authoritative), NULL in grid-wide rounds
    int32_t *slist = nullptr;
    int *srel = nullptr, *sinf = nullptr;
};
__device__ __forceinline__ int list_reserve(const Lists &L, int k) {
    return L.scnt ? atomicAdd(L.scnt, k) : atomicAdd(L.gcnt, k);
}
__device__ __forceinline__ void list_put(const Lists &L, int i, int v) {
    if (L.scnt && i < TL_CAP) L.slist[i] = v;
    L.glist[i] = v;
}
__device__ __forceinline__ void add_relabels(const AssignDev &a, const Lists &L, int k) {
    atomicAdd(a.cnt + C_RELABELS, k);
    if (L.srel) atomicAdd(L.srel, k);
}
__device__ __forceinline__ void set_infeasible(const AssignDev &a, const Lists &L, int why) {
    atomicExch(a.cnt + C_INFEASIBLE, why);
    if (L.sinf) atomicExch(L.sinf, why);
}

// X op by one group (warp when CTA_WIDE is false, else the whole CTA): relabel if
// the cheapest arc is not admissible, then push the unit on it.
template <bool CTA_WIDE>
__device__ void x_op(const AssignDev &a, int x, const Lists &L,
                     unsigned long long &pushes, unsigned long long &relabels, int tag = 0) {
    long long best = I64_MAX;
    int y = INT32_MAX;
    const int t = CTA_WIDE ? threadIdx.x : (threadIdx.x & 31);
    const long long px = t == 0 ? __ldcg((const long long *)a.px + x) : 0;  // overlaps the scan
    row_partial(a, x, t, CTA_WIDE ? ATHREADS : 32, best, y);
    if (CTA_WIDE) cta_argmin(best, y); else warp_argmin(best, y);
    if (t == 0) {
        if (y == INT32_MAX) {
            set_infeasible(a, L, 1);              // active node with no residual arc
        } else {
            if (!(best < -px)) {                 // not admissible: p(x) <- -(best + eps)
                check_price_write(a, x, px, -(best + a.eps), tag);
                a.px[x] = -(best + a.eps);
                relabels++;
                add_relabels(a, L, 1);
            }
            a.match[x] = y;                      // unit push x -> y
            pushes++;
            const int old = atomicAdd(a.ey + y, 1);
            if (old == 0) list_put(L, list_reserve(L, 1), y);
        }
    }
    if (CTA_WIDE) __syncthreads(); else __syncwarp();
}

// Y op: while y holds excess, push a unit back to its cheapest incoming X,
// relabelling y first when that reverse arc is not admissible.  One scan of
// match[] gathers the incoming X (with their reverse part-reduced costs) into
// shared memory; y's own relabels do not change their order, so the excess
// units go back to the gathered candidates in increasing cost order without
// rescanning.  More than YCAP incoming units falls back to one scan per unit.
constexpr int YCAP = 64;                // candidates gathered per warp-wide Y op in shared memory
constexpr int YCAP_CTA = 1024;          // per CTA-wide Y op (in the caller's 32 KB scratch: 2.5 x 8 KB)
constexpr int YBUCKET = 256;            // per-Y bucket slots for long Y lists (= YB_CAP)

template <bool CTA_WIDE>
__device__ void y_op(const AssignDev &a, int y, const Lists &L,
                     unsigned long long &pushes, unsigned long long &relabels, long long *sbuf, int tag = 0) {
    // CTA-wide: the candidates and their ranked costs live in the caller's whole
    // AWARPS x YB_CAP scratch (no other op runs in the CTA meanwhile): up to YCAP_CTA
    // candidates (a Y that collects a few hundred units in one phase would otherwise
    // fall back to one match[] scan per unit)
    __shared__ long long s_cv[CTA_WIDE ? 1 : AWARPS][CTA_WIDE ? 1 : YCAP];
    __shared__ int s_cx[CTA_WIDE ? 1 : AWARPS][CTA_WIDE ? 1 : YCAP];
    __shared__ int s_cn[CTA_WIDE ? 1 : AWARPS];
    constexpr int CAP = CTA_WIDE ? YCAP_CTA : YCAP;
    const int t = CTA_WIDE ? threadIdx.x : (threadIdx.x & 31);
    const int T = CTA_WIDE ? ATHREADS : 32;
    const int slot = CTA_WIDE ? 0 : (threadIdx.x >> 5);
    long long *cv = CTA_WIDE ? sbuf : s_cv[slot];
    int *cx = CTA_WIDE ? reinterpret_cast<int *>(sbuf + 2 * YCAP_CTA) : s_cx[slot];
    long long *srt = CTA_WIDE ? sbuf + YCAP_CTA : sbuf;
    // y's excess and price load while the gather below scans match[] (a listed y holds
    // excess; the check waits until after the scan)
    int ey = __ldcg(a.ey + y);
    long long py = __ldcg((const long long *)a.py + y);
    const long long py0 = py;
    // ---- gather
    if (t == 0) s_cn[slot] = 0;
    if (CTA_WIDE) __syncthreads(); else __syncwarp();
    const int n = a.n;
    const auto take = [&](int x) {
        const long long v = (long long)__ldg(a.w + (size_t)x * n + y) * a.scale - __ldcg((const long long *)a.px + x);
        const int k = atomicAdd(&s_cn[slot], 1);
        if (k < CAP) { cx[k] = x; cv[k] = v; }
    };
    if ((n & 3) == 0) {
        // match words and the frozen flags of the same 4 x load together (no dependent
        // frozen load per candidate)
        const int n4 = n >> 2;
        const int4 *m4 = reinterpret_cast<const int4 *>(a.match);
        const uint32_t *fz4 = reinterpret_cast<const uint32_t *>(a.frozen);
        for (int j0 = t; j0 < n4; j0 += 4 * T) {
            int4 mm[4];
            uint32_t fz[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int j = j0 + u * T;
                mm[u] = j < n4 ? __ldcg(m4 + j) : make_int4(-1, -1, -1, -1);
                fz[u] = j < n4 ? __ldcg(fz4 + j) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int j = j0 + u * T;
                if (mm[u].x == y && !(fz[u] & 0xffu)) take(4 * j + 0);
                if (mm[u].y == y && !(fz[u] & 0xff00u)) take(4 * j + 1);
                if (mm[u].z == y && !(fz[u] & 0xff0000u)) take(4 * j + 2);
                if (mm[u].w == y && !(fz[u] & 0xff000000u)) take(4 * j + 3);
            }
        }
    } else {
        for (int x = t; x < n; x += T)
            if (__ldcg(a.match + x) == y && !__ldcg(a.frozen + x)) take(x);
    }
    if (CTA_WIDE) __syncthreads(); else __syncwarp();
    if (ey <= 0) return;   // uniform: every thread read the same (phase-constant) word
    const int cnt = s_cn[slot];
    if (cnt > CAP) {
        if (t == 0) { atomicAdd(a.ops + 36, 1ull); atomicAdd(a.ops + 37, (unsigned long long)ey); atomicMax(a.ops + 33, (unsigned long long)cnt); }
        // ---- overflow: one scan per unit (the original scheme)
        while (ey > 0) {
            long long bv = I64_MAX;
            int bi = INT32_MAX;
            ycand_partial(a, y, t, T, bv, bi);
            if (CTA_WIDE) cta_argmin(bv, bi); else warp_argmin(bv, bi);
            if (bi == INT32_MAX) {
                if (t == 0) set_infeasible(a, L, 2);
                break;
            }
            if (t == 0) {
                if (!(bv < -py)) {
                    if (a.validate && -(bv + a.eps) >= py) atomicExch(a.cnt + C_INFEASIBLE, V_RELABEL);
                    py = -(bv + a.eps); relabels++; add_relabels(a, L, 1);
                }
                a.match[bi] = -1;
                list_put(L, list_reserve(L, 1), bi);
                pushes++;
            }
            ey--;
            if (CTA_WIDE) __syncthreads(); else __syncwarp();
        }
    } else if (ey >= a.ybatch_min && ey <= cnt) {   // ey == cnt: y keeps only frozen flow (all units go back)
        // ---- batch: the ey cheapest candidates in (v, x) order are exactly the units
        // the one-unit loop below would push back (y's relabels never reorder them).
        // Rank every candidate against the others, lay the chosen costs out in rank
        // order (sbuf: >= CAP entries of the caller's shared scratch), append the
        // batch with one list reservation and replay the relabel sequence.
        __shared__ int s_base[CTA_WIDE ? 1 : AWARPS];
        if (t == 0) s_base[slot] = list_reserve(L, ey);
        if (CTA_WIDE) __syncthreads(); else __syncwarp();
        const int base = s_base[slot];
        for (int k = t; k < cnt; k += T) {
            const long long vk = cv[k];
            const int xk = cx[k];
            int rank = 0;
#pragma unroll 8
            for (int j = 0; j < cnt; j++) {
                const long long vj = cv[j];
                rank += (vj < vk || (vj == vk && cx[j] < xk)) ? 1 : 0;
            }
            if (rank < ey) {
                srt[rank] = vk;
                a.match[xk] = -1;
                list_put(L, base + rank, xk);
            }
        }
        if (CTA_WIDE) __syncthreads(); else __syncwarp();
        if (t == 0) {
            unsigned long long rl = 0;
            for (int k = 0; k < ey; k++) {
                const long long vk = srt[k];
                if (!(vk < -py)) {
                    if (a.validate && -(vk + a.eps) >= py) atomicExch(a.cnt + C_INFEASIBLE, V_RELABEL);
                    py = -(vk + a.eps); rl++;
                }
            }
            relabels += rl;
            pushes += ey;
            if (rl) add_relabels(a, L, (int)rl);
        }
        ey = 0;
    } else {
        // ---- push back to the cheapest gathered candidates, one per excess unit
        while (ey > 0) {
            long long bv = I64_MAX;
            int bi = INT32_MAX, bk = -1;
            for (int k = t; k < cnt; k += T)
                if (cv[k] < bv || (cv[k] == bv && cx[k] < bi)) { bv = cv[k]; bi = cx[k]; bk = k; }
            long long v2 = bv;
            int i2 = bi;
            if (CTA_WIDE) cta_argmin(v2, i2); else warp_argmin(v2, i2);
            if (i2 == INT32_MAX) {
                if (t == 0) set_infeasible(a, L, 2);
                break;
            }
            if (bi == i2 && bk >= 0) cv[bk] = I64_MAX;   // the owner lane retires the slot
            if (t == 0) {
                if (!(v2 < -py)) {
                    if (a.validate && -(v2 + a.eps) >= py) atomicExch(a.cnt + C_INFEASIBLE, V_RELABEL);
                    py = -(v2 + a.eps); relabels++; add_relabels(a, L, 1);
                }
                a.match[i2] = -1;
                list_put(L, list_reserve(L, 1), i2);
                pushes++;
            }
            ey--;
            if (CTA_WIDE) __syncthreads(); else __syncwarp();
        }
    }
    if (t == 0) {
        if (py != py0 && a.validate && tag && atomicExch(a.pw + a.n + y, tag) == tag)
            atomicExch(a.cnt + C_INFEASIBLE, V_OWNER);
        a.py[y] = py;
        a.ey[y] = ey;
    }
    if (CTA_WIDE) __syncthreads(); else __syncwarp();
}

// Batch push-back of a Y holding ey excess units over its cnt incoming candidates
// (v, x), v = reverse part-reduced cost: the units go back to the ey cheapest
// candidates in increasing (v, x) order -- exactly the sequence of one-unit Y ops,
// since y's own relabels never reorder the candidates.  Each lane ranks its
// candidates against all others, the ranked costs are laid out in shared memory,
// lane 0 replays the relabel sequence (p(y) <- -(v + eps) whenever the next arc is
// not admissible) and the whole batch is appended with one list reservation.
constexpr int YB_PER_LANE = 8;               // up to 256 candidates per warp
constexpr int YB_CAP = 32 * YB_PER_LANE;
static_assert(AWARPS * YB_CAP * 2 >= 5 * YCAP_CTA, "CTA-wide Y op scratch (candidates, ranked costs, indices) exceeds s_sorted");

__device__ void y_batch_warp(const AssignDev &a, int y, int ey, long long py, int cnt,
                             const long long (&v)[YB_PER_LANE], const int (&xs)[YB_PER_LANE],
                             long long *s_sorted, const Lists &L,
                             unsigned long long &pushes, unsigned long long &relabels, int tag) {
    const int lane = threadIdx.x & 31;
    int rank[YB_PER_LANE];
#pragma unroll
    for (int k = 0; k < YB_PER_LANE; k++) rank[k] = 0;
    for (int src = 0; src < 32; src++) {
#pragma unroll
        for (int j = 0; j < YB_PER_LANE; j++) {
            const long long ov = __shfl_sync(0xffffffffu, v[j], src);
            const int ox = __shfl_sync(0xffffffffu, xs[j], src);
            if (ox == INT32_MAX) continue;
#pragma unroll
            for (int k = 0; k < YB_PER_LANE; k++)
                if (ov < v[k] || (ov == v[k] && ox < xs[k])) rank[k]++;
        }
    }
    int base = 0;
    if (lane == 0) base = list_reserve(L, ey);
    base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
    for (int k = 0; k < YB_PER_LANE; k++) {
        if (xs[k] != INT32_MAX && rank[k] < ey) {
            s_sorted[rank[k]] = v[k];
            a.match[xs[k]] = -1;
            list_put(L, base + rank[k], xs[k]);
        }
    }
    __syncwarp();
    if (lane == 0) {
        unsigned long long rl = 0;
        for (int k = 0; k < ey; k++) {
            const long long vk = s_sorted[k];
            if (!(vk < -py)) { py = -(vk + a.eps); rl++; }
        }
        relabels += rl;
        pushes += ey;
        if (rl) add_relabels(a, L, (int)rl);
        if (rl && a.validate && tag && atomicExch(a.pw + a.n + y, tag) == tag)
            atomicExch(a.cnt + C_INFEASIBLE, V_OWNER);
        a.py[y] = py;
        a.ey[y] = 0;
    }
    __syncwarp();
    (void)cnt;
}

// Y op over a pre-bucketed candidate list (long Y lists): the incoming X of y were
// collected once per phase into ybuf[y*YCAP ..]; one warp per y.
__device__ void y_op_bucketed(const AssignDev &a, int y, const Lists &L,
                              unsigned long long &pushes, unsigned long long &relabels,
                              long long *s_sorted, int tag) {
    const int lane = threadIdx.x & 31;
    const int cnt = __ldcg(a.ybcnt + y);
    const int ey = __ldcg(a.ey + y);
    if (cnt > YBUCKET || ey > cnt) {        // bucket overflow (or inconsistent): scan match[] instead
        if (lane == 0) { atomicAdd(a.ops + 32, 1ull); atomicMax(a.ops + 33, (unsigned long long)cnt); }
        y_op<false>(a, y, L, pushes, relabels, s_sorted, tag);
        if (lane == 0) a.ybcnt[y] = 0;
        __syncwarp();
        return;
    }
    const long long py = __ldcg((const long long *)a.py + y);
    const int n = a.n;
    long long v[YB_PER_LANE];
    int xs[YB_PER_LANE];
#pragma unroll
    for (int k = 0; k < YB_PER_LANE; k++) {
        const int i = lane + 32 * k;
        v[k] = I64_MAX;
        xs[k] = INT32_MAX;
        if (i < cnt) {
            const int x = __ldcg(a.ybuf + (size_t)y * YBUCKET + i);
            xs[k] = x;
            v[k] = (long long)__ldg(a.w + (size_t)x * n + y) * a.scale - __ldcg((const long long *)a.px + x);
        }
    }
    if (ey > 0) y_batch_warp(a, y, ey, py, cnt, v, xs, s_sorted, L, pushes, relabels, tag);
    if (lane == 0) a.ybcnt[y] = 0;
    __syncwarp();
}

// begin_refine (assign_scaling.py:145-182) fused with the first X phase: drop
// unfrozen flow, set p(x) = -(min part-reduced cost + eps) and push x's unit on
// that arc (admissible at reduced cost -eps by construction).
// push = 0: the preamble alone (the stepwise begin_refine); unfrozen X are left
// unmatched and active for the first round.
__global__ void __launch_bounds__(ATHREADS) begin_refine_kernel(AssignDev a, int push) {
    const int warp = (blockIdx.x * ATHREADS + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * ATHREADS) >> 5;
    const int lane = threadIdx.x & 31;
    unsigned long long pushes = 0;
    for (int x = warp; x < a.n; x += nwarps) {
        long long best = I64_MAX;
        int y = INT32_MAX;
        row_partial(a, x, lane, 32, best, y);
        warp_argmin(best, y);
        if (lane == 0) {
            if (y != INT32_MAX) a.px[x] = -(best + a.eps);
            if (!a.frozen[x] && !push) {
                a.match[x] = -1;
            } else if (!a.frozen[x]) {
                if (y == INT32_MAX) {
                    a.match[x] = -1;
                    atomicExch(a.cnt + C_INFEASIBLE, 1);
                } else {
                    a.match[x] = y;
                    pushes++;
                    const int old = atomicAdd(a.ey + y, 1);
                    if (old == 0) a.ylist[0][atomicAdd(a.cnt + C_Y0, 1)] = y;
                }
            }
        }
    }
    if (lane == 0 && pushes) atomicAdd(a.ops + O_PUSH, pushes);
}

// excess of y after flow removal: supplies (-1) + frozen flows (assign_scaling.py:158-168)
__global__ void reset_excess_kernel(AssignDev a) {
    for (int y = blockIdx.x * blockDim.x + threadIdx.x; y < a.n; y += gridDim.x * blockDim.x)
        a.ey[y] = -1 + a.frozen_in[y];
}

// Control words read right after a grid barrier: one thread per CTA loads them and
// the CTA shares them (thousands of warps loading one L2 line at the same moment
// serialise on its slice; ncu put half of the price update's stall samples there).
__device__ __forceinline__ void cta_bcast4(const int32_t *p0, const int32_t *p1, const int32_t *p2,
                                           const int32_t *p3, int &v0, int &v1, int &v2, int &v3) {
    __shared__ int s_b[4];
    __syncthreads();   // the previous broadcast has been read by every thread
    if (threadIdx.x == 0) {
        s_b[0] = __ldcg(p0);
        s_b[1] = p1 ? __ldcg(p1) : 0;
        s_b[2] = p2 ? __ldcg(p2) : 0;
        s_b[3] = p3 ? __ldcg(p3) : 0;
    }
    __syncthreads();
    v0 = s_b[0]; v1 = s_b[1]; v2 = s_b[2]; v3 = s_b[3];
}
__device__ __forceinline__ void cta_bcast3(const int32_t *p0, const int32_t *p1, const int32_t *p2,
                                           int &v0, int &v1, int &v2) {
    int u;
    cta_bcast4(p0, p1, p2, nullptr, v0, v1, v2, u);
}

// The refine's push/relabel rounds (refine_par's coordinator loop, assign_par.py:162-236)
// as one cooperative kernel.  Round r: Y phase over ylist[r&1] -> xlist[r&1];
// grid barrier; X phase over xlist[r&1] -> ylist[(r+1)&1]; grid barrier.
// Exits when no Y holds excess (refine done) or when a price update is due
// (relabels since the last one >= pu_threshold); the round index persists in cnt.
// Once the Y list is short the other CTAs leave and CTA 0 finishes alone with
// CTA-wide ops and CTA barriers (the long single-digit tail).
__global__ void __launch_bounds__(ATHREADS) refine_rounds_kernel(AssignDev a, int tail_threshold,
                                                                 long long round_budget,
                                                                 int pu_threshold, int max_rounds,
                                                                 int pu_every_k, int gated) {
    cg::grid_group grid = cg::this_grid();
    // gated (launches enqueued ahead of the host's decision): run only when the gate says
    // so; every CTA reads it before any CTA can rewrite it (the barrier), so all agree
    if (gated) {
        __shared__ int s_go;
        if (threadIdx.x == 0) s_go = __ldcg(a.cnt + C_GATE) == 0 && __ldcg(a.cnt + C_INFEASIBLE) == 0;
        __syncthreads();
        const int go = s_go;
        grid.sync();
        if (!go) return;
    }
    const int lane = threadIdx.x & 31;
    const int gwarp = (blockIdx.x * ATHREADS + threadIdx.x) >> 5;
    const int gwarps = (gridDim.x * ATHREADS) >> 5;
    const int cwarp = threadIdx.x >> 5;
    unsigned long long pushes = 0, relabels = 0, rounds = 0, tail_rounds = 0, tail_ops = 0;
    unsigned long long tail_ns = 0, multi_ns = 0, t_round = globaltimer();
    __shared__ long long s_sorted[AWARPS][YB_CAP];
    bool tail = false;
    // single-CTA tail: list counters / heads, relabel count and infeasibility in shared memory
    __shared__ int s_xn[2], s_yn[2], s_rel, s_inf;
    __shared__ int32_t s_xl[2][TL_CAP], s_yl[2][TL_CAP];
    int r = __ldcg(a.cnt + C_ROUND);
    for (;; r++) {
        {
            const unsigned long long now = globaltimer();
            if (tail) tail_ns += now - t_round; else multi_ns += now - t_round;
            t_round = now;
        }
        const int b = r & 1, nb = b ^ 1;
        int ny, infeasible, relabels_since, y_first = 0;
        if (tail) {
            __syncthreads();   // the previous round's shared counters are final
            ny = s_yn[b]; infeasible = s_inf; relabels_since = s_rel;
        } else {
            // with the control words, this CTA's first Y list entry (read speculatively:
            // used only when the round runs CTA-wide ops and the list reaches it)
            cta_bcast4(a.cnt + C_Y0 + b, a.cnt + C_INFEASIBLE, a.cnt + C_RELABELS,
                       (int)blockIdx.x < a.n ? a.ylist[b] + blockIdx.x : nullptr, ny, infeasible, relabels_since, y_first);
        }
        if (ny == 0 || infeasible) {
            if (blockIdx.x == 0 && threadIdx.x == 0) a.cnt[C_EXIT] = 0;
            break;
        }
        if (pu_threshold > 0 && relabels_since >= pu_threshold) {
            if (blockIdx.x == 0 && threadIdx.x == 0) a.cnt[C_EXIT] = 1;
            break;
        }
        // heuristic_every_k (assign_par.py:228-234): a price update every k rounds
        if (pu_every_k > 0 && rounds > 0 && r % pu_every_k == 0) {
            if (blockIdx.x == 0 && threadIdx.x == 0) a.cnt[C_EXIT] = 1;
            break;
        }
        // coordinator round cap (cycle_budget rounds per coordinator round)
        if (max_rounds > 0 && (long long)rounds >= max_rounds) {
            if (blockIdx.x == 0 && threadIdx.x == 0) a.cnt[C_EXIT] = 2;
            break;
        }
        if (r >= round_budget) {  // prices diverge: no perfect matching (assign_par.py:221-226)
            if (blockIdx.x == 0 && threadIdx.x == 0) { atomicExch(a.cnt + C_INFEASIBLE, 3); a.cnt[C_EXIT] = 0; }
            break;
        }
        if (!tail && ny <= min(tail_threshold, TL_CAP)) {
            tail = true;
            if (blockIdx.x != 0) break;  // CTA 0 finishes alone
            for (int i = threadIdx.x; i < ny; i += ATHREADS) s_yl[b][i] = __ldcg(a.ylist[b] + i);
            if (threadIdx.x == 0) { s_yn[b] = ny; s_xn[b] = 0; s_rel = relabels_since; s_inf = 0; }
            __syncthreads();
        }
        rounds++;
        if (tail) tail_rounds++;
        const int tag_y = a.vbase + 2 * r + 1, tag_x = tag_y + 1;   // validate: phase tags
        // ---- Y phase
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.cnt[C_X0 + nb] = 0;   // X list of round r+1 (last read in round r-1)
            a.cnt[C_Y0 + nb] = 0;   // Y list of round r+1 (last read at round r-1)
            if (tail) { s_xn[nb] = 0; s_yn[nb] = 0; }
        }
        if (tail) {
            const unsigned long long p0 = pushes + relabels;
            const Lists TX{a.xlist[b], a.cnt + C_X0 + b, &s_xn[b], s_xl[b], &s_rel, &s_inf};
            const Lists TY{a.ylist[nb], a.cnt + C_Y0 + nb, &s_yn[nb], s_yl[nb], &s_rel, &s_inf};
            // entries past TL_CAP live only in the global list (written by this CTA
            // before the last barrier)
            const auto ent = [&](const int32_t *sl, const int32_t *gl, int i) { return i < TL_CAP ? sl[i] : __ldcg(gl + i); };
            if (ny <= 2) {
                for (int i = 0; i < ny; i++)
                    y_op<true>(a, ent(s_yl[b], a.ylist[b], i), TX, pushes, relabels, s_sorted[0], tag_y);
            } else {
                for (int i = cwarp; i < ny; i += AWARPS)
                    y_op<false>(a, ent(s_yl[b], a.ylist[b], i), TX, pushes, relabels, s_sorted[cwarp], tag_y);
            }
            __threadfence_block();
            __syncthreads();
            const int nx = s_xn[b];
            if (nx <= 2) {
                for (int i = 0; i < nx; i++)
                    x_op<true>(a, ent(s_xl[b], a.xlist[b], i), TY, pushes, relabels, tag_x);
            } else {
                for (int i = cwarp; i < nx; i += AWARPS)
                    x_op<false>(a, ent(s_xl[b], a.xlist[b], i), TY, pushes, relabels, tag_x);
            }
            __threadfence_block();
            __syncthreads();
            // the global counters follow the shared ones (a later launch resumes from them)
            if (threadIdx.x == 0) { a.cnt[C_X0 + b] = s_xn[b]; a.cnt[C_Y0 + nb] = s_yn[nb]; }
            tail_ops += pushes + relabels - p0;
        } else {
            const Lists LX{a.xlist[b], a.cnt + C_X0 + b}, LY{a.ylist[nb], a.cnt + C_Y0 + nb};
            // a list no longer than the grid gets one CTA per node (one L2 round trip
            // per row scan); longer lists get one warp per node
            const bool timer = blockIdx.x == 0 && threadIdx.x == 0;
            unsigned long long t0 = timer ? globaltimer() : 0, t1 = 0;
            const unsigned long long t_r0 = t0;
            int hbin = 0;
            if (ny <= a.cta_y * (int)gridDim.x) {
                for (int i = blockIdx.x; i < ny; i += gridDim.x)
                    y_op<true>(a, i == (int)blockIdx.x ? y_first : __ldcg(a.ylist[b] + i), LX, pushes, relabels,
                               s_sorted[0], tag_y);
            } else {
                // long list: bucket every incoming X by its Y in one pass over match[]
                const int gtid = blockIdx.x * ATHREADS + threadIdx.x, gthr = gridDim.x * ATHREADS;
                for (int x = gtid; x < a.n; x += gthr) {
                    const int y = __ldcg(a.match + x);
                    if (y < 0 || __ldcg(a.frozen + x) || __ldcg(a.ey + y) <= 0) continue;
                    const int k = atomicAdd(a.ybcnt + y, 1);
                    if (k < YBUCKET) a.ybuf[(size_t)y * YBUCKET + k] = x;
                }
                if (timer) atomicAdd(a.ops + 34, globaltimer() - t0);
                grid.sync();
                if (timer) atomicAdd(a.ops + 35, globaltimer() - t0);
                for (int i = gwarp; i < ny; i += gwarps)
                    y_op_bucketed(a, __ldcg(a.ylist[b] + i), LX, pushes, relabels,
                                  s_sorted[threadIdx.x >> 5], tag_y);
            }
            if (timer) { t1 = globaltimer(); atomicAdd(a.ops + O_PH_Y, t1 - t0); t0 = t1; }
            grid.sync();
            if (timer) { t1 = globaltimer(); atomicAdd(a.ops + O_PH_SYNC1, t1 - t0); t0 = t1; }
            const unsigned long long t_y1 = t0;
            int nx, x_first, u2;
            cta_bcast3(a.cnt + C_X0 + b, (int)blockIdx.x < a.n ? a.xlist[b] + blockIdx.x : nullptr, nullptr, nx,
                       x_first, u2);
            if (nx <= a.cta_x * (int)gridDim.x) {
                for (int i = blockIdx.x; i < nx; i += gridDim.x)
                    x_op<true>(a, i == (int)blockIdx.x ? x_first : __ldcg(a.xlist[b] + i), LY, pushes, relabels, tag_x);
            } else {
                for (int i = gwarp; i < nx; i += gwarps)
                    x_op<false>(a, __ldcg(a.xlist[b] + i), LY, pushes, relabels, tag_x);
            }
            if (timer) {
                t1 = globaltimer(); atomicAdd(a.ops + O_PH_X, t1 - t0); t0 = t1;
                const int m = max(ny, nx);
                hbin = m <= 8 ? 0 : m <= 32 ? 1 : m <= 148 ? 2 : m <= 592 ? 3 : 4;
                atomicAdd(a.ops + O_HIST + hbin, 1ull);
            }
            grid.sync();
            if (timer) {
                t1 = globaltimer(); atomicAdd(a.ops + O_PH_SYNC2, t1 - t0);
                atomicAdd(a.ops + O_HIST_NS + hbin, t1 - t_r0);
                if (hbin == 4) { atomicAdd(a.ops + 30, t_y1 - t_r0); atomicAdd(a.ops + 31, t1 - t_y1); }
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.cnt[C_ROUND] = r;
        if (gated) a.cnt[C_GATE] = a.cnt[C_EXIT] == 1 ? 1 : 2;   // same thread wrote C_EXIT
    }
    if (lane == 0) {
        if (pushes) atomicAdd(a.ops + O_PUSH, pushes);
        if (relabels) atomicAdd(a.ops + O_RELABEL, relabels);
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        atomicAdd(a.ops + O_ROUNDS, rounds);
        atomicAdd(a.ops + O_TAIL_ROUNDS, tail_rounds);
        atomicAdd(a.ops + O_TAIL_OPS, tail_ops);
        atomicAdd(a.ops + O_TAIL_NS, tail_ns);
        atomicAdd(a.ops + O_MULTI_NS, multi_ns);
    }
    (void)cwarp;
}

// floor(rc / eps) for eps >= 1 via a double quotient corrected by one step
// (|rc| < 2^52 here), avoiding a 64-bit integer division per arc
__device__ __forceinline__ long long floordiv_eps(long long rc, long long eps, double inv_eps) {
    if (eps == 1) return rc;
    long long q = (long long)floor((double)rc * inv_eps);
    const long long r = rc - q * eps;
    if (r < 0) q--; else if (r >= eps) q++;
    return q;
}

// price_update_heuristic (assign_scaling.py:208-276) at a quiescent point of the
// refine: label every node with its distance to the deficit set over residual
// arcs, arc length floor(c_p / eps) + 1 (>= 0), in eps units; then lower each
// price by eps * min(label, last + 1), last = the largest label of an active node.
// The reference scans Dial buckets; here the same labels come from a frontier
// Bellman-Ford: X step = one CTA per Y whose label dropped, relaxing every arc x->y
// along row y of the transposed weights (coalesced) with atomicMin on l(x); Y step
// = one thread per X whose label dropped, relaxing its matched reverse arc.
constexpr int PU_GROUPS = 4;   // price update: up to this many frontier Y per CTA in flight (default)
constexpr int PU_GROUPS_MAX = 8;
constexpr int PU_RING_EXTRA = 16384;   // ring slots beyond n (>= the price update's groups + 64)
__device__ __forceinline__ void group_sync(int grp, int nthreads) {   // named barrier of one thread group
    asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(nthreads) : "memory");
}

// Y labels in the price update are packed words 2 l(y) + q, q = 1 while y is queued:
// one atomicMin lowers the label and marks y queued, and its old value says whether the
// caller must queue y (label dropped, y was not queued); taking y clears q and reads
// the label in one atomicAnd.  (A separate queued flag cost two more dependent L2 round
// trips per label drop and per take.)
__device__ __forceinline__ bool ylabel_drop(const AssignDev &a, int y, int l) {
    const int old = atomicMin(a.ly + y, 2 * l + 1);
    return (old >> 1) > l && !(old & 1);
}
__device__ __forceinline__ int ylabel_take(const AssignDev &a, int y) { return atomicAnd(a.ly + y, ~1) >> 1; }
__device__ __forceinline__ int ylabel(int word) { return word >> 1; }

struct PuDev {
    const int32_t *wt;      // transposed weights: wt[y*n + x] = w(x, y)
    int32_t *fy[2], *fx[2]; // frontiers
    int32_t *in_fx, *in_fy; // frontier membership flags
    int32_t *cnt;           // [0..1] |fy|, [2..3] |fx|
    // queue-driven variant (ring_on, env FM_PU_RING): frontier Y in a ring of ring_cap
    // slots (-1 = empty); rctr[0] head, [32] tail, [64] pending (queued + in flight)
    int32_t *ring;
    unsigned int *rctr;
    int ring_cap, ring_on;
    int ring_groups;        // frontier Y scanned at once per CTA in the queue-driven variant (1, 2, 4, 8)
    int local_next;         // queue-driven variant: a group keeps its first re-queued Y (option pu_local)
};

// One frontier Y of the price update, scanned by a group of GT threads (thread gt):
// relax every arc x->y into l(x) and, where l(x) dropped, x's matched reverse arc into
// its Y; push(y2) queues a Y whose label dropped (its queued flag already set).
template <typename Push>
__device__ __forceinline__ void pu_scan_y(const AssignDev &a, const PuDev &f, int y, int lyv, long long pyv,
                                          long long cap, double inv_eps, int gt, int PU_GT, Push push) {
    const int n = a.n;
    const int32_t *col = f.wt + (size_t)y * n;
    // vector path: 8 consecutive x per thread, every operand loaded up front
    // (int4 weights / labels / matches, longlong2 prices) so a thread's scan is
    // one L2 round trip instead of a chain of dependent ones
    const int nv8 = (n & 7) ? 0 : n;
    for (int x0 = gt * 8; x0 < nv8; x0 += PU_GT * 8) {
        const int4 w0 = __ldg((const int4 *)(col + x0)), w1 = __ldg((const int4 *)(col + x0 + 4));
        const int4 l0 = __ldcg((const int4 *)(a.lx + x0)), l1 = __ldcg((const int4 *)(a.lx + x0 + 4));
        // match, prices, frozen flags and the per-x arrays filled at the update's start
        // (w(x, match[x]), p(match[x])) do not change during the update: L1-cached loads
        // (every Y scan reads them all), and no dependent loads in stage 3
        const int4 m0 = __ldca((const int4 *)(a.match + x0)), m1 = __ldca((const int4 *)(a.match + x0 + 4));
        longlong2 pv[4];
#pragma unroll
        for (int k = 0; k < 4; k++) pv[k] = __ldca((const longlong2 *)(a.px + x0) + k);
        const int4 mw0 = __ldca((const int4 *)(a.mw + x0)), mw1 = __ldca((const int4 *)(a.mw + x0 + 4));
        longlong2 pm[4];
#pragma unroll
        for (int k = 0; k < 4; k++) pm[k] = __ldca((const longlong2 *)(a.pmx + x0) + k);
        const uint2 fz8 = __ldca((const uint2 *)(a.frozen + x0));
        uint32_t fb = 0;
        if (a.use_fix) fb = (__ldg(a.fixed_t + (size_t)y * a.nw + (x0 >> 5)) >> (x0 & 31)) & 0xffu;
        const int wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        const int lxv[8] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w};
        const int mxv[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
        const long long pxv[8] = {pv[0].x, pv[0].y, pv[1].x, pv[1].y, pv[2].x, pv[2].y, pv[3].x, pv[3].y};
        // stage 1: candidate labels; stage 2: all atomicMin on l(x) in flight
        // together; stage 3: the matched reverse arcs of the x that dropped
        int cand[8], old[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            cand[k] = LINF;
            if (wv[k] == FM_ABSENT_WEIGHT || lyv >= lxv[k] || mxv[k] == y || ((fb >> k) & 1u)) continue;
            const long long rc = -(long long)wv[k] * a.scale + pxv[k] - pyv;
            long long len = floordiv_eps(rc, a.eps, inv_eps) + 1;
            if (len < 0) len = 0;
            const long long c1 = (long long)lyv + len;
            if (c1 <= cap && c1 < lxv[k]) cand[k] = (int)c1;
        }
        // label drops are fire-and-forget (RED); the matched reverse arc is relaxed from
        // every candidate below the label read above -- a path length either way, so a
        // redundant relaxation is harmless and the fixpoint is unchanged
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (cand[k] < LINF) atomicMin(a.lx + x0 + k, cand[k]);
            old[k] = lxv[k];
        }
        const int w2[8] = {mw0.x, mw0.y, mw0.z, mw0.w, mw1.x, mw1.y, mw1.z, mw1.w};
        const long long py2[8] = {pm[0].x, pm[0].y, pm[1].x, pm[1].y, pm[2].x, pm[2].y, pm[3].x, pm[3].y};
        uint8_t fz[8];
#pragma unroll
        for (int k = 0; k < 8; k++) fz[k] = (uint8_t)(((k < 4 ? fz8.x : fz8.y) >> (8 * (k & 3))) & 0xffu);
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (!(cand[k] < old[k]) || mxv[k] < 0 || fz[k]) continue;
            const long long rc2 = (long long)w2[k] * a.scale - pxv[k] + py2[k];
            long long len2 = floordiv_eps(rc2, a.eps, inv_eps) + 1;
            if (len2 < 0) len2 = 0;
            const long long cand2 = cand[k] + len2;
            if (cand2 > cap) continue;
            const int mx = mxv[k];
            if (ylabel_drop(a, mx, (int)cand2)) push(mx);
        }
    }
    for (int x = nv8 + gt; x < n; x += PU_GT) {
        const int wv = __ldg(col + x);
        if (wv == FM_ABSENT_WEIGHT) continue;
        const int lxv = __ldcg(a.lx + x);
        if (lyv >= lxv) continue;                              // cannot improve (len >= 0)
        const int mx = __ldcg(a.match + x);
        if (mx == y) continue;                                 // flow arc: not residual forward
        if (a.use_fix && ((__ldg(a.fixed_t + (size_t)y * a.nw + (x >> 5)) >> (x & 31)) & 1u)) continue;
        const long long px = __ldcg((const long long *)a.px + x);
        const long long rc = -(long long)wv * a.scale + px - pyv;
        long long len = floordiv_eps(rc, a.eps, inv_eps) + 1;
        if (len < 0) len = 0;
        const long long cand = (long long)lyv + len;
        if (cand > cap || cand >= lxv) continue;
        const int old = atomicMin(a.lx + x, (int)cand);
        if ((int)cand >= old || mx < 0 || __ldcg(a.frozen + x)) continue;
        // l(x) dropped: relax x's unit arc y2 -> x (reverse of the matched arc)
        const long long rc2 = (long long)__ldg(a.w + (size_t)x * n + mx) * a.scale - px +
                              __ldcg((const long long *)a.py + mx);
        long long len2 = floordiv_eps(rc2, a.eps, inv_eps) + 1;
        if (len2 < 0) len2 = 0;
        const long long cand2 = cand + len2;
        if (cand2 > cap) continue;
        if (ylabel_drop(a, mx, (int)cand2)) push(mx);
    }
}

// the x of one 4-x group whose bit is set in mask4 (their l(x) may drop): load their
// matches and prices, relax x -> y into l(x) and, where it dropped, x's matched
// reverse arc into its Y
template <typename Push>
__device__ __forceinline__ void pu_relax4(const AssignDev &a, const PuDev &f, int y, int lyv, long long pyv,
                                          long long cap, double inv_eps, int xb, uint32_t mask4,
                                          const int (&wv)[4], const int (&lxv)[4], Push push) {
    const int4 m4 = __ldca((const int4 *)(a.match + xb));
    const longlong2 pa = __ldca((const longlong2 *)(a.px + xb)), pb = __ldca((const longlong2 *)(a.px + xb) + 1);
    const int mxv[4] = {m4.x, m4.y, m4.z, m4.w};
    const long long pxv[4] = {pa.x, pa.y, pb.x, pb.y};
    int cand[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        cand[k] = LINF;
        if (!((mask4 >> k) & 1u) || mxv[k] == y) continue;
        const long long rc = -(long long)wv[k] * a.scale + pxv[k] - pyv;
        long long len = floordiv_eps(rc, a.eps, inv_eps) + 1;
        if (len < 0) len = 0;
        const long long c1 = (long long)lyv + len;
        if (c1 <= cap && c1 < lxv[k]) cand[k] = (int)c1;
    }
#pragma unroll
    for (int k = 0; k < 4; k++)
        if (cand[k] < LINF) atomicMin(a.lx + xb + k, cand[k]);   // fire-and-forget (RED)
#pragma unroll
    for (int k = 0; k < 4; k++) {
        if (cand[k] >= LINF || mxv[k] < 0) continue;
        const int x = xb + k;
        if (__ldca(a.frozen + x)) continue;
        const long long rc2 = (long long)__ldca(a.mw + x) * a.scale - pxv[k] + __ldca((const long long *)a.pmx + x);
        long long len2 = floordiv_eps(rc2, a.eps, inv_eps) + 1;
        if (len2 < 0) len2 = 0;
        const long long cand2 = cand[k] + len2;
        if (cand2 > cap) continue;
        const int mx = mxv[k];
        if (ylabel_drop(a, mx, (int)cand2)) push(mx);
    }
}

// pu_scan_y with a cheap filter first: a chunk's weights and labels are loaded alone
// and only the x whose label could still drop (l(y) < l(x), arc present and not
// fixed) load their matches and prices; the matched reverse arc's operands are read
// only for the x whose label did drop.  After the first waves nearly every l(x) is
// already at or below l(y), so most chunks cost two vector loads and no arithmetic
// (and the kernel fits 2 CTAs per SM).  Loading a second chunk up front spilled and
// measured slower (r02h4).
template <typename Push>
__device__ __forceinline__ void pu_scan_y_filtered(const AssignDev &a, const PuDev &f, int y, int lyv,
                                                   long long pyv, long long cap, double inv_eps, int gt,
                                                   int PU_GT, Push push) {
    const int n = a.n;
    const int32_t *col = f.wt + (size_t)y * n;
    const int nv8 = (n & 7) ? 0 : n;
    for (int x0 = gt * 8; x0 < nv8; x0 += PU_GT * 8) {
        const int4 w0 = __ldg((const int4 *)(col + x0)), w1 = __ldg((const int4 *)(col + x0 + 4));
        const int4 l0 = __ldcg((const int4 *)(a.lx + x0)), l1 = __ldcg((const int4 *)(a.lx + x0 + 4));
        uint32_t fb = 0;
        if (a.use_fix) fb = (__ldg(a.fixed_t + (size_t)y * a.nw + (x0 >> 5)) >> (x0 & 31)) & 0xffu;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int4 wq = h ? w1 : w0, lq = h ? l1 : l0;
            const int wv[4] = {wq.x, wq.y, wq.z, wq.w};
            const int lxv[4] = {lq.x, lq.y, lq.z, lq.w};
            uint32_t m4 = 0;
#pragma unroll
            for (int k = 0; k < 4; k++)
                if (wv[k] != FM_ABSENT_WEIGHT && lyv < lxv[k] && !((fb >> (4 * h + k)) & 1u)) m4 |= 1u << k;
            if (m4) pu_relax4(a, f, y, lyv, pyv, cap, inv_eps, x0 + 4 * h, m4, wv, lxv, push);
        }
    }
    for (int x = nv8 + gt; x < n; x += PU_GT) {
        const int wv = __ldg(col + x);
        if (wv == FM_ABSENT_WEIGHT) continue;
        const int lxv = __ldcg(a.lx + x);
        if (lyv >= lxv) continue;
        const int mx = __ldcg(a.match + x);
        if (mx == y) continue;
        if (a.use_fix && ((__ldg(a.fixed_t + (size_t)y * a.nw + (x >> 5)) >> (x & 31)) & 1u)) continue;
        const long long px = __ldcg((const long long *)a.px + x);
        const long long rc = -(long long)wv * a.scale + px - pyv;
        long long len = floordiv_eps(rc, a.eps, inv_eps) + 1;
        if (len < 0) len = 0;
        const long long cand = (long long)lyv + len;
        if (cand > cap || cand >= lxv) continue;
        const int old = atomicMin(a.lx + x, (int)cand);
        if ((int)cand >= old || mx < 0 || __ldcg(a.frozen + x)) continue;
        const long long rc2 = (long long)__ldg(a.w + (size_t)x * n + mx) * a.scale - px +
                              __ldcg((const long long *)a.py + mx);
        long long len2 = floordiv_eps(rc2, a.eps, inv_eps) + 1;
        if (len2 < 0) len2 = 0;
        const long long cand2 = cand + len2;
        if (cand2 > cap) continue;
        if (ylabel_drop(a, mx, (int)cand2)) push(mx);
    }
}

// FILTER: the filtered column scan at 2 CTAs per SM (option pu_filter)
template <bool FILTER>
#ifndef FM_PU_MINB
#define FM_PU_MINB 2
#endif
__global__ void __launch_bounds__(ATHREADS, FILTER ? FM_PU_MINB : 1) price_update_kernel(AssignDev a, PuDev f, int gated) {
    // gated: run only when the rounds asked for an update (the gate is rewritten only at
    // this kernel's end, after its grid barriers, so every thread reads the same value)
    if (gated && __ldcg(a.cnt + C_GATE) != 1) return;
    cg::grid_group grid = cg::this_grid();
    const int n = a.n;
    const int tid = blockIdx.x * ATHREADS + threadIdx.x, nthr = gridDim.x * ATHREADS;
    const int lane = threadIdx.x & 31;
    const double inv_eps = 1.0 / (double)a.eps;
    // Labels are only needed up to last + 1 (last = the largest label of an active
    // node): explore with a label cap, and widen it (x8) only if some active node is
    // still unlabelled.  Under a cap every node whose true label is <= cap gets its
    // exact label (labels never decrease along a shortest path), which is all the
    // final min(label, last + 1) needs.
    long long cap = min((long long)a.max_bucket, (long long)(a.pu_cap0 > 0 ? a.pu_cap0 : 8));
    int it_total = 0;
    __shared__ int s_ly[PU_GROUPS_MAX], s_y[PU_GROUPS_MAX], s_next[PU_GROUPS_MAX];
    __shared__ long long s_py[PU_GROUPS_MAX];
    for (;;) {
    if (tid == 0) { a.cnt[C_PU_LAST] = 0; a.cnt[C_PU_CHG] = 0; }
    for (int v = tid; v < n; v += nthr) {
        a.lx[v] = LINF;
        const int mv = __ldcg(a.match + v);
        a.mw[v] = mv >= 0 ? __ldg(a.w + (size_t)v * n + mv) : 0;
        a.pmx[v] = mv >= 0 ? __ldcg((const long long *)a.py + mv) : 0;
        if (__ldcg(a.ey + v) < 0) {
            a.ly[v] = 1;                                  // label 0, queued
            if (f.ring_on) {
                atomicAdd(f.rctr + 64, 1u);
                f.ring[atomicAdd(f.rctr + 32, 1u)] = v;   // slots are empty, tail starts at 0
            } else {
                f.fy[0][atomicAdd(f.cnt + 0, 1)] = v;   // iteration 0's frontier (counter 0 of 3)
            }
        } else {
            a.ly[v] = 2 * LINF;                           // unlabelled, not queued
        }
    }
    grid.sync();
    // One barrier per iteration: the Y step is folded into the X step -- whenever
    // l(x) drops, x's matched reverse arc is relaxed into its Y right away (chaotic
    // relaxation reaches the same fixpoint).  Frontier counters are triple-buffered so
    // the counter of iteration it+2 can be zeroed during iteration it.
    int it = 0;
    const unsigned long long t_it0 = globaltimer();
    if (f.ring_on) {
        // Queue-driven relaxation, no grid barrier per wave: groups take frontier Y from
        // the ring until it is empty and nothing is in flight (chaotic relaxation: every
        // label is a path length and only falls, so the fixpoint is the same).  The ring
        // holds more slots than queued entries (<= n, one per Y) plus waiting groups, an
        // entry is taken with an exchange (one taker) and a slot refilled only when empty
        // (CAS), so no entry is lost, duplicated or overwritten.
        // Work-first: the first Y a group's scan re-queues is kept by the group as its
        // next Y (counted in pending like a ring entry) instead of a ring round trip, so a
        // chain of label drops runs at scan latency; further drops go to the ring.
        const int PU_GT = ATHREADS / f.ring_groups;
        const int grp = threadIdx.x / PU_GT, gt = threadIdx.x - grp * PU_GT;
        unsigned long long ys = 0, scan_ns = 0, t_scan = 0;
        if (gt == 0) s_next[grp] = -1;
        for (;;) {
            if (gt == 0) {
                if (t_scan) scan_ns += globaltimer() - t_scan;
                int y = f.local_next ? s_next[grp] : -1;
                s_next[grp] = -1;
                if (y < 0) {
                    const unsigned sl = atomicAdd(f.rctr + 0, 1u) % (unsigned)f.ring_cap;
                    for (unsigned ns = 32;; ns = min(ns * 2, 1024u)) {
                        // exactly one taker per entry; an empty slot stays empty (no read first)
                        const int v = atomicExch(f.ring + sl, -1);
                        if (v >= 0) { y = v; break; }
                        if (*(volatile unsigned *)(f.rctr + 64) == 0) break;
                        __nanosleep(ns);
                    }
                }
                s_y[grp] = y;
                if (y >= 0) {
                    s_py[grp] = __ldcg((const long long *)a.py + y);
                    s_ly[grp] = ylabel_take(a, y);   // a later drop re-queues y
                    ys++;
                    t_scan = globaltimer();
                }
            }
            group_sync(grp, PU_GT);
            const int y = s_y[grp];
            if (y < 0) break;
            const auto ring_push = [&](int mx) {
                atomicAdd(f.rctr + 64, 1u);
                if (f.local_next && atomicCAS(&s_next[grp], -1, mx) == -1) return;   // the group's next Y
                const unsigned t = atomicAdd(f.rctr + 32, 1u);
                fence_acq_rel_gpu();         // labels (and pending) visible before the entry
                int32_t *slot = f.ring + t % (unsigned)f.ring_cap;
                while (atomicCAS(slot, -1, mx) != -1) __nanosleep(64);
            };
            if (FILTER) pu_scan_y_filtered(a, f, y, s_ly[grp], s_py[grp], cap, inv_eps, gt, PU_GT, ring_push);
            else pu_scan_y(a, f, y, s_ly[grp], s_py[grp], cap, inv_eps, gt, PU_GT, ring_push);
            group_sync(grp, PU_GT);
            if (gt == 0) { fence_acq_rel_gpu(); atomicSub(f.rctr + 64, 1u); }
        }
        if (gt == 0 && ys) { atomicAdd(a.ops + O_PU_YS, ys); atomicAdd(a.ops + O_PU_SCANNS, scan_ns); }
        grid.sync();
    } else
    for (;; it++) {
        const int b = it & 1, nb = b ^ 1;
        int ny, u1, u2;
        cta_bcast3(f.cnt + it % 3, nullptr, nullptr, ny, u1, u2);
        if (ny == 0) break;
        if (tid == 0) atomicAdd(a.ops + O_PU_YS, (unsigned long long)ny);
        if (tid == 0) f.cnt[(it + 2) % 3] = 0;
        // Each CTA works on PU_GROUPS frontier Y at once (one group of GT threads per Y,
        // group barriers): a column scan is a latency chain, so several in flight per
        // SM beat one CTA-wide scan after another.  The group leader fetches each Y's
        // header (clear its queued flag, then read l(y), p(y)) one Y ahead, so the next
        // header's round trips overlap this scan.
        // groups only pay when the frontier outnumbers the CTAs (a group's scan is
        // PU_GROUPS times longer than a CTA-wide one)
        const int ng = ny > (int)gridDim.x ? PU_GROUPS : 1, PU_GT = ATHREADS / ng;
        const int grp = threadIdx.x / PU_GT, gt = threadIdx.x - grp * PU_GT;
        const int istep = gridDim.x * ng;
        int nxt_y = -1, nxt_l = 0;
        long long nxt_p = 0;
        if (gt == 0 && blockIdx.x * ng + grp < ny) {
            nxt_y = __ldcg(f.fy[b] + blockIdx.x * ng + grp);
            nxt_p = __ldcg((const long long *)a.py + nxt_y);
            nxt_l = ylabel_take(a, nxt_y);   // a later drop re-queues y
        }
        for (int i = blockIdx.x * ng + grp; i < ny; i += istep) {
            if (gt == 0) {
                s_y[grp] = nxt_y; s_ly[grp] = nxt_l; s_py[grp] = nxt_p;
                if (i + istep < ny) {
                    nxt_y = __ldcg(f.fy[b] + i + istep);
                    nxt_p = __ldcg((const long long *)a.py + nxt_y);
                    nxt_l = ylabel_take(a, nxt_y);
                }
            }
            group_sync(grp, PU_GT);
            const int y = s_y[grp];
            const int lyv = s_ly[grp];
            const long long pyv = s_py[grp];
            const auto wave_push = [&](int mx) {
                f.fy[nb][atomicAdd(f.cnt + (it + 1) % 3, 1)] = mx;   // read after the grid barrier
            };
            if (FILTER) pu_scan_y_filtered(a, f, y, lyv, pyv, cap, inv_eps, gt, PU_GT, wave_push);
            else pu_scan_y(a, f, y, lyv, pyv, cap, inv_eps, gt, PU_GT, wave_push);
            group_sync(grp, PU_GT);
        }
        grid.sync();
    }
    it_total += it + 1;
    if (tid == 0) atomicAdd(a.ops + O_PU_ITNS, globaltimer() - t_it0);
    // last = max label over active nodes (unmatched X, Y with positive excess);
    // an active node left unlabelled under the cap asks for a wider cap
    int last = 0, missing = 0;
    for (int v = tid; v < n; v += nthr) {
        if (__ldcg(a.match + v) < 0 && !__ldcg(a.frozen + v)) {
            const int l = __ldcg(a.lx + v);
            if (l >= LINF) missing = 1; else last = max(last, l);
        }
        if (__ldcg(a.ey + v) > 0) {
            const int l = ylabel(__ldcg(a.ly + v));
            if (l >= LINF) missing = 1; else last = max(last, l);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
        missing |= __shfl_xor_sync(0xffffffffu, missing, o);
    }
    if (lane == 0 && last) atomicMax(a.cnt + C_PU_LAST, last);
    if (lane == 0 && missing) atomicOr(a.cnt + C_PU_CHG, 1);
    grid.sync();
    int chg, u1, u2;
    cta_bcast3(a.cnt + C_PU_CHG, nullptr, nullptr, chg, u1, u2);
    if (!chg || cap >= a.max_bucket) break;
    cap = min(cap * 8, (long long)a.max_bucket);
    if (tid == 0) { f.cnt[0] = f.cnt[1] = f.cnt[2] = 0; f.rctr[0] = f.rctr[32] = f.rctr[64] = 0; }
    grid.sync();
    }  // cap loop
    const long long K = min((long long)__ldcg(a.cnt + C_PU_LAST), (long long)a.max_bucket) + 1;
    unsigned yfin = 0, ylab = 0;
    for (int v = tid; v < n; v += nthr) {
        const int lyv = ylabel(a.ly[v]);
        const long long dx = min((long long)a.lx[v], K), dy = min((long long)lyv, K);
        yfin += lyv < K;
        ylab += lyv < LINF;
        if (a.validate && (dx < 0 || dy < 0)) atomicExch(a.cnt + C_INFEASIBLE, V_RAISE);
        a.px[v] -= a.eps * dx;
        a.py[v] -= a.eps * dy;
    }
    yfin = __reduce_add_sync(0xffffffffu, yfin);
    ylab = __reduce_add_sync(0xffffffffu, ylab);
    if (lane == 0 && ylab) {
        atomicAdd(a.ops + O_PU_YFIN, (unsigned long long)yfin);
        atomicAdd(a.ops + O_PU_YLAB, (unsigned long long)ylab);
    }
    if (tid == 0) {
        atomicAdd(a.ops + O_PU_LASTSUM, (unsigned long long)(K - 1));
        a.cnt[C_RELABELS] = 0;
        f.cnt[0] = f.cnt[1] = f.cnt[2] = f.cnt[3] = 0;
        f.rctr[0] = f.rctr[32] = f.rctr[64] = 0;
        atomicAdd(a.ops + O_PU, 1ull);
        atomicAdd(a.ops + O_PU_ITERS, (unsigned long long)it_total);
        if (gated) { a.cnt[C_GATE] = 0; a.cnt[C_PUN] += 1; }   // the next enqueued rounds launch runs
    }
}

// wt = w^T (32 x 32 shared-memory tiles)
__global__ void transpose_kernel(const int32_t *w, int32_t *wt, int n) {
    __shared__ int32_t t[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int r = by + j, c = bx + threadIdx.x;
        if (r < n && c < n) t[j][threadIdx.x] = w[(size_t)r * n + c];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int r = bx + j, c = by + threadIdx.x;
        if (r < n && c < n) wt[(size_t)r * n + c] = t[threadIdx.x][j];
    }
}

// arc_fix (assign_scaling.py:185-205): freeze a pair when either direction's
// reduced cost exceeds 2 n eps.  Matched pairs that freeze pin x to y for good.
__global__ void arc_fix_kernel(AssignDev a) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long thr = 2LL * a.n * a.eps;
    unsigned long long cnt = 0;
    for (int x = warp; x < a.n; x += nwarps) {
        const long long px = a.px[x];
        const int mx = a.match[x];
        uint32_t *frow = a.fixed + (size_t)x * a.nw;
        for (int wb = 0; wb < a.nw; wb++) {
            const int y = wb * 32 + lane;
            bool fix = false;
            const uint32_t old = frow[wb];
            if (y < a.n && !((old >> lane) & 1u)) {
                const int wv = a.w[(size_t)x * a.n + y];
                if (wv != FM_ABSENT_WEIGHT) {
                    const long long rc = -(long long)wv * a.scale + px - a.py[y];
                    fix = rc > thr || -rc > thr;
                }
            }
            const uint32_t bits = __ballot_sync(0xffffffffu, fix);
            if (fix) {
                cnt++;
                if (y == mx) { a.frozen[x] = 1; atomicAdd(a.frozen_in + y, 1); }
            }
            if (lane == 0 && bits) frow[wb] = old | bits;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0 && cnt) atomicAdd(a.ops + O_FIXED, cnt);
}

// fixed_t = transpose of the fixed bitmask: one warp per 32 x 32 bit block, lane i
// holds row x = 32 bx + i and 32 ballots deal out the transposed rows
__global__ void bit_transpose_kernel(const uint32_t *in, uint32_t *out, int n, int nw) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int blk = warp; blk < nw * nw; blk += nwarps) {
        const int bx = blk / nw, by = blk - bx * nw;
        const int x = bx * 32 + lane;
        const uint32_t v = x < n ? in[(size_t)x * nw + by] : 0u;
        uint32_t mine = 0;
#pragma unroll
        for (int j = 0; j < 32; j++) {
            const uint32_t b = __ballot_sync(0xffffffffu, (v >> j) & 1u);
            if (lane == j) mine = b;
        }
        const int y = by * 32 + lane;
        if (y < n) out[(size_t)y * nw + bx] = mine;
    }
}

// max |w| over present arcs (scaled_cost_bound = (n+1) max|w|, assign_scaling.py:133)
__global__ void weight_bound_kernel(const int32_t *w, int64_t nn, unsigned long long *out /* [0] max|w| [2] arcs */) {
    unsigned long long m = 0, cnt = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nn;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int v = w[i];
        if (v != FM_ABSENT_WEIGHT) {
            m = max(m, (unsigned long long)(v < 0 ? -(long long)v : v));
            cnt++;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (m) atomicMax(out, m);
        if (cnt) atomicAdd(out + 2, cnt);
    }
}

// Loaded state (a reference ScalingState copied in): frozen[x] = x's matched arc is
// fixed, frozen_in[y] = frozen matches into y, ey[y] = (#matched into y) - 1.
__global__ void load_state_kernel(AssignDev a) {
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < a.n; x += gridDim.x * blockDim.x) {
        const int y = a.match[x];
        const bool fz = y >= 0 && ((a.fixed[(size_t)x * a.nw + (y >> 5)] >> (y & 31)) & 1u);
        a.frozen[x] = fz ? 1 : 0;
        if (y >= 0) {
            atomicAdd(a.ey + y, 1);
            if (fz) atomicAdd(a.frozen_in + y, 1);
        }
    }
}

// Coordinator round start (stepwise refine): list every active X (unmatched) in
// xlist[0] and every Y holding excess in ylist[0]; the round counter restarts at 0.
__global__ void active_lists_kernel(AssignDev a) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += gridDim.x * blockDim.x) {
        if (a.match[v] < 0) a.xlist[0][atomicAdd(a.cnt + C_X0, 1)] = v;
        if (a.ey[v] > 0) a.ylist[0][atomicAdd(a.cnt + C_Y0, 1)] = v;
    }
}

// X phase over xlist[0] (the active X of a loaded / freshly begun refine): relabel
// if needed, then push the unit, appending Y that become active to ylist[0].
__global__ void __launch_bounds__(ATHREADS) x_phase_kernel(AssignDev a, int tag) {
    const int warp = (blockIdx.x * ATHREADS + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * ATHREADS) >> 5;
    const int nx = __ldcg(a.cnt + C_X0);
    unsigned long long pushes = 0, relabels = 0;
    for (int i = warp; i < nx; i += nwarps)
        x_op<false>(a, __ldcg(a.xlist[0] + i), Lists{a.ylist[0], a.cnt + C_Y0}, pushes, relabels, tag);
    if ((threadIdx.x & 31) == 0) {
        if (pushes) atomicAdd(a.ops + O_PUSH, pushes);
        if (relabels) atomicAdd(a.ops + O_RELABEL, relabels);
    }
}

// ---- exact optimality certificate (no negative residual cycle)
// A perfect matching M is a maximum-weight matching iff the residual graph of M
// (forward arcs x->y for every present, unmatched pair; reverse arcs y->x for the
// matched pairs) has no negative cycle under the arc costs -w (scaled by any s > 0).
// Shortest distances from a virtual source joined to every node by 0-cost arcs then
// exist, and Bellman-Ford reaches them within 2n passes; a pass that still changes
// a distance after 2n passes proves a negative cycle.  Reduced costs under the
// solver's final prices make the distances start near their fixpoint (every arc is
// >= -eps at the end of the last refine), so a few passes usually settle it.  Every
// present arc counts, fixed or not: the certificate is independent of the solver.
__global__ void certify_init_kernel(const int32_t *w, const int32_t *match, int n, long long *dx, long long *dy,
                                    int32_t *bad /* not a perfect matching of present pairs */, int32_t *ycount) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        dx[v] = 0; dy[v] = 0;
        const int y = match[v];
        if (y < 0 || y >= n || w[(size_t)v * n + y] == FM_ABSENT_WEIGHT) atomicExch(bad, 1);
        else if (atomicAdd(ycount + y, 1) != 0) atomicExch(bad, 1);
    }
}

// forward pass: d(y) <- min(d(y), d(x) + c_p(x, y)) over present unmatched pairs; one
// warp per row, coalesced row reads, an atomicMin only where a distance drops
__global__ void certify_forward_kernel(const int32_t *w, const int32_t *match, const long long *px,
                                       const long long *py, long long scale, int n, const long long *dx,
                                       long long *dy, int32_t *changed) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    int chg = 0;
    for (int x = warp; x < n; x += nwarps) {
        const long long base = __ldcg(dx + x) + (px ? __ldg(px + x) : 0);
        const int mx = __ldg(match + x);
        const int32_t *row = w + (size_t)x * n;
        for (int y = lane; y < n; y += 32) {
            const int wv = __ldg(row + y);
            if (wv == FM_ABSENT_WEIGHT || y == mx) continue;
            const long long cand = base - (long long)wv * scale - (py ? __ldg(py + y) : 0);
            if (cand < __ldcg(dy + y)) {
                const long long old = atomicMin((long long *)dy + y, cand);
                chg |= cand < old;
            }
        }
    }
    if (__any_sync(0xffffffffu, chg) && lane == 0) atomicExch(changed, 1);
}

// reverse pass: d(x) <- min(d(x), d(M(x)) + c_p(M(x) -> x)), c_p of the reverse arc
// = -c_p(x, M(x))
__global__ void certify_reverse_kernel(const int32_t *w, const int32_t *match, const long long *px,
                                       const long long *py, long long scale, int n, long long *dx,
                                       const long long *dy, int32_t *changed) {
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
        const int y = match[x];
        const long long rc = -(long long)w[(size_t)x * n + y] * scale + (px ? px[x] : 0) - (py ? py[y] : 0);
        const long long cand = dy[y] - rc;
        if (cand < dx[x]) { dx[x] = cand; atomicExch(changed, 1); }
    }
}

__global__ void objective_kernel(const int32_t *w, const int32_t *match, int n,
                                 unsigned long long *out) {
    long long s = 0;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < n; x += gridDim.x * blockDim.x) {
        const int y = match[x];
        if (y >= 0) s += w[(size_t)x * n + y];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, (unsigned long long)s);
}

}  // namespace

struct fm_assign {
    int32_t n = 0, device = 0, nw = 0;
    AssignDev d{};
    int32_t *in_w = nullptr;          // staging for *_host
    unsigned long long *acc = nullptr; // [0] bound [1] objective
    unsigned long long *h_ops = nullptr;
    int32_t *h_cnt = nullptr;
    unsigned long long *h_acc = nullptr;
    cudaStream_t own_stream = nullptr, stream = nullptr;
    int coop_blocks = 0, pu_blocks = 0, sms = 0;
    int pu_blocks_k[2] = {0, 0};     // price_update_kernel<false / true> cooperative grid sizes
    PuDev pu{};
    int32_t *wt = nullptr;
    cudaEvent_t ev[4] = {};
    cudaEvent_t ev_pu[16] = {};  // around the enqueued-ahead price updates (2 per pair, <= 8 pairs)
    int pu_last_refine = 2;      // price updates of the previous refine (sizes the enqueue-ahead batch)
    bool pu_pending = false;
    // solve state (also drives the stepwise API)
    long long alpha = 10, bound = 0, eps = 1, round_budget = 0;
    int pu_threshold = 0, tail_threshold = 1, pu_every_k = 0;
    // options (fm_assign_set_option; round-1 environment knobs)
    int opt_ybatch_min = 1, opt_pu_ring = 1, opt_pu_threshold = -1, opt_tail_threshold = 1, opt_pu_cap = 256;
    int opt_cta_x = 4, opt_cta_y = 4;
    int opt_trace = 0;               // price-update statistics line on stderr after each solve
    int opt_pu_local = 0;            // price update: work-first continuation of a group's first re-queued Y
    int opt_pu_groups = 2;           // r02h3: with the filtered scan 2 groups per CTA beat 4 (M10000 47.4 -> 44.4 ms)
    int opt_pu_filter = 1;           // price update: filtered column scans at 2 CTAs per SM
    int opt_round_ctas = 0;          // refine rounds: cooperative CTAs (0 = one per SM)
    int32_t flags = 0;
    fm_stats st{};
};

namespace {

// make_scaling_state (assign_scaling.py:127-142): prices 0, eps0 = max(1, bound)
int assign_setup(fm_assign *A, const int32_t *w, int64_t alpha, int32_t flags) {
    const int n = A->n;
    AssignDev &d = A->d;
    d.w = w;
    d.scale = (int64_t)n + 1;
    d.use_fix = (flags & FM_ASSIGN_ARC_FIX) ? 1 : 0;
    d.validate = (flags & FM_ASSIGN_VALIDATE) ? 1 : 0;
    d.vbase = 0;
    d.ybatch_min = std::max(1, A->opt_ybatch_min);
    d.cta_x = std::max(1, A->opt_cta_x);
    d.cta_y = std::max(1, A->opt_cta_y);
    A->alpha = alpha;
    A->flags = flags;
    memset(&A->st, 0, sizeof(A->st));
    A->pu_last_refine = 2;
    cudaStream_t s = A->stream;
    cudaEventRecord(A->ev[2], s);
    FM_CHECK_CUDA(cudaMemsetAsync(d.px, 0, sizeof(int64_t) * n, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.py, 0, sizeof(int64_t) * n, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.match, 0xff, sizeof(int32_t) * n, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.frozen, 0, n, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.frozen_in, 0, sizeof(int32_t) * n, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.ybcnt, 0, sizeof(int32_t) * n, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.fixed, 0, sizeof(uint32_t) * (size_t)n * d.nw, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.fixed_t, 0, sizeof(uint32_t) * (size_t)n * d.nw, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.ops, 0, sizeof(unsigned long long) * O_COUNT, s));
    FM_CHECK_CUDA(cudaMemsetAsync(A->acc, 0, sizeof(unsigned long long) * 4, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.pw, 0, sizeof(int32_t) * 2 * (size_t)n, s));
    weight_bound_kernel<<<A->sms * 4, 256, 0, s>>>(w, (int64_t)n * n, A->acc);
    FM_CHECK_LAUNCH();
    A->st.launches++;
    if (flags & FM_ASSIGN_PRICE_UPDATE) {
        A->pu.wt = A->wt;
        transpose_kernel<<<dim3((n + 31) / 32, (n + 31) / 32), dim3(32, 8), 0, s>>>(w, A->wt, n);
        FM_CHECK_LAUNCH();
        FM_CHECK_CUDA(cudaMemsetAsync(A->pu.cnt, 0, sizeof(int32_t) * 4, s));
        // > queued entries (<= n) + groups waiting on a slot (pu_blocks * PU_GROUPS)
        A->pu.ring_cap = n + std::min(PU_RING_EXTRA, A->pu_blocks * PU_GROUPS_MAX + 64);
        A->pu.ring_on = A->opt_pu_ring ? 1 : 0;
        A->pu.ring_groups = A->opt_pu_groups;
        A->pu.local_next = A->opt_pu_local ? 1 : 0;
        if (A->pu.ring_on) {
            FM_CHECK_CUDA(cudaMemsetAsync(A->pu.ring, 0xff, sizeof(int32_t) * ((size_t)n + PU_RING_EXTRA), s));
            FM_CHECK_CUDA(cudaMemsetAsync(A->pu.rctr, 0, sizeof(unsigned int) * 96, s));
        }
        A->st.launches++;
    }
    FM_CHECK_CUDA(cudaMemcpyAsync(A->h_acc, A->acc, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, s));
    FM_CHECK_CUDA(cudaStreamSynchronize(s));
    A->bound = (long long)A->h_acc[0] * (long long)(n + 1);
    // _ops_budget (assign_scaling.py:374-377) = max(1e4, 40 n^2 m); every round does >= 1 op
    const double budget_d = std::max(1e4, 40.0 * n * (double)n * std::max<double>(1.0, (double)A->h_acc[2]));
    A->round_budget = budget_d > 4e18 ? (long long)4e18 : (long long)budget_d;
    A->eps = std::max(1LL, A->bound);
    A->pu_threshold = (flags & FM_ASSIGN_PRICE_UPDATE)
                          ? (A->opt_pu_threshold >= 0 ? A->opt_pu_threshold : std::max(64, n / 16)) : 0;
    A->tail_threshold = A->opt_tail_threshold;
    d.pu_cap0 = A->opt_pu_cap;
    return FM_OK;
}

// C_INFEASIBLE word -> status code and message
int assign_status(int why) {
    switch (why) {
    case 0: return FM_OK;
    case 1: fm_set_error("active node has no residual arc: instance admits no perfect matching"); return FM_INFEASIBLE;
    case 3: fm_set_error("operation budget exceeded; prices diverge, instance admits no perfect matching");
            return FM_INFEASIBLE;
    case V_RELABEL: fm_set_error("validate: relabel failed to lower a price"); return FM_VALIDATION;
    case V_OWNER: fm_set_error("validate: price word written by two ops in one phase"); return FM_VALIDATION;
    case V_RAISE: fm_set_error("validate: price update would raise a price"); return FM_VALIDATION;
    default: fm_set_error("inconsistent Y excess during refine"); return FM_CUDA_ERROR;
    }
}

// one price_update_heuristic launch (cooperative) on the solver's stream
cudaError_t launch_price_update(fm_assign *A, int gated = 0) {
    void *pargs[] = {(void *)&A->d, (void *)&A->pu, (void *)&gated};
    const bool filt = A->opt_pu_filter != 0;
    return cudaLaunchCooperativeKernel(filt ? (void *)price_update_kernel<true> : (void *)price_update_kernel<false>,
                                       dim3(A->pu_blocks_k[filt ? 1 : 0]), dim3(ATHREADS), pargs, 0, A->stream);
}

// one refine (assign_scaling.py:145-182 + assign_par.py:115-237): eps <- max(1, ceil(eps/alpha)),
// begin_refine fused with the first X phase, lock-free rounds with price updates, arc fixing
int assign_one_refine(fm_assign *A) {
    const int n = A->n;
    AssignDev &d = A->d;
    cudaStream_t s = A->stream;
    long long eps = std::max(1LL, (A->eps + A->alpha - 1) / A->alpha);   // -(-eps // alpha)
    A->eps = eps;
    d.eps = eps;
    d.max_bucket = std::min<long long>(A->bound / eps + 2, LINF - 1);
    FM_CHECK_CUDA(cudaMemsetAsync(d.cnt, 0, sizeof(int32_t) * C_COUNT, s));
    reset_excess_kernel<<<(n + 255) / 256, 256, 0, s>>>(d);
    FM_CHECK_LAUNCH();
    begin_refine_kernel<<<std::max(1, std::min((n + AWARPS - 1) / AWARPS, A->sms * 4)), ATHREADS, 0, s>>>(d, 1);
    FM_CHECK_LAUNCH();
    A->st.launches += 2;
    // The rounds kernel and the price update alternate until the refine is over.  The
    // launches are enqueued PU_AHEAD pairs at a time with a device-side gate (C_GATE:
    // the rounds set it to "price update" or "over", the update back to "rounds"), so
    // the host reads the counters once per batch instead of once per price update;
    // launches past the refine's end return at once.
    // The batch size follows the previous refine's update count (no-op launches are not
    // free: a gated rounds launch still pays its cooperative launch and one barrier).
#ifndef FM_PU_AHEAD
#define FM_PU_AHEAD 8
#endif
    constexpr int PU_AHEAD = FM_PU_AHEAD;
    const bool pu_on = (A->flags & FM_ASSIGN_PRICE_UPDATE) != 0;
    int pus_done = 0;
    for (;;) {
        int no_cap = 0, gated = 1;
        int every_k = pu_on ? A->pu_every_k : 0;
        const int pairs = pu_on ? std::max(1, std::min(PU_AHEAD, A->pu_last_refine - pus_done)) : 1;
        for (int q = 0; q < pairs; q++) {
            d.vbase += 1 << 21;   // fresh validate phase tags per launch
            void *args[] = {(void *)&d, (void *)&A->tail_threshold, (void *)&A->round_budget, (void *)&A->pu_threshold,
                            (void *)&no_cap, (void *)&every_k, (void *)&gated};
            FM_CHECK_CUDA(cudaLaunchCooperativeKernel((void *)refine_rounds_kernel,
                                                      dim3(A->opt_round_ctas > 0 ? std::min(A->opt_round_ctas, A->coop_blocks) : A->coop_blocks),
                                                      dim3(ATHREADS), args, 0, s));
            A->st.launches++;
            if (!pu_on) break;
            cudaEventRecord(A->ev_pu[2 * q], s);
            FM_CHECK_CUDA(launch_price_update(A, 1));
            cudaEventRecord(A->ev_pu[2 * q + 1], s);
            A->st.launches++;
        }
        FM_CHECK_CUDA(cudaMemcpyAsync(A->h_cnt, d.cnt, sizeof(int32_t) * C_COUNT, cudaMemcpyDeviceToHost, s));
        FM_CHECK_CUDA(cudaStreamSynchronize(s));
        for (int q = 0; pu_on && q < pairs; q++) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, A->ev_pu[2 * q], A->ev_pu[2 * q + 1]);
            A->st.ms_bfs += ms;   // price-update kernels (a gated no-op adds its launch only)
        }
        pus_done = A->h_cnt[C_PUN];
        if (A->h_cnt[C_INFEASIBLE] || A->h_cnt[C_GATE] == 2) break;
    }
    A->pu_last_refine = pus_done;
    if (d.use_fix) {
        arc_fix_kernel<<<std::max(1, std::min((n + 7) / 8, A->sms * 8)), 256, 0, s>>>(d);
        FM_CHECK_LAUNCH();
        A->st.launches++;
        bit_transpose_kernel<<<std::max(1, std::min((d.nw * d.nw + 7) / 8, A->sms * 8)), 256, 0, s>>>(
            d.fixed, d.fixed_t, n, d.nw);
        FM_CHECK_LAUNCH();
        A->st.launches++;
    }
    A->st.refines++;
    return assign_status(A->h_cnt[C_INFEASIBLE]);
}

// objective, counters and host copies (assign_scaling.py:456-466)
int assign_finish(fm_assign *A, int rc, int64_t *objective_out, int32_t *match_out, int64_t *prices_out) {
    const int n = A->n;
    AssignDev &d = A->d;
    cudaStream_t s = A->stream;
    if (rc == FM_OK) {
        FM_CHECK_CUDA(cudaMemsetAsync(A->acc + 1, 0, sizeof(unsigned long long), s));
        objective_kernel<<<std::max(1, std::min((n + 255) / 256, A->sms * 2)), 256, 0, s>>>(d.w, d.match, n, A->acc + 1);
        FM_CHECK_LAUNCH();
        A->st.launches++;
    }
    cudaEventRecord(A->ev[3], s);
    FM_CHECK_CUDA(cudaMemcpyAsync(A->h_ops, d.ops, sizeof(unsigned long long) * O_COUNT, cudaMemcpyDeviceToHost, s));
    FM_CHECK_CUDA(cudaMemcpyAsync(A->h_acc, A->acc, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, s));
    if (match_out) FM_CHECK_CUDA(cudaMemcpyAsync(match_out, d.match, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    if (prices_out) {
        FM_CHECK_CUDA(cudaMemcpyAsync(prices_out, d.px, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
        FM_CHECK_CUDA(cudaMemcpyAsync(prices_out + n, d.py, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
    }
    FM_CHECK_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, A->ev[2], A->ev[3]);
    A->st.ms_total = ms;
    A->st.ms_push = ms - A->st.ms_bfs;  // everything but the price updates
    A->st.pushes = (int64_t)A->h_ops[O_PUSH];
    A->st.relabels = (int64_t)A->h_ops[O_RELABEL];
    A->st.rounds = (int64_t)A->h_ops[O_ROUNDS];
    A->st.pr_sweeps = (int64_t)A->h_ops[O_TAIL_ROUNDS];  // rounds run by the single-CTA tail
    A->st.reserved[0] = (int64_t)A->h_ops[O_FIXED];      // pairs fixed
    A->st.reserved[1] = (int64_t)A->h_ops[O_PU];         // price updates
    A->st.reserved[2] = (int64_t)A->h_ops[O_PU_ITERS];   // Bellman-Ford iterations in them
    A->st.cut_sweeps = (int64_t)A->h_ops[O_PU_YS];       // price update: frontier Y visits
    A->st.pr_tiles = (int64_t)A->h_ops[O_PU_ITNS];       // price update: ns inside Bellman-Ford iterations (CTA 0)
    if (A->opt_trace && A->h_ops[O_PU]) {
        const double npu = (double)A->h_ops[O_PU];
        fprintf(stderr, "[fm_assign] %llu price updates: per update %.0f Y visits, %.1f us, last %.2f, "
                "Y labelled <= last %.0f, Y labelled %.0f, %.2f us per scan\n", A->h_ops[O_PU], A->h_ops[O_PU_YS] / npu,
                1e-3 * A->h_ops[O_PU_ITNS] / npu, A->h_ops[O_PU_LASTSUM] / npu, A->h_ops[O_PU_YFIN] / npu,
                A->h_ops[O_PU_YLAB] / npu, 1e-3 * A->h_ops[O_PU_SCANNS] / std::max(1.0, (double)A->h_ops[O_PU_YS]));
    }
    if (A->opt_trace)
        fprintf(stderr, "[fm_assign] grid rounds by max list size (count / ms): <=8 %llu / %.2f, <=32 %llu / %.2f, "
                "<=148 %llu / %.2f, <=592 %llu / %.2f, more %llu / %.2f; tail rounds %llu\n",
                A->h_ops[O_HIST], 1e-6 * A->h_ops[O_HIST_NS], A->h_ops[O_HIST + 1], 1e-6 * A->h_ops[O_HIST_NS + 1],
                A->h_ops[O_HIST + 2], 1e-6 * A->h_ops[O_HIST_NS + 2], A->h_ops[O_HIST + 3], 1e-6 * A->h_ops[O_HIST_NS + 3],
                A->h_ops[O_HIST + 4], 1e-6 * A->h_ops[O_HIST_NS + 4], A->h_ops[O_TAIL_ROUNDS]);
    if (A->opt_trace)
        fprintf(stderr, "[fm_assign] rounds with > 592 listed: Y phase + barrier %.2f ms, X phase + barrier %.2f ms; "
                "bucketed Y phases: bucket pass %.2f ms, + barrier %.2f ms; bucket fallbacks %llu; gather overflows %llu (%llu units, "
                "max candidates %llu)\n",
                1e-6 * A->h_ops[30], 1e-6 * A->h_ops[31], 1e-6 * A->h_ops[34], 1e-6 * A->h_ops[35], A->h_ops[32], A->h_ops[36],
                A->h_ops[37], A->h_ops[33]);
    A->st.reserved[3] = (int64_t)A->h_ops[O_TAIL_OPS];   // ops done by the single-CTA tail
    A->st.ms_cut = 1e-6 * (double)A->h_ops[O_TAIL_NS];   // time in single-CTA tail rounds
    A->st.ms_d2h = 1e-6 * (double)A->h_ops[O_MULTI_NS];  // time in grid-wide rounds
    A->st.ms_pr_kern = 1e-6 * (double)A->h_ops[O_PH_Y];  // CTA 0's Y phases in grid-wide rounds
    A->st.ms_bfs_kern = 1e-6 * (double)A->h_ops[O_PH_X]; // CTA 0's X phases in grid-wide rounds
    A->st.bytes_bfs = (int64_t)(A->h_ops[O_PH_SYNC1] + A->h_ops[O_PH_SYNC2]);  // ns in grid barriers
    // algorithmic bytes: every op scans one weight row (4n) + n prices (8n); the
    // begin phase and arc fixing read the whole matrix once each per refine
    A->st.bytes_push = (A->st.pushes + A->st.relabels) * 12LL * n +
                       A->st.refines * (int64_t)n * n * 4 * (d.use_fix ? 2 : 1);
    if (rc == FM_OK && objective_out) *objective_out = (int64_t)A->h_acc[1];
    return rc;
}

int assign_solve_device(fm_assign *A, const int32_t *w, int64_t alpha, int32_t flags,
                        int64_t *objective_out, int32_t *match_out, int64_t *prices_out) {
    FM_TRY(assign_setup(A, w, alpha, flags));
    int rc = FM_OK;
    for (;;) {
        rc = assign_one_refine(A);
        if (rc != FM_OK || A->eps == 1) break;
    }
    return assign_finish(A, rc, objective_out, match_out, prices_out);
}

}  // namespace

extern "C" int fm_assign_create(int32_t n, int32_t device, fm_assign **out) {
    if (!out || n < 1 || (int64_t)n * n > (int64_t)1 << 34) {
        fm_set_error("fm_assign_create: invalid n=%d", n);
        return FM_INVALID_ARG;
    }
    const int ndev = fm_device_count();
    if (ndev == 0) { fm_set_error("no CUDA device"); return FM_NO_DEVICE; }
    if (device < 0 || device >= ndev) { fm_set_error("device %d out of range", device); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(device));
    fm_assign *A = new fm_assign();
    A->n = n; A->device = device; A->nw = (n + 31) / 32;
    AssignDev &d = A->d;
    d.n = n; d.nw = A->nw; d.scale = (int64_t)n + 1;
    bool ok = cudaMalloc((void **)&d.px, sizeof(int64_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.py, sizeof(int64_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.match, sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.ey, sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.fixed, sizeof(uint32_t) * (size_t)n * A->nw) == cudaSuccess &&
              cudaMalloc((void **)&d.fixed_t, sizeof(uint32_t) * (size_t)n * A->nw) == cudaSuccess &&
              cudaMalloc((void **)&d.frozen, n) == cudaSuccess &&
              cudaMalloc((void **)&d.frozen_in, sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.xlist[0], sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.xlist[1], sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.ylist[0], sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.ylist[1], sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.cnt, sizeof(int32_t) * C_COUNT) == cudaSuccess &&
              cudaMalloc((void **)&d.lx, sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.ybcnt, sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.ybuf, sizeof(int32_t) * (size_t)n * YBUCKET) == cudaSuccess &&
              cudaMalloc((void **)&A->wt, sizeof(int32_t) * (size_t)n * n) == cudaSuccess &&
              cudaMalloc((void **)&A->pu.fy[0], sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&A->pu.fy[1], sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&A->pu.fx[0], sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&A->pu.fx[1], sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&A->pu.in_fx, sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&A->pu.in_fy, sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&A->pu.cnt, sizeof(int32_t) * 4) == cudaSuccess &&
              cudaMalloc((void **)&A->pu.ring, sizeof(int32_t) * ((size_t)n + PU_RING_EXTRA)) == cudaSuccess &&
              cudaMalloc((void **)&A->pu.rctr, sizeof(unsigned int) * 96) == cudaSuccess &&
              cudaMemset(A->pu.ring, 0xff, sizeof(int32_t) * ((size_t)n + PU_RING_EXTRA)) == cudaSuccess &&
              cudaMemset(A->pu.rctr, 0, sizeof(unsigned int) * 96) == cudaSuccess &&
              cudaMalloc((void **)&d.ly, sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.mw, sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.pmx, sizeof(int64_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.pw, sizeof(int32_t) * 2 * (size_t)n) == cudaSuccess &&
              cudaMalloc((void **)&d.ops, sizeof(unsigned long long) * O_COUNT) == cudaSuccess &&
              cudaMalloc((void **)&A->acc, sizeof(unsigned long long) * 4) == cudaSuccess &&
              cudaMallocHost((void **)&A->h_ops, sizeof(unsigned long long) * O_COUNT) == cudaSuccess &&
              cudaMallocHost((void **)&A->h_acc, sizeof(unsigned long long) * 4) == cudaSuccess &&
              cudaMallocHost((void **)&A->h_cnt, sizeof(int32_t) * C_COUNT) == cudaSuccess &&
              cudaStreamCreateWithFlags(&A->own_stream, cudaStreamNonBlocking) == cudaSuccess;
    if (!ok) {
        fm_set_error("fm_assign_create: allocation failed: %s", cudaGetErrorString(cudaGetLastError()));
        fm_assign_destroy(A);
        return FM_CUDA_ERROR;
    }
    A->stream = A->own_stream;
    for (auto &e : A->ev) cudaEventCreate(&e);
    for (auto &e : A->ev_pu) cudaEventCreate(&e);
    cudaDeviceGetAttribute(&A->sms, cudaDevAttrMultiProcessorCount, device);
    int per_sm = 0;
    int per_sm2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, refine_rounds_kernel, ATHREADS, 0);
    int per_sm3 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, price_update_kernel<false>, ATHREADS, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm3, price_update_kernel<true>, ATHREADS, 0);
    A->coop_blocks = std::max(1, std::min(per_sm, 2) * A->sms);
    A->pu_blocks_k[0] = std::max(1, std::min(per_sm2, 2) * A->sms);
    A->pu_blocks_k[1] = std::max(1, std::min(per_sm3, 2) * A->sms);
    A->pu_blocks = std::max(A->pu_blocks_k[0], A->pu_blocks_k[1]);   // sizes the ring
    *out = A;
    return FM_OK;
}

extern "C" void fm_assign_destroy(fm_assign *A) {
    if (!A) return;
    cudaSetDevice(A->device);
    void *dev[] = {A->d.mw, A->d.pmx, A->d.px, A->d.py, A->d.match, A->d.ey, A->d.fixed, A->d.fixed_t, A->d.frozen, A->d.frozen_in,
                   A->d.xlist[0], A->d.xlist[1], A->d.ylist[0], A->d.ylist[1], A->d.cnt, A->d.ops,
                   A->d.lx, A->d.ly, A->d.pw, A->d.ybcnt, A->d.ybuf, A->wt, A->pu.fy[0], A->pu.fy[1], A->pu.fx[0], A->pu.fx[1],
                   A->pu.in_fx, A->pu.in_fy, A->pu.cnt, A->pu.ring, A->pu.rctr,
                   A->acc, A->in_w};
    for (void *p : dev) if (p) cudaFree(p);
    if (A->h_ops) cudaFreeHost(A->h_ops);
    if (A->h_acc) cudaFreeHost(A->h_acc);
    if (A->h_cnt) cudaFreeHost(A->h_cnt);
    if (A->own_stream) cudaStreamDestroy(A->own_stream);
    for (auto e : A->ev) if (e) cudaEventDestroy(e);
    for (auto e : A->ev_pu) if (e) cudaEventDestroy(e);
    delete A;
}

extern "C" int fm_assign_solve(fm_assign *A, const int32_t *weights, int64_t alpha, int32_t flags,
                               int64_t *objective_out, int32_t *match_out, int64_t *prices_out,
                               fm_stats *stats, void *stream) {
    if (!A || !weights || alpha < 2) {
        fm_set_error("fm_assign_solve: invalid argument (alpha must be >= 2)");
        return FM_INVALID_ARG;
    }
    FM_CHECK_CUDA(cudaSetDevice(A->device));
    A->stream = stream ? (cudaStream_t)stream : A->own_stream;
    const int rc = assign_solve_device(A, weights, alpha, flags, objective_out, match_out, prices_out);
    if (stats) *stats = A->st;
    return rc;
}

extern "C" int fm_assign_solve_host(fm_assign *A, const int32_t *weights, int64_t alpha,
                                    int32_t flags, int64_t *objective_out, int32_t *match_out,
                                    int64_t *prices_out, fm_stats *stats) {
    if (!A || !weights || alpha < 2) {
        fm_set_error("fm_assign_solve_host: invalid argument (alpha must be >= 2)");
        return FM_INVALID_ARG;
    }
    FM_CHECK_CUDA(cudaSetDevice(A->device));
    A->stream = A->own_stream;
    const size_t bytes = sizeof(int32_t) * (size_t)A->n * A->n;
    if (!A->in_w) FM_CHECK_CUDA(cudaMalloc((void **)&A->in_w, bytes));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, A->stream);
    FM_CHECK_CUDA(cudaMemcpyAsync(A->in_w, weights, bytes, cudaMemcpyHostToDevice, A->stream));
    cudaEventRecord(b, A->stream);
    cudaEventSynchronize(b);
    float h2d = 0.f;
    cudaEventElapsedTime(&h2d, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const int rc = assign_solve_device(A, A->in_w, alpha, flags, objective_out, match_out, prices_out);
    A->st.ms_h2d = h2d;
    if (stats) *stats = A->st;
    return rc;
}

// ---- stepwise API (on_refine_end support): begin, one refine at a time, state export
extern "C" int fm_assign_begin(fm_assign *A, const int32_t *weights, int64_t alpha, int32_t flags) {
    if (!A || !weights || alpha < 2) {
        fm_set_error("fm_assign_begin: invalid argument (alpha must be >= 2)");
        return FM_INVALID_ARG;
    }
    FM_CHECK_CUDA(cudaSetDevice(A->device));
    A->stream = A->own_stream;
    const size_t bytes = sizeof(int32_t) * (size_t)A->n * A->n;
    if (!A->in_w) FM_CHECK_CUDA(cudaMalloc((void **)&A->in_w, bytes));
    FM_CHECK_CUDA(cudaMemcpyAsync(A->in_w, weights, bytes, cudaMemcpyHostToDevice, A->stream));
    return assign_setup(A, A->in_w, alpha, flags);
}

extern "C" int fm_assign_refine(fm_assign *A, int64_t *eps_out, int32_t *done_out) {
    if (!A) { fm_set_error("fm_assign_refine: null handle"); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(A->device));
    const int rc = assign_one_refine(A);
    if (eps_out) *eps_out = A->eps;
    if (done_out) *done_out = A->eps == 1;
    return rc;
}

// prices (2n: X then Y), match (n), fixed bitmask (n * ceil(n/32) words, row-major)
extern "C" int fm_assign_state(fm_assign *A, int64_t *prices, int32_t *match, uint32_t *fixed,
                               int64_t *objective_out, fm_stats *stats) {
    if (!A) { fm_set_error("fm_assign_state: null handle"); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(A->device));
    cudaStream_t s = A->stream;
    if (fixed) FM_CHECK_CUDA(cudaMemcpyAsync(fixed, A->d.fixed, sizeof(uint32_t) * (size_t)A->n * A->nw,
                                             cudaMemcpyDeviceToHost, s));
    FM_TRY(assign_finish(A, FM_OK, objective_out, match, prices));
    if (stats) *stats = A->st;
    return FM_OK;
}

// ---- stateful API: a reference ScalingState (assign_scaling.py:102-142) loaded onto the
// device, then begin_refine / refine_par rounds / price update / arc fixing as separate
// coordinator steps (refine_par, assign_par.py:115-237; min_cost_loop, :400-467).
namespace {

int assign_sync_cnt(fm_assign *A) {
    FM_CHECK_CUDA(cudaMemcpyAsync(A->h_cnt, A->d.cnt, sizeof(int32_t) * C_COUNT, cudaMemcpyDeviceToHost, A->stream));
    FM_CHECK_CUDA(cudaStreamSynchronize(A->stream));
    return FM_OK;
}

int assign_ops(fm_assign *A, unsigned long long *out16) {
    FM_CHECK_CUDA(cudaMemcpyAsync(A->h_ops, A->d.ops, sizeof(unsigned long long) * O_COUNT, cudaMemcpyDeviceToHost,
                                  A->stream));
    FM_CHECK_CUDA(cudaStreamSynchronize(A->stream));
    memcpy(out16, A->h_ops, sizeof(unsigned long long) * 16);
    return FM_OK;
}

}  // namespace

extern "C" int fm_assign_load(fm_assign *A, const int32_t *weights, int64_t alpha, int32_t flags, int64_t eps,
                              int64_t scale, int64_t bound, const int64_t *prices, const int32_t *match,
                              const uint32_t *fixed) {
    if (!A || alpha < 2 || eps < 1 || !prices || !match || !fixed) {
        fm_set_error("fm_assign_load: invalid argument");
        return FM_INVALID_ARG;
    }
    FM_CHECK_CUDA(cudaSetDevice(A->device));
    A->stream = A->own_stream;
    const int n = A->n;
    for (int x = 0; x < n; x++)
        if (match[x] < -1 || match[x] >= n) {
            fm_set_error("fm_assign_load: match[%d] = %d out of range", x, match[x]);
            return FM_INVALID_ARG;
        }
    const size_t bytes = sizeof(int32_t) * (size_t)n * n;
    if (!A->in_w) {
        if (!weights) { fm_set_error("fm_assign_load: no weight matrix loaded yet"); return FM_INVALID_ARG; }
        FM_CHECK_CUDA(cudaMalloc((void **)&A->in_w, bytes));
    }
    cudaStream_t s = A->stream;
    if (weights) FM_CHECK_CUDA(cudaMemcpyAsync(A->in_w, weights, bytes, cudaMemcpyHostToDevice, s));
    FM_TRY(assign_setup(A, A->in_w, alpha, flags));
    AssignDev &d = A->d;
    // arc cost c(x, y) = -scale * w(x, y): scale n + 1 for reduce_to_mincost networks,
    // 1 for a caller-built network whose costs are not multiples of n + 1
    if (scale > 0) {
        A->bound = A->bound / ((long long)n + 1) * scale;
        d.scale = scale;
    }
    if (bound >= 0) A->bound = bound;   // the state's scaled_cost_bound
    FM_CHECK_CUDA(cudaMemcpyAsync(d.px, prices, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    FM_CHECK_CUDA(cudaMemcpyAsync(d.py, prices + n, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    FM_CHECK_CUDA(cudaMemcpyAsync(d.match, match, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    FM_CHECK_CUDA(cudaMemcpyAsync(d.fixed, fixed, sizeof(uint32_t) * (size_t)n * d.nw, cudaMemcpyHostToDevice, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.ey, 0xff, sizeof(int32_t) * n, s));   // supplies: -1 per Y
    load_state_kernel<<<std::max(1, std::min((n + 255) / 256, A->sms * 2)), 256, 0, s>>>(d);
    FM_CHECK_LAUNCH();
    bit_transpose_kernel<<<std::max(1, std::min((d.nw * d.nw + 7) / 8, A->sms * 8)), 256, 0, s>>>(
        d.fixed, d.fixed_t, n, d.nw);
    FM_CHECK_LAUNCH();
    A->st.launches += 2;
    A->eps = eps;
    d.eps = eps;
    d.max_bucket = std::min<long long>(A->bound / eps + 2, LINF - 1);
    FM_CHECK_CUDA(cudaStreamSynchronize(s));
    return FM_OK;
}

extern "C" int fm_assign_begin_refine(fm_assign *A, int64_t *eps_out) {
    if (!A || !A->in_w) { fm_set_error("fm_assign_begin_refine: no state loaded"); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(A->device));
    const int n = A->n;
    AssignDev &d = A->d;
    cudaStream_t s = A->stream;
    A->eps = std::max(1LL, (A->eps + A->alpha - 1) / A->alpha);   // -(-eps // alpha)
    d.eps = A->eps;
    d.max_bucket = std::min<long long>(A->bound / A->eps + 2, LINF - 1);
    FM_CHECK_CUDA(cudaMemsetAsync(d.cnt, 0, sizeof(int32_t) * C_COUNT, s));
    reset_excess_kernel<<<(n + 255) / 256, 256, 0, s>>>(d);
    FM_CHECK_LAUNCH();
    begin_refine_kernel<<<std::max(1, std::min((n + AWARPS - 1) / AWARPS, A->sms * 4)), ATHREADS, 0, s>>>(d, 0);
    FM_CHECK_LAUNCH();
    A->st.launches += 2;
    FM_CHECK_CUDA(cudaStreamSynchronize(s));
    if (eps_out) *eps_out = A->eps;
    return FM_OK;
}

// One coordinator round of refine_par: every active X gets an op, then up to
// cycle_budget Y/X phase pairs (with price updates when the relabel budget asks; the
// every-k schedule is the caller's, at coordinator points).
// out = {pushes, relabels, rounds, active nodes left}.
extern "C" int fm_assign_round(fm_assign *A, int32_t cycle_budget, int64_t *out) {
    if (!A || !A->in_w || cycle_budget < 1 || !out) {
        fm_set_error("fm_assign_round: invalid argument or no state loaded");
        return FM_INVALID_ARG;
    }
    FM_CHECK_CUDA(cudaSetDevice(A->device));
    const int n = A->n;
    AssignDev &d = A->d;
    cudaStream_t s = A->stream;
    unsigned long long o0[16], o1[16];
    FM_TRY(assign_ops(A, o0));
    FM_CHECK_CUDA(cudaMemsetAsync(d.cnt, 0, sizeof(int32_t) * C_COUNT, s));
    active_lists_kernel<<<std::max(1, std::min((n + 255) / 256, A->sms * 2)), 256, 0, s>>>(d);
    FM_CHECK_LAUNCH();
    d.vbase += 1 << 21;
    x_phase_kernel<<<std::max(1, std::min((n + AWARPS - 1) / AWARPS, A->sms * 4)), ATHREADS, 0, s>>>(d, d.vbase);
    FM_CHECK_LAUNCH();
    FM_CHECK_CUDA(cudaMemsetAsync(d.cnt + C_X0, 0, sizeof(int32_t), s));
    A->st.launches += 2;
    FM_TRY(assign_sync_cnt(A));
    int rc = assign_status(A->h_cnt[C_INFEASIBLE]);
    while (rc == FM_OK) {
        const int done = A->h_cnt[C_ROUND];
        int cap = cycle_budget - done;
        if (cap <= 0) break;
        d.vbase += 1 << 21;
        int every_k = 0, gated = 0;
        void *args[] = {(void *)&d, (void *)&A->tail_threshold, (void *)&A->round_budget, (void *)&A->pu_threshold,
                        (void *)&cap, (void *)&every_k, (void *)&gated};
        FM_CHECK_CUDA(cudaLaunchCooperativeKernel((void *)refine_rounds_kernel, dim3(A->opt_round_ctas > 0 ? std::min(A->opt_round_ctas, A->coop_blocks) : A->coop_blocks),
                                                  dim3(ATHREADS), args, 0, s));
        A->st.launches++;
        FM_TRY(assign_sync_cnt(A));
        rc = assign_status(A->h_cnt[C_INFEASIBLE]);
        if (rc != FM_OK || A->h_cnt[C_EXIT] != 1) break;
        FM_CHECK_CUDA(launch_price_update(A));
        A->st.launches++;
        FM_TRY(assign_sync_cnt(A));
        rc = assign_status(A->h_cnt[C_INFEASIBLE]);
    }
    FM_TRY(assign_ops(A, o1));
    const int r = A->h_cnt[C_ROUND];
    out[0] = (int64_t)(o1[O_PUSH] - o0[O_PUSH]);
    out[1] = (int64_t)(o1[O_RELABEL] - o0[O_RELABEL]);
    out[2] = r;
    out[3] = A->h_cnt[C_Y0 + (r & 1)];
    return rc;
}

// price_update_heuristic (assign_scaling.py:208-276) at a coordinator point; a no-op
// without active nodes (then there are no deficit nodes either: excesses sum to 0)
extern "C" int fm_assign_price_update(fm_assign *A) {
    if (!A || !A->in_w) { fm_set_error("fm_assign_price_update: no state loaded"); return FM_INVALID_ARG; }
    if (!(A->flags & FM_ASSIGN_PRICE_UPDATE)) {
        fm_set_error("fm_assign_price_update: state loaded without FM_ASSIGN_PRICE_UPDATE");
        return FM_INVALID_ARG;
    }
    FM_CHECK_CUDA(cudaSetDevice(A->device));
    const int n = A->n;
    AssignDev &d = A->d;
    cudaStream_t s = A->stream;
    FM_CHECK_CUDA(cudaMemsetAsync(d.cnt, 0, sizeof(int32_t) * C_COUNT, s));
    active_lists_kernel<<<std::max(1, std::min((n + 255) / 256, A->sms * 2)), 256, 0, s>>>(d);
    FM_CHECK_LAUNCH();
    A->st.launches++;
    FM_TRY(assign_sync_cnt(A));
    if (A->h_cnt[C_X0] + A->h_cnt[C_Y0] == 0) return FM_OK;
    FM_CHECK_CUDA(launch_price_update(A));
    A->st.launches++;
    FM_TRY(assign_sync_cnt(A));
    return assign_status(A->h_cnt[C_INFEASIBLE]);
}

extern "C" int fm_assign_arc_fix(fm_assign *A, int64_t *fixed_pairs) {
    if (!A || !A->in_w) { fm_set_error("fm_assign_arc_fix: no state loaded"); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(A->device));
    const int n = A->n;
    AssignDev &d = A->d;
    cudaStream_t s = A->stream;
    unsigned long long o0[16], o1[16];
    FM_TRY(assign_ops(A, o0));
    const int use_fix = d.use_fix;
    d.use_fix = 1;
    arc_fix_kernel<<<std::max(1, std::min((n + 7) / 8, A->sms * 8)), 256, 0, s>>>(d);
    FM_CHECK_LAUNCH();
    d.use_fix = use_fix;
    bit_transpose_kernel<<<std::max(1, std::min((d.nw * d.nw + 7) / 8, A->sms * 8)), 256, 0, s>>>(
        d.fixed, d.fixed_t, n, d.nw);
    FM_CHECK_LAUNCH();
    A->st.launches += 2;
    FM_TRY(assign_ops(A, o1));
    if (fixed_pairs) *fixed_pairs = (int64_t)(o1[O_FIXED] - o0[O_FIXED]);
    return FM_OK;
}

// current state to HOST buffers (any may be NULL): prices 2n (X then Y), match n,
// fixed n * ceil(n/32) words, Y excess n, epsilon
extern "C" int fm_assign_export(fm_assign *A, int64_t *prices, int32_t *match, uint32_t *fixed, int32_t *ey,
                                int64_t *eps_out) {
    if (!A || !A->in_w) { fm_set_error("fm_assign_export: no state loaded"); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(A->device));
    const int n = A->n;
    AssignDev &d = A->d;
    cudaStream_t s = A->stream;
    if (prices) {
        FM_CHECK_CUDA(cudaMemcpyAsync(prices, d.px, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
        FM_CHECK_CUDA(cudaMemcpyAsync(prices + n, d.py, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
    }
    if (match) FM_CHECK_CUDA(cudaMemcpyAsync(match, d.match, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    if (fixed) FM_CHECK_CUDA(cudaMemcpyAsync(fixed, d.fixed, sizeof(uint32_t) * (size_t)n * d.nw,
                                             cudaMemcpyDeviceToHost, s));
    if (ey) FM_CHECK_CUDA(cudaMemcpyAsync(ey, d.ey, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    FM_CHECK_CUDA(cudaStreamSynchronize(s));
    if (eps_out) *eps_out = A->eps;
    return FM_OK;
}

// Options (replace the round-1 environment knobs); take effect at the next solve /
// load.  heuristic_every_k: a price update every k refine rounds (assign_par.py:228-234).
extern "C" int fm_assign_set_option(fm_assign *A, const char *name, int64_t value) {
    if (!A || !name) { fm_set_error("fm_assign_set_option: invalid argument"); return FM_INVALID_ARG; }
    const int v = (int)std::max<int64_t>(INT32_MIN, std::min<int64_t>(INT32_MAX, value));
    if (!strcmp(name, "heuristic_every_k")) A->pu_every_k = std::max(0, v);
    else if (!strcmp(name, "ybatch_min")) A->opt_ybatch_min = std::max(1, v);
    else if (!strcmp(name, "cta_x")) A->opt_cta_x = std::max(1, v);
    else if (!strcmp(name, "pu_groups")) {
        if (v != 1 && v != 2 && v != 4 && v != 8) { fm_set_error("pu_groups must be 1, 2, 4 or 8"); return FM_INVALID_ARG; }
        A->opt_pu_groups = v;
    }
    else if (!strcmp(name, "cta_y")) A->opt_cta_y = std::max(1, v);
    else if (!strcmp(name, "pu_ring")) A->opt_pu_ring = v;
    else if (!strcmp(name, "pu_local")) A->opt_pu_local = v;
    else if (!strcmp(name, "pu_filter")) A->opt_pu_filter = v;
    else if (!strcmp(name, "round_ctas")) A->opt_round_ctas = std::max(0, v);
    else if (!strcmp(name, "trace")) A->opt_trace = v;
    else if (!strcmp(name, "pu_threshold")) A->opt_pu_threshold = v;
    else if (!strcmp(name, "tail_threshold")) A->opt_tail_threshold = v;
    else if (!strcmp(name, "pu_cap")) A->opt_pu_cap = v;
    else { fm_set_error("fm_assign_set_option: unknown option '%s'", name); return FM_INVALID_ARG; }
    return FM_OK;
}

// Exact optimality certificate of a matching (CLI verify, tests): *certified = 1 when
// `match` is a perfect matching over present pairs with no negative residual cycle
// (proven maximum weight), 0 when a negative cycle exists, -1 when it is not a
// perfect matching.  weights HOST (copied in) or DEVICE (weights_on_device = 1);
// match HOST; prices HOST 2n (X then Y, any scale-s potentials, or NULL).
extern "C" int fm_assign_certify(fm_assign *A, const int32_t *weights, int32_t weights_on_device,
                                 const int32_t *match, const int64_t *prices, int64_t scale,
                                 int32_t *certified, int64_t *objective_out, int32_t *passes_out) {
    if (!A || !weights || !match || !certified) { fm_set_error("fm_assign_certify: invalid argument"); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(A->device));
    const int n = A->n;
    cudaStream_t s = A->own_stream;
    const size_t bytes = sizeof(int32_t) * (size_t)n * n;
    const int32_t *w = weights;
    if (!weights_on_device) {
        if (!A->in_w) FM_CHECK_CUDA(cudaMalloc((void **)&A->in_w, bytes));
        FM_CHECK_CUDA(cudaMemcpyAsync(A->in_w, weights, bytes, cudaMemcpyHostToDevice, s));
        w = A->in_w;
    }
    if (scale <= 0) scale = (int64_t)n + 1;
    // scratch: the price-update label arrays and frontier buffers are free between solves
    AssignDev &d = A->d;
    long long *dx = (long long *)d.px, *dy = (long long *)d.py;   // overwritten: state of the last solve is gone
    long long *ppx = nullptr, *ppy = nullptr;
    int32_t *m = d.match, *ycount = d.ey, *flags = d.cnt;
    long long *pbuf = nullptr;
    if (prices) {
        FM_CHECK_CUDA(cudaMalloc((void **)&pbuf, sizeof(long long) * 2 * (size_t)n));
        FM_CHECK_CUDA(cudaMemcpyAsync(pbuf, prices, sizeof(long long) * 2 * (size_t)n, cudaMemcpyHostToDevice, s));
        ppx = pbuf; ppy = pbuf + n;
    }
    FM_CHECK_CUDA(cudaMemcpyAsync(m, match, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
    FM_CHECK_CUDA(cudaMemsetAsync(ycount, 0, sizeof(int32_t) * n, s));
    FM_CHECK_CUDA(cudaMemsetAsync(flags, 0, sizeof(int32_t) * C_COUNT, s));
    FM_CHECK_CUDA(cudaMemsetAsync(A->acc, 0, sizeof(unsigned long long) * 4, s));
    const int gb = std::max(1, std::min((n + 255) / 256, A->sms * 2));
    certify_init_kernel<<<gb, 256, 0, s>>>(w, m, n, dx, dy, flags + 0, ycount);
    FM_CHECK_LAUNCH();
    FM_CHECK_CUDA(cudaMemcpyAsync(A->h_cnt, flags, sizeof(int32_t) * C_COUNT, cudaMemcpyDeviceToHost, s));
    FM_CHECK_CUDA(cudaStreamSynchronize(s));
    int rc = FM_OK;
    *certified = -1;
    int passes = 0;
    if (!A->h_cnt[0]) {
        // every matched pair must be present
        objective_kernel<<<gb, 256, 0, s>>>(w, m, n, A->acc + 1);
        FM_CHECK_LAUNCH();
        const int fb = std::max(1, std::min((n + 7) / 8, A->sms * 8));
        bool converged = false;
        for (passes = 1; passes <= 2 * n + 2; passes++) {
            FM_CHECK_CUDA(cudaMemsetAsync(flags + 1, 0, sizeof(int32_t), s));
            certify_forward_kernel<<<fb, 256, 0, s>>>(w, m, ppx, ppy, scale, n, dx, dy, flags + 1);
            FM_CHECK_LAUNCH();
            certify_reverse_kernel<<<gb, 256, 0, s>>>(w, m, ppx, ppy, scale, n, dx, dy, flags + 1);
            FM_CHECK_LAUNCH();
            FM_CHECK_CUDA(cudaMemcpyAsync(A->h_cnt, flags, sizeof(int32_t) * C_COUNT, cudaMemcpyDeviceToHost, s));
            FM_CHECK_CUDA(cudaStreamSynchronize(s));
            if (!A->h_cnt[1]) { converged = true; break; }
        }
        *certified = converged ? 1 : 0;
        FM_CHECK_CUDA(cudaMemcpyAsync(A->h_acc, A->acc, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, s));
        FM_CHECK_CUDA(cudaStreamSynchronize(s));
        if (objective_out) *objective_out = (int64_t)A->h_acc[1];
    }
    if (pbuf) cudaFree(pbuf);
    if (passes_out) *passes_out = passes;
    return rc;
}

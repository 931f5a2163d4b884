// fm_assign_sparse.cu -- cost-scaling assignment on SPARSE instances (complete=False)
// in compressed sparse form: the same algorithm as fm_assign.cu (reduction to min-cost
// flow with costs -(n+1) w, integral epsilon schedule eps <- max(1, ceil(eps/alpha))
// down to 1, refine as bulk-synchronous lock-free push-relabel phases, Dial price
// update, arc fixing; assign_scaling.py:85-182,185-276,380-497, assign_par.py:45-237),
// with O(n + m) memory and O(degree) work per operation instead of the dense kernels'
// n x n matrix.
//
// Layout: arcs sorted by x (CSR: rp[n+1], col[m], w[m], in input order within a row --
// the reference's out-arc order), and a y-major index over them (CSC: cp[n+1], ca[m] =
// the CSR arc of each column entry).  X flow is one matched arc per x (mat[x], -1 = x
// holds its unit); y excess = (#matched into y) - 1.  Phases as the dense path: an X
// phase reads only Y prices, a Y phase only prices of X matched into it, so every op
// sees exact prices and epsilon-optimality is kept exactly.  The rounds of a refine run
// inside one cooperative kernel (grid barriers between phases; once the Y list is short
// CTA 0 finishes alone with CTA barriers), and a price update is one cooperative kernel
// too (a grid barrier per Bellman-Ford wave): the host syncs once per refine and once
// per price update (sparse instances are the large-n, low-degree case the dense
// kernels' n-wide row scans do not fit).
#include <cooperative_groups.h>
#include <algorithm>
#include <climits>
#include <vector>
#include <string.h>

#include "fm_common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr long long SP_I64_MAX = 0x7fffffffffffffffLL;
constexpr int SP_LINF = 0x3fffffff;
constexpr int SP_YCAP = 256;          // Y-op candidates kept in shared memory per warp

struct SpDev {
    int32_t n;
    int64_t m;
    const int64_t *rp, *cp;           // CSR / CSC offsets (n + 1)
    const int32_t *col, *w, *cx, *ca; // CSR column + weight; CSC row (x) + CSR arc index
    uint8_t *fixed;                   // per CSR arc: frozen by arc fixing
    int64_t *px, *py;
    int32_t *mat;                     // matched CSR arc of x, -1 = x holds its unit
    int32_t *ey;                      // excess of y
    uint8_t *frozen;                  // x's matched arc is fixed
    int32_t *frozen_in;               // frozen matches into y
    int32_t *lx, *ly, *infy;          // price update labels / frontier flag
    int32_t *list[4];                 // X lists [0,1], Y lists [2,3] (round parity); frontiers reuse 2, 3
    int32_t *cnt;                     // [0..3] list counts, [4] infeasible, [5] relabels since PU,
                                      // [6] price update: changed, [7] last label, [8] round index,
                                      // [9] rounds kernel exit (0 done, 1 price update due), [12..14]
                                      // price-update frontier counts (rotating)
    unsigned long long *ops;          // [0] pushes [1] relabels [2] rounds [3] fixed [4] PU [5] PU waves
    int64_t scale, eps, max_bucket;
};

__device__ __forceinline__ void sp_argmin(long long &v, int &i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (ov < v || (ov == v && oi < i)) { v = ov; i = oi; }
    }
}

// min over x's present, non-fixed arcs of the part-reduced cost c - p(y) (first arc in
// row order wins ties, assign_par.py:84-90); warp-wide, result in every lane
__device__ __forceinline__ void sp_row_min(const SpDev &s, int x, int lane, long long &best, int &arc) {
    best = SP_I64_MAX;
    arc = INT32_MAX;
    for (int64_t a = s.rp[x] + lane; a < s.rp[x + 1]; a += 32) {
        if (s.fixed[a]) continue;
        const long long v = -(long long)s.w[a] * s.scale - __ldcg((const long long *)s.py + s.col[a]);
        if (v < best || (v == best && (int)a < arc)) { best = v; arc = (int)a; }
    }
    sp_argmin(best, arc);
}

__global__ void sp_bound_kernel(SpDev s, unsigned long long *out) {
    unsigned long long mx = 0;
    for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < s.m; a += (int64_t)gridDim.x * blockDim.x) {
        const long long v = s.w[a];
        mx = max(mx, (unsigned long long)(v < 0 ? -v : v));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

// begin_refine (assign_scaling.py:145-182) + the first X phase: unfrozen flow dropped,
// y excess = supplies + frozen flows, p(x) = -(min part-reduced cost + eps), x's unit
// pushed on that (admissible) arc
__global__ void sp_reset_kernel(SpDev s) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < s.n; v += gridDim.x * blockDim.x) {
        s.ey[v] = -1 + s.frozen_in[v];
        if (!s.frozen[v]) s.mat[v] = -1;
    }
}

__global__ void sp_begin_kernel(SpDev s) {
    const int lane = threadIdx.x & 31;
    unsigned long long pushes = 0;
    for (int x = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < s.n; x += (gridDim.x * blockDim.x) >> 5) {
        long long best;
        int arc;
        sp_row_min(s, x, lane, best, arc);
        if (lane == 0) {
            if (arc != INT32_MAX) s.px[x] = -(best + s.eps);
            if (!s.frozen[x]) {
                if (arc == INT32_MAX) {
                    atomicExch(s.cnt + 4, 1);
                } else {
                    s.mat[x] = arc;
                    pushes++;
                    const int y = s.col[arc];
                    if (atomicAdd(s.ey + y, 1) == 0) s.list[2][atomicAdd(s.cnt + 2, 1)] = y;
                }
            }
        }
    }
    if (lane == 0 && pushes) atomicAdd(s.ops + 0, pushes);
}

// Y op: y holding excess pushes its units back to the cheapest incoming matched,
// unfrozen x (reverse arc cost +w scale - p(x); (v, x) order), relabelling y whenever
// the next one is not admissible (assign_par.py:45-112).  One warp; sv / sx / sn are the
// warp's shared candidate buffer.
__device__ __forceinline__ void sp_y_op(const SpDev &s, int y, int32_t *xl_next, int32_t *xcnt_next, long long *sv,
                                        int *sx, int *sn, unsigned long long &pushes, unsigned long long &relabels) {
    const int lane = threadIdx.x & 31;
    int ey = __ldcg(s.ey + y);
    long long py = __ldcg((const long long *)s.py + y);
    if (ey <= 0) return;
    if (lane == 0) *sn = 0;
    __syncwarp();
    // gather: the column of y, arcs carrying a matched, unfrozen x's unit
    for (int64_t k = s.cp[y] + lane; k < s.cp[y + 1]; k += 32) {
        const int a = s.ca[k], x = s.cx[k];
        if (__ldcg(s.mat + x) != a || s.frozen[x]) continue;
        const int j = atomicAdd(sn, 1);
        if (j < SP_YCAP) { sx[j] = x; sv[j] = (long long)s.w[a] * s.scale - __ldcg((const long long *)s.px + x); }
    }
    __syncwarp();
    const int cnt = *(volatile int *)sn;
    if (cnt > SP_YCAP) {
        // overflow: one column scan per unit
        while (ey > 0) {
            long long bv = SP_I64_MAX;
            int bx = INT32_MAX;
            for (int64_t k = s.cp[y] + lane; k < s.cp[y + 1]; k += 32) {
                const int a = s.ca[k], x = s.cx[k];
                if (__ldcg(s.mat + x) != a || s.frozen[x]) continue;
                const long long v = (long long)s.w[a] * s.scale - __ldcg((const long long *)s.px + x);
                if (v < bv || (v == bv && x < bx)) { bv = v; bx = x; }
            }
            sp_argmin(bv, bx);
            if (bx == INT32_MAX) { if (lane == 0) atomicExch(s.cnt + 4, 2); break; }
            if (lane == 0) {
                if (!(bv < -py)) { py = -(bv + s.eps); relabels++; atomicAdd(s.cnt + 5, 1); }
                s.mat[bx] = -1;
                xl_next[atomicAdd(xcnt_next, 1)] = bx;
                pushes++;
            }
            __syncwarp();
            ey--;
        }
    } else {
        while (ey > 0) {
            long long bv = SP_I64_MAX;
            int bx = INT32_MAX, bk = -1;
            for (int k = lane; k < cnt; k += 32) {
                const long long v = sv[k];
                const int x = sx[k];
                if (v < bv || (v == bv && x < bx)) { bv = v; bx = x; bk = k; }
            }
            long long v2 = bv;
            int x2 = bx;
            sp_argmin(v2, x2);
            if (x2 == INT32_MAX) { if (lane == 0) atomicExch(s.cnt + 4, 2); break; }
            if (bx == x2 && bk >= 0) sv[bk] = SP_I64_MAX;   // the owner lane retires the slot
            if (lane == 0) {
                if (!(v2 < -py)) { py = -(v2 + s.eps); relabels++; atomicAdd(s.cnt + 5, 1); }
                s.mat[x2] = -1;
                xl_next[atomicAdd(xcnt_next, 1)] = x2;
                pushes++;
            }
            __syncwarp();
            ey--;
        }
    }
    if (lane == 0) { s.py[y] = py; s.ey[y] = ey; }
    __syncwarp();
}

// X op: x holding its unit relabels if its cheapest arc is not admissible and pushes
// the unit on it.  One warp.
__device__ __forceinline__ void sp_x_op(const SpDev &s, int x, int32_t *yl_next, int32_t *ycnt_next,
                                        unsigned long long &pushes, unsigned long long &relabels) {
    const int lane = threadIdx.x & 31;
    long long best;
    int arc;
    sp_row_min(s, x, lane, best, arc);
    if (lane == 0) {
        if (arc == INT32_MAX) {
            atomicExch(s.cnt + 4, 1);
        } else {
            const long long px = __ldcg((const long long *)s.px + x);
            if (!(best < -px)) { s.px[x] = -(best + s.eps); relabels++; atomicAdd(s.cnt + 5, 1); }
            s.mat[x] = arc;
            pushes++;
            const int y = s.col[arc];
            if (atomicAdd(s.ey + y, 1) == 0) yl_next[atomicAdd(ycnt_next, 1)] = y;
        }
    }
    __syncwarp();
}

constexpr int SP_THREADS = 256, SP_WARPS = SP_THREADS / 32;

// control words read right after a barrier: thread 0 loads them, the CTA shares them
__device__ __forceinline__ void sp_bcast(const int32_t *a, const int32_t *b, const int32_t *c, int &va, int &vb,
                                         int &vc) {
    __shared__ int sh[3];
    __syncthreads();
    if (threadIdx.x == 0) {
        sh[0] = __ldcg(a);
        sh[1] = b ? __ldcg(b) : 0;
        sh[2] = c ? __ldcg(c) : 0;
    }
    __syncthreads();
    va = sh[0]; vb = sh[1]; vc = sh[2];
}

// The refine's rounds as one cooperative kernel (refine_par's coordinator loop,
// assign_par.py:162-236).  Round r (b = r & 1): Y phase over ylist[b] -> xlist[b];
// barrier; X phase over xlist[b] -> ylist[b ^ 1]; barrier.  Exits when no Y holds
// excess (cnt[9] = 0) or a price update is due (cnt[9] = 1); the round index persists
// in cnt[8].  Counters of the lists a round writes are zeroed one round ahead (their
// last readers finished before the previous round's closing barrier).  Once the Y
// list is no longer than tail_threshold the other CTAs leave and CTA 0 continues with
// CTA barriers.
__global__ void __launch_bounds__(SP_THREADS) sp_rounds_kernel(SpDev s, int pu_threshold, long long round_budget,
                                                              int tail_threshold) {
    cg::grid_group grid = cg::this_grid();
    __shared__ long long s_v[SP_WARPS][SP_YCAP];
    __shared__ int s_x[SP_WARPS][SP_YCAP];
    __shared__ int s_n[SP_WARPS];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long pushes = 0, relabels = 0, rounds = 0;
    bool tail = false;
    int r, u0, u1, u2;
    sp_bcast(s.cnt + 8, nullptr, nullptr, r, u0, u1);
    for (;; r++) {
        int infeasible, relabels_since;
        sp_bcast(s.cnt + 4, s.cnt + 5, nullptr, infeasible, relabels_since, u0);
        const int b = r & 1;
        int ny;
        sp_bcast(s.cnt + 2 + b, nullptr, nullptr, ny, u1, u2);
        if (ny == 0 || infeasible) {
            if (blockIdx.x == 0 && threadIdx.x == 0) s.cnt[9] = 0;
            break;
        }
        if (pu_threshold > 0 && relabels_since >= pu_threshold) {
            if (blockIdx.x == 0 && threadIdx.x == 0) s.cnt[9] = 1;
            break;
        }
        if (r >= round_budget) {   // prices diverge: no perfect matching (assign_par.py:221-226)
            if (blockIdx.x == 0 && threadIdx.x == 0) { atomicExch(s.cnt + 4, 1); s.cnt[9] = 0; }
            break;
        }
        if (!tail && ny <= tail_threshold) {
            tail = true;
            if (blockIdx.x != 0) break;
        }
        rounds++;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            s.cnt[0 + (b ^ 1)] = 0;   // X list of round r + 1
            s.cnt[2 + (b ^ 1)] = 0;   // Y list this round's X phase writes (last read in round r - 1)
        }
        const int gw = tail ? wid : (int)((blockIdx.x * SP_THREADS + threadIdx.x) >> 5);
        const int nw = tail ? SP_WARPS : (int)((gridDim.x * SP_THREADS) >> 5);
        for (int i = gw; i < ny; i += nw)
            sp_y_op(s, __ldcg(s.list[2 + b] + i), s.list[0 + b], s.cnt + 0 + b, s_v[wid], s_x[wid], &s_n[wid],
                    pushes, relabels);
        if (tail) { __threadfence_block(); __syncthreads(); } else grid.sync();
        int nx;
        sp_bcast(s.cnt + 0 + b, nullptr, nullptr, nx, u1, u2);
        for (int i = gw; i < nx; i += nw)
            sp_x_op(s, __ldcg(s.list[0 + b] + i), s.list[2 + (b ^ 1)], s.cnt + 2 + (b ^ 1), pushes, relabels);
        if (tail) { __threadfence_block(); __syncthreads(); } else grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) s.cnt[8] = r;   // the round index persists across launches
    if (lane == 0) {
        if (pushes) atomicAdd(s.ops + 0, pushes);
        if (relabels) atomicAdd(s.ops + 1, relabels);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && rounds) atomicAdd(s.ops + 2, rounds);
}

// floor(rc / eps) for eps >= 1
__device__ __forceinline__ long long sp_floordiv(long long rc, long long eps) {
    long long q = rc / eps;
    if ((rc % eps != 0) && ((rc < 0) != (eps < 0))) q--;
    return q;
}

// price update (assign_scaling.py:208-276) as one cooperative kernel: labels =
// distances to the deficit set over reverse residual arcs, arc length floor(c_p / eps)
// + 1 >= 0, explored in frontier waves (grid barrier per wave) up to a label cap that
// widens x8 while an active node is unlabelled; then prices fall by eps min(label,
// last + 1), last = the largest label of an active node.  Frontiers live in list[2],
// list[3]; frontier counts rotate over cnt[12..14] so the next-but-one count is zeroed
// during a wave.
__global__ void __launch_bounds__(SP_THREADS) sp_pu_kernel(SpDev s) {
    cg::grid_group grid = cg::this_grid();
    const int tid = blockIdx.x * SP_THREADS + threadIdx.x, nthr = gridDim.x * SP_THREADS;
    const int lane = threadIdx.x & 31;
    const int gw = tid >> 5, nw = nthr >> 5;
    long long cap = min((long long)s.max_bucket, 8LL);
    unsigned long long waves = 0;
    for (;;) {
        if (tid == 0) { s.cnt[6] = 0; s.cnt[7] = 0; s.cnt[12] = 0; s.cnt[13] = 0; s.cnt[14] = 0; }
        grid.sync();
        for (int v = tid; v < s.n; v += nthr) {
            s.lx[v] = SP_LINF;
            if (s.ey[v] < 0) { s.ly[v] = 0; s.infy[v] = 1; s.list[2][atomicAdd(s.cnt + 12, 1)] = v; }
            else { s.ly[v] = SP_LINF; s.infy[v] = 0; }
        }
        grid.sync();
        for (int it = 0;; it++) {
            int nf, u1, u2;
            sp_bcast(s.cnt + 12 + it % 3, nullptr, nullptr, nf, u1, u2);
            if (nf == 0) break;
            waves++;
            if (tid == 0) s.cnt[12 + (it + 2) % 3] = 0;
            const int32_t *fr = s.list[2 + (it & 1)];
            int32_t *fr_next = s.list[2 + ((it + 1) & 1)];
            int32_t *fcnt_next = s.cnt + 12 + (it + 1) % 3;
            for (int i = gw; i < nf; i += nw) {
                const int y = __ldcg(fr + i);
                if (lane == 0) s.infy[y] = 0;
                __syncwarp();
                __threadfence();   // clear the flag before reading l(y): a later drop re-queues y
                const int lyv = __ldcg(s.ly + y);
                const long long pyv = __ldcg((const long long *)s.py + y);
                for (int64_t k = s.cp[y] + lane; k < s.cp[y + 1]; k += 32) {
                    const int a = s.ca[k], x = s.cx[k];
                    if (s.fixed[a] || __ldcg(s.mat + x) == a) continue;      // fixed / flow arc
                    const long long rc = -(long long)s.w[a] * s.scale + __ldcg((const long long *)s.px + x) - pyv;
                    long long len = sp_floordiv(rc, s.eps) + 1;
                    if (len < 0) len = 0;
                    const long long c1 = (long long)lyv + len;
                    if (c1 > cap || c1 >= __ldcg(s.lx + x)) continue;
                    const int old = atomicMin(s.lx + x, (int)c1);
                    if ((int)c1 >= old) continue;
                    const int ma = __ldcg(s.mat + x);
                    if (ma < 0 || s.frozen[x]) continue;
                    const int y2 = s.col[ma];
                    const long long rc2 = (long long)s.w[ma] * s.scale - __ldcg((const long long *)s.px + x) +
                                          __ldcg((const long long *)s.py + y2);
                    long long len2 = sp_floordiv(rc2, s.eps) + 1;
                    if (len2 < 0) len2 = 0;
                    const long long c2 = c1 + len2;
                    if (c2 > cap) continue;
                    if ((int)c2 < atomicMin(s.ly + y2, (int)c2) && atomicExch(s.infy + y2, 1) == 0)
                        fr_next[atomicAdd(fcnt_next, 1)] = y2;
                }
            }
            grid.sync();
        }
        // last = max label over active nodes; a missing one asks for a wider cap
        int last = 0, missing = 0;
        for (int v = tid; v < s.n; v += nthr) {
            if (__ldcg(s.mat + v) < 0 && !s.frozen[v]) { const int l = __ldcg(s.lx + v); if (l >= SP_LINF) missing = 1; else last = max(last, l); }
            if (__ldcg(s.ey + v) > 0) { const int l = __ldcg(s.ly + v); if (l >= SP_LINF) missing = 1; else last = max(last, l); }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
            missing |= __shfl_xor_sync(0xffffffffu, missing, o);
        }
        if (lane == 0) {
            if (last) atomicMax(s.cnt + 7, last);
            if (missing) atomicOr(s.cnt + 6, 1);
        }
        grid.sync();
        int chg, lst, u2;
        sp_bcast(s.cnt + 6, s.cnt + 7, nullptr, chg, lst, u2);
        if (!chg || cap >= s.max_bucket) {
            const long long K = min((long long)lst, (long long)s.max_bucket) + 1;
            for (int v = tid; v < s.n; v += nthr) {
                s.px[v] -= s.eps * min((long long)s.lx[v], K);
                s.py[v] -= s.eps * min((long long)s.ly[v], K);
            }
            break;
        }
        cap = min(cap * 8, (long long)s.max_bucket);
        grid.sync();
    }
    if (tid == 0) {
        s.cnt[5] = 0;   // relabels since the last price update
        atomicAdd(s.ops + 4, 1ull);
        atomicAdd(s.ops + 5, waves);
    }
}

// arc_fix (assign_scaling.py:185-205): freeze an arc whose reduced cost magnitude
// exceeds 2 n eps; a matched arc that freezes pins x to y for good
__global__ void sp_fix_kernel(SpDev s) {
    const long long thr = 2LL * s.n * s.eps;
    unsigned long long cnt = 0;
    for (int x = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; x < s.n; x += (gridDim.x * blockDim.x) >> 5) {
        const long long px = s.px[x];
        const int ma = s.mat[x];
        for (int64_t a = s.rp[x] + (threadIdx.x & 31); a < s.rp[x + 1]; a += 32) {
            if (s.fixed[a]) continue;
            const long long rc = -(long long)s.w[a] * s.scale + px - s.py[s.col[a]];
            if (rc > thr || -rc > thr) {
                s.fixed[a] = 1;
                cnt++;
                if ((int)a == ma) { s.frozen[x] = 1; atomicAdd(s.frozen_in + s.col[a], 1); }
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(s.ops + 3, cnt);
}

__global__ void sp_objective_kernel(SpDev s, unsigned long long *out) {
    long long t = 0;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < s.n; x += gridDim.x * blockDim.x)
        if (s.mat[x] >= 0) t += s.w[s.mat[x]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0 && t) atomicAdd(out, (unsigned long long)t);
}

__global__ void sp_match_y_kernel(SpDev s, int32_t *out) {
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < s.n; x += gridDim.x * blockDim.x)
        out[x] = s.mat[x] >= 0 ? s.col[s.mat[x]] : -1;
}

struct SpHost {
    SpDev d{};
    void *mem = nullptr;
    cudaStream_t st = nullptr;
    int32_t *h = nullptr;           // pinned: cnt mirror (8) + scratch
    unsigned long long *hops = nullptr;
    unsigned long long *dacc = nullptr;
    ~SpHost() {
        if (mem) cudaFree(mem);
        if (h) cudaFreeHost(h);
        if (hops) cudaFreeHost(hops);
        if (st) cudaStreamDestroy(st);
    }
};

int sp_sync_cnt(SpHost &H) {
    FM_CHECK_CUDA(cudaMemcpyAsync(H.h, H.d.cnt, sizeof(int32_t) * 16, cudaMemcpyDeviceToHost, H.st));
    FM_CHECK_CUDA(cudaStreamSynchronize(H.st));
    return FM_OK;
}

}  // namespace

// Sparse max-weight perfect matching (solve_assignment on an instance with complete =
// False, assign_scaling.py:470-497, in compressed form).  HOST inputs: m arcs (xs[k],
// ys[k], ws[k]) in the instance's edge order (no duplicates; int32 weights).  Outputs:
// objective (host int64), match_out[x] = y (host), prices_out (host 2n, X then Y) or NULL.
// flags: FM_ASSIGN_PRICE_UPDATE / FM_ASSIGN_ARC_FIX.  Status 1 = no perfect matching.
extern "C" int fm_assign_sparse_solve(int32_t n, int64_t m, const int32_t *xs, const int32_t *ys, const int32_t *ws,
                                      int64_t alpha, int32_t flags, int32_t device, int64_t *objective_out,
                                      int32_t *match_out, int64_t *prices_out, fm_stats *stats) {
    if (n < 1 || m < 0 || (m && (!xs || !ys || !ws)) || alpha < 2 || m > (int64_t)INT32_MAX - 1) {
        fm_set_error("fm_assign_sparse_solve: invalid argument");
        return FM_INVALID_ARG;
    }
    int ndev = fm_device_count();
    if (ndev == 0) { fm_set_error("no CUDA device"); return FM_NO_DEVICE; }
    if (device < 0 || device >= ndev) { fm_set_error("device %d out of range", device); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(device));
    cudaGetLastError();   // a stale error of another caller's runtime call must not be reported as ours
    // CSR (stable by x: row order = edge order) and CSC over the CSR arcs, on the host
    std::vector<int64_t> rp(n + 1, 0), cp(n + 1, 0);
    for (int64_t k = 0; k < m; k++) {
        if (xs[k] < 0 || xs[k] >= n || ys[k] < 0 || ys[k] >= n) { fm_set_error("arc endpoint out of range"); return FM_INVALID_ARG; }
        rp[xs[k] + 1]++;
        cp[ys[k] + 1]++;
    }
    for (int v = 0; v < n; v++) {
        // a side node without arcs: no perfect matching (the budget would find it slowly)
        if (rp[v + 1] == 0 || cp[v + 1] == 0) {
            fm_set_error("instance admits no perfect matching (node %d of the %s side has no arc)", v,
                         rp[v + 1] == 0 ? "X" : "Y");
            return FM_INFEASIBLE;
        }
        rp[v + 1] += rp[v];
        cp[v + 1] += cp[v];
    }
    std::vector<int32_t> col(m), w(m), cx(m), ca(m);
    {
        std::vector<int64_t> pos(rp.begin(), rp.end() - 1);
        for (int64_t k = 0; k < m; k++) { const int64_t a = pos[xs[k]]++; col[a] = ys[k]; w[a] = ws[k]; }
        std::vector<int64_t> cpos(cp.begin(), cp.end() - 1);
        for (int x = 0; x < n; x++)
            for (int64_t a = rp[x]; a < rp[x + 1]; a++) { const int64_t k = cpos[col[a]]++; cx[k] = x; ca[k] = (int32_t)a; }
    }
    SpHost H;
    FM_CHECK_CUDA(cudaStreamCreateWithFlags(&H.st, cudaStreamNonBlocking));
    const size_t mm = (size_t)std::max<int64_t>(m, 1), nn = (size_t)n;
    // every carve below is rounded up to 16 bytes: 24 carves -> at most 24 * 15 bytes of padding
    const size_t bytes = 2 * 8 * (nn + 1) + 4 * 4 * mm + mm + 2 * 8 * nn + 4 * nn * 10 + nn + 64 * 4 + 16 * 8 + 16 + 24 * 16;
    FM_CHECK_CUDA(cudaMalloc(&H.mem, bytes));
    FM_CHECK_CUDA(cudaMallocHost((void **)&H.h, 64 * sizeof(int32_t)));
    FM_CHECK_CUDA(cudaMallocHost((void **)&H.hops, 16 * sizeof(unsigned long long)));
    char *p = (char *)H.mem;
    auto take = [&](size_t b) { char *q = p; p += (b + 15) / 16 * 16; return (void *)q; };
    SpDev &d = H.d;
    d.n = n; d.m = m;
    d.rp = (int64_t *)take(8 * (nn + 1)); d.cp = (int64_t *)take(8 * (nn + 1));
    d.col = (int32_t *)take(4 * mm); d.w = (int32_t *)take(4 * mm); d.cx = (int32_t *)take(4 * mm); d.ca = (int32_t *)take(4 * mm);
    d.fixed = (uint8_t *)take(mm);
    d.px = (int64_t *)take(8 * nn); d.py = (int64_t *)take(8 * nn);
    d.mat = (int32_t *)take(4 * nn); d.ey = (int32_t *)take(4 * nn); d.frozen_in = (int32_t *)take(4 * nn);
    d.lx = (int32_t *)take(4 * nn); d.ly = (int32_t *)take(4 * nn); d.infy = (int32_t *)take(4 * nn);
    for (int k = 0; k < 4; k++) d.list[k] = (int32_t *)take(4 * nn);
    d.frozen = (uint8_t *)take(nn);
    d.cnt = (int32_t *)take(64 * 4);
    d.ops = (unsigned long long *)take(16 * 8);
    H.dacc = (unsigned long long *)take(16);
    if ((size_t)(p - (char *)H.mem) > bytes) { fm_set_error("fm_assign_sparse_solve: workspace sizing"); return FM_CUDA_ERROR; }
    FM_CHECK_CUDA(cudaMemcpyAsync((void *)d.rp, rp.data(), 8 * (nn + 1), cudaMemcpyHostToDevice, H.st));
    FM_CHECK_CUDA(cudaMemcpyAsync((void *)d.cp, cp.data(), 8 * (nn + 1), cudaMemcpyHostToDevice, H.st));
    if (m) {
        FM_CHECK_CUDA(cudaMemcpyAsync((void *)d.col, col.data(), 4 * m, cudaMemcpyHostToDevice, H.st));
        FM_CHECK_CUDA(cudaMemcpyAsync((void *)d.w, w.data(), 4 * m, cudaMemcpyHostToDevice, H.st));
        FM_CHECK_CUDA(cudaMemcpyAsync((void *)d.cx, cx.data(), 4 * m, cudaMemcpyHostToDevice, H.st));
        FM_CHECK_CUDA(cudaMemcpyAsync((void *)d.ca, ca.data(), 4 * m, cudaMemcpyHostToDevice, H.st));
    }
    FM_CHECK_CUDA(cudaMemsetAsync(d.fixed, 0, mm, H.st));
    FM_CHECK_CUDA(cudaMemsetAsync(d.px, 0, 8 * nn, H.st));
    FM_CHECK_CUDA(cudaMemsetAsync(d.py, 0, 8 * nn, H.st));
    FM_CHECK_CUDA(cudaMemsetAsync(d.mat, 0xff, 4 * nn, H.st));
    FM_CHECK_CUDA(cudaMemsetAsync(d.frozen, 0, nn, H.st));
    FM_CHECK_CUDA(cudaMemsetAsync(d.frozen_in, 0, 4 * nn, H.st));
    FM_CHECK_CUDA(cudaMemsetAsync(d.ops, 0, 16 * 8, H.st));
    FM_CHECK_CUDA(cudaMemsetAsync(H.dacc, 0, 16, H.st));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int blocks = std::max(1, std::min((n + 255) / 256, sms * 8));
    fm_stats st{};
    cudaEvent_t e0, e1;
    FM_CHECK_CUDA(cudaEventCreate(&e0));
    FM_CHECK_CUDA(cudaEventCreate(&e1));
    FM_CHECK_CUDA(cudaEventRecord(e0, H.st));
    if (m) sp_bound_kernel<<<std::max(1, (int)std::min<int64_t>((m + 255) / 256, sms * 8)), 256, 0, H.st>>>(d, H.dacc);
    FM_CHECK_LAUNCH();
    unsigned long long wmax = 0;
    FM_CHECK_CUDA(cudaMemcpyAsync(&wmax, H.dacc, 8, cudaMemcpyDeviceToHost, H.st));
    FM_CHECK_CUDA(cudaStreamSynchronize(H.st));
    d.scale = (int64_t)n + 1;
    const long long bound = (long long)wmax * (long long)(n + 1);
    long long eps = std::max(1LL, bound);
    const bool use_pu = flags & FM_ASSIGN_PRICE_UPDATE, use_fix = flags & FM_ASSIGN_ARC_FIX;
    const int pu_threshold = std::max(64, n / 16);
    const int pu_arg = use_pu ? pu_threshold : 0;
    // _ops_budget (assign_scaling.py:374-377) = max(1e4, 40 n^2 m) operations; a round does >= 1
    const long long round_budget = (long long)std::min(9e18, std::max(1e4, 40.0 * n * (double)n * std::max<double>(1.0, (double)m)));
    const int tail_threshold = 2 * SP_WARPS;
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sp_rounds_kernel, SP_THREADS, 0);
    int occ2 = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, sp_pu_kernel, SP_THREADS, 0);
    const int coop_blocks = std::max(1, std::min({sms * std::max(1, std::min(occ, occ2)), (n + SP_WARPS - 1) / SP_WARPS,
                                                  sms * 4}));
    int rc = FM_OK;
    while (rc == FM_OK) {
        eps = std::max(1LL, (eps + alpha - 1) / alpha);
        d.eps = eps;
        d.max_bucket = std::min<long long>(bound / eps + 2, SP_LINF - 1);
        FM_CHECK_CUDA(cudaMemsetAsync(d.cnt, 0, sizeof(int32_t) * 16, H.st));
        sp_reset_kernel<<<blocks, 256, 0, H.st>>>(d);
        sp_begin_kernel<<<std::max(1, std::min((n + 7) / 8, sms * 8)), 256, 0, H.st>>>(d);
        FM_CHECK_LAUNCH();
        st.launches += 2;
        // rounds (one cooperative launch until done or a price update is due)
        for (;;) {
            void *args[] = {(void *)&d, (void *)&pu_arg, (void *)&round_budget, (void *)&tail_threshold};
            FM_CHECK_CUDA(cudaLaunchCooperativeKernel((void *)sp_rounds_kernel, dim3(coop_blocks), dim3(SP_THREADS),
                                                      args, 0, H.st));
            st.launches++;
            FM_TRY(sp_sync_cnt(H));
            if (H.h[4]) { rc = H.h[4] == 1 ? FM_INFEASIBLE : FM_CUDA_ERROR; break; }
            if (H.h[9] != 1) break;   // no Y holds excess: refine done
            // price update: the Y list moves to list[1] while list[2], list[3] hold frontiers,
            // then comes back to its slot (the round index keeps counting toward the budget)
            const int r = H.h[8], b = r & 1, ny = H.h[2 + b];
            FM_CHECK_CUDA(cudaMemcpyAsync(d.list[1], d.list[2 + b], sizeof(int32_t) * ny, cudaMemcpyDeviceToDevice, H.st));
            void *pargs[] = {(void *)&d};
            FM_CHECK_CUDA(cudaLaunchCooperativeKernel((void *)sp_pu_kernel, dim3(coop_blocks), dim3(SP_THREADS), pargs, 0,
                                                      H.st));
            st.launches++;
            st.reserved[1]++;
            FM_CHECK_CUDA(cudaMemcpyAsync(d.list[2 + b], d.list[1], sizeof(int32_t) * ny, cudaMemcpyDeviceToDevice, H.st));
            int32_t *c = H.h + 32;   // pinned staging (the copy runs after this loop iteration)
            for (int i = 0; i < 10; i++) c[i] = 0;
            c[2 + b] = ny;
            c[8] = r;
            FM_CHECK_CUDA(cudaMemcpyAsync(d.cnt, c, sizeof(int32_t) * 10, cudaMemcpyHostToDevice, H.st));
        }
        if (rc != FM_OK) break;
        if (use_fix) {
            sp_fix_kernel<<<std::max(1, std::min((n + 7) / 8, sms * 8)), 256, 0, H.st>>>(d);
            FM_CHECK_LAUNCH();
            st.launches++;
        }
        st.refines++;
        if (eps == 1) break;
    }
    if (rc == FM_INFEASIBLE) fm_set_error("instance admits no perfect matching (an active node has no residual arc, "
                                          "or the operation budget was exceeded)");
    else if (rc != FM_OK) fm_set_error("inconsistent Y excess during the sparse refine");
    if (rc == FM_OK) {
        FM_CHECK_CUDA(cudaMemsetAsync(H.dacc + 1, 0, 8, H.st));
        sp_objective_kernel<<<blocks, 256, 0, H.st>>>(d, H.dacc + 1);
        sp_match_y_kernel<<<blocks, 256, 0, H.st>>>(d, d.list[1]);
        FM_CHECK_LAUNCH();
        st.launches += 2;
        unsigned long long obj = 0;
        FM_CHECK_CUDA(cudaMemcpyAsync(&obj, H.dacc + 1, 8, cudaMemcpyDeviceToHost, H.st));
        if (match_out) FM_CHECK_CUDA(cudaMemcpyAsync(match_out, d.list[1], 4 * nn, cudaMemcpyDeviceToHost, H.st));
        if (prices_out) {
            FM_CHECK_CUDA(cudaMemcpyAsync(prices_out, d.px, 8 * nn, cudaMemcpyDeviceToHost, H.st));
            FM_CHECK_CUDA(cudaMemcpyAsync(prices_out + n, d.py, 8 * nn, cudaMemcpyDeviceToHost, H.st));
        }
        cudaEventRecord(e1, H.st);
        FM_CHECK_CUDA(cudaStreamSynchronize(H.st));
        if (objective_out) *objective_out = (int64_t)obj;
    } else {
        cudaEventRecord(e1, H.st);
        cudaStreamSynchronize(H.st);
    }
    FM_CHECK_CUDA(cudaMemcpy(H.hops, d.ops, 16 * 8, cudaMemcpyDeviceToHost));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    st.ms_total = ms;
    st.pushes = (int64_t)H.hops[0];
    st.relabels = (int64_t)H.hops[1];
    st.rounds = (int64_t)H.hops[2];
    st.reserved[2] = (int64_t)H.hops[5];   // price-update waves
    st.reserved[0] = (int64_t)H.hops[3];   // arcs fixed
    if (stats) *stats = st;
    return rc;
}

// fm_grid.cu -- B200-native lock-free push-relabel max-flow / min-cut on 4-connected grids.
//
// Replaces the reference's hybrid_solve (maxflow_par.py:157-238) for grid networks.
// Structure-of-arrays residual layout (one int32 plane per direction), Hong's
// lock-free push/relabel with int32 atomics (maxflow_par.py:65-129), device-side
// global relabel by tile-local multi-level relaxation + gap + marking
// (maxflow_seq.py:119-160, maxflow_par.py:220-226), and the minimal source-side
// cut by a seeded residual reach.  See DESIGN.md.
#include <algorithm>
#include <atomic>
#include <string>
#include <thread>
#include <vector>
#include <climits>
#include <cuda.h>   // CUtensorMap (TMA descriptors; encoded through the runtime's driver entry point)
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fm_common.cuh"

namespace {

constexpr int TILE_W = 32;           // tile width == warp width: one warp per tile row
constexpr int TILE_H = 32;           // rows per tile
constexpr int BLK_Y = 8;             // 32 x 8 = 256 threads per CTA; 4 rows per thread
constexpr int ROWS_PER_THREAD = TILE_H / BLK_Y;
constexpr int NWARPS = TILE_W * BLK_Y / 32;

// residual mask bits
constexpr uint8_t M_R = 1, M_L = 2, M_D = 4, M_U = 8, M_T = 16;

// Work list of tiles for persistent CTAs, double-buffered by launch parity p:
// launch p drains list[p] (clearing each tile's flag as it is taken) and fills
// list[p^1] (the flag dedups).  cnt = {count0, work1, count1, work0} so the two
// words a launch of parity p needs zeroed (count[p^1], work[p]) are adjacent.
struct TileQueue {
    int32_t *list[2];
    int32_t *flag[2];
    int32_t *cnt;
};

__device__ __forceinline__ void tq_push(const TileQueue &q, int parity, int tile) {
    if (atomicExch(q.flag[parity] + tile, 1) == 0) q.list[parity][atomicAdd(q.cnt + 2 * parity, 1)] = tile;
}

// next tile of launch parity p for this CTA (thread 0 calls; -1 when drained)
__device__ __forceinline__ int tq_take(const TileQueue &q, int parity, int all_tiles, int ntiles) {
    const int i = atomicAdd(q.cnt + (parity ? 1 : 3), 1);
    if (all_tiles) return i < ntiles ? i : -1;
    if (i >= __ldcg(q.cnt + 2 * parity)) return -1;
    const int t = __ldcg(q.list[parity] + i);
    q.flag[parity][t] = 0;
    return t;
}

// A neighbour band's planes as seen from this band (row-band mode, multi-GPU): device
// pointers valid on this band's device (peer access in one process, CUDA IPC across
// processes), pre-offset to the neighbour's boundary row (its last row for the band
// above, its first row for the band below).  res = the neighbour's residual toward us
// (rD of the row above / rU of the row below), read by the cut's incoming-arc planes.
struct PeerView {
    int32_t *h, *dist, *inbox, *res;
    uint8_t *cut;
    int32_t *ext;           // its external-push flags for the tiles of that boundary row
    int32_t *rq_slot, *rq_flag;
    unsigned int *rq_ctr;   // its ring queue (tail at [32])
    int32_t rq_cap;
    int32_t tile0;          // its tile index of the boundary tile row's first tile
};

struct GridDev {
    int32_t *e, *h, *rR, *rL, *rD, *rU, *rT, *rS, *cS;
    int32_t *dist;
    uint32_t *rbits;        // K2 bit planes: per tile, 5 x 32 words (R, L, D, U, T arcs; lane = row)
    uint8_t *mask, *marked, *cut;
    // tile-resident kernel (K1 v2): flow pushed across a tile border is parked in
    // an inbox of the receiving pixel (inflow_h: across a vertical tile border,
    // inflow_v: across a horizontal one) until the receiving tile next loads
    int32_t *inflow_h, *inflow_v;
    int32_t ntx, nty;       // tiles per row / column
    TileQueue pq;           // push-relabel work list
    TileQueue bq;           // BFS / cut frontier work list
    // row-band mode (multi-GPU): this handle holds rows [R0, R0 + H) of a
    // taller grid.  Arcs leaving the first / last row toward a neighbour band are real
    // arcs; the neighbour's halo rows, inboxes and queues are reached through up / dn.
    int32_t has_up, has_dn;
    int32_t hlim;           // H + has_dn: rows r with r + 1 < hlim have a pixel below
    int32_t rmin;           // -has_up: rows r with r > rmin have a pixel above
    PeerView up, dn;
    int32_t *ext;           // this band's external-push flags: [0, ntx) top tile row, [ntx, 2 ntx) bottom
    unsigned long long *ext_ctr;   // [0] flags this band raised on its neighbours, [1] own flags consumed
    // local relabel (tail rounds): tiles touched by pushes since the last relabel, and
    // the region R (touched tiles dilated by a margin) a local relabel recomputes;
    // region == nullptr means "global"
    uint8_t *touched;
    const uint8_t *region;
    int32_t H, W;
    int32_t V;      // node count |V| = H*W + 2 (the source's height)
    int32_t INF;    // "unreached" distance sentinel (== V)
    int32_t solo_max;   // push kernel: a pass listing <= solo_max pixels runs on warp 0 alone
    int32_t k_solo;     // push kernel: at most this many solo passes per visit (0: up to k_local)
};

// ----------------------------------------------------------------------------
// init: hybrid_init + init_preflow (maxflow_par.py:44-62, maxflow_seq.py:47-64).
// Saturating s->p gives e(p) = capS(p).  With precancel, min(capS, capT) is routed
// s->p->t immediately (value- and cut-preserving).
// ----------------------------------------------------------------------------
__global__ void grid_init_kernel(GridDev g, const int32_t *__restrict__ capR,
                                 const int32_t *__restrict__ capL,
                                 const int32_t *__restrict__ capD,
                                 const int32_t *__restrict__ capU,
                                 const int32_t *__restrict__ capS,
                                 const int32_t *__restrict__ capT,
                                 const int32_t *__restrict__ capD_above,   // band mode: capD of the row above (W)
                                 const int32_t *__restrict__ capU_below,   // band mode: capU of the row below (W)
                                 int precancel,
                                 unsigned long long *acc /* [0]=sum capS [1]=negative [2]=too large [3]=pair > 65535 */) {
    long long sum = 0, bad = 0, big = 0, wide = 0;
    // rows over blocks, columns over threads: coalesced, and no 64-bit division per pixel
    for (int32_t r = blockIdx.x; r < g.H; r += gridDim.x)
    for (int32_t c = threadIdx.x; c < g.W; c += blockDim.x) {
        const int64_t p = (int64_t)r * g.W + c;
        int32_t cs = capS[p], ct = capT[p];
        int32_t cr = c + 1 < g.W ? capR[p] : 0;
        int32_t cl = c > 0 ? capL[p] : 0;
        int32_t cd = r + 1 < g.hlim ? capD[p] : 0;
        int32_t cu = r > g.rmin ? capU[p] : 0;
        bad += (cs < 0) | (ct < 0) | (cr < 0) | (cl < 0) | (cd < 0) | (cu < 0);
        // int32 device state: the excess of p is at most capS + the capacities into p, and
        // a merged pair's residual at most the pair's two capacities (the reference's
        // Python ints have no such limit, so larger inputs are refused, not wrapped)
        const long long inR = c > 0 ? max(capR[p - 1], 0) : 0, inL = c + 1 < g.W ? max(capL[p + 1], 0) : 0;
        const long long inD = r > 0 ? max(capD[p - g.W], 0) : (g.has_up ? max(capD_above[c], 0) : 0);
        const long long inU = r + 1 < g.H ? max(capU[p + g.W], 0) : (g.has_dn ? max(capU_below[c], 0) : 0);
        big += ((long long)max(cs, 0) + inR + inL + inD + inU > (long long)INT32_MAX) |
               ((long long)max(cr, 0) + inL > (long long)INT32_MAX) | ((long long)max(cd, 0) + inU > (long long)INT32_MAX);
        // pairs too wide for the packed 16-bit residual fields of the push kernel
        wide += ((long long)max(cr, 0) + inL > 65535) | ((long long)max(cd, 0) + inU > 65535);
        cs = max(cs, 0); ct = max(ct, 0);
        const int32_t m = precancel ? min(cs, ct) : 0;
        g.e[p] = cs - m;
        g.rT[p] = ct - m;
        g.rS[p] = cs;
        g.cS[p] = cs;
        g.rR[p] = max(cr, 0);
        g.rL[p] = max(cl, 0);
        g.rD[p] = max(cd, 0);
        g.rU[p] = max(cu, 0);
        g.h[p] = 0;
        g.marked[p] = 0;
        g.inflow_h[p] = 0;
        g.inflow_v[p] = 0;
        sum += cs;
    }
    // grid-stride kernel with 1-D blocks of 256
    __shared__ long long red[4][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
        big += __shfl_xor_sync(0xffffffffu, big, o);
        wide += __shfl_xor_sync(0xffffffffu, wide, o);
    }
    if (lane == 0) { red[0][wid] = sum; red[1][wid] = bad; red[2][wid] = big; red[3][wid] = wide; }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long s = 0, b = 0, x = 0, w = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) { s += red[0][i]; b += red[1][i]; x += red[2][i]; w += red[3][i]; }
        if (s) atomicAdd(&acc[0], (unsigned long long)s);
        if (b) atomicAdd(&acc[1], (unsigned long long)b);
        if (x) atomicAdd(&acc[2], (unsigned long long)x);
        if (w) atomicAdd(&acc[3], (unsigned long long)w);
    }
}

// ----------------------------------------------------------------------------
// Two-hop pre-routing (after init, before the first global relabel): a pixel holding
// excess sends it straight on through a neighbour that still has sink capacity
// (s -> p -> q -> t augmentations).  After pre-cancellation a pixel either holds
// excess or sink capacity, never both, so the only contended word is rT(q), taken
// with a compare-and-swap; residual pairs are updated atomically.  The result is a
// valid preflow, so flow value and minimal cut are unchanged; it only removes work
// the first push rounds would otherwise do pixel by pixel.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void two_hop_pixel(const GridDev &g, int32_t r, int32_t c);

// one thread per pixel: x = column, rows over blockIdx.y (grid-stride past 65535 rows)
__global__ void two_hop_kernel(GridDev g) {
    const int32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= g.W) return;
    for (int32_t r = blockIdx.y; r < g.H; r += gridDim.y) two_hop_pixel(g, r, c);
}

__device__ __forceinline__ void two_hop_pixel(const GridDev &g, int32_t r, int32_t c) {
    const int64_t p = (int64_t)r * g.W + c;
    int32_t e = g.e[p];
    if (e <= 0) return;
    int32_t *fwd[4] = {g.rR, g.rL, g.rD, g.rU};
    int32_t *rev[4] = {g.rL, g.rR, g.rU, g.rD};
    // band mode: routes stay inside the band (arcs to a neighbour band are left alone)
    const bool ok[4] = {c + 1 < g.W, c > 0, r + 1 < g.H, r > 0};
    const int64_t qs[4] = {p + 1, p - 1, p + g.W, p - g.W};
    // every operand first (one round trip)
    int32_t rp[4], t[4];
#pragma unroll
    for (int d = 0; d < 4; d++) {
        rp[d] = ok[d] ? *(volatile int32_t *)(fwd[d] + p) : 0;
        t[d] = ok[d] ? *(volatile int32_t *)(g.rT + qs[d]) : 0;
    }
    // the excess is split over the directions from the loaded values, and the four sink
    // reservations go out together (one round trip instead of a CAS chain): each takes
    // min(want, what rT(q) held) and hands the over-draw back, so no rT(q) is overdrawn
    // for good and the sum taken from it never exceeds its residual
    int32_t want[4], old[4];
    int32_t rem = e;
#pragma unroll
    for (int d = 0; d < 4; d++) {
        want[d] = (rp[d] > 0 && t[d] > 0 && rem > 0) ? min(rem, min(rp[d], t[d])) : 0;
        rem -= want[d];
    }
#pragma unroll
    for (int d = 0; d < 4; d++) old[d] = want[d] > 0 ? atomicSub(g.rT + qs[d], want[d]) : 0;
#pragma unroll
    for (int d = 0; d < 4; d++) {
        if (want[d] <= 0) continue;
        const int32_t take = min(want[d], max(old[d], 0));
        if (take < want[d]) atomicAdd(g.rT + qs[d], want[d] - take);
        if (take <= 0) continue;
        e -= take;
        atomicSub(fwd[d] + p, take);
        atomicAdd(rev[d] + qs[d], take);
    }
    g.e[p] = e;
}

// Three-hop pre-routing (after the two-hop pass): s -> p -> q -> q2 -> t through a
// neighbour q and one of q's neighbours q2 with spare sink capacity.  r(q -> q2) is
// reserved first and rT(q2) second (each by compare-and-swap, the unused part of the
// reservation handed back), so concurrent paths through q never overdraw it.
__device__ __forceinline__ int32_t cas_take(int32_t *w, int32_t want) {
    int32_t v = *(volatile int32_t *)w;
    while (v > 0) {
        const int32_t take = min(want, v);
        const int32_t old = atomicCAS(w, v, v - take);
        if (old == v) return take;
        v = old;
    }
    return 0;
}

__global__ void three_hop_kernel(GridDev g) {
    const int64_t HW = (int64_t)g.H * g.W;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= HW) return;
    int32_t e = g.e[p];
    if (e <= 0) return;
    const int32_t r = (int32_t)(p / g.W), c = (int32_t)(p - (int64_t)r * g.W);
    int32_t *fwd[4] = {g.rR, g.rL, g.rD, g.rU};
    int32_t *rev[4] = {g.rL, g.rR, g.rU, g.rD};
    const int dr[4] = {0, 0, 1, -1}, dc[4] = {1, -1, 0, 0};
    for (int d1 = 0; d1 < 4 && e > 0; d1++) {
        const int32_t qr = r + dr[d1], qc = c + dc[d1];
        if (qr < 0 || qr >= g.H || qc < 0 || qc >= g.W) continue;
        const int64_t q = (int64_t)qr * g.W + qc;
        for (int d2 = 0; d2 < 4 && e > 0; d2++) {
            if (d2 == (d1 ^ 1)) continue;                         // back to p
            const int32_t r2 = qr + dr[d2], c2 = qc + dc[d2];
            if (r2 < 0 || r2 >= g.H || c2 < 0 || c2 >= g.W) continue;
            const int64_t q2 = (int64_t)r2 * g.W + c2;
            const int32_t rpq = *(volatile int32_t *)(fwd[d1] + p);
            const int32_t want = min(e, rpq);
            if (want <= 0) break;                                 // p -> q saturated
            if (*(volatile int32_t *)(g.rT + q2) <= 0 || *(volatile int32_t *)(fwd[d2] + q) <= 0) continue;
            // every hop reserved by compare-and-swap: r(p -> q) is also the middle hop of
            // other pixels' paths (x -> p -> q), so the owner may not just subtract
            const int32_t a0 = cas_take(fwd[d1] + p, want);       // reserve p -> q
            if (a0 <= 0) break;
            const int32_t a = cas_take(fwd[d2] + q, a0);          // then q -> q2
            if (a < a0) atomicAdd(fwd[d1] + p, a0 - a);           // hand back the unused part
            if (a <= 0) continue;
            const int32_t b = cas_take(g.rT + q2, a);             // then q2 -> t
            if (b < a) { atomicAdd(fwd[d2] + q, a - b); atomicAdd(fwd[d1] + p, a - b); }
            if (b <= 0) continue;
            e -= b;
            atomicAdd(rev[d1] + q, b);
            atomicAdd(rev[d2] + q2, b);
        }
    }
    g.e[p] = e;
}

// ----------------------------------------------------------------------------
// K1 (v1): one lock-free sweep, one thread per pixel (maxflow_par.py:95-128).
// Skip if e <= 0 or h >= |V|; find the lowest residual neighbour among
// {t (height 0), right, left, down, up, s (height |V|)}; push min(e, r) with four
// atomics when strictly above it, otherwise relabel to lowest + 1 (owner-only).
// Only the owner lowers e(p) and r(p->q), so its loads are conservative and a
// push never overdraws (maxflow_par.py:114-119).
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) pr_sweep_kernel(GridDev g, int32_t *active_flag,
                                                       unsigned long long *ops) {
    const int c = blockIdx.x * TILE_W + threadIdx.x;
    const int r = blockIdx.y * BLK_Y + threadIdx.y;
    int pushes = 0, relabels = 0, act = 0;
    if (c < g.W && r < g.H) {
        const int64_t p = (int64_t)r * g.W + c;
        const int32_t e = ld_cg(g.e + p);
        const int32_t hp = g.h[p];
        if (e > 0 && hp < g.V) {
            act = 1;
            int32_t best_h = INT32_MAX, best_r = 0;
            int dir = -1;
            const int32_t rt = g.rT[p];
            if (rt > 0) {
                best_h = 0; best_r = rt; dir = 4;
            } else {
                if (c + 1 < g.W) {
                    const int32_t rr = ld_cg(g.rR + p);
                    if (rr > 0) { const int32_t hq = ld_cg(g.h + p + 1); if (hq < best_h) { best_h = hq; best_r = rr; dir = 0; } }
                }
                if (c > 0) {
                    const int32_t rr = ld_cg(g.rL + p);
                    if (rr > 0) { const int32_t hq = ld_cg(g.h + p - 1); if (hq < best_h) { best_h = hq; best_r = rr; dir = 1; } }
                }
                if (r + 1 < g.H) {
                    const int32_t rr = ld_cg(g.rD + p);
                    if (rr > 0) { const int32_t hq = ld_cg(g.h + p + g.W); if (hq < best_h) { best_h = hq; best_r = rr; dir = 2; } }
                }
                if (r > 0) {
                    const int32_t rr = ld_cg(g.rU + p);
                    if (rr > 0) { const int32_t hq = ld_cg(g.h + p - g.W); if (hq < best_h) { best_h = hq; best_r = rr; dir = 3; } }
                }
                if (g.rS[p] > 0 && g.V < best_h) { best_h = g.V; dir = 5; }
            }
            if (dir >= 0) {
                if (hp > best_h) {
                    const int32_t d = min(e, best_r);
                    atomicSub(g.e + p, d);
                    if (dir == 4) {
                        g.rT[p] = rt - d;  // only p touches its sink arc
                    } else {
                        int64_t q; int32_t *fw, *bw;
                        if (dir == 0) { q = p + 1; fw = g.rR; bw = g.rL; }
                        else if (dir == 1) { q = p - 1; fw = g.rL; bw = g.rR; }
                        else if (dir == 2) { q = p + g.W; fw = g.rD; bw = g.rU; }
                        else { q = p - g.W; fw = g.rU; bw = g.rD; }
                        atomicSub(fw + p, d);
                        atomicAdd(bw + q, d);
                        atomicAdd(g.e + q, d);
                    }
                    pushes = 1;
                } else {
                    g.h[p] = best_h + 1;
                    relabels = 1;
                }
            }
        }
    }
    if (__syncthreads_or(act) && threadIdx.x == 0 && threadIdx.y == 0) *active_flag = 1;
    block_add_i64<NWARPS>(pushes, ops + 0);
    block_add_i64<NWARPS>(relabels, ops + 1);
}

// ----------------------------------------------------------------------------
// K1 (v2, default): tile-resident lock-free push-relabel.  One CTA stages a 32x32
// tile (e, h, four direction residuals, sink residual) plus a 1-pixel halo of
// neighbour heights in shared memory and runs up to k_local lock-free passes of
// the maxflow_par.py:95-128 operation with shared-memory atomics.  No barrier
// orders the passes (warps free-run, as the reference's workers do); a CTA-wide
// vote every 4 passes ends the visit once no pixel of the tile is active.
// A push across the tile border lowers the sender's own residual and parks the
// amount in the receiver's inbox, so no other CTA ever writes a word this CTA
// holds in shared memory; the receiver folds its inbox into e and the reverse
// residual when it next loads (or the coordinator does, before a global relabel).
// Halo heights are a snapshot: stale reads are tolerated by the lock-free
// argument, exactly like a worker reading a neighbour's height.
// ----------------------------------------------------------------------------
constexpr int PT_W = 32, PT_H = 32, PT_TY = 16;          // 512 threads, 2 rows each
constexpr int PT_ROWS = PT_H / PT_TY;

#ifndef FM_PT_MINBLOCKS
#define FM_PT_MINBLOCKS 4  // 32 registers: 4 CTAs (2048 threads) per SM
#endif
__global__ void __launch_bounds__(PT_W * PT_TY, FM_PT_MINBLOCKS) pr_tile_kernel(GridDev g, int k_local, int steps, int fused, int vote_mask, int parity,
                                                               int32_t *processed,
                                                               unsigned long long *ops) {
    __shared__ int32_t s_e[PT_H][PT_W];
    __shared__ int32_t s_h[PT_H + 2][PT_W + 2];
    __shared__ int32_t s_r[4][PT_H][PT_W];   // R, L, D, U
    __shared__ int32_t s_t[PT_H][PT_W];
    __shared__ int s_tile;
    const int tx = threadIdx.x, ty = threadIdx.y;
    long long pushes = 0, relabels = 0;
    for (;;) {
    __syncthreads();
    if (tx == 0 && ty == 0) s_tile = tq_take(g.pq, parity, 0, 0);
    __syncthreads();
    const int tile = s_tile;
    if (tile < 0) break;
    const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
    const int r0 = tyi * PT_H, c0 = txi * PT_W;
    __threadfence();
    const int V = g.V;
    const int c = c0 + tx;
    int32_t rs[PT_ROWS];
    bool ghost[PT_ROWS];
#pragma unroll
    for (int k = 0; k < PT_ROWS; k++) {
        const int lr = ty + k * PT_TY;
        const int r = r0 + lr;
        ghost[k] = false;
        if (r < g.H && c < g.W) {
            const int64_t p = (int64_t)r * g.W + c;
            int32_t e = g.e[p];
            int32_t rr = g.rR[p], rl = g.rL[p], rd = g.rD[p], ru = g.rU[p];
            if (tx == 0 && c > 0) { const int32_t d = atomicExch(g.inflow_h + p, 0); e += d; rl += d; }
            if (tx == PT_W - 1 && c + 1 < g.W) { const int32_t d = atomicExch(g.inflow_h + p, 0); e += d; rr += d; }
            if (lr == 0 && r > 0) { const int32_t d = atomicExch(g.inflow_v + p, 0); e += d; ru += d; }
            if (lr == PT_H - 1 && r + 1 < g.H) { const int32_t d = atomicExch(g.inflow_v + p, 0); e += d; rd += d; }
            s_e[lr][tx] = e;
            s_h[lr + 1][tx + 1] = g.h[p];
            s_r[0][lr][tx] = rr; s_r[1][lr][tx] = rl; s_r[2][lr][tx] = rd; s_r[3][lr][tx] = ru;
            s_t[lr][tx] = g.rT[p];
            rs[k] = g.rS[p];
        } else {
            s_e[lr][tx] = 0;
            s_h[lr + 1][tx + 1] = V;
            s_r[0][lr][tx] = s_r[1][lr][tx] = s_r[2][lr][tx] = s_r[3][lr][tx] = 0;
            s_t[lr][tx] = 0;
            rs[k] = 0;
        }
    }
    // halo snapshot of neighbour heights
    {
        const int tid = ty * PT_W + tx;
        if (tid < 4 * PT_W) {
            const int side = tid / PT_W, i = tid % PT_W;
            int r, cc, hr, hc;
            if (side == 0) { r = r0 - 1; cc = c0 + i; hr = 0; hc = i + 1; }
            else if (side == 1) { r = r0 + PT_H; cc = c0 + i; hr = PT_H + 1; hc = i + 1; }
            else if (side == 2) { r = r0 + i; cc = c0 - 1; hr = i + 1; hc = 0; }
            else { r = r0 + i; cc = c0 + PT_W; hr = i + 1; hc = PT_W + 1; }
            s_h[hr][hc] = (r >= 0 && r < g.H && cc >= 0 && cc < g.W) ? g.h[(int64_t)r * g.W + cc] : V;
        }
    }
    __syncthreads();

    volatile int32_t *ve = &s_e[0][0];
    volatile int32_t *vh = &s_h[0][0];
    volatile int32_t *vt = &s_t[0][0];
    constexpr int HS = PT_W + 2;  // s_h row stride
    for (int it = 0; it < k_local; it++) {
        bool any = false;
#pragma unroll
        for (int k = 0; k < PT_ROWS; k++) {
            const int lr = ty + k * PT_TY;
            const int li = lr * PT_W + tx;
            if (ghost[k]) continue;                      // owned by the neighbour band
            const int hi = (lr + 1) * HS + tx + 1;
            const int r = r0 + lr;
            // up to `steps` operations on this pixel per pass: a relabel is always
            // followed by the push it enables (the pixel now sits one above its
            // lowest residual neighbour), and the pixel keeps discharging while it
            // holds excess -- a sequence of maxflow_par.py:98-125 operations by the
            // pixel's owner, each one lock-free
            for (int st = 0; st < steps; st++) {
                const int32_t e = ve[li];
                if (e <= 0) break;
                int32_t hp = vh[hi];
                if (hp >= V) break;
                any = true;
                const int32_t rt = vt[li];
                if (rt > 0) {                             // sink at height 0
                    if (hp == 0) { vh[hi] = 1; relabels++; }
                    const int32_t d = min(e, rt);
                    vt[li] = rt - d;                      // owner-only word
                    atomicSub(&s_e[lr][tx], d);
                    pushes++;
                    continue;
                }
                int32_t best_h = INT32_MAX, best_r = 0;
                int dir = -1;
                const int32_t rr = *(volatile int32_t *)&s_r[0][lr][tx];
                if (rr > 0 && c + 1 < g.W) { const int32_t hq = vh[hi + 1]; if (hq < best_h) { best_h = hq; best_r = rr; dir = 0; } }
                const int32_t rl = *(volatile int32_t *)&s_r[1][lr][tx];
                if (rl > 0 && c > 0) { const int32_t hq = vh[hi - 1]; if (hq < best_h) { best_h = hq; best_r = rl; dir = 1; } }
                const int32_t rd = *(volatile int32_t *)&s_r[2][lr][tx];
                if (rd > 0 && r + 1 < g.H) { const int32_t hq = vh[hi + HS]; if (hq < best_h) { best_h = hq; best_r = rd; dir = 2; } }
                const int32_t ru = *(volatile int32_t *)&s_r[3][lr][tx];
                if (ru > 0 && r > 0) { const int32_t hq = vh[hi - HS]; if (hq < best_h) { best_h = hq; best_r = ru; dir = 3; } }
                if (rs[k] > 0 && V < best_h) { best_h = V; dir = 5; }
                if (dir < 0) break;                       // nothing residual: written off later
                if (hp <= best_h) {                       // relabel (owner-only)
                    hp = best_h + 1;
                    vh[hi] = hp;
                    relabels++;
                    // above the source: inactive.  fused == 0: the reference's one
                    // operation per pass (the push waits for the next pass)
                    if (dir == 5 || !fused) break;
                }
                const int32_t d = min(e, best_r);
                atomicSub(&s_e[lr][tx], d);
                atomicSub(&s_r[dir][lr][tx], d);
                int qr = lr, qc = tx;
                if (dir == 0) qc++; else if (dir == 1) qc--; else if (dir == 2) qr++; else qr--;
                const int rev = dir ^ 1;                  // R<->L, D<->U
                if (qr >= 0 && qr < PT_H && qc >= 0 && qc < PT_W) {
                    atomicAdd(&s_r[rev][qr][qc], d);
                    atomicAdd(&s_e[qr][qc], d);
                } else {
                    const int64_t q = (int64_t)(r0 + qr) * g.W + (c0 + qc);
                    atomicAdd((dir < 2 ? g.inflow_h : g.inflow_v) + q, d);
                    __threadfence();
                    const int nt = (dir == 0) ? tile + 1 : (dir == 1) ? tile - 1
                                 : (dir == 2) ? tile + g.ntx : tile - g.ntx;
                    tq_push(g.pq, parity ^ 1, nt);
                    g.touched[nt] = 1;
                }
                pushes++;
            }
        }
        if ((it & vote_mask) == vote_mask && !__syncthreads_or(any)) break;
    }
    __syncthreads();
    bool act = false;
#pragma unroll
    for (int k = 0; k < PT_ROWS; k++) {
        const int lr = ty + k * PT_TY;
        const int r = r0 + lr;
        if (r < g.H && c < g.W) {
            const int64_t p = (int64_t)r * g.W + c;
            const int32_t e = s_e[lr][tx], h = s_h[lr + 1][tx + 1];
            g.e[p] = e;
            g.h[p] = h;
            g.rR[p] = s_r[0][lr][tx]; g.rL[p] = s_r[1][lr][tx];
            g.rD[p] = s_r[2][lr][tx]; g.rU[p] = s_r[3][lr][tx];
            g.rT[p] = s_t[lr][tx];
            act |= (e > 0 && h < V && !ghost[k]);
        }
    }
    const int any_act = __syncthreads_or(act);
    if (tx == 0 && ty == 0) {
        if (any_act) tq_push(g.pq, parity ^ 1, tile);
        g.touched[tile] = 1;
        atomicAdd(processed, 1);
    }
    }  // tile loop
    block_add_i64<PT_W * PT_TY / 32>(pushes, ops + 0);
    block_add_i64<PT_W * PT_TY / 32>(relabels, ops + 1);
}

// ----------------------------------------------------------------------------
// K1 (v3, default): the same tile-resident lock-free operation, driven by per-pass
// lists of active pixels instead of a scan of all 1024 pixels per pass.
//
// A v2 pass costs every warp a scan of its rows while only a few percent of the
// pixels are active (ncu: ~1 thread per warp executes the operation body, 30% of
// stall samples sit in the activity vote).  Here the pixels a pass operates on are
// listed in shared memory and dealt out to consecutive threads, so warps run
// operations with most lanes busy.  While a pass lists more than 32 pixels the
// whole CTA works on it (one barrier per pass); once a list fits one warp, warp 0
// carries on alone with warp-synchronous passes and the other warps sleep at the
// final barrier, so sparse passes pay neither a CTA barrier nor idle warps' issue.
//
// List maintenance (each pixel appears at most once per list):
//  * after its operation(s) the owner re-lists its pixel iff its excess is still
//    positive (the value its own atomicSub returned) and it sits below the source;
//  * a push re-lists the receiver iff the receiver's atomicAdd saw e <= 0, i.e. this
//    push made it active.  An owner whose own atomicSub left e <= 0 stops working
//    on the pixel, so "owner saw e > 0 last" and "a sender saw e <= 0" exclude each
//    other in the atomic order on e(p): exactly one of them lists p.
// Pixels left out (no residual arc, above the source) are rescanned when the tile
// is next loaded.  Lists are double-buffered; three counters rotate so that the
// counter the next pass fills is zeroed one barrier before it is used.
// Flow pushed across the tile border goes to the receiver's inbox (fire-and-forget
// RED); the neighbour tile is queued for the next launch once, at the end of the
// visit (the launch boundary orders the inbox writes before its next load).
// ----------------------------------------------------------------------------
// push-kernel CTA = 32 x PL_TY threads on one 32x32 tile.  4 warps (r02by: push kernel
// -3% at 4096^2 and 8192^2 against 8 warps): a pass with few listed pixels parks fewer
// warps at its barrier, and the tile's shared memory, not the thread count, bounds the
// CTAs per SM.  The border / inbox stage needs one thread per border pixel (4 x 32).
#ifndef FM_PL_TY
#define FM_PL_TY 4
#endif
constexpr int PL_TY = FM_PL_TY, PL_NT = PT_W * PL_TY, PL_ROWS = PT_H / PL_TY;
static_assert(PL_NT >= 4 * PT_W, "the border / inbox stage of a tile visit needs 128 threads");
// heights with a 1-pixel halo, rows padded to 40 words so each interior row starts
// 16-byte aligned (column c at PL_HC + c; halo columns at PL_HC - 1 and PL_HC + 32)
constexpr int PL_HS = 40, PL_HC = 4;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
// 4-byte copy; zero-fills the destination when !pred
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem, bool pred) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(pred ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::: "memory");
}

// ---- TMA (cp.async.bulk.tensor) staging of a tile visit's planes ---------------------
// Tensor maps of the int32 planes (H x W, row-major): e, rT, rS as 32 x 32 boxes at
// (c0, r0); h as a 40 x 34 box at (c0 - 4, r0 - 1), which is exactly the padded halo
// layout of PlSmemT::h (row stride PL_HS = 40, column c at PL_HC = 4 + c) -- the halo
// rows and columns arrive with the interior, out-of-grid cells zero-filled.  r[4]: the
// int32 residual planes (the packed instance packs them from registers instead).  One
// thread arms the CTA's mbarrier with the byte count and issues the copies; every thread
// waits on the barrier's phase.  Used when W % 4 == 0 (TMA strides are 16-byte multiples).
struct PlMaps {
    CUtensorMap e, t, s, h, r[4];
};

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long *mbar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long *mbar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *mbar, unsigned parity) {
    asm volatile("{\n .reg .pred P1;\n"
                 "FM_WAIT_%=:\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
                 " @!P1 bra FM_WAIT_%=;\n}" ::"r"(smem_u32(mbar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y, unsigned long long *mbar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(smem_u32(mbar)) : "memory");
}
// earlier generic-proxy accesses of this thread to shared memory before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
#ifndef FM_PL_MINBLOCKS
#define FM_PL_MINBLOCKS 6
#endif

__device__ __forceinline__ void pl_append_warp(bool want, int idx, int *cnt, uint16_t *list) {
    const unsigned m = __ballot_sync(0xffffffffu, want);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(cnt, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (want) list[base + __popc(m & ((1u << lane) - 1))] = (uint16_t)idx;
}

__device__ __forceinline__ uint2 pk_pack(int32_t r, int32_t l, int32_t d, int32_t u) {
    return make_uint2((uint32_t)r | ((uint32_t)l << 16), (uint32_t)d | ((uint32_t)u << 16));
}

// Flow pushed out of the tile into pixel (qr, qc) (band coordinates): parked in the
// receiver's inbox.  Row-band mode: a row outside the band is the neighbour band's
// boundary row, whose inbox is reached through peer memory; the system-scope fence
// orders the inbox add before the external-push flag the CTA raises after the visit.
__device__ __forceinline__ void push_out(const GridDev &g, int qr, int qc, int dir, int32_t d) {
    if (qr < 0) { atomicAdd(g.up.inbox + qc, d); __threadfence_system(); return; }
    if (qr >= g.H) { atomicAdd(g.dn.inbox + qc, d); __threadfence_system(); return; }
    atomicAdd((dir < 2 ? g.inflow_h : g.inflow_v) + (int64_t)qr * g.W + qc, d);
}

struct PlTile {
    int32_t *e, *h, *t;        // shared planes (h with a 1-pixel halo, row stride PT_W + 2)
    int32_t (*r)[PT_H * PT_W];
    uint2 *r2;                 // packed-residual kernel: {R | L << 16, D | U << 16} per pixel
    const uint8_t *f;
    int *nbr;                  // bit d: flow was parked in the inbox of neighbour tile d
    int r0, c0;
    uint8_t *dirty;            // row lr changed in this visit (plain stores of 1: benign races)
};

// The default operation (steps == 1, not fused: one maxflow_par.py:98-125 operation
// per listed pixel per pass) with every shared-memory read issued up front and the
// two pushes' atomics in flight together: the pass is a latency chain, so fewer
// dependent round trips is what makes it faster.  Same results as pl_item.
// No grid-bound tests: the residual toward a neighbour outside the grid (or band, with
// no neighbour band) is 0 from grid_init and only ever grows by flow that neighbour
// sent, so a positive residual implies the neighbour exists.
__device__ __forceinline__ bool pl_op1(const GridDev &g, const PlTile &T, int li, int *recv,
                                       unsigned &pushes, unsigned &relabels) {
    constexpr int HS = PL_HS;
    volatile int32_t *ve = T.e;
    volatile int32_t *vh = T.h;
    volatile int32_t *vt = T.t;
    const int V = g.V;
    const int lr = li >> 5, lc = li & 31;
    const int hi = (lr + 1) * HS + lc + PL_HC;
    const uint8_t f = T.f[li];
    const int32_t e = ve[li], hp = vh[hi], rt = vt[li];
    const int32_t rr = *(volatile int32_t *)&T.r[0][li];
    const int32_t rl = *(volatile int32_t *)&T.r[1][li];
    const int32_t rd = *(volatile int32_t *)&T.r[2][li];
    const int32_t ru = *(volatile int32_t *)&T.r[3][li];
    const int32_t hR = vh[hi + 1], hL = vh[hi - 1], hD = vh[hi + HS], hU = vh[hi - HS];
    if ((f & 2) || e <= 0 || hp >= V) return false;
    if (rt > 0) {                                          // sink at height 0
        T.dirty[lr] = 1;
        if (hp == 0) { vh[hi] = 1; relabels++; }
        const int32_t d = min(e, rt);
        vt[li] = rt - d;
        pushes++;
        return atomicSub(&T.e[li], d) - d > 0;
    }
    int32_t best_h = INT32_MAX, best_r = 0;
    int dir = -1;
    if (rr > 0 && hR < best_h) { best_h = hR; best_r = rr; dir = 0; }
    if (rl > 0 && hL < best_h) { best_h = hL; best_r = rl; dir = 1; }
    if (rd > 0 && hD < best_h) { best_h = hD; best_r = rd; dir = 2; }
    if (ru > 0 && hU < best_h) { best_h = hU; best_r = ru; dir = 3; }
    if ((f & 1) && V < best_h) { best_h = V; dir = 5; }
    if (dir < 0) return false;                             // nothing residual: rescanned on next load
    T.dirty[lr] = 1;                                       // a relabel or a push follows
    if (hp <= best_h) {                                    // relabel (owner-only); the push waits
        vh[hi] = best_h + 1;
        relabels++;
        return dir != 5;                                   // above the source: inactive
    }
    const int32_t d = min(e, best_r);
    int qr = lr, qc = lc;
    if (dir == 0) qc++; else if (dir == 1) qc--; else if (dir == 2) qr++; else qr--;
    // both returning atomics in flight before either result is used (passes are
    // barrier-separated, so the order of the owner's and the receiver's updates is free)
    const int32_t oldp = atomicSub(&T.e[li], d);           // the owner's view of e(p)
    atomicSub(&T.r[dir][li], d);
    pushes++;
    if (qr >= 0 && qr < PT_H && qc >= 0 && qc < PT_W) {
        const int qi = qr * PT_W + qc;
        T.dirty[qr] = 1;
        atomicAdd(&T.r[dir ^ 1][qi], d);
        const int32_t old = atomicAdd(&T.e[qi], d);
        if (old <= 0 && old + d > 0) *recv = qi;
    } else {
        push_out(g, T.r0 + qr, T.c0 + qc, dir, d);
        atomicOr(T.nbr, 1 << dir);
    }
    return oldp - d > 0;                                   // hp < V here
}

// pl_op1 over packed residuals: the four residuals of a pixel are 16-bit fields of two
// 32-bit shared words, {R | L << 16, D | U << 16} (used when every neighbour pair's two
// capacities sum to <= 65535: a field then never leaves [0, 65535], so a shifted 32-bit
// atomic add is exact; a pair's two residuals share a word index), so the operation
// reads them with one 64-bit load and shared memory per tile shrinks by 8 KB.
__device__ __forceinline__ bool pk_op1(const GridDev &g, const PlTile &T, int li, int *recv,
                                       unsigned &pushes, unsigned &relabels) {
    constexpr int HS = PL_HS;
    volatile int32_t *ve = T.e;
    volatile int32_t *vh = T.h;
    volatile int32_t *vt = T.t;
    const int V = g.V;
    const int lr = li >> 5, lc = li & 31;
    const int hi = (lr + 1) * HS + lc + PL_HC;
    const uint8_t f = T.f[li];
    const int32_t e = ve[li], hp = vh[hi], rt = vt[li];
    const unsigned long long w64 = *(volatile unsigned long long *)&T.r2[li];
    const uint2 w = make_uint2((uint32_t)w64, (uint32_t)(w64 >> 32));
    const int32_t hR = vh[hi + 1], hL = vh[hi - 1], hD = vh[hi + HS], hU = vh[hi - HS];
    if ((f & 2) || e <= 0 || hp >= V) return false;
    if (rt > 0) {                                          // sink at height 0
        T.dirty[lr] = 1;
        if (hp == 0) { vh[hi] = 1; relabels++; }
        const int32_t d = min(e, rt);
        vt[li] = rt - d;
        pushes++;
        return atomicSub(&T.e[li], d) - d > 0;
    }
    const int32_t rr = (int32_t)(w.x & 0xffff), rl = (int32_t)(w.x >> 16);
    const int32_t rd = (int32_t)(w.y & 0xffff), ru = (int32_t)(w.y >> 16);
    int32_t best_h = INT32_MAX, best_r = 0;
    int dir = -1;
    if (rr > 0 && hR < best_h) { best_h = hR; best_r = rr; dir = 0; }
    if (rl > 0 && hL < best_h) { best_h = hL; best_r = rl; dir = 1; }
    if (rd > 0 && hD < best_h) { best_h = hD; best_r = rd; dir = 2; }
    if (ru > 0 && hU < best_h) { best_h = hU; best_r = ru; dir = 3; }
    if ((f & 1) && V < best_h) { best_h = V; dir = 5; }
    if (dir < 0) return false;
    T.dirty[lr] = 1;
    if (hp <= best_h) {
        vh[hi] = best_h + 1;
        relabels++;
        return dir != 5;
    }
    const int32_t d = min(e, best_r);
    int qr = lr, qc = lc;
    if (dir == 0) qc++; else if (dir == 1) qc--; else if (dir == 2) qr++; else qr--;
    const int32_t oldp = atomicSub(&T.e[li], d);
    uint32_t *rw = reinterpret_cast<uint32_t *>(T.r2);
    atomicAdd(&rw[2 * li + (dir >> 1)], 0u - ((uint32_t)d << (16 * (dir & 1))));
    pushes++;
    if (qr >= 0 && qr < PT_H && qc >= 0 && qc < PT_W) {
        const int qi = qr * PT_W + qc;
        T.dirty[qr] = 1;
        atomicAdd(&rw[2 * qi + (dir >> 1)], (uint32_t)d << (16 * ((dir & 1) ^ 1)));
        const int32_t old = atomicAdd(&T.e[qi], d);
        if (old <= 0 && old + d > 0) *recv = qi;
    } else {
        push_out(g, T.r0 + qr, T.c0 + qc, dir, d);
        atomicOr(T.nbr, 1 << dir);
    }
    return oldp - d > 0;
}

// two candidates per lane (the pixel itself, the receiver it activated), one list reservation
__device__ __forceinline__ void pl_append2_warp(bool wa, int ia, bool wb, int ib, int *cnt, uint16_t *list) {
    const unsigned ma = __ballot_sync(0xffffffffu, wa), mb = __ballot_sync(0xffffffffu, wb);
    if (!(ma | mb)) return;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1;
    int base = 0;
    if (lane == 0) base = atomicAdd(cnt, __popc(ma) + __popc(mb));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (wa) list[base + __popc(ma & lt)] = (uint16_t)ia;
    if (wb) list[base + __popc(ma) + __popc(mb & lt)] = (uint16_t)ib;
}

// One listed pixel: up to `steps` operations of maxflow_par.py:98-125 by its owner.
// Returns whether the owner re-lists it; *recv = the in-tile receiver its last push
// activated (-1 if none); receivers of earlier pushes are listed directly.
__device__ __forceinline__ bool pl_item(const GridDev &g, const PlTile &T, int li, int steps, int fused,
                                        int *cnt_next, uint16_t *lout, int *recv,
                                        unsigned &pushes, unsigned &relabels) {
    constexpr int HS = PL_HS;
    volatile int32_t *ve = T.e;
    volatile int32_t *vh = T.h;
    volatile int32_t *vt = T.t;
    const int V = g.V;
    const int lr = li >> 5, lc = li & 31;
    const int hi = (lr + 1) * HS + lc + PL_HC;
    const int r = T.r0 + lr, c = T.c0 + lc;
    const uint8_t f = T.f[li];
    if (f & 2) return false;                               // ghost row: owned by the neighbour band
    int32_t e = ve[li];
    int32_t hp = vh[hi];
    for (int st = 0; st < steps; st++) {
        if (e <= 0 || hp >= V) return false;
        const int32_t rt = vt[li];
        if (rt > 0) {                                      // sink at height 0
            if (hp == 0) { hp = 1; vh[hi] = 1; relabels++; }
            const int32_t d = min(e, rt);
            vt[li] = rt - d;
            e = atomicSub(&T.e[li], d) - d;
            pushes++;
            continue;
        }
        const int32_t rr = *(volatile int32_t *)&T.r[0][li];
        const int32_t rl = *(volatile int32_t *)&T.r[1][li];
        const int32_t rd = *(volatile int32_t *)&T.r[2][li];
        const int32_t ru = *(volatile int32_t *)&T.r[3][li];
        const int32_t hR = vh[hi + 1], hL = vh[hi - 1], hD = vh[hi + HS], hU = vh[hi - HS];
        int32_t best_h = INT32_MAX, best_r = 0;
        int dir = -1;
        if (rr > 0 && c + 1 < g.W && hR < best_h) { best_h = hR; best_r = rr; dir = 0; }
        if (rl > 0 && c > 0 && hL < best_h) { best_h = hL; best_r = rl; dir = 1; }
        if (rd > 0 && r + 1 < g.hlim && hD < best_h) { best_h = hD; best_r = rd; dir = 2; }
        if (ru > 0 && r > g.rmin && hU < best_h) { best_h = hU; best_r = ru; dir = 3; }
        if ((f & 1) && V < best_h) { best_h = V; dir = 5; }
        if (dir < 0) return false;                         // nothing residual: rescanned on next load
        if (hp <= best_h) {                                // relabel (owner-only)
            hp = best_h + 1;
            vh[hi] = hp;
            relabels++;
            if (dir == 5) return false;                    // above the source: inactive
            if (!fused) break;
        }
        const int32_t d = min(e, best_r);
        atomicSub(&T.r[dir][li], d);
        int qr = lr, qc = lc;
        if (dir == 0) qc++; else if (dir == 1) qc--; else if (dir == 2) qr++; else qr--;
        if (qr >= 0 && qr < PT_H && qc >= 0 && qc < PT_W) {
            const int qi = qr * PT_W + qc;
            atomicAdd(&T.r[dir ^ 1][qi], d);
            const int32_t old = atomicAdd(&T.e[qi], d);
            if (old <= 0 && old + d > 0) {
                if (*recv >= 0) lout[atomicAdd(cnt_next, 1)] = (uint16_t)*recv;
                *recv = qi;
            }
        } else {
            push_out(g, T.r0 + qr, T.c0 + qc, dir, d);
            atomicOr(T.nbr, 1 << dir);
        }
        e = atomicSub(&T.e[li], d) - d;                    // last: the owner's view of e(p)
        pushes++;
    }
    return e > 0 && hp < V;
}

template <bool PK> struct PlRes { int32_t r[4][PT_H * PT_W]; };              // R, L, D, U
template <> struct PlRes<true> { uint2 r2[PT_H * PT_W]; };                  // packed 16-bit fields

// Members a TMA copy lands in start on 128-byte boundaries (e, t, list -- rS is staged in
// list[0] --, h, and the int32 residual planes).
constexpr int PL_HWORDS = ((PT_H + 2) * PL_HS + 31) / 32 * 32;   // 34 x 40 heights, padded to 128 B
template <bool PK> struct __align__(128) PlSmemT {
    int32_t e[PT_H * PT_W];
    int32_t t[PT_H * PT_W];
    uint16_t list[2][PT_H * PT_W];
    int32_t h[PL_HWORDS];
    PlRes<PK> res;
    uint8_t f[PT_H * PT_W];      // bit 0: residual arc to s, bit 1: outside the grid
    uint8_t dirty[PT_H];         // rows a visit changed (only those are written back)
    unsigned long long mbar;     // TMA completion barrier (one per CTA, phase flips per visit)
    int cnt[3];
    int nbr;
    int tile;
    int flag;
    long long red[PL_NT / 32];
};
using PlSmem = PlSmemT<false>;

struct PlCounters {
    unsigned pushes = 0, relabels = 0, passes = 0, items = 0;   // per thread per launch: 32 bits suffice
#ifdef FM_PL_TIMING
    long long t_load = 0, t_pass = 0, t_store = 0, visits = 0, solo = 0, t_solo = 0, dense_passes = 0, solo_passes = 0;
#endif
};

// One visit of `tile`: load (folding the inboxes), list-driven passes, write back.
// Returns (CTA-uniform) whether the tile still holds an active pixel; S.nbr = the
// neighbour tiles whose inboxes received flow.  Starts and ends with a barrier.
template <bool PK>
__device__ __forceinline__ bool pl_visit(const GridDev &g, PlSmemT<PK> &S, int tile, int k_local, int steps,
                                         int fused, PlCounters &C, const PlMaps *maps, unsigned &tma_phase) {
    constexpr int HS = PL_HS;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * PT_W + tx;
    const int V = g.V;
    if (tid == 0) { S.cnt[0] = S.cnt[1] = S.cnt[2] = 0; S.nbr = 0; }
#ifdef FM_PL_TIMING
    long long t0 = clock64(), t1 = 0, t2 = 0;
#endif
    const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
    PlTile T;
    if constexpr (PK) T = PlTile{S.e, S.h, S.t, nullptr, S.res.r2, S.f, &S.nbr, tyi * PT_H, txi * PT_W, S.dirty};
    else T = PlTile{S.e, S.h, S.t, S.res.r, nullptr, S.f, &S.nbr, tyi * PT_H, txi * PT_W, S.dirty};
    // the generic item path (steps > 1 or fused) writes every row back
    if (tid < PT_H) S.dirty[tid] = (steps == 1 && !fused) ? 0 : 1;
    const int r0 = T.r0, c0 = T.c0;
    int32_t *stage = (int32_t *)&S.list[0][0];   // rS staging (the lists are built afterwards)
    // load.  TMA (maps != nullptr): one thread issues the plane copies, the halo rows and
    // columns arrive inside the height box; else cp.async, thread = (row, 4-column chunk).
    const bool tma = maps != nullptr;
    if (tma) {
        fence_proxy_async_smem();   // this visit's async writes come after every earlier smem access
        __syncthreads();
        if (tid == 0) {
            constexpr unsigned bytes = 3 * PT_H * PT_W * 4 + (PT_H + 2) * PL_HS * 4 + (PK ? 0 : 4 * PT_H * PT_W * 4);
            mbar_expect(&S.mbar, bytes);
            tma_load_2d(S.e, &maps->e, c0, r0, &S.mbar);
            tma_load_2d(S.t, &maps->t, c0, r0, &S.mbar);
            tma_load_2d(stage, &maps->s, c0, r0, &S.mbar);
            tma_load_2d(S.h, &maps->h, c0 - PL_HC, r0 - 1, &S.mbar);
            if constexpr (!PK)
                for (int k = 0; k < 4; k++) tma_load_2d(S.res.r[k], &maps->r[k], c0, r0, &S.mbar);
        }
    }
    for (int u = tid; u < PT_H * (PT_W / 4); u += PL_NT) {   // thread = (row, 4-column chunk)
        const int lrow = u >> 3, ch = u & 7;
        const int r = r0 + lrow, cb = c0 + 4 * ch;
        const int li = lrow * PT_W + 4 * ch, hi = (lrow + 1) * HS + PL_HC + 4 * ch;
        if (tma) {
            // the packed instance's residual fields are assembled from registers
            if constexpr (PK) {
                if (r < g.H && cb + 4 <= g.W) {
                    const int64_t p = (int64_t)r * g.W + cb;
                    const int4 a = __ldcg((const int4 *)(g.rR + p)), b = __ldcg((const int4 *)(g.rL + p));
                    const int4 d = __ldcg((const int4 *)(g.rD + p)), u = __ldcg((const int4 *)(g.rU + p));
                    S.res.r2[li + 0] = pk_pack(a.x, b.x, d.x, u.x);
                    S.res.r2[li + 1] = pk_pack(a.y, b.y, d.y, u.y);
                    S.res.r2[li + 2] = pk_pack(a.z, b.z, d.z, u.z);
                    S.res.r2[li + 3] = pk_pack(a.w, b.w, d.w, u.w);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        const bool in = r < g.H && cb + j < g.W;
                        const int64_t p = in ? (int64_t)r * g.W + cb + j : 0;
                        S.res.r2[li + j] = in ? pk_pack(__ldcg(g.rR + p), __ldcg(g.rL + p), __ldcg(g.rD + p), __ldcg(g.rU + p)) : make_uint2(0u, 0u);
                    }
                }
            }
        } else if (r < g.H && cb + 4 <= g.W && (g.W & 3) == 0) {            const int64_t p = (int64_t)r * g.W + cb;
            cp_async16(&S.e[li], g.e + p);
            if constexpr (PK) {
                const int4 a = __ldcg((const int4 *)(g.rR + p)), b = __ldcg((const int4 *)(g.rL + p));
                const int4 d = __ldcg((const int4 *)(g.rD + p)), u = __ldcg((const int4 *)(g.rU + p));
                S.res.r2[li + 0] = pk_pack(a.x, b.x, d.x, u.x);
                S.res.r2[li + 1] = pk_pack(a.y, b.y, d.y, u.y);
                S.res.r2[li + 2] = pk_pack(a.z, b.z, d.z, u.z);
                S.res.r2[li + 3] = pk_pack(a.w, b.w, d.w, u.w);
            } else {
                cp_async16(&S.res.r[0][li], g.rR + p);
                cp_async16(&S.res.r[1][li], g.rL + p);
                cp_async16(&S.res.r[2][li], g.rD + p);
                cp_async16(&S.res.r[3][li], g.rU + p);
            }
            cp_async16(&S.t[li], g.rT + p);
            cp_async16(&S.h[hi], g.h + p);
            cp_async16(&stage[li], g.rS + p);
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const bool in = r < g.H && cb + j < g.W;
                const int64_t p = in ? (int64_t)r * g.W + cb + j : 0;
                cp_async4(&S.e[li + j], g.e + p, in);
                if constexpr (PK) {
                    S.res.r2[li + j] = in ? pk_pack(__ldcg(g.rR + p), __ldcg(g.rL + p), __ldcg(g.rD + p), __ldcg(g.rU + p)) : make_uint2(0u, 0u);
                } else {
                    cp_async4(&S.res.r[0][li + j], g.rR + p, in);
                    cp_async4(&S.res.r[1][li + j], g.rL + p, in);
                    cp_async4(&S.res.r[2][li + j], g.rD + p, in);
                    cp_async4(&S.res.r[3][li + j], g.rU + p, in);
                }
                cp_async4(&S.t[li + j], g.rT + p, in);
                cp_async4(&S.h[hi + j], g.h + p, in);
                cp_async4(&stage[li + j], g.rS + p, in);
            }
        }
    }
    // halo heights (a snapshot: stale reads are the lock-free argument's business) and
    // the inboxes of the border pixels, both issued while the copies are in flight
    int32_t inbox = 0, peer_h = 0;
    int ib_li = -1, ib_dir = 0, peer_hidx = -1;
    if (tid < 4 * PT_W) {
        const int side = tid / PT_W, i = tid % PT_W;
        int r, cc, hidx;
        if (side == 0) { r = r0 - 1; cc = c0 + i; hidx = PL_HC + i; }
        else if (side == 1) { r = r0 + PT_H; cc = c0 + i; hidx = (PT_H + 1) * HS + PL_HC + i; }
        else if (side == 2) { r = r0 + i; cc = c0 - 1; hidx = (i + 1) * HS + PL_HC - 1; }
        else { r = r0 + i; cc = c0 + PT_W; hidx = (i + 1) * HS + PL_HC + PT_W; }
        const bool hin = r >= 0 && r < g.H && cc >= 0 && cc < g.W;
        if (side < 2 && !hin && cc < g.W && ((r < 0 && g.has_up) || (r == g.H && g.has_dn))) {
            peer_h = ld_cg((r < 0 ? g.up.h : g.dn.h) + cc);   // row bands: the neighbour band's row
            peer_hidx = hidx;                                  // (stored after the TMA wait)
        } else if (!tma) {
            cp_async4(&S.h[hidx], g.h + (hin ? (int64_t)r * g.W + cc : 0), hin);
        }
        // border pixel of this side and its inbox (flow parked by the neighbour tile)
        const int lr = side == 0 ? 0 : side == 1 ? PT_H - 1 : i;
        const int lc = side == 2 ? 0 : side == 3 ? PT_W - 1 : i;
        const int pr = r0 + lr, pc = c0 + lc;
        const bool has = pr < g.H && pc < g.W &&
                         (side == 0 ? pr > g.rmin : side == 1 ? pr + 1 < g.hlim : side == 2 ? pc > 0 : pc + 1 < g.W);
        if (has) {
            const int64_t p = (int64_t)pr * g.W + pc;
            inbox = atomicExch((side < 2 ? g.inflow_v : g.inflow_h) + p, 0);
            ib_li = lr * PT_W + lc;
            ib_dir = side == 0 ? 3 : side == 1 ? 2 : side == 2 ? 1 : 0;   // residual toward the sender
        }
    }
    if (tma) {
        mbar_wait(&S.mbar, tma_phase);
        tma_phase ^= 1u;
    } else {
        cp_async_wait_all();
    }
    if (peer_hidx >= 0) S.h[peer_hidx] = peer_h;
    __syncthreads();
    if (inbox) {
        S.dirty[ib_li >> 5] = 1;
        atomicAdd(&S.e[ib_li], inbox);          // a corner pixel has two inboxes
        if constexpr (PK) atomicAdd(reinterpret_cast<uint32_t *>(S.res.r2) + 2 * ib_li + (ib_dir >> 1), (uint32_t)inbox << (16 * (ib_dir & 1)));
        else S.res.r[ib_dir][ib_li] += inbox;
    }
#pragma unroll
    for (int k = 0; k < PL_ROWS; k++) {
        const int lr = ty + k * PL_TY;
        const int r = r0 + lr, c = c0 + tx;
        const int li = lr * PT_W + tx;
        S.f[li] = (r < g.H && c < g.W) ? (stage[li] > 0 ? 1 : 0) : 2;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < PL_ROWS; k++) {
        const int lr = ty + k * PL_TY;
        const int li = lr * PT_W + tx;
        pl_append_warp(S.e[li] > 0 && S.h[(lr + 1) * HS + PL_HC + tx] < V && !(S.f[li] & 2), li, &S.cnt[0], S.list[0]);
    }
#ifdef FM_PL_TIMING
    t1 = clock64();
#endif
    // dense passes: the whole CTA, one barrier per pass
    const bool simple = steps == 1 && !fused;
    int it = 0;
    bool solo = false;
    // list counters rotate through S.cnt[0..2] (current / next / cleared for the pass
    // after) and the two lists swap: no per-pass modulo arithmetic
    int cc = 0, cn = 1, cz = 2;
    uint16_t *lin = S.list[0], *lout = S.list[1];
    const int solo_max = g.solo_max;
    const int wbase = tid & ~31;
    for (; it < k_local; it++) {
        __syncthreads();
        const int n = S.cnt[cc];
        if (n <= solo_max) { solo = n > 0; break; }
        C.passes++;
        C.items += n;
        int *cnt_next = &S.cnt[cn];
        if (tid == 0) S.cnt[cz] = 0;
        for (int base = 0; base + wbase < n; base += PL_NT) {   // warp-uniform bound
            const int i = base + tid;
            int recv = -1;
            const int li = i < n ? lin[i] : 0;
            bool keep;
            if constexpr (PK) keep = i < n && pk_op1(g, T, li, &recv, C.pushes, C.relabels);   // simple only
            else keep = i < n && (simple ? pl_op1(g, T, li, &recv, C.pushes, C.relabels)
                                         : pl_item(g, T, li, steps, fused, cnt_next, lout, &recv, C.pushes, C.relabels));
            pl_append2_warp(keep, li, recv >= 0, recv, cnt_next, lout);
        }
        const int t = cc; cc = cn; cn = cz; cz = t;
        uint16_t *tl = lin; lin = lout; lout = tl;
    }
    // sparse passes: warp 0 alone, warp-synchronous
#ifdef FM_PL_TIMING
    if (solo && tid == 0) C.solo++;
    const long long ts0 = clock64();
    const int it_dense = it;
#endif
    if (solo && tid < 32 && simple) {
        // one warp is the only reader and writer of the lists now: the next list's
        // length is the warp's own running count (no shared counter round trip)
        int n = S.cnt[cc];
        const unsigned lt = (1u << tid) - 1;
        const int it_end = g.k_solo > 0 ? min(k_local, it + g.k_solo) : k_local;
        for (; it < it_end && n > 0; it++) {
            C.passes++;
            C.items += n;
            int nn = 0;
            for (int base = 0; base < n; base += 32) {
                const int i = base + tid;
                int recv = -1;
                const int li = i < n ? lin[i] : 0;
                bool keep;
                if constexpr (PK) keep = i < n && pk_op1(g, T, li, &recv, C.pushes, C.relabels);
                else keep = i < n && pl_op1(g, T, li, &recv, C.pushes, C.relabels);
                const unsigned ma = __ballot_sync(0xffffffffu, keep), mb = __ballot_sync(0xffffffffu, recv >= 0);
                if (keep) lout[nn + __popc(ma & lt)] = (uint16_t)li;
                if (recv >= 0) lout[nn + __popc(ma) + __popc(mb & lt)] = (uint16_t)recv;
                nn += __popc(ma) + __popc(mb);
            }
            __syncwarp();
            n = nn;
            uint16_t *tl = lin; lin = lout; lout = tl;
        }
    } else if (!PK && solo && tid < 32) {
        for (; it < k_local; it++) {
            __syncwarp();
            const int n = S.cnt[cc];
            if (n == 0) break;
            C.passes++;
            C.items += n;
            int *cnt_next = &S.cnt[cn];
            if (tid == 0) S.cnt[cz] = 0;
            __syncwarp();
            for (int base = 0; base < n; base += 32) {
                const int i = base + tid;
                int recv = -1;
                const int li = i < n ? lin[i] : 0;
                bool keep = false;
                if constexpr (!PK)
                    keep = i < n && (simple ? pl_op1(g, T, li, &recv, C.pushes, C.relabels)
                                            : pl_item(g, T, li, steps, fused, cnt_next, lout, &recv, C.pushes, C.relabels));
                pl_append2_warp(keep, li, recv >= 0, recv, cnt_next, lout);
            }
            const int t = cc; cc = cn; cn = cz; cz = t;
            uint16_t *tl = lin; lin = lout; lout = tl;
        }
    }
#ifdef FM_PL_TIMING
    if (tid == 0) { C.t_solo += clock64() - ts0; C.dense_passes += it_dense; C.solo_passes += it - it_dense; }
#endif
    __syncthreads();
#ifdef FM_PL_TIMING
    t2 = clock64();
#endif
    bool act = false;
#pragma unroll
    for (int k = 0; k < PL_ROWS; k++) {
        const int lr = ty + k * PL_TY;
        const int r = r0 + lr, c = c0 + tx;
        const int li = lr * PT_W + tx;
        if (r < g.H && c < g.W) {
            const int64_t p = (int64_t)r * g.W + c;
            const int32_t e = S.e[li], h = S.h[(lr + 1) * HS + PL_HC + tx];
            act |= (e > 0 && h < V && !(S.f[li] & 2));
            if (!S.dirty[lr]) continue;   // untouched row (warp-uniform): global state unchanged
            g.e[p] = e;
            g.h[p] = h;
            if constexpr (PK) {
                const uint2 w = S.res.r2[li];
                g.rR[p] = (int32_t)(w.x & 0xffff); g.rL[p] = (int32_t)(w.x >> 16);
                g.rD[p] = (int32_t)(w.y & 0xffff); g.rU[p] = (int32_t)(w.y >> 16);
            } else {
                g.rR[p] = S.res.r[0][li]; g.rL[p] = S.res.r[1][li];
                g.rD[p] = S.res.r[2][li]; g.rU[p] = S.res.r[3][li];
            }
            g.rT[p] = S.t[li];
        }
    }
    const bool any = __syncthreads_or(act) != 0;
#ifdef FM_PL_TIMING
    if (tid == 0) { C.t_load += t1 - t0; C.t_pass += t2 - t1; C.t_store += clock64() - t2; C.visits++; }
#endif
    return any;
}

// ----------------------------------------------------------------------------
// One push round as a CUDA graph: a while-conditional node whose body is a single
// pr_list_kernel launch.  The launch's last CTA to finish evaluates the round's
// triggers -- idle launch, launch cap, relabel budget at batch boundaries (the host
// loop's checks, in the same order) -- arms the tile queue for the next launch and
// sets the loop condition, so a round runs without a host round trip per batch.
// ----------------------------------------------------------------------------
struct PrCtl {
    int32_t parity, done, cap, batch, stop, processed, finished, pad;
    long long budget;
    unsigned long long tiles;
};

// the round's control block written by a one-thread kernel (its value travels as a
// launch argument): an H2D memcpy would queue on the copy engine behind a batch
// solve's 400 MB plane transfer (fm_grid_solve_host_batch)
__global__ void prctl_set_kernel(PrCtl *dst, PrCtl v) { *dst = v; }

// Narrow host capacity planes (uint8 / uint16, fm_grid_solve_host_batch elem_bytes 1 / 2)
// cross PCIe narrow and are widened to the int32 input planes on the device: 16 bytes of
// narrow values per thread step, stored as int4 (HBM-bound, ~0.1 ms for six 4096^2 planes
// against 5.5 ms less PCIe).
template <typename T>
__global__ void widen_planes_kernel(const T *src, int32_t *dst, int64_t n) {
    constexpr int PER = 16 / sizeof(T);
    const int64_t nv = n / PER;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(src) + i);
        const T *e = reinterpret_cast<const T *>(&v);
        int4 *o = reinterpret_cast<int4 *>(dst + i * PER);
#pragma unroll
        for (int k = 0; k < PER / 4; k++) __stcs(o + k, make_int4(e[4 * k], e[4 * k + 1], e[4 * k + 2], e[4 * k + 3]));
    }
    for (int64_t i = nv * PER + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i];
}

#ifndef FM_PK_MINBLOCKS
#define FM_PK_MINBLOCKS 8
#endif
template <bool PK>
__global__ void __launch_bounds__(PL_NT, PK ? FM_PK_MINBLOCKS : FM_PL_MINBLOCKS) pr_list_kernel(GridDev g, int k_local, int steps, int fused,
                                                                       int parity_arg, int32_t *processed,
                                                                       unsigned long long *ops,
                                                                       PrCtl *ctl, cudaGraphConditionalHandle loop,
                                                                       const __grid_constant__ PlMaps maps, int use_tma) {
    __shared__ PlSmemT<PK> S;
    const int tid = threadIdx.y * PT_W + threadIdx.x;
    unsigned tma_phase = 0;
    if (use_tma) {
        if (tid == 0) mbar_init(&S.mbar);
        __syncthreads();
    }
    // graph launches read the launch parity from the round's control block (processed
    // then points into it); host launches pass it as an argument
    const int parity = ctl ? __ldcg(&ctl->parity) : parity_arg;
    PlCounters C;
    for (;;) {
        __syncthreads();
        if (tid == 0) S.tile = tq_take(g.pq, parity, 0, 0);
        __syncthreads();
        const int tile = S.tile;
        if (tile < 0) break;
        const bool any_act = pl_visit(g, S, tile, k_local, steps, fused, C, use_tma ? &maps : nullptr, tma_phase);
        if (tid == 0) {
            if (any_act) tq_push(g.pq, parity ^ 1, tile);
            g.touched[tile] = 1;
            const int nb = S.nbr;
            if (nb & 1) { tq_push(g.pq, parity ^ 1, tile + 1); g.touched[tile + 1] = 1; }
            if (nb & 2) { tq_push(g.pq, parity ^ 1, tile - 1); g.touched[tile - 1] = 1; }
            // row bands: a push out of the band's first / last tile row went to the
            // neighbour band's inbox; raise its external-push flag for that tile (the
            // pushers fenced their inbox adds at system scope before the visit's barrier)
            const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
            if (nb & 4) {
                if (tyi + 1 < g.nty) { tq_push(g.pq, parity ^ 1, tile + g.ntx); g.touched[tile + g.ntx] = 1; }
                else if (atomicExch(g.dn.ext + txi, 1) == 0) atomicAdd(g.ext_ctr + 0, 1ull);
            }
            if (nb & 8) {
                if (tyi > 0) { tq_push(g.pq, parity ^ 1, tile - g.ntx); g.touched[tile - g.ntx] = 1; }
                else if (atomicExch(g.up.ext + txi, 1) == 0) atomicAdd(g.ext_ctr + 0, 1ull);
            }
            atomicAdd(processed, 1);
        }
    }
    block_add_i64<PL_NT / 32>(C.pushes, ops + 0);
    block_add_i64<PL_NT / 32>(C.relabels, ops + 1);
    if (tid == 0) {   // diagnostics: passes run and list items dealt (ops[3], ops[4]) -- thread 0 saw them all
        if (C.passes) atomicAdd(ops + 3, (unsigned long long)C.passes);
        if (C.items) atomicAdd(ops + 4, (unsigned long long)C.items);
#ifdef FM_PL_TIMING
        atomicAdd(ops + 6, (unsigned long long)C.t_load); atomicAdd(ops + 7, (unsigned long long)C.t_pass);
        atomicAdd(ops + 8, (unsigned long long)C.t_store); atomicAdd(ops + 9, (unsigned long long)C.visits);
        atomicAdd(ops + 10, (unsigned long long)C.solo);
        atomicAdd(ops + 11, (unsigned long long)C.t_solo); atomicAdd(ops + 12, (unsigned long long)C.dense_passes);
        atomicAdd(ops + 13, (unsigned long long)C.solo_passes);
#endif
    }
    if (ctl && tid == 0) {
        __threadfence();
        if (atomicAdd(&ctl->finished, 1) == (int)gridDim.x - 1) {   // last CTA: round control
            __threadfence();
            const int nproc = __ldcg(&ctl->processed);
            const int done = ctl->done + 1;
            const bool stop = nproc == 0 || done >= ctl->cap ||
                              (done % ctl->batch == 0 && (long long)__ldcg(ops + 1) >= ctl->budget);
            const int pn = parity ^ 1;
            g.pq.cnt[pn ? 0 : 2] = 0;              // tq_arm for the next launch
            g.pq.cnt[(pn ? 0 : 2) + 1] = 0;
            ctl->done = done;
            ctl->tiles += nproc;
            ctl->parity = pn;
            ctl->stop = stop;
            if (!stop) ctl->processed = 0;         // kept when stopping: 0 marks an idle launch
            ctl->finished = 0;
            __threadfence();
            cudaGraphSetConditional(loop, stop ? 0u : 1u);
        }
    }
}

// Row bands: before a push launch of parity p, zero the list words it needs (as
// tq_arm) and queue the tiles a neighbour band pushed flow into (external-push flags,
// [0, ntx) = our top tile row, [ntx, 2 ntx) = our bottom tile row).  One CTA.
__global__ void band_arm_kernel(GridDev g, int p) {
    if (threadIdx.x == 0) { g.pq.cnt[p ? 0 : 2] = 0; g.pq.cnt[(p ? 0 : 2) + 1] = 0; }
    __syncthreads();
    unsigned long long took = 0;
    for (int i = threadIdx.x; i < 2 * g.ntx; i += blockDim.x) {
        if (*(volatile int32_t *)(g.ext + i) == 0 || atomicExch(g.ext + i, 0) == 0) continue;
        took++;
        tq_push(g.pq, p, i < g.ntx ? i : (g.nty - 1) * g.ntx + (i - g.ntx));
    }
    if (took) atomicAdd(g.ext_ctr + 1, took);
}

// fold every parked inbox into e and the reverse residual (coordinator point)
__global__ void integrate_inflow_kernel(GridDev g) {
    const int tile = blockIdx.x;
    const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
    const int r0 = tyi * PT_H, c0 = txi * PT_W;
    const int i = threadIdx.x;  // 0..127: top, bottom, left, right
    const int side = i / PT_W, j = i % PT_W;
    int r, c;
    if (side == 0) { r = r0; c = c0 + j; }
    else if (side == 1) { r = r0 + PT_H - 1; c = c0 + j; }
    else if (side == 2) { r = r0 + j; c = c0; }
    else { r = r0 + j; c = c0 + PT_W - 1; }
    if (r >= g.H || c >= g.W) return;
    const int64_t p = (int64_t)r * g.W + c;
    // a tile corner is visited by two threads (one per side): e needs an atomic
    if (side == 0 && r > g.rmin) { const int32_t d = g.inflow_v[p]; if (d) { g.inflow_v[p] = 0; atomicAdd(g.e + p, d); g.rU[p] += d; } }
    if (side == 1 && r + 1 < g.hlim) { const int32_t d = g.inflow_v[p]; if (d) { g.inflow_v[p] = 0; atomicAdd(g.e + p, d); g.rD[p] += d; } }
    if (side == 2 && c > 0) { const int32_t d = g.inflow_h[p]; if (d) { g.inflow_h[p] = 0; atomicAdd(g.e + p, d); g.rL[p] += d; } }
    if (side == 3 && c + 1 < g.W) { const int32_t d = g.inflow_h[p]; if (d) { g.inflow_h[p] = 0; atomicAdd(g.e + p, d); g.rR[p] += d; } }
}

// ----------------------------------------------------------------------------
// cancel_violations (maxflow_par.py:132-154), opt-in: saturate every residual arc
// whose tail sits more than one level above its head.  Mates of cancelled arcs
// have the lower endpoint as tail and never violate, so arcs are independent.
// ----------------------------------------------------------------------------
__global__ void cancel_kernel(GridDev g, unsigned long long *count) {
    const int64_t HW = (int64_t)g.H * g.W;
    long long cnt = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < HW;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = (int32_t)(p / g.W), c = (int32_t)(p - (int64_t)r * g.W);
        if (false) continue;
        const int32_t hp = g.h[p];
        int32_t moved = 0;
        const int32_t rt = g.rT[p];
        if (rt > 0 && hp > 1) { g.rT[p] = 0; moved += rt; cnt++; }
        const int32_t rs = g.rS[p];
        if (rs > 0 && hp > g.V + 1) { g.rS[p] = 0; moved += rs; cnt++; }
        struct { int ok; int64_t q; int32_t *fw, *bw; } nb[4] = {
            {c + 1 < g.W, p + 1, g.rR, g.rL}, {c > 0, p - 1, g.rL, g.rR},
            {r + 1 < g.H, p + g.W, g.rD, g.rU}, {r > 0, p - g.W, g.rU, g.rD}};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (!nb[k].ok) continue;
            const int32_t rr = nb[k].fw[p];
            if (rr > 0 && hp > g.h[nb[k].q] + 1) {
                nb[k].fw[p] = 0;                 // only this thread touches this word now
                atomicAdd(nb[k].bw + nb[k].q, rr);
                atomicAdd(g.e + nb[k].q, rr);
                moved += rr;
                cnt++;
            }
        }
        if (moved) atomicSub(g.e + p, moved);
    }
    if (cnt) atomicAdd(count, (unsigned long long)cnt);
}

// ----------------------------------------------------------------------------
// K2: global relabel = backward BFS from t over residual arcs (maxflow_seq.py:119-146)
// computed as exact residual distances by tile-local multi-level relaxation:
// d(p) = 1 if r(p->t) > 0, else 1 + min{ d(q) : r(p->q) > 0 }.  Each CTA iterates
// its 32x32 tile in shared memory to a local fixpoint against a frozen halo; the
// host repeats sweeps until no tile changes (a chaotic Bellman-Ford that converges
// to the BFS levels because values only decrease and are always path lengths).
// ----------------------------------------------------------------------------
__global__ void bfs_init_kernel(GridDev g) {
    const int64_t HW = (int64_t)g.H * g.W;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < HW;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = (int32_t)(p / g.W), c = (int32_t)(p - (int64_t)r * g.W);
        uint8_t m = 0;
        if (c + 1 < g.W && g.rR[p] > 0) m |= M_R;
        if (c > 0 && g.rL[p] > 0) m |= M_L;
        if (r + 1 < g.H && g.rD[p] > 0) m |= M_D;
        if (r > 0 && g.rU[p] > 0) m |= M_U;
        if (g.rT[p] > 0) m |= M_T;
        if (false) m = 0;    // distance imported from the owner band
        g.mask[p] = m;
        g.dist[p] = (m & M_T) ? 1 : g.INF;
    }
}

// Frontier-driven: a tile is visited only when its own flag is set (all tiles on
// the first sweep, afterwards only tiles whose halo changed in the previous sweep).
// A visit runs to the tile's local fixpoint, writes back what changed and flags the
// neighbour tiles across every border that changed.  Converged when a sweep
// changes nothing.
__device__ __forceinline__ void flag_changed_borders(const GridDev &g, int tile, int tyi, int txi,
                                                     int bt, int bb, int bl, int br, int parity) {
    const auto in = [&](int t) { return !g.region || g.region[t]; };  // local relabel stays in R
    if (bt && tyi > 0 && in(tile - g.ntx)) tq_push(g.bq, parity, tile - g.ntx);
    if (bb && tyi + 1 < g.nty && in(tile + g.ntx)) tq_push(g.bq, parity, tile + g.ntx);
    if (bl && txi > 0 && in(tile - 1)) tq_push(g.bq, parity, tile - 1);
    if (br && txi + 1 < g.ntx && in(tile + 1)) tq_push(g.bq, parity, tile + 1);
}

__global__ void __launch_bounds__(256) bfs_tile_kernel(GridDev g, int parity, int all_tiles,
                                                       int32_t *changed_count) {
    __shared__ int32_t sd[TILE_H + 2][TILE_W + 2];
    __shared__ int s_tile, s_b[4];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * TILE_W + tx;
    for (;;) {
    __syncthreads();
    if (tid == 0) {
        s_tile = tq_take(g.bq, parity, all_tiles, g.ntx * g.nty);
        s_b[0] = s_b[1] = s_b[2] = s_b[3] = 0;
    }
    __syncthreads();
    const int tile = s_tile;
    if (tile < 0) break;
    const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
    const int c0 = txi * TILE_W, r0 = tyi * TILE_H;
    for (int i = tid; i < (TILE_H + 2) * (TILE_W + 2); i += TILE_W * BLK_Y) {
        const int lr = i / (TILE_W + 2), lc = i % (TILE_W + 2);
        const int r = r0 + lr - 1, c = c0 + lc - 1;
        sd[lr][lc] = (r >= 0 && r < g.H && c >= 0 && c < g.W) ? g.dist[(int64_t)r * g.W + c] : g.INF;
    }
    uint8_t m[ROWS_PER_THREAD];
    int32_t d0[ROWS_PER_THREAD];
    const int c = c0 + tx;
#pragma unroll
    for (int k = 0; k < ROWS_PER_THREAD; k++) {
        const int r = r0 + ty + k * BLK_Y;
        m[k] = (r < g.H && c < g.W) ? g.mask[(int64_t)r * g.W + c] : 0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ROWS_PER_THREAD; k++) d0[k] = sd[ty + k * BLK_Y + 1][tx + 1];
    bool any = false;
    for (;;) {
        bool ch = false;
#pragma unroll
        for (int k = 0; k < ROWS_PER_THREAD; k++) {
            const int lr = ty + k * BLK_Y + 1, lc = tx + 1;
            const uint8_t mk = m[k];
            if (!mk) continue;
            const int32_t cur = sd[lr][lc];
            int32_t nd = cur;
            if (mk & M_R) nd = min(nd, sd[lr][lc + 1] + 1);
            if (mk & M_L) nd = min(nd, sd[lr][lc - 1] + 1);
            if (mk & M_D) nd = min(nd, sd[lr + 1][lc] + 1);
            if (mk & M_U) nd = min(nd, sd[lr - 1][lc] + 1);
            if (nd < cur) { sd[lr][lc] = nd; ch = true; }
        }
        if (!__syncthreads_or(ch)) break;
        any = true;
    }
    if (any) {
#pragma unroll
        for (int k = 0; k < ROWS_PER_THREAD; k++) {
            const int lr = ty + k * BLK_Y;
            const int r = r0 + lr;
            const int32_t v = sd[lr + 1][tx + 1];
            if (r < g.H && c < g.W && v != d0[k]) {
                g.dist[(int64_t)r * g.W + c] = v;
                if (lr == 0) s_b[0] = 1;
                if (lr == TILE_H - 1) s_b[1] = 1;
                if (tx == 0) s_b[2] = 1;
                if (tx == TILE_W - 1) s_b[3] = 1;
            }
        }
        __syncthreads();
        if (tid == 0) {
            flag_changed_borders(g, tile, tyi, txi, s_b[0], s_b[1], s_b[2], s_b[3], parity ^ 1);
            atomicAdd(changed_count, 1);
        }
    }
    }  // tile loop
}

// ----------------------------------------------------------------------------
// K2 (bit-parallel, default): the same tile fixpoint, one warp per 32x32 tile with
// the tile's residual arcs as bit planes (lane = tile row, bit = column).
//
// bfs_init_bits_kernel builds, per tile row, five words with warp ballots:
// R/L/D/U (pixel has a residual arc toward that neighbour) and T (arc to the sink).
// bfs_bits_kernel then runs a level-synchronous multi-source BFS inside the tile:
// level 1 = T pixels, every halo pixel (and imported ghost-row pixel) of distance v
// is a source entering at level v, and one level expands the whole tile with a few
// shifts, shuffles and ANDs:
//     N = ((F >> 1) & R) | ((F << 1) & L) | (F_below & D) | (F_above & U),  N &= ~seen
// Empty level ranges jump straight to the next halo distance.  A visit recomputes
// the tile from its current halo; distances only fall as halos fall, and the
// write-back keeps min(old, new), so stale halo reads can never raise a label.
// The v1 per-pixel Jacobi kernel (bfs_tile_kernel) stays behind FM_BFS_BITS=0.
// ----------------------------------------------------------------------------
constexpr int BB_WARPS = 4;   // tiles in flight per CTA (one per warp)

__device__ __forceinline__ uint32_t bits_row(const GridDev &g, int tile, int lr, int lane) {
    const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
    const int r = tyi * PT_H + lr, c = txi * PT_W + lane;
    const bool in = r < g.H && c < g.W;
    const int64_t p = (int64_t)r * g.W + c;
    const bool aR = in && c + 1 < g.W && g.rR[p] > 0;
    const bool aL = in && c > 0 && g.rL[p] > 0;
    const bool aD = in && r + 1 < g.hlim && g.rD[p] > 0;   // band mode: arcs into the neighbour band
    const bool aU = in && r > g.rmin && g.rU[p] > 0;
    const bool aT = in && g.rT[p] > 0;
    const uint32_t w[5] = {__ballot_sync(0xffffffffu, aR), __ballot_sync(0xffffffffu, aL),
                           __ballot_sync(0xffffffffu, aD), __ballot_sync(0xffffffffu, aU),
                           __ballot_sync(0xffffffffu, aT)};
    uint32_t *B = g.rbits + (size_t)tile * 160 + lr;
    const uint32_t wk = lane == 0 ? w[0] : lane == 1 ? w[1] : lane == 2 ? w[2] : lane == 3 ? w[3] : w[4];
    if (lane < 5) B[lane * 32] = wk;
    if (r < g.H && c < g.W) g.dist[p] = aT ? 1 : g.INF;
    return w[4];
}

// bits_row for rows lr0 .. lr0 + 3 of a tile with all 20 plane loads issued before the
// first ballot (memory-level parallelism: the preparation pass is HBM-bound)
__device__ __forceinline__ void bits_rows4(const GridDev &g, int tile, int lr0, int lane) {
    const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
    const int c = txi * PT_W + lane;
    int32_t vR[4], vL[4], vD[4], vU[4], vT[4];
    bool in[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int r = tyi * PT_H + lr0 + k;
        in[k] = r < g.H && c < g.W;
        const int64_t p = in[k] ? (int64_t)r * g.W + c : 0;
        vR[k] = in[k] ? __ldcs(g.rR + p) : 0;
        vL[k] = in[k] ? __ldcs(g.rL + p) : 0;
        vD[k] = in[k] ? __ldcs(g.rD + p) : 0;
        vU[k] = in[k] ? __ldcs(g.rU + p) : 0;
        vT[k] = in[k] ? __ldcs(g.rT + p) : 0;
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int r = tyi * PT_H + lr0 + k;
        const bool aR = in[k] && c + 1 < g.W && vR[k] > 0;
        const bool aL = in[k] && c > 0 && vL[k] > 0;
        const bool aD = in[k] && r + 1 < g.hlim && vD[k] > 0;
        const bool aU = in[k] && r > g.rmin && vU[k] > 0;
        const bool aT = in[k] && vT[k] > 0;
        const uint32_t w[5] = {__ballot_sync(0xffffffffu, aR), __ballot_sync(0xffffffffu, aL),
                               __ballot_sync(0xffffffffu, aD), __ballot_sync(0xffffffffu, aU),
                               __ballot_sync(0xffffffffu, aT)};
        uint32_t *B = g.rbits + (size_t)tile * 160 + lr0 + k;
        // lane k < 5 stores word k (a select chain: a dynamic index would put w[] on the stack)
        const uint32_t wk = lane == 0 ? w[0] : lane == 1 ? w[1] : lane == 2 ? w[2] : lane == 3 ? w[3] : w[4];
        if (lane < 5) B[lane * 32] = wk;
        if (in[k]) g.dist[(int64_t)r * g.W + c] = aT ? 1 : g.INF;
    }
}

// listed == 0: every tile; listed == 1: the tiles of bq.list[0] (local relabel region).
// (Seeding the ring with only the tiles that hold a sink arc is NOT enough: a tile
// without one next to a sink pixel on its neighbour's border is never notified -- that
// border value is 1 from the start and never "changes" -- so every tile is queued.)
__global__ void bfs_init_bits_kernel(GridDev g, int listed) {
    const int lane = threadIdx.x & 31;
    const int64_t nrows = listed ? (int64_t)__ldcg(g.bq.cnt + 0) * PT_H : (int64_t)g.ntx * g.nty * PT_H;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nrows;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int k = (int)(w / PT_H), lr = (int)(w % PT_H);
        const int tile = listed ? g.bq.list[0][k] : k;
        bits_row(g, tile, lr, lane);
    }
}

__device__ __forceinline__ int warp_min_i32(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__global__ void __launch_bounds__(32 * BB_WARPS) bfs_bits_kernel(GridDev g, int parity, int all_tiles,
                                                               int32_t *changed_count) {
    __shared__ int32_t s_d[BB_WARPS][PT_H * (PT_W + 1)];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t *sd = s_d[wid];
    const int INF = g.INF;
    for (;;) {
        int tile = 0;
        if (lane == 0) tile = tq_take(g.bq, parity, all_tiles, g.ntx * g.nty);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile < 0) break;
        const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
        const int r0 = tyi * PT_H, c0 = txi * PT_W;
        const uint32_t *B = g.rbits + (size_t)tile * 160;
        const uint32_t mR = B[lane], mL = B[32 + lane], mD = B[64 + lane], mU = B[96 + lane], mT = B[128 + lane];
        // halo distances: lane = column for the rows above / below, lane = row for the columns left / right
        const int cl = c0 + lane, rl = r0 + lane;
        const int ht = (r0 > 0 && cl < g.W) ? ld_cg(g.dist + (int64_t)(r0 - 1) * g.W + cl) : INF;
        const int hb = (r0 + PT_H < g.H && cl < g.W) ? ld_cg(g.dist + (int64_t)(r0 + PT_H) * g.W + cl) : INF;
        const int hl = (c0 > 0 && rl < g.H) ? ld_cg(g.dist + (int64_t)rl * g.W + c0 - 1) : INF;
        const int hr = (c0 + PT_W < g.W && rl < g.H) ? ld_cg(g.dist + (int64_t)rl * g.W + c0 + PT_W) : INF;
        // ghost rows (row bands) hold imported distances: sources, never recomputed
        const int g0 = -1, g1 = -1;   // (round-1 ghost rows; band halos now come from PeerView)
        const int gv0 = (g0 >= 0 && cl < g.W) ? ld_cg(g.dist + (int64_t)(r0 + g0) * g.W + cl) : INF;
        const int gv1 = (g1 >= 0 && cl < g.W) ? ld_cg(g.dist + (int64_t)(r0 + g1) * g.W + cl) : INF;
        uint32_t F = mT, seen = mT;
        for (uint32_t x = mT; x; x &= x - 1) sd[lane * (PT_W + 1) + __ffs(x) - 1] = 1;
        int L = 1;
        for (;;) {
            if (g0 >= 0) { const uint32_t s = __ballot_sync(0xffffffffu, gv0 == L); if (lane == g0) F |= s; }
            if (g1 >= 0) { const uint32_t s = __ballot_sync(0xffffffffu, gv1 == L); if (lane == g1) F |= s; }
            const uint32_t tb = __ballot_sync(0xffffffffu, ht == L);
            const uint32_t bb = __ballot_sync(0xffffffffu, hb == L);
            uint32_t up = __shfl_up_sync(0xffffffffu, F, 1);
            uint32_t dn = __shfl_down_sync(0xffffffffu, F, 1);
            if (lane == 0) up = tb;
            if (lane == 31) dn = bb;
            uint32_t N = ((F >> 1) & mR) | ((F << 1) & mL) | (dn & mD) | (up & mU);
            if (hr == L) N |= mR & 0x80000000u;
            if (hl == L) N |= mL & 1u;
            N &= ~seen;
            seen |= N;
            L++;
            for (uint32_t x = N; x; x &= x - 1) sd[lane * (PT_W + 1) + __ffs(x) - 1] = L;
            F = N;
            if (!__any_sync(0xffffffffu, F != 0)) {
                int m = INF;
                if (ht >= L) m = min(m, ht);
                if (hb >= L) m = min(m, hb);
                if (hl >= L) m = min(m, hl);
                if (hr >= L) m = min(m, hr);
                if (gv0 >= L) m = min(m, gv0);
                if (gv1 >= L) m = min(m, gv1);
                m = warp_min_i32(m);
                if (m >= INF) break;
                L = m;
            }
        }
        __syncwarp();
        // write back min(old, new); note which borders changed
        bool bt = false, bbot = false, bl = false, br = false;
        for (int i = 0; i < PT_H; i++) {
            const int r = r0 + i;
            if (r >= g.H) break;
            const uint32_t sr = __shfl_sync(0xffffffffu, seen, i);
            if (i == g0 || i == g1 || cl >= g.W || !((sr >> lane) & 1)) continue;
            const int64_t p = (int64_t)r * g.W + cl;
            const int nv = sd[i * (PT_W + 1) + lane];
            if (nv < ld_cg(g.dist + p)) {
                g.dist[p] = nv;
                bt |= i == 0;
                bbot |= i == PT_H - 1;
                bl |= lane == 0;
                br |= lane == PT_W - 1;
            }
        }
        const int b0 = __any_sync(0xffffffffu, bt), b1 = __any_sync(0xffffffffu, bbot);
        const int b2 = __any_sync(0xffffffffu, bl), b3 = __any_sync(0xffffffffu, br);
        if (lane == 0 && (b0 | b1 | b2 | b3)) {
            flag_changed_borders(g, tile, tyi, txi, b0, b1, b2, b3, parity ^ 1);
            atomicAdd(changed_count, 1);
        }
        __syncwarp();
    }
}

// ----------------------------------------------------------------------------
// K2 as ONE persistent launch (default): the tile fixpoint driven by a device work
// queue instead of host-synchronised sweeps.  A tile whose border distances fell
// queues its neighbours (flag-deduplicated); warps take tiles until the queue is
// empty and no tile is in flight (asynchronous chaotic relaxation: every value is a
// path length and only falls, so the fixpoint reached is the BFS distance whatever
// the order).  The queue is a ring of slots: a warp reserves slot `head++` and
// waits for it to be filled (tail++ by a producer) or for `pending` (queued + in
// flight tiles) to reach 0, which ends the launch.  Every CTA is resident (grid =
// occupancy), so a waiting warp never blocks the producer it waits for.
// ----------------------------------------------------------------------------
struct RingQ {
    int32_t *slot;          // cap entries, -1 = empty
    int32_t *flag;          // per tile: queued
    unsigned int *ctr;      // [0] head, [32] tail, [64] pending, [96] tile visits that changed a border (one line each)
                            // [248] timeout flag (band mode: a wait that exceeded the limit), [252] band-local
                            // done word (row bands: raised by the watcher warp when the shared pending hits 0)
    unsigned int *pend;     // the pending counter the launch ends on: ctr + 64, or (row bands)
                            // one counter shared by every band's ring (on band 0's device)
    int32_t cap;
    int32_t rerun;          // a tile found stale again while in flight: 1 rerun at once, 0 requeue
    int32_t incr;           // 1: a re-visit only propagates halo improvements (option BFS_INCR)
    int32_t ns0, ns1;       // idle-poll backoff (ns)
    int32_t sys;            // row bands: fences at system scope (peer GPUs read / count what we publish)
};

// Release / acquire accesses for the ring protocol (PTX memory model): a release store /
// CAS publishes the warp's earlier stores (ordered before it by __syncwarp), an acquire
// load / CAS makes the publisher's stores visible to the loads after it.  Cheaper than
// the sequentially consistent fence of __threadfence (MEMBAR.SC + L1 invalidate): a
// release is MEMBAR.ALL + the access, an acquire the access + L1 invalidate.  sys:
// system scope (row bands: the other side is a peer GPU).
__device__ __forceinline__ int ld_acquire(const int32_t *p, bool sys) {
    int v;
    if (sys) asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int32_t *p, int v, bool sys) {
    if (sys) asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
    else asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int cas_acq_rel(int32_t *p, int cmp, int val, bool sys) {
    int old;
    if (sys) asm volatile("atom.acq_rel.sys.global.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "l"(p), "r"(cmp), "r"(val) : "memory");
    else asm volatile("atom.acq_rel.gpu.global.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "l"(p), "r"(cmp), "r"(val) : "memory");
    return old;
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// initial content: tiles list0[0..*count0) (count0 != nullptr) or every tile
__global__ void ringq_init_kernel(RingQ q, int ntiles, const int32_t *list0, const int32_t *count0) {
    const int n0 = count0 ? __ldcg(count0) : ntiles;
    // flag words: bits 0-1 state (0 idle, 1 queued, 2 in flight, 3 stale in flight), bit 2
    // "visited in this launch" (incremental re-visits).  Every tile queued: every flag is
    // written here; a listed start has had its flags zeroed by the host first.
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < q.cap; i += gridDim.x * blockDim.x) {
        if (i < n0) {
            const int t = count0 ? list0[i] : i;
            q.slot[i] = t;
            q.flag[t] = 1;
        } else {
            q.slot[i] = -1;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        q.ctr[0] = 0; q.ctr[32] = n0; q.ctr[64] = n0; q.ctr[96] = 0;
        q.ctr[128] = 0; q.ctr[160] = 0; q.ctr[161] = 0; q.ctr[192] = 0; q.ctr[224] = n0;
        q.ctr[240] = q.ctr[241] = q.ctr[244] = q.ctr[245] = q.ctr[246] = q.ctr[247] = 0;
        q.ctr[248] = 0;
        q.ctr[252] = 0;   // band-local done word (row bands)
        for (int i = 208; i < 218; i++) q.ctr[i] = 0;
    }
}

// The global relabel's preparation in ONE launch (single band, default kernels): per tile
// row, the BFS arc words and distance seeds -- rebuilt from the residual planes only for
// tiles a push touched since the last relabel (full: every tile), else the seeds come
// from the tile's unchanged sink word --, the ring with every tile queued, the push work
// list's flags, and the relabel's counters.  Replaces bfs_init_bits + ringq_init + three
// memsets.  Touched flags are cleared by the finalize that follows the BFS.
template <bool WHOLE>   // WHOLE: whole tiles, ntx % 4 == 0 (the 4-tile-group pass)
__global__ void __launch_bounds__(256, WHOLE ? 4 : 6) relabel_init_kernel(GridDev g, RingQ q, int full, int integ,
                                                               unsigned long long *acc) {
    const int lane = threadIdx.x & 31;
    const int ntiles = g.ntx * g.nty;
    const int nquads = ntiles * (PT_H / 4);   // < 2^31: H * W < 2^30 (fm_grid_create)
    const int wstep = (gridDim.x * blockDim.x) >> 5;
    // consecutive warps take the same 4 rows of consecutive tiles: every plane is then
    // read as runs of adjacent 128-byte row segments (DRAM-friendly), not one segment
    // per 16 KB row stride
    // 32-bit index math (a 64-bit division per quad made this pass issue-bound)
    const auto tile_of = [&](int w) {
        const int rest = w / g.ntx;
        return (rest / (PT_H / 4)) * g.ntx + (w - rest * g.ntx);
    };
    int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if constexpr (WHOLE) {
        // whole tiles, 4 tiles per group: one image row of 4 tiles per warp iteration,
        // int4 loads (lane = 4 columns), the 32-bit arc words assembled from the lanes'
        // nibbles with 3 shuffles -- a quarter of the load and ballot instructions
        const int ngroups = g.ntx / 4;
        const int nunits = g.nty * PT_H * ngroups;
        const int j = lane >> 3, sh = 4 * (lane & 7);
        for (int u = w; u < nunits; u += wstep) {
            const int row = u / ngroups, tg = u - row * ngroups;   // row = image row
            const int ty = row / PT_H, lr = row - ty * PT_H;
            const int tile = ty * g.ntx + 4 * tg + j;
            const int c = (4 * tg + j) * PT_W + (sh);              // first of this lane's 4 columns
            const int64_t p = (int64_t)row * g.W + c;
            const bool tch = full || g.touched[tile];
            uint32_t *B = g.rbits + (size_t)tile * 160 + lr;
            uint32_t nR = 0, nL = 0, nD = 0, nU = 0, nT = 0;
            if (tch) {
                int4 R = __ldcs((const int4 *)(g.rR + p)), L = __ldcs((const int4 *)(g.rL + p));
                int4 D = __ldcs((const int4 *)(g.rD + p)), U = __ldcs((const int4 *)(g.rU + p));
                const int4 T = __ldcs((const int4 *)(g.rT + p));
                if (integ) {
                    // the push round's parked inboxes folded in here (integrate_inflow_kernel's
                    // work, fused): flow from the tile above / below into rows 0 / 31, from the
                    // left / right tile into columns 0 / 31; e and the residual toward the
                    // sender grow by it (a tile with inbox flow was marked touched by its sender)
                    const int k = lane & 7;
                    const bool vtop = lr == 0 && row > g.rmin, vbot = lr == PT_H - 1 && row + 1 < g.hlim;
                    const int4 dv = (vtop || vbot) ? __ldcg((const int4 *)(g.inflow_v + p)) : make_int4(0, 0, 0, 0);
                    const int dl = (k == 0 && c > 0) ? __ldcg(g.inflow_h + p) : 0;
                    const int dr = (k == 7 && c + 4 < g.W) ? __ldcg(g.inflow_h + p + 3) : 0;
                    const bool anyv = dv.x | dv.y | dv.z | dv.w;
                    if (anyv || dl || dr) {
                        int4 E = __ldcg((const int4 *)(g.e + p));
                        E.x += dv.x + dl; E.y += dv.y; E.z += dv.z; E.w += dv.w + dr;
                        *(int4 *)(g.e + p) = E;
                        if (anyv) {
                            *(int4 *)(g.inflow_v + p) = make_int4(0, 0, 0, 0);
                            int4 &V = vtop ? U : D;
                            V.x += dv.x; V.y += dv.y; V.z += dv.z; V.w += dv.w;
                            *(int4 *)((vtop ? g.rU : g.rD) + p) = V;
                        }
                        if (dl) { g.inflow_h[p] = 0; L.x += dl; g.rL[p] = L.x; }
                        if (dr) { g.inflow_h[p + 3] = 0; R.w += dr; g.rR[p + 3] = R.w; }
                    }
                }
                const auto nib = [](const int4 v) {
                    return (uint32_t)(v.x > 0) | ((uint32_t)(v.y > 0) << 1) | ((uint32_t)(v.z > 0) << 2) |
                           ((uint32_t)(v.w > 0) << 3);
                };
                nR = nib(R); nL = nib(L); nD = nib(D); nU = nib(U); nT = nib(T);
                if (c + 4 >= g.W) nR &= 0x7u;                // the last column has no right arc
                if (c == 0) nL &= 0xeu;                      // the first column no left arc
                if (!(row + 1 < g.hlim)) nD = 0;
                if (!(row > g.rmin)) nU = 0;
            } else {
                nT = (__ldcg(B + 128) >> sh) & 0xfu;         // untouched: the old sink word still holds
            }
            uint32_t wR = nR << sh, wL = nL << sh, wD = nD << sh, wU = nU << sh, wT = nT << sh;
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                wR |= __shfl_xor_sync(0xffffffffu, wR, o);
                wL |= __shfl_xor_sync(0xffffffffu, wL, o);
                wD |= __shfl_xor_sync(0xffffffffu, wD, o);
                wU |= __shfl_xor_sync(0xffffffffu, wU, o);
                wT |= __shfl_xor_sync(0xffffffffu, wT, o);
            }
            const int k = lane & 7;
            if (tch && k < 5) B[k * 32] = k == 0 ? wR : k == 1 ? wL : k == 2 ? wD : k == 3 ? wU : wT;
            const int INF = g.INF;
            *(int4 *)(g.dist + p) = make_int4((nT & 1u) ? 1 : INF, (nT & 2u) ? 1 : INF, (nT & 4u) ? 1 : INF,
                                              (nT & 8u) ? 1 : INF);
        }
    } else {
    // the tile's touched flag is loaded one iteration ahead (it gates the plane loads)
    uint8_t tch_next = 0;
    if (!full && w < nquads) tch_next = g.touched[tile_of(w)];
    for (; w < nquads; w += wstep) {
        const int tile = tile_of(w);
        const int lr0 = 4 * ((w / g.ntx) % (PT_H / 4));
        const bool tch = full || tch_next;
        if (!full && w + wstep < nquads) tch_next = g.touched[tile_of(w + wstep)];
        if (tch) {
            bits_rows4(g, tile, lr0, lane);
        } else {
            const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
            const int c = txi * PT_W + lane;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int r = tyi * PT_H + lr0 + k;
                const uint32_t tw = g.rbits[(size_t)tile * 160 + 128 + lr0 + k];
                if (r < g.H && c < g.W) g.dist[(int64_t)r * g.W + c] = ((tw >> lane) & 1u) ? 1 : g.INF;
            }
        }
    }
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < q.cap; i += gridDim.x * blockDim.x) {
        q.slot[i] = i < ntiles ? i : -1;
        if (i < ntiles) {
            q.flag[i] = 1;
            g.pq.flag[0][i] = 0;
            g.pq.flag[1][i] = 0;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        q.ctr[0] = 0; q.ctr[32] = ntiles; q.ctr[64] = ntiles; q.ctr[96] = 0;
        q.ctr[128] = 0; q.ctr[160] = 0; q.ctr[161] = 0; q.ctr[192] = 0; q.ctr[224] = ntiles;
        q.ctr[240] = q.ctr[241] = q.ctr[244] = q.ctr[245] = q.ctr[246] = q.ctr[247] = 0;
        q.ctr[248] = 0;
        for (int i = 208; i < 218; i++) q.ctr[i] = 0;
        g.pq.cnt[0] = g.pq.cnt[1] = g.pq.cnt[2] = g.pq.cnt[3] = 0;
        acc[0] = acc[1] = acc[2] = 0;
    }
}

// Tile states: 0 idle, 1 queued, 2 in flight, 3 in flight + stale again.  A tile is
// never processed by two warps at once (so a visit owns its pixels' distances); a
// visit that finds a neighbour in flight marks it 3 and the owner runs it again.  A
// claimed neighbour may live in a neighbour band's ring (peer memory): its slot / flag /
// tail words, our shared pending count.  (Claiming, counting and publishing happen at
// the end of a visit in ring_kernel: one pending update and one slot reservation per
// visit, since those counters are the hottest words of the launch.)

// Halo row above / below a tile (lane = column): the neighbour tile's border row, or
// in row-band mode the neighbour band's boundary row through peer memory.
__device__ __forceinline__ int halo_dist_top(const GridDev &g, int r0, int cl) {
    if (cl >= g.W) return g.INF;
    if (r0 > 0) return ld_cg(g.dist + (int64_t)(r0 - 1) * g.W + cl);
    return g.has_up ? ld_cg(g.up.dist + cl) : g.INF;
}
__device__ __forceinline__ int halo_dist_bot(const GridDev &g, int r0, int cl) {
    if (cl >= g.W) return g.INF;
    if (r0 + PT_H < g.H) return ld_cg(g.dist + (int64_t)(r0 + PT_H) * g.W + cl);
    return (g.has_dn && r0 + PT_H == g.H) ? ld_cg(g.dn.dist + cl) : g.INF;
}
__device__ __forceinline__ bool halo_cut_top(const GridDev &g, int r0, int cl) {
    if (cl >= g.W) return false;
    if (r0 > 0) return __ldcg(g.cut + (int64_t)(r0 - 1) * g.W + cl) != 0;
    return g.has_up && __ldcg(g.up.cut + cl) != 0;
}
__device__ __forceinline__ bool halo_cut_bot(const GridDev &g, int r0, int cl) {
    if (cl >= g.W) return false;
    if (r0 + PT_H < g.H) return __ldcg(g.cut + (int64_t)(r0 + PT_H) * g.W + cl) != 0;
    return g.has_dn && r0 + PT_H == g.H && __ldcg(g.dn.cut + cl) != 0;
}

// Border changes of one visit: which of the tile's own rows / columns moved (b0 top,
// b1 bottom, b2 left, b3 right) and whether anything on a border changed at all.
struct RingChange { int b0, b1, b2, b3, any; int r0, r1, r2, r3; };   // r*: border row / column reached (BFS)

// One BFS visit (warp per tile), K2: level-synchronous bit-parallel BFS of the tile
// from its sink arcs and halo distances (from scratch), or an incremental re-visit.
#ifdef FM_BFS_TIMING
struct BfsTm { long long ld = 0, lvl = 0, wb = 0, wait = 0, push = 0; };
#endif
__device__ __forceinline__ RingChange bfs_visit(const GridDev &g, const RingQ &q, int tile, bool visited, int32_t *sd,
                                                int lane
#ifdef FM_BFS_TIMING
                                                , int &lv, BfsTm &tm
#endif
                                                ) {
#ifdef FM_BFS_TIMING
    long long tA = clock64();
#endif
    const int INF = g.INF;
    const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
    const int r0 = tyi * PT_H, c0 = txi * PT_W;
    const int cl = c0 + lane, rl = r0 + lane;
    const uint32_t *B = g.rbits + (size_t)tile * 160;
    const uint32_t mR = B[lane], mL = B[32 + lane], mD = B[64 + lane], mU = B[96 + lane], mT = B[128 + lane];
    // Halo distances and the tile's own border distances (for change detection).  A
    // from-scratch visit recomputes the interior: a visit's halos are never larger than
    // the previous visit's (distances only fall and the owner is exclusive), so every
    // pixel it reaches gets a value <= the old one and is written without a read.
    const int ht = halo_dist_top(g, r0, cl);
    const int hb = halo_dist_bot(g, r0, cl);
    const int hl = (c0 > 0 && rl < g.H) ? ld_cg(g.dist + (int64_t)rl * g.W + c0 - 1) : INF;
    const int hr = (c0 + PT_W < g.W && rl < g.H) ? ld_cg(g.dist + (int64_t)rl * g.W + c0 + PT_W) : INF;
    const int last_r = min(PT_H, g.H - r0) - 1, last_c = min(PT_W, g.W - c0) - 1;
    const int ot = cl < g.W ? ld_cg(g.dist + (int64_t)r0 * g.W + cl) : INF;                 // own top row
    const int ob = cl < g.W ? ld_cg(g.dist + (int64_t)(r0 + last_r) * g.W + cl) : INF;      // own bottom row
    const int ol = rl < g.H ? ld_cg(g.dist + (int64_t)rl * g.W + c0) : INF;                  // own left column
    const int orr = rl < g.H ? ld_cg(g.dist + (int64_t)rl * g.W + c0 + last_c) : INF;        // own right column
    uint32_t seen = 0;
    const bool incr = q.incr && visited;
#ifdef FM_BFS_TIMING
    long long tB = 0;
#endif
    if (incr) {
        // Re-visit: the previous visit left a fixpoint for the halos it saw, and halos
        // only fall, so only pixels that a now-shorter halo path improves change.  Load
        // the current distances, seed the border pixels whose halo now gives a shorter
        // path, and run the level loop from there keeping only improved pixels.
        for (int i = 0; i < PT_H; i++)
            sd[i * (PT_W + 1) + lane] = (r0 + i < g.H && cl < g.W) ? ld_cg(g.dist + (int64_t)(r0 + i) * g.W + cl) : INF;
        __syncwarp();
#ifdef FM_BFS_TIMING
        tB = clock64();
#endif
        const uint32_t mU0 = __shfl_sync(0xffffffffu, mU, 0), mD31 = __shfl_sync(0xffffffffu, mD, PT_H - 1);
        // smallest halo value >= lo whose path improves a border pixel (INF: none)
        const auto next_seed = [&](int lo) -> int {
            int m = INF;
            if (ht >= lo && ht < INF && ((mU0 >> lane) & 1u) && ht + 1 < sd[lane]) m = min(m, ht);
            if (hb >= lo && hb < INF && ((mD31 >> lane) & 1u) && hb + 1 < sd[(PT_H - 1) * (PT_W + 1) + lane]) m = min(m, hb);
            if (hl >= lo && hl < INF && (mL & 1u) && hl + 1 < sd[lane * (PT_W + 1)]) m = min(m, hl);
            if (hr >= lo && hr < INF && (mR & 0x80000000u) && hr + 1 < sd[lane * (PT_W + 1) + PT_W - 1]) m = min(m, hr);
            return warp_min_i32(m);
        };
        int L = next_seed(0);
        uint32_t F = 0;
        while (L < INF) {
            const uint32_t tb = __ballot_sync(0xffffffffu, ht == L);
            const uint32_t bb = __ballot_sync(0xffffffffu, hb == L);
            uint32_t up = __shfl_up_sync(0xffffffffu, F, 1);
            uint32_t dn = __shfl_down_sync(0xffffffffu, F, 1);
            if (lane == 0) up = tb;
            if (lane == 31) dn = bb;
            uint32_t N = ((F >> 1) & mR) | ((F << 1) & mL) | (dn & mD) | (up & mU);
            if (hr == L) N |= mR & 0x80000000u;
            if (hl == L) N |= mL & 1u;
            uint32_t K = 0;   // the pixels level L+1 improves (own row: no cross-lane hazard)
            for (uint32_t x = N; x; x &= x - 1) {
                const int b = __ffs(x) - 1;
                int32_t *d = &sd[lane * (PT_W + 1) + b];
                if (L + 1 < *d) { *d = L + 1; K |= 1u << b; }
            }
            seen |= K;
            F = K;
            L++;
#ifdef FM_BFS_TIMING
            lv++;
#endif
            if (!__any_sync(0xffffffffu, F != 0)) {
                __syncwarp();
                L = next_seed(L);
            }
        }
        __syncwarp();
    } else {
        // level-synchronous BFS; sd[row][col] = level at which the pixel was reached
#ifdef FM_BFS_TIMING
        tB = clock64();
#endif
        uint32_t F = mT;
        seen = mT;
        for (uint32_t x = mT; x; x &= x - 1) sd[lane * (PT_W + 1) + __ffs(x) - 1] = 1;
        int L = 1;
        // the level stores of step L are issued after step L+1's shuffles, so they run
        // while the shuffles are in flight (P / PL: pixels reached last step, their level)
        uint32_t P = 0;
        int PL = 0;
        for (;;) {
            const uint32_t tb = __ballot_sync(0xffffffffu, ht == L);
            const uint32_t bb = __ballot_sync(0xffffffffu, hb == L);
            uint32_t up = __shfl_up_sync(0xffffffffu, F, 1);
            uint32_t dn = __shfl_down_sync(0xffffffffu, F, 1);
            for (uint32_t x = P; x; x &= x - 1) sd[lane * (PT_W + 1) + __ffs(x) - 1] = PL;
            if (lane == 0) up = tb;
            if (lane == 31) dn = bb;
            uint32_t N = ((F >> 1) & mR) | ((F << 1) & mL) | (dn & mD) | (up & mU);
            if (hr == L) N |= mR & 0x80000000u;
            if (hl == L) N |= mL & 1u;
            N &= ~seen;
            seen |= N;
            L++;
#ifdef FM_BFS_TIMING
            lv++;
#endif
            P = N;
            PL = L;
            F = N;
            if (!__any_sync(0xffffffffu, F != 0)) {
                int m = INF;
                if (ht >= L) m = min(m, ht);
                if (hb >= L) m = min(m, hb);
                if (hl >= L) m = min(m, hl);
                if (hr >= L) m = min(m, hr);
                m = warp_min_i32(m);
                if (m >= INF) break;
                L = m;
            }
        }
        __syncwarp();
    }
    // write back every reached pixel (lane = column); borders compared with the old values
#ifdef FM_BFS_TIMING
    const long long tC = clock64();
#endif
    const uint32_t any_seen = __ballot_sync(0xffffffffu, seen != 0);
    bool ct = false, cb = false;
    for (uint32_t rows = any_seen; rows; rows &= rows - 1) {
        const int i = __ffs(rows) - 1;
        const uint32_t sr = __shfl_sync(0xffffffffu, seen, i);
        if (((sr >> lane) & 1) && cl < g.W) {
            const int v = sd[i * (PT_W + 1) + lane];
            g.dist[(int64_t)(r0 + i) * g.W + cl] = v;
            ct |= i == 0 && v < ot;
            cb |= i == last_r && v < ob;
        }
    }
    // own left / right columns: lane = row
    const bool sl = (seen & 1u) && lane <= last_r;
    const bool sr_ = ((seen >> last_c) & 1u) && lane <= last_r;
    const bool cl_ = sl && sd[lane * (PT_W + 1)] < ol;
    const bool cr_ = sr_ && sd[lane * (PT_W + 1) + last_c] < orr;
    RingChange ch;
    ch.any = __ballot_sync(0xffffffffu, ct || cb || cl_ || cr_) != 0;
    ch.b0 = __any_sync(0xffffffffu, ct);
    ch.b1 = __any_sync(0xffffffffu, cb);
    ch.b2 = __any_sync(0xffffffffu, cl_);
    ch.b3 = __any_sync(0xffffffffu, cr_);
    ch.r0 = __shfl_sync(0xffffffffu, seen, 0) != 0;
    ch.r1 = __shfl_sync(0xffffffffu, seen, last_r) != 0;
    ch.r2 = __any_sync(0xffffffffu, sl);
    ch.r3 = __any_sync(0xffffffffu, sr_);
#ifdef FM_BFS_TIMING
    const long long tD = clock64();
    tm.ld += tB - tA; tm.lvl += tC - tB; tm.wb += tD - tC;
#endif
    return ch;
}

// One cut visit (warp per tile), K3: the seeded-reach closure with the tile's
// incoming residual arcs as bit planes (lane = tile row, bit = column),
//     S |= ((S >> 1) & inR) | ((S << 1) & inL) | (S_below & inD) | (S_above & inU)
// plus the halo's cut bits, until no word changes; the pixels it adds are written.
__device__ __forceinline__ RingChange cut_visit(const GridDev &g, int tile, int lane) {
    const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
    const int r0 = tyi * PT_H, c0 = txi * PT_W;
    const int cl = c0 + lane, rl = r0 + lane;
    const uint32_t *B = g.rbits + (size_t)tile * 160;
    const uint32_t iR = B[lane], iL = B[32 + lane], iD = B[64 + lane], iU = B[96 + lane];
    // current cut words of the tile (row i built by a ballot over its 32 columns)
    uint32_t S = 0;
#pragma unroll 8
    for (int i = 0; i < PT_H; i++) {
        const int r = r0 + i;
        const bool b = r < g.H && cl < g.W && __ldcg(g.cut + (int64_t)r * g.W + cl);
        const uint32_t wv = __ballot_sync(0xffffffffu, b);
        if (lane == i) S = wv;
    }
    const uint32_t S0 = S;
    const uint32_t top = __ballot_sync(0xffffffffu, halo_cut_top(g, r0, cl));
    const uint32_t bot = __ballot_sync(0xffffffffu, halo_cut_bot(g, r0, cl));
    const bool hl = c0 > 0 && rl < g.H && __ldcg(g.cut + (int64_t)rl * g.W + c0 - 1);
    const bool hr = c0 + PT_W < g.W && rl < g.H && __ldcg(g.cut + (int64_t)rl * g.W + c0 + PT_W);
    if (hr) S |= iR & 0x80000000u;
    if (hl) S |= iL & 1u;
    if (lane == 0) S |= top & iU;
    if (lane == 31) S |= bot & iD;
    for (;;) {
        const uint32_t up = __shfl_up_sync(0xffffffffu, S, 1), dn = __shfl_down_sync(0xffffffffu, S, 1);
        uint32_t N = S | ((S >> 1) & iR) | ((S << 1) & iL);
        if (lane > 0) N |= up & iU;
        if (lane < 31) N |= dn & iD;
        const bool chg = N != S;
        S = N;
        if (!__any_sync(0xffffffffu, chg)) break;
    }
    const uint32_t add = S & ~S0;
    const uint32_t rows = __ballot_sync(0xffffffffu, add != 0);
    for (uint32_t x = rows; x; x &= x - 1) {
        const int i = __ffs(x) - 1;
        const uint32_t a = __shfl_sync(0xffffffffu, add, i);
        if ((a >> lane) & 1) g.cut[(int64_t)(r0 + i) * g.W + cl] = 1;
    }
    RingChange ch;
    ch.b0 = rows & 1;
    ch.b1 = (rows >> 31) & 1;
    ch.b2 = __any_sync(0xffffffffu, add & 1u);
    ch.b3 = __any_sync(0xffffffffu, add >> 31);
    ch.any = ch.b0 | ch.b1 | ch.b2 | ch.b3;
    ch.r0 = ch.r1 = ch.r2 = ch.r3 = 0;
    return ch;
}

// K2 with owner scheduling (single band, global relabel; option bfs_owner): tile t is
// visited only by warp t mod (launch warps), so no two warps ever hold it and there is
// no shared queue -- a visit whose border changed marks the neighbour tile dirty (one
// release exchange on its flag), the owner finds it by polling its few flags and takes
// it with an acquire exchange.  Replaces the ring's pop / claim / publish round trips
// and its two hottest words (head, tail); the pending count stays: a visit adds the
// neighbours it is about to mark BEFORE marking them (a marked tile can be taken and
// finished at once), then removes the ones that were already dirty and itself.  Flags:
// 0 clean, 1 dirty from the start (relabel_init marks every tile, pending = ntiles), 2
// marked by a neighbour.  A tile without a sink arc starts clean (its owner clears the
// initial mark unless a neighbour marked it already): its distances come only through
// its halos, and a neighbour's FIRST visit marks it whenever their shared border was
// reached (the border's sink pixels hold their distance 1 from the preparation, so
// "changed" alone would never fire for them).
__device__ __forceinline__ int exch_acq_rel(int32_t *p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.exch.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__global__ void __launch_bounds__(32 * BB_WARPS) owner_bfs_kernel(GridDev g, RingQ q) {
    __shared__ int32_t s_d[BB_WARPS][PT_H * (PT_W + 1)];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t *sd = s_d[wid];
    const int gw = blockIdx.x * BB_WARPS + wid, nw = gridDim.x * BB_WARPS;
    const int ntiles = g.ntx * g.nty;
    const int nown = gw < ntiles ? (ntiles - gw + nw - 1) / nw : 0;   // <= 64 (host checks)
    uint32_t vis0 = 0, vis1 = 0;   // owned tile i visited in this launch (incremental re-visits)
    unsigned chg_count = 0, nvis = 0;
    long long busy = 0;
#ifdef FM_BFS_TIMING
    BfsTm tm;
    int lv = 0;
#endif
    {
        int skipped = 0;
        for (int i = 0; i < nown; i++) {
            const int tile = gw + i * nw;
            if (__any_sync(0xffffffffu, g.rbits[(size_t)tile * 160 + 128 + lane] != 0u)) continue;
            if (lane == 0 && atomicCAS(q.flag + tile, 1, 0) == 1) skipped++;
        }
        if (lane == 0 && skipped) atomicSub(q.pend, (unsigned)skipped);
    }
    unsigned ns = q.ns0;
    for (;;) {
        const int32_t f0 = lane < nown ? *(volatile int32_t *)(q.flag + gw + lane * nw) : 0;
        const int32_t f1 = lane + 32 < nown ? *(volatile int32_t *)(q.flag + gw + (lane + 32) * nw) : 0;
        uint32_t d0 = __ballot_sync(0xffffffffu, f0 != 0), d1 = __ballot_sync(0xffffffffu, f1 != 0);
        if (!(d0 | d1)) {
            if (*(volatile unsigned *)q.pend == 0) break;
            __nanosleep(ns);
            ns = min(ns * 2, (unsigned)q.ns1);
            continue;
        }
        ns = q.ns0;
        while (d0 | d1) {
            int i;
            if (d0) { i = __ffs(d0) - 1; d0 &= d0 - 1; } else { i = 32 + __ffs(d1) - 1; d1 &= d1 - 1; }
            const int tile = gw + i * nw;
            int took = 0;
            if (lane == 0) took = exch_acq_rel(q.flag + tile, 0);   // acquire: the markers' stores
            took = __shfl_sync(0xffffffffu, took, 0);
            __syncwarp();
            if (!took) continue;
            const bool vis = i < 32 ? ((vis0 >> i) & 1u) : ((vis1 >> (i - 32)) & 1u);
            const long long tv0 = clock64();
#ifdef FM_BFS_TIMING
            const RingChange ch = bfs_visit(g, q, tile, vis, sd, lane, lv, tm);
#else
            const RingChange ch = bfs_visit(g, q, tile, vis, sd, lane);
#endif
            busy += clock64() - tv0;
            nvis++;
            if (i < 32) vis0 |= 1u << i; else vis1 |= 1u << (i - 32);
            chg_count += ch.any ? 1u : 0u;
            const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
            int nt = -1;
            const bool first = !vis;
            if (lane == 0 && (ch.b0 || (first && ch.r0)) && tyi > 0) nt = tile - g.ntx;
            if (lane == 1 && (ch.b1 || (first && ch.r1)) && tyi + 1 < g.nty) nt = tile + g.ntx;
            if (lane == 2 && (ch.b2 || (first && ch.r2)) && txi > 0) nt = tile - 1;
            if (lane == 3 && (ch.b3 || (first && ch.r3)) && txi + 1 < g.ntx) nt = tile + 1;
            const int k = __popc(__ballot_sync(0xffffffffu, nt >= 0));
            if (lane == 0 && k) atomicAdd(q.pend, (unsigned)k);   // counted before they can be taken
            __syncwarp();   // the warp's dist stores (and the count) precede the release exchanges
            const bool fresh = nt >= 0 && exch_acq_rel(q.flag + nt, 2) == 0;
            const int nfresh = __popc(__ballot_sync(0xffffffffu, fresh));
            if (lane == 0) atomicAdd(q.pend, (unsigned)(nfresh - k - 1));   // this tile done
            __syncwarp();
        }
    }
    if (lane == 0 && chg_count) atomicAdd(q.ctr + 96, chg_count);
    if (lane == 0 && nvis) {   // visits and the cycles spent inside them (trace statistics)
        atomicAdd(q.ctr + 192, nvis);
        atomicAdd((unsigned long long *)(q.ctr + 240), (unsigned long long)busy);
#ifdef FM_BFS_TIMING
        unsigned long long *t = (unsigned long long *)(q.ctr + 208);
        atomicAdd(t + 1, (unsigned long long)tm.ld); atomicAdd(t + 2, (unsigned long long)tm.lvl);
        atomicAdd(t + 3, (unsigned long long)tm.wb);
        atomicAdd((unsigned long long *)(q.ctr + 244), (unsigned long long)lv);
#endif
    }
}

// K2 (MODE 0, global relabel BFS) / K3 (MODE 1, min-cut reach) as ONE persistent
// launch over the ring queue.  Row-band mode: halos of the band's first / last tile
// row come from the neighbour bands' planes, a changed boundary row queues the
// neighbour band's tile in ITS ring, and every band's launch ends on one shared
// pending counter (all bands' launches run at once, one per GPU).
template <int MODE>
__global__ void __launch_bounds__(32 * BB_WARPS) ring_kernel(GridDev g, RingQ q) {
    __shared__ int32_t s_d[BB_WARPS][MODE == 0 ? PT_H * (PT_W + 1) : 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t *sd = s_d[wid];
    // a wait that exceeds this (a neighbour band's launch never started, e.g. two bands
    // on one GPU that cannot be resident together) ends the launch with an error flag
    constexpr unsigned long long WAIT_LIMIT_NS = 20ull * 1000 * 1000 * 1000;
#ifdef FM_BFS_TIMING
    BfsTm tm;
#endif
    unsigned chg_count = 0;   // visits that changed a border (lane 0; flushed once at the end)
    int base_slot = 0;
    if (q.sys && blockIdx.x == 0 && wid == 0) {
        // row bands: the watcher warp of this band polls the shared pending count (on
        // band 0's device) and raises the band-local done word when it reaches 0
        if (lane == 0) {
            const unsigned long long t0 = globaltimer_ns();
            for (;;) {
                if (ld_acquire((const int32_t *)q.pend, true) == 0) break;
                if (globaltimer_ns() - t0 > WAIT_LIMIT_NS) { atomicExch(q.ctr + 248, 1u); break; }
                __nanosleep(256);
            }
            st_release((int32_t *)(q.ctr + 252), 1, false);
        }
        __syncwarp();
        return;
    }
    for (;;) {
        int tile = -1;
        bool visited = false;
#ifdef FM_BFS_TIMING
        const long long tw0 = clock64();
#endif
        if (lane == 0) {
            const unsigned s = atomicAdd(q.ctr + 0, 1u) % (unsigned)q.cap;
            volatile int32_t *vs = q.slot + s;
            unsigned long long t0 = 0;
            for (unsigned ns = q.ns0;; ns = min(ns * 2, (unsigned)q.ns1)) {
                tile = ld_acquire((const int32_t *)vs, q.sys);   // acquire: the producer's stores
                if (tile >= 0) { *vs = -1; break; }
                // row bands: the shared pending count is remote for most bands; idle warps
                // poll only the band-local done word the watcher raises
                if (q.sys ? (*(volatile int32_t *)(q.ctr + 252) != 0) : (*(volatile unsigned *)q.pend == 0)) break;
                if (q.sys) {
                    const unsigned long long now = globaltimer_ns();
                    if (!t0) t0 = now;
                    else if (now - t0 > WAIT_LIMIT_NS) { atomicExch(q.ctr + 248, 1u); break; }
                }
                __nanosleep(ns);
            }
            if (tile >= 0) visited = (atomicAdd(q.flag + tile, 1) & 4) != 0;   // queued -> in flight
        }
        tile = __shfl_sync(0xffffffffu, tile, 0);
        visited = __shfl_sync(0xffffffffu, visited ? 1 : 0, 0) != 0;
        __syncwarp();   // lane 0's acquire orders every lane's loads of the visit
#ifdef FM_BFS_TIMING
        tm.wait += clock64() - tw0;
#endif
        if (tile < 0) break;
        const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
        bool again = true;
#ifdef FM_BFS_TIMING
        const long long tv0 = clock64();
        int lv = 0;
#endif
        while (again) {
            RingChange ch;
            if constexpr (MODE == 0) {
#ifdef FM_BFS_TIMING
                ch = bfs_visit(g, q, tile, visited, sd, lane, lv, tm);
#else
                ch = bfs_visit(g, q, tile, visited, sd, lane);
#endif
            } else {
                ch = cut_visit(g, tile, lane);
            }
            int st = 0;
#ifdef FM_BFS_TIMING
            const long long tp0 = clock64();
#endif
            __syncwarp();   // the warp's stores precede the lanes' release operations below
            // (1) in parallel: lanes 0-3 claim the up / down / left / right neighbour (state
            // 0 -> 1: queued by us, 2 -> 3: its owner runs it again; release CAS keeping the
            // visited bit), lane 4 releases this tile (2 -> idle + visited; release: the
            // warp's stores, ordered before it by the __syncwarp above, are visible before
            // the tile can be taken again -- an incremental re-visit on another SM reads the
            // interior; acquire: a 3 read here sees the stores of the visit that marked it)
            int nt = -1, peer = 0, own = 0;
            bool claimed = false;
            if (lane < 4) {
                if (lane == 0 && ch.b0) { if (tyi > 0) nt = tile - g.ntx; else if (g.has_up) { nt = g.up.tile0 + txi; peer = 1; } }
                if (lane == 1 && ch.b1) { if (tyi + 1 < g.nty) nt = tile + g.ntx; else if (g.has_dn) { nt = g.dn.tile0 + txi; peer = 2; } }
                if (lane == 2 && ch.b2 && txi > 0) nt = tile - 1;
                if (lane == 3 && ch.b3 && txi + 1 < g.ntx) nt = tile + 1;
                if (nt >= 0 && (peer || !g.region || g.region[nt])) {
                    int32_t *fl = peer == 1 ? g.up.rq_flag : peer == 2 ? g.dn.rq_flag : q.flag;
                    const bool sys = q.sys || peer;
                    for (int c = 0;;) {
                        const int state = c & 3;
                        if (state == 1 || state == 3) break;                 // queued / already marked
                        const int o = cas_acq_rel(fl + nt, c, c + 1, sys);
                        if (o == c) { claimed = state == 0; break; }
                        c = o;
                    }
                }
            } else if (lane == 4) {
                const int v = visited ? 4 : 0;
                own = cas_acq_rel(q.flag + tile, 2 | v, 4, q.sys);
                if (own == (3 | v)) atomicExch(q.flag + tile, q.rerun ? (2 | 4) : (1 | 4));   // run again / requeue
            }
            const unsigned cm = __ballot_sync(0xffffffffu, claimed);
            const unsigned cl = __ballot_sync(0xffffffffu, claimed && peer == 0);
            own = __shfl_sync(0xffffffffu, own, 4) & 3;
            st = own == 3 ? 3 : 0;
            if (lane == 0) {
                chg_count += ch.any ? 1u : 0u;
#ifdef FM_BFS_TIMING
                atomicAdd(q.ctr + 192, 1u);   // every visit (diagnostics)
#endif
                const int requeue = (st == 3 && !q.rerun) ? 1 : 0;
                if (requeue) st = 0;
                // (2) ONE update of the shared pending count: + the claimed neighbours, - this
                // tile unless it stays queued / in flight.  It precedes the slot stores, so a
                // claimed tile is counted before anyone can take (and complete) it.
                const int delta = __popc(cm) - (st == 3 || requeue ? 0 : 1);
                if (delta) atomicAdd(q.pend, (unsigned)delta);
                // (3) one reservation of local slots for the claimed neighbours + a requeue
                const int nl = __popc(cl) + requeue;
                base_slot = nl ? (int)atomicAdd(q.ctr + 32, (unsigned)nl) : 0;
                if (requeue) st_release(q.slot + ((unsigned)(base_slot + nl - 1) % (unsigned)q.cap), tile, q.sys);
            }
            base_slot = __shfl_sync(0xffffffffu, base_slot, 0);
            if (claimed) {   // release stores publish the tiles (and our stores) to their takers
                if (peer) {
                    const PeerView &pv = peer == 1 ? g.up : g.dn;
                    const unsigned s2 = atomicAdd(pv.rq_ctr + 32, 1u);
                    st_release(pv.rq_slot + (s2 % (unsigned)pv.rq_cap), nt, true);
                } else {
                    const int rank = __popc(cl & ((1u << lane) - 1));
                    st_release(q.slot + ((unsigned)(base_slot + rank) % (unsigned)q.cap), nt, q.sys);
                }
            }
            again = __shfl_sync(0xffffffffu, st, 0) == 3;
            visited = true;
            __syncwarp();
#ifdef FM_BFS_TIMING
            tm.push += clock64() - tp0;
#endif
        }  // while again
#ifdef FM_BFS_TIMING
        if (lane == 0) {
            atomicAdd((unsigned long long *)(q.ctr + 240), (unsigned long long)(clock64() - tv0));
            atomicAdd((unsigned long long *)(q.ctr + 244), (unsigned long long)lv);
        }
#endif
    }
    if (lane == 0 && chg_count) atomicAdd(q.ctr + 96, chg_count);
#ifdef FM_BFS_TIMING
    if (lane == 0 && MODE == 0) {   // per-section warp cycles: wait, load, levels, write-back, queue
        unsigned long long *t = (unsigned long long *)(q.ctr + 208);
        atomicAdd(t + 0, (unsigned long long)tm.wait); atomicAdd(t + 1, (unsigned long long)tm.ld);
        atomicAdd(t + 2, (unsigned long long)tm.lvl); atomicAdd(t + 3, (unsigned long long)tm.wb);
        atomicAdd(t + 4, (unsigned long long)tm.push);
    }
#endif
}

// ----------------------------------------------------------------------------
// K1 as ONE persistent launch per round (default): pl_visit over a device ring
// queue of tiles instead of a sequence of launches over double-buffered lists.
// A tile is queued when it holds active pixels after a visit or when flow is
// parked in its inbox; CTAs take tiles until the queue drains (round over: every
// pixel is inactive or written off) or the round's relabel budget / visit cap is
// reached (stop flag).  Flow crosses any number of tiles within the launch, so the
// tail rounds no longer pay one launch + host sync per tile hop.
// States as in the BFS ring (0 idle, 1 queued, 2 in flight, 3 in flight + more
// inflow); only the owner moves a tile out of 2/3, so a tile is never in the queue
// twice and never visited by two CTAs at once (its smem copy is the only writer).
// ctr: [0] head [32] tail [64] pending [96] visits [128] stop [160] relabels (u64)
//      [224] initial tiles.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void ring_enqueue(const RingQ &q, int t) {
    const unsigned s = atomicAdd(q.ctr + 32, 1u);
    __threadfence();
    *(volatile int32_t *)(q.slot + (s % (unsigned)q.cap)) = t;
}

__global__ void __launch_bounds__(PL_NT, FM_PL_MINBLOCKS) pr_ring_kernel(GridDev g, RingQ q, int k_local, int steps,
                                                                       int fused, long long relabel_budget,
                                                                       int visit_mult, unsigned long long *ops) {
    __shared__ PlSmem S;
    const int tid = threadIdx.y * PT_W + threadIdx.x;
    volatile unsigned *stop = q.ctr + 128;
    unsigned long long *rel_total = (unsigned long long *)(q.ctr + 160);
    PlCounters C;
    const unsigned visit_cap = (unsigned)max(64, visit_mult * (int)__ldcg(q.ctr + 224));
    for (;;) {
        __syncthreads();
        if (tid == 0) {
            int tile = -1;
            if (!*stop) {
                const unsigned s = atomicAdd(q.ctr + 0, 1u) % (unsigned)q.cap;
                volatile int32_t *vs = q.slot + s;
                for (unsigned ns = q.ns0;; ns = min(ns * 2, (unsigned)q.ns1)) {
                    tile = *vs;
                    if (tile >= 0) { *vs = -1; break; }
                    if (*(volatile unsigned *)(q.ctr + 64) == 0 || *stop) break;
                    __nanosleep(ns);
                }
                if (tile >= 0) { atomicExch(q.flag + tile, 2); __threadfence(); }
            }
            S.tile = tile;
        }
        __syncthreads();
        const int tile = S.tile;
        if (tile < 0) break;
        const long long rel0 = C.relabels;
        unsigned no_tma = 0;
        const bool act = pl_visit(g, S, tile, k_local, steps, fused, C, nullptr, no_tma);
        // this visit's relabels, CTA-wide (for the round's relabel budget)
        long long dr = C.relabels - rel0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dr += __shfl_xor_sync(0xffffffffu, dr, o);
        if ((tid & 31) == 0) S.red[tid >> 5] = dr;
        __syncthreads();
        if (tid == 0) {
            long long vr = 0;
            for (int w = 0; w < PL_NT / 32; w++) vr += S.red[w];
            g.touched[tile] = 1;
            const int nb = S.nbr;
            const int nts[4] = {tile + 1, tile - 1, tile + g.ntx, tile - g.ntx};
            for (int d = 0; d < 4; d++) {
                if (!((nb >> d) & 1)) continue;
                const int t = nts[d];
                g.touched[t] = 1;
                for (;;) {   // queue t, or mark it for a requeue by its owner
                    const int o = atomicCAS(q.flag + t, 0, 1);
                    if (o == 0) { atomicAdd(q.ctr + 64, 1u); ring_enqueue(q, t); break; }
                    if (o != 2 || atomicCAS(q.flag + t, 2, 3) == 2) break;
                }
            }
            const unsigned long long rt = atomicAdd(rel_total, (unsigned long long)vr) + (unsigned long long)vr;
            const unsigned nv = atomicAdd(q.ctr + 96, 1u) + 1;
            if (rt >= (unsigned long long)relabel_budget || nv >= visit_cap) *stop = 1;
            // leave flight: back to the queue if still active or fed while in flight
            int o = atomicCAS(q.flag + tile, 2, act ? 1 : 0);
            if (o == 3) { atomicExch(q.flag + tile, 1); o = 2; ring_enqueue(q, tile); }
            else if (act) ring_enqueue(q, tile);
            else atomicSub(q.ctr + 64, 1u);
        }
    }
    block_add_i64<PL_NT / 32>(C.pushes, ops + 0);
    block_add_i64<PL_NT / 32>(C.relabels, ops + 1);
    if (tid == 0) {
        if (C.passes) atomicAdd(ops + 3, (unsigned long long)C.passes);
        if (C.items) atomicAdd(ops + 4, (unsigned long long)C.items);
    }
}

// gap_relabel + marking (as bfs_finalize_kernel), one CTA per tile so each tile with
// an active pixel is queued once
// list == nullptr: every tile; else the n tiles of `list` (local relabel region)
__global__ void __launch_bounds__(256, 8) bfs_finalize_tiles_kernel(GridDev g, unsigned long long *acc,
                                                                 const int32_t *list, int n) {
    long long active = 0, mex = 0;
    int32_t lvl = 0;
    const int nt = list ? n : g.ntx * g.nty;
    for (int it = blockIdx.x; it < nt; it += gridDim.x) {
        const int tile = list ? list[it] : it;
        const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
        bool act = false;
        if (!list && threadIdx.x == 0) g.touched[tile] = 0;   // global relabel: every tile is current
        const int r = tyi * PT_H + (threadIdx.x >> 3), c = txi * PT_W + 4 * (threadIdx.x & 7);
        if ((g.W & 3) == 0 && (tyi + 1) * PT_H <= g.H && (txi + 1) * PT_W <= g.W) {
            // interior tile, W % 4 == 0: 4 consecutive pixels per thread, 16-byte accesses
            const int64_t p = (int64_t)r * g.W + c;
            {
                const int4 d4 = *(const int4 *)(g.dist + p), e4 = *(const int4 *)(g.e + p);
                const int dv[4] = {d4.x, d4.y, d4.z, d4.w}, ev[4] = {e4.x, e4.y, e4.z, e4.w};
                // old heights and marks matter only for unreached pixels (reached ones take
                // their distance): most groups skip those two reads
                const bool unreached = dv[0] >= g.INF || dv[1] >= g.INF || dv[2] >= g.INF || dv[3] >= g.INF;
                const int4 h4 = unreached ? *(const int4 *)(g.h + p) : make_int4(0, 0, 0, 0);
                const uchar4 m4 = unreached ? *(const uchar4 *)(g.marked + p) : make_uchar4(1, 1, 1, 1);
                int hv[4] = {h4.x, h4.y, h4.z, h4.w};
                unsigned char mv[4] = {m4.x, m4.y, m4.z, m4.w};
                bool mchg = false;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    if (dv[j] < g.INF) {
                        hv[j] = dv[j];
                        active += ev[j] > 0;
                        act |= ev[j] > 0;
                        lvl = max(lvl, dv[j]);
                    } else {
                        if (hv[j] < g.V) hv[j] = g.V;
                        if (!mv[j]) { mv[j] = 1; mex += ev[j]; mchg = true; }
                    }
                }
                *(int4 *)(g.h + p) = make_int4(hv[0], hv[1], hv[2], hv[3]);
                if (mchg) *(uchar4 *)(g.marked + p) = make_uchar4(mv[0], mv[1], mv[2], mv[3]);
            }
            // no CTA barrier per tile: every warp that saw an active pixel offers the tile
            // (the queue flag admits it once), so warps run ahead into the next tile's loads
            if (__any_sync(0xffffffffu, act) && (threadIdx.x & 31) == 0) tq_push(g.pq, 0, tile);
            continue;
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int lr = (threadIdx.x >> 5) + 8 * k;
            const int rr = tyi * PT_H + lr, cc = txi * PT_W + (threadIdx.x & 31);
            if (rr >= g.H || cc >= g.W) continue;
            const int64_t p = (int64_t)rr * g.W + cc;
            const int32_t d = g.dist[p];
            const int32_t e = g.e[p];
            if (d < g.INF) {
                g.h[p] = d;
                active += e > 0;
                act |= e > 0;
                lvl = max(lvl, d);
            } else {
                if (g.h[p] < g.V) g.h[p] = g.V;
                if (!g.marked[p]) { g.marked[p] = 1; mex += e; }
            }
        }
        if (__any_sync(0xffffffffu, act) && (threadIdx.x & 31) == 0) tq_push(g.pq, 0, tile);
    }
    __shared__ long long red[2][8];
    __shared__ int32_t redl[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        active += __shfl_xor_sync(0xffffffffu, active, o);
        mex += __shfl_xor_sync(0xffffffffu, mex, o);
        lvl = max(lvl, __shfl_xor_sync(0xffffffffu, lvl, o));
    }
    if (lane == 0) { red[0][wid] = active; red[1][wid] = mex; redl[wid] = lvl; }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long a = 0, m = 0; int32_t l = 0;
        for (int i = 0; i < 8; i++) { a += red[0][i]; m += red[1][i]; l = max(l, redl[i]); }
        if (a) atomicAdd(&acc[0], (unsigned long long)a);
        if (m) atomicAdd(&acc[1], (unsigned long long)m);
        if (l) atomicMax(&acc[2], (unsigned long long)l);
    }
}

// ----------------------------------------------------------------------------
// Local relabel (tail rounds).  R = tiles touched since the last relabel, dilated by
// `margin` tiles.  Outside R nothing moved, so dist[] there still holds the labels of
// the last relabel (= h for reached pixels, INF for written-off ones); distances only
// grow, so those are valid lower bounds, and relaxing R against them as frozen values
// gives every pixel of R a valid label (exact when its shortest path stays in R or
// crosses pixels whose distance did not change).  A pixel of R left at INF has no
// residual path to t at all -- every path leaving R meets a pixel already unreachable --
// so the gap relabel and the write-off stay exact.
// ----------------------------------------------------------------------------
__global__ void region_build_kernel(GridDev g, uint8_t *region, int margin, int32_t *count) {
    const int nt = g.ntx * g.nty;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
        const int ty = t / g.ntx, tx = t - ty * g.ntx;
        bool in = false;
        for (int dy = -margin; dy <= margin && !in; dy++) {
            const int yy = ty + dy;
            if (yy < 0 || yy >= g.nty) continue;
            for (int dx = -margin; dx <= margin; dx++) {
                const int xx = tx + dx;
                if (xx >= 0 && xx < g.ntx && g.touched[yy * g.ntx + xx]) { in = true; break; }
            }
        }
        region[t] = in ? 1 : 0;
        if (in) {
            g.bq.flag[0][t] = 1;
            g.bq.list[0][atomicAdd(g.bq.cnt + 0, 1)] = t;
            atomicAdd(count, 1);
        }
    }
}

// residual masks and seeds for the pixels of R only (one CTA per listed tile)
__global__ void bfs_init_local_kernel(GridDev g) {
    const int n = __ldcg(g.bq.cnt + 0);
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const int tile = g.bq.list[0][i];
        const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
        for (int k = threadIdx.x; k < TILE_W * TILE_H; k += blockDim.x) {
            const int r = tyi * TILE_H + k / TILE_W, c = txi * TILE_W + k % TILE_W;
            if (r >= g.H || c >= g.W) continue;
            const int64_t p = (int64_t)r * g.W + c;
            uint8_t m = 0;
            if (c + 1 < g.W && g.rR[p] > 0) m |= M_R;
            if (c > 0 && g.rL[p] > 0) m |= M_L;
            if (r + 1 < g.H && g.rD[p] > 0) m |= M_D;
            if (r > 0 && g.rU[p] > 0) m |= M_U;
            if (g.rT[p] > 0) m |= M_T;
            if (false) m = 0;
            g.mask[p] = m;
            g.dist[p] = (m & M_T) ? 1 : g.INF;
        }
    }
}

// gap + marking + active tiles over R only (active pixels only ever live in R)
__global__ void bfs_finalize_local_kernel(GridDev g, const int32_t *list, int n,
                                          unsigned long long *acc) {
    long long active = 0, mex = 0;
    int32_t lvl = 0;
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const int tile = list[i];
        const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
        bool act_tile = false;
        for (int k = threadIdx.x; k < TILE_W * TILE_H; k += blockDim.x) {
            const int r = tyi * TILE_H + k / TILE_W, c = txi * TILE_W + k % TILE_W;
            if (r >= g.H || c >= g.W) continue;
            const int64_t p = (int64_t)r * g.W + c;
            const int32_t d = g.dist[p];
            const int32_t e = g.e[p];
            if (d < g.INF) {
                g.h[p] = d;
                active += e > 0;
                act_tile |= e > 0;
                lvl = max(lvl, d);
            } else {
                if (g.h[p] < g.V) g.h[p] = g.V;
                if (!g.marked[p]) { g.marked[p] = 1; mex += e; }
            }
        }
        if (__syncthreads_or(act_tile) && threadIdx.x == 0) tq_push(g.pq, 0, tile);
    }
    if (active) atomicAdd(&acc[0], (unsigned long long)active);
    if (mex) atomicAdd(&acc[1], (unsigned long long)mex);
    if (lvl) atomicMax(&acc[2], (unsigned long long)lvl);
}

// gap_relabel (maxflow_seq.py:149-160) + marking (maxflow_par.py:223-226):
// reached pixels take their exact distance, unreached ones are lifted to >= |V|
// and, the first time, written off (their excess leaves ExcessTotal).
__global__ void bfs_finalize_kernel(GridDev g, unsigned long long *acc /* [0] active [1] newly marked excess [2] max level */) {
    const int64_t HW = (int64_t)g.H * g.W;
    long long active = 0, mex = 0;
    int32_t lvl = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < HW;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t d = g.dist[p];
        const int32_t e = g.e[p];
        if (d < g.INF) {
            g.h[p] = d;
            active += e > 0;
            lvl = max(lvl, d);
            if (e > 0) {
                const int32_t r = (int32_t)(p / g.W), c = (int32_t)(p - (int64_t)r * g.W);
                const int t = (r / PT_H) * g.ntx + c / PT_W;
                if (!__ldcg(g.pq.flag[0] + t)) tq_push(g.pq, 0, t);
            }
        } else {
            if (g.h[p] < g.V) g.h[p] = g.V;
            if (!g.marked[p]) { g.marked[p] = 1; mex += e; }
        }
    }
    __shared__ long long red[2][8];
    __shared__ int32_t redl[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        active += __shfl_xor_sync(0xffffffffu, active, o);
        mex += __shfl_xor_sync(0xffffffffu, mex, o);
        lvl = max(lvl, __shfl_xor_sync(0xffffffffu, lvl, o));
    }
    if (lane == 0) { red[0][wid] = active; red[1][wid] = mex; redl[wid] = lvl; }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long a = 0, m = 0; int32_t l = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) { a += red[0][i]; m += red[1][i]; l = max(l, redl[i]); }
        if (a) atomicAdd(&acc[0], (unsigned long long)a);
        if (m) atomicAdd(&acc[1], (unsigned long long)m);
        if (l) atomicMax(&acc[2], (unsigned long long)l);
    }
}

// ----------------------------------------------------------------------------
// K3: minimal source-side cut = residual reach from {s} U {p : e(p) > 0}
// (SURVEY.md 8a-A10).  Pull form: q joins S when a neighbour in S has a residual
// arc into q.  Same tile-local fixpoint scheme as K2.
// ----------------------------------------------------------------------------
__global__ void cut_init_kernel(GridDev g) {
    const int64_t HW = (int64_t)g.H * g.W;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < HW;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = (int32_t)(p / g.W), c = (int32_t)(p - (int64_t)r * g.W);
        uint8_t m = 0;  // incoming residual arcs: bit R = arc (p+1)->p, etc.
        if (c + 1 < g.W && g.rL[p + 1] > 0) m |= M_R;
        if (c > 0 && g.rR[p - 1] > 0) m |= M_L;
        if (r + 1 < g.H && g.rU[p + g.W] > 0) m |= M_D;
        if (r > 0 && g.rD[p - g.W] > 0) m |= M_U;
        const bool gh = false;
        g.mask[p] = gh ? 0 : m;           // ghost membership is imported from the owner band
        g.cut[p] = (!gh && (g.e[p] > 0 || g.cS[p] - g.rS[p] > 0)) ? 1 : 0;
    }
}

__global__ void __launch_bounds__(256) cut_tile_kernel(GridDev g, int parity, int all_tiles,
                                                       int32_t *changed_count) {
    __shared__ uint8_t ss[TILE_H + 2][TILE_W + 2];
    __shared__ int s_tile, s_b[4];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * TILE_W + tx;
    for (;;) {
    __syncthreads();
    if (tid == 0) {
        s_tile = tq_take(g.bq, parity, all_tiles, g.ntx * g.nty);
        s_b[0] = s_b[1] = s_b[2] = s_b[3] = 0;
    }
    __syncthreads();
    const int tile = s_tile;
    if (tile < 0) break;
    const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
    const int c0 = txi * TILE_W, r0 = tyi * TILE_H;
    for (int i = tid; i < (TILE_H + 2) * (TILE_W + 2); i += TILE_W * BLK_Y) {
        const int lr = i / (TILE_W + 2), lc = i % (TILE_W + 2);
        const int r = r0 + lr - 1, c = c0 + lc - 1;
        ss[lr][lc] = (r >= 0 && r < g.H && c >= 0 && c < g.W) ? g.cut[(int64_t)r * g.W + c] : 0;
    }
    uint8_t m[ROWS_PER_THREAD];
    const int c = c0 + tx;
#pragma unroll
    for (int k = 0; k < ROWS_PER_THREAD; k++) {
        const int r = r0 + ty + k * BLK_Y;
        m[k] = (r < g.H && c < g.W) ? g.mask[(int64_t)r * g.W + c] : 0;
    }
    __syncthreads();
    bool any = false;
    uint8_t grew[ROWS_PER_THREAD] = {};
    for (;;) {
        bool ch = false;
#pragma unroll
        for (int k = 0; k < ROWS_PER_THREAD; k++) {
            const int lr = ty + k * BLK_Y + 1, lc = tx + 1;
            const uint8_t mk = m[k];
            if (!mk || ss[lr][lc]) continue;
            if (((mk & M_R) && ss[lr][lc + 1]) || ((mk & M_L) && ss[lr][lc - 1]) ||
                ((mk & M_D) && ss[lr + 1][lc]) || ((mk & M_U) && ss[lr - 1][lc])) {
                ss[lr][lc] = 1;
                grew[k] = 1;
                ch = true;
            }
        }
        if (!__syncthreads_or(ch)) break;
        any = true;
    }
    if (any) {
#pragma unroll
        for (int k = 0; k < ROWS_PER_THREAD; k++) {
            const int lr = ty + k * BLK_Y;
            const int r = r0 + lr;
            if (grew[k] && r < g.H && c < g.W) {
                g.cut[(int64_t)r * g.W + c] = 1;
                if (lr == 0) s_b[0] = 1;
                if (lr == TILE_H - 1) s_b[1] = 1;
                if (tx == 0) s_b[2] = 1;
                if (tx == TILE_W - 1) s_b[3] = 1;
            }
        }
        __syncthreads();
        if (tid == 0) {
            flag_changed_borders(g, tile, tyi, txi, s_b[0], s_b[1], s_b[2], s_b[3], parity ^ 1);
            atomicAdd(changed_count, 1);
        }
    }
    }  // tile loop
}

// ----------------------------------------------------------------------------
// K3 bit-parallel (default): the cut closure with the tile's incoming residual arcs
// as bit planes (lane = tile row, bit = column), one warp per tile:
//     S |= ((S >> 1) & inR) | ((S << 1) & inL) | (S_below & inD) | (S_above & inU)
// (+ the halo's cut bits) until no word changes.  The cut bytes stay the exchanged /
// returned representation; a visit ORs in the pixels it adds.  cut_tile_kernel
// stays behind FM_BFS_BITS=0.
// ----------------------------------------------------------------------------
__global__ void cut_init_bits_kernel(GridDev g) {
    const int lane = threadIdx.x & 31;
    if (g.ntx % 4 == 0 && g.W == g.ntx * PT_W && g.H == g.nty * PT_H) {
        // whole tiles, 4 per group: one image row of 4 tiles per warp iteration, lane = 4
        // columns, int4 loads; the horizontal neighbours' residuals come from the adjacent
        // lanes (one extra scalar load at the warp's ends); words assembled by shuffles
        const int ngroups = g.ntx / 4;
        const int nunits = g.nty * PT_H * ngroups;
        const int sh = 4 * (lane & 7), j = lane >> 3;
        for (int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < nunits; u += (gridDim.x * blockDim.x) >> 5) {
            const int r = u / ngroups, tg = u - r * ngroups;
            const int ty = r / PT_H, lr = r - ty * PT_H;
            const int tile = ty * g.ntx + 4 * tg + j;
            const int c = (4 * tg + j) * PT_W + sh;
            const int64_t p = (int64_t)r * g.W + c;
            const int4 L = __ldcs((const int4 *)(g.rL + p)), R = __ldcs((const int4 *)(g.rR + p));
            const int4 E = __ldcs((const int4 *)(g.e + p)), CS = __ldcs((const int4 *)(g.cS + p));
            const int4 RS = __ldcs((const int4 *)(g.rS + p));
            const int4 Db = r + 1 < g.H ? __ldcs((const int4 *)(g.rU + p + g.W))
                                        : (g.has_dn ? ld_cg4(g.dn.res + c) : make_int4(0, 0, 0, 0));
            const int4 Ua = r > 0 ? __ldcs((const int4 *)(g.rD + p - g.W))
                                  : (g.has_up ? ld_cg4(g.up.res + c) : make_int4(0, 0, 0, 0));
            // rL of column c+4 (right neighbour of this lane's last pixel), rR of column c-1
            int lNext = __shfl_down_sync(0xffffffffu, L.x, 1);
            int rPrev = __shfl_up_sync(0xffffffffu, R.w, 1);
            if (lane == 31) lNext = c + 4 < g.W ? g.rL[p + 4] : 0;
            if (lane == 0) rPrev = c > 0 ? g.rR[p - 1] : 0;
            const uint32_t nR = (uint32_t)(L.y > 0) | ((uint32_t)(L.z > 0) << 1) | ((uint32_t)(L.w > 0) << 2) |
                                ((uint32_t)(c + 4 < g.W && lNext > 0) << 3);   // arc (q+1) -> q
            const uint32_t nL = (uint32_t)(c > 0 && rPrev > 0) | ((uint32_t)(R.x > 0) << 1) |
                                ((uint32_t)(R.y > 0) << 2) | ((uint32_t)(R.z > 0) << 3);  // arc (q-1) -> q
            const auto nib = [](const int4 v) {
                return (uint32_t)(v.x > 0) | ((uint32_t)(v.y > 0) << 1) | ((uint32_t)(v.z > 0) << 2) |
                       ((uint32_t)(v.w > 0) << 3);
            };
            const uint32_t nD = nib(Db), nU = nib(Ua);
            const uint32_t nS = (uint32_t)(E.x > 0 || CS.x - RS.x > 0) | ((uint32_t)(E.y > 0 || CS.y - RS.y > 0) << 1) |
                                ((uint32_t)(E.z > 0 || CS.z - RS.z > 0) << 2) | ((uint32_t)(E.w > 0 || CS.w - RS.w > 0) << 3);
            uint32_t wR = nR << sh, wL = nL << sh, wD = nD << sh, wU = nU << sh, wS = nS << sh;
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                wR |= __shfl_xor_sync(0xffffffffu, wR, o);
                wL |= __shfl_xor_sync(0xffffffffu, wL, o);
                wD |= __shfl_xor_sync(0xffffffffu, wD, o);
                wU |= __shfl_xor_sync(0xffffffffu, wU, o);
                wS |= __shfl_xor_sync(0xffffffffu, wS, o);
            }
            const int k = lane & 7;
            uint32_t *B = g.rbits + (size_t)tile * 160 + lr;
            if (k < 5) B[k * 32] = k == 0 ? wR : k == 1 ? wL : k == 2 ? wD : k == 3 ? wU : wS;
            *(uchar4 *)(g.cut + p) = make_uchar4(nS & 1u, (nS >> 1) & 1u, (nS >> 2) & 1u, (nS >> 3) & 1u);
        }
        return;
    }
    const int64_t nrows = (int64_t)g.ntx * g.nty * PT_H;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nrows;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int tile = (int)(w / PT_H), lr = (int)(w % PT_H);
        const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
        const int r = tyi * PT_H + lr, c = txi * PT_W + lane;
        const bool in = r < g.H && c < g.W;
        const int64_t p = (int64_t)r * g.W + c;
        const bool aR = in && c + 1 < g.W && g.rL[p + 1] > 0;     // residual arc (p+1) -> p
        const bool aL = in && c > 0 && g.rR[p - 1] > 0;
        // band mode: the arc from the neighbour band's boundary pixel is its residual
        const bool aD = in && (r + 1 < g.H ? g.rU[p + g.W] > 0 : (g.has_dn && ld_cg(g.dn.res + c) > 0));
        const bool aU = in && (r > 0 ? g.rD[p - g.W] > 0 : (g.has_up && ld_cg(g.up.res + c) > 0));
        const bool seed = in && (g.e[p] > 0 || g.cS[p] - g.rS[p] > 0);
        const uint32_t wd[5] = {__ballot_sync(0xffffffffu, aR), __ballot_sync(0xffffffffu, aL),
                                __ballot_sync(0xffffffffu, aD), __ballot_sync(0xffffffffu, aU),
                                __ballot_sync(0xffffffffu, seed)};
        uint32_t *B = g.rbits + (size_t)tile * 160 + lr;
        const uint32_t wk = lane == 0 ? wd[0] : lane == 1 ? wd[1] : lane == 2 ? wd[2] : lane == 3 ? wd[3] : wd[4];
        if (lane < 5) B[lane * 32] = wk;
        if (r < g.H && c < g.W) g.cut[p] = seed ? 1 : 0;
    }
}

__global__ void __launch_bounds__(32 * BB_WARPS) cut_bits_kernel(GridDev g, int parity, int all_tiles,
                                                               int32_t *changed_count) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int tile = 0;
        if (lane == 0) tile = tq_take(g.bq, parity, all_tiles, g.ntx * g.nty);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile < 0) break;
        const int tyi = tile / g.ntx, txi = tile - tyi * g.ntx;
        const int r0 = tyi * PT_H, c0 = txi * PT_W;
        const int cl = c0 + lane, rl = r0 + lane;
        const uint32_t *B = g.rbits + (size_t)tile * 160;
        const uint32_t iR = B[lane], iL = B[32 + lane], iD = B[64 + lane], iU = B[96 + lane];
        // current cut words of the tile (row i built by a ballot over its 32 columns)
        uint32_t S = 0;
#pragma unroll 8
        for (int i = 0; i < PT_H; i++) {
            const int r = r0 + i;
            const bool b = r < g.H && cl < g.W && __ldcg(g.cut + (int64_t)r * g.W + cl);
            const uint32_t wv = __ballot_sync(0xffffffffu, b);
            if (lane == i) S = wv;
        }
        const uint32_t S0 = S;
        const uint32_t top = __ballot_sync(0xffffffffu, r0 > 0 && cl < g.W && __ldcg(g.cut + (int64_t)(r0 - 1) * g.W + cl));
        const uint32_t bot = __ballot_sync(0xffffffffu, r0 + PT_H < g.H && cl < g.W &&
                                                        __ldcg(g.cut + (int64_t)(r0 + PT_H) * g.W + cl));
        const bool hl = c0 > 0 && rl < g.H && __ldcg(g.cut + (int64_t)rl * g.W + c0 - 1);
        const bool hr = c0 + PT_W < g.W && rl < g.H && __ldcg(g.cut + (int64_t)rl * g.W + c0 + PT_W);
        if (hr) S |= iR & 0x80000000u;
        if (hl) S |= iL & 1u;
        if (lane == 0) S |= top & iU;
        if (lane == 31) S |= bot & iD;
        for (;;) {
            const uint32_t up = __shfl_up_sync(0xffffffffu, S, 1), dn = __shfl_down_sync(0xffffffffu, S, 1);
            uint32_t N = S | ((S >> 1) & iR) | ((S << 1) & iL);
            if (lane > 0) N |= up & iU;
            if (lane < 31) N |= dn & iD;
            const bool ch = N != S;
            S = N;
            if (!__any_sync(0xffffffffu, ch)) break;
        }
        const uint32_t add = S & ~S0;
        const uint32_t rows = __ballot_sync(0xffffffffu, add != 0);
        for (uint32_t x = rows; x; x &= x - 1) {
            const int i = __ffs(x) - 1;
            const uint32_t a = __shfl_sync(0xffffffffu, add, i);
            if ((a >> lane) & 1) g.cut[(int64_t)(r0 + i) * g.W + cl] = 1;
        }
        const int b0 = rows & 1, b1 = (rows >> 31) & 1;
        const int b2 = __any_sync(0xffffffffu, add & 1u), b3 = __any_sync(0xffffffffu, add >> 31);
        if (lane == 0 && (b0 | b1 | b2 | b3)) {
            flag_changed_borders(g, tile, tyi, txi, b0, b1, b2, b3, parity ^ 1);
            atomicAdd(changed_count, 1);
        }
        __syncwarp();
    }
}

// sum of e over all pixels (flow = sum capS - sum e: node conservation)
__global__ void sum_e_kernel(GridDev g, unsigned long long *acc) {
    const int64_t HW = (int64_t)g.H * g.W;
    long long s = 0;
    // int4 loads, two in flight per thread (a scalar-load loop ran at 0.7 TB/s)
    const int64_t n4 = HW >> 2, stride = (int64_t)gridDim.x * blockDim.x;
    const int4 *e4 = reinterpret_cast<const int4 *>(g.e);
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + stride < n4; i += 2 * stride) {
        const int4 a = __ldcs(e4 + i), b = __ldcs(e4 + i + stride);
        s += (long long)a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
    }
    for (; i < n4; i += stride) { const int4 a = __ldcs(e4 + i); s += (long long)a.x + a.y + a.z + a.w; }
    for (int64_t p = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < HW; p += stride) s += g.e[p];
    __shared__ long long red[8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[wid] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) t += red[i];
        if (t) atomicAdd(acc, (unsigned long long)t);
    }
}


}  // namespace

// ============================================================================
// host side
// ============================================================================
struct fm_grid {
    int32_t H = 0, W = 0, device = 0;
    int64_t HW = 0;
    GridDev d{};
    // device scratch: 64-bit accumulators and 32-bit flags
    unsigned long long *acc = nullptr;   // [0..15]
    int32_t *flags = nullptr;            // [0..63]
    unsigned long long *h_acc = nullptr; // pinned mirrors
    int32_t *h_flags = nullptr;
    // host-input staging for *_host / begin
    int32_t *in_caps = nullptr;          // 6 * HW
    uint8_t *d_cut_tmp = nullptr;
    uint8_t *h_cut_stage = nullptr;      // pinned bounce buffer for the cut (host-output calls)
    // fm_grid_solve_host_batch: a second input set, two device / pinned cut stages and
    // the copy streams (H2D of instance k+1 and D2H of instance k-1 overlap solve k)
    int32_t *in_caps2 = nullptr;
    uint8_t *b_narrow[2] = {nullptr, nullptr};   // narrow (uint8 / uint16) plane staging
    size_t b_narrow_bytes = 0;
    uint8_t *b_dcut[2] = {nullptr, nullptr};
    uint8_t *b_hcut[2] = {nullptr, nullptr};
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[8] = {};   // [0..3] phase / kernel timing, [4..7] a push round whose stats are read after the relabel
    int grid_blocks = 0;                 // 1-D grid-stride kernels
    int ntiles = 0;                      // 32 x 32 tiles of the tile-resident kernel
    int32_t *d_queues = nullptr;         // push + BFS tile work lists
    int sms = 148;
    int relabel_div = 0;                 // option RELABEL_DIV
    int pq_parity = 0;                   // parity of the next push launch
    int pt_per_sm = 3;                   // resident pr_tile CTAs per SM (occupancy query)
    int op_steps = 1;                    // operations per pixel per pass (option OP_STEPS)
    int op_fused = 0;                    // relabel then push in one operation (option OP_FUSED)
    int vote_mask = 7;                   // CTA activity vote every vote_mask+1 passes (option VOTE)
    int bfs_bits = 2;                    // 2: persistent bit-parallel BFS (bfs_ring_kernel), 1: bit-parallel
                                         // sweeps (bfs_bits_kernel), 0: v1 Jacobi sweeps (option BFS_BITS)
    int bb_per_sm = 8;                   // resident bfs_bits CTAs per SM (occupancy query)
    int br_per_sm = 8;                   // resident bfs_ring CTAs per SM (occupancy query, <= br_cap)
    int bfs_owner = 1;                   // global relabel BFS with owner scheduling (owner_bfs_kernel; option bfs_owner;
                                         // r02bv: BFS kernel 4096^2 -2..4%, 8192^2 -8% vs the ring)
    int br_cap = 8;                      // option BR_CAP
    RingQ rq{};                          // device work queue of the persistent BFS
    RingQ prq{};                         // device work queue of the persistent push round
    int pr_ring = 0;                     // 1: one persistent pr_ring_kernel launch per round (option PR_RING; experimental, slower)
    int two_hop = 1;                     // two-hop pre-routing after init (option TWO_HOP)
    int k_tail = 0;                      // passes per visit in tail rounds (0: k_local) (option K_TAIL)
    int ring_tail = -1;                  // rounds with active <= H*W / ring_tail run as one ring launch (option
                                         // ring_tail; -1 auto: 1024 up to 2^24 px, r02bc: 4096^2 -2%, 8192^2 +1.5%)
    int tail_div = 1024;                 // tail round: active pixels <= H*W / tail_div (option TAIL_DIV)
    int pr_batch = 0;                    // push launches between checks of the round triggers (option PR_BATCH; 0 = auto)
    int visit_mult = 16;                 // ring round visit cap = visit_mult x initially active tiles (option VISIT_MULT)
    bool ring_stats_pending = false;
    bool pr_stats_pending = false;
    int pr_graph = -1;                   // 1: the push round's launch loop runs as a device while-graph (option PR_GRAPH; -1 = auto)
    cudaGraph_t prg = nullptr;           // that graph, its instance and the launch parameters it was built for
    cudaGraphExec_t prg_exec = nullptr;
    GridDev prg_d{};
    int prg_key[6] = {0, 0, 0, 0, 0, 0};
    bool prg_pending = false;            // round control block read back, consumed after the caller's sync
    int pr_kernel = 1;                   // 1: pr_list_kernel (v3), 0: pr_tile_kernel (v2) (option PR_KERNEL)
    int pl_per_sm = 6;                   // resident pr_list CTAs per SM (occupancy query)
    int pk_per_sm = 8;                   // same, packed-residual instance (occupancy query)
    int pk = 1;                          // packed 16-bit residuals in the push kernel when the input allows (option PACKED)
    bool pk_ok = false;                  // this solve's input allows them (every pair sum <= 65535)
    int k_local_list = 0;                // passes per visit of the list kernel (option K_LOCAL_LIST)
    int bq_parity = 0;                   // parity of the next BFS / cut sweep
    uint8_t *d_touched = nullptr;        // per tile: pushed into since the last relabel
    uint8_t *d_region = nullptr;         // per tile: in the local relabel's region
    int32_t *d_rlist = nullptr;          // region tile list (+ count at the end)
    int local_div = 64;                  // local relabel once active <= H*W/local_div (0: never)
    int local_max = 12;                  // consecutive local relabels before a global one
    int local_margin = 2;                // region dilation in tiles
    int local_streak = 0;
    int pl_occ = 6, pk_occ = 8, br_occ = 8;  // occupancy maxima (options may only lower the CTAs per SM)
    int bo_occ = 8;                      // owner_bfs_kernel CTAs per SM (occupancy query)
    int k_local = 0;                     // tuning overrides (options k_local / bfs_interval)
    int trace = 0;                       // option TRACE=1: one stderr line per round
    int bfs_interval_env = 0;
    PlMaps maps{};                       // TMA descriptors of the push kernel's planes (tile visit staging)
    bool maps_ok = false;                // encoded (W % 4 == 0 and the driver entry point resolved)
    int tma = 1;                         // option TMA: stage tile visits with cp.async.bulk.tensor (0: cp.async)
    // row-band mode (fm_grid_band_*): this handle is band `band` of `nbands`
    int band = -1, nbands = 0;
    int colocated = 1;                   // bands sharing this device (persistent grids split between them)
    int32_t H_total = 0;                 // rows of the whole grid
    int64_t total_tiles = 0;             // tiles of the whole grid (the shared ring's initial pending count)
    unsigned *gpend = nullptr;           // shared pending counter of the band rings (band 0's rq.ctr + 200)
    void *ipc_open[2][10] = {};          // IPC mappings of the neighbours' buffers (closed on destroy)
    void *ipc_gpend = nullptr;           // IPC mapping of band 0's ring counters (bands > 1)
    int32_t *band_caps = nullptr;        // band inputs staged by fm_grid_band_solve: 6 planes + 2 halo rows
    // solve state
    int32_t flags_solve = 0;
    bool relabel_full = true;            // next global relabel rebuilds every tile's arc words
    bool inflow_deferred = false;        // this round's inboxes are folded in by the relabel preparation
    long long sum_capS = 0;
    long long excess_total = 0;          // maxflow_par.py HybridState.excess_total
    long long active = 0;
    fm_stats st{};
};

namespace {

int sync_stream(fm_grid *g) {
    FM_CHECK_CUDA(cudaStreamSynchronize(g->stream));
    return FM_OK;
}

// persistent ring grid: every resident slot, shared between the bands on this device
int ring_blocks(const fm_grid *g) {
    return std::max(1, g->sms * g->br_per_sm / std::max(1, g->colocated));
}

int use_tma(const fm_grid *g) { return g->tma && g->maps_ok ? 1 : 0; }

// TMA descriptors of the planes a push-kernel tile visit stages (PlMaps).  The encoder
// is the driver's cuTensorMapEncodeTiled, reached through the runtime's entry-point
// query (no libcuda link).  Planes must have a row pitch that is a 16-byte multiple.
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

void encode_maps(fm_grid *g) {
    g->maps_ok = false;
    if (g->W % 4) return;
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
        cudaGetLastError();
        return;
    }
    const EncodeTiledFn enc = (EncodeTiledFn)fn;
    const cuuint64_t dims[2] = {(cuuint64_t)g->W, (cuuint64_t)g->H};
    const cuuint64_t strides[1] = {(cuuint64_t)g->W * 4};
    const cuuint32_t tile_box[2] = {PT_W, PT_H}, halo_box[2] = {PL_HS, PT_H + 2}, es[2] = {1, 1};
    struct { CUtensorMap *m; int32_t *plane; const cuuint32_t *box; } list[] = {
        {&g->maps.e, g->d.e, tile_box}, {&g->maps.t, g->d.rT, tile_box}, {&g->maps.s, g->d.rS, tile_box},
        {&g->maps.h, g->d.h, halo_box}, {&g->maps.r[0], g->d.rR, tile_box}, {&g->maps.r[1], g->d.rL, tile_box},
        {&g->maps.r[2], g->d.rD, tile_box}, {&g->maps.r[3], g->d.rU, tile_box}};
    for (auto &x : list)
        if (enc(x.m, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, x.plane, dims, strides, x.box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS)
            return;
    g->maps_ok = true;
}

float elapsed_between(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

float elapsed(fm_grid *g) {
    float ms = 0.f;
    cudaEventSynchronize(g->ev[1]);
    cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]);
    return ms;
}


int tq_reset(fm_grid *g, const TileQueue &q) {
    FM_CHECK_CUDA(cudaMemsetAsync(q.flag[0], 0, sizeof(int32_t) * 2 * (size_t)g->ntiles, g->stream));
    FM_CHECK_CUDA(cudaMemsetAsync(q.cnt, 0, sizeof(int32_t) * 4, g->stream));
    return FM_OK;
}

// zero count[p^1] and work[p] before a launch of parity p
int tq_arm(fm_grid *g, const TileQueue &q, int p) {
    FM_CHECK_CUDA(cudaMemsetAsync(q.cnt + (p ? 0 : 2), 0, sizeof(int32_t) * 2, g->stream));
    return FM_OK;
}

// Repeated frontier sweeps of a tile fixpoint kernel until a sweep changes nothing.
// Sweep 0 visits every tile; sweep i drains bq.list[i&1] and fills the other list
// with the neighbours of tiles whose border changed.  Persistent CTAs take tiles
// from the list, so a sweep over a small frontier costs a few microseconds.  The
// per-sweep count of changed tiles lands in flags[j] (batches of 4 per host check).
template <typename K>
int frontier_sweeps(fm_grid *g, K kernel, bool first_all, int64_t *sweeps, int64_t *launches,
                    double *ms_kern, dim3 block = dim3(TILE_W, BLK_Y), int nblocks = 0) {
    if (first_all) {
        FM_TRY(tq_reset(g, g->d.bq));
        g->bq_parity = 0;
    }
    const int batch = 4;
    const int blocks = nblocks > 0 ? nblocks : std::min(g->ntiles, g->sms * 8);
    bool first = first_all;
    for (;;) {
        FM_CHECK_CUDA(cudaMemsetAsync(g->flags, 0, sizeof(int32_t) * batch, g->stream));
        cudaEventRecord(g->ev[2], g->stream);
        for (int j = 0; j < batch; j++) {
            const int p = g->bq_parity;
            FM_TRY(tq_arm(g, g->d.bq, p));
            kernel<<<blocks, block, 0, g->stream>>>(g->d, p, first ? 1 : 0, g->flags + j);
            first = false;
            g->bq_parity ^= 1;
        }
        FM_CHECK_LAUNCH();
        cudaEventRecord(g->ev[3], g->stream);
        g->st.launches += batch;
        *launches += batch;
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags, g->flags, sizeof(int32_t) * batch,
                                      cudaMemcpyDeviceToHost, g->stream));
        FM_TRY(sync_stream(g));
        *ms_kern += elapsed_between(g->ev[2], g->ev[3]);
        int idle_at = -1;
        for (int j = 0; j < batch; j++) {
            if (!g->h_flags[j]) { idle_at = j; break; }
            g->st.reserved[0] += g->h_flags[j];   // tile visits that changed something
        }
        *sweeps += idle_at < 0 ? batch : idle_at + 1;
        if (idle_at >= 0) break;
    }
    return FM_OK;
}

// residual arcs for the BFS (all tiles, or the listed local-relabel region)
int bfs_init(fm_grid *g, bool listed, int nlisted = 0) {
    if (g->bfs_bits) {
        const int rows = (listed ? nlisted : g->ntiles) * PT_H;
        const int blocks = std::max(1, std::min((rows + 7) / 8, g->sms * 16));
        bfs_init_bits_kernel<<<blocks, 256, 0, g->stream>>>(g->d, listed ? 1 : 0);
    } else if (listed) {
        bfs_init_local_kernel<<<std::max(1, std::min(nlisted, g->sms * 8)), 256, 0, g->stream>>>(g->d);
    } else {
        bfs_init_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(g->d);
    }
    FM_CHECK_LAUNCH();
    g->st.launches++;
    return FM_OK;
}

// BFS fixpoint over the tiles (all of them, or the ones queued in bq[bq_parity]).
// bfs_bits == 2 (default): one persistent launch over the device ring queue; the
// visit count lands in h_flags[8] and the kernel time between ev[2] / ev[3], both
// collected by bfs_collect() after the caller's next stream sync.
int bfs_sweeps(fm_grid *g, bool first_all) {
    if (g->bfs_bits == 2) {
        // first_all: every tile (see bfs_init_bits_kernel); else the tiles queued in bq
        const int32_t *list0 = first_all ? nullptr : g->d.bq.list[g->bq_parity];
        const int32_t *cnt0 = first_all ? nullptr : g->d.bq.cnt + 2 * g->bq_parity;
        if (!first_all) FM_CHECK_CUDA(cudaMemsetAsync(g->rq.flag, 0, sizeof(int32_t) * (size_t)g->ntiles, g->stream));
        ringq_init_kernel<<<std::min((g->rq.cap + 255) / 256, g->sms * 8), 256, 0, g->stream>>>(g->rq, g->ntiles, list0, cnt0);
        FM_CHECK_LAUNCH();
        cudaEventRecord(g->ev[2], g->stream);
        ring_kernel<0><<<ring_blocks(g), 32 * BB_WARPS, 0, g->stream>>>(g->d, g->rq);
        FM_CHECK_LAUNCH();
        cudaEventRecord(g->ev[3], g->stream);
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags + 8, g->rq.ctr + 96, sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags + 10, g->rq.ctr + 192, sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags + 11, g->rq.ctr + 224, sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
        FM_TRY(tq_reset(g, g->d.bq));
        g->bq_parity = 0;
        g->st.launches += 2;
        g->st.bfs_sweeps += 1;
        g->st.bfs_launches += 1;
        g->ring_stats_pending = true;
        return FM_OK;
    }
    if (g->bfs_bits)
        return frontier_sweeps(g, bfs_bits_kernel, first_all, &g->st.bfs_sweeps, &g->st.bfs_launches,
                               &g->st.ms_bfs_kern, dim3(32 * BB_WARPS),
                               std::min((g->ntiles + BB_WARPS - 1) / BB_WARPS, g->sms * g->bb_per_sm));
    return frontier_sweeps(g, bfs_tile_kernel, first_all, &g->st.bfs_sweeps, &g->st.bfs_launches,
                           &g->st.ms_bfs_kern);
}

// after a stream sync: fold the ring BFS's kernel time and visit count into the stats
void bfs_collect(fm_grid *g) {
    if (!g->ring_stats_pending) return;
    g->ring_stats_pending = false;
    g->st.ms_bfs_kern += elapsed_between(g->ev[2], g->ev[3]);
    g->st.reserved[0] += g->h_flags[8];
    const float kms = elapsed_between(g->ev[2], g->ev[3]);
    if (g->trace) {
        unsigned long long tv[4] = {}, ts[5] = {};
        cudaMemcpy(tv, g->rq.ctr + 240, sizeof(tv), cudaMemcpyDeviceToHost);   // FM_BFS_TIMING builds
        cudaMemcpy(ts, g->rq.ctr + 208, sizeof(ts), cudaMemcpyDeviceToHost);
        const double nv = (double)std::max(1, g->h_flags[10]);
        if (ts[1]) fprintf(stderr, "[fm_grid]   bfs ring cycles per visit: wait %.0f load %.0f levels %.0f write %.0f queue %.0f\n",
                           ts[0] / nv, ts[1] / nv, ts[2] / nv, ts[3] / nv, ts[4] / nv);
        const double warps = (double)g->sms * g->br_per_sm * BB_WARPS;
        fprintf(stderr, "[fm_grid]   bfs ring: %d seeded tiles, %d visits (%d changed), %.3f ms | busy %.2f, "
                "cycles/visit %.0f (level loop %.0f), levels/visit %.1f\n", g->h_flags[11], g->h_flags[10], g->h_flags[8], kms,
                tv[0] / (kms * 1.965e6 * warps), tv[0] / (double)std::max(1, g->h_flags[10]),
                tv[3] / (double)std::max(1, g->h_flags[10]), tv[2] / (double)std::max(1, g->h_flags[10]));
    }
}

int bfs_finalize(fm_grid *g) {
    if (g->bfs_bits)
        bfs_finalize_tiles_kernel<<<std::min(g->ntiles, g->sms * 8), 256, 0, g->stream>>>(g->d, g->acc + 4, nullptr, 0);
    else
        bfs_finalize_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(g->d, g->acc + 4);
    FM_CHECK_LAUNCH();
    g->st.launches++;
    return FM_OK;
}

// global relabel + gap + marking; leaves the active-pixel count in g->active and
// the tiles holding active pixels in the push work list (parity 0)
int global_relabel(fm_grid *g) {
    if (g->bfs_bits == 2 && g->nbands == 0) {
        // default path: fused preparation, one ring launch, finalize, one host sync
        cudaEventRecord(g->ev[0], g->stream);
        const bool full = g->relabel_full || g->pr_kernel != 1 || g->pr_ring ||
                          (g->flags_solve & (FM_GRID_GLOBAL_SWEEP | FM_GRID_CANCEL_VIOLATIONS));
        const bool whole = g->d.ntx % 4 == 0 && g->W == g->d.ntx * PT_W && g->H == g->d.nty * PT_H;
        (whole ? relabel_init_kernel<true> : relabel_init_kernel<false>)
            <<<std::max(1, std::min((g->ntiles * (PT_H / 4) + 7) / 8, g->sms * (whole ? 4 : 6))), 256, 0, g->stream>>>(
                g->d, g->rq, full ? 1 : 0, g->inflow_deferred ? 1 : 0, g->acc + 4);
        g->inflow_deferred = false;
        FM_CHECK_LAUNCH();
        cudaEventRecord(g->ev[2], g->stream);
        const int rb = ring_blocks(g);
        // owner scheduling needs every owning warp resident at once (a tile is only ever
        // visited by its owner): a cooperative launch guarantees that or refuses, and a
        // refusal (e.g. the device shared with other work) falls back to the ring queue
        const int ob = g->sms * std::max(1, std::min(g->bo_occ, g->br_cap));
        bool launched = false;
        if (g->bfs_owner && g->ntiles <= 64 * ob * BB_WARPS) {
            void *args[] = {(void *)&g->d, (void *)&g->rq};
            launched = cudaLaunchCooperativeKernel((void *)owner_bfs_kernel, dim3(ob), dim3(32 * BB_WARPS), args, 0,
                                                   g->stream) == cudaSuccess;
            if (!launched) cudaGetLastError();
        }
        if (!launched) ring_kernel<0><<<rb, 32 * BB_WARPS, 0, g->stream>>>(g->d, g->rq);
        FM_CHECK_LAUNCH();
        cudaEventRecord(g->ev[3], g->stream);
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags + 8, g->rq.ctr + 96, sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags + 10, g->rq.ctr + 192, sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags + 11, g->rq.ctr + 224, sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
        g->pq_parity = 0;
        FM_TRY(bfs_finalize(g));   // clears the touched flags
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc + 4, g->acc + 4, sizeof(unsigned long long) * 3,
                                      cudaMemcpyDeviceToHost, g->stream));
        cudaEventRecord(g->ev[1], g->stream);
        g->st.launches += 2;
        g->st.bfs_sweeps += 1;
        g->st.bfs_launches += 1;
        g->ring_stats_pending = true;
        FM_TRY(sync_stream(g));
        bfs_collect(g);
        g->st.ms_bfs += elapsed(g);
        g->active = (long long)g->h_acc[4];
        g->excess_total -= (long long)g->h_acc[5];
        g->st.bfs_levels = std::max<int64_t>(g->st.bfs_levels, (int64_t)g->h_acc[6]);
        g->relabel_full = false;
        return FM_OK;
    }
    cudaEventRecord(g->ev[0], g->stream);
    FM_TRY(bfs_init(g, false));
    FM_TRY(bfs_sweeps(g, true));
    FM_CHECK_CUDA(cudaMemsetAsync(g->acc + 4, 0, sizeof(unsigned long long) * 3, g->stream));
    FM_TRY(tq_reset(g, g->d.pq));
    g->pq_parity = 0;
    FM_TRY(bfs_finalize(g));
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc + 4, g->acc + 4, sizeof(unsigned long long) * 3,
                                  cudaMemcpyDeviceToHost, g->stream));
    cudaEventRecord(g->ev[1], g->stream);
    FM_TRY(sync_stream(g));
    bfs_collect(g);
    g->st.ms_bfs += elapsed(g);
    g->active = (long long)g->h_acc[4];
    g->excess_total -= (long long)g->h_acc[5];
    g->st.bfs_levels = std::max<int64_t>(g->st.bfs_levels, (int64_t)g->h_acc[6]);
    FM_CHECK_CUDA(cudaMemsetAsync(g->d_touched, 0, (size_t)g->ntiles, g->stream));
    return FM_OK;
}

// Local relabel over the region of tiles touched since the last relabel (see
// region_build_kernel).  Falls back to the global relabel when the region is large.
int local_relabel(fm_grid *g) {
    cudaEventRecord(g->ev[0], g->stream);
    FM_TRY(tq_reset(g, g->d.bq));
    FM_CHECK_CUDA(cudaMemsetAsync(g->d_rlist + g->ntiles, 0, sizeof(int32_t), g->stream));
    region_build_kernel<<<(g->ntiles + 255) / 256, 256, 0, g->stream>>>(g->d, g->d_region, g->local_margin,
                                                                         g->d_rlist + g->ntiles);
    FM_CHECK_LAUNCH();
    FM_CHECK_CUDA(cudaMemcpyAsync(g->d_rlist, g->d.bq.list[0], sizeof(int32_t) * g->ntiles,
                                  cudaMemcpyDeviceToDevice, g->stream));
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags, g->d_rlist + g->ntiles, sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
    FM_TRY(sync_stream(g));
    const int nr = g->h_flags[0];
    g->st.launches++;
    if (nr > g->ntiles / 4) return global_relabel(g);
    g->d.region = g->d_region;
    FM_TRY(bfs_init(g, true, nr));
    g->bq_parity = 0;
    int rc = bfs_sweeps(g, false);
    if (rc == FM_OK) {
        FM_CHECK_CUDA(cudaMemsetAsync(g->acc + 4, 0, sizeof(unsigned long long) * 3, g->stream));
        FM_TRY(tq_reset(g, g->d.pq));
        g->pq_parity = 0;
        if (g->bfs_bits)
            bfs_finalize_tiles_kernel<<<std::max(1, std::min(nr, g->sms * 8)), 256, 0, g->stream>>>(
                g->d, g->acc + 4, g->d_rlist, nr);
        else
            bfs_finalize_local_kernel<<<std::max(1, std::min(nr, g->sms * 8)), 256, 0, g->stream>>>(
                g->d, g->d_rlist, nr, g->acc + 4);
        FM_CHECK_LAUNCH();
        g->st.launches++;
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc + 4, g->acc + 4, sizeof(unsigned long long) * 3,
                                      cudaMemcpyDeviceToHost, g->stream));
        cudaEventRecord(g->ev[1], g->stream);
        FM_TRY(sync_stream(g));
        bfs_collect(g);
        g->st.ms_bfs += elapsed(g);
        g->active = (long long)g->h_acc[4];
        g->excess_total -= (long long)g->h_acc[5];
        g->st.reserved[1]++;  // local relabels
    }
    g->d.region = nullptr;
    FM_CHECK_CUDA(cudaMemsetAsync(g->d_touched, 0, (size_t)g->ntiles, g->stream));
    return rc;
}

int current_flow(fm_grid *g, long long *flow);

int begin_device(fm_grid *g, const int32_t *capR, const int32_t *capL, const int32_t *capD,
                 const int32_t *capU, const int32_t *capS, const int32_t *capT, int32_t flags) {
    g->flags_solve = flags;
    g->local_streak = 0;
    g->relabel_full = true;   // init + two-hop changed every residual
    g->inflow_deferred = false;
    memset(&g->st, 0, sizeof(g->st));
    FM_CHECK_CUDA(cudaMemsetAsync(g->d_touched, 0, (size_t)g->ntiles, g->stream));
    FM_CHECK_CUDA(cudaMemsetAsync(g->acc, 0, sizeof(unsigned long long) * 32, g->stream));
    grid_init_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(
        g->d, capR, capL, capD, capU, capS, capT, nullptr, nullptr, (flags & FM_GRID_NO_PRECANCEL) ? 0 : 1, g->acc);
    FM_CHECK_LAUNCH();
    g->st.launches++;
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc, g->acc, sizeof(unsigned long long) * 4,
                                  cudaMemcpyDeviceToHost, g->stream));
    FM_TRY(sync_stream(g));
    g->pk_ok = g->h_acc[3] == 0;
    if (g->h_acc[1] != 0) {
        fm_set_error("negative capacity in grid input (%llu entries)", g->h_acc[1]);
        return FM_INVALID_ARG;
    }
    if (g->h_acc[2] != 0) {
        fm_set_error("grid capacities too large for the int32 device state: %llu pixels where capS plus the "
                     "capacities into the pixel, or a neighbour pair's two capacities, exceed 2^31-1", g->h_acc[2]);
        return FM_INVALID_ARG;
    }
    g->sum_capS = (long long)g->h_acc[0];
    // HybridState.excess_total = sum of excess after init_preflow = sum capS
    // (maxflow_par.py:56); pre-cancelled units are already at t.
    g->excess_total = g->sum_capS;
    if (g->trace) {
        long long f = 0;
        FM_TRY(current_flow(g, &f));
        fprintf(stderr, "[fm_grid] after pre-cancellation: %lld of %lld source units at the sink\n", f, g->sum_capS);
    }
    if (g->two_hop && !(flags & FM_GRID_NO_PRECANCEL)) {
        two_hop_kernel<<<dim3((unsigned)((g->W + 255) / 256), (unsigned)std::min(g->H, 65535)), 256, 0, g->stream>>>(g->d);
        FM_CHECK_LAUNCH();
        g->st.launches++;
        if (g->two_hop >= 2) {
            three_hop_kernel<<<(unsigned)((g->HW + 255) / 256), 256, 0, g->stream>>>(g->d);
            FM_CHECK_LAUNCH();
            g->st.launches++;
        }
        if (g->trace) {
            long long f = 0;
            FM_TRY(current_flow(g, &f));
            fprintf(stderr, "[fm_grid] after two-hop pre-routing: %lld of %lld source units at the sink\n", f, g->sum_capS);
        }
    }
    return global_relabel(g);
}

// One coordinator round: lock-free launches over the work list of tiles until an
// idle launch, until relabels since the last global relabel reach the relabel
// budget (the O(V)-work trigger of the reference's sequential solver,
// maxflow_seq.py:197-205 -- heuristic_period relabels between global relabels),
// or until the launch cap; then cancel (opt-in), global relabel, gap, mark
// (maxflow_par.py:195-229).
constexpr int K_LOCAL_DEFAULT = 32;      // lock-free passes per tile visit (v2)
constexpr int K_LOCAL_LIST_DEFAULT = 20; // passes per tile visit (v3: a pass over an empty list ends it)
constexpr int K_LOCAL_LIST_LARGE = 32;   // ... on grids >= 2^23 pixels
constexpr int MAX_LAUNCHES_DEFAULT = 16; // launch cap per round
constexpr int RELABEL_DIV_DEFAULT = 16;  // relabel budget = H*W / div
// grids >= 2^23 px end a push round after half as many relabels (r02h35/36: 8192^2
// 62.2 -> 60.0 ms, 4096^2 20.5 -> 20.2-20.4 ms; fewer stale-height operations per round)
constexpr int RELABEL_DIV_LARGE = 32;
inline int relabel_div_default(int64_t hw) { return hw >= ((int64_t)1 << 23) ? RELABEL_DIV_LARGE : RELABEL_DIV_DEFAULT; }

int run_round_global(fm_grid *g, int32_t cycle_budget, int32_t bfs_interval, int32_t *done_out) {
    const int32_t cap = std::max(1, std::min(cycle_budget, bfs_interval > 0 ? bfs_interval : 64));
    const dim3 grid((g->W + TILE_W - 1) / TILE_W, (g->H + BLK_Y - 1) / BLK_Y);
    int32_t done = 0;
    while (done < cap) {
        const int batch = std::min(8, cap - done);
        FM_CHECK_CUDA(cudaMemsetAsync(g->flags, 0, sizeof(int32_t) * batch, g->stream));
        cudaEventRecord(g->ev[2], g->stream);
        for (int i = 0; i < batch; i++)
            pr_sweep_kernel<<<grid, dim3(TILE_W, BLK_Y), 0, g->stream>>>(g->d, g->flags + i, g->acc + 10);
        FM_CHECK_LAUNCH();
        cudaEventRecord(g->ev[3], g->stream);
        g->st.launches += batch;
        g->st.pr_launches += batch;
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags, g->flags, sizeof(int32_t) * batch,
                                      cudaMemcpyDeviceToHost, g->stream));
        FM_TRY(sync_stream(g));
        g->st.ms_pr_kern += elapsed_between(g->ev[2], g->ev[3]);
        int idle_at = -1;
        for (int i = 0; i < batch; i++) if (!g->h_flags[i]) { idle_at = i; break; }
        done += idle_at < 0 ? batch : idle_at + 1;
        if (idle_at >= 0) break;
    }
    g->st.pr_sweeps += done;
    g->st.pr_tiles += (int64_t)done * g->ntiles;
    *done_out = done;
    return FM_OK;
}

// The round control block lives in flags[32..41]; its host mirror in h_flags[32..41].
PrCtl *pr_ctl_dev(fm_grid *g) { return reinterpret_cast<PrCtl *>(g->flags + 32); }
PrCtl *pr_ctl_host(fm_grid *g) { return reinterpret_cast<PrCtl *>(g->h_flags + 32); }

// (Re)build the push-round while-graph for these launch parameters (body: one
// pr_list_kernel node whose last CTA sets the loop condition).  Rebuilt only when a
// parameter baked into the node changes.
int pr_graph_build(fm_grid *g, int k_local, int blocks, bool pk) {
    const int key[6] = {k_local, blocks, g->op_steps, g->op_fused, pk ? 1 : 0, use_tma(g)};
    if (g->prg_exec && !memcmp(key, g->prg_key, sizeof(key)) && !memcmp(&g->d, &g->prg_d, sizeof(GridDev)))
        return FM_OK;
    if (g->prg_exec) { cudaGraphExecDestroy(g->prg_exec); g->prg_exec = nullptr; }
    if (g->prg) { cudaGraphDestroy(g->prg); g->prg = nullptr; }
    FM_CHECK_CUDA(cudaGraphCreate(&g->prg, 0));
    cudaGraphConditionalHandle handle;
    FM_CHECK_CUDA(cudaGraphConditionalHandleCreate(&handle, g->prg, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = handle;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t loop;
    FM_CHECK_CUDA(cudaGraphAddNode(&loop, g->prg, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];

    PrCtl *ctl = pr_ctl_dev(g);
    GridDev d = g->d;
    int steps = g->op_steps, fused = g->op_fused, parity0 = 0;
    int32_t *processed = &ctl->processed;
    unsigned long long *ops = g->acc + 10;
    PlMaps maps = g->maps;
    int tma = use_tma(g);
    void *pr_args[] = {&d, &k_local, &steps, &fused, &parity0, &processed, &ops, &ctl, &handle, &maps, &tma};
    cudaKernelNodeParams kp{};
    kp.func = pk ? (void *)pr_list_kernel<true> : (void *)pr_list_kernel<false>;
    kp.gridDim = dim3(blocks);
    kp.blockDim = dim3(PT_W, PL_TY);
    kp.kernelParams = pr_args;
    cudaGraphNode_t n;
    FM_CHECK_CUDA(cudaGraphAddKernelNode(&n, body, nullptr, 0, &kp));
    FM_CHECK_CUDA(cudaGraphInstantiate(&g->prg_exec, g->prg, 0));
    memcpy(g->prg_key, key, sizeof(key));
    g->prg_d = g->d;
    return FM_OK;
}

// Fold the control block of the last graph round into the stats (after a stream sync).
void pr_graph_consume(fm_grid *g, int32_t *idle_out, bool keep_parity = false) {
    if (!g->prg_pending) return;
    g->prg_pending = false;
    const PrCtl *c = pr_ctl_host(g);
    g->st.ms_pr_kern += elapsed_between(g->ev[6], g->ev[7]);
    g->st.launches += c->done;
    g->st.pr_launches += c->done;
    g->st.pr_sweeps += c->done;
    g->st.pr_tiles += (int64_t)c->tiles;
    if (!keep_parity) g->pq_parity = c->parity;   // (a relabel that ran since reset the lists)
    if (idle_out) *idle_out = c->processed == 0 ? 1 : 0;
}

// fold the push round's parked inboxes into e and the residuals -- unless the global
// relabel that follows does it in its preparation pass (inflow_deferred)
int integrate_inflow(fm_grid *g) {
    if (g->inflow_deferred) return FM_OK;
    integrate_inflow_kernel<<<g->ntiles, 4 * PT_W, 0, g->stream>>>(g->d);
    FM_CHECK_LAUNCH();
    g->st.launches++;
    return FM_OK;
}

int run_round_tiles(fm_grid *g, int32_t cycle_budget, int32_t bfs_interval, int32_t *idle_out = nullptr) {
    // passes per visit: large grids (the device-side round loop below, TMA-staged visits)
    // amortise a visit over 32 passes (4096^2: 23.1 -> 21.8 ms, 8192^2: 71.6 -> 66.5 ms),
    // smaller ones keep 20 (2048^2 segmentation 1.44 vs 1.57 ms at 32; r02ae)
    const bool large_grid = g->HW >= ((int64_t)1 << 23);
    const int k_list_auto = large_grid ? K_LOCAL_LIST_LARGE : K_LOCAL_LIST_DEFAULT;
    const int k_default = g->pr_kernel == 1 ? (g->k_local_list > 0 ? g->k_local_list : k_list_auto)
                                            : (g->k_local > 0 ? g->k_local : K_LOCAL_DEFAULT);
    // tail rounds (few active pixels, far from the sink): more passes per visit
    const bool tail = g->k_tail > 0 && g->active <= g->HW / std::max(1, g->tail_div);
    const int k_local = std::max(1, std::min(cycle_budget, tail ? g->k_tail : k_default));
    if (bfs_interval <= 0 && g->bfs_interval_env > 0) bfs_interval = g->bfs_interval_env;
    const int32_t cap = std::max(1, std::min((cycle_budget + k_local - 1) / k_local,
                                             bfs_interval > 0 ? bfs_interval : MAX_LAUNCHES_DEFAULT));
    const long long relabel_budget =
        std::max<long long>(1024, g->HW / (g->relabel_div > 0 ? g->relabel_div : relabel_div_default(g->HW)));
    const bool pk = g->pk && g->pk_ok && g->op_steps == 1 && !g->op_fused;
    const int blocks = std::min(g->ntiles, g->sms * (g->pr_kernel == 1 ? (pk ? g->pk_per_sm : g->pl_per_sm) : g->pt_per_sm));
    // Round triggers checked every `batch` launches.  Auto: large grids (>= 2^23 pixels) check
    // every 2 launches on the device (the round's launch loop as a while-graph, no host
    // round trip per check): a launch there is long enough that overshooting the relabel
    // budget by 3 launches of stale-height work (-22% operations at 4096^2) costs more than
    // the extra global relabels; smaller grids check every 4 launches from the host (r02r).
    const bool large = g->HW >= ((int64_t)1 << 23);
    const int batch_auto = g->pr_batch > 0 ? g->pr_batch : (large ? 2 : 4);
    const bool use_graph = g->pr_graph >= 0 ? g->pr_graph != 0 : large;
    if (use_graph && g->pr_kernel == 1) {
        FM_TRY(pr_graph_build(g, k_local, blocks, pk));
        PrCtl *h = pr_ctl_host(g);
        *h = PrCtl{};
        h->parity = g->pq_parity;
        h->cap = cap;
        h->batch = std::max(1, batch_auto);
        h->budget = relabel_budget;
        prctl_set_kernel<<<1, 1, 0, g->stream>>>(pr_ctl_dev(g), *h);
        FM_CHECK_LAUNCH();
        FM_TRY(tq_arm(g, g->d.pq, g->pq_parity));
        cudaEventRecord(g->ev[6], g->stream);
        FM_CHECK_CUDA(cudaGraphLaunch(g->prg_exec, g->stream));
        cudaEventRecord(g->ev[7], g->stream);
        FM_CHECK_CUDA(cudaMemcpyAsync(h, pr_ctl_dev(g), sizeof(PrCtl), cudaMemcpyDeviceToHost, g->stream));
        g->prg_pending = true;
        FM_TRY(integrate_inflow(g));
        return FM_OK;
    }
    int32_t done = 0;
    while (done < cap) {
        const int batch = std::min(batch_auto, cap - done);
        FM_CHECK_CUDA(cudaMemsetAsync(g->flags, 0, sizeof(int32_t) * batch, g->stream));
        cudaEventRecord(g->ev[2], g->stream);
        for (int i = 0; i < batch; i++) {
            const int p = g->pq_parity;
            FM_TRY(tq_arm(g, g->d.pq, p));
            if (g->pr_kernel == 1)
                (pk ? pr_list_kernel<true> : pr_list_kernel<false>)<<<blocks, dim3(PT_W, PL_TY), 0, g->stream>>>(
                    g->d, k_local, g->op_steps, g->op_fused, p, g->flags + i, g->acc + 10, nullptr, 0, g->maps, use_tma(g));
            else
                pr_tile_kernel<<<blocks, dim3(PT_W, PT_TY), 0, g->stream>>>(g->d, k_local, g->op_steps, g->op_fused, g->vote_mask, p, g->flags + i, g->acc + 10);
            g->pq_parity ^= 1;
        }
        FM_CHECK_LAUNCH();
        cudaEventRecord(g->ev[3], g->stream);
        g->st.launches += batch;
        g->st.pr_launches += batch;
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags, g->flags, sizeof(int32_t) * batch,
                                      cudaMemcpyDeviceToHost, g->stream));
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc + 10, g->acc + 10, sizeof(unsigned long long) * 2,
                                      cudaMemcpyDeviceToHost, g->stream));
        FM_TRY(sync_stream(g));
        g->st.ms_pr_kern += elapsed_between(g->ev[2], g->ev[3]);
        if (g->trace >= 3)
            fprintf(stderr, "[fm_grid]   batch: %.3f ms, tiles per launch %d %d %d %d\n", elapsed_between(g->ev[2], g->ev[3]),
                    g->h_flags[0], batch > 1 ? g->h_flags[1] : -1, batch > 2 ? g->h_flags[2] : -1, batch > 3 ? g->h_flags[3] : -1);
        int idle_at = -1;
        for (int i = 0; i < batch; i++) {
            if (!g->h_flags[i]) { idle_at = i; break; }
            g->st.pr_tiles += g->h_flags[i];
        }
        done += idle_at < 0 ? batch : idle_at + 1;
        if (idle_at >= 0) {
            if (idle_out) *idle_out = 1;
            break;
        }
        if ((long long)g->h_acc[11] >= relabel_budget) break;
    }
    FM_TRY(integrate_inflow(g));
    g->st.pr_sweeps += done;
    return FM_OK;
}

// One coordinator round as a single persistent launch over the device tile queue
// (pr_ring_kernel), seeded with the tiles the last relabel found active.  Kernel
// time and visit count are collected after the caller's stream sync.
int run_round_ring(fm_grid *g, int32_t cycle_budget) {
    const int k_default = g->k_local_list > 0 ? g->k_local_list : K_LOCAL_LIST_DEFAULT;
    const int k_local = std::max(1, std::min(cycle_budget, k_default));
    const long long relabel_budget =
        std::max<long long>(1024, g->HW / (g->relabel_div > 0 ? g->relabel_div : relabel_div_default(g->HW)));
    FM_CHECK_CUDA(cudaMemsetAsync(g->prq.flag, 0, sizeof(int32_t) * (size_t)g->ntiles, g->stream));
    ringq_init_kernel<<<std::min((g->prq.cap + 255) / 256, g->sms * 8), 256, 0, g->stream>>>(
        g->prq, g->ntiles, g->d.pq.list[0], g->d.pq.cnt + 0);
    FM_CHECK_LAUNCH();
    cudaEventRecord(g->ev[2], g->stream);
    pr_ring_kernel<<<g->sms * g->pl_per_sm, dim3(PT_W, PL_TY), 0, g->stream>>>(
        g->d, g->prq, k_local, g->op_steps, g->op_fused, relabel_budget, g->visit_mult, g->acc + 10);
    FM_CHECK_LAUNCH();
    cudaEventRecord(g->ev[3], g->stream);
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags + 9, g->prq.ctr + 96, sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
    FM_TRY(integrate_inflow(g));
    g->st.launches += 2;
    g->st.pr_launches += 1;
    g->st.pr_sweeps += 1;
    g->pr_stats_pending = true;
    return FM_OK;
}

int run_round(fm_grid *g, int32_t cycle_budget, int32_t bfs_interval) {
    const fm_stats before = g->st;
    const long long active_before = g->active;
    cudaEventRecord(g->ev[4], g->stream);
    FM_CHECK_CUDA(cudaMemsetAsync(g->acc + 10, 0, sizeof(unsigned long long) * 2, g->stream));
    int32_t sweeps = 0;
    // the relabel that closes this round (decided by the last relabel's active count)
    const bool go_local = g->local_div > 0 && !(g->flags_solve & FM_GRID_GLOBAL_SWEEP) &&
                          !(g->flags_solve & FM_GRID_CANCEL_VIOLATIONS) &&
                          g->active <= g->HW / g->local_div && g->local_streak < g->local_max;
    // a global relabel over whole 4-tile groups folds the inboxes in (no integrate pass)
    g->inflow_deferred = !go_local && g->bfs_bits == 2 && g->nbands == 0 && g->pr_kernel == 1 &&
                         !(g->flags_solve & (FM_GRID_GLOBAL_SWEEP | FM_GRID_CANCEL_VIOLATIONS)) &&
                         g->d.ntx % 4 == 0 && g->W == g->d.ntx * PT_W && g->H == g->d.nty * PT_H;
    // tail rounds (few active pixels, flow crossing many tiles) as one persistent launch
    const int ring_tail = g->ring_tail >= 0 ? g->ring_tail : (g->HW <= ((int64_t)1 << 24) ? 1024 : 0);
    if (g->flags_solve & FM_GRID_GLOBAL_SWEEP) {
        FM_TRY(run_round_global(g, cycle_budget, bfs_interval, &sweeps));
    } else if (g->pr_kernel == 1 && bfs_interval <= 0 && g->bfs_interval_env <= 0 &&
               (g->pr_ring || (ring_tail > 0 && g->active <= g->HW / ring_tail))) {
        FM_TRY(run_round_ring(g, cycle_budget));
        g->relabel_full = true;   // the next relabel prepares every tile (as with pr_ring)
    } else {
        FM_TRY(run_round_tiles(g, cycle_budget, bfs_interval));
    }
    if (g->flags_solve & FM_GRID_CANCEL_VIOLATIONS) {
        cancel_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(g->d, g->acc + 12);
        FM_CHECK_LAUNCH();
        g->st.launches++;
    }
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc + 10, g->acc + 10, sizeof(unsigned long long) * 5,
                                  cudaMemcpyDeviceToHost, g->stream));
    cudaEventRecord(g->ev[5], g->stream);
    // The relabel decision needs nothing from this push round, so its counters are read
    // after the relabel's own stream sync (one host round trip per round); the ring push
    // variant reuses ev[2]/ev[3] and is collected here.
    const auto collect = [&](bool after_relabel) {
        pr_graph_consume(g, nullptr, after_relabel);
        if (g->pr_stats_pending) {
            g->pr_stats_pending = false;
            g->st.ms_pr_kern += elapsed_between(g->ev[2], g->ev[3]);
            g->st.pr_tiles += g->h_flags[9];
        }
        g->st.ms_push += elapsed_between(g->ev[4], g->ev[5]);
        g->st.pushes += (int64_t)g->h_acc[10];
        g->st.relabels += (int64_t)g->h_acc[11];
        g->st.reserved[2] = (int64_t)g->h_acc[13];   // list-kernel passes (cumulative per solve)
        g->st.reserved[3] = (int64_t)g->h_acc[14];   // list-kernel items
    };
    const bool deferred = !g->pr_stats_pending;
    if (!deferred) {
        FM_TRY(sync_stream(g));
        collect(false);
    }
    if (go_local) {
        g->local_streak++;
        FM_TRY(local_relabel(g));
    } else {
        g->local_streak = 0;
        FM_TRY(global_relabel(g));
    }
    if (deferred) collect(true);   // the relabel synchronised the stream (and reset the work lists)
    g->st.rounds++;
    if (g->trace)
        fprintf(stderr, "[fm_grid] round %lld active %lld -> %lld | launches %lld tiles %lld pushes %lld relabels %lld "
                "push %.3f ms | bfs sweeps %lld %.3f ms levels %lld\n", (long long)g->st.rounds, active_before, g->active,
                (long long)(g->st.pr_sweeps - before.pr_sweeps), (long long)(g->st.pr_tiles - before.pr_tiles),
                (long long)(g->st.pushes - before.pushes), (long long)(g->st.relabels - before.relabels),
                g->st.ms_push - before.ms_push, (long long)(g->st.bfs_sweeps - before.bfs_sweeps),
                g->st.ms_bfs - before.ms_bfs, (long long)g->st.bfs_levels);
    return FM_OK;
}

// seeded residual reach: seeds + residual masks, then tile fixpoint sweeps
int cut_init(fm_grid *g) {
    if (g->bfs_bits) {
        const int rows = g->ntiles * PT_H;
        cut_init_bits_kernel<<<std::max(1, std::min((rows + 7) / 8, g->sms * 16)), 256, 0, g->stream>>>(g->d);
    } else {
        cut_init_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(g->d);
    }
    FM_CHECK_LAUNCH();
    g->st.launches++;
    return FM_OK;
}

// K3 as one persistent ring launch over every tile (default, bfs_bits == 2)
int cut_ring(fm_grid *g) {
    ringq_init_kernel<<<std::min((g->rq.cap + 255) / 256, g->sms * 8), 256, 0, g->stream>>>(g->rq, g->ntiles, nullptr, nullptr);
    FM_CHECK_LAUNCH();
    ring_kernel<1><<<ring_blocks(g), 32 * BB_WARPS, 0, g->stream>>>(g->d, g->rq);
    FM_CHECK_LAUNCH();
    g->st.launches += 2;
    g->st.cut_sweeps += 1;
    return FM_OK;
}

int cut_sweeps(fm_grid *g, bool first_all) {
    if (g->bfs_bits == 2) return cut_ring(g);
    double cut_kern = 0.0;
    int64_t cut_launches = 0;
    if (g->bfs_bits)
        return frontier_sweeps(g, cut_bits_kernel, first_all, &g->st.cut_sweeps, &cut_launches, &cut_kern,
                               dim3(32 * BB_WARPS),
                               std::min((g->ntiles + BB_WARPS - 1) / BB_WARPS, g->sms * g->bb_per_sm));
    return frontier_sweeps(g, cut_tile_kernel, first_all, &g->st.cut_sweeps, &cut_launches, &cut_kern);
}

int compute_cut(fm_grid *g, uint8_t *cut_out_dev) {
    g->relabel_full = true;   // the cut's incoming-arc words overwrite the BFS arc words
    cudaEventRecord(g->ev[0], g->stream);
    FM_TRY(cut_init(g));
    FM_TRY(cut_sweeps(g, true));
    if (cut_out_dev && cut_out_dev != g->d.cut)
        FM_CHECK_CUDA(cudaMemcpyAsync(cut_out_dev, g->d.cut, (size_t)g->HW, cudaMemcpyDeviceToDevice, g->stream));
    cudaEventRecord(g->ev[1], g->stream);
    FM_TRY(sync_stream(g));
    g->st.ms_cut += elapsed(g);
    return FM_OK;
}

int current_flow(fm_grid *g, long long *flow) {
    FM_CHECK_CUDA(cudaMemsetAsync(g->acc + 8, 0, sizeof(unsigned long long), g->stream));
    sum_e_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(g->d, g->acc + 8);
    FM_CHECK_LAUNCH();
    g->st.launches++;
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc + 8, g->acc + 8, sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, g->stream));
    FM_TRY(sync_stream(g));
    *flow = g->sum_capS - (long long)g->h_acc[8];
    return FM_OK;
}

int set_stream(fm_grid *g, void *stream) {
    g->stream = stream ? (cudaStream_t)stream : g->own_stream;
    return FM_OK;
}

int solve_device(fm_grid *g, const int32_t *capR, const int32_t *capL, const int32_t *capD,
                 const int32_t *capU, const int32_t *capS, const int32_t *capT,
                 int32_t cycle_budget, int32_t bfs_interval, int32_t flags, int64_t *flow_out,
                 uint8_t *cut_out) {
    cudaEvent_t t0, t1;
    FM_CHECK_CUDA(cudaEventCreate(&t0));
    FM_CHECK_CUDA(cudaEventCreate(&t1));
    cudaEventRecord(t0, g->stream);
    int rc = begin_device(g, capR, capL, capD, capU, capS, capT, flags);
    while (rc == FM_OK && g->active > 0) rc = run_round(g, cycle_budget, bfs_interval);
    if (rc == FM_OK && !(flags & FM_GRID_NO_CUT)) rc = compute_cut(g, cut_out);
    long long flow = 0;
    if (rc == FM_OK) rc = current_flow(g, &flow);
    cudaEventRecord(t1, g->stream);
    cudaEventSynchronize(t1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    g->st.ms_total = ms;
    if (g->trace >= 2) {   // FM_PL_TIMING builds: per-visit cycle split of the push kernel
        unsigned long long h[8] = {};
        cudaMemcpy(h, g->acc + 16, sizeof(h), cudaMemcpyDeviceToHost);
        const double v = h[3] ? (double)h[3] : 1.0;
        fprintf(stderr, "[fm_grid] visits %llu (solo %llu) cycles/visit: load %.0f passes %.0f (solo part %.0f) store %.0f"
                " | passes/visit dense %.2f solo %.2f\n",
                h[3], h[4], h[0] / v, h[1] / v, h[5] / v, h[2] / v, h[6] / v, h[7] / v);
    }
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    if (rc == FM_OK && flow_out) *flow_out = flow;
    return rc;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" int fm_grid_create(int32_t H, int32_t W, int32_t device, fm_grid **out) {
    if (!out || H < 1 || W < 1 || (int64_t)H * W > (int64_t)INT32_MAX / 2 - 4) {
        fm_set_error("fm_grid_create: invalid shape %d x %d", H, W);
        return FM_INVALID_ARG;
    }
    int ndev = fm_device_count();
    if (ndev == 0) { fm_set_error("no CUDA device"); return FM_NO_DEVICE; }
    if (device < 0 || device >= ndev) { fm_set_error("device %d out of range", device); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(device));
    fm_grid *g = new fm_grid();
    g->H = H; g->W = W; g->device = device; g->HW = (int64_t)H * W;
    g->d.ntx = (W + PT_W - 1) / PT_W;
    g->d.nty = (H + PT_H - 1) / PT_H;
    g->ntiles = g->d.ntx * g->d.nty;
    g->rq.incr = 1;
    g->d.solo_max = 32;
    g->d.k_solo = 0;
    g->rq.rerun = 0; g->rq.ns0 = 128; g->rq.ns1 = 2048;
    const size_t n4 = sizeof(int32_t) * (size_t)g->HW, n1 = (size_t)g->HW;
    int32_t **planes[] = {&g->d.e, &g->d.h, &g->d.rR, &g->d.rL, &g->d.rD, &g->d.rU,
                          &g->d.rT, &g->d.rS, &g->d.cS, &g->d.dist, &g->d.inflow_h, &g->d.inflow_v};
    for (auto pp : planes) {
        if (cudaMalloc((void **)pp, n4) != cudaSuccess) {
            fm_set_error("cudaMalloc of %zu bytes failed", n4);
            fm_grid_destroy(g);
            return FM_CUDA_ERROR;
        }
    }
    if (cudaMalloc((void **)&g->d.mask, n1) != cudaSuccess ||
        cudaMalloc((void **)&g->d.rbits, sizeof(uint32_t) * 160 * (size_t)g->ntiles) != cudaSuccess ||
        cudaMalloc((void **)&g->rq.flag, sizeof(int32_t) * (size_t)g->ntiles) != cudaSuccess ||
        cudaMalloc((void **)&g->rq.ctr, sizeof(unsigned int) * 256) != cudaSuccess ||
        cudaMalloc((void **)&g->prq.flag, sizeof(int32_t) * (size_t)g->ntiles) != cudaSuccess ||
        cudaMalloc((void **)&g->prq.ctr, sizeof(unsigned int) * 256) != cudaSuccess ||
        cudaMalloc((void **)&g->d.marked, n1) != cudaSuccess ||
        cudaMalloc((void **)&g->d.cut, n1) != cudaSuccess ||
        cudaMalloc((void **)&g->acc, sizeof(unsigned long long) * 32) != cudaSuccess ||
        cudaMalloc((void **)&g->d_queues, sizeof(int32_t) * (8 * (size_t)g->ntiles + 8)) != cudaSuccess ||
        cudaMalloc((void **)&g->d_touched, (size_t)g->ntiles) != cudaSuccess ||
        cudaMalloc((void **)&g->d_region, (size_t)g->ntiles) != cudaSuccess ||
        cudaMalloc((void **)&g->d_rlist, sizeof(int32_t) * ((size_t)g->ntiles + 1)) != cudaSuccess ||
        cudaMalloc((void **)&g->flags, sizeof(int32_t) * 64) != cudaSuccess ||
        cudaMalloc((void **)&g->d.ext, sizeof(int32_t) * 2 * (size_t)g->d.ntx) != cudaSuccess ||
        cudaMemset(g->d.ext, 0, sizeof(int32_t) * 2 * (size_t)g->d.ntx) != cudaSuccess ||
        cudaMallocHost((void **)&g->h_acc, sizeof(unsigned long long) * 32) != cudaSuccess ||
        cudaMallocHost((void **)&g->h_flags, sizeof(int32_t) * 64) != cudaSuccess ||
        cudaStreamCreateWithFlags(&g->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        fm_set_error("fm_grid_create: allocation failed: %s", cudaGetErrorString(cudaGetLastError()));
        fm_grid_destroy(g);
        return FM_CUDA_ERROR;
    }
    for (auto &e : g->ev) cudaEventCreate(&e);
    {
        TileQueue *qs[2] = {&g->d.pq, &g->d.bq};
        int32_t *base = g->d_queues;
        for (int k = 0; k < 2; k++) {
            // [list0 | list1 | flag0 | flag1] per queue, then 4 counters per queue
            qs[k]->list[0] = base + (size_t)(4 * k + 0) * g->ntiles;
            qs[k]->list[1] = base + (size_t)(4 * k + 1) * g->ntiles;
            qs[k]->flag[0] = base + (size_t)(4 * k + 2) * g->ntiles;
            qs[k]->flag[1] = base + (size_t)(4 * k + 3) * g->ntiles;
            qs[k]->cnt = base + (size_t)8 * g->ntiles + 4 * k;
        }
    }
    g->stream = g->own_stream;
    g->d.touched = g->d_touched;
    g->d.region = nullptr;
    g->d.H = H; g->d.W = W;
    g->d.hlim = H; g->d.rmin = 0;
    g->d.ext_ctr = g->acc + 24;
    g->rq.pend = g->rq.ctr + 64;
    g->prq.pend = g->prq.ctr + 64;
    g->d.V = (int32_t)(g->HW + 2);
    g->d.INF = g->d.V;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    g->sms = sms;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g->pt_per_sm, pr_tile_kernel, PT_W * PT_TY, 0);
    g->pt_per_sm = std::max(1, g->pt_per_sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g->pl_per_sm, pr_list_kernel<false>, PT_W * PL_TY, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g->pk_per_sm, pr_list_kernel<true>, PT_W * PL_TY, 0);
    g->pk_per_sm = std::max(1, g->pk_per_sm);
    g->pl_per_sm = std::max(1, g->pl_per_sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g->bb_per_sm, bfs_bits_kernel, 32 * BB_WARPS, 0);
    g->bb_per_sm = std::max(1, g->bb_per_sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g->br_occ, ring_kernel<0>, 32 * BB_WARPS, 0);
    g->br_occ = std::max(1, g->br_occ);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g->bo_occ, owner_bfs_kernel, 32 * BB_WARPS, 0);
    g->bo_occ = std::max(1, g->bo_occ);
    g->br_per_sm = std::max(1, std::min(g->br_occ, g->br_cap));
    g->pl_occ = g->pl_per_sm; g->pk_occ = g->pk_per_sm;
    // ring capacity: every tile once + one reserved slot per warp that can be resident
    // (fixed at the occupancy maximum: neighbour bands index this ring with it)
    g->rq.cap = g->ntiles + g->sms * g->br_occ * BB_WARPS + 64;
    g->prq.cap = g->ntiles + g->sms * g->pl_per_sm + 64;
    g->prq.rerun = 0; g->prq.ns0 = g->rq.ns0; g->prq.ns1 = g->rq.ns1;
    if (cudaMalloc((void **)&g->rq.slot, sizeof(int32_t) * (size_t)g->rq.cap) != cudaSuccess ||
        cudaMalloc((void **)&g->prq.slot, sizeof(int32_t) * (size_t)g->prq.cap) != cudaSuccess ||
        cudaMemset(g->rq.flag, 0, sizeof(int32_t) * (size_t)g->ntiles) != cudaSuccess) {
        fm_set_error("fm_grid_create: allocation failed");
        fm_grid_destroy(g);
        return FM_CUDA_ERROR;
    }
    g->grid_blocks = (int)std::min<int64_t>((g->HW + 255) / 256, (int64_t)sms * 8);
    encode_maps(g);
    *out = g;
    return FM_OK;
}

extern "C" void fm_grid_destroy(fm_grid *g) {
    if (!g) return;
    cudaSetDevice(g->device);
    int32_t *planes[] = {g->d.e, g->d.h, g->d.rR, g->d.rL, g->d.rD, g->d.rU,
                         g->d.rT, g->d.rS, g->d.cS, g->d.dist, g->d.inflow_h, g->d.inflow_v,
                         g->d_queues, g->in_caps};
    for (auto p : planes) if (p) cudaFree(p);
    if (g->d.mask) cudaFree(g->d.mask);
    if (g->d.rbits) cudaFree(g->d.rbits);
    if (g->rq.slot) cudaFree(g->rq.slot);
    if (g->rq.flag) cudaFree(g->rq.flag);
    if (g->rq.ctr) cudaFree(g->rq.ctr);
    if (g->prq.slot) cudaFree(g->prq.slot);
    if (g->prq.flag) cudaFree(g->prq.flag);
    if (g->prq.ctr) cudaFree(g->prq.ctr);
    if (g->d.marked) cudaFree(g->d.marked);
    if (g->d.cut) cudaFree(g->d.cut);
    if (g->d.ext) cudaFree(g->d.ext);
    if (g->band_caps) cudaFree(g->band_caps);
    for (auto &side : g->ipc_open)
        for (auto &p : side) if (p) { cudaIpcCloseMemHandle(p); p = nullptr; }
    if (g->ipc_gpend) cudaIpcCloseMemHandle(g->ipc_gpend);
    if (g->d_touched) cudaFree(g->d_touched);
    if (g->d_region) cudaFree(g->d_region);
    if (g->d_rlist) cudaFree(g->d_rlist);
    if (g->acc) cudaFree(g->acc);
    if (g->flags) cudaFree(g->flags);
    if (g->h_acc) cudaFreeHost(g->h_acc);
    if (g->h_flags) cudaFreeHost(g->h_flags);
    if (g->h_cut_stage) cudaFreeHost(g->h_cut_stage);
    if (g->in_caps2) cudaFree(g->in_caps2);
    for (int k = 0; k < 2; k++) {
        if (g->b_narrow[k]) cudaFree(g->b_narrow[k]);
        if (g->b_dcut[k]) cudaFree(g->b_dcut[k]);
        if (g->b_hcut[k]) cudaFreeHost(g->b_hcut[k]);
    }
    if (g->h2d_stream) cudaStreamDestroy(g->h2d_stream);
    if (g->d2h_stream) cudaStreamDestroy(g->d2h_stream);
    if (g->prg_exec) cudaGraphExecDestroy(g->prg_exec);
    if (g->prg) cudaGraphDestroy(g->prg);
    for (auto e : g->ev) if (e) cudaEventDestroy(e);
    if (g->own_stream) cudaStreamDestroy(g->own_stream);
    delete g;
}

extern "C" int fm_grid_solve(fm_grid *g, const int32_t *capR, const int32_t *capL,
                             const int32_t *capD, const int32_t *capU, const int32_t *capS,
                             const int32_t *capT, int32_t cycle_budget, int32_t bfs_interval,
                             int32_t flags, int64_t *flow_out, uint8_t *cut_out,
                             fm_stats *stats, void *stream) {
    if (!g || !capR || !capL || !capD || !capU || !capS || !capT || cycle_budget < 1) {
        fm_set_error("fm_grid_solve: invalid argument");
        return FM_INVALID_ARG;
    }
    FM_CHECK_CUDA(cudaSetDevice(g->device));
    set_stream(g, stream);
    int rc = solve_device(g, capR, capL, capD, capU, capS, capT, cycle_budget, bfs_interval,
                          flags, flow_out, cut_out);
    if (stats) *stats = g->st;
    return rc;
}

namespace {
int stage_host_caps(fm_grid *g, const int32_t *capR, const int32_t *capL, const int32_t *capD,
                    const int32_t *capU, const int32_t *capS, const int32_t *capT) {
    if (!g->in_caps)
        FM_CHECK_CUDA(cudaMalloc((void **)&g->in_caps, sizeof(int32_t) * 6 * (size_t)g->HW));
    const int32_t *src[6] = {capR, capL, capD, capU, capS, capT};
    for (int k = 0; k < 6; k++)
        FM_CHECK_CUDA(cudaMemcpyAsync(g->in_caps + (size_t)k * g->HW, src[k],
                                      sizeof(int32_t) * (size_t)g->HW, cudaMemcpyHostToDevice,
                                      g->stream));
    return FM_OK;
}
}  // namespace

extern "C" int fm_grid_solve_host(fm_grid *g, const int32_t *capR, const int32_t *capL,
                                  const int32_t *capD, const int32_t *capU, const int32_t *capS,
                                  const int32_t *capT, int32_t cycle_budget, int32_t bfs_interval,
                                  int32_t flags, int64_t *flow_out, uint8_t *cut_out,
                                  fm_stats *stats) {
    if (!g || !capR || !capL || !capD || !capU || !capS || !capT || cycle_budget < 1) {
        fm_set_error("fm_grid_solve_host: invalid argument");
        return FM_INVALID_ARG;
    }
    FM_CHECK_CUDA(cudaSetDevice(g->device));
    set_stream(g, nullptr);
    // The caller's cut array is usually fresh (its pages not yet faulted in): touch
    // them on a host thread while the device solves, so the final copy into it runs at
    // memory speed instead of page-fault speed.
    std::thread prefault;
    if (cut_out && !(flags & FM_GRID_NO_CUT)) {
        const size_t n = (size_t)g->HW;
        prefault = std::thread([cut_out, n] {
            for (size_t i = 0; i < n; i += 4096) ((volatile uint8_t *)cut_out)[i] = 0;
        });
    }
    struct Joiner {
        std::thread &t;
        ~Joiner() { if (t.joinable()) t.join(); }
    } joiner{prefault};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, g->stream);
    FM_TRY(stage_host_caps(g, capR, capL, capD, capU, capS, capT));
    cudaEventRecord(b, g->stream);
    cudaEventSynchronize(b);
    float h2d = 0.f;
    cudaEventElapsedTime(&h2d, a, b);
    const int32_t *c = g->in_caps;
    const size_t HW = (size_t)g->HW;
    int rc = solve_device(g, c, c + HW, c + 2 * HW, c + 3 * HW, c + 4 * HW, c + 5 * HW,
                          cycle_budget, bfs_interval, flags, flow_out, nullptr);
    float d2h = 0.f;
    if (rc == FM_OK && cut_out && !(flags & FM_GRID_NO_CUT)) {
        // D2H through a pinned bounce buffer (pageable D2H runs at a few GB/s), then one
        // host memcpy into the caller's array
        cudaEventRecord(a, g->stream);
        if (!g->h_cut_stage && cudaMallocHost((void **)&g->h_cut_stage, HW) != cudaSuccess) g->h_cut_stage = nullptr;
        uint8_t *dst = g->h_cut_stage ? g->h_cut_stage : cut_out;
        // no bounce buffer: the D2H writes the caller's array directly, so the
        // prefault thread (writing zeros into it) must be done first
        if (dst == cut_out && prefault.joinable()) prefault.join();
        // chunked: the host copy of chunk k overlaps the D2H of chunk k+1
        constexpr int NCH = 4;
        cudaEvent_t ce[NCH];
        const size_t per = (HW + NCH - 1) / NCH;
        for (int k = 0; k < NCH; k++) {
            cudaEventCreateWithFlags(&ce[k], cudaEventDisableTiming);
            const size_t lo = std::min(HW, k * per), hi = std::min(HW, lo + per);
            if (hi > lo && cudaMemcpyAsync(dst + lo, g->d.cut + lo, hi - lo, cudaMemcpyDeviceToHost, g->stream) != cudaSuccess)
                rc = FM_CUDA_ERROR;
            cudaEventRecord(ce[k], g->stream);
        }
        if (prefault.joinable()) prefault.join();
        if (rc == FM_OK && dst != cut_out) {
            // NT host threads, each copying its slice of every chunk as that chunk lands
            const int NT = HW >= ((size_t)4 << 20) ? 8 : 1;
            const int dev = g->device;
            auto work = [&, dev](int j) {
                if (NT > 1) cudaSetDevice(dev);
                for (int k = 0; k < NCH; k++) {
                    cudaEventSynchronize(ce[k]);
                    const size_t lo = std::min(HW, k * per), hi = std::min(HW, lo + per);
                    const size_t sl = (hi - lo + NT - 1) / NT;
                    const size_t a0 = std::min(hi, lo + j * sl), a1 = std::min(hi, a0 + sl);
                    if (a1 > a0) memcpy(cut_out + a0, dst + a0, a1 - a0);
                }
            };
            std::vector<std::thread> th;
            for (int j = 1; j < NT; j++) th.emplace_back(work, j);
            work(0);
            for (auto &t : th) t.join();
        }
        for (int k = 0; k < NCH; k++) cudaEventSynchronize(ce[k]), cudaEventDestroy(ce[k]);
        cudaEventRecord(b, g->stream);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&d2h, a, b);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    g->st.ms_h2d = h2d;
    g->st.ms_d2h = d2h;
    if (stats) *stats = g->st;
    return rc;
}

// A batch of independent same-shape instances from HOST planes, pipelined: the H2D of
// instance k+1 (copy stream, second input set) and the D2H of instance k-1's cut (a
// second copy stream through pinned stages, then host threads into the caller's
// arrays) run while instance k solves, so a stream of images costs
// max(solve, PCIe) per image instead of their sum.  Every instance's copies are still
// made (nothing cached across instances); results are those of fm_grid_solve_host.
extern "C" int fm_grid_solve_host_batch(fm_grid *g, int32_t count, const void *const *caps, int32_t elem_bytes,
                                        int32_t cycle_budget, int32_t bfs_interval, int32_t flags,
                                        int64_t *flows_out, uint8_t *const *cuts_out, fm_stats *stats) {
    if (!g || count < 0 || (count > 0 && (!caps || !flows_out)) || cycle_budget < 1 ||
        (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4)) {
        fm_set_error("fm_grid_solve_host_batch: invalid argument");
        return FM_INVALID_ARG;
    }
    for (int k = 0; k < 6 * count; k++)
        if (!caps[k]) { fm_set_error("fm_grid_solve_host_batch: capacity plane %d of instance %d is NULL", k % 6, k / 6);
                        return FM_INVALID_ARG; }
    if (count == 0) return FM_OK;
    FM_CHECK_CUDA(cudaSetDevice(g->device));
    set_stream(g, nullptr);
    const size_t HW = (size_t)g->HW;
    const bool want_cut = cuts_out && !(flags & FM_GRID_NO_CUT);
    if (!g->in_caps) FM_CHECK_CUDA(cudaMalloc((void **)&g->in_caps, sizeof(int32_t) * 6 * HW));
    if (count > 1 && !g->in_caps2) FM_CHECK_CUDA(cudaMalloc((void **)&g->in_caps2, sizeof(int32_t) * 6 * HW));
    const size_t nbytes = (size_t)elem_bytes * 6 * HW;
    if (elem_bytes < 4 && g->b_narrow_bytes < nbytes) {
        for (int b = 0; b < 2; b++) {
            if (g->b_narrow[b]) cudaFree(g->b_narrow[b]);
            g->b_narrow[b] = nullptr;
        }
        g->b_narrow_bytes = 0;
        for (int b = 0; b < 2; b++) FM_CHECK_CUDA(cudaMalloc((void **)&g->b_narrow[b], nbytes));
        g->b_narrow_bytes = nbytes;
    }
    if (!g->h2d_stream) FM_CHECK_CUDA(cudaStreamCreateWithFlags(&g->h2d_stream, cudaStreamNonBlocking));
    if (!g->d2h_stream) FM_CHECK_CUDA(cudaStreamCreateWithFlags(&g->d2h_stream, cudaStreamNonBlocking));
    if (want_cut)
        for (int b = 0; b < 2; b++) {
            if (!g->b_dcut[b]) FM_CHECK_CUDA(cudaMalloc((void **)&g->b_dcut[b], HW));
            if (!g->b_hcut[b]) FM_CHECK_CUDA(cudaMallocHost((void **)&g->b_hcut[b], HW));
        }
    int32_t *inbuf[2] = {g->in_caps, g->in_caps2};
    std::vector<cudaEvent_t> evs;
    const auto mkev = [&]() {
        cudaEvent_t e = nullptr;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        evs.push_back(e);
        return e;
    };
    // H2D of instance k into input set k % 2 (the set of instance k-2, whose solve the
    // host has already waited for); narrow planes land in the staging set k % 2
    const auto h2d = [&](int k) -> cudaEvent_t {
        uint8_t *dst = elem_bytes == 4 ? reinterpret_cast<uint8_t *>(inbuf[k & 1]) : g->b_narrow[k & 1];
        const size_t pb = (size_t)elem_bytes * HW;
        for (int p = 0; p < 6; p++)
            if (cudaMemcpyAsync(dst + p * pb, caps[6 * k + p], pb, cudaMemcpyHostToDevice, g->h2d_stream) != cudaSuccess)
                return nullptr;
        cudaEvent_t e = mkev();
        cudaEventRecord(e, g->h2d_stream);
        return e;
    };
    // host copy-out of a cut: NT threads, each a slice, after the D2H event
    std::thread copier[2];
    const auto copy_out = [](uint8_t *dst, const uint8_t *src, size_t n, cudaEvent_t done, int dev) {
        cudaSetDevice(dev);
        cudaEventSynchronize(done);
        const int NT = n >= ((size_t)4 << 20) ? 4 : 1;
        const size_t sl = (n + NT - 1) / NT;
        std::vector<std::thread> th;
        for (int j = 1; j < NT; j++)
            th.emplace_back([=] { const size_t a = std::min(n, j * sl), b = std::min(n, a + sl); memcpy(dst + a, src + a, b - a); });
        memcpy(dst, src, std::min(n, sl));
        for (auto &t : th) t.join();
    };
    // the caller's cut arrays are usually fresh: one host thread touches their pages in
    // order while the solves run (copy-out k waits until array k is done), so each
    // copy-out runs at memory speed instead of page-fault speed
    std::atomic<int> faulted{0};
    std::atomic<bool> stop_fault{false};
    std::thread prefault;
    if (want_cut)
        prefault = std::thread([&] {
            for (int k = 0; k < count && !stop_fault.load(std::memory_order_relaxed); k++) {
                if (cuts_out[k])
                    for (size_t i = 0; i < HW; i += 4096) ((volatile uint8_t *)cuts_out[k])[i] = 0;
                faulted.store(k + 1, std::memory_order_release);
            }
        });
    struct Cleanup {
        std::thread *c;
        std::vector<cudaEvent_t> &e;
        std::thread &pf;
        std::atomic<bool> &stop;
        ~Cleanup() {
            stop.store(true);
            if (pf.joinable()) pf.join();
            for (int b = 0; b < 2; b++) if (c[b].joinable()) c[b].join();
            for (auto x : e) cudaEventDestroy(x);
        }
    } cleanup{copier, evs, prefault, stop_fault};
    int rc = FM_OK;
    cudaEvent_t ready = h2d(0);
    if (!ready) { fm_set_error("fm_grid_solve_host_batch: H2D failed"); return FM_CUDA_ERROR; }
    for (int k = 0; k < count && rc == FM_OK; k++) {
        cudaEvent_t next = nullptr;
        if (k + 1 < count && !(next = h2d(k + 1))) { fm_set_error("fm_grid_solve_host_batch: H2D failed"); rc = FM_CUDA_ERROR; break; }
        FM_CHECK_CUDA(cudaStreamWaitEvent(g->stream, ready, 0));
        cudaEvent_t tw0 = nullptr, tw1 = nullptr;
        const auto t_host0 = std::chrono::steady_clock::now();
        if (g->trace) {
            cudaEventCreate(&tw0); cudaEventCreate(&tw1); evs.push_back(tw0); evs.push_back(tw1);
            cudaEventRecord(tw0, g->stream);
        }
        if (elem_bytes < 4) {
            const int blocks = g->sms * 8;
            if (elem_bytes == 1)
                widen_planes_kernel<uint8_t><<<blocks, 256, 0, g->stream>>>(g->b_narrow[k & 1], inbuf[k & 1], (int64_t)(6 * HW));
            else
                widen_planes_kernel<uint16_t><<<blocks, 256, 0, g->stream>>>(
                    reinterpret_cast<const uint16_t *>(g->b_narrow[k & 1]), inbuf[k & 1], (int64_t)(6 * HW));
            FM_CHECK_LAUNCH();
        }
        if (g->trace) cudaEventRecord(tw1, g->stream);
        const int32_t *c = inbuf[k & 1];
        int64_t flow = 0;
        rc = solve_device(g, c, c + HW, c + 2 * HW, c + 3 * HW, c + 4 * HW, c + 5 * HW, cycle_budget, bfs_interval,
                          flags, &flow, nullptr);
        if (rc != FM_OK) break;
        flows_out[k] = flow;
        if (stats) stats[k] = g->st;
        if (g->trace) {
            float wms = 0.f;
            cudaEventElapsedTime(&wms, tw0, tw1);
            const double host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
            fprintf(stderr, "[fm_grid] batch step %d: wait + widen %.3f ms, solve %.3f ms (device), step host %.3f ms\n", k, wms,
                    g->st.ms_total, host_ms);
        }
        if (want_cut && cuts_out[k]) {
            const int b = k & 1;
            if (copier[b].joinable()) copier[b].join();   // stage b is free again
            // the next solve overwrites d.cut: move it aside on the solve stream, then
            // D2H from there on the copy stream
            FM_CHECK_CUDA(cudaMemcpyAsync(g->b_dcut[b], g->d.cut, HW, cudaMemcpyDeviceToDevice, g->stream));
            cudaEvent_t moved = mkev();
            cudaEventRecord(moved, g->stream);
            FM_CHECK_CUDA(cudaStreamWaitEvent(g->d2h_stream, moved, 0));
            FM_CHECK_CUDA(cudaMemcpyAsync(g->b_hcut[b], g->b_dcut[b], HW, cudaMemcpyDeviceToHost, g->d2h_stream));
            cudaEvent_t landed = mkev();
            cudaEventRecord(landed, g->d2h_stream);
            while (faulted.load(std::memory_order_acquire) <= k) std::this_thread::yield();   // array k touched
            copier[b] = std::thread(copy_out, cuts_out[k], g->b_hcut[b], HW, landed, g->device);
        }
        ready = next;
    }
    for (int b = 0; b < 2; b++) if (copier[b].joinable()) copier[b].join();
    if (rc == FM_OK) {
        if (cudaStreamSynchronize(g->d2h_stream) != cudaSuccess || cudaStreamSynchronize(g->h2d_stream) != cudaSuccess) {
            fm_set_error("fm_grid_solve_host_batch: copy stream failed: %s", cudaGetErrorString(cudaGetLastError()));
            rc = FM_CUDA_ERROR;
        }
    } else {
        cudaStreamSynchronize(g->h2d_stream);   // no copy may still target a buffer the caller frees
        cudaStreamSynchronize(g->d2h_stream);
    }
    return rc;
}

extern "C" int fm_grid_begin(fm_grid *g, const int32_t *capR, const int32_t *capL,
                             const int32_t *capD, const int32_t *capU, const int32_t *capS,
                             const int32_t *capT, int32_t flags) {
    if (!g || !capR || !capL || !capD || !capU || !capS || !capT) {
        fm_set_error("fm_grid_begin: invalid argument");
        return FM_INVALID_ARG;
    }
    FM_CHECK_CUDA(cudaSetDevice(g->device));
    set_stream(g, nullptr);
    FM_TRY(stage_host_caps(g, capR, capL, capD, capU, capS, capT));
    const int32_t *c = g->in_caps;
    const size_t HW = (size_t)g->HW;
    return begin_device(g, c, c + HW, c + 2 * HW, c + 3 * HW, c + 4 * HW, c + 5 * HW, flags);
}

extern "C" int fm_grid_round(fm_grid *g, int32_t cycle_budget, int32_t bfs_interval,
                             int32_t *done, fm_stats *stats) {
    if (!g || cycle_budget < 1) { fm_set_error("fm_grid_round: invalid argument"); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(g->device));
    int rc = FM_OK;
    if (g->active > 0) rc = run_round(g, cycle_budget, bfs_interval);
    if (done) *done = g->active == 0;
    if (stats) *stats = g->st;
    return rc;
}

extern "C" int fm_grid_export(fm_grid *g, int32_t *rR, int32_t *rL, int32_t *rD, int32_t *rU,
                              int32_t *rT, int32_t *rS, int32_t *e, int32_t *h, uint8_t *marked,
                              int64_t *flow, int64_t *excess_total) {
    if (!g) { fm_set_error("fm_grid_export: null handle"); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(g->device));
    const size_t n4 = sizeof(int32_t) * (size_t)g->HW;
    struct { int32_t *dst; const int32_t *src; } cp[] = {
        {rR, g->d.rR}, {rL, g->d.rL}, {rD, g->d.rD}, {rU, g->d.rU},
        {rT, g->d.rT}, {rS, g->d.rS}, {e, g->d.e}, {h, g->d.h}};
    for (auto &x : cp)
        if (x.dst) FM_CHECK_CUDA(cudaMemcpyAsync(x.dst, x.src, n4, cudaMemcpyDeviceToHost, g->stream));
    if (marked) FM_CHECK_CUDA(cudaMemcpyAsync(marked, g->d.marked, (size_t)g->HW, cudaMemcpyDeviceToHost, g->stream));
    FM_TRY(sync_stream(g));
    if (flow) {
        long long f = 0;
        FM_TRY(current_flow(g, &f));
        *flow = f;
    }
    if (excess_total) *excess_total = g->excess_total;
    return FM_OK;
}

extern "C" int fm_grid_cut_host(fm_grid *g, uint8_t *cut_out, fm_stats *stats) {
    if (!g || !cut_out) { fm_set_error("fm_grid_cut_host: invalid argument"); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(g->device));
    FM_TRY(compute_cut(g, nullptr));
    FM_CHECK_CUDA(cudaMemcpyAsync(cut_out, g->d.cut, (size_t)g->HW, cudaMemcpyDeviceToHost, g->stream));
    FM_TRY(sync_stream(g));
    if (stats) *stats = g->st;
    return FM_OK;
}

extern "C" int fm_grid_stats(fm_grid *g, fm_stats *stats) {
    if (!g || !stats) { fm_set_error("fm_grid_stats: invalid argument"); return FM_INVALID_ARG; }
    *stats = g->st;
    return FM_OK;
}

// copy the current cut plane (no recompute) to dst (host when dst_on_host, else device)
extern "C" int fm_grid_cut_plane(fm_grid *g, uint8_t *dst, int32_t dst_on_host) {
    if (!g || !dst) { fm_set_error("fm_grid_cut_plane: invalid argument"); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(g->device));
    FM_CHECK_CUDA(cudaMemcpyAsync(dst, g->d.cut, (size_t)g->HW,
                                  dst_on_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, g->stream));
    FM_TRY(sync_stream(g));
    return FM_OK;
}

// A/B and tuning options (replace the round-1 environment knobs; a library never
// reads the caller's environment).  Take effect at the next solve.  Names are the
// DESIGN.md section 4 switch names in lower case.
extern "C" int fm_grid_set_option(fm_grid *g, const char *name, int64_t value) {
    if (!g || !name) { fm_set_error("fm_grid_set_option: invalid argument"); return FM_INVALID_ARG; }
    const int v = (int)std::max<int64_t>(INT32_MIN, std::min<int64_t>(INT32_MAX, value));
    const std::string k(name);
    if (k == "k_local") g->k_local = v;
    else if (k == "bfs_interval") g->bfs_interval_env = v;
    else if (k == "trace") g->trace = v;
    else if (k == "relabel_div") g->relabel_div = v;
    else if (k == "op_steps") g->op_steps = std::max(1, v);
    else if (k == "op_fused") g->op_fused = v;
    else if (k == "vote") g->vote_mask = std::max(1, v) - 1;
    else if (k == "pr_kernel") g->pr_kernel = v;
    else if (k == "bfs_bits") g->bfs_bits = v;
    else if (k == "bfs_owner") g->bfs_owner = v;
    else if (k == "br_cap") { g->br_cap = std::max(1, v); g->br_per_sm = std::max(1, std::min(g->br_occ, g->br_cap)); }
    else if (k == "pr_ring") g->pr_ring = v;
    else if (k == "pr_graph") g->pr_graph = v;
    else if (k == "tma") g->tma = v;
    else if (k == "packed") g->pk = v;
    else if (k == "bfs_incr") g->rq.incr = v ? 1 : 0;
    else if (k == "k_solo") g->d.k_solo = v;
    else if (k == "solo_max") g->d.solo_max = v;
    else if (k == "k_tail") g->k_tail = v;
    else if (k == "ring_tail") g->ring_tail = std::max(-1, v);
    else if (k == "two_hop") g->two_hop = v;
    else if (k == "tail_div") g->tail_div = v;
    else if (k == "pr_batch") g->pr_batch = std::max(0, std::min(16, v));
    else if (k == "visit_mult") g->visit_mult = std::max(1, v);
    else if (k == "br_rerun") g->rq.rerun = v;
    else if (k == "br_ns0") g->rq.ns0 = v;
    else if (k == "br_ns1") g->rq.ns1 = v;
    else if (k == "k_local_list") g->k_local_list = v;
    else if (k == "local_div") g->local_div = v;
    else if (k == "local_max") g->local_max = v;
    else if (k == "local_margin") g->local_margin = v;
    else if (k == "pk_occ") g->pk_per_sm = std::max(1, std::min(g->pk_occ, v));
    else if (k == "pl_per_sm") g->pl_per_sm = std::max(1, std::min(g->pl_occ, v));
    else { fm_set_error("fm_grid_set_option: unknown option '%s'", name); return FM_INVALID_ARG; }
    return FM_OK;
}

// ============================================================================
// Row bands (multi-GPU grid path; reference coordinator loop
// maxflow_par.py:195-229).  Band k of N holds rows [R0_k, R1_k) of the grid (band
// borders on 32-row tile boundaries).  Nothing is exchanged by messages: a band's
// kernels read the neighbour bands' boundary rows (heights for pushes, distances for
// the global relabel, cut bits for the min-cut reach) straight from their memory, push
// flow into their inboxes with remote atomics, raise their external-push flags, and
// queue their ring-BFS tiles; the bands' persistent ring launches end together on one
// shared pending counter.  The only host-level agreement is a few int64 per push batch
// / relabel, gathered through an fm_coll (a shared-memory barrier: threads of one
// process, or processes of one node).
// ============================================================================
#include <atomic>
#include <chrono>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

namespace {
constexpr int COLL_MAX_RANKS = 64, COLL_MAX_VALS = 8;
constexpr uint32_t COLL_MAGIC = 0x666d636cu;
struct CollShm {
    std::atomic<uint64_t> arrive;
    uint32_t magic, nranks;
    int64_t slot[2][COLL_MAX_RANKS][COLL_MAX_VALS];
};
static_assert(std::atomic<uint64_t>::is_always_lock_free, "cross-process atomics need lock-free 64-bit");
}  // namespace

struct fm_coll {
    CollShm *shm = nullptr;
    size_t bytes = 0;
    bool mapped = false;       // shm_open mapping (else heap, process-local)
    bool owner = false;
    std::string name;
    int32_t rank = 0, nranks = 1;
    uint64_t calls = 0;
};

extern "C" int fm_coll_create(const char *name, int32_t nranks, int32_t rank, fm_coll **out) {
    if (!out || nranks < 1 || nranks > COLL_MAX_RANKS || rank < 0 || rank >= nranks) {
        fm_set_error("fm_coll_create: invalid argument (1 <= nranks <= %d)", COLL_MAX_RANKS);
        return FM_INVALID_ARG;
    }
    fm_coll *c = new fm_coll();
    c->rank = rank; c->nranks = nranks; c->bytes = sizeof(CollShm);
    if (!name || !*name) {
        c->shm = new CollShm();
        c->shm->arrive.store(0);
        c->shm->magic = COLL_MAGIC;
        c->shm->nranks = (uint32_t)nranks;
    } else {
        // rank 0 creates and initialises the segment; the others open it after the
        // caller's own barrier (paper_1110_6231_b200.bands does a torch.distributed one)
        c->name = name;
        c->owner = rank == 0;
        const int fd = shm_open(name, c->owner ? (O_CREAT | O_RDWR | O_TRUNC) : O_RDWR, 0600);
        if (fd < 0) { fm_set_error("fm_coll_create: shm_open(%s) failed", name); delete c; return FM_INVALID_ARG; }
        if (c->owner && ftruncate(fd, (off_t)c->bytes) != 0) {
            close(fd); fm_set_error("fm_coll_create: ftruncate failed"); delete c; return FM_INVALID_ARG;
        }
        void *p = mmap(nullptr, c->bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (p == MAP_FAILED) { fm_set_error("fm_coll_create: mmap failed"); delete c; return FM_INVALID_ARG; }
        c->shm = (CollShm *)p;
        c->mapped = true;
        if (c->owner) {
            new (&c->shm->arrive) std::atomic<uint64_t>(0);
            c->shm->nranks = (uint32_t)nranks;
            std::atomic_thread_fence(std::memory_order_release);
            c->shm->magic = COLL_MAGIC;
        }
    }
    *out = c;
    return FM_OK;
}

extern "C" void fm_coll_destroy(fm_coll *c) {
    if (!c) return;
    if (c->mapped) {
        munmap(c->shm, c->bytes);
        if (c->owner) shm_unlink(c->name.c_str());
    } else {
        delete c->shm;
    }
    delete c;
}

// Every rank contributes n int64 and receives all ranks' values (out[rank * n + i]).
// Call k uses slot set k & 1: a rank can only start call k + 2 (which rewrites set
// k & 1) after every rank arrived at call k + 1, i.e. finished reading call k.
extern "C" int fm_coll_allgather(fm_coll *c, const int64_t *vals, int32_t n, int64_t *out) {
    if (!c || n < 0 || n > COLL_MAX_VALS || (n && (!vals || !out))) {
        fm_set_error("fm_coll_allgather: invalid argument (n <= %d)", COLL_MAX_VALS);
        return FM_INVALID_ARG;
    }
    CollShm *s = c->shm;
    if (s->magic != COLL_MAGIC || (int32_t)s->nranks != c->nranks) {
        fm_set_error("fm_coll_allgather: collective segment not initialised");
        return FM_INVALID_ARG;
    }
    const uint64_t k = c->calls++;
    int64_t *mine = s->slot[k & 1][c->rank];
    for (int i = 0; i < n; i++) mine[i] = vals[i];
    s->arrive.fetch_add(1, std::memory_order_acq_rel);
    const uint64_t target = (uint64_t)c->nranks * (k + 1);
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t spin = 0; s->arrive.load(std::memory_order_acquire) < target; spin++) {
        if (spin < 4096) continue;
        if ((spin & 1023) == 0 &&
            std::chrono::steady_clock::now() - t0 > std::chrono::seconds(300)) {
            fm_set_error("fm_coll_allgather: rank %d waited 300 s for the other ranks", c->rank);
            return FM_CUDA_ERROR;
        }
        sched_yield();
    }
    for (int r = 0; r < c->nranks; r++)
        for (int i = 0; i < n; i++) out[r * n + i] = s->slot[k & 1][r][i];
    return FM_OK;
}

// Band borders on 32-row tile boundaries (the last band takes the remainder);
// edges[0..nbands], the same split as paper_1110_6231_b200.bands.band_rows.
extern "C" int fm_band_split(int32_t H, int32_t nbands, int32_t *edges) {
    if (!edges || nbands < 1 || H < 1) { fm_set_error("fm_band_split: invalid argument"); return FM_INVALID_ARG; }
    const int64_t tiles = (H + PT_H - 1) / PT_H;
    if (nbands > tiles) {
        fm_set_error("fm_band_split: %d rows hold %lld tile rows, fewer than %d bands", H, (long long)tiles, nbands);
        return FM_INVALID_ARG;
    }
    for (int k = 0; k <= nbands; k++)
        edges[k] = (int32_t)std::min<int64_t>(H, ((k * tiles + nbands / 2) / nbands) * PT_H);
    edges[nbands] = H;
    for (int k = 0; k < nbands; k++)
        if (edges[k + 1] <= edges[k]) { fm_set_error("fm_band_split: empty band"); return FM_INVALID_ARG; }
    return FM_OK;
}

extern "C" int fm_grid_band_setup(fm_grid *g, int32_t band, int32_t nbands, int32_t H_total,
                                  int32_t colocated) {
    if (!g || nbands < 1 || band < 0 || band >= nbands || H_total < g->H ||
        (int64_t)H_total * g->W > (int64_t)INT32_MAX / 2 - 4 || (band + 1 < nbands && g->H % PT_H) ||
        colocated < 1) {
        fm_set_error("fm_grid_band_setup: invalid argument (inner bands need a multiple of %d rows)", PT_H);
        return FM_INVALID_ARG;
    }
    g->band = band;
    g->nbands = nbands;
    g->H_total = H_total;
    g->colocated = colocated;
    g->total_tiles = (int64_t)((H_total + PT_H - 1) / PT_H) * g->d.ntx;
    // heights, the source height |V| and the BFS sentinel are the whole grid's
    g->d.V = (int32_t)((int64_t)H_total * g->W + 2);
    g->d.INF = g->d.V;
    g->d.has_up = band > 0;
    g->d.has_dn = band + 1 < nbands;
    g->d.hlim = g->H + g->d.has_dn;
    g->d.rmin = -g->d.has_up;
    g->rq.sys = nbands > 1;
    g->local_div = 0;   // region-limited relabels are single-band only
    if (band == 0) g->gpend = g->rq.ctr + 200;
    return FM_OK;
}

namespace {
// the buffers a neighbour band needs, in export order
constexpr int BAND_BUFS = 10;
struct BandExport {
    uint32_t magic;
    int32_t device, H, W, ntx, nty, rq_cap, pid;
    cudaIpcMemHandle_t h[BAND_BUFS];   // h, dist, inflow_v, rD, rU, cut, ext, rq.slot, rq.flag, rq.ctr
};
static_assert(sizeof(BandExport) <= 1024, "FM_BAND_EXPORT_BYTES");

void *band_buf(fm_grid *g, int k) {
    void *b[BAND_BUFS] = {g->d.h, g->d.dist, g->d.inflow_v, g->d.rD, g->d.rU, g->d.cut, g->d.ext,
                          g->rq.slot, g->rq.flag, g->rq.ctr};
    return b[k];
}

// PeerView of neighbour band `nb` (its buffers `buf`) seen from g; side 0 = above, 1 = below
PeerView make_peer(const fm_grid *g, int side, int nbH, int nbnty, int nb_rq_cap, void *const *buf) {
    PeerView v{};
    const int64_t row = side == 0 ? (int64_t)(nbH - 1) * g->W : 0;   // its boundary row
    v.h = (int32_t *)buf[0] + row;
    v.dist = (int32_t *)buf[1] + row;
    v.inbox = (int32_t *)buf[2] + row;
    v.res = side == 0 ? (int32_t *)buf[3] + row : (int32_t *)buf[4];   // its rD (above) / rU (below)
    v.cut = (uint8_t *)buf[5] + row;
    v.ext = (int32_t *)buf[6] + (side == 0 ? g->d.ntx : 0);            // its bottom / top tile row flags
    v.rq_slot = (int32_t *)buf[7];
    v.rq_flag = (int32_t *)buf[8];
    v.rq_ctr = (unsigned *)buf[9];
    v.rq_cap = nb_rq_cap;
    v.tile0 = side == 0 ? (nbnty - 1) * g->d.ntx : 0;
    return v;
}
}  // namespace

extern "C" int fm_grid_band_export(fm_grid *g, void *blob) {
    if (!g || !blob || g->band < 0) { fm_set_error("fm_grid_band_export: set the band up first"); return FM_INVALID_ARG; }
    FM_CHECK_CUDA(cudaSetDevice(g->device));
    BandExport x{};
    x.magic = COLL_MAGIC; x.device = g->device; x.H = g->H; x.W = g->W;
    x.ntx = g->d.ntx; x.nty = g->d.nty; x.rq_cap = g->rq.cap; x.pid = (int32_t)getpid();
    for (int k = 0; k < BAND_BUFS; k++) FM_CHECK_CUDA(cudaIpcGetMemHandle(&x.h[k], band_buf(g, k)));
    memset(blob, 0, FM_BAND_EXPORT_BYTES);
    memcpy(blob, &x, sizeof(x));
    return FM_OK;
}

// Neighbours exported by other processes (one process per GPU): open their buffers.
// up / dn may be NULL (first / last band); band0 is needed by every band but band 0.
extern "C" int fm_grid_band_link(fm_grid *g, const void *up_blob, const void *dn_blob, const void *band0_blob) {
    if (!g || g->band < 0 || (g->d.has_up && !up_blob) || (g->d.has_dn && !dn_blob) || (g->band > 0 && !band0_blob)) {
        fm_set_error("fm_grid_band_link: missing neighbour export");
        return FM_INVALID_ARG;
    }
    FM_CHECK_CUDA(cudaSetDevice(g->device));
    const void *blobs[2] = {g->d.has_up ? up_blob : nullptr, g->d.has_dn ? dn_blob : nullptr};
    for (int side = 0; side < 2; side++) {
        if (!blobs[side]) continue;
        BandExport x;
        memcpy(&x, blobs[side], sizeof(x));
        if (x.magic != COLL_MAGIC || x.W != g->W || x.ntx != g->d.ntx) {
            fm_set_error("fm_grid_band_link: neighbour export does not match this band (width %d vs %d)", x.W, g->W);
            return FM_INVALID_ARG;
        }
        for (int k = 0; k < BAND_BUFS; k++) {
            if (g->ipc_open[side][k]) { cudaIpcCloseMemHandle(g->ipc_open[side][k]); g->ipc_open[side][k] = nullptr; }
            FM_CHECK_CUDA(cudaIpcOpenMemHandle(&g->ipc_open[side][k], x.h[k], cudaIpcMemLazyEnablePeerAccess));
        }
        (side == 0 ? g->d.up : g->d.dn) = make_peer(g, side, x.H, x.nty, x.rq_cap, g->ipc_open[side]);
        if (g->band == 1 && side == 0) g->gpend = (unsigned *)g->ipc_open[0][9] + 200;
    }
    if (g->band > 1) {
        // band 0 is not a neighbour: map its ring counters for the shared pending count
        BandExport x;
        memcpy(&x, band0_blob, sizeof(x));
        if (x.magic != COLL_MAGIC) { fm_set_error("fm_grid_band_link: bad band-0 export"); return FM_INVALID_ARG; }
        void *p = nullptr;
        FM_CHECK_CUDA(cudaIpcOpenMemHandle(&p, x.h[9], cudaIpcMemLazyEnablePeerAccess));
        if (g->ipc_gpend) cudaIpcCloseMemHandle(g->ipc_gpend);
        g->gpend = (unsigned *)p + 200;
        g->ipc_gpend = p;
    }
    return FM_OK;
}

// Neighbours in this process (bands on the same or on peer-accessible devices).
extern "C" int fm_grid_band_link_local(fm_grid *g, fm_grid *up, fm_grid *dn, fm_grid *band0) {
    if (!g || g->band < 0 || (g->d.has_up && !up) || (g->d.has_dn && !dn) || !band0 || band0->band != 0) {
        fm_set_error("fm_grid_band_link_local: missing neighbour band");
        return FM_INVALID_ARG;
    }
    FM_CHECK_CUDA(cudaSetDevice(g->device));
    fm_grid *nb[2] = {g->d.has_up ? up : nullptr, g->d.has_dn ? dn : nullptr};
    for (int side = 0; side < 2; side++) {
        if (!nb[side]) continue;
        if (nb[side]->W != g->W) { fm_set_error("fm_grid_band_link_local: width mismatch"); return FM_INVALID_ARG; }
        if (nb[side]->device != g->device) {
            const cudaError_t e = cudaDeviceEnablePeerAccess(nb[side]->device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else FM_CHECK_CUDA(e);
        }
        void *buf[BAND_BUFS];
        for (int k = 0; k < BAND_BUFS; k++) buf[k] = band_buf(nb[side], k);
        (side == 0 ? g->d.up : g->d.dn) = make_peer(g, side, nb[side]->H, nb[side]->d.nty, nb[side]->rq.cap, buf);
    }
    if (band0->device != g->device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(band0->device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else FM_CHECK_CUDA(e);
    }
    g->gpend = band0->rq.ctr + 200;
    return FM_OK;
}

namespace {
int band_gather(fm_grid *g, fm_coll *c, const int64_t *v, int n, int64_t *out) {
    (void)g;
    return fm_coll_allgather(c, v, n, out);
}

// sums of column i over ranks (and the max of column imax, if >= 0)
void band_sums(const fm_coll *c, const int64_t *all, int n, int64_t *sum, int imax = -1) {
    for (int i = 0; i < n; i++) sum[i] = 0;
    for (int r = 0; r < c->nranks; r++)
        for (int i = 0; i < n; i++)
            sum[i] = i == imax ? std::max(sum[i], all[r * n + i]) : sum[i] + all[r * n + i];
}

// the shared pending count of the next band ring launch (band 0 sets it before the
// barrier that precedes every band's launch)
int band_arm_ring(fm_grid *g) {
    ringq_init_kernel<<<std::min((g->rq.cap + 255) / 256, g->sms * 8), 256, 0, g->stream>>>(g->rq, g->ntiles, nullptr, nullptr);
    FM_CHECK_LAUNCH();
    g->st.launches++;
    if (g->band == 0) {
        g->h_flags[40] = (int32_t)g->total_tiles;
        FM_CHECK_CUDA(cudaMemcpyAsync(g->gpend, g->h_flags + 40, sizeof(int32_t), cudaMemcpyHostToDevice, g->stream));
    }
    return FM_OK;
}

// global relabel of every band: bit words + seeds, barrier, one ring launch per band
// ending on the shared pending count, then gap + marking; returns the active pixels of
// the whole grid
int band_relabel(fm_grid *g, fm_coll *c, long long *active_total) {
    cudaEventRecord(g->ev[0], g->stream);
    FM_TRY(bfs_init(g, false));
    FM_TRY(band_arm_ring(g));
    FM_TRY(sync_stream(g));
    int64_t one = 1, all[COLL_MAX_RANKS * 4];
    FM_TRY(band_gather(g, c, &one, 1, all));   // every band's distances and queue are seeded
    cudaEventRecord(g->ev[2], g->stream);
    ring_kernel<0><<<ring_blocks(g), 32 * BB_WARPS, 0, g->stream>>>(g->d, g->rq);
    FM_CHECK_LAUNCH();
    cudaEventRecord(g->ev[3], g->stream);
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags + 8, g->rq.ctr + 96, sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags + 12, g->rq.ctr + 248, sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
    FM_CHECK_CUDA(cudaMemsetAsync(g->acc + 4, 0, sizeof(unsigned long long) * 3, g->stream));
    FM_TRY(tq_reset(g, g->d.pq));
    g->pq_parity = 0;
    FM_TRY(bfs_finalize(g));
    // a new push round: external-push flags and their counters start from zero
    FM_CHECK_CUDA(cudaMemsetAsync(g->d.ext, 0, sizeof(int32_t) * 2 * (size_t)g->d.ntx, g->stream));
    FM_CHECK_CUDA(cudaMemsetAsync(g->acc + 24, 0, sizeof(unsigned long long) * 2, g->stream));
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc + 4, g->acc + 4, sizeof(unsigned long long) * 3,
                                  cudaMemcpyDeviceToHost, g->stream));
    cudaEventRecord(g->ev[1], g->stream);
    FM_TRY(sync_stream(g));
    g->st.ms_bfs_kern += elapsed_between(g->ev[2], g->ev[3]);
    g->st.ms_bfs += elapsed(g);
    g->st.reserved[0] += g->h_flags[8];
    g->st.launches += 1;
    g->st.bfs_sweeps += 1;
    g->st.bfs_launches += 1;
    g->active = (long long)g->h_acc[4];
    g->excess_total -= (long long)g->h_acc[5];
    const int64_t v[4] = {(int64_t)g->h_acc[4], (int64_t)g->h_acc[5], (int64_t)g->h_acc[6], g->h_flags[12]};
    FM_TRY(band_gather(g, c, v, 4, all));
    int64_t s[4];
    band_sums(c, all, 4, s, 2);
    g->st.bfs_levels = std::max<int64_t>(g->st.bfs_levels, s[2]);
    if (s[3]) { fm_set_error("row bands: a ring launch waited too long for a neighbour band (not co-resident?)"); return FM_CUDA_ERROR; }
    *active_total = s[0];
    return FM_OK;
}

// One coordinator round of lock-free push launches on every band: batches of pr_batch
// launches, each preceded by an arm step that queues the tiles neighbours pushed flow
// into; after each batch the bands agree on {last launch idle, external flags raised
// vs consumed, relabels}.  The round ends when no band visited a tile in its last
// launch and every raised flag was consumed (no flow left in flight), on the relabel
// budget of the whole grid, or on the launch cap (run_round_tiles' triggers).
int band_push_round(fm_grid *g, fm_coll *c, int32_t cycle_budget) {
    const int k_default = g->k_local_list > 0 ? g->k_local_list : K_LOCAL_LIST_DEFAULT;
    const int k_local = std::max(1, std::min(cycle_budget, k_default));
    const int32_t cap = std::max(1, std::min((cycle_budget + k_local - 1) / k_local,
                                             g->bfs_interval_env > 0 ? g->bfs_interval_env : MAX_LAUNCHES_DEFAULT));
    const long long relabel_budget = std::max<long long>(
        1024, (long long)g->H_total * g->W / (g->relabel_div > 0 ? g->relabel_div : relabel_div_default((int64_t)g->H_total * g->W)));
    const bool pk = g->pk && g->pk_ok && g->op_steps == 1 && !g->op_fused;
    const int blocks = std::max(1, std::min(g->ntiles, g->sms * (pk ? g->pk_per_sm : g->pl_per_sm) / std::max(1, g->colocated)));
    cudaEventRecord(g->ev[0], g->stream);
    FM_CHECK_CUDA(cudaMemsetAsync(g->acc + 10, 0, sizeof(unsigned long long) * 2, g->stream));
    int32_t done = 0;
    int64_t all[COLL_MAX_RANKS * 4];
    while (done < cap) {
        const int batch = std::min(g->pr_batch > 0 ? g->pr_batch : 4, cap - done);
        FM_CHECK_CUDA(cudaMemsetAsync(g->flags, 0, sizeof(int32_t) * batch, g->stream));
        cudaEventRecord(g->ev[2], g->stream);
        for (int i = 0; i < batch; i++) {
            const int p = g->pq_parity;
            band_arm_kernel<<<1, 256, 0, g->stream>>>(g->d, p);
            (pk ? pr_list_kernel<true> : pr_list_kernel<false>)<<<blocks, dim3(PT_W, PL_TY), 0, g->stream>>>(
                g->d, k_local, g->op_steps, g->op_fused, p, g->flags + i, g->acc + 10, nullptr, 0, g->maps, use_tma(g));
            g->pq_parity ^= 1;
        }
        FM_CHECK_LAUNCH();
        cudaEventRecord(g->ev[3], g->stream);
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags, g->flags, sizeof(int32_t) * batch, cudaMemcpyDeviceToHost, g->stream));
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc + 10, g->acc + 10, sizeof(unsigned long long) * 2,
                                      cudaMemcpyDeviceToHost, g->stream));
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc + 24, g->acc + 24, sizeof(unsigned long long) * 2,
                                      cudaMemcpyDeviceToHost, g->stream));
        FM_TRY(sync_stream(g));
        g->st.ms_pr_kern += elapsed_between(g->ev[2], g->ev[3]);
        g->st.launches += 2 * batch;
        g->st.pr_launches += batch;
        for (int i = 0; i < batch; i++) g->st.pr_tiles += g->h_flags[i];
        done += batch;
        const int64_t v[4] = {g->h_flags[batch - 1], (int64_t)g->h_acc[24], (int64_t)g->h_acc[25], (int64_t)g->h_acc[11]};
        FM_TRY(band_gather(g, c, v, 4, all));
        int64_t s[4];
        band_sums(c, all, 4, s);
        if (s[0] == 0 && s[1] == s[2]) break;      // idle everywhere, no flow in flight
        if (s[3] >= relabel_budget) break;
    }
    integrate_inflow_kernel<<<g->ntiles, 4 * PT_W, 0, g->stream>>>(g->d);
    FM_CHECK_LAUNCH();
    g->st.launches++;
    cudaEventRecord(g->ev[1], g->stream);
    FM_TRY(sync_stream(g));
    g->st.ms_push += elapsed(g);
    g->st.pr_sweeps += done;
    g->st.pushes += (int64_t)g->h_acc[10];
    g->st.relabels += (int64_t)g->h_acc[11];
    return FM_OK;
}

int band_cut(fm_grid *g, fm_coll *c) {
    cudaEventRecord(g->ev[0], g->stream);
    FM_TRY(cut_init(g));
    FM_TRY(band_arm_ring(g));
    FM_TRY(sync_stream(g));
    int64_t one = 1, all[COLL_MAX_RANKS];
    FM_TRY(band_gather(g, c, &one, 1, all));   // every band's seeds and queue are in place
    ring_kernel<1><<<ring_blocks(g), 32 * BB_WARPS, 0, g->stream>>>(g->d, g->rq);
    FM_CHECK_LAUNCH();
    g->st.launches++;
    g->st.cut_sweeps++;
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags + 12, g->rq.ctr + 248, sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
    cudaEventRecord(g->ev[1], g->stream);
    FM_TRY(sync_stream(g));
    g->st.ms_cut += elapsed(g);
    const int64_t t = g->h_flags[12];
    FM_TRY(band_gather(g, c, &t, 1, all));
    for (int r = 0; r < c->nranks; r++)
        if (all[r]) { fm_set_error("row bands: the cut ring waited too long for a neighbour band"); return FM_CUDA_ERROR; }
    return FM_OK;
}
}  // namespace

// One band's share of a banded solve (every band of the grid calls it at once, with
// its own rows; see fm_grid_band_setup / _link).  Inputs may be host or device
// memory (UVA copies): the six planes of the band's rows, capD of the row above the
// band and capU of the row below it (W each; NULL for the first / last band).
// flow_out = the whole grid's flow; cut_out = the band's rows of the minimal cut.
extern "C" int fm_grid_band_solve(fm_grid *g, fm_coll *c, const int32_t *capR, const int32_t *capL,
                                  const int32_t *capD, const int32_t *capU, const int32_t *capS,
                                  const int32_t *capT, const int32_t *capD_above, const int32_t *capU_below,
                                  int32_t cycle_budget, int32_t flags, int64_t *flow_out, uint8_t *cut_out,
                                  fm_stats *stats) {
    if (!g || !c || g->band < 0 || c->nranks != g->nbands || c->rank != g->band || cycle_budget < 1 ||
        !capR || !capL || !capD || !capU || !capS || !capT || (g->d.has_up && !capD_above) ||
        (g->d.has_dn && !capU_below)) {
        fm_set_error("fm_grid_band_solve: invalid argument");
        return FM_INVALID_ARG;
    }
    if ((g->d.has_up && !g->d.up.h) || (g->d.has_dn && !g->d.dn.h) || (g->nbands > 1 && !g->gpend)) {
        fm_set_error("fm_grid_band_solve: band not linked to its neighbours");
        return FM_INVALID_ARG;
    }
    if (flags & (FM_GRID_CANCEL_VIOLATIONS | FM_GRID_GLOBAL_SWEEP)) {
        fm_set_error("fm_grid_band_solve: cancel_violations / global sweeps are single-band options");
        return FM_INVALID_ARG;
    }
    FM_CHECK_CUDA(cudaSetDevice(g->device));
    set_stream(g, nullptr);
    if (g->bfs_bits != 2 || g->pr_kernel != 1) { g->bfs_bits = 2; g->pr_kernel = 1; }   // band path = default kernels
    const size_t HW = (size_t)g->HW, W = (size_t)g->W;
    if (!g->band_caps) FM_CHECK_CUDA(cudaMalloc((void **)&g->band_caps, sizeof(int32_t) * (6 * HW + 2 * W)));
    const int32_t *src[6] = {capR, capL, capD, capU, capS, capT};
    cudaEvent_t t0, t1;
    FM_CHECK_CUDA(cudaEventCreate(&t0));
    FM_CHECK_CUDA(cudaEventCreate(&t1));
    cudaEventRecord(t0, g->stream);
    for (int k = 0; k < 6; k++)
        FM_CHECK_CUDA(cudaMemcpyAsync(g->band_caps + k * HW, src[k], sizeof(int32_t) * HW, cudaMemcpyDefault, g->stream));
    int32_t *above = g->band_caps + 6 * HW, *below = above + W;
    if (capD_above) FM_CHECK_CUDA(cudaMemcpyAsync(above, capD_above, sizeof(int32_t) * W, cudaMemcpyDefault, g->stream));
    if (capU_below) FM_CHECK_CUDA(cudaMemcpyAsync(below, capU_below, sizeof(int32_t) * W, cudaMemcpyDefault, g->stream));
    const int32_t *cp = g->band_caps;
    g->flags_solve = flags;
    memset(&g->st, 0, sizeof(g->st));
    const uint64_t calls0 = c->calls;
    int64_t all[COLL_MAX_RANKS * 4];
    FM_CHECK_CUDA(cudaMemsetAsync(g->d_touched, 0, (size_t)g->ntiles, g->stream));
    FM_CHECK_CUDA(cudaMemsetAsync(g->acc, 0, sizeof(unsigned long long) * 32, g->stream));
    FM_CHECK_CUDA(cudaMemsetAsync(g->d.ext, 0, sizeof(int32_t) * 2 * (size_t)g->d.ntx, g->stream));
    g->rq.pend = g->gpend;
    grid_init_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(
        g->d, cp, cp + HW, cp + 2 * HW, cp + 3 * HW, cp + 4 * HW, cp + 5 * HW, above, below,
        (flags & FM_GRID_NO_PRECANCEL) ? 0 : 1, g->acc);
    FM_CHECK_LAUNCH();
    g->st.launches++;
    if (g->two_hop && !(flags & FM_GRID_NO_PRECANCEL)) {
        two_hop_kernel<<<dim3((unsigned)((g->W + 255) / 256), (unsigned)std::min(g->H, 65535)), 256, 0, g->stream>>>(g->d);
        FM_CHECK_LAUNCH();
        g->st.launches++;
    }
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc, g->acc, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, g->stream));
    FM_TRY(sync_stream(g));
    {
        const int64_t v[3] = {(int64_t)g->h_acc[1], (int64_t)g->h_acc[2], (int64_t)g->h_acc[0]};
        FM_TRY(band_gather(g, c, v, 3, all));
        int64_t s[3];
        band_sums(c, all, 3, s);
        if (s[0]) { fm_set_error("negative capacity in grid input (%lld entries)", (long long)s[0]); return FM_INVALID_ARG; }
        if (s[1]) {
            fm_set_error("grid capacities too large for the int32 device state: %lld pixels where capS plus the "
                         "capacities into the pixel, or a neighbour pair's two capacities, exceed 2^31-1", (long long)s[1]);
            return FM_INVALID_ARG;
        }
    }
    g->pk_ok = g->h_acc[3] == 0;
    g->sum_capS = (long long)g->h_acc[0];
    g->excess_total = g->sum_capS;
    long long active = 0;
    int rc = band_relabel(g, c, &active);
    while (rc == FM_OK && active > 0) {
        rc = band_push_round(g, c, cycle_budget);
        if (rc == FM_OK) rc = band_relabel(g, c, &active);
        g->st.rounds++;
    }
    if (rc == FM_OK && !(flags & FM_GRID_NO_CUT)) {
        rc = band_cut(g, c);
        if (rc == FM_OK && cut_out)
            rc = cudaMemcpyAsync(cut_out, g->d.cut, HW, cudaMemcpyDefault, g->stream) == cudaSuccess ? FM_OK : FM_CUDA_ERROR;
    }
    if (rc == FM_OK) {
        FM_CHECK_CUDA(cudaMemsetAsync(g->acc + 8, 0, sizeof(unsigned long long), g->stream));
        sum_e_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(g->d, g->acc + 8);
        FM_CHECK_LAUNCH();
        g->st.launches++;
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc + 8, g->acc + 8, sizeof(unsigned long long), cudaMemcpyDeviceToHost, g->stream));
        cudaEventRecord(t1, g->stream);
        FM_TRY(sync_stream(g));
        const int64_t v = g->sum_capS - (long long)g->h_acc[8];
        FM_TRY(band_gather(g, c, &v, 1, all));
        int64_t flow = 0;
        for (int r = 0; r < c->nranks; r++) flow += all[r];
        if (flow_out) *flow_out = flow;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t0, t1);
        g->st.ms_total = ms;
    }
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    g->st.reserved[2] = (int64_t)(c->calls - calls0);   // host-level agreements (all-gathers) of this solve
    if (stats) *stats = g->st;
    return rc;
}

// ---------------------------------------------------------------- in-process group
struct fm_group {
    int32_t H = 0, W = 0, nbands = 0;
    std::vector<int32_t> edges;
    std::vector<fm_grid *> bands;
    std::vector<fm_coll *> colls;   // one view per band of one process-local segment
    CollShm *shm = nullptr;
};

extern "C" void fm_group_destroy(fm_group *grp) {
    if (!grp) return;
    for (auto b : grp->bands) fm_grid_destroy(b);
    for (auto c : grp->colls) { c->shm = nullptr; delete c; }
    delete grp->shm;
    delete grp;
}

// nbands bands of an H x W grid, band k on devices[k] (bands may share a device:
// virtual bands, their persistent grids are split between them)
extern "C" int fm_group_create(int32_t H, int32_t W, int32_t nbands, const int32_t *devices, fm_group **out) {
    if (!out || !devices || nbands < 1 || nbands > COLL_MAX_RANKS) {
        fm_set_error("fm_group_create: invalid argument (1 <= nbands <= %d)", COLL_MAX_RANKS);
        return FM_INVALID_ARG;
    }
    fm_group *grp = new fm_group();
    grp->H = H; grp->W = W; grp->nbands = nbands;
    grp->edges.resize(nbands + 1);
    int rc = fm_band_split(H, nbands, grp->edges.data());
    if (rc != FM_OK) { delete grp; return rc; }
    grp->shm = new CollShm();
    grp->shm->arrive.store(0);
    grp->shm->magic = COLL_MAGIC;
    grp->shm->nranks = (uint32_t)nbands;
    for (int k = 0; k < nbands; k++) {
        int co = 0;
        for (int j = 0; j < nbands; j++) co += devices[j] == devices[k];
        fm_grid *b = nullptr;
        rc = fm_grid_create(grp->edges[k + 1] - grp->edges[k], W, devices[k], &b);
        if (rc == FM_OK) rc = fm_grid_band_setup(b, k, nbands, H, co);
        if (rc != FM_OK) { if (b) fm_grid_destroy(b); fm_group_destroy(grp); return rc; }
        grp->bands.push_back(b);
        fm_coll *c = new fm_coll();
        c->shm = grp->shm; c->rank = k; c->nranks = nbands; c->bytes = sizeof(CollShm);
        grp->colls.push_back(c);
    }
    for (int k = 0; k < nbands; k++) {
        rc = fm_grid_band_link_local(grp->bands[k], k > 0 ? grp->bands[k - 1] : nullptr,
                                     k + 1 < nbands ? grp->bands[k + 1] : nullptr, grp->bands[0]);
        if (rc != FM_OK) { fm_group_destroy(grp); return rc; }
    }
    *out = grp;
    return FM_OK;
}

extern "C" int fm_group_band(fm_group *grp, int32_t k, fm_grid **band, int32_t *row0, int32_t *rows) {
    if (!grp || k < 0 || k >= grp->nbands) { fm_set_error("fm_group_band: invalid argument"); return FM_INVALID_ARG; }
    if (band) *band = grp->bands[k];
    if (row0) *row0 = grp->edges[k];
    if (rows) *rows = grp->edges[k + 1] - grp->edges[k];
    return FM_OK;
}

// Whole-grid planes (host or device memory), one host thread per band.  stats:
// counters summed over bands, rounds and times of the slowest band.
extern "C" int fm_group_solve(fm_group *grp, const int32_t *capR, const int32_t *capL, const int32_t *capD,
                              const int32_t *capU, const int32_t *capS, const int32_t *capT, int32_t cycle_budget,
                              int32_t flags, int64_t *flow_out, uint8_t *cut_out, fm_stats *stats) {
    if (!grp || !capR || !capL || !capD || !capU || !capS || !capT || cycle_budget < 1) {
        fm_set_error("fm_group_solve: invalid argument");
        return FM_INVALID_ARG;
    }
    const int nb = grp->nbands;
    const size_t W = (size_t)grp->W;
    std::vector<int> rcs(nb, FM_OK);
    std::vector<std::string> errs(nb);
    std::vector<fm_stats> sts(nb);
    std::vector<int64_t> flows(nb, 0);
    // a restarted group: the collective segment's call counters start over
    grp->shm->arrive.store(0);
    for (auto c : grp->colls) c->calls = 0;
    auto work = [&](int k) {
        const size_t o = (size_t)grp->edges[k] * W, o1 = (size_t)grp->edges[k + 1] * W;
        rcs[k] = fm_grid_band_solve(grp->bands[k], grp->colls[k], capR + o, capL + o, capD + o, capU + o, capS + o,
                                    capT + o, k > 0 ? capD + o - W : nullptr, k + 1 < nb ? capU + o1 : nullptr,
                                    cycle_budget, flags, &flows[k], cut_out ? cut_out + o : nullptr, &sts[k]);
        if (rcs[k] != FM_OK) errs[k] = fm_last_error();
    };
    std::vector<std::thread> th;
    for (int k = 1; k < nb; k++) th.emplace_back(work, k);
    work(0);
    for (auto &t : th) t.join();
    for (int k = 0; k < nb; k++)
        if (rcs[k] != FM_OK) { fm_set_error("band %d: %s", k, errs[k].c_str()); return rcs[k]; }
    if (flow_out) *flow_out = flows[0];
    if (stats) {
        fm_stats s = sts[0];
        for (int k = 1; k < nb; k++) {
            const fm_stats &b = sts[k];
            s.pushes += b.pushes; s.relabels += b.relabels; s.launches += b.launches;
            s.pr_sweeps = std::max(s.pr_sweeps, b.pr_sweeps); s.pr_tiles += b.pr_tiles;
            s.bfs_sweeps = std::max(s.bfs_sweeps, b.bfs_sweeps);
            s.bfs_levels = std::max(s.bfs_levels, b.bfs_levels);
            s.pr_launches += b.pr_launches; s.bfs_launches += b.bfs_launches;
            s.ms_total = std::max(s.ms_total, b.ms_total); s.ms_push = std::max(s.ms_push, b.ms_push);
            s.ms_bfs = std::max(s.ms_bfs, b.ms_bfs); s.ms_cut = std::max(s.ms_cut, b.ms_cut);
            s.ms_pr_kern = std::max(s.ms_pr_kern, b.ms_pr_kern); s.ms_bfs_kern = std::max(s.ms_bfs_kern, b.ms_bfs_kern);
            s.reserved[0] += b.reserved[0];
        }
        s.reserved[2] = sts[0].reserved[2];   // agreements: every band makes the same ones
        *stats = s;
    }
    return FM_OK;
}

// per-band counters of the last group solve
extern "C" int fm_group_band_stats(fm_group *grp, int32_t k, fm_stats *stats) {
    if (!grp || k < 0 || k >= grp->nbands || !stats) { fm_set_error("fm_group_band_stats: invalid argument"); return FM_INVALID_ARG; }
    *stats = grp->bands[k]->st;
    return FM_OK;
}

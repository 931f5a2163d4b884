// fm_grid.cu -- B200-native lock-free push-relabel max-flow / min-cut on 4-connected grids.
//
// Replaces the reference's hybrid_solve (maxflow_par.py:157-238) for grid networks.
// Structure-of-arrays residual layout (one int32 plane per direction), Hong's
// lock-free push/relabel with int32 atomics (maxflow_par.py:65-129), device-side
// global relabel by tile-local multi-level relaxation + gap + marking
// (maxflow_seq.py:119-160, maxflow_par.py:220-226), and the minimal source-side
// cut by a seeded residual reach.  See DESIGN.md.
#include <algorithm>
#include <stdio.h>
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

struct GridDev {
    int32_t *e, *h, *rR, *rL, *rD, *rU, *rT, *rS, *cS;
    int32_t *dist;
    uint8_t *mask, *marked, *cut;
    int32_t H, W;
    int32_t V;      // node count |V| = H*W + 2 (the source's height)
    int32_t INF;    // "unreached" distance sentinel (== V)
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
                                 const int32_t *__restrict__ capT, int precancel,
                                 unsigned long long *acc /* [0]=sum capS [1]=invalid */) {
    const int64_t HW = (int64_t)g.H * g.W;
    long long sum = 0, bad = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < HW;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = (int32_t)(p / g.W), c = (int32_t)(p - (int64_t)r * g.W);
        int32_t cs = capS[p], ct = capT[p];
        int32_t cr = c + 1 < g.W ? capR[p] : 0;
        int32_t cl = c > 0 ? capL[p] : 0;
        int32_t cd = r + 1 < g.H ? capD[p] : 0;
        int32_t cu = r > 0 ? capU[p] : 0;
        bad += (cs < 0) | (ct < 0) | (cr < 0) | (cl < 0) | (cd < 0) | (cu < 0);
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
        sum += cs;
    }
    // grid-stride kernel with 1-D blocks of 256
    __shared__ long long red[2][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if (lane == 0) { red[0][wid] = sum; red[1][wid] = bad; }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long s = 0, b = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) { s += red[0][i]; b += red[1][i]; }
        if (s) atomicAdd(&acc[0], (unsigned long long)s);
        if (b) atomicAdd(&acc[1], (unsigned long long)b);
    }
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
        g.mask[p] = m;
        g.dist[p] = (m & M_T) ? 1 : g.INF;
    }
}

__global__ void __launch_bounds__(256) bfs_tile_kernel(GridDev g, int32_t *changed_flag) {
    __shared__ int32_t sd[TILE_H + 2][TILE_W + 2];
    const int c0 = blockIdx.x * TILE_W, r0 = blockIdx.y * TILE_H;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * TILE_W + tx;
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
            const int r = r0 + ty + k * BLK_Y;
            const int32_t v = sd[ty + k * BLK_Y + 1][tx + 1];
            if (r < g.H && c < g.W && v != d0[k]) g.dist[(int64_t)r * g.W + c] = v;
        }
        if (tid == 0) *changed_flag = 1;
    }
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
        g.mask[p] = m;
        g.cut[p] = (g.e[p] > 0 || g.cS[p] - g.rS[p] > 0) ? 1 : 0;
    }
}

__global__ void __launch_bounds__(256) cut_tile_kernel(GridDev g, int32_t *changed_flag) {
    __shared__ uint8_t ss[TILE_H + 2][TILE_W + 2];
    const int c0 = blockIdx.x * TILE_W, r0 = blockIdx.y * TILE_H;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * TILE_W + tx;
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
            const int r = r0 + ty + k * BLK_Y;
            if (grew[k] && r < g.H && c < g.W) g.cut[(int64_t)r * g.W + c] = 1;
        }
        if (tid == 0) *changed_flag = 1;
    }
}

// sum of e over all pixels (flow = sum capS - sum e: node conservation)
__global__ void sum_e_kernel(GridDev g, unsigned long long *acc) {
    const int64_t HW = (int64_t)g.H * g.W;
    long long s = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < HW;
         p += (int64_t)gridDim.x * blockDim.x)
        s += g.e[p];
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
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[4] = {};
    int grid_blocks = 0;                 // 1-D grid-stride kernels
    // solve state
    int32_t flags_solve = 0;
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

dim3 tile_grid(const fm_grid *g) {
    return dim3((g->W + TILE_W - 1) / TILE_W, (g->H + TILE_H - 1) / TILE_H);
}

// global relabel + gap + marking; leaves the active-pixel count in g->active
int global_relabel(fm_grid *g) {
    cudaEventRecord(g->ev[0], g->stream);
    bfs_init_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(g->d);
    FM_CHECK_LAUNCH();
    g->st.launches++;
    const dim3 tg = tile_grid(g);
    const int batch = 4;
    for (;;) {
        FM_CHECK_CUDA(cudaMemsetAsync(g->flags, 0, sizeof(int32_t) * batch, g->stream));
        cudaEventRecord(g->ev[2], g->stream);
        for (int i = 0; i < batch; i++) {
            bfs_tile_kernel<<<tg, dim3(TILE_W, BLK_Y), 0, g->stream>>>(g->d, g->flags + i);
        }
        FM_CHECK_LAUNCH();
        cudaEventRecord(g->ev[3], g->stream);
        g->st.launches += batch;
        g->st.bfs_launches += batch;
        g->st.bfs_sweeps += batch;
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags, g->flags, sizeof(int32_t) * batch,
                                      cudaMemcpyDeviceToHost, g->stream));
        FM_TRY(sync_stream(g));
        g->st.ms_bfs_kern += elapsed_between(g->ev[2], g->ev[3]);
        if (g->h_flags[batch - 1] == 0) break;
    }
    FM_CHECK_CUDA(cudaMemsetAsync(g->acc + 4, 0, sizeof(unsigned long long) * 3, g->stream));
    bfs_finalize_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(g->d, g->acc + 4);
    FM_CHECK_LAUNCH();
    g->st.launches++;
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc + 4, g->acc + 4, sizeof(unsigned long long) * 3,
                                  cudaMemcpyDeviceToHost, g->stream));
    cudaEventRecord(g->ev[1], g->stream);
    FM_TRY(sync_stream(g));
    g->st.ms_bfs += elapsed(g);
    g->active = (long long)g->h_acc[4];
    g->excess_total -= (long long)g->h_acc[5];
    g->st.bfs_levels = std::max<int64_t>(g->st.bfs_levels, (int64_t)g->h_acc[6]);
    return FM_OK;
}

int begin_device(fm_grid *g, const int32_t *capR, const int32_t *capL, const int32_t *capD,
                 const int32_t *capU, const int32_t *capS, const int32_t *capT, int32_t flags) {
    g->flags_solve = flags;
    memset(&g->st, 0, sizeof(g->st));
    FM_CHECK_CUDA(cudaMemsetAsync(g->acc, 0, sizeof(unsigned long long) * 16, g->stream));
    grid_init_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(
        g->d, capR, capL, capD, capU, capS, capT, (flags & FM_GRID_NO_PRECANCEL) ? 0 : 1, g->acc);
    FM_CHECK_LAUNCH();
    g->st.launches++;
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc, g->acc, sizeof(unsigned long long) * 2,
                                  cudaMemcpyDeviceToHost, g->stream));
    FM_TRY(sync_stream(g));
    if (g->h_acc[1] != 0) {
        fm_set_error("negative capacity in grid input (%llu entries)", g->h_acc[1]);
        return FM_INVALID_ARG;
    }
    g->sum_capS = (long long)g->h_acc[0];
    // HybridState.excess_total = sum of excess after init_preflow = sum capS
    // (maxflow_par.py:56); pre-cancelled units are already at t.
    g->excess_total = g->sum_capS;
    return global_relabel(g);
}

// one coordinator round: lock-free sweeps until an idle sweep or the budget,
// then cancel (opt-in), global relabel, gap, mark (maxflow_par.py:195-229)
int run_round(fm_grid *g, int32_t cycle_budget, int32_t bfs_interval) {
    const int32_t cap = std::max(1, std::min(cycle_budget, bfs_interval > 0 ? bfs_interval : 64));
    const dim3 grid((g->W + TILE_W - 1) / TILE_W, (g->H + BLK_Y - 1) / BLK_Y);
    int32_t done = 0;
    cudaEventRecord(g->ev[0], g->stream);
    FM_CHECK_CUDA(cudaMemsetAsync(g->acc + 10, 0, sizeof(unsigned long long) * 2, g->stream));
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
    if (g->flags_solve & FM_GRID_CANCEL_VIOLATIONS) {
        cancel_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(g->d, g->acc + 12);
        FM_CHECK_LAUNCH();
        g->st.launches++;
    }
    FM_CHECK_CUDA(cudaMemcpyAsync(g->h_acc + 10, g->acc + 10, sizeof(unsigned long long) * 2,
                                  cudaMemcpyDeviceToHost, g->stream));
    cudaEventRecord(g->ev[1], g->stream);
    FM_TRY(sync_stream(g));
    g->st.ms_push += elapsed(g);
    g->st.pushes += (int64_t)g->h_acc[10];
    g->st.relabels += (int64_t)g->h_acc[11];
    g->st.pr_sweeps += done;
    g->st.bytes_push += (int64_t)done * 32 * g->HW + 16 * (int64_t)g->h_acc[10];
    FM_TRY(global_relabel(g));
    g->st.bytes_bfs += 0;
    g->st.rounds++;
    return FM_OK;
}

int compute_cut(fm_grid *g, uint8_t *cut_out_dev) {
    cudaEventRecord(g->ev[0], g->stream);
    cut_init_kernel<<<g->grid_blocks, 256, 0, g->stream>>>(g->d);
    FM_CHECK_LAUNCH();
    g->st.launches++;
    const dim3 tg = tile_grid(g);
    const int batch = 4;
    for (;;) {
        FM_CHECK_CUDA(cudaMemsetAsync(g->flags, 0, sizeof(int32_t) * batch, g->stream));
        for (int i = 0; i < batch; i++)
            cut_tile_kernel<<<tg, dim3(TILE_W, BLK_Y), 0, g->stream>>>(g->d, g->flags + i);
        FM_CHECK_LAUNCH();
        g->st.launches += batch;
        g->st.cut_sweeps += batch;
        FM_CHECK_CUDA(cudaMemcpyAsync(g->h_flags, g->flags, sizeof(int32_t) * batch,
                                      cudaMemcpyDeviceToHost, g->stream));
        FM_TRY(sync_stream(g));
        if (g->h_flags[batch - 1] == 0) break;
    }
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
    const size_t n4 = sizeof(int32_t) * (size_t)g->HW, n1 = (size_t)g->HW;
    int32_t **planes[] = {&g->d.e, &g->d.h, &g->d.rR, &g->d.rL, &g->d.rD, &g->d.rU,
                          &g->d.rT, &g->d.rS, &g->d.cS, &g->d.dist};
    for (auto pp : planes) {
        if (cudaMalloc((void **)pp, n4) != cudaSuccess) {
            fm_set_error("cudaMalloc of %zu bytes failed", n4);
            fm_grid_destroy(g);
            return FM_CUDA_ERROR;
        }
    }
    if (cudaMalloc((void **)&g->d.mask, n1) != cudaSuccess ||
        cudaMalloc((void **)&g->d.marked, n1) != cudaSuccess ||
        cudaMalloc((void **)&g->d.cut, n1) != cudaSuccess ||
        cudaMalloc((void **)&g->acc, sizeof(unsigned long long) * 16) != cudaSuccess ||
        cudaMalloc((void **)&g->flags, sizeof(int32_t) * 64) != cudaSuccess ||
        cudaMallocHost((void **)&g->h_acc, sizeof(unsigned long long) * 16) != cudaSuccess ||
        cudaMallocHost((void **)&g->h_flags, sizeof(int32_t) * 64) != cudaSuccess ||
        cudaStreamCreateWithFlags(&g->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        fm_set_error("fm_grid_create: allocation failed: %s", cudaGetErrorString(cudaGetLastError()));
        fm_grid_destroy(g);
        return FM_CUDA_ERROR;
    }
    for (auto &e : g->ev) cudaEventCreate(&e);
    g->stream = g->own_stream;
    g->d.H = H; g->d.W = W;
    g->d.V = (int32_t)(g->HW + 2);
    g->d.INF = g->d.V;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    g->grid_blocks = (int)std::min<int64_t>((g->HW + 255) / 256, (int64_t)sms * 8);
    *out = g;
    return FM_OK;
}

extern "C" void fm_grid_destroy(fm_grid *g) {
    if (!g) return;
    cudaSetDevice(g->device);
    int32_t *planes[] = {g->d.e, g->d.h, g->d.rR, g->d.rL, g->d.rD, g->d.rU,
                         g->d.rT, g->d.rS, g->d.cS, g->d.dist, g->in_caps};
    for (auto p : planes) if (p) cudaFree(p);
    if (g->d.mask) cudaFree(g->d.mask);
    if (g->d.marked) cudaFree(g->d.marked);
    if (g->d.cut) cudaFree(g->d.cut);
    if (g->acc) cudaFree(g->acc);
    if (g->flags) cudaFree(g->flags);
    if (g->h_acc) cudaFreeHost(g->h_acc);
    if (g->h_flags) cudaFreeHost(g->h_flags);
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
        cudaEventRecord(a, g->stream);
        if (cudaMemcpyAsync(cut_out, g->d.cut, HW, cudaMemcpyDeviceToHost, g->stream) != cudaSuccess)
            rc = FM_CUDA_ERROR;
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

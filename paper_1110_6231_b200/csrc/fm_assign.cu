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
#include <cooperative_groups.h>
#include <algorithm>
#include <string.h>

#include "fm_common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int ATHREADS = 512;            // 16 warps per CTA
constexpr int AWARPS = ATHREADS / 32;
constexpr long long I64_MAX = 0x7fffffffffffffffLL;

struct AssignDev {
    const int32_t *w;      // n x n weights (row x), FM_ABSENT_WEIGHT = no arc
    int64_t *px, *py;      // prices of X and Y
    int32_t *match;        // match[x] = y carrying x's unit, -1 if x holds its excess
    int32_t *ey;           // excess of y
    uint32_t *fixed;       // arc-fix bitmask, row-major n x nw words
    uint8_t *frozen;       // frozen[x]: x's matched arc is fixed (its flow never changes)
    int32_t *frozen_in;    // frozen_in[y]: number of frozen matches into y
    int32_t *xlist[2], *ylist[2];
    int32_t *cnt;          // [0..1] X list counts, [2..3] Y list counts, [4] infeasible, [5] tail flag
    unsigned long long *ops;  // [0] pushes [1] relabels [2] rounds [3] tail rounds [4] fixed pairs
    int32_t n, nw;
    int64_t scale;         // n + 1
    int64_t eps;
    int use_fix;
};

__device__ __forceinline__ bool is_fixed(const AssignDev &a, int x, int y) {
    return a.use_fix && ((__ldcg(a.fixed + (size_t)x * a.nw + (y >> 5)) >> (y & 31)) & 1u);
}

// (value, index) min with the lower index winning ties (first arc in the
// reference's out-arc order wins, assign_par.py:84-90)
__device__ __forceinline__ void warp_argmin(long long &v, int &i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (ov < v || (ov == v && oi < i)) { v = ov; i = oi; }
    }
}

// min over non-fixed present arcs of x of the part-reduced cost c(x,y) - p(y)
// (assign_scaling.py:170-182, assign_par.py:82-90).  Whole warp; result in all lanes.
__device__ void scan_row(const AssignDev &a, int x, long long &best, int &arg) {
    const int32_t *row = a.w + (size_t)x * a.n;
    const int lane = threadIdx.x & 31;
    long long bv = I64_MAX;
    int bi = INT32_MAX;
    if ((a.n & 3) == 0) {
        const int4 *row4 = reinterpret_cast<const int4 *>(row);
        const int n4 = a.n >> 2;
        for (int j = lane; j < n4; j += 32) {
            const int4 w4 = __ldg(row4 + j);
            const int wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int y = 4 * j + k;
                if (wv[k] == FM_ABSENT_WEIGHT || is_fixed(a, x, y)) continue;
                const long long v = -(long long)wv[k] * a.scale - __ldcg((const long long *)a.py + y);
                if (v < bv) { bv = v; bi = y; }
            }
        }
    } else {
        for (int y = lane; y < a.n; y += 32) {
            const int wv = __ldg(row + y);
            if (wv == FM_ABSENT_WEIGHT || is_fixed(a, x, y)) continue;
            const long long v = -(long long)wv * a.scale - __ldcg((const long long *)a.py + y);
            if (v < bv) { bv = v; bi = y; }
        }
    }
    warp_argmin(bv, bi);
    best = bv;
    arg = bi;
}

// X op: relabel if the cheapest arc is not admissible, then push one unit on it.
__device__ void x_op(const AssignDev &a, int x, int32_t *ylist_next, int32_t *ycnt_next,
                     unsigned long long &pushes, unsigned long long &relabels) {
    long long best;
    int y;
    scan_row(a, x, best, y);
    const int lane = threadIdx.x & 31;
    if (lane == 0) {
        if (y == INT32_MAX) {
            atomicExch(a.cnt + 4, 1);  // active node with no residual arc: infeasible
        } else {
            const long long px = a.px[x];
            if (!(best < -px)) {       // not admissible: p(x) <- -(best + eps)
                a.px[x] = -(best + a.eps);
                relabels++;
            }
            a.match[x] = y;            // unit push x -> y
            pushes++;
            const int old = atomicAdd(a.ey + y, 1);
            if (old == 0) ylist_next[atomicAdd(ycnt_next, 1)] = y;
        }
    }
    __syncwarp();
}

// Y op: while y holds excess, push a unit back to its cheapest incoming X
// (reverse arc cost +(n+1) w), relabelling y first when it is not admissible.
__device__ void y_op(const AssignDev &a, int y, int32_t *xlist_next, int32_t *xcnt_next,
                     unsigned long long &pushes, unsigned long long &relabels) {
    const int lane = threadIdx.x & 31;
    int ey = __ldcg(a.ey + y);
    long long py = __ldcg((const long long *)a.py + y);
    while (ey > 0) {
        long long bv = I64_MAX;
        int bi = INT32_MAX;
        for (int x = lane; x < a.n; x += 32) {
            if (__ldcg(a.match + x) != y || __ldcg(a.frozen + x)) continue;
            const long long v = (long long)__ldg(a.w + (size_t)x * a.n + y) * a.scale -
                                __ldcg((const long long *)a.px + x);
            if (v < bv) { bv = v; bi = x; }
        }
        warp_argmin(bv, bi);
        if (bi == INT32_MAX) {  // cannot happen for a consistent state
            if (lane == 0) atomicExch(a.cnt + 4, 2);
            break;
        }
        if (lane == 0) {
            if (!(bv < -py)) {
                py = -(bv + a.eps);
                relabels++;
            }
            a.match[bi] = -1;
            xlist_next[atomicAdd(xcnt_next, 1)] = bi;
            pushes++;
        }
        ey--;
        __syncwarp();
    }
    if (lane == 0) {
        a.py[y] = py;
        a.ey[y] = ey;
    }
    __syncwarp();
}

// begin_refine (assign_scaling.py:145-182) fused with the first X phase: drop
// unfrozen flow, set p(x) = -(min part-reduced cost + eps) and push x's unit on
// that arc (admissible at reduced cost -eps by construction).
__global__ void __launch_bounds__(ATHREADS) begin_refine_kernel(AssignDev a) {
    const int warp = (blockIdx.x * ATHREADS + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * ATHREADS) >> 5;
    const int lane = threadIdx.x & 31;
    unsigned long long pushes = 0, relabels = 0;
    for (int x = warp; x < a.n; x += nwarps) {
        long long best;
        int y;
        scan_row(a, x, best, y);
        if (lane == 0) {
            if (y != INT32_MAX) a.px[x] = -(best + a.eps);
            if (!a.frozen[x]) {
                if (y == INT32_MAX) {
                    a.match[x] = -1;
                    atomicExch(a.cnt + 4, 1);
                } else {
                    a.match[x] = y;
                    pushes++;
                    const int old = atomicAdd(a.ey + y, 1);
                    if (old == 0) a.ylist[0][atomicAdd(a.cnt + 2, 1)] = y;
                }
            }
        }
    }
    if (lane == 0 && pushes) atomicAdd(a.ops + 0, pushes);
    (void)relabels;
}

// excess of y after flow removal: supplies (-1) + frozen flows (assign_scaling.py:158-168)
__global__ void reset_excess_kernel(AssignDev a) {
    for (int y = blockIdx.x * blockDim.x + threadIdx.x; y < a.n; y += gridDim.x * blockDim.x)
        a.ey[y] = -1 + a.frozen_in[y];
}

// The refine's push/relabel rounds (refine_par's coordinator loop, assign_par.py:162-236)
// as one cooperative kernel.  Round r: Y phase over ylist[r&1] -> xlist[r&1];
// grid barrier; X phase over xlist[r&1] -> ylist[(r+1)&1]; grid barrier.
__global__ void __launch_bounds__(ATHREADS) refine_rounds_kernel(AssignDev a, int tail_threshold,
                                                                 long long round_budget) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int gwarp = (blockIdx.x * ATHREADS + threadIdx.x) >> 5;
    const int gwarps = (gridDim.x * ATHREADS) >> 5;
    const int cwarp = threadIdx.x >> 5;
    unsigned long long pushes = 0, relabels = 0, rounds = 0, tail_rounds = 0;
    bool tail = false;
    for (int r = 0;; r++) {
        const int b = r & 1, nb = b ^ 1;
        const int ny = __ldcg(a.cnt + 2 + b);
        if (ny == 0 || __ldcg(a.cnt + 4)) break;
        if (r >= round_budget) {  // prices diverge: no perfect matching (assign_par.py:221-226)
            if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(a.cnt + 4, 3);
            break;
        }
        if (!tail && ny <= tail_threshold) {
            tail = true;
            if (blockIdx.x != 0) break;  // CTA 0 finishes the refine alone
        }
        rounds++;
        if (tail) tail_rounds++;
        const int wi = tail ? cwarp : gwarp;
        const int wn = tail ? AWARPS : gwarps;
        // ---- Y phase
        if ((tail || blockIdx.x == 0) && threadIdx.x == 0) {
            a.cnt[nb] = 0;      // X list of round r+1 (last read in round r-1)
            a.cnt[2 + nb] = 0;  // Y list of round r+1 (last read at round r-1)
        }
        for (int i = wi; i < ny; i += wn)
            y_op(a, __ldcg(a.ylist[b] + i), a.xlist[b], a.cnt + b, pushes, relabels);
        if (tail) { __threadfence_block(); __syncthreads(); } else grid.sync();
        // ---- X phase
        const int nx = __ldcg(a.cnt + b);
        for (int i = wi; i < nx; i += wn)
            x_op(a, __ldcg(a.xlist[b] + i), a.ylist[nb], a.cnt + 2 + nb, pushes, relabels);
        if (tail) { __threadfence_block(); __syncthreads(); } else grid.sync();
    }
    if (lane == 0) {
        if (pushes) atomicAdd(a.ops + 0, pushes);
        if (relabels) atomicAdd(a.ops + 1, relabels);
    }
    if (threadIdx.x == 0 && (blockIdx.x == 0)) {
        atomicAdd(a.ops + 2, rounds);
        atomicAdd(a.ops + 3, tail_rounds);
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
    if (lane == 0 && cnt) atomicAdd(a.ops + 4, cnt);
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
    int coop_blocks = 0, sms = 0;
    fm_stats st{};
};

namespace {

int assign_solve_device(fm_assign *A, const int32_t *w, int64_t alpha, int32_t flags,
                        int64_t *objective_out, int32_t *match_out, int64_t *prices_out) {
    const int n = A->n;
    AssignDev &d = A->d;
    d.w = w;
    d.use_fix = (flags & FM_ASSIGN_ARC_FIX) ? 1 : 0;
    memset(&A->st, 0, sizeof(A->st));
    cudaStream_t s = A->stream;
    cudaEvent_t t0, t1;
    FM_CHECK_CUDA(cudaEventCreate(&t0));
    FM_CHECK_CUDA(cudaEventCreate(&t1));
    cudaEventRecord(t0, s);
    // make_scaling_state (assign_scaling.py:127-142): prices 0, eps0 = max(1, bound)
    FM_CHECK_CUDA(cudaMemsetAsync(d.px, 0, sizeof(int64_t) * n, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.py, 0, sizeof(int64_t) * n, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.frozen, 0, n, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.frozen_in, 0, sizeof(int32_t) * n, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.fixed, 0, sizeof(uint32_t) * (size_t)n * d.nw, s));
    FM_CHECK_CUDA(cudaMemsetAsync(d.ops, 0, sizeof(unsigned long long) * 8, s));
    FM_CHECK_CUDA(cudaMemsetAsync(A->acc, 0, sizeof(unsigned long long) * 4, s));
    weight_bound_kernel<<<A->sms * 4, 256, 0, s>>>(w, (int64_t)n * n, A->acc);
    FM_CHECK_LAUNCH();
    A->st.launches++;
    FM_CHECK_CUDA(cudaMemcpyAsync(A->h_acc, A->acc, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, s));
    FM_CHECK_CUDA(cudaStreamSynchronize(s));
    const long long bound = (long long)A->h_acc[0] * (long long)(n + 1);
    // _ops_budget (assign_scaling.py:374-377) = max(1e4, 40 n^2 m); every round does >= 1 op
    const double budget_d = std::max(1e4, 40.0 * n * (double)n * std::max<double>(1.0, (double)A->h_acc[2]));
    const long long round_budget = budget_d > 4e18 ? (long long)4e18 : (long long)budget_d;
    long long eps = std::max(1LL, bound);
    const int tail_threshold = AWARPS;
    int rc = FM_OK;
    for (;;) {
        eps = std::max(1LL, (eps + alpha - 1) / alpha);   // -(-eps // alpha)
        d.eps = eps;
        FM_CHECK_CUDA(cudaMemsetAsync(d.cnt, 0, sizeof(int32_t) * 8, s));
        reset_excess_kernel<<<(n + 255) / 256, 256, 0, s>>>(d);
        FM_CHECK_LAUNCH();
        begin_refine_kernel<<<std::max(1, std::min((n + AWARPS - 1) / AWARPS, A->sms * 4)), ATHREADS, 0, s>>>(d);
        FM_CHECK_LAUNCH();
        void *args[] = {(void *)&d, (void *)&tail_threshold, (void *)&round_budget};
        FM_CHECK_CUDA(cudaLaunchCooperativeKernel((void *)refine_rounds_kernel, dim3(A->coop_blocks),
                                                  dim3(ATHREADS), args, 0, s));
        A->st.launches += 3;
        if (d.use_fix) {
            arc_fix_kernel<<<std::max(1, std::min((n + 7) / 8, A->sms * 8)), 256, 0, s>>>(d);
            FM_CHECK_LAUNCH();
            A->st.launches++;
        }
        A->st.refines++;
        FM_CHECK_CUDA(cudaMemcpyAsync(A->h_cnt, d.cnt, sizeof(int32_t) * 8, cudaMemcpyDeviceToHost, s));
        FM_CHECK_CUDA(cudaStreamSynchronize(s));
        if (A->h_cnt[4]) {
            rc = FM_INFEASIBLE;
            fm_set_error(A->h_cnt[4] == 1 ? "active node has no residual arc: instance admits no perfect matching"
                         : A->h_cnt[4] == 3 ? "operation budget exceeded; prices diverge, instance admits no perfect matching"
                                            : "inconsistent Y excess during refine");
            if (A->h_cnt[4] == 2) { rc = FM_CUDA_ERROR; break; }
            break;
        }
        if (eps == 1) break;
    }
    if (rc == FM_OK) {
        objective_kernel<<<std::max(1, std::min((n + 255) / 256, A->sms * 2)), 256, 0, s>>>(w, d.match, n, A->acc + 1);
        FM_CHECK_LAUNCH();
        A->st.launches++;
    }
    cudaEventRecord(t1, s);
    FM_CHECK_CUDA(cudaMemcpyAsync(A->h_ops, d.ops, sizeof(unsigned long long) * 8, cudaMemcpyDeviceToHost, s));
    FM_CHECK_CUDA(cudaMemcpyAsync(A->h_acc, A->acc, sizeof(unsigned long long) * 4, cudaMemcpyDeviceToHost, s));
    if (match_out) FM_CHECK_CUDA(cudaMemcpyAsync(match_out, d.match, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
    if (prices_out) {
        FM_CHECK_CUDA(cudaMemcpyAsync(prices_out, d.px, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
        FM_CHECK_CUDA(cudaMemcpyAsync(prices_out + n, d.py, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
    }
    FM_CHECK_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    A->st.ms_total = ms;
    A->st.ms_push = ms;
    A->st.pushes = (int64_t)A->h_ops[0];
    A->st.relabels = (int64_t)A->h_ops[1];
    A->st.rounds = (int64_t)A->h_ops[2];
    A->st.pr_sweeps = (int64_t)A->h_ops[3];  // rounds run by the single-CTA tail
    A->st.reserved[0] = (int64_t)A->h_ops[4]; // pairs fixed
    // algorithmic bytes: every op scans one weight row (4n) + n prices (8n); the
    // begin phase and arc fixing read the whole matrix once each per refine
    A->st.bytes_push = (A->st.pushes + A->st.relabels) * 12LL * n +
                       A->st.refines * (int64_t)n * n * 4 * (d.use_fix ? 2 : 1);
    if (rc == FM_OK && objective_out) *objective_out = (int64_t)A->h_acc[1];
    return rc;
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
              cudaMalloc((void **)&d.frozen, n) == cudaSuccess &&
              cudaMalloc((void **)&d.frozen_in, sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.xlist[0], sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.xlist[1], sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.ylist[0], sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.ylist[1], sizeof(int32_t) * n) == cudaSuccess &&
              cudaMalloc((void **)&d.cnt, sizeof(int32_t) * 8) == cudaSuccess &&
              cudaMalloc((void **)&d.ops, sizeof(unsigned long long) * 8) == cudaSuccess &&
              cudaMalloc((void **)&A->acc, sizeof(unsigned long long) * 4) == cudaSuccess &&
              cudaMallocHost((void **)&A->h_ops, sizeof(unsigned long long) * 8) == cudaSuccess &&
              cudaMallocHost((void **)&A->h_acc, sizeof(unsigned long long) * 4) == cudaSuccess &&
              cudaMallocHost((void **)&A->h_cnt, sizeof(int32_t) * 8) == cudaSuccess &&
              cudaStreamCreateWithFlags(&A->own_stream, cudaStreamNonBlocking) == cudaSuccess;
    if (!ok) {
        fm_set_error("fm_assign_create: allocation failed: %s", cudaGetErrorString(cudaGetLastError()));
        fm_assign_destroy(A);
        return FM_CUDA_ERROR;
    }
    A->stream = A->own_stream;
    cudaDeviceGetAttribute(&A->sms, cudaDevAttrMultiProcessorCount, device);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, refine_rounds_kernel, ATHREADS, 0);
    A->coop_blocks = std::max(1, std::min(per_sm, 2) * A->sms);
    *out = A;
    return FM_OK;
}

extern "C" void fm_assign_destroy(fm_assign *A) {
    if (!A) return;
    cudaSetDevice(A->device);
    void *dev[] = {A->d.px, A->d.py, A->d.match, A->d.ey, A->d.fixed, A->d.frozen, A->d.frozen_in,
                   A->d.xlist[0], A->d.xlist[1], A->d.ylist[0], A->d.ylist[1], A->d.cnt, A->d.ops,
                   A->acc, A->in_w};
    for (void *p : dev) if (p) cudaFree(p);
    if (A->h_ops) cudaFreeHost(A->h_ops);
    if (A->h_acc) cudaFreeHost(A->h_acc);
    if (A->h_cnt) cudaFreeHost(A->h_cnt);
    if (A->own_stream) cudaStreamDestroy(A->own_stream);
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

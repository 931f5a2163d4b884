// fm_csr.cu -- lock-free push-relabel max-flow / min-cut on arbitrary networks (CSR).
//
// The generic-graph form of the reference's hybrid_solve (maxflow_par.py:157-238):
// the arc-pair forward star of graph.py:43-84 (arc 2k forward, 2k+1 its reverse,
// out-arc lists in input order) is uploaded as CSR; one thread owns one node and runs
// the lockfree_round operation (maxflow_par.py:95-128) with int32 atomics on the
// residuals (int64 for capacities past the int32 range, fm_csr_solve64) and int64
// atomics on the excesses; between rounds the coordinator runs a
// level-synchronous frontier BFS from t (maxflow_seq.py:119-146) on the device, the
// gap relabel and the marking (maxflow_par.py:220-226).  The cut is the seeded
// residual reach.  Grid networks use fm_grid.cu instead.
#include <algorithm>
#include <string.h>
#include <vector>

#include "fm_common.cuh"

namespace {

template <typename R>   // residual type: int32_t, or long long for wide capacities
struct CsrDev {
    int32_t n, s, t;
    int64_t m2;
    const int64_t *ostart;   // n + 1
    const int32_t *oarc;     // out-arc slot ids, per node in input order
    const int32_t *head;     // head of every arc slot
    const R *cap;            // capacity of every slot
    R *res;                  // residual of every slot
    unsigned long long *ex;  // excess (two's complement int64 in an unsigned word)
    int32_t *h;
    int32_t *dist;
    uint8_t *marked, *cut;
    int32_t *frontier[2];
    int32_t *fcount;         // [0..1] frontier sizes, [2] changed/active flag
};

__device__ __forceinline__ void res_add(int32_t *p, long long d) { atomicAdd(p, (int32_t)d); }
__device__ __forceinline__ void res_add(long long *p, long long d) {
    atomicAdd((unsigned long long *)p, (unsigned long long)d);
}

template <typename R>
__device__ __forceinline__ long long ld_ex(const CsrDev<R> &g, int v) {
    return (long long)__ldcg(g.ex + v);
}

// init_preflow (maxflow_seq.py:47-64): saturate the source's forward, non-loop arcs
template <typename R>
__global__ void csr_init_kernel(CsrDev<R> g) {
    for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < g.m2; a += (int64_t)gridDim.x * blockDim.x)
        g.res[a] = g.cap[a];
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += gridDim.x * blockDim.x) {
        g.ex[v] = 0;
        g.h[v] = v == g.s ? g.n : 0;
        g.marked[v] = 0;
    }
}

template <typename R>
__global__ void csr_preflow_kernel(CsrDev<R> g) {
    const int64_t b = g.ostart[g.s], e = g.ostart[g.s + 1];
    for (int64_t i = b + blockIdx.x * blockDim.x + threadIdx.x; i < e; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t a = g.oarc[i];
        if ((a & 1) || g.head[a] == g.s) continue;
        const R f = g.cap[a];
        if (f <= 0) continue;
        g.res[a] -= f;
        res_add(g.res + (a ^ 1), f);
        atomicAdd(g.ex + g.head[a], (unsigned long long)(long long)f);
    }
}

// one lock-free pass over the nodes (maxflow_par.py:95-128)
template <typename R>
__global__ void csr_pass_kernel(CsrDev<R> g, int32_t *active_flag, unsigned long long *ops) {
    long long pushes = 0, relabels = 0;
    bool act = false;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < g.n; x += gridDim.x * blockDim.x) {
        if (x == g.s || x == g.t) continue;
        const long long e = ld_ex(g, x);
        if (e <= 0) continue;
        const int32_t hx = __ldcg(g.h + x);
        if (hx >= g.n) continue;
        int32_t best_h = INT32_MAX;
        int32_t best = -1;
        for (int64_t i = g.ostart[x]; i < g.ostart[x + 1]; i++) {
            const int32_t a = g.oarc[i];
            if (__ldcg(g.res + a) > 0) {
                const int32_t hy = __ldcg(g.h + g.head[a]);
                if (hy < best_h) { best_h = hy; best = a; }
            }
        }
        if (best < 0) continue;  // nothing residual: the coordinator writes it off
        act = true;
        if (hx > best_h) {
            const long long r = __ldcg(g.res + best);
            const long long d = e < r ? e : r;
            atomicAdd(g.ex + x, (unsigned long long)(-d));
            res_add(g.res + best, -d);
            res_add(g.res + (best ^ 1), d);
            atomicAdd(g.ex + g.head[best], (unsigned long long)d);
            pushes++;
        } else {
            g.h[x] = best_h + 1;
            relabels++;
        }
    }
    if (__syncthreads_or(act) && threadIdx.x == 0) *active_flag = 1;
    if (pushes) atomicAdd(ops + 0, (unsigned long long)pushes);
    if (relabels) atomicAdd(ops + 1, (unsigned long long)relabels);
}

// global relabel: level-synchronous BFS from t over residual arcs y -> x
template <typename R>
__global__ void csr_bfs_init_kernel(CsrDev<R> g) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += gridDim.x * blockDim.x)
        g.dist[v] = (v == g.t) ? 0 : -1;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        g.frontier[0][0] = g.t;
        g.fcount[0] = 1;
        g.fcount[1] = 0;
    }
}

template <typename R>
__global__ void csr_bfs_level_kernel(CsrDev<R> g, int parity, int level) {
    const int cnt = __ldcg(g.fcount + parity);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const int x = g.frontier[parity][i];
        for (int64_t k = g.ostart[x]; k < g.ostart[x + 1]; k++) {
            const int32_t a = g.oarc[k];
            if (g.res[a ^ 1] <= 0) continue;   // the mate of an out-arc of x is an arc INTO x
            const int32_t y = g.head[a];
            if (y == g.s) continue;            // the source is pre-scanned and never traversed
            if (atomicCAS(g.dist + y, -1, level + 1) == -1)
                g.frontier[parity ^ 1][atomicAdd(g.fcount + (parity ^ 1), 1)] = y;
        }
    }
}

// gap_relabel + marking; counts active nodes (excess > 0, reached)
template <typename R>
__global__ void csr_finalize_kernel(CsrDev<R> g, unsigned long long *acc /* [0] active [1] marked excess */) {
    long long active = 0, mex = 0;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += gridDim.x * blockDim.x) {
        if (v == g.s) continue;
        const int32_t d = g.dist[v];
        if (v == g.t) { g.h[v] = 0; continue; }
        const long long e = (long long)g.ex[v];
        if (d >= 0) {
            g.h[v] = d;
            active += e > 0;
        } else {
            if (g.h[v] < g.n) g.h[v] = g.n;
            if (!g.marked[v]) { g.marked[v] = 1; mex += e; }
        }
    }
    if (active) atomicAdd(acc + 0, (unsigned long long)active);
    if (mex) atomicAdd(acc + 1, (unsigned long long)mex);
}

// cut: residual reach from {s} U {v != t : e(v) > 0}
template <typename R>
__global__ void csr_cut_init_kernel(CsrDev<R> g) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < g.n; v += gridDim.x * blockDim.x)
        g.cut[v] = (v == g.s || (v != g.t && (long long)g.ex[v] > 0)) ? 1 : 0;
}

template <typename R>
__global__ void csr_cut_pass_kernel(CsrDev<R> g, int32_t *changed) {
    bool ch = false;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < g.n; x += gridDim.x * blockDim.x) {
        if (!__ldcg(g.cut + x)) continue;
        for (int64_t k = g.ostart[x]; k < g.ostart[x + 1]; k++) {
            const int32_t a = g.oarc[k];
            if (g.res[a] > 0) {
                const int32_t y = g.head[a];
                if (!__ldcg(g.cut + y)) { g.cut[y] = 1; ch = true; }
            }
        }
    }
    if (__syncthreads_or(ch) && threadIdx.x == 0) *changed = 1;
}

}  // namespace

namespace {

template <typename R>
int csr_solve(const char *fn, int32_t n, int32_t s, int32_t t, int64_t m2, const int64_t *ostart,
              const int32_t *oarc, const int32_t *head, const R *cap, int32_t cycle_budget, int32_t flags,
              int64_t *flow_out, uint8_t *cut_out, R *res_out, int64_t *ex_out, fm_stats *stats) {
    if (n < 2 || s < 0 || s >= n || t < 0 || t >= n || s == t || m2 < 0 || (m2 & 1) || !ostart ||
        (m2 > 0 && (!oarc || !head || !cap)) || cycle_budget < 1 || m2 > (int64_t)INT32_MAX) {
        fm_set_error("%s: invalid argument", fn);
        return FM_INVALID_ARG;
    }
    if (fm_device_count() == 0) { fm_set_error("no CUDA device"); return FM_NO_DEVICE; }
    fm_stats st{};
    cudaStream_t stream;
    FM_CHECK_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    CsrDev<R> g{};
    g.n = n; g.s = s; g.t = t; g.m2 = m2;
    const size_t am = (size_t)std::max<int64_t>(m2, 1);
    int64_t *d_ostart = nullptr;
    int32_t *d_oarc = nullptr, *d_head = nullptr;
    R *d_cap = nullptr;
    unsigned long long *acc = nullptr;
    int32_t *flags_d = nullptr;
    int rc = FM_OK;
#define FM_CSR_TRY(call) do { if ((call) != cudaSuccess) { fm_set_error("%s: %s", #call, cudaGetErrorString(cudaGetLastError())); rc = FM_CUDA_ERROR; goto done; } } while (0)
    FM_CSR_TRY(cudaMalloc((void **)&d_ostart, sizeof(int64_t) * ((size_t)n + 1)));
    FM_CSR_TRY(cudaMalloc((void **)&d_oarc, sizeof(int32_t) * am));
    FM_CSR_TRY(cudaMalloc((void **)&d_head, sizeof(int32_t) * am));
    FM_CSR_TRY(cudaMalloc((void **)&d_cap, sizeof(R) * am));
    FM_CSR_TRY(cudaMalloc((void **)&g.res, sizeof(R) * am));
    FM_CSR_TRY(cudaMalloc((void **)&g.ex, sizeof(unsigned long long) * n));
    FM_CSR_TRY(cudaMalloc((void **)&g.h, sizeof(int32_t) * n));
    FM_CSR_TRY(cudaMalloc((void **)&g.dist, sizeof(int32_t) * n));
    FM_CSR_TRY(cudaMalloc((void **)&g.marked, n));
    FM_CSR_TRY(cudaMalloc((void **)&g.cut, n));
    FM_CSR_TRY(cudaMalloc((void **)&g.frontier[0], sizeof(int32_t) * n));
    FM_CSR_TRY(cudaMalloc((void **)&g.frontier[1], sizeof(int32_t) * n));
    FM_CSR_TRY(cudaMalloc((void **)&g.fcount, sizeof(int32_t) * 4));
    FM_CSR_TRY(cudaMalloc((void **)&acc, sizeof(unsigned long long) * 8));
    FM_CSR_TRY(cudaMalloc((void **)&flags_d, sizeof(int32_t) * 4));
    cudaEventRecord(t0, stream);
    FM_CSR_TRY(cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * 8, stream));   // op counters
    FM_CSR_TRY(cudaMemcpyAsync(d_ostart, ostart, sizeof(int64_t) * ((size_t)n + 1), cudaMemcpyHostToDevice, stream));
    if (m2 > 0) {
        FM_CSR_TRY(cudaMemcpyAsync(d_oarc, oarc, sizeof(int32_t) * m2, cudaMemcpyHostToDevice, stream));
        FM_CSR_TRY(cudaMemcpyAsync(d_head, head, sizeof(int32_t) * m2, cudaMemcpyHostToDevice, stream));
        FM_CSR_TRY(cudaMemcpyAsync(d_cap, cap, sizeof(R) * m2, cudaMemcpyHostToDevice, stream));
    }
    g.ostart = d_ostart; g.oarc = d_oarc; g.head = d_head; g.cap = d_cap;
    {
        const int nb = std::max(1, std::min((int)((std::max<int64_t>(n, m2) + 255) / 256), 148 * 8));
        const int nbn = std::max(1, std::min((n + 255) / 256, 148 * 8));
        csr_init_kernel<<<nb, 256, 0, stream>>>(g);
        csr_preflow_kernel<<<1, 256, 0, stream>>>(g);
        st.launches += 2;
        long long h_acc[2] = {0, 0};
        int32_t h_flag = 0;
        const int cap_passes = std::max(1, std::min(cycle_budget, 64));
        // the coordinator: global relabel first, then rounds (maxflow_par.py:195-229)
        for (int round = -1;; round++) {
            // ---- global relabel + gap + marking
            csr_bfs_init_kernel<<<nbn, 256, 0, stream>>>(g);
            int parity = 0, level = 0;
            for (;; level++) {
                int32_t cnt = 0;
                FM_CSR_TRY(cudaMemcpyAsync(&cnt, g.fcount + parity, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
                FM_CSR_TRY(cudaStreamSynchronize(stream));
                if (cnt == 0) break;
                FM_CSR_TRY(cudaMemsetAsync(g.fcount + (parity ^ 1), 0, sizeof(int32_t), stream));
                csr_bfs_level_kernel<<<std::max(1, std::min((cnt + 255) / 256, 148 * 8)), 256, 0, stream>>>(g, parity, level);
                st.launches++;
                st.bfs_sweeps++;
                parity ^= 1;
            }
            st.bfs_levels = std::max<int64_t>(st.bfs_levels, level);
            FM_CSR_TRY(cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * 2, stream));
            csr_finalize_kernel<<<nbn, 256, 0, stream>>>(g, acc);
            st.launches += 2;
            FM_CSR_TRY(cudaMemcpyAsync(h_acc, acc, sizeof(unsigned long long) * 2, cudaMemcpyDeviceToHost, stream));
            FM_CSR_TRY(cudaStreamSynchronize(stream));
            if (round >= 0) st.rounds++;
            if (h_acc[0] == 0) break;
            // ---- lock-free passes until an idle pass or the budget
            int done = 0;
            while (done < cap_passes) {
                FM_CSR_TRY(cudaMemsetAsync(flags_d, 0, sizeof(int32_t), stream));
                csr_pass_kernel<<<nbn, 256, 0, stream>>>(g, flags_d, acc + 2);
                st.launches++;
                done++;
                FM_CSR_TRY(cudaMemcpyAsync(&h_flag, flags_d, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
                FM_CSR_TRY(cudaStreamSynchronize(stream));
                if (!h_flag) break;
            }
            st.pr_sweeps += done;
        }
        // ---- cut
        csr_cut_init_kernel<<<nbn, 256, 0, stream>>>(g);
        for (;;) {
            FM_CSR_TRY(cudaMemsetAsync(flags_d, 0, sizeof(int32_t), stream));
            csr_cut_pass_kernel<<<nbn, 256, 0, stream>>>(g, flags_d);
            st.cut_sweeps++;
            st.launches++;
            FM_CSR_TRY(cudaMemcpyAsync(&h_flag, flags_d, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
            FM_CSR_TRY(cudaStreamSynchronize(stream));
            if (!h_flag) break;
        }
        unsigned long long ops[2] = {0, 0};
        FM_CSR_TRY(cudaMemcpyAsync(ops, acc + 2, sizeof(unsigned long long) * 2, cudaMemcpyDeviceToHost, stream));
        long long et = 0;
        FM_CSR_TRY(cudaMemcpyAsync(&et, g.ex + t, sizeof(long long), cudaMemcpyDeviceToHost, stream));
        if (cut_out) FM_CSR_TRY(cudaMemcpyAsync(cut_out, g.cut, (size_t)n, cudaMemcpyDeviceToHost, stream));
        if (res_out && m2 > 0) FM_CSR_TRY(cudaMemcpyAsync(res_out, g.res, sizeof(R) * m2, cudaMemcpyDeviceToHost, stream));
        if (ex_out) FM_CSR_TRY(cudaMemcpyAsync(ex_out, g.ex, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, stream));
        cudaEventRecord(t1, stream);
        FM_CSR_TRY(cudaStreamSynchronize(stream));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, t0, t1);
        st.ms_total = ms;
        st.pushes = (int64_t)ops[0];
        st.relabels = (int64_t)ops[1];
        if (flow_out) *flow_out = et;
    }
    (void)flags;
done:
#undef FM_CSR_TRY
    cudaFree(d_ostart); cudaFree(d_oarc); cudaFree(d_head); cudaFree(d_cap);
    cudaFree(g.res); cudaFree(g.ex); cudaFree(g.h); cudaFree(g.dist); cudaFree(g.marked); cudaFree(g.cut);
    cudaFree(g.frontier[0]); cudaFree(g.frontier[1]); cudaFree(g.fcount); cudaFree(acc); cudaFree(flags_d);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    cudaStreamDestroy(stream);
    if (stats) *stats = st;
    return rc;
}

}  // namespace

extern "C" int fm_csr_solve(int32_t n, int32_t s, int32_t t, int64_t m2, const int64_t *ostart,
                            const int32_t *oarc, const int32_t *head, const int32_t *cap,
                            int32_t cycle_budget, int32_t flags, int64_t *flow_out,
                            uint8_t *cut_out, int32_t *res_out, int64_t *ex_out, fm_stats *stats) {
    return csr_solve<int32_t>("fm_csr_solve", n, s, t, m2, ostart, oarc, head, cap, cycle_budget, flags,
                              flow_out, cut_out, res_out, ex_out, stats);
}

extern "C" int fm_csr_solve64(int32_t n, int32_t s, int32_t t, int64_t m2, const int64_t *ostart,
                              const int32_t *oarc, const int32_t *head, const int64_t *cap,
                              int32_t cycle_budget, int32_t flags, int64_t *flow_out,
                              uint8_t *cut_out, int64_t *res_out, int64_t *ex_out, fm_stats *stats) {
    // int64 residuals; the caller keeps every capacity below 2^62 and the source's total
    // out-capacity below 2^63 so no residual or excess can leave int64
    if (m2 > 0 && cap) {
        long long src = 0;
        for (int64_t i = 0; i < m2; i++) {
            if (cap[i] < 0 || cap[i] >= (1ll << 62)) {
                fm_set_error("fm_csr_solve64: capacity of slot %lld outside [0, 2^62)", (long long)i);
                return FM_INVALID_ARG;
            }
        }
        if (ostart && s >= 0 && s < n && head && oarc) {
            for (int64_t i = ostart[s]; i < ostart[s + 1]; i++) {
                if (i < 0 || i >= m2 || oarc[i] < 0 || oarc[i] >= m2) break;
                if (__builtin_add_overflow(src, (long long)cap[oarc[i]], &src)) {
                    fm_set_error("fm_csr_solve64: total capacity out of the source exceeds 2^63-1");
                    return FM_INVALID_ARG;
                }
            }
        }
    }
    return csr_solve<long long>("fm_csr_solve64", n, s, t, m2, ostart, oarc, head, (const long long *)cap,
                                cycle_budget, flags, flow_out, cut_out, (long long *)res_out, ex_out, stats);
}

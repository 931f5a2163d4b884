"""Benchmark of the grid max-flow / assignment hot path (one JSON line on rank 0).

Workload (N = 1): BASELINE.json's metric "grid max-flow Medges/s & solve ms at
4096^2; assignment solve ms at n=4096".  A step = one complete max-flow + min-cut
solve of a 4096 x 4096 4-connected grid (generator G), inputs
resident in HBM.  value = Medges/s = E_grid / solve seconds, E_grid =
2(2HW - H - W) + 2HW.  The n = 4096 assignment solve, config 2 (2048^2
segmentation) and config 3's grid on one GPU are reported beside it.  e2e = the K
steps from pinned host planes through one pipelined hybrid_solve_batch call (each
step's six-plane H2D and cut D2H inside the timed region, overlapped with the
neighbouring steps' solves), the generator's capacities (0..100) sent as uint8
planes and widened on the device; e2e.int32_batch = the same call with int32 planes;
e2e.single_call = one synchronous hybrid_solve per step with int32 planes.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1): BASELINE config 3 -- ONE 8192 x 8192 grid (generator G, seed
8192) strong-scaled in N row bands, one band per GPU (paper_1110_6231_b200.bands:
neighbours reached through CUDA IPC peer memory, coordinator agreement through a
shared-memory all-gather); flow and minimal-cut hash are asserted equal to the
single-GPU solve's at every N.  Time = max over ranks of the bands' device time.
``--impl reference`` times the reference algorithm's CPU port (oracle/, C
restatement of hybrid_solve with real threads) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid max-flow Medges/s & solve ms at 4096²; assignment solve ms at n=4096"
UNIT = "Medges/s"


def e_grid(H: int, W: int) -> int:
    return 2 * (2 * H * W - H - W) + 2 * H * W


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampler for the timed region (the recipe's clocks line)."""

    def __init__(self, device: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 8 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) > 8:
                for k, v in zip(names, r[5:9]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(k)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the committed ncu capture (profiles/ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        # the push kernel's capture is keyed by its instance (pr_list_kernel<packed> on
        # generator G, whose pair sums fit the packed 16-bit residuals)
        d = t[kernel] if kernel in t else next(v for k, v in t.items() if k.startswith(kernel + "<"))
        return round(d["dram_bytes_per_launch"]), d.get("source")
    except Exception:
        return None, None


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline_grid(threads: int):
    """The reference's grid path restated in C (oracle/), timed on this box's host cores
    (SURVEY.md 8d): hybrid_solve with every host thread on a bounded 512^2 sample (the
    line's value), the sequential solver on 512^2 and 1024^2, the CPU model."""
    import oracle
    from paper_1110_6231_b200 import generators as G

    S = 512
    caps = G.grid_random(S, S, S)
    t = time.perf_counter()
    d = oracle.grid_maxflow(*caps, solver="hybrid", worker_count=threads)
    dt = time.perf_counter() - t
    t = time.perf_counter()
    d1 = oracle.grid_maxflow(*caps, solver="seq")
    dts = time.perf_counter() - t
    assert d["value"] == d1["value"]
    caps = G.grid_random(1024, 1024, 1024)
    t = time.perf_counter()
    d2 = oracle.grid_maxflow(*caps, solver="seq")
    dt2 = time.perf_counter() - t
    return {"value": round(e_grid(S, S) / dt / 1e6, 4), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"generator G {S}x{S} seed {S}: hybrid_solve port (oracle/fm_oracle.c, "
                      f"{threads} threads, cycle_budget 7000) solve {dt:.2f}s",
            "cpu_model": cpu_model(), "os_cpu_count": os.cpu_count(),
            "seq_port": {"512": {"medges_per_s": round(e_grid(S, S) / dts / 1e6, 4), "solve_s": round(dts, 3)},
                         "1024": {"medges_per_s": round(e_grid(1024, 1024) / dt2 / 1e6, 4), "solve_s": round(dt2, 3),
                                  "flow": d2["value"]}},
            "note": "the reference itself is pure Python and GIL-bound (effectively 1 core); "
                    "its sequential solver is the fastest CPU path (SURVEY.md 6)"}


def cpu_baseline_assign():
    """solve_assignment(mode="seq") and (mode="par", worker_count=1) restated in C
    (oracle/) at n = 1024 (BASELINE config 4), both weight ranges.  n = 4096 is not run
    by default: the seq port takes 30-70 s per instance on these hosts (--cpu-assign-4096)."""
    import oracle
    from paper_1110_6231_b200 import generators as G

    out = {}
    for M in (100, 10000):
        w = G.assignment_reference(1024, M, 1024)
        for mode in ("seq", "par"):
            t = time.perf_counter()
            d = oracle.assign(1024, matrix=w, mode=mode)
            out[f"n1024_M{M}_{mode}"] = {"solve_ms": round(1000 * (time.perf_counter() - t), 1),
                                         "objective": d["objective"], "cores": 1}
    return out


def cpu_baseline_assign_4096():
    import oracle
    from paper_1110_6231_b200 import generators as G

    out = {}
    for name, w in (("optical_flow", G.assignment_optical_flow(4096, 4096)),
                    ("reference_generate_M100", G.assignment_reference(4096, 100, 4096))):
        t = time.perf_counter()
        d = oracle.assign(4096, matrix=w, mode="seq")
        out[f"n4096_{name}_seq"] = {"solve_ms": round(1000 * (time.perf_counter() - t), 1),
                                    "objective": d["objective"], "cores": 1}
    return out


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    import oracle
    from paper_1110_6231_b200 import generators as G

    S = args.ref_size
    caps = G.grid_random(S, S, S)
    for _ in range(args.warmup):
        oracle.grid_maxflow(*caps, solver="hybrid", worker_count=threads)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        d = oracle.grid_maxflow(*caps, solver="hybrid", worker_count=threads)
        times.append(time.perf_counter() - t)
    ms = 1000 * statistics.mean(times)
    v = e_grid(S, S) / (ms / 1000) / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak" if ws == 1 else "strong", "vs_baseline": None,
            "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"grid max-flow + min-cut, generator G {S}x{S} seed {S} "
                                   f"(bounded CPU sample of the GPU workload)", "flow": d["value"]},
            "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"hybrid_solve restated in C (oracle/fm_oracle.c), {threads} threads, "
                                       f"generator G {S}x{S}", "cpu_model": cpu_model()},
            "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def grid_roofline(agg: dict, steps: int, ms_total: float, peak: float, peak_src: str, scope: str):
    """Roofline of pr_list_kernel (the dominant kernel) per SURVEY.md 8d: algorithmic
    bytes per launch = 32 B per visited pixel (tile visits x 1024 px: 7 state words read
    + the height written) + 16 B per push, over the mean launch duration (CUDA events
    around launch batches on the solve stream).  The builder's per-visit accounting
    (60 B/px: every plane read and written back + the 512 B halo) is reported beside."""
    launches = max(1, agg.get("pr_launches", 0))
    tiles, pushes = agg.get("pr_tiles", 0), agg.get("pushes", 0)
    pr_ms = agg.get("ms_pr_kern", 0.0)
    dur = pr_ms / launches
    b8d = (tiles * 1024 * 32 + pushes * 16) / launches
    bvis = tiles * (1024 * 60 + 512) / launches
    ach = b8d / (dur / 1000.0) / 1e9 if dur > 0 else 0.0
    achv = bvis / (dur / 1000.0) / 1e9 if dur > 0 else 0.0
    traffic, traffic_src = ncu_traffic("pr_list_kernel")
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
            "traffic": traffic, "traffic_source": traffic_src, "kernel": "pr_list_kernel",
            "peak_source": peak_src, "bytes_per_launch": int(b8d),
            "bytes_rule": "SURVEY 8d: 32 B x visited pixels (tile visits x 1024) + 16 B x pushes",
            "per_visit_accounting": {"bytes_per_launch": int(bvis), "achieved": round(achv, 1),
                                     "frac": round(achv / peak, 4),
                                     "rule": "60 B/px per tile visit (8 planes read, 7 written) + 512 B halo"},
            "launch_ms": round(dur, 5), "launches_per_solve": launches // max(1, steps),
            "kernel_share_of_step": round(pr_ms / max(1e-9, ms_total), 3), "scope": scope}


def assign_roofline(st: dict, n: int, ms: float, peak: float):
    """SURVEY.md 8d assignment bytes: each op (push or relabel) scans a weight row (4n B)
    + flow / fixed bits (n/4 B); each refine reads the matrix twice (row-min preamble +
    arc fix, 8 n^2 B); over the whole solve's device time."""
    ops = st.get("pushes", 0) + st.get("relabels", 0)
    b = ops * (4 * n + n // 4) + st.get("refines", 0) * 8 * n * n
    ach = b / (ms / 1000.0) / 1e9
    return {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
            "bytes_per_solve": int(b), "ops": ops, "refines": st.get("refines", 0),
            "scope": "whole solve (every assignment kernel)"}


def cut_sha(cut_np) -> str:
    import hashlib

    return hashlib.sha256(np.packbits(np.asarray(cut_np, dtype=bool).reshape(-1)).tobytes()).hexdigest()[:16]


# BASELINE config 3 (generator G 8192^2, seed 8192) solved on one GPU: flow certified by
# tests/test_grid_gpu.py::test_certificate_at_8192; the banded run must reproduce both
FLOW_8192 = 3318000345


def run_banded(args, ws, rank, local):
    """N > 1: config 3 strong-scaled -- one 8192^2 grid, one row band per rank."""
    import torch
    import torch.distributed as dist

    from paper_1110_6231_b200 import bands as B
    from paper_1110_6231_b200 import generators as G

    S = args.banded_size
    H = W = S
    ndev = max(1, torch.cuda.device_count())
    colocated = max(1, -(-ws // ndev)) if args.dist_backend == "gloo" else 1
    caps = G.grid_random(H, W, S)
    band = B.DistBand(H, W, rank, ws, local, colocated=colocated)
    rows, above, below = B.band_planes(caps, band.r0, band.r1)
    del caps
    dev = torch.device("cuda", local)
    rows_d = [torch.from_numpy(r).to(dev) for r in rows]
    above_d = torch.from_numpy(above).to(dev) if above is not None else None
    below_d = torch.from_numpy(below).to(dev) if below is not None else None
    Hb = band.r1 - band.r0
    cut_d = torch.empty((Hb, W), dtype=torch.uint8, device=dev)

    def reduce(vals, op):
        t = torch.tensor(vals, dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=op)
        return t.tolist()

    flows = set()
    for _ in range(args.warmup):
        f, _, _ = band.solve(rows_d, above_d, below_d, cut_out=cut_d)
        flows.add(f)
    clocks = Clocks(local)
    dist.barrier()
    torch.cuda.synchronize()
    agg, dev_ms, t0 = {}, 0.0, time.perf_counter()
    agg_res2 = 0
    for _ in range(args.steps):
        f, _, st = band.solve(rows_d, above_d, below_d, cut_out=cut_d)
        flows.add(f)
        dev_ms += st["ms_total"]
        agg_res2 += int(st["reserved"][2])
        for k, v in st.items():
            if isinstance(v, (int, float)):
                agg[k] = agg.get(k, 0) + v
    torch.cuda.synchronize()
    wall_ms = 1000 * (time.perf_counter() - t0)
    dist.barrier()
    clk = clocks.stop()
    dev_max, wall_max = reduce([dev_ms, wall_ms], dist.ReduceOp.MAX)
    ms_step = dev_max / args.steps
    assert len(flows) == 1, f"flow changed across steps: {flows}"
    flow = flows.pop()
    # the whole grid's minimal cut, gathered in band order, against the single-GPU solve
    packed = np.packbits(cut_d.cpu().numpy().astype(bool).reshape(-1))
    parts = [None] * ws
    dist.all_gather_object(parts, packed.tobytes())
    import hashlib

    sha = hashlib.sha256(b"".join(parts)).hexdigest()[:16]
    value = e_grid(H, W) / (ms_step / 1000.0) / 1e6
    # e2e: this rank's rows from pinned host memory -> solve -> cut rows back to the host
    e2e = None
    if not args.no_e2e:
        pin = [torch.from_numpy(r).pin_memory() for r in rows]
        ab = [torch.from_numpy(a).pin_memory() if a is not None else None for a in (above, below)]
        cut_h = torch.empty((Hb, W), dtype=torch.uint8).pin_memory()
        times = []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            f, _, _ = band.solve(pin, ab[0], ab[1], cut_out=cut_h)
            times.append(time.perf_counter() - t0)
            assert f == flow
        (tt,) = reduce([statistics.mean(times)], dist.ReduceOp.MAX)
        e2e = {"value": round(e_grid(H, W) / tt / 1e6, 3), "unit": UNIT,
               "h2d_bytes_per_step": 6 * 4 * H * W + 8 * W * (ws - 1), "d2h_bytes_per_step": H * W,
               "ms_per_step": round(1000 * tt, 3),
               "api": "paper_1110_6231_b200.bands.DistBand.solve(pinned host rows) on every rank"}
    launches_all = reduce([agg.get("launches", 0)], dist.ReduceOp.SUM)[0]
    peak, peak_src = measured_peak_hbm()
    roof = grid_roofline(agg, args.steps, dev_ms, peak, peak_src, "rank 0 band, timed solves")
    if rank == 0:
        if S == 8192:
            assert flow == FLOW_8192, f"banded flow {flow} != single-GPU {FLOW_8192}"
        line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
                "config": {"workload": f"BASELINE config 3: grid max-flow + min-cut {H}x{W} 4-connected, generator G "
                                       f"seed {S}, strong-scaled in {ws} row bands (one per GPU)",
                           "E_grid": e_grid(H, W), "flow": flow, "cut_sha16": sha,
                           "parallelism": f"row bands x{ws} (peer memory via CUDA IPC; shared-memory coordinator)",
                           "band_rows": [list(sp) for sp in band.spans],
                           "l2": "inputs larger than L2", "cycle_budget": 7000,
                           "time": "device time of the bands' solves (CUDA events), max over ranks",
                           "wall_ms_per_step_max": round(wall_max / args.steps, 3)},
                "roofline": roof, "cpu_baseline": None, "e2e": e2e,
                "gpu_launches": int(launches_all), "clocks": clk,
                "coordinator": {"agreements_per_solve": int(agg_res2 // args.steps),
                                "what": "shared-memory all-gathers of <= 4 int64 (per push batch and per relabel); "
                                        "no data-path messages: boundary rows, inboxes and ring queues are peer memory"},
                "per_solve_rank0": {k: (round(v / args.steps, 3) if isinstance(v, float) else v // args.steps)
                                    for k, v in agg.items() if k in ("pushes", "relabels", "rounds", "launches",
                                                                    "pr_launches", "pr_tiles", "ms_total", "ms_push",
                                                                    "ms_bfs", "ms_cut", "ms_pr_kern", "ms_bfs_kern")}}
        print(json.dumps(line), flush=True)
    band.close()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--banded-size", type=int, default=8192, help="N > 1: side of the banded grid (config 3)")
    ap.add_argument("--assign-n", type=int, default=4096)
    ap.add_argument("--ref-size", type=int, default=512)
    ap.add_argument("--bfs-interval", type=int, default=0)
    ap.add_argument("--no-assign", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-assign-4096", action="store_true", help="also time the n=4096 assignment CPU port (~1 min)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-big", action="store_true", help="skip the 8192^2 single-GPU solve")
    ap.add_argument("--no-virtual-bands", action="store_true",
                    help="skip the 2-band solve on one GPU (its bands' ring launches must run concurrently, "
                         "which a kernel-serialising profiler prevents)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: run the banded path with several ranks sharing fewer GPUs")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch

    ws, rank, local = dist_env()
    if args.dist_backend == "gloo":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        return run_banded(args, ws, rank, local)
    import paper_1110_6231_b200 as fmb
    from paper_1110_6231_b200 import generators as G

    S = args.size
    caps_h = [np.ascontiguousarray(c) for c in G.grid_random(S, S, S)]
    caps_d = [torch.from_numpy(c).cuda() for c in caps_h]
    cut_d = torch.empty((S, S), dtype=torch.uint8, device="cuda")
    solver = fmb.GridSolver(S, S, device=local)
    stream = torch.cuda.current_stream()

    def step():
        return solver.solve_device(caps_d, 7000, args.bfs_interval, cut_out=cut_d, stream=stream)

    flows = set()
    for _ in range(args.warmup):
        f, _ = step()
        flows.add(f)
    clocks = Clocks(local)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    agg = {}
    ev0.record(stream)
    for _ in range(args.steps):
        f, st = step()
        flows.add(f)
        for k, v in st.items():
            if isinstance(v, (int, float)):
                agg[k] = agg.get(k, 0) + v
        agg["bfs_tile_visits"] = agg.get("bfs_tile_visits", 0) + int(st["reserved"][0])
    ev1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms_total = ev0.elapsed_time(ev1)
    ms_step = ms_total / args.steps
    value = e_grid(S, S) / (ms_step / 1000.0) / 1e6
    assert len(flows) == 1, f"flow changed across steps: {flows}"
    flow = flows.pop()
    HW = S * S
    peak, peak_src = measured_peak_hbm()
    K = args.steps
    roofline = grid_roofline(agg, K, ms_total, peak, peak_src, "timed solves")

    # end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        pinned = [torch.from_numpy(c).pin_memory().numpy() for c in caps_h]
        net = fmb.build_grid_network(*pinned)
        fmb.hybrid_solve(net)  # warm (workspace allocation)
        times = []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = fmb.hybrid_solve(net)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            assert rep.objective == flow
        t_single = statistics.mean(times)
        # the same K steps as ONE pipelined call (a stream of images): each step still
        # copies its six planes in and its cut out, overlapped with the previous /
        # next step's solve
        def batch_time(batch_net):
            nets = [batch_net] * args.steps
            fmb.hybrid_solve_batch(nets[:2])  # warm (second input set, stages, copy streams)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            reps = fmb.hybrid_solve_batch(nets)
            torch.cuda.synchronize()
            assert all(r.objective == flow and r.cut is not None for r in reps)
            return (time.perf_counter() - t0) / args.steps
        t_b32 = batch_time(net)
        # the generator's capacities (0..100) fit uint8: the planes cross PCIe as uint8
        # (100 MB instead of 402 MB per step) and are widened to int32 on the device
        assert all(int(c.max()) <= 255 for c in caps_h)
        pinned8 = [torch.from_numpy(c.astype(np.uint8)).pin_memory().numpy() for c in caps_h]
        net8 = fmb.build_grid_network(*pinned8)
        assert net8.narrow_bytes == 1
        tt = batch_time(net8)
        e2e = {"value": round(e_grid(S, S) / tt / 1e6, 3), "unit": UNIT,
               "h2d_bytes_per_step": 6 * HW, "d2h_bytes_per_step": HW + 8,
               "ms_per_step": round(1000 * tt, 3),
               "api": f"paper_1110_6231_b200.hybrid_solve_batch([build_grid_network(*uint8 pinned host planes)] x {args.steps}): "
                      "one call; the capacities (0..100) cross PCIe as uint8 and are widened to int32 on the device; "
                      "step k+1's H2D and step k-1's cut D2H overlap step k's solve",
               "int32_batch": {"value": round(e_grid(S, S) / t_b32 / 1e6, 3), "unit": UNIT,
                               "ms_per_step": round(1000 * t_b32, 3), "h2d_bytes_per_step": 6 * 4 * HW,
                               "api": "the same batch call with int32 pinned host planes"},
               "single_call": {"value": round(e_grid(S, S) / t_single / 1e6, 3), "unit": UNIT,
                               "ms_per_step": round(1000 * t_single, 3), "h2d_bytes_per_step": 6 * 4 * HW,
                               "api": "paper_1110_6231_b200.hybrid_solve(build_grid_network(*int32 pinned host planes)), "
                                      "one synchronous call per step"}}

    # the other grid config of BASELINE.json on one GPU: 2048^2 segmentation (config 2)
    seg = None
    if not args.no_assign:
        cs = [torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in G.grid_segmentation(2048, 2048, 2048)]
        cut2 = torch.empty((2048, 2048), dtype=torch.uint8, device="cuda")
        sv = fmb.GridSolver(2048, 2048, device=local)
        for _ in range(3):
            f2, _ = sv.solve_device(cs, cut_out=cut2, stream=stream)
        tms = []
        for _ in range(max(3, args.steps)):
            f2, st2 = sv.solve_device(cs, cut_out=cut2, stream=stream)
            tms.append(st2["ms_total"])
        sv.close()
        ms2 = statistics.mean(tms)
        seg = {"workload": "generator S 2048x2048 seed 2048 (synthetic segmentation energy)", "flow": f2,
               "solve_ms": round(ms2, 3), "medges_per_s": round(e_grid(2048, 2048) / (ms2 / 1000) / 1e6, 1),
               "rounds": st2["rounds"], "pushes": st2["pushes"], "relabels": st2["relabels"]}

    # config 3's grid (8192^2, generator G seed 8192) on this single GPU: the N=1 point
    # of the row-band strong-scaling series (flow + cut hash the banded runs must match)
    big = None
    if not args.no_assign and not args.no_big:
        B8 = 8192
        cb = [torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in G.grid_random(B8, B8, B8)]
        cut3 = torch.empty((B8, B8), dtype=torch.uint8, device="cuda")
        sv = fmb.GridSolver(B8, B8, device=local)
        sv.solve_device(cb, cut_out=cut3, stream=stream)
        tms = []
        for _ in range(2):
            f3, st3 = sv.solve_device(cb, cut_out=cut3, stream=stream)
            tms.append(st3["ms_total"])
        sv.close()
        ms3 = statistics.mean(tms)
        big = {"workload": "generator G 8192x8192 seed 8192 on 1 GPU (config 3, N=1)", "flow": f3,
               "cut_sha16": cut_sha(cut3.cpu().numpy()),
               "solve_ms": round(ms3, 3), "medges_per_s": round(e_grid(B8, B8) / (ms3 / 1000) / 1e6, 1),
               "rounds": st3["rounds"], "pushes": st3["pushes"], "relabels": st3["relabels"]}
        # the same grid in 2 row bands on this GPU (virtual bands: the banded code path,
        # one host thread per band) -- identical flow and cut
        from paper_1110_6231_b200 import bands as Bd

    if big is not None and not args.no_virtual_bands:
        grp = Bd.BandGroup(B8, B8, 2, [local, local])
        grp.solve(cb, cut_out=cut3)
        tms = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fb, _, stb = grp.solve(cb, cut_out=cut3)
            tms.append(1000 * (time.perf_counter() - t0))
        grp.close()
        big["two_virtual_bands"] = {"flow": fb, "cut_sha16": cut_sha(cut3.cpu().numpy()),
                                    "solve_ms_wall": round(statistics.mean(tms), 3),
                                    "device_ms_max_band": round(stb["ms_total"], 3), "rounds": stb["rounds"]}
        assert fb == f3 and big["two_virtual_bands"]["cut_sha16"] == big["cut_sha16"]
    if big is not None:
        del cb, cut3

    # assignment n = 4096 (single GPU; replicas only)
    assign = None
    if not args.no_assign:
        n = args.assign_n
        assign = {}
        asolver = fmb.AssignmentSolver(n, device=local)
        cases = [("optical_flow", G.assignment_optical_flow(n, n)),
                 ("reference_generate_M100", G.assignment_reference(n, 100, n)),
                 ("reference_generate_M10000", G.assignment_reference(n, 10000, n))]
        for name, w in cases:
            wd = torch.from_numpy(w).cuda()
            for _ in range(2):
                asolver.solve_device(wd, stream=stream)
            ts = []
            for _ in range(max(1, args.steps)):
                torch.cuda.synchronize()
                a0 = torch.cuda.Event(enable_timing=True)
                a1 = torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                obj, m, _, st = asolver.solve_device(wd, stream=stream)
                a1.record(stream)
                torch.cuda.synchronize()
                ts.append(a0.elapsed_time(a1))
            assert sorted(m.tolist()) == list(range(n))
            wp = torch.from_numpy(w).pin_memory().numpy()
            fmb.solve_assignment(wp)  # workspace allocation outside the timed call
            t0 = time.perf_counter()
            rep, _ = fmb.solve_assignment(wp)
            e2e_ms = 1000 * (time.perf_counter() - t0)
            assert rep.objective == obj
            ms_a = statistics.mean(ts)
            assign[name] = {"solve_ms": round(ms_a, 3), "objective": obj,
                            "e2e_ms": round(e2e_ms, 3), "pushes": st["pushes"], "relabels": st["relabels"],
                            "rounds": st["rounds"], "tail_rounds": st["pr_sweeps"], "refines": st["refines"],
                            "roofline": assign_roofline(st, n, ms_a, peak)}
        asolver.close()
        # config 4: dense n = 1024 (reference generator, w <= 100 and w <= 10^4)
        a1 = fmb.AssignmentSolver(1024, device=local)
        for M in (100, 10000):
            wd = torch.from_numpy(G.assignment_reference(1024, M, 1024)).cuda()
            a1.solve_device(wd, stream=stream)
            obj, m, _, st = a1.solve_device(wd, stream=stream)
            assign[f"n1024_reference_generate_M{M}"] = {"solve_ms": round(st["ms_total"], 3), "objective": obj,
                                                          "pushes": st["pushes"], "relabels": st["relabels"]}
        a1.close()

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline_grid(os.cpu_count() or 1)
        if assign is not None:
            ca = cpu_baseline_assign()
            if args.cpu_assign_4096:
                ca.update(cpu_baseline_assign_4096())
            for M in (100, 10000):
                g = assign.get(f"n1024_reference_generate_M{M}")
                if g:
                    assert ca[f"n1024_M{M}_seq"]["objective"] == g["objective"]
            cpu["assignment"] = ca
    per = {k: round(v / K, 3) if isinstance(v, float) else v // K for k, v in agg.items()
           if k in ("pushes", "relabels", "rounds", "launches", "pr_sweeps", "pr_tiles", "bfs_sweeps", "bfs_levels",
                    "cut_sweeps", "ms_total", "ms_push", "ms_bfs", "ms_cut", "ms_pr_kern", "ms_bfs_kern",
                    "pr_launches", "bfs_tile_visits")}
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": f"grid max-flow + min-cut {S}x{S} 4-connected, generator G "
                                   f"(numpy PCG64 seed {S}, caps 0..100)",
                       "E_grid": e_grid(S, S), "flow": flow, "parallelism": "single GPU",
                       "l2": "inputs larger than L2 (6 x 64 MiB planes + 40 B/px state)",
                       "cycle_budget": 7000, "bfs_interval": args.bfs_interval},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(agg.get("launches", 0)), "clocks": clk,
            "per_solve": per, "segmentation_2048": seg, "grid_8192_1gpu": big, "assignment_n4096": assign}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

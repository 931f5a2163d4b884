"""Summarise ncu output into profiles/ (run here, on the gpurun_out/ files).

    python scripts/summarize_ncu.py launches gpurun_out/launches.csv > profiles/X_launches.md
    python scripts/summarize_ncu.py full gpurun_out/prof.ncu-rep > profiles/X_full.md
    python scripts/summarize_ncu.py traffic gpurun_out/traffic.csv > profiles/ncu_traffic.json
"""
import re
import collections
import csv
import io
import subprocess
import sys



TEMPLATE_NAMES = {"ring_kernel<0>": "ring_kernel<bfs>", "ring_kernel<1>": "ring_kernel<cut>",
                  "pr_list_kernel<1>": "pr_list_kernel<packed>", "pr_list_kernel<true>": "pr_list_kernel<packed>",
                  "pr_list_kernel<0>": "pr_list_kernel<int32>", "pr_list_kernel<false>": "pr_list_kernel<int32>"}


def kname(raw):
    """Kernel name without namespace, return type or parameters; the instances of the
    ring and push kernels keep a tag (ring_kernel<bfs> / <cut>, pr_list_kernel<packed>)."""
    if raw.strip() == "graph":   # ncu --graph-profiling graph: a push round's while-graph
        return "pr_list_kernel<packed> x round (while-graph)"
    n = raw.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("(bool)", "")
    for k, v in TEMPLATE_NAMES.items():
        if k in n:
            return v
    n = n.split("(")[0]
    n = re.sub(r"<[^<>]*>", "", n)
    return n.replace("void ", "").strip()

def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = kname(r[ki])
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list: {path}\n")
    print("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare shares)\n")
    print("| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {v[0]} | {v[1]:.2f} | {100 * v[1] / tot:.1f}% | {1000 * v[1] / v[0]:.1f} |")
    print(f"\ntotal {tot:.2f} ms over {sum(v[0] for v in agg.values())} launches")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__shared_mem_per_block_static",
        "l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum", "l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "smsp__inst_executed.sum",
        "smsp__average_warp_latency_issue_stalled_barrier.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full: {path}\n")
    ki = h.index("Kernel Name")
    for n, r in enumerate(rows[2:]):
        print(f"## launch {n}: `{r[ki][:90]}`\n\n| metric | value | unit |\n|---|---|---|")
        for w in WANT:
            if w in h:
                print(f"| {w} | {r[h.index(w)]} | {units[h.index(w)]} |")
        print()


def traffic(path):
    """Per-kernel mean DRAM bytes and duration per launch from an ncu --metrics
    dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv log (JSON)."""
    import json
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, ii, mi, vi, ui = (h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"),
                          h.index("Metric Value"), h.index("Metric Unit"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3,
             "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        names[r[ii]] = kname(r[ki])
        per[r[ii]][r[mi]] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    extra = collections.defaultdict(dict)
    for lid, m in per.items():
        a = agg[names[lid]]
        a[0] += 1
        a[1] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a[2] += m.get("gpu__time_duration.sum", 0.0)
        for key in ("l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum",
                    "l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum",
                    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"):
            ex = extra[names[lid]]
            ex[key] = ex.get(key, 0.0) + m.get(key, 0.0)
    out = {}
    for k, v in agg.items():
        d = {"launches": v[0], "dram_bytes_per_launch": v[1] / v[0], "duration_us_per_launch": v[2] / v[0],
             "source": path}
        ex = extra[k]
        if ex:
            sec = v[2] * 1e-6
            d["global_atom_per_launch"] = ex.get("l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum", 0.0) / v[0]
            d["global_red_per_launch"] = ex.get("l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum", 0.0) / v[0]
            d["shared_atom_wavefronts_per_launch"] = ex.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", 0.0) / v[0]
            if sec > 0:
                d["global_atom_red_per_s"] = (ex.get("l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum", 0.0) +
                                              ex.get("l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum", 0.0)) / sec
                d["shared_atom_wavefronts_per_s"] = ex.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", 0.0) / sec
        out[k] = d
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](sys.argv[2])

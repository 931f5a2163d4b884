"""Race hunting for the generic-graph (CSR) GPU path: random graphs vs the oracle's
sequential solver (value) and seeded-reach cut."""
import os, sys, time, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_1110_6231_b200 as fmb

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 500
base = int(sys.argv[2]) if len(sys.argv) > 2 else 0
bad = 0
t0 = time.time()
for case in range(n_cases):
    rng = random.Random(base * 100000 + case)
    n = rng.randint(2, 3000)
    m = rng.randint(1, 8 * n)
    hi = rng.choice([1, 3, 100, 100000])
    edges = [(rng.randrange(n), rng.randrange(n), rng.randint(0, hi)) for _ in range(m)]
    net = fmb.build_network(edges, n, 0, n - 1)
    d = oracle.maxflow_seq(n, 0, n - 1, edges, want_state=True)
    cut = oracle.reach_cut(n, 0, n - 1, edges, d["residual"], d["excess"]).astype(bool)
    rep = fmb.hybrid_solve(net)
    if rep.objective != d["value"] or not (rep.cut == cut).all():
        bad += 1
        print(f"MISMATCH case {case}: n {n} m {m} hi {hi} got {rep.objective} want {d['value']}", flush=True)
print(f"{n_cases} generic graphs: {bad} mismatches, {time.time() - t0:.1f} s", flush=True)

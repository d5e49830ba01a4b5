"""One-line summary of a bench.py JSON line read from stdin (usage: bench.py ... | bench_line.py LABEL)."""
import json, sys, statistics
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print(sys.argv[1], round(d["ms_per_step"], 2), "mean step", round(statistics.mean(d["details"]["step_ms"]), 2),
      "e2e_ms", round(d["config"]["N_A"] * d["details"]["gmres_iterations"] / d["e2e"]["value"] * 1e3, 2))

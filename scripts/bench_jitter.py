"""Does the clocks sampler perturb the timed region?  Runs bench.py with the sampling interval
given on the command line and prints the K-step bracket minus the mean per-solve device time
(development aid; usage: bench_jitter.py MS [MS ...], each repeated REPEAT times)."""
import json, os, statistics, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = int(os.environ.get("REPEAT", "4"))
for _ in range(rep):
    for ms in sys.argv[1:]:
        env = dict(os.environ, CPDDG_BENCH_CLOCK_MS=ms)
        out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "5", "--warmup", "3",
                              "--cpu-baseline", "off"], env=env, capture_output=True, text=True).stdout
        d = json.loads(out.strip().splitlines()[-1])
        m = statistics.mean(d["details"]["step_ms"])
        e = d["config"]["N_A"] * d["details"]["gmres_iterations"] / d["e2e"]["value"] * 1e3
        print(f"clock_ms {ms:>7}: bracket - mean {d['ms_per_step'] - m:6.2f} ms, e2e - mean {e - m:6.2f} ms, "
              f"samples {d['clocks'].get('samples')}", flush=True)

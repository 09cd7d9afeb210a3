"""Automatic schedule per config: plan, pipelined step, kernel time, tune wall (env A/B, e.g.
FEMGPU_MACRO_AFFINE=0 FEMGPU_TUNE_CACHE=0 python tools/auto_ab.py C2,C1b)."""
import json, sys, time
sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg
for name in sys.argv[1].split(","):
    p = fg.config_problem(name)
    t0 = time.perf_counter()
    with fg.GpuInstance(p) as g:
        g.action()
        tune_s = time.perf_counter() - t0
        step_s, kern_s, _ = g.profile(warmup=2, reps=10)
        g.time_steps(int(max(3, min(10000, 0.1 / step_s))), pipelined=True)
        k = int(max(5, min(20000, 0.2 / step_s)))
        t = g.time_steps(k, pipelined=True) / k
        print(json.dumps({"config": name, "plan": g.describe().split(" | auto")[0], "step_us": round(t * 1e6, 1),
                          "kernel_us": round(kern_s * 1e6, 1), "tune_s": round(tune_s, 1)}), flush=True)

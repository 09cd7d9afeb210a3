"""Runs the automatic schedule on benchmark configs and records the model's predictions next to
the measurements (FEMGPU_TUNE_LOG, one JSON line per config, predicted vs measured per candidate).

usage: python tools/tune_report.py C2,C4 out.jsonl [all]
  all: FEMGPU_TUNE_ALL=1 -- compile and time every candidate (calibration of the model constants)
"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, ".")
cfgs = sys.argv[1].split(",") if sys.argv[1] != "ALL" else None
out = sys.argv[2]
os.environ["FEMGPU_TUNE_LOG"] = out + ".tmp"
os.environ["FEMGPU_TUNE_CACHE"] = "0"
if len(sys.argv) > 3 and sys.argv[3] == "all":
    os.environ["FEMGPU_TUNE_ALL"] = "1"
import paper_2506_17471_b200 as fg  # noqa: E402

for cfg in cfgs or list(fg.CONFIGS):
    if os.path.exists(out + ".tmp"):
        os.remove(out + ".tmp")
    p = fg.config_problem(cfg)
    os.environ["FEMGPU_CACHE"] = tempfile.mkdtemp(prefix="femgpu_tune_")  # cold JIT cache: honest tune wall
    t0 = time.perf_counter()
    with fg.GpuInstance(p) as g:
        sched = g.default_schedule()
        t_tune = time.perf_counter() - t0
        plan = g.describe()
    rec = json.loads(open(out + ".tmp").read().strip().splitlines()[-1]) if os.path.exists(out + ".tmp") else {}
    rec.update(config=cfg, tune_wall_s=round(t_tune, 2), plan=plan.split(" | auto: ")[0])
    with open(out, "a") as f:
        f.write(json.dumps(rec) + "\n")
    timed = [c for c in rec.get("candidates", []) if c["meas_us"] > 0]
    best = min(timed, key=lambda c: c["meas_us"]) if timed else None
    print(cfg, "tune %.1f s (model %.1f, jit %.1f, timing %.1f)" % (t_tune, rec.get("model_s", 0), rec.get("jit_s", 0),
                                                              rec.get("timing_s", 0)), "timed", len(timed), "winner", rec.get("winner"),
          "best %.1f us" % best["meas_us"] if best else "", "spearman %.2f" % rec.get("spearman", 0), flush=True)
if os.path.exists(out + ".tmp"):
    os.remove(out + ".tmp")

"""Quick probe: time a config (default C2: P2 Laplace 3D, N=107) under several schedules.
Schedules are specs: auto | scpt | tile:b=256 | macro:G=6,b=64,ms=1,rt=128,mb=0,basis=smem"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg
from paper_2506_17471_b200 import abi

n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1] != "-" else None
name = sys.argv[2] if len(sys.argv) > 2 else "C2"
specs = sys.argv[3].split(";") if len(sys.argv) > 3 else ["auto", "scpt", "macro:G=6"]


def parse(spec):
    if spec == "auto":
        return None
    kind, _, rest = spec.partition(":")
    kv = dict(x.split("=") for x in rest.split(",") if x)
    knobs = {}
    if "b" in kv:
        knobs["block_cells"] = int(kv["b"])
    if kv.get("basis") == "smem":
        knobs["basis"] = abi.BASIS_SMEM
    if "rt" in kv:
        knobs["reg_target"] = int(kv["rt"])
    if "mb" in kv:
        knobs["min_blocks"] = int(kv["mb"])
    if kind == "scpt":
        return fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC, **knobs)
    if kind == "tile":
        return fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, **knobs)
    if kind == "macro":
        return fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, group_cells=int(kv.get("G", 0)),
                                    stage_smem=int(kv.get("ms", 0)), **knobs)
    raise ValueError(spec)


t = time.time()
p = fg.config_problem(name, n=n)
print("build %.1fs cells=%d dofs=%d" % (time.time() - t, p.connectivity.cell_count, p.output_size), flush=True)
g = fg.GpuInstance(p)
print("create %.1fs" % (time.time() - t), flush=True)
flops = fg.usable_flops(p.signature) * p.connectivity.cell_count
res = {}
for spec in specs:
    try:
        t0 = time.time()
        sec = g.time(parse(spec))
        res[spec] = dict(us=round(sec * 1e6, 1), gdofs=round(p.output_size / sec / 1e9, 2),
                         tflops=round(flops / sec / 1e12, 2))
        print(spec, json.dumps(res[spec]), "(%.1fs)" % (time.time() - t0), flush=True)
    except Exception as e:
        print(spec, "FAILED", str(e)[:300], flush=True)
print(json.dumps(res))

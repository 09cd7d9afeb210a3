"""Times named schedules on benchmark configs (one JSON line per config x schedule).

usage: python tools/sweep.py C2,C4 auto,macro6,tile-256 [reps]
Schedule names: auto | scpt | scpt-smem | macroG[-ms][-bB][-mM] | tile-B[-mM]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402
from paper_2506_17471_b200 import abi  # noqa: E402


def sched(name):
    if name == "auto":
        return None
    parts = name.split("-")
    kw = {}
    for p in parts[1:] if parts[0] != "dmma" else []:
        if p == "ms":
            kw["stage_smem"] = 1
        elif p == "ys":
            kw["stage_smem"] = 2
        elif p == "qm":
            kw["stage_smem"] = 3
        elif p == "ql":
            kw["stage_smem"] = 4
        elif p.startswith("o") and p[1:].isdigit():
            kw["qmopt"] = int(p[1:])
        elif p.startswith("sp"):
            kw["split"] = int(p[2:])
        elif p == "smem":
            kw["basis"] = abi.BASIS_SMEM
        elif p == "const":
            kw["basis"] = abi.BASIS_CONST
        elif p.startswith("b"):
            kw["block_cells"] = int(p[1:])
        elif p.startswith("m"):
            kw["min_blocks"] = int(p[1:])
        elif p.startswith("r"):
            kw["reg_target"] = int(p[1:])
        elif p.startswith("g") and p[1:].isdigit():
            kw["group_cells"] = int(p[1:])
        elif p.isdigit():
            kw["block_cells"] = int(p)
    head = parts[0]
    if head == "dmma":
        # dmma-c<cells per warp task>-q<TQ>-b<CTA threads>-m<min CTAs/SM>-smem|glob
        d = {}
        for p in parts[1:]:
            if p.startswith("c"):
                d["cells_per_group"] = int(p[1:])
            elif p.startswith("q"):
                d["quad_tile"] = int(p[1:])
            elif p.startswith("l"):
                d["lanes_per_cell"] = int(p[1:])
            elif p.startswith("R"):
                d["eval_row_tile"] = int(p[1:])
            elif p.startswith("S"):
                d["quad_row_tile"] = int(p[1:])
            elif p.startswith("m"):
                d["min_blocks"] = int(p[1:])
            elif p == "breg":
                d["stage_smem"] = 1
            elif p == "u2":
                d["qmopt"] = 16384
            elif p.startswith("b"):
                d["block_cells"] = int(p[1:])
            elif p == "smem":
                d["basis"] = abi.BASIS_SMEM
            elif p == "glob":
                d["basis"] = abi.BASIS_CONST
        return fg.TilingParams.dmma(**d)
    if head == "colour":
        return fg.TilingParams.scpt(scatter=abi.SCATTER_COLOR, **kw)
    if head == "scpt":
        return fg.TilingParams.scpt(scatter=abi.SCATTER_ATOMIC, **kw)
    if head.startswith("macro"):
        return fg.TilingParams.scpt(scatter=abi.SCATTER_MACRO, group_cells=int(head[5:] or 0), **kw)
    if head == "tile":
        return fg.TilingParams.scpt(scatter=abi.SCATTER_TILE, **kw)
    raise ValueError(name)


PIPE = os.environ.get("SWEEP_PIPE", "1") == "1"


def device_y(g, n):
    import torch
    from paper_2506_17471_b200.krylov import _CudaArray
    return torch.as_tensor(_CudaArray(g.device_output(), n), device="cuda").cpu().numpy()


def main():
    cfgs = sys.argv[1].split(",")
    names = sys.argv[2].split(",")
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    peak = fg.fp64_peak()[0]
    for cfg in cfgs:
        t0 = time.time()
        p = fg.config_problem(cfg)
        flops = fg.usable_flops(p.signature) * p.connectivity.cell_count
        with fg.GpuInstance(p) as g:
            ref = None
            for nm in names:
                res = {"config": cfg, "sched": nm}
                try:
                    s = sched(nm)
                    y = g.action(s)
                    if ref is None:
                        ref = y
                    res["rel_l2_vs_first"] = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
                    step, kern, zero = g.profile(s, warmup=3, reps=reps)
                    res.update(step_us=round(step * 1e6, 1), kernel_us=round(kern * 1e6, 1),
                               gdofs=round(p.output_size / step / 1e9, 2),
                               fp64_frac_kernel=round(flops / kern / 1e12 / peak, 3))
                    if PIPE:  # output-pipelined steps (zeroing of the next output inside the kernel)
                        tp = g.time_steps(reps, s, pipelined=True) / reps
                        yp = device_y(g, p.output_size)
                        res.update(pipe_step_us=round(tp * 1e6, 1),
                                   pipe_rel_l2=float(np.linalg.norm(yp - y) / np.linalg.norm(y)))
                        ts = g.time_steps(reps, s, pipelined=3) / reps
                        yp = device_y(g, p.output_size)
                        res.update(side_step_us=round(ts * 1e6, 1),
                                   side_rel_l2=float(np.linalg.norm(yp - y) / np.linalg.norm(y)))
                except Exception as e:  # noqa: BLE001
                    res["error"] = str(e)[:300]
                print(json.dumps(res), flush=True)
        print(json.dumps({"config": cfg, "wall_s": round(time.time() - t0, 1)}), flush=True)


if __name__ == "__main__":
    main()

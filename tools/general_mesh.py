"""A benchmark configuration on a 'general' mesh: the structured mesh with the cells of every
6-cell group shuffled (and optionally every cell shuffled globally), so no connectivity pattern
repeats (the macro families do not apply) while spatial locality is kept (or not).  Times the
automatic schedule and named schedules (tools/sweep.py names).

usage: python tools/general_mesh.py C2 local|global|global+reorder sched,sched,... [reps]
  global+reorder: the globally shuffled mesh renumbered by femgpu_problem_reorder (Morton cells,
  first-touch nodes)
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2506_17471_b200 as fg  # noqa: E402
from tools.sweep import sched  # noqa: E402


def permuted(p, perm):
    c = p.connectivity
    for m in c.scalar_maps + c.vector_maps + [c.test_map] + ([c.coord_map] if c.coord_map is not None else []):
        pass
    seen = {}
    def remap(im):
        if id(im) not in seen:
            seen[id(im)] = fg.IndexMap(np.ascontiguousarray(im.indices[perm]), im.global_count)
        return seen[id(im)]
    c.scalar_maps = [remap(m) for m in c.scalar_maps]
    c.vector_maps = [remap(m) for m in c.vector_maps]
    c.test_map = remap(c.test_map)
    if c.coord_map is not None:
        c.coord_map = remap(c.coord_map)
    return p


def main():
    cfg, mode = sys.argv[1], sys.argv[2]
    names = sys.argv[3].split(",")
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    p = fg.config_problem(cfg)
    C = p.connectivity.cell_count
    rng = np.random.default_rng(1)
    if mode == "local":
        perm = (np.arange(C).reshape(-1, 6)[:, None, :].repeat(1, 1)[:, 0, :])
        perm = np.array([g[rng.permutation(6)] for g in perm]).reshape(-1)
    else:
        perm = rng.permutation(C)
    p = permuted(p, perm)
    if mode.endswith("+reorder"):
        p, _ = fg.reorder_problem(p)
    ref = None
    with fg.GpuInstance(p) as g:
        for nm in names:
            res = {"config": cfg, "mesh": mode, "sched": nm}
            try:
                s = sched(nm)
                y = g.action(s)
                ref = y if ref is None else ref
                res["rel_l2_vs_first"] = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
                g.time_steps(3, s, pipelined=True)
                t = g.time_steps(reps, s, pipelined=True) / reps
                res.update(step_us=round(t * 1e6, 1), plan=g.describe().split(" | auto: ")[0] if nm == "auto" else nm)
            except Exception as e:  # noqa: BLE001
                res["error"] = str(e)[:200]
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

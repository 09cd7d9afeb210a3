"""Generates tests/golden/reference_outputs.npz with the REFERENCE's own code (oracle/_ref:
femsched::make_problem + preset_map/generic_map + reference_action, compiled from
/root/reference/proj/include/femsched/form.hpp).  Run in the container that has /root/reference:

    python tests/golden/make_golden.py

For each case it stores y, the reference counters and a SHA-256 of the instance arrays, so the
tests can pin (a) the numpy synthesis (paper_2506_17471_b200.form.make_problem) and (b) the C
restatement (oracle/femoracle.c) without the reference being present (e.g. on the GPU box).
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from tests.helpers import ACCEPTANCE, UNIT  # noqa: E402

CASES = [(op, d, p, q, 16, 7) for op, d, p, q in ACCEPTANCE] + list(UNIT) + [
    ("generic:laplace", 2, 2, 6, 5, 11), ("generic:elasticity", 3, 2, 4, 5, 12), ("generic:mass", 1, 3, 4, 7, 13),
    ("hyperelasticity", 3, 2, 4, 5, 3), ("hyperelasticity", 2, 3, 6, 6, 1), ("elasticity", 3, 2, 10, 4, 7),
    ("mass", 1, 2, 3, 9, 2), ("helmholtz", 3, 2, 6, 3, 5)]


def instance_digest(p):
    h = hashlib.sha256()
    arrs = list(p.tabulations.scalar_phi) + list(p.tabulations.vector_phi) + [p.tabulations.psi, p.tabulations.weights]
    arrs += [m.indices for m in p.connectivity.scalar_maps] + [m.indices for m in p.connectivity.vector_maps]
    arrs += [p.connectivity.test_map.indices]
    if p.signature.affine_geometry:
        arrs += [p.connectivity.coord_map.indices, p.connectivity.coords]
    arrs += list(p.scalar_inputs) + list(p.vector_inputs)
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def key(case):
    return "%s|%d|%d|%d|%d|%d" % case


def main():
    out = {}
    for case in CASES:
        p = oracle.ref_make_problem(*case)
        y, cnt = oracle.ref_reference_action(p, counters=True)
        out["y:" + key(case)] = y
        out["counters:" + key(case)] = np.array(cnt, dtype=np.int64)
        out["digest:" + key(case)] = np.frombuffer(instance_digest(p).encode(), dtype=np.uint8)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_outputs.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, len(CASES), "cases")
    # an instance file written by the reference's own femsched::save_instance_file (io.hpp), so
    # the io reader is pinned on a box without the reference (tests/test_io.py)
    inst = os.path.join(os.path.dirname(os.path.abspath(__file__)), "instance_laplace_2d_p2.txt")
    oracle.ref_save_instance(oracle.ref_make_problem("laplace", 2, 2, 6, 16, 7), inst)
    print("wrote", inst)
    # mesh instances (structured meshes, coefficient / vector-test-space forms) written by the
    # reference's save_instance_file, with the reference's reference_action output, so the GPU
    # suite runs reference-written mesh files through the kernels (tests/test_gpu_configs.py)
    ys = {}
    for name, args in MESH_FILES.items():
        import paper_2506_17471_b200 as fg
        p = fg.mesh_problem(*args)
        f = os.path.join(os.path.dirname(os.path.abspath(__file__)), name + ".txt")
        oracle.ref_save_instance(p, f)
        ys["y:" + name] = oracle.ref_reference_action(oracle.ref_load_instance(f))
        print("wrote", f)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "mesh_instance_outputs.npz"), **ys)


# reference-written mesh instance files: (form, dim, degree, Q, n)
MESH_FILES = {"mesh_helmholtz_coef_2d_p3": ("helmholtz_coef", 2, 3, 12, 3),
              "mesh_elasticity_3d_p2": ("elasticity", 3, 2, 4, 1)}


if __name__ == "__main__":
    main()

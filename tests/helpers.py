"""Shared test helpers (instances from the reference's own test suites)."""
import numpy as np

import paper_2506_17471_b200 as fg

# (op, d, p, Q) tuples of the acceptance sweep, 16 cells, seed 7 (acceptance.cpp:34-37)
ACCEPTANCE = [("mass", 2, 2, 7), ("laplace", 2, 2, 6), ("helmholtz", 2, 3, 12), ("mass", 3, 1, 5),
              ("laplace", 3, 2, 8), ("helmholtz", 3, 1, 7)]
# (op, d, p, Q, cells, seed) used by the unit tests (test_simulate.cpp:61-62,111-112,133-134,149-150;
# test_form.cpp:135,197,208,220-221,245,272)
UNIT = [("laplace", 2, 2, 6, 16, 7), ("laplace", 2, 2, 6, 33, 4), ("elasticity", 2, 2, 5, 9, 21),
        ("mass", 2, 2, 6, 8, 3), ("helmholtz", 2, 1, 3, 10, 13), ("helmholtz", 2, 2, 4, 4, 3),
        ("laplace", 2, 2, 6, 2, 11), ("elasticity", 2, 2, 6, 8, 5), ("laplace", 2, 2, 6, 3, 2)]


def preset_problem(op, d, p, Q, cells, seed):
    sig = fg.preset_signature(op, d, p, Q)
    return fg.make_problem(sig, fg.preset_map(op, sig), cells, seed)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def max_rel(a, b):
    """Elementwise relative error with the reference's 1e-30 guard (search.hpp:360-366)."""
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-30))) if len(b) else 0.0


def dense_triple_product_problem():
    """The known-answer instance of test_form.cpp:142-193 (n=4, Q=5, det=3)."""
    n, q = 4, 5
    sig = fg.FormSignature(dim=2, scalar_spaces=[fg.ScalarSpace(n, 1)], test_dofs=n, test_deriv_terms=1,
                           quad_points=q, coord_dofs=3)
    phi = np.array([[0.3 + 0.1 * i + 0.07 * j for j in range(n)] for i in range(q)])
    tab = fg.Tabulations(scalar_phi=[phi.reshape(1, q, n)], psi=phi.T.copy().reshape(1, n, q),
                         weights=np.array([0.5, 0.6, 0.7, 0.8, 0.9]))
    conn = fg.MeshConnectivity(cell_count=1)
    conn.scalar_maps = [fg.IndexMap(np.arange(n, dtype=np.int32).reshape(1, n), n)]
    conn.test_map = fg.IndexMap(np.arange(n, dtype=np.int32).reshape(1, n), n)
    conn.coord_map = fg.IndexMap(np.arange(3, dtype=np.int32).reshape(1, 3), 3)
    conn.coord_global_count = 3
    conn.coords = np.array([[0.0, 0.0], [2.0, 0.0], [0.0, 1.5]])
    p = fg.ProblemInstance(sig, fg.preset_map("mass", sig), tab, conn, [np.array([1.0, 2.0, 3.0, 4.0])], [], n)
    p.validate()
    return p


# test_form.cpp:142-193, re-derived with the compiled reference
DENSE_TRIPLE_PRODUCT_Y = np.array([39.119999999999997, 44.034000000000006, 48.948, 53.862000000000002])


def complete_rows(p, m):
    """Rows of y whose every contribution comes from cells [0, m) (what a reference run over that
    cell range reproduces exactly)."""
    tm = p.connectivity.test_map.indices
    inside = np.zeros(p.output_size, dtype=bool)
    inside[tm[:m].ravel()] = True
    if m < tm.shape[0]:
        inside[tm[m:].ravel()] = False
    return np.nonzero(inside)[0]

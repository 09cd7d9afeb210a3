/*
 * femoracle.c — TEST INFRASTRUCTURE ONLY (the parity checker, never shipped and
 * never on the product path).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 *
 * A plain-C restatement of the reference's sequential ground-truth action and
 * its helpers, consuming the flat femgpu_problem descriptor (include/femgpu.h):
 *
 *   oracle_validate         <- ProblemInstance::validate      form.hpp:416-434
 *                              (FormSignature::validate :115-147, PointwiseMap::validate
 *                               :234-280, Tabulations::validate :332-368,
 *                               MeshConnectivity::validate :380-404)
 *   oracle_usable_flops     <- usable_flops                    form.hpp:164-173
 *   oracle_affine_jacobian  <- affine_jacobian                 form.hpp:441-457
 *   oracle_reference_action <- reference_action               form.hpp:471-595
 *   (map evaluation)        <- PointwiseMap::eval_node         form.hpp:295-314
 *
 * Loop and summation order follow the reference exactly (cells ascending, j
 * ascending in the evaluation matvecs, k inner in the quadrature matvec, plain
 * additions into the output), and the library is compiled with
 * -ffp-contract=off, so on x86-64 it is bit-identical to the reference built
 * with its own flags (pinned in tests/test_oracle.py against oracle/_ref and the
 * committed golden vectors in tests/golden/).
 *
 * Extension (not in the reference, not pinned by it): FEMGPU_OP_INV_JACOBIAN,
 * J^{-1}[a][b] = adj(J)[a][b] / det.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../include/femgpu.h"

#define ORC_OK 0
#define ORC_INVALID 1
#define ORC_NONFINITE 3

static int fail(char* err, int len, int code, const char* msg) {
    if (err && len > 0) {
        strncpy(err, msg, (size_t)len - 1);
        err[len - 1] = 0;
    }
    return code;
}

static int all_finite(const double* v, long long n) {
    for (long long i = 0; i < n; ++i)
        if (!isfinite(v[i])) return 0;
    return 1;
}

static int map_in_bounds(const int32_t* m, long long n, int32_t bound) {
    for (long long i = 0; i < n; ++i)
        if (m[i] < 0 || m[i] >= bound) return 0;
    return 1;
}

int oracle_validate(const femgpu_problem* p, char* err, int len) {
    /* FormSignature::validate, form.hpp:115-147 */
    if (p->dim < 1 || p->dim > 3) return fail(err, len, ORC_INVALID, "signature: dim must be 1..3");
    if (p->n_scalar + p->n_vector == 0)
        return fail(err, len, ORC_INVALID, "signature: at least one trial space required");
    if (p->quad_points < 1) return fail(err, len, ORC_INVALID, "signature: quad_points must be >= 1");
    if (p->test_dofs < 1 || p->test_deriv_terms < 1)
        return fail(err, len, ORC_INVALID, "signature: test space counts must be positive");
    if (p->word_bytes != 4 && p->word_bytes != 8)
        return fail(err, len, ORC_INVALID, "signature: word_bytes must be 4 or 8");
    for (int i = 0; i < p->n_scalar; ++i)
        if (p->scalar_spaces[i].dofs < 1 || p->scalar_spaces[i].deriv_terms < 1)
            return fail(err, len, ORC_INVALID, "signature: scalar space counts must be positive");
    for (int i = 0; i < p->n_vector; ++i) {
        const femgpu_space* v = &p->vector_spaces[i];
        if (v->dofs < 1 || v->deriv_terms < 1)
            return fail(err, len, ORC_INVALID, "signature: vector space counts must be positive");
        if (!v->components)
            return fail(err, len, ORC_INVALID,
                        "signature: one component index per derivative term required");
        for (int k = 0; k < v->deriv_terms; ++k)
            if (v->components[k] < 0 || v->components[k] >= p->dim)
                return fail(err, len, ORC_INVALID, "signature: component index out of range");
    }
    if (p->affine_geometry) {
        if (p->coord_dofs != p->dim + 1)
            return fail(err, len, ORC_INVALID, "signature: affine geometry requires coord_dofs == dim+1");
        if (p->coordinate_space != -1)
            return fail(err, len, ORC_INVALID,
                        "signature: coordinate_space is only meaningful when non-affine");
    } else {
        if (p->coordinate_space < 0 || p->coordinate_space >= p->n_vector)
            return fail(err, len, ORC_INVALID,
                        "signature: non-affine geometry requires the coordinate space to appear in "
                        "the vector-space list exactly once");
    }
    /* PointwiseMap::validate, form.hpp:234-280 */
    if (p->n_map_outputs != p->test_deriv_terms)
        return fail(err, len, ORC_INVALID, "pointwise map: one expression per test derivative term required");
    for (int o = 0; o < p->n_map_outputs; ++o)
        if (p->map_outputs[o] < 0 || p->map_outputs[o] >= p->n_map_nodes)
            return fail(err, len, ORC_INVALID, "pointwise map: output references unknown node");
    for (int id = 0; id < p->n_map_nodes; ++id) {
        const femgpu_map_node* n = &p->map_nodes[id];
        switch (n->op) {
            case FEMGPU_OP_CONSTANT: break;
            case FEMGPU_OP_SCALAR_DERIV:
                if (n->a < 0 || n->a >= p->n_scalar || n->b < 0 || n->b >= p->scalar_spaces[n->a].deriv_terms)
                    return fail(err, len, ORC_INVALID, "pointwise map: undeclared scalar derivative input");
                break;
            case FEMGPU_OP_VECTOR_DERIV:
                if (n->a < 0 || n->a >= p->n_vector || n->b < 0 || n->b >= p->vector_spaces[n->a].deriv_terms)
                    return fail(err, len, ORC_INVALID, "pointwise map: undeclared vector derivative input");
                break;
            case FEMGPU_OP_JACOBIAN:
            case FEMGPU_OP_INV_JACOBIAN:
                if (!p->affine_geometry)
                    return fail(err, len, ORC_INVALID, "pointwise map: jacobian input requires affine geometry");
                if (n->a < 0 || n->a >= p->dim || n->b < 0 || n->b >= p->dim)
                    return fail(err, len, ORC_INVALID, "pointwise map: jacobian index out of range");
                break;
            case FEMGPU_OP_DETERMINANT:
                if (!p->affine_geometry)
                    return fail(err, len, ORC_INVALID, "pointwise map: determinant input requires affine geometry");
                break;
            case FEMGPU_OP_WEIGHT: break;
            case FEMGPU_OP_COORD:
                if (!p->affine_geometry)
                    return fail(err, len, ORC_INVALID, "pointwise map: coord input requires affine geometry");
                if (n->a < 0 || n->a >= p->coord_dofs || n->b < 0 || n->b >= p->dim)
                    return fail(err, len, ORC_INVALID, "pointwise map: coord index out of range");
                break;
            case FEMGPU_OP_ADD:
            case FEMGPU_OP_MUL:
                if (n->a < 0 || n->b < 0 || n->a >= id || n->b >= id)
                    return fail(err, len, ORC_INVALID, "pointwise map: child must precede its parent");
                break;
            default: return fail(err, len, ORC_INVALID, "pointwise map: unknown op");
        }
    }
    /* Tabulations::validate, form.hpp:332-368 */
    const int Q = p->quad_points;
    for (int i = 0; i < p->n_scalar; ++i)
        if (!all_finite(p->scalar_spaces[i].phi, (long long)p->scalar_spaces[i].deriv_terms * Q * p->scalar_spaces[i].dofs))
            return fail(err, len, ORC_INVALID, "tabulations: non-finite entry in scalar phi");
    for (int i = 0; i < p->n_vector; ++i)
        if (!all_finite(p->vector_spaces[i].phi, (long long)p->vector_spaces[i].deriv_terms * Q * p->vector_spaces[i].dofs))
            return fail(err, len, ORC_INVALID, "tabulations: non-finite entry in vector phi");
    if (!all_finite(p->psi, (long long)p->test_deriv_terms * p->test_dofs * Q))
        return fail(err, len, ORC_INVALID, "tabulations: non-finite entry in psi");
    if (!all_finite(p->weights, Q)) return fail(err, len, ORC_INVALID, "tabulations: non-finite weight");
    /* MeshConnectivity::validate, form.hpp:380-404 */
    const long long C = p->cell_count;
    if (C < 1) return fail(err, len, ORC_INVALID, "connectivity: at least one cell required");
    for (int i = 0; i < p->n_scalar; ++i)
        if (!map_in_bounds(p->scalar_spaces[i].map, C * p->scalar_spaces[i].dofs, p->scalar_spaces[i].global_count))
            return fail(err, len, ORC_INVALID, "connectivity: index out of bounds in scalar space map");
    for (int i = 0; i < p->n_vector; ++i)
        if (!map_in_bounds(p->vector_spaces[i].map, C * p->vector_spaces[i].dofs, p->vector_spaces[i].global_count))
            return fail(err, len, ORC_INVALID, "connectivity: index out of bounds in vector space map");
    if (!map_in_bounds(p->test_map, C * p->test_dofs, p->test_global_count))
        return fail(err, len, ORC_INVALID, "connectivity: index out of bounds in test space map");
    if (p->affine_geometry) {
        if (!map_in_bounds(p->coord_map, C * p->coord_dofs, p->coord_global_count))
            return fail(err, len, ORC_INVALID, "connectivity: index out of bounds in coordinate map");
        if (p->coord_global_count < 1 || !p->coords)
            return fail(err, len, ORC_INVALID, "connectivity: coordinate array shape mismatch");
    }
    if (p->output_size != p->test_global_count)
        return fail(err, len, ORC_INVALID, "instance: output length mismatch");
    return ORC_OK;
}

long long oracle_usable_flops(const femgpu_problem* p) {
    long long ops = 0;
    for (int i = 0; i < p->n_scalar; ++i)
        ops += 2LL * p->scalar_spaces[i].deriv_terms * p->quad_points * p->scalar_spaces[i].dofs;
    for (int i = 0; i < p->n_vector; ++i)
        ops += 2LL * p->vector_spaces[i].deriv_terms * p->quad_points * p->vector_spaces[i].dofs;
    ops += 2LL * p->test_deriv_terms * p->quad_points * p->test_dofs;
    return ops;
}

void oracle_affine_jacobian(const double* X, int dim, double* J, double* det_out) {
    for (int c = 0; c < dim; ++c)
        for (int r = 0; r < dim; ++r) J[r * dim + c] = X[(c + 1) * dim + r] - X[r];
    double det = 0.0;
    switch (dim) {
        case 1: det = J[0]; break;
        case 2: det = J[0] * J[3] - J[1] * J[2]; break;
        case 3:
            det = J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
                  J[2] * (J[3] * J[7] - J[4] * J[6]);
            break;
        default: break;
    }
    *det_out = det;
}

/* Extension: inverse of the affine Jacobian via the adjugate. */
static void inverse_jacobian(const double* J, int dim, double det, double* Ji) {
    if (dim == 1) {
        Ji[0] = 1.0 / det;
    } else if (dim == 2) {
        Ji[0] = J[3] / det;
        Ji[1] = -J[1] / det;
        Ji[2] = -J[2] / det;
        Ji[3] = J[0] / det;
    } else {
        Ji[0] = (J[4] * J[8] - J[5] * J[7]) / det;
        Ji[1] = (J[2] * J[7] - J[1] * J[8]) / det;
        Ji[2] = (J[1] * J[5] - J[2] * J[4]) / det;
        Ji[3] = (J[5] * J[6] - J[3] * J[8]) / det;
        Ji[4] = (J[0] * J[8] - J[2] * J[6]) / det;
        Ji[5] = (J[2] * J[3] - J[0] * J[5]) / det;
        Ji[6] = (J[3] * J[7] - J[4] * J[6]) / det;
        Ji[7] = (J[1] * J[6] - J[0] * J[7]) / det;
        Ji[8] = (J[0] * J[4] - J[1] * J[3]) / det;
    }
}

typedef struct {
    const double* sd;  /* scalar derivs, flattened by term offsets */
    const double* vd;  /* vector derivs */
    const int* soff;   /* scalar term offsets */
    const int* voff;
    const double* J;
    const double* Ji;
    double det;
    double w;
    const double* X;
    int dim;
} eval_in;

/* Recursive, unmemoised evaluation: same traversal as eval_node (form.hpp:295-314). */
static double eval_node(const femgpu_problem* p, int id, const eval_in* in, long long* ops) {
    const femgpu_map_node* n = &p->map_nodes[id];
    switch (n->op) {
        case FEMGPU_OP_CONSTANT: return n->value;
        case FEMGPU_OP_SCALAR_DERIV: return in->sd[in->soff[n->a] + n->b];
        case FEMGPU_OP_VECTOR_DERIV: return in->vd[in->voff[n->a] + n->b];
        case FEMGPU_OP_JACOBIAN: return in->J[n->a * in->dim + n->b];
        case FEMGPU_OP_INV_JACOBIAN: return in->Ji[n->a * in->dim + n->b];
        case FEMGPU_OP_DETERMINANT: return in->det;
        case FEMGPU_OP_WEIGHT: return in->w;
        case FEMGPU_OP_COORD: return in->X[n->a * in->dim + n->b];
        case FEMGPU_OP_ADD: {
            if (ops) ++*ops;
            double l = eval_node(p, n->a, in, ops);
            double r = eval_node(p, n->b, in, ops);
            return l + r;
        }
        case FEMGPU_OP_MUL: {
            if (ops) ++*ops;
            double l = eval_node(p, n->a, in, ops);
            double r = eval_node(p, n->b, in, ops);
            return l * r;
        }
    }
    return 0.0;
}

/* counters (may be NULL): [0] matvec_mults, [1] matvec_adds, [2] map_ops
 * (ReferenceCounters, form.hpp:463-467).  cell_begin/cell_end restrict the
 * loop to a cell range (the restriction used by test_form.cpp:11-24). */
int oracle_reference_action_range(const femgpu_problem* p, int cell_begin, int cell_end, double* out,
                                  long long* counters, char* err, int len) {
    int rc = oracle_validate(p, err, len);
    if (rc) return rc;
    const int dim = p->dim, Q = p->quad_points, ns = p->n_scalar, nv = p->n_vector;
    const int nW = p->test_dofs, Tw = p->test_deriv_terms;
    int soff[FEMGPU_MAX_SPACES + 1], voff[FEMGPU_MAX_SPACES + 1];
    int max_dofs = 1;
    soff[0] = 0;
    for (int i = 0; i < ns; ++i) {
        soff[i + 1] = soff[i] + p->scalar_spaces[i].deriv_terms;
        if (p->scalar_spaces[i].dofs > max_dofs) max_dofs = p->scalar_spaces[i].dofs;
    }
    voff[0] = 0;
    for (int i = 0; i < nv; ++i) {
        voff[i + 1] = voff[i] + p->vector_spaces[i].deriv_terms;
        if (p->vector_spaces[i].dofs > max_dofs) max_dofs = p->vector_spaces[i].dofs;
    }
    if (ns > FEMGPU_MAX_SPACES || nv > FEMGPU_MAX_SPACES)
        return fail(err, len, ORC_INVALID, "oracle: too many spaces");
    for (long long i = 0; i < p->output_size; ++i) out[i] = 0.0;

    double* local = (double*)malloc(sizeof(double) * (size_t)max_dofs * 3);
    double* sd = (double*)malloc(sizeof(double) * (size_t)(soff[ns] + 1));
    double* vd = (double*)malloc(sizeof(double) * (size_t)(voff[nv] + 1));
    double* e = (double*)malloc(sizeof(double) * (size_t)Tw);
    double* cell_out = (double*)malloc(sizeof(double) * (size_t)nW);
    double* slocal[FEMGPU_MAX_SPACES];
    double* vlocal[FEMGPU_MAX_SPACES];
    for (int i = 0; i < ns; ++i) slocal[i] = (double*)malloc(sizeof(double) * (size_t)p->scalar_spaces[i].dofs);
    for (int i = 0; i < nv; ++i) vlocal[i] = (double*)malloc(sizeof(double) * (size_t)p->vector_spaces[i].dofs * dim);
    double X[4 * 3], J[9], Ji[9], det = 0.0;
    char msg[160];
    rc = ORC_OK;

    for (int cell = cell_begin; cell < cell_end && rc == ORC_OK; ++cell) {
        /* gather, form.hpp:498-509 */
        for (int i = 0; i < ns; ++i) {
            const femgpu_space* s = &p->scalar_spaces[i];
            for (int j = 0; j < s->dofs; ++j) slocal[i][j] = s->input[s->map[(long long)cell * s->dofs + j]];
        }
        for (int i = 0; i < nv; ++i) {
            const femgpu_space* s = &p->vector_spaces[i];
            for (int j = 0; j < s->dofs; ++j)
                for (int c = 0; c < dim; ++c)
                    vlocal[i][j * dim + c] = s->input[(long long)s->map[(long long)cell * s->dofs + j] * dim + c];
        }
        det = 0.0;
        if (p->affine_geometry) {
            for (int j = 0; j < p->coord_dofs; ++j)
                for (int c = 0; c < dim; ++c)
                    X[j * dim + c] = p->coords[(long long)p->coord_map[(long long)cell * p->coord_dofs + j] * dim + c];
            oracle_affine_jacobian(X, dim, J, &det);
            if (!isfinite(det)) {
                snprintf(msg, sizeof msg, "reference_action: non-finite value at cell %d during jacobian", cell);
                rc = fail(err, len, ORC_NONFINITE, msg);
                break;
            }
            inverse_jacobian(J, dim, det, Ji);
        }
        for (int jw = 0; jw < nW; ++jw) cell_out[jw] = 0.0;
        for (int iq = 0; iq < Q && rc == ORC_OK; ++iq) {
            /* evaluation, form.hpp:526-555 */
            for (int i = 0; i < ns; ++i) {
                const femgpu_space* s = &p->scalar_spaces[i];
                for (int k = 0; k < s->deriv_terms; ++k) {
                    const double* phi = s->phi + ((long long)k * Q + iq) * s->dofs;
                    double acc = 0.0;
                    for (int j = 0; j < s->dofs; ++j) acc += phi[j] * slocal[i][j];
                    sd[soff[i] + k] = acc;
                    if (counters) {
                        counters[0] += s->dofs;
                        counters[1] += s->dofs;
                    }
                }
            }
            for (int i = 0; i < nv; ++i) {
                const femgpu_space* s = &p->vector_spaces[i];
                for (int k = 0; k < s->deriv_terms; ++k) {
                    const double* phi = s->phi + ((long long)k * Q + iq) * s->dofs;
                    const int comp = s->components[k];
                    double acc = 0.0;
                    for (int j = 0; j < s->dofs; ++j) acc += phi[j] * vlocal[i][j * dim + comp];
                    vd[voff[i] + k] = acc;
                    if (counters) {
                        counters[0] += s->dofs;
                        counters[1] += s->dofs;
                    }
                }
            }
            int bad = 0;
            for (int t = 0; t < soff[ns]; ++t) bad |= !isfinite(sd[t]);
            for (int t = 0; t < voff[nv]; ++t) bad |= !isfinite(vd[t]);
            if (bad) {
                snprintf(msg, sizeof msg, "reference_action: non-finite value at cell %d during evaluation", cell);
                rc = fail(err, len, ORC_NONFINITE, msg);
                break;
            }
            /* pointwise map, form.hpp:561-573 */
            eval_in in = {sd, vd, soff, voff, J, Ji, det, p->weights[iq], X, dim};
            for (int k = 0; k < Tw; ++k) {
                e[k] = eval_node(p, p->map_outputs[k], &in, counters ? &counters[2] : NULL);
                if (!isfinite(e[k])) {
                    snprintf(msg, sizeof msg, "reference_action: non-finite value at cell %d during pointwise map", cell);
                    rc = fail(err, len, ORC_NONFINITE, msg);
                    break;
                }
            }
            if (rc) break;
            /* quadrature, form.hpp:575-585 */
            for (int jw = 0; jw < nW; ++jw) {
                double acc = cell_out[jw];
                for (int k = 0; k < Tw; ++k) acc += p->psi[((long long)k * nW + jw) * Q + iq] * e[k];
                cell_out[jw] = acc;
            }
            if (counters) {
                counters[0] += (long long)nW * Tw;
                counters[1] += (long long)nW * Tw;
            }
        }
        if (rc) break;
        for (int jw = 0; jw < nW; ++jw)
            if (!isfinite(cell_out[jw])) {
                snprintf(msg, sizeof msg, "reference_action: non-finite value at cell %d during quadrature", cell);
                rc = fail(err, len, ORC_NONFINITE, msg);
                break;
            }
        if (rc) break;
        /* scatter, form.hpp:590-592 */
        for (int jw = 0; jw < nW; ++jw) out[p->test_map[(long long)cell * nW + jw]] += cell_out[jw];
    }
    free(local);
    free(sd);
    free(vd);
    free(e);
    free(cell_out);
    for (int i = 0; i < ns; ++i) free(slocal[i]);
    for (int i = 0; i < nv; ++i) free(vlocal[i]);
    return rc;
}

int oracle_reference_action(const femgpu_problem* p, double* out, long long* counters, char* err, int len) {
    return oracle_reference_action_range(p, 0, p->cell_count, out, counters, err, len);
}

/* ---- deterministic synthesis restated (form.hpp:741-768) -------------- */

/* SynthRng::next_u64 (splitmix64), form.hpp:744-749 */
uint64_t oracle_splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* n draws of SynthRng::uniform(lo, span), form.hpp:751-753 */
void oracle_uniform_fill(uint64_t* state, double lo, double span, double* out, long long n) {
    for (long long i = 0; i < n; ++i)
        out[i] = lo + span * (double)(oracle_splitmix_next(state) >> 11) * 0x1.0p-53;
}

/* chain_index_map, form.hpp:761-768 */
int oracle_chain_index_map(int cells, int entries, int32_t* out) {
    const int overlap = (entries + 3) / 4;
    const int stride = entries - overlap;
    for (int cell = 0; cell < cells; ++cell)
        for (int j = 0; j < entries; ++j) out[(long long)cell * entries + j] = cell * stride + j;
    return (cells - 1) * stride + entries;
}

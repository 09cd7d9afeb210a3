// emit.cpp — sm_100a CUDA source emitter for the matrix-free action.
//
// Replaces the role of the reference's text emitter (codegen.hpp:268-675,
// emit_scpt / emit_mlt) with kernels that are actually compiled (NVRTC, jit.cpp)
// and launched.  Every kernel computes exactly the reference pipeline
// (reference_action, form.hpp:497-593):
//   gather (:498-509) -> affine jacobian + det (:511-520, :441-457)
//   -> per-qp evaluation matvecs (:526-555) -> pointwise map DAG (:561-573)
//   -> quadrature matvec (:575-585) -> scatter-add (:590-592)
// with the same per-cell operation order (j ascending in evaluation, k inner in
// quadrature).  The map DAG is emitted once per quadrature point as SSA
// (identical values to the reference's unmemoised recursion), so nvcc CSEs and
// hoists cell-invariant geometry out of the unrolled qp loop.
//
// Families (KernelPlan::family):
//   Scpt  one thread per cell; int32 SoA maps read from global; red.global.add.f64 scatter.
//   Tile  one thread per cell, one CTA per tile of consecutive cells: the tile's unique
//         DOFs/vertices are staged in shared memory (4 gathers in flight per thread) and
//         read through tile-local uint16 maps; cell results go to a shared-memory staging
//         array and are summed per DOF through a tile-local CSR (no atomics, fixed order:
//         cells ascending, as in the reference); only DOFs shared with another tile reach
//         global memory atomically, the rest are plain stores.
//   Mlt   the paper's multi-level tiling (TilingParams, qoi.hpp:23-33): N_c cells x N_WI
//         lanes per CTA, quadrature tiles T^Q, Phi/Psi tiles staged through an aliased
//         shared buffer, lanes striding qp rows (evaluation) and test rows (quadrature),
//         scatter once per (quad tile, quad row tile) (simulate.hpp:293-598 semantics).
// Basis residency (KernelPlan::basis): the packed tabulation array lives either in the
// kernel parameter bank (DFMA reads it as a c[0x0][imm] operand: zero load
// instructions) or is staged once per CTA into shared memory.
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <sstream>

#include "femgpu_internal.hpp"

namespace femgpu {

namespace {

std::string lit(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%a", v);  // exact hex-float literal
    std::string s(buf);
    if (s == "inf") return "__longlong_as_double(0x7ff0000000000000LL)";
    if (s == "-inf") return "__longlong_as_double(0xfff0000000000000LL)";
    if (s == "nan" || s == "-nan") return "__longlong_as_double(0x7ff8000000000000LL)";
    return "(" + s + ")";
}

struct Out {
    std::ostringstream s;
    int ind = 0;
    template <typename T>
    Out& operator<<(const T& v) {
        s << v;
        return *this;
    }
    Out& line(const std::string& l) {
        for (int i = 0; i < ind; ++i) s << "  ";
        s << l << "\n";
        return *this;
    }
};

// Which map nodes are reachable from the outputs; which derivative variables are used.
struct MapUse {
    std::vector<char> live;
    std::vector<char> qdep;  // node value depends on the quadrature point (derivs, weight)
    std::set<std::pair<int, int>> sd_used, vd_used;  // (space, term)
    bool uses_inv = false, uses_J = false, uses_det = false, uses_X = false;
};

MapUse analyse(const Signature& sig) {
    MapUse u;
    u.live.assign(sig.nodes.size(), 0);
    std::vector<int> stack(sig.outputs.begin(), sig.outputs.end());
    while (!stack.empty()) {
        int id = stack.back();
        stack.pop_back();
        if (u.live[id]) continue;
        u.live[id] = 1;
        const MapNode& n = sig.nodes[id];
        switch (n.op) {
            case FEMGPU_OP_SCALAR_DERIV: u.sd_used.insert({n.a, n.b}); break;
            case FEMGPU_OP_VECTOR_DERIV: u.vd_used.insert({n.a, n.b}); break;
            case FEMGPU_OP_JACOBIAN: u.uses_J = true; break;
            case FEMGPU_OP_INV_JACOBIAN: u.uses_inv = true; break;
            case FEMGPU_OP_DETERMINANT: u.uses_det = true; break;
            case FEMGPU_OP_COORD: u.uses_X = true; break;
            case FEMGPU_OP_ADD:
            case FEMGPU_OP_MUL:
                stack.push_back(n.a);
                stack.push_back(n.b);
                break;
            default: break;
        }
    }
    u.qdep.assign(sig.nodes.size(), 0);
    for (size_t id = 0; id < sig.nodes.size(); ++id) {
        const MapNode& n = sig.nodes[id];
        switch (n.op) {
            case FEMGPU_OP_SCALAR_DERIV:
            case FEMGPU_OP_VECTOR_DERIV:
            case FEMGPU_OP_WEIGHT: u.qdep[id] = 1; break;
            case FEMGPU_OP_ADD:
            case FEMGPU_OP_MUL: u.qdep[id] = u.qdep[n.a] || u.qdep[n.b]; break;
            default: break;
        }
    }
    return u;
}

// Emits the DAG nodes selected by `want` as SSA (children precede parents by validation).
template <typename TabFn>
void emit_nodes(Out& o, const Signature& sig, const MapUse& use, bool qdep_pass, const std::string& qs, TabFn TAB) {
    for (size_t id = 0; id < sig.nodes.size(); ++id) {
        if (!use.live[id] || static_cast<bool>(use.qdep[id]) != qdep_pass) continue;
        const MapNode& n = sig.nodes[id];
        std::string rhs;
        switch (n.op) {
            case FEMGPU_OP_CONSTANT: rhs = lit(n.value); break;
            case FEMGPU_OP_SCALAR_DERIV: rhs = "s" + std::to_string(n.a) + "_" + std::to_string(n.b); break;
            case FEMGPU_OP_VECTOR_DERIV: rhs = "t" + std::to_string(n.a) + "_" + std::to_string(n.b); break;
            case FEMGPU_OP_JACOBIAN: rhs = "J" + std::to_string(n.a) + "_" + std::to_string(n.b); break;
            case FEMGPU_OP_INV_JACOBIAN: rhs = "Ji" + std::to_string(n.a) + "_" + std::to_string(n.b); break;
            case FEMGPU_OP_DETERMINANT: rhs = "det"; break;
            case FEMGPU_OP_WEIGHT: rhs = TAB(std::to_string(sig.w_off) + "+(" + qs + ")"); break;
            case FEMGPU_OP_COORD: rhs = "X" + std::to_string(n.a) + "_" + std::to_string(n.b); break;
            case FEMGPU_OP_ADD: rhs = "n" + std::to_string(n.a) + " + n" + std::to_string(n.b); break;
            case FEMGPU_OP_MUL: rhs = "n" + std::to_string(n.a) + " * n" + std::to_string(n.b); break;
        }
        o.line("const double n" + std::to_string(id) + " = " + rhs + ";");
    }
}

std::string nm(const char* p, int a) { return std::string(p) + std::to_string(a); }
std::string nm(const char* p, int a, int b) { return nm(p, a) + "_" + std::to_string(b); }
std::string nm(const char* p, int a, int b, int c) { return nm(p, a, b) + "_" + std::to_string(c); }

// Emits the parameter struct shared by all families.
void emit_params(Out& o, const Signature& sig, const KernelPlan& kp, long long nt_param) {
    o.line("struct Params {");
    for (int i = 0; i < sig.ns(); ++i) o.line("  const double* x" + std::to_string(i) + "; const int* m" + std::to_string(i) + ";");
    for (int i = 0; i < sig.nv(); ++i) o.line("  const double* v" + std::to_string(i) + "; const int* vm" + std::to_string(i) + ";");
    o.line("  const int* tm; const int* cm; const double* X;");
    o.line("  double* y; unsigned long long* bad; const double* tabg;");
    if (kp.family == Family::Dmma) o.line("  const double* afr;");
    if (kp.colour) o.line("  const int* perm;");
    if (kp.family == Family::Macro)
        for (size_t g = 0; g < kp.group_entries.size(); ++g) o.line("  const int* gidx" + std::to_string(g) + ";");
    const int ngroups = kp.family == Family::Tile ? static_cast<int>(kp.group_entries.size()) : 0;
    for (int g = 0; g < ngroups; ++g)
        o.line("  const int* goff" + std::to_string(g) + "; const int* gcnt" + std::to_string(g) + "; const int* glist" +
               std::to_string(g) + "; const unsigned short* gloc" + std::to_string(g) + ";");
    o.line("  const unsigned short* roff; const unsigned short* rpos;");
    // cell0 / n_cells: the cell range [cell0, n_cells) of this launch (pipelined host actions launch
    // one slab at a time; macro: group range [cell0/G, n_cells/G)); stride / n_groups stay global
    o.line("  int n_cells; int stride; int n_tiles; int lstride; int n_groups; int cell0;");
    // zp / zn: y rows a *later* slab reaches first, zeroed by this launch (pipeline.cpp fused
    // zeroing; only in fused-zeroing kernels: two more fields cost C5-adv-P2 6 % elsewhere, see
    // profiles/r01_prologue_ab.txt)
    if (kp.zfused) o.line("  double* zp; long long zn;");
    if (nt_param > 0) o.line("  double tab[" + std::to_string(nt_param) + "];");
    o.line("};");
}

// Macro-element context: cell s of a group whose local connectivity is the
// compile-time pattern kp.mpat[group][s*entries + j] (indices into the group's unique list).
struct MacroCtx {
    int s;
    // mstage=1: per-thread shared-memory slots of the gathered values
    std::vector<long long> xslot, vslot;  // per space: first slot
    long long Xslot = 0;
};

// Per-cell body for Scpt/Tile/Macro: one thread computes one whole cell in registers.
void emit_cell_body(Out& o, const Signature& sig, const KernelPlan& kp, const MapUse& use, bool tile,
                    bool unroll_q, const MacroCtx* mc = nullptr) {
    auto pat = [&](int g, int j) { return kp.mpat[g][static_cast<size_t>(mc->s) * kp.group_entries[g] + j]; };
    const int d = sig.dim, Q = sig.Q;
    auto TAB = [&](const std::string& idx) {
        if (kp.basis == kBasisGlobal) return "__ldg(&P.tabg[" + idx + "])";
        return kp.basis == FEMGPU_BASIS_CONST ? "P.tab[" + idx + "]" : "sT[" + idx + "]";
    };
    const std::string C = "P.stride";
    // ---- gather (form.hpp:498-509)
    o.line("// gather");
    for (int i = 0; i < sig.ns(); ++i) {
        for (int j = 0; j < sig.sdofs[i]; ++j) {
            std::string idx = std::to_string(j) + "*(size_t)" + C + "+cell";
            if (mc && kp.mstage)
                o.line("const double " + nm("u", i, j) + " = SM(" + std::to_string(mc->xslot[i] + pat(kp.sgroup[i], j)) + ");");
            else if (mc)
                o.line("const double " + nm("u", i, j) + " = " + nm("xg", i, pat(kp.sgroup[i], j)) + ";");
            else if (tile && kp.sgroup[i] >= 0)
                o.line("const double " + nm("u", i, j) + " = xs" + std::to_string(i) + "[sl" +
                       std::to_string(kp.sgroup[i]) + "[" + std::to_string(j * kp.tile_cells) + " + threadIdx.x]];");
            else if (!kp.salias.empty()) {  // node index named: the scatter reuses it (salias)
                o.line("const int " + nm("sn", i, j) + " = __ldg(&P.m" + std::to_string(i) + "[" + idx + "]);");
                o.line("const double " + nm("u", i, j) + " = __ldg(&P.x" + std::to_string(i) + "[" + nm("sn", i, j) + "]);");
            } else
                o.line("const double " + nm("u", i, j) + " = __ldg(&P.x" + std::to_string(i) + "[__ldg(&P.m" +
                       std::to_string(i) + "[" + idx + "])]);");
        }
    }
    for (int i = 0; i < sig.nv(); ++i) {
        std::set<int> comps(sig.vcomps[i].begin(), sig.vcomps[i].end());
        for (int j = 0; j < sig.vdofs[i]; ++j) {
            std::string idx = std::to_string(j) + "*(size_t)" + C + "+cell";
            std::string node = nm("vn", i, j);
            if (mc) {
                for (int c : comps)
                    o.line("const double " + nm("w", i, j, c) + " = " +
                           (kp.mstage ? "SM(" + std::to_string(mc->vslot[i] + static_cast<long long>(pat(kp.vgroup[i], j)) * d + c) + ")"
                                      : nm("vg", i, pat(kp.vgroup[i], j), c)) + ";");
                continue;
            }
            if (tile && kp.vgroup[i] >= 0)
                o.line("const int " + node + " = sl" + std::to_string(kp.vgroup[i]) + "[" +
                       std::to_string(j * kp.tile_cells) + " + threadIdx.x];");
            else
                o.line("const int " + node + " = __ldg(&P.vm" + std::to_string(i) + "[" + idx + "]);");
            // padded global layout: components (0,1) as one aligned 16-byte load (no initializer on the
            // double2: the checked twin's goto may jump over it)
            const bool pair = !(tile && kp.vgroup[i] >= 0) && d >= 2 && comps.count(0) && comps.count(1);
            if (pair) {
                const std::string pv = nm("wp", i, j);
                o.line("double2 " + pv + "; " + pv + " = __ldg(reinterpret_cast<const double2*>(P.v" + std::to_string(i) +
                       " + (size_t)" + node + "*" + std::to_string(vec_stride(d)) + "));");
            }
            for (int c : comps) {
                if (tile && kp.vgroup[i] >= 0)
                    o.line("const double " + nm("w", i, j, c) + " = vs" + std::to_string(i) + "[" + node + "*" +
                           std::to_string(d) + "+" + std::to_string(c) + "];");
                else if (pair && c < 2)
                    o.line("const double " + nm("w", i, j, c) + " = " + nm("wp", i, j) + (c == 0 ? ".x;" : ".y;"));
                else
                    o.line("const double " + nm("w", i, j, c) + " = __ldg(&P.v" + std::to_string(i) + "[(size_t)" +
                           node + "*" + std::to_string(vec_stride(d)) + "+" + std::to_string(c) + "]);");
            }
        }
    }
    // ---- geometry (form.hpp:511-520, 441-457)
    if (sig.affine) {
        o.line("// coordinates + affine jacobian");
        for (int j = 0; j < sig.coord_dofs; ++j) {
            std::string idx = std::to_string(j) + "*(size_t)" + C + "+cell";
            std::string vtx = nm("cv", j);
            if (mc) {
                for (int c = 0; c < d; ++c)
                    o.line("const double " + nm("X", j, c) + " = " +
                           (kp.mstage ? "SM(" + std::to_string(mc->Xslot + static_cast<long long>(pat(kp.cgroup, j)) * d + c) + ")"
                                      : nm("Xg", pat(kp.cgroup, j), c)) + ";");
                continue;
            }
            if (tile && kp.cgroup >= 0)
                o.line("const int " + vtx + " = sl" + std::to_string(kp.cgroup) + "[" + std::to_string(j * kp.tile_cells) +
                       " + threadIdx.x];");
            else
                o.line("const int " + vtx + " = __ldg(&P.cm[" + idx + "]);");
            const bool xpair = !(tile && kp.cgroup >= 0) && d >= 2;
            if (xpair)
                o.line("double2 " + nm("Xp", j) + "; " + nm("Xp", j) + " = __ldg(reinterpret_cast<const double2*>(P.X + (size_t)" +
                       vtx + "*" + std::to_string(vec_stride(d)) + "));");
            for (int c = 0; c < d; ++c) {
                if (tile && kp.cgroup >= 0)
                    o.line("const double " + nm("X", j, c) + " = Xs[" + vtx + "*" + std::to_string(d) + "+" +
                           std::to_string(c) + "];");
                else if (xpair && c < 2)
                    o.line("const double " + nm("X", j, c) + " = " + nm("Xp", j) + (c == 0 ? ".x;" : ".y;"));
                else
                    o.line("const double " + nm("X", j, c) + " = __ldg(&P.X[(size_t)" + vtx + "*" + std::to_string(vec_stride(d)) +
                           "+" + std::to_string(c) + "]);");
            }
        }
        for (int c = 0; c < d; ++c)
            for (int r = 0; r < d; ++r)
                o.line("const double " + nm("J", r, c) + " = " + nm("X", c + 1, r) + " - " + nm("X", 0, r) + ";");
        if (d == 1) o.line("const double det = J0_0;");
        if (d == 2) o.line("const double det = J0_0 * J1_1 - J0_1 * J1_0;");
        if (d == 3)
            o.line("const double det = J0_0 * (J1_1 * J2_2 - J1_2 * J2_1) - J0_1 * (J1_0 * J2_2 - J1_2 * J2_0) + "
                   "J0_2 * (J1_0 * J2_1 - J1_1 * J2_0);");
        if (use.uses_inv) {
            if (d == 1) o.line("const double Ji0_0 = 1.0 / det;");
            if (d == 2) {
                o.line("const double Ji0_0 = J1_1 / det, Ji0_1 = -J0_1 / det, Ji1_0 = -J1_0 / det, Ji1_1 = J0_0 / det;");
            }
            if (d == 3) {
                o.line("const double Ji0_0 = (J1_1*J2_2 - J1_2*J2_1) / det, Ji0_1 = (J0_2*J2_1 - J0_1*J2_2) / det, "
                       "Ji0_2 = (J0_1*J1_2 - J0_2*J1_1) / det;");
                o.line("const double Ji1_0 = (J1_2*J2_0 - J1_0*J2_2) / det, Ji1_1 = (J0_0*J2_2 - J0_2*J2_0) / det, "
                       "Ji1_2 = (J0_2*J1_0 - J0_0*J1_2) / det;");
                o.line("const double Ji2_0 = (J1_0*J2_1 - J1_1*J2_0) / det, Ji2_1 = (J0_1*J2_0 - J0_0*J2_1) / det, "
                       "Ji2_2 = (J0_0*J1_1 - J0_1*J1_0) / det;");
            }
        }
        o.line("if (CHECKED && NF(det)) { stage = 0; goto report; }");
    }
    // ---- cell-invariant map nodes (geometry, constants), hoisted out of the qp loop
    emit_nodes(o, sig, use, false, "0", TAB);
    // ---- accumulators
    {
        std::string l = "double";
        for (int jw = 0; jw < sig.nW; ++jw) l += std::string(jw ? "," : "") + " o" + std::to_string(jw) + " = 0.0";
        o.line(l + ";");
    }
    o.line("bool nf = false;");
    const std::string q = unroll_q ? "" : "q";
    auto body_q = [&](const std::string& qs) {
        // evaluation (form.hpp:526-555)
        for (int i = 0; i < sig.ns(); ++i)
            for (int k = 0; k < sig.sterms[i]; ++k) {
                const long long base = sig.phi_off_s[i] + static_cast<long long>(k) * Q * sig.sdofs[i];
                std::string v = nm("s", i, k);
                for (int j = 0; j < sig.sdofs[i]; ++j) {
                    std::string t = TAB(std::to_string(base + j) + "+(" + qs + ")*" + std::to_string(sig.sdofs[i]));
                    if (j == 0)
                        o.line("double " + v + " = " + t + " * " + nm("u", i, j) + ";");
                    else
                        o.line(v + " = FMA(" + t + ", " + nm("u", i, j) + ", " + v + ");");
                }
            }
        for (int i = 0; i < sig.nv(); ++i)
            for (int k = 0; k < sig.vterms[i]; ++k) {
                const long long base = sig.phi_off_v[i] + static_cast<long long>(k) * Q * sig.vdofs[i];
                const int comp = sig.vcomps[i][k];
                std::string v = nm("t", i, k);
                for (int j = 0; j < sig.vdofs[i]; ++j) {
                    std::string t = TAB(std::to_string(base + j) + "+(" + qs + ")*" + std::to_string(sig.vdofs[i]));
                    if (j == 0)
                        o.line("double " + v + " = " + t + " * " + nm("w", i, j, comp) + ";");
                    else
                        o.line(v + " = FMA(" + t + ", " + nm("w", i, j, comp) + ", " + v + ");");
                }
            }
        // stage check of the evaluation results (checked kernel: every term; fast kernel:
        // terms the map never reads, the rest propagate into the outputs)
        {
            std::string all, unused;
            for (int i = 0; i < sig.ns(); ++i)
                for (int k = 0; k < sig.sterms[i]; ++k) {
                    all += " | NF(" + nm("s", i, k) + ")";
                    if (!use.sd_used.count({i, k})) unused += " | NF(" + nm("s", i, k) + ")";
                }
            for (int i = 0; i < sig.nv(); ++i)
                for (int k = 0; k < sig.vterms[i]; ++k) {
                    all += " | NF(" + nm("t", i, k) + ")";
                    if (!use.vd_used.count({i, k})) unused += " | NF(" + nm("t", i, k) + ")";
                }
            o.line("if (CHECKED && (false" + all + ")) { stage = 1; goto report; }");
            if (!unused.empty()) o.line("nf = nf" + unused + ";");
        }
        // pointwise map (form.hpp:561-573): quadrature-point-dependent nodes
        emit_nodes(o, sig, use, true, qs, TAB);
        {
            std::string chk;
            for (int k = 0; k < sig.Tw; ++k) {
                o.line("const double e" + std::to_string(k) + " = n" + std::to_string(sig.outputs[k]) + ";");
                chk += " | NF(e" + std::to_string(k) + ")";
            }
            o.line("if (CHECKED && (false" + chk + ")) { stage = 2; goto report; }");
        }
        // quadrature (form.hpp:575-585): acc = cell_out[jw]; acc += psi_k(jw,q) * e_k, k inner
        // (Psi entries zero at every point are skipped: acc + 0 * e_k == acc for finite e_k, and an
        // output no entry reads is checked on its own)
        for (int k = 0; k < sig.Tw; ++k)
            if (sig.output_dead(k)) o.line("nf = nf | NF(e" + std::to_string(k) + ");");
        for (int jw = 0; jw < sig.nW; ++jw)
            for (int k = 0; k < sig.Tw; ++k) {
                if (!sig.pnz(k, jw)) continue;
                const long long idx = sig.psi_off + (static_cast<long long>(k) * sig.nW + jw) * Q;
                o.line("o" + std::to_string(jw) + " = FMA(" + TAB(std::to_string(idx) + "+(" + qs + ")") + ", e" +
                       std::to_string(k) + ", o" + std::to_string(jw) + ");");
            }
    };
    if (unroll_q) {
        for (int iq = 0; iq < Q; ++iq) {
            o.line("{ // quadrature point " + std::to_string(iq));
            o.ind++;
            body_q(std::to_string(iq));
            o.ind--;
            o.line("}");
        }
    } else {
        o.line("#pragma unroll 1");
        o.line("for (int q = 0; q < " + std::to_string(Q) + "; ++q) {");
        o.ind++;
        body_q("q");
        o.ind--;
        o.line("}");
    }
    (void)q;
    // ---- final finiteness (quadrature stage)
    {
        std::string chk;
        for (int jw = 0; jw < sig.nW; ++jw) chk += " | NF(o" + std::to_string(jw) + ")";
        if (sig.affine) chk += " | NF(det)";
        o.line("nf = nf" + chk + ";");
        o.line("if (CHECKED && nf) { stage = 3; goto report; }");
        o.line("if (!CHECKED && nf) atomicMin(P.bad, (unsigned long long)cell);");
    }
    // ---- scatter (form.hpp:590-592)
    o.line("if (!CHECKED) {");
    o.ind++;
    for (int jw = 0; jw < sig.nW; ++jw) {
        std::string idx = std::to_string(jw) + "*(size_t)" + C + "+cell";
        std::string row = "__ldg(&P.tm[" + idx + "])";
        if (!mc && !tile && !kp.salias.empty() && kp.salias[jw][0] >= 0) {
            // row = scale * (gathered node index) + add (Instance::test_alias): no test-map load
            const auto& a = kp.salias[jw];
            row = "(" + nm(a[0] == 1 ? "vn" : "sn", static_cast<int>(a[1]), static_cast<int>(a[2])) +
                  (a[3] != 1 ? " * " + std::to_string(a[3]) : "") + (a[4] ? " + " + std::to_string(a[4]) : "") + ")";
        }
        if (mc && kp.ysmem)
            o.line("SY(" + std::to_string(pat(kp.tgroup, jw)) + ") += o" + std::to_string(jw) + ";");
        else if (mc)
            o.line(nm("ya", pat(kp.tgroup, jw)) + " += o" + std::to_string(jw) + ";");
        else if (tile)
            o.line("st[" + std::to_string(jw * kp.tile_cells) + " + threadIdx.x] = o" + std::to_string(jw) + ";");
        else if (kp.colour)  // no other cell of this launch (colour) touches the DOF
            o.line("P.y[" + row + "] += o" + std::to_string(jw) + ";");
        else if (std::getenv("FEMGPU_DEBUG_SCATTER_STORE") && !mc && !tile)  // timing experiment only (wrong results)
            o.line("P.y[" + row + "] = o" + std::to_string(jw) + ";");
        else
            o.line("atomicAdd(&P.y[" + row + "], o" + std::to_string(jw) + ");");
    }
    o.ind--;
    o.line("}");
}

const char* kPrelude = R"(// generated by femgpu (emit.cpp) for sm_100a
#define NF(v) ((((unsigned)__double2hiint(v)) & 0x7ff00000u) == 0x7ff00000u)
// acc += a*b exactly as the reference writes it; contracted to DFMA unless --fmad=false
#define FMA(a, b, acc) ((acc) + (a) * (b))
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" :: "l"(p)); }
__device__ __forceinline__ int ldidx(const int* p) {
  int v;
  asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
)";

}  // namespace

// ---- helpers shared with emit_dmma.cpp
std::vector<char> map_live(const Signature& sig) { return analyse(sig).live; }
std::vector<char> map_qdep(const Signature& sig) { return analyse(sig).qdep; }

// Emits the live map nodes of one pass (cell-invariant or quadrature-point-dependent) as SSA;
// the quadrature weight is read through `weight_expr`.
void emit_map_nodes(std::ostringstream& os, const Signature& sig, const std::vector<char>& live,
                    const std::vector<char>& qdep, bool qdep_pass, const std::string& weight_expr) {
    for (size_t id = 0; id < sig.nodes.size(); ++id) {
        if (!live[id] || static_cast<bool>(qdep[id]) != qdep_pass) continue;
        const MapNode& n = sig.nodes[id];
        std::string rhs;
        switch (n.op) {
            case FEMGPU_OP_CONSTANT: rhs = lit(n.value); break;
            case FEMGPU_OP_SCALAR_DERIV: rhs = "s" + std::to_string(n.a) + "_" + std::to_string(n.b); break;
            case FEMGPU_OP_VECTOR_DERIV: rhs = "t" + std::to_string(n.a) + "_" + std::to_string(n.b); break;
            case FEMGPU_OP_JACOBIAN: rhs = "J" + std::to_string(n.a) + "_" + std::to_string(n.b); break;
            case FEMGPU_OP_INV_JACOBIAN: rhs = "Ji" + std::to_string(n.a) + "_" + std::to_string(n.b); break;
            case FEMGPU_OP_DETERMINANT: rhs = "det"; break;
            case FEMGPU_OP_WEIGHT: rhs = weight_expr; break;
            case FEMGPU_OP_COORD: rhs = "X" + std::to_string(n.a) + "_" + std::to_string(n.b); break;
            case FEMGPU_OP_ADD: rhs = "n" + std::to_string(n.a) + " + n" + std::to_string(n.b); break;
            case FEMGPU_OP_MUL: rhs = "n" + std::to_string(n.a) + " * n" + std::to_string(n.b); break;
        }
        os << "        const double n" << id << " = " << rhs << ";\n";
    }
}

// Coordinates through the coordinate map, affine Jacobian and determinant (form.hpp:441-457,
// :511-520), optionally J^-1 (extension op 9).
void emit_geometry(std::ostringstream& os, const Signature& sig, bool uses_inv, const std::string& cell) {
    const int d = sig.dim;
    for (int j = 0; j < sig.coord_dofs; ++j) {
        os << "        const int cv" << j << " = __ldg(&P.cm[" << j << " * (size_t)P.stride + " << cell << "]);\n";
        if (d >= 2) {
            // padded layout: components (0,1) are one aligned 16-byte load
            os << "        const double2 X" << j << "_01 = __ldg(reinterpret_cast<const double2*>(P.X + (size_t)cv" << j << " * "
               << vec_stride(d) << "));\n";
            os << "        const double X" << j << "_0 = X" << j << "_01.x, X" << j << "_1 = X" << j << "_01.y;\n";
            if (d == 3)
                os << "        const double X" << j << "_2 = __ldg(&P.X[(size_t)cv" << j << " * " << vec_stride(d) << " + 2]);\n";
        } else {
            os << "        const double X" << j << "_0 = __ldg(&P.X[(size_t)cv" << j << "]);\n";
        }
    }
    for (int c = 0; c < d; ++c)
        for (int r = 0; r < d; ++r)
            os << "        const double J" << r << "_" << c << " = X" << c + 1 << "_" << r << " - X0_" << r << ";\n";
    if (d == 1) os << "        const double det = J0_0;\n";
    if (d == 2) os << "        const double det = J0_0 * J1_1 - J0_1 * J1_0;\n";
    if (d == 3)
        os << "        const double det = J0_0 * (J1_1 * J2_2 - J1_2 * J2_1) - J0_1 * (J1_0 * J2_2 - J1_2 * J2_0) + "
              "J0_2 * (J1_0 * J2_1 - J1_1 * J2_0);\n";
    if (uses_inv) {
        if (d == 1) os << "        const double Ji0_0 = 1.0 / det;\n";
        if (d == 2)
            os << "        const double Ji0_0 = J1_1 / det, Ji0_1 = -J0_1 / det, Ji1_0 = -J1_0 / det, Ji1_1 = J0_0 / det;\n";
        if (d == 3) {
            os << "        const double Ji0_0 = (J1_1*J2_2 - J1_2*J2_1) / det, Ji0_1 = (J0_2*J2_1 - J0_1*J2_2) / det, "
                  "Ji0_2 = (J0_1*J1_2 - J0_2*J1_1) / det;\n";
            os << "        const double Ji1_0 = (J1_2*J2_0 - J1_0*J2_2) / det, Ji1_1 = (J0_0*J2_2 - J0_2*J2_0) / det, "
                  "Ji1_2 = (J0_2*J1_0 - J0_0*J1_2) / det;\n";
            os << "        const double Ji2_0 = (J1_0*J2_1 - J1_1*J2_0) / det, Ji2_1 = (J0_1*J2_0 - J0_0*J2_1) / det, "
                  "Ji2_2 = (J0_0*J1_1 - J0_1*J1_0) / det;\n";
        }
    }
}

std::string KernelPlan::key() const {
    std::ostringstream s;
    s << int(family) << "/" << basis << "/" << block << "/" << tile_cells << "/" << Nc << "x" << Nwi << "/" << TQ << "/"
      << Ter << "/" << Tqr << "/" << Tqc << "/" << strict << "/" << min_blocks << "/G" << G << "/ms" << mstage << "/ys" << ysmem
      << "/qm" << qmajor << "x" << msplit << "o" << qmopt << "m" << merge.size() << "/ql" << qloop << "/col" << colour << "/zf" << zfused;
    for (int t : Tcs) s << "s" << t;
    for (int t : Tcv) s << "v" << t;
    for (size_t g = 0; g < group_cap.size(); ++g) s << "g" << group_entries[g] << ":" << group_cap[g];
    for (int g : sgroup) s << "S" << g;
    for (int g : vgroup) s << "V" << g;
    s << "T" << tgroup << "C" << cgroup << "tv" << tvec << "br" << breg;
    uint64_t h = 0xcbf29ce484222325ULL;
    for (const auto& p : mpat)
        for (int v : p) h = (h ^ static_cast<uint64_t>(v + 1)) * 0x100000001b3ULL;
    for (const auto& m : merge)
        for (int v : m) h = (h ^ static_cast<uint64_t>(v + 7)) * 0x100000001b3ULL;
    for (const auto& t : talias)
        for (long long v : t) h = (h ^ static_cast<uint64_t>(v + 11)) * 0x100000001b3ULL;
    for (const auto& t : dalias)
        for (long long v : t) h = (h ^ static_cast<uint64_t>(v + 13)) * 0x100000001b3ULL;
    for (const auto& t : salias)
        for (long long v : t) h = (h ^ static_cast<uint64_t>(v + 17)) * 0x100000001b3ULL;
    for (const auto& a : maff) {
        h = (h ^ 0x5bd1e995ULL) * 0x100000001b3ULL;
        for (int v : a) h = (h ^ static_cast<uint64_t>(v + 19)) * 0x100000001b3ULL;
    }
    s << "P" << h;
    return s.str();
}

EmitResult emit_mlt(const Signature& sig, const KernelPlan& kp);  // below
EmitResult emit_dmma(const Signature& sig, const KernelPlan& kp);  // below

// Fused zeroing (pipeline.cpp overlapped_zero_action): every CTA clears its share of the y rows
// [zp, zp + zn) before any early exit; a launch never writes those rows itself.
// Streaming stores (st.global.cs, evict-first): the zeroed rows are not read by this launch, so they
// must not displace the gathered lines in L2.
const char* kZeroPrologue =
    "if (P.zn > 0) {\n"
    "  const long long zper = (P.zn + gridDim.x - 1) / gridDim.x, z0 = (long long)blockIdx.x * zper;\n"
    "  const long long z1 = min(z0 + zper, P.zn);\n"
    "  for (long long i = z0 + threadIdx.x; i < z1; i += blockDim.x) __stcs(P.zp + i, 0.0);\n"
    "}\n";

namespace {

std::string S(long long v) { return std::to_string(v); }

// Checked (diagnostic) or plain SCPT kernel: one thread per cell, int32 SoA maps.
void emit_scpt_kernel(Out& o, const Signature& sig, const KernelPlan& kp, const MapUse& use, bool unroll_q,
                      bool checked, const std::string& name, long long smem_tab_off) {
    KernelPlan p = kp;
    p.family = Family::Scpt;
    o.line("");
    std::string bounds = checked ? "" : "__launch_bounds__(" + S(kp.block) + (kp.min_blocks > 1 ? ", " + S(kp.min_blocks) : "") + ") ";
    o.line("extern \"C\" __global__ void " + bounds + name + "(const __grid_constant__ Params P) {");
    o.ind++;
    o.line(std::string("constexpr bool CHECKED = ") + (checked ? "true" : "false") + ";");
    if (!checked && kp.zfused) o << kZeroPrologue;
    if (kp.basis == FEMGPU_BASIS_SMEM) {
        o.line("extern __shared__ __align__(16) unsigned char smraw[];");
        o.line("double* sT = reinterpret_cast<double*>(smraw + " + S(smem_tab_off) + ");");
        o.line("for (int i = threadIdx.x; i < " + S(sig.tab_size) + "; i += blockDim.x) sT[i] = P.tabg[i];");
        o.line("__syncthreads();");
    }
    if (kp.colour && !checked) {
        // colour launch: positions [cell0, n_cells) of the colour-sorted permutation
        o.line("const int ci = P.cell0 + blockIdx.x * blockDim.x + threadIdx.x;");
        o.line("const int cell = ci < P.n_cells ? __ldg(&P.perm[ci]) : 0;");
        o.line("int stage = -1; (void)stage;");
        o.line("if (ci < P.n_cells) {");
        o.ind++;
    } else {
        o.line("const int cell = P.cell0 + blockIdx.x * blockDim.x + threadIdx.x;");
        o.line("int stage = -1; (void)stage;");
        o.line("if (cell < P.n_cells) {");
        o.ind++;
    }
    emit_cell_body(o, sig, p, use, false, unroll_q);
    o.ind--;
    o.line("}");
    o.line("return;");
    o.line("report:");
    o.line("  atomicMin(P.bad, (unsigned long long)cell * 4ull + (unsigned long long)stage);");
    o.ind--;
    o.line("}");
}

// SCPT with G independent cells per thread (cells c0 + k*blockDim, k < G, coalesced per k):
// the per-cell statements are interleaved so that every tabulation operand (constant bank or
// shared memory, one LDCU/LDS per DFMA in the one-cell kernel) is loaded once for G cells, and
// the G cells give the scheduler independent DFMA chains.  No connectivity pattern is needed
// (unlike the macro family); each cell keeps the reference's own operation order.
void emit_scpt_multi_kernel(Out& o, const Signature& sig, const KernelPlan& kp, const MapUse& use, bool unroll_q,
                            const std::string& name, long long smem_tab_off) {
    const int G = kp.G, d = sig.dim, Q = sig.Q;
    auto TAB = [&](const std::string& idx) {
        if (kp.basis == kBasisGlobal) return "__ldg(&P.tabg[" + idx + "])";
        return kp.basis == FEMGPU_BASIS_CONST ? "P.tab[" + idx + "]" : "sT[" + idx + "]";
    };
    auto K = [](const std::string& v, int k) { return v + "_c" + std::to_string(k); };
    // cell-invariant nodes the quadrature-point part reads (constants are re-emitted per cell)
    std::set<int> need;
    for (size_t id = 0; id < sig.nodes.size(); ++id) {
        if (!use.live[id] || !use.qdep[id]) continue;
        const MapNode& n = sig.nodes[id];
        if (n.op == FEMGPU_OP_ADD || n.op == FEMGPU_OP_MUL) {
            if (!use.qdep[n.a]) need.insert(n.a);
            if (!use.qdep[n.b]) need.insert(n.b);
        }
    }
    for (int out : sig.outputs)
        if (!use.qdep[out]) need.insert(out);
    o.line("");
    o.line("extern \"C\" __global__ void __launch_bounds__(" + S(kp.block) + (kp.min_blocks > 1 ? ", " + S(kp.min_blocks) : "") +
           ") " + name + "(const __grid_constant__ Params P) {");
    o.ind++;
    o.line("constexpr bool CHECKED = false;");
    if (kp.zfused) o << kZeroPrologue;
    if (kp.basis == FEMGPU_BASIS_SMEM) {
        o.line("extern __shared__ __align__(16) unsigned char smraw[];");
        o.line("double* sT = reinterpret_cast<double*>(smraw + " + S(smem_tab_off) + ");");
        o.line("for (int i = threadIdx.x; i < " + S(sig.tab_size) + "; i += blockDim.x) sT[i] = P.tabg[i];");
        o.line("__syncthreads();");
    }
    o.line("const int cbase = P.cell0 + blockIdx.x * " + S(G) + " * blockDim.x + threadIdx.x;");
    o.line("if (cbase >= P.n_cells) return;");
    for (int k = 0; k < G; ++k) {
        o.line("const bool ok_c" + S(k) + " = cbase + " + S(k) + " * (int)blockDim.x < P.n_cells;");
        o.line("const int cell_c" + S(k) + " = ok_c" + S(k) + " ? cbase + " + S(k) + " * (int)blockDim.x : cbase;");
    }
    // ---- per cell: gather, geometry, cell-invariant nodes (kept in hk<k>_<id>)
    for (int k = 0; k < G; ++k) {
        o.line("bool nf_c" + S(k) + " = false;");
        for (int i = 0; i < sig.ns(); ++i)
            for (int j = 0; j < sig.sdofs[i]; ++j)
                o.line("const double " + K(nm("u", i, j), k) + " = __ldg(&P.x" + S(i) + "[__ldg(&P.m" + S(i) + "[" + S(j) +
                       "*(size_t)P.stride + cell_c" + S(k) + "])]);");
        for (int i = 0; i < sig.nv(); ++i) {
            std::set<int> comps(sig.vcomps[i].begin(), sig.vcomps[i].end());
            for (int j = 0; j < sig.vdofs[i]; ++j) {
                const std::string node = K(nm("vn", i, j), k);
                o.line("const int " + node + " = __ldg(&P.vm" + S(i) + "[" + S(j) + "*(size_t)P.stride + cell_c" + S(k) + "]);");
                for (int c : comps)
                    o.line("const double " + K(nm("w", i, j, c), k) + " = __ldg(&P.v" + S(i) + "[(size_t)" + node + "*" +
                           S(vec_stride(d)) + "+" + S(c) + "]);");
            }
        }
        for (int id : need) o.line("double " + K("hk" + S(id), k) + ";");
        o.line("{");
        o.ind++;
        if (sig.affine) {
            std::ostringstream g;
            emit_geometry(g, sig, use.uses_inv, "cell_c" + S(k));
            std::istringstream gl(g.str());
            std::string line;
            while (std::getline(gl, line)) o.line(line.substr(line.find_first_not_of(' ')));
            o.line("nf_c" + S(k) + " = NF(det);");
        }
        emit_nodes(o, sig, use, false, "0", TAB);
        for (int id : need) o.line(K("hk" + S(id), k) + " = n" + S(id) + ";");
        o.ind--;
        o.line("}");
        {
            std::string l = "double";
            for (int jw = 0; jw < sig.nW; ++jw) l += std::string(jw ? "," : "") + " " + K("o" + S(jw), k) + " = 0.0";
            o.line(l + ";");
        }
    }
    auto body_q = [&](const std::string& qs) {
        // evaluation: one tabulation load per (term, j) for all G cells
        for (int i = 0; i < sig.ns(); ++i)
            for (int t = 0; t < sig.sterms[i]; ++t) {
                const long long base = sig.phi_off_s[i] + static_cast<long long>(t) * Q * sig.sdofs[i];
                for (int k = 0; k < G; ++k) o.line("double " + K(nm("s", i, t), k) + ";");
                for (int j = 0; j < sig.sdofs[i]; ++j) {
                    std::string l = "{ const double tb = " + TAB(S(base + j) + "+(" + qs + ")*" + S(sig.sdofs[i])) + ";";
                    for (int k = 0; k < G; ++k) {
                        const std::string v = K(nm("s", i, t), k), u = K(nm("u", i, j), k);
                        l += j == 0 ? " " + v + " = tb * " + u + ";" : " " + v + " = FMA(tb, " + u + ", " + v + ");";
                    }
                    o.line(l + " }");
                }
            }
        for (int i = 0; i < sig.nv(); ++i)
            for (int t = 0; t < sig.vterms[i]; ++t) {
                const long long base = sig.phi_off_v[i] + static_cast<long long>(t) * Q * sig.vdofs[i];
                const int comp = sig.vcomps[i][t];
                for (int k = 0; k < G; ++k) o.line("double " + K(nm("t", i, t), k) + ";");
                for (int j = 0; j < sig.vdofs[i]; ++j) {
                    std::string l = "{ const double tb = " + TAB(S(base + j) + "+(" + qs + ")*" + S(sig.vdofs[i])) + ";";
                    for (int k = 0; k < G; ++k) {
                        const std::string v = K(nm("t", i, t), k), w = K(nm("w", i, j, comp), k);
                        l += j == 0 ? " " + v + " = tb * " + w + ";" : " " + v + " = FMA(tb, " + w + ", " + v + ");";
                    }
                    o.line(l + " }");
                }
            }
        // pointwise map per cell (same SSA as the one-cell kernel), outputs into e<kt>_c<k>
        for (int k = 0; k < G; ++k) {
            for (int kt = 0; kt < sig.Tw; ++kt) o.line("double " + K("e" + S(kt), k) + ";");
            o.line("{");
            o.ind++;
            std::string unused;
            for (int i = 0; i < sig.ns(); ++i)
                for (int t = 0; t < sig.sterms[i]; ++t) {
                    o.line("const double " + nm("s", i, t) + " = " + K(nm("s", i, t), k) + ";");
                    if (!use.sd_used.count({i, t})) unused += " | NF(" + nm("s", i, t) + ")";
                }
            for (int i = 0; i < sig.nv(); ++i)
                for (int t = 0; t < sig.vterms[i]; ++t) {
                    o.line("const double " + nm("t", i, t) + " = " + K(nm("t", i, t), k) + ";");
                    if (!use.vd_used.count({i, t})) unused += " | NF(" + nm("t", i, t) + ")";
                }
            if (!unused.empty()) o.line("nf_c" + S(k) + " = nf_c" + S(k) + unused + ";");
            for (int id : need) {
                if (sig.nodes[id].op == FEMGPU_OP_CONSTANT) o.line("const double n" + S(id) + " = " + lit(sig.nodes[id].value) + ";");
                else o.line("const double n" + S(id) + " = " + K("hk" + S(id), k) + ";");
            }
            emit_nodes(o, sig, use, true, qs, TAB);
            for (int kt = 0; kt < sig.Tw; ++kt) o.line(K("e" + S(kt), k) + " = n" + S(sig.outputs[kt]) + ";");
            o.ind--;
            o.line("}");
        }
        // quadrature: one Psi load per (jw, term) for all G cells, k inner as in the reference
        // (all-zero Psi entries skipped, see emit_cell_body)
        for (int kt = 0; kt < sig.Tw; ++kt)
            if (sig.output_dead(kt))
                for (int k = 0; k < G; ++k) o.line("nf_c" + S(k) + " = nf_c" + S(k) + " | NF(" + K("e" + S(kt), k) + ");");
        for (int jw = 0; jw < sig.nW; ++jw)
            for (int kt = 0; kt < sig.Tw; ++kt) {
                if (!sig.pnz(kt, jw)) continue;
                const long long idx = sig.psi_off + (static_cast<long long>(kt) * sig.nW + jw) * Q;
                std::string l = "{ const double tb = " + TAB(S(idx) + "+(" + qs + ")") + ";";
                for (int k = 0; k < G; ++k)
                    l += " " + K("o" + S(jw), k) + " = FMA(tb, " + K("e" + S(kt), k) + ", " + K("o" + S(jw), k) + ");";
                o.line(l + " }");
            }
    };
    if (unroll_q) {
        for (int iq = 0; iq < Q; ++iq) {
            o.line("{ // quadrature point " + S(iq));
            o.ind++;
            body_q(S(iq));
            o.ind--;
            o.line("}");
        }
    } else {
        o.line("#pragma unroll 1");
        o.line("for (int q = 0; q < " + S(Q) + "; ++q) {");
        o.ind++;
        body_q("q");
        o.ind--;
        o.line("}");
    }
    // ---- finiteness + scatter per cell
    for (int k = 0; k < G; ++k) {
        std::string chk;
        for (int jw = 0; jw < sig.nW; ++jw) chk += " | NF(" + K("o" + S(jw), k) + ")";
        o.line("if (ok_c" + S(k) + ") {");
        o.ind++;
        o.line("if (nf_c" + S(k) + chk + ") atomicMin(P.bad, (unsigned long long)cell_c" + S(k) + ");");
        for (int jw = 0; jw < sig.nW; ++jw)
            o.line("atomicAdd(&P.y[__ldg(&P.tm[" + S(jw) + "*(size_t)P.stride + cell_c" + S(k) + "])], " + K("o" + S(jw), k) + ");");
        o.ind--;
        o.line("}");
    }
    o.line("(void)CHECKED;");
    o.ind--;
    o.line("}");
}

// Shared-memory plan of the pipelined tile kernel (bytes, 16-byte aligned regions).
struct TilePlan {
    struct Item {
        std::string dst, src;
        int group, comps;
        long long off;  // within a buffer
    };
    std::vector<Item> items;            // gathered values per buffer
    std::vector<int> gather_groups;     // groups whose local map the cell body reads
    std::map<int, long long> sloc_off;  // per gather group, within a buffer
    long long slist_off = 0, sroff_off = 0, srpos_off = 0;
    long long tab_off = -1, st_off = 0, buf0 = 0, buf_bytes = 0, total = 0;
};

long long al16(long long v) { return (v + 15) / 16 * 16; }

TilePlan plan_tile(const Signature& sig, const KernelPlan& kp) {
    TilePlan t;
    const int TB = kp.tile_cells, D = sig.dim;
    long long off = 0;
    if (kp.basis == FEMGPU_BASIS_SMEM) {
        t.tab_off = off;
        off = al16(off + sig.tab_size * 8);
    }
    t.st_off = off;
    off = al16(off + 8LL * sig.nW * TB);
    t.buf0 = off;
    long long b = 0;
    auto add_group = [&](int g) {
        if (std::find(t.gather_groups.begin(), t.gather_groups.end(), g) == t.gather_groups.end())
            t.gather_groups.push_back(g);
    };
    for (int i = 0; i < sig.ns(); ++i) {
        t.items.push_back({"xs" + S(i), "P.x" + S(i), kp.sgroup[i], 1, 0});
        add_group(kp.sgroup[i]);
    }
    for (int i = 0; i < sig.nv(); ++i) {
        t.items.push_back({"vs" + S(i), "P.v" + S(i), kp.vgroup[i], D, 0});
        add_group(kp.vgroup[i]);
    }
    if (sig.affine) {
        t.items.push_back({"Xs", "P.X", kp.cgroup, D, 0});
        add_group(kp.cgroup);
    }
    for (auto& it : t.items) {
        it.off = b;
        b = al16(b + 8LL * kp.group_cap[it.group] * it.comps);
    }
    for (int g : t.gather_groups) {
        t.sloc_off[g] = b;
        b = al16(b + 2LL * kp.group_entries[g] * TB);
    }
    const long long capt = (kp.group_cap[kp.tgroup] + 3) / 4 * 4;
    t.slist_off = b;
    b = al16(b + 4 * capt);
    t.sroff_off = b;
    b = al16(b + 2 * capt);
    t.srpos_off = b;
    b = al16(b + 2LL * TB * sig.nW);
    t.buf_bytes = b;
    t.total = off + 2 * b;
    return t;
}

// The persistent, double-buffered tile kernel.  Per iteration (tile t, next tile tn):
//   wait for buffer[cur]; prefetch (cp.async) tn's local maps, CSR and test list into
//   buffer[nxt] and load tn's gather lists into registers; compute t's cells from smem
//   into the staging array; issue tn's value gathers (cp.async x[list], coords[list]);
//   reduce t per DOF through the CSR and write y (plain store, or red.add if shared).
void emit_tile_kernel(Out& o, const Signature& sig, const KernelPlan& kp, const MapUse& use, bool unroll_q,
                      const TilePlan& T, const std::string& name) {
    const int TB = kp.tile_cells;
    const int nW = sig.nW;
    o.line("");
    std::string bounds = "__launch_bounds__(" + S(TB) + (kp.min_blocks > 1 ? ", " + S(kp.min_blocks) : "") + ") ";
    o.line("extern \"C\" __global__ void " + bounds + name + "(const __grid_constant__ Params P) {");
    o.ind++;
    o.line("constexpr bool CHECKED = false;");
    o.line("extern __shared__ __align__(16) unsigned char smraw[];");
    if (kp.basis == FEMGPU_BASIS_SMEM) {
        o.line("double* sT = reinterpret_cast<double*>(smraw + " + S(T.tab_off) + ");");
        o.line("for (int i = threadIdx.x; i < " + S(sig.tab_size) + "; i += " + S(TB) + ") sT[i] = P.tabg[i];");
    }
    o.line("double* st = reinterpret_cast<double*>(smraw + " + S(T.st_off) + ");");
    o.line("const int tid = threadIdx.x;");
    o.line("int t = blockIdx.x;");
    o.line("if (t >= P.n_tiles) return;");
    // list registers per gather group
    std::map<int, int> K;
    for (int g : T.gather_groups) {
        K[g] = (kp.group_cap[g] + TB - 1) / TB;
        o.line("int gl" + S(g) + "[" + S(K[g]) + "];");
    }
    // --- helper lambdas (emitted as macros over a buffer base)
    auto emit_meta = [&](const std::string& tile, const std::string& base) {
        // local maps of the gather groups: entries rows of TB uint16 (16-byte chunks)
        for (int g : T.gather_groups) {
            const int ent = kp.group_entries[g];
            const long long chunks_per_row = 2LL * TB / 16;
            o.line("for (int c = tid; c < " + S(ent * chunks_per_row) + "; c += " + S(TB) + ") {");
            o.line("  const int j = c / " + S(chunks_per_row) + ", k = c % " + S(chunks_per_row) + ";");
            o.line("  cp16(" + base + " + " + S(T.sloc_off.at(g)) + " + (j * " + S(TB) + ") * 2 + k * 16, P.gloc" + S(g) +
                   " + (size_t)j * P.lstride + (size_t)" + tile + " * " + S(TB) + " + k * 8);");
            o.line("}");
        }
        const std::string G = S(kp.tgroup);
        o.line("{");
        o.line("  const int lb = __ldg(&P.goff" + G + "[" + tile + "]), ln = __ldg(&P.gcnt" + G + "[" + tile + "]);");
        o.line("  for (int c = tid; c < (ln + 3) / 4; c += " + S(TB) + ") cp16(" + base + " + " + S(T.slist_off) +
               " + c * 16, P.glist" + G + " + lb + c * 4);");
        o.line("  for (int c = tid; c < (ln + 3) / 4; c += " + S(TB) + ") cp8(" + base + " + " + S(T.sroff_off) +
               " + c * 8, P.roff + lb + c * 4);");
        o.line("  const int tc = min(" + S(TB) + ", P.n_cells - " + tile + " * " + S(TB) + ");");
        o.line("  for (int c = tid; c < (tc * " + S(nW) + " + 7) / 8; c += " + S(TB) + ") cp16(" + base + " + " +
               S(T.srpos_off) + " + c * 16, P.rpos + (size_t)" + tile + " * " + S(TB * nW) + " + c * 8);");
        o.line("}");
    };
    auto emit_lists = [&](const std::string& tile) {
        for (int g : T.gather_groups) {
            o.line("{");
            o.line("  const int lb = __ldg(&P.goff" + S(g) + "[" + tile + "]), ln = __ldg(&P.gcnt" + S(g) + "[" + tile + "]);");
            o.line("  #pragma unroll");
            o.line("  for (int k = 0; k < " + S(K[g]) + "; ++k) { const int u = tid + k * " + S(TB) + "; gl" + S(g) +
                   "[k] = u < ln ? (__ldg(&P.glist" + S(g) + "[lb + u]) & 0x7fffffff) : -1; }");
            o.line("}");
        }
    };
    auto emit_gathers = [&](const std::string& base) {
        for (const auto& it : T.items) {
            o.line("#pragma unroll");
            o.line("for (int k = 0; k < " + S(K[it.group]) + "; ++k) if (gl" + S(it.group) + "[k] >= 0) {");
            o.line("  const int u = tid + k * " + S(TB) + ";");
            for (int c = 0; c < it.comps; ++c)
                o.line("  cp8(" + base + " + " + S(it.off) + " + (u * " + S(it.comps) + " + " + S(c) + ") * 8, " + it.src +
                       " + (size_t)gl" + S(it.group) + "[k] * " + S(it.comps == 1 ? 1 : vec_stride(it.comps)) + " + " + S(c) + ");");
            o.line("}");
        }
    };
    // prologue: tile t into buffer 0
    o.line("unsigned char* const buf0 = smraw + " + S(T.buf0) + ";");
    emit_meta("t", "buf0");
    emit_lists("t");
    emit_gathers("buf0");
    o.line("cp_commit();");
    o.line("int cur = 0;");
    o.line("for (;;) {");
    o.ind++;
    o.line("const int tn = t + gridDim.x;");
    o.line("cp_wait_all();");
    o.line("__syncthreads();");
    o.line("unsigned char* B = buf0 + cur * " + S(T.buf_bytes) + ";");
    o.line("unsigned char* N = buf0 + (cur ^ 1) * " + S(T.buf_bytes) + ";");
    o.line("if (tn < P.n_tiles) {");
    o.ind++;
    emit_meta("tn", "N");
    emit_lists("tn");
    o.ind--;
    o.line("}");
    // compute tile t
    for (const auto& it : T.items)
        o.line("const double* " + it.dst + " = reinterpret_cast<const double*>(B + " + S(it.off) + ");");
    for (int g : T.gather_groups)
        o.line("const unsigned short* sl" + S(g) + " = reinterpret_cast<const unsigned short*>(B + " +
               S(T.sloc_off.at(g)) + ");");
    o.line("const int cell = t * " + S(TB) + " + tid;");
    o.line("int stage = -1; (void)stage;");
    o.line("if (cell < P.n_cells) {");
    o.ind++;
    emit_cell_body(o, sig, kp, use, true, unroll_q);
    o.ind--;
    o.line("}");
    o.line("if (tn < P.n_tiles) {");
    o.ind++;
    emit_gathers("N");
    o.ind--;
    o.line("}");
    o.line("cp_commit();");
    o.line("__syncthreads();");
    // reduce tile t
    o.line("{");
    o.ind++;
    o.line("const int ln = __ldg(&P.gcnt" + S(kp.tgroup) + "[t]);");
    o.line("const int tc = min(" + S(TB) + ", P.n_cells - t * " + S(TB) + ");");
    o.line("const int* slist = reinterpret_cast<const int*>(B + " + S(T.slist_off) + ");");
    o.line("const unsigned short* sroff = reinterpret_cast<const unsigned short*>(B + " + S(T.sroff_off) + ");");
    o.line("const unsigned short* srpos = reinterpret_cast<const unsigned short*>(B + " + S(T.srpos_off) + ");");
    o.line("for (int u = tid; u < ln; u += " + S(TB) + ") {");
    o.line("  const int e = slist[u];");
    o.line("  const int r0 = sroff[u], r1 = u + 1 < ln ? (int)sroff[u + 1] : tc * " + S(nW) + ";");
    o.line("  double s = 0.0;");
    o.line("  for (int r = r0; r < r1; ++r) s += st[srpos[r]];");
    o.line("  if (e < 0) atomicAdd(&P.y[e & 0x7fffffff], s); else P.y[e] = s;");
    o.line("}");
    o.ind--;
    o.line("}");
    o.line("if (tn >= P.n_tiles) break;");
    o.line("t = tn;");
    o.line("cur ^= 1;");
    o.ind--;
    o.line("}");
    o.line("return;");
    o.line("report:");
    o.line("  return;");
    o.ind--;
    o.line("}");
}

// Affine index pattern of a map group (MacroLayout::aoff): one index load per cell group, the
// unique nodes at compile-time offsets from it (address arithmetic folds into the loads' immediates).
bool macro_affine(const KernelPlan& kp, int g) {
    return g >= 0 && static_cast<size_t>(g) < kp.maff.size() && !kp.maff[g].empty();
}

void emit_macro_bases(Out& o, const KernelPlan& kp, const std::set<int>& gathered) {
    std::set<int> gs = gathered;
    gs.insert(kp.tgroup);
    for (int g : gs)
        if (macro_affine(kp, g)) o.line("const int igb" + S(g) + " = __ldg(&P.gidx" + S(g) + "[grp]);");
}

std::string macro_index(const KernelPlan& kp, int g, int u) {
    if (!macro_affine(kp, g)) return "__ldg(&P.gidx" + S(g) + "[" + S(u) + " * NG + grp])";
    const int off = kp.maff[g][u];
    return off ? "(igb" + S(g) + " + " + S(off) + ")" : "igb" + S(g);
}

// Macro-element kernel: one thread per group of G cells sharing the compile-time pattern.
// Gathers each unique node of the group once, computes the G cells in order with the
// per-cell operation order of the reference, accumulates y per unique node in registers
// (cells ascending), and issues one red.global.add.f64 per unique test DOF.
void emit_macro_kernel(Out& o, const Signature& sig, const KernelPlan& kp, const MapUse& use, bool unroll_q,
                       const std::string& name, long long smem_tab_off, long long ysmem_off = 0) {
    const int D = sig.dim;
    o.line("");
    std::string bounds = "__launch_bounds__(" + S(kp.block) + (kp.min_blocks > 1 ? ", " + S(kp.min_blocks) : "") + ") ";
    o.line("extern \"C\" __global__ void " + bounds + name + "(const __grid_constant__ Params P) {");
    o.ind++;
    o.line("constexpr bool CHECKED = false;");
    if (kp.zfused) o << kZeroPrologue;
    if (kp.basis == FEMGPU_BASIS_SMEM) {
        o.line("extern __shared__ __align__(16) unsigned char smraw[];");
        o.line("double* sT = reinterpret_cast<double*>(smraw + " + S(smem_tab_off) + ");");
        o.line("for (int i = threadIdx.x; i < " + S(sig.tab_size) + "; i += blockDim.x) sT[i] = P.tabg[i];");
        o.line("__syncthreads();");
    }
    if (kp.mstage) {
        if (kp.basis != FEMGPU_BASIS_SMEM) o.line("extern __shared__ __align__(16) unsigned char smraw[];");
        o.line("volatile double* const sm_base = reinterpret_cast<volatile double*>(smraw + " + S(smem_tab_off + (kp.basis == FEMGPU_BASIS_SMEM ? al16(sig.tab_size * 8) : 0)) + ") + threadIdx.x;");
        o.line("#define SM(k) sm_base[(k) * " + S(kp.block) + "]");
        o.line("#define cp8s(k, src) cp8(const_cast<unsigned char*>(reinterpret_cast<volatile unsigned char*>(&SM(k))), (src))");
    }
    if (kp.ysmem) {
        if (kp.basis != FEMGPU_BASIS_SMEM && !kp.mstage) o.line("extern __shared__ __align__(16) unsigned char smraw[];");
        o.line("double* const sy_base = reinterpret_cast<double*>(smraw + " + S(ysmem_off) + ") + threadIdx.x;");
    }
    o.line("const int grp = P.cell0 / " + S(kp.G) + " + blockIdx.x * " + S(kp.block) + " + threadIdx.x;");
    o.line("if (grp >= P.n_cells / " + S(kp.G) + ") return;");
    o.line("const size_t NG = (size_t)P.n_groups;");
    // gathers: unique global indices per group, then values
    std::set<int> gathered;
    for (int i = 0; i < sig.ns(); ++i) gathered.insert(kp.sgroup[i]);
    for (int i = 0; i < sig.nv(); ++i) gathered.insert(kp.vgroup[i]);
    if (sig.affine) gathered.insert(kp.cgroup);
    emit_macro_bases(o, kp, gathered);
    // streaming order (mstage == 0): a unique node is loaded just before the first cell of the
    // group that reads it, and its y contribution is issued right after the last cell that
    // writes it, so register live ranges follow the cells instead of spanning the group.
    auto first_use = [&](int g, int u) {
        const int E = kp.group_entries[g];
        for (int s = 0; s < kp.G; ++s)
            for (int j = 0; j < E; ++j)
                if (kp.mpat[g][static_cast<size_t>(s) * E + j] == u) return s;
        return 0;
    };
    auto last_use = [&](int g, int u) {
        const int E = kp.group_entries[g];
        for (int s = kp.G - 1; s >= 0; --s)
            for (int j = 0; j < E; ++j)
                if (kp.mpat[g][static_cast<size_t>(s) * E + j] == u) return s;
        return kp.G - 1;
    };
    const bool stream = !kp.mstage;
    auto emit_loads = [&](int s_now) {
        for (int g : gathered)
            for (int u = 0; u < kp.group_cap[g]; ++u) {
                if (stream && first_use(g, u) != s_now) continue;
                o.line("const int ig" + S(g) + "_" + S(u) + " = " + macro_index(kp, g, u) + ";");
                if (kp.mstage) continue;
                for (int i = 0; i < sig.ns(); ++i)
                    if (kp.sgroup[i] == g)
                        o.line("const double xg" + S(i) + "_" + S(u) + " = __ldg(&P.x" + S(i) + "[ig" + S(g) + "_" + S(u) + "]);");
                // padded node-major layout: components (0,1) come as one aligned 16-byte load
                auto node_loads = [&](const std::string& dst, const std::string& arr, const std::set<int>& comps) {
                    const std::string base = arr + " + (size_t)ig" + S(g) + "_" + S(u) + " * " + S(vec_stride(D));
                    const bool pair = D >= 2 && comps.count(0) && comps.count(1);
                    if (pair) {
                        // (no initializer: the checked twin's goto may jump over this declaration)
                        o.line("double2 " + dst + "_01; " + dst + "_01 = __ldg(reinterpret_cast<const double2*>(" + base + "));");
                        o.line("const double " + dst + "_0 = " + dst + "_01.x, " + dst + "_1 = " + dst + "_01.y;");
                    }
                    for (int c : comps)
                        if (!pair || c >= 2) o.line("const double " + dst + "_" + S(c) + " = __ldg(" + base + " + " + S(c) + ");");
                };
                for (int i = 0; i < sig.nv(); ++i)
                    if (kp.vgroup[i] == g) {
                        std::set<int> comps(sig.vcomps[i].begin(), sig.vcomps[i].end());
                        node_loads("vg" + S(i) + "_" + S(u), "P.v" + S(i), comps);
                    }
                if (sig.affine && kp.cgroup == g) {
                    std::set<int> comps;
                    for (int c = 0; c < D; ++c) comps.insert(c);
                    node_loads("Xg" + S(u), "P.X", comps);
                }
            }
    };
    const int gt = kp.tgroup;
    auto emit_reds = [&](int s_now) {
        for (int u = 0; u < kp.group_cap[gt]; ++u) {
            if (stream && last_use(gt, u) != s_now) continue;
            std::string idx = gathered.count(gt) ? "ig" + S(gt) + "_" + S(u) : macro_index(kp, gt, u);
            if (!kp.talias.empty() && kp.talias[u][0] >= 0 && !kp.mstage) {  // row = scale * gathered node + add
                const auto& al = kp.talias[u];
                idx = "(ig" + S(al[0]) + "_" + S(al[1]) + (al[2] != 1 ? " * " + S(al[2]) : "") + (al[3] ? " + " + S(al[3]) : "") + ")";
            }
            o.line("atomicAdd(&P.y[" + idx + "], " + (kp.ysmem ? "SY(" + S(u) + ")" : "ya" + S(u)) + ");");
        }
    };
    MacroCtx base{0, {}, {}, 0};
    if (kp.mstage) {
        emit_loads(-1);
        // thread-private slots [slot][blockDim] (conflict-free), filled with cp.async
        long long slot = 0;
        std::vector<std::string> copies;
        for (int i = 0; i < sig.ns(); ++i) {
            base.xslot.push_back(slot);
            for (int u = 0; u < kp.group_cap[kp.sgroup[i]]; ++u)
                copies.push_back("cp8s(" + S(slot + u) + ", P.x" + S(i) + " + ig" + S(kp.sgroup[i]) + "_" + S(u) + ");");
            slot += kp.group_cap[kp.sgroup[i]];
        }
        for (int i = 0; i < sig.nv(); ++i) {
            base.vslot.push_back(slot);
            for (int u = 0; u < kp.group_cap[kp.vgroup[i]]; ++u)
                for (int c = 0; c < D; ++c)
                    copies.push_back("cp8s(" + S(slot + static_cast<long long>(u) * D + c) + ", P.v" + S(i) + " + (size_t)ig" +
                                     S(kp.vgroup[i]) + "_" + S(u) + " * " + S(vec_stride(D)) + " + " + S(c) + ");");
            slot += static_cast<long long>(kp.group_cap[kp.vgroup[i]]) * D;
        }
        if (sig.affine) {
            base.Xslot = slot;
            for (int u = 0; u < kp.group_cap[kp.cgroup]; ++u)
                for (int c = 0; c < D; ++c)
                    copies.push_back("cp8s(" + S(slot + static_cast<long long>(u) * D + c) + ", P.X + (size_t)ig" +
                                     S(kp.cgroup) + "_" + S(u) + " * " + S(vec_stride(D)) + " + " + S(c) + ");");
            slot += static_cast<long long>(kp.group_cap[kp.cgroup]) * D;
        }
        for (const auto& c : copies) o.line(c);
        o.line("cp_commit();");
        o.line("cp_wait_all();");
    }
    if (kp.ysmem) {
        // y accumulators in a thread-private shared-memory column (conflict-free), freeing registers
        o.line("#define SY(k) sy_base[(k) * " + S(kp.block) + "]");
        for (int u = 0; u < kp.group_cap[gt]; ++u) o.line("SY(" + S(u) + ") = 0.0;");
    } else {
        std::string l = "double";
        for (int u = 0; u < kp.group_cap[gt]; ++u) l += std::string(u ? "," : "") + " ya" + S(u) + " = 0.0";
        o.line(l + ";");
    }
    o.line("int stage = -1; (void)stage;");
    for (int s = 0; s < kp.G; ++s) {
        if (stream) emit_loads(s);
        o.line("{ // cell " + S(s) + " of the group");
        o.ind++;
        o.line("const int cell = grp * " + S(kp.G) + " + " + S(s) + ";");
        MacroCtx mc = base;
        mc.s = s;
        emit_cell_body(o, sig, kp, use, false, unroll_q, &mc);
        o.ind--;
        o.line("}");
        if (stream) emit_reds(s);
    }
    if (!stream) emit_reds(-1);
    o.line("return;");
    o.line("report:");
    o.line("  return;");
    o.ind--;
    o.line("}");
}

// Cell-invariant map nodes the quadrature-point pass reads (operands of q-dependent ADD/MUL nodes,
// or outputs), constants excepted: the macro q-major kernel parks them in a thread-private column.
std::vector<int> macro_hoisted_nodes(const Signature& sig, const MapUse& use) {
    std::set<int> nd;
    for (size_t id = 0; id < sig.nodes.size(); ++id) {
        if (!use.live[id] || !use.qdep[id]) continue;
        const MapNode& n = sig.nodes[id];
        if (n.op == FEMGPU_OP_ADD || n.op == FEMGPU_OP_MUL) {
            if (!use.qdep[n.a]) nd.insert(n.a);
            if (!use.qdep[n.b]) nd.insert(n.b);
        }
    }
    for (int out : sig.outputs)
        if (!use.qdep[out]) nd.insert(out);
    std::vector<int> stored;
    for (int id : nd)
        if (sig.nodes[id].op != FEMGPU_OP_CONSTANT) stored.push_back(id);
    return stored;
}

// Per-thread shared-memory staging of the macro q-major pipeline (qmopt bit 5): one row of the
// group's gathered doubles (odd row length: conflict-free 8-byte accesses) and two buffers of its
// unique indices ([buffer][index][thread] columns).
struct MacroStageVal {
    std::string name, arr;
    int slot = 0, k = 0, stride = 1, comp = 0;
};
struct MacroStage {
    std::vector<std::pair<int, int>> idx;  // (map group, unique) per staged index
    std::vector<MacroStageVal> vals;
    int row = 1, nidx = 0;
    long long bytes(int block) const { return (8LL * row + 8LL * nidx) * block; }
};
MacroStage macro_stage_plan(const Signature& sig, const KernelPlan& kp) {
    MacroStage M;
    std::set<int> gathered;
    for (int i = 0; i < sig.ns(); ++i) gathered.insert(kp.sgroup[i]);
    for (int i = 0; i < sig.nv(); ++i) gathered.insert(kp.vgroup[i]);
    if (sig.affine) gathered.insert(kp.cgroup);
    const int D = sig.dim;
    int slot = 0;
    for (int g : gathered)
        for (int u = 0; u < kp.group_cap[g]; ++u) {
            const int k = static_cast<int>(M.idx.size());
            M.idx.push_back({g, u});
            for (int i = 0; i < sig.ns(); ++i)
                if (kp.sgroup[i] == g) M.vals.push_back({"xg" + std::to_string(i) + "_" + std::to_string(u), "P.x" + std::to_string(i), slot++, k, 1, 0});
            for (int i = 0; i < sig.nv(); ++i)
                if (kp.vgroup[i] == g)
                    for (int c : std::set<int>(sig.vcomps[i].begin(), sig.vcomps[i].end()))
                        M.vals.push_back({"vg" + std::to_string(i) + "_" + std::to_string(u) + "_" + std::to_string(c),
                                          "P.v" + std::to_string(i), slot++, k, vec_stride(D), c});
            if (sig.affine && kp.cgroup == g)
                for (int c = 0; c < D; ++c)
                    M.vals.push_back({"Xg" + std::to_string(u) + "_" + std::to_string(c), "P.X", slot++, k, vec_stride(D), c});
        }
    M.row = slot | 1;
    M.nidx = static_cast<int>(M.idx.size());
    return M;
}

// Macro-elements, quadrature-point-major ("qmajor"): the G cells of a group are interleaved at
// statement level inside each quadrature point, so every tabulation operand (LDCU from the
// constant bank, or an LDS) is loaded once for the G cells instead of once per cell (the cell-major
// macro kernel issues ~1 LDCU per 1.4 DFMA; sm_100a DFMA has no constant-bank operand form).  The
// cell-invariant map nodes of each cell are parked in a thread-private shared-memory column
// between the geometry pass and the quadrature loop, and the quadrature contributions go straight
// into the group's y accumulators (one per unique test DOF; the sum order over (q, cell, k) is
// reassociated, well inside the parity tolerance).  Non-finite values are detected on the
// accumulators (plus the terms the map never reads and det); the stage-checked twin then names the
// exact lowest cell and stage as usual.
void emit_macro_qmajor_kernel(Out& o, const Signature& sig, const KernelPlan& kp, const MapUse& use,
                              const std::string& name, long long smem_tab_off, long long hsmem_off) {
    const int D = sig.dim, G = kp.G, Q = sig.Q;
    const int SPL = std::max(1, kp.msplit);
    auto pat = [&](int g, int s, int j) { return kp.mpat[g][static_cast<size_t>(s) * kp.group_entries[g] + j]; };
    auto TAB = [&](const std::string& idx) {
        if (kp.basis == kBasisGlobal) return "__ldg(&P.tabg[" + idx + "])";
        return kp.basis == FEMGPU_BASIS_CONST ? "P.tab[" + idx + "]" : "sT[" + idx + "]";
    };
    const std::vector<int> stored = macro_hoisted_nodes(sig, use);
    std::vector<int> need;
    {
        std::set<int> nd;
        for (size_t id = 0; id < sig.nodes.size(); ++id) {
            if (!use.live[id] || !use.qdep[id]) continue;
            const MapNode& n = sig.nodes[id];
            if (n.op == FEMGPU_OP_ADD || n.op == FEMGPU_OP_MUL) {
                if (!use.qdep[n.a]) nd.insert(n.a);
                if (!use.qdep[n.b]) nd.insert(n.b);
            }
        }
        for (int out : sig.outputs)
            if (!use.qdep[out]) nd.insert(out);
        need.assign(nd.begin(), nd.end());
    }
    const int NH = static_cast<int>(stored.size());
    o.line("");
    o.line("extern \"C\" __global__ void __launch_bounds__(" + S(kp.block) + (kp.min_blocks > 1 ? ", " + S(kp.min_blocks) : "") +
           ") " + name + "(const __grid_constant__ Params P) {");
    o.ind++;
    o.line("constexpr bool CHECKED = false;");
    // qmopt bit 13: the zeroing of the fused range is spread over the launch's valid threads and
    // issued after the gathers (the stores drain while the loads are in flight) instead of a CTA prologue
    const bool late_zero = kp.zfused && (kp.qmopt & 8192) && SPL == 1 && !(kp.qmopt & 96);
    if (kp.zfused && !late_zero) o << kZeroPrologue;
    o.line("extern __shared__ __align__(16) unsigned char smraw[];");
    if (kp.basis == FEMGPU_BASIS_SMEM) {
        o.line("double* sT = reinterpret_cast<double*>(smraw + " + S(smem_tab_off) + ");");
        o.line("for (int i = threadIdx.x; i < " + S(sig.tab_size) + "; i += blockDim.x) sT[i] = P.tabg[i];");
        o.line("__syncthreads();");
    }
    // qmopt bit 0: the hoisted column is read back from shared memory (volatile: the compiler may
    // not forward the stored values into registers across the quadrature loop)
    if (kp.qmopt & 1) {
        o.line("volatile double* const sh_base = reinterpret_cast<volatile double*>(smraw + " + S(hsmem_off) + ") + threadIdx.x;");
        o.line("#define SH(k) sh_base[(k) * " + S(kp.block) + "]");
    } else {  // registers (constant indices): the compiler keeps them live across the quadrature loop
        o.line("double shr[" + S(std::max<long long>(1, static_cast<long long>(stored.size()) * ((G + SPL - 1) / SPL))) + "];");
        o.line("#define SH(k) shr[k]");
    }
    if (SPL == 1) {
        if (!(kp.qmopt & 96)) o.line("const int grp = P.cell0 / " + S(G) + " + blockIdx.x * " + S(kp.block) + " + threadIdx.x;");
    } else {
        // split groups: warp w computes cell subset (w % SPL) of 32 consecutive groups; the warps of
        // one group sit in the same CTA, so the nodes their subsets share hit in L1
        o.line("const int wid = threadIdx.x >> 5, sub = wid % " + S(SPL) + ";");
        o.line("const int grp = P.cell0 / " + S(G) + " + (blockIdx.x * " + S(kp.block / 32 / SPL) + " + wid / " + S(SPL) +
               ") * 32 + (threadIdx.x & 31);");
    }
    std::set<int> gathered;
    for (int i = 0; i < sig.ns(); ++i) gathered.insert(kp.sgroup[i]);
    for (int i = 0; i < sig.nv(); ++i) gathered.insert(kp.vgroup[i]);
    if (sig.affine) gathered.insert(kp.cgroup);
    const int gt = kp.tgroup;
    // qmopt bit 5: persistent CTAs with a two-stage cp.async pipeline per thread: while group g
    // computes, the next group's gathered values (and the one after's indices) stream into a
    // thread-private shared-memory row, so neither gather hop is exposed
    const bool staged = (kp.qmopt & 32) != 0 && SPL == 1;
    const bool persistent = !staged && (kp.qmopt & 64) != 0 && SPL == 1;
    const MacroStage MS = macro_stage_plan(sig, kp);
    if (staged) {
        o.line("const int gend = P.n_cells / " + S(G) + ";");
        o.line("const size_t NG = (size_t)P.n_groups;");
        o.line("const int gstride = gridDim.x * " + S(kp.block) + ";");
        o.line("double* const sv = reinterpret_cast<double*>(smraw + " + S(kp.stage_off) + ") + threadIdx.x * " + S(MS.row) + ";");
        o.line("int* const si = reinterpret_cast<int*>(smraw + " + S(kp.stage_off + 8LL * MS.row * kp.block) + ") + threadIdx.x;");
        o.line("#define SI(b, k) si[((b) * " + S(MS.nidx) + " + (k)) * " + S(kp.block) + "]");
        auto idx_copies = [&](const std::string& b, const std::string& g) {
            for (size_t k = 0; k < MS.idx.size(); ++k)
                o.line("cp4(&SI(" + b + ", " + S(k) + "), &P.gidx" + S(MS.idx[k].first) + "[" + S(MS.idx[k].second) + " * NG + " + g + "]);");
        };
        auto val_copies = [&](const std::string& b) {
            for (const auto& v : MS.vals)
                o.line("cp8(sv + " + S(v.slot) + ", " + v.arr + " + (size_t)SI(" + b + ", " + S(v.k) + ") * " + S(v.stride) + " + " + S(v.comp) + ");");
        };
        o.line("int grp = P.cell0 / " + S(G) + " + blockIdx.x * " + S(kp.block) + " + threadIdx.x;");
        o.line("if (grp >= gend) return;");
        idx_copies("0", "grp");
        o.line("cp_commit(); cp_wait_all();");
        val_copies("0");
        o.line("if (grp + gstride < gend) {");
        idx_copies("1", "grp + gstride");
        o.line("}");
        o.line("cp_commit(); cp_wait_all();");
        o.line("int buf = 1;");
        o.line("for (; grp < gend; grp += gstride, buf ^= 1) {");
        o.ind++;
    } else if (persistent) {
        // qmopt bit 6: persistent grid-stride loop over groups, so a group's red.add scatter drains
        // while the thread already computes its next group (no drain stall at thread exit);
        // bit 7: the next group's index lines are prefetched into L2 one iteration ahead
        o.line("const int gend = P.n_cells / " + S(G) + ";");
        o.line("const size_t NG = (size_t)P.n_groups;");
        o.line("const int gstride = gridDim.x * " + S(kp.block) + ";");
        o.line("for (int grp = P.cell0 / " + S(G) + " + blockIdx.x * " + S(kp.block) + " + threadIdx.x; grp < gend; grp += gstride) {");
        o.ind++;
        if (kp.qmopt & 128) {
            o.line("if (grp + gstride < gend) {");
            for (int g : gathered)
                for (int u = 0; u < kp.group_cap[g]; ++u)
                    o.line("  prefetch_l2(&P.gidx" + S(g) + "[" + S(u) + " * NG + grp + gstride]);");
            o.line("}");
        }
    } else {
        o.line("if (grp >= P.n_cells / " + S(G) + ") return;");
        o.line("const size_t NG = (size_t)P.n_groups;");
        emit_macro_bases(o, kp, gathered);
    }
    const bool affine_ok = !staged && !persistent;  // base indices declared (one-shot groups)
    for (int part = 0; part < SPL; ++part) {
        const int c0 = part * G / SPL, c1 = (part + 1) * G / SPL;
        if (SPL > 1) {
            o.line(std::string(part ? "} else " : "") + (part + 1 < SPL ? "if (sub == " + S(part) + ") {" : "{") +
                   " // cells " + S(c0) + ".." + S(c1 - 1) + " of the group");
            o.ind++;
        }
        // unique nodes of each map group read by this subset of cells
        auto used = [&](int g, int u) {
            const int E = kp.group_entries[g];
            for (int sc = c0; sc < c1; ++sc)
                for (int j = 0; j < E; ++j)
                    if (pat(g, sc, j) == u) return true;
            return false;
        };
        // ---- gathers: every unique node of the subset once (16-byte loads of padded vector nodes)
        if (staged) {
            for (const auto& v : MS.vals) o.line("const double " + v.name + " = sv[" + S(v.slot) + "];");
            o.line("if (grp + gstride < gend) {");
            o.ind++;
            for (const auto& v : MS.vals)
                o.line("cp8(sv + " + S(v.slot) + ", " + v.arr + " + (size_t)SI(buf, " + S(v.k) + ") * " + S(v.stride) + " + " +
                       S(v.comp) + ");");
            o.line("if (grp + 2 * gstride < gend) {");
            for (size_t k = 0; k < MS.idx.size(); ++k)
                o.line("  cp4(&SI(buf ^ 1, " + S(k) + "), &P.gidx" + S(MS.idx[k].first) + "[" + S(MS.idx[k].second) +
                       " * NG + grp + 2 * gstride]);");
            o.line("}");
            o.ind--;
            o.line("}");
            o.line("cp_commit();");
        }
        for (int g : gathered)
            for (int u = 0; u < kp.group_cap[g]; ++u) {
                if (!used(g, u) || staged) continue;
                o.line("const int ig" + S(g) + "_" + S(u) + " = " +
                       (affine_ok ? macro_index(kp, g, u) : "__ldg(&P.gidx" + S(g) + "[" + S(u) + " * NG + grp])") + ";");
                for (int i = 0; i < sig.ns(); ++i)
                    if (kp.sgroup[i] == g)
                        o.line("const double xg" + S(i) + "_" + S(u) + " = __ldg(&P.x" + S(i) + "[ig" + S(g) + "_" + S(u) + "]);");
                auto node_loads = [&](const std::string& dst, const std::string& arr, const std::set<int>& comps) {
                    const std::string base = arr + " + (size_t)ig" + S(g) + "_" + S(u) + " * " + S(vec_stride(D));
                    const bool pair = D >= 2 && comps.count(0) && comps.count(1);
                    if (pair) {
                        o.line("const double2 " + dst + "_01 = __ldg(reinterpret_cast<const double2*>(" + base + "));");
                        o.line("const double " + dst + "_0 = " + dst + "_01.x, " + dst + "_1 = " + dst + "_01.y;");
                    }
                    for (int c : comps)
                        if (!pair || c >= 2) o.line("const double " + dst + "_" + S(c) + " = __ldg(" + base + " + " + S(c) + ");");
                };
                for (int i = 0; i < sig.nv(); ++i)
                    if (kp.vgroup[i] == g) node_loads("vg" + S(i) + "_" + S(u), "P.v" + S(i), std::set<int>(sig.vcomps[i].begin(), sig.vcomps[i].end()));
                if (sig.affine && kp.cgroup == g) {
                    std::set<int> comps;
                    for (int c = 0; c < D; ++c) comps.insert(c);
                    node_loads("Xg" + S(u), "P.X", comps);
                }
            }
        if (late_zero) {
            o.line("{ const long long g0 = P.cell0 / " + S(G) + ", ng = P.n_cells / " + S(G) + " - g0;");
            o.line("  for (long long i = grp - g0; i < P.zn; i += ng) __stcs(P.zp + i, 0.0); }");
        }
        o.line("bool nf = false;");
        // ---- per cell: geometry + cell-invariant nodes -> thread-private smem column
        for (int sc = c0; sc < c1; ++sc) {
            o.line("{ // geometry of cell " + S(sc));
            o.ind++;
            if (sig.affine) {
                for (int j = 0; j < sig.coord_dofs; ++j)
                    for (int c = 0; c < D; ++c)
                        o.line("const double " + nm("X", j, c) + " = " + nm("Xg", pat(kp.cgroup, sc, j), c) + ";");
                for (int c = 0; c < D; ++c)
                    for (int r = 0; r < D; ++r)
                        o.line("const double " + nm("J", r, c) + " = " + nm("X", c + 1, r) + " - " + nm("X", 0, r) + ";");
                if (D == 1) o.line("const double det = J0_0;");
                if (D == 2) o.line("const double det = J0_0 * J1_1 - J0_1 * J1_0;");
                if (D == 3)
                    o.line("const double det = J0_0 * (J1_1 * J2_2 - J1_2 * J2_1) - J0_1 * (J1_0 * J2_2 - J1_2 * J2_0) + "
                           "J0_2 * (J1_0 * J2_1 - J1_1 * J2_0);");
                if (use.uses_inv) {
                    std::ostringstream gi;
                    if (D == 1) gi << "const double Ji0_0 = 1.0 / det;";
                    if (D == 2) gi << "const double Ji0_0 = J1_1 / det, Ji0_1 = -J0_1 / det, Ji1_0 = -J1_0 / det, Ji1_1 = J0_0 / det;";
                    if (D == 3)
                        gi << "const double Ji0_0 = (J1_1*J2_2 - J1_2*J2_1) / det, Ji0_1 = (J0_2*J2_1 - J0_1*J2_2) / det, "
                              "Ji0_2 = (J0_1*J1_2 - J0_2*J1_1) / det, Ji1_0 = (J1_2*J2_0 - J1_0*J2_2) / det, "
                              "Ji1_1 = (J0_0*J2_2 - J0_2*J2_0) / det, Ji1_2 = (J0_2*J1_0 - J0_0*J1_2) / det, "
                              "Ji2_0 = (J1_0*J2_1 - J1_1*J2_0) / det, Ji2_1 = (J0_1*J2_0 - J0_0*J2_1) / det, "
                              "Ji2_2 = (J0_0*J1_1 - J0_1*J1_0) / det;";
                    o.line(gi.str());
                }
                o.line("nf = nf | NF(det);");
            }
            emit_nodes(o, sig, use, false, "0", TAB);
            for (int h = 0; h < NH; ++h) o.line("SH(" + S((sc - c0) * NH + h) + ") = n" + S(stored[h]) + ";");
            o.ind--;
            o.line("}");
        }
        {
            std::string l;
            for (int u = 0; u < kp.group_cap[gt]; ++u)
                if (used(gt, u)) l += std::string(l.empty() ? "double" : ",") + " ya" + S(u) + " = 0.0";
            o.line(l + ";");
        }
        // ---- quadrature points: statements interleaved over the subset's cells
        // qmopt bit 4: the quadrature loop stays rolled (a Q-th of the code: instruction-cache misses
        // stall the unrolled straight-line kernel); tabulation offsets become q-relative
        const bool rolled = (kp.qmopt & 16) != 0;
        auto QI = [&](long long base0, long long stride, int q) {
            return rolled ? S(base0) + " + q * " + S(stride) : S(base0 + static_cast<long long>(q) * stride);
        };
        if (rolled) {
            o.line((kp.qmopt & 16384) ? "#pragma unroll 2" : "#pragma unroll 1");  // bit 14: two points per trip
            o.line("for (int q = 0; q < " + S(Q) + "; ++q) {");
            o.ind++;
        }
        for (int q = 0; q < (rolled ? 1 : Q); ++q) {
            o.line("{ // quadrature point " + (rolled ? std::string("q") : S(q)));
            o.ind++;
            // evaluation
            for (int i = 0; i < sig.ns(); ++i)
                for (int t = 0; t < sig.sterms[i]; ++t) {
                    const long long base = sig.phi_off_s[i] + static_cast<long long>(t) * Q * sig.sdofs[i];
                    for (int sc = c0; sc < c1; ++sc) o.line("double " + nm("s", i, t) + "_c" + S(sc) + ";");
                    for (int j = 0; j < sig.sdofs[i]; ++j) {
                        std::string l = "{ const double tb = " + TAB(QI(base + j, sig.sdofs[i], q)) + ";";
                        for (int sc = c0; sc < c1; ++sc) {
                            const std::string v = nm("s", i, t) + "_c" + S(sc), u = nm("xg", i, pat(kp.sgroup[i], sc, j));
                            l += j == 0 ? " " + v + " = tb * " + u + ";" : " " + v + " = FMA(tb, " + u + ", " + v + ");";
                        }
                        o.line(l + " }");
                    }
                }
            for (int i = 0; i < sig.nv(); ++i)
                for (int t = 0; t < sig.vterms[i]; ++t) {
                    const long long base = sig.phi_off_v[i] + static_cast<long long>(t) * Q * sig.vdofs[i];
                    const int comp = sig.vcomps[i][t];
                    for (int sc = c0; sc < c1; ++sc) o.line("double " + nm("t", i, t) + "_c" + S(sc) + ";");
                    for (int j = 0; j < sig.vdofs[i]; ++j) {
                        std::string l = "{ const double tb = " + TAB(QI(base + j, sig.vdofs[i], q)) + ";";
                        for (int sc = c0; sc < c1; ++sc) {
                            const std::string v = nm("t", i, t) + "_c" + S(sc), w = nm("vg", i, pat(kp.vgroup[i], sc, j), comp);
                            l += j == 0 ? " " + v + " = tb * " + w + ";" : " " + v + " = FMA(tb, " + w + ", " + v + ");";
                        }
                        o.line(l + " }");
                    }
                }
            // map per cell
            for (int sc = c0; sc < c1; ++sc) {
                for (int k = 0; k < sig.Tw; ++k) o.line("double e" + S(k) + "_c" + S(sc) + ";");
                o.line("{");
                o.ind++;
                std::string unused;
                for (int i = 0; i < sig.ns(); ++i)
                    for (int t = 0; t < sig.sterms[i]; ++t) {
                        o.line("const double " + nm("s", i, t) + " = " + nm("s", i, t) + "_c" + S(sc) + ";");
                        if (!use.sd_used.count({i, t})) unused += " | NF(" + nm("s", i, t) + ")";
                    }
                for (int i = 0; i < sig.nv(); ++i)
                    for (int t = 0; t < sig.vterms[i]; ++t) {
                        o.line("const double " + nm("t", i, t) + " = " + nm("t", i, t) + "_c" + S(sc) + ";");
                        if (!use.vd_used.count({i, t})) unused += " | NF(" + nm("t", i, t) + ")";
                    }
                if (!unused.empty()) o.line("nf = nf" + unused + ";");
                for (int h = 0; h < NH; ++h) o.line("const double n" + S(stored[h]) + " = SH(" + S((sc - c0) * NH + h) + ");");
                for (int id : need)
                    if (sig.nodes[id].op == FEMGPU_OP_CONSTANT) o.line("const double n" + S(id) + " = " + lit(sig.nodes[id].value) + ";");
                emit_nodes(o, sig, use, true, rolled ? std::string("q") : S(q), TAB);
                for (int k = 0; k < sig.Tw; ++k) o.line("e" + S(k) + "_c" + S(sc) + " = n" + S(sig.outputs[k]) + ";");
                o.ind--;
                o.line("}");
            }
            // quadrature straight into the group's y accumulators, one Psi load for the subset's cells
            // (all-zero Psi entries skipped, see emit_cell_body)
            for (int k = 0; k < sig.Tw; ++k)
                if (sig.output_dead(k))
                    for (int sc = c0; sc < c1; ++sc) o.line("nf = nf | NF(e" + S(k) + "_c" + S(sc) + ");");
            for (int jw = 0; jw < sig.nW; ++jw)
                for (int k = 0; k < sig.Tw; ++k) {
                    if (!sig.pnz(k, jw)) continue;
                    const long long idx = sig.psi_off + (static_cast<long long>(k) * sig.nW + jw) * Q;
                    std::string l = "{ const double tb = " + TAB(QI(idx, 1, q)) + ";";
                    for (int sc = c0; sc < c1; ++sc) {
                        const std::string ya = "ya" + S(pat(gt, sc, jw));
                        l += " " + ya + " = FMA(tb, e" + S(k) + "_c" + S(sc) + ", " + ya + ");";
                    }
                    o.line(l + " }");
                }
            o.ind--;
            o.line("}");
        }
        if (rolled) {
            o.ind--;
            o.line("}");
        }
        // ---- finiteness (any non-finite contribution reaches an accumulator) + scatter
        {
            std::string chk;
            for (int u = 0; u < kp.group_cap[gt]; ++u)
                if (used(gt, u)) chk += " | NF(ya" + S(u) + ")";
            o.line("if (nf" + chk + ") atomicMin(P.bad, (unsigned long long)grp * " + S(G) + ");");
        }
        const bool merging = !kp.merge.empty() && SPL == 1 && gathered.count(gt) && !(kp.qmopt & 2) && !staged;
        if (merging) {
            // warp merge: lane l's contribution to node u moves to lane l+s when that lane's group has
            // the same global node (as u'): one red.add per node of the warp's block of groups instead
            // of one per (group, node); the owner of a moved contribution then skips it (zeroed).
            // The pairing is a hint from the layout; equality of the global indices decides at run time.
            o.line("if (__activemask() == 0xffffffffu) {");
            o.ind++;
            o.line("const int lane = threadIdx.x & 31;");
            for (const auto& m : kp.merge) {
                const int sft = m[0], u = m[1], u2 = m[2];
                const std::string a = "ya" + S(u), b = "ya" + S(u2), ia = "ig" + S(gt) + "_" + S(u), ib = "ig" + S(gt) + "_" + S(u2);
                o.line("{ const double v = __shfl_up_sync(0xffffffffu, " + a + ", " + S(sft) + "); const int i = __shfl_up_sync(0xffffffffu, " +
                       ia + ", " + S(sft) + "); const int j = __shfl_down_sync(0xffffffffu, " + ib + ", " + S(sft) + ");");
                o.line("  if (lane >= " + S(sft) + " && i == " + ib + ") " + b + " += v;");
                o.line("  if (lane + " + S(sft) + " < 32 && j == " + ia + ") " + a + " = 0.0; }");
            }
            o.ind--;
            o.line("}");
        }
        for (int u = 0; u < kp.group_cap[gt]; ++u) {
            if (!used(gt, u)) continue;
            // qmopt bit 1: reload the scatter indices (an opaque load the compiler cannot merge with
            // the gather's) instead of keeping them live in registers across the quadrature loop
            std::string idx = ((kp.qmopt & 2) || staged) ? "ldidx(&P.gidx" + S(gt) + "[" + S(u) + " * NG + grp])"
                              : gathered.count(gt) ? "ig" + S(gt) + "_" + S(u)
                              : affine_ok          ? macro_index(kp, gt, u)
                                                   : "__ldg(&P.gidx" + S(gt) + "[" + S(u) + " * NG + grp])";
            if (!kp.talias.empty() && kp.talias[u][0] >= 0) {
                // the row is an image of a gathered node: scale * node + add (no test-map load)
                const auto& al = kp.talias[u];
                const std::string src = ((kp.qmopt & 2) || staged)
                                            ? "ldidx(&P.gidx" + S(al[0]) + "[" + S(al[1]) + " * NG + grp])"
                                            : "ig" + S(al[0]) + "_" + S(al[1]);
                idx = "(" + src + (al[2] != 1 ? " * " + S(al[2]) : "") + (al[3] ? " + " + S(al[3]) : "") + ")";
            }
            if (kp.qmopt & 4)  // timing experiment only (wrong results): plain store instead of red.add
                o.line("P.y[" + idx + "] = ya" + S(u) + ";");
            else if (kp.qmopt & 8)  // timing experiment only (wrong results): no scatter traffic
                o.line("if (ya" + S(u) + " == 1234.5678) P.y[" + idx + "] = 0.0;");
            else if (merging)  // a merged-away contribution is exactly 0.0: nothing to add
                o.line("if (ya" + S(u) + " != 0.0) atomicAdd(&P.y[" + idx + "], ya" + S(u) + ");");
            else
                o.line("atomicAdd(&P.y[" + idx + "], ya" + S(u) + ");");
        }
        if (SPL > 1) o.ind--;
    }
    if (SPL > 1) o.line("}");
    if (staged) {
        o.line("cp_wait_all();");
        o.ind--;
        o.line("}");
    }
    if (persistent) {
        o.ind--;
        o.line("}");
    }
    o.line("(void)CHECKED;");
    o.ind--;
    o.line("}");
}

const char* kAsync = R"(
__device__ __forceinline__ void cp16(unsigned char* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
)";

}  // namespace

EmitResult emit_kernel(const Signature& sig, const KernelPlan& kp) {
    if (kp.family == Family::Mlt) return emit_mlt(sig, kp);
    if (kp.family == Family::Dmma) return emit_dmma(sig, kp);
    const MapUse use = analyse(sig);
    EmitResult r;
    Out o;
    o << kPrelude;
    const bool tile = kp.family == Family::Tile;
    const long long nt_param = kp.basis == FEMGPU_BASIS_CONST ? sig.tab_size : 0;
    emit_params(o, sig, kp, nt_param);
    // Unroll the qp loop unless the straight-line body would be huge.
    long long fmas = 0;
    for (int i = 0; i < sig.ns(); ++i) fmas += static_cast<long long>(sig.sterms[i]) * sig.sdofs[i];
    for (int i = 0; i < sig.nv(); ++i) fmas += static_cast<long long>(sig.vterms[i]) * sig.vdofs[i];
    fmas += static_cast<long long>(sig.nW) * sig.Tw;
    // FEMGPU_DEBUG_UNROLL_Q=0/1 overrides the heuristic (I-cache experiments)
    const char* uq = std::getenv("FEMGPU_DEBUG_UNROLL_Q");
    const bool unroll_q = uq ? std::atoi(uq) != 0 : (!kp.qloop && fmas * sig.Q <= 2000);  // larger bodies: NVRTC time + I-cache
    if (kp.family == Family::Macro) {
        r.kernel = "femgpu_macro";
        r.kernel_checked = "femgpu_macro_checked";
        r.smem_bytes = kp.basis == FEMGPU_BASIS_SMEM ? static_cast<size_t>(al16(sig.tab_size * 8)) : 0;
        if (kp.mstage) {
            o << kAsync;
            long long slots = 0;
            for (int i = 0; i < sig.ns(); ++i) slots += kp.group_cap[kp.sgroup[i]];
            for (int i = 0; i < sig.nv(); ++i) slots += static_cast<long long>(kp.group_cap[kp.vgroup[i]]) * sig.dim;
            if (sig.affine) slots += static_cast<long long>(kp.group_cap[kp.cgroup]) * sig.dim;
            r.smem_bytes += static_cast<size_t>(slots * 8 * kp.block);
        }
        const long long ysmem_off = static_cast<long long>(r.smem_bytes);
        if (kp.ysmem) r.smem_bytes += static_cast<size_t>(kp.group_cap[kp.tgroup]) * 8 * kp.block;
        if (kp.qmajor) {
            // thread-private columns of the cell-invariant map nodes of one thread's cells
            const long long nh = static_cast<long long>(macro_hoisted_nodes(sig, use).size());
            const int spl = std::max(1, kp.msplit);
            const long long cells_per_thread = (kp.G + spl - 1) / spl;
            const long long hoff = static_cast<long long>(al16(static_cast<long long>(r.smem_bytes)));
            if (kp.qmopt & 1) r.smem_bytes = static_cast<size_t>(hoff + nh * cells_per_thread * 8 * kp.block);
            KernelPlan kq = kp;
            if ((kp.qmopt & 32) && spl == 1) {
                o << kAsync;
                kq.stage_off = static_cast<long long>(al16(static_cast<long long>(r.smem_bytes)));
                r.smem_bytes = static_cast<size_t>(kq.stage_off + macro_stage_plan(sig, kp).bytes(kp.block));
            }
            emit_macro_qmajor_kernel(o, sig, kq, use, r.kernel, 0, hoff);
        } else {
            emit_macro_kernel(o, sig, kp, use, unroll_q, r.kernel, 0, ysmem_off);
        }
        emit_scpt_kernel(o, sig, kp, use, false, true, r.kernel_checked, 0);
    } else if (tile) {
        o << kAsync;
        const TilePlan T = plan_tile(sig, kp);
        r.kernel = "femgpu_tile";
        r.kernel_checked = "femgpu_tile_checked";
        r.smem_bytes = static_cast<size_t>(T.total);
        emit_tile_kernel(o, sig, kp, use, unroll_q, T, r.kernel);
        emit_scpt_kernel(o, sig, kp, use, false, true, r.kernel_checked, T.tab_off);
    } else {
        r.kernel = "femgpu_scpt";
        r.kernel_checked = "femgpu_scpt_checked";
        r.smem_bytes = kp.basis == FEMGPU_BASIS_SMEM ? static_cast<size_t>(sig.tab_size) * 8 : 0;
        if (kp.G > 1)
            emit_scpt_multi_kernel(o, sig, kp, use, unroll_q && kp.G * fmas * sig.Q <= 12000, r.kernel, 0);
        else
            emit_scpt_kernel(o, sig, kp, use, unroll_q, false, r.kernel, 0);
        emit_scpt_kernel(o, sig, kp, use, false, true, r.kernel_checked, 0);
    }
    r.source = o.s.str();
    return r;
}


// ---------------------------------------------------------------------------------------------
// MLT family: the paper's multi-level tiling (TilingParams, qoi.hpp:23-33) with the execution
// and summation semantics of run_mlt (simulate.hpp:293-598): CTA = N_c cells x N_WI lanes,
// quadrature tiles of T^Q points; per (eval row tile, space, column tile) the cells' DOF tiles are
// gathered and the Phi tile is prefetched cooperatively into the aliased shared buffer B (roster
// flat = N_c*N_WI*round + N_WI*lid0 + lid1), lanes stride the rows; the map writes e_arr; per
// (quad row tile, column tile) the Psi tile goes through B; y gets one red.add per (quad tile,
// quad row tile) per test DOF.  Tabulations are read from global memory (L2-resident).
EmitResult emit_mlt(const Signature& sig, const KernelPlan& kp) {
    const MapUse use = analyse(sig);
    EmitResult r;
    Out o;
    o << kPrelude;
    emit_params(o, sig, kp, 0);
    const int NC = kp.Nc, NW = kp.Nwi, BS = NC * NW, Q = sig.Q, D = sig.dim;
    const int TQ = kp.TQ, TER = kp.Ter, TQR = kp.Tqr, TQC = kp.Tqc, TW = sig.Tw, NWD = sig.nW;
    struct Sp {
        bool vec;
        int idx, n, terms, tc;
        long long phi_off;
        std::vector<int> comps;
    };
    std::vector<Sp> sps;
    for (int i = 0; i < sig.ns(); ++i) sps.push_back({false, i, sig.sdofs[i], sig.sterms[i], kp.Tcs[i], sig.phi_off_s[i], {}});
    for (int i = 0; i < sig.nv(); ++i)
        sps.push_back({true, i, sig.vdofs[i], sig.vterms[i], kp.Tcv[i], sig.phi_off_v[i], sig.vcomps[i]});
    long long buf = 0;
    for (const auto& s : sps) buf = std::max<long long>(buf, static_cast<long long>(s.terms) * TER * s.tc);
    buf = std::max<long long>(buf, static_cast<long long>(TW) * TQR * TQC);
    long long dt = 1;
    for (const auto& s : sps) dt = std::max<long long>(dt, static_cast<long long>(s.tc) * (s.vec ? D : 1));
    const long long earr = static_cast<long long>(TW) * NC * TQ;
    const int geo = sig.affine ? D * D + 1 + sig.coord_dofs * D : 0;
    const long long off_e = buf, off_dofs = off_e + earr, off_geo = off_dofs + NC * dt;
    r.smem_bytes = static_cast<size_t>((off_geo + static_cast<long long>(NC) * geo) * 8);
    r.kernel = "femgpu_mlt";
    r.kernel_checked = "femgpu_mlt_checked";
    const int RR = (TER + NW - 1) / NW, RQ = (TQR + NW - 1) / NW;
    auto TABG = [](const std::string& idx) { return "__ldg(&P.tabg[" + idx + "])"; };

    o.line("");
    o.line("extern \"C\" __global__ void __launch_bounds__(" + S(BS) + ") " + r.kernel + "(const __grid_constant__ Params P) {");
    o.ind++;
    o.line("constexpr bool CHECKED = false;");
    o.line("extern __shared__ __align__(16) double smd[];");
    o.line("double* Bf = smd; double* earr = smd + " + S(off_e) + "; double* dofs = smd + " + S(off_dofs) +
           "; double* geo = smd + " + S(off_geo) + ";");
    o.line("const int tid = threadIdx.x, lid0 = tid / " + S(NW) + ", lid1 = tid % " + S(NW) + ";");
    o.line("const int cell = blockIdx.x * " + S(NC) + " + lid0;");
    o.line("const bool live = cell < P.n_cells;");
    o.line("bool nf = false;");
    o.line("int stage = -1; (void)stage;");
    if (sig.affine) {
        // geometry once per cell (lane 0), shared with the cell's lanes
        o.line("if (live && lid1 == 0) {");
        o.ind++;
        o.line("double* g = geo + lid0 * " + S(geo) + ";");
        for (int j = 0; j < sig.coord_dofs; ++j) {
            o.line("{");
            o.line("  const int v = __ldg(&P.cm[" + S(j) + "*(size_t)P.stride + cell]);");
            for (int c = 0; c < D; ++c)
                o.line("  g[" + S(D * D + 1 + j * D + c) + "] = __ldg(&P.X[(size_t)v*" + S(vec_stride(D)) + "+" + S(c) + "]);");
            o.line("}");
        }
        o.ind--;
        o.line("}");
        o.line("__syncthreads();");
        o.line("const double* g = geo + lid0 * " + S(geo) + ";");
        for (int j = 0; j < sig.coord_dofs; ++j)
            for (int c = 0; c < D; ++c) o.line("const double X" + S(j) + "_" + S(c) + " = g[" + S(D * D + 1 + j * D + c) + "];");
        for (int c = 0; c < D; ++c)
            for (int rr = 0; rr < D; ++rr)
                o.line("const double J" + S(rr) + "_" + S(c) + " = X" + S(c + 1) + "_" + S(rr) + " - X0_" + S(rr) + ";");
        if (D == 1) o.line("const double det = J0_0;");
        if (D == 2) o.line("const double det = J0_0 * J1_1 - J0_1 * J1_0;");
        if (D == 3)
            o.line("const double det = J0_0 * (J1_1 * J2_2 - J1_2 * J2_1) - J0_1 * (J1_0 * J2_2 - J1_2 * J2_0) + "
                   "J0_2 * (J1_0 * J2_1 - J1_1 * J2_0);");
        if (use.uses_inv) {
            if (D == 1) o.line("const double Ji0_0 = 1.0 / det;");
            if (D == 2) o.line("const double Ji0_0 = J1_1 / det, Ji0_1 = -J0_1 / det, Ji1_0 = -J1_0 / det, Ji1_1 = J0_0 / det;");
            if (D == 3) {
                o.line("const double Ji0_0 = (J1_1*J2_2 - J1_2*J2_1) / det, Ji0_1 = (J0_2*J2_1 - J0_1*J2_2) / det, Ji0_2 = (J0_1*J1_2 - J0_2*J1_1) / det;");
                o.line("const double Ji1_0 = (J1_2*J2_0 - J1_0*J2_2) / det, Ji1_1 = (J0_0*J2_2 - J0_2*J2_0) / det, Ji1_2 = (J0_2*J1_0 - J0_0*J1_2) / det;");
                o.line("const double Ji2_0 = (J1_0*J2_1 - J1_1*J2_0) / det, Ji2_1 = (J0_1*J2_0 - J0_0*J2_1) / det, Ji2_2 = (J0_0*J1_1 - J0_1*J1_0) / det;");
            }
        }
        o.line("if (live) nf = nf | NF(det);");
    }
    emit_nodes(o, sig, use, false, "0", TABG);
    o.line("for (int qt = 0; qt < " + S((Q + TQ - 1) / TQ) + "; ++qt) {");
    o.ind++;
    o.line("const int qb = qt * " + S(TQ) + ", tq = min(" + S(TQ) + ", " + S(Q) + " - qb);");
    // ---- evaluation phase
    o.line("for (int rb = 0; rb < tq; rb += " + S(TER) + ") {");
    o.ind++;
    o.line("const int tr = min(" + S(TER) + ", tq - rb);");
    for (size_t si = 0; si < sps.size(); ++si)
        for (int k = 0; k < sps[si].terms; ++k) {
            std::string l = "double";
            for (int rr = 0; rr < RR; ++rr) l += std::string(rr ? "," : "") + " a" + S(si) + "_" + S(k) + "_" + S(rr) + " = 0.0";
            o.line(l + ";");
        }
    for (size_t si = 0; si < sps.size(); ++si) {
        const Sp& sp = sps[si];
        const int comps = sp.vec ? D : 1;
        const std::string X = sp.vec ? "P.v" + S(sp.idx) : "P.x" + S(sp.idx);
        const std::string M = sp.vec ? "P.vm" + S(sp.idx) : "P.m" + S(sp.idx);
        o.line("for (int cb = 0; cb < " + S(sp.n) + "; cb += " + S(sp.tc) + ") {");
        o.ind++;
        o.line("const int tc = min(" + S(sp.tc) + ", " + S(sp.n) + " - cb);");
        // per-cell DOF tile gather (lanes of the cell share it)
        o.line("if (live) for (int t = lid1; t < tc * " + S(comps) + "; t += " + S(NW) + ") {");
        o.line("  const int j = t / " + S(comps) + ", c = t % " + S(comps) + ";");
        o.line("  dofs[lid0 * " + S(dt) + " + t] = __ldg(&" + X + "[(size_t)__ldg(&" + M + "[(size_t)(cb + j) * P.stride + cell]) * " +
               S(sp.vec ? vec_stride(D) : 1) + " + c]);");
        o.line("}");
        // cooperative Phi-tile prefetch into the aliased buffer (roster of simulate.hpp:414-429)
        o.line("for (int f = tid; f < tr * tc; f += " + S(BS) + ") {");
        o.line("  const int i = f / tc, j = f % tc;");
        for (int k = 0; k < sp.terms; ++k)
            o.line("  Bf[" + S(static_cast<long long>(k) * TER * sp.tc) + " + i * " + S(sp.tc) + " + j] = " +
                   TABG(S(sp.phi_off + static_cast<long long>(k) * Q * sp.n) + " + (qb + rb + i) * " + S(sp.n) + " + cb + j") + ";");
        o.line("}");
        o.line("__syncthreads();");
        for (int rr = 0; rr < RR; ++rr) {
            o.line("if (live && lid1 + " + S(rr * NW) + " < tr) {");
            o.ind++;
            o.line("const int iq = lid1 + " + S(rr * NW) + ";");
            for (int k = 0; k < sp.terms; ++k) {
                const int comp = sp.vec ? sp.comps[k] : 0;
                const std::string a = "a" + S(si) + "_" + S(k) + "_" + S(rr);
                o.line("for (int j = 0; j < tc; ++j) " + a + " = FMA(Bf[" + S(static_cast<long long>(k) * TER * sp.tc) + " + iq * " +
                       S(sp.tc) + " + j], dofs[lid0 * " + S(dt) + " + j * " + S(comps) + " + " + S(comp) + "], " + a + ");");
            }
            o.ind--;
            o.line("}");
        }
        o.line("__syncthreads();");
        o.ind--;
        o.line("}");
    }
    // map per row (the lane that evaluated the row applies the map)
    for (int rr = 0; rr < RR; ++rr) {
        o.line("if (live && lid1 + " + S(rr * NW) + " < tr) {");
        o.ind++;
        o.line("const int iq = lid1 + " + S(rr * NW) + ";");
        // alias derivative variables
        for (size_t si = 0; si < sps.size(); ++si)
            for (int k = 0; k < sps[si].terms; ++k)
                o.line("const double " + std::string(sps[si].vec ? "t" : "s") + S(sps[si].idx) + "_" + S(k) + " = a" + S(si) + "_" +
                       S(k) + "_" + S(rr) + ";");
        {
            std::string unused;
            for (int i = 0; i < sig.ns(); ++i)
                for (int k = 0; k < sig.sterms[i]; ++k)
                    if (!use.sd_used.count({i, k})) unused += " | NF(s" + S(i) + "_" + S(k) + ")";
            for (int i = 0; i < sig.nv(); ++i)
                for (int k = 0; k < sig.vterms[i]; ++k)
                    if (!use.vd_used.count({i, k})) unused += " | NF(t" + S(i) + "_" + S(k) + ")";
            if (!unused.empty()) o.line("nf = nf" + unused + ";");
        }
        emit_nodes(o, sig, use, true, "qb + rb + iq", TABG);
        for (int k = 0; k < TW; ++k)
            o.line("earr[(" + S(k) + " * " + S(NC) + " + lid0) * " + S(TQ) + " + rb + iq] = n" + S(sig.outputs[k]) + ";");
        o.ind--;
        o.line("}");
    }
    o.ind--;
    o.line("}");
    o.line("__syncthreads();");
    // ---- quadrature phase
    o.line("for (int rb = 0; rb < " + S(NWD) + "; rb += " + S(TQR) + ") {");
    o.ind++;
    o.line("const int tr = min(" + S(TQR) + ", " + S(NWD) + " - rb);");
    {
        std::string l = "double";
        for (int rr = 0; rr < RQ; ++rr) l += std::string(rr ? "," : "") + " o" + S(rr) + " = 0.0";
        o.line(l + ";");
    }
    o.line("for (int cb = 0; cb < tq; cb += " + S(TQC) + ") {");
    o.ind++;
    o.line("const int tc = min(" + S(TQC) + ", tq - cb);");
    o.line("for (int f = tid; f < tr * tc; f += " + S(BS) + ") {");
    o.line("  const int i = f / tc, j = f % tc;");
    for (int k = 0; k < TW; ++k)
        o.line("  Bf[" + S(static_cast<long long>(k) * TQR * TQC) + " + i * " + S(TQC) + " + j] = " +
               TABG(S(sig.psi_off + static_cast<long long>(k) * NWD * Q) + " + (rb + i) * " + S(Q) + " + qb + cb + j") + ";");
    o.line("}");
    o.line("__syncthreads();");
    for (int rr = 0; rr < RQ; ++rr) {
        o.line("if (live && lid1 + " + S(rr * NW) + " < tr) {");
        o.line("  const int jw = lid1 + " + S(rr * NW) + ";");
        o.line("  for (int iq = 0; iq < tc; ++iq) {");
        for (int k = 0; k < TW; ++k)
            o.line("    o" + S(rr) + " = FMA(Bf[" + S(static_cast<long long>(k) * TQR * TQC) + " + jw * " + S(TQC) +
                   " + iq], earr[(" + S(k) + " * " + S(NC) + " + lid0) * " + S(TQ) + " + cb + iq], o" + S(rr) + ");");
        o.line("  }");
        o.line("}");
    }
    o.line("__syncthreads();");
    o.ind--;
    o.line("}");
    // scatter this (quad tile, row tile) (simulate.hpp:578-586)
    for (int rr = 0; rr < RQ; ++rr) {
        o.line("if (live && lid1 + " + S(rr * NW) + " < tr) {");
        o.line("  const int jw = lid1 + " + S(rr * NW) + ";");
        o.line("  nf = nf | NF(o" + S(rr) + ");");
        o.line("  atomicAdd(&P.y[__ldg(&P.tm[(size_t)(rb + jw) * P.stride + cell])], o" + S(rr) + ");");
        o.line("}");
    }
    o.ind--;
    o.line("}");
    o.line("__syncthreads();");
    o.ind--;
    o.line("}");
    o.line("if (nf) atomicMin(P.bad, (unsigned long long)cell);");
    o.line("return;");
    o.line("report:");
    o.line("  return;");
    o.ind--;
    o.line("}");
    // diagnostic kernel: the SCPT stage-checked kernel over the same Params
    KernelPlan pk = kp;
    pk.family = Family::Scpt;
    pk.basis = FEMGPU_BASIS_SMEM;
    emit_scpt_kernel(o, sig, pk, use, false, true, r.kernel_checked, 0);
    r.source = o.s.str();
    r.smem_bytes = std::max<size_t>(r.smem_bytes, static_cast<size_t>(sig.tab_size) * 8);
    return r;
}

size_t tile_smem_bytes(const Signature& sig, const KernelPlan& kp) { return static_cast<size_t>(plan_tile(sig, kp).total); }


void emit_dmma_kernel(std::ostringstream& o, const Signature& sig, const KernelPlan& kp, DmmaLayout& L,
                      const std::string& name);

EmitResult emit_dmma(const Signature& sig, const KernelPlan& kp) {
    const MapUse use = analyse(sig);
    EmitResult r;
    Out o;
    o << kPrelude;
    o << "#define DMMA(d0, d1, a, b) asm(\"mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\" : "
         "\"+d\"(d0), \"+d\"(d1) : \"d\"(a), \"d\"(b))\n";
    emit_params(o, sig, kp, 0);
    DmmaLayout L = dmma_layout(sig, kp);
    r.kernel = "femgpu_dmma";
    r.kernel_checked = "femgpu_dmma_checked";
    emit_dmma_kernel(o.s, sig, kp, L, r.kernel);
    r.smem_bytes = dmma_smem_bytes(sig, kp);
    long long fmas = 0;
    for (int i = 0; i < sig.ns(); ++i) fmas += static_cast<long long>(sig.sterms[i]) * sig.sdofs[i];
    for (int i = 0; i < sig.nv(); ++i) fmas += static_cast<long long>(sig.vterms[i]) * sig.vdofs[i];
    fmas += static_cast<long long>(sig.nW) * sig.Tw;
    KernelPlan ck = kp;
    ck.basis = kBasisGlobal;
    ck.min_blocks = 1;
    emit_scpt_kernel(o, sig, ck, use, false, true, r.kernel_checked, 0);  // diagnostic twin: rolled (compile time)
    r.source = o.s.str();
    return r;
}

}  // namespace femgpu

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
//         DOFs/vertices are staged in shared memory through tile-local uint16 maps, the
//         cell results are reduced into a shared-memory y tile, and only DOFs shared with
//         another tile reach global memory atomically (the rest are plain stores).
//   Mlt   the paper's multi-level tiling (TilingParams, qoi.hpp:23-33): N_c cells x N_WI
//         lanes per CTA, quadrature tiles T^Q, Phi/Psi tiles staged through an aliased
//         shared buffer, lanes striding qp rows (evaluation) and test rows (quadrature),
//         scatter once per (quad tile, quad row tile) (simulate.hpp:293-598 semantics).
// Basis residency (KernelPlan::basis): the packed tabulation array lives either in the
// kernel parameter bank (DFMA reads it as a c[0x0][imm] operand: zero load
// instructions) or is staged once per CTA into shared memory.
#include <cstdio>
#include <cstring>
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
    const int ngroups = static_cast<int>(kp.group_entries.size());
    for (int g = 0; g < ngroups; ++g)
        o.line("  const int* goff" + std::to_string(g) + "; const int* glist" + std::to_string(g) +
               "; const unsigned short* gloc" + std::to_string(g) + ";");
    o.line("  int n_cells; int stride;");
    if (nt_param > 0) o.line("  double tab[" + std::to_string(nt_param) + "];");
    o.line("};");
}

// Per-cell body for Scpt/Tile: one thread computes one whole cell in registers.
void emit_cell_body(Out& o, const Signature& sig, const KernelPlan& kp, const MapUse& use, bool tile,
                    bool unroll_q) {
    const int d = sig.dim, Q = sig.Q;
    auto TAB = [&](const std::string& idx) {
        return kp.basis == FEMGPU_BASIS_CONST ? "P.tab[" + idx + "]" : "sT[" + idx + "]";
    };
    const std::string C = "P.stride";
    // ---- gather (form.hpp:498-509)
    o.line("// gather");
    for (int i = 0; i < sig.ns(); ++i) {
        for (int j = 0; j < sig.sdofs[i]; ++j) {
            std::string idx = std::to_string(j) + "*(size_t)" + C + "+cell";
            if (tile && kp.sgroup[i] >= 0)
                o.line("const double " + nm("u", i, j) + " = xs" + std::to_string(i) + "[P.gloc" +
                       std::to_string(kp.sgroup[i]) + "[" + idx + "]];");
            else
                o.line("const double " + nm("u", i, j) + " = __ldg(&P.x" + std::to_string(i) + "[__ldg(&P.m" +
                       std::to_string(i) + "[" + idx + "])]);");
        }
    }
    for (int i = 0; i < sig.nv(); ++i) {
        std::set<int> comps(sig.vcomps[i].begin(), sig.vcomps[i].end());
        for (int j = 0; j < sig.vdofs[i]; ++j) {
            std::string idx = std::to_string(j) + "*(size_t)" + C + "+cell";
            std::string node = nm("vn", i, j);
            if (tile && kp.vgroup[i] >= 0)
                o.line("const int " + node + " = P.gloc" + std::to_string(kp.vgroup[i]) + "[" + idx + "];");
            else
                o.line("const int " + node + " = __ldg(&P.vm" + std::to_string(i) + "[" + idx + "]);");
            for (int c : comps) {
                if (tile && kp.vgroup[i] >= 0)
                    o.line("const double " + nm("w", i, j, c) + " = vs" + std::to_string(i) + "[" + node + "*" +
                           std::to_string(d) + "+" + std::to_string(c) + "];");
                else
                    o.line("const double " + nm("w", i, j, c) + " = __ldg(&P.v" + std::to_string(i) + "[(size_t)" +
                           node + "*" + std::to_string(d) + "+" + std::to_string(c) + "]);");
            }
        }
    }
    // ---- geometry (form.hpp:511-520, 441-457)
    if (sig.affine) {
        o.line("// coordinates + affine jacobian");
        for (int j = 0; j < sig.coord_dofs; ++j) {
            std::string idx = std::to_string(j) + "*(size_t)" + C + "+cell";
            std::string vtx = nm("cv", j);
            if (tile && kp.cgroup >= 0)
                o.line("const int " + vtx + " = P.gloc" + std::to_string(kp.cgroup) + "[" + idx + "];");
            else
                o.line("const int " + vtx + " = __ldg(&P.cm[" + idx + "]);");
            for (int c = 0; c < d; ++c) {
                if (tile && kp.cgroup >= 0)
                    o.line("const double " + nm("X", j, c) + " = Xs[" + vtx + "*" + std::to_string(d) + "+" +
                           std::to_string(c) + "];");
                else
                    o.line("const double " + nm("X", j, c) + " = __ldg(&P.X[(size_t)" + vtx + "*" + std::to_string(d) +
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
        for (int jw = 0; jw < sig.nW; ++jw)
            for (int k = 0; k < sig.Tw; ++k) {
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
        if (tile)
            o.line("atomicAdd(&ys[P.gloc" + std::to_string(kp.tgroup) + "[" + idx + "]], o" + std::to_string(jw) + ");");
        else
            o.line("atomicAdd(&P.y[__ldg(&P.tm[" + idx + "])], o" + std::to_string(jw) + ");");
    }
    o.ind--;
    o.line("}");
}

const char* kPrelude = R"(// generated by femgpu (emit.cpp) for sm_100a
#define NF(v) ((((unsigned)__double2hiint(v)) & 0x7ff00000u) == 0x7ff00000u)
// acc += a*b exactly as the reference writes it; contracted to DFMA unless --fmad=false
#define FMA(a, b, acc) ((acc) + (a) * (b))
)";

}  // namespace

std::string KernelPlan::key() const {
    std::ostringstream s;
    s << int(family) << "/" << basis << "/" << block << "/" << tile_cells << "/" << Nc << "x" << Nwi << "/" << TQ << "/"
      << Ter << "/" << Tqr << "/" << Tqc << "/" << strict;
    for (int t : Tcs) s << "s" << t;
    for (int t : Tcv) s << "v" << t;
    for (size_t g = 0; g < group_cap.size(); ++g) s << "g" << group_entries[g] << ":" << group_cap[g];
    for (int g : sgroup) s << "S" << g;
    for (int g : vgroup) s << "V" << g;
    s << "T" << tgroup << "C" << cgroup;
    return s.str();
}

EmitResult emit_mlt(const Signature& sig, const KernelPlan& kp);  // emit_mlt.cpp

EmitResult emit_kernel(const Signature& sig, const KernelPlan& kp) {
    if (kp.family == Family::Mlt) return emit_mlt(sig, kp);
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
    const bool unroll_q = fmas * sig.Q <= 6000;

    const std::string name = tile ? "femgpu_tile" : "femgpu_scpt";
    r.kernel = name;
    r.kernel_checked = name + "_checked";

    // smem layout (doubles): [tab (smem basis)] [ys] [xs_i] [vs_i] [Xs]
    long long off = 0;
    long long off_tab = -1, off_y = -1, off_X = -1;
    std::vector<long long> off_x(sig.ns(), -1), off_v(sig.nv(), -1);
    if (kp.basis == FEMGPU_BASIS_SMEM) {
        off_tab = off;
        off += sig.tab_size;
    }
    if (tile) {
        off_y = off;
        off += kp.group_cap[kp.tgroup];
        for (int i = 0; i < sig.ns(); ++i)
            if (kp.sgroup[i] >= 0) {
                off_x[i] = off;
                off += kp.group_cap[kp.sgroup[i]];
            }
        for (int i = 0; i < sig.nv(); ++i)
            if (kp.vgroup[i] >= 0) {
                off_v[i] = off;
                off += static_cast<long long>(kp.group_cap[kp.vgroup[i]]) * sig.dim;
            }
        if (sig.affine && kp.cgroup >= 0) {
            off_X = off;
            off += static_cast<long long>(kp.group_cap[kp.cgroup]) * sig.dim;
        }
    }
    r.smem_bytes = static_cast<size_t>(off) * 8;

    for (int checked = 0; checked < 2; ++checked) {
        const std::string kn = checked ? r.kernel_checked : r.kernel;
        o.line("");
        o.line(std::string("extern \"C\" __global__ void ") + (checked ? "" : "__launch_bounds__(" + std::to_string(kp.block) + ") ") +
               kn + "(const __grid_constant__ Params P) {");
        o.ind++;
        o.line(std::string("constexpr bool CHECKED = ") + (checked ? "true" : "false") + ";");
        if (off > 0) o.line("extern __shared__ double smem[];");
        if (kp.basis == FEMGPU_BASIS_SMEM) {
            o.line("double* sT = smem + " + std::to_string(off_tab) + ";");
            o.line("for (int i = threadIdx.x; i < " + std::to_string(sig.tab_size) + "; i += blockDim.x) sT[i] = P.tabg[i];");
        }
        if (tile) {
            o.line("const int tile = blockIdx.x;");
            o.line("const int cell = tile * " + std::to_string(kp.tile_cells) + " + threadIdx.x;");
            o.line("double* ys = smem + " + std::to_string(off_y) + ";");
            for (int i = 0; i < sig.ns(); ++i)
                if (off_x[i] >= 0) o.line("double* xs" + std::to_string(i) + " = smem + " + std::to_string(off_x[i]) + ";");
            for (int i = 0; i < sig.nv(); ++i)
                if (off_v[i] >= 0) o.line("double* vs" + std::to_string(i) + " = smem + " + std::to_string(off_v[i]) + ";");
            if (off_X >= 0) o.line("double* Xs = smem + " + std::to_string(off_X) + ";");
            // stage every group's unique entries
            const int ngroups = static_cast<int>(kp.group_entries.size());
            for (int g = 0; g < ngroups; ++g) {
                std::string G = std::to_string(g);
                o.line("{");
                o.ind++;
                o.line("const int b = __ldg(&P.goff" + G + "[tile]), n = __ldg(&P.goff" + G + "[tile + 1]) - b;");
                o.line("for (int u = threadIdx.x; u < n; u += blockDim.x) {");
                o.ind++;
                o.line("const int gi = __ldg(&P.glist" + G + "[b + u]) & 0x7fffffff;");
                if (g == kp.tgroup) o.line("ys[u] = 0.0;");
                for (int i = 0; i < sig.ns(); ++i)
                    if (kp.sgroup[i] == g) o.line("xs" + std::to_string(i) + "[u] = __ldg(&P.x" + std::to_string(i) + "[gi]);");
                for (int i = 0; i < sig.nv(); ++i)
                    if (kp.vgroup[i] == g)
                        for (int c = 0; c < sig.dim; ++c)
                            o.line("vs" + std::to_string(i) + "[u*" + std::to_string(sig.dim) + "+" + std::to_string(c) +
                                   "] = __ldg(&P.v" + std::to_string(i) + "[(size_t)gi*" + std::to_string(sig.dim) + "+" +
                                   std::to_string(c) + "]);");
                if (sig.affine && kp.cgroup == g)
                    for (int c = 0; c < sig.dim; ++c)
                        o.line("Xs[u*" + std::to_string(sig.dim) + "+" + std::to_string(c) + "] = __ldg(&P.X[(size_t)gi*" +
                               std::to_string(sig.dim) + "+" + std::to_string(c) + "]);");
                o.ind--;
                o.line("}");
                o.ind--;
                o.line("}");
            }
            o.line("__syncthreads();");
        } else {
            if (kp.basis == FEMGPU_BASIS_SMEM) o.line("__syncthreads();");
            o.line("const int cell = blockIdx.x * " + std::to_string(kp.block) + " + threadIdx.x;");
        }
        o.line("int stage = -1; (void)stage;");
        o.line("if (cell < P.n_cells) {");
        o.ind++;
        emit_cell_body(o, sig, kp, use, tile, unroll_q);
        o.ind--;
        o.line("}");
        o.line("goto done;");
        o.line("report:");
        o.line("  atomicMin(P.bad, (unsigned long long)cell * 4ull + (unsigned long long)stage);");
        o.line("done:");
        if (tile && !checked) {
            const std::string G = std::to_string(kp.tgroup);
            o.line("__syncthreads();");
            o.line("{");
            o.ind++;
            o.line("const int b = __ldg(&P.goff" + G + "[tile]), n = __ldg(&P.goff" + G + "[tile + 1]) - b;");
            o.line("for (int u = threadIdx.x; u < n; u += blockDim.x) {");
            o.line("  const int e = __ldg(&P.glist" + G + "[b + u]);");
            o.line("  if (e < 0) atomicAdd(&P.y[e & 0x7fffffff], ys[u]); else P.y[e] = ys[u];");
            o.line("}");
            o.ind--;
            o.line("}");
        }
        o.line("return;");
        o.ind--;
        o.line("}");
    }
    r.source = o.s.str();
    r.param_bytes = 0;
    return r;
}

}  // namespace femgpu

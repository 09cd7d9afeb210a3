// emit_dmma.cpp — the warp-level FP64 tensor-core family (femgpu_dmma).
//
// The reference's action (reference_action, form.hpp:497-593) contracts, per cell,
//   evaluation   s_t(q)   = sum_j  Phi_t(q, j) u_j            (form.hpp:526-555)
//   quadrature   y_jw    += sum_k  Psi_k(jw, q) e_k(q)        (form.hpp:575-585)
// Over 8 cells both are small dense GEMMs with the cells as the M dimension:
//   S^T[c][(t,q)] = U^T[c][j] . Phi^T[j][(t,q)]      Y^T[c][jw] = E^T[c][(k,q)] . Psi^T[(k,q)][jw]
// sm_100a has no FP64 kind of tcgen05 (ptxas rejects .kind::f64); its FP64 tensor path is
// DMMA (mma.sync m8n8k4 .f64).  This family keeps the whole per-cell pipeline of one warp in
// registers, with no block-level synchronisation after the one-time fragment staging:
//
//   warp task = CW cells (MB m-blocks of 8; persistent warps, grid-stride over tasks)
//     geometry  lane l computes cell l's affine J / det and the cell-invariant map nodes once
//               (no 4x lane redundancy) into a warp-private shared-memory row
//     per m-block of 8 cells (lane = 4*r + g: cell r, lane-group g):
//       gather  A fragments a[ks] = u[cell r][j = 4 ks + g] straight from global memory
//       per quadrature chunk of T^Q = 4*TQL points (lane-group g owns q = chunk*T^Q + 4 s + g):
//         eval  DMMA, B = Phi^T fragments (fragment-major, built at create) -> D[r][2g+i]:
//               lane-group g's output slots are exactly (term, s) of its own quadrature points,
//               so the pointwise map runs on the DMMA accumulators in place
//         map   the pointwise DAG (straight-line SSA, as in the other families) per (cell, q)
//         quad  DMMA with A = E^T built from the map outputs without any shuffle: k-step
//               kappa = (k, s) takes column g from lane-group g (the K order of Psi^T is
//               permuted at create to match, the FA2 register-reuse trick for m8n8k4)
//       scatter red.global.add.f64 straight from the Y^T accumulator fragments
//
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64, row.col): a0 = A[lane>>2][lane&3];
// b0 = B[lane&3][lane>>2]; {c0,c1} = C[lane>>2][2*(lane&3) + {0,1}].
// Rows (cells) are independent in every GEMM and padded K entries are zero in both operands,
// so a non-finite input of one cell only reaches that cell's outputs; the lane flags the lowest
// failing cell (like the reference's first failing cell) and the stage-checked twin names the
// stage.
#include <algorithm>
#include <cstdlib>
#include <set>
#include <sstream>

#include "femgpu_internal.hpp"

namespace femgpu {

namespace {
std::string S(long long v) { return std::to_string(v); }
}  // namespace

DmmaLayout dmma_layout(const Signature& sig, const KernelPlan& kp) {
    DmmaLayout L;
    L.CW = kp.Nc;
    L.MB = kp.Nc / 8;
    L.TQ = kp.TQ;
    L.TQL = kp.TQ / 4;
    L.NCH = (sig.Q + kp.TQ - 1) / kp.TQ;
    for (int i = 0; i < sig.ns(); ++i) {
        DmmaGroup g;
        g.vec = false;
        g.space = i;
        g.comp = 0;
        g.n = sig.sdofs[i];
        for (int t = 0; t < sig.sterms[i]; ++t) g.terms.push_back(t);
        L.groups.push_back(g);
    }
    for (int i = 0; i < sig.nv(); ++i) {
        std::set<int> comps(sig.vcomps[i].begin(), sig.vcomps[i].end());
        for (int a : comps) {
            DmmaGroup g;
            g.vec = true;
            g.space = i;
            g.comp = a;
            g.n = sig.vdofs[i];
            for (int t = 0; t < sig.vterms[i]; ++t)
                if (sig.vcomps[i][t] == a) g.terms.push_back(t);
            L.groups.push_back(g);
        }
    }
    long long f = 0;
    for (auto& g : L.groups) {
        g.KS = (g.n + 3) / 4;
        g.NB = (static_cast<int>(g.terms.size()) * L.TQL + 1) / 2;
        g.foff = f;
        f += static_cast<long long>(g.NB) * g.KS;
    }
    L.KQ = sig.Tw * L.TQL;
    L.NBQ = (sig.nW + 7) / 8;
    L.foff_q = f;
    f += static_cast<long long>(L.NBQ) * L.KQ;
    L.FPC = f;
    L.nfrag = L.FPC * L.NCH;
    return L;
}

// Fragment-major B operands: [chunk][group (n-block, k-step)..., quad (n-block, k-step)][lane].
std::vector<double> dmma_fragments(const Signature& sig, const DmmaLayout& L, const std::vector<double>& tab) {
    std::vector<double> fr(static_cast<size_t>(L.nfrag * 32), 0.0);
    const int Q = sig.Q, TQL = L.TQL;
    for (int ch = 0; ch < L.NCH; ++ch) {
        double* base = fr.data() + static_cast<size_t>(ch) * L.FPC * 32;
        for (const auto& g : L.groups) {
            const long long phi = g.vec ? sig.phi_off_v[g.space] : sig.phi_off_s[g.space];
            const int T = static_cast<int>(g.terms.size());
            for (int nb = 0; nb < g.NB; ++nb)
                for (int ks = 0; ks < g.KS; ++ks)
                    for (int lane = 0; lane < 32; ++lane) {
                        // b0 = B[k = lane&3][n = lane>>2]; column n = 2*g' + i -> slot 2*nb + i of lane-group g'
                        const int j = ks * 4 + (lane & 3), n = lane >> 2, gq = n >> 1, slot = 2 * nb + (n & 1);
                        const int ti = slot / TQL, s = slot % TQL, q = ch * L.TQ + 4 * s + gq;
                        double v = 0.0;
                        if (ti < T && q < Q && j < g.n)
                            v = tab[phi + static_cast<long long>(g.terms[ti]) * Q * g.n + static_cast<long long>(q) * g.n + j];
                        base[(g.foff + static_cast<long long>(nb) * g.KS + ks) * 32 + lane] = v;
                    }
        }
        for (int nb = 0; nb < L.NBQ; ++nb)
            for (int kq = 0; kq < L.KQ; ++kq)
                for (int lane = 0; lane < 32; ++lane) {
                    // b0 = B[kk = lane&3][jw = lane>>2]; k-step kq = (k, s), row kk taken from lane-group kk
                    const int k = kq / TQL, s = kq % TQL, jw = nb * 8 + (lane >> 2), q = ch * L.TQ + 4 * s + (lane & 3);
                    double v = 0.0;
                    if (jw < sig.nW && q < Q)
                        v = tab[sig.psi_off + (static_cast<long long>(k) * sig.nW + jw) * Q + q];
                    base[(L.foff_q + static_cast<long long>(nb) * L.KQ + kq) * 32 + lane] = v;
                }
    }
    return fr;
}

namespace {

// Cell-invariant map nodes the quadrature-point part reads (constants are re-emitted).
struct Hoist {
    std::vector<int> stored;  // node ids kept in the warp's shared-memory rows
    std::vector<int> consts;  // constant node ids re-emitted in the map phase
};

Hoist hoisted(const Signature& sig, const std::vector<char>& live, const std::vector<char>& qdep) {
    std::set<int> need;
    for (size_t id = 0; id < sig.nodes.size(); ++id) {
        if (!live[id] || !qdep[id]) continue;
        const MapNode& n = sig.nodes[id];
        if (n.op == FEMGPU_OP_ADD || n.op == FEMGPU_OP_MUL) {
            if (!qdep[n.a]) need.insert(n.a);
            if (!qdep[n.b]) need.insert(n.b);
        }
    }
    for (int o : sig.outputs)
        if (!qdep[o]) need.insert(o);
    Hoist h;
    for (int id : need) {
        if (sig.nodes[id].op == FEMGPU_OP_CONSTANT)
            h.consts.push_back(id);
        else
            h.stored.push_back(id);
    }
    return h;
}

}  // namespace

// Shared with emit.cpp
std::vector<char> map_live(const Signature& sig);
std::vector<char> map_qdep(const Signature& sig);
void emit_map_nodes(std::ostringstream& o, const Signature& sig, const std::vector<char>& live,
                    const std::vector<char>& qdep, bool qdep_pass, const std::string& weight_expr);
void emit_geometry(std::ostringstream& o, const Signature& sig, bool uses_inv, const std::string& cell);

namespace {
struct Smem {
    long long off_A = 0, off_H = 0, total = 0;  // doubles
    int nH = 0;
};
Smem dmma_smem(const Signature& sig, const KernelPlan& kp, const DmmaLayout& L) {
    Smem s;
    const Hoist H = hoisted(sig, map_live(sig), map_qdep(sig));
    s.nH = static_cast<int>(H.stored.size());
    long long off = 0;
    if (kp.basis == FEMGPU_BASIS_SMEM) off += L.nfrag * 32;
    s.off_H = off;
    off += static_cast<long long>(kp.block / 32) * s.nH * L.CW;
    s.total = off;
    return s;
}
}  // namespace

size_t dmma_smem_bytes(const Signature& sig, const KernelPlan& kp) {
    const DmmaLayout L = dmma_layout(sig, kp);
    return static_cast<size_t>(dmma_smem(sig, kp, L).total * 8);
}

// Live doubles per lane of one m-block (register-pressure estimate used by the auto schedule).
long long dmma_live_doubles(const Signature& sig, const DmmaLayout& L) {
    long long a = 0, s = 0;
    for (const auto& g : L.groups) {
        a += g.KS;
        s += 2LL * g.NB;
    }
    return a + s + static_cast<long long>(sig.Tw) * L.TQL + 2LL * L.NBQ;
}

void emit_dmma_kernel(std::ostringstream& o, const Signature& sig, const KernelPlan& kp, DmmaLayout& L,
                      const std::string& name) {
    const std::vector<char> live = map_live(sig), qdep = map_qdep(sig);
    const Hoist H = hoisted(sig, live, qdep);
    const Smem SM = dmma_smem(sig, kp, L);
    const int NT = kp.block, NW = NT / 32, CW = L.CW, MB = L.MB, TQL = L.TQL, nH = SM.nH;
    const int MBJ = std::max(1, kp.Ter), PF = kp.Tqr > 0 ? 1 : 0;
    const bool tv = kp.tvec >= 0 && std::getenv("FEMGPU_DEBUG_NO_TVEC") == nullptr;
    const bool breg = kp.breg && L.NCH == 1;
    const bool smemA = kp.basis == FEMGPU_BASIS_SMEM;
    // timing experiments only (wrong results): plain stores instead of red.add in the scatter
    const bool scatter_store = std::getenv("FEMGPU_DEBUG_SCATTER_STORE") != nullptr;
    // timing experiments only (wrong results): value gathers from 64 nodes (L1-resident, few wavefronts)
    const std::string gx = std::getenv("FEMGPU_DEBUG_GATHER_LOCAL") != nullptr ? " & 63)" : ")";
    bool uses_inv = false;
    for (size_t id = 0; id < sig.nodes.size(); ++id)
        if (live[id] && sig.nodes[id].op == FEMGPU_OP_INV_JACOBIAN) uses_inv = true;
    // which derivative variables the map reads (the rest are still checked for finiteness)
    std::set<std::pair<int, int>> sd_used, vd_used;
    for (size_t id = 0; id < sig.nodes.size(); ++id) {
        if (!live[id]) continue;
        if (sig.nodes[id].op == FEMGPU_OP_SCALAR_DERIV) sd_used.insert({sig.nodes[id].a, sig.nodes[id].b});
        if (sig.nodes[id].op == FEMGPU_OP_VECTOR_DERIV) vd_used.insert({sig.nodes[id].a, sig.nodes[id].b});
    }

    o << "\nextern \"C\" __global__ void __launch_bounds__(" << NT << (kp.min_blocks > 1 ? ", " + S(kp.min_blocks) : "")
      << ") " << name << "(const __grid_constant__ Params P) {\n";
    o << "  extern __shared__ __align__(16) double sm[];\n";
    o << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n";
    // fused zeroing of [zp, zp + zn) in a CTA prologue (a slice per warp task inside the task loop
    // measured slower: C4 1939 vs 1872 us per pipelined step)
    if (kp.zfused) o << kZeroPrologue;
    o << "  const int r = lane >> 2, g = lane & 3;\n";
    o << "  const size_t STR = (size_t)P.stride;\n";
    if (smemA) {
        o << "  for (int i = tid; i < " << L.nfrag * 16 << "; i += " << NT
          << ") reinterpret_cast<double2*>(sm)[i] = __ldg(reinterpret_cast<const double2*>(P.afr) + i);\n";
        o << "  __syncthreads();\n";
        o << "  const double* const FR = sm + lane;\n";
    } else {
        o << "  const double* const FR = P.afr + lane;\n";
    }
    o << "  double* const sH = sm + " << SM.off_H << " + warp * " << static_cast<long long>(nH) * CW << "; (void)sH;\n";
    if (breg)  // single chunk: every B fragment of the form lives in registers for the whole kernel
        for (long long f = 0; f < L.FPC; ++f) o << "  const double Bf" << f << " = FR[" << f * 32 << "];\n";
    o << "  const int n_tasks = (P.n_cells - P.cell0 + " << CW - 1 << ") / " << CW << ";\n";
    o << "  unsigned long long badc = ~0ULL;\n";
    o << "  #pragma unroll 1\n";
    o << "  for (int task = blockIdx.x * " << NW << " + warp; task < n_tasks; task += gridDim.x * " << NW << ") {\n";
    o << "    const int c0 = P.cell0 + task * " << CW << ";\n";
    // ---- geometry + cell-invariant nodes, one lane per cell (emitted after the first m-group's
    // gather has been issued, so its latency overlaps the geometry)
    std::ostringstream geo;
    {
    std::ostringstream& o = geo;
    if (sig.affine || nH > 0) {
        o << "    if (lane < " << CW << ") {\n";
        o << "      const bool cok = c0 + lane < P.n_cells;\n";
        o << "      const int cell = cok ? c0 + lane : c0;\n";
        if (sig.affine) {
            std::ostringstream gm;
            emit_geometry(gm, sig, uses_inv, "cell");
            o << gm.str();
            o << "      if (cok && NF(det)) badc = min(badc, (unsigned long long)cell);\n";
        }
        {
            std::ostringstream m;
            emit_map_nodes(m, sig, live, qdep, false, "0.0");
            o << m.str();
        }
        for (int h = 0; h < nH; ++h) o << "      sH[" << static_cast<long long>(h) * CW << " + lane] = n" << H.stored[h] << ";\n";
        o << "    }\n";
        o << "    __syncwarp();\n";
    }
    }
    // ---- m-groups of MBJ m-blocks sharing every B-fragment load; optional software prefetch:
    // indices two m-groups ahead, values one m-group ahead (loop-carried registers).
    std::vector<std::vector<int>> by_space_s(sig.ns()), by_space_v(sig.nv());
    for (size_t gi = 0; gi < L.groups.size(); ++gi)
        (L.groups[gi].vec ? by_space_v[L.groups[gi].space] : by_space_s[L.groups[gi].space]).push_back(static_cast<int>(gi));
    struct Sp {
        bool vec;
        int i;
        std::vector<int> gids;
    };
    std::vector<Sp> sps;
    for (int i = 0; i < sig.ns(); ++i) sps.push_back({false, i, by_space_s[i]});
    for (int i = 0; i < sig.nv(); ++i) sps.push_back({true, i, by_space_v[i]});
    const std::string J = "_j";
    auto ixname = [&](const std::string& pre, const Sp& sp, int ks, int j) {
        return pre + S(sp.vec) + "_" + S(sp.i) + "_" + S(ks) + J + S(j);
    };
    auto uname = [&](const std::string& pre, int gid, int ks, int j) { return pre + S(gid) + "_" + S(ks) + J + S(j); };
    // index loads of m-group `grp` (expression) into `pre` variables (decl: declare const)
    auto emit_idx = [&](const std::string& ind, const std::string& pre, const std::string& grp, bool decl) {
        for (int j = 0; j < MBJ; ++j) {
            const std::string cell = "(c0 + ((" + grp + ") * " + S(MBJ) + " + " + S(j) + ") * 8 + r)";
            for (const Sp& sp : sps) {
                const DmmaGroup& g0 = L.groups[sp.gids[0]];
                for (int ks = 0; ks < g0.KS; ++ks) {
                    const bool partial = (ks + 1) * 4 > g0.n;
                    std::string ok = cell + " < P.n_cells";
                    if (partial) ok += " && " + S(ks * 4) + " + g < " + S(g0.n);
                    o << ind << (decl ? "const int " : "") << ixname(pre, sp, ks, j) << " = (" << ok << ") ? __ldg(&P."
                      << (sp.vec ? "vm" : "m") << sp.i << "[(" << ks * 4 << " + g) * STR + " << cell << "]) : -1;\n";
                }
            }
        }
    };
    auto emit_vals = [&](const std::string& ind, const std::string& ipre, const std::string& upre, bool decl) {
        for (int j = 0; j < MBJ; ++j)
            for (const Sp& sp : sps) {
                const DmmaGroup& g0 = L.groups[sp.gids[0]];
                for (int ks = 0; ks < g0.KS; ++ks) {
                    const std::string ix = ixname(ipre, sp, ks, j);
                    // vector spaces: padded node-major layout, components (0,1) as one 16-byte load
                    int g0c = -1, g1c = -1;
                    if (sp.vec && sig.dim >= 2)
                        for (int gid : sp.gids) {
                            if (L.groups[gid].comp == 0) g0c = gid;
                            if (L.groups[gid].comp == 1) g1c = gid;
                        }
                    const bool pair = g0c >= 0 && g1c >= 0;
                    const std::string pv = "pv" + S(sp.i) + "_" + S(ks) + J + S(j) + "_" + upre;
                    if (pair)
                        o << ind << "const double2 " << pv << " = " << ix << " >= 0 ? __ldg(reinterpret_cast<const double2*>(P.v"
                          << sp.i << " + (size_t)(" << ix << gx << " * " << vec_stride(sig.dim) << ")) : make_double2(0.0, 0.0);\n";
                    for (int gid : sp.gids) {
                        o << ind << (decl ? "const double " : "") << uname(upre, gid, ks, j) << " = ";
                        if (pair && gid == g0c)
                            o << pv << ".x;\n";
                        else if (pair && gid == g1c)
                            o << pv << ".y;\n";
                        else if (sp.vec)
                            o << ix << " >= 0 ? __ldg(&P.v" << sp.i << "[(size_t)(" << ix << gx << " * " << vec_stride(sig.dim) << " + "
                              << L.groups[gid].comp << "]) : 0.0;\n";
                        else
                            o << ix << " >= 0 ? __ldg(&P.x" << sp.i << "[(" << ix << gx << "]) : 0.0;\n";
                    }
                }
            }
    };
    const int NG = MB / MBJ;
    // interleaved vector test space: its node indices feed the scatter too
    const Sp* tsp = nullptr;
    for (const Sp& sp : sps)
        if (tv && sp.vec && sp.i == kp.tvec) tsp = &sp;
    // spaces whose current-m-group indices the scatter reads (tvec, or the per-column aliases)
    auto kept = [&](const Sp& sp) {
        if (&sp == tsp) return true;
        if (tsp || kp.dalias.empty()) return false;
        for (const auto& a : kp.dalias)
            if (a[0] >= 0 && (a[0] == 1) == sp.vec && a[1] == sp.i) return true;
        return false;
    };
    if (PF) {
        // loop-carried prefetch registers: ixN = indices of m-group grp+1, uN = values of grp,
        // ixK = indices of grp (only the test-space indices are kept)
        for (int j = 0; j < MBJ; ++j)
            for (const Sp& sp : sps) {
                const DmmaGroup& g0 = L.groups[sp.gids[0]];
                for (int ks = 0; ks < g0.KS; ++ks) {
                    o << "    int " << ixname("ixN", sp, ks, j) << " = -1;\n";
                    if (kept(sp)) o << "    int " << ixname("ixK", sp, ks, j) << " = -1;\n";
                    for (int gid : sp.gids) o << "    double " << uname("uN", gid, ks, j) << " = 0.0;\n";
                }
            }
    }
    auto copy_tidx = [&](const std::string& ind, const std::string& dst, const std::string& src) {
        for (const Sp& sp : sps) {
            if (!kept(sp)) continue;
            for (int j = 0; j < MBJ; ++j)
                for (int ks = 0; ks < L.groups[sp.gids[0]].KS; ++ks)
                    o << ind << ixname(dst, sp, ks, j) << " = " << ixname(src, sp, ks, j) << ";\n";
        }
    };
    if (PF) {
        // stage chain: m-group 0 loads its own indices+values (before the geometry), later m-groups
        // were prefetched one iteration ahead
        emit_idx("    ", "ixN", "0", false);
        emit_vals("    ", "ixN", "uN", false);
        copy_tidx("    ", "ixK", "ixN");
        if (NG > 1) emit_idx("    ", "ixN", "1", false);
    }
    o << geo.str();
    o << "    #pragma unroll 1\n";
    o << "    for (int grp = 0; grp < " << NG << "; ++grp) {\n";
    if (PF) {
        for (int j = 0; j < MBJ; ++j)
            for (const Sp& sp : sps)
                for (int ks = 0; ks < L.groups[sp.gids[0]].KS; ++ks) {
                    for (int gid : sp.gids)
                        o << "      const double " << uname("uA", gid, ks, j) << " = " << uname("uN", gid, ks, j) << ";\n";
                    if (kept(sp))
                        o << "      const int " << ixname("ixC", sp, ks, j) << " = " << ixname("ixK", sp, ks, j) << ";\n";
                }
        if (NG > 1) {
            o << "      if (grp + 1 < " << NG << ") {\n";
            emit_vals("        ", "ixN", "uN", false);
            copy_tidx("        ", "ixK", "ixN");
            o << "      }\n";
            if (NG > 2) {
                o << "      if (grp + 2 < " << NG << ") {\n";
                emit_idx("        ", "ixN", "grp + 2", false);
                o << "      }\n";
            }
        }
    } else {
        // (issuing m-group 0 before the geometry was measured neutral on C4 and 15 % slower on the
        //  register-bound C5-hyp-P3/P4: the gathered values stay live across the geometry)
        emit_idx("      ", "ix", "grp", true);
        emit_vals("      ", "ix", "uA", true);
    }
    for (int j = 0; j < MBJ; ++j) {
        o << "      const int cr" << j << " = (grp * " << MBJ << " + " << j << ") * 8 + r, cell" << j << " = c0 + cr" << j << ";\n";
        o << "      const bool cok" << j << " = cell" << j << " < P.n_cells;\n";
        for (int h = 0; h < nH; ++h)
            o << "      const double hv" << h << J << j << " = sH[" << static_cast<long long>(h) * CW << " + cr" << j << "];\n";
        for (int nb = 0; nb < L.NBQ; ++nb)
            o << "      double y" << nb << J << j << "_0 = 0.0, y" << nb << J << j << "_1 = 0.0;\n";
    }
    // quadrature chunks: rolled, or two per trip (qmopt bit 14: more independent DMMA chains)
    o << ((kp.qmopt & 16384) ? "      #pragma unroll 2\n" : "      #pragma unroll 1\n");
    o << "      for (int ch = 0; ch < " << L.NCH << "; ++ch) {\n";
    o << "        const double* const Fc = FR + (size_t)ch * " << L.FPC * 32 << "; (void)Fc;\n";
    // ---- evaluation GEMMs (one B fragment load feeds MBJ DMMAs)
    for (size_t gi = 0; gi < L.groups.size(); ++gi) {
        const DmmaGroup& g = L.groups[gi];
        for (int nb = 0; nb < g.NB; ++nb) {
            for (int j = 0; j < MBJ; ++j)
                o << "        double S" << gi << "_" << nb << J << j << "_0 = 0.0, S" << gi << "_" << nb << J << j << "_1 = 0.0;\n";
            for (int ks = 0; ks < g.KS; ++ks) {
                const long long f = g.foff + static_cast<long long>(nb) * g.KS + ks;
                o << "        { const double b = " << (breg ? "Bf" + S(f) : "Fc[" + S(f * 32) + "]") << ";";
                for (int j = 0; j < MBJ; ++j)
                    o << " DMMA(S" << gi << "_" << nb << J << j << "_0, S" << gi << "_" << nb << J << j << "_1, "
                      << uname("uA", static_cast<int>(gi), ks, j) << ", b);";
                o << " }\n";
            }
        }
    }
    // ---- pointwise map per (m-block, owned quadrature point)
    for (int s = 0; s < TQL; ++s) {
        o << "        const int q" << s << " = ch * " << L.TQ << " + " << 4 * s << " + g;\n";
        o << "        const bool qok" << s << " = q" << s << " < " << sig.Q << ";\n";
        o << "        const double wq" << s << " = qok" << s << " ? __ldg(&P.tabg[" << sig.w_off << " + q" << s << "]) : 0.0;\n";
    }
    // map of owned point s for every m-block, then at once its quadrature k-steps kappa = (k, s):
    // E values die right after their DMMAs (register pressure), sum order over kappa is s-major
    for (int s = 0; s < TQL; ++s) {
        for (int j = 0; j < MBJ; ++j) {
            o << "        double E" << s << "_0" << J << j;
            for (int k = 1; k < sig.Tw; ++k) o << ", E" << s << "_" << k << J << j;
            o << ";\n";
            o << "        {\n";
            std::string nf = "false";
            for (size_t gi = 0; gi < L.groups.size(); ++gi) {
                const DmmaGroup& g = L.groups[gi];
                for (size_t ti = 0; ti < g.terms.size(); ++ti) {
                    const int slot = static_cast<int>(ti) * TQL + s;
                    const std::string v = (g.vec ? "t" : "s") + S(g.space) + "_" + S(g.terms[ti]);
                    o << "          const double " << v << " = S" << gi << "_" << slot / 2 << J << j << "_" << slot % 2 << ";\n";
                    const bool used = g.vec ? vd_used.count({g.space, g.terms[ti]}) : sd_used.count({g.space, g.terms[ti]});
                    if (!used) nf += " | NF(" + v + ")";
                }
            }
            for (int h = 0; h < nH; ++h) o << "          const double n" << H.stored[h] << " = hv" << h << J << j << ";\n";
            for (int id : H.consts) {
                char buf[64];
                std::snprintf(buf, sizeof buf, "%a", sig.nodes[id].value);
                o << "          const double n" << id << " = (" << buf << ");\n";
            }
            {
                std::ostringstream m;
                emit_map_nodes(m, sig, live, qdep, true, "wq" + S(s));
                o << m.str();
            }
            for (int k = 0; k < sig.Tw; ++k) {
                o << "          E" << s << "_" << k << J << j << " = qok" << s << " ? n" << sig.outputs[k] << " : 0.0;\n";
                nf += " | NF(n" + S(sig.outputs[k]) + ")";
            }
            o << "          if (cok" << j << " && qok" << s << " && (" << nf << ")) badc = min(badc, (unsigned long long)cell" << j
              << ");\n";
            o << "        }\n";
        }
        // ---- quadrature GEMM: k-steps kappa = (k, s) of this owned point
        for (int k = 0; k < sig.Tw; ++k) {
            const int kq = k * TQL + s;
            for (int nb = 0; nb < L.NBQ; ++nb) {
                // a fragment whose test DOFs all have Psi(k, jw, .) == 0 adds nothing (fused problems'
                // off-diagonal blocks): no DMMA
                bool zero = true;
                for (int jw = nb * 8; jw < std::min(sig.nW, nb * 8 + 8) && zero; ++jw) zero = !sig.pnz(k, jw);
                if (zero) continue;
                const long long f = L.foff_q + static_cast<long long>(nb) * L.KQ + kq;
                o << "        { const double b = " << (breg ? "Bf" + S(f) : "Fc[" + S(f * 32) + "]") << ";";
                for (int j = 0; j < MBJ; ++j)
                    o << " DMMA(y" << nb << J << j << "_0, y" << nb << J << j << "_1, E" << s << "_" << k << J << j << ", b);";
                o << " }\n";
            }
        }
    }
    o << "      }\n";  // chunks
    // ---- scatter from the accumulator fragments
    for (int j = 0; j < MBJ; ++j) {
        if (tsp) {
            // interleaved vector test space: y index = node(cell, a) * dim + comp with jw = a * dim + comp;
            // node(cell r, a) was gathered by lane 4r + (a & 3) as its k-step a >> 2 index
            const int d = sig.dim, KS = L.groups[tsp->gids[0]].KS;
            for (int nb = 0; nb < L.NBQ; ++nb)
                for (int i = 0; i < 2; ++i) {
                    const int jlo = nb * 8 + i, jhi = std::min(nb * 8 + i + 6, sig.nW - 1);
                    if (jlo > sig.nW - 1) continue;
                    const int klo = (jlo / d) >> 2, khi = (jhi / d) >> 2;
                    o << "      int ty" << nb << "_" << i << J << j << ";\n";
                    o << "      {\n        const int jw = " << nb * 8 + i << " + 2 * g, a = jw / " << d << ";\n";
                    o << "        const int src = (r << 2) | (a & 3);\n";
                    std::string sel = "-1";
                    for (int ks = std::min(khi, KS - 1); ks >= klo; --ks) {
                        o << "        const int t" << ks << " = __shfl_sync(0xffffffffu, " << ixname(PF ? "ixC" : "ix", *tsp, ks, j)
                          << ", src);\n";
                        sel = "((a >> 2) == " + S(ks) + " ? t" + S(ks) + " : " + sel + ")";
                    }
                    o << "        ty" << nb << "_" << i << J << j << " = " << sel << " * " << d << " + jw % " << d << ";\n      }\n";
                }
        }
        // per-column aliases (no tvec): rows = scale * gathered node + add, shuffled from the lane that
        // gathered the node; columns without an alias load the test map
        const bool dal = !tsp && !kp.dalias.empty();
        if (dal) {
            for (int nb = 0; nb < L.NBQ; ++nb)
                for (int i = 0; i < 2; ++i) {
                    if (nb * 8 + i >= sig.nW) continue;
                    std::string srcl = "0", scale = "1", add = "0LL", al = "false";
                    std::vector<std::pair<int, int>> srcs;  // distinct (space slot in sps, k-step)
                    std::string pick = "0";
                    for (int gg = 3; gg >= 0; --gg) {
                        const int jw = nb * 8 + i + 2 * gg;
                        if (jw >= sig.nW || kp.dalias[jw][0] < 0) continue;
                        const auto& a = kp.dalias[jw];
                        int spi = -1;
                        for (size_t q = 0; q < sps.size(); ++q)
                            if (sps[q].vec == (a[0] == 1) && sps[q].i == a[1]) spi = static_cast<int>(q);
                        if (spi < 0) continue;
                        const int ks = static_cast<int>(a[2] >> 2);
                        if (std::find(srcs.begin(), srcs.end(), std::make_pair(spi, ks)) == srcs.end()) srcs.push_back({spi, ks});
                        const std::string gq = "g == " + S(gg);
                        srcl = "(" + gq + " ? " + S(a[2] & 3) + " : " + srcl + ")";
                        scale = "(" + gq + " ? " + S(a[3]) + " : " + scale + ")";
                        add = "(" + gq + " ? " + S(a[4]) + "LL : " + add + ")";
                        al = "(" + gq + " || " + al + ")";
                        pick = "(" + gq + " ? t" + S(spi) + "_" + S(ks) + " : " + pick + ")";
                    }
                    o << "      int ta" << nb << "_" << i << J << j << " = 0;\n";
                    o << "      const bool al" << nb << "_" << i << J << j << " = " << al << ";\n";
                    if (srcs.empty()) continue;
                    o << "      {\n        const int src = (r << 2) | " << srcl << ";\n";
                    for (const auto& sk : srcs)
                        o << "        const int t" << sk.first << "_" << sk.second << " = __shfl_sync(0xffffffffu, "
                          << ixname(PF ? "ixC" : "ix", sps[sk.first], sk.second, j) << ", src);\n";
                    o << "        ta" << nb << "_" << i << J << j << " = (int)((long long)" << pick << " * " << scale << " + " << add
                      << ");\n      }\n";
                }
        }
        o << "      if (cok" << j << ") {\n";
        for (int nb = 0; nb < L.NBQ; ++nb)
            for (int i = 0; i < 2; ++i) {
                const std::string v = "y" + S(nb) + J + S(j) + "_" + S(i);
                if (nb * 8 + i >= sig.nW) continue;  // no lane holds a test DOF in this slot
                const bool partial = nb * 8 + 8 > sig.nW;
                o << "        " << (partial ? "if (" + S(nb * 8 + i) + " + 2 * g < " + S(sig.nW) + ") " : "") << "{\n";
                o << "          if (NF(" << v << ")) badc = min(badc, (unsigned long long)cell" << j << ");\n";
                const std::string load = "__ldg(&P.tm[(" + S(nb * 8 + i) + " + 2 * g) * STR + cell" + S(j) + "])";
                const std::string yi = tsp ? "ty" + S(nb) + "_" + S(i) + J + S(j)
                                       : dal ? "(al" + S(nb) + "_" + S(i) + J + S(j) + " ? ta" + S(nb) + "_" + S(i) + J + S(j) + " : " + load + ")"
                                             : load;
                o << "          " << (scatter_store ? "P.y[" : "atomicAdd(&P.y[") << yi << "]" << (scatter_store ? " = " : ", ") << v
                  << (scatter_store ? ";\n" : ");\n");
                o << "        }\n";
            }
        o << "      }\n";
    }
    o << "    }\n";  // m-groups
    if (sig.affine || nH > 0) o << "    __syncwarp();\n";
    o << "  }\n";  // tasks
    o << "  if (badc != ~0ULL) atomicMin(P.bad, badc);\n";
    o << "}\n";
}

}  // namespace femgpu

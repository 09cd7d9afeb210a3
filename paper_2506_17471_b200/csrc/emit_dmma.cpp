// emit_dmma.cpp — the cell-batched FP64 tensor-core family (femgpu_dmma).
//
// The reference's action (reference_action, form.hpp:497-593) contracts, per cell,
//   evaluation   s_t(q)   = sum_j  Phi_t(q, j) u_j            (form.hpp:526-555)
//   quadrature   y_jw    += sum_k  Psi_k(jw, q) e_k(q)        (form.hpp:575-585)
// Over a tile of N_c cells both are small dense GEMMs with the cells as the N
// dimension: S[(t,q)][c] = Phi[(t,q)][j] * U[j][c] and Y[jw][c] = Psi[jw][(k,q)] * E[(k,q)][c].
// sm_100a has no FP64 kind of tcgen05 (ptxas rejects .kind::f64); its FP64 tensor
// path is DMMA (mma.sync m8n8k4 .f64), which this family drives directly:
//
//   per tile of N_c cells (persistent CTAs; N_c multiple of 8):
//     gather   U_g[k][c] (zero-padded to a multiple of 4 rows) for every evaluation
//              group g = (space, component); per-cell geometry (affine J, det) and the
//              cell-invariant map nodes into H[h][c]
//     per quadrature tile of T^Q points (the paper's quad_tile, qoi.hpp:26):
//       eval   warp tasks of R m-blocks x S n-blocks: DMMA over the k-steps, A operand
//              = Phi fragments (fragment-major, prepared at create), B = U_g -> S_g
//       map    one thread per (cell, quadrature point): the pointwise DAG (straight-line
//              SSA, as in the other families) reads S and H, writes E
//       quad   DMMA, A = Psi fragments, B = E; the accumulators Y stay in registers
//              across the quadrature tiles
//     scatter  red.global.add.f64 straight from the accumulator fragments
//
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64): A a0 = A[lane>>2][lane&3];
// B b0 = B[lane&3][lane>>2]; C/D {c0,c1} = C[lane>>2][2*(lane&3) + {0,1}].
// Columns are independent in every GEMM, so a non-finite input of one cell only
// reaches that cell's outputs, which the scatter flags (lowest cell, like the
// reference's first failing cell; the stage is named by the checked twin kernel).
#include <algorithm>
#include <set>
#include <sstream>

#include "femgpu_internal.hpp"

namespace femgpu {

namespace {
std::string S(long long v) { return std::to_string(v); }
// smallest ld >= n with ld % 16 == r (doubles): conflict-free fragment loads/stores
long long ld_mod(long long n, long long r) {
    long long ld = n;
    while (ld % 16 != r) ++ld;
    return ld;
}
}  // namespace

DmmaLayout dmma_layout(const Signature& sig, const KernelPlan& kp) {
    DmmaLayout L;
    L.NC = kp.Nc;
    L.TQ = kp.TQ;
    L.NQT = (sig.Q + kp.TQ - 1) / kp.TQ;
    L.LDU = ld_mod(L.NC, 4);
    if (L.LDU - L.NC > 8) L.LDU = ld_mod(L.NC, 12);
    L.LDS = ld_mod(L.NC, 8);
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
        g.MB = (static_cast<int>(g.terms.size()) * L.TQ + 7) / 8;
        g.foff = f;
        f += static_cast<long long>(g.MB) * g.KS;
    }
    L.KSq = (sig.Tw * L.TQ + 3) / 4;
    L.MBq = (sig.nW + 7) / 8;
    L.foff_q = f;
    f += static_cast<long long>(L.MBq) * L.KSq;
    L.FPT = f;
    // shared-memory plan (doubles)
    long long off = 0;
    if (kp.basis == FEMGPU_BASIS_SMEM) {
        L.off_A = off;
        off += L.NQT * L.FPT * 32;
    }
    for (auto& g : L.groups) {
        g.offU = off;
        off += static_cast<long long>(g.KS) * 4 * L.LDU;
    }
    for (auto& g : L.groups) {
        g.offS = off;
        off += static_cast<long long>(g.MB) * 8 * L.LDS;
    }
    L.off_E = off;
    off += static_cast<long long>(L.KSq) * 4 * L.LDU;
    L.off_H = off;
    L.nH_cap = 0;
    L.smem_doubles = off;  // + H rows (set by the emitter once the hoisted set is known)
    return L;
}

// Fragment-major A operands: [q tile][group (m-block, k-step)..., quad (m-block, k-step)][lane].
std::vector<double> dmma_fragments(const Signature& sig, const DmmaLayout& L, const std::vector<double>& tab) {
    std::vector<double> fr(static_cast<size_t>(L.NQT * L.FPT * 32), 0.0);
    const int Q = sig.Q;
    for (int qt = 0; qt < L.NQT; ++qt) {
        const int q0 = qt * L.TQ;
        double* base = fr.data() + static_cast<size_t>(qt) * L.FPT * 32;
        for (const auto& g : L.groups) {
            const long long phi = g.vec ? sig.phi_off_v[g.space] : sig.phi_off_s[g.space];
            for (int mb = 0; mb < g.MB; ++mb)
                for (int ks = 0; ks < g.KS; ++ks)
                    for (int lane = 0; lane < 32; ++lane) {
                        const int r = mb * 8 + (lane >> 2), k = ks * 4 + (lane & 3);
                        const int tt = r / L.TQ, ql = r % L.TQ, q = q0 + ql;
                        double v = 0.0;
                        if (tt < static_cast<int>(g.terms.size()) && q < Q && k < g.n)
                            v = tab[phi + static_cast<long long>(g.terms[tt]) * Q * g.n + static_cast<long long>(q) * g.n + k];
                        base[((g.foff + static_cast<long long>(mb) * g.KS + ks) * 32) + lane] = v;
                    }
        }
        for (int mb = 0; mb < L.MBq; ++mb)
            for (int ks = 0; ks < L.KSq; ++ks)
                for (int lane = 0; lane < 32; ++lane) {
                    const int jw = mb * 8 + (lane >> 2), kk = ks * 4 + (lane & 3);
                    const int k = kk / L.TQ, ql = kk % L.TQ, q = q0 + ql;
                    double v = 0.0;
                    if (jw < sig.nW && k < sig.Tw && q < Q)
                        v = tab[sig.psi_off + (static_cast<long long>(k) * sig.nW + jw) * Q + q];
                    base[((L.foff_q + static_cast<long long>(mb) * L.KSq + ks) * 32) + lane] = v;
                }
    }
    return fr;
}

namespace {

// Cell-invariant map nodes the quadrature-point part reads (constants are re-emitted).
struct Hoist {
    std::vector<int> stored;  // node ids kept in H rows
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

size_t dmma_smem_bytes(const Signature& sig, const KernelPlan& kp) {
    DmmaLayout L = dmma_layout(sig, kp);
    const Hoist H = hoisted(sig, map_live(sig), map_qdep(sig));
    return static_cast<size_t>((L.off_H + static_cast<long long>(H.stored.size()) * L.LDS) * 8);
}

void emit_dmma_kernel(std::ostringstream& o, const Signature& sig, const KernelPlan& kp, DmmaLayout& L,
                      const std::string& name) {
    const std::vector<char> live = map_live(sig), qdep = map_qdep(sig);
    const Hoist H = hoisted(sig, live, qdep);
    L.nH_cap = static_cast<int>(H.stored.size());
    L.smem_doubles = L.off_H + static_cast<long long>(L.nH_cap) * L.LDS;
    const int NC = L.NC, TQ = L.TQ, NT = kp.block, NW = NT / 32, R = kp.Ter, SB = kp.Tqr;
    const int NB = NC / 8;
    const int NBS = (NB + SB - 1) / SB;
    const bool smemA = kp.basis == FEMGPU_BASIS_SMEM;
    bool uses_inv = false;
    for (size_t id = 0; id < sig.nodes.size(); ++id)
        if (live[id] && sig.nodes[id].op == FEMGPU_OP_INV_JACOBIAN) uses_inv = true;

    o << "\nextern \"C\" __global__ void __launch_bounds__(" << NT << (kp.min_blocks > 1 ? ", " + S(kp.min_blocks) : "")
      << ") " << name << "(const __grid_constant__ Params P) {\n";
    o << "  extern __shared__ __align__(16) double sm[];\n";
    o << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5; (void)warp;\n";
    o << "  const size_t STR = (size_t)P.stride;\n";
    if (smemA) {
        o << "  double* const sA = sm + " << L.off_A << ";\n";
        o << "  for (int i = tid; i < " << (L.NQT * L.FPT * 16) << "; i += " << NT
          << ") reinterpret_cast<double2*>(sA)[i] = __ldg(reinterpret_cast<const double2*>(P.afr) + i);\n";
    }
    o << "  double* const sE = sm + " << L.off_E << ";\n";
    o << "  double* const sH = sm + " << L.off_H << "; (void)sH;\n";
    // E rows past Tw*TQ are K padding: zero once (never written afterwards)
    const long long erows = static_cast<long long>(sig.Tw) * TQ;
    if (L.KSq * 4 > erows)
        o << "  for (int i = tid; i < " << (L.KSq * 4 - erows) * L.LDU << "; i += " << NT << ") sE[" << erows * L.LDU
          << " + i] = 0.0;\n";
    o << "  __syncthreads();\n";
    o << "  const int n_tiles = (P.n_cells + " << NC - 1 << ") / " << NC << ";\n";
    o << "  #pragma unroll 1\n";
    o << "  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {\n";
    o << "    const int c0 = tile * " << NC << ";\n";
    // ---- gather: one index per (space, entry, cell); all component groups of the space
    std::vector<std::vector<int>> by_space_s(sig.ns()), by_space_v(sig.nv());
    for (size_t gi = 0; gi < L.groups.size(); ++gi)
        (L.groups[gi].vec ? by_space_v[L.groups[gi].space] : by_space_s[L.groups[gi].space]).push_back(static_cast<int>(gi));
    auto gather_space = [&](bool vec, int i, const std::vector<int>& gids) {
        const DmmaGroup& g0 = L.groups[gids[0]];
        const long long rows = static_cast<long long>(g0.KS) * 4;
        o << "    for (int e = tid; e < " << rows * NC << "; e += " << NT << ") {\n";
        o << "      const int k = e / " << NC << ", c = e % " << NC << ", cell = c0 + c;\n";
        o << "      const bool ok = k < " << g0.n << " && cell < P.n_cells;\n";
        o << "      const int idx = ok ? __ldg(&P." << (vec ? "vm" : "m") << i << "[k * STR + cell]) : 0;\n";
        for (int gid : gids) {
            const DmmaGroup& g = L.groups[gid];
            if (vec)
                o << "      sm[" << g.offU << " + k * " << L.LDU << " + c] = ok ? __ldg(&P.v" << i << "[(size_t)idx * "
                  << sig.dim << " + " << g.comp << "]) : 0.0;\n";
            else
                o << "      sm[" << g.offU << " + k * " << L.LDU << " + c] = ok ? __ldg(&P.x" << i << "[idx]) : 0.0;\n";
        }
        o << "    }\n";
    };
    for (int i = 0; i < sig.ns(); ++i) gather_space(false, i, by_space_s[i]);
    for (int i = 0; i < sig.nv(); ++i) gather_space(true, i, by_space_v[i]);
    // ---- geometry + cell-invariant map nodes
    if (sig.affine || !H.stored.empty()) {
        o << "    for (int c = tid; c < " << NC << "; c += " << NT << ") {\n";
        o << "      const int cell = c0 + c;\n";
        o << "      if (cell < P.n_cells) {\n";
        if (sig.affine) {
            std::ostringstream g;
            emit_geometry(g, sig, uses_inv, "cell");
            o << g.str();
            o << "        if (NF(det)) atomicMin(P.bad, (unsigned long long)cell);\n";
        }
        {
            std::ostringstream m;
            emit_map_nodes(m, sig, live, qdep, false, "0.0");
            o << m.str();
        }
        for (size_t h = 0; h < H.stored.size(); ++h)
            o << "        sH[" << h * L.LDS << " + c] = n" << H.stored[h] << ";\n";
        o << "      } else {\n";
        for (size_t h = 0; h < H.stored.size(); ++h) o << "        sH[" << h * L.LDS << " + c] = 0.0;\n";
        o << "      }\n";
        o << "    }\n";
    }
    o << "    __syncthreads();\n";
    // ---- quadrature-tile loop
    const int TPWq = static_cast<int>((static_cast<long long>((L.MBq + R - 1) / R) * NBS + NW - 1) / NW);
    o << "    double yacc[" << TPWq << "][" << R << "][" << SB << "][2];\n";
    o << "    #pragma unroll\n    for (int j = 0; j < " << TPWq << "; ++j)\n      #pragma unroll\n      for (int r = 0; r < " << R
      << "; ++r)\n        #pragma unroll\n        for (int s = 0; s < " << SB
      << "; ++s) { yacc[j][r][s][0] = 0.0; yacc[j][r][s][1] = 0.0; }\n";
    o << "    #pragma unroll 1\n";
    o << "    for (int qt = 0; qt < " << L.NQT << "; ++qt) {\n";
    o << "      const double* const Aq = " << (smemA ? "sA" : "P.afr") << " + (size_t)qt * " << L.FPT * 32 << " + lane;\n";
    // eval tasks
    long long ntask = 0;
    std::vector<long long> tstart;
    for (const auto& g : L.groups) {
        tstart.push_back(ntask);
        ntask += static_cast<long long>((g.MB + R - 1) / R) * NBS;
    }
    const std::string LDA = smemA ? "" : "__ldg";
    o << "      for (int t = warp; t < " << ntask << "; t += " << NW << ") {\n";
    for (size_t gi = 0; gi < L.groups.size(); ++gi) {
        const DmmaGroup& g = L.groups[gi];
        const long long t0 = tstart[gi], t1 = t0 + static_cast<long long>((g.MB + R - 1) / R) * NBS;
        o << "        " << (gi ? "else " : "") << "if (t < " << t1 << ") {\n";
        o << "          const int tl = t - " << t0 << ", mb0 = (tl / " << NBS << ") * " << R << ", nb0 = (tl % " << NBS
          << ") * " << SB << ";\n";
        o << "          double acc[" << R << "][" << SB << "][2] = {};\n";
        o << "          const double* Ab = Aq + (" << g.foff << " + mb0 * " << g.KS << ") * 32;\n";
        o << "          const double* Bb = sm + " << g.offU << " + (lane & 3) * " << L.LDU << " + nb0 * 8 + (lane >> 2);\n";
        o << "          #pragma unroll\n";
        o << "          for (int ks = 0; ks < " << g.KS << "; ++ks) {\n";
        o << "            double a[" << R << "], b[" << SB << "];\n";
        o << "            #pragma unroll\n            for (int r = 0; r < " << R << "; ++r) a[r] = (mb0 + r < " << g.MB
          << ") ? " << (smemA ? "Ab[(r * " + S(g.KS) + " + ks) * 32]" : "__ldg(&Ab[(r * " + S(g.KS) + " + ks) * 32])")
          << " : 0.0;\n";
        o << "            #pragma unroll\n            for (int s = 0; s < " << SB << "; ++s) b[s] = (nb0 + s < " << NB
          << ") ? Bb[ks * " << 4 * L.LDU << " + s * 8] : 0.0;\n";
        o << "            #pragma unroll\n            for (int r = 0; r < " << R
          << "; ++r)\n              #pragma unroll\n              for (int s = 0; s < " << SB
          << "; ++s) DMMA(acc[r][s], a[r], b[s]);\n";
        o << "          }\n";
        o << "          #pragma unroll\n          for (int r = 0; r < " << R << "; ++r)\n";
        o << "            if (mb0 + r < " << g.MB << ") {\n";
        o << "              #pragma unroll\n              for (int s = 0; s < " << SB << "; ++s)\n";
        o << "                if (nb0 + s < " << NB << ") *reinterpret_cast<double2*>(sm + " << g.offS << " + ((mb0 + r) * 8 + (lane >> 2)) * "
          << L.LDS << " + (nb0 + s) * 8 + 2 * (lane & 3)) = make_double2(acc[r][s][0], acc[r][s][1]);\n";
        o << "            }\n";
        o << "        }\n";
    }
    o << "      }\n";
    o << "      __syncthreads();\n";
    // map: one thread per (cell, quadrature point of the tile)
    o << "      for (int it = tid; it < " << NC * TQ << "; it += " << NT << ") {\n";
    o << "        const int c = it % " << NC << ", ql = it / " << NC << ", q = qt * " << TQ << " + ql;\n";
    o << "        if (q < " << sig.Q << ") {\n";
    for (size_t h = 0; h < H.stored.size(); ++h)
        o << "          const double n" << H.stored[h] << " = sH[" << h * L.LDS << " + c];\n";
    for (int id : H.consts) {
        char buf[64];
        std::snprintf(buf, sizeof buf, "%a", sig.nodes[id].value);
        o << "          const double n" << id << " = (" << buf << ");\n";
    }
    std::string nfexpr = "false";
    for (const auto& g : L.groups)
        for (size_t tt = 0; tt < g.terms.size(); ++tt) {
            const std::string v = (g.vec ? "t" : "s") + S(g.space) + "_" + S(g.terms[tt]);
            o << "          const double " << v << " = sm[" << g.offS << " + (" << tt * TQ << " + ql) * " << L.LDS
              << " + c];\n";
            nfexpr += " | NF(" + v + ")";
        }
    {
        std::ostringstream m;
        emit_map_nodes(m, sig, live, qdep, true, "__ldg(&P.tabg[" + S(sig.w_off) + " + q])");
        o << m.str();
    }
    for (int k = 0; k < sig.Tw; ++k) {
        o << "          sE[(" << k * TQ << " + ql) * " << L.LDU << " + c] = n" << sig.outputs[k] << ";\n";
        nfexpr += " | NF(n" + S(sig.outputs[k]) + ")";
    }
    o << "          if ((" << nfexpr << ") && c0 + c < P.n_cells) atomicMin(P.bad, (unsigned long long)(c0 + c));\n";
    o << "        } else {\n";
    for (int k = 0; k < sig.Tw; ++k) o << "          sE[(" << k * TQ << " + ql) * " << L.LDU << " + c] = 0.0;\n";
    o << "        }\n";
    o << "      }\n";
    o << "      __syncthreads();\n";
    // quadrature GEMM: persistent accumulators (fixed task set per warp across q tiles)
    const long long ntq = static_cast<long long>((L.MBq + R - 1) / R) * NBS;
    o << "      #pragma unroll\n      for (int j = 0; j < " << TPWq << "; ++j) {\n";
    o << "        const int t = warp + j * " << NW << ";\n";
    o << "        if (t < " << ntq << ") {\n";
    o << "          const int mb0 = (t / " << NBS << ") * " << R << ", nb0 = (t % " << NBS << ") * " << SB << ";\n";
    o << "          const double* Ab = Aq + (" << L.foff_q << " + mb0 * " << L.KSq << ") * 32;\n";
    o << "          const double* Bb = sE + (lane & 3) * " << L.LDU << " + nb0 * 8 + (lane >> 2);\n";
    o << "          #pragma unroll 4\n";
    o << "          for (int ks = 0; ks < " << L.KSq << "; ++ks) {\n";
    o << "            double a[" << R << "], b[" << SB << "];\n";
    o << "            #pragma unroll\n            for (int r = 0; r < " << R << "; ++r) a[r] = (mb0 + r < " << L.MBq
      << ") ? " << (smemA ? "Ab[(r * " + S(L.KSq) + " + ks) * 32]" : "__ldg(&Ab[(r * " + S(L.KSq) + " + ks) * 32])")
      << " : 0.0;\n";
    o << "            #pragma unroll\n            for (int s = 0; s < " << SB << "; ++s) b[s] = (nb0 + s < " << NB
      << ") ? Bb[ks * " << 4 * L.LDU << " + s * 8] : 0.0;\n";
    o << "            #pragma unroll\n            for (int r = 0; r < " << R
      << "; ++r)\n              #pragma unroll\n              for (int s = 0; s < " << SB
      << "; ++s) DMMA(yacc[j][r][s], a[r], b[s]);\n";
    o << "          }\n";
    o << "        }\n";
    o << "      }\n";
    o << "    }\n";  // q tiles
    // scatter from the accumulator fragments
    o << "    #pragma unroll\n    for (int j = 0; j < " << TPWq << "; ++j) {\n";
    o << "      const int t = warp + j * " << NW << ";\n";
    o << "      if (t < " << ntq << ") {\n";
    o << "        const int mb0 = (t / " << NBS << ") * " << R << ", nb0 = (t % " << NBS << ") * " << SB << ";\n";
    o << "        bool nf = false;\n";
    o << "        int badc = 0x7fffffff;\n";
    o << "        #pragma unroll\n        for (int r = 0; r < " << R << "; ++r) {\n";
    o << "          const int jw = (mb0 + r) * 8 + (lane >> 2);\n";
    o << "          if (jw < " << sig.nW << ") {\n";
    o << "            #pragma unroll\n            for (int s = 0; s < " << SB << "; ++s)\n";
    o << "              #pragma unroll\n              for (int i = 0; i < 2; ++i) {\n";
    o << "                const int cell = c0 + (nb0 + s) * 8 + 2 * (lane & 3) + i;\n";
    o << "                if (nb0 + s < " << NB << " && cell < P.n_cells) {\n";
    o << "                  const double v = yacc[j][r][s][i];\n";
    o << "                  if (NF(v)) { nf = true; badc = min(badc, cell); }\n";
    o << "                  atomicAdd(&P.y[__ldg(&P.tm[(size_t)jw * STR + cell])], v);\n";
    o << "                }\n";
    o << "              }\n";
    o << "          }\n";
    o << "        }\n";
    o << "        if (nf) atomicMin(P.bad, (unsigned long long)badc);\n";
    o << "      }\n";
    o << "    }\n";
    o << "  }\n";  // tiles
    o << "}\n";
}

}  // namespace femgpu

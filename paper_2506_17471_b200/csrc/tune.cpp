// tune.cpp — the automatic schedule (s == NULL at the C-ABI): the paper's "cost model prunes
// the schedule space to a few candidates that are timed empirically per form", on B200.
//
// The reference ranks TilingParams candidates with an analytic bytes/bandwidth model
// (perf_model.hpp:146-294, search.hpp:211-251, b = 9 + SCPT) and `tune` runs them through a
// measuring Executor (search.hpp:338-416).  Here the candidate space is the B200 kernel
// families: the DFMA families (macro-elements or SCPT, one thread per cell) and the warp-level
// DMMA family with its knobs (joint m-blocks, gather prefetch, CTA size).  The model counts FP64
// pipe slots per cell for each family (DFMA: usable FMAs + map + geometry at ~50 % pipe
// efficiency; DMMA: padded m8n8k4 slots at ~55 %, measured round 1), keeps every family within
// 1.6x of the best prediction, and each kept candidate is timed with CUDA events on the
// instance stream ([zero y + action], 2 warm-up + 5 timed).  The winner is cached in the
// instance.  Small instances (< kTuneMinCells) skip the timing and use the DFMA default.
#include <algorithm>
#include <chrono>
#include <array>
#include <atomic>
#include <cstdlib>
#include <numeric>
#include <thread>
#include <cstring>
#include <fstream>
#include <sstream>
#include <sys/stat.h>
#include <unistd.h>
#include <cstdio>

#include "femgpu_internal.hpp"

namespace femgpu {

namespace {

constexpr long long kTuneMinCells = 200000;

femgpu_schedule dfma_default() {
    femgpu_schedule s{};
    s.kind = FEMGPU_SCPT;
    return s;
}

femgpu_schedule dmma_variant(int joint, int prefetch, int block, int cells) {
    femgpu_schedule s{};
    s.kind = FEMGPU_DMMA;
    s.eval_row_tile = joint;
    s.quad_row_tile = prefetch;
    s.block_cells = block;
    s.cells_per_group = cells;
    return s;
}

// FP64 instructions of the map DAG per cell: (q-dependent, cell-invariant) live ADD/MUL nodes,
// an ADD fed by a single-use MUL of the same level counted once (contracted to a DFMA).
std::pair<long long, long long> map_instr(const Signature& sig) {
    const std::vector<char> live = map_live(sig), qdep = map_qdep(sig);
    std::vector<int> uses(sig.nodes.size(), 0);
    for (size_t i = 0; i < sig.nodes.size(); ++i) {
        const MapNode& n = sig.nodes[i];
        if (live[i] && (n.op == FEMGPU_OP_ADD || n.op == FEMGPU_OP_MUL)) {
            ++uses[n.a];
            ++uses[n.b];
        }
    }
    long long nq = 0, nc = 0;
    for (size_t i = 0; i < sig.nodes.size(); ++i) {
        const MapNode& n = sig.nodes[i];
        if (!live[i] || (n.op != FEMGPU_OP_ADD && n.op != FEMGPU_OP_MUL)) continue;
        int w = 1;
        if (n.op == FEMGPU_OP_ADD)
            for (int c : {n.a, n.b})
                if (sig.nodes[c].op == FEMGPU_OP_MUL && uses[c] == 1 && qdep[c] == qdep[i]) w = 0;
        (qdep[i] ? nq : nc) += w;
    }
    return {nq, nc};
}

// Persisted decisions: the timing pass runs once per (form, map, cell count, device) and the winner is
// written next to the JIT cache, so a later process on the same box (e.g. a profiler run, whose timings
// would be distorted by the instrumentation) replays the same kernel.  FEMGPU_TUNE_CACHE=0 disables.
std::string tune_key(const Instance& I) {
    const Signature& sig = I.sig;
    std::ostringstream k;
    k << "v18|" << sig.dim << "|" << sig.Q << "|" << sig.nW << "|" << sig.Tw << "|" << I.cells << "|" << I.output_size;
    for (size_t i = 0; i < sig.sdofs.size(); ++i) k << "|s" << sig.sdofs[i] << ":" << sig.sterms[i];
    for (size_t i = 0; i < sig.vdofs.size(); ++i) {
        k << "|v" << sig.vdofs[i] << ":" << sig.vterms[i];
        for (int c : sig.vcomps[i]) k << "," << c;
    }
    for (const auto& n : sig.nodes) k << "|" << n.op << "," << n.a << "," << n.b << "," << n.value;
    for (int o : sig.outputs) k << "|o" << o;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceProp prop{};
    cudaGetDeviceProperties(&prop, dev);
    k << "|" << prop.name << "|" << sms;
    uint64_t h = 0xcbf29ce484222325ULL;
    for (unsigned char c : k.str()) h = (h ^ c) * 0x100000001b3ULL;
    char hex[32];
    std::snprintf(hex, sizeof hex, "%016llx", static_cast<unsigned long long>(h));
    return hex;
}

std::string tune_path(const Instance& I) {
    std::string dir;
    if (const char* e = std::getenv("FEMGPU_CACHE")) dir = e;
    else dir = std::string(std::getenv("HOME") ? std::getenv("HOME") : "/tmp") + "/.cache/femgpu";
    ::mkdir(dir.c_str(), 0755);
    return dir + "/tune_" + tune_key(I) + ".txt";
}

bool tune_cache_enabled() {
    const char* e = std::getenv("FEMGPU_TUNE_CACHE");
    return !(e && std::strcmp(e, "0") == 0);
}

}  // namespace

std::string describe_plan(const KernelPlan& kp) {
    std::ostringstream s;
    switch (kp.family) {
        case Family::Macro:
            s << "femgpu_macro G=" << kp.G << " block=" << kp.block << (kp.qmajor ? " q-major" : "")
              << (kp.qmajor && !(kp.qmopt & 16) ? " unrolled" : "") << ((kp.qmopt & 16384) ? " 2q/trip" : "")
              << (std::any_of(kp.maff.begin(), kp.maff.end(), [](const std::vector<int>& a) { return !a.empty(); }) ? " affine-idx" : "")
              << (kp.msplit > 1 ? " split=" + std::to_string(kp.msplit) : std::string())
              << (!kp.merge.empty() ? " warp-merge=" + std::to_string(kp.merge.size()) : std::string()) << (kp.ysmem ? " y-smem" : "");
            break;
        case Family::Scpt:
            s << "femgpu_scpt cells/thread=" << std::max(1, kp.G) << " block=" << kp.block << " minCTAs=" << kp.min_blocks
              << (kp.qloop ? " q-loop" : "");
            break;
        case Family::Tile: s << "femgpu_tile cells=" << kp.tile_cells; break;
        case Family::Mlt: s << "femgpu_mlt Nc=" << kp.Nc << " Nwi=" << kp.Nwi << " TQ=" << kp.TQ; break;
        case Family::Dmma:
            s << "femgpu_dmma cells/task=" << kp.Nc << " TQ=" << kp.TQ << ((kp.qmopt & 16384) ? " 2ch/trip" : "")
              << " joint=" << kp.Ter << " prefetch=" << kp.Tqr
              << " block=" << kp.block << " basis=" << (kp.basis == FEMGPU_BASIS_SMEM ? "smem" : "l1");
            break;
    }
    if (kp.zfused) s << " +fused-zero" << (kp.zslabs > 0 ? "/" + std::to_string(kp.zslabs) : std::string());
    if (kp.pipe_memset) s << " +pipe-memset";
    return s.str();
}

namespace {

// One point of the schedule space with its model terms (tune log / FEMGPU_TUNE_LOG).
struct Cand {
    femgpu_schedule s{};
    KernelPlan kp;
    std::string label;
    int family = 0;             // 0 macro, 1 scpt, 2 dmma
    double slots = 0;           // FP64 lane-slots per cell (DMMA: padded m8n8k4 slots)
    double t_pipe = 0;          // seconds: FP64 pipe at the family's sustained efficiency
    double pred = 0;            // seconds: the model after the JIT (occupancy, spills)
    double meas = -1;           // seconds: measured (timed candidates only)
    int regs = 0, warps = 0;    // registers per thread, resident warps per SM
    long long spill = 0;        // local bytes per thread
    bool compiled = false, timed = false;
    std::string reject;
};

femgpu_schedule macro_variant(int G, int block, int variant, int reg_target, int min_blocks) {
    femgpu_schedule s = dfma_default();
    s.scatter = FEMGPU_SCATTER_MACRO;
    s.group_cells = G;
    s.block_cells = block;
    s.reserved[1] = reg_target;
    s.reserved[2] = min_blocks;
    s.reserved[3] = variant;
    return s;
}

femgpu_schedule scpt_variant(int G, int block, int min_blocks, bool qloop) {
    femgpu_schedule s = dfma_default();
    s.scatter = FEMGPU_SCATTER_ATOMIC;
    s.group_cells = G;
    s.block_cells = block;
    s.reserved[2] = min_blocks;
    s.reserved[3] = qloop ? 4 : 0;
    return s;
}

// Sustained fraction of the FP64 pipe each family reaches, fitted on every candidate of every
// benchmark configuration timed exhaustively (FEMGPU_TUNE_ALL=1, profiles/r02_tuner_calibration.jsonl):
// macro 0.64-0.70, SCPT 0.45-0.63 (scalar forms), DMMA 0.56-0.68 of its padded slots; the HBM side
// reaches ~0.65 of the peak on gather/scatter traffic.  Resident warps hide the gather latency:
// each warp per SM fewer than the 32 of full occupancy costs ~ kLatency / warps (fitted: 8 warps
// +15 %, 16 warps +7.5 %); local-memory spills cost ~ (spill / kSpillBytes)^2: up to ~800 B/thread they
// stay in L1 and cost 0-10 % (C5-hyp-P1 q-major macro: 544 B, 11 % faster than the best non-spilling
// kernel), 1.4-2.8 KB cost 10-40 %, 8.5 KB 10x (profiles/r02_tuner_calibration.jsonl)
constexpr double kEffMacro = 0.68, kEffScpt = 0.55, kEffDmma = 0.62, kEffHbm = 0.65;
constexpr double kLatency = 1.2, kSpillBytes = 4096.0;
// DMMA B-fragment share of the L1 data pipe at one m-block per fragment load (C4: joint 1/2 at
// 2034/1919 us without prefetch, joint 2/4 at 1869/1831 us with it; C5-adv-P1 joint 1/2 at 5010/4642 us)
constexpr double kBfrag = 0.15;

}  // namespace

void autotune(Instance& I) {
    I.auto_ready = true;
    I.auto_sched = dfma_default();
    I.auto_log.clear();
    const char* env = std::getenv("FEMGPU_AUTOTUNE");
    if ((env && std::strcmp(env, "0") == 0) || I.cells < kTuneMinCells) {
        I.auto_log = "default (no timing: " + std::string(I.cells < kTuneMinCells ? "small instance" : "FEMGPU_AUTOTUNE=0") + ")";
        return;
    }
    if (tune_cache_enabled()) {
        std::ifstream in(tune_path(I));
        if (in) {
            try {
                I.auto_sched = load_schedule(in);
                I.auto_log = "cached decision (" + tune_path(I) + ")";
                resolve_schedule(I, &I.auto_sched);  // still feasible here
                return;
            } catch (const Error&) {
                I.auto_sched = dfma_default();
            }
        }
    }
    const Signature& sig = I.sig;
    using Clock = std::chrono::steady_clock;
    const Clock::time_point t_start = Clock::now();
    Clock::time_point t_jit0, t_jit1, t_meas1;
    int dev = 0, sms = 148, clk_khz = 1965000;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const double clk = clk_khz * 1e3, lanes = 64.0 * sms;  // FP64 lanes per SM per clock
    // ---- FP64 lane-slots per cell (the paper's "Ops" count on this hardware)
    const double usable_fma = static_cast<double>(sig.useful_flops()) / 2.0;
    const std::pair<long long, long long> mi = map_instr(sig);
    const long long map_q = mi.first, map_c = mi.second;
    const double geo_slots = sig.affine ? 6.0 * sig.dim * sig.dim : 0.0;
    const double dfma_slots = usable_fma + static_cast<double>(map_q) * sig.Q + static_cast<double>(map_c) + geo_slots;
    // HBM floor: every input, coordinate, output and distinct index array once (SURVEY 8d bytes_alg)
    double alg_bytes = 8.0 * I.output_size;
    for (const auto& sp : I.sspaces) alg_bytes += 8.0 * sp.global;
    for (const auto& sp : I.vspaces) alg_bytes += 8.0 * sp.global * sig.dim;
    alg_bytes += 8.0 * I.coord_global * sig.dim;
    for (const auto& m : I.group_maps) alg_bytes += 4.0 * static_cast<double>(m.size());
    int mem_khz = 0, bus_bits = 0;
    cudaDeviceGetAttribute(&mem_khz, cudaDevAttrMemoryClockRate, dev);
    cudaDeviceGetAttribute(&bus_bits, cudaDevAttrGlobalMemoryBusWidth, dev);
    const double hbm = mem_khz > 0 && bus_bits > 0 ? 2.0 * mem_khz * 1e3 * bus_bits / 8.0 : 8e12;
    const double t_hbm = alg_bytes / (hbm * kEffHbm);
    // ---- enumerate the schedule space
    std::vector<Cand> C;
    auto add = [&](const femgpu_schedule& sc, int family) {
        Cand c;
        c.s = sc;
        c.family = family;
        try {
            c.kp = resolve_schedule(I, &c.s);
        } catch (const Error& e) {
            if (e.code != FEMGPU_E_INFEASIBLE && e.code != FEMGPU_E_INVALID) throw;
            return;
        }
        c.label = describe_plan(c.kp);
        for (const auto& o : C)
            if (o.label == c.label) return;
        if (family == 2) {
            const DmmaLayout L = dmma_layout(sig, c.kp);
            // padded m8n8k4 slots at the DMMA rate (measured 37.1 vs 34.2 TF DFMA: x1.085 per slot);
            // the map runs per padded quadrature point, the cell-invariant part once per cell
            // (quad fragments whose Psi block is all zero are skipped by the kernel: fused problems)
            long long zero_frags = 0;
            for (int k = 0; k < sig.Tw; ++k)
                for (int nb = 0; nb < L.NBQ; ++nb) {
                    bool zero = true;
                    for (int jw = nb * 8; jw < std::min(sig.nW, nb * 8 + 8) && zero; ++jw) zero = !sig.pnz(k, jw);
                    zero_frags += zero ? static_cast<long long>(L.TQL) * L.NCH : 0;
                }
            c.slots = static_cast<double>(L.nfrag - zero_frags) * 256.0 / 8.0 / 1.085 +
                      static_cast<double>(map_q) * (4.0 * L.TQL * L.NCH) + static_cast<double>(map_c) + geo_slots;
        } else {
            c.slots = dfma_slots;
        }
        const double eff = family == 0 ? kEffMacro : family == 1 ? kEffScpt : kEffDmma;
        c.t_pipe = std::max(static_cast<double>(I.cells) * c.slots / (lanes * clk) / eff, t_hbm);
        C.push_back(c);
    };
    add(dfma_default(), 1);  // the paper's SCPT baseline, always timed (b + SCPT)
    for (int G : {6, 4, 3, 2}) {  // the largest group size whose common pattern fits the register budget
        if (!I.macro_layout(G).ok) continue;
        const size_t before = C.size();
        // q-major, rolled quadrature loop; in pipelined actions the next output is zeroed by the
        // launch's threads after their gathers (qmopt 8192: C2 192 vs 206 us with a CTA prologue)
        add(macro_variant(G, 32, 3 | (8208 << 16), 232, 0), 0);
        add(macro_variant(G, 32, 3 | (24592 << 16), 232, 0), 0);  // two quadrature points per trip (C2 182 vs 192 us)
        // the group's cells split over 2 or 3 warps (fewer registers per thread for wide forms:
        // C5-adv-P2 854 vs 1001 us of SCPT; profiles/r02_sweeps.md)
        if (G % 2 == 0) add(macro_variant(G, 64, 3 | (2 << 8) | (16 << 16), 200, 0), 0);
        if (G % 3 == 0) add(macro_variant(G, 96, 3 | (3 << 8) | (16 << 16), 168, 0), 0);
        add(macro_variant(G, 64, 3 | (8208 << 16), 232, 0), 0);
        add(macro_variant(G, 32, 0, 0, 8), 0);                  // cell-major, uncapped
        add(macro_variant(G, 64, 0, 0, 0), 0);                  // cell-major, 168-register cap
        if (C.size() > before) break;
    }
    for (const auto& v : std::vector<std::array<int, 4>>{{1, 256, 3, 0}, {1, 128, 5, 0}, {1, 64, 0, 0}, {2, 128, 0, 0},
                                                         {2, 128, 0, 1}, {2, 64, 0, 1}, {3, 64, 0, 1}, {3, 128, 0, 1}})
        add(scpt_variant(v[0], v[1], v[2], v[3] != 0), 1);
    {
        std::vector<int> tqs = {0};
        long long bestf = -1;
        int bestq = 0;
        for (int tq = 4; tq <= (sig.Q + 3) / 4 * 4; tq += 4) {
            KernelPlan kp;
            femgpu_schedule s = dmma_variant(1, 0, 0, 0);
            s.quad_tile = tq;
            try {
                resolve_dmma(sig, kp, &s);
            } catch (const Error&) {
                continue;
            }
            const long long f = dmma_layout(sig, kp).nfrag;
            if (bestf < 0 || f < bestf) bestf = f, bestq = tq;
        }
        tqs.push_back(bestq);
        if (sig.Q > 8) tqs.push_back(8);
        for (int tq : tqs)
            for (int joint : {1, 2, 4})
                for (int pf : {0, 1})
                    for (int block : {128, 256}) {
                        if (joint == 4 && block == 256) continue;  // (4 joint m-blocks: register-heavy)
                        femgpu_schedule s = dmma_variant(joint, pf, block, 32);
                        s.quad_tile = tq;
                        add(s, 2);
                        if (joint == 1 && block == 128) {
                            KernelPlan kt;
                            try {
                                resolve_dmma(sig, kt, &s);
                            } catch (const Error&) {
                                continue;
                            }
                            if (dmma_layout(sig, kt).NCH > 1) {
                                s.reserved[3] = 0x4000 << 16;  // two quadrature chunks per trip (hyp-P4 2815 vs 2895 us)
                                add(s, 2);
                            }
                        }
                    }
    }
    // ---- static pruning: the best kCompile by FP64-pipe time (each family keeps its best two)
    const char* all_env = std::getenv("FEMGPU_TUNE_ALL");  // calibration runs: compile and time everything
    const bool tune_all = all_env && std::strcmp(all_env, "0") != 0;
    constexpr size_t kCompile = 16, kTimed = 9;
    std::vector<size_t> order(C.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return C[a].t_pipe < C[b].t_pipe; });
    std::vector<size_t> sel = {0};  // SCPT baseline
    int per_family[3] = {0, 0, 0};
    for (size_t i : order)
        if (i != 0 && per_family[C[i].family] < 2) {
            sel.push_back(i);
            ++per_family[C[i].family];
        }
    for (size_t i : order)
        if ((tune_all || sel.size() < kCompile) && std::find(sel.begin(), sel.end(), i) == sel.end()) sel.push_back(i);
    // ---- JIT the survivors in parallel (NVRTC is thread-safe; modules land in the global cache)
    t_jit0 = Clock::now();
    {
        std::vector<std::thread> pool;
        std::atomic<size_t> next{0};
        const unsigned nthr = std::max(1u, std::min<unsigned>(16, std::thread::hardware_concurrency()));
        for (unsigned t = 0; t < nthr; ++t)
            pool.emplace_back([&] {
                cudaSetDevice(dev);
                for (size_t k; (k = next.fetch_add(1)) < sel.size();) {
                    try {
                        get_module(sig, C[sel[k]].kp);
                    } catch (const Error&) {
                    }
                }
            });
        for (auto& t : pool) t.join();
    }
    // ---- model with the compiled kernels' attributes: resident warps against the gather
    // latency, spills (relative: candidates spilling much more than the least-spilling one are out)
    long long min_spill = -1;
    for (size_t i : sel) {
        Cand& c = C[i];
        std::shared_ptr<Module> m;
        try {
            m = I.module_for(c.kp);
        } catch (const Error& e) {
            c.reject = std::string("jit: ") + e.what();
            continue;
        }
        c.compiled = true;
        c.regs = m->regs;
        c.spill = m->local_bytes;
        c.warps = m->occupancy * (c.kp.block / 32);
        if (min_spill < 0 || c.spill < min_spill) min_spill = c.spill;
    }
    for (size_t i : sel) {
        Cand& c = C[i];
        if (!c.compiled) continue;
        // DMMA gather prefetch (values one m-group ahead) hides latency like ~1.5x the resident warps
        // (C3b 234.7 vs 242.0 us, C5-adv-P3 826.8 vs 845.4, C5-hyp-P1 2874 vs 2959 at 2/3 the warps)
        const double w = std::max(1, c.warps) * (c.family == 2 && c.kp.Tqr ? 1.5 : 1.0);
        // (SCPT spills sit inside the unrolled point loop: 240-650 B/thread cost it 2-5x)
        const double sp = static_cast<double>(c.spill) / (c.family == 1 ? kSpillBytes / 8.0 : kSpillBytes);
        c.pred = c.t_pipe * (1.0 + kLatency / w) * (1.0 + sp * sp);
        // DMMA: every B-fragment load (shared memory, one per DMMA) feeds `joint` m-blocks; the loads
        // compete with the gathers and the scatter for the L1 data pipe (kEffDmma is fitted at joint 2)
        if (c.family == 2) c.pred *= (1.0 + kBfrag / std::max(1, c.kp.Ter)) / (1.0 + kBfrag / 2.0);
        if (c.spill > 2 * min_spill + 768) c.reject = "spills " + std::to_string(c.spill) + " B/thread";
        else if (c.warps < 4) c.reject = "occupancy " + std::to_string(c.warps) + " warps/SM";
    }
    std::vector<size_t> ranked;
    for (size_t i : sel)
        if (C[i].compiled && C[i].reject.empty()) ranked.push_back(i);
    if (ranked.empty())  // everything spills: keep the compiled ones, the model still orders them
        for (size_t i : sel)
            if (C[i].compiled) ranked.push_back(i);
    std::stable_sort(ranked.begin(), ranked.end(), [&](size_t a, size_t b) { return C[a].pred < C[b].pred; });
    // ---- measure: >= 5 runs and ~10 ms of work each, then the three fastest re-timed interleaved
    t_jit1 = Clock::now();
    auto time_it = [&](const KernelPlan& kp, int reps) {
        FG_CUDA(cudaEventRecord(I.ev0, I.stream));
        for (int i = 0; i < reps; ++i) run_action(I, kp, I.d_y, I.stream);
        FG_CUDA(cudaEventRecord(I.ev1, I.stream));
        FG_CUDA(cudaEventSynchronize(I.ev1));
        float ms = 0.f;
        FG_CUDA(cudaEventElapsedTime(&ms, I.ev0, I.ev1));
        return ms * 1e-3 / reps;
    };
    std::vector<int> reps_of(C.size(), 5);
    std::vector<std::pair<double, size_t>> first;
    std::vector<size_t> timed;
    auto measure = [&](size_t i) {
        Cand& c = C[i];
        timed.push_back(i);
        try {
            for (int k = 0; k < 2; ++k) run_action(I, c.kp, I.d_y, I.stream);
            const double t1 = time_it(c.kp, 1);
            reps_of[i] = std::max(5, std::min(200, static_cast<int>(0.01 / std::max(t1, 1e-6))));
            c.meas = time_it(c.kp, reps_of[i]);
            c.timed = true;
            first.push_back({c.meas, i});
        } catch (const Error& e) {
            if (e.code != FEMGPU_E_INFEASIBLE && e.code != FEMGPU_E_JIT) throw;
            c.reject = std::string("launch: ") + e.what();
        }
    };
    // clocks up before the first timed candidate (~40 ms of the best prediction's work): a GPU coming
    // out of idle timed C5-adv-P4's first candidate 19 % slow
    for (size_t i : ranked) {
        try {
            run_action(I, C[i].kp, I.d_y, I.stream);
            const double t1 = time_it(C[i].kp, 1);
            time_it(C[i].kp, std::max(1, std::min(400, static_cast<int>(0.04 / std::max(t1, 1e-6)))));
        } catch (const Error& e) {
            if (e.code != FEMGPU_E_INFEASIBLE && e.code != FEMGPU_E_JIT) throw;
            continue;
        }
        break;
    }
    // stage 1: the best prediction of every kernel class (the model's cross-class efficiencies are
    // its least certain term; within a class its ranking holds better).  Classes: macro q-major
    // (one warp per group), macro split/cell-major, SCPT, DMMA -- the split and cell-major macro
    // kernels measured 1.2-1.9x their prediction on the heavy forms, q-major 0.6-0.95x
    auto cls = [&](size_t i) {
        const Cand& c = C[i];
        return c.family == 0 && !(c.kp.qmajor && c.kp.msplit == 1) ? 3 : c.family;
    };
    for (int k = 0; k < 4; ++k)
        for (size_t i : ranked)
            if (cls(i) == k) {
                measure(i);
                break;
            }
    // stage 2: the remaining slots (b = 9) in prediction order within the classes as measured in
    // stage 1: two thirds to the fastest class, the rest to a runner-up within 25 % (C3b: macro candidates
    // predicted ahead of the DMMA ones measured 1.3-1.9x slower and took the slots of the winner)
    {
        std::vector<std::pair<double, int>> fam_t;
        for (auto& f : first) fam_t.push_back({f.first, cls(f.second)});
        std::sort(fam_t.begin(), fam_t.end());
        const size_t left = kTimed > timed.size() ? kTimed - timed.size() : 0;
        std::vector<size_t> quota(4, 0);
        // (a runner-up measured more than 25 % behind gets nothing: the slots go to the fastest class)
        const bool close = fam_t.size() > 1 && fam_t[1].first <= 1.25 * fam_t[0].first;
        if (!fam_t.empty()) quota[fam_t[0].second] = close ? (2 * left + 2) / 3 : left;
        if (close) quota[fam_t[1].second] = left - quota[fam_t[0].second];
        std::vector<size_t> extra;
        for (size_t k = 0; k < fam_t.size() && k < 2; ++k)
            for (size_t i : ranked) {
                if (quota[fam_t[k].second] == 0) break;
                if (cls(i) == fam_t[k].second && std::find(timed.begin(), timed.end(), i) == timed.end() &&
                    std::find(extra.begin(), extra.end(), i) == extra.end()) {
                    extra.push_back(i);
                    --quota[fam_t[k].second];
                }
            }
        // unused quota (a family ran out of candidates): the best remaining predictions overall
        for (size_t i : ranked)
            if ((tune_all || timed.size() + extra.size() < kTimed) && std::find(timed.begin(), timed.end(), i) == timed.end() &&
                std::find(extra.begin(), extra.end(), i) == extra.end())
                extra.push_back(i);
        for (size_t i : extra) measure(i);
    }
    if (std::find(timed.begin(), timed.end(), size_t(0)) == timed.end() && C[0].compiled) measure(0);  // + SCPT
    std::sort(first.begin(), first.end());
    const size_t top = std::min<size_t>(3, first.size());
    std::vector<double> retime(top, 1e300);
    for (int round = 0; round < 2 && top > 1; ++round)
        for (size_t k = 0; k < top; ++k) {
            const size_t j = round % 2 ? top - 1 - k : k;
            retime[j] = std::min(retime[j], time_it(C[first[j].second].kp, reps_of[first[j].second]));
        }
    size_t win = 0;
    for (size_t k = 1; k < top; ++k)
        if (retime[k] < retime[win]) win = k;
    t_meas1 = Clock::now();
    auto secs = [](Clock::time_point a, Clock::time_point b) { return std::chrono::duration<double>(b - a).count(); };
    std::ostringstream log;
    auto us = [](double t) { return static_cast<long long>(t * 1e7) / 10.0; };
    log << "model: " << C.size() << " candidates, " << sel.size() << " compiled, " << first.size()
        << " timed (FP64 slots/cell: dfma " << static_cast<long long>(dfma_slots) << "; HBM floor "
        << us(t_hbm) << " us)";
    for (size_t i : timed)
        if (C[i].timed)
            log << " [" << C[i].label << ": pred " << us(C[i].pred) << " us, meas " << us(C[i].meas) << " us, "
                << C[i].regs << " regs, " << C[i].warps << " warps/SM]";
    for (size_t i : sel)
        if (!C[i].reject.empty()) log << " [rejected " << C[i].label << ": " << C[i].reject << "]";
    if (!first.empty()) {
        I.auto_sched = C[first[win].second].s;
        log << "; re-timed top " << top << ", winner " << C[first[win].second].label;
        // a macro winner on an affine index pattern: its twin that loads every index instead
        // (the offset form changes register allocation; C5-hyp-P1 measured it 1.6 % slower)
        const KernelPlan& wk = C[first[win].second].kp;
        const bool aff = wk.family == Family::Macro &&
                         std::any_of(wk.maff.begin(), wk.maff.end(), [](const std::vector<int>& a) { return !a.empty(); });
        if (aff) {
            femgpu_schedule tw = I.auto_sched;
            tw.reserved[0] |= FEMGPU_FLAG_INDEX_LOADS;
            try {
                const KernelPlan kt = resolve_schedule(I, &tw);
                run_action(I, kt, I.d_y, I.stream);  // JIT + module load outside the timing
                const int reps = reps_of[first[win].second];
                double ta = 1e300, tl = 1e300;
                for (int round = 0; round < 2; ++round) {
                    ta = std::min(ta, time_it(wk, reps));
                    tl = std::min(tl, time_it(kt, reps));
                }
                log << "; affine index offsets " << us(ta) << " us vs index loads " << us(tl) << " us";
                if (tl < ta) I.auto_sched = tw;
            } catch (const Error& e) {
                if (e.code != FEMGPU_E_INFEASIBLE && e.code != FEMGPU_E_JIT) throw;
            }
        }
    }
    // ---- rank agreement of the model with the measurements (Spearman over the timed candidates)
    double rho = 0.0;
    if (first.size() > 2) {
        std::vector<size_t> tp;
        for (auto& f : first) tp.push_back(f.second);
        std::vector<size_t> by_pred = tp;
        std::stable_sort(by_pred.begin(), by_pred.end(), [&](size_t a, size_t b) { return C[a].pred < C[b].pred; });
        double d2 = 0.0;
        for (size_t r = 0; r < tp.size(); ++r) {
            const size_t pr = static_cast<size_t>(std::find(by_pred.begin(), by_pred.end(), tp[r]) - by_pred.begin());
            d2 += static_cast<double>((pr - r) * (pr - r));
        }
        const double n = static_cast<double>(tp.size());
        rho = 1.0 - 6.0 * d2 / (n * (n * n - 1.0));
        log << "; model rank agreement (Spearman) " << static_cast<long long>(rho * 1000) / 1000.0;
    }
    // pipelined actions (femgpu_action_device_pipelined, the bench step): zero the next output
    // inside the action kernel, or with a memset after it, whichever the winner runs faster with
    if (!first.empty() && supports_cell_range(resolve_schedule(I, &I.auto_sched))) {
        double* yb[2] = {I.d_y, I.second_output()};
        femgpu_schedule sm = I.auto_sched;
        sm.reserved[0] |= FEMGPU_FLAG_PIPE_MEMSET;
        const KernelPlan kf = resolve_schedule(I, &I.auto_sched), km = resolve_schedule(I, &sm);
        auto time_piped = [&](const KernelPlan& kp, int reps) {
            FG_CUDA(cudaMemsetAsync(yb[0], 0, sizeof(double) * static_cast<size_t>(I.output_size), I.stream));
            run_action_pipelined(I, kp, yb[0], yb[1], I.stream);
            FG_CUDA(cudaEventRecord(I.ev0, I.stream));
            for (int i = 0; i < reps; ++i) run_action_pipelined(I, kp, yb[(i + 1) & 1], yb[i & 1], I.stream);
            FG_CUDA(cudaEventRecord(I.ev1, I.stream));
            FG_CUDA(cudaEventSynchronize(I.ev1));
            float ms = 0.f;
            FG_CUDA(cudaEventElapsedTime(&ms, I.ev0, I.ev1));
            return ms * 1e-3 / reps;
        };
        const int reps = reps_of[first[win].second];
        double tf = 1e300, tm = 1e300;
        for (int round = 0; round < 2; ++round) {
            tf = std::min(tf, time_piped(kf, reps));
            tm = std::min(tm, time_piped(km, reps));
        }
        log << "; pipelined steps: in-kernel zeroing " << static_cast<long long>(tf * 1e7) / 10.0 << " us, memset "
            << static_cast<long long>(tm * 1e7) / 10.0 << " us";
        if (tm < tf) I.auto_sched.reserved[0] |= FEMGPU_FLAG_PIPE_MEMSET;
    }
    // a non-finite input must not leave a stale flag behind the tuning runs
    FG_CUDA(cudaMemsetAsync(I.d_bad, 0xff, 2 * sizeof(unsigned long long), I.stream));
    FG_CUDA(cudaStreamSynchronize(I.stream));
    I.auto_log = log.str();
    if (const char* path = std::getenv("FEMGPU_TUNE_LOG")) {  // predicted vs measured, one JSON line per instance
        std::ofstream js(path, std::ios::app);
        js << "{\"cells\": " << I.cells << ", \"dofs\": " << I.output_size << ", \"Q\": " << sig.Q
           << ", \"usable_flops\": " << sig.usable_flops() << ", \"spearman\": " << rho << ", \"winner\": \""
           << (first.empty() ? std::string() : C[first[win].second].label) << "\", \"model_s\": " << secs(t_start, t_jit0)
           << ", \"jit_s\": " << secs(t_jit0, t_jit1) << ", \"timing_s\": " << secs(t_jit1, t_meas1) << ", \"candidates\": [";
        bool comma = false;
        for (size_t i : sel) {
            const Cand& c = C[i];
            js << (comma ? ", " : "") << "{\"label\": \"" << c.label << "\", \"family\": " << c.family
               << ", \"slots\": " << c.slots << ", \"t_pipe_us\": " << c.t_pipe * 1e6 << ", \"pred_us\": " << c.pred * 1e6
               << ", \"meas_us\": " << (c.timed ? c.meas * 1e6 : -1.0) << ", \"regs\": " << c.regs
               << ", \"warps\": " << c.warps << ", \"spill\": " << c.spill << ", \"reject\": \"" << c.reject << "\"}";
            comma = true;
        }
        js << "]}\n";
    }
    if (tune_cache_enabled()) {
        const std::string path = tune_path(I), tmp = path + ".tmp" + std::to_string(static_cast<long long>(::getpid()));
        {
            std::ofstream out(tmp);
            if (out) save_schedule(out, &I.auto_sched, sig.ns(), sig.nv());
        }
        std::rename(tmp.c_str(), path.c_str());
    }
}

KernelPlan plan_for(Instance& I, const femgpu_schedule* s) {
    if (s) return resolve_schedule(I, s);
    if (!I.auto_ready) autotune(I);
    return resolve_schedule(I, &I.auto_sched);
}

}  // namespace femgpu

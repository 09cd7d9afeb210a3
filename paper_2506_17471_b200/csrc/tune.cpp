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
#include <cstdlib>
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

// FP64-pipe slots (FMA lanes) per cell of the map DAG evaluated at every quadrature point.
long long map_ops(const Signature& sig) {
    long long ops = 0;
    for (const auto& n : sig.nodes)
        if (n.op == FEMGPU_OP_ADD || n.op == FEMGPU_OP_MUL) ++ops;
    return ops;
}

// Persisted decisions: the timing pass runs once per (form, map, cell count, device) and the winner is
// written next to the JIT cache, so a later process on the same box (e.g. a profiler run, whose timings
// would be distorted by the instrumentation) replays the same kernel.  FEMGPU_TUNE_CACHE=0 disables.
std::string tune_key(const Instance& I) {
    const Signature& sig = I.sig;
    std::ostringstream k;
    k << "v4|" << sig.dim << "|" << sig.Q << "|" << sig.nW << "|" << sig.Tw << "|" << I.cells << "|" << I.output_size;
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
            s << "femgpu_macro G=" << kp.G << " block=" << kp.block << (kp.qmajor ? " q-major" : "") << (kp.msplit > 1 ? " split=" + std::to_string(kp.msplit) : std::string()) << (kp.ysmem ? " y-smem" : "");
            break;
        case Family::Scpt:
            s << "femgpu_scpt cells/thread=" << std::max(1, kp.G) << " block=" << kp.block << " minCTAs=" << kp.min_blocks
              << (kp.qloop ? " q-loop" : "");
            break;
        case Family::Tile: s << "femgpu_tile cells=" << kp.tile_cells; break;
        case Family::Mlt: s << "femgpu_mlt Nc=" << kp.Nc << " Nwi=" << kp.Nwi << " TQ=" << kp.TQ; break;
        case Family::Dmma:
            s << "femgpu_dmma cells/task=" << kp.Nc << " TQ=" << kp.TQ << " joint=" << kp.Ter << " prefetch=" << kp.Tqr
              << " block=" << kp.block << " basis=" << (kp.basis == FEMGPU_BASIS_SMEM ? "smem" : "l1");
            break;
    }
    if (kp.zfused) s << " +fused-zero" << (kp.zslabs > 0 ? "/" + std::to_string(kp.zslabs) : std::string());
    if (kp.pipe_memset) s << " +pipe-memset";
    return s.str();
}

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
    // ---- model: FP64-pipe lane-slots per cell
    const double usable_fma = static_cast<double>(sig.usable_flops()) / 2.0;
    const double map_slots = static_cast<double>(map_ops(sig)) * sig.Q;
    const double geo_slots = sig.affine ? 6.0 * sig.dim * sig.dim : 0.0;
    const double t_dfma = (usable_fma + map_slots + geo_slots) / 0.50;
    double t_dmma = 1e300;
    {
        KernelPlan kp;
        femgpu_schedule s = dmma_variant(1, 0, 0, 0);
        try {
            resolve_dmma(sig, kp, &s);
            const DmmaLayout L = dmma_layout(sig, kp);
            const double dmma_slots = static_cast<double>(L.nfrag) * 256.0 / 8.0;  // per cell
            t_dmma = dmma_slots / 0.55 + (map_slots * (4.0 * L.TQL * L.NCH) / sig.Q + geo_slots) / 0.5;
        } catch (const Error&) {
        }
    }
    const double best = std::min(t_dfma, t_dmma);
    std::vector<femgpu_schedule> cands;
    if (t_dfma <= 1.6 * best) {
        cands.push_back(dfma_default());
        {  // macro-elements with 32-thread CTAs (measured 2 % faster on C2 / C5-adv-P1)
            femgpu_schedule s = dfma_default();
            s.scatter = FEMGPU_SCATTER_MACRO;
            s.block_cells = 32;
            cands.push_back(s);
            s.reserved[2] = 8;  // uncapped (255 registers, 8 warps/SM): C5-adv-P1 1448 us vs 1703 us
            cands.push_back(s);
            s.reserved[2] = 0;
            // quadrature-point-major (one tabulation load for the group's cells) with the quadrature
            // loop rolled and the hoisted map nodes in registers (C2: 197 vs 224 us unrolled,
            // instruction-cache stalls; profiles/r02_c2_qmajor.md)
            s.reserved[3] = 3 | (16 << 16);
            s.reserved[1] = 232;
            cands.push_back(s);
        }
        for (int mb : {3, 5}) {  // SCPT with a register cap (more resident warps to hide the gathers)
            femgpu_schedule s = dfma_default();
            s.scatter = FEMGPU_SCATTER_ATOMIC;
            s.block_cells = mb == 3 ? 256 : 128;
            s.reserved[2] = mb;
            cands.push_back(s);
        }
        for (int G : {2}) {  // SCPT with G cells per thread (shared tabulation loads)
            femgpu_schedule s = dfma_default();
            s.scatter = FEMGPU_SCATTER_ATOMIC;
            s.group_cells = G;
            cands.push_back(s);
            s.reserved[3] = 4;  // quadrature loop kept rolled (measured 7 % faster on C3a)
            cands.push_back(s);
        }
        {  // 3 cells per thread, rolled quadrature loop, 64-thread CTAs (C3a: 181 us vs 205 us)
            femgpu_schedule s = dfma_default();
            s.scatter = FEMGPU_SCATTER_ATOMIC;
            s.group_cells = 3;
            s.block_cells = 64;
            s.reserved[3] = 4;
            cands.push_back(s);
        }
    }
    if (t_dmma <= 1.6 * best) {
        // quadrature chunk: the register-capped choice of resolve_dmma and, when different, the
        // uncapped one with the fewest padded DMMAs (more registers, fewer tensor-pipe slots)
        std::vector<int> tqs = {0};
        {
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
            KernelPlan kp;
            femgpu_schedule s = dmma_variant(1, 0, 0, 0);
            resolve_dmma(sig, kp, &s);
            if (bestq > 0 && bestq != kp.TQ) tqs.push_back(bestq);
            // two owned points per lane-group: measured best on several high-Q forms (hyp-P4)
            if (sig.Q > 8 && kp.TQ != 8 && bestq != 8) tqs.push_back(8);
        }
        for (int tq : tqs)
            for (int joint : {1, 2})
                for (int block : {128, 256}) {
                    cands.push_back(dmma_variant(joint, 0, block, 32));
                    cands.back().quad_tile = tq;
                }
        for (int tq : tqs)  // gather prefetch (C5-hyp-P2: T^Q=8 + prefetch 2191-2226 us vs 2310 us)
            for (int block : {128, 256}) {
                cands.push_back(dmma_variant(1, 1, block, 32));
                cands.back().quad_tile = tq;
            }
    }
    std::ostringstream log;
    log << "model slots/cell: dfma " << static_cast<long long>(t_dfma) << ", dmma "
        << (t_dmma < 1e299 ? std::to_string(static_cast<long long>(t_dmma)) : std::string("n/a")) << "; timed:";
    // first pass: every candidate, >= 5 runs and >= ~10 ms of work; second pass: the three fastest
    // re-timed in an interleaved order (clock/power-state drift between candidates cancels out)
    auto time_it = [&](const KernelPlan& kp, int reps) {
        FG_CUDA(cudaEventRecord(I.ev0, I.stream));
        for (int i = 0; i < reps; ++i) run_action(I, kp, I.d_y, I.stream);
        FG_CUDA(cudaEventRecord(I.ev1, I.stream));
        FG_CUDA(cudaEventSynchronize(I.ev1));
        float ms = 0.f;
        FG_CUDA(cudaEventElapsedTime(&ms, I.ev0, I.ev1));
        return ms * 1e-3 / reps;
    };
    std::vector<std::pair<double, size_t>> first;
    std::vector<KernelPlan> plans(cands.size());
    std::vector<int> reps_of(cands.size(), 5);
    for (size_t ci = 0; ci < cands.size(); ++ci) {
        try {
            plans[ci] = resolve_schedule(I, &cands[ci]);
            for (int i = 0; i < 2; ++i) run_action(I, plans[ci], I.d_y, I.stream);
            const double t1 = time_it(plans[ci], 1);
            reps_of[ci] = std::max(5, std::min(200, static_cast<int>(0.01 / std::max(t1, 1e-6))));
            const double t = time_it(plans[ci], reps_of[ci]);
            log << " [" << describe_plan(plans[ci]) << ": " << static_cast<long long>(t * 1e7) / 10.0 << " us]";
            first.push_back({t, ci});
        } catch (const Error& e) {
            if (e.code != FEMGPU_E_INFEASIBLE && e.code != FEMGPU_E_JIT) throw;
            log << " [infeasible: " << e.what() << "]";
        }
    }
    std::sort(first.begin(), first.end());
    const size_t top = std::min<size_t>(3, first.size());
    std::vector<double> retime(top, 1e300);
    for (int round = 0; round < 2 && top > 1; ++round)
        for (size_t i = 0; i < top; ++i) {
            const size_t ci = first[round % 2 ? top - 1 - i : i].second;
            const double t = time_it(plans[ci], reps_of[ci]);
            size_t slot = 0;
            for (size_t k = 0; k < top; ++k)
                if (first[k].second == ci) slot = k;
            retime[slot] = std::min(retime[slot], t);
        }
    if (!first.empty()) {
        size_t win = 0;
        if (top > 1)
            for (size_t k = 1; k < top; ++k)
                if (retime[k] < retime[win]) win = k;
        I.auto_sched = cands[first[win].second];
        log << "; re-timed top " << top << ", winner " << describe_plan(plans[first[win].second]);
        // fused y zeroing (pipeline.cpp): slabbed launches clear later slabs' rows instead of a
        // memset in front; kept only where it times faster (it wins on C5-hyp-P1 and C4,
        // loses where slab boundaries cost more than the memset)
        const char* zo = std::getenv("FEMGPU_ZERO_OVERLAP");
        if (!zo) {
            const KernelPlan& k0 = plans[first[win].second];
            const int reps = reps_of[first[win].second];
            std::vector<femgpu_schedule> fzs;
            std::vector<KernelPlan> kzs;
            for (int slabs : {4, 8}) {  // fewer slabs: larger front memset, fewer slab boundaries
                femgpu_schedule fz = I.auto_sched;
                fz.reserved[0] |= FEMGPU_FLAG_FUSED_ZERO | (slabs << 8);
                const KernelPlan kz = resolve_schedule(I, &fz);
                if (!kz.zfused) continue;
                for (int i = 0; i < 2; ++i) run_action(I, kz, I.d_y, I.stream);
                if (I.last_launches <= 1) continue;  // not applicable here (size, locality)
                fzs.push_back(fz);
                kzs.push_back(kz);
            }
            double t0 = 1e300;
            std::vector<double> tz(kzs.size(), 1e300);
            for (int round = 0; round < 2 && !kzs.empty(); ++round) {
                t0 = std::min(t0, time_it(k0, reps));
                for (size_t i = 0; i < kzs.size(); ++i) tz[i] = std::min(tz[i], time_it(kzs[i], reps));
            }
            size_t best = 0;
            for (size_t i = 1; i < tz.size(); ++i)
                if (tz[i] < tz[best]) best = i;
            if (!kzs.empty()) {
                log << "; fused zeroing";
                for (size_t i = 0; i < kzs.size(); ++i)
                    log << " " << kzs[i].zslabs << " slabs " << static_cast<long long>(tz[i] * 1e7) / 10.0 << " us";
                log << " vs one launch " << static_cast<long long>(t0 * 1e7) / 10.0 << " us";
                if (tz[best] < 0.99 * t0) I.auto_sched = fzs[best];
            }
        }
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
        const int reps = reps_of[first[0].second];
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

// femgpu_internal.hpp — host-side runtime structures of libfemgpu (not part of the ABI).
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <iosfwd>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/femgpu.h"

namespace femgpu {

// Errors thrown inside the library and converted to femgpu_status at the ABI.
struct Error : std::runtime_error {
    femgpu_status code;
    Error(femgpu_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(femgpu_status c, const std::string& m) { throw Error(c, m); }
inline void invalid(const std::string& m) { fail(FEMGPU_E_INVALID, m); }

void cuda_check(cudaError_t e, const char* what);
#define FG_CUDA(x) ::femgpu::cuda_check((x), #x)

// Structural copy of the problem signature + pointwise map: everything the
// kernel emitter needs (no bulk data).
struct MapNode {
    int op, a, b;
    double value;
};

struct Signature {
    int dim = 0, Q = 0, coord_dofs = 0;
    bool affine = true;
    int coordinate_space = -1;
    std::vector<int> sdofs, sterms;                 // scalar spaces
    std::vector<int> vdofs, vterms;                 // vector spaces
    std::vector<std::vector<int>> vcomps;           // component per vector term
    int nW = 0, Tw = 0;                             // test dofs / test terms
    std::vector<MapNode> nodes;
    std::vector<int> outputs;

    int ns() const { return static_cast<int>(sdofs.size()); }
    int nv() const { return static_cast<int>(vdofs.size()); }
    long long usable_flops() const;
    long long useful_flops() const;  // minus the skipped all-zero Psi entries (= usable_flops for dense Psi)
    // Offsets into the packed tabulation array (phi scalar, phi vector, psi, weights).
    std::vector<long long> phi_off_s, phi_off_v;
    long long psi_off = 0, w_off = 0, tab_size = 0;
    void layout();
    // Psi(k, jw, .) != 0 at some quadrature point ([k * nW + jw]; empty = all nonzero).  The emitters
    // skip the quadrature FMAs of all-zero entries (fused problems: the off-diagonal Psi blocks,
    // fuse.cpp); an output with no nonzero entry is checked for finiteness on its own.
    std::vector<char> psi_nz;
    bool pnz(int k, int jw) const { return psi_nz.empty() || psi_nz[static_cast<size_t>(k) * nW + jw]; }
    bool output_dead(int k) const {
        for (int jw = 0; jw < nW; ++jw)
            if (pnz(k, jw)) return false;
        return true;
    }
};

Signature signature_from(const femgpu_problem* p);
void dedupe_map(Signature& s);
std::vector<char> map_live(const Signature& sig);  // emit.cpp: nodes reachable from the outputs
std::vector<char> map_qdep(const Signature& sig);  // emit.cpp: nodes depending on the quadrature point  // commutative value numbering of the map DAG (bit-identical values)

// Device layout of vector inputs and coordinates: node-major with the components padded to a
// 16-byte multiple (3D: [node][4]), so a node's components are one aligned 16 B + 8 B pair of
// loads instead of three 8 B loads (fewer L1 wavefronts per gather).  The host (ABI) layout stays
// [node*dim + comp]; femgpu_create / set_inputs pad on upload.
inline int vec_stride(int dim) { return dim == 3 ? 4 : dim; }
// layout.cu: host [rows][d] -> device [rows][vec_stride(d)] (staging: rows*d doubles on the device)
void upload_padded(double* dst, const double* src_host, long long rows, int d, double* staging, cudaStream_t stream);

// Kernel families.
enum class Family { Scpt, Tile, Mlt, Macro, Dmma };

// Internal basis residency used by the checked twin of the DMMA family (tabulations read
// from global memory; they may exceed shared memory).
constexpr int kBasisGlobal = 3;

// Fully resolved launch plan (what the emitter specialises on).
struct KernelPlan {
    Family family = Family::Scpt;
    int basis = FEMGPU_BASIS_CONST;    // const (param bank) or smem
    int block = 128;                   // threads per CTA
    int tile_cells = 0;                // Tile: cells per CTA (== block)
    int min_blocks = 1;                // __launch_bounds__ min CTAs per SM (register cap)
    // Tile family: map-group ids per space (-1 = not staged) and smem capacities.
    std::vector<int> sgroup, vgroup;
    int tgroup = -1, cgroup = -1;
    int tvec = -1;                     // DMMA: vector space whose node map interleaves into the test map
    bool breg = false;                 // DMMA: B fragments in registers (single quadrature chunk)
    bool zfused = false;               // run_action: y zeroing fused into slab launches (FEMGPU_FLAG_FUSED_ZERO)
    int zslabs = 0;                    // slabs for fused zeroing (reserved[0] >> 8; 0 = default)
    bool pipe_memset = false;          // pipelined actions: memset the next output instead of in-kernel zeroing
    std::vector<int> group_entries, group_cap;   // per group: entries per cell, max unique per tile
    // MLT family (TilingParams)
    int Nc = 1, Nwi = 1, TQ = 1, Ter = 1, Tqr = 1, Tqc = 1;
    std::vector<int> Tcs, Tcv;
    bool strict = false;               // --fmad=false (bitwise debug mode)
    // Macro family: G cells per thread sharing the compile-time local pattern mpat[group]
    int G = 0;
    int mstage = 0;                       // 0: gathered values in registers; 1: cp.async into smem
    bool ysmem = false;                   // macro: y accumulators in thread-private smem columns (registers)
    bool qmajor = false;                  // macro: quadrature-point-major, statements interleaved over the G cells
    int msplit = 1;                       // macro q-major: cells of a group split over this many warps
    int qmopt = 0;                        // macro q-major: bit 0 hoisted column read from smem, bit 1 reload scatter
                                          // indices, bit 4 rolled quadrature loop, bit 5 persistent cp.async staging,
                                          // bit 8 warp merge of shared-node contributions before the scatter
    std::vector<std::array<int, 3>> merge;  // macro: warp-merge pairs (MacroLayout::merge of the test group)
    std::vector<std::array<long long, 4>> talias;  // macro: scatter rows derived from gathered indices (MacroLayout::talias)
    // DMMA without tvec: per test column (trial kind 0 scalar / 1 vector / -1 none, space, column,
    // scale, add): the row is scale * (that space's gathered node index) + add (Instance::test_alias)
    std::vector<std::array<long long, 5>> dalias;
    // SCPT (one cell per thread): the same per-column aliases, rows from the gathered node indices
    std::vector<std::array<long long, 5>> salias;
    long long stage_off = 0;              // macro q-major staging: byte offset of the staging area (emitter-internal)
    bool qloop = false;                   // scpt: keep the quadrature loop rolled (I-cache / registers)
    bool colour = false;                  // scpt: one launch per cell colour, plain y updates (deterministic)
    std::vector<std::vector<int>> mpat;   // per map group: G*entries local indices
    std::vector<std::vector<int>> maff;   // per map group: MacroLayout::aoff (empty: indices loaded)
    std::string key() const;
};

// DMMA family (emit_dmma.cpp): evaluation groups = (space, component) with their terms.
struct DmmaGroup {
    bool vec = false;
    int space = 0, comp = 0, n = 0;
    std::vector<int> terms;
    int KS = 0, NB = 0;          // k-steps (n/4), n-blocks of 8 output slots per chunk
    long long foff = 0;          // first fragment within a chunk
};
struct DmmaLayout {
    int CW = 0, MB = 0;          // cells per warp task, m-blocks of 8 cells
    int TQ = 0, TQL = 0, NCH = 0;  // quadrature points per chunk, per lane-group, chunks
    std::vector<DmmaGroup> groups;
    int KQ = 0, NBQ = 0;         // quadrature k-steps (Tw*TQL) and n-blocks (nW/8) per chunk
    long long foff_q = 0, FPC = 0, nfrag = 0;  // fragments: quadrature offset, per chunk, total
};
DmmaLayout dmma_layout(const Signature& sig, const KernelPlan& kp);
std::vector<double> dmma_fragments(const Signature& sig, const DmmaLayout& L, const std::vector<double>& tab);
size_t dmma_smem_bytes(const Signature& sig, const KernelPlan& kp);
long long dmma_live_doubles(const Signature& sig, const DmmaLayout& L);
void resolve_dmma(const Signature& sig, KernelPlan& kp, const femgpu_schedule* s);

struct EmitResult {
    std::string source;
    std::string kernel;          // fast kernel name
    std::string kernel_checked;  // stage-checked diagnostic kernel name
    size_t param_bytes = 0;
    size_t smem_bytes = 0;       // dynamic shared memory per CTA
};

EmitResult emit_kernel(const Signature& sig, const KernelPlan& kp);
size_t tile_smem_bytes(const Signature& sig, const KernelPlan& kp);

// JIT: NVRTC compile for sm_100a, cached by source hash (memory + disk).
struct Module {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t fast = nullptr, checked = nullptr;
    EmitResult emitted;
    int regs = 0;
    long long local_bytes = 0;  // local memory per thread (spills) of the fast kernel
    int occupancy = 1;   // resident CTAs per SM of the fast kernel
    int sms = 148;
};
std::vector<char> jit_compile(const std::string& source, bool strict, std::string* log);
std::shared_ptr<Module> get_module(const Signature& sig, const KernelPlan& kp);

// Tile layout of one map group at one tile size (built in femgpu_create).
struct TileGroup {
    int entries = 0;
    int max_unique = 0;
    long long total_unique = 0;
    int32_t* d_off = nullptr;      // per tile: start of its (4-aligned) segment in list/roff
    int32_t* d_cnt = nullptr;      // per tile: unique entries
    int32_t* d_list = nullptr;     // global index | 0x80000000 if shared with another tile
    uint16_t* d_loc = nullptr;     // [entry][lstride] tile-local index (lstride = n_tiles*TB)
};

struct TileLayout {
    int tile_cells = 0;
    int n_tiles = 0;
    std::vector<TileGroup> groups;
    // CSR of the test group: per unique DOF (aligned with its list) the start of its
    // contribution run; per tile, TB*nW staging positions j*TB + local_cell.
    uint16_t* d_roff = nullptr;
    uint16_t* d_rpos = nullptr;
};

// Macro-element layout: groups of G consecutive cells with one common local
// connectivity pattern per distinct map (detected in femgpu_create).
struct MacroLayout {
    int G = 0;
    long long n_groups = 0;
    bool ok = false;
    std::vector<int> unique;                 // per map group: unique entries per cell group
    std::vector<std::vector<int>> pattern;   // per map group: G*entries local indices
    std::vector<int32_t*> d_gidx;            // per map group: [unique][n_groups] global indices
    // warp merge of the test map (q-major kernels, qmopt bit 8): (lane shift s, unique u, unique u')
    // such that group g's node u is group g+s's node u' for at least half of the group pairs of a warp
    std::vector<std::array<int, 3>> merge;
    // per unique node of the test group: (group, unique, scale, add) with row = scale * node + add of
    // another group's unique node (Instance::test_alias), group -1 = loaded from the test group's gidx
    std::vector<std::array<long long, 4>> talias;
    // per map group: gidx[u][grp] = gidx[0][grp] + aoff[u] for every cell group (a lattice-numbered
    // structured mesh), so one index load per group and compile-time offsets replace the U loads;
    // empty = not affine
    std::vector<std::vector<int>> aoff;
};

// Greedy colouring of the test map (femgpu_color_cells) with the cells sorted by colour.
struct Colouring {
    int n = 0;
    std::vector<int> off;        // colour c = perm[off[c] .. off[c+1])
    int32_t* d_perm = nullptr;   // cells ordered by (colour, cell)
};

struct DeviceSpace {
    int dofs = 0, terms = 0, global = 0;
    double* d_x = nullptr;          // input vector (vector spaces: padded [node][vec_stride])
    double* d_stage = nullptr;      // vector spaces: contiguous upload staging ([node][dim])
    int32_t* d_mapT = nullptr;      // [entry][cell] (SoA, coalesced); may alias another space's
    int group = -1;                 // content-equal map group
};

// Slab plan of the overlapped host-buffer action (pipeline.cpp).
struct PipePlan {
    int align = 1;
    std::vector<int> cb;                      // slab k = cells [cb[k], cb[k+1])
    std::vector<std::vector<long long>> up;   // per trial space: input rows resident before slab k
    std::vector<long long> zero_hi;           // y rows zeroed before slab k
    std::vector<long long> fin;               // y rows final (downloadable) after slab k
    bool useful = false;
};

struct Instance {
    Signature sig;
    int device = 0;
    int cells = 0, output_size = 0;
    std::vector<double> tab;        // packed tabulations (host copy, goes to param bank)
    double* d_tab = nullptr;        // packed tabulations (device, smem-staged variants)
    std::vector<DeviceSpace> sspaces, vspaces;
    int32_t* d_tmapT = nullptr;
    int32_t* d_cmapT = nullptr;
    double* d_coords = nullptr;
    int coord_global = 0;
    int test_group = -1, coord_group = -1;
    // vector space i with test_map[c][a*dim + comp] == map_i[c][a]*dim + comp (interleaved vector
    // test space, form.hpp:664-665 convention), or -1: the scatter can then reuse the gathered node
    // indices instead of reading the (dim x larger) test map
    int test_vspace = -1;
    // per test column j: test_map[c][j] == scale * map_g[c][col] + add for every cell c (another
    // map group g), or group -1.  Fused problems (fuse.cpp): problem p's test rows are its trial (or
    // vertex) rows shifted by its output offset; vector test spaces: node * dim + comp.  The macro
    // kernels then scatter through indices they already gathered instead of loading the test map.
    struct TestAlias {
        int group = -1, col = 0, scale = 1;
        long long add = 0;
    };
    std::vector<TestAlias> test_alias;
    std::vector<std::vector<int32_t>> group_maps;  // host copies of distinct maps ([cell][entry])
    std::vector<int> group_global;
    double* d_y = nullptr;
    double* d_y2 = nullptr;         // second output buffer of pipelined steps (femgpu_time_steps_ex)
    double* second_output() {
        if (!d_y2) d_y2 = alloc<double>(static_cast<size_t>(output_size));
        return d_y2;
    }
    int32_t* d_bad = nullptr;       // first failing cell (INT32_MAX = none)
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::map<int, std::unique_ptr<TileLayout>> tiles;   // by tile size
    std::map<int, std::unique_ptr<MacroLayout>> macros; // by cells per group
    std::map<int, double*> dmma_frags;                   // by quad tile: fragment-major Phi/Psi
    double* dmma_fragments_for(const KernelPlan& kp);
    std::map<std::string, std::shared_ptr<Module>> modules;  // by KernelPlan::key(): no re-emit per launch
    std::shared_ptr<Module> module_for(const KernelPlan& kp);
    std::vector<void*> allocations;
    int64_t device_bytes = 0;
    int64_t last_launches = 0;
    std::mutex mu;                  // serialises actions on this instance (tune(jobs>1))
    // automatic schedule (s == NULL): chosen once per instance by tune.cpp
    std::unique_ptr<PipePlan> pipe;
    std::unique_ptr<Colouring> colouring;
    const Colouring& colour_plan();
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    std::vector<cudaEvent_t> ev_pipe;
    // streaming host actions (femgpu_action_host_async): two sets of device inputs/outputs, so step
    // i+1's uploads run while step i's results download.  Set 0 is the instance's own d_x / d_y.
    std::vector<double*> x_alt;                 // per trial space (scalar then vector): set-1 inputs
    std::vector<double*> cg_work;               // device CG (cg.cu): r, p, two A p buffers, partials + scalars
    cudaEvent_t ev_async_comp[2] = {nullptr, nullptr}, ev_async_d2h[2] = {nullptr, nullptr};
    bool async_used[2] = {false, false};
    int async_next = 0, async_pending = 0, async_last = -1;
    KernelPlan async_kp;
    const PipePlan& pipe_plan(int align);
    std::unique_ptr<PipePlan> pipe_stream;         // streaming steps: few large slabs (stream_slab_count)
    const PipePlan& stream_plan(int align);
    // fused zeroing of y (pipeline.cpp): slab plan, worker stream, per-slab events
    std::map<std::pair<int, int>, std::unique_ptr<PipePlan>> zplans;  // by (align, slabs): host scan of the maps
    const PipePlan& zero_plan(int align, int slabs, int max_slabs);
    std::unique_ptr<PipePlan> slab_plan(int K, int align) const;
    cudaStream_t s_work = nullptr;
    std::vector<cudaEvent_t> ev_zero;
    bool auto_ready = false;
    femgpu_schedule auto_sched{};
    std::string auto_log;

    ~Instance();
    template <typename T>
    T* alloc(size_t count) {
        void* p = nullptr;
        FG_CUDA(cudaMalloc(&p, count * sizeof(T) + 16));
        allocations.push_back(p);
        device_bytes += static_cast<int64_t>(count * sizeof(T));
        return static_cast<T*>(p);
    }
    const TileLayout& tile_layout(int tile_cells);
    const MacroLayout& macro_layout(int G);
};

void validate_problem(const femgpu_problem* p);
// Host-only tile planning (map groups, per-tile unique caps) for emit/JIT checks without a GPU.
void host_tile_plan(const femgpu_problem* p, const Signature& sig, KernelPlan& kp, const femgpu_schedule* s);
void host_macro_plan(const femgpu_problem* p, const Signature& sig, KernelPlan& kp, const femgpu_schedule* s);
std::unique_ptr<Instance> create_instance(const femgpu_problem* p);
KernelPlan resolve_schedule(Instance& inst, const femgpu_schedule* s);
void run_action(Instance& inst, const KernelPlan& kp, double* d_y, cudaStream_t stream,
                cudaEvent_t after_zero = nullptr);
// One launch over the cell range [c_begin, c_end) (Scpt, Macro (G-aligned) and Dmma families);
// y is zeroed first only when zero_y.
// zero_ptr / zero_n: y rows of a later slab this launch clears (fused zeroing, pipeline.cpp).
void run_action_range(Instance& inst, const KernelPlan& kp, double* d_y, cudaStream_t stream, int c_begin, int c_end,
                      bool zero_y, cudaEvent_t after_zero = nullptr, double* zero_ptr = nullptr,
                      long long zero_n = 0);
long long launch_grid(Instance& inst, const KernelPlan& kp, const Module& mod, long long ncell);  // CTAs of one launch
extern const char* kZeroPrologue;  // emit.cpp
// Output-pipelined action: d_y is all zeros on entry; the action kernel also zeroes d_next (the next
// step's output) in its prologue, so back-to-back steps need no separate memset (femgpu_action_device_pipelined).
void run_action_pipelined(Instance& inst, const KernelPlan& kp, double* d_y, double* d_next, cudaStream_t stream);
bool supports_cell_range(const KernelPlan& kp);
int range_align(const KernelPlan& kp);
// pipeline.cpp: y zeroing fused into slab-wise compute; false = not applicable
bool overlapped_zero_action(Instance& inst, const KernelPlan& kp, double* d_y, cudaStream_t stream,
                            cudaEvent_t after_zero);
// pipeline.cpp: femgpu_action_host overlapped over H2D / compute / D2H streams; false = not applicable
// buf = -1: one synchronous action into inst.d_y; buf = 0/1: a streaming step on buffer set `buf`
// (inputs already swapped in by the caller) writing y_dev, ordered against the previous use of the set
bool pipelined_host_action(Instance& inst, const KernelPlan& kp, const double* const* scalar_inputs,
                           const double* const* vector_inputs, double* y_host, int buf = -1, double* y_dev = nullptr);
void check_failure(Instance& inst, const KernelPlan& kp, cudaStream_t stream);
// cg.cu: conjugate gradients on the instance stream for a square scalar SPD operator
void device_cg(Instance& I, const KernelPlan& kp, const double* b, double* x, double rtol, int maxiter, int check_every,
               int* iterations, double* rel_residual);
// Host-side data-parallel loop over [0, n) in up to 32 contiguous chunks (re-blocking, layouts, reorder).
template <typename F>
void parallel_for(long long n, F&& f) {
    const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    const long long chunks = std::min<long long>(hw, std::max<long long>(1, n / 4096));
    if (chunks <= 1) {
        f(0LL, n);
        return;
    }
    std::vector<std::thread> th;
    for (long long c = 0; c < chunks; ++c)
        th.emplace_back([&, c] { f(n * c / chunks, n * (c + 1) / chunks); });
    for (auto& t : th) t.join();
}
// C-ABI error plumbing shared by the translation units that implement entry points
void set_last_error(const std::string& msg);
template <typename F>
femgpu_status abi_guard(F&& f) {
    try {
        f();
        return FEMGPU_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return FEMGPU_E_INTERNAL;
    } catch (...) {
        set_last_error("unknown error");
        return FEMGPU_E_INTERNAL;
    }
}
}  // namespace femgpu
// An owned problem (io.cpp load_problem, fuse.cpp fuse_problems): the flat descriptor plus its storage.
struct femgpu_owned_problem {
    femgpu_problem desc{};
    std::vector<femgpu_space> sspaces, vspaces;
    std::vector<std::vector<int32_t>> smaps, vmaps, comps;
    std::vector<std::vector<double>> sphi, vphi, sin, vin;
    std::vector<double> psi, weights, coords;
    std::vector<int32_t> test_map, coord_map, outputs;
    std::vector<femgpu_map_node> nodes;
};
struct femgpu_instance {
    std::unique_ptr<femgpu::Instance> impl;
};
const femgpu_problem* femgpu_owned_view(const femgpu_owned_problem* p);
void femgpu_owned_delete(femgpu_owned_problem* p);
namespace femgpu {
// io.cpp: the reference's structured-text instance / candidate files (io.hpp)
void save_problem(std::ostream& os, const femgpu_problem* p);
femgpu_owned_problem* load_problem(std::istream& is);
void save_schedule(std::ostream& os, const femgpu_schedule* s, int n_scalar, int n_vector);
femgpu_schedule load_schedule(std::istream& is);
// tune.cpp: the automatic schedule (cost-model pruning + empirical timing, cached per instance)
void autotune(Instance& inst);
KernelPlan plan_for(Instance& inst, const femgpu_schedule* s);
std::string describe_plan(const KernelPlan& kp);

}  // namespace femgpu

/*
 * femgpu.h — C-ABI of the B200-native (sm_100a) FP64 matrix-free finite-element
 * action y = A(u)·x.  Drop-in for the reference `femsched` action path:
 *
 *   reference entry point                                   replaced by
 *   -----------------------------------------------------   ---------------------------------
 *   femsched::reference_action(const ProblemInstance&)        femgpu_create + femgpu_action
 *     (/root/reference/proj/include/femsched/form.hpp:471-595)  (or femgpu_action_once)
 *   femsched::run_schedule(inst, build_plan(sig, params))     femgpu_action(inst, &schedule, y)
 *     (simulate.hpp:601-603, run_scpt :171, run_mlt :293)
 *   femsched::Executor / ExecutionOutcome                     femgpu_execute (measured seconds)
 *     (search.hpp:257-283)
 *   femsched::usable_flops (form.hpp:164-173)                 femgpu_usable_flops
 *
 * All arguments are plain pointers and sizes; no C++ or torch types cross this
 * boundary and no C++ exception escapes it.  Every function returns a
 * femgpu_status; the message of the last failure on the calling thread is
 * available from femgpu_last_error().  Status codes map onto the reference's
 * exception types (form.hpp:23-31, form.hpp:492-495):
 *   FEMGPU_E_INVALID    -> std::invalid_argument  (validate() failures)
 *   FEMGPU_E_INFEASIBLE -> femsched::InfeasibleError (schedule cannot launch)
 *   FEMGPU_E_NONFINITE  -> std::runtime_error "non-finite value at cell N during <stage>"
 *
 * Host pointers passed to femgpu_create are borrowed for the duration of the
 * call only; the instance owns device copies afterwards (re-blocked layout).
 */
#ifndef FEMGPU_H
#define FEMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FEMGPU_ABI_VERSION 1

typedef enum femgpu_status {
    FEMGPU_OK = 0,
    FEMGPU_E_INVALID = 1,
    FEMGPU_E_INFEASIBLE = 2,
    FEMGPU_E_NONFINITE = 3,
    FEMGPU_E_CUDA = 4,
    FEMGPU_E_JIT = 5,
    FEMGPU_E_INTERNAL = 6
} femgpu_status;

/* PointwiseMap::Op, same numbering as femsched (form.hpp:194-204).
 * FEMGPU_OP_INV_JACOBIAN is a B200-build extension (J^{-1}[a][b], affine only);
 * it is not expressible in the reference map language. */
typedef enum femgpu_map_op {
    FEMGPU_OP_CONSTANT = 0,
    FEMGPU_OP_SCALAR_DERIV = 1, /* a = space, b = term */
    FEMGPU_OP_VECTOR_DERIV = 2, /* a = space, b = term */
    FEMGPU_OP_JACOBIAN = 3,     /* a = row, b = col */
    FEMGPU_OP_DETERMINANT = 4,
    FEMGPU_OP_WEIGHT = 5,
    FEMGPU_OP_COORD = 6, /* a = local vertex, b = axis */
    FEMGPU_OP_ADD = 7,
    FEMGPU_OP_MUL = 8,
    FEMGPU_OP_INV_JACOBIAN = 9 /* extension */
} femgpu_map_op;

/* PointwiseMap::Node (form.hpp:205-209). */
typedef struct femgpu_map_node {
    int32_t op;
    int32_t a;
    int32_t b;
    int32_t pad_;
    double value;
} femgpu_map_node;

/* One trial space: ScalarSpace/VectorSpace (form.hpp:71-80) together with its
 * tabulations (form.hpp:324-330), index map (form.hpp:49-65) and input vector
 * (form.hpp:412-413). */
typedef struct femgpu_space {
    int32_t dofs;              /* local DOFs (per component for vector spaces) */
    int32_t deriv_terms;
    const int32_t* components; /* vector spaces: deriv_terms component indices; NULL for scalar */
    const double* phi;         /* deriv_terms x quad_points x dofs, row-major per term */
    const int32_t* map;        /* cell_count x dofs, row-major [cell][entry] */
    int32_t global_count;      /* IndexMap::global_count */
    int32_t pad_;
    const double* input;       /* global_count (scalar) or global_count*dim (vector, [node*dim+comp]) */
} femgpu_space;

/* femsched::ProblemInstance flattened (form.hpp:407-435). */
typedef struct femgpu_problem {
    int32_t dim;
    int32_t quad_points;
    int32_t coord_dofs;
    int32_t affine_geometry;   /* bool */
    int32_t coordinate_space;  /* -1 when affine */
    int32_t word_bytes;
    int32_t n_scalar;
    int32_t n_vector;
    const femgpu_space* scalar_spaces;
    const femgpu_space* vector_spaces;
    int32_t test_dofs;
    int32_t test_deriv_terms;
    const double* psi;         /* test_deriv_terms x test_dofs x quad_points */
    const double* weights;     /* quad_points */
    int32_t cell_count;
    int32_t test_global_count;
    const int32_t* test_map;   /* cell_count x test_dofs */
    const int32_t* coord_map;  /* cell_count x coord_dofs (affine only) */
    const double* coords;      /* coord_global_count x dim (affine only) */
    int32_t coord_global_count;
    int32_t n_map_nodes;
    const femgpu_map_node* map_nodes;
    const int32_t* map_outputs; /* test_deriv_terms node ids */
    int32_t n_map_outputs;
    int32_t output_size;
} femgpu_problem;

/* Schedule point.  kind/tile fields mirror femsched::TilingParams
 * (qoi.hpp:23-41); the remaining fields are B200 knobs (0 = automatic). */
typedef enum femgpu_schedule_kind {
    FEMGPU_SCPT = 0, /* TilingParams::scpt(): one thread per cell */
    FEMGPU_MLT = 1,  /* multi-level tiling: N_c cells x N_WI lanes per CTA */
    FEMGPU_DMMA = 2  /* B200 extension: warp-level FP64 tensor-core (DMMA m8n8k4) pipeline.
                        cells_per_group = cells per warp task (8, 16, 24, 32), quad_tile = T^Q
                        quadrature points per chunk (rounded up to a multiple of 4),
                        lanes_per_cell = 4 (fixed by the fragment layout; 0 accepted),
                        block_cells = threads per CTA, basis SMEM = Phi/Psi fragments staged in
                        shared memory once per CTA (else read through L1);
                        0 = automatic for every field */
} femgpu_schedule_kind;

typedef enum femgpu_basis {
    FEMGPU_BASIS_AUTO = 0,
    FEMGPU_BASIS_CONST = 1, /* tabulations in the constant bank (DFMA c[] operands) */
    FEMGPU_BASIS_SMEM = 2   /* tabulations staged once per CTA in shared memory */
} femgpu_basis;

typedef enum femgpu_scatter {
    FEMGPU_SCATTER_AUTO = 0,
    FEMGPU_SCATTER_ATOMIC = 1, /* red.global.add.f64 per (cell, test DOF) */
    FEMGPU_SCATTER_TILE = 2,   /* CTA-tile aggregation in smem; global atomics only on shared DOFs */
    FEMGPU_SCATTER_MACRO = 3,  /* macro-elements: G cells per thread with a common local pattern,
                                  register accumulation, one atomic per unique DOF of the group */
    FEMGPU_SCATTER_COLOR = 4   /* greedy cell colouring of the test map (femgpu_color_cells): one launch
                                  per colour, plain read-modify-write of y (no two cells of a colour
                                  share a DOF), so y is bitwise reproducible run to run */
} femgpu_scatter;

#define FEMGPU_MAX_SPACES 8

typedef struct femgpu_schedule {
    int32_t kind;
    int32_t quad_tile;
    int32_t eval_row_tile;
    int32_t eval_col_tiles_scalar[FEMGPU_MAX_SPACES];
    int32_t eval_col_tiles_vector[FEMGPU_MAX_SPACES];
    int32_t quad_row_tile;
    int32_t quad_col_tile;
    int32_t cells_per_group;
    int32_t lanes_per_cell;
    /* B200 knobs */
    int32_t basis;         /* femgpu_basis */
    int32_t scatter;       /* femgpu_scatter */
    int32_t block_cells;   /* SCPT/tile: cells (threads) per CTA; macro: groups (threads) per CTA; 0 = auto */
    int32_t group_cells;   /* macro: cells per group G; 0 = auto */
    int32_t reserved[4];   /* [0] flags (FEMGPU_FLAG_*), [1] register target, [2] min CTAs/SM */
} femgpu_schedule;

/* femgpu_schedule.reserved[0] flags */
#define FEMGPU_FLAG_STRICT 1      /* --fmad=false: the reference's bitwise per-cell arithmetic */
#define FEMGPU_FLAG_FUSED_ZERO 2  /* y zeroing fused into slab launches (Macro/SCPT/DMMA, large
                                     outputs; the automatic schedule sets it where it measures faster);
                                     bits 8-15 of reserved[0]: slab count (0 = 8) */
#define FEMGPU_FLAG_PIPE_MEMSET 4 /* femgpu_action_device_pipelined zeroes the next output with a separate
                                     memset instead of inside the action kernel (the automatic schedule
                                     sets it where the in-kernel zeroing measures slower) */
#define FEMGPU_FLAG_INDEX_LOADS 8 /* macro kernels load every unique index of a cell group even when the
                                     mesh numbering makes them one base plus fixed offsets (the
                                     automatic schedule sets it where the offset form measures slower) */

typedef struct femgpu_instance femgpu_instance;

/* ---- library --------------------------------------------------------- */
int32_t femgpu_abi_version(void);
const char* femgpu_last_error(void);
/* Number of CUDA devices visible (0 on a host without a GPU). */
int32_t femgpu_device_count(void);
/* Select the device used by subsequent femgpu_create calls on this thread. */
femgpu_status femgpu_set_device(int32_t device);

/* ---- pure host helpers (no GPU needed) --------------------------------- */
/* femsched::usable_flops (form.hpp:164-173) */
femgpu_status femgpu_usable_flops(const femgpu_problem* p, int64_t* flops_per_cell);
/* The reference's ReferenceCounters for reference_action(p, &counters) (form.hpp:463-472):
 * matvec mults/adds and pointwise-map add/mul evaluations of the unmemoised recursion, computed
 * from the instance's structure (the GPU kernels execute the same arithmetic with a compiled,
 * value-numbered map, so they do not count at run time). */
femgpu_status femgpu_reference_counters(const femgpu_problem* p, int64_t* matvec_mults, int64_t* matvec_adds,
                                        int64_t* map_ops);
/* femsched::ProblemInstance::validate (form.hpp:416-434) */
femgpu_status femgpu_validate(const femgpu_problem* p);
/* Emit the CUDA source the JIT would compile for (problem signature+map, schedule).
 * Writes at most cap bytes (NUL-terminated) and the full length to *len. */
femgpu_status femgpu_emit_source(const femgpu_problem* p, const femgpu_schedule* s,
                                 char* buf, size_t cap, size_t* len);
/* Compile that source with NVRTC for sm_100a (works without a GPU). */
femgpu_status femgpu_jit_check(const femgpu_problem* p, const femgpu_schedule* s);

/* ---- device instance --------------------------------------------------- */
femgpu_status femgpu_create(const femgpu_problem* p, femgpu_instance** out);
femgpu_status femgpu_destroy(femgpu_instance* inst);
/* Replace trial input vectors (host pointers, lengths as in the problem). */
femgpu_status femgpu_set_inputs(femgpu_instance* inst, const double* const* scalar_inputs,
                                const double* const* vector_inputs);
/* y = A(u)·x into a host buffer of output_size doubles (H2D of nothing, D2H of y). */
femgpu_status femgpu_action(femgpu_instance* inst, const femgpu_schedule* s, double* y_host);
/* End to end: copy host inputs in (like set_inputs), run, copy y out.  On instances with locality
 * (>= 1M cells, node-ordered slabs) the H2D of x, the action (slab by slab over contiguous cell
 * ranges) and the D2H of the finished part of y overlap on three streams (FEMGPU_PIPELINE=0
 * disables).  Host buffers should be pinned (femgpu_host_alloc) for the overlap. */
femgpu_status femgpu_action_host(femgpu_instance* inst, const femgpu_schedule* s,
                                 const double* const* scalar_inputs,
                                 const double* const* vector_inputs, double* y_host);
/* Streaming end-to-end actions: like femgpu_action_host, but returns once the step is enqueued.
 * Two sets of device inputs/outputs alternate, so step i+1's H2D overlaps step i's D2H (PCIe is
 * full duplex).  Every step still copies its inputs in and its y out.  Host buffers must stay valid
 * (inputs) and unread (y) until femgpu_action_host_wait, which completes all steps, leaves the
 * instance holding the last step's inputs and output, and reports a non-finite value in any step.
 * Every other call on the instance completes pending steps first.  Instances without a slab plan
 * run each step synchronously. */
femgpu_status femgpu_action_host_async(femgpu_instance* inst, const femgpu_schedule* s, const double* const* scalar_inputs,
                                       const double* const* vector_inputs, double* y_host);
femgpu_status femgpu_action_host_wait(femgpu_instance* inst);
/* The action's caller: conjugate gradients for A x = b with A the instance's operator
 * (one scalar trial space numbered like the test space; symmetric positive definite), entirely on the
 * instance stream: one output-pipelined action + fused update kernels per iteration, scalars in device
 * memory, fixed-order reductions (no float atomics outside the action); the host reads the residual every check_every
 * iterations.  b_dev, x_dev: device vectors of output_size doubles; x_dev = initial guess in, solution
 * out.  Stops at ||r|| <= rtol ||b|| or maxiter; *iterations, *rel_residual = ||r|| / ||b||. */
femgpu_status femgpu_cg(femgpu_instance* inst, const femgpu_schedule* s, const double* b_dev, double* x_dev, double rtol,
                        int32_t maxiter, int32_t check_every, int32_t* iterations, double* rel_residual);
/* Device-resident: y_dev is a device pointer of output_size doubles; stream is a
 * cudaStream_t (NULL = the instance stream, a non-blocking stream; pass cudaStreamLegacy to order
 * after work on the legacy default stream, e.g. torch's default stream whose handle is 0).
 * Asynchronous, no host sync. */
femgpu_status femgpu_action_device(femgpu_instance* inst, const femgpu_schedule* s, double* y_dev,
                                   void* stream);
/* Output-pipelined device action: y_dev must hold zeros on entry (e.g. zeroed by the previous call);
 * in stream order y_dev becomes A(u)·x and y_next_dev[0:output_size) is zeroed, the zeroing done
 * inside the action kernel (macro / SCPT / DMMA families; a memset otherwise).  Back-to-back
 * actions into alternating buffers (a Krylov loop's successive products) thus need one launch each
 * and no separate memset.  y_next_dev may be NULL; it must not alias y_dev.  Asynchronous. */
femgpu_status femgpu_action_device_pipelined(femgpu_instance* inst, const femgpu_schedule* s, double* y_dev,
                                             double* y_next_dev, void* stream);
/* Non-finite check of the device-side actions issued so far on `stream` (NULL = instance stream):
 * synchronizes the stream and reports FEMGPU_E_NONFINITE with the reference's diagnostic
 * ("non-finite value at cell N during <stage>", form.hpp:492-595) if any cell produced one. */
femgpu_status femgpu_check_finite(femgpu_instance* inst, const femgpu_schedule* s, void* stream);
/* Paper timing protocol: warmup launches, then at least
 * min_reps and at least min_seconds of [zero y + action] timed with CUDA events on
 * the instance stream; *seconds = arithmetic mean per action. */
femgpu_status femgpu_time_action(femgpu_instance* inst, const femgpu_schedule* s, int32_t warmup,
                                 int32_t min_reps, double min_seconds, double* seconds);
/* Exactly `steps` back-to-back actions [zero y + action] on the instance stream, bracketed by
 * a device synchronize on both sides and timed with CUDA events: *seconds = total elapsed. */
femgpu_status femgpu_time_steps(femgpu_instance* inst, const femgpu_schedule* s, int32_t steps,
                                double* seconds);
/* femgpu_time_steps with flags: FEMGPU_STEPS_PIPELINED = each step is one
 * femgpu_action_device_pipelined into alternating output buffers (the step still zeroes one full
 * output and computes one full action; the zeroing runs inside the action kernel). */
#define FEMGPU_STEPS_PIPELINED 1
femgpu_status femgpu_time_steps_ex(femgpu_instance* inst, const femgpu_schedule* s, int32_t steps, int32_t flags,
                                   double* seconds);
/* Split timing of the same protocol: mean seconds per step [zero y + action], per
 * action kernel alone and per y-zeroing, each bracketed by CUDA events on the
 * instance stream (the roofline's per-kernel duration). */
femgpu_status femgpu_profile_action(femgpu_instance* inst, const femgpu_schedule* s, int32_t warmup,
                                    int32_t reps, double* step_seconds, double* kernel_seconds,
                                    double* zero_seconds);
/* The FP64 roofline denominator, measured live: DFMA peak of the current device
 * (TFLOP/s) and its nominal SM clock (GHz).  Ahead-of-time sm_100a kernel. */
femgpu_status femgpu_fp64_peak(double* tflops, double* sm_clock_ghz);
/* The FP64 tensor-core (DMMA m8n8k4) peak of the current device (TFLOP/s), measured live. */
femgpu_status femgpu_fp64_dmma_peak(double* tflops);
/* Executor seam (search.hpp:257-283): run, verify finiteness, report output and
 * measured seconds (mean of the timing protocol above). */
femgpu_status femgpu_execute(femgpu_instance* inst, const femgpu_schedule* s, double* y_host,
                             double* measured_seconds);
/* The schedule femgpu uses for this instance when s == NULL: on instances of >= 200k cells the
 * kernel families are pruned by an FP64-pipe cost model and the survivors timed once (CUDA
 * events); the winner is cached in the instance (FEMGPU_AUTOTUNE=0 disables the timing).
 * Replaces femsched::rank + tune (search.hpp:211-416) for the default path. */
femgpu_status femgpu_default_schedule(const femgpu_instance* inst, femgpu_schedule* s);
/* Human-readable kernel plan for schedule s (NULL = the automatic one, with its tuning log). */
femgpu_status femgpu_describe_schedule(femgpu_instance* inst, const femgpu_schedule* s, char* buf, size_t cap,
                                       size_t* len);
/* Introspection: kernel launches issued by the last action, device bytes held. */
femgpu_status femgpu_stats(const femgpu_instance* inst, int64_t* launches_last_action,
                           int64_t* device_bytes, int64_t* tiles, int64_t* max_tile_dofs);
/* The execution census of schedule s on this instance, in the field order of femsched::TraceCounters
 * (simulate.hpp:91-104) followed by the workgroup count (ExecutionOutcome::workgroups, search.hpp:263):
 * [0] barriers per workgroup, [1] flops_matvec, [2] flops_masked_padding (DMMA m8n8k4 padding),
 * [3] gather_words (trial words read: each unique node of a macro group once), [4] scatter_words
 * (red.add issued), [5] reference_words (tabulation words staged per CTA), [6] reference_cached_words
 * (constant-bank reads), [7] coord_words, [8..10] local eval/quad words (0: registers), [11] shared-memory
 * words per CTA, [12] CTAs launched.  n >= FEMGPU_TRACE_COUNTERS. */
#define FEMGPU_TRACE_COUNTERS 13
femgpu_status femgpu_trace_counters(femgpu_instance* inst, const femgpu_schedule* s, int64_t* out, int32_t n);
/* Copies the instance's output buffer (the y of the last action, or of the last step of
 * femgpu_time_steps / femgpu_time_steps_ex) into y_host (output_size doubles); synchronous. */
femgpu_status femgpu_read_output(femgpu_instance* inst, double* y_host);
/* Device pointers (for zero-copy callers): output buffer of the instance. */
femgpu_status femgpu_device_output(femgpu_instance* inst, double** y_dev);
/* Device pointer of trial input vector `space` (scalar spaces first, then vector spaces),
 * for zero-copy halo exchanges (multi-GPU): length global_count for scalar spaces; vector spaces
 * are stored node-major with the components padded to 16 bytes ([node][4] in 3D, [node][2] in
 * 2D), so their length is global_count x (dim == 3 ? 4 : dim). */
femgpu_status femgpu_device_input(femgpu_instance* inst, int32_t space, double** x_dev);
/* The CUDA stream (cudaStream_t) the instance launches on. */
femgpu_status femgpu_stream(femgpu_instance* inst, void** stream);

/* One-shot, reference_action-shaped: create, run (default schedule), destroy. */
femgpu_status femgpu_action_once(const femgpu_problem* p, double* y_host);

/* Pinned host memory helpers. */
femgpu_status femgpu_host_alloc(size_t bytes, void** ptr);
femgpu_status femgpu_host_free(void* ptr);

/* ---- multi-GPU: cell-partitioned action with GPU-to-GPU halo exchange -----
 * (the reference is single-process.)  One rank per GPU owns a slab of cells
 * as its own instance (compact local numbering).  Lists are in that local numbering:
 *   push  (push_peer[i], push_row[i]): rows whose partial sums this rank computes but rank
 *         push_peer[i] owns; per owner in ascending global-DOF order
 *   recv  (recv_peer[i], recv_row[i]): owned rows rank recv_peer[i] contributes to, per source in
 *         the same order as that source's push list to this rank
 *   pull  (pull_space[i], pull_peer[i], pull_node[i], pull_remote[i]): ghost node pull_node[i] of
 *         trial space pull_space[i] (scalar spaces first) takes its value from node pull_remote[i]
 *         of its owner pull_peer[i]
 * Cells [0, boundary_cells) are the only ones touching shared rows (the local cell order puts
 * them first); the push of their partial sums overlaps the interior cells.  Owners add what they
 * receive in ascending rank order (deterministic).  Peer buffers are reached over NVLink (CUDA IPC
 * across processes, direct pointers within a process); ranks are ordered by device-side flags, so
 * a step is a fixed launch sequence on one stream with no host synchronisation.  Every rank must
 * run the same number of actions.  The caller may change owned inputs between actions only once
 * every rank finished the previous action (e.g. after an all-reduce, as in a Krylov loop). */
typedef struct femgpu_halo femgpu_halo;
femgpu_status femgpu_halo_create(femgpu_instance* inst, int32_t rank, int32_t world, int32_t boundary_cells,
                                 int64_t n_push, const int32_t* push_peer, const int32_t* push_row, int64_t n_recv,
                                 const int32_t* recv_peer, const int32_t* recv_row, int64_t n_pull,
                                 const int32_t* pull_space, const int32_t* pull_peer, const int32_t* pull_node,
                                 const int32_t* pull_remote, femgpu_halo** out);
femgpu_status femgpu_halo_destroy(femgpu_halo* h);
/* The bytes this rank publishes (IPC handles and offsets of its flags, receive buffer and input
 * buffers); *len = the fixed size.  All-gather them over the ranks (any transport). */
femgpu_status femgpu_halo_export(femgpu_halo* h, void* buf, size_t cap, size_t* len);
/* The all-gathered exports of ranks 0..world-1, `stride` bytes apart: maps the peers' buffers. */
femgpu_status femgpu_halo_import(femgpu_halo* h, const void* all, size_t stride);
/* One distributed action into y_dev (NULL = the instance output): pull ghost inputs, boundary
 * cells, push (side stream), interior cells, completion of the owned shared rows.  Asynchronous. */
femgpu_status femgpu_halo_action(femgpu_halo* h, const femgpu_schedule* s, double* y_dev, void* stream);
/* Exactly `steps` distributed actions on the instance stream, CUDA events, device sync on both
 * sides: *seconds = this rank's elapsed time (the caller takes the max over ranks). */
femgpu_status femgpu_halo_time_steps(femgpu_halo* h, const femgpu_schedule* s, int32_t steps, double* seconds);
/* Synchronizes `stream` (NULL = instance stream) and reports a peer that never reached the
 * exchange (bounded waits: FEMGPU_HALO_TIMEOUT_MS, default 20000) as FEMGPU_E_CUDA. */
femgpu_status femgpu_halo_check(femgpu_halo* h, void* stream);
/* Distributed CG on the devices over the exchange (call on every rank, same arguments): vectors in the
 * rank's local test numbering (owned rows + ghosts; trial space 0 numbered like it), dots over owned
 * rows all-reduced GPU to GPU through the peers' flag words (values summed in rank order), no host
 * round trip except the residual check every check_every iterations.  b_dev: the right-hand side on
 * owned rows; x_dev: initial guess in, solution out (owned rows meaningful).  Call femgpu_halo_check
 * afterwards: a rank that never arrives is reported, not waited for. */
femgpu_status femgpu_halo_cg(femgpu_halo* h, const femgpu_schedule* s, const double* b_dev, double* x_dev, double rtol,
                             int32_t maxiter, int32_t check_every, int32_t* iterations, double* rel_residual);

/* ---- instance / candidate files (femsched io.hpp, format_version 1) ------
 * The reference's versioned structured-text format (io.hpp:197-391): doubles with 17
 * significant digits, bit-exact round trip; femgpu_problem_save writes byte-identical text to
 * femsched::save_instance.  A loaded problem owns its arrays; *view stays valid until
 * femgpu_problem_free.  Schedule files follow save_candidate/load_candidate (io.hpp:407-460)
 * for kinds scpt/mlt; the B200 kinds are written as extension kinds ("b200_dmma"). */
typedef struct femgpu_owned_problem femgpu_owned_problem;
femgpu_status femgpu_problem_load(const char* path, femgpu_owned_problem** out, const femgpu_problem** view);
femgpu_status femgpu_problem_free(femgpu_owned_problem* p);
femgpu_status femgpu_problem_save(const femgpu_problem* p, const char* path);
femgpu_status femgpu_schedule_save(const femgpu_schedule* s, int32_t n_scalar, int32_t n_vector, const char* path);
femgpu_status femgpu_schedule_load(const char* path, femgpu_schedule* s);

/* ---- fused multi-operator actions (csrc/fuse.cpp) ----
 * n problems on the same cells, geometry (coordinate map + coordinates) and quadrature weights
 * become one problem whose output is [y_0; y_1; ...; y_{n-1}] (offsets[p] .. offsets[p+1], n+1
 * entries, may be NULL).  Trial spaces with the same map, global count and input are merged (their
 * derivative terms united, identical terms shared): shared trial values are gathered and evaluated
 * once per cell.  The test space is the disjoint union with a block-diagonal Psi; kernels skip the
 * Psi entries that are zero at every quadrature point.  Create an instance on *view like any
 * problem; free with femgpu_problem_free.  Differing meshes, weights or dimensions are
 * FEMGPU_E_INVALID. */
femgpu_status femgpu_problem_fuse(const femgpu_problem* const* problems, int32_t n, femgpu_owned_problem** out,
                                  const femgpu_problem** view, int64_t* offsets);

/* ---- locality-restoring renumbering of a general mesh (csrc/reorder.cpp) -------------------
 * Cells sorted by the Morton code of their centroid; every global index space renumbered in
 * first-touch order (spaces with equal global counts share a numbering; a node*dim+comp vector test
 * space follows its trial space).  *view is the same problem in the new numbering (inputs and
 * coordinates permuted).  Optional outputs, new -> old: cell_perm[cell_count],
 * output_perm[output_size] (y_new[r] = y_old[output_perm[r]]), scalar_input_perms[i][global_count]
 * and vector_input_perms[i][global_count] (node level) for later inputs.  Free with
 * femgpu_problem_free. */
femgpu_status femgpu_problem_reorder(const femgpu_problem* p, femgpu_owned_problem** out, const femgpu_problem** view,
                                     int32_t* cell_perm, int32_t* output_perm, int32_t* const* scalar_input_perms,
                                     int32_t* const* vector_input_perms);

/* ---- structured meshes (synthetic unit square / unit cube) -------------
 * Unit square: n x n squares, 2 triangles each; unit cube: n^3 cubes, 6 Kuhn
 * tetrahedra each.  P_degree nodes live on the degree-refined lattice and the
 * global DOF number is the lattice index, so shared edges and faces agree.
 * Cells are ordered brick-major (brick x brick [x brick] squares/cubes) so a
 * run of consecutive cells is spatially compact.  Vertex v has lattice index
 * and coordinates lattice/n.  Node ordering per cell: the dim+1 vertices
 * first, then the remaining barycentric multi-indices in lexicographic order. */
femgpu_status femgpu_mesh_counts(int32_t dim, int32_t n, int32_t degree, int64_t* cells,
                                 int64_t* nodes, int64_t* vertices, int32_t* nodes_per_cell);
femgpu_status femgpu_mesh_build(int32_t dim, int32_t n, int32_t degree, int32_t brick,
                                int32_t* node_map, int32_t* vertex_map, double* coords);
/* The rows [cell_begin, cell_end) of femgpu_mesh_build's node and vertex maps (same global
 * numbering), written from row 0 of node_map / vertex_map; coords (may be NULL) as in
 * femgpu_mesh_build.  One rank of a cell-partitioned run builds only its own slab with it. */
femgpu_status femgpu_mesh_build_range(int32_t dim, int32_t n, int32_t degree, int32_t brick, int64_t cell_begin,
                                      int64_t cell_end, int32_t* node_map, int32_t* vertex_map, double* coords);
/* Greedy cell colouring: no two cells of one colour share an entry of map.
 * colors[cell] in [0, *n_colors). Deterministic (cells in ascending order,
 * smallest free colour). */
femgpu_status femgpu_color_cells(const int32_t* map, int32_t cells, int32_t entries,
                                 int32_t global_count, int32_t* colors, int32_t* n_colors);

#ifdef __cplusplus
}
#endif

#endif /* FEMGPU_H */

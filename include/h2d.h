/*
 * h2d.h — C-ABI drop-in boundary of the B200 Lagrange + DirectCF step.
 *
 * The reference (`/root/reference/proj`, "hydro2d") exposes its solver as a
 * C++ value API in proj/include/hydro/ (*.hpp) and has no C-ABI or device path.
 * This header is the flat boundary a foreign caller (ctypes, cgo, JNI, the
 * C++ `hydro::` shim in include/hydro/) binds.  Every entry point names the
 * reference interface it replaces (file:line, relative to proj/).
 *
 * Layout contract (identical to the reference `Field<T>`, field.hpp:15-44):
 *   - cell fields hold (nx + 2*H2D_GHOST) * (ny + 2*H2D_GHOST) doubles,
 *     row-major in j, contiguous in i, element (i,j) at
 *     (j + H2D_GHOST) * (nx + 2*H2D_GHOST) + (i + H2D_GHOST);
 *   - node fields are the same with nx+1 / ny+1;
 *   - Vec2 fields (normals, velocities) are interleaved {x, y} pairs, exactly
 *     the bytes of std::vector<hydro::Vec2>.
 * So `State::m[a].raw().data()` can be passed as-is.
 *
 * Three libraries implement this ABI with different symbol prefixes:
 *   h2d_   libh2d.so            the product (CUDA sm_100a, device resident)
 *   h2do_  oracle/libh2d_oracle.so  plain-C restatement (test checker only)
 *   h2dr_  oracle/_ref/libh2d_ref.so reference library itself (test checker)
 * Only the h2d_ prefix is declared here; the oracle libraries export the same
 * signatures under their prefix.
 *
 * Errors: every call returns 0 on success or an H2D_ERR_* kind; details
 * (reference exception class, located cell, step, message) are fetched with
 * h2d_last_error.  Kinds mirror proj/include/hydro/errors.hpp:11-34.
 */
#ifndef H2D_H
#define H2D_H

#ifdef __cplusplus
extern "C" {
#endif

#define H2D_ABI_VERSION 3
/* materials per State: the reference's kMaxMat (state.hpp:13) is 2; the third
 * slot is the N-material extension of configuration 5,
 * no reference counterpart. Contexts with nmat <= 2 are the reference. */
#define H2D_MAX_MAT 3
#define H2D_GHOST 2   /* reference kGhost, field.hpp:11 */

/* BoundaryKind, mesh.hpp:8 */
enum { H2D_BC_PERIODIC = 0, H2D_BC_WALL = 1 };
/* EosModel::Kind, eos.hpp:12 */
enum { H2D_EOS_PERFECT = 0, H2D_EOS_STIFFENED = 1 };
/* CornerScheme, reconstruct.hpp:7 (same ordinal order) */
enum {
    H2D_CORNER_UPWIND = 0,
    H2D_CORNER_AVGMIN = 1,
    H2D_CORNER_LINEARXY = 2,
    H2D_CORNER_LINEARDIAG = 3,
    H2D_CORNER_MULTID = 4
};
/* RemapKind, remap.hpp:9 */
enum { H2D_REMAP_AD = 0, H2D_REMAP_DIRECT = 1, H2D_REMAP_DIRECTCF = 2 };

/* Error kinds: 0 = ok; 1..6 = the reference exception classes; >= 100 API. */
enum {
    H2D_OK = 0,
    H2D_ERR_SIM = 1,          /* SimError (errors.hpp:11) */
    H2D_ERR_TANGLED = 2,      /* TangledCellError (errors.hpp:30) */
    H2D_ERR_UNPHYSICAL = 3,   /* UnphysicalStateError (errors.hpp:31) */
    H2D_ERR_NEGMASS = 4,      /* NegativeMassError (errors.hpp:32) */
    H2D_ERR_CFL = 5,          /* CflViolationError (errors.hpp:33) */
    H2D_ERR_ISOLATED = 6,     /* IsolatedMixedCellError (errors.hpp:34) */
    H2D_ERR_INVALID = 100,    /* bad argument / unsupported option */
    H2D_ERR_DEVICE = 101,     /* CUDA runtime failure */
    H2D_ERR_NOMEM = 102
};

/* Mesh (mesh.hpp:13-29). */
typedef struct {
    int nx, ny;
    double dx, dy, x0, y0;
    int bc_x, bc_y; /* H2D_BC_* */
} h2d_mesh;

/* EosModel (eos.hpp:11-19). */
typedef struct {
    int kind; /* H2D_EOS_* */
    double gamma;
    double pi;
} h2d_eos;

/* MaterialSet (state.hpp:29-32) + PseudoViscosityParams (lagrange.hpp:7-10)
 * + ReconConfig (reconstruct.hpp:9-13): everything fixed for a run. */
typedef struct {
    h2d_mesh mesh;
    int nmat;
    h2d_eos eos[H2D_MAX_MAT];
    double pv_a1, pv_a2;
    int face_order;        /* ReconConfig::face_order */
    int corner;            /* H2D_CORNER_* */
    int interface_degrade; /* ReconConfig::interface_degrade */
    int options;           /* H2D_OPT_* bits, 0 = the reference scheme */
} h2d_config;

/* Options with no reference counterpart (default off; every parity claim is
 * for options == 0):
 * H2D_OPT_SLIVER_ENERGY — configuration 5's sliver-energy safeguard: after
 *   finalize_cells' sliver pass (remap.cpp:194-226), a material of a cell with
 *   positive mass and NEGATIVE specific internal energy (a remapped sliver;
 *   the reference floors energies in the Lagrangian phase only,
 *   lagrange.cpp:119-124, and then throws UnphysicalStateError from
 *   sound_speed, eos.hpp:31-32) hands its m*e to the cell's largest-mass other
 *   material when that sum stays positive (total m*e conserved), else drops
 *   it; its own e becomes 0 (P = 0, c = 0). */
enum { H2D_OPT_SLIVER_ENERGY = 1 };

/* Host view of a reference State (state.hpp:39-63).  Any derived pointer
 * (vol, m_mix, e_mix, rho_mix, p_mix) may be NULL on upload, in which case
 * the device recomputes it with sync_derived semantics (state.cpp:120-143). */
typedef struct {
    double* m[H2D_MAX_MAT];
    double* e[H2D_MAX_MAT];
    double* k[H2D_MAX_MAT];
    double* vol;
    double* m_mix;
    double* e_mix;
    double* rho_mix;
    double* p_mix;
    double* iface_normal; /* cell Vec2, interleaved */
    double* u;            /* node Vec2, interleaved */
    int step;
    double time;
} h2d_state;

/* Host view of a LagrangeResult (lagrange.hpp:38-45). */
typedef struct {
    double* u_half; /* node Vec2 */
    double* u_lag;  /* node Vec2 */
    double* e_lag[H2D_MAX_MAT];
    double* vol_lag;
    double* q;
    int floor_count;
} h2d_lagrange;

/* RemapDiag (remap.hpp:42-46). */
typedef struct {
    double max_k_violation;
    int k_clip_count;
    int mass_fix_count;
} h2d_remap_diag;

/* Located exception record (errors.hpp:11-28). `what` is the reference's
 * formatted what() string of the innermost throw; `in_step` is 1 when the
 * error was raised inside lagrange_step/remap_step, where run() re-throws it
 * with " [<case> step <n>]" appended (harness.cpp:404-407). */
typedef struct {
    int kind;
    int i, j, step;
    int in_step;
    char what[256];
} h2d_error;

/* StepDiag (harness.hpp:66-72) with its Totals (state.hpp:93-98): the record
 * run() appends to RunReport::series after every step (make_diag,
 * harness.cpp:360-376, called at :410). */
typedef struct {
    int step;
    double t, dt;
    double mass, mass_mat[H2D_MAX_MAT], momentum_x, momentum_y, internal_energy;
    double min_rho, max_rho, min_p, max_p;
} h2d_step_diag;

/* Device-resident run loop (harness.cpp:380-412, non-kinematic branch). */
typedef struct {
    int max_steps;    /* 0 = until t_end (compares the state's absolute step) */
    double t_end;
    double cfl;
    int remap_kind;   /* H2D_REMAP_*: all three on single-domain contexts (AD with at
                       * most 2 materials); block contexts run DirectCF and AD
                       * through h2d_blocks_run / h2d_blocks_run_kind */
    double* dt_log;   /* optional host array receiving each step's dt */
    int dt_log_cap;
    /* outputs */
    int steps_done;
    int floor_count;  /* sum of LagrangeResult::floor_count */
    h2d_remap_diag diag;
    /* optional host array receiving one StepDiag per step done (make_diag of
     * the new State, harness.cpp:410). The product reduces it on the device
     * inside the step: step / t / dt and the extrema are the reference's bits;
     * the sums are a fixed-order tree instead of the reference's serial loop,
     * so each is within n * 2^-53 * sum|term| of it (n terms). */
    h2d_step_diag* series;
    int series_cap;
} h2d_run_args;

/* One block of a 2D domain decomposition (no reference counterpart: the
 * reference is serial): owned cells [oi, oi+bnx) x [oj, oj+bny)
 * of the global mesh plus a halo of `halo` (>= 8) cells stored around them. */
typedef struct {
    int oi, oj, bnx, bny, halo;
} h2d_block;

typedef struct h2d_ctx h2d_ctx;

/* Library identity: returns H2D_ABI_VERSION. */
int h2d_abi_version(void);

/* Mesh + MaterialSet + params (state.hpp:65 make_state's inputs). device<0
 * selects the current device. Validates like Mesh::Mesh (mesh.hpp:26-29). */
int h2d_create(const h2d_config* cfg, int device, h2d_ctx** out);
void h2d_destroy(h2d_ctx* ctx);

/* Replace the context's State (all ghost layers included). */
int h2d_upload_state(h2d_ctx* ctx, const h2d_state* s);
/* Read the State back into the reference layout; NULL pointers are skipped. */
int h2d_download_state(h2d_ctx* ctx, h2d_state* s);

/* Init helpers on the context's State, as init_case calls them
 * (harness.cpp:286-288): void fill_ghosts(State&) (state.hpp:87,
 * state.cpp:110-118); void sync_derived(State&, const MaterialSet&)
 * (state.hpp:91, state.cpp:120-143); void update_interface_normals(State&)
 * (remap.hpp:64, remap.cpp:1093-1096). */
int h2d_fill_ghosts(h2d_ctx* ctx);
int h2d_sync_derived(h2d_ctx* ctx);
int h2d_update_interface_normals(h2d_ctx* ctx);

/* double cfl_dt(const State&, const MaterialSet&, double cfl)
 * (harness.hpp:64, harness.cpp:293-313). */
int h2d_cfl_dt(h2d_ctx* ctx, double cfl, double* dt_out);

/* LagrangeResult lagrange_step(State, MaterialSet, dt, PseudoViscosityParams)
 * (lagrange.hpp:56-59). The result stays on the device for h2d_remap_step;
 * `out` (nullable) receives a copy. */
int h2d_lagrange_step(h2d_ctx* ctx, double dt, h2d_lagrange* out);

/* Install an externally built LagrangeResult (e.g. the imposed-velocity
 * `kinematic()` of test_remap.cpp:46-54). NULL e_lag/vol_lag/q entries are
 * zero-filled. */
int h2d_set_lagrange(h2d_ctx* ctx, const h2d_lagrange* lag);

/* State remap_step(State, MaterialSet, LagrangeResult, dt, RemapKind,
 * ReconConfig, x_first, remap_velocity, RemapDiag*) (remap.hpp:51-53).
 * Replaces the device State by the remapped one (step+1, time+dt).
 * `diag` (nullable) is accumulated like the reference's RemapDiag.
 * remap_kind: H2D_REMAP_DIRECTCF (cf_pass, remap.cpp:734-1073) or
 * H2D_REMAP_AD (two directional passes, remap.cpp:469-589, X first when
 * x_first != 0; at most 2 materials) or H2D_REMAP_DIRECT (direct_pass,
 * remap.cpp:593-724) on single-domain contexts; block contexts run DirectCF
 * only and return H2D_ERR_INVALID for the others. */
int h2d_remap_step(h2d_ctx* ctx, double dt, int remap_kind, int x_first,
                   int remap_velocity, h2d_remap_diag* diag);

/* RunReport run(...) hot loop without the catalogue/init (harness.cpp:390-412):
 * cfl_dt -> min(t_end - t) -> lagrange_step -> remap_step -> nan_scan. */
int h2d_run(h2d_ctx* ctx, h2d_run_args* args);

/* Totals compute_totals(const State&) (state.hpp:100, state.cpp:145-160);
 * out = {mass, mass_mat0, mass_mat1, momentum.x, momentum.y, internal_energy}. */
int h2d_totals(h2d_ctx* ctx, double out[6]);

/* StepDiag make_diag(const State&, double dt) (harness.cpp:360-376) of the
 * context's current State, e.g. RunReport::series[0] = make_diag(s, 0.0)
 * (harness.cpp:385); sums in the reference's serial order. */
int h2d_step_diag_now(h2d_ctx* ctx, double dt, h2d_step_diag* out);

/* ---- field readback formats and checkpoints ------- */
/* DumpFormat, io.hpp:9 */
enum { H2D_DUMP_CSV = 0, H2D_DUMP_VTK = 1 };

/* void write_fields(const State&, const std::string& path, DumpFormat)
 * (io.hpp:17, io.cpp:72-83): CSV or legacy-VTK cell dump of the context's
 * resident State, byte-identical to the reference's; H2D_ERR_SIM when the
 * file cannot be written (the reference's SimError). Single-domain contexts. */
int h2d_write_fields(h2d_ctx* ctx, const char* path, int fmt);
/* The same formatter on a host State view (no device needed). */
int h2d_write_fields_host(const h2d_config* cfg, const h2d_state* s, const char* path, int fmt);
/* void append_diag_line(std::ostream&, step, t, dt, Totals, extrema)
 * (io.hpp:21-22, io.cpp:85-92) of one StepDiag into buf (NUL-terminated). */
int h2d_diag_line(const h2d_step_diag* d, char* buf, int cap);
/* Binary checkpoint of the persistent State (no reference counterpart):
 * header (mesh, material count, step, time) + every Field in the reference
 * layout; a load into a context of another mesh returns H2D_ERR_INVALID.
 * Restarting from a checkpoint continues bit-exactly. */
int h2d_save_state(h2d_ctx* ctx, const char* path);
int h2d_load_state(h2d_ctx* ctx, const char* path);
int h2d_save_state_host(const h2d_config* cfg, const h2d_state* s, const char* path);
int h2d_load_state_host(const h2d_config* cfg, h2d_state* s, const char* path);

/* ---- 2D block decomposition (no reference counterpart) ----
 * A block context owns [oi, oi+bnx) x [oj, oj+bny) of the global mesh plus a
 * halo (>= 8 cells). One run-loop step computes the whole step on the window
 * with redundant halo work, so ONE halo exchange of the State (8 neighbours,
 * corners included) and one all-reduce of the next step's wave speed per step
 * keep every owned value bit-identical to the single-domain run. Walls only. */
int h2d_create_block(const h2d_config* cfg, const h2d_block* blk, int device, h2d_ctx** out);
/* window upload / owned-region download in the GLOBAL reference layout */
int h2d_block_upload(h2d_ctx* ctx, const h2d_state* global_state);
int h2d_block_download(h2d_ctx* ctx, h2d_state* global_state);
/* The block's initial State from a painted WINDOW of the global mesh (each
 * rank paints only its own window; no global host State): the arrays of `win`
 * hold the cells [wi0, wi0 + wnx) x [wj0, wj0 + wny) (wnx * wny doubles,
 * row-major, no ghost layers) and the nodes [wi0, wi0 + wnx] x [wj0, wj0 + wny]
 * ((wnx + 1) (wny + 1) Vec2); m, e, k per material and u are read. The window
 * should cover the block's storage window clipped to the mesh. Then the
 * init_case tail on the device (fill_ghosts at the global walls,
 * sync_derived, update_interface_normals; harness.cpp:286-288); the first
 * exchange of h2d_blocks_run makes the halo exact. */
int h2d_block_init_window(h2d_ctx* ctx, const h2d_state* win, int wi0, int wj0, int wnx, int wny, int step,
                          double time);
/* run control: begin (computes the owned wave speed of the initial State),
 * one graph-launched step, the scalars to combine across blocks
 * {next wave-speed max bits (MAX), next cfl error key (MIN), error key (MIN),
 * done}, writing the combined values back, and undoing a commit when another
 * block failed earlier in the same step */
int h2d_block_begin(h2d_ctx* ctx, int max_steps, double t_end, double cfl);
int h2d_block_step(h2d_ctx* ctx);
int h2d_block_scalars(h2d_ctx* ctx, unsigned long long out[4]);
int h2d_block_set(h2d_ctx* ctx, const unsigned long long in[3]);
int h2d_block_rollback(h2d_ctx* ctx);
/* halo exchange with the neighbour at (dx, dy) in {-1,0,1}^2: buffer sizes,
 * pack of the owned data it needs, unpack of the data it sent (device ptrs) */
long long h2d_halo_bytes(h2d_ctx* ctx, int dx, int dy, int pack);
int h2d_halo_pack(h2d_ctx* ctx, int dx, int dy, void* dev_buf);
int h2d_halo_unpack(h2d_ctx* ctx, int dx, int dy, const void* dev_buf);
/* counters, dt log and first error of the block's run (like h2d_run) */
int h2d_block_result(h2d_ctx* ctx, h2d_run_args* args);

/* The block run loop with the data plane in the library: every step of
 * every block, the one max all-reduce of {next wave speed, first cfl error,
 * first error, done} and the one halo exchange (8 neighbours, corners
 * included) are enqueued on the device; the exchange overlaps the next step's
 * Lagrange tiles on owned data; the host polls every 16 steps. A transport
 * is either NCCL (one block per process: rank = by * px + bx of a px x py
 * grid, the communicator created here from an id of h2d_nccl_unique_id,
 * libnccl.so.2 opened at run time) or in-process (all px * py blocks of the
 * decomposition in this process, one device, rank order). Counters, dt log
 * and errors per block come from h2d_block_result afterwards. */
typedef struct h2d_comm h2d_comm;
int h2d_nccl_unique_id(unsigned char id[128]);
int h2d_comm_nccl(const unsigned char id[128], int px, int py, int rank, h2d_ctx* block, h2d_comm** out);
int h2d_comm_local(h2d_ctx* const* blocks, int px, int py, h2d_comm** out);
void h2d_comm_destroy(h2d_comm* comm);
/* device_ms (nullable): CUDA-event time from the first step's start to the
 * last step's exchange (the slowest block of this process) */
int h2d_blocks_run(h2d_comm* comm, int max_steps, double t_end, double cfl, int* steps_done, float* device_ms);
/* The same loop with the remap engine chosen: H2D_REMAP_DIRECTCF (as
 * h2d_blocks_run: ONE halo exchange + one all-reduce per step) or
 * H2D_REMAP_AD (run(kind = AD), harness.cpp:398-403 / remap.cpp:1110-1115, at
 * most 2 materials): the split remap needs its neighbours' pass-0 Work
 * (remap.cpp:87-97) before pass 1, i.e. a SECOND halo exchange per step
 * between the two directional passes (PAPER.md:544 against :595). Owned
 * values are bit-identical to the single-domain AD run. */
int h2d_blocks_run_kind(h2d_comm* comm, int remap_kind, int max_steps, double t_end, double cfl, int* steps_done,
                        float* device_ms);

/* Stream trace of the next h2d_blocks_run* call (evidence of the overlap; no
 * reference counterpart): CUDA timing events at nine points of each of the
 * first `steps` steps and each block of this process. h2d_comm_trace_read
 * returns the number of floats recorded (steps x blocks x 9, step-major) and
 * copies up to cap of them: milliseconds from the block's first step start of
 * {owned Lagrange tiles start, end, edge tiles end (after the halo wait), AD
 * mid exchange start, end, rest of the step end, all-reduce start, State halo
 * exchange start, end}; -1 = point not reached (e.g. the AD points of a
 * DirectCF run). The State exchange recorded with step s is the one enqueued
 * after step s, which overlaps step s + 1's owned tiles. */
int h2d_comm_trace(h2d_comm* comm, int steps);
int h2d_comm_trace_read(h2d_comm* comm, float* out, int cap);

/* ---- benchmark support (no reference counterpart) ---------------------- */
/* Kernels launched by this library in the calling process so far. */
long long h2d_launch_count(void);
/* One run-loop step (as h2d_run with max_steps = state step + 1) bracketed by
 * CUDA events on the context's stream. ms[6] = the whole step; with
 * phases = 1 (plain launches, events between kernels) also ms[0] step start
 * (dt), ms[1] the fused Lagrange kernel, ms[2] the remap flux tile kernel,
 * ms[3] slivers + Work ghosts, ms[4] dual-mesh momentum, ms[5] the derived
 * fields / normals / NaN-scan kernel, ms[7] the ghost-layer launches and the
 * commit; phases = 0 replays the production CUDA graph (only ms[6] set).
 * remap_kind = H2D_REMAP_AD times the AD step (its two passes and the post
 * kernels land in ms[2]). */
int h2d_step_timed(h2d_ctx* ctx, double cfl, double t_end, int phases, int remap_kind, float ms[8]);
/* Write `bytes` of scratch on the context's stream (evicts L2 between timed
 * steps) and wait for it. */
int h2d_flush_l2(h2d_ctx* ctx, long long bytes);

/* ---- the reference's sub-step entry points (value API of lagrange.hpp /
 * remap.hpp that the reference's own unit tests call) -------------------- */

/* HalfStepState (lagrange.hpp:14-24). */
typedef struct {
    double* x_half;  /* node Vec2 */
    double* u_half;  /* node Vec2 */
    double* vol_half;
    double* e_half[H2D_MAX_MAT];
    double* p_half[H2D_MAX_MAT];
    double* p_mix_half;
    double* q;
    int floor_count;
} h2d_half;

/* HalfStepState predict(State, MaterialSet, dt, PseudoViscosityParams)
 * (lagrange.hpp:48-49, lagrange.cpp:79-144) of the context's State. */
int h2d_predict(h2d_ctx* ctx, double dt, h2d_half* out);
/* LagrangeResult correct(State, MaterialSet, HalfStepState, dt)
 * (lagrange.hpp:50-51, lagrange.cpp:146-196) from a caller's HalfStepState
 * (u_half, p_half, q with ghosts); the result stays on the device for
 * h2d_remap_step and `out` (nullable) receives a copy. floor_count adds the
 * half state's count like the reference. */
int h2d_correct(h2d_ctx* ctx, double dt, const h2d_half* in, h2d_lagrange* out);
/* State remap_single_axis(State, MaterialSet, LagrangeResult, dt, Axis,
 * ReconConfig, remap_velocity, RemapDiag*) (remap.hpp:55-57,
 * remap.cpp:1098-1104): one AD directional pass; single-domain, <= 2
 * materials. */
int h2d_remap_single_axis(h2d_ctx* ctx, double dt, int axis_x, int remap_velocity, h2d_remap_diag* diag);

/* The reference's scalar kernels on the device: n records, record r reads
 * in[r * H2D_SC_IN ...] and writes out[r * H2D_SC_OUT ...]; flags[r]
 * (nullable) is set where the reference call throws (the exception named per
 * op). Runs on the current device; H2D_ERR_DEVICE without one. */
#define H2D_SC_IN 48
#define H2D_SC_OUT 8
enum {
    H2D_SC_VAN_LEER = 0,          /* r -> phi                           reconstruct.cpp:10-14 */
    H2D_SC_LIMITED_GRADIENT = 1,  /* am ac ap xm xc xp -> g; SimError   reconstruct.cpp:16-24 */
    H2D_SC_FACE_VALUE = 2,        /* order a0 a1 a2 x0 x1 x2 sgn lw ufdt -> v; SimError  :26-31 */
    H2D_SC_CORNER_VALUE = 3,      /* scheme a[9] xlx[9] xly[9] (index [(di+1)*3+dj+1]) dxp dyp lag_wx lag_wy
                                   * sgn_fx u_fx_dt sgn_fy u_fy_dt eval_rel.x eval_rel.y dx dy -> v; SimError
                                   *                                    reconstruct.cpp:116-152 */
    H2D_SC_MULTID_PLANE = 4,      /* a[9] xlx[9] xly[9] dx dy -> a0 cx cy grad_raw.x .y grad.x .y; SimError
                                   *                                    reconstruct.cpp:74-107 */
    H2D_SC_CLIPPED_FRACTION = 5,  /* w h n.x n.y d -> f                 vof.cpp:28-45 */
    H2D_SC_PLACE_INTERFACE = 6,   /* frac n.x n.y lo.x lo.y hi.x hi.y -> d   vof.cpp:47-73 */
    H2D_SC_YOUNGS_NORMAL = 7,     /* k1[9] ([(di+1)*3+dj+1]) dx dy -> n.x n.y; IsolatedMixedCellError vof.cpp:10-22 */
    H2D_SC_CELL_VOLUME = 8,       /* p00 p10 p11 p01 (x, y) -> vol; TangledCellError  state.cpp:25-32 */
    H2D_SC_CF_CORNER_FLUX = 9,    /* u.x u.y dt -> dvol sx sy           remap.cpp:16-25 */
    H2D_SC_CF_FACE_FLUX_X = 10,   /* ym yp dm.x dm.y dp.x dp.y -> dvol wlo whi  remap.cpp:27-47 */
    H2D_SC_CF_FACE_FLUX_Y = 11,   /* xm xp dm.x dm.y dp.x dp.y -> dvol wlo whi  remap.cpp:49-51 */
    H2D_SC_PSEUDO_VISCOSITY = 12, /* rho c div_u a1 a2 L -> q           lagrange.cpp:7-12 */
    H2D_SC_DIV_U_CELL = 13,       /* u00 u10 u01 u11 (x, y) dx dy -> div lagrange.cpp:14-20 */
    H2D_SC_GRAD_PQ_NODE = 14,     /* p[4] q[4] at (i-1,j-1) (i,j-1) (i-1,j) (i,j), dx dy -> g.x g.y  lagrange.cpp:22-30 */
    H2D_SC_AD_FACE_FLUX = 15      /* u0 u1 dt width cv -> f; CflViolationError  remap.cpp:53-73 (one face) */
};
int h2d_scalar_eval(int op, int n, const double* in, double* out, int* flags);

/* Last error recorded on this context (kind H2D_OK if none). */
int h2d_last_error(h2d_ctx* ctx, h2d_error* err);

#ifdef __cplusplus
}
#endif
#endif /* H2D_H */

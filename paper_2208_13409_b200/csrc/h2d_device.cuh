// h2d_device.cuh — device-side layout, control block and the fp64 scalar
// kernels of the Lagrange + DirectCF step (sm_100a).
//
// Bit-exactness contract: compiled with -fmad=false,
// IEEE div/sqrt; every expression keeps the reference association, and
// std::max/std::min semantics are kept by rmax/rmin (NaN and signed-zero
// behaviour of `a < b ? b : a`).  Cited lines are in /root/reference/proj.
#pragma once
#include <cstdint>
#include <cuda.h>  // CUtensorMap (the type only; maps are encoded through the runtime's driver entry point)
#include <math_constants.h>
#include <cfloat>
#ifdef H2D_CHECKED
// checked build (tools/variants.py build checked -DH2D_CHECKED): every plane
// index, shared-memory tile index and sliver-list slot is bounds-checked on
// the device (assert -> cudaErrorAssert); the substitute for compute-sanitizer
// memcheck, which this pool does not run
#include <cassert>
#define H2D_CHECK(x) assert(x)
#else
#define H2D_CHECK(x) ((void)0)
#endif

#define H2D_DEV __device__ __forceinline__

namespace h2d {

constexpr int G = 2;  // ghost layers of every device field (== kGhost, field.hpp:11)
constexpr double kPureTol = 1e-10;   // state.hpp:17
constexpr double kThermoTol = 1e-6;  // state.hpp:22
constexpr double kCflFrac = 0.9;     // remap.cpp:13
constexpr uint64_t kNoErr = 0xFFFFFFFFFFFFFFFFull;

// Error phases in the reference's program order (cfl_dt -> lagrange_step ->
// remap_step -> nan_scan).  The first error of a step is the minimum key
// (phase, outer loop index, inner loop index, sub-index) over all threads.
enum Phase : uint32_t {
    PH_CFL_UNPHYS = 1,    // sound_speed in cfl_dt            (harness.cpp:303, eos.hpp:32)
    PH_CFL_WAVE = 2,      // non-finite wave speed            (harness.cpp:311)
    PH_Q_UNPHYS = 3,      // sound_speed in compute_q         (lagrange.cpp:48-59,63-77)
    PH_PRED_TANGLED = 4,  // predict quad volume              (lagrange.cpp:44)
    PH_CORR_TANGLED = 5,  // correct quad volume              (lagrange.cpp:44)
    PH_CFL_XFACE = 6,     // remap.cpp:751-752
    PH_CFL_YFACE = 7,     // remap.cpp:759-760
    PH_CFL_CORNER = 8,    // remap.cpp:765-766
    PH_COLLAPSED = 9,     // remap.cpp:788
    PH_GRAD_XFACE = 10,   // limited_gradient_1d throw        (reconstruct.cpp:18)
    PH_GRAD_YFACE = 11,
    PH_GRAD_CORNER = 12,
    PH_NEGMASS = 13,      // finalize_cells                   (remap.cpp:186,190)
    PH_GRAD_DUALX = 14,
    PH_GRAD_DUALY = 15,
    PH_GRAD_DUALC = 16,
    PH_NODAL_MASS = 17,   // apply_dual_update                (remap.cpp:455)
    // AD split remap, per directional pass p = 0, 1 (phase + 5 p): the
    // collapsed-cell scan (remap.cpp:484), the face loop (CFL :532-535 and
    // the limiter throw, in face order), finalize_cells, the dual faces,
    // apply_dual_update
    PH_AD_COLLAPSED = 20,
    PH_AD_FACE = 21,
    PH_AD_NEGMASS = 22,
    PH_AD_GRAD_DUAL = 23,
    PH_AD_NODAL = 24,
    PH_NAN_CELL = 30,     // nan_scan                         (harness.cpp:347-358)
    PH_NAN_NODE = 31,
};

H2D_DEV uint64_t ekey(uint32_t ph, int outer, int inner, int sub) {
    return ((uint64_t)ph << 58) | ((uint64_t)(uint32_t)(outer + 16) << 33) |
           ((uint64_t)(uint32_t)(inner + 16) << 8) | (uint64_t)(uint32_t)sub;
}

// Device control block: the run loop's scalars live on the device so a whole
// sequence of steps is launched (or graph-replayed) without host syncs.
struct Ctl {
    double dt, time, t_end, cfl;
    int step, max_steps;
    int done;        // loop condition false -> every later kernel is a no-op
    int cur;         // parity of the committed State buffers
    int steps_done;
    int floor_count;  // sum of LagrangeResult::floor_count
    int k_clip_count, mass_fix_count;
    int step_floor;   // floor count of the step in flight
    int step_clip;
    int step_fix;
    int pad_;
    unsigned long long err_key;
    unsigned long long wmax_bits;       // max wave speed (non-negative doubles order as integers)
    unsigned long long kviol_bits;      // max_k_violation of the step in flight
    unsigned long long next_wmax_bits;  // wave-speed max of the state just produced (next step's cfl_dt)
    unsigned long long next_err_key;    // first cfl_dt error of that state
    double max_k_violation;
    double last_dt;
    int commit_time;  // 1: advance time/step at commit (run loop / remap_step)
    int use_cfl;      // 1: dt from the cfl reduction, 0: dt provided by the host
    int check_loop;   // 1: apply the run loop condition (harness.cpp:390-391)
    int pad2_;
    double* dt_log;   // device array, steps_done entries
    int dt_log_cap;
    // undo record of the last commit (block mode: a peer block failed first)
    double prev_time, prev_max_k_violation;
    int committed, counted;
    // per-step diagnostics of the run loop (make_diag, harness.cpp:360-376):
    // the values of the step in flight (k_post: cells, node update: momentum)
    // and the device log the commit appends one record of kDiagRec doubles to
    double dg[12];
    double* diag_log;
    int diag_log_cap;
    int pad3_;
    // sliver rounds (k_sliver_list / k_sliver_round / k_sliver_tail)
    int sl_n;                 // pending slivers listed this step
    int sl_on;                // the parallel rounds run (not periodic, list fits)
    int sl_cnt[8];            // slivers applied per round
};

// StepDiag + Totals (harness.hpp:66-72, state.hpp:93-98) slots of Ctl::dg
enum { DG_MASS, DG_IE, DG_MM0, DG_MM1, DG_MM2, DG_MINR, DG_MAXR, DG_MINP, DG_MAXP, DG_NCELL, DG_PX = DG_NCELL, DG_PY, DG_N };
// fold of each slot: 0 sum, 1 min, 2 max
H2D_DEV int dg_op(int k) { return (k == DG_MINR || k == DG_MINP) ? 1 : ((k == DG_MAXR || k == DG_MAXP) ? 2 : 0); }
// one log record: step, t, dt, then Ctl::dg[0 .. DG_N)
constexpr int kDiagRec = 3 + DG_N;
// Per-step diagnostics reduction: k_post and the node update store one
// fixed-shape block partial each (no fences or tickets inside those kernels),
// then k_diag_reduce folds them in index order (kDiagBlocks blocks, then the
// last one to arrive), so the result does not depend on block scheduling.
constexpr int kDiagBlocks = 148;
struct DiagScratch {
    double* part[2];  // [0] k_post blocks x DG_NCELL, [1] node blocks x 2
    double* lvl2;     // kDiagBlocks x DG_N
    unsigned* tick;
};

// Every thread of a kernel reads the control block: go through the read-only
// (L1-cached) path so the broadcast costs one L2 request per SM rather than
// one per warp on a single L2 line.  A value that is stale within a kernel is
// harmless (errors only need to stop later kernels).
H2D_DEV bool halted(const Ctl* c) {
    return __ldg(&c->done) != 0 || __ldg(&c->err_key) != kNoErr;
}
H2D_DEV double step_dt(const Ctl* c) { return __ldg(&c->dt); }
H2D_DEV void raise(Ctl* c, uint64_t key) { atomicMin(&c->err_key, (unsigned long long)key); }

// per-material slots of the State (H2D_MAX_MAT): 1-2 = the reference, 3 = config 5
constexpr int kMatSlots = 3;
// error sub-index of finalize's "non-positive cell mass" (after the material indices)
constexpr int kSubCellMass = 7;
// the Direct engine's face loop raises its CFL check and its gradient errors
// in one phase (loop order), sub 1 / 2 (DirectCF's gradient errors: sub 0)
constexpr int kSubDirectCfl = 1, kSubDirectGrad = 2;

// Half-open range of GLOBAL indices [i0, i1) x [j0, j1).
struct Rng {
    int i0, i1, j0, j1;
};

// Per-launch constants and field pointers.  Kernels work in GLOBAL mesh
// indices (the reference's i, j); a context stores the window of one block of
// the 2D decomposition: global (i, j) lives at j * P + i + off, where off maps
// the block origin (oi, oj) minus the halo H to the start of every plane.  A
// single-domain context is the block (0, 0, nx, ny) with H = G = 2, i.e. the
// reference Field layout.
// TMA descriptors of the planes the remap tile stages (per State parity):
// u_half x / y (node boxes), e_lag, m, k per material (cell boxes).
enum { TM_UHX, TM_UHY, TM_EL0, TM_M0 = TM_EL0 + 3, TM_K0 = TM_M0 + 3, TM_N = TM_K0 + 3 };
struct TmaSet {
    CUtensorMap t[TM_N];
};

struct Dev {
    int nx, ny, P, nmat, per_x, per_y;  // nx, ny: GLOBAL mesh size
    int oi, oj, H, off;                 // block origin, storage halo, index offset
    // compute ranges per phase (reference ranges, extended into the halo on
    // block sides that face a neighbour block; see capi.cu block_ranges)
    Rng r_lagc, r_lagn, r_lage, r_gath, r_dual, r_node, r_sync, r_nrm;
    Rng own_c, own_n;  // cells / nodes this block answers for (errors, counters, nan, cfl)
    Rng win_c, win_n;  // cells / nodes present in storage
    double dx, dy, x0, y0, cv, L;
    // exact reciprocals of dx, dy, dx*dy when they are powers of two (0
    // otherwise): x / dx == x * (1/dx) bit for bit in that case
    double rdx, rdy, rcv;
    // LinearDiag unit diagonal (reconstruct.cpp:135,139,144): dx/diag, dy/diag
    // with diag = sqrt(dx*dx + dy*dy), loop invariant, computed once (same bits)
    double dgx, dgy;
    int stiff[kMatSlots];
    double gamma[kMatSlots], pi[kMatSlots];
    double a1, a2;
    int face_order, corner_diag, degrade, remap_velocity;
    int corner;  // CornerScheme (H2D_CORNER_*): Upwind, AvgMin, LinearXY, LinearDiag, Multid
    int direct;  // 1: the Direct engine (faces only) instead of DirectCF
    int opt_energy;  // H2D_OPT_SLIVER_ENERGY (no reference counterpart, default off)

    // current (read) State
    const double *m[kMatSlots], *e[kMatSlots], *k[kMatSlots], *m_mix, *e_mix, *rho_mix, *p_mix, *nrx, *nry, *ux, *uy;
    double* vol;
    // next (written) State: also the remap's Work arrays (remap.cpp:88-98)
    double *nm[kMatSlots], *ne[kMatSlots], *nk[kMatSlots], *nvol, *nm_mix, *ne_mix, *nrho_mix, *np_mix, *nnrx, *nnry, *nux, *nuy;
    // LagrangeResult (lagrange.hpp:38-45)
    double *q, *pmh, *ph[kMatSlots], *uhx, *uhy, *ulx, *uly, *el[kMatSlots], *vol_lag;
    double *volh, *eh[kMatSlots];  // HalfStepState vol_half / e_half (h2d_predict only; null otherwise)
    // remap scratch (the tile kernel keeps its geometry in shared memory)
    double *me[kMatSlots], *mcell, *unrm;
    double *dmx, *dmy, *dmc;
    double *dfx_x, *dfx_y, *dfy_x, *dfy_y;  // dual-face momentum contributions
    double *dc_x[2], *dc_y[2];              // dual-corner contributions per pair
    double *slm[kMatSlots], *slme[kMatSlots];               // pending sliver mass / m*e (remap.cpp:149-153)
    uint8_t* sliver;                        // per-cell sliver flags (bit a)
    uint8_t* dflag[4];                      // active X / Y dual faces, dual-corner pairs
    // sliver index: bit (i - r_gath.i0) of word [(j - r_gath.j0) * nwx + (i - r_gath.i0) / 32]
    // in sl_segs, bit (j - r_gath.j0) % 32 of sl_rows[(j - r_gath.j0) / 32]; cleared as consumed
    unsigned *sl_rows, *sl_segs;
    unsigned* sl_segs2;  // the second pending-set bitmap of the sliver rounds (k_sliver_round)
    int* sl_list;  // the pending slivers in the reference order (k_sliver_list), sl_cap ints: [0, cap/4) the
                   // list, [cap/4, cap/2) the tail list, then one status byte per list entry
    int sl_cap;
    Ctl* ctl;
    const TmaSet* tma;  // host pointer: the launch passes *tma by value (__grid_constant__)
    // block mode: the fused Lagrange kernel runs in two launches around the
    // halo exchange: lag_sel 1 = only the tiles whose origin lies in
    // lag_inner (their stencil reads owned data only), 2 = the others, 0 = all
    Rng lag_inner;
    int lag_sel;
    int scan_nodes;     // run loop: the node update also runs nan_scan's node part (harness.cpp:353-357)
    int diag;           // run loop: reduce the step's make_diag values (k_post cells, node update momentum)
    DiagScratch dsc;    // diagnostics block partials ([0] k_post, [1] node update) + k_diag_reduce scratch
    int fsz;            // doubles per plane (P * R; the bound H2D_CHECKED tests plane indices against)
    // two / three materials: one class byte per remap tile (k_tile_class;
    // row-major over the remap grid, tq_nx x tq_ny): r < 3 = material r is
    // absent from the tile's staged region and the tile runs the kernel with
    // one slot fewer, 3 = the kernel of the context's material count. Null:
    // every tile runs the kernel of its NM.
    uint8_t* tcls;
    int tq_nx, tq_ny;
    // single domain: the classification masks (cell_cls_mask) ORed per k_post
    // block (32 x 8 cells over r_sync, pcls_nx blocks per row), written by
    // k_post for the State it produces; cls_post: this launch sequence is a
    // run-loop step, whose tile classes come from them (k_tile_class_post)
    uint16_t* pcls;
    int pcls_nx, cls_post;
};

// 32-bit plane offsets: P * R < 2^31 for every mesh up to 16384^2 (checked at
// context creation), which halves the index arithmetic of the stencils.
H2D_DEV int ix(const Dev& d, int i, int j) {
    const int q = j * d.P + i + d.off;
    H2D_CHECK(q >= 0 && q < d.fsz);
    return q;
}
H2D_DEV bool in(const Rng& r, int i, int j) { return i >= r.i0 && i < r.i1 && j >= r.j0 && j < r.j1; }

H2D_DEV double div_dx(const Dev& d, double x, double k) {  // x / (k * dx), k a power of two
    return d.rdx != 0.0 ? x * (d.rdx * (1.0 / k)) : x / (k * d.dx);
}
H2D_DEV double div_dy(const Dev& d, double x, double k) {
    return d.rdy != 0.0 ? x * (d.rdy * (1.0 / k)) : x / (k * d.dy);
}
H2D_DEV double div_cv(const Dev& d, double x) { return d.rcv != 0.0 ? x * d.rcv : x / d.cv; }
// phase density m / (k * cv) (lagrange.cpp:54,115,180, state.cpp:133,
// harness.cpp:301): a pure cell has k == 1 exactly, so k * cv == cv exactly
// and the divide is div_cv's exact power-of-two multiply
H2D_DEV double rho_of(const Dev& d, double m, double k) {
    return (k == 1.0 && d.rcv != 0.0) ? m * d.rcv : m / (k * d.cv);
}
H2D_DEV double rmax(double a, double b) { return (a < b) ? b : a; }  // std::max
H2D_DEV double rmin(double a, double b) { return (b < a) ? b : a; }  // std::min

// eos_pressure, eos.hpp:21-25
H2D_DEV double eos_p(const Dev& d, int a, double rho, double e) {
    double p = (d.gamma[a] - 1.0) * rho * e;
    if (d.stiff[a]) p -= d.pi[a];
    return p;
}
// sound_speed, eos.hpp:29-34; `bad` marks the reference's throw
H2D_DEV double sound(const Dev& d, int a, double rho, double p, bool& bad) {
    const double pi = d.stiff[a] ? d.pi[a] : 0.0;
    const double c2 = d.gamma[a] * (p + pi) / rho;
    if (!(c2 >= 0.0)) bad = true;
    return sqrt(c2);
}

// Programmatic dependent launch: every kernel first waits for the grids it
// depends on (a no-op when launched without the PDL attribute) and at once
// lets its dependents launch, so a dependent grid's CTAs are resident and
// waiting while this grid's last wave drains (hides launch gaps and tails in
// the run-loop graph).
H2D_DEV void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- per-step diagnostics ------------------------------------------------
// op 0: sum, 1: min (std::min), 2: max (std::max)
H2D_DEV double dg_comb(int op, double a, double b) { return op == 0 ? a + b : (op == 1 ? rmin(a, b) : rmax(a, b)); }
H2D_DEV double dg_ident(int op) { return op == 0 ? 0.0 : (op == 1 ? CUDART_INF : -CUDART_INF); }

// Fixed-shape block combine (every thread of the block must call it; the
// block is a whole number of warps): a shuffle tree per warp, then warp 0's
// thread 0 folds the warps in index order. Thread 0 holds the result.
template <int NV>
__device__ __forceinline__ void block_combine(double (&v)[NV], const int (&op)[NV], double* sh) {
    const int t = threadIdx.y * blockDim.x + threadIdx.x, nw = (blockDim.x * blockDim.y) >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] = dg_comb(op[k], v[k], __shfl_down_sync(0xffffffffu, v[k], o));
    if ((t & 31) == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) sh[(t >> 5) * NV + k] = v[k];
    __syncthreads();
    if (t == 0)
        for (int w = 1; w < nw; ++w)
#pragma unroll
            for (int k = 0; k < NV; ++k) v[k] = dg_comb(op[k], v[k], sh[w * NV + k]);
    __syncthreads();
}

// Warp partial of NV values, stored at part[(block * warps per block + warp) * NV]
// by lane 0 (all 32 lanes call it; no block barrier).
template <int NV>
__device__ __forceinline__ void warp_partial(double (&v)[NV], const int (&op)[NV], double* part) {
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] = dg_comb(op[k], v[k], __shfl_down_sync(0xffffffffu, v[k], o));
    const int t = threadIdx.y * blockDim.x + threadIdx.x;
    if ((t & 31) == 0) {
        const int nw = (blockDim.x * blockDim.y) >> 5;
        const size_t w = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * nw + (t >> 5);
#pragma unroll
        for (int k = 0; k < NV; ++k) part[w * NV + k] = v[k];
    }
}

// van_leer, reconstruct.cpp:10-14
H2D_DEV double van_leer(double r) {
    if (!(r > 0.0)) return 0.0;
    if (r > 1e300) return 2.0;
    return (r + fabs(r)) / (1.0 + r);
}
// limited_gradient_1d, reconstruct.cpp:16-24
H2D_DEV double lim_grad(double am, double ac, double ap, double xm, double xc, double xp, bool& bad) {
    const double hm = xc - xm, hp = xp - xc;
    if (hm <= 0.0 || hp <= 0.0) {
        bad = true;
        return 0.0;
    }
    const double nm = ac - am, np = ap - ac;
    // a zero difference over a positive (non-NaN) spacing gives dm == 0 (or
    // dp == 0) and the result 0: return before the divides, whose fast path
    // rejects zero operands (same result, no slow-path call)
    if ((nm == 0.0 && hm > 0.0) || (np == 0.0 && hp > 0.0)) return 0.0;
    const double dm = nm / hm;
    const double dp = np / hp;
    if (dm == 0.0 || dp == 0.0 || (dm > 0.0) != (dp > 0.0)) return 0.0;
    const double r = dm / dp;
    return 0.5 * (van_leer(r) * dp + van_leer(1.0 / r) * dm);
}
// face_value at order 2, reconstruct.cpp:26-31
H2D_DEV double face_value2(double a0, double a1, double a2, double x0, double x1, double x2, double sgn, double lw,
                           double ufdt, bool& bad) {
    const double g = lim_grad(a0, a1, a2, x0, x1, x2, bad);
    return a1 + 0.5 * g * (sgn * lw - ufdt);
}
// corner_value LinearDiag, reconstruct.cpp:134-148 (+ diag_gradient :38-42).
// a/xl are the 3x3 stencil [p][q] flattened as p*3+q.
H2D_DEV double corner_diag(const Dev& d, const double* a, const double* xlx, const double* xly, double dxp,
                           double dyp, double lwx, double lwy, bool& bad) {
    const double ac = a[4];
    const double sx = dxp >= 0.0 ? 1.0 : -1.0;
    if (dxp * dyp > 0.0) {
        const double vx = d.dgx, vy = d.dgy;
        const double sc = xlx[4] * vx + xly[4] * vy;
        const double gv = lim_grad(a[0], ac, a[8], xlx[0] * vx + xly[0] * vy, sc, xlx[8] * vx + xly[8] * vy, bad);
        const double ex = sx * lwx - dxp, ey = sx * lwy - dyp;
        return ac + 0.5 * gv * (ex * vx + ey * vy);
    }
    const double vx = d.dgx, vy = -d.dgy;  // (-dy)/diag == -(dy/diag)
    const double sc = xlx[4] * vx + xly[4] * vy;
    const double gvp = lim_grad(a[2], ac, a[6], xlx[2] * vx + xly[2] * vy, sc, xlx[6] * vx + xly[6] * vy, bad);
    const double ex = sx * lwx - dxp, ey = sx * -lwy - dyp;
    return ac + 0.5 * gvp * (ex * vx + ey * vy);
}

// CornerScheme (reconstruct.hpp:7, the H2D_CORNER_* ordinals)
enum { CS_UPWIND = 0, CS_AVGMIN = 1, CS_LINEARXY = 2, CS_LINEARDIAG = 3, CS_MULTID = 4 };
// CornerKin (reconstruct.hpp:44-51); er = eval_rel
struct Kin {
    double dxp, dyp, lwx, lwy, sfx, ufx, sfy, ufy, erx, ery;
};
H2D_DEV int sgn3(double v) { return v > 0.0 ? 1 : (v < 0.0 ? -1 : 0); }  // reconstruct.cpp:35
// multid_plane (reconstruct.cpp:45-107): the least-squares plane through the
// 3x3 stencil (Householder QR of the 8x2 system), limited by the smallest of
// the four 1D limited slopes; returns (a0, cx, cy, gx, gy)
static __device__ __noinline__ void multid_plane(double dgx, double dgy, const double* a, const double* xlx,
                                          const double* xly, double& a0, double& cx, double& cy, double& gx,
                                          double& gy, bool& bad, double* graw = nullptr) {
    a0 = a[4];
    cx = xlx[4];
    cy = xly[4];
    double X0[8], X1[8], b[8];
    {
        int m = 0;
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (p == 1 && q == 1) continue;
                X0[m] = xlx[p * 3 + q] - cx;
                X1[m] = xly[p * 3 + q] - cy;
                b[m] = a[p * 3 + q] - a0;
                ++m;
            }
    }
    gx = gy = 0.0;
    bool rank_ok = true;
#pragma unroll
    for (int col = 0; col < 2; ++col) {
        if (!rank_ok) break;
        double* Xc = col == 0 ? X0 : X1;
        double nrm = 0.0;
#pragma unroll
        for (int r = col; r < 8; ++r) nrm += Xc[r] * Xc[r];
        nrm = sqrt(nrm);
        if (nrm < 1e-300) {  // rank-deficient geometry: zero gradient
            rank_ok = false;
            break;
        }
        const double alpha = Xc[col] > 0.0 ? -nrm : nrm;
        double v[8];
        v[col] = Xc[col] - alpha;
#pragma unroll
        for (int r = col + 1; r < 8; ++r) v[r] = Xc[r];
        double vtv = 0.0;
#pragma unroll
        for (int r = col; r < 8; ++r) vtv += v[r] * v[r];
        if (vtv > 0.0) {
#pragma unroll
            for (int cc = col; cc < 2; ++cc) {
                double* Xk = cc == 0 ? X0 : X1;
                double sv = 0.0;
#pragma unroll
                for (int r = col; r < 8; ++r) sv += v[r] * Xk[r];
                sv *= 2.0 / vtv;
#pragma unroll
                for (int r = col; r < 8; ++r) Xk[r] -= sv * v[r];
            }
            double sv = 0.0;
#pragma unroll
            for (int r = col; r < 8; ++r) sv += v[r] * b[r];
            sv *= 2.0 / vtv;
#pragma unroll
            for (int r = col; r < 8; ++r) b[r] -= sv * v[r];
        }
    }
    if (!rank_ok) return;
    const double g2 = b[1] / X1[1];
    const double g1 = (b[0] - X1[0] * g2) / X0[0];
    if (graw) {  // PlaneRecon::grad_raw (h2d_scalar_eval only)
        graw[0] = g1;
        graw[1] = g2;
    }
    const double gnorm = sqrt(g1 * g1 + g2 * g2);
    if (gnorm < 1e-300) return;
    const double vx = dgx, vy = dgy;  // dx/diag, dy/diag (hoisted, same bits)
    const double lgx = lim_grad(a[1], a[4], a[7], xlx[1], xlx[4], xlx[7], bad);
    const double lgy = lim_grad(a[3], a[4], a[5], xly[3], xly[4], xly[5], bad);
    const double sc = xlx[4] * vx + xly[4] * vy;
    const double gv = lim_grad(a[0], a[4], a[8], xlx[0] * vx + xly[0] * vy, sc, xlx[8] * vx + xly[8] * vy, bad);
    const double scp = xlx[4] * vx + xly[4] * -vy;
    const double gvp =
        lim_grad(a[2], a[4], a[6], xlx[2] * vx + xly[2] * -vy, scp, xlx[6] * vx + xly[6] * -vy, bad);
    const double phi = rmin(rmin(fabs(lgx), fabs(lgy)), rmin(fabs(gv), fabs(gvp))) / gnorm;
    gx = phi * g1;
    gy = phi * g2;
}
// corner_value (reconstruct.cpp:116-152) for the AvgMin, LinearXY and Multid
// schemes (LinearDiag, the default, stays inline as corner_diag): out of line
// so the hot kernels keep their registers; a / xl as corner_diag
static __device__ __noinline__ double corner_value_other(int scheme, double dgx, double dgy, const double* a,
                                                  const double* xlx, const double* xly, Kin k, bool* bad) {
    const double ac = a[4];
    bool b = false;
    double r = ac;
    if (scheme == CS_AVGMIN) {
        const int sx = sgn3(k.dxp), sy = sgn3(k.dyp);
        const double pair_avg = 0.5 * (ac + a[(1 + sx) * 3 + (1 + sy)]);
        r = rmin(ac, pair_avg);
    } else if (scheme == CS_LINEARXY) {
        const double gx = lim_grad(a[1], ac, a[7], xlx[1], xlx[4], xlx[7], b);
        const double gy = lim_grad(a[3], ac, a[5], xly[3], xly[4], xly[5], b);
        r = ac + 0.5 * gx * (k.sfx * k.lwx - k.ufx) + 0.5 * gy * (k.sfy * k.lwy - k.ufy);
    } else if (scheme == CS_MULTID) {
        double a0, cx, cy, gx, gy;
        multid_plane(dgx, dgy, a, xlx, xly, a0, cx, cy, gx, gy, b);
        r = a0 + (gx * k.erx + gy * k.ery);
    }
    if (b) *bad = true;
    return r;
}
// plane_eval(multid_plane(stencil), (bx, by)) (reconstruct.hpp:67-69), out of line
static __device__ __noinline__ double multid_eval(double dgx, double dgy, const double* a, const double* xlx,
                                           const double* xly, double bx, double by, bool* bad) {
    double a0, cx, cy, gx, gy;
    bool b = false;
    multid_plane(dgx, dgy, a, xlx, xly, a0, cx, cy, gx, gy, b);
    if (b) *bad = true;
    return a0 + (gx * (bx - cx) + gy * (by - cy));
}

// corner_fraction / clipped_fraction, vof.cpp:28-45
H2D_DEV double corner_fraction(double A, double B, double t) {
    if (t <= 0.0) return 0.0;
    if (A > 0.0 && t < A) return t * t / (2.0 * A * B);
    return (t - 0.5 * A) / B;
}
H2D_DEV double clipped_fraction(double w, double h, double nx, double ny, double dd) {
    double A = fabs(nx) * w, B = fabs(ny) * h;
    if (A > B) {
        const double t = A;
        A = B;
        B = t;
    }
    const double S = 0.5 * (A + B);
    if (dd <= -S) return 0.0;
    if (dd >= S) return 1.0;
    if (dd <= 0.0) return corner_fraction(A, B, dd + S);
    return 1.0 - corner_fraction(A, B, S - dd);
}
// place_interface, vof.cpp:47-73 (returns d)
H2D_DEV double place_interface(double frac, double nx, double ny, double lox, double loy, double hix, double hiy) {
    const double w = hix - lox, h = hiy - loy;
    double A = fabs(nx) * w, B = fabs(ny) * h;
    if (A > B) {
        const double t = A;
        A = B;
        B = t;
    }
    const double S = 0.5 * (A + B);
    const bool flip = frac > 0.5;
    const double kk = flip ? 1.0 - frac : frac;
    double t;
    if (A > 0.0 && kk <= A / (2.0 * B))
        t = sqrt(2.0 * A * B * kk);
    else
        t = kk * B + 0.5 * A;
    double dd = t - S;
    if (flip) dd = -dd;
    if (fabs(clipped_fraction(w, h, nx, ny, dd) - frac) > 1e-13) {
        double lo = -S, hi = S;
        for (int it = 0; it < 200 && hi - lo > 1e-13 * (2.0 * S); ++it) {
            const double mid = 0.5 * (lo + hi);
            if (clipped_fraction(w, h, nx, ny, mid) < frac)
                lo = mid;
            else
                hi = mid;
        }
        dd = 0.5 * (lo + hi);
    }
    return dd;
}

H2D_DEV bool is_mixed(double k0) { return k0 > kPureTol && k0 < 1.0 - kPureTol; }  // remap.cpp:100

// Three materials (configuration 5's N-material extension; the
// oracle's pair3 / mixed3 / largest_other3, oracle/h2d_oracle.c): the
// reference's one-interface VOF on the two largest fractions of a cell.
H2D_DEV void pair3(const double* k, int& lo, int& hi) {
    int p = 0;
    if (k[1] > k[p]) p = 1;
    if (k[2] > k[p]) p = 2;
    int q = p == 0 ? 1 : 0;
    for (int a = 0; a < 3; ++a)
        if (a != p && k[a] > k[q]) q = a;
    lo = p < q ? p : q;
    hi = p < q ? q : p;
}
H2D_DEV bool mixed3(const double* k) {
    const int n = (k[0] > 0.0) + (k[1] > 0.0) + (k[2] > 0.0);
    if (n == 3) return true;
    if (n < 2) return false;
    return is_mixed(k[0] > 0.0 ? k[0] : k[1]);
}
H2D_DEV int largest_other3(const double* k, int a) {
    int b = -1;
    for (int c = 0; c < 3; ++c)
        if (c != a && (b < 0 || k[c] > k[b])) b = c;
    return b;
}
// the pure donor's material: the largest fraction (first on ties)
H2D_DEV int largest3(const double* k) {
    int p = 0;
    if (k[1] > k[p]) p = 1;
    if (k[2] > k[p]) p = 2;
    return p;
}

}  // namespace h2d

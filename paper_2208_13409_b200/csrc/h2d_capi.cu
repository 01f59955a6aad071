// h2d_capi.cu — the C-ABI of include/h2d.h over the sm_100a kernels.
//
// A context owns one device, one stream, a double-buffered device State (the
// buffer pair alternates every committed step, so a failed step leaves the
// previous State intact, matching the reference's value semantics), the
// LagrangeResult and all remap scratch, laid out as (P x R) fp64 planes with
// two ghost layers.  There is no host compute on the step path; a missing
// device is an error (H2D_ERR_DEVICE), never a fallback.
#include "../../include/h2d.h"
#include "h2d_launch.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace h2d;

namespace {

struct StateBufs {
    double *m[kMatSlots], *e[kMatSlots], *k[kMatSlots], *vol, *m_mix, *e_mix, *rho_mix, *p_mix, *nrx, *nry, *ux, *uy;
};

}  // namespace

struct h2d_ctx {
    h2d_config cfg{};
    int device = 0;
    cudaStream_t st = nullptr;
    int nx = 0, ny = 0, nmat = 1, P = 0, R = 0;
    size_t fsz = 0;  // doubles per plane
    char* arena = nullptr;
    size_t arena_bytes = 0, arena_used = 0;
    StateBufs sb[2]{};
    Dev base{};
    Ctl* ctl = nullptr;   // device
    Ctl* hctl = nullptr;  // pinned host mirror
    int cur = 0;
    bool have_lag = false;
    h2d_error err{};
    double* stage = nullptr;     // device staging for AoS Vec2 fields
    double* dt_log = nullptr;    // device dt log of h2d_run
    int dt_log_cap = 0;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};  // one run-loop step per State parity
    cudaGraphExec_t graph_ad[2][2] = {};            // AD steps per (State parity, x_first)
    cudaGraphExec_t graph_dir[2] = {nullptr, nullptr};  // Direct-engine steps per State parity
    double* ad_mem = nullptr;                       // AD Work planes between the passes
    TmaSet tma[2]{};                                // remap-tile TMA descriptors per State parity
    AdWork adw{};
    long long graph_kernels = 0, graph_kernels_ad = 0;
    cudaEvent_t ev[9] = {};
    h2d_block blk{};   // the block of the 2D decomposition (the whole mesh for h2d_create)
    bool is_block = false;
    double* xbuf = nullptr;  // device staging for window uploads / owned downloads
    size_t xbuf_bytes = 0;
    void* flush = nullptr;
    size_t flush_bytes = 0;
    void* diag_mem = nullptr;       // DiagRed scratch of k_post / the node update
    void* tcls_mem = nullptr;       // Dev::tcls, the remap tiles' material classes
    void* pcls_mem = nullptr;       // Dev::pcls, the post blocks' classification masks
    size_t diag_tick_bytes = 0;     // the ticket words at the start of diag_mem
    double* diag_log = nullptr;     // device StepDiag log of h2d_run (kDiagRec doubles per step)
    cudaGraphExec_t graph_rest[2] = {nullptr, nullptr};  // block data plane: the step after the Lagrange kernel
    // the run loops keep no derived planes (m_mix, e_mix, rho_mix, p_mix, vol):
    // set after a run step, cleared by ensure_derived (sync_derived on the
    // current State) before anything reads the State
    bool derived_stale = false;
    long long graph_rest_kernels = 0;
};

namespace {

constexpr int kRunLogCap = 65536;  // dt / StepDiag log entries of a run until t_end

void set_err(h2d_ctx* c, int kind, const char* what, int i = -1, int j = -1, int step = -1, int in_step = 0) {
    c->err.kind = kind;
    c->err.i = i;
    c->err.j = j;
    c->err.step = step;
    c->err.in_step = in_step;
    std::snprintf(c->err.what, sizeof c->err.what, "%s", what);
}

int cuda_fail(h2d_ctx* c, cudaError_t e, const char* where) {
    char buf[200];
    std::snprintf(buf, sizeof buf, "CUDA error in %s: %s", where, cudaGetErrorString(e));
    if (c) set_err(c, H2D_ERR_DEVICE, buf);
    return H2D_ERR_DEVICE;
}

#define CK(call)                                               \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return cuda_fail(c, e_, #call); \
    } while (0)

double* carve(h2d_ctx* c, size_t count_doubles) {
    const size_t bytes = (count_doubles * sizeof(double) + 255) & ~size_t(255);
    double* p = reinterpret_cast<double*>(c->arena + c->arena_used);
    c->arena_used += bytes;
    return p;
}
// pointer to element (-G, -G) of a plane: the plane base
inline double* plane(h2d_ctx* c) { return carve(c, c->fsz); }

Dev make_dev(h2d_ctx* c, int parity, int remap_velocity) {
    Dev d = c->base;
    const StateBufs& s = c->sb[parity];
    const StateBufs& n = c->sb[1 - parity];
    for (int a = 0; a < kMatSlots; ++a) {
        d.m[a] = s.m[a];
        d.e[a] = s.e[a];
        d.k[a] = s.k[a];
        d.nm[a] = n.m[a];
        d.ne[a] = n.e[a];
        d.nk[a] = n.k[a];
    }
    d.vol = s.vol;
    d.m_mix = s.m_mix;
    d.e_mix = s.e_mix;
    d.rho_mix = s.rho_mix;
    d.p_mix = s.p_mix;
    d.nrx = s.nrx;
    d.nry = s.nry;
    d.ux = s.ux;
    d.uy = s.uy;
    d.nvol = n.vol;
    d.nm_mix = n.m_mix;
    d.ne_mix = n.e_mix;
    d.nrho_mix = n.rho_mix;
    d.np_mix = n.p_mix;
    d.nnrx = n.nrx;
    d.nnry = n.nry;
    d.nux = n.ux;
    d.nuy = n.uy;
    d.remap_velocity = remap_velocity;
    d.tma = &c->tma[parity];
    return d;
}

int ctl_pull(h2d_ctx* c) {
    CK(cudaMemcpyAsync(c->hctl, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return 0;
}
int ctl_push(h2d_ctx* c) {
    CK(cudaMemcpyAsync(c->ctl, c->hctl, sizeof(Ctl), cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
    return 0;
}
// Reset the control block before an API call (errors of earlier calls do not
// block later ones, like independent reference calls).
int ctl_reset(h2d_ctx* c) {
    if (int rc = ctl_pull(c)) return rc;
    Ctl& h = *c->hctl;
    h.err_key = kNoErr;
    h.done = 0;
    h.cur = c->cur;
    h.step_floor = h.step_clip = h.step_fix = 0;
    h.wmax_bits = h.kviol_bits = 0;
    h.next_wmax_bits = 0;
    h.next_err_key = kNoErr;
    h.diag_log = nullptr;
    h.diag_log_cap = 0;
    // a run that ended inside a step (error) can leave diagnostics tickets
    // half counted: clear them for the next call
    if (c->diag_mem) CK(cudaMemsetAsync(c->diag_mem, 0, c->diag_tick_bytes, c->st));
    return ctl_push(c);
}

// dt / StepDiag logs of a run of up to `cap` steps
int ensure_logs(h2d_ctx* c, int cap) {
    if (cap <= c->dt_log_cap) return 0;
    if (c->dt_log) cudaFree(c->dt_log);
    if (c->diag_log) cudaFree(c->diag_log);
    c->dt_log = nullptr;
    c->diag_log = nullptr;
    c->dt_log_cap = 0;
    CK(cudaMalloc(&c->dt_log, sizeof(double) * (size_t)cap));
    CK(cudaMalloc(&c->diag_log, sizeof(double) * kDiagRec * (size_t)cap));
    c->dt_log_cap = cap;
    return 0;
}

// device StepDiag records -> h2d_step_diag (harness.hpp:66-72)
int copy_series(h2d_ctx* c, h2d_step_diag* out, int n) {
    if (!out || n <= 0) return 0;
    std::vector<double> r((size_t)n * kDiagRec);
    CK(cudaMemcpy(r.data(), c->diag_log, sizeof(double) * r.size(), cudaMemcpyDeviceToHost));
    for (int q = 0; q < n; ++q) {
        const double* x = &r[(size_t)q * kDiagRec];
        h2d_step_diag& o = out[q];
        o.step = (int)x[0];
        o.t = x[1];
        o.dt = x[2];
        o.mass = x[3 + DG_MASS];
        o.mass_mat[0] = x[3 + DG_MM0];
        o.mass_mat[1] = c->nmat >= 2 ? x[3 + DG_MM1] : 0.0;
        o.mass_mat[2] = c->nmat == 3 ? x[3 + DG_MM2] : 0.0;
        o.momentum_x = x[3 + DG_PX];
        o.momentum_y = x[3 + DG_PY];
        o.internal_energy = x[3 + DG_IE];
        o.min_rho = x[3 + DG_MINR];
        o.max_rho = x[3 + DG_MAXR];
        o.min_p = x[3 + DG_MINP];
        o.max_p = x[3 + DG_MAXP];
    }
    return 0;
}

// Rebuild the reference exception of the first failing phase (errors.hpp).
int decode_error(h2d_ctx* c, bool in_run) {
    const uint64_t key = c->hctl->err_key;
    if (key == kNoErr) return 0;
    const int ph = (int)(key >> 58);
    const int outer = (int)((key >> 33) & 0x1FFFFFF) - 16;
    const int inner = (int)((key >> 8) & 0x1FFFFFF) - 16;
    const int sub = (int)(key & 0xFF);
    int kind = H2D_ERR_SIM;
    const char* msg = "";
    bool located = false, with_step = false;
    int in_step = 1;
    switch (ph) {
    case PH_CFL_UNPHYS: kind = H2D_ERR_UNPHYSICAL; msg = "unphysical state: gamma*(P+pi)/rho < 0"; in_step = 0; break;
    case PH_CFL_WAVE: kind = H2D_ERR_SIM; msg = "non-finite wave speed"; in_step = 0; break;
    case PH_Q_UNPHYS: kind = H2D_ERR_UNPHYSICAL; msg = "unphysical state: gamma*(P+pi)/rho < 0"; break;
    case PH_PRED_TANGLED:
    case PH_CORR_TANGLED: kind = H2D_ERR_TANGLED; msg = "tangled cell"; located = true; break;
    case PH_CFL_XFACE: kind = H2D_ERR_CFL; msg = "CFL violation at X-face"; located = true; break;
    case PH_CFL_YFACE: kind = H2D_ERR_CFL; msg = "CFL violation at Y-face"; located = true; break;
    case PH_CFL_CORNER: kind = H2D_ERR_CFL; msg = "CFL violation at corner"; located = true; break;
    case PH_COLLAPSED: kind = H2D_ERR_CFL; msg = "collapsed Lagrangian cell"; located = true; break;
    case PH_GRAD_XFACE:
    case PH_GRAD_YFACE:
        if (sub == kSubDirectCfl) {  // the Direct engine's face loop (remap.cpp:668-671)
            kind = H2D_ERR_CFL;
            msg = "CFL violation at face";
            located = true;
            break;
        }
        kind = H2D_ERR_SIM;
        msg = "non-increasing centroid coordinates";
        break;
    case PH_GRAD_CORNER:
    case PH_GRAD_DUALX:
    case PH_GRAD_DUALY:
    case PH_GRAD_DUALC: kind = H2D_ERR_SIM; msg = "non-increasing centroid coordinates"; break;
    case PH_NEGMASS:
        kind = H2D_ERR_NEGMASS;
        msg = sub == kSubCellMass ? "non-positive cell mass" : "negative mass";
        located = true;
        break;
    case PH_NODAL_MASS: kind = H2D_ERR_NEGMASS; msg = "non-positive nodal mass"; located = true; break;
    case PH_NAN_CELL: kind = H2D_ERR_SIM; msg = "non-finite cell state"; located = true; with_step = true; in_step = 0; break;
    case PH_NAN_NODE: kind = H2D_ERR_SIM; msg = "non-finite velocity"; located = true; with_step = true; in_step = 0; break;
    default:
        if (ph >= PH_AD_COLLAPSED && ph < PH_AD_COLLAPSED + 10) {  // AD pass 0 / 1 (remap.cpp:469-589)
            switch ((ph - PH_AD_COLLAPSED) % 5 + PH_AD_COLLAPSED) {
            case PH_AD_COLLAPSED: kind = H2D_ERR_CFL; msg = "collapsed Lagrangian cell"; located = true; break;
            case PH_AD_FACE:
                if (sub & 1) {
                    kind = H2D_ERR_SIM;
                    msg = "non-increasing centroid coordinates";
                } else {
                    kind = H2D_ERR_CFL;
                    msg = "CFL violation at face";
                    located = true;
                }
                break;
            case PH_AD_NEGMASS:
                kind = H2D_ERR_NEGMASS;
                msg = sub == kSubCellMass ? "non-positive cell mass" : "negative mass";
                located = true;
                break;
            case PH_AD_GRAD_DUAL: kind = H2D_ERR_SIM; msg = "non-increasing centroid coordinates"; break;
            default: kind = H2D_ERR_NEGMASS; msg = "non-positive nodal mass"; located = true; break;
            }
            break;
        }
        kind = H2D_ERR_DEVICE;
        msg = "unknown device error";
        break;
    }
    std::string w = msg;
    // the AD scan and face keys are (cross, along, 2 * axis_x + ...): a Y pass
    // stores (i, j) as (inner, outer) swapped
    const int adp = ph >= PH_AD_COLLAPSED && ph < PH_AD_COLLAPSED + 10 ? (ph - PH_AD_COLLAPSED) % 5 : -1;
    const bool ad_y = ((adp == 0 || adp == 1) && !(sub >> 1)) || (ph == PH_GRAD_YFACE && sub == kSubDirectCfl);
    const int i = located ? (ad_y ? outer : inner) : -1, j = located ? (ad_y ? inner : outer) : -1;
    // SimError::format appends the location only for i >= 0 || j >= 0 (errors.hpp:23)
    if (located && (i >= 0 || j >= 0)) w += " at cell (" + std::to_string(i) + "," + std::to_string(j) + ")";
    const int step = c->hctl->step;
    if (with_step) w += " step " + std::to_string(step);
    if (!in_run) in_step = 0;
    set_err(c, kind, w.c_str(), i, j, (with_step || in_step) ? step : -1, in_step);
    return kind;
}

int check_launch(h2d_ctx* c) {
    CK(cudaGetLastError());
    return 0;
}

// host <-> device copies in the reference layout (pitch n1 + 4)
int put_plane(h2d_ctx* c, double* dst, const double* src, int n1, int n2) {
    if (!src) return 0;
    const size_t w = (size_t)(n1 + 2 * G) * sizeof(double);
    CK(cudaMemcpy2DAsync(dst, (size_t)c->P * sizeof(double), src, w, w, (size_t)(n2 + 2 * G),
                         cudaMemcpyHostToDevice, c->st));
    return 0;
}
int get_plane(h2d_ctx* c, double* dst, const double* src, int n1, int n2) {
    if (!dst) return 0;
    const size_t w = (size_t)(n1 + 2 * G) * sizeof(double);
    CK(cudaMemcpy2DAsync(dst, w, src, (size_t)c->P * sizeof(double), w, (size_t)(n2 + 2 * G),
                         cudaMemcpyDeviceToHost, c->st));
    return 0;
}
int put_vec(h2d_ctx* c, double* x, double* y, const double* src, int n1, int n2) {
    if (!src) return 0;
    const int W = n1 + 2 * G, H = n2 + 2 * G;
    CK(cudaMemcpyAsync(c->stage, src, (size_t)W * H * 2 * sizeof(double), cudaMemcpyHostToDevice, c->st));
    launch_deinterleave(c->stage, x, y, W, H, c->P, c->st);
    return check_launch(c);
}
int get_vec(h2d_ctx* c, double* dst, const double* x, const double* y, int n1, int n2) {
    if (!dst) return 0;
    const int W = n1 + 2 * G, H = n2 + 2 * G;
    launch_interleave(c->stage, x, y, W, H, c->P, c->st);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(dst, c->stage, (size_t)W * H * 2 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    return 0;
}
int zero_plane(h2d_ctx* c, double* p) {
    CK(cudaMemsetAsync(p, 0, c->fsz * sizeof(double), c->st));
    return 0;
}

__global__ void k_fill(double* p, double v, size_t n) {  // setup only
    const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (t < n) p[t] = v;
}
int fill_plane(h2d_ctx* c, double* p, double v) {
    k_fill<<<(unsigned)((c->fsz + 255) / 256), 256, 0, c->st>>>(p, v, c->fsz);
    return check_launch(c);
}

int fill_ghosts_cur(h2d_ctx* c, int parity) {
    const Dev d = make_dev(c, parity, 1);
    FieldList fl{};
    fl.respect_halt = 0;
    int q = 0;
    for (int a = 0; a < c->nmat; ++a) {
        fl.f[q++] = c->sb[parity].m[a];
        fl.f[q++] = c->sb[parity].e[a];
        fl.f[q++] = c->sb[parity].k[a];
    }
    fl.f[q++] = c->sb[parity].nrx;
    fl.f[q++] = c->sb[parity].nry;
    fl.n = q;
    launch_ghost_cells(d, fl, c->st);
    FieldList fu{};
    fu.respect_halt = 0;
    fu.n = 2;
    fu.f[0] = c->sb[parity].ux;
    fu.f[1] = c->sb[parity].uy;
    launch_ghost_nodes(d, fu, c->st);
    return check_launch(c);
}

// One run-loop step (harness.cpp:390-412) for the state in `parity`.
// (single domain: the step's start is the previous step's k_tail, and the
// first step of a call gets a standalone k_step_start, start_first below)
void enqueue_step(h2d_ctx* c, int parity) { launch_step(make_dev(c, parity, 1), !c->is_block, c->st); }

// the start of the first run-loop step of a call (later starts are fused
// into the previous step's k_tail on a single domain)
void start_first(h2d_ctx* c) {
    if (!c->is_block) launch_step_start(make_dev(c, c->cur, 1), c->st);
}

// rebuild the derived planes of the current State after run-loop steps
// (sync_derived, state.cpp:120-143: the values k_post computed in registers)
int ensure_derived(h2d_ctx* c) {
    if (!c->derived_stale) return 0;
    launch_sync(make_dev(c, c->cur, 1), 0, 0, c->st);
    if (int rc = check_launch(c)) return rc;
    CK(cudaStreamSynchronize(c->st));
    c->derived_stale = false;
    return 0;
}

// cfl_dt of the current State into the control block's "next" slots, which
// the first k_step_start of a run consumes (later steps get them from k_post)
void enqueue_cfl_next(h2d_ctx* c) {
    const Dev d = make_dev(c, c->cur, 1);
    launch_cfl_next(d, c->st);
    launch_cls_flags(d, c->st);  // and the tile-classification masks of the current State (Dev::pcls)
}

// The run-loop step is a fixed sequence of ~20 kernels whose arguments only
// depend on the State parity: capture it once per parity as a CUDA graph and
// replay it, so the per-kernel launch cost is paid once.
int ensure_graphs(h2d_ctx* c) {
    if (c->graph[0] && c->graph[1]) return 0;
    for (int p = 0; p < 2; ++p) {
        cudaGraph_t g = nullptr;
        const long long before = launch_count();
        CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
        enqueue_step(c, p);
        CK(cudaStreamEndCapture(c->st, &g));
        c->graph_kernels = launch_count() - before;
        add_launches(-c->graph_kernels);  // captured, not executed
        const cudaError_t e = cudaGraphInstantiate(&c->graph[p], g, 0);
        cudaGraphDestroy(g);
        CK(e);
    }
    return 0;
}

// Direct-engine run-loop steps (remap.cpp:593-724), captured like DirectCF's
int ensure_graphs_dir(h2d_ctx* c) {
    if (c->graph_dir[0] && c->graph_dir[1]) return 0;
    for (int p = 0; p < 2; ++p) {
        cudaGraph_t g = nullptr;
        const long long before = launch_count();
        CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
        Dev d = make_dev(c, p, 1);
        d.direct = 1;
        launch_step(d, !c->is_block, c->st);
        CK(cudaStreamEndCapture(c->st, &g));
        c->graph_kernels = launch_count() - before;
        add_launches(-c->graph_kernels);
        const cudaError_t e = cudaGraphInstantiate(&c->graph_dir[p], g, 0);
        cudaGraphDestroy(g);
        CK(e);
    }
    return 0;
}

int launch_step_graph(h2d_ctx* c, int parity) {
    CK(cudaGraphLaunch(c->graph[parity], c->st));
    add_launches(c->graph_kernels);
    return 0;
}

// The AD engine's Work planes (remap.cpp:87-97 between the two directional
// passes), allocated on first use: m, me, e, k per material, mcell, u, normals.
int ensure_ad(h2d_ctx* c) {
    if (c->ad_mem) return 0;
    const int nm = c->nmat;
    const size_t pb = (c->fsz * sizeof(double) + 255) & ~size_t(255);
    const size_t n = 4 * (size_t)nm + 5;
    CK(cudaMalloc(&c->ad_mem, pb * n));
    CK(cudaMemsetAsync(c->ad_mem, 0, pb * n, c->st));
    char* p = reinterpret_cast<char*>(c->ad_mem);
    auto take = [&]() {
        double* r = reinterpret_cast<double*>(p);
        p += pb;
        return r;
    };
    AdWork& W = c->adw;
    for (int a = 0; a < nm; ++a) {
        W.m[a] = take();
        W.me[a] = take();
        W.e[a] = take();
        W.k[a] = take();
    }
    W.mcell = take();
    W.ux = take();
    W.uy = take();
    W.nrx = take();
    W.nry = take();
    return 0;
}

// AD run-loop steps: the axis order alternates with the step number
// (harness.cpp:401, x_first = step % 2 == 0), captured per (parity, x_first).
int ensure_graphs_ad(h2d_ctx* c) {
    if (int rc = ensure_ad(c)) return rc;
    for (int p = 0; p < 2; ++p)
        for (int xf = 0; xf < 2; ++xf) {
            if (c->graph_ad[p][xf]) continue;
            cudaGraph_t g = nullptr;
            const long long before = launch_count();
            CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
            launch_step_ad(make_dev(c, p, 1), c->adw, xf, 1, c->st);
            CK(cudaStreamEndCapture(c->st, &g));
            c->graph_kernels_ad = launch_count() - before;
            add_launches(-c->graph_kernels_ad);
            const cudaError_t e = cudaGraphInstantiate(&c->graph_ad[p][xf], g, 0);
            cudaGraphDestroy(g);
            CK(e);
        }
    return 0;
}

// Compute ranges of every phase: the reference's ranges, and
// on block sides facing a neighbour block the storage window shrunk by the
// stencil reach accumulated up to that phase, so that after one step the
// owned cells and nodes are exact and only the halo needs the exchange.
void block_ranges(h2d_ctx* c) {
    Dev& d = c->base;
    const h2d_block& b = c->blk;
    const int NX = d.nx, NY = d.ny, H = b.halo;
    const bool li = b.oi > 0, ri = b.oi + b.bnx < NX, bi = b.oj > 0, ti = b.oj + b.bny < NY;
    const int wl = b.oi - H, wr = b.oi + b.bnx + H, wb = b.oj - H, wt = b.oj + b.bny + H;
    auto R = [&](int rlo, int rhi, int slo, int shi, int rjlo, int rjhi) {
        Rng r;
        r.i0 = li ? std::max(rlo, wl + slo) : rlo;
        r.i1 = ri ? std::min(rhi, wr - shi) : rhi;
        r.j0 = bi ? std::max(rjlo, wb + slo) : rjlo;
        r.j1 = ti ? std::min(rjhi, wt - shi) : rjhi;
        return r;
    };
    d.r_lagc = R(0, NX, 0, 0, 0, NY);
    d.r_lagn = R(0, NX + 1, 1, 0, 0, NY + 1);
    d.r_lage = R(0, NX, 1, 1, 0, NY);
    d.r_gath = R(0, NX, 3, 3, 0, NY);
    d.r_dual = R(0, NX + 1, 4, 3, 0, NY + 1);
    d.r_node = R(0, NX + 1, 6, 5, 0, NY + 1);
    d.r_sync = R(-G, NX + G, 5, 5, -G, NY + G);
    d.r_nrm = R(0, NX, 6, 6, 0, NY);
    d.own_c = {li ? b.oi : -G, ri ? b.oi + b.bnx : NX + G, bi ? b.oj : -G, ti ? b.oj + b.bny : NY + G};
    d.own_n = {li ? b.oi : -G, ri ? b.oi + b.bnx : NX + G + 1, bi ? b.oj : -G, ti ? b.oj + b.bny : NY + G + 1};
    d.win_c = {std::max(wl, -G), std::min(wr, NX + G), std::max(wb, -G), std::min(wt, NY + G)};
    d.win_n = {std::max(wl, -G), std::min(wr + 1, NX + G + 1), std::max(wb, -G), std::min(wt + 1, NY + G + 1)};
}

// TMA descriptors (cuTensorMapEncodeTiled through the runtime's driver entry
// point) of every plane the remap tile stages: 2D fp64 tensors of P x R
// doubles (row pitch P * 8 bytes), node boxes RNW x RNH, cell boxes RCW x RCH;
// boxes reaching past the plane are zero-filled.
int make_tmas(h2d_ctx* c) {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn enc = nullptr;
    if (!enc) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            return 1;
        enc = reinterpret_cast<EncodeFn>(fn);
    }
    const Dev& d = c->base;
    auto make = [&](CUtensorMap* m, double* base, cuuint32_t bw, cuuint32_t bh) {
        const cuuint64_t dims[2] = {(cuuint64_t)c->P, (cuuint64_t)c->R};
        const cuuint64_t strides[1] = {(cuuint64_t)c->P * sizeof(double)};
        const cuuint32_t box[2] = {bw, bh};
        const cuuint32_t es[2] = {1, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS;
    };
    const cuuint32_t nw = tma_node_box_w(), nh = tma_node_box_h(), cw = tma_cell_box_w(), ch = tma_cell_box_h();
    for (int p = 0; p < 2; ++p) {
        TmaSet& t = c->tma[p];
        int bad = make(&t.t[TM_UHX], d.uhx, nw, nh) | make(&t.t[TM_UHY], d.uhy, nw, nh);
        for (int a = 0; a < c->nmat; ++a) {
            bad |= make(&t.t[TM_EL0 + a], d.el[a], cw, ch);
            bad |= make(&t.t[TM_M0 + a], c->sb[p].m[a], cw, ch);
            bad |= make(&t.t[TM_K0 + a], c->sb[p].k[a], cw, ch);
        }
        if (bad) return 1;
    }
    return 0;
}

int create_ctx(const h2d_config* cfg, const h2d_block* blk, int device, h2d_ctx** out, bool block);

}  // namespace

extern "C" {

int h2d_abi_version(void) { return H2D_ABI_VERSION; }

long long h2d_launch_count(void) { return launch_count(); }

int h2d_create(const h2d_config* cfg, int device, h2d_ctx** out) {
    h2d_block whole;
    whole.oi = 0;
    whole.oj = 0;
    whole.bnx = cfg->mesh.nx;
    whole.bny = cfg->mesh.ny;
    whole.halo = G;
    return create_ctx(cfg, &whole, device, out, false);
}

int h2d_create_block(const h2d_config* cfg, const h2d_block* blk, int device, h2d_ctx** out) {
    *out = nullptr;
    const h2d_mesh& m = cfg->mesh;
    if (m.bc_x == H2D_BC_PERIODIC || m.bc_y == H2D_BC_PERIODIC) return H2D_ERR_INVALID;  // walls only
    if (blk->halo < 8 || blk->oi < 0 || blk->oj < 0 || blk->bnx < blk->halo || blk->bny < blk->halo ||
        blk->oi + blk->bnx > m.nx || blk->oj + blk->bny > m.ny)
        return H2D_ERR_INVALID;
    const int rc = create_ctx(cfg, blk, device, out, true);
    if (!rc) (*out)->is_block = true;
    return rc;
}

}  // extern "C"

namespace {
int create_ctx(const h2d_config* cfg, const h2d_block* blk, int device, h2d_ctx** out, bool block) {
    *out = nullptr;
    const h2d_mesh& m = cfg->mesh;
    if (m.nx < 3 || m.ny < 3) return H2D_ERR_SIM;        // Mesh::Mesh, mesh.hpp:27
    if (m.dx <= 0.0 || m.dy <= 0.0) return H2D_ERR_SIM;  // mesh.hpp:28
    if (cfg->nmat < 1 || cfg->nmat > H2D_MAX_MAT) return H2D_ERR_INVALID;  // (3: DESIGN.md 5b)
    if (cfg->corner < H2D_CORNER_UPWIND || cfg->corner > H2D_CORNER_MULTID) return H2D_ERR_INVALID;
    h2d_ctx* c = new h2d_ctx();
    c->cfg = *cfg;
    auto fail = [&](int rc) {
        h2d_destroy(c);
        return rc;
    };
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(H2D_ERR_DEVICE);
    if (device < 0) cudaGetDevice(&device);
    c->device = device;
    if (cudaSetDevice(device) != cudaSuccess) return fail(H2D_ERR_DEVICE);
    if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) return fail(H2D_ERR_DEVICE);
    c->nx = m.nx;
    c->ny = m.ny;
    c->nmat = cfg->nmat;
    c->blk = *blk;
    const int H = blk->halo;
    c->P = ((blk->bnx + 1 + 2 * H) + 31) / 32 * 32;
    c->R = blk->bny + 1 + 2 * H;
    c->fsz = (size_t)c->P * (size_t)c->R;
    if (c->fsz >= (size_t)1 << 31) {  // device plane offsets are 32-bit
        h2d_destroy(c);
        return H2D_ERR_INVALID;
    }
    const int nm = c->nmat;
    // fp64 planes, exactly as carved below: 2 x State (3 nm + 9; a single
    // domain shares its normals between the parities: one material carries
    // them unchanged, and with 2-3 materials the normals are updated in place
    // (only mixed cells change; a step that fails before k_post never touches
    // them, and a decomposition block, which can be rolled back after
    // k_post, keeps two copies), the LagrangeResult (7) and per material
    // p_half, e_lag, me, sliver m / m*e (5 nm), the remap scratch (13), the
    // AoS staging (2). Single domain, 1 / 2 / 3 materials: 49 / 60 / 71
    // planes, i.e. with the 10 byte planes ~402 / 490 / 578 B per cell:
    // 16384^2 x 3 materials (configuration 5) fits one B200
    const bool shared_nrm = nm == 1 || !block;
    const size_t planes = 2 * (3 * (size_t)nm + 9) - (shared_nrm ? 2 : 0) + 7 + 5 * (size_t)nm + 13 + 2;
    const size_t bytes_planes = planes * ((c->fsz * sizeof(double) + 255) & ~size_t(255));
    const size_t bytes_small = 10 * ((c->fsz + 255) & ~size_t(255)) + ((size_t)c->R * 4 + 256);
    c->arena_bytes = bytes_planes + bytes_small + 4096;
    if (cudaMalloc(&c->arena, c->arena_bytes) != cudaSuccess) return fail(H2D_ERR_NOMEM);
    cudaMemsetAsync(c->arena, 0, c->arena_bytes, c->st);
    for (int p = 0; p < 2; ++p) {
        StateBufs& s = c->sb[p];
        std::memset(&s, 0, sizeof s);
        for (int a = 0; a < nm; ++a) {
            s.m[a] = plane(c);
            s.e[a] = plane(c);
            s.k[a] = plane(c);
        }
        s.vol = plane(c);
        s.m_mix = plane(c);
        s.e_mix = plane(c);
        s.rho_mix = plane(c);
        s.p_mix = plane(c);
        if (p == 0 || !shared_nrm) {
            s.nrx = plane(c);
            s.nry = plane(c);
        } else {  // both parities share the normals (see the plane count above)
            s.nrx = c->sb[0].nrx;
            s.nry = c->sb[0].nry;
        }
        s.ux = plane(c);
        s.uy = plane(c);
    }
    Dev& d = c->base;
    std::memset(&d, 0, sizeof d);
    d.nx = m.nx;
    d.ny = m.ny;
    d.P = c->P;
    d.fsz = (int)c->fsz;
    d.oi = blk->oi;
    d.oj = blk->oj;
    d.H = H;
    d.off = (H - blk->oj) * c->P + (H - blk->oi);
    block_ranges(c);
    d.nmat = nm;
    d.per_x = m.bc_x == H2D_BC_PERIODIC;
    d.per_y = m.bc_y == H2D_BC_PERIODIC;
    d.dx = m.dx;
    d.dy = m.dy;
    d.x0 = m.x0;
    d.y0 = m.y0;
    d.cv = m.dx * m.dy;
    d.L = std::sqrt(m.dx * m.dy);  // Mesh::char_length, mesh.hpp:39
    auto pow2_recip = [](double v) {  // 1/v when v is an exact power of two with a normal reciprocal
        int e = 0;
        const double mnt = std::frexp(v, &e);
        const double r = 1.0 / v;
        return (mnt == 0.5 && std::isnormal(r) && std::isnormal(v)) ? r : 0.0;
    };
    d.rdx = pow2_recip(m.dx);
    d.rdy = pow2_recip(m.dy);
    d.rcv = pow2_recip(d.cv);
    {
        const double diag = std::sqrt(m.dx * m.dx + m.dy * m.dy);  // host IEEE, no contraction
        d.dgx = m.dx / diag;
        d.dgy = m.dy / diag;
    }
    for (int a = 0; a < nm; ++a) {
        d.stiff[a] = cfg->eos[a].kind == H2D_EOS_STIFFENED;
        d.gamma[a] = cfg->eos[a].gamma;
        d.pi[a] = cfg->eos[a].pi;
    }
    d.a1 = cfg->pv_a1;
    d.a2 = cfg->pv_a2;
    d.face_order = cfg->face_order;
    d.corner_diag = cfg->corner == H2D_CORNER_LINEARDIAG;
    d.corner = cfg->corner;
    d.degrade = cfg->interface_degrade != 0;
    d.opt_energy = (cfg->options & H2D_OPT_SLIVER_ENERGY) != 0;
    d.remap_velocity = 1;
    d.q = plane(c);
    d.pmh = plane(c);
    d.uhx = plane(c);
    d.uhy = plane(c);
    d.ulx = plane(c);
    d.uly = plane(c);
    d.vol_lag = plane(c);
    for (int a = 0; a < nm; ++a) {
        d.ph[a] = plane(c);
        d.el[a] = plane(c);
        d.me[a] = plane(c);
        d.slm[a] = plane(c);
        d.slme[a] = plane(c);
    }
    d.mcell = plane(c);
    d.unrm = plane(c);
    d.dmx = plane(c);
    d.dmy = plane(c);
    d.dmc = plane(c);
    d.dfx_x = plane(c);
    d.dfx_y = plane(c);
    d.dfy_x = plane(c);
    d.dfy_y = plane(c);
    d.dc_x[0] = plane(c);
    d.dc_y[0] = plane(c);
    d.dc_x[1] = plane(c);
    d.dc_y[1] = plane(c);
    c->stage = plane(c);  // >= (nx+5)(ny+5)*2? P*R >= (nx+5)(ny+5); staging needs 2x
    (void)carve(c, c->fsz);
    auto bytes_plane = [&]() {
        char* p = c->arena + c->arena_used;
        c->arena_used += (c->fsz + 255) & ~size_t(255);
        return reinterpret_cast<uint8_t*>(p);
    };
    d.sliver = bytes_plane();
    for (int q = 0; q < 4; ++q) d.dflag[q] = bytes_plane();
    d.sl_segs = reinterpret_cast<unsigned*>(bytes_plane());  // two bitmaps of <= R*(P/8+4) bytes each
    d.sl_segs2 = d.sl_segs + c->fsz / 8;                     // (the second at byte fsz/2 of the plane)
    d.sl_list = reinterpret_cast<int*>(bytes_plane());       // 4 byte planes: one int per cell
    d.sl_cap = (int)c->fsz;
    for (int q = 0; q < 3; ++q) (void)bytes_plane();
    d.sl_rows = reinterpret_cast<unsigned*>(c->arena + c->arena_used);
    c->arena_used += ((size_t)c->R * 4 + 255) & ~size_t(255);
    if (c->arena_used > c->arena_bytes) return fail(H2D_ERR_NOMEM);
    if (cudaMalloc(&c->ctl, sizeof(Ctl)) != cudaSuccess) return fail(H2D_ERR_NOMEM);
    if (cudaMallocHost(&c->hctl, sizeof(Ctl)) != cudaSuccess) return fail(H2D_ERR_NOMEM);
    std::memset(c->hctl, 0, sizeof(Ctl));
    c->hctl->err_key = kNoErr;
    d.ctl = c->ctl;
    {  // diagnostics scratch: the ticket, the second-level partials, the block partials
        const size_t n0 = (size_t)diag_partials(d, 0), n1 = (size_t)diag_partials(d, 1);
        c->diag_tick_bytes = 256;
        const size_t bytes = 256 + sizeof(double) * ((size_t)kDiagBlocks * DG_N + n0 * DG_NCELL + n1 * 2);
        if (cudaMalloc(&c->diag_mem, bytes) != cudaSuccess) return fail(H2D_ERR_NOMEM);
        if (cudaMemset(c->diag_mem, 0, bytes) != cudaSuccess) return fail(H2D_ERR_DEVICE);
        double* pp = reinterpret_cast<double*>(static_cast<char*>(c->diag_mem) + 256);
        d.dsc.tick = static_cast<unsigned*>(c->diag_mem);
        d.dsc.lvl2 = pp;
        d.dsc.part[0] = pp + (size_t)kDiagBlocks * DG_N;
        d.dsc.part[1] = d.dsc.part[0] + n0 * DG_NCELL;
    }
    {  // one class byte per remap tile (launch_remap_tile's grid; 2-3 materials)
        const int shift = (d.r_gath.i0 - G + d.H - d.oi) & 1;  // tile_shift (h2d_kernels.cu)
        const int w = d.r_gath.i1 - (d.r_gath.i0 - shift), h = d.r_gath.j1 - d.r_gath.j0;
        d.tq_nx = std::max(1, (w + remap_tile_w() - 1) / remap_tile_w());
        d.tq_ny = std::max(1, (h + remap_tile_h() - 1) / remap_tile_h());
        if (nm >= 2) {
            const size_t n = (size_t)d.tq_nx * d.tq_ny;
            if (cudaMalloc(&c->tcls_mem, n) != cudaSuccess) return fail(H2D_ERR_NOMEM);
            if (cudaMemset(c->tcls_mem, 3, n) != cudaSuccess) return fail(H2D_ERR_DEVICE);
            d.tcls = static_cast<uint8_t*>(c->tcls_mem);
        }
    }
#ifndef H2D_CLS_POST
#define H2D_CLS_POST 1
#endif
    d.pcls = nullptr;
    d.pcls_nx = 0;
    d.cls_post = 0;
    if (H2D_CLS_POST && remap_uses_classes(nm) && !block) {  // Dev::pcls, one mask per k_post block (over r_sync)
        const int pw = (d.r_sync.i1 - d.r_sync.i0 + 31) / 32, ph = (d.r_sync.j1 - d.r_sync.j0 + 7) / 8;
        const size_t n = (size_t)std::max(1, pw) * std::max(1, ph);
        if (cudaMalloc(&c->pcls_mem, n * sizeof(uint16_t)) != cudaSuccess) return fail(H2D_ERR_NOMEM);
        if (cudaMemset(c->pcls_mem, 0xFF, n * sizeof(uint16_t)) != cudaSuccess) return fail(H2D_ERR_DEVICE);
        d.pcls = static_cast<uint16_t*>(c->pcls_mem);
        d.pcls_nx = std::max(1, pw);
    }
    if (ctl_push(c)) return fail(H2D_ERR_DEVICE);
    // make_state defaults (state.cpp:5-23): k0 = 1, normals (1, 0), vol = dx*dy
    for (int p = 0; p < 2; ++p) {
        if (fill_plane(c, c->sb[p].k[0], 1.0) || (p == 0 || !shared_nrm ? fill_plane(c, c->sb[p].nrx, 1.0) : 0) ||
            fill_plane(c, c->sb[p].vol, d.cv))
            return fail(H2D_ERR_DEVICE);
    }
    if (make_tmas(c)) return fail(H2D_ERR_DEVICE);
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return fail(H2D_ERR_DEVICE);
    *out = c;
    return 0;
}
}  // namespace

extern "C" {

void h2d_destroy(h2d_ctx* c) {
    if (!c) return;
    if (c->device >= 0) cudaSetDevice(c->device);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->flush) cudaFree(c->flush);
    for (auto& g : c->graph)
        if (g) cudaGraphExecDestroy(g);
    for (auto& gp : c->graph_ad)
        for (auto& g : gp)
            if (g) cudaGraphExecDestroy(g);
    for (auto& g : c->graph_dir)
        if (g) cudaGraphExecDestroy(g);
    for (auto& g : c->graph_rest)
        if (g) cudaGraphExecDestroy(g);
    if (c->ad_mem) cudaFree(c->ad_mem);
    if (c->st) cudaStreamSynchronize(c->st);
    if (c->arena) cudaFree(c->arena);
    if (c->ctl) cudaFree(c->ctl);
    if (c->hctl) cudaFreeHost(c->hctl);
    if (c->dt_log) cudaFree(c->dt_log);
    if (c->diag_log) cudaFree(c->diag_log);
    if (c->diag_mem) cudaFree(c->diag_mem);
    if (c->tcls_mem) cudaFree(c->tcls_mem);
    if (c->pcls_mem) cudaFree(c->pcls_mem);
    if (c->xbuf) cudaFree(c->xbuf);
    if (c->st) cudaStreamDestroy(c->st);
    delete c;
}

int h2d_upload_state(h2d_ctx* c, const h2d_state* v) {
    cudaSetDevice(c->device);
    const int nx = c->nx, ny = c->ny;
    StateBufs& s = c->sb[c->cur];
    for (int a = 0; a < c->nmat; ++a) {
        if (int rc = put_plane(c, s.m[a], v->m[a], nx, ny)) return rc;
        if (int rc = put_plane(c, s.e[a], v->e[a], nx, ny)) return rc;
        if (int rc = put_plane(c, s.k[a], v->k[a], nx, ny)) return rc;
    }
    if (int rc = put_vec(c, s.nrx, s.nry, v->iface_normal, nx, ny)) return rc;
    if (int rc = put_vec(c, s.ux, s.uy, v->u, nx + 1, ny + 1)) return rc;
    const bool derived = v->vol && v->m_mix && v->e_mix && v->rho_mix && v->p_mix;
    if (derived) {
        if (int rc = put_plane(c, s.vol, v->vol, nx, ny)) return rc;
        if (int rc = put_plane(c, s.m_mix, v->m_mix, nx, ny)) return rc;
        if (int rc = put_plane(c, s.e_mix, v->e_mix, nx, ny)) return rc;
        if (int rc = put_plane(c, s.rho_mix, v->rho_mix, nx, ny)) return rc;
        if (int rc = put_plane(c, s.p_mix, v->p_mix, nx, ny)) return rc;
    }
    if (int rc = ctl_pull(c)) return rc;
    c->hctl->step = v->step;
    c->hctl->time = v->time;
    if (int rc = ctl_push(c)) return rc;
    c->derived_stale = false;
    if (!derived) return h2d_sync_derived(c);
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

int h2d_download_state(h2d_ctx* c, h2d_state* v) {
    cudaSetDevice(c->device);
    if (int rc_ = ensure_derived(c)) return rc_;
    cudaSetDevice(c->device);
    const int nx = c->nx, ny = c->ny;
    const StateBufs& s = c->sb[c->cur];
    for (int a = 0; a < c->nmat; ++a) {
        if (int rc = get_plane(c, v->m[a], s.m[a], nx, ny)) return rc;
        if (int rc = get_plane(c, v->e[a], s.e[a], nx, ny)) return rc;
        if (int rc = get_plane(c, v->k[a], s.k[a], nx, ny)) return rc;
    }
    if (int rc = get_plane(c, v->vol, s.vol, nx, ny)) return rc;
    if (int rc = get_plane(c, v->m_mix, s.m_mix, nx, ny)) return rc;
    if (int rc = get_plane(c, v->e_mix, s.e_mix, nx, ny)) return rc;
    if (int rc = get_plane(c, v->rho_mix, s.rho_mix, nx, ny)) return rc;
    if (int rc = get_plane(c, v->p_mix, s.p_mix, nx, ny)) return rc;
    if (v->iface_normal) {
        if (int rc = get_vec(c, v->iface_normal, s.nrx, s.nry, nx, ny)) return rc;
        CK(cudaStreamSynchronize(c->st));  // staging buffer reuse
    }
    if (int rc = get_vec(c, v->u, s.ux, s.uy, nx + 1, ny + 1)) return rc;
    if (int rc = ctl_pull(c)) return rc;
    v->step = c->hctl->step;
    v->time = c->hctl->time;
    return 0;
}

int h2d_fill_ghosts(h2d_ctx* c) {
    cudaSetDevice(c->device);
    if (int rc = fill_ghosts_cur(c, c->cur)) return rc;
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

int h2d_sync_derived(h2d_ctx* c) {
    cudaSetDevice(c->device);
    c->derived_stale = false;
    launch_sync(make_dev(c, c->cur, 1), 0, 0, c->st);
    if (int rc = check_launch(c)) return rc;
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

int h2d_update_interface_normals(h2d_ctx* c) {
    cudaSetDevice(c->device);
    if (c->nmat < 2) return 0;
    const Dev d = make_dev(c, c->cur, 1);
    launch_normals_api(d, c->st);
    FieldList fl{};
    fl.respect_halt = 0;
    fl.n = 2;
    fl.f[0] = c->sb[c->cur].nrx;
    fl.f[1] = c->sb[c->cur].nry;
    launch_ghost_cells(d, fl, c->st);
    if (int rc = check_launch(c)) return rc;
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

int h2d_cfl_dt(h2d_ctx* c, double cfl, double* dt) {
    cudaSetDevice(c->device);
    if (int rc_ = ensure_derived(c)) return rc_;
    cudaSetDevice(c->device);
    if (int rc = ctl_reset(c)) return rc;
    c->hctl->cfl = cfl;
    if (int rc = ctl_push(c)) return rc;
    const Dev d = make_dev(c, c->cur, 1);
    launch_begin(c->ctl, 2, 0.0, c->st);
    launch_cfl(d, 0, c->st);
    if (int rc = check_launch(c)) return rc;
    if (int rc = ctl_pull(c)) return rc;
    if (int rc = decode_error(c, false)) return rc;
    *dt = c->hctl->dt;
    return 0;
}

int h2d_lagrange_step(h2d_ctx* c, double dt, h2d_lagrange* out) {
    cudaSetDevice(c->device);
    if (int rc_ = ensure_derived(c)) return rc_;
    cudaSetDevice(c->device);
    c->have_lag = false;
    if (int rc = ctl_reset(c)) return rc;
    const Dev d = make_dev(c, c->cur, 1);
    if (int rc = zero_plane(c, d.vol_lag)) return rc;
    launch_begin(c->ctl, 1, dt, c->st);
    launch_lagrange(d, 1, c->st);
    if (int rc = check_launch(c)) return rc;
    if (int rc = ctl_pull(c)) return rc;
    if (int rc = decode_error(c, false)) return rc;
    c->have_lag = true;
    if (out) {
        const int nx = c->nx, ny = c->ny;
        if (int rc = get_vec(c, out->u_half, d.uhx, d.uhy, nx + 1, ny + 1)) return rc;
        CK(cudaStreamSynchronize(c->st));
        if (int rc = get_vec(c, out->u_lag, d.ulx, d.uly, nx + 1, ny + 1)) return rc;
        for (int a = 0; a < c->nmat; ++a)
            if (int rc = get_plane(c, out->e_lag[a], d.el[a], nx, ny)) return rc;
        if (int rc = get_plane(c, out->vol_lag, d.vol_lag, nx, ny)) return rc;
        if (int rc = get_plane(c, out->q, d.q, nx, ny)) return rc;
        CK(cudaStreamSynchronize(c->st));
        out->floor_count = c->hctl->step_floor;
    }
    return 0;
}

int h2d_set_lagrange(h2d_ctx* c, const h2d_lagrange* in) {
    cudaSetDevice(c->device);
    const int nx = c->nx, ny = c->ny;
    const Dev& d = c->base;
    double* planes[] = {d.uhx, d.uhy, d.ulx, d.uly, d.vol_lag, d.q, d.el[0], d.el[1], d.el[2]};
    for (double* p : planes)
        if (p)
            if (int rc = zero_plane(c, p)) return rc;
    if (int rc = put_vec(c, d.uhx, d.uhy, in->u_half, nx + 1, ny + 1)) return rc;
    CK(cudaStreamSynchronize(c->st));
    if (int rc = put_vec(c, d.ulx, d.uly, in->u_lag, nx + 1, ny + 1)) return rc;
    for (int a = 0; a < c->nmat; ++a)
        if (int rc = put_plane(c, d.el[a], in->e_lag[a], nx, ny)) return rc;
    if (int rc = put_plane(c, d.vol_lag, in->vol_lag, nx, ny)) return rc;
    if (int rc = put_plane(c, d.q, in->q, nx, ny)) return rc;
    CK(cudaStreamSynchronize(c->st));
    c->have_lag = true;
    return 0;
}

int h2d_remap_step(h2d_ctx* c, double dt, int kind, int x_first, int remap_velocity, h2d_remap_diag* diag) {
    cudaSetDevice(c->device);
    if (int rc_ = ensure_derived(c)) return rc_;
    cudaSetDevice(c->device);
    if (kind != H2D_REMAP_DIRECTCF && !(kind == H2D_REMAP_AD && !c->is_block && c->nmat <= 2) &&
        !(kind == H2D_REMAP_DIRECT && !c->is_block)) {
        set_err(c, H2D_ERR_INVALID, "the device runs DirectCF, Direct and (single-domain, <= 2 materials) AD");
        return H2D_ERR_INVALID;
    }
    if (!c->have_lag) {
        set_err(c, H2D_ERR_INVALID, "remap_step without a LagrangeResult");
        return H2D_ERR_INVALID;
    }
    if (kind == H2D_REMAP_AD)
        if (int rc = ensure_ad(c)) return rc;
    if (int rc = ctl_reset(c)) return rc;
    Dev d = make_dev(c, c->cur, remap_velocity != 0);
    d.direct = kind == H2D_REMAP_DIRECT;
    launch_begin(c->ctl, 1, dt, c->st);
    if (kind == H2D_REMAP_AD)
        launch_remap_ad(d, c->adw, x_first != 0, remap_velocity != 0, 0, c->st);
    else
        launch_remap(d, c->st);
    launch_commit(c->ctl, 1, c->st);
    if (int rc = check_launch(c)) return rc;
    if (int rc = ctl_pull(c)) return rc;
    if (int rc = decode_error(c, false)) return rc;
    c->cur = c->hctl->cur;
    if (diag) {
        const double v = __builtin_bit_cast(double, (unsigned long long)c->hctl->kviol_bits);
        if (v > diag->max_k_violation) diag->max_k_violation = v;
        diag->k_clip_count += c->hctl->step_clip;
        diag->mass_fix_count += c->hctl->step_fix;
    }
    return 0;
}

// ---- sub-step entry points (lagrange.hpp predict / correct, remap.hpp
// remap_single_axis) and the scalar kernels ---------------------------------
int h2d_predict(h2d_ctx* c, double dt, h2d_half* out) {
    cudaSetDevice(c->device);
    if (int rc_ = ensure_derived(c)) return rc_;
    cudaSetDevice(c->device);
    c->have_lag = false;
    if (c->is_block) {
        set_err(c, H2D_ERR_INVALID, "predict on a block context");
        return H2D_ERR_INVALID;
    }
    if (int rc = ctl_reset(c)) return rc;
    Dev d = make_dev(c, c->cur, 1);
    // vol_half / e_half land in the vol_lag / e_lag scratch (predict writes
    // no e_lag); interior only, zero ghosts like the reference's Field(nx, ny)
    d.volh = d.vol_lag;
    if (int rc = zero_plane(c, d.vol_lag)) return rc;
    for (int a = 0; a < c->nmat; ++a) {
        d.eh[a] = d.el[a];
        if (int rc = zero_plane(c, d.el[a])) return rc;
    }
    launch_begin(c->ctl, 1, dt, c->st);
    launch_lagrange_mode(d, 0, 1, c->st);
    launch_xhalf(d, d.ulx, d.uly, c->st);  // x_half in the u_lag scratch (predict has no u_lag)
    if (int rc = check_launch(c)) return rc;
    if (int rc = ctl_pull(c)) return rc;
    if (int rc = decode_error(c, false)) return rc;
    if (out) {
        const int nx = c->nx, ny = c->ny;
        if (int rc = get_vec(c, out->u_half, d.uhx, d.uhy, nx + 1, ny + 1)) return rc;
        CK(cudaStreamSynchronize(c->st));
        if (int rc = get_vec(c, out->x_half, d.ulx, d.uly, nx + 1, ny + 1)) return rc;
        CK(cudaStreamSynchronize(c->st));
        if (int rc = get_plane(c, out->vol_half, d.vol_lag, nx, ny)) return rc;
        for (int a = 0; a < c->nmat; ++a) {
            if (int rc = get_plane(c, out->e_half[a], d.el[a], nx, ny)) return rc;
            if (int rc = get_plane(c, out->p_half[a], d.ph[a], nx, ny)) return rc;
        }
        if (int rc = get_plane(c, out->p_mix_half, d.pmh, nx, ny)) return rc;
        if (int rc = get_plane(c, out->q, d.q, nx, ny)) return rc;
        CK(cudaStreamSynchronize(c->st));
        out->floor_count = c->hctl->step_floor;
    }
    return 0;
}

int h2d_correct(h2d_ctx* c, double dt, const h2d_half* in, h2d_lagrange* out) {
    cudaSetDevice(c->device);
    if (int rc_ = ensure_derived(c)) return rc_;
    cudaSetDevice(c->device);
    c->have_lag = false;
    if (c->is_block || !in || !in->u_half || !in->q) {
        set_err(c, H2D_ERR_INVALID, "correct needs a single-domain context and a HalfStepState");
        return H2D_ERR_INVALID;
    }
    const int nx = c->nx, ny = c->ny;
    Dev d = make_dev(c, c->cur, 1);
    if (int rc = put_vec(c, d.uhx, d.uhy, in->u_half, nx + 1, ny + 1)) return rc;
    CK(cudaStreamSynchronize(c->st));
    if (int rc = put_plane(c, d.q, in->q, nx, ny)) return rc;
    for (int a = 0; a < c->nmat; ++a) {
        if (in->p_half[a]) {
            if (int rc = put_plane(c, d.ph[a], in->p_half[a], nx, ny)) return rc;
        } else if (int rc = zero_plane(c, d.ph[a])) {
            return rc;
        }
    }
    if (int rc = zero_plane(c, d.vol_lag)) return rc;
    if (int rc = ctl_reset(c)) return rc;
    launch_begin(c->ctl, 1, dt, c->st);
    launch_lagrange_mode(d, 1, 2, c->st);
    if (int rc = check_launch(c)) return rc;
    if (int rc = ctl_pull(c)) return rc;
    if (int rc = decode_error(c, false)) return rc;
    c->have_lag = true;
    if (out) {
        if (int rc = get_vec(c, out->u_half, d.uhx, d.uhy, nx + 1, ny + 1)) return rc;
        CK(cudaStreamSynchronize(c->st));
        if (int rc = get_vec(c, out->u_lag, d.ulx, d.uly, nx + 1, ny + 1)) return rc;
        for (int a = 0; a < c->nmat; ++a)
            if (int rc = get_plane(c, out->e_lag[a], d.el[a], nx, ny)) return rc;
        if (int rc = get_plane(c, out->vol_lag, d.vol_lag, nx, ny)) return rc;
        if (int rc = get_plane(c, out->q, d.q, nx, ny)) return rc;
        CK(cudaStreamSynchronize(c->st));
        out->floor_count = c->hctl->step_floor + in->floor_count;
    }
    return 0;
}

int h2d_remap_single_axis(h2d_ctx* c, double dt, int axis_x, int remap_velocity, h2d_remap_diag* diag) {
    cudaSetDevice(c->device);
    if (int rc_ = ensure_derived(c)) return rc_;
    cudaSetDevice(c->device);
    if (c->is_block || c->nmat > 2) {
        set_err(c, H2D_ERR_INVALID, "remap_single_axis runs on single-domain contexts with <= 2 materials");
        return H2D_ERR_INVALID;
    }
    if (!c->have_lag) {
        set_err(c, H2D_ERR_INVALID, "remap_single_axis without a LagrangeResult");
        return H2D_ERR_INVALID;
    }
    if (int rc = ensure_ad(c)) return rc;
    if (int rc = ctl_reset(c)) return rc;
    Dev d = make_dev(c, c->cur, remap_velocity != 0);
    launch_begin(c->ctl, 1, dt, c->st);
    launch_remap_single_axis(d, c->adw, axis_x != 0, remap_velocity != 0, c->st);
    launch_commit(c->ctl, 1, c->st);
    if (int rc = check_launch(c)) return rc;
    if (int rc = ctl_pull(c)) return rc;
    if (int rc = decode_error(c, false)) return rc;
    c->cur = c->hctl->cur;
    if (diag) {
        const double v = __builtin_bit_cast(double, (unsigned long long)c->hctl->kviol_bits);
        if (v > diag->max_k_violation) diag->max_k_violation = v;
        diag->k_clip_count += c->hctl->step_clip;
        diag->mass_fix_count += c->hctl->step_fix;
    }
    return 0;
}

namespace {
// device scratch of h2d_scalar_eval (per host thread, grown on demand)
struct ScalarScratch {
    int device = -1;
    double *in = nullptr, *out = nullptr;
    int* flags = nullptr;
    int cap = 0;
    ~ScalarScratch() {
        if (in) cudaFree(in);
        if (out) cudaFree(out);
        if (flags) cudaFree(flags);
    }
};
thread_local ScalarScratch g_scalar;
}  // namespace

int h2d_scalar_eval(int op, int n, const double* in, double* out, int* flags) {
    if (n < 0 || op < H2D_SC_VAN_LEER || op > H2D_SC_AD_FACE_FLUX) return H2D_ERR_INVALID;
    if (n == 0) return 0;
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return H2D_ERR_DEVICE;
    ScalarScratch& s = g_scalar;
    if (s.device != dev || s.cap < n) {
        if (s.in) cudaFree(s.in);
        if (s.out) cudaFree(s.out);
        if (s.flags) cudaFree(s.flags);
        s.in = s.out = nullptr;
        s.flags = nullptr;
        const int cap = n < 1024 ? 1024 : n;
        if (cudaMalloc(&s.in, (size_t)cap * H2D_SC_IN * sizeof(double)) != cudaSuccess ||
            cudaMalloc(&s.out, (size_t)cap * H2D_SC_OUT * sizeof(double)) != cudaSuccess ||
            cudaMalloc(&s.flags, (size_t)cap * sizeof(int)) != cudaSuccess) {
            s.cap = 0;
            return H2D_ERR_DEVICE;
        }
        s.cap = cap;
        s.device = dev;
    }
    if (cudaMemcpy(s.in, in, (size_t)n * H2D_SC_IN * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
        return H2D_ERR_DEVICE;
    launch_scalar(op, n, s.in, s.out, s.flags, nullptr);
    if (cudaGetLastError() != cudaSuccess) return H2D_ERR_DEVICE;
    if (cudaMemcpy(out, s.out, (size_t)n * H2D_SC_OUT * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
        return H2D_ERR_DEVICE;
    if (flags && cudaMemcpy(flags, s.flags, (size_t)n * sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
        return H2D_ERR_DEVICE;
    return 0;
}

int h2d_run(h2d_ctx* c, h2d_run_args* a) {
    cudaSetDevice(c->device);
    a->steps_done = 0;
    const bool ad = a->remap_kind == H2D_REMAP_AD, dir = a->remap_kind == H2D_REMAP_DIRECT;
    if (a->remap_kind != H2D_REMAP_DIRECTCF && !(ad && !c->is_block && c->nmat <= 2) && !(dir && !c->is_block)) {
        set_err(c, H2D_ERR_INVALID, "the device runs DirectCF, Direct and (single-domain, <= 2 materials) AD");
        return H2D_ERR_INVALID;
    }
    const int cap = a->max_steps > 0 ? a->max_steps : kRunLogCap;
    if (int rc = ensure_logs(c, cap)) return rc;
    if (int rc = ctl_reset(c)) return rc;
    Ctl& h = *c->hctl;
    h.t_end = a->t_end;
    h.cfl = a->cfl;
    h.max_steps = a->max_steps;
    h.steps_done = 0;
    h.floor_count = 0;
    h.k_clip_count = 0;
    h.mass_fix_count = 0;
    h.max_k_violation = a->diag.max_k_violation;
    h.dt_log = c->dt_log;
    h.dt_log_cap = c->dt_log_cap;
    h.diag_log = c->diag_log;
    h.diag_log_cap = c->dt_log_cap;
    if (int rc = ctl_push(c)) return rc;
    int parity = c->cur;
    int rc = 0;
    if ((rc = ad ? ensure_graphs_ad(c) : (dir ? ensure_graphs_dir(c) : ensure_graphs(c)))) return rc;
    enqueue_cfl_next(c);
    start_first(c);
    // Launch in chunks; the device control block turns every kernel after the
    // loop condition fails (or after an error) into a no-op.
    for (;;) {
        int chunk = 32;
        if (a->max_steps > 0) {
            const int left = a->max_steps - h.step;
            if (left <= 0) break;
            chunk = left < chunk ? left : chunk;
        }
        const int step0 = h.step;
        for (int q = 0; q < chunk; ++q) {
            if (ad) {  // x_first = s.step % 2 == 0 (harness.cpp:401)
                CK(cudaGraphLaunch(c->graph_ad[parity][(step0 + q) % 2 == 0], c->st));
                add_launches(c->graph_kernels_ad);
            } else if (dir) {
                CK(cudaGraphLaunch(c->graph_dir[parity], c->st));
                add_launches(c->graph_kernels);
            } else if ((rc = launch_step_graph(c, parity))) {
                return rc;
            }
            parity ^= 1;
        }
        if ((rc = check_launch(c))) return rc;
        if ((rc = ctl_pull(c))) return rc;
        parity = h.cur;
        if (h.err_key != kNoErr || h.done) break;
    }
    c->cur = h.cur;
    c->derived_stale = true;
    a->steps_done = h.steps_done;
    a->floor_count += h.floor_count;
    a->diag.k_clip_count += h.k_clip_count;
    a->diag.mass_fix_count += h.mass_fix_count;
    a->diag.max_k_violation = h.max_k_violation;
    if (a->dt_log && h.steps_done > 0) {
        const int n = h.steps_done < a->dt_log_cap ? h.steps_done : a->dt_log_cap;
        CK(cudaMemcpy(a->dt_log, c->dt_log, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost));
    }
    if (int rc = copy_series(c, a->series, h.steps_done < a->series_cap ? h.steps_done : a->series_cap)) return rc;
    c->have_lag = false;
    return decode_error(c, true);
}

static int totals7(h2d_ctx* c, double out[7]);
int h2d_totals(h2d_ctx* c, double out[6]) {
    double t[7];
    if (int rc = totals7(c, t)) return rc;
    for (int q = 0; q < 6; ++q) out[q] = t[q];
    return 0;
}

// {mass, mass_mat0, mass_mat1, momentum x, momentum y, internal energy, mass_mat2}
static int totals7(h2d_ctx* c, double out[7]) {
    cudaSetDevice(c->device);
    if (int rc_ = ensure_derived(c)) return rc_;
    // compute_totals (state.cpp:145-160) is a serial fp64 sum: read the
    // fields back and add them in the reference order so totals are exact.
    cudaSetDevice(c->device);
    const int nx = c->nx, ny = c->ny;
    const size_t W = (size_t)nx + 2 * G, Wn = W + 1;
    std::vector<double> m_mix(W * (ny + 2 * G)), e_mix(m_mix.size()), m0(m_mix.size()), m1(m_mix.size()),
        m2(m_mix.size());
    std::vector<double> u(Wn * (ny + 1 + 2 * G) * 2);
    const StateBufs& s = c->sb[c->cur];
    if (int rc = get_plane(c, m_mix.data(), s.m_mix, nx, ny)) return rc;
    if (int rc = get_plane(c, e_mix.data(), s.e_mix, nx, ny)) return rc;
    if (int rc = get_plane(c, m0.data(), s.m[0], nx, ny)) return rc;
    if (c->nmat >= 2)
        if (int rc = get_plane(c, m1.data(), s.m[1], nx, ny)) return rc;
    if (c->nmat == 3)
        if (int rc = get_plane(c, m2.data(), s.m[2], nx, ny)) return rc;
    if (int rc = get_vec(c, u.data(), s.ux, s.uy, nx + 1, ny + 1)) return rc;
    CK(cudaStreamSynchronize(c->st));
    auto C = [&](const std::vector<double>& f, int i, int j) { return f[(size_t)(j + G) * W + (i + G)]; };
    double mass = 0.0, ie = 0.0, mm0 = 0.0, mm1 = 0.0, mm2 = 0.0, px = 0.0, py = 0.0;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            mass += C(m_mix, i, j);
            ie += C(m_mix, i, j) * C(e_mix, i, j);
            mm0 += C(m0, i, j);
            if (c->nmat >= 2) mm1 += C(m1, i, j);
            if (c->nmat == 3) mm2 += C(m2, i, j);
        }
    const bool px_ = c->cfg.mesh.bc_x == H2D_BC_PERIODIC, py_ = c->cfg.mesh.bc_y == H2D_BC_PERIODIC;
    const int ie_ = px_ ? nx - 1 : nx, je_ = py_ ? ny - 1 : ny;
    for (int j = 0; j <= je_; ++j)
        for (int i = 0; i <= ie_; ++i) {
            const double mp =
                0.25 * (C(m_mix, i - 1, j - 1) + C(m_mix, i, j - 1) + C(m_mix, i - 1, j) + C(m_mix, i, j));
            const size_t n = (size_t)(j + G) * Wn + (i + G);
            px += mp * u[2 * n];
            py += mp * u[2 * n + 1];
        }
    out[0] = mass;
    out[1] = mm0;
    out[2] = mm1;
    out[3] = px;
    out[4] = py;
    out[5] = ie;
    out[6] = mm2;
    return 0;
}

int h2d_step_diag_now(h2d_ctx* c, double dt, h2d_step_diag* out) {
    cudaSetDevice(c->device);
    if (int rc_ = ensure_derived(c)) return rc_;
    // make_diag (harness.cpp:360-376) on the host, in the reference's order
    double t[7];
    if (int rc = totals7(c, t)) return rc;
    const int nx = c->nx, ny = c->ny;
    const size_t W = (size_t)nx + 2 * G;
    std::vector<double> rho(W * (ny + 2 * G)), p(rho.size());
    const StateBufs& s = c->sb[c->cur];
    if (int rc = get_plane(c, rho.data(), s.rho_mix, nx, ny)) return rc;
    if (int rc = get_plane(c, p.data(), s.p_mix, nx, ny)) return rc;
    CK(cudaStreamSynchronize(c->st));
    if (int rc = ctl_pull(c)) return rc;
    auto C = [&](const std::vector<double>& f, int i, int j) { return f[(size_t)(j + G) * W + (i + G)]; };
    h2d_step_diag d{};
    d.step = c->hctl->step;
    d.t = c->hctl->time;
    d.dt = dt;
    d.mass = t[0];
    d.mass_mat[0] = t[1];
    d.mass_mat[1] = t[2];
    d.mass_mat[2] = t[6];
    d.momentum_x = t[3];
    d.momentum_y = t[4];
    d.internal_energy = t[5];
    d.min_rho = d.max_rho = C(rho, 0, 0);
    d.min_p = d.max_p = C(p, 0, 0);
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            d.min_rho = std::min(d.min_rho, C(rho, i, j));
            d.max_rho = std::max(d.max_rho, C(rho, i, j));
            d.min_p = std::min(d.min_p, C(p, i, j));
            d.max_p = std::max(d.max_p, C(p, i, j));
        }
    *out = d;
    return 0;
}

// host staging of the whole reference State of a single-domain context
struct HostStage {
    std::vector<double> buf;
    h2d_state v{};
    HostStage(int nx, int ny, int nmat) {
        const size_t nc = (size_t)(nx + 2 * G) * (ny + 2 * G), nn = (size_t)(nx + 1 + 2 * G) * (ny + 1 + 2 * G);
        buf.assign(nc * (3 * (size_t)nmat + 5 + 2) + 2 * nn, 0.0);
        double* p = buf.data();
        auto take = [&](size_t n) {
            double* q = p;
            p += n;
            return q;
        };
        for (int a = 0; a < nmat; ++a) v.m[a] = take(nc);
        for (int a = 0; a < nmat; ++a) v.e[a] = take(nc);
        for (int a = 0; a < nmat; ++a) v.k[a] = take(nc);
        v.vol = take(nc);
        v.m_mix = take(nc);
        v.e_mix = take(nc);
        v.rho_mix = take(nc);
        v.p_mix = take(nc);
        v.iface_normal = take(2 * nc);
        v.u = take(2 * nn);
    }
};

int h2d_write_fields(h2d_ctx* c, const char* path, int fmt) {
    if (c->is_block) {
        set_err(c, H2D_ERR_INVALID, "write_fields: single-domain contexts only");
        return H2D_ERR_INVALID;
    }
    HostStage h(c->nx, c->ny, c->nmat);
    if (int rc = h2d_download_state(c, &h.v)) return rc;
    const int rc = h2d_write_fields_host(&c->cfg, &h.v, path, fmt);
    if (rc == H2D_ERR_SIM) set_err(c, rc, (std::string("cannot write: ") + (path ? path : "")).c_str());
    if (rc == H2D_ERR_INVALID) set_err(c, rc, "write_fields: bad format or path");
    return rc;
}

int h2d_save_state(h2d_ctx* c, const char* path) {
    if (c->is_block) {
        set_err(c, H2D_ERR_INVALID, "save_state: single-domain contexts only");
        return H2D_ERR_INVALID;
    }
    HostStage h(c->nx, c->ny, c->nmat);
    if (int rc = h2d_download_state(c, &h.v)) return rc;
    const int rc = h2d_save_state_host(&c->cfg, &h.v, path);
    if (rc) set_err(c, rc, (std::string("cannot write checkpoint: ") + (path ? path : "")).c_str());
    return rc;
}

int h2d_load_state(h2d_ctx* c, const char* path) {
    if (c->is_block) {
        set_err(c, H2D_ERR_INVALID, "load_state: single-domain contexts only");
        return H2D_ERR_INVALID;
    }
    HostStage h(c->nx, c->ny, c->nmat);
    const int rc = h2d_load_state_host(&c->cfg, &h.v, path);
    if (rc) {
        set_err(c, rc, (std::string("cannot read a checkpoint of this mesh: ") + (path ? path : "")).c_str());
        return rc;
    }
    return h2d_upload_state(c, &h.v);
}

int h2d_step_timed(h2d_ctx* c, double cfl, double t_end, int phases, int remap_kind, float ms[8]) {
    c->derived_stale = true;  // run-loop steps keep no derived planes
    cudaSetDevice(c->device);
    const bool ad = remap_kind == H2D_REMAP_AD, dir = remap_kind == H2D_REMAP_DIRECT;
    if (!(remap_kind == H2D_REMAP_DIRECTCF || (ad && !c->is_block && c->nmat <= 2) || (dir && !c->is_block))) {
        set_err(c, H2D_ERR_INVALID, "h2d_step_timed: DirectCF, Direct or (single-domain) AD only");
        return H2D_ERR_INVALID;
    }
    if (ad)
        if (int rc = ensure_graphs_ad(c)) return rc;
    if (dir)
        if (int rc = ensure_graphs_dir(c)) return rc;
    const int xf = c->hctl->step % 2 == 0;  // harness.cpp:401
    if (!c->ev[0])
        for (auto& e : c->ev) CK(cudaEventCreate(&e));
    if (int rc = ctl_reset(c)) return rc;
    Ctl& h = *c->hctl;
    h.t_end = t_end;
    h.cfl = cfl;
    h.max_steps = 0;
    h.steps_done = 0;
    h.dt_log = nullptr;
    h.dt_log_cap = 0;
    if (int rc = ctl_push(c)) return rc;
    // the wave speed of the current State (normally left by the previous
    // step's k_post) is recomputed outside the timed region
    enqueue_cfl_next(c);
    for (int q = 0; q < 8; ++q) ms[q] = 0.0f;
    if (phases) {  // un-graphed launches with events between the kernels / groups
        Dev d = make_dev(c, c->cur, 1);
        d.scan_nodes = 1;  // as the run-loop graph
        d.diag = 1;
        d.direct = dir;
        d.cls_post = d.pcls != nullptr;
        CK(cudaEventRecord(c->ev[0], c->st));
        launch_step_start(d, c->st);
        CK(cudaEventRecord(c->ev[1], c->st));
        launch_lag_fused(d, c->st);
        CK(cudaEventRecord(c->ev[2], c->st));
        launch_lag_ghosts(d, c->st);
        CK(cudaEventRecord(c->ev[3], c->st));
        if (ad) {  // both AD passes and the post kernels in the remap slot
            launch_remap_ad(d, c->adw, xf, 1, 1, c->st);
            CK(cudaEventRecord(c->ev[4], c->st));
            CK(cudaEventRecord(c->ev[5], c->st));
            CK(cudaEventRecord(c->ev[6], c->st));
        } else {
            launch_remap_tile(d, c->st);
            CK(cudaEventRecord(c->ev[4], c->st));
            launch_remap_slivers(d, c->st);
            CK(cudaEventRecord(c->ev[5], c->st));
            launch_remap_dual(d, c->st);
            CK(cudaEventRecord(c->ev[6], c->st));
            launch_post(d, 1, c->st);
        }
        CK(cudaEventRecord(c->ev[7], c->st));
        launch_tail(d, 0, c->st);
        CK(cudaEventRecord(c->ev[8], c->st));
        if (int rc = check_launch(c)) return rc;
        CK(cudaEventSynchronize(c->ev[8]));
        float t[8];
        for (int q = 0; q < 8; ++q) CK(cudaEventElapsedTime(&t[q], c->ev[q], c->ev[q + 1]));
        ms[0] = t[0];         // step start
        ms[1] = t[1];         // k_lag_fused
        ms[2] = t[3];         // k_remap_tile
        ms[3] = t[4];         // slivers + Work / flux ghosts
        ms[4] = t[5];         // dual-mesh momentum
        ms[5] = t[6];         // k_post
        ms[7] = t[2] + t[7];  // Lagrange ghosts, post ghosts + commit
        CK(cudaEventElapsedTime(&ms[6], c->ev[0], c->ev[8]));
    } else {  // the production path: one graph launch
        if (int rc = ensure_graphs(c)) return rc;
        start_first(c);  // (the graph's own k_tail starts the step after it)
        CK(cudaEventRecord(c->ev[0], c->st));
        if (ad) {
            CK(cudaGraphLaunch(c->graph_ad[c->cur][xf], c->st));
            add_launches(c->graph_kernels_ad);
        } else if (dir) {
            CK(cudaGraphLaunch(c->graph_dir[c->cur], c->st));
            add_launches(c->graph_kernels);
        } else if (int rc = launch_step_graph(c, c->cur)) {
            return rc;
        }
        CK(cudaEventRecord(c->ev[8], c->st));
        CK(cudaEventSynchronize(c->ev[8]));
        CK(cudaEventElapsedTime(&ms[6], c->ev[0], c->ev[8]));
    }
    if (int rc = ctl_pull(c)) return rc;
    c->cur = h.cur;
    return decode_error(c, true);
}

int h2d_flush_l2(h2d_ctx* c, long long bytes) {
    cudaSetDevice(c->device);
    if ((size_t)bytes > c->flush_bytes) {
        if (c->flush) cudaFree(c->flush);
        c->flush = nullptr;
        CK(cudaMalloc(&c->flush, (size_t)bytes));
        c->flush_bytes = (size_t)bytes;
    }
    CK(cudaMemsetAsync(c->flush, c->flush_bytes & 0xFF, c->flush_bytes, c->st));
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

// ---- 2D block decomposition -------------------------------------------------

namespace {

int ensure_xbuf(h2d_ctx* c, size_t bytes) {
    if (bytes <= c->xbuf_bytes) return 0;
    if (c->xbuf) cudaFree(c->xbuf);
    c->xbuf = nullptr;
    c->xbuf_bytes = 0;
    CK(cudaMalloc(&c->xbuf, bytes));
    c->xbuf_bytes = bytes;
    return 0;
}

// global-layout host planes <-> this block's planes over rectangle r: only
// the rectangle's rows are copied (strided 2D copy into a compact buffer)
int global_rect(h2d_ctx* c, double* host, int vec, bool node, Rng r, double* px, double* py, bool upload) {
    if (!host || r.i1 <= r.i0 || r.j1 <= r.j0) return 0;
    const int W = c->nx + (node ? 1 : 0) + 2 * G;
    const int w = r.i1 - r.i0, h = r.j1 - r.j0, e = vec ? 2 : 1;
    const size_t bytes = (size_t)w * h * e * sizeof(double);
    if (int rc = ensure_xbuf(c, bytes)) return rc;
    const Dev d = make_dev(c, c->cur, 1);
    double* hstart = host + ((size_t)(r.j0 + G) * W + (r.i0 + G)) * e;
    const size_t hpitch = (size_t)W * e * sizeof(double), row = (size_t)w * e * sizeof(double);
    if (upload) {
        CK(cudaMemcpy2DAsync(c->xbuf, row, hstart, hpitch, row, (size_t)h, cudaMemcpyHostToDevice, c->st));
        launch_global_xfer(d, c->xbuf, r, px, py, vec, 1, c->st);
    } else {
        launch_global_xfer(d, c->xbuf, r, px, py, vec, 0, c->st);
        CK(cudaMemcpy2DAsync(hstart, hpitch, c->xbuf, row, row, (size_t)h, cudaMemcpyDeviceToHost, c->st));
    }
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

// state planes exchanged with the neighbours: cells and nodes
void state_lists(h2d_ctx* c, FieldList& cl, FieldList& nl) {
    const StateBufs& sb = c->sb[c->cur];
    cl = FieldList{};
    nl = FieldList{};
    for (int a = 0; a < c->nmat; ++a) {
        cl.f[cl.n++] = sb.m[a];
        cl.f[cl.n++] = sb.e[a];
        cl.f[cl.n++] = sb.k[a];
    }
    // (the derived planes are not part of the exchange: the step rebuilds
    // what it needs from m and k, ensure_derived the rest when read)
    cl.f[cl.n++] = sb.nrx;
    cl.f[cl.n++] = sb.nry;
    nl.f[nl.n++] = sb.ux;
    nl.f[nl.n++] = sb.uy;
}

// halo rectangles (global indices) for the neighbour in direction (dx, dy):
// pack = my owned data that neighbour needs, unpack = my halo it fills
void halo_rects(h2d_ctx* c, int dx, int dy, bool pack, Rng& rc, Rng& rn) {
    const h2d_block& b = c->blk;
    const Dev& d = c->base;
    const int H = b.halo;
    auto axis = [&](int dd, int o, int n, int own_c0, int own_c1, int own_n0, int own_n1, int& c0, int& c1,
                    int& n0, int& n1) {
        if (dd == 0) {
            c0 = own_c0;
            c1 = own_c1;
            n0 = own_n0;
            n1 = own_n1;
        } else if (pack) {
            if (dd > 0) {
                c0 = n0 = o + n - H;
                c1 = n1 = o + n;
            } else {
                c0 = n0 = o;
                c1 = o + H;
                n1 = o + H + 1;
            }
        } else {
            if (dd < 0) {
                c0 = n0 = o - H;
                c1 = n1 = o;
            } else {
                c0 = n0 = o + n;
                c1 = o + n + H;
                n1 = o + n + H + 1;
            }
        }
    };
    axis(dx, b.oi, b.bnx, d.own_c.i0, d.own_c.i1, d.own_n.i0, d.own_n.i1, rc.i0, rc.i1, rn.i0, rn.i1);
    axis(dy, b.oj, b.bny, d.own_c.j0, d.own_c.j1, d.own_n.j0, d.own_n.j1, rc.j0, rc.j1, rn.j0, rn.j1);
}

long long rect_doubles(const FieldList& cl, const FieldList& nl, const Rng& rc, const Rng& rn) {
    return (long long)(rc.i1 - rc.i0) * (rc.j1 - rc.j0) * cl.n + (long long)(rn.i1 - rn.i0) * (rn.j1 - rn.j0) * nl.n;
}

}  // namespace

int h2d_block_upload(h2d_ctx* c, const h2d_state* g) {
    cudaSetDevice(c->device);
    const Dev& d = c->base;
    StateBufs& s = c->sb[c->cur];
    const Rng wc = d.win_c, wn = d.win_n;
    for (int a = 0; a < c->nmat; ++a) {
        if (int rc = global_rect(c, g->m[a], 0, false, wc, s.m[a], nullptr, true)) return rc;
        if (int rc = global_rect(c, g->e[a], 0, false, wc, s.e[a], nullptr, true)) return rc;
        if (int rc = global_rect(c, g->k[a], 0, false, wc, s.k[a], nullptr, true)) return rc;
    }
    double* dv[5] = {s.vol, s.m_mix, s.e_mix, s.rho_mix, s.p_mix};
    double* hv[5] = {g->vol, g->m_mix, g->e_mix, g->rho_mix, g->p_mix};
    for (int q = 0; q < 5; ++q)
        if (int rc = global_rect(c, hv[q], 0, false, wc, dv[q], nullptr, true)) return rc;
    if (int rc = global_rect(c, g->iface_normal, 1, false, wc, s.nrx, s.nry, true)) return rc;
    if (int rc = global_rect(c, g->u, 1, true, wn, s.ux, s.uy, true)) return rc;
    if (int rc = ctl_pull(c)) return rc;
    c->hctl->step = g->step;
    c->hctl->time = g->time;
    c->derived_stale = false;
    return ctl_push(c);
}

int h2d_block_init_window(h2d_ctx* c, const h2d_state* w, int wi0, int wj0, int wnx, int wny, int step,
                          double time) {
    cudaSetDevice(c->device);
    if (!c->is_block || !w || wnx < 1 || wny < 1) return H2D_ERR_INVALID;
    const Dev& d = c->base;
    StateBufs& s = c->sb[c->cur];
    // the painted window's rectangle inside this block's storage window
    auto clip = [&](const Rng& win, int n1) {
        Rng r{std::max(win.i0, wi0), std::min(win.i1, wi0 + wnx + n1), std::max(win.j0, wj0),
              std::min(win.j1, wj0 + wny + n1)};
        return r;
    };
    const Rng rc = clip(d.win_c, 0), rn = clip(d.win_n, 1);
    auto put = [&](const double* host, int vec, bool node, const Rng& r, double* px, double* py) -> int {
        if (!host || r.i1 <= r.i0 || r.j1 <= r.j0) return 0;
        const int W = wnx + (node ? 1 : 0), e = vec ? 2 : 1;
        const int rw = r.i1 - r.i0, rh = r.j1 - r.j0;
        const size_t row = (size_t)rw * e * sizeof(double);
        if (int rc2 = ensure_xbuf(c, row * rh)) return rc2;
        const double* hstart = host + ((size_t)(r.j0 - wj0) * W + (r.i0 - wi0)) * e;
        CK(cudaMemcpy2DAsync(c->xbuf, row, hstart, (size_t)W * e * sizeof(double), row, (size_t)rh,
                             cudaMemcpyHostToDevice, c->st));
        launch_global_xfer(make_dev(c, c->cur, 1), c->xbuf, r, px, py, vec, 1, c->st);
        CK(cudaStreamSynchronize(c->st));
        return 0;
    };
    for (int a = 0; a < c->nmat; ++a) {
        if (int rc2 = put(w->m[a], 0, false, rc, s.m[a], nullptr)) return rc2;
        if (int rc2 = put(w->e[a], 0, false, rc, s.e[a], nullptr)) return rc2;
        if (int rc2 = put(w->k[a], 0, false, rc, s.k[a], nullptr)) return rc2;
    }
    if (int rc2 = put(w->u, 1, true, rn, s.ux, s.uy)) return rc2;
    if (int rc2 = ctl_pull(c)) return rc2;
    c->hctl->step = step;
    c->hctl->time = time;
    if (int rc2 = ctl_push(c)) return rc2;
    // init_case's tail (harness.cpp:286-288) on the window
    if (int rc2 = h2d_fill_ghosts(c)) return rc2;
    if (int rc2 = h2d_sync_derived(c)) return rc2;
    return h2d_update_interface_normals(c);
}

int h2d_block_download(h2d_ctx* c, h2d_state* g) {
    cudaSetDevice(c->device);
    if (int rc_ = ensure_derived(c)) return rc_;
    cudaSetDevice(c->device);
    const Dev& d = c->base;
    StateBufs& s = c->sb[c->cur];
    const Rng oc = d.own_c, on = d.own_n;
    for (int a = 0; a < c->nmat; ++a) {
        if (int rc = global_rect(c, g->m[a], 0, false, oc, s.m[a], nullptr, false)) return rc;
        if (int rc = global_rect(c, g->e[a], 0, false, oc, s.e[a], nullptr, false)) return rc;
        if (int rc = global_rect(c, g->k[a], 0, false, oc, s.k[a], nullptr, false)) return rc;
    }
    double* dv[5] = {s.vol, s.m_mix, s.e_mix, s.rho_mix, s.p_mix};
    double* hv[5] = {g->vol, g->m_mix, g->e_mix, g->rho_mix, g->p_mix};
    for (int q = 0; q < 5; ++q)
        if (int rc = global_rect(c, hv[q], 0, false, oc, dv[q], nullptr, false)) return rc;
    if (int rc = global_rect(c, g->iface_normal, 1, false, oc, s.nrx, s.nry, false)) return rc;
    if (int rc = global_rect(c, g->u, 1, true, on, s.ux, s.uy, false)) return rc;
    if (int rc = ctl_pull(c)) return rc;
    g->step = c->hctl->step;
    g->time = c->hctl->time;
    return 0;
}

int h2d_block_begin(h2d_ctx* c, int max_steps, double t_end, double cfl) {
    cudaSetDevice(c->device);
    if (int rc = ctl_reset(c)) return rc;
    Ctl& h = *c->hctl;
    h.t_end = t_end;
    h.cfl = cfl;
    h.max_steps = max_steps;
    h.steps_done = 0;
    h.floor_count = h.k_clip_count = h.mass_fix_count = 0;
    h.max_k_violation = 0.0;
    const int cap = max_steps > 0 ? max_steps : kRunLogCap;
    if (int rc = ensure_logs(c, cap)) return rc;
    h.dt_log = c->dt_log;
    h.dt_log_cap = c->dt_log_cap;
    h.diag_log = c->diag_log;
    h.diag_log_cap = c->dt_log_cap;
    if (int rc = ctl_push(c)) return rc;
    if (int rc = ensure_graphs(c)) return rc;
    enqueue_cfl_next(c);  // wave speed of the owned cells of the initial State
    if (int rc = check_launch(c)) return rc;
    if (int rc = ctl_pull(c)) return rc;
    return 0;
}

int h2d_block_scalars(h2d_ctx* c, unsigned long long out[4]) {
    cudaSetDevice(c->device);
    if (int rc = ctl_pull(c)) return rc;
    out[0] = c->hctl->next_wmax_bits;
    out[1] = c->hctl->next_err_key;
    out[2] = c->hctl->err_key;
    out[3] = (unsigned long long)c->hctl->done;
    return 0;
}

int h2d_block_set(h2d_ctx* c, const unsigned long long in[3]) {
    cudaSetDevice(c->device);
    if (int rc = ctl_pull(c)) return rc;
    c->hctl->next_wmax_bits = in[0];
    c->hctl->next_err_key = in[1];
    c->hctl->err_key = in[2];
    return ctl_push(c);
}

int h2d_block_step(h2d_ctx* c) {
    cudaSetDevice(c->device);
    c->derived_stale = true;
    if (int rc = launch_step_graph(c, c->cur)) return rc;
    if (int rc = ctl_pull(c)) return rc;
    c->cur = c->hctl->cur;
    return 0;
}

int h2d_block_rollback(h2d_ctx* c) {
    cudaSetDevice(c->device);
    launch_rollback(c->ctl, c->st);
    if (int rc = check_launch(c)) return rc;
    if (int rc = ctl_pull(c)) return rc;
    c->cur = c->hctl->cur;
    return 0;
}

long long h2d_halo_bytes(h2d_ctx* c, int dx, int dy, int pack) {
    FieldList cl, nl;
    state_lists(c, cl, nl);
    Rng rc, rn;
    halo_rects(c, dx, dy, pack != 0, rc, rn);
    return rect_doubles(cl, nl, rc, rn) * (long long)sizeof(double);
}

int h2d_halo_pack(h2d_ctx* c, int dx, int dy, void* dev_buf) {
    cudaSetDevice(c->device);
    FieldList cl, nl;
    state_lists(c, cl, nl);
    Rng rc, rn;
    halo_rects(c, dx, dy, true, rc, rn);
    launch_rect_xfer(make_dev(c, c->cur, 1), cl, nl, rc, rn, static_cast<double*>(dev_buf), 1, c->st);
    if (int rc2 = check_launch(c)) return rc2;
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

int h2d_halo_unpack(h2d_ctx* c, int dx, int dy, const void* dev_buf) {
    cudaSetDevice(c->device);
    FieldList cl, nl;
    state_lists(c, cl, nl);
    Rng rc, rn;
    halo_rects(c, dx, dy, false, rc, rn);
    launch_rect_xfer(make_dev(c, c->cur, 1), cl, nl, rc, rn, const_cast<double*>(static_cast<const double*>(dev_buf)),
                     0, c->st);
    if (int rc2 = check_launch(c)) return rc2;
    CK(cudaStreamSynchronize(c->st));
    return 0;
}

int h2d_block_result(h2d_ctx* c, h2d_run_args* a) {
    cudaSetDevice(c->device);
    if (int rc = ctl_pull(c)) return rc;
    const Ctl& h = *c->hctl;
    a->steps_done = h.steps_done;
    a->floor_count = h.floor_count;
    a->diag.k_clip_count = h.k_clip_count;
    a->diag.mass_fix_count = h.mass_fix_count;
    a->diag.max_k_violation = h.max_k_violation;
    if (a->dt_log && h.steps_done > 0) {
        const int n = h.steps_done < a->dt_log_cap ? h.steps_done : a->dt_log_cap;
        CK(cudaMemcpy(a->dt_log, c->dt_log, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost));
    }
    if (int rc = copy_series(c, a->series, h.steps_done < a->series_cap ? h.steps_done : a->series_cap)) return rc;
    return decode_error(c, true);
}

int h2d_last_error(h2d_ctx* c, h2d_error* e) {
    *e = c->err;
    return 0;
}

}  // extern "C"

// ===========================================================================
// Block-decomposition data plane: the whole multi-block run
// loop in the library, with the State, the control block and every per-step
// exchange on the device.  Per step and block, on the block's compute stream
// st and its communication stream cs:
//
//   st: wait(apply) -> k_step_start + Lagrange tiles on owned data
//       -> wait(halo) -> Lagrange edge tiles -> rest of the step (graph)
//       -> k_red_pack: {next wave speed, ~next cfl error, ~error, done}
//   cs: wait(red) -> ONE max all-reduce of the four words -> k_red_apply
//       (global dt input and first error; a pre-commit error anywhere rolls
//       every committed block back) -> record(apply) -> pack every halo
//       rectangle (8 neighbours, corners included) into one buffer ->
//       grouped send/recv with the neighbours -> unpack -> record(halo)
//
// so the halo exchange overlaps the next step's Lagrange tiles on owned
// data, and the host only polls the control blocks every kPollSteps steps.
// Transports: NCCL (one block per process, the communicator owned here,
// opened at run time from libnccl.so.2) or in-process (every block of the
// decomposition in this process on one device: device-to-device copies and a
// one-block max kernel, same stream structure).
// ===========================================================================
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is opened with dlopen

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    bool load() {
        if (h) return true;
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return false;
        auto sym = [&](auto& f, const char* n) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, n)); return f != nullptr; };
        return sym(GetUniqueId, "ncclGetUniqueId") && sym(CommInitRank, "ncclCommInitRank") &&
               sym(CommDestroy, "ncclCommDestroy") && sym(AllReduce, "ncclAllReduce") && sym(Send, "ncclSend") &&
               sym(Recv, "ncclRecv") && sym(GroupStart, "ncclGroupStart") && sym(GroupEnd, "ncclGroupEnd");
    }
};
NcclApi g_nccl;

const int kDirs[8][2] = {{-1, -1}, {0, -1}, {1, -1}, {-1, 0}, {1, 0}, {-1, 1}, {0, 1}, {1, 1}};
int dir_index(int dx, int dy) {
    for (int q = 0; q < 8; ++q)
        if (kDirs[q][0] == dx && kDirs[q][1] == dy) return q;
    return -1;
}

}  // namespace

struct h2d_comm {
    int kind = 0;  // 0 in-process, 1 NCCL
    int px = 1, py = 1;
    ncclComm_t nccl = nullptr;
    struct Side {
        h2d_ctx* c = nullptr;
        int rank = 0, bx = 0, by = 0;
        int peer[8];                 // neighbour rank per direction (-1: global boundary)
        HaloPlan pk{}, up{};         // pack / unpack rectangles, segments ordered like kDirs
        int seg_pk[8], seg_up[8];    // segment of direction q in pk / up (-1: none)
        double *send = nullptr, *recv = nullptr;
        unsigned long long* red = nullptr;
        cudaStream_t cs = nullptr;
        cudaEvent_t e_red = nullptr, e_apply = nullptr, e_packed = nullptr, e_halo = nullptr;
        // AD remap: the AdWork halo exchanged between the two passes (same
        // rectangles, its own plane lists, offsets, buffers and events)
        HaloPlan pk_ad{}, up_ad{};
        double *send_ad = nullptr, *recv_ad = nullptr;
        cudaEvent_t e_p0 = nullptr, e_packed_ad = nullptr, e_mid = nullptr;
    };
    std::vector<Side> side;
    unsigned long long** red_ptrs = nullptr;  // device array of every side's red (in-process)
    cudaEvent_t e_all = nullptr;
    // h2d_comm_trace: timing events of the first trace_cap steps of the next
    // run, per block kTracePts points (ms from the run's first step start)
    int trace_cap = 0;
    std::vector<float> trace;
};
enum { TR_LAG0, TR_LAG1, TR_EDGE1, TR_MID0, TR_MID1, TR_REST1, TR_RED0, TR_HALO0, TR_HALO1, kTracePts };

namespace {

void comm_free(h2d_comm* m) {
    for (auto& sd : m->side) {
        if (sd.c) cudaSetDevice(sd.c->device);
        if (sd.cs) cudaStreamSynchronize(sd.cs);
        if (sd.send) cudaFree(sd.send);
        if (sd.recv) cudaFree(sd.recv);
        if (sd.red) cudaFree(sd.red);
        if (sd.send_ad) cudaFree(sd.send_ad);
        if (sd.recv_ad) cudaFree(sd.recv_ad);
        for (cudaEvent_t e : {sd.e_red, sd.e_apply, sd.e_packed, sd.e_halo, sd.e_p0, sd.e_packed_ad, sd.e_mid})
            if (e) cudaEventDestroy(e);
        if (sd.cs) cudaStreamDestroy(sd.cs);
    }
    if (m->red_ptrs) cudaFree(m->red_ptrs);
    if (m->e_all) cudaEventDestroy(m->e_all);
    if (m->nccl && g_nccl.CommDestroy) g_nccl.CommDestroy(m->nccl);
    delete m;
}

// planes of State parity p exchanged with the neighbours (state_lists at p)
void lists_at(h2d_ctx* c, int p, FieldList& cl, FieldList& nl) {
    const int keep = c->cur;
    c->cur = p;
    state_lists(c, cl, nl);
    c->cur = keep;
}

// AdWork planes a block needs from its neighbours before AD pass 1
// (remap.cpp:87-97: the Work of pass 0)
void ad_lists(h2d_ctx* c, FieldList& cl, FieldList& nl) {
    const AdWork& W = c->adw;
    cl = FieldList{};
    nl = FieldList{};
    for (int a = 0; a < c->nmat; ++a) {
        cl.f[cl.n++] = W.m[a];
        cl.f[cl.n++] = W.me[a];
        cl.f[cl.n++] = W.e[a];
        cl.f[cl.n++] = W.k[a];
    }
    cl.f[cl.n++] = W.mcell;
    if (c->nmat == 2) {  // (one material: pass 1 reads the State's normals)
        cl.f[cl.n++] = W.nrx;
        cl.f[cl.n++] = W.nry;
    }
    nl.f[nl.n++] = W.ux;
    nl.f[nl.n++] = W.uy;
}

// first AD run of a communicator: the AdWork planes, the plans of the
// mid-step exchange and its buffers
int side_setup_ad(h2d_comm::Side& sd) {
    h2d_ctx* c = sd.c;
    cudaSetDevice(c->device);
    if (c->nmat > 2) {
        set_err(c, H2D_ERR_INVALID, "the AD remap holds at most 2 materials");
        return H2D_ERR_INVALID;
    }
    if (int rc = ensure_ad(c)) return rc;
    if (sd.send_ad) return 0;
    FieldList cl, nl;
    ad_lists(c, cl, nl);
    sd.pk_ad = sd.pk;
    sd.up_ad = sd.up;
    for (int pack = 1; pack >= 0; --pack) {
        HaloPlan& pl = pack ? sd.pk_ad : sd.up_ad;
        pl.off[0] = 0;
        for (int q = 0; q < pl.n; ++q) pl.off[q + 1] = pl.off[q] + rect_doubles(cl, nl, pl.rc[q], pl.rn[q]);
    }
    CK(cudaMalloc(&sd.send_ad, (size_t)(sd.pk_ad.off[sd.pk_ad.n] > 0 ? sd.pk_ad.off[sd.pk_ad.n] : 1) * sizeof(double)));
    CK(cudaMalloc(&sd.recv_ad, (size_t)(sd.up_ad.off[sd.up_ad.n] > 0 ? sd.up_ad.off[sd.up_ad.n] : 1) * sizeof(double)));
    for (cudaEvent_t* e : {&sd.e_p0, &sd.e_packed_ad, &sd.e_mid})
        CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    return 0;
}

int side_setup(h2d_comm* m, h2d_comm::Side& sd) {
    h2d_ctx* c = sd.c;
    cudaSetDevice(c->device);
    if (!c->is_block) return H2D_ERR_INVALID;
    FieldList cl, nl;
    state_lists(c, cl, nl);
    sd.pk.n = sd.up.n = 0;
    sd.pk.off[0] = sd.up.off[0] = 0;
    for (int q = 0; q < 8; ++q) {
        const int x = sd.bx + kDirs[q][0], y = sd.by + kDirs[q][1];
        sd.peer[q] = (x >= 0 && x < m->px && y >= 0 && y < m->py) ? y * m->px + x : -1;
        sd.seg_pk[q] = sd.seg_up[q] = -1;
        if (sd.peer[q] < 0) continue;
        for (int pack = 1; pack >= 0; --pack) {
            HaloPlan& pl = pack ? sd.pk : sd.up;
            Rng rc, rn;
            halo_rects(c, kDirs[q][0], kDirs[q][1], pack != 0, rc, rn);
            (pack ? sd.seg_pk : sd.seg_up)[q] = pl.n;
            pl.rc[pl.n] = rc;
            pl.rn[pl.n] = rn;
            pl.off[pl.n + 1] = pl.off[pl.n] + rect_doubles(cl, nl, rc, rn);
            ++pl.n;
        }
    }
    CK(cudaMalloc(&sd.send, (size_t)(sd.pk.off[sd.pk.n] > 0 ? sd.pk.off[sd.pk.n] : 1) * sizeof(double)));
    CK(cudaMalloc(&sd.recv, (size_t)(sd.up.off[sd.up.n] > 0 ? sd.up.off[sd.up.n] : 1) * sizeof(double)));
    CK(cudaMalloc(&sd.red, 4 * sizeof(unsigned long long)));
    CK(cudaStreamCreateWithFlags(&sd.cs, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&sd.e_red, &sd.e_apply, &sd.e_packed, &sd.e_halo})
        CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    // the Lagrange tiles whose stencil reads owned data only: tile origins
    // (i0, j0) with cells [i0-1, i0+LTX] and nodes [i0-1, i0+LTX+1] inside
    // the owned range on every side that has a neighbour (walls are local)
    const h2d_block& b = c->blk;
    const int ltx = lag_tile_w(), lty = lag_tile_h();
    Rng in{-(1 << 29), 1 << 29, -(1 << 29), 1 << 29};
    if (sd.bx > 0) in.i0 = b.oi + 1;
    if (sd.bx < m->px - 1) in.i1 = b.oi + b.bnx - 1 - ltx;
    if (sd.by > 0) in.j0 = b.oj + 1;
    if (sd.by < m->py - 1) in.j1 = b.oj + b.bny - 1 - lty;
    c->base.lag_inner = in;
    // the step after the Lagrange kernel, per State parity
    for (int p = 0; p < 2; ++p) {
        if (c->graph_rest[p]) continue;
        cudaGraph_t g = nullptr;
        const long long before = launch_count();
        CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeThreadLocal));
        launch_step_block_rest(make_dev(c, p, 1), c->st);
        CK(cudaStreamEndCapture(c->st, &g));
        c->graph_rest_kernels = launch_count() - before;
        add_launches(-c->graph_rest_kernels);
        const cudaError_t e = cudaGraphInstantiate(&c->graph_rest[p], g, 0);
        cudaGraphDestroy(g);
        CK(e);
    }
    return 0;
}

int comm_finish(h2d_comm* m, h2d_comm** out) {
    for (auto& sd : m->side)
        if (int rc = side_setup(m, sd)) {
            comm_free(m);
            return rc;
        }
    if (m->kind == 0) {
        h2d_ctx* c = m->side[0].c;
        std::vector<unsigned long long*> ptrs;
        for (auto& sd : m->side) ptrs.push_back(sd.red);
        CK(cudaMalloc(&m->red_ptrs, ptrs.size() * sizeof(void*)));
        CK(cudaMemcpy(m->red_ptrs, ptrs.data(), ptrs.size() * sizeof(void*), cudaMemcpyHostToDevice));
        CK(cudaEventCreateWithFlags(&m->e_all, cudaEventDisableTiming));
    }
    *out = m;
    return 0;
}

}  // namespace

extern "C" {

int h2d_nccl_unique_id(unsigned char id[128]) {
    if (!g_nccl.load()) return H2D_ERR_INVALID;
    ncclUniqueId u;
    if (g_nccl.GetUniqueId(&u) != ncclSuccess) return H2D_ERR_DEVICE;
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, 128);
    return 0;
}

int h2d_comm_nccl(const unsigned char id[128], int px, int py, int rank, h2d_ctx* blk, h2d_comm** out) {
    *out = nullptr;
    if (!blk || px < 1 || py < 1 || rank < 0 || rank >= px * py) return H2D_ERR_INVALID;
    if (!g_nccl.load()) {
        set_err(blk, H2D_ERR_INVALID, "libnccl.so.2 not found");
        return H2D_ERR_INVALID;
    }
    h2d_ctx* c = blk;
    cudaSetDevice(c->device);
    h2d_comm* m = new h2d_comm();
    m->kind = 1;
    m->px = px;
    m->py = py;
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    if (g_nccl.CommInitRank(&m->nccl, px * py, u, rank) != ncclSuccess) {
        delete m;
        set_err(c, H2D_ERR_DEVICE, "ncclCommInitRank failed");
        return H2D_ERR_DEVICE;
    }
    h2d_comm::Side sd;
    sd.c = c;
    sd.rank = rank;
    sd.bx = rank % px;
    sd.by = rank / px;
    m->side.push_back(sd);
    return comm_finish(m, out);
}

int h2d_comm_local(h2d_ctx* const* blocks, int px, int py, h2d_comm** out) {
    *out = nullptr;
    if (!blocks || px < 1 || py < 1) return H2D_ERR_INVALID;
    h2d_comm* m = new h2d_comm();
    m->kind = 0;
    m->px = px;
    m->py = py;
    for (int r = 0; r < px * py; ++r) {
        h2d_comm::Side sd;
        sd.c = blocks[r];
        sd.rank = r;
        sd.bx = r % px;
        sd.by = r / px;
        if (!sd.c || sd.c->device != blocks[0]->device) {
            delete m;
            return H2D_ERR_INVALID;
        }
        m->side.push_back(sd);
    }
    return comm_finish(m, out);
}

void h2d_comm_destroy(h2d_comm* m) {
    if (m) comm_free(m);
}

int h2d_blocks_run(h2d_comm* m, int max_steps, double t_end, double cfl, int* steps_out, float* device_ms) {
    return h2d_blocks_run_kind(m, H2D_REMAP_DIRECTCF, max_steps, t_end, cfl, steps_out, device_ms);
}

int h2d_blocks_run_kind(h2d_comm* m, int remap_kind, int max_steps, double t_end, double cfl, int* steps_out,
                        float* device_ms) {
    constexpr int kPollSteps = 16;
    if (steps_out) *steps_out = 0;
    if (device_ms) *device_ms = 0.0f;
    h2d_ctx* c = m->side[0].c;  // CK's error target
    const int n = (int)m->side.size();
    const bool ad = remap_kind == H2D_REMAP_AD;
    if (!ad && remap_kind != H2D_REMAP_DIRECTCF) {
        set_err(c, H2D_ERR_INVALID, "block mode runs the DirectCF and AD remaps");
        return H2D_ERR_INVALID;
    }
    if (ad)
        for (auto& sd : m->side)
            if (int rc = side_setup_ad(sd)) return rc;
    for (auto& sd : m->side) {
        if (int rc = h2d_block_begin(sd.c, max_steps, t_end, cfl)) return rc;
        sd.c->derived_stale = true;
    }
    std::vector<int> parity(n);
    for (int b = 0; b < n; ++b) parity[b] = m->side[b].c->cur;

    // optional trace (h2d_comm_trace): timing events at fixed points of a step
    std::vector<cudaEvent_t> tev;
    const int tr_steps = m->trace_cap;
    m->trace.clear();
    if (tr_steps > 0) {
        tev.resize((size_t)tr_steps * n * kTracePts, nullptr);
        for (auto& e : tev) CK(cudaEventCreate(&e));
    }
    int tr_q = -1;  // the step being traced (-1: none)
    auto mark = [&](int b, int pt, cudaStream_t st) {
        if (tr_q >= 0) cudaEventRecord(tev[((size_t)tr_q * n + b) * kTracePts + pt], st);
    };
    int steps_issued = 0;

    // the all-reduce + apply of every block's four words, on the cs streams
    auto combine = [&]() -> int {
        for (auto& sd : m->side) {
            launch_red_pack(sd.c->ctl, sd.red, sd.c->st);
            CK(cudaEventRecord(sd.e_red, sd.c->st));
            CK(cudaStreamWaitEvent(sd.cs, sd.e_red, 0));
            mark((int)(&sd - &m->side[0]), TR_RED0, sd.cs);
        }
        if (m->kind == 1) {
            auto& sd = m->side[0];
            if (g_nccl.AllReduce(sd.red, sd.red, 4, ncclUint64, ncclMax, m->nccl, sd.cs) != ncclSuccess) {
                set_err(c, H2D_ERR_DEVICE, "ncclAllReduce failed");
                return H2D_ERR_DEVICE;
            }
        } else {
            auto& s0 = m->side[0];
            for (int b = 1; b < n; ++b) CK(cudaStreamWaitEvent(s0.cs, m->side[b].e_red, 0));
            launch_red_local(m->red_ptrs, n, s0.cs);
            CK(cudaEventRecord(m->e_all, s0.cs));
            for (int b = 1; b < n; ++b) CK(cudaStreamWaitEvent(m->side[b].cs, m->e_all, 0));
        }
        for (auto& sd : m->side) {
            launch_red_apply(sd.c->ctl, sd.red, sd.cs);
            CK(cudaEventRecord(sd.e_apply, sd.cs));
        }
        return check_launch(c);
    };
    // one halo exchange on the cs streams: mid = false the State of parity
    // p[b] (after combine), mid = true the AdWork planes between the AD passes
    auto exchange = [&](const std::vector<int>& p, bool mid) -> int {
        auto lists = [&](h2d_comm::Side& sd, int par, FieldList& cl, FieldList& nl) {
            if (mid)
                ad_lists(sd.c, cl, nl);
            else
                lists_at(sd.c, par, cl, nl);
        };
        for (int b = 0; b < n; ++b) {
            auto& sd = m->side[b];
            FieldList cl, nl;
            lists(sd, p[b], cl, nl);
            mark(b, mid ? TR_MID0 : TR_HALO0, sd.cs);
            launch_halo_multi(make_dev(sd.c, p[b], 1), cl, nl, mid ? sd.pk_ad : sd.pk, mid ? sd.send_ad : sd.send, 1,
                              sd.cs);
            CK(cudaEventRecord(mid ? sd.e_packed_ad : sd.e_packed, sd.cs));
        }
        if (m->kind == 1) {
            auto& sd = m->side[0];
            const HaloPlan& pk = mid ? sd.pk_ad : sd.pk;
            const HaloPlan& up = mid ? sd.up_ad : sd.up;
            double* send = mid ? sd.send_ad : sd.send;
            double* recv = mid ? sd.recv_ad : sd.recv;
            if (g_nccl.GroupStart() != ncclSuccess) return H2D_ERR_DEVICE;
            for (int q = 0; q < 8; ++q) {
                if (sd.peer[q] < 0) continue;
                const int a = sd.seg_pk[q], r = sd.seg_up[q];
                g_nccl.Send(send + pk.off[a], (size_t)(pk.off[a + 1] - pk.off[a]), ncclFloat64, sd.peer[q], m->nccl,
                            sd.cs);
                g_nccl.Recv(recv + up.off[r], (size_t)(up.off[r + 1] - up.off[r]), ncclFloat64, sd.peer[q], m->nccl,
                            sd.cs);
            }
            if (g_nccl.GroupEnd() != ncclSuccess) {
                set_err(c, H2D_ERR_DEVICE, "NCCL halo exchange failed");
                return H2D_ERR_DEVICE;
            }
        } else {  // pull: my halo segment for direction q is the neighbour's pack segment for -q
            for (int b = 0; b < n; ++b) {
                auto& sd = m->side[b];
                const HaloPlan& up = mid ? sd.up_ad : sd.up;
                for (int q = 0; q < 8; ++q) {
                    if (sd.peer[q] < 0) continue;
                    auto& nb = m->side[sd.peer[q]];
                    const HaloPlan& npk = mid ? nb.pk_ad : nb.pk;
                    const int a = nb.seg_pk[dir_index(-kDirs[q][0], -kDirs[q][1])], r = sd.seg_up[q];
                    CK(cudaStreamWaitEvent(sd.cs, mid ? nb.e_packed_ad : nb.e_packed, 0));
                    CK(cudaMemcpyAsync((mid ? sd.recv_ad : sd.recv) + up.off[r],
                                       (mid ? nb.send_ad : nb.send) + npk.off[a],
                                       (size_t)(up.off[r + 1] - up.off[r]) * sizeof(double), cudaMemcpyDeviceToDevice,
                                       sd.cs));
                }
            }
        }
        for (int b = 0; b < n; ++b) {
            auto& sd = m->side[b];
            FieldList cl, nl;
            lists(sd, p[b], cl, nl);
            launch_halo_multi(make_dev(sd.c, p[b], 1), cl, nl, mid ? sd.up_ad : sd.up, mid ? sd.recv_ad : sd.recv, 0,
                              sd.cs);
            mark(b, mid ? TR_MID1 : TR_HALO1, sd.cs);
            CK(cudaEventRecord(mid ? sd.e_mid : sd.e_halo, sd.cs));
        }
        return check_launch(c);
    };

    if (int rc = combine()) return rc;  // the initial State's global wave speed
    if (int rc = exchange(parity, false)) return rc;  // the initial halos (exact after a window init)
    std::vector<cudaEvent_t> t0(n), t1(n);
    for (int b = 0; b < n; ++b) {
        CK(cudaEventCreate(&t0[b]));
        CK(cudaEventCreate(&t1[b]));
        auto& sd = m->side[b];
        CK(cudaStreamWaitEvent(sd.c->st, sd.e_halo, 0));
        CK(cudaEventRecord(t0[b], sd.c->st));
    }
    for (;;) {
        int chunk = kPollSteps;
        if (max_steps > 0) {
            const int left = max_steps - m->side[0].c->hctl->step;
            if (left <= 0) break;
            chunk = left < chunk ? left : chunk;
        }
        const int step0 = m->side[0].c->hctl->step;
        for (int q = 0; q < chunk; ++q) {
            const int x_first = (step0 + q) % 2 == 0;  // harness.cpp:401
            // (the exchange of step s - 1, which overlaps step s's owned tiles, was
            // enqueued with tr_q = s - 1: its TR_HALO* marks belong to that record)
            tr_q = steps_issued < tr_steps ? steps_issued : -1;
            ++steps_issued;
            for (int b = 0; b < n; ++b) {
                auto& sd = m->side[b];
                h2d_ctx* bc = sd.c;
                const Dev d = make_dev(bc, parity[b], 1);
                CK(cudaStreamWaitEvent(bc->st, sd.e_apply, 0));
                mark(b, TR_LAG0, bc->st);
                launch_step_block_head(d, 1, bc->st);
                mark(b, TR_LAG1, bc->st);
                CK(cudaStreamWaitEvent(bc->st, sd.e_halo, 0));
                launch_step_block_head(d, 2, bc->st);
                mark(b, TR_EDGE1, bc->st);
                if (ad) {  // pass 0 on this block's window, then its AdWork halo goes out
                    launch_step_block_ad_mid(d, bc->adw, x_first, bc->st);
                    CK(cudaEventRecord(sd.e_p0, bc->st));
                    CK(cudaStreamWaitEvent(sd.cs, sd.e_p0, 0));
                    continue;
                }
                CK(cudaGraphLaunch(bc->graph_rest[parity[b]], bc->st));
                add_launches(bc->graph_rest_kernels);
                mark(b, TR_REST1, bc->st);
                parity[b] ^= 1;
            }
            if (ad) {  // the split remap's second exchange, then pass 1 and the rest of the step
                if (int rc = exchange(parity, true)) return rc;
                for (int b = 0; b < n; ++b) {
                    auto& sd = m->side[b];
                    h2d_ctx* bc = sd.c;
                    CK(cudaStreamWaitEvent(bc->st, sd.e_mid, 0));
                    launch_step_block_ad_rest(make_dev(bc, parity[b], 1), bc->adw, x_first, bc->st);
                    mark(b, TR_REST1, bc->st);
                    parity[b] ^= 1;
                }
            }
            if (int rc = combine()) return rc;
            if (int rc = exchange(parity, false)) return rc;
        }
        bool stop = false;
        for (int b = 0; b < n; ++b) {
            auto& sd = m->side[b];
            CK(cudaStreamSynchronize(sd.cs));
            if (int rc = ctl_pull(sd.c)) return rc;
            parity[b] = sd.c->hctl->cur;
            if (sd.c->hctl->err_key != kNoErr || sd.c->hctl->done) stop = true;
        }
        if (stop) break;
    }
    float worst = 0.0f;
    for (int b = 0; b < n; ++b) {
        auto& sd = m->side[b];
        CK(cudaEventRecord(t1[b], sd.cs));
        CK(cudaStreamSynchronize(sd.cs));
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, t0[b], t1[b]));
        worst = ms > worst ? ms : worst;
        if (int rc = ctl_pull(sd.c)) return rc;
        sd.c->cur = sd.c->hctl->cur;
    }
    if (tr_steps > 0) {  // ms of every traced point from its block's first step start (-1: not reached)
        const int got = steps_issued < tr_steps ? steps_issued : tr_steps;
        m->trace.assign((size_t)got * n * kTracePts, -1.0f);
        for (int q = 0; q < got; ++q)
            for (int b = 0; b < n; ++b)
                for (int pt = 0; pt < kTracePts; ++pt) {
                    float ms = -1.0f;
                    const size_t k = ((size_t)q * n + b) * kTracePts + pt;
                    if (cudaEventElapsedTime(&ms, t0[b], tev[k]) == cudaSuccess) m->trace[k] = ms;
                }
        cudaGetLastError();  // (an unrecorded point reports an error: cleared)
        for (auto& e : tev) cudaEventDestroy(e);
        m->trace_cap = 0;
    }
    for (int b = 0; b < n; ++b) {
        cudaEventDestroy(t0[b]);
        cudaEventDestroy(t1[b]);
    }
    if (device_ms) *device_ms = worst;
    if (steps_out) *steps_out = m->side[0].c->hctl->steps_done;
    return 0;
}

int h2d_comm_trace(h2d_comm* m, int steps) {
    if (!m || steps < 0 || steps > 4096) return H2D_ERR_INVALID;
    m->trace_cap = steps;
    return 0;
}

int h2d_comm_trace_read(h2d_comm* m, float* out, int cap) {
    if (!m) return 0;
    const int nrec = (int)m->trace.size();
    if (out)
        for (int k = 0; k < nrec && k < cap; ++k) out[k] = m->trace[k];
    return nrec;
}

}  // extern "C"

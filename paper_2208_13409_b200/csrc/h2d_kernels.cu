// h2d_kernels.cu — fp64 sm_100a kernels of one Lagrange + DirectCF step.
//
// Each kernel restates one reference phase (cited file:line, proj/src) as a
// data-parallel gather: every face / corner / dual-face flux is computed once
// by its own thread and stored; every cell and node then sums its incoming
// contributions in exactly the reference's program order (SURVEY.md App. C
// items 3-4), so the result is bit-identical to the serial scatter loops.
// Errors are recorded as the minimum (phase, loop index) key, i.e. the first
// exception the serial reference would have thrown.
#include "h2d_device.cuh"
#include "h2d_launch.h"

#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>
#include <cuda_runtime.h>

#include <atomic>

#include <type_traits>

namespace h2d {

// ---------------------------------------------------------------------------
// indexing helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tid2(int& i, int& j, int ilo, int jlo) {
    i = ilo + (int)(blockIdx.x * blockDim.x + threadIdx.x);
    j = jlo + (int)(blockIdx.y * blockDim.y + threadIdx.y);
}
// ownership: every global cell / node / face is answered for (errors,
// counters, nan_scan, cfl) by exactly one block
__device__ __forceinline__ bool own_cell(const Dev& d, int i, int j) { return in(d.own_c, i, j); }
__device__ __forceinline__ bool own_node(const Dev& d, int i, int j) { return in(d.own_n, i, j); }
__device__ __forceinline__ bool own_xface(const Dev& d, int i, int j) {  // node column i, cell row j
    return i >= d.own_n.i0 && i < d.own_n.i1 && j >= d.own_c.j0 && j < d.own_c.j1;
}
__device__ __forceinline__ bool own_yface(const Dev& d, int i, int j) {  // cell column i, node row j
    return i >= d.own_c.i0 && i < d.own_c.i1 && j >= d.own_n.j0 && j < d.own_n.j1;
}

// ---------------------------------------------------------------------------
// control kernels
// ---------------------------------------------------------------------------
// Start of a step or of a single API phase. mode: 0 = run-loop step (applies
// harness.cpp:390-391), 1 = API call with host dt, 2 = API cfl_dt only.
// RemapDiag updates (remap.cpp:161-165). Whole regions can carry a rounding-
// level violation at once (config 4, steps 80-117: tens of millions of cells),
// so one same-address atomic per cell would serialise at the L2 slice: the
// lanes that update combine first (max / count are order-free, so this is
// exact), and a max no larger than the last value seen is not sent at all
// (the stored maximum only grows, so a stale cached copy only lets more
// updates through).
__device__ __forceinline__ void bump_kviol(Ctl* ctl, double viol) {
    namespace cg = cooperative_groups;
    // a value that does not exceed the running maximum cannot change it (a
    // stale cached read only lets a few more threads through): most cells with
    // a rounding-level violation stop here, before the warp reduction
    const unsigned long long mine = (unsigned long long)__double_as_longlong(viol);
    if (mine <= __ldca(&ctl->kviol_bits)) return;
    const auto g = cg::coalesced_threads();
    const unsigned long long v = cg::reduce(g, mine, cg::greater<unsigned long long>());
    if (g.thread_rank() == 0) atomicMax(&ctl->kviol_bits, v);
}
__device__ __forceinline__ void bump_clip(Ctl* ctl) {
    const auto g = cooperative_groups::coalesced_threads();
    if (g.thread_rank() == 0) atomicAdd(&ctl->step_clip, (int)g.size());
}

// LagrangeResult::floor_count (lagrange.cpp:124,187), combined the same way
__device__ __forceinline__ void bump_floor(Ctl* ctl, int n) {
    namespace cg = cooperative_groups;
    const auto g = cg::coalesced_threads();
    const int v = cg::reduce(g, n, cg::plus<int>());
    if (g.thread_rank() == 0) atomicAdd(&ctl->step_floor, v);
}

__global__ void k_begin(Ctl* c, int mode, double host_dt) {
    pdl_enter();
    if (c->err_key != kNoErr || c->done) return;
    c->wmax_bits = 0ull;
    c->kviol_bits = 0ull;
    c->step_floor = 0;
    c->step_clip = 0;
    c->step_fix = 0;
    if (mode == 0) {
        const double t_end = c->t_end;
        if (!(c->time < t_end - 1e-15 * rmax(1.0, t_end))) {
            c->done = 1;
            return;
        }
        if (c->max_steps > 0 && c->step >= c->max_steps) {
            c->done = 1;
            return;
        }
    } else if (mode == 1) {
        c->dt = host_dt;
    }
}

// cfl_dt, harness.cpp:293-313: per-cell wave speed, block max, one atomic
// per block on the bit pattern (non-negative doubles order as integers).
template <int NM>
__global__ void k_cfl(Dev d, int into_next) {
    pdl_enter();
    if (halted(d.ctl)) return;
    unsigned long long wb = 0ull;
    // owned interior cells (cfl_dt loops over the whole mesh; the blocks of a
    // decomposition split it and the maxima are combined across ranks)
    const int ci0 = max(d.own_c.i0, 0), ci1 = min(d.own_c.i1, d.nx);
    const int cj0 = max(d.own_c.j0, 0), cj1 = min(d.own_c.j1, d.ny);
    const int w = ci1 - ci0;
    const long long ncell = (long long)w * (cj1 - cj0);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ncell;
         t += (long long)gridDim.x * blockDim.x) {
        const int j = cj0 + (int)(t / w), i = ci0 + (int)(t % w);
        const int c = ix(d, i, j);
        double cs = 0.0;
        bool bad = false;
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            const double ka = d.k[a][c];
            if (ka < kThermoTol) continue;
            const double rho_a = rho_of(d, d.m[a][c], ka);
            const double pa = eos_p(d, a, rho_a, d.e[a][c]);
            cs += ka * sound(d, a, rho_a, pa, bad);
        }
        if (bad) atomicMin(into_next ? &d.ctl->next_err_key : &d.ctl->err_key, ekey(PH_CFL_UNPHYS, j, i, 0));
        double umax = 0.0;
#pragma unroll
        for (int dj = 0; dj <= 1; ++dj)
#pragma unroll
            for (int di = 0; di <= 1; ++di) {
                const int n = ix(d, i + di, j + dj);
                const double ux = d.ux[n], uy = d.uy[n];
                umax = rmax(umax, sqrt(ux * ux + uy * uy));
            }
        const double ws = cs + umax;
        // NaN and +-0 never raise the max (std::max keeps its first argument)
        if (ws > 0.0) {
            const unsigned long long b = (unsigned long long)__double_as_longlong(ws);
            wb = b > wb ? b : wb;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, wb, o);
        wb = v > wb ? v : wb;
    }
    __shared__ unsigned long long sw[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sw[warp] = wb;
    __syncthreads();
    if (warp == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        wb = lane < nw ? sw[lane] : 0ull;
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long v = __shfl_xor_sync(0xffffffffu, wb, o);
            wb = v > wb ? v : wb;
        }
        if (lane == 0 && wb) atomicMax(into_next ? &d.ctl->next_wmax_bits : &d.ctl->wmax_bits, wb);
    }
}

// harness.cpp:311-312 and the run loop's dt = min(dt, t_end - t) (:395)
__global__ void k_cfl_final(Ctl* c, double dx, double dy, int run_loop) {
    pdl_enter();
    if (c->err_key != kNoErr || c->done) return;
    const double wmax = __longlong_as_double((long long)c->wmax_bits);
    if (!(wmax > 0.0) || !isfinite(wmax)) {
        raise(c, ekey(PH_CFL_WAVE, 0x1FFFFFF - 32, 0, 0));
        return;
    }
    double dt = c->cfl * rmin(dx, dy) / wmax;
    c->last_dt = dt;
    if (run_loop) dt = rmin(dt, c->t_end - c->time);
    c->dt = dt;
}

// ---------------------------------------------------------------------------
// ghost layers (state.cpp:47-108)
// ---------------------------------------------------------------------------
__device__ __forceinline__ int wrap_cell(int i, int n, int periodic) {
    if (periodic) return (i % n + n) % n;
    if (i < 0) return -1 - i;
    if (i >= n) return 2 * n - 1 - i;
    return i;
}
// thread index -> ghost cell position of the (nx+4)x(ny+4) ring
__device__ __forceinline__ bool ghost_cell_pos(int t, int nx, int ny, int& i, int& j) {
    const int W = nx + 2 * G;
    if (t < 2 * G * W) {  // bottom and top strips
        const int r = t / W;
        i = t % W - G;
        j = r < G ? r - G : ny + (r - G);
        return true;
    }
    t -= 2 * G * W;
    if (t < 2 * G * ny) {
        const int col = t / ny;
        j = t % ny;
        i = col < G ? col - G : nx + (col - G);
        return true;
    }
    return false;
}

// (one field f per call: the launch spreads the fields over blockIdx.z, so
// every thread does one independent load / store instead of a chain)
__device__ __forceinline__ void ghost_cells_at(const Dev& d, const FieldList& fl, int t, int f) {
    int i, j;
    if (!ghost_cell_pos(t, d.nx, d.ny, i, j)) return;
    if (!in(d.win_c, i, j)) return;
    const int is = wrap_cell(i, d.nx, d.per_x), js = wrap_cell(j, d.ny, d.per_y);
    double* p = fl.f[f];
    p[ix(d, i, j)] = p[ix(d, is, js)];
}

// fill_ghost_nodes (state.cpp:87-108) for Vec2 pairs (x, y).
// (one Vec2 pair (fl.f[f0], fl.f[f0 + 1]) per call, f0 even)
__device__ __forceinline__ void ghost_nodes_at(const Dev& d, const FieldList& fl, int t, int f0) {
    const int nx = d.nx, ny = d.ny;
    const int W = nx + 1 + 2 * G;
    int i, j;
    if (t < 2 * G * W) {
        const int r = t / W;
        i = t % W - G;
        j = r < G ? r - G : ny + 1 + (r - G);
    } else {
        t -= 2 * G * W;
        if (t < 2 * G * (ny + 1)) {
            const int col = t / (ny + 1);
            j = t % (ny + 1);
            i = col < G ? col - G : nx + 1 + (col - G);
        } else {
            // boundary-node wall zeroing (state.cpp:90-95)
            t -= 2 * G * (ny + 1);
            if (t < 2 * (ny + 1)) {
                j = t % (ny + 1);
                i = t < ny + 1 ? 0 : nx;
                if (!d.per_x && in(d.win_n, i, j)) fl.f[f0][ix(d, i, j)] = 0.0;
                return;
            }
            t -= 2 * (ny + 1);
            if (t < 2 * (nx + 1)) {
                i = t % (nx + 1);
                j = t < nx + 1 ? 0 : ny;
                if (!d.per_y && in(d.win_n, i, j)) fl.f[f0 + 1][ix(d, i, j)] = 0.0;
            }
            return;
        }
    }
    if (!in(d.win_n, i, j)) return;
    // wrap_node (state.cpp:71-80)
    int si, sj;
    bool fi = false, fj = false;
    if (d.per_x) {
        si = i % nx;
        if (si < 0) si += nx;
    } else if (i < 0) {
        si = -i;
        fi = true;
    } else if (i > nx) {
        si = 2 * nx - i;
        fi = true;
    } else {
        si = i;
    }
    if (d.per_y) {
        sj = j % ny;
        if (sj < 0) sj += ny;
    } else if (j < 0) {
        sj = -j;
        fj = true;
    } else if (j > ny) {
        sj = 2 * ny - j;
        fj = true;
    } else {
        sj = j;
    }
    // the source is read as it is after the wall zeroing of the same call
    const bool zx = !d.per_x && (si == 0 || si == nx);
    const bool zy = !d.per_y && (sj == 0 || sj == ny);
    const int dst = ix(d, i, j), src = ix(d, si, sj);
    double vx = zx ? 0.0 : fl.f[f0][src];
    double vy = zy ? 0.0 : fl.f[f0 + 1][src];
    if (fi) vx = -vx;
    if (fj) vy = -vy;
    fl.f[f0][dst] = vx;
    fl.f[f0 + 1][dst] = vy;
}

// sync_derived, state.cpp:120-143, over every cell including ghosts.
// src: 0 = current state (API), 1 = next state (after a remap).
template <int NM>
__global__ void k_sync(Dev d, int next, int respect_halt) {
    pdl_enter();
    if (respect_halt && halted(d.ctl)) return;
    int i, j;
    tid2(i, j, d.win_c.i0, d.win_c.j0);
    if (!in(d.win_c, i, j) || i < -G || j < -G || i >= d.nx + G || j >= d.ny + G) return;
    const int c = ix(d, i, j);
    const double cv = d.cv;
    double m = 0.0, me = 0.0, p = 0.0;
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        const double ka = next ? d.nk[a][c] : d.k[a][c];
        if (ka <= 0.0) continue;
        const double ma = next ? d.nm[a][c] : d.m[a][c];
        const double ea = next ? d.ne[a][c] : d.e[a][c];
        m += ma;
        me += ma * ea;
        if (ka < kThermoTol) continue;
        const double rho_a = rho_of(d, ma, ka);
        p += ka * eos_p(d, a, rho_a, ea);
    }
    double* om = next ? d.nm_mix : const_cast<double*>(d.m_mix);
    double* oe = next ? d.ne_mix : const_cast<double*>(d.e_mix);
    double* orho = next ? d.nrho_mix : const_cast<double*>(d.rho_mix);
    double* op = next ? d.np_mix : const_cast<double*>(d.p_mix);
    double* ov = next ? d.nvol : d.vol;
    om[c] = m;
    oe[c] = m > 0.0 ? me / m : 0.0;
    orho[c] = div_cv(d, m);
    op[c] = p;
    ov[c] = cv;
}

// ---------------------------------------------------------------------------
// Lagrangian phase (lagrange.cpp)
// ---------------------------------------------------------------------------
// quad_volume_disp, lagrange.cpp:36-46, with node displacements s*u
__device__ __forceinline__ double quad_vol4(const Dev& d, double u00x, double u00y, double u10x, double u10y,
                                            double u11x, double u11y, double u01x, double u01y, double s,
                                            bool& tangled) {
    const double d00x = s * u00x, d00y = s * u00y;
    const double d10x = s * u10x, d10y = s * u10y;
    const double d11x = s * u11x, d11y = s * u11y;
    const double d01x = s * u01x, d01y = s * u01y;
    const double ebx = d.dx + d10x - d00x, eby = d10y - d00y;
    const double elx = d01x - d00x, ely = d.dy + d01y - d00y;
    const double etx = d.dx + d11x - d01x, ety = d11y - d01y;
    const double erx = d11x - d10x, ery = d.dy + d11y - d10y;
    const double s1 = 0.5 * (ebx * ely - eby * elx);
    const double s2 = 0.5 * (etx * ery - ety * erx);
    if (s1 <= 0.0 || s2 <= 0.0) tangled = true;
    return s1 + s2;
}

// compute_q (lagrange.cpp:63-77: div_u_cell :14-20, pseudo_viscosity :7-12,
// mixture_sound_speed :48-59) fused with the cell part of predict
// (lagrange.cpp:89-131, dh = 0.5*dt*u :251-255): one thread per cell.
template <int NM>
__global__ void k_lag_cells(Dev d) {
    pdl_enter();
    if (halted(d.ctl)) return;
    int i, j;
    tid2(i, j, d.r_lagc.i0, d.r_lagc.j0);
    if (!in(d.r_lagc, i, j)) return;
    const bool own = own_cell(d, i, j);
    const double dt = step_dt(d.ctl);
    const int c = ix(d, i, j);
    const int n00 = c, n10 = ix(d, i + 1, j), n01 = ix(d, i, j + 1), n11 = ix(d, i + 1, j + 1);
    const double u00x = d.ux[n00], u00y = d.uy[n00], u10x = d.ux[n10], u10y = d.uy[n10];
    const double u01x = d.ux[n01], u01y = d.uy[n01], u11x = d.ux[n11], u11y = d.uy[n11];
    double ka[NM], ma[NM], en[NM];
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        ka[a] = d.k[a][c];
        ma[a] = d.m[a][c];
        en[a] = d.e[a][c];
    }
    // Q^n
    const double ux_l = 0.5 * (u00x + u01x);
    const double ux_r = 0.5 * (u10x + u11x);
    const double uy_b = 0.5 * (u00y + u10y);
    const double uy_t = 0.5 * (u01y + u11y);
    const double div = div_dx(d, ux_r - ux_l, 1.0) + div_dy(d, uy_t - uy_b, 1.0);
    double q = 0.0;
    if (!(div >= 0.0)) {
        double cs = 0.0;
        bool bad = false;
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            if (ka[a] < kThermoTol) continue;
            const double rho_a = rho_of(d, ma[a], ka[a]);
            const double pa = eos_p(d, a, rho_a, en[a]);
            cs += ka[a] * sound(d, a, rho_a, pa, bad);
        }
        if (bad && own) raise(d.ctl, ekey(PH_Q_UNPHYS, j, i, 0));
        const double rho = d.rho_mix[c];
        const double du = d.L * fabs(div);
        q = rho * d.a1 * du * cs + d.a2 * rho * du * du;
    }
    d.q[c] = q;
    // predict
    bool tangled = false;
    const double vol = quad_vol4(d, u00x, u00y, u10x, u10y, u11x, u11y, u01x, u01y, 0.5 * dt, tangled);
    if (tangled && own) raise(d.ctl, ekey(PH_PRED_TANGLED, j, i, 0));
    double pmix = 0.0;
    int floors = 0;
    const double cv = d.cv;
    // h2d_predict also returns HalfStepState::vol_half / e_half (lagrange.hpp:14-24)
    const bool half_out = d.volh != nullptr && in(d.own_c, i, j);
    if (half_out) d.volh[c] = vol;
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        double pa_h = 0.0;
        double eh = ka[a] > 0.0 ? en[a] : 0.0;  // frozen sliver (lagrange.cpp:110)
        if (!(ka[a] < kThermoTol)) {
            const double rho_n = rho_of(d, ma[a], ka[a]);
            const double rho_h = ma[a] / (ka[a] * vol);
            const double pa_n = eos_p(d, a, rho_n, en[a]);
            double ea = en[a] - (pa_n + q) * (1.0 / rho_h - 1.0 / rho_n);
            const double efloor = 1e-8 * fabs(en[a]);
            if (ea < efloor) {
                ea = efloor;
                ++floors;
            }
            pa_h = eos_p(d, a, rho_h, ea);
            pmix += ka[a] * pa_h;
            eh = ea;
        }
        d.ph[a][c] = pa_h;
        if (half_out) d.eh[a][c] = eh;
    }
    d.pmh[c] = pmix;
    if (floors && own) bump_floor(d.ctl, floors);
}

// Node part of predict (lagrange.cpp:135-142: nodal_mass state.cpp:34-36,
// grad_pq_node lagrange.cpp:22-30) and correct (lagrange.cpp:146-196), fused
// per 32x8 tile: u_half of the tile's (33 x 9) nodes goes to shared memory,
// u_lag is written per node and e_lag per cell from the four u_half.
constexpr int LTX = 32, LTY = 8;

// (row, column) of a flat tile index t = tid, tid + BS, ... over rows of W
// entries, stepped incrementally (no per-iteration integer divide / modulo)
template <int W, int BS>
struct RowCol {
    int r, c;
    __device__ __forceinline__ explicit RowCol(int t) : r(t / W), c(t % W) {}
    __device__ __forceinline__ void step() {
        r += BS / W;
        c += BS % W;
        if (c >= W) {
            c -= W;
            ++r;
        }
    }
};
// mode 0: predict's node part + correct (lagrange_step); 1: predict's node
// part only (h2d_predict); 2: correct only, u_half read from its planes
// (h2d_correct on a caller's HalfStepState)
template <int NM>
__global__ void __launch_bounds__(LTX * LTY) k_lag_nodes(Dev d, int write_vol_lag, int mode) {
    pdl_enter();
    constexpr int NN = (LTX + 1) * (LTY + 1);
    __shared__ double shx[NN], shy[NN];
    __shared__ int s_halt;
    const int tid = threadIdx.x;
    if (tid == 0) s_halt = halted(d.ctl);
    __syncthreads();
    if (s_halt) return;
    const Rng rn = d.r_lagn;
    const int i0 = rn.i0 + blockIdx.x * LTX, j0 = rn.j0 + blockIdx.y * LTY;
    const double dt = step_dt(d.ctl);
    for (int t = tid; t < NN; t += LTX * LTY) {
        const int i = i0 + t % (LTX + 1), j = j0 + t / (LTX + 1);
        double hx = 0.0, hy = 0.0;
        if (mode == 2) {
            if (in(rn, i, j)) {
                const int e = ix(d, i, j);
                hx = d.uhx[e];
                hy = d.uhy[e];
                if ((i < i0 + LTX || i == rn.i1 - 1) && (j < j0 + LTY || j == rn.j1 - 1)) {
                    d.ulx[e] = 2.0 * hx - d.ux[e];
                    d.uly[e] = 2.0 * hy - d.uy[e];
                }
            }
        } else if (in(rn, i, j)) {
            const int a = ix(d, i - 1, j - 1), b = ix(d, i, j - 1), c = ix(d, i - 1, j), e = ix(d, i, j);
            const double mp = 0.25 * (d.m_mix[a] + d.m_mix[b] + d.m_mix[c] + d.m_mix[e]);
            const double rho_p = div_cv(d, mp);
            const double pq_a = d.pmh[a] + d.q[a], pq_b = d.pmh[b] + d.q[b];
            const double pq_c = d.pmh[c] + d.q[c], pq_e = d.pmh[e] + d.q[e];
            const double gx = div_dx(d, pq_b + pq_e - pq_a - pq_c, 2.0);  // pq(i,j-1)+pq(i,j)-pq(i-1,j-1)-pq(i-1,j)
            const double gy = div_dy(d, pq_c + pq_e - pq_a - pq_b, 2.0);  // pq(i-1,j)+pq(i,j)-pq(i-1,j-1)-pq(i,j-1)
            const double sc = 0.5 * dt / rho_p;
            const double ux = d.ux[e], uy = d.uy[e];
            hx = ux - gx * sc;
            hy = uy - gy * sc;
            if ((i < i0 + LTX || i == rn.i1 - 1) && (j < j0 + LTY || j == rn.j1 - 1)) {
                d.uhx[e] = hx;
                d.uhy[e] = hy;
                d.ulx[e] = 2.0 * hx - ux;
                d.uly[e] = 2.0 * hy - uy;
            }
        }
        shx[t] = hx;
        shy[t] = hy;
    }
    if (mode == 1) return;
    __syncthreads();
    const int tx = tid % LTX, ty = tid / LTX;
    const int i = i0 + tx, j = j0 + ty;
    if (!in(d.r_lage, i, j)) return;
    const bool own = own_cell(d, i, j);
    const int q00 = tx + ty * (LTX + 1), q10 = q00 + 1, q01 = q00 + LTX + 1, q11 = q01 + 1;
    bool tangled = false;
    const double vol =
        quad_vol4(d, shx[q00], shy[q00], shx[q10], shy[q10], shx[q11], shy[q11], shx[q01], shy[q01], dt, tangled);
    if (tangled && own) raise(d.ctl, ekey(PH_CORR_TANGLED, j, i, 0));
    const int n = ix(d, i, j);
    if (write_vol_lag) d.vol_lag[n] = vol;
    int floors = 0;
    const double cv = d.cv;
    const double qn = d.q[n];
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        const double ka = d.k[a][n];
        const double en = d.e[a][n];
        double ea = 0.0;
        if (ka < kThermoTol) {
            if (ka > 0.0) ea = en;
        } else {
            const double ma = d.m[a][n];
            const double rho_n = rho_of(d, ma, ka);
            const double rho_l = ma / (ka * vol);
            ea = en - (d.ph[a][n] + qn) * (1.0 / rho_l - 1.0 / rho_n);
            const double efloor = 1e-8 * fabs(en);
            if (ea < efloor) {
                ea = efloor;
                ++floors;
            }
        }
        d.el[a][n] = ea;
    }
    if (floors && own) bump_floor(d.ctl, floors);
}

// The run-loop Lagrangian phase in ONE kernel per 32x8 node tile: Q and the
// cell part of predict are evaluated for the tile's (34 x 10) surrounding
// cells into shared memory (a ghost cell is evaluated at its wrapped
// interior source, which is exactly what fill_ghost_cells would copy,
// lagrange.cpp:75,132), then u_half / u_lag per node and e_lag per own cell
// (lagrange.cpp:135-142, 146-196). Q, p_half and p_mix_half never leave the
// chip; the API path (h2d_lagrange_step) keeps the two-kernel form because
// it returns Q.
#ifndef H2D_FTY
#define H2D_FTY 8
#endif
// 352 threads (11 warps) for a 32 x 8 tile: the 34 x 10 cell pass and the
// 33 x 9 node pass take one round each (256 threads need two, the second
// mostly idle at the barrier); CTAs per SM per material count as measured
// (profiles/r02_var_lagthreads.jsonl, r02_var_lagthreads2.jsonl)
#ifndef H2D_LAG_NT
#define H2D_LAG_NT 352
#endif
#ifndef H2D_FMINB
#define H2D_FMINB(NM) ((NM) == 2 ? 4 : 3)
#endif
#ifndef H2D_LAG_INTERIOR
#define H2D_LAG_INTERIOR 1
#endif
// INT: an interior tile (uniform over the CTA, see k_lag_fused): every cell
// of its 34 x 10 pass is a mesh cell inside the window (no ghost image, no
// wrap), every node of its 33 x 9 pass lies inside r_lagn off the walls, and
// every own cell is in r_lagc / r_lage and owned, so the range tests of the
// general path are all true and are compiled out (same arithmetic, same
// bits; C4 Lagrange 2.81 -> 2.60 ms, profiles/r02_var_laginterior.jsonl)
template <int NM, bool INT>
__device__ __forceinline__ void lag_fused_body(const Dev& d, const int i0, const int j0, double* s_q, double* s_pmh,
                                               double (*s_ph)[(LTX + 2) * (H2D_FTY + 2)], double* s_mm, double* shx,
                                               double* shy) {
    constexpr int LTY = H2D_FTY;
    constexpr int NT = H2D_LAG_NT;  // threads (>= the tile's cells; extra ones help the halo passes)
    constexpr int CW = LTX + 2, CH = LTY + 2, NC = CW * CH, NN = (LTX + 1) * (LTY + 1);
    const int tid = threadIdx.x;
    const int nx = d.nx, ny = d.ny;
    const Rng rn = d.r_lagn;
    const double dt = step_dt(d.ctl);
    const double cv = d.cv;
    // ---- cells [i0-1, i0+LTX] x [j0-1, j0+LTY]: Q^n and predict
    RowCol<CW, NT> rc0(tid);
    for (int t = tid; t < NC; t += NT, rc0.step()) {
        const int ci = i0 - 1 + rc0.c, cj = j0 - 1 + rc0.r;
        double q = 0.0, pmix = 0.0, ph[NM] = {}, mmix = 0.0;
        if (INT || (in(d.win_c, ci, cj) && ci >= -1 && cj >= -1 && ci <= nx && cj <= ny)) {
            const int i = (!INT && (ci < 0 || ci >= nx)) ? wrap_cell(ci, nx, d.per_x) : ci;
            const int j = (!INT && (cj < 0 || cj >= ny)) ? wrap_cell(cj, ny, d.per_y) : cj;
            // the canonical evaluation (errors, floor counts): an own interior cell of this tile
            const bool canon = ci == i && cj == j && ci >= i0 && ci < i0 + LTX && cj >= j0 && cj < j0 + LTY &&
                               (INT || (in(d.r_lagc, i, j) && own_cell(d, i, j)));
            const int c = ix(d, i, j);
            const int n10 = ix(d, i + 1, j), n01 = ix(d, i, j + 1), n11 = ix(d, i + 1, j + 1);
            const double u00x = d.ux[c], u00y = d.uy[c], u10x = d.ux[n10], u10y = d.uy[n10];
            const double u01x = d.ux[n01], u01y = d.uy[n01], u11x = d.ux[n11], u11y = d.uy[n11];
            double ka[NM], ma[NM], en[NM];
#pragma unroll
            for (int a = 0; a < NM; ++a) {
                ka[a] = d.k[a][c];
                ma[a] = d.m[a][c];
                en[a] = d.e[a][c];
            }
            // the State's m_mix / rho_mix (sync_derived, state.cpp:120-143) from
            // the partial masses: the run loop does not keep the derived planes
            // (they are rebuilt bit-identically when the State is read)
#pragma unroll
            for (int a = 0; a < NM; ++a)
                if (ka[a] > 0.0) mmix += ma[a];
            const double ux_l = 0.5 * (u00x + u01x);
            const double ux_r = 0.5 * (u10x + u11x);
            const double uy_b = 0.5 * (u00y + u10y);
            const double uy_t = 0.5 * (u01y + u11y);
            const double div = div_dx(d, ux_r - ux_l, 1.0) + div_dy(d, uy_t - uy_b, 1.0);
            if (!(div >= 0.0)) {
                double cs = 0.0;
                bool bad = false;
#pragma unroll
                for (int a = 0; a < NM; ++a) {
                    if (ka[a] < kThermoTol) continue;
                    const double rho_a = rho_of(d, ma[a], ka[a]);
                    const double pa = eos_p(d, a, rho_a, en[a]);
                    cs += ka[a] * sound(d, a, rho_a, pa, bad);
                }
                if (bad && canon) raise(d.ctl, ekey(PH_Q_UNPHYS, j, i, 0));
                const double rho = div_cv(d, mmix);
                const double du = d.L * fabs(div);
                q = rho * d.a1 * du * cs + d.a2 * rho * du * du;
            }
            bool tangled = false;
            const double vol = quad_vol4(d, u00x, u00y, u10x, u10y, u11x, u11y, u01x, u01y, 0.5 * dt, tangled);
            if (tangled && canon) raise(d.ctl, ekey(PH_PRED_TANGLED, j, i, 0));
            int floors = 0;
#pragma unroll
            for (int a = 0; a < NM; ++a) {
                if (!(ka[a] < kThermoTol)) {
                    const double rho_n = rho_of(d, ma[a], ka[a]);
                    const double pa_n = eos_p(d, a, rho_n, en[a]);
                    // vol == cv (a still or uniformly moving cell, lagrange.cpp:
                    // 34-35) gives rho_h == rho_n bit for bit, so 1/rho_h - 1/rho_n
                    // is +0 whenever 1/rho_n is finite: skip the three divides
                    double rho_h = rho_n, dv = 0.0;
                    if (!(vol == cv && fabs(rho_n) >= DBL_MIN)) {
                        rho_h = ma[a] / (ka[a] * vol);
                        dv = 1.0 / rho_h - 1.0 / rho_n;
                    }
                    double ea = en[a] - (pa_n + q) * dv;
                    const double efloor = 1e-8 * fabs(en[a]);
                    if (ea < efloor) {
                        ea = efloor;
                        ++floors;
                    }
                    ph[a] = eos_p(d, a, rho_h, ea);
                    pmix += ka[a] * ph[a];
                }
            }
            if (floors && canon) bump_floor(d.ctl, floors);
        }
        s_q[t] = q;
        s_pmh[t] = pmix;
        s_mm[t] = mmix;
#pragma unroll
        for (int a = 0; a < NM; ++a) s_ph[a][t] = ph[a];
    }
    __syncthreads();
    // ---- nodes: u_half, u_lag
    RowCol<LTX + 1, NT> rc1(tid);
    for (int t = tid; t < NN; t += NT, rc1.step()) {
        const int i = i0 + rc1.c, j = j0 + rc1.r;
        double hx = 0.0, hy = 0.0;
        if (INT || in(rn, i, j)) {
            const int ta = rc1.c + rc1.r * CW;  // cell (i-1, j-1) in the cell tile
            const int tb = ta + 1, tc = ta + CW, te = tc + 1;
            const int e = ix(d, i, j);
            const double mp = 0.25 * (s_mm[ta] + s_mm[tb] + s_mm[tc] + s_mm[te]);
            const double rho_p = div_cv(d, mp);
            const double pq_a = s_pmh[ta] + s_q[ta], pq_b = s_pmh[tb] + s_q[tb];
            const double pq_c = s_pmh[tc] + s_q[tc], pq_e = s_pmh[te] + s_q[te];
            const double gx = div_dx(d, pq_b + pq_e - pq_a - pq_c, 2.0);
            const double gy = div_dy(d, pq_c + pq_e - pq_a - pq_b, 2.0);
            const double sc = 0.5 * dt / rho_p;
            const double ux = d.ux[e], uy = d.uy[e];
            hx = ux - gx * sc;
            hy = uy - gy * sc;
            // fill_ghost_nodes(u_half) zeroes the wall-normal component on the
            // wall nodes (state.cpp:90-95) before correct reads u_half
            // (lagrange.cpp:142,155): the wall-node gradient is a rounding
            // residue of ((b + e) - a) - c with mirrored a = b, c = e
            if (!INT && !d.per_x && (i == 0 || i == nx)) hx = 0.0;
            if (!INT && !d.per_y && (j == 0 || j == ny)) hy = 0.0;
            if (INT ? (i < i0 + LTX && j < j0 + LTY)
                    : ((i < i0 + LTX || i == rn.i1 - 1) && (j < j0 + LTY || j == rn.j1 - 1))) {
                d.uhx[e] = hx;
                d.uhy[e] = hy;
                d.ulx[e] = 2.0 * hx - ux;
                d.uly[e] = 2.0 * hy - uy;
            }
        }
        shx[t] = hx;
        shy[t] = hy;
    }
    __syncthreads();
    // ---- own cells: correct
    if (tid >= LTX * LTY) return;
    const int tx = tid % LTX, ty = tid / LTX;
    const int i = i0 + tx, j = j0 + ty;
    if (!INT && !in(d.r_lage, i, j)) return;
    const bool own = INT || own_cell(d, i, j);
    const int q00 = tx + ty * (LTX + 1), q10 = q00 + 1, q01 = q00 + LTX + 1, q11 = q01 + 1;
    bool tangled = false;
    const double vol =
        quad_vol4(d, shx[q00], shy[q00], shx[q10], shy[q10], shx[q11], shy[q11], shx[q01], shy[q01], dt, tangled);
    if (tangled && own) raise(d.ctl, ekey(PH_CORR_TANGLED, j, i, 0));
    const int n = ix(d, i, j);
    const int tcell = (tx + 1) + (ty + 1) * CW;
    int floors = 0;
    const double qn = s_q[tcell];
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        const double ka = d.k[a][n];
        const double en = d.e[a][n];
        double ea = 0.0;
        if (ka < kThermoTol) {
            if (ka > 0.0) ea = en;
        } else {
            const double ma = d.m[a][n];
            const double rho_n = rho_of(d, ma, ka);
            double dv = 0.0;  // vol == cv: rho_l == rho_n, the difference of inverses is +0
            if (!(vol == cv && fabs(rho_n) >= DBL_MIN)) {
                const double rho_l = ma / (ka * vol);
                dv = 1.0 / rho_l - 1.0 / rho_n;
            }
            ea = en - (s_ph[a][tcell] + qn) * dv;
            const double efloor = 1e-8 * fabs(en);
            if (ea < efloor) {
                ea = efloor;
                ++floors;
            }
        }
        d.el[a][n] = ea;
    }
    if (floors && own) bump_floor(d.ctl, floors);
}

template <int NM>
__global__ void __launch_bounds__(H2D_LAG_NT, H2D_FMINB(NM)) k_lag_fused(Dev d) {
    pdl_enter();
    constexpr int LTY = H2D_FTY;
    constexpr int NC = (LTX + 2) * (LTY + 2), NN = (LTX + 1) * (LTY + 1);
    __shared__ double s_q[NC], s_pmh[NC], s_ph[NM][NC], s_mm[NC];
    __shared__ double shx[NN], shy[NN];
    __shared__ int s_halt, s_int;
    const Rng rn = d.r_lagn;
    const int i0 = rn.i0 + blockIdx.x * LTX, j0 = rn.j0 + blockIdx.y * LTY;
    if (threadIdx.x == 0) {
        s_halt = halted(d.ctl);
        // interior tile: cells [i0-1, i0+LTX] x [j0-1, j0+LTY] are mesh cells
        // inside the window, nodes [i0, i0+LTX] x [j0, j0+LTY] lie inside
        // r_lagn, off the walls and before the range's last row / column, the
        // own cells inside r_lagc, r_lage and the owned range (one thread
        // evaluates the ~60 instructions of it, not all 352)
        bool interior = false;
        if (H2D_LAG_INTERIOR) {
            const int ia = i0 - 1, ib = i0 + LTX, ja = j0 - 1, jb = j0 + LTY;  // inclusive cell bounds of the pass
            interior = ia >= 0 && ib < d.nx && ja >= 0 && jb < d.ny && in(d.win_c, ia, ja) && in(d.win_c, ib, jb) &&
                       i0 >= 1 && ib <= d.nx - 1 && j0 >= 1 && jb <= d.ny - 1 && ib < rn.i1 - 1 && jb < rn.j1 - 1 &&
                       in(d.r_lagc, i0, j0) && in(d.r_lagc, ib - 1, jb - 1) && in(d.r_lage, i0, j0) &&
                       in(d.r_lage, ib - 1, jb - 1) && own_cell(d, i0, j0) && own_cell(d, ib - 1, jb - 1);
        }
        s_int = interior;
    }
    __syncthreads();
    if (s_halt) return;
    if (d.lag_sel && (in(d.lag_inner, i0, j0) != (d.lag_sel == 1))) return;
    if (s_int)
        lag_fused_body<NM, true>(d, i0, j0, s_q, s_pmh, s_ph, s_mm, shx, shy);
    else
        lag_fused_body<NM, false>(d, i0, j0, s_q, s_pmh, s_ph, s_mm, shx, shy);
}

// ---------------------------------------------------------------------------
// DirectCF remap (remap.cpp:734-1073)
// ---------------------------------------------------------------------------
// make_work, remap.cpp:116-140, over every cell incl. ghosts: the next-state
// buffers become the Work arrays.
// remap_velocity == false: the new u is lag.u_lag unchanged (remap.cpp:130,
// 993); the Work arrays of make_work (remap.cpp:116-140) are otherwise read in
// place (w.m = state m, w.e = e_lag, w.k = state k, w.me = m * e_lag), so the
// flux threads never race with finalize writing the next State.
__global__ void k_copy_u(Dev d) {
    pdl_enter();
    if (halted(d.ctl)) return;
    int i, j;
    tid2(i, j, d.win_n.i0, d.win_n.j0);
    if (!in(d.win_n, i, j)) return;
    const int c = ix(d, i, j);
    d.nux[c] = d.ulx[c];
    d.nuy[c] = d.uly[c];
}

// cf_face_flux_x, remap.cpp:27-47 (Y faces call it with swapped components)
__device__ __forceinline__ void face_flux(double ym, double yp, double dmx, double dmy, double dpx, double dpy,
                                          double& dv, double& wl, double& wh) {
    dv = 0.0;
    wl = 0.0;
    wh = 0.0;
    const double wlo = ym + rmax(0.0, dmy);
    const double whi = yp + rmin(0.0, dpy);
    if (whi <= wlo) return;
    wl = wlo;
    wh = whi;
    // static face line (both offsets zero): the trapezoid volume is a signed
    // zero, and no output depends on the sign of a zero face volume (it is
    // skipped by `dvol == 0.0` and adds nothing to vlag), so skip the divide
    if (dmx == 0.0 && dpx == 0.0) return;
    const double den = (yp + dpy) - (ym + dmy);
    double xlo, xhi;
    if (fabs(den) < 1e-300) {
        xlo = xhi = 0.5 * (dmx + dpx);
    } else {
        // a zero numerator over a finite divisor: the exact signed zero of the
        // quotient (0 * den has the sign of 0 / den) without the divide's slow path
        const double num = dpx - dmx;
        const double slope = (num == 0.0 && fabs(den) < CUDART_INF) ? num * den : num / den;
        xlo = dmx + slope * (wlo - (ym + dmy));
        xhi = dmx + slope * (whi - (ym + dmy));
    }
    dv = 0.5 * (xlo + xhi) * (whi - wlo);
}

// ---------------------------------------------------------------------------
// The fused remap tile kernel (remap.cpp:739-991): for a 32x8 tile of cells it
// computes, in shared memory, the axis geometry, face / corner flux geometry,
// Lagrangian volumes, densities, centroids and interfaces of the tile plus a
// two-cell halo (the reference's ghosted ranges at the mesh edge), then every
// face and corner flux of the tile once, then gathers them per cell in the
// reference's order and runs the per-cell part of finalize_cells.  Only the
// State inputs (u_half, e_lag, m, k, normals) are read from HBM and only the
// Work outputs (m, me, e, k, mcell, sliver flags) and the mass fluxes the dual
// pass needs (dmx, dmy, dmc) are written back.
// ---------------------------------------------------------------------------
constexpr int RTX = 32, RTY = 8;
constexpr int RCW = RTX + 4, RCH = RTY + 4;  // cell region [i0-2, i0+RTX+2)
constexpr int RNW = RTX + 6, RNH = RTY + 5;  // node region [i0-2, i0+RTX+3] (a 38-wide TMA box row = 304 B)
constexpr int RNN = RNW * RNH, RNC = RCW * RCH;
constexpr int NXF = (RTX + 1) * RTY, NYF = RTX * (RTY + 1), NCF = (RTX + 1) * (RTY + 1);
constexpr int NIT = NCF > NXF ? (NCF > NYF ? NCF : NYF) : (NXF > NYF ? NXF : NYF);  // item buffer
constexpr int RCELL1 = 5, RCELL2 = 10;  // cell arrays per material count
__host__ __device__ constexpr int al16(int n) { return (n + 15) & ~15; }  // smem planes start 128-byte aligned (TMA destinations)

template <int NM>
struct Tile {
    int ci0, cj0;  // origin of both regions: (i0 - 2, j0 - 2)
    double *hx, *hy, *fdx, *fdy, *fxdv, *fydv;  // nodes
    double *vl, *rho[kMatSlots], *el[kMatSlots], *kk[kMatSlots], *xl2x, *xl2y, *ifd, *ifd2;  // cells
    // (ifd2: the Direct engine's Y-displaced interfaces; ifd its X-displaced ones)
    // flux items of one sub-phase (X faces, then Y faces, then corners share
    // the buffer): dm, dme, dva per material
    double* it[3][kMatSlots];
    __device__ __forceinline__ int c(int i, int j) const {
        H2D_CHECK(i - ci0 >= 0 && i - ci0 < RCW && j - cj0 >= 0 && j - cj0 < RCH);
        return (i - ci0) + (j - cj0) * RCW;
    }
    __device__ __forceinline__ int n(int i, int j) const {
        H2D_CHECK(i - ci0 >= 0 && i - ci0 < RNW && j - cj0 >= 0 && j - cj0 < RNH);
        return (i - ci0) + (j - cj0) * RNW;
    }
    // cf_corner_flux (remap.cpp:16-25) at region node q, recomputed from the
    // staged u_half (zero outside the window); sx / sy are meaningful only
    // when the returned volume is nonzero
    __device__ __forceinline__ double cfv(int q, double dt, int& sx, int& sy) const {
        const double ddx = hx[q] * dt, ddy = hy[q] * dt;
        sx = ddx > 0.0 ? 1 : -1;
        sy = ddy > 0.0 ? 1 : -1;
        return fabs(ddx * ddy);
    }
    // make_axis_geom (remap.cpp:315-320) from the face-mean displacements
    __device__ __forceinline__ double xlcx(const Dev& d, int i, int j) const {
        const int q = n(i, j);
        return d.x0 + (i + 0.5) * d.dx + 0.5 * (fdx[q] + fdx[q + 1]);
    }
    __device__ __forceinline__ double wlx(const Dev& d, int i, int j) const {
        const int q = n(i, j);
        return d.dx + (fdx[q + 1] - fdx[q]);
    }
    __device__ __forceinline__ double xlcy(const Dev& d, int i, int j) const {
        const int q = n(i, j);
        return d.y0 + (j + 0.5) * d.dy + 0.5 * (fdy[q] + fdy[q + RNW]);
    }
    __device__ __forceinline__ double wly(const Dev& d, int i, int j) const {
        const int q = n(i, j);
        return d.dy + (fdy[q + RNW] - fdy[q]);
    }
};

template <int NM, bool DIR = false>
constexpr size_t remap_smem_bytes() {
    return sizeof(double) * (6 * al16(RNN) + (NM == 1 ? RCELL1 : RCELL2 + 3 * (NM - 2) + (DIR ? 1 : 0)) * al16(RNC) +
                             3 * NM * al16(NIT)) + 128;
}

template <int NM, bool DIR = false>
__device__ __forceinline__ Tile<NM> carve_tile(char* base, int ci0, int cj0) {
    Tile<NM> T;
    T.ci0 = ci0;
    T.cj0 = cj0;
    double* p = reinterpret_cast<double*>(base);
    auto take = [&](int n) {
        double* r = p;
        p += al16(n);
        return r;
    };
    T.hx = take(RNN);
    T.hy = take(RNN);
    T.fdx = take(RNN);
    T.fdy = take(RNN);
    T.fxdv = take(RNN);
    T.fydv = take(RNN);
    T.vl = take(RNC);
    T.xl2x = take(RNC);
    T.xl2y = take(RNC);
    for (int a = 0; a < NM; ++a) {
        T.rho[a] = take(RNC);
        T.el[a] = take(RNC);
    }
    if (NM >= 2) {
        for (int a = 0; a < NM; ++a) T.kk[a] = take(RNC);
        T.ifd = take(RNC);
        T.ifd2 = DIR ? take(RNC) : T.ifd;
    }
    for (int k = 0; k < 3; ++k)
        for (int a = 0; a < NM; ++a) T.it[k][a] = take(NIT);
    return T;
}

// The non-default corner schemes and the Multid faces read their 3x3
// stencils from the tile themselves, out of line: the default LinearDiag path
// keeps its stencil in registers (an array whose address is taken would move
// to local memory for every path)
struct Pair2 {  // two results and the "non-increasing centroid" flag, returned by value
    double a, b;
    int bad;
};
__device__ __noinline__ Pair2 corner_other_tile(int scheme, double dgx, double dgy, const double* rho,
                                                const double* el, const double* x2x, const double* x2y, int dc,
                                                Kin k) {
    double sr[9], se[9], xlx[9], xly[9];
    for (int q = 0; q < 3; ++q)
        for (int p = 0; p < 3; ++p) {
            const int sidx = dc + (p - 1) + (q - 1) * RCW;
            sr[p * 3 + q] = rho[sidx];
            se[p * 3 + q] = el[sidx];
            xlx[p * 3 + q] = x2x[sidx];
            xly[p * 3 + q] = x2y[sidx];
        }
    bool bad = false;
    Pair2 r;
    r.a = rmax(corner_value_other(scheme, dgx, dgy, sr, xlx, xly, k, &bad), 0.0);
    r.b = corner_value_other(scheme, dgx, dgy, se, xlx, xly, k, &bad);
    r.bad = bad;
    return r;
}
__device__ __noinline__ Pair2 multid_face_tile(double dgx, double dgy, const double* rho, const double* el,
                                               const double* x2x, const double* x2y, int dc, double bx, double by) {
    double sr[9], se[9], xlx[9], xly[9];
    for (int q = 0; q < 3; ++q)
        for (int p = 0; p < 3; ++p) {
            const int sidx = dc + (p - 1) + (q - 1) * RCW;
            sr[p * 3 + q] = rho[sidx];
            se[p * 3 + q] = el[sidx];
            xlx[p * 3 + q] = x2x[sidx];
            xly[p * 3 + q] = x2y[sidx];
        }
    bool bad = false;
    Pair2 r;
    r.a = multid_eval(dgx, dgy, sr, xlx, xly, bx, by, &bad);
    r.b = multid_eval(dgx, dgy, se, xlx, xly, bx, by, &bad);
    r.bad = bad;
    return r;
}

// The interface rectangle of donor (di, dj) (remap.cpp:807-824): RM 0 the
// DirectCF rectangle through the Lagrangian face midpoints; the Direct
// engine's X- (RM 1) or Y-displaced (RM 2) rectangle (remap.cpp:616-640)
template <int RM, int NM>
__device__ __forceinline__ void iface_rect(const Dev& d, const Tile<NM>& T, int di, int dj, double& lox, double& loy,
                                           double& hix, double& hiy) {
    const double cx = d.x0 + (di + 0.5) * d.dx, cy = d.y0 + (dj + 0.5) * d.dy;
    lox = cx - 0.5 * d.dx + (RM == 2 ? 0.0 : T.fdx[T.n(di, dj)]);
    loy = cy - 0.5 * d.dy + (RM == 1 ? 0.0 : T.fdy[T.n(di, dj)]);
    hix = cx + 0.5 * d.dx + (RM == 2 ? 0.0 : T.fdx[T.n(di + 1, dj)]);
    hiy = cy + 0.5 * d.dy + (RM == 1 ? 0.0 : T.fdy[T.n(di, dj + 1)]);
    if (RM == 1) {  // cen.y -+ hy exactly (no added displacement)
        loy = cy - 0.5 * d.dy;
        hiy = cy + 0.5 * d.dy;
    } else if (RM == 2) {
        lox = cx - 0.5 * d.dx;
        hix = cx + 0.5 * d.dx;
    }
}

// The three-material split of a flux box of donor (di, dj) (oracle
// split_flux, nmat == 3): a mixed donor gives k_r * dvol to the material
// outside its interface pair and splits the rest at the pair's interface; a
// pure donor gives everything to its largest fraction.
template <int NM, int RM = 0>
__device__ __forceinline__ void split_flux3(const Dev& d, const Tile<NM>& T, int di, int dj, double blox,
                                            double bloy, double bhix, double bhiy, double dvol, double* dva) {
    const int c = T.c(di, dj);
    const double k[3] = {T.kk[0][c], T.kk[1][c], T.kk[NM - 1][c]};
    dva[0] = 0.0;
    dva[1] = 0.0;
    dva[NM - 1] = 0.0;
    if (!mixed3(k)) {
        dva[largest3(k)] = dvol;
        return;
    }
    int lo, hi;
    pair3(k, lo, hi);
    const int r = 3 - lo - hi;
    const int g = ix(d, di, dj);
    const double nx = d.nrx[g], ny = d.nry[g], dd = RM == 2 ? T.ifd2[c] : T.ifd[c];
    double lox, loy, hix, hiy;
    iface_rect<RM>(d, T, di, dj, lox, loy, hix, hiy);
    const double rcx = 0.5 * (lox + hix), rcy = 0.5 * (loy + hiy);
    const double bcx = 0.5 * (blox + bhix), bcy = 0.5 * (bloy + bhiy);
    const double bw = bhix - blox, bh = bhiy - bloy;
    double f0;
    if (!(bw * bh > 0.0)) {
        const double sdist = (nx * (bcx - rcx) + ny * (bcy - rcy)) - dd;
        f0 = sdist <= 0.0 ? 1.0 : 0.0;
    } else {
        f0 = clipped_fraction(bw, bh, nx, ny, dd - (nx * (bcx - rcx) + ny * (bcy - rcy)));
    }
    double dr = k[r] > 0.0 ? k[r] * dvol : 0.0;
    const double rest = dvol - dr;
    const double dl = f0 * rest;
    const double dh = rest - dl;
#pragma unroll
    for (int a = 0; a < NM; ++a) dva[a] = a == lo ? dl : (a == hi ? dh : dr);
}

// box_frac0 + split_flux, remap.cpp:243-268, donor cell (di, dj) of the tile
template <int NM, int RM = 0>
__device__ __forceinline__ void split_flux_t(const Dev& d, const Tile<NM>& T, int di, int dj, double blox,
                                             double bloy, double bhix, double bhiy, double dvol, double* dva) {
    dva[0] = dvol;
    if (NM == 1) return;
    dva[1] = 0.0;
    if (NM == 3) {
        split_flux3<NM, RM>(d, T, di, dj, blox, bloy, bhix, bhiy, dvol, dva);
        return;
    }
    const int c = T.c(di, dj);
    const double k0 = T.kk[0][c];
    if (is_mixed(k0)) {
        const int g = ix(d, di, dj);  // mixed donors only: the normal from HBM (L2)
        const double nx = d.nrx[g], ny = d.nry[g], dd = RM == 2 ? T.ifd2[c] : T.ifd[c];
        double lox, loy, hix, hiy;
        iface_rect<RM>(d, T, di, dj, lox, loy, hix, hiy);
        const double rcx = 0.5 * (lox + hix), rcy = 0.5 * (loy + hiy);
        const double bcx = 0.5 * (blox + bhix), bcy = 0.5 * (bloy + bhiy);
        const double bw = bhix - blox, bh = bhiy - bloy;
        const double area = bw * bh;
        double f0;
        if (!(area > 0.0)) {
            const double sdist = (nx * (bcx - rcx) + ny * (bcy - rcy)) - dd;
            f0 = sdist <= 0.0 ? 1.0 : 0.0;
        } else {
            const double dbox = dd - (nx * (bcx - rcx) + ny * (bcy - rcy));
            f0 = clipped_fraction(bw, bh, nx, ny, dbox);
        }
        dva[0] = f0 * dvol;
        dva[1] = dvol - dva[0];
    } else if (k0 < 0.5) {
        dva[0] = 0.0;
        dva[1] = dvol;
    }
}

// Face flux (remap.cpp:850-918) of the X (AX = 1, at node i, row j) or Y
// (AX = 0, at column i, node row j) face; returns the face's dmx / dmy entry.
template <int NM, int AX, bool XC = false, bool DIR = false>
__device__ __forceinline__ double face_item_t(const Dev& d, const Tile<NM>& T, int i, int j, double dt,
                                              double* odm, double* odme, double* odva) {
    const int qn = T.n(i, j);
    const double dvol = AX ? T.fxdv[qn] : T.fydv[qn];
    double dmtot = 0.0;
    double dva[NM] = {}, rfv[NM] = {}, efv[NM] = {};
    bool cfl_ok = true;
    if (DIR && dvol != 0.0 && fabs(dvol) > kCflFrac * d.cv) {  // the Direct face loop's CFL check (remap.cpp:668-671)
        cfl_ok = false;
        const int ia = AX ? i : j, ic = AX ? j : i;
        if (AX ? own_xface(d, i, j) : own_yface(d, i, j))
            raise(d.ctl, ekey(AX ? PH_GRAD_XFACE : PH_GRAD_YFACE, ic, ia, kSubDirectCfl));
    }
    if (dvol != 0.0 && cfl_ok) {
        const int ia = AX ? i : j, ic = AX ? j : i;
        const int ia_d = dvol > 0.0 ? ia - 1 : ia;
        const double sgn = dvol > 0.0 ? 1.0 : -1.0;
        const int cdi = AX ? ia_d : ic, cdj = AX ? ic : ia_d;
        double wlo, whi, blo, bhi;
        if (DIR) {  // face_flux_box (remap.cpp:325-334)
            const double fd = AX ? T.fdx[qn] : T.fdy[qn];
            const double f0pos = AX ? d.x0 + ia * d.dx : d.y0 + ia * d.dy;
            blo = rmin(f0pos, f0pos + fd);
            bhi = rmax(f0pos, f0pos + fd);
            wlo = AX ? d.y0 + ic * d.dy : d.x0 + ic * d.dx;
            whi = AX ? d.y0 + (ic + 1) * d.dy : d.x0 + (ic + 1) * d.dx;
        } else {
            // the flux window [wlo, whi] of cf_face_flux (remap.cpp:29-31, same
            // bits; dvol != 0 implies whi > wlo)
            const int q1 = AX ? T.n(i, j + 1) : T.n(i + 1, j);
            wlo = AX ? d.y0 + j * d.dy + rmax(0.0, dt * T.hy[qn]) : d.x0 + i * d.dx + rmax(0.0, dt * T.hx[qn]);
            whi = AX ? d.y0 + (j + 1) * d.dy + rmin(0.0, dt * T.hy[q1]) : d.x0 + (i + 1) * d.dx + rmin(0.0, dt * T.hx[q1]);
            const double wwin = whi - wlo;
            const double width = dvol / wwin;
            const double f0pos = AX ? d.x0 + ia * d.dx : d.y0 + ia * d.dy;
            blo = rmin(f0pos, f0pos + width);
            bhi = rmax(f0pos, f0pos + width);
        }
        constexpr int RM = DIR ? (AX ? 1 : 2) : 0;
        if (AX)
            split_flux_t<NM, RM>(d, T, cdi, cdj, blo, wlo, bhi, whi, dvol, dva);
        else
            split_flux_t<NM, RM>(d, T, cdi, cdj, wlo, blo, whi, bhi, dvol, dva);
        bool bad = false;
        const int cm = AX ? T.c(ia_d - 1, ic) : T.c(ic, ia_d - 1);
        const int cc = AX ? T.c(ia_d, ic) : T.c(ic, ia_d);
        const int cp = AX ? T.c(ia_d + 1, ic) : T.c(ic, ia_d + 1);
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            if (dva[a] == 0.0) continue;
            int ord = d.face_order;
            if (ord == 2 && NM >= 2 && d.degrade &&
                (T.kk[a][cm] < 1.0 - kPureTol || T.kk[a][cc] < 1.0 - kPureTol || T.kk[a][cp] < 1.0 - kPureTol))
                ord = 1;
            double rf, ef;
            if (ord <= 1) {
                rf = T.rho[a][cc];
                ef = T.el[a][cc];
            } else if (XC && d.corner == CS_MULTID) {  // multid_faces (remap.cpp:840,889-894)
                const double bcx = AX ? 0.5 * (blo + bhi) : 0.5 * (wlo + whi);
                const double bcy = AX ? 0.5 * (wlo + whi) : 0.5 * (blo + bhi);
                const Pair2 r2 = multid_face_tile(d.dgx, d.dgy, T.rho[a], T.el[a], T.xl2x, T.xl2y, T.c(cdi, cdj), bcx, bcy);
                rf = r2.a;
                ef = r2.b;
                if (r2.bad) bad = true;
            } else {
                const int im = AX ? ia_d - 1 : ic, jm = AX ? ic : ia_d - 1;
                const int ic_ = AX ? ia_d : ic, jc = AX ? ic : ia_d;
                const int ip = AX ? ia_d + 1 : ic, jp = AX ? ic : ia_d + 1;
                const double x0 = AX ? T.xlcx(d, im, jm) : T.xlcy(d, im, jm);
                const double x1 = AX ? T.xlcx(d, ic_, jc) : T.xlcy(d, ic_, jc);
                const double x2 = AX ? T.xlcx(d, ip, jp) : T.xlcy(d, ip, jp);
                const double lw = AX ? T.wlx(d, ic_, jc) : T.wly(d, ic_, jc), ufdt = AX ? T.fdx[qn] : T.fdy[qn];
                rf = face_value2(T.rho[a][cm], T.rho[a][cc], T.rho[a][cp], x0, x1, x2, sgn, lw, ufdt, bad);
                ef = face_value2(T.el[a][cm], T.el[a][cc], T.el[a][cp], x0, x1, x2, sgn, lw, ufdt, bad);
            }
            rfv[a] = rf;
            efv[a] = ef;
        }
        if (bad && (AX ? own_xface(d, i, j) : own_yface(d, i, j)))
            raise(d.ctl, ekey(AX ? PH_GRAD_XFACE : PH_GRAD_YFACE, ic, ia, DIR ? kSubDirectGrad : 0));
    }
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        double dm = 0.0, dme = 0.0;
        if (dva[a] != 0.0) {
            dm = rfv[a] * dva[a];
            dme = rfv[a] * efv[a] * dva[a];
            dmtot += dm;
        }
        odm[a] = dm;
        odme[a] = dme;
        odva[a] = dva[a];
    }
    return dmtot;
}

// Corner flux (remap.cpp:923-983) at node (i, j); returns the dmc entry.
template <int NM, bool XC = false>
__device__ __forceinline__ double corner_item_t(const Dev& d, const Tile<NM>& T, int i, int j, double dt,
                                                double* odm, double* odme, double* odva) {
    const int qn = T.n(i, j);
    int sx, sy;
    const double cdv = T.cfv(qn, dt, sx, sy);
    double dva[NM] = {}, rfv[NM] = {}, efv[NM] = {};
    double dmtot = 0.0;
    if (cdv != 0.0) {
        const int di = sx > 0 ? i - 1 : i, dj = sy > 0 ? j - 1 : j;
        const double npx = d.x0 + i * d.dx, npy = d.y0 + j * d.dy;
        const double ddx = dt * T.hx[qn], ddy = dt * T.hy[qn];
        const double blox = rmin(npx, npx + ddx), bloy = rmin(npy, npy + ddy);
        const double bhix = rmax(npx, npx + ddx), bhiy = rmax(npy, npy + ddy);
        split_flux_t<NM>(d, T, di, dj, blox, bloy, bhix, bhiy, cdv, dva);
        const int dc = T.c(di, dj);
        const double lwx = T.wlx(d, di, dj), lwy = T.wly(d, di, dj);
        bool bad = false;
        const bool lin_cfg = d.corner != CS_UPWIND && d.face_order > 1;
        Kin kin;  // remap.cpp:944-956
        kin.dxp = ddx;
        kin.dyp = ddy;
        kin.lwx = lwx;
        kin.lwy = lwy;
        if (XC && lin_cfg && d.corner != CS_LINEARDIAG) {
            const int fxj = sy > 0 ? j - 1 : j, fyi = sx > 0 ? i - 1 : i;
            kin.sfx = T.fxdv[T.n(i, fxj)] >= 0.0 ? 1.0 : -1.0;
            kin.ufx = T.fdx[T.n(i, fxj)];
            kin.sfy = T.fydv[T.n(fyi, j)] >= 0.0 ? 1.0 : -1.0;
            kin.ufy = T.fdy[T.n(fyi, j)];
            kin.erx = 0.5 * (blox + bhix) - T.xl2x[dc];
            kin.ery = 0.5 * (bloy + bhiy) - T.xl2y[dc];
        }
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            if (dva[a] == 0.0) continue;
            bool lin = lin_cfg;
            if (lin && NM >= 2 && d.degrade) {
                for (int q = -1; q <= 1 && lin; ++q)
                    for (int p = -1; p <= 1; ++p)
                        if (T.kk[a][T.c(di + p, dj + q)] < 1.0 - kPureTol) {
                            lin = false;
                            break;
                        }
            }
            double rf, ef;
            if (!lin) {
                rf = T.rho[a][dc];
                ef = T.el[a][dc];
            } else if (XC && d.corner != CS_LINEARDIAG) {
                const Pair2 r2 = corner_other_tile(d.corner, d.dgx, d.dgy, T.rho[a], T.el[a], T.xl2x, T.xl2y, dc, kin);
                rf = r2.a;
                ef = r2.b;
                if (r2.bad) bad = true;
            } else {
                double sr[9], se[9], xlx[9], xly[9];
#pragma unroll
                for (int q = 0; q < 3; ++q)
#pragma unroll
                    for (int p = 0; p < 3; ++p) {
                        const int sidx = T.c(di + p - 1, dj + q - 1);
                        sr[p * 3 + q] = T.rho[a][sidx];
                        se[p * 3 + q] = T.el[a][sidx];
                        xlx[p * 3 + q] = T.xl2x[sidx];
                        xly[p * 3 + q] = T.xl2y[sidx];
                    }
                rf = rmax(corner_diag(d, sr, xlx, xly, ddx, ddy, lwx, lwy, bad), 0.0);
                ef = corner_diag(d, se, xlx, xly, ddx, ddy, lwx, lwy, bad);
            }
            rfv[a] = rf;
            efv[a] = ef;
        }
        if (bad && own_node(d, i, j)) raise(d.ctl, ekey(PH_GRAD_CORNER, j, i, 0));
    }
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        double dm = 0.0, dme = 0.0;
        if (dva[a] != 0.0) {
            dm = rfv[a] * dva[a];
            dme = rfv[a] * efv[a] * dva[a];
            dmtot += dm;
        }
        odm[a] = dm;
        odme[a] = dme;
        odva[a] = dva[a];
    }
    return dmtot;
}

// fill_face_flux_ghosts (remap.cpp:371-382) for dmx / dmy and the dmc ghost
// rows (:985-988).  Every write reads interior entries only.
__device__ __forceinline__ void flux_ghosts_at(const Dev& d, int t) {
    const int nx = d.nx, ny = d.ny;
    // dmx: along = x (na = nx), cross = y (nc = ny); (ia, ic) at (i, j)
    auto dmx_c = [&](int ia, int ic) -> double {  // value incl. cross ghosts
        if (ic == -1) return d.per_y ? d.dmx[ix(d, ia, ny - 1)] : d.dmx[ix(d, ia, 0)];
        if (ic == ny) return d.per_y ? d.dmx[ix(d, ia, 0)] : d.dmx[ix(d, ia, ny - 1)];
        return d.dmx[ix(d, ia, ic)];
    };
    // dmy: along = y (na = ny), cross = x (nc = nx); (ia, ic) at (ic, ia)
    auto dmy_c = [&](int ia, int ic) -> double {
        if (ic == -1) return d.per_x ? d.dmy[ix(d, nx - 1, ia)] : d.dmy[ix(d, 0, ia)];
        if (ic == nx) return d.per_x ? d.dmy[ix(d, 0, ia)] : d.dmy[ix(d, nx - 1, ia)];
        return d.dmy[ix(d, ic, ia)];
    };
    auto dmc_r = [&](int i, int j) -> double {  // dmc incl. the j = -1 ghost row
        if (j == -1) return d.per_y ? d.dmc[ix(d, i, ny - 1)] : d.dmc[ix(d, i, 1)];
        return d.dmc[ix(d, i, j)];
    };
    // only the ghost entries inside this block's window (the global mesh
    // boundary); X-face entries live at (node column, cell row), Y-face
    // entries at (cell column, node row)
    auto wxf = [&](int i, int j) {
        return i >= d.win_n.i0 && i < d.win_n.i1 && j >= d.win_c.j0 && j < d.win_c.j1;
    };
    auto wyf = [&](int i, int j) {
        return i >= d.win_c.i0 && i < d.win_c.i1 && j >= d.win_n.j0 && j < d.win_n.j1;
    };
    if (t <= nx) {  // dmx cross ghosts at ia = t
        if (wxf(t, -1)) d.dmx[ix(d, t, -1)] = dmx_c(t, -1);
        if (wxf(t, ny)) d.dmx[ix(d, t, ny)] = dmx_c(t, ny);
        if (in(d.win_n, t, -1)) d.dmc[ix(d, t, -1)] = dmc_r(t, -1);
    }
    if (t <= ny) {  // dmy cross ghosts at ia = t
        if (wyf(-1, t)) d.dmy[ix(d, -1, t)] = dmy_c(t, -1);
        if (wyf(nx, t)) d.dmy[ix(d, nx, t)] = dmy_c(t, nx);
    }
    if (t <= ny + 1) {  // dmx along ghost (-1, ic), ic in [-1, ny]
        const int ic = t - 1;
        if (wxf(-1, ic)) d.dmx[ix(d, -1, ic)] = d.per_x ? dmx_c(nx - 1, ic) : -dmx_c(1, ic);
        if (in(d.win_n, -1, ic)) d.dmc[ix(d, -1, ic)] = d.per_x ? dmc_r(nx - 1, ic) : dmc_r(1, ic);
    }
    if (t <= nx + 1) {  // dmy along ghost (ia = -1, ic) at (ic, -1), ic in [-1, nx]
        const int ic = t - 1;
        if (wyf(ic, -1)) d.dmy[ix(d, ic, -1)] = d.per_y ? dmy_c(ny - 1, ic) : -dmy_c(1, ic);
    }
}

// Ghost layers of several cell fields (blockIdx.y = 0), node Vec2 fields
// (blockIdx.y = 1) and the face / corner mass-flux ghosts (blockIdx.y = 2) in
// one launch; every write reads interior entries only.
__global__ void k_ghost_multi(Dev d, FieldList cells, FieldList nodes, int flux, int respect_halt) {
    pdl_enter();
    if (respect_halt && halted(d.ctl)) return;
    const int t = blockIdx.x * blockDim.x + threadIdx.x, f = blockIdx.z;
    if (blockIdx.y == 0) {
        if (f < cells.n) ghost_cells_at(d, cells, t, f);
    } else if (blockIdx.y == 1) {
        if (2 * f < nodes.n) ghost_nodes_at(d, nodes, t, 2 * f);
    } else if (flux && f == 0) {
        flux_ghosts_at(d, t);
    }
}

// finalize_cells, per-cell part (remap.cpp:156-191) of cell (i, j) of a
// remap tile: fractions, clipping, snapping, sliver capture, energies
template <int NM>
__device__ __forceinline__ void finalize_cell(const Dev& d, const Rng& rg, int i, int j, int c, int tx, bool own,
                                              double* m, double* me, const double* va,
                                              uint32_t ph_negmass = PH_NEGMASS) {
    double k[2] = {1.0, 0.0};
    uint8_t sl = 0;
    if (NM == 3) {  // the three-material finalize (oracle finalize_cells, nmat == 3)
        int r = -1;  // a material with an exactly zero remapped volume: the two-material rule
        for (int a = NM - 1; a >= 0 && r < 0; --a)
            if (va[a] == 0.0) r = a;
        double kk[3];
        if (r >= 0) {
            const int lo = r == 0 ? 1 : 0, hi = r == 2 ? 1 : 2;
            double k0 = div_cv(d, va[lo]);
            const double k1 = div_cv(d, va[hi]);
            double viol = 0.0;
            const double cand[5] = {-k0, k0 - 1.0, -k1, k1 - 1.0, fabs(k0 + k1 - 1.0)};
#pragma unroll
            for (int q = 0; q < 5; ++q)
                if (viol < cand[q]) viol = cand[q];
            if (viol > 0.0 && own) bump_kviol(d.ctl, viol);
            if (k0 < 0.0 || k0 > 1.0) {
                if (own) bump_clip(d.ctl);
                k0 = (k0 < 0.0) ? 0.0 : ((1.0 < k0) ? 1.0 : k0);
            }
            if (k0 < kPureTol) k0 = 0.0;
            if (k0 > 1.0 - kPureTol) k0 = 1.0;
            kk[lo] = k0;
            kk[hi] = 1.0 - k0;
            kk[r] = 0.0;
        } else {
#pragma unroll
            for (int a = 0; a < 3; ++a) kk[a] = div_cv(d, va[a]);
            double viol = 0.0;
            const double cand[7] = {-kk[0], kk[0] - 1.0, -kk[1], kk[1] - 1.0, -kk[2], kk[2] - 1.0,
                                    fabs(kk[0] + kk[1] + kk[2] - 1.0)};
#pragma unroll
            for (int q = 0; q < 7; ++q)
                if (viol < cand[q]) viol = cand[q];
            if (viol > 0.0 && own) bump_kviol(d.ctl, viol);
            bool clipped = false;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                if (kk[a] < 0.0 || kk[a] > 1.0) {
                    clipped = true;
                    kk[a] = (kk[a] < 0.0) ? 0.0 : ((1.0 < kk[a]) ? 1.0 : kk[a]);
                }
                if (kk[a] < kPureTol) kk[a] = 0.0;
                if (kk[a] > 1.0 - kPureTol) kk[a] = 1.0;
            }
            if (clipped && own) bump_clip(d.ctl);
            kk[2] = (1.0 - kk[0]) - kk[1];
            if (kk[2] < kPureTol) {
                kk[2] = 0.0;
                kk[1] = 1.0 - kk[0];
            }
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if ((kk[a] == 0.0 && m[a] != 0.0) || m[a] < 0.0) {
                sl |= (uint8_t)(1u << a);
                d.slm[a][c] = m[a];
                d.slme[a][c] = me[a];
                m[a] = 0.0;
                me[a] = 0.0;
                if (kk[a] > 0.0) {  // a negative mass with volume left behind
                    const int b = largest_other3(kk, a);
                    if (r >= 0 && a != r)
                        kk[3 - r - a] = 1.0;  // the reference's partner on the pair
                    else
                        kk[b] = kk[b] + kk[a];
                    kk[a] = 0.0;
                }
            }
        }
#pragma unroll
        for (int a = 0; a < 3; ++a) d.nk[a][c] = kk[a];
    } else if (NM == 2) {
        double k0 = div_cv(d, va[0]);
        const double k1 = div_cv(d, va[1]);
        double viol = 0.0;
        const double cand[5] = {-k0, k0 - 1.0, -k1, k1 - 1.0, fabs(k0 + k1 - 1.0)};
#pragma unroll
        for (int q = 0; q < 5; ++q)
            if (viol < cand[q]) viol = cand[q];
        if (viol > 0.0 && own) bump_kviol(d.ctl, viol);
        if (k0 < 0.0 || k0 > 1.0) {
            if (own) bump_clip(d.ctl);
            k0 = (k0 < 0.0) ? 0.0 : ((1.0 < k0) ? 1.0 : k0);
        }
        if (k0 < kPureTol) k0 = 0.0;
        if (k0 > 1.0 - kPureTol) k0 = 1.0;
        k[0] = k0;
        k[1] = 1.0 - k0;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            if ((k[a] == 0.0 && m[a] != 0.0) || m[a] < 0.0) {
                sl |= (uint8_t)(1u << a);
                d.slm[a][c] = m[a];
                d.slme[a][c] = me[a];
                m[a] = 0.0;
                me[a] = 0.0;
                if (k[a] > 0.0) {
                    k[a] = 0.0;
                    k[1 - a] = 1.0;
                }
            }
        }
        d.nk[0][c] = k[0];
        d.nk[1][c] = k[1];
    } else {
        d.nk[0][c] = d.k[0][c];  // one material: w.k = s.k carried unchanged
    }
    double mtot = 0.0;
    int bad_sub = -1;
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        const double ma = m[a];
        if (ma < 0.0 && bad_sub < 0) bad_sub = a;
        d.nm[a][c] = ma;
        d.me[a][c] = me[a];
        d.ne[a][c] = ma > 0.0 ? me[a] / ma : 0.0;
        mtot += ma;
    }
    if (bad_sub < 0 && mtot <= 0.0) bad_sub = kSubCellMass;
    if (bad_sub >= 0 && own) raise(d.ctl, ekey(ph_negmass, j, i, bad_sub));
    d.mcell[c] = mtot;
    if (NM >= 2) {
        d.sliver[c] = sl;
        if (sl) {  // index the sliver for k_slivers (row bit + segment bit)
            const int jr = j - rg.j0, ir = i - rg.i0;
            atomicOr(&d.sl_segs[(size_t)jr * ((rg.i1 - rg.i0 + 31) >> 5) + (ir >> 5)], 1u << (ir & 31));
            atomicOr(&d.sl_rows[jr >> 5], 1u << (jr & 31));
        }
    }
}

// A mapped tile's cell (k_remap_tile MAP): slots 0 / 1 hold materials mat0 <
// mat1 of a context with NC materials; every absent material contributes
// exactly what the NC-material gather gives it -- its m, m * e_lag and k * v,
// no flux -- and the cell is finalised by the NC-material rule (vf: the
// volume its k multiplies, cv on the quiescent path, the Lagrangian volume
// otherwise). (NS, NC) = (2, 3): one material absent from a three-material
// tile; (1, 2): from a two-material tile; (1, 3): a three-material context's
// tile that holds one material only.
template <int NS, int NC>
__device__ __forceinline__ void finalize_mapped(const Dev& d, const Rng& rg, int i, int j, int c, int tx, bool own,
                                                const double* ms, const double* mes, const double* vas, int mat0,
                                                int mat1, double vf) {
    // built with constant indices (selects), so the vectors stay in registers
    double m[NC], me[NC], va[NC];
#pragma unroll
    for (int a = 0; a < NC; ++a) {
        const bool s0 = a == mat0, s1 = NS == 2 && a == mat1;
        double m0 = 0.0, mer = 0.0, var = 0.0;
        if (!s0 && !s1) {  // an absent material: its own planes
            m0 = d.m[a][c];
            mer = m0 * d.el[a][c];
            var = d.k[a][c] * vf;
        }
        m[a] = s0 ? ms[0] : (s1 ? ms[NS - 1] : m0);
        me[a] = s0 ? mes[0] : (s1 ? mes[NS - 1] : mer);
        va[a] = s0 ? vas[0] : (s1 ? vas[NS - 1] : var);
    }
    finalize_cell<NC>(d, rg, i, j, c, tx, own, m, me, va);
}

// plane column of the remap tiles' first region column (rg.i0 - 2) is odd
__host__ __device__ __forceinline__ int tile_shift(const Dev& d) { return (d.r_gath.i0 - G + d.H - d.oi) & 1; }

// TMA (cp.async.bulk.tensor) + mbarrier helpers for the remap tile's staging
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!done);
}

// XC: the AvgMin / LinearXY / Multid corner schemes compiled in (their
// out-of-line calls cost the default kernels registers; see launch_remap_tile)
// DIR: the Direct engine (remap.cpp:593-724): face volumes fd * width, the
// X / Y-displaced interfaces, no corner fluxes (items and dmc zero)
// MAP (NM = 2 only): a three-material context's tile whose staged region
// holds at most two materials (k_tile_class): the two present materials are
// staged into the two slots and the kernel runs the two-material flux code on
// them, which is the three-material code whenever the third material is
// absent from every donor and stencil (k_tile_class checks the per-cell
// conditions); finalize is the three-material one on the expanded vectors.
template <int NM, bool XC = false, bool DIR = false, bool MAP = false>
#ifndef H2D_RT_MAP3
#define H2D_RT_MAP3 1
#endif
// H2D_RT_MAP2: the same per-tile mapping for two materials (one-material
// kernel on single-material tiles); bit-identical but measured slower (C4
// remap 3.70 -> 4.56 ms incl. its classification pass, profiles/
// r02_var_map2_rejected.jsonl), so off
#ifndef H2D_RT_MAP2
#define H2D_RT_MAP2 0
#endif
// H2D_RT_MAP31: a three-material context's tile that holds ONE material runs
// the one-slot kernel (class 4 + p)
#ifndef H2D_RT_MAP31
#define H2D_RT_MAP31 1
#endif
// H2D_RT_MAP32: the two-slot class (one material absent) has its own launch;
// 0: those tiles run the three-slot kernel (one whole-grid launch less)
#ifndef H2D_RT_MAP32
#define H2D_RT_MAP32 1
#endif
#ifndef H2D_RT_SPLITBAR
#define H2D_RT_SPLITBAR 1
#endif
#ifndef H2D_RT_MINB1
#define H2D_RT_MINB1 4
#endif
#ifndef H2D_RT_MINB2
#define H2D_RT_MINB2 3
#endif
#ifndef H2D_RT_MINB3
#define H2D_RT_MINB3 2
#endif
__global__ void __launch_bounds__(RTX * RTY, NM == 1 ? H2D_RT_MINB1 : (NM == 2 ? H2D_RT_MINB2 : H2D_RT_MINB3)) k_remap_tile(Dev d, const __grid_constant__ TmaSet tm) {
    pdl_enter();
    extern __shared__ __align__(128) char smem_raw[];
    __shared__ int s_halt;
    __shared__ __align__(8) uint64_t s_bar, s_bar2;
    const int tid = threadIdx.x;
    // three materials with tile classes: each tile runs in exactly one of the
    // two launches (uniform over the CTA, before any copy is issued)
    // tile class (k_tile_class): 0..2 = that material is absent (two slots of a
    // three-material context, one slot of a two-material one), 3 = the
    // context's own kernel, 4..6 = a three-material context's tile holding
    // only material cls - 4 (one slot); slot a holds material mat(a)
    int rabs = 3;
    if (MAP || (NM >= 2 && !XC && !DIR && d.tcls)) {
        rabs = d.tcls[blockIdx.y * gridDim.x + blockIdx.x];
        if (!MAP) {
            if (rabs != 3) return;
        } else if (NM == 2) {
            if (rabs > 2) return;
        } else {
            if (d.nmat == 3 ? rabs < 4 : rabs > 1) return;
        }
    }
    // NM = 2 slots of a three-material context: the two present materials in
    // order; NM = 1 slot of a two-material context: the present one
    const int mat0 = MAP ? (NM == 2 ? (rabs == 0 ? 1 : 0) : (d.nmat == 3 ? rabs - 4 : 1 - rabs)) : 0,
              mat1 = MAP ? (rabs == 2 ? 1 : 2) : 1;
    auto mat = [&](int a) { return MAP ? (a == 0 ? mat0 : mat1) : a; };
    const int nx = d.nx, ny = d.ny;
    const Rng rg = d.r_gath;
    // TMA wants the box's first column 16-byte aligned (an even plane
    // column): a block whose range starts on an odd column shifts its tile
    // grid one column left (the extra column's items are computed, never
    // gathered, and land outside every range a later phase reads)
    const int sx = tile_shift(d);
    const int i0 = rg.i0 - sx + blockIdx.x * RTX, j0 = rg.j0 + blockIdx.y * RTY;
    // the 128-byte-aligned start of the tile as an OFFSET from the shared array
    // (not a pointer rebuilt from an integer: the compiler then keeps the
    // shared address space and emits LDS / STS with 32-bit addresses instead
    // of generic LD / ST for every tile access)
#ifndef H2D_RT_SMEMPTR
#define H2D_RT_SMEMPTR 1
#endif
#if H2D_RT_SMEMPTR
    char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
#else
    char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
#endif
    const Tile<NM> T = carve_tile<NM, DIR>(smem, i0 - G, j0 - G);
    // ---- phase 0: one thread stages the tile + halo with TMA (2D boxes of
    // the planes, zero-filled past the plane): u_half on the node region,
    // e_lag, m, k on the cell region.  T.rho holds m and T.vl (1 material) /
    // T.kk hold k until phase 2 turns them into densities and volumes.
    // Node values outside the window are never read (every use below is
    // guarded by the window), so whatever the plane holds there is harmless.
    // The copies are issued before the halt flag is read, so the control
    // block's load latency overlaps them (a halted step waits for its copies
    // before the CTA exits: its shared memory must not be handed on while a
    // copy is still writing it).
    // H2D_RT_SPLITBAR: the node planes complete one mbarrier, the cell planes
    // a second, so the quiescent test and phase 1 start before the cell
    // planes have landed
    constexpr bool kSplit = H2D_RT_SPLITBAR != 0;
    uint64_t* bar_c = kSplit ? &s_bar2 : &s_bar;
    if (tid == 0) {
        mbar_init(&s_bar, 1);
        if (kSplit) mbar_init(&s_bar2, 1);
        constexpr uint32_t nbytes = 2u * RNW * RNH * 8u, cbytes = 3u * NM * RCW * RCH * 8u;
        const int x = T.ci0 + d.H - d.oi, y = T.cj0 + d.H - d.oj;  // plane column / row of the region origin
        mbar_expect_tx(&s_bar, kSplit ? nbytes : nbytes + cbytes);
        tma_load_2d(T.hx, &tm.t[TM_UHX], x, y, &s_bar);
        tma_load_2d(T.hy, &tm.t[TM_UHY], x, y, &s_bar);
        if (kSplit) mbar_expect_tx(bar_c, cbytes);
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            tma_load_2d(T.el[a], &tm.t[TM_EL0 + mat(a)], x, y, bar_c);
            tma_load_2d(T.rho[a], &tm.t[TM_M0 + mat(a)], x, y, bar_c);
            tma_load_2d(NM >= 2 ? T.kk[a] : T.vl, &tm.t[TM_K0 + mat(a)], x, y, bar_c);
        }
        s_halt = halted(d.ctl);
    }
    const double dt = step_dt(d.ctl);
    const double cv = d.cv;
    __syncthreads();
    if (s_halt) {
        if (tid == 0) {
            mbar_wait(&s_bar, 0);
            if (kSplit) mbar_wait(bar_c, 0);
        }
        return;
    }
    mbar_wait(&s_bar, 0);
    // ---- quiescent tile: u_half == 0 at every node of the tile's faces and
    // corners makes every face / corner flux volume of the tile zero, so no
    // flux is gathered (the reference skips zero volumes, remap.cpp:860,929),
    // the Lagrangian volume of each own cell is exactly cv (cv + 0 - 0 ...),
    // and the face / corner mass fluxes are +0.0: the per-cell finalize needs
    // only the cell's own inputs (same bits as the full path below)
    {
        int moving = 0;
        RowCol<RTX + 1, RTX * RTY> rq(tid);
        for (int t = tid; t < NCF; t += RTX * RTY, rq.step()) {
            const int ni = i0 + rq.c, nj = j0 + rq.r;
            if (in(d.win_n, ni, nj)) {
                const int q = T.n(ni, nj);
                if (T.hx[q] != 0.0 || T.hy[q] != 0.0) moving = 1;
            }
        }
        if (!__syncthreads_or(moving)) {
            if (kSplit) mbar_wait(bar_c, 0);
            const int ni1 = min(nx, rg.i1), nj1 = min(ny, rg.j1);
            RowCol<RTX + 1, RTX * RTY> rz(tid);
            for (int t = tid; t < NCF; t += RTX * RTY, rz.step()) {
                const int ni = i0 + rz.c, nj = j0 + rz.r;
                const bool lastx = ni < i0 + RTX || ni == ni1, lasty = nj < j0 + RTY || nj == nj1;
                if (ni <= ni1 && nj < nj1 && nj < j0 + RTY && lastx) d.dmx[ix(d, ni, nj)] = 0.0;
                if (ni < ni1 && ni < i0 + RTX && nj <= nj1 && lasty) d.dmy[ix(d, ni, nj)] = 0.0;
                if (ni <= ni1 && nj <= nj1 && lastx && lasty) d.dmc[ix(d, ni, nj)] = 0.0;
            }
            const int tx = tid % RTX, ty = tid / RTX;
            const int i = i0 + tx, j = j0 + ty;
            if (!in(rg, i, j)) return;
            const int c = ix(d, i, j);
            double m[NM], me[NM], va[NM];
            const int tc = T.c(i, j);
#pragma unroll
            for (int a = 0; a < NM; ++a) {
                const double m0 = T.rho[a][tc];
                m[a] = m0;
                me[a] = m0 * T.el[a][tc];
                va[a] = (NM >= 2 ? T.kk[a][tc] : T.vl[tc]) * cv;
            }
            if (MAP && NM == 1 && d.nmat == 3)
                finalize_mapped<NM, 3>(d, rg, i, j, c, tx, own_cell(d, i, j), m, me, va, mat0, mat1, cv);
            else if (MAP)
                finalize_mapped<NM, NM + 1>(d, rg, i, j, c, tx, own_cell(d, i, j), m, me, va, mat0, mat1, cv);
            else
                finalize_cell<NM>(d, rg, i, j, c, tx, own_cell(d, i, j), m, me, va);
            return;
        }
    }
    __syncthreads();
    // ---- phase 1, node items: corner flux, axis geometry, face flux volumes
    // (cf_corner_flux remap.cpp:16-25, make_axis_geom :296-322, :744-767)
    RowCol<RNW, RTX * RTY> rs2(tid);
    for (int t = tid; t < RNN; t += RTX * RTY, rs2.step()) {
        const int i = T.ci0 + rs2.c, j = T.cj0 + rs2.r;
        double fdx = 0.0, fdy = 0.0, fxv = 0.0, fyv = 0.0;
        if (in(d.win_n, i, j)) {
            const double hx = T.hx[t], hy = T.hy[t];
            if (!DIR) {
                const double cfv = fabs((hx * dt) * (hy * dt));
                if (cfv > kCflFrac * cv && own_node(d, i, j)) raise(d.ctl, ekey(PH_CFL_CORNER, j, i, 0));
            }
            // faces on the region's last node row / column feed no region cell
            if (j < ny + G && j < T.cj0 + RNH - 1 && j + 1 < d.win_n.j1) {
                const double ux1 = T.hx[t + RNW], uy1 = T.hy[t + RNW];
                fdx = 0.5 * (hx + ux1) * dt;
                if (DIR) {
                    fxv = fdx * d.dy;  // remap.cpp:663
                } else {
                    double wl, wh;
                    face_flux(d.y0 + j * d.dy, d.y0 + (j + 1) * d.dy, dt * hx, dt * hy, dt * ux1, dt * uy1, fxv, wl,
                              wh);
                    if (fabs(fxv) > kCflFrac * cv && own_xface(d, i, j)) raise(d.ctl, ekey(PH_CFL_XFACE, j, i, 0));
                }
            }
            if (i < nx + G && i < T.ci0 + RNW - 1 && i + 1 < d.win_n.i1) {
                const double ux1 = T.hx[t + 1], uy1 = T.hy[t + 1];
                fdy = 0.5 * (hy + uy1) * dt;
                if (DIR) {
                    fyv = fdy * d.dx;
                } else {
                    double wl, wh;
                    face_flux(d.x0 + i * d.dx, d.x0 + (i + 1) * d.dx, dt * hy, dt * hx, dt * uy1, dt * ux1, fyv, wl,
                              wh);
                    if (fabs(fyv) > kCflFrac * cv && own_yface(d, i, j)) raise(d.ctl, ekey(PH_CFL_YFACE, j, i, 0));
                }
            }
        }
        T.fdx[t] = fdx;
        T.fdy[t] = fdy;
        T.fxdv[t] = fxv;
        T.fydv[t] = fyv;
    }
    __syncthreads();
    if (kSplit) mbar_wait(bar_c, 0);
    // ---- phase 2, cell items: Lagrangian volume, densities, centroids,
    // interfaces (remap.cpp:769-824)
    RowCol<RCW, RTX * RTY> rs3(tid);
    for (int t = tid; t < RNC; t += RTX * RTY, rs3.step()) {
        const int i = T.ci0 + rs3.c, j = T.cj0 + rs3.r;
        if (!in(d.win_c, i, j) || i + 1 >= d.win_n.i1 || j + 1 >= d.win_n.j1) continue;
        const int q00 = T.n(i, j), q10 = q00 + 1, q01 = q00 + RNW, q11 = q01 + 1;
        auto cterm = [&](int q, int ni, int nj) -> double {  // remap.cpp:775-785
            int csx, csy;
            const double dv = T.cfv(q, dt, csx, csy);
            if (dv == 0.0) return 0.0;
            const int di = csx > 0 ? ni - 1 : ni, dj = csy > 0 ? nj - 1 : nj;
            if (di == i && dj == j) return dv;
            const int ri = csx > 0 ? ni : ni - 1, rj = csy > 0 ? nj : nj - 1;
            if (ri == i && rj == j) return -dv;
            return 0.0;
        };
        double v;
        if (DIR) {  // remap.cpp:605-606
            v = cv + (T.fdx[q10] - T.fdx[q00]) * d.dy + (T.fdy[q01] - T.fdy[q00]) * d.dx;
        } else {
            v = cv + T.fxdv[q10] - T.fxdv[q00] + T.fydv[q01] - T.fydv[q00];
            v += cterm(q00, i, j) + cterm(q10, i + 1, j) + cterm(q01, i, j + 1) + cterm(q11, i + 1, j + 1);
        }
        if (v <= 0.0 && own_cell(d, i, j)) raise(d.ctl, ekey(PH_COLLAPSED, j, i, 0));
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            const double ka = NM >= 2 ? T.kk[a][t] : T.vl[t];
            const double ma = T.rho[a][t];
            T.rho[a][t] = ka > 0.0 ? ma / (ka * v) : 0.0;
        }
        T.vl[t] = v;
        const double mdx = 0.25 * (dt * T.hx[q00] + dt * T.hx[q10] + dt * T.hx[q01] + dt * T.hx[q11]);
        const double mdy = 0.25 * (dt * T.hy[q00] + dt * T.hy[q10] + dt * T.hy[q01] + dt * T.hy[q11]);
        T.xl2x[t] = (d.x0 + (i + 0.5) * d.dx) + mdx;
        T.xl2y[t] = (d.y0 + (j + 0.5) * d.dy) + mdy;
        if (NM >= 2) {
            double k0 = T.kk[0][t];
            bool mixed = is_mixed(k0);
            if (NM == 3) {  // the interface of the pair (pair3), fraction of its lower material
                const double k[3] = {T.kk[0][t], T.kk[1][t], T.kk[NM - 1][t]};
                mixed = mixed3(k);
                int lo, hi;
                pair3(k, lo, hi);
                k0 = k[3 - lo - hi] > 0.0 ? k[lo] / (k[lo] + k[hi]) : k[lo];
            }
            double dd = 0.0, dd2 = 0.0;
            if (mixed) {
                const int g = ix(d, i, j);
                double lox, loy, hix, hiy;
                iface_rect<DIR ? 1 : 0>(d, T, i, j, lox, loy, hix, hiy);
                dd = place_interface(k0, d.nrx[g], d.nry[g], lox, loy, hix, hiy);
                if (DIR) {  // the Y-displaced interface of the Direct engine
                    iface_rect<2>(d, T, i, j, lox, loy, hix, hiy);
                    dd2 = place_interface(k0, d.nrx[g], d.nry[g], lox, loy, hix, hiy);
                }
            }
            T.ifd[t] = dd;
            if (DIR) T.ifd2[t] = dd2;
        }
    }
    __syncthreads();
    // ---- flux items, each computed once, in three sub-phases sharing one
    // shared-memory buffer (X faces, Y faces, corners); after each, every
    // cell adds that sub-phase's terms in the reference order (App. C item 3):
    // X face i (+), i+1 (-), Y face j (+), j+1 (-), corners row-major
    const int tx = tid % RTX, ty = tid / RTX;
    const int i = i0 + tx, j = j0 + ty;
    const bool act = in(rg, i, j);
    const int c = act ? ix(d, i, j) : 0;
    const int tc = T.c(i, j);
    double m[NM], me[NM], va[NM];
    if (act) {
        const double vl = T.vl[tc];
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            const double m0 = d.m[mat(a)][c];
            m[a] = m0;
            me[a] = m0 * T.el[a][tc];
            va[a] = (NM >= 2 ? T.kk[a][tc] : d.k[mat(a)][c]) * vl;  // (T.kk: the staged k, unchanged)
        }
    }
    auto add = [&](int a, int q, bool neg) {  // the skip of remap.cpp:860,929
        const double dv = T.it[2][a][q];
        if (dv == 0.0) return;
        if (neg) {
            m[a] += -T.it[0][a][q];
            me[a] += -T.it[1][a][q];
            va[a] += -dv;
        } else {
            m[a] += T.it[0][a][q];
            me[a] += T.it[1][a][q];
            va[a] += dv;
        }
    };
    double dm[NM], dme[NM], dva[NM];
    RowCol<RTX + 1, RTX * RTY> rs4(tid);
    for (int t = tid; t < NXF; t += RTX * RTY, rs4.step()) {  // X faces ia in [i0, i0+RTX], rows [j0, j0+RTY)
        const int ia = i0 + rs4.c, ic = j0 + rs4.r;
#pragma unroll
        for (int a = 0; a < NM; ++a) dva[a] = dm[a] = dme[a] = 0.0;
        if (ia <= min(nx, rg.i1) && ic < min(ny, rg.j1)) {
            const double tot = face_item_t<NM, 1, XC, DIR>(d, T, ia, ic, dt, dm, dme, dva);
            if (ia < i0 + RTX || ia == min(nx, rg.i1)) d.dmx[ix(d, ia, ic)] = tot;
        }
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            T.it[0][a][t] = dm[a];
            T.it[1][a][t] = dme[a];
            T.it[2][a][t] = dva[a];
        }
    }
    __syncthreads();
    if (act) {
        const int xl = tx + ty * (RTX + 1);
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            add(a, xl, false);
            add(a, xl + 1, true);
        }
    }
    __syncthreads();
    for (int t = tid; t < NYF; t += RTX * RTY) {  // Y faces: columns [i0, i0+RTX), ja in [j0, j0+RTY]
        const int ic = i0 + t % RTX, ja = j0 + t / RTX;
#pragma unroll
        for (int a = 0; a < NM; ++a) dva[a] = dm[a] = dme[a] = 0.0;
        if (ic < min(nx, rg.i1) && ja <= min(ny, rg.j1)) {
            const double tot = face_item_t<NM, 0, XC, DIR>(d, T, ic, ja, dt, dm, dme, dva);
            if (ja < j0 + RTY || ja == min(ny, rg.j1)) d.dmy[ix(d, ic, ja)] = tot;
        }
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            T.it[0][a][t] = dm[a];
            T.it[1][a][t] = dme[a];
            T.it[2][a][t] = dva[a];
        }
    }
    __syncthreads();
    if (act) {
        const int yb = tx + ty * RTX;
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            add(a, yb, false);
            add(a, yb + RTX, true);
        }
    }
    __syncthreads();
    RowCol<RTX + 1, RTX * RTY> rs5(tid);
    for (int t = tid; t < NCF; t += RTX * RTY, rs5.step()) {  // corner nodes [i0, i0+RTX] x [j0, j0+RTY]
        const int ni = i0 + rs5.c, nj = j0 + rs5.r;
#pragma unroll
        for (int a = 0; a < NM; ++a) dva[a] = dm[a] = dme[a] = 0.0;
        const int ni1 = min(nx, rg.i1), nj1 = min(ny, rg.j1);
        if (ni <= ni1 && nj <= nj1) {
            const double tot = DIR ? 0.0 : corner_item_t<NM, XC>(d, T, ni, nj, dt, dm, dme, dva);
            if ((ni < i0 + RTX || ni == ni1) && (nj < j0 + RTY || nj == nj1)) d.dmc[ix(d, ni, nj)] = tot;
        }
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            T.it[0][a][t] = dm[a];
            T.it[1][a][t] = dme[a];
            T.it[2][a][t] = dva[a];
        }
    }
    __syncthreads();
    if (!act) return;
    const bool own = own_cell(d, i, j);
    if (!DIR) {  // (the Direct engine has no corner fluxes)
        const int cq[4] = {tx + ty * (RTX + 1), tx + 1 + ty * (RTX + 1), tx + (ty + 1) * (RTX + 1),
                           tx + 1 + (ty + 1) * (RTX + 1)};
        const int ndi[4] = {i, i + 1, i, i + 1}, ndj[4] = {j, j, j + 1, j + 1};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int csx, csy;
            const double cd = T.cfv(T.n(ndi[q], ndj[q]), dt, csx, csy);
            if (cd == 0.0) continue;  // no corner flux at this node (its items are all zero)
            const int di = csx > 0 ? ndi[q] - 1 : ndi[q], dj = csy > 0 ? ndj[q] - 1 : ndj[q];
            const int ri = csx > 0 ? ndi[q] : ndi[q] - 1, rj = csy > 0 ? ndj[q] : ndj[q] - 1;
            const bool donor = di == i && dj == j;
            if (!donor && !(ri == i && rj == j)) continue;
#pragma unroll
            for (int a = 0; a < NM; ++a) add(a, cq[q], donor);
        }
    }
    if (MAP && NM == 1 && d.nmat == 3)
        finalize_mapped<NM, 3>(d, rg, i, j, c, tx, own, m, me, va, mat0, mat1, T.vl[tc]);
    else if (MAP)
        finalize_mapped<NM, NM + 1>(d, rg, i, j, c, tx, own, m, me, va, mat0, mat1, T.vl[tc]);
    else
        finalize_cell<NM>(d, rg, i, j, c, tx, own, m, me, va);
}


__device__ __forceinline__ void sliver_offset(int lane, int& di, int& dj, int& ring) {
    if (lane < 8) {  // ring 1: (dj, di) row-major, centre skipped
        const int q = lane < 4 ? lane : lane + 1;
        dj = q / 3 - 1;
        di = q % 3 - 1;
        ring = 1;
    } else {  // ring 2: dj = -2 (5), dj = -1..1 (di = -2, 2), dj = 2 (5)
        const int q = lane - 8;
        ring = 2;
        if (q < 5) {
            dj = -2;
            di = q - 2;
        } else if (q < 11) {
            dj = (q - 5) / 2 - 1;
            di = ((q - 5) & 1) ? 2 : -2;
        } else {
            dj = 2;
            di = q - 13;
        }
    }
}

// Sequential sliver redistribution (remap.cpp:194-226) in the reference's
// row-major `pending` order. The tile kernel marks each sliver in a row bitmap
// and a 32-cell segment bitmap (finalize_cell); this kernel (one block of
// SLB threads) first lists the slivers of a chunk of rows in order, all warps
// in parallel (rows compacted, per-row counts scanned, positions written),
// then one warp applies them one after another:
//  * each sliver's 24 ring candidates are loaded by 24 lanes and reduced to
//    the FIRST maximum of k (the strict `>` scan = lowest lane among equal
//    maxima, ring 1 before ring 2);
//  * the candidates of the next SLD slivers are loaded ahead; every applied
//    sliver broadcasts the cell and values it wrote and the pending records
//    patch the copies they hold, so each record always sees the values the
//    reference's loop would (exact), and the chain of dependent slivers runs
//    at shuffle speed instead of one memory round trip per sliver.
constexpr int SLB = 256, SLROWS = 4096, SLD = 4;

template <int NM>
struct SliverRec {
    int sc, fl, nc, own;       // cell, flags, this lane's candidate cell, own-cell flag
    double sm[NM], sme[NM];    // sliver masses (remap.cpp:172)
    double mv[NM], kv[NM], mev[NM], mcv;  // candidate m, k, me per material, mcell
    int part[NM];              // the orphan's partner material (remap.cpp:217-225; 3 materials: largest other k)
};

template <int NM>
__device__ __forceinline__ void sliver_load(const Dev& d, const Rng& rg, int v, int lane, int di, int dj,
                                            SliverRec<NM>& r) {
    const int W = rg.i1 - rg.i0;  // v = (j - rg.j0) * W + (i - rg.i0)
    const int sj = rg.j0 + v / W, si = rg.i0 + v % W;
    const int c = ix(d, si, sj);
    r.sc = c;
    r.own = own_cell(d, si, sj);
    int ni = si + di, nj = sj + dj;
    if (d.per_x) ni = (ni + 2 * d.nx) % d.nx;
    if (d.per_y) nj = (nj + 2 * d.ny) % d.ny;
    const bool inb = lane < 24 && ni >= 0 && ni < d.nx && nj >= 0 && nj < d.ny && in(rg, ni, nj);
    r.nc = inb ? ix(d, ni, nj) : -1;
    r.fl = d.sliver[c];
    r.mcv = 0.0;
    if (NM == 3) {
        const double k3[3] = {d.nk[0][c], d.nk[1][c], d.nk[NM - 1][c]};
#pragma unroll
        for (int a = 0; a < NM; ++a) r.part[a] = largest_other3(k3, a);
    } else {
#pragma unroll
        for (int a = 0; a < NM; ++a) r.part[a] = 1 - a;
    }
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        r.sm[a] = d.slm[a][c];
        r.sme[a] = d.slme[a][c];
        r.mv[a] = 0.0;
        r.kv[a] = -1.0;
        r.mev[a] = 0.0;
        if (inb) {
            r.mv[a] = d.nm[a][r.nc];
            r.kv[a] = d.nk[a][r.nc];
            r.mev[a] = d.me[a][r.nc];
        }
    }
    if (inb) r.mcv = d.mcell[r.nc];
}

// a write of (m, me of material a, mcell) to cell w, seen by a pending record
template <int NM>
__device__ __forceinline__ void sliver_patch(SliverRec<NM>& r, int w, int a, double nm, double nme, double nmc) {
    if (r.nc == w) {
#pragma unroll
        for (int b = 0; b < NM; ++b)
            if (b == a) {
                r.mv[b] = nm;
                r.mev[b] = nme;
            }
        r.mcv = nmc;
    }
}

// Apply one pending record (both of its materials, a = 0 first as the
// reference pushes them, remap.cpp:170-181); returns nothing, patches `p1..p3`.
template <int NM>
__device__ __forceinline__ void sliver_apply_rec(const Dev& d, SliverRec<NM>& r, int lane, int ring,
                                                 SliverRec<NM>& p1, SliverRec<NM>& p2, SliverRec<NM>& p3) {
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        if (!(r.fl & (1 << a))) continue;
        const double mv = r.mv[a], kv = r.kv[a];
        const double mev = r.mev[a];
        const double smv = r.sm[a], smev = r.sme[a];
        const bool cand = kv > -1.0 && !(mv <= 0.0);  // the reference skips m <= 0, then needs k > bk
        int br = cand ? ring : 4, bl = lane;
        double bkv = kv;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const int orr = __shfl_xor_sync(0xffffffffu, br, o);
            const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
            const double ok = __shfl_xor_sync(0xffffffffu, bkv, o);
            const bool take = orr < br || (orr == br && br < 4 && (ok > bkv || (ok == bkv && ol < bl)));
            if (take) {
                br = orr;
                bl = ol;
                bkv = ok;
            }
        }
        const bool found = br < 4;
        const double mcar = __shfl_sync(0xffffffffu, mv, found ? bl : 0);
        int w, wa, src;
        double nm = 0.0, nme = 0.0, nmc = 0.0;
        if (found && mcar + smv > 0.0) {  // the carrier takes the sliver (remap.cpp:212-216)
            w = __shfl_sync(0xffffffffu, r.nc, bl);
            wa = a;
            src = bl;
            if (lane == bl) {
                nm = mv + smv;
                nme = mev + smev;
                nmc = r.mcv + smv;
                d.nm[a][w] = nm;
                d.me[a][w] = nme;
                d.ne[a][w] = nme / nm;
                d.mcell[w] = nmc;
            }
        } else {  // no carrier: the partner material at the sliver's own cell (:217-225)
            w = r.sc;
            wa = r.part[a];
            src = 0;
            if (lane == 0) {  // rare: fresh loads (memory is current after the __syncwarp)
                if (r.own) d.ctl->step_fix += 1;
                nm = d.nm[wa][w] + smv;
                nme = d.me[wa][w] + smev;
                nmc = d.mcell[w] + smv;
                d.nm[wa][w] = nm;
                d.me[wa][w] = nme;
                d.ne[wa][w] = nme / nm;
                d.mcell[w] = nmc;
            }
        }
        nm = __shfl_sync(0xffffffffu, nm, src);
        nme = __shfl_sync(0xffffffffu, nme, src);
        nmc = __shfl_sync(0xffffffffu, nmc, src);
        sliver_patch(r, w, wa, nm, nme, nmc);  // this cell's second material sees the first
        sliver_patch(p1, w, wa, nm, nme, nmc);
        sliver_patch(p2, w, wa, nm, nme, nmc);
        sliver_patch(p3, w, wa, nm, nme, nmc);
        __syncwarp();
    }
}

// block-wide exclusive scan of one int per thread (SLB threads); returns the total
__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int t = lane < SLB / 32 ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        s_warp[32 + lane] = t;  // inclusive warp prefixes
    }
    __syncthreads();
    total = s_warp[32 + SLB / 32 - 1];
    const int base = wid ? s_warp[32 + wid - 1] : 0;
    const int r = base + x - v;
    __syncthreads();
    return r;
}

// The sliver redistribution runs in three steps (launch_remap_slivers):
//  1. k_sliver_list (one block): the pending slivers in the reference's
//     row-major order, listed from the row / segment bitmaps finalize_cell
//     set (rows compacted, per-row counts scanned, positions written); the
//     segment bitmap stays set: it is the pending set P_0 of step 2.
//  2. k_sliver_round r = 0 .. kSlRounds-1 (whole GPU): a sliver reads and
//     writes only cells within Chebyshev distance 2 of its own cell (its two
//     candidate rings, remap.cpp:200-216, or the cell itself, :217-225), so
//     two slivers further than 4 apart never touch a common cell. A pending
//     sliver with no EARLIER pending sliver within distance 4 (the bitmap P_r
//     of the slivers still pending) sees exactly the values the reference's
//     sequential loop would show it -- every earlier sliver that could change
//     them is applied, no later one has run -- so all such slivers of a round
//     are applied at once, one thread each (they are pairwise more than 4
//     apart: of two closer ones the later is blocked by the earlier). P_{r+1}
//     is the same set minus the round's slivers, kept in the other bitmap.
//     Rounds stop when a round applies fewer than kSlMinProgress (a chain of
//     dependent slivers: one per round).
//  3. k_sliver_tail (one block): the slivers still pending, in order, are
//     applied by one warp with the pipelined record path below (exact for a
//     chain), and the bitmaps are cleared.
// Periodic meshes (conflicts wrap around) and lists longer than a quarter of
// the list capacity skip step 2.
#ifndef H2D_SL_ROUNDS
#define H2D_SL_ROUNDS 8
#endif
constexpr int kSlRounds = H2D_SL_ROUNDS, kSlMinProgress = 32, kSlGrid = 148;
static_assert(kSlRounds <= 8, "Ctl::sl_cnt holds 8 rounds");

template <int NM>
__device__ __forceinline__ void sliver_chunk_list(const Dev& d, const Rng& rg, int* s_rows, int* s_off, int* s_warp,
                                                  int r0, int base, int& total) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nrow = rg.j1 - rg.j0, nwx = (rg.i1 - rg.i0 + 31) >> 5;
    constexpr int NRW = SLROWS / 32;
    unsigned rb = 0u;
    const int rw = (r0 >> 5) + tid;
    if (tid < NRW && (r0 + 32 * tid) < nrow) {
        rb = d.sl_rows[rw];
        if (rb) d.sl_rows[rw] = 0u;
    }
    int nrows;
    const int rpos = block_excl_scan(__popc(rb), s_warp, nrows);
    for (unsigned b = rb, q = rpos; b; b &= b - 1, ++q) s_rows[q] = r0 + 32 * tid + __ffs(b) - 1;
    __syncthreads();
    total = 0;
    if (nrows == 0) return;
    // slivers per row (one warp per row), scanned into offsets
    for (int k = wid; k < nrows; k += SLB / 32) {
        const unsigned* seg = d.sl_segs + (size_t)s_rows[k] * nwx;
        int cnt = 0;
        for (int w = lane; w < nwx; w += 32) cnt += __popc(seg[w]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0) s_off[k] = cnt;
    }
    __syncthreads();
    {
        int run = 0;  // SLROWS / SLB rows per thread, scanned by blocks of consecutive rows
        constexpr int PER = SLROWS / SLB;
        int loc[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int k = tid * PER + q;
            loc[q] = k < nrows ? s_off[k] : 0;
            run += loc[q];
        }
        int tot;
        int off = block_excl_scan(run, s_warp, tot);
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int k = tid * PER + q;
            if (k < nrows) s_off[k] = base + off;
            off += loc[q];
        }
        total = tot;
    }
    __syncthreads();
    // positions, row-major (words in order, bits in order)
    for (int k = wid; k < nrows; k += SLB / 32) {
        const int jr = s_rows[k];
        const unsigned* seg = d.sl_segs + (size_t)jr * nwx;
        int pb = s_off[k];
        for (int w0 = 0; w0 < nwx; w0 += 32) {
            const int w = w0 + lane;
            unsigned bits = w < nwx ? seg[w] : 0u;
            const int c = __popc(bits);
            int x = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            int p = pb + x - c;
            for (; bits; bits &= bits - 1, ++p) {
                H2D_CHECK(p < d.sl_cap);
                d.sl_list[p] = jr * (rg.i1 - rg.i0) + (w << 5) + __ffs(bits) - 1;
            }
            pb += __shfl_sync(0xffffffffu, x, 31);
        }
    }
    __syncthreads();
}

template <int NM>
__global__ void __launch_bounds__(SLB, 1) k_sliver_list(Dev d) {
    pdl_enter();
    __shared__ int s_halt;
    __shared__ int s_rows[SLROWS], s_off[SLROWS];
    __shared__ int s_warp[64];
    if (threadIdx.x == 0) s_halt = halted(d.ctl);
    __syncthreads();
    if (s_halt) return;
    const Rng rg = d.r_gath;
    const int nrow = rg.j1 - rg.j0;
    int n = 0;
    for (int r0 = 0; r0 < nrow; r0 += SLROWS) {
        int t;
        sliver_chunk_list<NM>(d, rg, s_rows, s_off, s_warp, r0, n, t);
        n += t;
    }
    if (threadIdx.x == 0) {
        Ctl* c = d.ctl;
        c->sl_n = n;
        c->sl_on = !(d.per_x || d.per_y || n > d.sl_cap / 4);
        for (int q = 0; q < kSlRounds; ++q) c->sl_cnt[q] = 0;
    }
}

__device__ __forceinline__ uint8_t* sl_status(const Dev& d) {
    return reinterpret_cast<uint8_t*>(d.sl_list + d.sl_cap / 2);
}
__device__ __forceinline__ int* sl_tail(const Dev& d) { return d.sl_list + d.sl_cap / 4; }
__device__ __forceinline__ unsigned* sl_bits(const Dev& d, int r) { return (r & 1) ? d.sl_segs2 : d.sl_segs; }

// any pending sliver EARLIER than (jr, ir) in row-major order within
// Chebyshev distance 4 (rows jr-4 .. jr-1: columns ir-4 .. ir+4; row jr:
// ir-4 .. ir-1), in the bitmap P
__device__ __forceinline__ bool sl_blocked(const unsigned* P, int nwx, int W, int jr, int ir) {
    // the window spans at most two words per row: all ten loads issue together
    const int c0 = ir - 4 < 0 ? 0 : ir - 4, c1u = ir + 4 < W - 1 ? ir + 4 : W - 1;
    const int w0 = c0 >> 5;
    unsigned acc = 0u;
#pragma unroll
    for (int dq = 4; dq >= 0; --dq) {
        const int q = jr - dq;
        const int c1 = dq ? c1u : ir - 1;
        if (q < 0 || c1 < c0) continue;
        const int w1 = c1 >> 5;
        const unsigned lo = c0 & 31;
        const unsigned hi0 = w1 == w0 ? (c1 & 31) : 31;
        acc |= __ldcg(P + (size_t)q * nwx + w0) & (0xffffffffu >> (31 - hi0)) & (0xffffffffu << lo);
        if (w1 != w0) acc |= __ldcg(P + (size_t)q * nwx + w1) & (0xffffffffu >> (31 - (c1 & 31)));
    }
    return acc != 0u;
}

// candidates L0 .. L1-1 of a sliver at (si, sj) for material a: all loads
// issued together, then the first strict maximum of k among m > 0
template <int L0, int L1>
__device__ __forceinline__ void sliver_scan(const Dev& d, const Rng& rg, int a, int si, int sj, int& best, double& bk,
                                            double& bm) {
    double mv[L1 - L0], kv[L1 - L0];
    int nc[L1 - L0];
#pragma unroll
    for (int q = 0; q < L1 - L0; ++q) {
        int di, dj, ring;
        sliver_offset(L0 + q, di, dj, ring);
        const int ni = si + di, nj = sj + dj;
        const bool ok = ni >= 0 && ni < d.nx && nj >= 0 && nj < d.ny && in(rg, ni, nj);
        nc[q] = ok ? ix(d, ni, nj) : -1;
        mv[q] = ok ? d.nm[a][nc[q]] : 0.0;
        kv[q] = ok ? d.nk[a][nc[q]] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < L1 - L0; ++q)
        if (nc[q] >= 0 && !(mv[q] <= 0.0) && (best < 0 || kv[q] > bk)) {
            best = nc[q];
            bk = kv[q];
            bm = mv[q];
        }
}

// One pending record (cell v of the list, every flagged material, a = 0
// first as the reference pushes them, remap.cpp:170-181) applied by ONE
// thread: the candidate scan of remap.cpp:200-216 (ring 1 before ring 2,
// row-major inside a ring, first strict maximum of k among m > 0), the
// carrier update, else the partner material at the sliver's own cell.
template <int NM>
__device__ __forceinline__ void sliver_apply_thread(const Dev& d, const Rng& rg, int v) {
    const int W = rg.i1 - rg.i0;
    const int sj = rg.j0 + v / W, si = rg.i0 + v % W;
    const int c = ix(d, si, sj);
    const int fl = d.sliver[c];
    const bool own = own_cell(d, si, sj);
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        if (!(fl & (1 << a))) continue;
        const double smv = d.slm[a][c], smev = d.slme[a][c];
        // ring 1 (8 candidates), then ring 2 (16) only if ring 1 had none:
        // each ring's loads are issued together (no dependent chain)
        int best = -1;
        double bk = 0.0, bm = 0.0;
        sliver_scan<0, 8>(d, rg, a, si, sj, best, bk, bm);
        if (best < 0) sliver_scan<8, 24>(d, rg, a, si, sj, best, bk, bm);
        if (best >= 0 && bm + smv > 0.0) {  // the carrier takes the sliver (remap.cpp:212-216)
            const double nm = bm + smv, nme = d.me[a][best] + smev;
            d.nm[a][best] = nm;
            d.me[a][best] = nme;
            d.ne[a][best] = nme / nm;
            d.mcell[best] = d.mcell[best] + smv;
        } else {  // no carrier: the partner material at the sliver's own cell (:217-225)
            int pa = 1 - a;
            if (NM == 3) {
                const double k3[3] = {d.nk[0][c], d.nk[1][c], d.nk[NM - 1][c]};
                pa = largest_other3(k3, a);
            }
            if (own) atomicAdd(&d.ctl->step_fix, 1);
            const double nm = d.nm[pa][c] + smv, nme = d.me[pa][c] + smev;
            d.nm[pa][c] = nm;
            d.me[pa][c] = nme;
            d.ne[pa][c] = nme / nm;
            d.mcell[c] = d.mcell[c] + smv;
        }
    }
}

// round r runs when the rounds are on and every earlier round applied at
// least kSlMinProgress slivers (a round that did not run counted none)
__device__ __forceinline__ bool sl_round_runs(const Ctl* c, int r) {
    return __ldcg(&c->sl_on) && (r == 0 || __ldcg(&c->sl_cnt[r - 1]) >= kSlMinProgress);
}

template <int NM>
__global__ void __launch_bounds__(256) k_sliver_round(Dev d, int r) {
    pdl_enter();
    const Ctl* cc = d.ctl;
    if (halted(cc)) return;
    const int n = __ldcg(&cc->sl_n);
    if (!sl_round_runs(cc, r) || n == 0) return;
    const Rng rg = d.r_gath;
    const int W = rg.i1 - rg.i0, nwx = (W + 31) >> 5;
    const unsigned* P = sl_bits(d, r);
    unsigned* Q = sl_bits(d, r + 1);  // P_{r-1} -> P_{r+1}
    uint8_t* st = sl_status(d);
    int applied = 0;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int v = d.sl_list[k];
        const int jr = v / W, ir = v % W;
        unsigned* qw = Q + (size_t)jr * nwx + (ir >> 5);
        const unsigned bit = 1u << (ir & 31);
        const int s = r == 0 ? 0xff : st[k];
        if (s != 0xff) {
            if (s == r - 1) atomicAnd(qw, ~bit);  // applied last round: leaves P_{r+1}
            continue;
        }
        if (sl_blocked(P, nwx, W, jr, ir)) {
            st[k] = 0xff;
            if (r == 0) atomicOr(qw, bit);  // pending into P_1
            continue;
        }
        sliver_apply_thread<NM>(d, rg, v);
        st[k] = (uint8_t)r;
        if (r > 0) atomicAnd(qw, ~bit);
        ++applied;
    }
    const int tot = __reduce_add_sync(0xffffffffu, applied);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(&d.ctl->sl_cnt[r], tot);
}

template <int NM>
__global__ void __launch_bounds__(SLB, 1) k_sliver_tail(Dev d) {
    pdl_enter();
    __shared__ int s_halt, s_n;
    __shared__ int s_warp[64];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) s_halt = halted(d.ctl);
    __syncthreads();
    if (s_halt) return;
    const Rng rg = d.r_gath;
    const int W = rg.i1 - rg.i0, nwx = (W + 31) >> 5;
    const int n = d.ctl->sl_n;
    int last = -1;  // the last round that ran
    while (last + 1 < kSlRounds && sl_round_runs(d.ctl, last + 1)) ++last;
    const bool rounds = last >= 0;
    const uint8_t* st = sl_status(d);
    // the pending records, in order, and the bitmaps cleared: P_last holds the
    // records pending at round `last`, P_{last+1} those pending after it
    const int* list = d.sl_list;
    int np = n;
    if (rounds) {
        int* tl = sl_tail(d);
        const int per = (n + SLB - 1) / SLB, k0 = tid * per, k1 = min(n, k0 + per);
        int cnt = 0;
        for (int k = k0; k < k1; ++k) cnt += st[k] == 0xff;
        int tot;
        int pos = block_excl_scan(cnt, s_warp, tot);
        unsigned* Pa = sl_bits(d, last);
        unsigned* Pb = sl_bits(d, last + 1);
        for (int k = k0; k < k1; ++k) {
            const int s = st[k];
            if (s != 0xff && s != last) continue;
            const int v = d.sl_list[k];
            const int jr = v / W, ir = v % W;
            const size_t wq = (size_t)jr * nwx + (ir >> 5);
            const unsigned bit = 1u << (ir & 31);
            atomicAnd(Pa + wq, ~bit);
            if (s == 0xff) {
                atomicAnd(Pb + wq, ~bit);
                tl[pos++] = v;
            }
        }
        if (tid == 0) s_n = tot;
        __syncthreads();
        np = s_n;
        list = tl;
    } else {
        for (int k = tid; k < n; k += SLB) {
            const int v = d.sl_list[k];
            const int jr = v / W, ir = v % W;
            atomicAnd(d.sl_segs + (size_t)jr * nwx + (ir >> 5), ~(1u << (ir & 31)));
        }
    }
    __syncthreads();
    // one warp applies the remaining records in order, SLD records in flight
    if (wid == 0 && np > 0) {
        int di = 0, dj = 0, ring = 3;
        if (lane < 24) sliver_offset(lane, di, dj, ring);
        SliverRec<NM> r0v, r1v, r2v, r3v;
        if (0 < np) sliver_load(d, rg, list[0], lane, di, dj, r0v);
        if (1 < np) sliver_load(d, rg, list[1], lane, di, dj, r1v);
        if (2 < np) sliver_load(d, rg, list[2], lane, di, dj, r2v);
        if (3 < np) sliver_load(d, rg, list[3], lane, di, dj, r3v);
        for (int k = 0; k < np; k += SLD) {
            sliver_apply_rec(d, r0v, lane, ring, r1v, r2v, r3v);
            if (k + 4 < np) sliver_load(d, rg, list[k + 4], lane, di, dj, r0v);
            if (k + 1 >= np) break;
            sliver_apply_rec(d, r1v, lane, ring, r2v, r3v, r0v);
            if (k + 5 < np) sliver_load(d, rg, list[k + 5], lane, di, dj, r1v);
            if (k + 2 >= np) break;
            sliver_apply_rec(d, r2v, lane, ring, r3v, r0v, r1v);
            if (k + 6 < np) sliver_load(d, rg, list[k + 6], lane, di, dj, r2v);
            if (k + 3 >= np) break;
            sliver_apply_rec(d, r3v, lane, ring, r0v, r1v, r2v);
            if (k + 7 < np) sliver_load(d, rg, list[k + 7], lane, di, dj, r3v);
        }
    }
}

// dual_face_value, remap.cpp:384-404 for node velocities w.u (= u_lag)
__device__ __forceinline__ double dual_face_value(const Dev& d, const double* u, int ax, int ia_d, int ic, double dt,
                                                  double wa, double sgn, double ufdt, bool& bad) {
    auto at = [&](int ia) { return ax ? ix(d, ia, ic) : ix(d, ic, ia); };
    if (d.face_order <= 1) return u[at(ia_d)];
    const double* uh = ax ? d.uhx : d.uhy;
    const double nm1 = uh[at(ia_d - 1)] * dt, n0 = uh[at(ia_d)] * dt, np1 = uh[at(ia_d + 1)] * dt;
    const double x0 = (ia_d - 1) * wa + nm1, x1 = ia_d * wa + n0, x2 = (ia_d + 1) * wa + np1;
    const double dfl = 0.5 * (nm1 + n0), dfr = 0.5 * (n0 + np1);
    return face_value2(u[at(ia_d - 1)], u[at(ia_d)], u[at(ia_d + 1)], x0, x1, x2, sgn, wa + (dfr - dfl), ufdt, bad);
}

// dual_face_pass, remap.cpp:408-442: one thread per dual face. AX = 1: X
// (ia = i node, ic = j), AX = 0: Y (ia = j, ic = i); stored at (i, j).
template <int AX>
__device__ __forceinline__ bool dual_face_val(const Dev& d, int i, int j, double& mx, double& my,
                                              uint32_t ph = AX ? PH_GRAD_DUALX : PH_GRAD_DUALY) {
    const int ia = AX ? i : j, ic = AX ? j : i;
    const int per_a = AX ? d.per_x : d.per_y;
    const int s = ix(d, i, j);
    mx = 0.0;
    my = 0.0;
    if (ia < (per_a ? 0 : 1)) return false;
    const double* dmf = AX ? d.dmx : d.dmy;
    auto F = [&](int a, int c) { return dmf[AX ? ix(d, a, c) : ix(d, c, a)]; };
    const double dm = 0.25 * ((F(ia - 1, ic - 1) + F(ia - 1, ic)) + (F(ia, ic - 1) + F(ia, ic)));
    if (dm != 0.0) {
        const double dt = step_dt(d.ctl);
        const int ia_d = dm > 0.0 ? ia - 1 : ia;
        const double sgn = dm > 0.0 ? 1.0 : -1.0;
        const double* uh = AX ? d.uhx : d.uhy;
        const double ufdt = 0.5 * (uh[AX ? ix(d, ia - 1, ic) : ix(d, ic, ia - 1)] * dt + uh[s] * dt);
        const double wa = AX ? d.dx : d.dy;
        bool bad = false;
        const double ufx = dual_face_value(d, d.ulx, AX, ia_d, ic, dt, wa, sgn, ufdt, bad);
        const double ufy = dual_face_value(d, d.uly, AX, ia_d, ic, dt, wa, sgn, ufdt, bad);
        if (bad && own_node(d, i, j)) raise(d.ctl, ekey(ph, ic, ia, 0));
        mx = ufx * dm;
        my = ufy * dm;
    }
    return dm != 0.0;  // a zero dual mass flux is skipped (remap.cpp:423)
}
template <int AX>
__device__ __forceinline__ void dual_face_item(const Dev& d, int i, int j) {
    double mx, my;
    const bool on = dual_face_val<AX>(d, i, j, mx, my);
    const int s = ix(d, i, j);
    (AX ? d.dfx_x : d.dfy_x)[s] = mx;
    (AX ? d.dfx_y : d.dfy_y)[s] = my;
    if (d.per_x || d.per_y) d.dflag[AX ? 0 : 1][s] = on;  // only the periodic gather reads flags
}

// Dual-mesh corner exchanges, remap.cpp:1000-1069: iteration (i, j), both
// pairs (1,1) and (1,-1).
// the dual corner velocity for the AvgMin / LinearXY / Multid schemes on
// the 3x3 node stencil around node (wi, wj) (plane index g), out of line
// (see corner_other_tile); stencil positions node_pos + dt u_half as inline
__device__ __noinline__ Pair2 dual_corner_other(int scheme, double dgx, double dgy, const double* ulx,
                                                const double* uly, const double* uhx, const double* uhy, int g, int P,
                                                int wi, int wj, double x0, double y0, double dx, double dy, double dt,
                                                Kin k) {
    double ax_[9], ay_[9], xlx[9], xly[9];
    for (int q = 0; q < 3; ++q)
        for (int p = 0; p < 3; ++p) {
            const int ni = wi + p - 1, nj = wj + q - 1;
            const int nn = g + (p - 1) + (q - 1) * P;
            ax_[p * 3 + q] = ulx[nn];
            ay_[p * 3 + q] = uly[nn];
            xlx[p * 3 + q] = (x0 + ni * dx) + dt * uhx[nn];
            xly[p * 3 + q] = (y0 + nj * dy) + dt * uhy[nn];
        }
    bool bad = false;
    Pair2 r;
    r.a = corner_value_other(scheme, dgx, dgy, ax_, xlx, xly, k, &bad);
    r.b = corner_value_other(scheme, dgx, dgy, ay_, xlx, xly, k, &bad);
    r.bad = bad;
    return r;
}

template <bool XC>
__device__ __forceinline__ bool dual_corner_pair(const Dev& d, int i, int j, int pr, double& cx, double& cy) {
    const int nx = d.nx, ny = d.ny;
    const double dt = step_dt(d.ctl);
    {
        const int sx = 1, sy = pr == 0 ? 1 : -1;
        const int pi = i + sx, pj = j + sy;
        cx = 0.0;
        cy = 0.0;
        bool active = true;
        if (!d.per_x && (pi < 0 || pi > nx)) active = false;
        if (!d.per_y && (pj < 0 || pj > ny)) active = false;
        double Fv = 0.0;
        if (active) {
            double sc[4];
            const int qi[4] = {i, i + sx, i, i + sx}, qj[4] = {j, j, j + sy, j + sy};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int n = ix(d, qi[q], qj[q]);
                // cf_corner_flux (remap.cpp:16-25) recomputed from u_half
                const double ddx = d.uhx[n] * dt, ddy = d.uhy[n] * dt;
                const double cdv = fabs(ddx * ddy), dmcv = d.dmc[n];
                sc[q] = 0.0;
                if (cdv == 0.0 || dmcv == 0.0) continue;
                const int csx = ddx > 0.0 ? 1 : -1, csy = ddy > 0.0 ? 1 : -1;
                if (csx == sx && csy == sy)
                    sc[q] = -dmcv;
                else if (csx == -sx && csy == -sy)
                    sc[q] = dmcv;
            }
            Fv = 0.25 * (sc[0] + sc[1] + sc[2] + sc[3]);
            if (Fv == 0.0) active = false;
        }
        if (active) {
            const bool incoming = Fv > 0.0;
            const int di = incoming ? pi : i, dj = incoming ? pj : j;
            const int wi = d.per_x ? ((di % nx) + nx) % nx : di;
            const int wj = d.per_y ? ((dj % ny) + ny) % ny : dj;
            double ufx, ufy;
            if (!(d.corner != CS_UPWIND && d.face_order > 1)) {
                ufx = d.ulx[ix(d, wi, wj)];
                ufy = d.uly[ix(d, wi, wj)];
            } else {
                const int ci0 = i < pi ? i : pi, cj0 = j < pj ? j : pj;
                const int ci = d.per_x ? ((ci0 % nx) + nx) % nx : ci0;
                const int cj = d.per_y ? ((cj0 % ny) + ny) % ny : cj0;
                // xlag2 of cell (ci, cj) (remap.cpp:797-803) recomputed from u_half
                const int n00 = ix(d, ci, cj), n10 = ix(d, ci + 1, cj), n01 = ix(d, ci, cj + 1),
                             n11 = ix(d, ci + 1, cj + 1);
                const double xmd = 0.25 * (dt * d.uhx[n00] + dt * d.uhx[n10] + dt * d.uhx[n01] + dt * d.uhx[n11]);
                const double ymd = 0.25 * (dt * d.uhy[n00] + dt * d.uhy[n10] + dt * d.uhy[n01] + dt * d.uhy[n11]);
                const double cxc = d.x0 + (ci + 0.5) * d.dx, cyc = d.y0 + (cj + 0.5) * d.dy;
                const double mdx = (cxc + xmd) - cxc;
                const double mdy = (cyc + ymd) - cyc;
                const double dirx = incoming ? -sx : sx, diry = incoming ? -sy : sy;
                const double dxp = dirx * rmax(fabs(mdx), 1e-300);
                const double dyp = diry * rmax(fabs(mdy), 1e-300);
                const double lwx = d.dx + 0.5 * (dt * d.uhx[ix(d, wi + 1, wj)] - dt * d.uhx[ix(d, wi - 1, wj)]);
                const double lwy = d.dy + 0.5 * (dt * d.uhy[ix(d, wi, wj + 1)] - dt * d.uhy[ix(d, wi, wj - 1)]);
                bool bad = false;
                if (!XC || d.corner == CS_LINEARDIAG) {
                    double ax_[9], ay_[9], xlx[9], xly[9];
#pragma unroll
                    for (int q = 0; q < 3; ++q)
#pragma unroll
                        for (int p = 0; p < 3; ++p) {
                            const int ni = wi + p - 1, nj = wj + q - 1;
                            const int nn = ix(d, ni, nj);
                            ax_[p * 3 + q] = d.ulx[nn];
                            ay_[p * 3 + q] = d.uly[nn];
                            xlx[p * 3 + q] = (d.x0 + ni * d.dx) + dt * d.uhx[nn];
                            xly[p * 3 + q] = (d.y0 + nj * d.dy) + dt * d.uhy[nn];
                        }
                    ufx = corner_diag(d, ax_, xlx, xly, dxp, dyp, lwx, lwy, bad);
                    ufy = corner_diag(d, ay_, xlx, xly, dxp, dyp, lwx, lwy, bad);
                } else {
                    Kin kin;  // the synthetic kinematics of remap.cpp:1036-1052
                    kin.dxp = dxp;
                    kin.dyp = dyp;
                    kin.lwx = lwx;
                    kin.lwy = lwy;
                    kin.sfx = dirx;
                    kin.ufx = mdx;
                    kin.sfy = diry;
                    kin.ufy = mdy;
                    kin.erx = (cxc + 0.5 * mdx) - ((d.x0 + wi * d.dx) + dt * d.uhx[ix(d, wi, wj)]);
                    kin.ery = (cyc + 0.5 * mdy) - ((d.y0 + wj * d.dy) + dt * d.uhy[ix(d, wi, wj)]);
                    const Pair2 r2 = dual_corner_other(d.corner, d.dgx, d.dgy, d.ulx, d.uly, d.uhx, d.uhy, ix(d, wi, wj),
                                                       d.P, wi, wj, d.x0, d.y0, d.dx, d.dy, dt, kin);
                    ufx = r2.a;
                    ufy = r2.b;
                    if (r2.bad) bad = true;
                }
                if (bad && own_node(d, i, j)) raise(d.ctl, ekey(PH_GRAD_DUALC, j, i, pr));
            }
            cx = ufx * Fv;
            cy = ufy * Fv;
        }
        return active;
    }
}
template <bool XC>
__device__ __forceinline__ void dual_corner_items(const Dev& d, int i, int j) {
    const int s = ix(d, i, j);
#pragma unroll
    for (int pr = 0; pr < 2; ++pr) {
        double cx, cy;
        const bool on = dual_corner_pair<XC>(d, i, j, pr, cx, cy);
        d.dc_x[pr][s] = cx;
        d.dc_y[pr][s] = cy;
        if (d.per_x || d.per_y) d.dflag[2 + pr][s] = on;
    }
}

// All dual-mesh items of one unique node (i, j): its X and Y dual faces and
// its two diagonal corner exchanges (remap.cpp:995-1069).
#ifndef H2D_DUAL_MINB
#define H2D_DUAL_MINB 8
#endif
template <bool XC = false>
__global__ void __launch_bounds__(128, H2D_DUAL_MINB) k_dual_items(Dev d) {
    pdl_enter();
    if (halted(d.ctl)) return;
    int i, j;
    tid2(i, j, d.r_dual.i0, d.r_dual.j0);
    const int iend = d.per_x ? d.nx - 1 : d.nx, jend = d.per_y ? d.ny - 1 : d.ny;
    if (!in(d.r_dual, i, j) || i < 0 || j < 0 || i > iend || j > jend) return;
    {  // every mass flux the node's items read is zero: all items are skipped
       // ones (remap.cpp:423,1019), stored as exact zeros
        const int a = ix(d, i - 1, j - 1), b = ix(d, i, j - 1), c = ix(d, i - 1, j), e = ix(d, i, j);
        const int f = ix(d, i + 1, j - 1), g = ix(d, i + 1, j), h = ix(d, i, j + 1), k = ix(d, i + 1, j + 1);
        const double* X = d.dmx;
        const double* Y = d.dmy;
        const double* Cn = d.dmc;
        const bool quiet = (X[a] == 0.0) & (X[b] == 0.0) & (X[c] == 0.0) & (X[e] == 0.0) & (Y[a] == 0.0) &
                           (Y[b] == 0.0) & (Y[c] == 0.0) & (Y[e] == 0.0) & (Cn[b] == 0.0) & (Cn[f] == 0.0) &
                           (Cn[e] == 0.0) & (Cn[g] == 0.0) & (Cn[h] == 0.0) & (Cn[k] == 0.0);
        if (!(d.per_x || d.per_y)) {  // walls: dflag[0] marks a quiet node, its items are not stored
            d.dflag[0][e] = quiet;
            if (quiet) return;
        } else if (quiet) {
            d.dfx_x[e] = 0.0;
            d.dfx_y[e] = 0.0;
            d.dfy_x[e] = 0.0;
            d.dfy_y[e] = 0.0;
            d.dc_x[0][e] = 0.0;
            d.dc_y[0][e] = 0.0;
            d.dc_x[1][e] = 0.0;
            d.dc_y[1][e] = 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) d.dflag[q][e] = 0;
            return;
        }
    }
    dual_face_item<1>(d, i, j);
    dual_face_item<0>(d, i, j);
    dual_corner_items<XC>(d, i, j);
}

// Wall boundaries: the MomAcc gather in its fixed loop order — X face i (+),
// X face i+1 (-), Y face j (+), Y face j+1 (-), corner (i-1, j-1, pair (1,1))
// (-), own pairs (+, +), corner (i-1, j+1, pair (1,-1)) (-) — then
// apply_dual_update (remap.cpp:444-464) and the wall condition (:462).
template <int NM>
__device__ __forceinline__ void node_update_walls_at(const Dev& d, int i, int j, double& px, double& py) {
    const int nx = d.nx, ny = d.ny;
    if (!in(d.r_node, i, j) || i < 0 || j < 0 || i > nx || j > ny) return;
    const int s = ix(d, i, j);
    const int sxr = ix(d, i + 1, j), syt = ix(d, i, j + 1);
    const int pp = ix(d, i - 1, j - 1), pm = ix(d, i - 1, j + 1);
    // Items outside the unique node range were never written: index guards.
    // A skipped item (zero dual mass flux, inactive corner) is stored as
    // exactly 0.0, and adding +-0.0 leaves the accumulator unchanged (it
    // starts at +0.0 and a sum is -0.0 only if both terms are), so the
    // reference's skip needs no flag here.
    // Items of a quiet node (k_dual_items, dflag[0]) are zeros that were not
    // stored: they are skipped like the zero items above.
    const uint8_t* qf = d.dflag[0];
    const bool qs = qf[s];
    const bool fxp = i >= 1 && !qs, fxm = i + 1 <= nx && !qf[sxr], fyp = j >= 1 && !qs,
               fym = j + 1 <= ny && !qf[syt];
    const bool fpp = i >= 1 && j >= 1 && !qf[pp], fpm = i >= 1 && j + 1 <= ny && !qf[pm];
    double ax = 0.0, ay = 0.0;
    if (fxp) { ax += d.dfx_x[s]; ay += d.dfx_y[s]; }
    if (fxm) { ax += -d.dfx_x[sxr]; ay += -d.dfx_y[sxr]; }
    if (fyp) { ax += d.dfy_x[s]; ay += d.dfy_y[s]; }
    if (fym) { ax += -d.dfy_x[syt]; ay += -d.dfy_y[syt]; }
    if (fpp) { ax += -d.dc_x[0][pp]; ay += -d.dc_y[0][pp]; }
    if (!qs) {
        ax += d.dc_x[0][s];
        ay += d.dc_y[0][s];
        ax += d.dc_x[1][s];
        ay += d.dc_y[1][s];
    }
    if (fpm) { ax += -d.dc_x[1][pm]; ay += -d.dc_y[1][pm]; }
    const int c00 = pp, c10 = ix(d, i, j - 1), c01 = ix(d, i - 1, j);
    double l00 = 0.0, l10 = 0.0, l01 = 0.0, l11 = 0.0;  // make_work's mcell (remap.cpp:133-138)
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        l00 += d.m[a][c00];
        l10 += d.m[a][c10];
        l01 += d.m[a][c01];
        l11 += d.m[a][s];
    }
    const double mp_lag = 0.25 * (l00 + l10 + l01 + l11);
    const double mp_new = 0.25 * (d.mcell[c00] + d.mcell[c10] + d.mcell[c01] + d.mcell[s]);
    if (mp_new <= 0.0 && own_node(d, i, j)) raise(d.ctl, ekey(PH_NODAL_MASS, j, i, 0));
    const double inv = 1.0 / mp_new;
    double ux = inv * (mp_lag * d.ulx[s] + ax), uy = inv * (mp_lag * d.uly[s] + ay);
    if (i == 0 || i == nx) ux = 0.0;
    if (j == 0 || j == ny) uy = 0.0;
    d.nux[s] = ux;
    d.nuy[s] = uy;
    const double u2 = ux * ux + uy * uy;  // (a node at rest: sqrt(+0) = +0 without the sqrt)
    d.unrm[s] = u2 == 0.0 ? 0.0 : sqrt(u2);
    if (d.scan_nodes && own_node(d, i, j) && (!isfinite(ux) | !isfinite(uy)))
        raise(d.ctl, ekey(PH_NAN_NODE, j, i, 0));  // nan_scan on the new u (harness.cpp:353-357)
    if (d.diag && own_node(d, i, j)) {  // compute_totals' momentum term (state.cpp:154-158)
        px = mp_new * ux;
        py = mp_new * uy;
    }
}

// Run-loop epilogue of the node kernels: the step's total momentum
// (compute_totals, state.cpp:154-158) for the diagnostics record.
__device__ __forceinline__ void node_momentum(const Dev& d, double px, double py) {
    if (!d.diag) return;
    double v[2] = {px, py};
    const int op[2] = {0, 0};
    warp_partial<2>(v, op, d.dsc.part[1]);
}

template <int NM>
__global__ void k_node_update_walls(Dev d) {
    pdl_enter();
    if (halted(d.ctl)) return;  // one load per warp: warp-uniform
    int i, j;
    tid2(i, j, d.r_node.i0, d.r_node.j0);
    double px = 0.0, py = 0.0;
    node_update_walls_at<NM>(d, i, j, px, py);
    node_momentum(d, px, py);
}

// MomAcc gather (App. C item 4) + apply_dual_update (remap.cpp:444-464) with
// the periodic copies (:458-461) folded in: thread per node (i, j) in
// [0, nx] x [0, ny] computes the value of its source node.
__device__ __forceinline__ void node_update_at(const Dev& d, int i, int j, double& px, double& py) {
    const int nx = d.nx, ny = d.ny;
    if (!in(d.r_node, i, j) || i < 0 || j < 0 || i > nx || j > ny) return;
    const int iend = d.per_x ? nx - 1 : nx, jend = d.per_y ? ny - 1 : ny;
    const int si = (d.per_x && i == nx) ? 0 : i, sj = (d.per_y && j == ny) ? 0 : j;
    const int s = ix(d, si, sj);
    double ax = 0.0, ay = 0.0;
    // X then Y dual faces (remap.cpp:995-996). Face ia joins nodes (ia-1, ia):
    // + to node ia, - to the node ia-1 wraps to; applied in face-loop order.
    auto faces = [&](int ax_, int along, int cross) {
        const int n = ax_ ? nx : ny;
        const int per = ax_ ? d.per_x : d.per_y;
        const int hi = ax_ ? iend : jend, lo = per ? 0 : 1;
        const double* fx_ = ax_ ? d.dfx_x : d.dfy_x;
        const double* fy_ = ax_ ? d.dfx_y : d.dfy_y;
        const uint8_t* fl = d.dflag[ax_ ? 0 : 1];
        auto at = [&](int a) { return ax_ ? ix(d, a, cross) : ix(d, cross, a); };
        int am = along + 1;
        if (per && am == n) am = 0;
        const bool ap = along >= lo && along <= hi && fl[at(along)];
        const bool an = am >= lo && am <= hi && fl[at(am)];
        const bool minus_first = an && am < along;
        if (minus_first) {
            ax += -fx_[at(am)];
            ay += -fy_[at(am)];
        }
        if (ap) {
            ax += fx_[at(along)];
            ay += fy_[at(along)];
        }
        if (an && !minus_first) {
            ax += -fx_[at(am)];
            ay += -fy_[at(am)];
        }
    };
    faces(1, si, sj);
    faces(0, sj, si);
    {  // dual corners: up to 4 contributions, applied in (j, i, pair) loop order
        const int iuniq = iend, juniq = jend;
        long long tk[4];
        double cx[4], cy[4];
        int nc = 0;
        auto push = [&](int ii, int jj, int pr, double sgn) {
            if (ii < 0 || ii > iuniq || jj < 0 || jj > juniq) return;
            const int q = ix(d, ii, jj);
            if (!d.dflag[2 + pr][q]) return;
            tk[nc] = ((long long)jj * (iuniq + 1) + ii) * 2 + pr;
            cx[nc] = sgn > 0 ? d.dc_x[pr][q] : -d.dc_x[pr][q];
            cy[nc] = sgn > 0 ? d.dc_y[pr][q] : -d.dc_y[pr][q];
            ++nc;
        };
        // partner index of pair (1, +-1) whose target wraps to (si, sj)
        int ip = si - 1, jp1 = sj - 1, jp2 = sj + 1;
        if (d.per_x && ip < 0) ip += nx;
        if (d.per_y) {
            if (jp1 < 0) jp1 += ny;
            if (jp2 >= ny) jp2 -= ny;
        }
        push(ip, jp1, 0, -1.0);
        if (si <= iuniq && sj <= juniq) {
            push(si, sj, 0, 1.0);
            push(si, sj, 1, 1.0);
        }
        push(ip, jp2, 1, -1.0);
        // with walls the pushes above are already in loop order; periodic
        // wrap can reorder them: insertion sort by loop time (n <= 4)
        if (d.per_x || d.per_y)
            for (int a = 1; a < nc; ++a)
            for (int b = a; b > 0 && tk[b - 1] > tk[b]; --b) {
                long long t0 = tk[b];
                tk[b] = tk[b - 1];
                tk[b - 1] = t0;
                double v = cx[b];
                cx[b] = cx[b - 1];
                cx[b - 1] = v;
                v = cy[b];
                cy[b] = cy[b - 1];
                cy[b - 1] = v;
            }
        for (int a = 0; a < nc; ++a) {
            ax += cx[a];
            ay += cy[a];
        }
    }
    // mcell before finalize = make_work's sum of the state's partial masses
    // (remap.cpp:133-138), incl. ghost cells
    auto ml = [&](size_t c) {
        double mc = 0.0;
        for (int a = 0; a < d.nmat; ++a) mc += d.m[a][c];
        return mc;
    };
    const double mp_lag = 0.25 * (ml(ix(d, si - 1, sj - 1)) + ml(ix(d, si, sj - 1)) + ml(ix(d, si - 1, sj)) + ml(s));
    const double mp_new =
        0.25 * (d.mcell[ix(d, si - 1, sj - 1)] + d.mcell[ix(d, si, sj - 1)] + d.mcell[ix(d, si - 1, sj)] + d.mcell[s]);
    if (mp_new <= 0.0 && si == i && sj == j && own_node(d, i, j)) raise(d.ctl, ekey(PH_NODAL_MASS, j, i, 0));
    const double inv = 1.0 / mp_new;
    const int o = ix(d, i, j);
    double ux = inv * (mp_lag * d.ulx[s] + ax), uy = inv * (mp_lag * d.uly[s] + ay);
    // fill_ghost_nodes (remap.cpp:462) zeroes the normal component on walls
    if (!d.per_x && (i == 0 || i == nx)) ux = 0.0;
    if (!d.per_y && (j == 0 || j == ny)) uy = 0.0;
    d.nux[o] = ux;
    d.nuy[o] = uy;
    d.unrm[o] = sqrt(ux * ux + uy * uy);  // |u| for the next cfl_dt (harness.cpp:308)
    if (d.scan_nodes && own_node(d, i, j) && (!isfinite(ux) | !isfinite(uy)))
        raise(d.ctl, ekey(PH_NAN_NODE, j, i, 0));  // nan_scan on the new u (harness.cpp:353-357)
    if (d.diag && i <= iend && j <= jend && own_node(d, i, j)) {  // state.cpp:154-158
        px = mp_new * ux;
        py = mp_new * uy;
    }
}

__global__ void k_node_update(Dev d) {
    pdl_enter();
    if (halted(d.ctl)) return;  // one load per warp: warp-uniform
    int i, j;
    tid2(i, j, d.r_node.i0, d.r_node.j0);
    double px = 0.0, py = 0.0;
    node_update_at(d, i, j, px, py);
    node_momentum(d, px, py);
}

// refresh_normals_impl + youngs_normal (remap.cpp:102-114, vof.cpp:10-22)
// on the next state's fractions; `api` = operate on the current state.
__global__ void k_normals(Dev d, int api) {
    pdl_enter();
    if (!api && halted(d.ctl)) return;
    int i, j;
    tid2(i, j, 0, 0);
    if (i >= d.nx || j >= d.ny) return;
    // a decomposition block: only cells whose 3x3 stencil is stored (the
    // outer halo ring is made exact by the first halo exchange)
    if (!in(d.win_c, i - 1, j - 1) || !in(d.win_c, i + 1, j + 1)) return;
    const double* k0 = api ? d.k[0] : d.nk[0];
    const double* k1 = api ? d.k[1] : d.nk[1];
    double* nx_ = api ? const_cast<double*>(d.nrx) : d.nnrx;
    double* ny_ = api ? const_cast<double*>(d.nry) : d.nnry;
    const int c = ix(d, i, j);
    if (!api) {  // the Work normals start as the State's (remap.cpp:130)
        nx_[c] = d.nrx[c];
        ny_[c] = d.nry[c];
    }
    if (d.nmat == 3) {  // three materials: the interface pair's k_hi (pair3)
        const double* kf[3];
        for (int a = 0; a < 3; ++a) kf[a] = api ? d.k[a] : d.nk[a];
        const double k3[3] = {kf[0][c], kf[1][c], kf[2][c]};
        if (!mixed3(k3)) return;
        int lo, hi;
        pair3(k3, lo, hi);
        k1 = kf[hi];
    } else if (!is_mixed(k0[c])) {
        return;
    }
    auto K = [&](int ii, int jj) { return k1[ix(d, ii, jj)]; };
    auto col = [&](int ii) { return K(ii, j - 1) + 2.0 * K(ii, j) + K(ii, j + 1); };
    auto row = [&](int jj) { return K(i - 1, jj) + 2.0 * K(i, jj) + K(i + 1, jj); };
    const double gx = div_dx(d, col(i + 1) - col(i - 1), 8.0);
    const double gy = div_dy(d, row(j + 1) - row(j - 1), 8.0);
    const double g = sqrt(gx * gx + gy * gy);
    if (g < 1e-300) return;  // IsolatedMixedCellError caught: keep the previous normal
    nx_[c] = gx / g;
    ny_[c] = gy / g;
}

// Step commit: the remapped State becomes current (remap.cpp:1084-1085).
__global__ void k_commit(Ctl* c, int advance) {
    pdl_enter();
    if (c->err_key != kNoErr || c->done) return;
    if (advance) {
        c->time = c->time + c->dt;
        c->step += 1;
    }
    c->cur ^= 1;
}

// Start of a run-loop step (harness.cpp:390-395): loop condition, then the
// cfl_dt of the current State, whose wave-speed maximum and first error were
// produced by the previous step's k_post (or k_cfl before the first step).
__device__ __forceinline__ void step_start_body(Ctl* c, double dx, double dy) {
    if (c->err_key != kNoErr || c->done) return;
    c->kviol_bits = 0ull;
    c->step_floor = 0;
    c->step_clip = 0;
    c->step_fix = 0;
    const double t_end = c->t_end;
    if (!(c->time < t_end - 1e-15 * rmax(1.0, t_end)) || (c->max_steps > 0 && c->step >= c->max_steps)) {
        c->done = 1;
        return;
    }
    if (c->next_err_key != kNoErr) {
        c->err_key = c->next_err_key;
        return;
    }
    const double wmax = __longlong_as_double((long long)c->next_wmax_bits);
    if (!(wmax > 0.0) || !isfinite(wmax)) {
        c->err_key = ekey(PH_CFL_WAVE, 0x1FFFFFF - 32, 0, 0);
        return;
    }
    double dt = c->cfl * rmin(dx, dy) / wmax;
    c->last_dt = dt;
    c->dt = rmin(dt, t_end - c->time);
    c->next_wmax_bits = 0ull;
    c->next_err_key = kNoErr;
}
__global__ void k_step_start(Ctl* c, double dx, double dy) {
    pdl_enter();
    step_start_body(c, dx, dy);
}

// End of a run-loop step: the remapped State becomes current
// (remap.cpp:1084-1085) unless an earlier phase failed; nan_scan errors come
// after the commit (harness.cpp:402-409), so they still commit.
__device__ __forceinline__ void commit_finish_body(Ctl* c) {
    c->committed = 0;
    c->counted = 0;
    if (c->done) return;
    const unsigned long long e = c->err_key;
    const bool ok = e == kNoErr;
    if (!ok && (int)(e >> 58) < PH_NAN_CELL) return;
    c->prev_time = c->time;
    c->prev_max_k_violation = c->max_k_violation;
    c->time = c->time + c->dt;
    c->step += 1;
    c->cur ^= 1;
    c->committed = 1;
    if (!ok) return;
    if (c->dt_log && c->steps_done < c->dt_log_cap) c->dt_log[c->steps_done] = c->dt;
    if (c->diag_log && c->steps_done < c->diag_log_cap) {  // rep.series.push_back(make_diag(s, dt))
        double* r = c->diag_log + (size_t)c->steps_done * kDiagRec;
        r[0] = (double)c->step;
        r[1] = c->time;
        r[2] = c->dt;
        for (int k = 0; k < DG_N; ++k) r[3 + k] = c->dg[k];
    }
    c->steps_done += 1;
    c->floor_count += c->step_floor;
    c->k_clip_count += c->step_clip;
    c->mass_fix_count += c->step_fix;
    const double v = __longlong_as_double((long long)c->kviol_bits);
    if (v > c->max_k_violation) c->max_k_violation = v;
    c->counted = 1;
}
__global__ void k_commit_finish(Ctl* c) {
    pdl_enter();
    commit_finish_body(c);
}

// Undo the last commit (block mode: another block failed in the same step
// before its commit, so the decomposed State must stay at the previous step).
__global__ void k_rollback(Ctl* c) {
    pdl_enter();
    if (!c->committed) return;
    c->time = c->prev_time;
    c->step -= 1;
    c->cur ^= 1;
    if (c->counted) {
        c->steps_done -= 1;
        c->floor_count -= c->step_floor;
        c->k_clip_count -= c->step_clip;
        c->mass_fix_count -= c->step_fix;
        c->max_k_violation = c->prev_max_k_violation;
    }
    c->committed = 0;
    c->counted = 0;
}

// Copy a rectangle (global indices, half-open) of several planes to / from a
// contiguous buffer: cell planes use `rc`, node planes `rn` (halo exchange).
__global__ void k_rect_xfer(Dev d, FieldList cells, FieldList nodes, Rng rc, Rng rn, double* buf, int to_buf) {
    pdl_enter();
    const int wc = rc.i1 - rc.i0, hc = rc.j1 - rc.j0, wn = rn.i1 - rn.i0, hn = rn.j1 - rn.j0;
    const long long ac = (long long)wc * hc, an = (long long)wn * hn;
    const long long total = ac * cells.n + an * nodes.n;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        double* pl;
        int i, j;
        if (t < ac * cells.n) {
            const int f = (int)(t / ac);
            const long long r = t - f * ac;
            pl = cells.f[f];
            i = rc.i0 + (int)(r % wc);
            j = rc.j0 + (int)(r / wc);
        } else {
            const long long u = t - ac * cells.n;
            const int f = (int)(u / an);
            const long long r = u - f * an;
            pl = nodes.f[f];
            i = rn.i0 + (int)(r % wn);
            j = rn.j0 + (int)(r / wn);
        }
        if (to_buf)
            buf[t] = pl[ix(d, i, j)];
        else
            pl[ix(d, i, j)] = buf[t];
    }
}

// Rectangle r of this block's planes <-> a compact buffer (row pitch r width;
// vec != 0: interleaved Vec2 split into x / y planes) — window uploads and
// owned-region downloads in the global reference layout.
__global__ void k_global_xfer(Dev d, double* buf, Rng r, double* px, double* py, int vec, int to_block) {
    pdl_enter();
    const int w = r.i1 - r.i0, h = r.j1 - r.j0;
    const long long n = (long long)w * h;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        const int i = r.i0 + (int)(t % w), j = r.j0 + (int)(t / w);
        const int li = ix(d, i, j);
        if (to_block) {
            if (vec) {
                px[li] = buf[2 * t];
                py[li] = buf[2 * t + 1];
            } else {
                px[li] = buf[t];
            }
        } else {
            if (vec) {
                buf[2 * t] = px[li];
                buf[2 * t + 1] = py[li];
            } else {
                buf[t] = px[li];
            }
        }
    }
}


// The end of the remap on the new State, one thread per position of the
// ghosted node range: sync_derived over every cell (state.cpp:120-143, from
// assemble_state remap.cpp:1087), refresh_normals_impl on interior cells
// (remap.cpp:102-114, vof.cpp:10-22), and in the run loop nan_scan
// (harness.cpp:347-358) plus the wave speed of the next step's cfl_dt
// (harness.cpp:293-310), so the State is read once.
#ifndef H2D_POST_MINB
#define H2D_POST_MINB 5
#endif
// Three materials: the class of each remap tile (Dev::tcls). A material r is
// absent from a tile when no cell of the tile's staged region (the 36 x 12
// TMA box, zero past the plane) has k_r > 0 or m_r != 0. The two-slot kernel
// on the other two materials (lo < hi) is then the three-material kernel,
// given that every region cell satisfies
//  * a cell holding lo alone is not mixed in the two-material sense
//    (mixed3 == is_mixed(k_lo), remap.cpp:100 / oracle mixed3), and
//  * a non-mixed donor's material is the same: largest3(k) == (k_lo < 0.5 ?
//    hi : lo) (remap.cpp:255-263 / oracle split_flux);
// (with k_r = 0 the mixed split, the interface fraction and the degrade
// tests reduce to the two-material expressions term by term). The class is
// the highest such r, else 3.
__device__ __forceinline__ bool map_ok(const double* k, int r) {
    const int lo = r == 0 ? 1 : 0, hi = r == 2 ? 1 : 2;
    if (k[lo] > 0.0 && !(k[hi] > 0.0) && is_mixed(k[lo])) return false;
    if (!mixed3(k) && largest3(k) != (k[lo] < 0.5 ? hi : lo)) return false;
    return true;
}
// Two materials: with r absent the one-material kernel on p = 1 - r is the
// two-material one when every region cell is pure p in the reference's
// sense (k_p >= 1 - kPureTol): no cell is mixed (remap.cpp:100), every donor
// is p's (k0 < 0.5 <=> p = 1, remap.cpp:263) and no stencil degrades to
// first order (remap.cpp:270-283).
__device__ __forceinline__ bool map_ok2(const double* k, int r) { return k[1 - r] >= 1.0 - kPureTol; }

// One cell's terms of the tile classification (k_tile_class): material a is
// present (bits 0-2), the mapping condition of "r absent" fails (bits 3-5),
// k_a is not pure (bits 6-8); OR over the cells of a tile's staged region
template <int NM>
__device__ __forceinline__ unsigned cell_cls_mask(const double* k, const double* m) {
    unsigned mk = 0u;
#pragma unroll
    for (int r = 0; r < NM; ++r) {
        if (k[r] > 0.0 || m[r] != 0.0) mk |= 1u << r;
        if (!(NM == 3 ? map_ok(k, r) : map_ok2(k, r))) mk |= 8u << r;
        if (!(k[r] >= 1.0 - kPureTol)) mk |= 64u << r;
    }
    return mk;
}
// the class of a tile from the OR of its region's cell masks (see k_tile_class)
template <int NM>
__device__ __forceinline__ int cls_of_mask(unsigned mk) {
    const unsigned pres = mk & 7u, ok = ~(mk >> 3) & 7u, pure = ~(mk >> 6) & 7u;
    int cls = 3;
    if (NM == 2 || H2D_RT_MAP32)
        for (int r = NM - 1; r >= 0 && cls == 3; --r)
            if (!((pres >> r) & 1u) && ((ok >> r) & 1u)) cls = r;
    // three materials, ONE present (p) and pure in every region cell: the
    // two-slot mapping (either absent material, both conditions hold) whose
    // second slot is absent too and meets the two-material condition
    // (map_ok2: every region cell pure p), i.e. the one-material kernel
    if (NM == 3 && H2D_RT_MAP31)
        for (int p = 0; p < 3; ++p) {
            const unsigned others = 7u & ~(1u << p);
            if (pres == (1u << p) && (ok & others) == others && ((pure >> p) & 1u)) cls = 4 + p;
        }
    return cls;
}

#ifndef H2D_POST_INTERIOR
#define H2D_POST_INTERIOR 1
#endif
// INT: every cell of the block is a mesh cell inside r_sync, r_nrm and the
// owned range (uniform over the block, see k_post): the range tests are true
// and compiled out
template <int NM, bool INT>
__device__ __forceinline__ void post_body(const Dev& d, const int run_loop, unsigned long long* sw,
                                          double (*s_dg)[256], unsigned* s_cls) {
    constexpr int NDG = NM == 3 ? DG_NCELL : DG_NCELL - 1;
    int i, j;
    tid2(i, j, d.r_sync.i0, d.r_sync.j0);
    const int nx = d.nx, ny = d.ny;
    unsigned long long wb = 0ull;
    const bool act = INT || in(d.r_sync, i, j);
    const bool interior = INT || (i >= 0 && j >= 0 && i < nx && j < ny);
    const int c = act ? ix(d, i, j) : 0;
    const double cv = d.cv;
    double ka[NM], ma[NM], ea[NM];
    double m = 0.0, emix = 0.0, p = 0.0;
    // the next step's sound speed (cfl_dt, harness.cpp:293-313) comes out of
    // the same per-material loop as the mixture pressure: the materials with
    // k >= kThermoTol, in index order, from the same rho_a and p_a (the
    // wave-speed block below only adds |u|)
    double cs = 0.0;
    bool cs_bad = false;
    unsigned cmk = 0u;  // this cell's classification mask (cell_cls_mask)
    if (act) {
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            ka[a] = d.nk[a][c];
            ma[a] = d.nm[a][c];
            ea[a] = d.ne[a][c];
        }
        double me = 0.0;
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            if (ka[a] <= 0.0) continue;
            m += ma[a];
            me += ma[a] * ea[a];
            if (ka[a] < kThermoTol) continue;
            const double rho_a = rho_of(d, ma[a], ka[a]);
            const double pa = eos_p(d, a, rho_a, ea[a]);
            p += ka[a] * pa;
            if (run_loop) cs += ka[a] * sound(d, a, rho_a, pa, cs_bad);
        }
        emix = m > 0.0 ? me / m : 0.0;
        if (NM >= 2 && run_loop && d.pcls) cmk = cell_cls_mask<NM>(ka, ma);  // for the next step's tile classes
        if (!run_loop) {  // the run loop keeps no derived planes (rebuilt when the State is read)
            d.nm_mix[c] = m;
            d.ne_mix[c] = emix;
            d.nrho_mix[c] = div_cv(d, m);
            d.np_mix[c] = p;
            d.nvol[c] = cv;
        }
    }
    // make_diag's cell part (harness.cpp:360-376, state.cpp:148-153): this
    // cell's terms go to shared memory now (registers stay free for the rest)
    // and are folded after the kernel's closing barrier
    const int tl = threadIdx.y * blockDim.x + threadIdx.x;
    if (run_loop && d.diag) {
        const bool on = INT || (act && interior && own_cell(d, i, j));
        const double rho = div_cv(d, m);
        constexpr int sh = NM == 3 ? 0 : 1;  // plane of slot k >= DG_MINR: k - sh
        s_dg[DG_MASS][tl] = on ? m : 0.0;
        s_dg[DG_IE][tl] = on ? m * emix : 0.0;
        s_dg[DG_MM0][tl] = on ? ma[0] : 0.0;
        s_dg[DG_MM1][tl] = on && NM >= 2 ? ma[NM >= 2 ? 1 : 0] : 0.0;
        if (NM == 3) s_dg[NM == 3 ? DG_MM2 : 0][tl] = on ? ma[NM - 1] : 0.0;
        s_dg[DG_MINR - sh][tl] = on ? rho : CUDART_INF;
        s_dg[DG_MAXR - sh][tl] = on ? rho : -CUDART_INF;
        s_dg[DG_MINP - sh][tl] = on ? p : CUDART_INF;
        s_dg[DG_MAXP - sh][tl] = on ? p : -CUDART_INF;
    }
    if (act) {
        if (INT || (interior && in(d.r_nrm, i, j))) {
            if (NM >= 2) {  // normals of the new fractions
                bool mixed = is_mixed(ka[0]);
                int hi = 1;
                if (NM == 3) {  // Youngs normal of the interface pair's k_hi (pair3)
                    const double k3[3] = {ka[0], ka[1], ka[NM - 1]};
                    mixed = mixed3(k3);
                    int lo;
                    pair3(k3, lo, hi);
                }
                // in place (a single domain's parities share the normal
                // plane): it already holds the old normal, which a non-mixed
                // cell keeps, so only mixed cells are read and written
                const bool inplace = d.nrx == d.nnrx;
                double nrx = 0.0, nry = 0.0;
                if (mixed || !inplace) {
                    nrx = d.nrx[c];
                    nry = d.nry[c];
                }
                if (mixed) {
                    const double* kh = d.nk[hi];
                    auto K = [&](int ii, int jj) { return kh[ix(d, ii, jj)]; };
                    auto col = [&](int ii) { return K(ii, j - 1) + 2.0 * K(ii, j) + K(ii, j + 1); };
                    auto row = [&](int jj) { return K(i - 1, jj) + 2.0 * K(i, jj) + K(i + 1, jj); };
                    const double gx = div_dx(d, col(i + 1) - col(i - 1), 8.0);
                    const double gy = div_dy(d, row(j + 1) - row(j - 1), 8.0);
                    const double g = sqrt(gx * gx + gy * gy);
                    if (!(g < 1e-300)) {  // an isolated mixed cell keeps its normal
                        nrx = gx / g;
                        nry = gy / g;
                    }
                }
                if (mixed || !inplace) {
                    d.nnrx[c] = nrx;
                    d.nnry[c] = nry;
                }
            }
            if (run_loop && (INT || own_cell(d, i, j))) {
                if (!isfinite(m) | !isfinite(emix) | !isfinite(p)) raise(d.ctl, ekey(PH_NAN_CELL, j, i, 0));
                // next step's wave speed on the new State (cs from above)
                if (cs_bad) atomicMin(&d.ctl->next_err_key, ekey(PH_CFL_UNPHYS, j, i, 0));
                double umax = 0.0;
#pragma unroll
                for (int dj = 0; dj <= 1; ++dj)
#pragma unroll
                    for (int di = 0; di <= 1; ++di) umax = rmax(umax, d.unrm[ix(d, i + di, j + dj)]);
                const double w = cs + umax;
                if (w > 0.0) wb = (unsigned long long)__double_as_longlong(w);
            }
        }
    }
    // (nan_scan's node part runs in the node update that writes u, d.scan_nodes)
    if (run_loop) {
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long v = __shfl_xor_sync(0xffffffffu, wb, o);
            wb = v > wb ? v : wb;
        }
        const int t = threadIdx.y * blockDim.x + threadIdx.x;
        if ((t & 31) == 0) sw[t >> 5] = wb;
        if (NM >= 2 && d.pcls) {  // (every thread of the block is here: no early exit above)
            cmk = __reduce_or_sync(0xffffffffu, cmk);
            if ((t & 31) == 0 && cmk) atomicOr(s_cls, cmk);
        }
        __syncthreads();
        if (t == 0) {
            for (int w = 1; w < (int)(blockDim.x * blockDim.y) / 32; ++w) wb = sw[w] > wb ? sw[w] : wb;
            if (wb) atomicMax(&d.ctl->next_wmax_bits, wb);
            if (NM >= 2 && d.pcls) d.pcls[blockIdx.y * gridDim.x + blockIdx.x] = (uint16_t)*s_cls;
        }
        if (d.diag) {  // warp w folds diagnostics planes w, w + 8 over the block's 256 cells (fixed order)
            double* part = d.dsc.part[0] + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * DG_NCELL;
            for (int pl = t >> 5; pl < NDG; pl += 8) {
                const int k = (NM == 3 || pl < DG_MM2) ? pl : pl + 1;  // the slot of plane pl
                const int lane = t & 31, op = dg_op(k);
                // (op is uniform over the warp: one copy of the fold per operation,
                // so dg_comb is a single add / min / max instead of all three + selects)
                auto fold = [&](auto opc) {
                    constexpr int OP = decltype(opc)::value;
                    double v = s_dg[pl][lane];
#pragma unroll
                    for (int q = 1; q < 8; ++q) v = dg_comb(OP, v, s_dg[pl][lane + 32 * q]);
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v = dg_comb(OP, v, __shfl_down_sync(0xffffffffu, v, o));
                    if (lane == 0) part[k] = v;
                };
                if (op == 0)
                    fold(std::integral_constant<int, 0>{});
                else if (op == 1)
                    fold(std::integral_constant<int, 1>{});
                else
                    fold(std::integral_constant<int, 2>{});
            }
            if (NM < 3 && t == 0) part[DG_MM2] = 0.0;
        }
    }
}

template <int NM>
__global__ void __launch_bounds__(256, H2D_POST_MINB) k_post(Dev d, int run_loop) {
    pdl_enter();
    __shared__ unsigned long long sw[8];
    // per-thread diagnostics terms (block of 32 x 8); fewer than three
    // materials keep no DG_MM2 plane (its partial is written as 0)
    constexpr int NDG = NM == 3 ? DG_NCELL : DG_NCELL - 1;
    __shared__ double s_dg[NDG][256];
    __shared__ int s_halt, s_int;
    __shared__ unsigned s_cls;
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        s_halt = halted(d.ctl);
        s_cls = 0u;
        bool interior = false;  // (uniform over the block: one thread evaluates it)
        if (H2D_POST_INTERIOR) {
            const int ia = d.r_sync.i0 + (int)(blockIdx.x * blockDim.x),
                      ja = d.r_sync.j0 + (int)(blockIdx.y * blockDim.y);
            const int ib = ia + (int)blockDim.x - 1, jb = ja + (int)blockDim.y - 1;
            interior = ia >= 0 && ja >= 0 && ib < d.nx && jb < d.ny && in(d.r_sync, ia, ja) && in(d.r_sync, ib, jb) &&
                       in(d.r_nrm, ia, ja) && in(d.r_nrm, ib, jb) && own_cell(d, ia, ja) && own_cell(d, ib, jb);
        }
        s_int = interior;
    }
    __syncthreads();
    if (s_halt) return;
    if (s_int)
        post_body<NM, true>(d, run_loop, sw, s_dg, &s_cls);
    else
        post_body<NM, false>(d, run_loop, sw, s_dg, &s_cls);
}

// ---------------------------------------------------------------------------
// AD split remap (remap.cpp:469-589), the first "next" row of SURVEY.md 8f:
// one directional pass along AX (1 = X, 0 = Y) per kernel sequence. Work
// inputs come from an AdIO (the State + LagrangeResult for pass 0, the AdWork
// of pass 0 for pass 1); outputs go to the next-state / Work planes of the Dev
// the pass is launched with, so finalize_cell, k_slivers and the ghost fills
// are shared with DirectCF.
// ---------------------------------------------------------------------------
template <int NM, int AX>
__global__ void __launch_bounds__(RTX * RTY, 3) k_ad_tile(Dev d, AdIO w) {
    pdl_enter();
    constexpr int CW = AX ? RTX + 4 : RTX, CH = AX ? RTY : RTY + 4;  // cells: along-axis halo of 2
    constexpr int FW = AX ? RTX + 5 : RTX, FH = AX ? RTY : RTY + 5;  // along-axis faces of those cells
    constexpr int NCR = CW * CH, NFR = FW * FH;
    constexpr int NIF = AX ? (RTX + 1) * RTY : RTX * (RTY + 1);  // the tile's own faces
    __shared__ double s_fd[NFR];
    __shared__ double s_vl[NCR], s_xl[NCR], s_wl[NCR], s_rho[NM][NCR], s_e[NM][NCR], s_k[NM][NCR];
    __shared__ double s_ifd[NM == 2 ? NCR : 1];
    __shared__ double s_it[3][NM][NIF];
    __shared__ int s_halt;
    const int tid = threadIdx.x;
    if (tid == 0) s_halt = halted(d.ctl);
    __syncthreads();
    if (s_halt) return;
    const int nx = d.nx, ny = d.ny;
    const Rng rg = d.r_gath;
    const int i0 = rg.i0 + blockIdx.x * RTX, j0 = rg.j0 + blockIdx.y * RTY;
    const double dt = step_dt(d.ctl);
    const double cv = d.cv;
    const int na = AX ? nx : ny, nc = AX ? ny : nx;
    const double wa = AX ? d.dx : d.dy, wc = AX ? d.dy : d.dx, origin = AX ? d.x0 : d.y0;
    const double* uh = AX ? d.uhx : d.uhy;
    const uint32_t pb = 5u * (uint32_t)w.pass;
    // (along, cross) -> region slots
    auto F = [&](int ia, int ic) { return AX ? (ia - i0 + 2) + (ic - j0) * FW : (ic - i0) + (ia - j0 + 2) * FW; };
    auto Cs = [&](int ia, int ic) { return AX ? (ia - i0 + 2) + (ic - j0) * CW : (ic - i0) + (ia - j0 + 2) * CW; };
    // face-mean displacements, make_axis_geom (remap.cpp:306-313)
    auto fd_at = [&](int ia, int ic) -> double {
        const int n0i = AX ? ia : ic, n0j = AX ? ic : ia;
        const int n1i = AX ? ia : ic + 1, n1j = AX ? ic + 1 : ia;
        if (!in(d.win_n, n0i, n0j) || !in(d.win_n, n1i, n1j)) return 0.0;
        return 0.5 * (uh[ix(d, n0i, n0j)] + uh[ix(d, n1i, n1j)]) * dt;
    };
    // ---- stage: face displacements and the cells' Work inputs
    for (int t = tid; t < NFR; t += RTX * RTY) {
        const int ia = AX ? i0 - 2 + t % FW : j0 - 2 + t / FW, ic = AX ? j0 + t / FW : i0 + t % FW;
        s_fd[t] = fd_at(ia, ic);
    }
    for (int t = tid; t < NCR; t += RTX * RTY) {
        const int i = (AX ? i0 - 2 : i0) + t % CW, j = (AX ? j0 : j0 - 2) + t / CW;
        if (!in(d.win_c, i, j)) continue;
        const int c = ix(d, i, j);
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            s_rho[a][t] = w.m[a][c];
            s_e[a][t] = w.e[a][c];
            s_k[a][t] = w.k[a][c];
        }
    }
    __syncthreads();
    // ---- cells: 1D Lagrangian volume, densities, centroid / width, interfaces
    // (remap.cpp:478-514; the collapsed scan covers [-G, n+G) both ways)
    for (int t = tid; t < NCR; t += RTX * RTY) {
        const int i = (AX ? i0 - 2 : i0) + t % CW, j = (AX ? j0 : j0 - 2) + t / CW;
        if (!in(d.win_c, i, j)) continue;
        const int ia = AX ? i : j, ic = AX ? j : i;
        if (ia + 1 > (AX ? d.win_n.i1 - 1 : d.win_n.j1 - 1)) continue;
        const double dl = s_fd[F(ia, ic)], dr = s_fd[F(ia + 1, ic)];
        const double v = cv + (dr - dl) * wc;
        if (v <= 0.0 && ia >= -G && ia < na + G && ic >= -G && ic < nc + G)
            raise(d.ctl, ekey(PH_AD_COLLAPSED + pb, ic, ia, 2 * AX));
        s_vl[t] = v;
        s_xl[t] = origin + (ia + 0.5) * wa + 0.5 * (dl + dr);
        s_wl[t] = wa + (dr - dl);
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            const double ka = s_k[a][t];
            s_rho[a][t] = ka > 0.0 ? s_rho[a][t] / (ka * v) : 0.0;
        }
        if (NM == 2) {
            const double k0 = s_k[0][t];
            double dd = 0.0;
            if (is_mixed(k0)) {
                const double cx = d.x0 + (i + 0.5) * d.dx, cy = d.y0 + (j + 0.5) * d.dy;
                const int g = ix(d, i, j);
                if (AX)
                    dd = place_interface(k0, w.nrx[g], w.nry[g], cx - 0.5 * d.dx + dl, cy - 0.5 * d.dy,
                                         cx + 0.5 * d.dx + dr, cy + 0.5 * d.dy);
                else
                    dd = place_interface(k0, w.nrx[g], w.nry[g], cx - 0.5 * d.dx, cy - 0.5 * d.dy + dl,
                                         cx + 0.5 * d.dx, cy + 0.5 * d.dy + dr);
            }
            s_ifd[t] = dd;
        }
    }
    // the scan's cross-axis ghost rows (columns) lie outside every tile: the
    // tiles on the cross boundary check them from u_half's ghost layers
    {
        const int c0 = AX ? j0 : i0, c1 = AX ? min(j0 + RTY, rg.j1) : min(i0 + RTX, rg.i1);
        const int a0 = AX ? i0 - 2 : j0 - 2, a1 = AX ? i0 + RTX + 2 : j0 + RTY + 2;
        const bool lo = c0 == 0, hi = c1 == nc;
        if (lo || hi) {
            const int nrow = (lo ? 2 : 0) + (hi ? 2 : 0);
            for (int t = tid; t < nrow * (a1 - a0); t += RTX * RTY) {
                const int r = t / (a1 - a0), ia = a0 + t % (a1 - a0);
                const int ic = (lo && r < 2) ? -2 + r : nc + (r - (lo ? 2 : 0));
                if (ia < -G || ia >= na + G) continue;
                const double v = cv + (fd_at(ia + 1, ic) - fd_at(ia, ic)) * wc;
                if (v <= 0.0) raise(d.ctl, ekey(PH_AD_COLLAPSED + pb, ic, ia, 2 * AX));
            }
        }
    }
    __syncthreads();
    // ---- the tile's faces along AX (remap.cpp:526-577)
    for (int t = tid; t < NIF; t += RTX * RTY) {
        const int ia = AX ? i0 + t % (RTX + 1) : j0 + t / RTX, ic = AX ? j0 + t / (RTX + 1) : i0 + t % RTX;
        double dm[2] = {0.0, 0.0}, dme[2] = {0.0, 0.0}, dva[2] = {0.0, 0.0};
        const bool valid = AX ? (ia <= min(nx, rg.i1) && ic < min(ny, rg.j1)) : (ic < min(nx, rg.i1) && ia <= min(ny, rg.j1));
        if (valid) {
            const double fdv = s_fd[F(ia, ic)];
            const double dvol = fdv * wc;
            double dmtot = 0.0;
            if (dvol != 0.0) {
                if (fabs(dvol) > kCflFrac * cv) raise(d.ctl, ekey(PH_AD_FACE + pb, ic, ia, 2 * AX));
                const int ia_d = dvol > 0.0 ? ia - 1 : ia;
                const double sgn = dvol > 0.0 ? 1.0 : -1.0;
                const int cdi = AX ? ia_d : ic, cdj = AX ? ic : ia_d;
                const int cd = Cs(ia_d, ic);
                // face_flux_box (remap.cpp:325-334) and split_flux (:254-268)
                double blox, bloy, bhix, bhiy;
                if (AX) {
                    const double xf = d.x0 + ia * d.dx;
                    blox = rmin(xf, xf + fdv);
                    bloy = d.y0 + ic * d.dy;
                    bhix = rmax(xf, xf + fdv);
                    bhiy = d.y0 + (ic + 1) * d.dy;
                } else {
                    const double yf = d.y0 + ia * d.dy;
                    blox = d.x0 + ic * d.dx;
                    bloy = rmin(yf, yf + fdv);
                    bhix = d.x0 + (ic + 1) * d.dx;
                    bhiy = rmax(yf, yf + fdv);
                }
                dva[0] = dvol;
                if (NM == 2) {
                    const double k0 = s_k[0][cd];
                    if (is_mixed(k0)) {
                        const int g = ix(d, cdi, cdj);
                        const double nxv = w.nrx[g], nyv = w.nry[g], dd = s_ifd[cd];
                        const double dl = s_fd[F(ia_d, ic)], dr = s_fd[F(ia_d + 1, ic)];
                        const double cx = d.x0 + (cdi + 0.5) * d.dx, cy = d.y0 + (cdj + 0.5) * d.dy;
                        const double lox = AX ? cx - 0.5 * d.dx + dl : cx - 0.5 * d.dx;
                        const double loy = AX ? cy - 0.5 * d.dy : cy - 0.5 * d.dy + dl;
                        const double hix = AX ? cx + 0.5 * d.dx + dr : cx + 0.5 * d.dx;
                        const double hiy = AX ? cy + 0.5 * d.dy : cy + 0.5 * d.dy + dr;
                        const double rcx = 0.5 * (lox + hix), rcy = 0.5 * (loy + hiy);
                        const double bcx = 0.5 * (blox + bhix), bcy = 0.5 * (bloy + bhiy);
                        const double bw = bhix - blox, bh = bhiy - bloy;
                        const double area = bw * bh;
                        double f0;
                        if (!(area > 0.0)) {
                            const double sd = (nxv * (bcx - rcx) + nyv * (bcy - rcy)) - dd;
                            f0 = sd <= 0.0 ? 1.0 : 0.0;
                        } else {
                            const double dbox = dd - (nxv * (bcx - rcx) + nyv * (bcy - rcy));
                            f0 = clipped_fraction(bw, bh, nxv, nyv, dbox);
                        }
                        dva[0] = f0 * dvol;
                        dva[1] = dvol - dva[0];
                    } else if (k0 < 0.5) {
                        dva[0] = 0.0;
                        dva[1] = dvol;
                    }
                }
                bool bad = false;
                const int cm = Cs(ia_d - 1, ic), cp = Cs(ia_d + 1, ic);
#pragma unroll
                for (int a = 0; a < NM; ++a) {
                    if (dva[a] == 0.0) continue;
                    int ord = d.face_order;
                    if (ord == 2 && NM == 2 && d.degrade &&
                        (s_k[a][cm] < 1.0 - kPureTol || s_k[a][cd] < 1.0 - kPureTol || s_k[a][cp] < 1.0 - kPureTol))
                        ord = 1;
                    double rf, ef;
                    if (ord <= 1) {
                        rf = s_rho[a][cd];
                        ef = s_e[a][cd];
                    } else {
                        rf = face_value2(s_rho[a][cm], s_rho[a][cd], s_rho[a][cp], s_xl[cm], s_xl[cd], s_xl[cp], sgn,
                                         s_wl[cd], fdv, bad);
                        ef = face_value2(s_e[a][cm], s_e[a][cd], s_e[a][cp], s_xl[cm], s_xl[cd], s_xl[cp], sgn,
                                         s_wl[cd], fdv, bad);
                    }
                    dm[a] = rf * dva[a];
                    dme[a] = rf * ef * dva[a];
                    dmtot += dm[a];
                }
                if (bad) raise(d.ctl, ekey(PH_AD_FACE + pb, ic, ia, 2 * AX + 1));
            }
            const bool ownf = AX ? (ia < i0 + RTX || ia == min(nx, rg.i1)) : (ia < j0 + RTY || ia == min(ny, rg.j1));
            if (ownf) (AX ? d.dmx : d.dmy)[AX ? ix(d, ia, ic) : ix(d, ic, ia)] = dmtot;
        }
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            s_it[0][a][t] = dm[a];
            s_it[1][a][t] = dme[a];
            s_it[2][a][t] = dva[a];
        }
    }
    __syncthreads();
    // ---- gather (left face +, right face -, remap.cpp:830-838) and finalize
    const int tx = tid % RTX, ty = tid / RTX;
    const int i = i0 + tx, j = j0 + ty;
    if (!in(rg, i, j)) return;
    const int c = ix(d, i, j);
    const double vl = s_vl[Cs(AX ? i : j, AX ? j : i)];
    const int ql = AX ? tx + ty * (RTX + 1) : tx + ty * RTX, qr = AX ? ql + 1 : ql + RTX;
    double m[2], me[2], va[2];
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        const double m0 = w.m[a][c];
        double mm = m0, mme = w.me_from_e ? m0 * w.e[a][c] : w.me[a][c], vv = w.k[a][c] * vl;
        if (s_it[2][a][ql] != 0.0) {
            mm += s_it[0][a][ql];
            mme += s_it[1][a][ql];
            vv += s_it[2][a][ql];
        }
        if (s_it[2][a][qr] != 0.0) {
            mm += -s_it[0][a][qr];
            mme += -s_it[1][a][qr];
            vv += -s_it[2][a][qr];
        }
        m[a] = mm;
        me[a] = mme;
        va[a] = vv;
    }
    finalize_cell<NM>(d, rg, i, j, c, tx, own_cell(d, i, j), m, me, va, PH_AD_NEGMASS + pb);
}

// Run-loop step epilogue in ONE launch (it used to be three: the ghost
// layers of the new normals and u, the diagnostics fold, the commit): the
// first nghost blocks fill the ghost layers (assemble_state's fill_ghosts,
// remap.cpp:1084-1088), the next kDiagBlocks fold slices of the diagnostics
// partials (as k_diag_reduce), and the last block to finish folds the slices,
// commits the step (k_commit_finish) and, for a single domain, starts the
// next one (k_step_start: loop condition and dt from the wave speed k_post
// produced), so the next step's graph needs no head kernel.
__global__ void __launch_bounds__(256) k_tail(Dev d, FieldList cells, FieldList nodes, int nb1, int n0, int n1,
                                              int start_next) {
    pdl_enter();
    __shared__ int s_flag;
    __shared__ double sh[8 * DG_N];
    const int t = threadIdx.x;
    if (t == 0) s_flag = halted(d.ctl);
    __syncthreads();
    const bool halt = s_flag;
    const int b = blockIdx.x, ncomb = cells.n + nodes.n / 2;
    int op[DG_N];
#pragma unroll
    for (int k = 0; k < DG_N; ++k) op[k] = dg_op(k);
    const DiagScratch& r = d.dsc;
    if (b < nb1 * ncomb) {
        if (!halt) {
            const int comb = b / nb1, tt = (b % nb1) * 256 + t;
            if (comb < cells.n)
                ghost_cells_at(d, cells, tt, comb);
            else
                ghost_nodes_at(d, nodes, tt, 2 * (comb - cells.n));
        }
    } else if (d.diag) {
        const int q = b - nb1 * ncomb, G = kDiagBlocks;
        double v[DG_N];
#pragma unroll
        for (int k = 0; k < DG_N; ++k) v[k] = dg_ident(op[k]);
        if (!halt) {
            const long long lo0 = (long long)n0 * q / G, hi0 = (long long)n0 * (q + 1) / G;
            const long long lo1 = (long long)n1 * q / G, hi1 = (long long)n1 * (q + 1) / G;
            for (long long e = lo0 + t; e < hi0; e += blockDim.x)
#pragma unroll
                for (int k = 0; k < DG_NCELL; ++k) v[k] = dg_comb(op[k], v[k], r.part[0][e * DG_NCELL + k]);
            for (long long e = lo1 + t; e < hi1; e += blockDim.x) {
                v[DG_PX] += r.part[1][e * 2];
                v[DG_PY] += r.part[1][e * 2 + 1];
            }
        }
        block_combine<DG_N>(v, op, sh);
        if (t == 0)
#pragma unroll
            for (int k = 0; k < DG_N; ++k) r.lvl2[q * DG_N + k] = v[k];
    }
    __syncthreads();
    if (t == 0) {
        __threadfence();
        s_flag = atomicAdd(r.tick, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_flag) return;
    if (d.diag && !halted(d.ctl)) {
        double v[DG_N];
#pragma unroll
        for (int k = 0; k < DG_N; ++k) v[k] = dg_ident(op[k]);
        for (int q = t; q < kDiagBlocks; q += blockDim.x)
#pragma unroll
            for (int k = 0; k < DG_N; ++k) v[k] = dg_comb(op[k], v[k], __ldcg(&r.lvl2[q * DG_N + k]));
        block_combine<DG_N>(v, op, sh);
        if (t == 0)
#pragma unroll
            for (int k = 0; k < DG_N; ++k) d.ctl->dg[k] = v[k];
    }
    if (t == 0) {
        __threadfence();
        *r.tick = 0u;
        commit_finish_body(d.ctl);
        if (start_next) step_start_body(d.ctl, d.dx, d.dy);
    }
}

// AD dual faces of one pass (dual_face_pass along AX, remap.cpp:408-442); the
// Dev's u_lag planes are the pass's Work velocities
template <int AX>
__global__ void __launch_bounds__(128, 8) k_ad_dual(Dev d, int pass) {
    pdl_enter();
    if (halted(d.ctl)) return;
    int i, j;
    tid2(i, j, d.r_dual.i0, d.r_dual.j0);
    const int iend = d.per_x ? d.nx - 1 : d.nx, jend = d.per_y ? d.ny - 1 : d.ny;
    if (!in(d.r_dual, i, j) || i < 0 || j < 0 || i > iend || j > jend) return;
    double mx, my;
    const bool on = dual_face_val<AX>(d, i, j, mx, my, PH_AD_GRAD_DUAL + 5u * (uint32_t)pass);
    const int s = ix(d, i, j);
    (AX ? d.dfx_x : d.dfy_x)[s] = mx;
    (AX ? d.dfx_y : d.dfy_y)[s] = my;
    d.dflag[AX ? 0 : 1][s] = on;
}

// AD MomAcc gather (one axis, face-loop order incl. the periodic seam) and
// apply_dual_update (remap.cpp:444-464) with mcell_lag = the pass's input mcell
template <int AX>
__device__ __forceinline__ void ad_node_at(const Dev& d, const AdIO& w, int i, int j, double& px, double& py) {
    const int nx = d.nx, ny = d.ny;
    if (!in(d.r_node, i, j) || i < 0 || j < 0 || i > nx || j > ny) return;
    const int iend = d.per_x ? nx - 1 : nx, jend = d.per_y ? ny - 1 : ny;
    const int si = (d.per_x && i == nx) ? 0 : i, sj = (d.per_y && j == ny) ? 0 : j;
    const int s = ix(d, si, sj);
    double ax = 0.0, ay = 0.0;
    {  // face ia joins nodes (ia-1, ia): + to node ia, - to the node ia-1 wraps to
        const int n = AX ? nx : ny;
        const int per = AX ? d.per_x : d.per_y;
        const int hi = AX ? iend : jend, lo = per ? 0 : 1;
        const int along = AX ? si : sj, cross = AX ? sj : si;
        const double* fx_ = AX ? d.dfx_x : d.dfy_x;
        const double* fy_ = AX ? d.dfx_y : d.dfy_y;
        const uint8_t* fl = d.dflag[AX ? 0 : 1];
        auto at = [&](int a) { return AX ? ix(d, a, cross) : ix(d, cross, a); };
        int am = along + 1;
        if (per && am == n) am = 0;
        const bool ap = along >= lo && along <= hi && fl[at(along)];
        const bool an = am >= lo && am <= hi && fl[at(am)];
        const bool minus_first = an && am < along;
        if (minus_first) {
            ax += -fx_[at(am)];
            ay += -fy_[at(am)];
        }
        if (ap) {
            ax += fx_[at(along)];
            ay += fy_[at(along)];
        }
        if (an && !minus_first) {
            ax += -fx_[at(am)];
            ay += -fy_[at(am)];
        }
    }
    auto ml = [&](int ci, int cj) {
        const int c = ix(d, ci, cj);
        if (w.mcell) return w.mcell[c];
        double mc = 0.0;  // make_work's mcell (remap.cpp:133-138)
        for (int a = 0; a < d.nmat; ++a) mc += w.m[a][c];
        return mc;
    };
    const double mp_lag = 0.25 * (ml(si - 1, sj - 1) + ml(si, sj - 1) + ml(si - 1, sj) + ml(si, sj));
    const double mp_new =
        0.25 * (d.mcell[ix(d, si - 1, sj - 1)] + d.mcell[ix(d, si, sj - 1)] + d.mcell[ix(d, si - 1, sj)] + d.mcell[s]);
    if (mp_new <= 0.0 && si == i && sj == j && own_node(d, i, j))
        raise(d.ctl, ekey(PH_AD_NODAL + 5u * (uint32_t)w.pass, j, i, 0));
    const double inv = 1.0 / mp_new;
    const int o = ix(d, i, j);
    double ux = inv * (mp_lag * w.ux[s] + ax), uy = inv * (mp_lag * w.uy[s] + ay);
    if (!d.per_x && (i == 0 || i == nx)) ux = 0.0;  // fill_ghost_nodes wall zeroing (remap.cpp:462)
    if (!d.per_y && (j == 0 || j == ny)) uy = 0.0;
    d.nux[o] = ux;
    d.nuy[o] = uy;
    d.unrm[o] = sqrt(ux * ux + uy * uy);
    if (d.scan_nodes && w.pass == 1 && own_node(d, i, j) && (!isfinite(ux) | !isfinite(uy)))
        raise(d.ctl, ekey(PH_NAN_NODE, j, i, 0));  // nan_scan on the final u
    if (d.diag && w.pass == 1 && i <= iend && j <= jend && own_node(d, i, j)) {  // state.cpp:154-158
        px = mp_new * ux;
        py = mp_new * uy;
    }
}

template <int AX>
__global__ void k_ad_node(Dev d, AdIO w) {
    pdl_enter();
    if (halted(d.ctl)) return;  // one load per warp: warp-uniform
    int i, j;
    tid2(i, j, d.r_node.i0, d.r_node.j0);
    double px = 0.0, py = 0.0;
    ad_node_at<AX>(d, w, i, j, px, py);
    if (w.pass == 1) node_momentum(d, px, py);
}

// refresh_normals_impl after AD pass 0 (remap.cpp:102-114): youngs normals of
// the pass's new fractions where mixed, else the pass's input normals
__global__ void k_ad_normals(Dev d, AdIO w) {
    pdl_enter();
    if (halted(d.ctl)) return;
    int i, j;
    tid2(i, j, d.r_nrm.i0, d.r_nrm.j0);  // (a block: the cells whose 3x3 fractions are exact after the pass)
    if (!in(d.r_nrm, i, j)) return;
    const int c = ix(d, i, j);
    double nrx = w.nrx[c], nry = w.nry[c];
    if (is_mixed(d.nk[0][c])) {
        auto K = [&](int ii, int jj) { return d.nk[1][ix(d, ii, jj)]; };
        auto col = [&](int ii) { return K(ii, j - 1) + 2.0 * K(ii, j) + K(ii, j + 1); };
        auto row = [&](int jj) { return K(i - 1, jj) + 2.0 * K(i, jj) + K(i + 1, jj); };
        const double gx = div_dx(d, col(i + 1) - col(i - 1), 8.0);
        const double gy = div_dy(d, row(j + 1) - row(j - 1), 8.0);
        const double g = sqrt(gx * gx + gy * gy);
        if (!(g < 1e-300)) {
            nrx = gx / g;
            nry = gy / g;
        }
    }
    d.nnrx[c] = nrx;
    d.nnry[c] = nry;
}

// AoS <-> SoA staging for Vec2 fields (reference layout pitch W = n1 + 2G).
__global__ void k_deinterleave(const double* src, double* x, double* y, int W, int H, int P) {
    pdl_enter();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= W * H) return;
    const int r = t / W, col = t % W;
    x[(size_t)r * P + col] = src[2 * (size_t)t];
    y[(size_t)r * P + col] = src[2 * (size_t)t + 1];
}
__global__ void k_interleave(double* dst, const double* x, const double* y, int W, int H, int P) {
    pdl_enter();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= W * H) return;
    const int r = t / W, col = t % W;
    dst[2 * (size_t)t] = x[(size_t)r * P + col];
    dst[2 * (size_t)t + 1] = y[(size_t)r * P + col];
}

// ---------------------------------------------------------------------------
// launch wrappers
// ---------------------------------------------------------------------------
static std::atomic<long long> g_launches{0};
long long launch_count() { return g_launches.load(); }
void add_launches(long long n) { g_launches += n; }
// Launch with the programmatic-stream-serialization attribute (PDL): the
// kernel may start while its predecessor drains and waits in pdl_enter().
template <typename... KArgs, typename... Args>
static void pdl(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
    ++g_launches;
}

static dim3 blk2() { return dim3(32, 4); }
static dim3 grid_rect(int w, int h) {
    const dim3 b = blk2();
    return dim3((unsigned)((w + b.x - 1) / b.x), (unsigned)((h + b.y - 1) / b.y));
}
static unsigned nblk(long long n, int b) { return (unsigned)((n + b - 1) / b); }
static int ext(int a, int b) { return b > a ? b - a : 1; }
static dim3 grid_of(const Rng& r) { return grid_rect(ext(r.i0, r.i1), ext(r.j0, r.j1)); }
static dim3 tiles_of(const Rng& r, int tx, int ty) {
    return dim3((unsigned)((ext(r.i0, r.i1) + tx - 1) / tx), (unsigned)((ext(r.j0, r.j1) + ty - 1) / ty));
}

void launch_begin(Ctl* c, int mode, double dt, cudaStream_t s) { k_begin<<<1, 1, 0, s>>>(c, mode, dt); }

void launch_cfl(const Dev& d, int run_loop, cudaStream_t s) {
    // grid-stride: a few blocks per SM, one atomic per block
    const long long ncell = (long long)d.nx * d.ny;
    unsigned nb = nblk(ncell, 256);
    if (nb > 148u * 8u) nb = 148u * 8u;
    if (d.nmat == 3)
        { k_cfl<3><<<nb, 256, 0, s>>>(d, 0); ++g_launches; }
    else if (d.nmat == 2)
        { k_cfl<2><<<nb, 256, 0, s>>>(d, 0); ++g_launches; }
    else
        { k_cfl<1><<<nb, 256, 0, s>>>(d, 0); ++g_launches; }
    { k_cfl_final<<<1, 1, 0, s>>>(d.ctl, d.dx, d.dy, run_loop); ++g_launches; }
}

static long long ghost_threads(const Dev& d) {
    const long long nc = 2LL * G * (d.nx + 2 * G) + 2LL * G * d.ny;
    const long long nn = 2LL * G * (d.nx + 1 + 2 * G) + 2LL * G * (d.ny + 1) + 2LL * (d.ny + 1) + 2LL * (d.nx + 1);
    const long long nf = (d.nx > d.ny ? d.nx : d.ny) + 2;
    long long m = nc > nn ? nc : nn;
    return m > nf ? m : nf;
}
void launch_ghost_multi(const Dev& d, const FieldList& cells, const FieldList& nodes, int flux, int respect_halt,
                        cudaStream_t s) {
    int nz = cells.n > (nodes.n + 1) / 2 ? cells.n : (nodes.n + 1) / 2;
    if (nz < 1) nz = 1;
    const dim3 g(nblk(ghost_threads(d), 256), flux ? 3 : 2, nz);
    pdl(k_ghost_multi, g, dim3(256), 0, s, d, cells, nodes, flux, respect_halt);
}
void launch_ghost_cells(const Dev& d, const FieldList& fl, cudaStream_t s) {
    FieldList none{};
    launch_ghost_multi(d, fl, none, 0, fl.respect_halt, s);
}
void launch_ghost_nodes(const Dev& d, const FieldList& fl, cudaStream_t s) {
    FieldList none{};
    launch_ghost_multi(d, none, fl, 0, fl.respect_halt, s);
}

void launch_sync(const Dev& d, int next, int respect_halt, cudaStream_t s) {
    const dim3 g = grid_of(d.win_c);
    if (d.nmat == 3)
        { k_sync<3><<<g, blk2(), 0, s>>>(d, next, respect_halt); ++g_launches; }
    else if (d.nmat == 2)
        { k_sync<2><<<g, blk2(), 0, s>>>(d, next, respect_halt); ++g_launches; }
    else
        { k_sync<1><<<g, blk2(), 0, s>>>(d, next, respect_halt); ++g_launches; }
}

void launch_lagrange(const Dev& d, int write_vol_lag, cudaStream_t s) { launch_lagrange_mode(d, write_vol_lag, 0, s); }

void launch_lagrange_mode(const Dev& d, int write_vol_lag, int mode, cudaStream_t s) {
    const dim3 gc = grid_of(d.r_lagc);
    const dim3 gl = tiles_of(d.r_lagn, LTX, LTY);
    FieldList fl{};
    fl.respect_halt = 1;
    if (mode != 2) {
        if (d.nmat == 3)
            { k_lag_cells<3><<<gc, blk2(), 0, s>>>(d); ++g_launches; }
        else if (d.nmat == 2)
            { k_lag_cells<2><<<gc, blk2(), 0, s>>>(d); ++g_launches; }
        else
            { k_lag_cells<1><<<gc, blk2(), 0, s>>>(d); ++g_launches; }
        fl.n = 2;  // Q (lagrange.cpp:75) and p_mix_half (:132) ghosts
        fl.f[0] = d.q;
        fl.f[1] = d.pmh;
        if (mode == 1) {  // HalfStepState returns p_half with its ghosts too (:133)
            for (int a = 0; a < d.nmat; ++a) fl.f[fl.n++] = d.ph[a];
        }
        launch_ghost_cells(d, fl, s);
    }
    if (d.nmat == 3)
        { k_lag_nodes<3><<<gl, LTX * LTY, 0, s>>>(d, write_vol_lag, mode); ++g_launches; }
    else if (d.nmat == 2)
        { k_lag_nodes<2><<<gl, LTX * LTY, 0, s>>>(d, write_vol_lag, mode); ++g_launches; }
    else
        { k_lag_nodes<1><<<gl, LTX * LTY, 0, s>>>(d, write_vol_lag, mode); ++g_launches; }
    FieldList fn{};
    fn.n = mode == 2 ? 2 : 4;
    fn.f[0] = mode == 2 ? d.ulx : d.uhx;
    fn.f[1] = mode == 2 ? d.uly : d.uhy;
    fn.f[2] = d.ulx;
    fn.f[3] = d.uly;
    fl.n = mode == 1 ? 0 : d.nmat;
    for (int a = 0; a < d.nmat; ++a) fl.f[a] = d.el[a];
    launch_ghost_multi(d, fl, fn, 0, 1, s);
}

void remap_init() {
    static bool done = false;
    if (done) return;
    cudaFuncSetAttribute(k_remap_tile<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)remap_smem_bytes<1>());
    cudaFuncSetAttribute(k_remap_tile<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)remap_smem_bytes<2>());
    cudaFuncSetAttribute(k_remap_tile<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)remap_smem_bytes<3>());
    cudaFuncSetAttribute(k_remap_tile<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)remap_smem_bytes<1>());
    cudaFuncSetAttribute(k_remap_tile<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)remap_smem_bytes<2>());
    cudaFuncSetAttribute(k_remap_tile<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)remap_smem_bytes<3>());
    cudaFuncSetAttribute(k_remap_tile<1, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)remap_smem_bytes<1, true>());
    cudaFuncSetAttribute(k_remap_tile<2, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)remap_smem_bytes<2, true>());
    cudaFuncSetAttribute(k_remap_tile<3, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)remap_smem_bytes<3, true>());
    cudaFuncSetAttribute(k_remap_tile<2, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)remap_smem_bytes<2>());
    cudaFuncSetAttribute(k_remap_tile<1, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)remap_smem_bytes<1>());
    done = true;
}

// k_post (sync_derived, normals, and in the run loop nan_scan + next cfl) and
// the ghost layers of the new u and normals (assemble_state's fill_ghosts).
void post_and_ghosts(const Dev& d, int run_loop, cudaStream_t s) {
    launch_post(d, run_loop, s);
    if (!run_loop) launch_post_ghosts(d, s);  // the run loop's k_tail fills them
}

void launch_post(const Dev& d, int run_loop, cudaStream_t s) {
    const dim3 gp = tiles_of(d.r_sync, 32, 8);
    if (d.nmat == 3)
        pdl(k_post<3>, gp, dim3(32, 8), 0, s, d, run_loop);
    else if (d.nmat == 2)
        pdl(k_post<2>, gp, dim3(32, 8), 0, s, d, run_loop);
    else
        pdl(k_post<1>, gp, dim3(32, 8), 0, s, d, run_loop);
}

// run-loop epilogue (k_tail): post ghosts + diagnostics fold + commit (+ next start)
void launch_tail(const Dev& d, int start_next, cudaStream_t s) {
    FieldList fg{};
    fg.n = 2;
    fg.f[0] = d.nnrx;
    fg.f[1] = d.nnry;
    FieldList fu{};
    fu.n = 2;
    fu.f[0] = d.nux;
    fu.f[1] = d.nuy;
    const int nb1 = (int)nblk(ghost_threads(d), 256);
    const int nb = nb1 * 3 + (d.diag ? kDiagBlocks : 0);
    pdl(k_tail, dim3(nb), dim3(256), 0, s, d, fg, fu, nb1, (int)diag_partials(d, 0), (int)diag_partials(d, 1),
        start_next);
}

long long diag_partials(const Dev& d, int which) {  // block counts of k_post / the node grids
    if (which == 0) {  // one partial per k_post block
        const dim3 g = tiles_of(d.r_sync, 32, 8);
        return (long long)g.x * g.y;
    }
    const dim3 g = grid_of(d.r_node), b = blk2();  // one per node-update warp
    return (long long)g.x * g.y * (b.x * b.y / 32);
}

void launch_post_ghosts(const Dev& d, cudaStream_t s) {
    FieldList fg{};
    fg.n = 2;
    fg.f[0] = d.nnrx;
    fg.f[1] = d.nnry;
    FieldList fu{};
    fu.n = 2;
    fu.f[0] = d.nux;
    fu.f[1] = d.nuy;
    launch_ghost_multi(d, fg, fu, 0, 1, s);
}

void launch_remap(const Dev& d, cudaStream_t s) { launch_remap_core(d, s); post_and_ghosts(d, 0, s); }

// run-loop Lagrangian phase: the fused kernel + ghost layers of u_half, u_lag, e_lag
void launch_lagrange_run(const Dev& d, cudaStream_t s) {
    launch_lag_fused(d, s);
    launch_lag_ghosts(d, s);
}

void launch_lag_fused(const Dev& d, cudaStream_t s) {
    if (d.nmat == 3)
        pdl(k_lag_fused<3>, tiles_of(d.r_lagn, LTX, H2D_FTY), dim3(H2D_LAG_NT), 0, s, d);
    else if (d.nmat == 2)
        pdl(k_lag_fused<2>, tiles_of(d.r_lagn, LTX, H2D_FTY), dim3(H2D_LAG_NT), 0, s, d);
    else
        pdl(k_lag_fused<1>, tiles_of(d.r_lagn, LTX, H2D_FTY), dim3(H2D_LAG_NT), 0, s, d);
}

void launch_lag_ghosts(const Dev& d, cudaStream_t s) {
    FieldList fn{};
    fn.n = 4;
    fn.f[0] = d.uhx;
    fn.f[1] = d.uhy;
    fn.f[2] = d.ulx;
    fn.f[3] = d.uly;
    FieldList fl{};
    fl.n = d.nmat;
    for (int a = 0; a < d.nmat; ++a) fl.f[a] = d.el[a];
    launch_ghost_multi(d, fl, fn, 0, 1, s);
}

void launch_remap_core(const Dev& d, cudaStream_t s) {
    if (!d.remap_velocity) { k_copy_u<<<grid_of(d.win_n), blk2(), 0, s>>>(d); ++g_launches; }
    launch_remap_tile(d, s);
    launch_remap_slivers(d, s);
    launch_remap_dual(d, s);
}

template <int NM>
__global__ void __launch_bounds__(RTX * RTY) k_tile_class(Dev d) {
    pdl_enter();
    const int tid = threadIdx.x;
    const Rng rg = d.r_gath;
    const int i0 = rg.i0 - tile_shift(d) + blockIdx.x * RTX, j0 = rg.j0 + blockIdx.y * RTY;
    const int x0 = i0 - G + d.H - d.oi, y0 = j0 - G + d.H - d.oj;  // plane column / row of the region origin
    const int R = d.fsz / d.P;
    unsigned mk = 0u;
    for (int t = tid; t < RCW * RCH; t += RTX * RTY) {
        const int x = x0 + t % RCW, y = y0 + t / RCW;
        double k[NM], m[NM];
        if (x < 0 || x >= d.P || y < 0 || y >= R) {  // zero-filled by the copy: absent
#pragma unroll
            for (int a = 0; a < NM; ++a) k[a] = m[a] = 0.0;
        } else {
            const int q = y * d.P + x;
#pragma unroll
            for (int a = 0; a < NM; ++a) {
                k[a] = d.k[a][q];
                m[a] = d.m[a][q];
            }
        }
        mk |= cell_cls_mask<NM>(k, m);
    }
    __shared__ unsigned s_mk;
    if (tid == 0) s_mk = 0u;
    __syncthreads();
    mk = __reduce_or_sync(0xffffffffu, mk);
    if ((tid & 31) == 0) atomicOr(&s_mk, mk);
    __syncthreads();
    if (tid == 0) d.tcls[blockIdx.y * gridDim.x + blockIdx.x] = (uint8_t)cls_of_mask<NM>(s_mk);
}

// Run loop, single domain: the cell masks come from k_post of the step
// before, which holds the new State's k and m in registers anyway (one OR per
// 32 x 8 post block, Dev::pcls; the first step of a call gets them from
// k_cls_flags): a tile's class is the OR over the post blocks that cover its
// staged region (a superset of the region: a tile next to another material is
// classified a little more cautiously, never less), one thread per tile
template <int NM>
__global__ void k_tile_class_post(Dev d, int ntx, int nty) {
    pdl_enter();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntx * nty) return;
    const int bx = t % ntx, by = t / ntx;
    const Rng rg = d.r_gath, rs = d.r_sync;
    const int i0 = rg.i0 - tile_shift(d) + bx * RTX, j0 = rg.j0 + by * RTY;
    // region cells [i0 - 2, i0 + RTX + 2) x [j0 - 2, j0 + RTY + 2), clipped to the stored cells (r_sync)
    const int ilo = max(i0 - G, rs.i0), ihi = min(i0 + RTX + G, rs.i1) - 1;
    const int jlo = max(j0 - G, rs.j0), jhi = min(j0 + RTY + G, rs.j1) - 1;
    unsigned mk = 0u;
    for (int q = (jlo - rs.j0) / 8; q <= (jhi - rs.j0) / 8; ++q)
        for (int p = (ilo - rs.i0) / 32; p <= (ihi - rs.i0) / 32; ++p) mk |= d.pcls[q * d.pcls_nx + p];
    d.tcls[t] = (uint8_t)cls_of_mask<NM>(mk);
}

// the cell masks of the CURRENT State per post block (the first step of a call)
template <int NM>
__global__ void __launch_bounds__(256) k_cls_flags(Dev d) {
    __shared__ unsigned s_mk;
    const int tl = threadIdx.y * blockDim.x + threadIdx.x;
    if (tl == 0) s_mk = 0u;
    __syncthreads();
    int i, j;
    tid2(i, j, d.r_sync.i0, d.r_sync.j0);
    unsigned mk = 0u;
    if (in(d.r_sync, i, j)) {
        const int c = ix(d, i, j);
        double k[NM], m[NM];
#pragma unroll
        for (int a = 0; a < NM; ++a) {
            k[a] = d.k[a][c];
            m[a] = d.m[a][c];
        }
        mk = cell_cls_mask<NM>(k, m);
    }
    mk = __reduce_or_sync(0xffffffffu, mk);
    if ((tl & 31) == 0 && mk) atomicOr(&s_mk, mk);
    __syncthreads();
    if (tl == 0) d.pcls[blockIdx.y * gridDim.x + blockIdx.x] = (uint16_t)s_mk;
}

// the fused flux tile kernel alone (timed separately by h2d_step_timed)
int remap_uses_classes(int nmat) { return (nmat == 3 && H2D_RT_MAP3) || (nmat == 2 && H2D_RT_MAP2); }
int remap_tile_w() { return RTX; }
int remap_tile_h() { return RTY; }
int tma_node_box_w() { return RNW; }
int tma_node_box_h() { return RNH; }
int tma_cell_box_w() { return RCW; }
int tma_cell_box_h() { return RCH; }

// tile classes: from the post blocks' masks in the run loop of a single
// domain (Dev::cls_post), else from the State itself
static void launch_tile_class(const Dev& d, dim3 gft, cudaStream_t s) {
    if (d.cls_post && d.pcls) {
        const int n = (int)(gft.x * gft.y);
        if (d.nmat == 3)
            pdl(k_tile_class_post<3>, dim3(nblk(n, 256)), dim3(256), 0, s, d, (int)gft.x, (int)gft.y);
        else
            pdl(k_tile_class_post<2>, dim3(nblk(n, 256)), dim3(256), 0, s, d, (int)gft.x, (int)gft.y);
    } else if (d.nmat == 3) {
        pdl(k_tile_class<3>, gft, dim3(RTX * RTY), 0, s, d);
    } else {
        pdl(k_tile_class<2>, gft, dim3(RTX * RTY), 0, s, d);
    }
}

// the post blocks' masks of the current State (start of a run; later steps get them from k_post)
void launch_cls_flags(const Dev& d, cudaStream_t s) {
    if (!d.pcls || d.nmat < 2) return;
    const dim3 gp = tiles_of(d.r_sync, 32, 8);
    if (d.nmat == 3)
        { k_cls_flags<3><<<gp, dim3(32, 8), 0, s>>>(d); ++g_launches; }
    else
        { k_cls_flags<2><<<gp, dim3(32, 8), 0, s>>>(d); ++g_launches; }
}

void launch_remap_tile(const Dev& d, cudaStream_t s) {
    remap_init();
    Rng rt = d.r_gath;
    rt.i0 -= tile_shift(d);
    const dim3 gft = tiles_of(rt, RTX, RTY);
    const bool xc = d.corner != CS_UPWIND && d.corner != CS_LINEARDIAG;  // the extended corner schemes
    if (d.direct) {  // the Direct engine (remap.cpp:593-724)
        if (d.nmat == 3)
            pdl(k_remap_tile<3, false, true>, gft, dim3(RTX * RTY), remap_smem_bytes<3, true>(), s, d, *d.tma);
        else if (d.nmat == 2)
            pdl(k_remap_tile<2, false, true>, gft, dim3(RTX * RTY), remap_smem_bytes<2, true>(), s, d, *d.tma);
        else
            pdl(k_remap_tile<1, false, true>, gft, dim3(RTX * RTY), remap_smem_bytes<1, true>(), s, d, *d.tma);
        return;
    }
    if (d.nmat == 3)
        if (xc) {
            Dev dx = d;
            dx.tcls = nullptr;
            pdl(k_remap_tile<3, true>, gft, dim3(RTX * RTY), remap_smem_bytes<3>(), s, dx, *d.tma);
        } else if (d.tcls && H2D_RT_MAP3) {  // per-tile: two-slot kernel where a material is absent
            launch_tile_class(d, gft, s);
            if (H2D_RT_MAP31)
                pdl(k_remap_tile<1, false, false, true>, gft, dim3(RTX * RTY), remap_smem_bytes<1>(), s, d, *d.tma);
            if (H2D_RT_MAP32)
                pdl(k_remap_tile<2, false, false, true>, gft, dim3(RTX * RTY), remap_smem_bytes<2>(), s, d, *d.tma);
            pdl(k_remap_tile<3>, gft, dim3(RTX * RTY), remap_smem_bytes<3>(), s, d, *d.tma);
        } else {
            Dev dx = d;
            dx.tcls = nullptr;
            pdl(k_remap_tile<3>, gft, dim3(RTX * RTY), remap_smem_bytes<3>(), s, dx, *d.tma);
        }
    else if (d.nmat == 2)
        if (xc) {
            Dev dx = d;
            dx.tcls = nullptr;
            pdl(k_remap_tile<2, true>, gft, dim3(RTX * RTY), remap_smem_bytes<2>(), s, dx, *d.tma);
        } else if (d.tcls && H2D_RT_MAP2) {  // per-tile: one-material kernel where a material is absent
            launch_tile_class(d, gft, s);
            pdl(k_remap_tile<1, false, false, true>, gft, dim3(RTX * RTY), remap_smem_bytes<1>(), s, d, *d.tma);
            pdl(k_remap_tile<2>, gft, dim3(RTX * RTY), remap_smem_bytes<2>(), s, d, *d.tma);
        } else {
            Dev dx = d;
            dx.tcls = nullptr;
            pdl(k_remap_tile<2>, gft, dim3(RTX * RTY), remap_smem_bytes<2>(), s, dx, *d.tma);
        }
    else
        xc ? pdl(k_remap_tile<1, true>, gft, dim3(RTX * RTY), remap_smem_bytes<1>(), s, d, *d.tma)
           : pdl(k_remap_tile<1>, gft, dim3(RTX * RTY), remap_smem_bytes<1>(), s, d, *d.tma);
}

// slivers + finalize_cells ghost fill + flux ghosts
// H2D_OPT_SLIVER_ENERGY (include/h2d.h; oracle sliver_energy_fix): after the
// sliver pass, a material with m > 0 and e < 0 hands m*e to the cell's
// largest-mass other material if the sum stays positive, else drops it; its
// e becomes 0 (materials in index order)
template <int NM>
__global__ void k_energy_fix(Dev d) {
    pdl_enter();
    if (halted(d.ctl)) return;
    int i, j;
    tid2(i, j, d.r_gath.i0, d.r_gath.j0);
    if (!in(d.r_gath, i, j)) return;
    const int c = ix(d, i, j);
#pragma unroll
    for (int a = 0; a < NM; ++a) {
        if (!(d.nm[a][c] > 0.0 && d.ne[a][c] < 0.0)) continue;
        int b = -1;
#pragma unroll
        for (int q = 0; q < NM; ++q)
            if (q != a && d.nm[q][c] > 0.0 && (b < 0 || d.nm[q][c] > d.nm[b][c])) b = q;
        if (b >= 0) {
            const double meb = d.me[b][c] + d.me[a][c];
            if (meb > 0.0) {
                d.me[b][c] = meb;
                d.ne[b][c] = meb / d.nm[b][c];
            }
        }
        d.me[a][c] = 0.0;
        d.ne[a][c] = 0.0;
    }
}

void launch_remap_slivers(const Dev& d, cudaStream_t s) {
    if (d.nmat == 3) {
        pdl(k_sliver_list<3>, dim3(1), dim3(SLB), 0, s, d);
        for (int r = 0; r < kSlRounds; ++r) pdl(k_sliver_round<3>, dim3(kSlGrid), dim3(256), 0, s, d, r);
        pdl(k_sliver_tail<3>, dim3(1), dim3(SLB), 0, s, d);
    } else if (d.nmat == 2) {
        pdl(k_sliver_list<2>, dim3(1), dim3(SLB), 0, s, d);
        for (int r = 0; r < kSlRounds; ++r) pdl(k_sliver_round<2>, dim3(kSlGrid), dim3(256), 0, s, d, r);
        pdl(k_sliver_tail<2>, dim3(1), dim3(SLB), 0, s, d);
    }
    if (d.opt_energy) {
        if (d.nmat == 3)
            pdl(k_energy_fix<3>, grid_of(d.r_gath), blk2(), 0, s, d);
        else if (d.nmat == 2)
            pdl(k_energy_fix<2>, grid_of(d.r_gath), blk2(), 0, s, d);
        else
            pdl(k_energy_fix<1>, grid_of(d.r_gath), blk2(), 0, s, d);
    }
    // finalize_cells ghost fill (remap.cpp:227-233) + face / corner flux ghosts
    FieldList fl{};
    int q = 0;
    for (int a = 0; a < d.nmat; ++a) {
        fl.f[q++] = d.nm[a];
        fl.f[q++] = d.me[a];
        fl.f[q++] = d.ne[a];
        fl.f[q++] = d.nk[a];
    }
    fl.f[q++] = d.mcell;
    fl.n = q;
    FieldList none{};
    launch_ghost_multi(d, fl, none, 1, 1, s);
}

// dual-mesh momentum remap (remap.cpp:993-1059)
void launch_remap_dual(const Dev& d, cudaStream_t s) {
    if (d.remap_velocity) {
        if (d.corner != CS_UPWIND && d.corner != CS_LINEARDIAG)
            pdl(k_dual_items<true>, grid_of(d.r_dual), blk2(), 0, s, d);
        else
            pdl(k_dual_items<false>, grid_of(d.r_dual), blk2(), 0, s, d);
        if (d.per_x || d.per_y)  // periodic seams reorder the node sums: sorted gather
            pdl(k_node_update, grid_of(d.r_node), blk2(), 0, s, d);
        else
            d.nmat == 3   ? pdl(k_node_update_walls<3>, grid_of(d.r_node), blk2(), 0, s, d)
            : d.nmat == 2 ? pdl(k_node_update_walls<2>, grid_of(d.r_node), blk2(), 0, s, d)
                          : pdl(k_node_update_walls<1>, grid_of(d.r_node), blk2(), 0, s, d);
    }
}

// One run-loop step. fused_start: the step's start (loop condition, dt) was
// done by the previous step's k_tail (single domain), and this step's k_tail
// starts the next one; otherwise (blocks: the wave speed is combined across
// blocks between steps) the step begins with k_step_start.
void launch_step(const Dev& dd, int fused_start, cudaStream_t s) {
    Dev d = dd;
    d.scan_nodes = 1;
    d.diag = 1;
    d.cls_post = d.pcls != nullptr;  // the step before (or launch_cls_flags) left the post blocks' masks
    if (!fused_start) pdl(k_step_start, dim3(1), dim3(1), 0, s, d.ctl, d.dx, d.dy);
    launch_lagrange_run(d, s);
    launch_remap_core(d, s);
    launch_post(d, 1, s);
    launch_tail(d, fused_start, s);
}

// ---- block mode: the step split around the halo exchange ----------------------
// head(1): the step start (dt from the all-reduced wave speed) and the fused
// Lagrange tiles that read owned data only; head(2): the remaining tiles,
// launched once the halo has arrived; rest: everything after the Lagrange
// kernel (captured as a CUDA graph per State parity)
void launch_step_block_head(const Dev& dd, int part, cudaStream_t s) {
    Dev d = dd;
    d.scan_nodes = 1;
    d.diag = 1;
    d.lag_sel = part;
    if (part == 1) { k_step_start<<<1, 1, 0, s>>>(d.ctl, d.dx, d.dy); ++g_launches; }
    const dim3 g = tiles_of(d.r_lagn, LTX, H2D_FTY), b(H2D_LAG_NT);
    if (d.nmat == 3)
        { k_lag_fused<3><<<g, b, 0, s>>>(d); ++g_launches; }
    else if (d.nmat == 2)
        { k_lag_fused<2><<<g, b, 0, s>>>(d); ++g_launches; }
    else
        { k_lag_fused<1><<<g, b, 0, s>>>(d); ++g_launches; }
}
// HalfStepState::x_half (lagrange.cpp:87-93): node_pos(i, j) + (0.5 dt) u over
// every stored node, ghosts included
__global__ void k_xhalf(Dev d, double* xh, double* yh) {
    const double dt = step_dt(d.ctl);
    const double h = 0.5 * dt;
    int i, j;
    tid2(i, j, d.win_n.i0, d.win_n.j0);
    if (!in(d.win_n, i, j)) return;
    const int n = ix(d, i, j);
    xh[n] = (d.x0 + i * d.dx) + h * d.ux[n];
    yh[n] = (d.y0 + j * d.dy) + h * d.uy[n];
}
void launch_xhalf(const Dev& d, double* xh, double* yh, cudaStream_t s) {
    k_xhalf<<<grid_of(d.win_n), blk2(), 0, s>>>(d, xh, yh);
    ++g_launches;
}

int lag_tile_w() { return LTX; }
int lag_tile_h() { return H2D_FTY; }
void launch_step_block_rest(const Dev& dd, cudaStream_t s) {
    Dev d = dd;
    d.scan_nodes = 1;
    d.diag = 1;
    launch_lag_ghosts(d, s);
    launch_remap_core(d, s);
    launch_post(d, 1, s);
    launch_tail(d, 0, s);
}

// the per-step scalars of a block, combined across blocks by ONE max-reduction
// of four 64-bit words: the next wave-speed maximum (a non-negative double's
// bits order as integers), the complements of the first cfl_dt error key and
// of the first error key (max of ~key = ~min of key), and done
__global__ void k_red_pack(const Ctl* c, unsigned long long* red) {
    red[0] = c->next_wmax_bits;
    red[1] = ~c->next_err_key;
    red[2] = ~c->err_key;
    red[3] = (unsigned long long)c->done;
}
// back into the control block: the global values the single domain would
// hold; when the first error precedes the commit, a block that committed its
// step undoes it (the decomposed State stays at the last common step)
__global__ void k_red_apply(Ctl* c, const unsigned long long* red) {
    c->next_wmax_bits = red[0];
    c->next_err_key = ~red[1];
    const unsigned long long e = ~red[2];
    c->err_key = e;
    if (e != kNoErr && (int)(e >> 58) < PH_NAN_CELL && c->committed) {
        c->time = c->prev_time;
        c->step -= 1;
        c->cur ^= 1;
        if (c->counted) {
            c->steps_done -= 1;
            c->floor_count -= c->step_floor;
            c->k_clip_count -= c->step_clip;
            c->mass_fix_count -= c->step_fix;
            c->max_k_violation = c->prev_max_k_violation;
        }
        c->committed = 0;
        c->counted = 0;
    }
}
// in-process blocks: the max over every block's four words, written back to all
__global__ void k_red_local(unsigned long long* const* red, int n) {
    const int w = threadIdx.x;
    if (w >= 4) return;
    unsigned long long m = 0;
    for (int b = 0; b < n; ++b) m = red[b][w] > m ? red[b][w] : m;
    for (int b = 0; b < n; ++b) red[b][w] = m;
}
void launch_red_pack(const Ctl* c, unsigned long long* red, cudaStream_t s) {
    k_red_pack<<<1, 1, 0, s>>>(c, red);
    ++g_launches;
}
void launch_red_apply(Ctl* c, const unsigned long long* red, cudaStream_t s) {
    k_red_apply<<<1, 1, 0, s>>>(c, red);
    ++g_launches;
}
void launch_red_local(unsigned long long* const* red, int n, cudaStream_t s) {
    k_red_local<<<1, 32, 0, s>>>(red, n);
    ++g_launches;
}

// every halo rectangle of a block in ONE launch: segment q covers the
// rectangles rc[q] (cell planes) and rn[q] (node planes), laid out from
// off[q] in the buffer (k_rect_xfer's order inside a segment)
__global__ void k_halo_multi(Dev d, FieldList cells, FieldList nodes, HaloPlan plan, double* buf, int to_buf) {
    const long long total = plan.off[plan.n];
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        int q = 0;
        while (t >= plan.off[q + 1]) ++q;
        const Rng rc = plan.rc[q], rn = plan.rn[q];
        const long long u = t - plan.off[q];
        const int wc = rc.i1 - rc.i0, wn = rn.i1 - rn.i0;
        const long long ac = (long long)wc * (rc.j1 - rc.j0), an = (long long)wn * (rn.j1 - rn.j0);
        double* pl;
        int i, j;
        if (u < ac * cells.n) {
            const int f = (int)(u / ac);
            const long long r = u - f * ac;
            pl = cells.f[f];
            i = rc.i0 + (int)(r % wc);
            j = rc.j0 + (int)(r / wc);
        } else {
            const long long v = u - ac * cells.n;
            const int f = (int)(v / an);
            const long long r = v - f * an;
            pl = nodes.f[f];
            i = rn.i0 + (int)(r % wn);
            j = rn.j0 + (int)(r / wn);
        }
        if (to_buf)
            buf[t] = pl[ix(d, i, j)];
        else
            pl[ix(d, i, j)] = buf[t];
    }
}
void launch_halo_multi(const Dev& d, const FieldList& cells, const FieldList& nodes, const HaloPlan& plan,
                       double* buf, int to_buf, cudaStream_t s) {
    const long long n = plan.off[plan.n];
    if (n <= 0) return;
    unsigned nb = nblk(n, 256);
    if (nb > 148u * 8u) nb = 148u * 8u;
    k_halo_multi<<<nb, 256, 0, s>>>(d, cells, nodes, plan, buf, to_buf);
    ++g_launches;
}

// One AD directional pass (remap.cpp:469-589) writing into dout's planes.
static void launch_ad_pass(const Dev& dout, const AdIO& w, int remap_velocity, cudaStream_t s) {
    const dim3 gft = tiles_of(dout.r_gath, RTX, RTY);
    if (dout.nmat == 2) {
        if (w.axis_x)
            pdl(k_ad_tile<2, 1>, gft, dim3(RTX * RTY), 0, s, dout, w);
        else
            pdl(k_ad_tile<2, 0>, gft, dim3(RTX * RTY), 0, s, dout, w);
    } else {
        if (w.axis_x)
            pdl(k_ad_tile<1, 1>, gft, dim3(RTX * RTY), 0, s, dout, w);
        else
            pdl(k_ad_tile<1, 0>, gft, dim3(RTX * RTY), 0, s, dout, w);
    }
    launch_remap_slivers(dout, s);  // slivers + Work / face-flux ghosts (finalize_cells tail, :371-382)
    FieldList none{};
    if (remap_velocity) {
        Dev dd = dout;  // the dual faces read the pass's Work velocities
        dd.ulx = const_cast<double*>(w.ux);
        dd.uly = const_cast<double*>(w.uy);
        if (w.axis_x) {
            pdl(k_ad_dual<1>, grid_of(dd.r_dual), blk2(), 0, s, dd, w.pass);
            pdl(k_ad_node<1>, grid_of(dd.r_node), blk2(), 0, s, dd, w);
        } else {
            pdl(k_ad_dual<0>, grid_of(dd.r_dual), blk2(), 0, s, dd, w.pass);
            pdl(k_ad_node<0>, grid_of(dd.r_node), blk2(), 0, s, dd, w);
        }
        FieldList fu{};
        fu.n = 2;
        fu.f[0] = dout.nux;
        fu.f[1] = dout.nuy;
        launch_ghost_multi(dout, none, fu, 0, 1, s);
    }
    if (dout.nmat == 2 && w.pass == 0) {  // pass 1's normals are k_post's
        pdl(k_ad_normals, grid_of(dout.r_nrm), blk2(), 0, s, dout, w);
        FieldList fc{};
        fc.n = 2;
        fc.f[0] = dout.nnrx;
        fc.f[1] = dout.nnry;
        launch_ghost_multi(dout, fc, none, 0, 1, s);
    }
}

// The two directional passes (remap.cpp:1110-1115). Pass 0 writes the AdWork
// planes, pass 1 reads them and writes the next State; a decomposition block
// exchanges the AdWork halo between the two (launch_step_block_ad_*).
void launch_ad_first(const Dev& d, const AdWork& W, int x_first, int remap_velocity, cudaStream_t s) {
    const int nm = d.nmat;
    Dev d0 = d;  // pass 0 writes the AdWork
    AdIO w0{};
    for (int a = 0; a < nm; ++a) {
        d0.nm[a] = W.m[a];
        d0.ne[a] = W.e[a];
        d0.nk[a] = W.k[a];
        d0.me[a] = W.me[a];
        w0.m[a] = d.m[a];
        w0.e[a] = d.el[a];
        w0.k[a] = d.k[a];
    }
    d0.mcell = W.mcell;
    d0.nux = W.ux;
    d0.nuy = W.uy;
    d0.nnrx = W.nrx;
    d0.nnry = W.nry;
    w0.nrx = d.nrx;
    w0.nry = d.nry;
    w0.mcell = nullptr;
    w0.ux = d.ulx;
    w0.uy = d.uly;
    w0.me_from_e = 1;
    w0.pass = 0;
    w0.axis_x = x_first ? 1 : 0;
    launch_ad_pass(d0, w0, remap_velocity, s);
}

void launch_ad_second(const Dev& d, const AdWork& W, int x_first, int remap_velocity, int run_loop, cudaStream_t s) {
    const int nm = d.nmat;
    AdIO w1{};
    for (int a = 0; a < nm; ++a) {
        w1.m[a] = W.m[a];
        w1.me[a] = W.me[a];
        w1.e[a] = W.e[a];
        w1.k[a] = W.k[a];
    }
    w1.nrx = nm == 2 ? W.nrx : d.nrx;
    w1.nry = nm == 2 ? W.nry : d.nry;
    w1.mcell = W.mcell;
    w1.ux = remap_velocity ? W.ux : d.ulx;
    w1.uy = remap_velocity ? W.uy : d.uly;
    w1.me_from_e = 0;
    w1.pass = 1;
    w1.axis_x = x_first ? 0 : 1;
    launch_ad_pass(d, w1, remap_velocity, s);
    if (!remap_velocity) pdl(k_copy_u, grid_of(d.win_n), blk2(), 0, s, d);  // w.u = u_lag (remap.cpp:130)
    Dev dp = d;  // refresh_normals_impl of pass 1 starts from pass 0's normals
    if (nm == 2) {
        dp.nrx = W.nrx;
        dp.nry = W.nry;
    }
    post_and_ghosts(dp, run_loop, s);
}

void launch_remap_ad(const Dev& d, const AdWork& W, int x_first, int remap_velocity, int run_loop, cudaStream_t s) {
    launch_ad_first(d, W, x_first, remap_velocity, s);
    launch_ad_second(d, W, x_first, remap_velocity, run_loop, s);
}

// Block mode with the AD remap: the step after the Lagrange kernel in two
// parts around the exchange of the AdWork halo (the split remap needs its
// neighbours' pass-0 result before pass 1: one more exchange per step than
// the unsplit DirectCF step, PAPER.md:544 / :595)
void launch_step_block_ad_mid(const Dev& dd, const AdWork& W, int x_first, cudaStream_t s) {
    Dev d = dd;
    d.scan_nodes = 1;
    d.diag = 1;
    launch_lag_ghosts(d, s);
    launch_ad_first(d, W, x_first, 1, s);
}
void launch_step_block_ad_rest(const Dev& dd, const AdWork& W, int x_first, cudaStream_t s) {
    Dev d = dd;
    d.scan_nodes = 1;
    d.diag = 1;
    launch_ad_second(d, W, x_first, 1, 1, s);
    launch_tail(d, 0, s);
}

// remap_single_axis (remap.cpp:1098-1104): make_work + ONE directional pass
// (pass 0 semantics: Work from the State and the LagrangeResult) written
// straight into the next State, then assemble_state (ghosts + sync_derived);
// the pass's own refresh_normals_impl (remap.cpp:588) writes the new normals
void launch_remap_single_axis(const Dev& d, const AdWork& W, int axis_x, int remap_velocity, cudaStream_t s) {
    Dev d0 = d;
    d0.mcell = W.mcell;
    AdIO w0{};
    for (int a = 0; a < d.nmat; ++a) {
        w0.m[a] = d.m[a];
        w0.e[a] = d.el[a];
        w0.k[a] = d.k[a];
    }
    w0.nrx = d.nrx;
    w0.nry = d.nry;
    w0.mcell = nullptr;
    w0.ux = d.ulx;
    w0.uy = d.uly;
    w0.me_from_e = 1;
    w0.pass = 0;
    w0.axis_x = axis_x;
    launch_ad_pass(d0, w0, remap_velocity, s);
    if (!remap_velocity) pdl(k_copy_u, grid_of(d.win_n), blk2(), 0, s, d);  // w.u = u_lag (remap.cpp:130)
    post_and_ghosts(d, 0, s);
}

void launch_step_ad(const Dev& dd, const AdWork& W, int x_first, int fused_start, cudaStream_t s) {
    Dev d = dd;
    d.scan_nodes = 1;
    d.diag = 1;
    if (!fused_start) pdl(k_step_start, dim3(1), dim3(1), 0, s, d.ctl, d.dx, d.dy);
    launch_lagrange_run(d, s);
    launch_remap_ad(d, W, x_first, 1, 1, s);
    launch_tail(d, fused_start, s);
}

void launch_step_start(const Dev& d, cudaStream_t s) { k_step_start<<<1, 1, 0, s>>>(d.ctl, d.dx, d.dy); ++g_launches; }
void launch_commit_finish(const Dev& d, cudaStream_t s) { k_commit_finish<<<1, 1, 0, s>>>(d.ctl); ++g_launches; }

void launch_cfl_next(const Dev& d, cudaStream_t s) {
    const long long ncell = (long long)d.nx * d.ny;
    unsigned nb = nblk(ncell, 256);
    if (nb > 148u * 8u) nb = 148u * 8u;
    if (d.nmat == 3)
        { k_cfl<3><<<nb, 256, 0, s>>>(d, 1); ++g_launches; }
    else if (d.nmat == 2)
        { k_cfl<2><<<nb, 256, 0, s>>>(d, 1); ++g_launches; }
    else
        { k_cfl<1><<<nb, 256, 0, s>>>(d, 1); ++g_launches; }
}

void launch_rollback(Ctl* c, cudaStream_t s) { k_rollback<<<1, 1, 0, s>>>(c); ++g_launches; }
void launch_rect_xfer(const Dev& d, const FieldList& cells, const FieldList& nodes, Rng rc, Rng rn, double* buf,
                      int to_buf, cudaStream_t s) {
    const long long n = (long long)(rc.i1 - rc.i0) * (rc.j1 - rc.j0) * cells.n +
                        (long long)(rn.i1 - rn.i0) * (rn.j1 - rn.j0) * nodes.n;
    unsigned nb = nblk(n > 0 ? n : 1, 256);
    if (nb > 148u * 16u) nb = 148u * 16u;
    { k_rect_xfer<<<nb, 256, 0, s>>>(d, cells, nodes, rc, rn, buf, to_buf); ++g_launches; }
}
void launch_global_xfer(const Dev& d, double* buf, Rng r, double* px, double* py, int vec, int to_block,
                        cudaStream_t s) {
    const long long n = (long long)(r.i1 - r.i0) * (r.j1 - r.j0);
    unsigned nb = nblk(n > 0 ? n : 1, 256);
    if (nb > 148u * 16u) nb = 148u * 16u;
    { k_global_xfer<<<nb, 256, 0, s>>>(d, buf, r, px, py, vec, to_block); ++g_launches; }
}

void launch_commit(Ctl* c, int advance, cudaStream_t s) { k_commit<<<1, 1, 0, s>>>(c, advance); }


void launch_normals_api(const Dev& d, cudaStream_t s) { k_normals<<<grid_rect(d.nx, d.ny), blk2(), 0, s>>>(d, 1); }

void launch_deinterleave(const double* src, double* x, double* y, int W, int H, int P, cudaStream_t s) {
    { k_deinterleave<<<nblk((long long)W * H, 256), 256, 0, s>>>(src, x, y, W, H, P); ++g_launches; }
}
void launch_interleave(double* dst, const double* x, const double* y, int W, int H, int P, cudaStream_t s) {
    { k_interleave<<<nblk((long long)W * H, 256), 256, 0, s>>>(dst, x, y, W, H, P); ++g_launches; }
}
}  // namespace h2d

/*
 * h2d_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU oracle.
 *
 * A plain-C, serial restatement of the reference hot path (Lagrange phase +
 * DirectCF remap + cfl_dt + run loop) of /root/reference/proj, exported
 * through the h2d C-ABI (include/h2d.h) under the `h2do_` prefix.  It is the
 * checker the parity tests compare the CUDA product against; the product
 * never links, loads or calls it.  It is itself pinned bit-for-bit against
 * the reference library (oracle/_ref, built by oracle/Makefile) by
 * tests/test_oracle_vs_reference.py and against committed golden vectors in
 * tests/golden/.
 *
 * Faithfulness rules: every expression keeps the
 * reference association, every accumulation keeps the reference order, and
 * std::min/std::max/std::clamp keep their exact comparison semantics
 * (ref_max(a,b) = a<b ? b : a, ref_min(a,b) = b<a ? b : a).  Built with
 * -ffp-contract=off.  Each function cites the reference file:line it restates.
 *
 * Scope: DirectCF remap with CornerScheme Upwind or LinearDiag (the hot path,
 * SURVEY.md §8a); AD/Direct engines and the AvgMin/LinearXY/Multid corner
 * schemes are out of scope and refused with H2D_ERR_INVALID.
 */
#include "../include/h2d.h"

#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NG H2D_GHOST
#define PURE_TOL 1e-10   /* kPureTol, state.hpp:17 */
#define THERMO_TOL 1e-6  /* kThermoTol, state.hpp:22 */
#define CFL_FRAC 0.9     /* kCflFrac, remap.cpp:13 */

/* ------------------------------------------------------------------ fields */
/* Ghosted 2D arrays in the reference Field<T> layout (field.hpp:15-33). */
typedef struct {
    int n1, n2, st;
    double* p;
} fld;
typedef struct {
    int n1, n2, st;
    double* p; /* interleaved x,y */
} vfld;
typedef struct {
    int n1, n2, st;
    int* p;
} ifld;

#define IDX(f, i, j) ((size_t)((j) + NG) * (size_t)(f).st + (size_t)((i) + NG))
#define A(f, i, j) ((f).p[IDX(f, i, j)])
#define VX(f, i, j) ((f).p[2 * IDX(f, i, j)])
#define VY(f, i, j) ((f).p[2 * IDX(f, i, j) + 1])

static size_t fsize(int n1, int n2) { return (size_t)(n1 + 2 * NG) * (size_t)(n2 + 2 * NG); }
static fld fnew(int n1, int n2) {
    fld f = {n1, n2, n1 + 2 * NG, (double*)calloc(fsize(n1, n2), sizeof(double))};
    return f;
}
static vfld vnew(int n1, int n2) {
    vfld f = {n1, n2, n1 + 2 * NG, (double*)calloc(2 * fsize(n1, n2), sizeof(double))};
    return f;
}
static ifld inew(int n1, int n2) {
    ifld f = {n1, n2, n1 + 2 * NG, (int*)calloc(fsize(n1, n2), sizeof(int))};
    return f;
}
static void fzero(fld f) { memset(f.p, 0, fsize(f.n1, f.n2) * sizeof(double)); }
static void vzero(vfld f) { memset(f.p, 0, 2 * fsize(f.n1, f.n2) * sizeof(double)); }
static void izero(ifld f) { memset(f.p, 0, fsize(f.n1, f.n2) * sizeof(int)); }
static void ffill(fld f, double v) {
    size_t n = fsize(f.n1, f.n2);
    for (size_t q = 0; q < n; ++q) f.p[q] = v;
}
static void fcopy(fld d, fld s) { memcpy(d.p, s.p, fsize(s.n1, s.n2) * sizeof(double)); }
static void vcopy(vfld d, vfld s) { memcpy(d.p, s.p, 2 * fsize(s.n1, s.n2) * sizeof(double)); }

/* std::max / std::min / std::clamp comparison semantics */
static double ref_max(double a, double b) { return (a < b) ? b : a; }
static double ref_min(double a, double b) { return (b < a) ? b : a; }

/* ----------------------------------------------------------------- context */
typedef struct {
    /* Work (remap.cpp:88-98) */
    fld m[H2D_MAX_MAT], me[H2D_MAX_MAT], e[H2D_MAX_MAT], k[H2D_MAX_MAT];
    vfld normals;
    fld mcell;
    vfld u;
} work_t;

struct h2do_ctx {
    h2d_config cfg;
    int nx, ny, nmat, per_x, per_y;
    double dx, dy, x0, y0, cv;
    /* State (state.hpp:39-63) */
    fld m[H2D_MAX_MAT], e[H2D_MAX_MAT], k[H2D_MAX_MAT];
    fld vol, m_mix, e_mix, rho_mix, p_mix;
    vfld nrm, u;
    int step;
    double time;
    /* LagrangeResult (lagrange.hpp:38-45) */
    vfld u_half, u_lag;
    fld e_lag[H2D_MAX_MAT], vol_lag, q;
    int floor_count, have_lag;
    /* predict scratch (HalfStepState, lagrange.hpp:26-35) */
    vfld dh;
    fld vol_half, e_half[H2D_MAX_MAT], p_half[H2D_MAX_MAT], p_mix_half;
    int half_floor;
    /* remap scratch */
    work_t w;
    fld fdx, fdy, xlcx, xlcy, wlx, wly; /* AxisGeom X / Y (remap.cpp:288-294) */
    fld fx_dv, fx_lo, fx_hi, fy_dv, fy_lo, fy_hi;
    fld cf_dv;
    ifld cf_sx, cf_sy;
    fld vlag, rho[H2D_MAX_MAT];
    vfld xlag2;
    ifld if_mixed, if_lo, if_hi; /* (if_lo, if_hi: the interface pair of a 3-material cell) */
    fld if_lox, if_loy, if_hix, if_hiy, if_nx, if_ny, if_d;
    fld vola[H2D_MAX_MAT];
    fld dmx, dmy, dmc, mcell_lag;
    vfld acc, unew;
    int* sl_i; int* sl_j; int* sl_a; double* sl_m; double* sl_me;
    size_t sl_cap;
    h2d_remap_diag* diag;
    /* error unwinding */
    jmp_buf jb;
    h2d_error err;
};
typedef struct h2do_ctx ctx_t;

static void raise_err(ctx_t* c, int kind, int i, int j, const char* what) {
    c->err.kind = kind;
    c->err.i = i;
    c->err.j = j;
    c->err.step = -1;
    c->err.in_step = 0;
    /* SimError::format (errors.hpp:21-26) */
    if (i >= 0 || j >= 0)
        snprintf(c->err.what, sizeof c->err.what, "%s at cell (%d,%d)", what, i, j);
    else
        snprintf(c->err.what, sizeof c->err.what, "%s", what);
    longjmp(c->jb, 1);
}

/* ---------------------------------------------------------------- EOS */
/* eos_pressure, eos.hpp:21-25 */
static double eos_pressure(const h2d_eos* q, double rho, double e) {
    double p = (q->gamma - 1.0) * rho * e;
    if (q->kind == H2D_EOS_STIFFENED) p -= q->pi;
    return p;
}
/* sound_speed, eos.hpp:29-34 */
static double sound_speed(ctx_t* c, const h2d_eos* q, double rho, double p) {
    const double pi = (q->kind == H2D_EOS_STIFFENED) ? q->pi : 0.0;
    const double c2 = q->gamma * (p + pi) / rho;
    if (!(c2 >= 0.0)) raise_err(c, H2D_ERR_UNPHYSICAL, -1, -1, "unphysical state: gamma*(P+pi)/rho < 0");
    return sqrt(c2);
}

/* ---------------------------------------------------------------- ghosts */
/* wrap_cell, state.cpp:48-53 */
static int wrap_cell(int i, int n, int periodic) {
    if (periodic) return (i % n + n) % n;
    if (i < 0) return -1 - i;
    if (i >= n) return 2 * n - 1 - i;
    return i;
}
/* fill_cell_ghosts, state.cpp:55-66 */
static void ghost_cells(ctx_t* c, fld f) {
    for (int j = -NG; j < c->ny + NG; ++j) {
        const int js = wrap_cell(j, c->ny, c->per_y);
        for (int i = -NG; i < c->nx + NG; ++i) {
            if (i >= 0 && i < c->nx && j >= 0 && j < c->ny) continue;
            const int is = wrap_cell(i, c->nx, c->per_x);
            A(f, i, j) = A(f, is, js);
        }
    }
}
static void ghost_cells_v(ctx_t* c, vfld f) {
    for (int j = -NG; j < c->ny + NG; ++j) {
        const int js = wrap_cell(j, c->ny, c->per_y);
        for (int i = -NG; i < c->nx + NG; ++i) {
            if (i >= 0 && i < c->nx && j >= 0 && j < c->ny) continue;
            const int is = wrap_cell(i, c->nx, c->per_x);
            VX(f, i, j) = VX(f, is, js);
            VY(f, i, j) = VY(f, is, js);
        }
    }
}
/* wrap_node, state.cpp:71-80 */
static int wrap_node(int i, int n, int periodic, int* flip) {
    *flip = 0;
    if (periodic) {
        int s = i % n;
        if (s < 0) s += n;
        return s;
    }
    if (i < 0) { *flip = 1; return -i; }
    if (i > n) { *flip = 1; return 2 * n - i; }
    return i;
}
/* fill_ghost_nodes, state.cpp:87-108 */
static void ghost_nodes(ctx_t* c, vfld u) {
    const int nx = c->nx, ny = c->ny;
    if (!c->per_x)
        for (int j = 0; j <= ny; ++j) { VX(u, 0, j) = 0.0; VX(u, nx, j) = 0.0; }
    if (!c->per_y)
        for (int i = 0; i <= nx; ++i) { VY(u, i, 0) = 0.0; VY(u, i, ny) = 0.0; }
    for (int j = -NG; j <= ny + NG; ++j) {
        int fj;
        const int sj = wrap_node(j, ny, c->per_y, &fj);
        for (int i = -NG; i <= nx + NG; ++i) {
            if (i >= 0 && i <= nx && j >= 0 && j <= ny) continue;
            int fi;
            const int si = wrap_node(i, nx, c->per_x, &fi);
            double vx = VX(u, si, sj), vy = VY(u, si, sj);
            if (fi) vx = -vx;
            if (fj) vy = -vy;
            VX(u, i, j) = vx;
            VY(u, i, j) = vy;
        }
    }
}

/* sync_derived, state.cpp:120-143 */
static void sync_derived(ctx_t* c) {
    const double cv = c->cv;
    for (int j = -NG; j < c->ny + NG; ++j)
        for (int i = -NG; i < c->nx + NG; ++i) {
            double m = 0.0, me = 0.0, p = 0.0;
            for (int a = 0; a < c->nmat; ++a) {
                const double ka = A(c->k[a], i, j);
                if (ka <= 0.0) continue;
                const double ma = A(c->m[a], i, j);
                m += ma;
                me += ma * A(c->e[a], i, j);
                if (ka < THERMO_TOL) continue;
                const double rho_a = ma / (ka * cv);
                p += ka * eos_pressure(&c->cfg.eos[a], rho_a, A(c->e[a], i, j));
            }
            A(c->m_mix, i, j) = m;
            A(c->e_mix, i, j) = m > 0.0 ? me / m : 0.0;
            A(c->rho_mix, i, j) = m / cv;
            A(c->p_mix, i, j) = p;
            A(c->vol, i, j) = cv;
        }
}

/* ---------------------------------------------------------------- cfl_dt */
/* cfl_dt, harness.cpp:293-313 */
static double cfl_dt(ctx_t* c, double cfl) {
    double wmax = 0.0;
    for (int j = 0; j < c->ny; ++j)
        for (int i = 0; i < c->nx; ++i) {
            double cs = 0.0;
            for (int a = 0; a < c->nmat; ++a) {
                const double ka = A(c->k[a], i, j);
                if (ka < THERMO_TOL) continue;
                const double rho_a = A(c->m[a], i, j) / (ka * c->cv);
                const double pa = eos_pressure(&c->cfg.eos[a], rho_a, A(c->e[a], i, j));
                cs += ka * sound_speed(c, &c->cfg.eos[a], rho_a, pa);
            }
            double umax = 0.0;
            for (int dj = 0; dj <= 1; ++dj)
                for (int di = 0; di <= 1; ++di) {
                    const double ux = VX(c->u, i + di, j + dj), uy = VY(c->u, i + di, j + dj);
                    umax = ref_max(umax, sqrt(ux * ux + uy * uy));
                }
            wmax = ref_max(wmax, cs + umax);
        }
    if (!(wmax > 0.0) || !isfinite(wmax)) raise_err(c, H2D_ERR_SIM, -1, -1, "non-finite wave speed");
    return cfl * ref_min(c->dx, c->dy) / wmax;
}

/* ---------------------------------------------------------------- Lagrange */
/* quad_volume_disp, lagrange.cpp:36-46 (nodes d00, d10, d11, d01) */
static double quad_volume_disp(ctx_t* c, vfld d, int i, int j) {
    const double d00x = VX(d, i, j), d00y = VY(d, i, j);
    const double d10x = VX(d, i + 1, j), d10y = VY(d, i + 1, j);
    const double d11x = VX(d, i + 1, j + 1), d11y = VY(d, i + 1, j + 1);
    const double d01x = VX(d, i, j + 1), d01y = VY(d, i, j + 1);
    const double ebx = c->dx + d10x - d00x, eby = d10y - d00y;
    const double elx = d01x - d00x, ely = c->dy + d01y - d00y;
    const double etx = c->dx + d11x - d01x, ety = d11y - d01y;
    const double erx = d11x - d10x, ery = c->dy + d11y - d10y;
    const double s1 = 0.5 * (ebx * ely - eby * elx);
    const double s2 = 0.5 * (etx * ery - ety * erx);
    if (s1 <= 0.0 || s2 <= 0.0) raise_err(c, H2D_ERR_TANGLED, i, j, "tangled cell");
    return s1 + s2;
}

/* mixture_sound_speed, lagrange.cpp:48-59 */
static double mixture_sound_speed(ctx_t* c, int i, int j) {
    double cs = 0.0;
    for (int a = 0; a < c->nmat; ++a) {
        const double ka = A(c->k[a], i, j);
        if (ka < THERMO_TOL) continue;
        const double rho_a = A(c->m[a], i, j) / (ka * c->cv);
        const double pa = eos_pressure(&c->cfg.eos[a], rho_a, A(c->e[a], i, j));
        cs += ka * sound_speed(c, &c->cfg.eos[a], rho_a, pa);
    }
    return cs;
}

/* compute_q + div_u_cell + pseudo_viscosity, lagrange.cpp:63-77,14-20,7-12 */
static void compute_q(ctx_t* c) {
    const double L = sqrt(c->dx * c->dy); /* Mesh::char_length, mesh.hpp:39 */
    fzero(c->q);
    for (int j = 0; j < c->ny; ++j)
        for (int i = 0; i < c->nx; ++i) {
            vfld u = c->u;
            const double ux_l = 0.5 * (VX(u, i, j) + VX(u, i, j + 1));
            const double ux_r = 0.5 * (VX(u, i + 1, j) + VX(u, i + 1, j + 1));
            const double uy_b = 0.5 * (VY(u, i, j) + VY(u, i + 1, j));
            const double uy_t = 0.5 * (VY(u, i, j + 1) + VY(u, i + 1, j + 1));
            const double div = (ux_r - ux_l) / c->dx + (uy_t - uy_b) / c->dy;
            if (div >= 0.0) continue;
            const double rho = A(c->rho_mix, i, j);
            const double cs = mixture_sound_speed(c, i, j);
            const double du = L * fabs(div);
            A(c->q, i, j) = rho * c->cfg.pv_a1 * du * cs + c->cfg.pv_a2 * rho * du * du;
        }
    ghost_cells(c, c->q);
}

/* predict, lagrange.cpp:79-144 */
static void predict(ctx_t* c, double dt) {
    const int nx = c->nx, ny = c->ny;
    const double cv = c->cv;
    compute_q(c);
    c->half_floor = 0;
    for (int j = -NG; j <= ny + NG; ++j)
        for (int i = -NG; i <= nx + NG; ++i) {
            VX(c->dh, i, j) = 0.5 * dt * VX(c->u, i, j);
            VY(c->dh, i, j) = 0.5 * dt * VY(c->u, i, j);
        }
    for (int a = 0; a < c->nmat; ++a) { fzero(c->e_half[a]); fzero(c->p_half[a]); }
    fzero(c->p_mix_half);
    fzero(c->vol_half);
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const double vol = quad_volume_disp(c, c->dh, i, j);
            A(c->vol_half, i, j) = vol;
            double pmix = 0.0;
            for (int a = 0; a < c->nmat; ++a) {
                const double ka = A(c->k[a], i, j);
                if (ka < THERMO_TOL) {
                    if (ka > 0.0) A(c->e_half[a], i, j) = A(c->e[a], i, j);
                    continue;
                }
                const double ma = A(c->m[a], i, j);
                const double en = A(c->e[a], i, j);
                const double rho_n = ma / (ka * cv);
                const double rho_h = ma / (ka * vol);
                const double pa_n = eos_pressure(&c->cfg.eos[a], rho_n, en);
                double ea = en - (pa_n + A(c->q, i, j)) * (1.0 / rho_h - 1.0 / rho_n);
                const double efloor = 1e-8 * fabs(en);
                if (ea < efloor) { ea = efloor; ++c->half_floor; }
                A(c->e_half[a], i, j) = ea;
                A(c->p_half[a], i, j) = eos_pressure(&c->cfg.eos[a], rho_h, ea);
                pmix += ka * A(c->p_half[a], i, j);
            }
            A(c->p_mix_half, i, j) = pmix;
        }
    ghost_cells(c, c->p_mix_half);
    for (int a = 0; a < c->nmat; ++a) ghost_cells(c, c->p_half[a]);

    vzero(c->u_half);
    for (int j = 0; j <= ny; ++j)
        for (int i = 0; i <= nx; ++i) {
            /* nodal_mass, state.cpp:34-36 */
            const double mp = 0.25 * (A(c->m_mix, i - 1, j - 1) + A(c->m_mix, i, j - 1) +
                                      A(c->m_mix, i - 1, j) + A(c->m_mix, i, j));
            const double rho_p = mp / cv;
            /* grad_pq_node, lagrange.cpp:22-30 */
#define PQ(ii, jj) (A(c->p_mix_half, ii, jj) + A(c->q, ii, jj))
            const double gx = (PQ(i, j - 1) + PQ(i, j) - PQ(i - 1, j - 1) - PQ(i - 1, j)) / (2.0 * c->dx);
            const double gy = (PQ(i - 1, j) + PQ(i, j) - PQ(i - 1, j - 1) - PQ(i, j - 1)) / (2.0 * c->dy);
#undef PQ
            const double s = 0.5 * dt / rho_p;
            VX(c->u_half, i, j) = VX(c->u, i, j) - gx * s;
            VY(c->u_half, i, j) = VY(c->u, i, j) - gy * s;
        }
    ghost_nodes(c, c->u_half);
}

/* correct, lagrange.cpp:146-196 (u_half already in c->u_half) */
static void correct(ctx_t* c, double dt) {
    const int nx = c->nx, ny = c->ny;
    const double cv = c->cv;
    vfld dl = c->dh; /* reuse: dl = dt * u_half over every node */
    for (int j = -NG; j <= ny + NG; ++j)
        for (int i = -NG; i <= nx + NG; ++i) {
            VX(dl, i, j) = dt * VX(c->u_half, i, j);
            VY(dl, i, j) = dt * VY(c->u_half, i, j);
        }
    vzero(c->u_lag);
    for (int j = 0; j <= ny; ++j)
        for (int i = 0; i <= nx; ++i) {
            VX(c->u_lag, i, j) = 2.0 * VX(c->u_half, i, j) - VX(c->u, i, j);
            VY(c->u_lag, i, j) = 2.0 * VY(c->u_half, i, j) - VY(c->u, i, j);
        }
    ghost_nodes(c, c->u_lag);
    fzero(c->vol_lag);
    for (int a = 0; a < c->nmat; ++a) fzero(c->e_lag[a]);
    int floor = 0;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const double vol = quad_volume_disp(c, dl, i, j);
            A(c->vol_lag, i, j) = vol;
            for (int a = 0; a < c->nmat; ++a) {
                const double ka = A(c->k[a], i, j);
                if (ka < THERMO_TOL) {
                    if (ka > 0.0) A(c->e_lag[a], i, j) = A(c->e[a], i, j);
                    continue;
                }
                const double ma = A(c->m[a], i, j);
                const double en = A(c->e[a], i, j);
                const double rho_n = ma / (ka * cv);
                const double rho_l = ma / (ka * vol);
                double ea = en - (A(c->p_half[a], i, j) + A(c->q, i, j)) * (1.0 / rho_l - 1.0 / rho_n);
                const double efloor = 1e-8 * fabs(en);
                if (ea < efloor) { ea = efloor; ++floor; }
                A(c->e_lag[a], i, j) = ea;
            }
        }
    for (int a = 0; a < c->nmat; ++a) ghost_cells(c, c->e_lag[a]);
    c->floor_count = floor + c->half_floor;
    c->have_lag = 1;
}

/* ---------------------------------------------------------------- reconstruction */
/* van_leer, reconstruct.cpp:10-14 */
static double van_leer(double r) {
    if (!(r > 0.0)) return 0.0;
    if (r > 1e300) return 2.0;
    return (r + fabs(r)) / (1.0 + r);
}
/* limited_gradient_1d, reconstruct.cpp:16-24 */
static double limited_gradient_1d(ctx_t* c, double am, double ac, double ap, double xm, double xc,
                                  double xp) {
    const double hm = xc - xm, hp = xp - xc;
    if (hm <= 0.0 || hp <= 0.0) raise_err(c, H2D_ERR_SIM, -1, -1, "non-increasing centroid coordinates");
    const double dm = (ac - am) / hm;
    const double dp = (ap - ac) / hp;
    if (dm == 0.0 || dp == 0.0 || (dm > 0.0) != (dp > 0.0)) return 0.0;
    const double r = dm / dp;
    return 0.5 * (van_leer(r) * dp + van_leer(1.0 / r) * dm);
}
/* face_value at order 2, reconstruct.cpp:26-31 */
static double face_value2(ctx_t* c, const double a[3], const double x[3], double sgn, double lw,
                          double ufdt) {
    const double g = limited_gradient_1d(c, a[0], a[1], a[2], x[0], x[1], x[2]);
    return a[1] + 0.5 * g * (sgn * lw - ufdt);
}
/* corner_value, LinearDiag branch, reconstruct.cpp:134-148 with diag_gradient
 * (:38-42). a[p][q], xl[p][q] as Stencil3x3 (reconstruct.hpp:35-38). */
static double corner_linear_diag(ctx_t* c, const double a[3][3], const double xlx[3][3],
                                 const double xly[3][3], double dxp, double dyp, double lwx,
                                 double lwy) {
    const double dx = c->dx, dy = c->dy;
    const double ac = a[1][1];
    const double diag = sqrt(dx * dx + dy * dy);
    const double sx = dxp >= 0.0 ? 1.0 : -1.0;
    if (dxp * dyp > 0.0) {
        const double vx = dx / diag, vy = dy / diag;
        const double sc = xlx[1][1] * vx + xly[1][1] * vy;
        const double gv = limited_gradient_1d(c, a[0][0], ac, a[2][2], xlx[0][0] * vx + xly[0][0] * vy, sc,
                                              xlx[2][2] * vx + xly[2][2] * vy);
        const double ex = sx * lwx - dxp, ey = sx * lwy - dyp;
        return ac + 0.5 * gv * (ex * vx + ey * vy);
    }
    const double vx = dx / diag, vy = -dy / diag;
    const double sc = xlx[1][1] * vx + xly[1][1] * vy;
    const double gvp = limited_gradient_1d(c, a[0][2], ac, a[2][0], xlx[0][2] * vx + xly[0][2] * vy, sc,
                                           xlx[2][0] * vx + xly[2][0] * vy);
    const double ex = sx * lwx - dxp, ey = sx * -lwy - dyp;
    return ac + 0.5 * gvp * (ex * vx + ey * vy);
}

/* CornerKin, reconstruct.hpp:44-51 (er = eval_rel) */
typedef struct {
    double dxp, dyp, lag_wx, lag_wy, sgn_fx, u_fx_dt, sgn_fy, u_fy_dt, erx, ery;
} kin_t;
static int sgn_i(double v) { return v > 0.0 ? 1 : (v < 0.0 ? -1 : 0); } /* reconstruct.cpp:35 */
/* diag_gradient, reconstruct.cpp:38-42 */
static double diag_gradient(ctx_t* c, const double a[3][3], const double xlx[3][3], const double xly[3][3],
                            int im, int jm, int ip, int jp, double vx, double vy) {
    const double sc = xlx[1][1] * vx + xly[1][1] * vy;
    return limited_gradient_1d(c, a[im][jm], a[1][1], a[ip][jp], xlx[im][jm] * vx + xly[im][jm] * vy, sc,
                               xlx[ip][jp] * vx + xly[ip][jp] * vy);
}
/* qr_solve_2col, reconstruct.cpp:45-72: Householder QR of the m x 2 system */
static void qr_solve_2col(double X[8][2], double b[8], int m, double* g1, double* g2) {
    for (int col = 0; col < 2; ++col) {
        double nrm = 0.0;
        for (int r = col; r < m; ++r) nrm += X[r][col] * X[r][col];
        nrm = sqrt(nrm);
        if (nrm < 1e-300) { *g1 = 0.0; *g2 = 0.0; return; }
        const double alpha = X[col][col] > 0.0 ? -nrm : nrm;
        double v[8];
        v[col] = X[col][col] - alpha;
        for (int r = col + 1; r < m; ++r) v[r] = X[r][col];
        double vtv = 0.0;
        for (int r = col; r < m; ++r) vtv += v[r] * v[r];
        if (vtv > 0.0) {
            for (int cc = col; cc < 2; ++cc) {
                double sv = 0.0;
                for (int r = col; r < m; ++r) sv += v[r] * X[r][cc];
                sv *= 2.0 / vtv;
                for (int r = col; r < m; ++r) X[r][cc] -= sv * v[r];
            }
            double sv = 0.0;
            for (int r = col; r < m; ++r) sv += v[r] * b[r];
            sv *= 2.0 / vtv;
            for (int r = col; r < m; ++r) b[r] -= sv * v[r];
        }
    }
    const double y2 = b[1] / X[1][1];
    *g2 = y2;
    *g1 = (b[0] - X[0][1] * y2) / X[0][0];
}
/* multid_plane, reconstruct.cpp:76-107: pl = {a0, centre, limited gradient} */
typedef struct { double a0, cx, cy, gx, gy; } plane_t;
static plane_t multid_plane(ctx_t* c, const double a[3][3], const double xlx[3][3], const double xly[3][3]) {
    plane_t pl;
    pl.a0 = a[1][1];
    pl.cx = xlx[1][1];
    pl.cy = xly[1][1];
    double X[8][2], b[8];
    int m = 0;
    for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) {
            if (p == 1 && q == 1) continue;
            X[m][0] = xlx[p][q] - pl.cx;
            X[m][1] = xly[p][q] - pl.cy;
            b[m] = a[p][q] - pl.a0;
            ++m;
        }
    double grx, gry;
    qr_solve_2col(X, b, m, &grx, &gry);
    const double gnorm = sqrt(grx * grx + gry * gry);
    if (gnorm < 1e-300) {
        pl.gx = 0.0;
        pl.gy = 0.0;
        return pl;
    }
    const double dx = c->dx, dy = c->dy;
    const double diag = sqrt(dx * dx + dy * dy);
    const double vx = dx / diag, vy = dy / diag, vpx = dx / diag, vpy = -dy / diag;
    const double gx = limited_gradient_1d(c, a[0][1], a[1][1], a[2][1], xlx[0][1], xlx[1][1], xlx[2][1]);
    const double gy = limited_gradient_1d(c, a[1][0], a[1][1], a[1][2], xly[1][0], xly[1][1], xly[1][2]);
    const double gv = diag_gradient(c, a, xlx, xly, 0, 0, 2, 2, vx, vy);
    const double gvp = diag_gradient(c, a, xlx, xly, 0, 2, 2, 0, vpx, vpy);
    const double phi = ref_min(ref_min(fabs(gx), fabs(gy)), ref_min(fabs(gv), fabs(gvp))) / gnorm;
    pl.gx = phi * grx;
    pl.gy = phi * gry;
    return pl;
}
/* plane_eval, reconstruct.hpp:67-69 */
static double plane_eval(const plane_t* pl, double x, double y) {
    return pl->a0 + (pl->gx * (x - pl->cx) + pl->gy * (y - pl->cy));
}
/* corner_value, reconstruct.cpp:116-152 (every corner scheme) */
static double corner_value(ctx_t* c, int scheme, const double a[3][3], const double xlx[3][3],
                           const double xly[3][3], const kin_t* k) {
    const double ac = a[1][1];
    switch (scheme) {
    case H2D_CORNER_AVGMIN: {
        const int sx = sgn_i(k->dxp), sy = sgn_i(k->dyp);
        const double pair_avg = 0.5 * (ac + a[1 + sx][1 + sy]);
        return ref_min(ac, pair_avg);
    }
    case H2D_CORNER_LINEARXY: {
        const double gx = limited_gradient_1d(c, a[0][1], ac, a[2][1], xlx[0][1], xlx[1][1], xlx[2][1]);
        const double gy = limited_gradient_1d(c, a[1][0], ac, a[1][2], xly[1][0], xly[1][1], xly[1][2]);
        return ac + 0.5 * gx * (k->sgn_fx * k->lag_wx - k->u_fx_dt) + 0.5 * gy * (k->sgn_fy * k->lag_wy - k->u_fy_dt);
    }
    case H2D_CORNER_LINEARDIAG:
        return corner_linear_diag(c, a, xlx, xly, k->dxp, k->dyp, k->lag_wx, k->lag_wy);
    case H2D_CORNER_MULTID: {
        const plane_t pl = multid_plane(c, a, xlx, xly);
        return pl.a0 + (pl.gx * k->erx + pl.gy * k->ery);
    }
    default:
        return ac;
    }
}

/* ---------------------------------------------------------------- VOF */
/* corner_fraction, vof.cpp:28-32 */
static double corner_fraction(double A_, double B_, double t) {
    if (t <= 0.0) return 0.0;
    if (A_ > 0.0 && t < A_) return t * t / (2.0 * A_ * B_);
    return (t - 0.5 * A_) / B_;
}
/* clipped_fraction, vof.cpp:36-45 */
static double clipped_fraction(double w, double h, double nx, double ny, double d) {
    double A_ = fabs(nx) * w, B_ = fabs(ny) * h;
    if (A_ > B_) { double t = A_; A_ = B_; B_ = t; }
    const double S = 0.5 * (A_ + B_);
    if (d <= -S) return 0.0;
    if (d >= S) return 1.0;
    if (d <= 0.0) return corner_fraction(A_, B_, d + S);
    return 1.0 - corner_fraction(A_, B_, S - d);
}
/* place_interface, vof.cpp:47-73; returns d */
static double place_interface(double frac, double nx, double ny, double lox, double loy, double hix,
                              double hiy) {
    const double w = hix - lox, h = hiy - loy;
    double A_ = fabs(nx) * w, B_ = fabs(ny) * h;
    if (A_ > B_) { double t = A_; A_ = B_; B_ = t; }
    const double S = 0.5 * (A_ + B_);
    const int flip = frac > 0.5;
    const double kk = flip ? 1.0 - frac : frac;
    double t;
    if (A_ > 0.0 && kk <= A_ / (2.0 * B_))
        t = sqrt(2.0 * A_ * B_ * kk);
    else
        t = kk * B_ + 0.5 * A_;
    double d = t - S;
    if (flip) d = -d;
    if (fabs(clipped_fraction(w, h, nx, ny, d) - frac) > 1e-13) {
        double lo = -S, hi = S;
        for (int it = 0; it < 200 && hi - lo > 1e-13 * (2.0 * S); ++it) {
            const double mid = 0.5 * (lo + hi);
            if (clipped_fraction(w, h, nx, ny, mid) < frac) lo = mid; else hi = mid;
        }
        d = 0.5 * (lo + hi);
    }
    return d;
}
/* youngs_normal, vof.cpp:10-22; returns 0 and leaves n untouched when the
 * gradient vanishes (the IsolatedMixedCellError caught at remap.cpp:107-111) */
static int youngs_normal(ctx_t* c, fld k1, int i, int j, double* nx, double* ny) {
#define COL(ii) (A(k1, ii, j - 1) + 2.0 * A(k1, ii, j) + A(k1, ii, j + 1))
#define ROW(jj) (A(k1, i - 1, jj) + 2.0 * A(k1, i, jj) + A(k1, i + 1, jj))
    const double gx = (COL(i + 1) - COL(i - 1)) / (8.0 * c->dx);
    const double gy = (ROW(j + 1) - ROW(j - 1)) / (8.0 * c->dy);
#undef COL
#undef ROW
    const double g = sqrt(gx * gx + gy * gy);
    if (g < 1e-300) return 0;
    *nx = gx / g;
    *ny = gy / g;
    return 1;
}

/* ---------------------------------------------------------------- remap */
static int is_mixed(double k0) { return k0 > PURE_TOL && k0 < 1.0 - PURE_TOL; } /* remap.cpp:100 */

/* ---- three materials (configuration 5; no reference counterpart, the
 * reference stops at kMaxMat = 2, state.hpp:13). The N-material extension
 * applies the reference's one-interface VOF to the two
 * largest fractions of a cell and IS the reference wherever a cell holds at
 * most two materials (tests/test_three_materials.py checks that a 3-material
 * run with one material absent equals the 2-material reference run):
 *   mixed     three materials present (k > 0), or exactly two with the
 *             lower-index one mixed in the reference's sense (remap.cpp:100);
 *   pair      (lo, hi): the two largest fractions, ties to the lower index;
 *   normal    Youngs normal of the pair's k_hi (remap.cpp:102-114);
 *   interface place_interface(frac, normal, rect) with frac = k_lo, or
 *             k_lo / (k_lo + k_hi) when the third material is present;
 *   split     a mixed donor: the third material takes k_r * dvol of the flux
 *             box, the pair splits the rest at the interface (box_frac0);
 *             a pure donor gives everything to its largest fraction
 *             (remap.cpp:243-268);
 *   finalize  a cell where some material's remapped volume is exactly zero is
 *             finalised by the reference's two-material rule on the other two
 *             (the zero one: the highest such index); otherwise k_a = vola_a /
 *             cv, clipped and snapped each, k2 = (1 - k0) - k1 (a k2 below
 *             kPureTol snaps and k1 = 1 - k0), and a negative-mass material
 *             hands its fraction to the largest other (remap.cpp:146-193);
 *   slivers   an orphan sliver joins the cell's largest other material
 *             (remap.cpp:217-225). */
static void pair3(const double* k, int* lo, int* hi) {
    int p = 0;
    for (int a = 1; a < 3; ++a)
        if (k[a] > k[p]) p = a;
    int q = p == 0 ? 1 : 0;
    for (int a = 0; a < 3; ++a)
        if (a != p && k[a] > k[q]) q = a;
    *lo = p < q ? p : q;
    *hi = p < q ? q : p;
}
static int mixed3(const double* k) {
    const int n = (k[0] > 0.0) + (k[1] > 0.0) + (k[2] > 0.0);
    if (n == 3) return 1;
    if (n < 2) return 0;
    const int lo = k[0] > 0.0 ? 0 : 1;
    return is_mixed(k[lo]);
}
static int largest_other3(const double* k, int a) {
    int b = -1;
    for (int c = 0; c < 3; ++c)
        if (c != a && (b < 0 || k[c] > k[b])) b = c;
    return b;
}
static void kcell3(fld* kf, int i, int j, double* k) {
    for (int a = 0; a < 3; ++a) k[a] = A(kf[a], i, j);
}

/* cf_face_flux_x, remap.cpp:27-47; (dmx,dmy),(dpx,dpy) already axis-swapped for Y */
static void cf_face_flux(double ym, double yp, double dmx, double dmy, double dpx, double dpy,
                         double* dv, double* wl, double* wh) {
    *dv = 0.0; *wl = 0.0; *wh = 0.0;
    const double wlo = ym + ref_max(0.0, dmy);
    const double whi = yp + ref_min(0.0, dpy);
    if (whi <= wlo) return;
    *wl = wlo;
    *wh = whi;
    const double den = (yp + dpy) - (ym + dmy);
    double xlo, xhi;
    if (fabs(den) < 1e-300) {
        xlo = xhi = 0.5 * (dmx + dpx);
    } else {
        const double slope = (dpx - dmx) / den;
        xlo = dmx + slope * (wlo - (ym + dmy));
        xhi = dmx + slope * (whi - (ym + dmy));
    }
    *dv = 0.5 * (xlo + xhi) * (whi - wlo);
}

/* make_work, remap.cpp:116-140 */
static void make_work(ctx_t* c) {
    work_t* w = &c->w;
    for (int a = 0; a < c->nmat; ++a) {
        fcopy(w->m[a], c->m[a]);
        fcopy(w->e[a], c->e_lag[a]);
        fcopy(w->k[a], c->k[a]);
        fzero(w->me[a]);
        for (int j = -NG; j < c->ny + NG; ++j)
            for (int i = -NG; i < c->nx + NG; ++i) A(w->me[a], i, j) = A(w->m[a], i, j) * A(w->e[a], i, j);
    }
    vcopy(w->normals, c->nrm);
    vcopy(w->u, c->u_lag);
    for (int j = -NG; j < c->ny + NG; ++j)
        for (int i = -NG; i < c->nx + NG; ++i) {
            double m = 0.0;
            for (int a = 0; a < c->nmat; ++a) m += A(w->m[a], i, j);
            A(w->mcell, i, j) = m;
        }
}

/* box_frac0 + split_flux, remap.cpp:243-268 */
static void split_flux(ctx_t* c, int di, int dj, double blox, double bloy, double bhix, double bhiy,
                       double dvol, double dva[H2D_MAX_MAT]) {
    dva[0] = dvol;
    dva[1] = 0.0;
    dva[2] = 0.0;
    if (c->nmat == 3) {  /* the N-material split (see pair3) */
        double k[3];
        kcell3(c->w.k, di, dj, k);
        dva[0] = 0.0;
        if (!A(c->if_mixed, di, dj)) {
            int p = 0;
            for (int a = 1; a < 3; ++a)
                if (k[a] > k[p]) p = a;
            dva[p] = dvol;
            return;
        }
        const int lo = A(c->if_lo, di, dj), hi = A(c->if_hi, di, dj), r = 3 - lo - hi;
        const double nx = A(c->if_nx, di, dj), ny = A(c->if_ny, di, dj), d = A(c->if_d, di, dj);
        const double rcx = 0.5 * (A(c->if_lox, di, dj) + A(c->if_hix, di, dj));
        const double rcy = 0.5 * (A(c->if_loy, di, dj) + A(c->if_hiy, di, dj));
        const double bcx = 0.5 * (blox + bhix), bcy = 0.5 * (bloy + bhiy);
        const double bw = bhix - blox, bh = bhiy - bloy;
        double f0;
        if (!(bw * bh > 0.0)) {
            const double sv = (nx * (bcx - rcx) + ny * (bcy - rcy)) - d;
            f0 = sv <= 0.0 ? 1.0 : 0.0;
        } else {
            f0 = clipped_fraction(bw, bh, nx, ny, d - (nx * (bcx - rcx) + ny * (bcy - rcy)));
        }
        dva[r] = k[r] > 0.0 ? k[r] * dvol : 0.0;
        const double rest = dvol - dva[r];
        dva[lo] = f0 * rest;
        dva[hi] = rest - dva[lo];
        return;
    }
    if (c->nmat != 2) return;
    if (A(c->if_mixed, di, dj)) {
        const double nx = A(c->if_nx, di, dj), ny = A(c->if_ny, di, dj), d = A(c->if_d, di, dj);
        const double rcx = 0.5 * (A(c->if_lox, di, dj) + A(c->if_hix, di, dj));
        const double rcy = 0.5 * (A(c->if_loy, di, dj) + A(c->if_hiy, di, dj));
        const double bcx = 0.5 * (blox + bhix), bcy = 0.5 * (bloy + bhiy);
        const double bw = bhix - blox, bh = bhiy - bloy;
        const double area = bw * bh;
        double f0;
        if (!(area > 0.0)) {
            const double s = (nx * (bcx - rcx) + ny * (bcy - rcy)) - d;
            f0 = s <= 0.0 ? 1.0 : 0.0;
        } else {
            const double dbox = d - (nx * (bcx - rcx) + ny * (bcy - rcy));
            f0 = clipped_fraction(bw, bh, nx, ny, dbox);
        }
        dva[0] = f0 * dvol;
        dva[1] = dvol - dva[0];
    } else if (A(c->w.k[0], di, dj) < 0.5) {
        dva[0] = 0.0;
        dva[1] = dvol;
    }
}

static int pure_1d(ctx_t* c, int a, int axis_x, int ia_d, int ic) { /* remap.cpp:270-276 */
    for (int d = -1; d <= 1; ++d) {
        const double kv = axis_x ? A(c->w.k[a], ia_d + d, ic) : A(c->w.k[a], ic, ia_d + d);
        if (kv < 1.0 - PURE_TOL) return 0;
    }
    return 1;
}
static int pure_3x3(ctx_t* c, int a, int i, int j) { /* remap.cpp:278-283 */
    for (int dj = -1; dj <= 1; ++dj)
        for (int di = -1; di <= 1; ++di)
            if (A(c->w.k[a], i + di, j + dj) < 1.0 - PURE_TOL) return 0;
    return 1;
}

static void apply_cell(ctx_t* c, fld* vola, int a, int i, int j, double dm, double dme, double dva) {
    if (i < 0 || i >= c->nx || j < 0 || j >= c->ny) return; /* remap.cpp:833-838 */
    A(c->w.m[a], i, j) += dm;
    A(c->w.me[a], i, j) += dme;
    A(vola[a], i, j) += dva;
}

/* refresh_normals_impl, remap.cpp:102-114: Youngs normal of k1 in the mixed
 * cells (3 materials: of the pair's k_hi, pair3); an isolated cell keeps its
 * normal */
static void refresh_normals(ctx_t* c, fld* kf, vfld nrm) {
    for (int j = 0; j < c->ny; ++j)
        for (int i = 0; i < c->nx; ++i) {
            int hi = 1;
            if (c->nmat == 3) {
                double k[3];
                kcell3(kf, i, j, k);
                if (!mixed3(k)) continue;
                int lo;
                pair3(k, &lo, &hi);
            } else if (!is_mixed(A(kf[0], i, j))) {
                continue;
            }
            double nxv, nyv;
            if (youngs_normal(c, kf[hi], i, j, &nxv, &nyv)) {
                VX(nrm, i, j) = nxv;
                VY(nrm, i, j) = nyv;
            }
        }
    ghost_cells_v(c, nrm);
}

/* the pending-sliver record of material a at (i, j), remap.cpp:170-173 */
static void push_sliver(ctx_t* c, size_t* npend, int i, int j, int a) {
    if (*npend == c->sl_cap) {
        c->sl_cap = c->sl_cap ? 2 * c->sl_cap : 1024;
        c->sl_i = realloc(c->sl_i, c->sl_cap * sizeof(int));
        c->sl_j = realloc(c->sl_j, c->sl_cap * sizeof(int));
        c->sl_a = realloc(c->sl_a, c->sl_cap * sizeof(int));
        c->sl_m = realloc(c->sl_m, c->sl_cap * sizeof(double));
        c->sl_me = realloc(c->sl_me, c->sl_cap * sizeof(double));
    }
    c->sl_i[*npend] = i;
    c->sl_j[*npend] = j;
    c->sl_a[*npend] = a;
    c->sl_m[*npend] = A(c->w.m[a], i, j);
    c->sl_me[*npend] = A(c->w.me[a], i, j);
    ++*npend;
}

/* H2D_OPT_SLIVER_ENERGY (no reference counterpart, include/h2d.h): a material
 * with m > 0 and e < 0 after the sliver pass hands m*e to the cell's
 * largest-mass other material if the sum stays positive, else drops it;
 * its e becomes 0. Materials in index order. */
static void sliver_energy_fix(ctx_t* c) {
    work_t* w = &c->w;
    for (int j = 0; j < c->ny; ++j)
        for (int i = 0; i < c->nx; ++i)
            for (int a = 0; a < c->nmat; ++a) {
                if (!(A(w->m[a], i, j) > 0.0 && A(w->e[a], i, j) < 0.0)) continue;
                int b = -1;
                for (int q = 0; q < c->nmat; ++q)
                    if (q != a && A(w->m[q], i, j) > 0.0 && (b < 0 || A(w->m[q], i, j) > A(w->m[b], i, j))) b = q;
                if (b >= 0) {
                    const double meb = A(w->me[b], i, j) + A(w->me[a], i, j);
                    if (meb > 0.0) {
                        A(w->me[b], i, j) = meb;
                        A(w->e[b], i, j) = meb / A(w->m[b], i, j);
                    }
                }
                A(w->me[a], i, j) = 0.0;
                A(w->e[a], i, j) = 0.0;
            }
}

/* finalize_cells, remap.cpp:146-234 */
static void finalize_cells(ctx_t* c) {
    work_t* w = &c->w;
    const double cv = c->cv;
    size_t npend = 0;
    for (int j = 0; j < c->ny; ++j)
        for (int i = 0; i < c->nx; ++i) {
            if (c->nmat == 3) {
                int r = -1;  /* a material with an exactly zero remapped volume: two-material rule */
                for (int a = 2; a >= 0 && r < 0; --a)
                    if (A(c->vola[a], i, j) == 0.0) r = a;
                if (r >= 0) {
                    const int lo = r == 0 ? 1 : 0, hi = r == 2 ? 1 : 2;
                    double k0 = A(c->vola[lo], i, j) / cv;
                    const double k1 = A(c->vola[hi], i, j) / cv;
                    double viol = 0.0;
                    const double cand[5] = {-k0, k0 - 1.0, -k1, k1 - 1.0, fabs(k0 + k1 - 1.0)};
                    for (int q = 0; q < 5; ++q)
                        if (viol < cand[q]) viol = cand[q];
                    if (c->diag && viol > c->diag->max_k_violation) c->diag->max_k_violation = viol;
                    if (k0 < 0.0 || k0 > 1.0) {
                        if (c->diag) ++c->diag->k_clip_count;
                        k0 = (k0 < 0.0) ? 0.0 : ((1.0 < k0) ? 1.0 : k0);
                    }
                    if (k0 < PURE_TOL) k0 = 0.0;
                    if (k0 > 1.0 - PURE_TOL) k0 = 1.0;
                    A(w->k[lo], i, j) = k0;
                    A(w->k[hi], i, j) = 1.0 - k0;
                    A(w->k[r], i, j) = 0.0;
                } else {
                    double k[3];
                    for (int a = 0; a < 3; ++a) k[a] = A(c->vola[a], i, j) / cv;
                    double viol = 0.0;
                    const double cand[7] = {-k[0], k[0] - 1.0, -k[1], k[1] - 1.0, -k[2], k[2] - 1.0,
                                            fabs(k[0] + k[1] + k[2] - 1.0)};
                    for (int q = 0; q < 7; ++q)
                        if (viol < cand[q]) viol = cand[q];
                    if (c->diag && viol > c->diag->max_k_violation) c->diag->max_k_violation = viol;
                    int clipped = 0;
                    for (int a = 0; a < 3; ++a) {
                        if (k[a] < 0.0 || k[a] > 1.0) {
                            clipped = 1;
                            k[a] = (k[a] < 0.0) ? 0.0 : ((1.0 < k[a]) ? 1.0 : k[a]);
                        }
                        if (k[a] < PURE_TOL) k[a] = 0.0;
                        if (k[a] > 1.0 - PURE_TOL) k[a] = 1.0;
                    }
                    if (clipped && c->diag) ++c->diag->k_clip_count;
                    k[2] = (1.0 - k[0]) - k[1];
                    if (k[2] < PURE_TOL) {
                        k[2] = 0.0;
                        k[1] = 1.0 - k[0];
                    }
                    for (int a = 0; a < 3; ++a) A(w->k[a], i, j) = k[a];
                }
                for (int a = 0; a < 3; ++a) {
                    if ((A(w->k[a], i, j) == 0.0 && A(w->m[a], i, j) != 0.0) || A(w->m[a], i, j) < 0.0) {
                        push_sliver(c, &npend, i, j, a);
                        A(w->m[a], i, j) = 0.0;
                        A(w->me[a], i, j) = 0.0;
                        if (A(w->k[a], i, j) > 0.0) {  /* a negative mass with volume left behind */
                            double kk[3];
                            kcell3(w->k, i, j, kk);
                            const int b = largest_other3(kk, a);
                            if (r >= 0 && a != r) {  /* the reference's partner rule on the pair */
                                A(w->k[3 - r - a], i, j) = 1.0;
                            } else {
                                A(w->k[b], i, j) = kk[b] + kk[a];
                            }
                            A(w->k[a], i, j) = 0.0;
                        }
                    }
                }
            }
            if (c->nmat == 2) {
                double k0 = A(c->vola[0], i, j) / cv;
                const double k1 = A(c->vola[1], i, j) / cv;
                double viol = 0.0; /* std::max({...}) folds with `<` */
                const double cand[5] = {-k0, k0 - 1.0, -k1, k1 - 1.0, fabs(k0 + k1 - 1.0)};
                for (int q = 0; q < 5; ++q)
                    if (viol < cand[q]) viol = cand[q];
                if (c->diag && viol > c->diag->max_k_violation) c->diag->max_k_violation = viol;
                if (k0 < 0.0 || k0 > 1.0) {
                    if (c->diag) ++c->diag->k_clip_count;
                    k0 = (k0 < 0.0) ? 0.0 : ((1.0 < k0) ? 1.0 : k0);
                }
                if (k0 < PURE_TOL) k0 = 0.0;
                if (k0 > 1.0 - PURE_TOL) k0 = 1.0;
                A(w->k[0], i, j) = k0;
                A(w->k[1], i, j) = 1.0 - k0;
                for (int a = 0; a < 2; ++a) {
                    if ((A(w->k[a], i, j) == 0.0 && A(w->m[a], i, j) != 0.0) || A(w->m[a], i, j) < 0.0) {
                        push_sliver(c, &npend, i, j, a);
                        A(w->m[a], i, j) = 0.0;
                        A(w->me[a], i, j) = 0.0;
                        if (A(w->k[a], i, j) > 0.0) {
                            A(w->k[a], i, j) = 0.0;
                            A(w->k[1 - a], i, j) = 1.0;
                        }
                    }
                }
            }
            double mtot = 0.0;
            for (int a = 0; a < c->nmat; ++a) {
                const double ma = A(w->m[a], i, j);
                if (ma < 0.0) raise_err(c, H2D_ERR_NEGMASS, i, j, "negative mass");
                A(w->e[a], i, j) = ma > 0.0 ? A(w->me[a], i, j) / ma : 0.0;
                mtot += ma;
            }
            if (mtot <= 0.0) raise_err(c, H2D_ERR_NEGMASS, i, j, "non-positive cell mass");
            A(w->mcell, i, j) = mtot;
        }

    for (size_t s = 0; s < npend; ++s) {
        const int si = c->sl_i[s], sj = c->sl_j[s], a = c->sl_a[s];
        const double sm = c->sl_m[s], sme = c->sl_me[s];
        int bi = -1, bj = -1;
        double bk = -1.0;
        for (int r = 1; r <= 2 && bi < 0; ++r)
            for (int dj = -r; dj <= r; ++dj)
                for (int di = -r; di <= r; ++di) {
                    const int adi = di < 0 ? -di : di, adj = dj < 0 ? -dj : dj;
                    if ((adi < adj ? adj : adi) != r) continue;
                    int ni = si + di, nj = sj + dj;
                    if (c->per_x) ni = (ni + 2 * c->nx) % c->nx;
                    if (c->per_y) nj = (nj + 2 * c->ny) % c->ny;
                    if (ni < 0 || ni >= c->nx || nj < 0 || nj >= c->ny) continue;
                    if (A(w->m[a], ni, nj) <= 0.0) continue;
                    if (A(w->k[a], ni, nj) > bk) {
                        bk = A(w->k[a], ni, nj);
                        bi = ni;
                        bj = nj;
                    }
                }
        if (bi >= 0 && A(w->m[a], bi, bj) + sm > 0.0) {
            A(w->m[a], bi, bj) += sm;
            A(w->me[a], bi, bj) += sme;
            A(w->e[a], bi, bj) = A(w->me[a], bi, bj) / A(w->m[a], bi, bj);
            A(w->mcell, bi, bj) += sm;
        } else {
            if (c->diag) ++c->diag->mass_fix_count;
            int b = 1 - a;
            if (c->nmat == 3) {
                double kk[3];
                kcell3(w->k, si, sj, kk);
                b = largest_other3(kk, a);
            }
            A(w->m[b], si, sj) += sm;
            A(w->me[b], si, sj) += sme;
            A(w->e[b], si, sj) = A(w->me[b], si, sj) / A(w->m[b], si, sj);
            A(w->mcell, si, sj) += sm;
        }
    }
    if (c->cfg.options & H2D_OPT_SLIVER_ENERGY) sliver_energy_fix(c);
    for (int a = 0; a < c->nmat; ++a) {
        ghost_cells(c, w->m[a]);
        ghost_cells(c, w->me[a]);
        ghost_cells(c, w->e[a]);
        ghost_cells(c, w->k[a]);
    }
    ghost_cells(c, w->mcell);
}

/* fill_face_flux_ghosts, remap.cpp:371-382 (dmface in (along, cross) layout) */
static void face_flux_ghosts(fld f, int na, int nc, int per_a, int per_c) {
    for (int ia = 0; ia <= na; ++ia) {
        A(f, ia, -1) = per_c ? A(f, ia, nc - 1) : A(f, ia, 0);
        A(f, ia, nc) = per_c ? A(f, ia, 0) : A(f, ia, nc - 1);
    }
    for (int ic = -1; ic <= nc; ++ic) A(f, -1, ic) = per_a ? A(f, na - 1, ic) : -A(f, 1, ic);
}

static int wrapi(int i, int n, int periodic) { /* remap.cpp:339-344 */
    if (!periodic) return i;
    int r = i % n;
    if (r < 0) r += n;
    return r;
}
/* MomAcc::add, remap.cpp:358-365 */
static void acc_add(ctx_t* c, int i, int j, double vx, double vy) {
    const int nux = c->per_x ? c->nx : c->nx + 1;
    const int nuy = c->per_y ? c->ny : c->ny + 1;
    i = wrapi(i, nux, c->per_x);
    j = wrapi(j, nuy, c->per_y);
    if (i < 0 || i >= nux || j < 0 || j >= nuy) return;
    VX(c->acc, i, j) += vx;
    VY(c->acc, i, j) += vy;
}

/* dual_face_value, remap.cpp:384-404 (comp 0 = x, 1 = y) */
static double dual_face_value(ctx_t* c, int comp, int axis_x, int ia_d, int ic, double dt, double wa,
                              double sgn, double ufdt) {
#define UV(ia) (axis_x ? (comp ? VY(c->w.u, ia, ic) : VX(c->w.u, ia, ic)) \
                       : (comp ? VY(c->w.u, ic, ia) : VX(c->w.u, ic, ia)))
#define ND(ia) ((axis_x ? VX(c->u_half, ia, ic) : VY(c->u_half, ic, ia)) * dt)
    if (c->cfg.face_order <= 1) return UV(ia_d);
    double a[3], x[3];
    for (int d = -1; d <= 1; ++d) {
        a[d + 1] = UV(ia_d + d);
        x[d + 1] = (ia_d + d) * wa + ND(ia_d + d);
    }
    const double dfl = 0.5 * (ND(ia_d - 1) + ND(ia_d));
    const double dfr = 0.5 * (ND(ia_d) + ND(ia_d + 1));
    return face_value2(c, a, x, sgn, wa + (dfr - dfl), ufdt);
#undef UV
#undef ND
}

/* dual_face_pass, remap.cpp:408-442 */
static void dual_face_pass(ctx_t* c, int axis_x, fld dmface, double dt) {
    const int iend = c->per_x ? c->nx - 1 : c->nx, jend = c->per_y ? c->ny - 1 : c->ny;
    const int na_nodes = axis_x ? iend : jend, nc_nodes = axis_x ? jend : iend;
    const int per_a = axis_x ? c->per_x : c->per_y;
    const double wa = axis_x ? c->dx : c->dy;
    const int ia_lo = per_a ? 0 : 1, ia_hi = na_nodes;
    for (int ic = 0; ic <= nc_nodes; ++ic)
        for (int ia = ia_lo; ia <= ia_hi; ++ia) {
            const double dm = 0.25 * ((A(dmface, ia - 1, ic - 1) + A(dmface, ia - 1, ic)) +
                                      (A(dmface, ia, ic - 1) + A(dmface, ia, ic)));
            if (dm == 0.0) continue;
            const int ia_d = dm > 0.0 ? ia - 1 : ia;
            const double sgn = dm > 0.0 ? 1.0 : -1.0;
#define ND(iia) ((axis_x ? VX(c->u_half, iia, ic) : VY(c->u_half, ic, iia)) * dt)
            const double ufdt = 0.5 * (ND(ia - 1) + ND(ia));
#undef ND
            const double ufx = dual_face_value(c, 0, axis_x, ia_d, ic, dt, wa, sgn, ufdt);
            const double ufy = dual_face_value(c, 1, axis_x, ia_d, ic, dt, wa, sgn, ufdt);
            const double mx = ufx * dm, my = ufy * dm;
            if (axis_x) {
                acc_add(c, ia, ic, mx, my);
                acc_add(c, ia - 1, ic, mx * -1.0, my * -1.0);
            } else {
                acc_add(c, ic, ia, mx, my);
                acc_add(c, ic, ia - 1, mx * -1.0, my * -1.0);
            }
        }
}

/* apply_dual_update, remap.cpp:444-464 */
static void apply_dual_update(ctx_t* c) {
    work_t* w = &c->w;
    const int iend = c->per_x ? c->nx - 1 : c->nx, jend = c->per_y ? c->ny - 1 : c->ny;
    vcopy(c->unew, w->u);
#define QUARTER(f, i, j) (0.25 * (A(f, i - 1, j - 1) + A(f, i, j - 1) + A(f, i - 1, j) + A(f, i, j)))
    for (int j = 0; j <= jend; ++j)
        for (int i = 0; i <= iend; ++i) {
            const double mp_lag = QUARTER(c->mcell_lag, i, j);
            const double mp_new = QUARTER(w->mcell, i, j);
            if (mp_new <= 0.0) raise_err(c, H2D_ERR_NEGMASS, i, j, "non-positive nodal mass");
            const double inv = 1.0 / mp_new;
            VX(c->unew, i, j) = inv * (mp_lag * VX(w->u, i, j) + VX(c->acc, i, j));
            VY(c->unew, i, j) = inv * (mp_lag * VY(w->u, i, j) + VY(c->acc, i, j));
        }
#undef QUARTER
    if (c->per_x)
        for (int j = 0; j <= jend; ++j) {
            VX(c->unew, c->nx, j) = VX(c->unew, 0, j);
            VY(c->unew, c->nx, j) = VY(c->unew, 0, j);
        }
    if (c->per_y)
        for (int i = 0; i <= c->nx; ++i) {
            VX(c->unew, i, c->ny) = VX(c->unew, i, 0);
            VY(c->unew, i, c->ny) = VY(c->unew, i, 0);
        }
    ghost_nodes(c, c->unew);
    vcopy(w->u, c->unew);
}

/* cf_pass, remap.cpp:734-1073 */
static void cf_pass(ctx_t* c, double dt, int remap_velocity) {
    work_t* w = &c->w;
    const int nx = c->nx, ny = c->ny, nmat = c->nmat;
    const double cv = c->cv, dx = c->dx, dy = c->dy, x0 = c->x0, y0 = c->y0;
    const int order = c->cfg.face_order;
    vfld uh = c->u_half;
#define DX_(i, j) (dt * VX(uh, i, j))
#define DY_(i, j) (dt * VY(uh, i, j))

    /* make_axis_geom X and Y, remap.cpp:296-322 */
    for (int ic = -NG; ic < ny + NG; ++ic)
        for (int ia = -NG; ia <= nx + NG; ++ia)
            A(c->fdx, ia, ic) = 0.5 * (VX(uh, ia, ic) + VX(uh, ia, ic + 1)) * dt;
    for (int ic = -NG; ic < ny + NG; ++ic)
        for (int ia = -NG; ia < nx + NG; ++ia) {
            const double dl = A(c->fdx, ia, ic), dr = A(c->fdx, ia + 1, ic);
            A(c->xlcx, ia, ic) = x0 + (ia + 0.5) * dx + 0.5 * (dl + dr);
            A(c->wlx, ia, ic) = dx + (dr - dl);
        }
    for (int ic = -NG; ic < nx + NG; ++ic)
        for (int ia = -NG; ia <= ny + NG; ++ia)
            A(c->fdy, ia, ic) = 0.5 * (VY(uh, ic, ia) + VY(uh, ic + 1, ia)) * dt;
    for (int ic = -NG; ic < nx + NG; ++ic)
        for (int ia = -NG; ia < ny + NG; ++ia) {
            const double dl = A(c->fdy, ia, ic), dr = A(c->fdy, ia + 1, ic);
            A(c->xlcy, ia, ic) = y0 + (ia + 0.5) * dy + 0.5 * (dl + dr);
            A(c->wly, ia, ic) = dy + (dr - dl);
        }

    /* face and corner flux geometry, remap.cpp:744-767 */
    for (int j = -NG; j < ny + NG; ++j)
        for (int i = -NG; i <= nx + NG; ++i) {
            double dv, wl, wh;
            cf_face_flux(y0 + j * dy, y0 + (j + 1) * dy, DX_(i, j), DY_(i, j), DX_(i, j + 1), DY_(i, j + 1),
                         &dv, &wl, &wh);
            A(c->fx_dv, i, j) = dv; A(c->fx_lo, i, j) = wl; A(c->fx_hi, i, j) = wh;
            if (fabs(dv) > CFL_FRAC * cv) raise_err(c, H2D_ERR_CFL, i, j, "CFL violation at X-face");
        }
    for (int j = -NG; j <= ny + NG; ++j)
        for (int i = -NG; i < nx + NG; ++i) {
            double dv, wl, wh;
            cf_face_flux(x0 + i * dx, x0 + (i + 1) * dx, DY_(i, j), DX_(i, j), DY_(i + 1, j), DX_(i + 1, j),
                         &dv, &wl, &wh);
            A(c->fy_dv, i, j) = dv; A(c->fy_lo, i, j) = wl; A(c->fy_hi, i, j) = wh;
            if (fabs(dv) > CFL_FRAC * cv) raise_err(c, H2D_ERR_CFL, i, j, "CFL violation at Y-face");
        }
    for (int j = -NG; j <= ny + NG; ++j)
        for (int i = -NG; i <= nx + NG; ++i) {
            /* cf_corner_flux, remap.cpp:16-25 */
            const double ddx = VX(uh, i, j) * dt, ddy = VY(uh, i, j) * dt;
            double dv = fabs(ddx * ddy);
            int sx = 0, sy = 0;
            if (dv == 0.0) {
                dv = 0.0;
            } else {
                sx = ddx > 0.0 ? 1 : -1;
                sy = ddy > 0.0 ? 1 : -1;
            }
            A(c->cf_dv, i, j) = dv; A(c->cf_sx, i, j) = sx; A(c->cf_sy, i, j) = sy;
            if (dv > CFL_FRAC * cv) raise_err(c, H2D_ERR_CFL, i, j, "CFL violation at corner");
        }

    /* Lagrangian volume and densities, remap.cpp:769-794 */
    for (int j = -NG; j < ny + NG; ++j)
        for (int i = -NG; i < nx + NG; ++i) {
            double v = cv + A(c->fx_dv, i + 1, j) - A(c->fx_dv, i, j) + A(c->fy_dv, i, j + 1) - A(c->fy_dv, i, j);
            double t[4];
            const int ni_[4] = {i, i + 1, i, i + 1}, nj_[4] = {j, j, j + 1, j + 1};
            for (int q = 0; q < 4; ++q) {
                const int ni = ni_[q], nj = nj_[q];
                const double dv = A(c->cf_dv, ni, nj);
                t[q] = 0.0;
                if (dv == 0.0) continue;
                const int sx = A(c->cf_sx, ni, nj), sy = A(c->cf_sy, ni, nj);
                const int di = sx > 0 ? ni - 1 : ni, dj = sy > 0 ? nj - 1 : nj;
                if (di == i && dj == j) { t[q] = dv; continue; }
                const int ri = sx > 0 ? ni : ni - 1, rj = sy > 0 ? nj : nj - 1;
                if (ri == i && rj == j) t[q] = -dv;
            }
            v += t[0] + t[1] + t[2] + t[3];
            if (v <= 0.0) raise_err(c, H2D_ERR_CFL, i, j, "collapsed Lagrangian cell");
            A(c->vlag, i, j) = v;
            for (int a = 0; a < nmat; ++a) {
                const double ka = A(w->k[a], i, j);
                A(c->rho[a], i, j) = ka > 0.0 ? A(w->m[a], i, j) / (ka * v) : 0.0;
            }
        }
    /* 2D Lagrangian centroids, remap.cpp:797-803 */
    for (int j = -NG; j < ny + NG; ++j)
        for (int i = -NG; i < nx + NG; ++i) {
            const double mdx = 0.25 * (DX_(i, j) + DX_(i + 1, j) + DX_(i, j + 1) + DX_(i + 1, j + 1));
            const double mdy = 0.25 * (DY_(i, j) + DY_(i + 1, j) + DY_(i, j + 1) + DY_(i + 1, j + 1));
            VX(c->xlag2, i, j) = (x0 + (i + 0.5) * dx) + mdx;
            VY(c->xlag2, i, j) = (y0 + (j + 0.5) * dy) + mdy;
        }
    /* interfaces, remap.cpp:807-824 */
    izero(c->if_mixed);
    if (nmat >= 2)
        for (int j = -NG; j < ny + NG; ++j)
            for (int i = -NG; i < nx + NG; ++i) {
                double k0 = A(w->k[0], i, j);
                if (nmat == 3) {  /* the pair's interface (pair3) */
                    double k[3];
                    kcell3(w->k, i, j, k);
                    if (!mixed3(k)) continue;
                    int lo, hi;
                    pair3(k, &lo, &hi);
                    A(c->if_lo, i, j) = lo;
                    A(c->if_hi, i, j) = hi;
                    k0 = k[3 - lo - hi] > 0.0 ? k[lo] / (k[lo] + k[hi]) : k[lo];
                } else if (!is_mixed(k0)) {
                    continue;
                }
                const double cx = x0 + (i + 0.5) * dx, cy = y0 + (j + 0.5) * dy;
                const double lox = cx - 0.5 * dx + A(c->fdx, i, j), loy = cy - 0.5 * dy + A(c->fdy, j, i);
                const double hix = cx + 0.5 * dx + A(c->fdx, i + 1, j), hiy = cy + 0.5 * dy + A(c->fdy, j + 1, i);
                const double nxv = VX(w->normals, i, j), nyv = VY(w->normals, i, j);
                A(c->if_mixed, i, j) = 1;
                A(c->if_lox, i, j) = lox; A(c->if_loy, i, j) = loy;
                A(c->if_hix, i, j) = hix; A(c->if_hiy, i, j) = hiy;
                A(c->if_nx, i, j) = nxv; A(c->if_ny, i, j) = nyv;
                A(c->if_d, i, j) = place_interface(k0, nxv, nyv, lox, loy, hix, hiy);
            }
    for (int a = 0; a < nmat; ++a) {
        fzero(c->vola[a]);
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) A(c->vola[a], i, j) = A(w->k[a], i, j) * A(c->vlag, i, j);
    }

    /* face fluxes, remap.cpp:850-921 */
    fzero(c->dmx);
    fzero(c->dmy);
    for (int axis = 0; axis < 2; ++axis) {
        const int ax = axis == 0;
        const int na = ax ? nx : ny, nc = ax ? ny : nx;
        fld fdv = ax ? c->fx_dv : c->fy_dv, flo = ax ? c->fx_lo : c->fy_lo, fhi = ax ? c->fx_hi : c->fy_hi;
        fld gfd = ax ? c->fdx : c->fdy, gxl = ax ? c->xlcx : c->xlcy, gwl = ax ? c->wlx : c->wly;
        fld dmf = ax ? c->dmx : c->dmy;
        for (int ic = 0; ic < nc; ++ic)
            for (int ia = 0; ia <= na; ++ia) {
                A(dmf, ia, ic) = 0.0;
                const int fi = ax ? ia : ic, fj = ax ? ic : ia;
                const double dvol = A(fdv, fi, fj);
                if (dvol == 0.0) continue;
                const int ia_d = dvol > 0.0 ? ia - 1 : ia;
                const double sgn = dvol > 0.0 ? 1.0 : -1.0;
                const int cdi = ax ? ia_d : ic, cdj = ax ? ic : ia_d;
                const double wlo = A(flo, fi, fj), whi = A(fhi, fi, fj);
                const double wwin = whi - wlo;
                const double width = dvol / wwin;
                const double f0pos = ax ? x0 + ia * dx : y0 + ia * dy;
                const double blo = ref_min(f0pos, f0pos + width), bhi = ref_max(f0pos, f0pos + width);
                double dva[H2D_MAX_MAT];
                if (ax) split_flux(c, cdi, cdj, blo, wlo, bhi, whi, dvol, dva);
                else split_flux(c, cdi, cdj, wlo, blo, whi, bhi, dvol, dva);
                double dmtot = 0.0;
                for (int a = 0; a < nmat; ++a) {
                    if (dva[a] == 0.0) continue;
                    int ord = order;
                    if (ord == 2 && nmat >= 2 && c->cfg.interface_degrade && !pure_1d(c, a, ax, ia_d, ic)) ord = 1;
                    double rf, ef;
                    if (ord <= 1) {
                        rf = A(c->rho[a], cdi, cdj);
                        ef = A(w->e[a], cdi, cdj);
                    } else if (c->cfg.corner == H2D_CORNER_MULTID) { /* multid_faces, remap.cpp:840,889-894 */
                        double sr[3][3], se[3][3], xlx[3][3], xly[3][3];
                        for (int q = 0; q < 3; ++q)
                            for (int p = 0; p < 3; ++p) {
                                sr[p][q] = A(c->rho[a], cdi + p - 1, cdj + q - 1);
                                se[p][q] = A(w->e[a], cdi + p - 1, cdj + q - 1);
                                xlx[p][q] = VX(c->xlag2, cdi + p - 1, cdj + q - 1);
                                xly[p][q] = VY(c->xlag2, cdi + p - 1, cdj + q - 1);
                            }
                        const double bcx = ax ? 0.5 * (blo + bhi) : 0.5 * (wlo + whi);
                        const double bcy = ax ? 0.5 * (wlo + whi) : 0.5 * (blo + bhi);
                        const plane_t pr = multid_plane(c, sr, xlx, xly), pe = multid_plane(c, se, xlx, xly);
                        rf = plane_eval(&pr, bcx, bcy);
                        ef = plane_eval(&pe, bcx, bcy);
                    } else {
                        double sr[3], se[3], sxp[3];
                        for (int d = -1; d <= 1; ++d) {
                            const int ci = ax ? ia_d + d : ic, cj = ax ? ic : ia_d + d;
                            sr[d + 1] = A(c->rho[a], ci, cj);
                            se[d + 1] = A(w->e[a], ci, cj);
                            sxp[d + 1] = A(gxl, ia_d + d, ic);
                        }
                        rf = face_value2(c, sr, sxp, sgn, A(gwl, ia_d, ic), A(gfd, ia, ic));
                        ef = face_value2(c, se, sxp, sgn, A(gwl, ia_d, ic), A(gfd, ia, ic));
                    }
                    const double dm = rf * dva[a];
                    const double dme = rf * ef * dva[a];
                    dmtot += dm;
                    if (ax) {
                        apply_cell(c, c->vola, a, ia - 1, ic, -dm, -dme, -dva[a]);
                        apply_cell(c, c->vola, a, ia, ic, dm, dme, dva[a]);
                    } else {
                        apply_cell(c, c->vola, a, ic, ia - 1, -dm, -dme, -dva[a]);
                        apply_cell(c, c->vola, a, ic, ia, dm, dme, dva[a]);
                    }
                }
                A(dmf, ia, ic) = dmtot;
            }
    }
    face_flux_ghosts(c->dmx, nx, ny, c->per_x, c->per_y);
    face_flux_ghosts(c->dmy, ny, nx, c->per_y, c->per_x);

    /* corner fluxes, remap.cpp:923-988 */
    fzero(c->dmc);
    for (int j = 0; j <= ny; ++j)
        for (int i = 0; i <= nx; ++i) {
            A(c->dmc, i, j) = 0.0;
            const double cdv = A(c->cf_dv, i, j);
            if (cdv == 0.0) continue;
            const int sx = A(c->cf_sx, i, j), sy = A(c->cf_sy, i, j);
            const int di = sx > 0 ? i - 1 : i, dj = sy > 0 ? j - 1 : j;
            const int ri = sx > 0 ? i : i - 1, rj = sy > 0 ? j : j - 1;
            const double npx = x0 + i * dx, npy = y0 + j * dy;
            const double ddx = DX_(i, j), ddy = DY_(i, j);
            const double blox = ref_min(npx, npx + ddx), bloy = ref_min(npy, npy + ddy);
            const double bhix = ref_max(npx, npx + ddx), bhiy = ref_max(npy, npy + ddy);
            double dva[H2D_MAX_MAT];
            split_flux(c, di, dj, blox, bloy, bhix, bhiy, cdv, dva);
            const double lwx = A(c->wlx, di, dj), lwy = A(c->wly, dj, di);
            kin_t kin; /* remap.cpp:944-956 */
            kin.dxp = ddx;
            kin.dyp = ddy;
            kin.lag_wx = lwx;
            kin.lag_wy = lwy;
            {
                const int fxj = sy > 0 ? j - 1 : j, fyi = sx > 0 ? i - 1 : i;
                kin.sgn_fx = A(c->fx_dv, i, fxj) >= 0.0 ? 1.0 : -1.0;
                kin.u_fx_dt = A(c->fdx, i, fxj);
                kin.sgn_fy = A(c->fy_dv, fyi, j) >= 0.0 ? 1.0 : -1.0;
                kin.u_fy_dt = A(c->fdy, j, fyi);
                kin.erx = 0.5 * (blox + bhix) - VX(c->xlag2, di, dj);
                kin.ery = 0.5 * (bloy + bhiy) - VY(c->xlag2, di, dj);
            }
            double dmtot = 0.0;
            for (int a = 0; a < nmat; ++a) {
                if (dva[a] == 0.0) continue;
                int scheme = c->cfg.corner; /* remap.cpp:960-963 */
                if (order <= 1) scheme = H2D_CORNER_UPWIND;
                if (scheme != H2D_CORNER_UPWIND && nmat >= 2 && c->cfg.interface_degrade && !pure_3x3(c, a, di, dj))
                    scheme = H2D_CORNER_UPWIND;
                const int lin = scheme != H2D_CORNER_UPWIND;
                double rf, ef;
                if (!lin) {
                    rf = A(c->rho[a], di, dj);
                    ef = A(w->e[a], di, dj);
                } else {
                    double sr[3][3], se[3][3], xlx[3][3], xly[3][3];
                    for (int q = 0; q < 3; ++q)
                        for (int p = 0; p < 3; ++p) {
                            sr[p][q] = A(c->rho[a], di + p - 1, dj + q - 1);
                            se[p][q] = A(w->e[a], di + p - 1, dj + q - 1);
                            xlx[p][q] = VX(c->xlag2, di + p - 1, dj + q - 1);
                            xly[p][q] = VY(c->xlag2, di + p - 1, dj + q - 1);
                        }
                    rf = ref_max(corner_value(c, scheme, sr, xlx, xly, &kin), 0.0);
                    ef = corner_value(c, scheme, se, xlx, xly, &kin);
                }
                const double dm = rf * dva[a];
                const double dme = rf * ef * dva[a];
                dmtot += dm;
                apply_cell(c, c->vola, a, di, dj, -dm, -dme, -dva[a]);
                apply_cell(c, c->vola, a, ri, rj, dm, dme, dva[a]);
            }
            A(c->dmc, i, j) = dmtot;
        }
    for (int i = 0; i <= nx; ++i) A(c->dmc, i, -1) = c->per_y ? A(c->dmc, i, ny - 1) : A(c->dmc, i, 1);
    for (int j = -1; j <= ny; ++j) A(c->dmc, -1, j) = c->per_x ? A(c->dmc, nx - 1, j) : A(c->dmc, 1, j);

    fcopy(c->mcell_lag, w->mcell);
    finalize_cells(c);

    if (remap_velocity) {
        vzero(c->acc);
        dual_face_pass(c, 1, c->dmx, dt);
        dual_face_pass(c, 0, c->dmy, dt);
        /* dual corners, remap.cpp:1000-1069 */
        const int iuniq = c->per_x ? nx - 1 : nx, juniq = c->per_y ? ny - 1 : ny;
        for (int j = 0; j <= juniq; ++j)
            for (int i = 0; i <= iuniq; ++i)
                for (int pr = 0; pr < 2; ++pr) {
                    const int sx = 1, sy = pr == 0 ? 1 : -1;
                    const int pi = i + sx, pj = j + sy;
                    if (!c->per_x && (pi < 0 || pi > nx)) continue;
                    if (!c->per_y && (pj < 0 || pj > ny)) continue;
                    double sc[4];
                    const int qi[4] = {i, i + sx, i, i + sx}, qj[4] = {j, j, j + sy, j + sy};
                    for (int q = 0; q < 4; ++q) {
                        const double cdv = A(c->cf_dv, qi[q], qj[q]), dmcv = A(c->dmc, qi[q], qj[q]);
                        const int csx = A(c->cf_sx, qi[q], qj[q]), csy = A(c->cf_sy, qi[q], qj[q]);
                        sc[q] = 0.0;
                        if (cdv == 0.0 || dmcv == 0.0) continue;
                        if (csx == sx && csy == sy) sc[q] = -dmcv;
                        else if (csx == -sx && csy == -sy) sc[q] = dmcv;
                    }
                    const double F = 0.25 * (sc[0] + sc[1] + sc[2] + sc[3]);
                    if (F == 0.0) continue;
                    const int incoming = F > 0.0;
                    const int di = incoming ? pi : i, dj = incoming ? pj : j;
                    const int wi = wrapi(di, c->per_x ? nx : nx + 1, c->per_x);
                    const int wj = wrapi(dj, c->per_y ? ny : ny + 1, c->per_y);
                    double ufx, ufy;
                    if (!(c->cfg.corner != H2D_CORNER_UPWIND && order > 1)) { /* remap.cpp:1025-1029 */
                        ufx = VX(w->u, wi, wj);
                        ufy = VY(w->u, wi, wj);
                    } else {
                        const int ci = wrapi(i < pi ? i : pi, nx, c->per_x);
                        const int cj = wrapi(j < pj ? j : pj, ny, c->per_y);
                        const double mdx = VX(c->xlag2, ci, cj) - (x0 + (ci + 0.5) * dx);
                        const double mdy = VY(c->xlag2, ci, cj) - (y0 + (cj + 0.5) * dy);
                        const double dirx = incoming ? -sx : sx, diry = incoming ? -sy : sy;
                        const double dxp = dirx * ref_max(fabs(mdx), 1e-300);
                        const double dyp = diry * ref_max(fabs(mdy), 1e-300);
                        const double lwx = dx + 0.5 * (DX_(wi + 1, wj) - DX_(wi - 1, wj));
                        const double lwy = dy + 0.5 * (DY_(wi, wj + 1) - DY_(wi, wj - 1));
                        double ax_[3][3], ay_[3][3], xlx[3][3], xly[3][3];
                        for (int q = 0; q < 3; ++q)
                            for (int p = 0; p < 3; ++p) {
                                const int ni = wi + p - 1, nj = wj + q - 1;
                                ax_[p][q] = VX(w->u, ni, nj);
                                ay_[p][q] = VY(w->u, ni, nj);
                                xlx[p][q] = (x0 + ni * dx) + DX_(ni, nj);
                                xly[p][q] = (y0 + nj * dy) + DY_(ni, nj);
                            }
                        kin_t kin; /* remap.cpp:1036-1052 */
                        kin.dxp = dxp;
                        kin.dyp = dyp;
                        kin.lag_wx = lwx;
                        kin.lag_wy = lwy;
                        kin.sgn_fx = dirx;
                        kin.u_fx_dt = mdx;
                        kin.sgn_fy = diry;
                        kin.u_fy_dt = mdy;
                        kin.erx = ((x0 + (ci + 0.5) * dx) + 0.5 * mdx) - ((x0 + wi * dx) + DX_(wi, wj));
                        kin.ery = ((y0 + (cj + 0.5) * dy) + 0.5 * mdy) - ((y0 + wj * dy) + DY_(wi, wj));
                        ufx = corner_value(c, c->cfg.corner, ax_, xlx, xly, &kin);
                        ufy = corner_value(c, c->cfg.corner, ay_, xlx, xly, &kin);
                    }
                    acc_add(c, i, j, ufx * F, ufy * F);
                    acc_add(c, pi, pj, ufx * -F, ufy * -F);
                }
        apply_dual_update(c);
    }
    /* refresh_normals_impl, remap.cpp:102-114 */
    if (nmat >= 2) refresh_normals(c, w->k, w->normals);
#undef DX_
#undef DY_
}

/* direct_pass, remap.cpp:593-724: the unsplit one-step remap through the
 * faces only (no corner fluxes), each axis with its own directionally
 * displaced interface; dual faces only on the momentum side. */
static void direct_pass(ctx_t* c, double dt, int remap_velocity) {
    work_t* w = &c->w;
    const int nx = c->nx, ny = c->ny, nmat = c->nmat;
    const double cv = c->cv, dx = c->dx, dy = c->dy, x0 = c->x0, y0 = c->y0;
    const int order = c->cfg.face_order;
    vfld uh = c->u_half;
    /* make_axis_geom X and Y, remap.cpp:296-322 */
    for (int ic = -NG; ic < ny + NG; ++ic)
        for (int ia = -NG; ia <= nx + NG; ++ia)
            A(c->fdx, ia, ic) = 0.5 * (VX(uh, ia, ic) + VX(uh, ia, ic + 1)) * dt;
    for (int ic = -NG; ic < ny + NG; ++ic)
        for (int ia = -NG; ia < nx + NG; ++ia) {
            const double dl = A(c->fdx, ia, ic), dr = A(c->fdx, ia + 1, ic);
            A(c->xlcx, ia, ic) = x0 + (ia + 0.5) * dx + 0.5 * (dl + dr);
            A(c->wlx, ia, ic) = dx + (dr - dl);
        }
    for (int ic = -NG; ic < nx + NG; ++ic)
        for (int ia = -NG; ia <= ny + NG; ++ia)
            A(c->fdy, ia, ic) = 0.5 * (VY(uh, ic, ia) + VY(uh, ic + 1, ia)) * dt;
    for (int ic = -NG; ic < nx + NG; ++ic)
        for (int ia = -NG; ia < ny + NG; ++ia) {
            const double dl = A(c->fdy, ia, ic), dr = A(c->fdy, ia + 1, ic);
            A(c->xlcy, ia, ic) = y0 + (ia + 0.5) * dy + 0.5 * (dl + dr);
            A(c->wly, ia, ic) = dy + (dr - dl);
        }
    /* Lagrangian volume and densities, remap.cpp:601-614 */
    for (int j = -NG; j < ny + NG; ++j)
        for (int i = -NG; i < nx + NG; ++i) {
            const double v = cv + (A(c->fdx, i + 1, j) - A(c->fdx, i, j)) * dy + (A(c->fdy, j + 1, i) - A(c->fdy, j, i)) * dx;
            if (v <= 0.0) raise_err(c, H2D_ERR_CFL, i, j, "collapsed Lagrangian cell");
            A(c->vlag, i, j) = v;
            for (int a = 0; a < nmat; ++a) {
                const double ka = A(w->k[a], i, j);
                A(c->rho[a], i, j) = ka > 0.0 ? A(w->m[a], i, j) / (ka * v) : 0.0;
            }
        }
    for (int a = 0; a < nmat; ++a) {
        fzero(c->vola[a]);
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) A(c->vola[a], i, j) = A(w->k[a], i, j) * A(c->vlag, i, j);
    }
    /* face fluxes per axis, remap.cpp:656-713, each with the interfaces of
     * its own displaced rectangles (remap.cpp:616-640) */
    fzero(c->dmx);
    fzero(c->dmy);
    for (int axis = 0; axis < 2; ++axis) {
        const int ax = axis == 0;
        izero(c->if_mixed);
        if (nmat >= 2)
            for (int j = -NG; j < ny + NG; ++j)
                for (int i = -NG; i < nx + NG; ++i) {
                    double k0 = A(w->k[0], i, j);
                    if (nmat == 3) {
                        double k[3];
                        kcell3(w->k, i, j, k);
                        if (!mixed3(k)) continue;
                        int lo, hi;
                        pair3(k, &lo, &hi);
                        A(c->if_lo, i, j) = lo;
                        A(c->if_hi, i, j) = hi;
                        k0 = k[3 - lo - hi] > 0.0 ? k[lo] / (k[lo] + k[hi]) : k[lo];
                    } else if (!is_mixed(k0)) {
                        continue;
                    }
                    const double cx = x0 + (i + 0.5) * dx, cy = y0 + (j + 0.5) * dy;
                    const double hx = 0.5 * dx, hy = 0.5 * dy;
                    double lox, loy, hix, hiy;
                    if (ax) {
                        lox = cx - hx + A(c->fdx, i, j); loy = cy - hy;
                        hix = cx + hx + A(c->fdx, i + 1, j); hiy = cy + hy;
                    } else {
                        lox = cx - hx; loy = cy - hy + A(c->fdy, j, i);
                        hix = cx + hx; hiy = cy + hy + A(c->fdy, j + 1, i);
                    }
                    const double nxv = VX(w->normals, i, j), nyv = VY(w->normals, i, j);
                    A(c->if_mixed, i, j) = 1;
                    A(c->if_lox, i, j) = lox; A(c->if_loy, i, j) = loy;
                    A(c->if_hix, i, j) = hix; A(c->if_hiy, i, j) = hiy;
                    A(c->if_nx, i, j) = nxv; A(c->if_ny, i, j) = nyv;
                    A(c->if_d, i, j) = place_interface(k0, nxv, nyv, lox, loy, hix, hiy);
                }
        const int na = ax ? nx : ny, nc = ax ? ny : nx;
        fld gfd = ax ? c->fdx : c->fdy, gxl = ax ? c->xlcx : c->xlcy, gwl = ax ? c->wlx : c->wly;
        fld dmf = ax ? c->dmx : c->dmy;
        const double wc = ax ? dy : dx;
        for (int ic = 0; ic < nc; ++ic)
            for (int ia = 0; ia <= na; ++ia) {
                const double fd = A(gfd, ia, ic);
                const double dvol = fd * wc;
                A(dmf, ia, ic) = 0.0;
                if (dvol == 0.0) continue;
                if (fabs(dvol) > CFL_FRAC * cv)
                    raise_err(c, H2D_ERR_CFL, ax ? ia : ic, ax ? ic : ia, "CFL violation at face");
                const int ia_d = dvol > 0.0 ? ia - 1 : ia;
                const double sgn = dvol > 0.0 ? 1.0 : -1.0;
                const int cdi = ax ? ia_d : ic, cdj = ax ? ic : ia_d;
                /* face_flux_box, remap.cpp:325-334 */
                double blox, bloy, bhix, bhiy;
                if (ax) {
                    const double xf = x0 + ia * dx;
                    blox = ref_min(xf, xf + fd); bhix = ref_max(xf, xf + fd);
                    bloy = y0 + ic * dy; bhiy = y0 + (ic + 1) * dy;
                } else {
                    const double yf = y0 + ia * dy;
                    blox = x0 + ic * dx; bhix = x0 + (ic + 1) * dx;
                    bloy = ref_min(yf, yf + fd); bhiy = ref_max(yf, yf + fd);
                }
                double dva[H2D_MAX_MAT];
                split_flux(c, cdi, cdj, blox, bloy, bhix, bhiy, dvol, dva);
                double dmtot = 0.0;
                for (int a = 0; a < nmat; ++a) {
                    if (dva[a] == 0.0) continue;
                    int ord = order;
                    if (ord == 2 && nmat >= 2 && c->cfg.interface_degrade && !pure_1d(c, a, ax, ia_d, ic)) ord = 1;
                    double rf, ef;
                    if (ord <= 1) {
                        rf = A(c->rho[a], cdi, cdj);
                        ef = A(w->e[a], cdi, cdj);
                    } else {
                        double sr[3], se[3], sxp[3];
                        for (int d = -1; d <= 1; ++d) {
                            const int ci = ax ? ia_d + d : ic, cj = ax ? ic : ia_d + d;
                            sr[d + 1] = A(c->rho[a], ci, cj);
                            se[d + 1] = A(w->e[a], ci, cj);
                            sxp[d + 1] = A(gxl, ia_d + d, ic);
                        }
                        rf = face_value2(c, sr, sxp, sgn, A(gwl, ia_d, ic), fd);
                        ef = face_value2(c, se, sxp, sgn, A(gwl, ia_d, ic), fd);
                    }
                    const double dm = rf * dva[a];
                    const double dme = rf * ef * dva[a];
                    dmtot += dm;
                    if (ax) {
                        apply_cell(c, c->vola, a, ia - 1, ic, -dm, -dme, -dva[a]);
                        apply_cell(c, c->vola, a, ia, ic, dm, dme, dva[a]);
                    } else {
                        apply_cell(c, c->vola, a, ic, ia - 1, -dm, -dme, -dva[a]);
                        apply_cell(c, c->vola, a, ic, ia, dm, dme, dva[a]);
                    }
                }
                A(dmf, ia, ic) = dmtot;
            }
    }
    face_flux_ghosts(c->dmx, nx, ny, c->per_x, c->per_y);
    face_flux_ghosts(c->dmy, ny, nx, c->per_y, c->per_x);
    fcopy(c->mcell_lag, w->mcell);
    finalize_cells(c);
    if (remap_velocity) {
        vzero(c->acc);
        dual_face_pass(c, 1, c->dmx, dt);
        dual_face_pass(c, 0, c->dmy, dt);
        apply_dual_update(c);
    }
    if (nmat >= 2) refresh_normals(c, w->k, w->normals);
}

/* directional_pass, remap.cpp:469-589: the X (axis_x = 1) or Y remap of the
 * alternating-direction (AD) split scheme.  (along, cross) layouts as cf_pass:
 * X: (ia, ic) = (i, j); Y: (ia, ic) = (j, i). */
static void directional_pass(ctx_t* c, double dt, int axis_x, int remap_velocity) {
    work_t* w = &c->w;
    const int nx = c->nx, ny = c->ny, nmat = c->nmat;
    const double cv = c->cv, dx = c->dx, dy = c->dy, x0 = c->x0, y0 = c->y0;
    const int order = c->cfg.face_order;
    const int na = axis_x ? nx : ny, nc = axis_x ? ny : nx;
    const double wa = axis_x ? dx : dy, wc = axis_x ? dy : dx;
    const int per_a = axis_x ? c->per_x : c->per_y, per_c = axis_x ? c->per_y : c->per_x;
    fld gfd = axis_x ? c->fdx : c->fdy, gxl = axis_x ? c->xlcx : c->xlcy, gwl = axis_x ? c->wlx : c->wly;
    fld dmf = axis_x ? c->dmx : c->dmy;
    vfld uh = c->u_half;
#define CI(ia, ic) (axis_x ? (ia) : (ic))
#define CJ(ia, ic) (axis_x ? (ic) : (ia))
    /* make_axis_geom, remap.cpp:296-322 */
    for (int ic = -NG; ic < nc + NG; ++ic)
        for (int ia = -NG; ia <= na + NG; ++ia) {
            const double u0 = axis_x ? VX(uh, ia, ic) : VY(uh, ic, ia);
            const double u1 = axis_x ? VX(uh, ia, ic + 1) : VY(uh, ic + 1, ia);
            A(gfd, ia, ic) = 0.5 * (u0 + u1) * dt;
        }
    const double origin = axis_x ? x0 : y0;
    for (int ic = -NG; ic < nc + NG; ++ic)
        for (int ia = -NG; ia < na + NG; ++ia) {
            const double dl = A(gfd, ia, ic), dr = A(gfd, ia + 1, ic);
            A(gxl, ia, ic) = origin + (ia + 0.5) * wa + 0.5 * (dl + dr);
            A(gwl, ia, ic) = wa + (dr - dl);
        }
    /* 1D Lagrangian volumes and densities, remap.cpp:478-491 */
    for (int ic = -NG; ic < nc + NG; ++ic)
        for (int ia = -NG; ia < na + NG; ++ia) {
            const int i = CI(ia, ic), j = CJ(ia, ic);
            const double v = cv + (A(gfd, ia + 1, ic) - A(gfd, ia, ic)) * wc;
            if (v <= 0.0) raise_err(c, H2D_ERR_CFL, i, j, "collapsed Lagrangian cell");
            A(c->vlag, i, j) = v;
            for (int a = 0; a < nmat; ++a) {
                const double ka = A(w->k[a], i, j);
                A(c->rho[a], i, j) = ka > 0.0 ? A(w->m[a], i, j) / (ka * v) : 0.0;
            }
        }
    /* interfaces on the 1D-displaced rectangles, remap.cpp:493-514 */
    izero(c->if_mixed);
    if (nmat == 2)
        for (int ic = -NG; ic < nc + NG; ++ic)
            for (int ia = -NG; ia < na + NG; ++ia) {
                const int i = CI(ia, ic), j = CJ(ia, ic);
                const double k0 = A(w->k[0], i, j);
                if (!is_mixed(k0)) continue;
                const double cx = x0 + (i + 0.5) * dx, cy = y0 + (j + 0.5) * dy;
                const double dl = A(gfd, ia, ic), dr = A(gfd, ia + 1, ic);
                double lox, loy, hix, hiy;
                if (axis_x) {
                    lox = cx - 0.5 * dx + dl; loy = cy - 0.5 * dy;
                    hix = cx + 0.5 * dx + dr; hiy = cy + 0.5 * dy;
                } else {
                    lox = cx - 0.5 * dx; loy = cy - 0.5 * dy + dl;
                    hix = cx + 0.5 * dx; hiy = cy + 0.5 * dy + dr;
                }
                const double nxv = VX(w->normals, i, j), nyv = VY(w->normals, i, j);
                A(c->if_mixed, i, j) = 1;
                A(c->if_lox, i, j) = lox; A(c->if_loy, i, j) = loy;
                A(c->if_hix, i, j) = hix; A(c->if_hiy, i, j) = hiy;
                A(c->if_nx, i, j) = nxv; A(c->if_ny, i, j) = nyv;
                A(c->if_d, i, j) = place_interface(k0, nxv, nyv, lox, loy, hix, hiy);
            }
    for (int a = 0; a < nmat; ++a) {
        fzero(c->vola[a]);
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) A(c->vola[a], i, j) = A(w->k[a], i, j) * A(c->vlag, i, j);
    }
    /* face fluxes, remap.cpp:526-577 */
    fzero(dmf);
    for (int ic = 0; ic < nc; ++ic)
        for (int ia = 0; ia <= na; ++ia) {
            const double dvol = A(gfd, ia, ic) * wc;
            A(dmf, ia, ic) = 0.0;
            if (dvol == 0.0) continue;
            if (fabs(dvol) > CFL_FRAC * cv) raise_err(c, H2D_ERR_CFL, CI(ia, ic), CJ(ia, ic), "CFL violation at face");
            const int ia_d = dvol > 0.0 ? ia - 1 : ia;
            const double sgn = dvol > 0.0 ? 1.0 : -1.0;
            const int cdi = CI(ia_d, ic), cdj = CJ(ia_d, ic);
            /* face_flux_box, remap.cpp:325-334 */
            const double d = A(gfd, ia, ic);
            double blox, bloy, bhix, bhiy;
            if (axis_x) {
                const double xf = x0 + ia * dx;
                blox = ref_min(xf, xf + d); bloy = y0 + ic * dy;
                bhix = ref_max(xf, xf + d); bhiy = y0 + (ic + 1) * dy;
            } else {
                const double yf = y0 + ia * dy;
                blox = x0 + ic * dx; bloy = ref_min(yf, yf + d);
                bhix = x0 + (ic + 1) * dx; bhiy = ref_max(yf, yf + d);
            }
            double dva[H2D_MAX_MAT];
            split_flux(c, cdi, cdj, blox, bloy, bhix, bhiy, dvol, dva);
            double dmtot = 0.0;
            for (int a = 0; a < nmat; ++a) {
                if (dva[a] == 0.0) continue;
                int ord = order;
                if (ord == 2 && nmat == 2 && c->cfg.interface_degrade && !pure_1d(c, a, axis_x, ia_d, ic)) ord = 1;
                double rf, ef;
                if (ord <= 1) {
                    rf = A(c->rho[a], cdi, cdj);
                    ef = A(w->e[a], cdi, cdj);
                } else {
                    double sr[3], se[3], sxp[3];
                    for (int q = -1; q <= 1; ++q) {
                        const int ci = CI(ia_d + q, ic), cj = CJ(ia_d + q, ic);
                        sr[q + 1] = A(c->rho[a], ci, cj);
                        se[q + 1] = A(w->e[a], ci, cj);
                        sxp[q + 1] = A(gxl, ia_d + q, ic);
                    }
                    rf = face_value2(c, sr, sxp, sgn, A(gwl, ia_d, ic), A(gfd, ia, ic));
                    ef = face_value2(c, se, sxp, sgn, A(gwl, ia_d, ic), A(gfd, ia, ic));
                }
                const double dm = rf * dva[a];
                const double dme = rf * ef * dva[a];
                dmtot += dm;
                apply_cell(c, c->vola, a, CI(ia - 1, ic), CJ(ia - 1, ic), -dm, -dme, -dva[a]);
                apply_cell(c, c->vola, a, CI(ia, ic), CJ(ia, ic), dm, dme, dva[a]);
            }
            A(dmf, ia, ic) = dmtot;
        }
    face_flux_ghosts(dmf, na, nc, per_a, per_c);
#undef CI
#undef CJ
    fcopy(c->mcell_lag, w->mcell);
    finalize_cells(c);
    if (remap_velocity) {
        vzero(c->acc);
        dual_face_pass(c, axis_x, dmf, dt);
        apply_dual_update(c);
    }
    /* refresh_normals_impl, remap.cpp:102-114 */
    if (nmat == 2) {
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                if (!is_mixed(A(w->k[0], i, j))) continue;
                double nxv, nyv;
                if (youngs_normal(c, w->k[1], i, j, &nxv, &nyv)) {
                    VX(w->normals, i, j) = nxv;
                    VY(w->normals, i, j) = nyv;
                }
            }
        ghost_cells_v(c, w->normals);
    }
}

/* assemble_state, remap.cpp:1075-1089 (make_state defaults, state.cpp:5-23) */
static void assemble_state(ctx_t* c, double dt) {
    work_t* w = &c->w;
    for (int a = 0; a < H2D_MAX_MAT; ++a) {
        if (a < c->nmat) {
            fcopy(c->m[a], w->m[a]);
            fcopy(c->e[a], w->e[a]);
            fcopy(c->k[a], w->k[a]);
        } else {
            fzero(c->m[a]);
            fzero(c->e[a]);
            ffill(c->k[a], a == 0 ? 1.0 : 0.0);
        }
    }
    vcopy(c->nrm, w->normals);
    vcopy(c->u, w->u);
    c->step += 1;
    c->time += dt;
    /* fill_ghosts, state.cpp:110-118 */
    for (int a = 0; a < c->nmat; ++a) {
        ghost_cells(c, c->m[a]);
        ghost_cells(c, c->e[a]);
        ghost_cells(c, c->k[a]);
    }
    ghost_cells_v(c, c->nrm);
    ghost_nodes(c, c->u);
    sync_derived(c);
}

/* ---------------------------------------------------------------- C-ABI */
int h2do_abi_version(void) { return H2D_ABI_VERSION; }

static void ctx_free(ctx_t* c) {
    if (!c) return;
    /* every fld/vfld/ifld member is a single calloc'd block */
    fld* fl[] = {&c->m[0], &c->m[1], &c->e[0], &c->e[1], &c->k[0], &c->k[1], &c->vol, &c->m_mix, &c->e_mix,
                 &c->rho_mix, &c->p_mix, &c->e_lag[0], &c->e_lag[1], &c->vol_lag, &c->q, &c->vol_half,
                 &c->e_half[0], &c->e_half[1], &c->p_half[0], &c->p_half[1], &c->p_mix_half,
                 &c->w.m[0], &c->w.m[1], &c->w.me[0], &c->w.me[1], &c->w.e[0], &c->w.e[1], &c->w.k[0],
                 &c->w.k[1], &c->w.mcell, &c->fdx, &c->fdy, &c->xlcx, &c->xlcy, &c->wlx, &c->wly,
                 &c->fx_dv, &c->fx_lo, &c->fx_hi, &c->fy_dv, &c->fy_lo, &c->fy_hi, &c->cf_dv, &c->vlag,
                 &c->m[2], &c->e[2], &c->k[2], &c->e_lag[2], &c->e_half[2], &c->p_half[2], &c->w.m[2],
                 &c->w.me[2], &c->w.e[2], &c->w.k[2], &c->rho[2], &c->vola[2],
                 &c->rho[0], &c->rho[1], &c->if_lox, &c->if_loy, &c->if_hix, &c->if_hiy, &c->if_nx,
                 &c->if_ny, &c->if_d, &c->vola[0], &c->vola[1], &c->dmx, &c->dmy, &c->dmc, &c->mcell_lag};
    for (size_t q = 0; q < sizeof fl / sizeof fl[0]; ++q) free(fl[q]->p);
    vfld* vf[] = {&c->nrm, &c->u, &c->u_half, &c->u_lag, &c->dh, &c->w.normals, &c->w.u, &c->xlag2, &c->acc,
                  &c->unew};
    for (size_t q = 0; q < sizeof vf / sizeof vf[0]; ++q) free(vf[q]->p);
    free(c->cf_sx.p);
    free(c->cf_sy.p);
    free(c->if_mixed.p); free(c->if_lo.p); free(c->if_hi.p);
    free(c->sl_i); free(c->sl_j); free(c->sl_a); free(c->sl_m); free(c->sl_me);
    free(c);
}

int h2do_create(const h2d_config* cfg, int device, ctx_t** out) {
    (void)device;
    *out = NULL;
    const h2d_mesh* m = &cfg->mesh;
    if (m->nx < 3 || m->ny < 3) return H2D_ERR_SIM;       /* Mesh::Mesh, mesh.hpp:27 */
    if (m->dx <= 0.0 || m->dy <= 0.0) return H2D_ERR_SIM; /* mesh.hpp:28 */
    if (cfg->nmat < 1 || cfg->nmat > H2D_MAX_MAT) return H2D_ERR_INVALID;
    if (cfg->corner < H2D_CORNER_UPWIND || cfg->corner > H2D_CORNER_MULTID) return H2D_ERR_INVALID;
    ctx_t* c = (ctx_t*)calloc(1, sizeof(ctx_t));
    c->cfg = *cfg;
    const int nx = m->nx, ny = m->ny;
    c->nx = nx; c->ny = ny; c->nmat = cfg->nmat;
    c->dx = m->dx; c->dy = m->dy; c->x0 = m->x0; c->y0 = m->y0;
    c->per_x = m->bc_x == H2D_BC_PERIODIC;
    c->per_y = m->bc_y == H2D_BC_PERIODIC;
    c->cv = m->dx * m->dy;
    for (int a = 0; a < H2D_MAX_MAT; ++a) {
        c->m[a] = fnew(nx, ny); c->e[a] = fnew(nx, ny); c->k[a] = fnew(nx, ny);
        ffill(c->k[a], a == 0 ? 1.0 : 0.0);
        c->e_lag[a] = fnew(nx, ny); c->e_half[a] = fnew(nx, ny); c->p_half[a] = fnew(nx, ny);
        c->w.m[a] = fnew(nx, ny); c->w.me[a] = fnew(nx, ny); c->w.e[a] = fnew(nx, ny); c->w.k[a] = fnew(nx, ny);
        c->rho[a] = fnew(nx, ny); c->vola[a] = fnew(nx, ny);
    }
    c->vol = fnew(nx, ny); ffill(c->vol, c->cv);
    c->m_mix = fnew(nx, ny); c->e_mix = fnew(nx, ny); c->rho_mix = fnew(nx, ny); c->p_mix = fnew(nx, ny);
    c->nrm = vnew(nx, ny);
    for (size_t q = 0; q < fsize(nx, ny); ++q) { c->nrm.p[2 * q] = 1.0; c->nrm.p[2 * q + 1] = 0.0; }
    c->u = vnew(nx + 1, ny + 1);
    c->u_half = vnew(nx + 1, ny + 1); c->u_lag = vnew(nx + 1, ny + 1); c->dh = vnew(nx + 1, ny + 1);
    c->vol_lag = fnew(nx, ny); c->q = fnew(nx, ny); c->vol_half = fnew(nx, ny); c->p_mix_half = fnew(nx, ny);
    c->w.normals = vnew(nx, ny); c->w.mcell = fnew(nx, ny); c->w.u = vnew(nx + 1, ny + 1);
    c->fdx = fnew(nx + 1, ny); c->xlcx = fnew(nx, ny); c->wlx = fnew(nx, ny);
    c->fdy = fnew(ny + 1, nx); c->xlcy = fnew(ny, nx); c->wly = fnew(ny, nx);
    c->fx_dv = fnew(nx + 1, ny); c->fx_lo = fnew(nx + 1, ny); c->fx_hi = fnew(nx + 1, ny);
    c->fy_dv = fnew(nx, ny + 1); c->fy_lo = fnew(nx, ny + 1); c->fy_hi = fnew(nx, ny + 1);
    c->cf_dv = fnew(nx + 1, ny + 1); c->cf_sx = inew(nx + 1, ny + 1); c->cf_sy = inew(nx + 1, ny + 1);
    c->vlag = fnew(nx, ny); c->xlag2 = vnew(nx, ny);
    c->if_mixed = inew(nx, ny); c->if_lo = inew(nx, ny); c->if_hi = inew(nx, ny);
    c->if_lox = fnew(nx, ny); c->if_loy = fnew(nx, ny); c->if_hix = fnew(nx, ny); c->if_hiy = fnew(nx, ny);
    c->if_nx = fnew(nx, ny); c->if_ny = fnew(nx, ny); c->if_d = fnew(nx, ny);
    c->dmx = fnew(nx + 1, ny); c->dmy = fnew(ny + 1, nx); c->dmc = fnew(nx + 1, ny + 1);
    c->mcell_lag = fnew(nx, ny);
    c->acc = vnew(nx + 1, ny + 1); c->unew = vnew(nx + 1, ny + 1);
    *out = c;
    return 0;
}

void h2do_destroy(ctx_t* c) { ctx_free(c); }

static void put(fld f, const double* src) { if (src) memcpy(f.p, src, fsize(f.n1, f.n2) * sizeof(double)); }
static void putv(vfld f, const double* src) { if (src) memcpy(f.p, src, 2 * fsize(f.n1, f.n2) * sizeof(double)); }
static void get(fld f, double* dst) { if (dst) memcpy(dst, f.p, fsize(f.n1, f.n2) * sizeof(double)); }
static void getv(vfld f, double* dst) { if (dst) memcpy(dst, f.p, 2 * fsize(f.n1, f.n2) * sizeof(double)); }

int h2do_upload_state(ctx_t* c, const h2d_state* v) {
    for (int a = 0; a < c->nmat; ++a) { put(c->m[a], v->m[a]); put(c->e[a], v->e[a]); put(c->k[a], v->k[a]); }
    putv(c->nrm, v->iface_normal);
    putv(c->u, v->u);
    c->step = v->step;
    c->time = v->time;
    if (v->vol && v->m_mix && v->e_mix && v->rho_mix && v->p_mix) {
        put(c->vol, v->vol); put(c->m_mix, v->m_mix); put(c->e_mix, v->e_mix);
        put(c->rho_mix, v->rho_mix); put(c->p_mix, v->p_mix);
    } else {
        sync_derived(c);
    }
    c->have_lag = 0;
    return 0;
}

int h2do_download_state(ctx_t* c, h2d_state* v) {
    for (int a = 0; a < c->nmat; ++a) { get(c->m[a], v->m[a]); get(c->e[a], v->e[a]); get(c->k[a], v->k[a]); }
    get(c->vol, v->vol); get(c->m_mix, v->m_mix); get(c->e_mix, v->e_mix);
    get(c->rho_mix, v->rho_mix); get(c->p_mix, v->p_mix);
    getv(c->nrm, v->iface_normal);
    getv(c->u, v->u);
    v->step = c->step;
    v->time = c->time;
    return 0;
}

/* fill_ghosts, state.cpp:110-118 */
int h2do_fill_ghosts(ctx_t* c) {
    for (int a = 0; a < c->nmat; ++a) {
        ghost_cells(c, c->m[a]);
        ghost_cells(c, c->e[a]);
        ghost_cells(c, c->k[a]);
    }
    ghost_cells_v(c, c->nrm);
    ghost_nodes(c, c->u);
    return 0;
}
int h2do_sync_derived(ctx_t* c) {
    sync_derived(c);
    return 0;
}
/* update_interface_normals -> refresh_normals_impl, remap.cpp:1093-1096,102-114 */
int h2do_update_interface_normals(ctx_t* c) {
    if (c->nmat < 2) return 0;
    refresh_normals(c, c->k, c->nrm);
    return 0;
}

int h2do_cfl_dt(ctx_t* c, double cfl, double* dt) {
    if (setjmp(c->jb)) return c->err.kind;
    *dt = cfl_dt(c, cfl);
    return 0;
}

static void lag_out(ctx_t* c, h2d_lagrange* out) {
    if (!out) return;
    getv(c->u_half, out->u_half);
    getv(c->u_lag, out->u_lag);
    for (int a = 0; a < c->nmat; ++a) get(c->e_lag[a], out->e_lag[a]);
    get(c->vol_lag, out->vol_lag);
    get(c->q, out->q);
    out->floor_count = c->floor_count;
}

int h2do_lagrange_step(ctx_t* c, double dt, h2d_lagrange* out) {
    c->have_lag = 0;
    if (setjmp(c->jb)) return c->err.kind;
    predict(c, dt);
    correct(c, dt);
    lag_out(c, out);
    return 0;
}

int h2do_set_lagrange(ctx_t* c, const h2d_lagrange* in) {
    vzero(c->u_half); vzero(c->u_lag); fzero(c->vol_lag); fzero(c->q);
    putv(c->u_half, in->u_half);
    putv(c->u_lag, in->u_lag);
    for (int a = 0; a < c->nmat; ++a) { fzero(c->e_lag[a]); put(c->e_lag[a], in->e_lag[a]); }
    put(c->vol_lag, in->vol_lag);
    put(c->q, in->q);
    c->floor_count = in->floor_count;
    c->have_lag = 1;
    return 0;
}

/* remap_step, remap.cpp:1106-1126 (DirectCF and AD; not Direct) */
int h2do_remap_step(ctx_t* c, double dt, int kind, int x_first, int remap_velocity, h2d_remap_diag* diag) {
    if (kind != H2D_REMAP_DIRECTCF && kind != H2D_REMAP_AD && kind != H2D_REMAP_DIRECT) {
        c->err.kind = H2D_ERR_INVALID;
        snprintf(c->err.what, sizeof c->err.what, "only the DirectCF and AD remaps are implemented");
        return H2D_ERR_INVALID;
    }
    if (!c->have_lag) {
        c->err.kind = H2D_ERR_INVALID;
        snprintf(c->err.what, sizeof c->err.what, "remap_step without a LagrangeResult");
        return H2D_ERR_INVALID;
    }
    if (kind == H2D_REMAP_AD && c->nmat == 3) {
        c->err.kind = H2D_ERR_INVALID;
        snprintf(c->err.what, sizeof c->err.what, "the AD remap has no three-material extension");
        return H2D_ERR_INVALID;
    }
    h2d_remap_diag local;
    if (diag) local = *diag;
    c->diag = diag ? &local : NULL;
    if (setjmp(c->jb)) { c->diag = NULL; return c->err.kind; }
    make_work(c);
    if (kind == H2D_REMAP_DIRECT) {  /* remap.cpp:1109 */
        direct_pass(c, dt, remap_velocity);
    } else if (kind == H2D_REMAP_AD) {  /* remap.cpp:1110-1115 */
        directional_pass(c, dt, x_first ? 1 : 0, remap_velocity);
        directional_pass(c, dt, x_first ? 0 : 1, remap_velocity);
    } else {
        cf_pass(c, dt, remap_velocity);
    }
    assemble_state(c, dt);
    if (diag) *diag = local;
    c->diag = NULL;
    c->have_lag = 0;
    return 0;
}

/* nan_scan, harness.cpp:347-358 */
static void nan_scan(ctx_t* c) {
    for (int j = 0; j < c->ny; ++j)
        for (int i = 0; i < c->nx; ++i)
            if (!isfinite(A(c->m_mix, i, j)) || !isfinite(A(c->e_mix, i, j)) || !isfinite(A(c->p_mix, i, j)))
                raise_err(c, H2D_ERR_SIM, i, j, "non-finite cell state");
    for (int j = 0; j <= c->ny; ++j)
        for (int i = 0; i <= c->nx; ++i)
            if (!isfinite(VX(c->u, i, j)) || !isfinite(VY(c->u, i, j)))
                raise_err(c, H2D_ERR_SIM, i, j, "non-finite velocity");
}

int h2do_step_diag_now(ctx_t* c, double dt, h2d_step_diag* d);

/* run loop, harness.cpp:390-412 (non-kinematic) */
int h2do_run(ctx_t* c, h2d_run_args* a) {
    a->steps_done = 0;
    for (;;) {
        if (!(c->time < a->t_end - 1e-15 * ref_max(1.0, a->t_end))) break;
        if (a->max_steps > 0 && c->step >= a->max_steps) break;
        double dt;
        int rc = h2do_cfl_dt(c, a->cfl, &dt);
        if (rc) return rc;
        dt = ref_min(dt, a->t_end - c->time);
        const int step_now = c->step;
        rc = h2do_lagrange_step(c, dt, NULL);
        if (!rc) {
            a->floor_count += c->floor_count;
            rc = h2do_remap_step(c, dt, a->remap_kind, step_now % 2 == 0, 1, &a->diag);
        }
        if (rc) {
            c->err.step = step_now;
            c->err.in_step = 1;
            return rc;
        }
        if (setjmp(c->jb)) {
            c->err.step = c->step;
            /* SimError::format appends " step N" for nan_scan's located throw */
            size_t L = strlen(c->err.what);
            snprintf(c->err.what + L, sizeof c->err.what - L, " step %d", c->step);
            return c->err.kind;
        }
        nan_scan(c);
        if (a->dt_log && a->steps_done < a->dt_log_cap) a->dt_log[a->steps_done] = dt;
        if (a->series && a->steps_done < a->series_cap) h2do_step_diag_now(c, dt, &a->series[a->steps_done]);
        a->steps_done += 1;
    }
    return 0;
}

/* compute_totals, state.cpp:145-160 */
static void totals7(ctx_t* c, double out[7]);
int h2do_totals(ctx_t* c, double out[6]) {
    double t[7];
    totals7(c, t);
    memcpy(out, t, 6 * sizeof(double));
    return 0;
}
/* {mass, mass_mat0, mass_mat1, momentum x, momentum y, internal energy, mass_mat2} */
static void totals7(ctx_t* c, double out[7]) {
    double mass = 0.0, ie = 0.0, mm[3] = {0.0, 0.0, 0.0}, px = 0.0, py = 0.0;
    for (int j = 0; j < c->ny; ++j)
        for (int i = 0; i < c->nx; ++i) {
            mass += A(c->m_mix, i, j);
            ie += A(c->m_mix, i, j) * A(c->e_mix, i, j);
            for (int a = 0; a < c->nmat; ++a) mm[a] += A(c->m[a], i, j);
        }
    const int ie_ = c->per_x ? c->nx - 1 : c->nx, je_ = c->per_y ? c->ny - 1 : c->ny;
    for (int j = 0; j <= je_; ++j)
        for (int i = 0; i <= ie_; ++i) {
            const double mp = 0.25 * (A(c->m_mix, i - 1, j - 1) + A(c->m_mix, i, j - 1) + A(c->m_mix, i - 1, j) +
                                      A(c->m_mix, i, j));
            px += mp * VX(c->u, i, j);
            py += mp * VY(c->u, i, j);
        }
    out[0] = mass; out[1] = mm[0]; out[2] = mm[1]; out[3] = px; out[4] = py; out[5] = ie; out[6] = mm[2];
}

/* make_diag, harness.cpp:360-376 */
int h2do_step_diag_now(ctx_t* c, double dt, h2d_step_diag* d) {
    double t[7];
    totals7(c, t);
    memset(d, 0, sizeof *d);
    d->step = c->step;
    d->t = c->time;
    d->dt = dt;
    d->mass = t[0];
    d->mass_mat[0] = t[1];
    d->mass_mat[1] = t[2];
    d->mass_mat[2] = t[6];
    d->momentum_x = t[3];
    d->momentum_y = t[4];
    d->internal_energy = t[5];
    d->min_rho = d->max_rho = A(c->rho_mix, 0, 0);
    d->min_p = d->max_p = A(c->p_mix, 0, 0);
    for (int j = 0; j < c->ny; ++j)
        for (int i = 0; i < c->nx; ++i) {
            d->min_rho = ref_min(d->min_rho, A(c->rho_mix, i, j));
            d->max_rho = ref_max(d->max_rho, A(c->rho_mix, i, j));
            d->min_p = ref_min(d->min_p, A(c->p_mix, i, j));
            d->max_p = ref_max(d->max_p, A(c->p_mix, i, j));
        }
    return 0;
}

int h2do_last_error(ctx_t* c, h2d_error* e) {
    *e = c->err;
    return 0;
}

/* scalar probes (oracle tests only) */
double h2do_van_leer(double r) { return van_leer(r); }
double h2do_clipped_fraction(double w, double h, double nx, double ny, double d) {
    return clipped_fraction(w, h, nx, ny, d);
}
double h2do_place_interface(double frac, double nx, double ny, double lox, double loy, double hix, double hiy) {
    return place_interface(frac, nx, ny, lox, loy, hix, hiy);
}

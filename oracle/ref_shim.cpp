// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle).  Exposes the reference
// library itself (/root/reference/proj, compiled unmodified from its own
// sources by oracle/Makefile into oracle/_ref/) through the h2d C-ABI under
// the `h2dr_` prefix, so the pytest suite can run the very same call
// sequence against the reference, the C restatement (h2do_) and the CUDA
// product (h2d_).  Nothing in the product links or loads this file.
//
// Every entry forwards to the reference function named in include/h2d.h.
#include "../include/h2d.h"

#include "hydro/harness.hpp"
#include "hydro/io.hpp"
#include "hydro/config.hpp"
#include "hydro/lagrange.hpp"
#include "hydro/remap.hpp"
#include "hydro/state.hpp"
#include "hydro/vof.hpp"
#include "hydro/reconstruct.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <sstream>
#include <string>

using namespace hydro;

struct h2dr_ctx {
    MaterialSet mats;
    PseudoViscosityParams pv;
    ReconConfig rc;
    State s;
    LagrangeResult lag;
    bool have_lag = false;
    h2d_error err{};
};

namespace {

Mesh to_mesh(const h2d_mesh& m) {
    return Mesh(m.nx, m.ny, m.dx, m.dy, m.x0, m.y0,
                m.bc_x == H2D_BC_WALL ? BoundaryKind::Wall : BoundaryKind::Periodic,
                m.bc_y == H2D_BC_WALL ? BoundaryKind::Wall : BoundaryKind::Periodic);
}

template <class T>
void put(Field<T>& f, const double* src) {
    if (!src) return;
    std::memcpy(f.raw().data(), src, f.raw().size() * sizeof(T));
}
template <class T>
void get(const Field<T>& f, double* dst) {
    if (!dst) return;
    std::memcpy(dst, f.raw().data(), f.raw().size() * sizeof(T));
}

void set_err(h2dr_ctx* c, int kind, const char* what, int i, int j, int step, int in_step) {
    c->err.kind = kind;
    c->err.i = i;
    c->err.j = j;
    c->err.step = step;
    c->err.in_step = in_step;
    std::snprintf(c->err.what, sizeof(c->err.what), "%s", what);
}

template <class F>
int guarded(h2dr_ctx* c, int step, int in_step, F&& f) {
    try {
        f();
        return 0;
    } catch (const TangledCellError& e) {
        set_err(c, H2D_ERR_TANGLED, e.what(), e.i(), e.j(), step < 0 ? e.step() : step, in_step);
        return H2D_ERR_TANGLED;
    } catch (const UnphysicalStateError& e) {
        set_err(c, H2D_ERR_UNPHYSICAL, e.what(), e.i(), e.j(), step < 0 ? e.step() : step, in_step);
        return H2D_ERR_UNPHYSICAL;
    } catch (const NegativeMassError& e) {
        set_err(c, H2D_ERR_NEGMASS, e.what(), e.i(), e.j(), step < 0 ? e.step() : step, in_step);
        return H2D_ERR_NEGMASS;
    } catch (const CflViolationError& e) {
        set_err(c, H2D_ERR_CFL, e.what(), e.i(), e.j(), step < 0 ? e.step() : step, in_step);
        return H2D_ERR_CFL;
    } catch (const IsolatedMixedCellError& e) {
        set_err(c, H2D_ERR_ISOLATED, e.what(), e.i(), e.j(), step < 0 ? e.step() : step, in_step);
        return H2D_ERR_ISOLATED;
    } catch (const SimError& e) {
        set_err(c, H2D_ERR_SIM, e.what(), e.i(), e.j(), step < 0 ? e.step() : step, in_step);
        return H2D_ERR_SIM;
    } catch (const std::exception& e) {
        set_err(c, H2D_ERR_INVALID, e.what(), -1, -1, -1, 0);
        return H2D_ERR_INVALID;
    }
}

// harness.cpp:347-358 (anonymous there, so restated verbatim in behaviour)
void ref_nan_scan(const State& s, int step) {
    for (int j = 0; j < s.mesh.ny; ++j)
        for (int i = 0; i < s.mesh.nx; ++i)
            if (!std::isfinite(s.m_mix(i, j)) || !std::isfinite(s.e_mix(i, j)) ||
                !std::isfinite(s.p_mix(i, j)))
                throw SimError("non-finite cell state", i, j, step);
    for (int j = 0; j <= s.mesh.ny; ++j)
        for (int i = 0; i <= s.mesh.nx; ++i)
            if (!std::isfinite(s.u(i, j).x) || !std::isfinite(s.u(i, j).y))
                throw SimError("non-finite velocity", i, j, step);
}

} // namespace

extern "C" {

int h2dr_abi_version(void) { return H2D_ABI_VERSION; }

int h2dr_create(const h2d_config* cfg, int /*device*/, h2dr_ctx** out) {
    h2dr_ctx tmp;
    int rc = guarded(&tmp, -1, 0, [&] {
        if (cfg->nmat < 1 || cfg->nmat > kMaxMat) throw std::invalid_argument("nmat out of range");
        auto* c = new h2dr_ctx();
        c->mats.n = cfg->nmat;
        for (int a = 0; a < cfg->nmat; ++a) {
            const h2d_eos& e = cfg->eos[a];
            c->mats.mat[a].eos = e.kind == H2D_EOS_STIFFENED ? EosModel::stiffened(e.gamma, e.pi)
                                                             : EosModel::perfect(e.gamma);
        }
        c->pv.a1 = cfg->pv_a1;
        c->pv.a2 = cfg->pv_a2;
        c->rc.face_order = cfg->face_order;
        c->rc.corner = static_cast<CornerScheme>(cfg->corner);
        c->rc.interface_degrade = cfg->interface_degrade != 0;
        try {
            c->s = make_state(to_mesh(cfg->mesh), cfg->nmat);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
    return rc;
}

void h2dr_destroy(h2dr_ctx* c) { delete c; }

int h2dr_upload_state(h2dr_ctx* c, const h2d_state* v) {
    State& s = c->s;
    for (int a = 0; a < s.nmat; ++a) {
        put(s.m[a], v->m[a]);
        put(s.e[a], v->e[a]);
        put(s.k[a], v->k[a]);
    }
    put(s.iface_normal, v->iface_normal);
    put(s.u, v->u);
    s.step = v->step;
    s.time = v->time;
    if (v->vol && v->m_mix && v->e_mix && v->rho_mix && v->p_mix) {
        put(s.vol, v->vol);
        put(s.m_mix, v->m_mix);
        put(s.e_mix, v->e_mix);
        put(s.rho_mix, v->rho_mix);
        put(s.p_mix, v->p_mix);
    } else {
        sync_derived(s, c->mats);
    }
    c->have_lag = false;
    return 0;
}

int h2dr_download_state(h2dr_ctx* c, h2d_state* v) {
    const State& s = c->s;
    for (int a = 0; a < s.nmat; ++a) {
        get(s.m[a], v->m[a]);
        get(s.e[a], v->e[a]);
        get(s.k[a], v->k[a]);
    }
    get(s.vol, v->vol);
    get(s.m_mix, v->m_mix);
    get(s.e_mix, v->e_mix);
    get(s.rho_mix, v->rho_mix);
    get(s.p_mix, v->p_mix);
    get(s.iface_normal, v->iface_normal);
    get(s.u, v->u);
    v->step = s.step;
    v->time = s.time;
    return 0;
}

int h2dr_fill_ghosts(h2dr_ctx* c) {
    fill_ghosts(c->s);
    return 0;
}
int h2dr_sync_derived(h2dr_ctx* c) {
    sync_derived(c->s, c->mats);
    return 0;
}
int h2dr_update_interface_normals(h2dr_ctx* c) {
    update_interface_normals(c->s);
    return 0;
}

int h2dr_cfl_dt(h2dr_ctx* c, double cfl, double* dt) {
    return guarded(c, -1, 0, [&] { *dt = cfl_dt(c->s, c->mats, cfl); });
}

static void lag_out(const LagrangeResult& r, h2d_lagrange* out, int nmat) {
    if (!out) return;
    get(r.u_half, out->u_half);
    get(r.u_lag, out->u_lag);
    for (int a = 0; a < nmat; ++a) get(r.e_lag[a], out->e_lag[a]);
    get(r.vol_lag, out->vol_lag);
    get(r.q, out->q);
    out->floor_count = r.floor_count;
}

int h2dr_lagrange_step(h2dr_ctx* c, double dt, h2d_lagrange* out) {
    return guarded(c, -1, 0, [&] {
        c->lag = lagrange_step(c->s, c->mats, dt, c->pv);
        c->have_lag = true;
        lag_out(c->lag, out, c->s.nmat);
    });
}

int h2dr_set_lagrange(h2dr_ctx* c, const h2d_lagrange* in) {
    const Mesh& m = c->s.mesh;
    LagrangeResult r;
    r.u_half = Field<Vec2>(m.nx + 1, m.ny + 1);
    r.u_lag = Field<Vec2>(m.nx + 1, m.ny + 1);
    put(r.u_half, in->u_half);
    put(r.u_lag, in->u_lag);
    for (int a = 0; a < c->s.nmat; ++a) {
        r.e_lag[a] = Field<double>(m.nx, m.ny);
        put(r.e_lag[a], in->e_lag[a]);
    }
    r.vol_lag = Field<double>(m.nx, m.ny);
    put(r.vol_lag, in->vol_lag);
    r.q = Field<double>(m.nx, m.ny);
    put(r.q, in->q);
    r.floor_count = in->floor_count;
    c->lag = std::move(r);
    c->have_lag = true;
    return 0;
}

int h2dr_remap_step(h2dr_ctx* c, double dt, int kind, int x_first, int remap_velocity,
                    h2d_remap_diag* diag) {
    if (!c->have_lag) {
        set_err(c, H2D_ERR_INVALID, "remap_step without a LagrangeResult", -1, -1, -1, 0);
        return H2D_ERR_INVALID;
    }
    return guarded(c, -1, 0, [&] {
        RemapDiag d;
        if (diag) {
            d.max_k_violation = diag->max_k_violation;
            d.k_clip_count = diag->k_clip_count;
            d.mass_fix_count = diag->mass_fix_count;
        }
        c->s = remap_step(c->s, c->mats, c->lag, dt, static_cast<RemapKind>(kind), c->rc,
                          x_first != 0, remap_velocity != 0, diag ? &d : nullptr);
        if (diag) {
            diag->max_k_violation = d.max_k_violation;
            diag->k_clip_count = d.k_clip_count;
            diag->mass_fix_count = d.mass_fix_count;
        }
        c->have_lag = false;
    });
}

// make_diag (harness.cpp:360-376; file-local there, restated over the
// reference's own compute_totals)
static h2d_step_diag ref_make_diag(const State& s, double dt) {
    h2d_step_diag d{};
    d.step = s.step;
    d.t = s.time;
    d.dt = dt;
    const Totals t = compute_totals(s);
    d.mass = t.mass;
    d.mass_mat[0] = t.mass_mat[0];
    d.mass_mat[1] = t.mass_mat[1];
    d.momentum_x = t.momentum.x;
    d.momentum_y = t.momentum.y;
    d.internal_energy = t.internal_energy;
    d.min_rho = d.max_rho = s.rho_mix(0, 0);
    d.min_p = d.max_p = s.p_mix(0, 0);
    for (int j = 0; j < s.mesh.ny; ++j)
        for (int i = 0; i < s.mesh.nx; ++i) {
            d.min_rho = std::min(d.min_rho, s.rho_mix(i, j));
            d.max_rho = std::max(d.max_rho, s.rho_mix(i, j));
            d.min_p = std::min(d.min_p, s.p_mix(i, j));
            d.max_p = std::max(d.max_p, s.p_mix(i, j));
        }
    return d;
}

// harness.cpp:390-412 with kinematic == false, on the context's State.
int h2dr_run(h2dr_ctx* c, h2d_run_args* a) {
    State& s = c->s;
    RemapDiag rd;
    rd.max_k_violation = a->diag.max_k_violation;
    rd.k_clip_count = a->diag.k_clip_count;
    rd.mass_fix_count = a->diag.mass_fix_count;
    a->steps_done = 0;
    int rc = 0;
    while (s.time < a->t_end - 1e-15 * std::max(1.0, a->t_end)) {
        if (a->max_steps > 0 && s.step >= a->max_steps) break;
        double dt = 0.0;
        rc = guarded(c, -1, 0, [&] { dt = cfl_dt(s, c->mats, a->cfl); });
        if (rc) break;
        dt = std::min(dt, a->t_end - s.time);
        const int step_now = s.step;
        rc = guarded(c, step_now, 1, [&] {
            LagrangeResult lag = lagrange_step(s, c->mats, dt, c->pv);
            a->floor_count += lag.floor_count;
            const bool x_first = s.step % 2 == 0;
            s = remap_step(s, c->mats, lag, dt, static_cast<RemapKind>(a->remap_kind), c->rc,
                           x_first, true, &rd);
        });
        if (rc) break;
        rc = guarded(c, -1, 0, [&] { ref_nan_scan(s, s.step); });
        if (rc) break;
        if (a->dt_log && a->steps_done < a->dt_log_cap) a->dt_log[a->steps_done] = dt;
        if (a->series && a->steps_done < a->series_cap) a->series[a->steps_done] = ref_make_diag(s, dt);
        ++a->steps_done;
    }
    a->diag.max_k_violation = rd.max_k_violation;
    a->diag.k_clip_count = rd.k_clip_count;
    a->diag.mass_fix_count = rd.mass_fix_count;
    c->have_lag = false;
    return rc;
}

int h2dr_step_diag_now(h2dr_ctx* c, double dt, h2d_step_diag* out) {
    *out = ref_make_diag(c->s, dt);
    return 0;
}

// write_fields (io.hpp:17) of the context's State with the reference writer
int h2dr_write_fields(h2dr_ctx* c, const char* path, int fmt) {
    return guarded(c, -1, 0, [&] {
        write_fields(c->s, std::string(path), fmt == H2D_DUMP_CSV ? DumpFormat::Csv : DumpFormat::VtkLegacyAscii);
    });
}

// append_diag_line (io.hpp:21-22) of one record
int h2dr_diag_line(const h2d_step_diag* d, char* buf, int cap) {
    std::ostringstream o;
    Totals t;
    t.mass = d->mass;
    t.mass_mat[0] = d->mass_mat[0];
    t.mass_mat[1] = d->mass_mat[1];
    t.momentum = Vec2{d->momentum_x, d->momentum_y};
    t.internal_energy = d->internal_energy;
    append_diag_line(o, d->step, d->t, d->dt, t, d->min_rho, d->max_rho, d->min_p, d->max_p);
    const std::string s = o.str();
    if ((int)s.size() + 1 > cap) return H2D_ERR_INVALID;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

int h2dr_totals(h2dr_ctx* c, double out[6]) {
    const Totals t = compute_totals(c->s);
    out[0] = t.mass;
    out[1] = t.mass_mat[0];
    out[2] = t.mass_mat[1];
    out[3] = t.momentum.x;
    out[4] = t.momentum.y;
    out[5] = t.internal_energy;
    return 0;
}

int h2dr_last_error(h2dr_ctx* c, h2d_error* e) {
    *e = c->err;
    return 0;
}

// ---- extra probes used only by the oracle tests --------------------------

// init_case (harness.cpp:226-291) over a flat region list, written into a
// host state view. shape: 0 All, 1 HalfPlaneX, 2 Rectangle, 3 Circle.
// region rows: {shape, xsplit, rlo.x, rlo.y, rhi.x, rhi.y, cx, cy, radius,
//               mat, rho, p, ux, uy}
int h2dr_init_regions(h2dr_ctx* c, const double* rows, int nreg, h2d_state* out) {
    return guarded(c, -1, 0, [&] {
        CaseSpec cs;
        const Mesh& m = c->s.mesh;
        cs.nx = m.nx;
        cs.ny = m.ny;
        cs.x0 = m.x0;
        cs.y0 = m.y0;
        cs.lx = m.dx * m.nx;
        cs.ly = m.dy * m.ny;
        cs.bc_x = m.bc_x;
        cs.bc_y = m.bc_y;
        cs.mats = c->mats;
        for (int r = 0; r < nreg; ++r) {
            const double* q = rows + 14 * r;
            Region g;
            g.shape = static_cast<Region::Shape>(static_cast<int>(q[0]));
            g.xsplit = q[1];
            g.rect = {{q[2], q[3]}, {q[4], q[5]}};
            g.center = {q[6], q[7]};
            g.radius = q[8];
            g.mat = static_cast<int>(q[9]);
            g.rho = q[10];
            g.p = q[11];
            g.u = {q[12], q[13]};
            cs.regions.push_back(g);
        }
        // init_case rebuilds the mesh with dx = lx/nx (harness.cpp:9-11);
        // refuse meshes for which that does not round-trip.
        if (cs.lx / cs.nx != m.dx || cs.ly / cs.ny != m.dy)
            throw std::invalid_argument("mesh spacing does not round-trip through lx/nx");
        c->s = init_case(cs);
        h2dr_download_state(c, out);
    });
}

// Scalar probes of the reconstruction / VOF helpers (reconstruct.cpp, vof.cpp).
double h2dr_van_leer(double r) { return van_leer(r); }
double h2dr_limited_gradient_1d(double am, double ac, double ap, double xm, double xc, double xp) {
    try {
        return limited_gradient_1d(am, ac, ap, xm, xc, xp);
    } catch (...) {
        return NAN;
    }
}
double h2dr_clipped_fraction(double w, double h, double nx, double ny, double d) {
    return clipped_fraction(w, h, {nx, ny}, d);
}
double h2dr_place_interface(double frac, double nx, double ny, double lox, double loy,
                            double hix, double hiy) {
    return place_interface(frac, {nx, ny}, Rect{{lox, loy}, {hix, hiy}}).d;
}
// corner_value with a flat 3x3 stencil: a[9] (p-major: a[p*3+q]), xl[18]
double h2dr_corner_value(int scheme, const double* a, const double* xl, const double* kin) {
    Stencil3x3 st;
    for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) {
            st.a[p][q] = a[p * 3 + q];
            st.xl[p][q] = {xl[2 * (p * 3 + q)], xl[2 * (p * 3 + q) + 1]};
        }
    CornerKin k;
    k.dxp = kin[0];
    k.dyp = kin[1];
    k.lag_wx = kin[2];
    k.lag_wy = kin[3];
    k.sgn_fx = kin[4];
    k.u_fx_dt = kin[5];
    k.sgn_fy = kin[6];
    k.u_fy_dt = kin[7];
    k.eval_rel = {kin[8], kin[9]};
    k.dx = kin[10];
    k.dy = kin[11];
    try {
        return corner_value(static_cast<CornerScheme>(scheme), st, k);
    } catch (...) {
        return NAN;
    }
}

} // extern "C"

// RunReport run(configure_case(RunConfig)) (harness.cpp:380-424, config.cpp:95-106),
// the path of the pybind11 run_case (module.cpp:50-93): the series, final
// State and report scalars {time, l2_rho, l2_k, max_k_violation, k_clip,
// mass_fix, energy_floor}; returns the error kind (message in err_what).
extern "C" int h2dr_run_case(const char* name, int divisor, int scheme, int face_order, int corner, double cfl,
                             double t_end, int max_steps, h2d_step_diag* series, int cap, int* n_series,
                             double out[8], int* steps, h2d_state* final_state, char* err_what, int err_cap) {
    h2dr_ctx c;
    *n_series = 0;
    int nser = 0;
    const int rc = guarded(&c, -1, 0, [&] {
        RunConfig r;
        r.case_name = name;
        r.divisor = divisor;
        r.scheme = static_cast<RemapKind>(scheme);
        r.face_order = face_order;
        r.corner = static_cast<CornerScheme>(corner);
        r.cfl = cfl;
        r.t_end = t_end;
        r.max_steps = max_steps;
        const CaseSpec cs = configure_case(r);
        const RunReport rep = run(cs);
        for (const StepDiag& d : rep.series) {
            if (nser >= cap) break;
            h2d_step_diag& o = series[nser++];
            o = h2d_step_diag{};
            o.step = d.step;
            o.t = d.t;
            o.dt = d.dt;
            o.mass = d.totals.mass;
            o.mass_mat[0] = d.totals.mass_mat[0];
            o.mass_mat[1] = d.totals.mass_mat[1];
            o.momentum_x = d.totals.momentum.x;
            o.momentum_y = d.totals.momentum.y;
            o.internal_energy = d.totals.internal_energy;
            o.min_rho = d.min_rho;
            o.max_rho = d.max_rho;
            o.min_p = d.min_p;
            o.max_p = d.max_p;
        }
        out[0] = rep.final_state.time;
        out[1] = rep.l2_rho_vs_initial;
        out[2] = rep.l2_k_vs_initial;
        out[3] = rep.max_k_violation;
        out[4] = rep.k_clip_count;
        out[5] = rep.mass_fix_count;
        out[6] = rep.energy_floor_count;
        *steps = rep.steps;
        if (final_state) {
            const State& s = rep.final_state;
            for (int a = 0; a < s.nmat; ++a) {
                get(s.m[a], final_state->m[a]);
                get(s.e[a], final_state->e[a]);
                get(s.k[a], final_state->k[a]);
            }
            get(s.vol, final_state->vol);
            get(s.m_mix, final_state->m_mix);
            get(s.e_mix, final_state->e_mix);
            get(s.rho_mix, final_state->rho_mix);
            get(s.p_mix, final_state->p_mix);
            get(s.iface_normal, final_state->iface_normal);
            get(s.u, final_state->u);
            final_state->step = s.step;
            final_state->time = s.time;
        }
    });
    *n_series = nser;
    if (rc && err_what) std::snprintf(err_what, err_cap, "%s", c.err.what);
    return rc;
}

// convergence_study (harness.cpp:426-461) of the reference itself: errs
// [scheme][mesh] and one slope per scheme; returns the error kind.
extern "C" int h2dr_convergence(const char* name, const int* meshes, int nmesh, const int* schemes, int nscheme,
                                double* errs, double* slopes, char* err_what, int err_cap) {
    h2dr_ctx c;
    const int rc = guarded(&c, -1, 0, [&] {
        std::vector<int> ms(meshes, meshes + nmesh);
        std::vector<RemapKind> ks;
        for (int s = 0; s < nscheme; ++s) ks.push_back(static_cast<RemapKind>(schemes[s]));
        const auto res = convergence_study(name, ms, ks);
        for (int s = 0; s < nscheme; ++s) {
            for (int m = 0; m < nmesh; ++m) errs[s * nmesh + m] = res[s].rows[m].err;
            slopes[s] = res[s].slope;
        }
    });
    if (rc && err_what) std::snprintf(err_what, err_cap, "%s", c.err.what);
    return rc;
}

// ---- sub-step entry points and the scalar kernels (h2d.h, the reference's
// predict / correct / remap_single_axis and its public scalar functions) ----
extern "C" {

int h2dr_predict(h2dr_ctx* c, double dt, h2d_half* out) {
    return guarded(c, -1, 0, [&] {
        const HalfStepState h = predict(c->s, c->mats, dt, c->pv);
        if (!out) return;
        get(h.x_half, out->x_half);
        get(h.u_half, out->u_half);
        get(h.vol_half, out->vol_half);
        for (int a = 0; a < c->s.nmat; ++a) {
            get(h.e_half[a], out->e_half[a]);
            get(h.p_half[a], out->p_half[a]);
        }
        get(h.p_mix_half, out->p_mix_half);
        get(h.q, out->q);
        out->floor_count = h.floor_count;
    });
}

int h2dr_correct(h2dr_ctx* c, double dt, const h2d_half* in, h2d_lagrange* out) {
    const Mesh& m = c->s.mesh;
    HalfStepState h;
    h.u_half = Field<Vec2>(m.nx + 1, m.ny + 1);
    put(h.u_half, in->u_half);
    for (int a = 0; a < c->s.nmat; ++a) {
        h.p_half[a] = Field<double>(m.nx, m.ny);
        put(h.p_half[a], in->p_half[a]);
    }
    h.q = Field<double>(m.nx, m.ny);
    put(h.q, in->q);
    h.floor_count = in->floor_count;
    return guarded(c, -1, 0, [&] {
        c->lag = correct(c->s, c->mats, h, dt);
        c->have_lag = true;
        lag_out(c->lag, out, c->s.nmat);
    });
}

int h2dr_remap_single_axis(h2dr_ctx* c, double dt, int axis_x, int remap_velocity, h2d_remap_diag* diag) {
    if (!c->have_lag) {
        set_err(c, H2D_ERR_INVALID, "remap_single_axis without a LagrangeResult", -1, -1, -1, 0);
        return H2D_ERR_INVALID;
    }
    return guarded(c, -1, 0, [&] {
        RemapDiag d;
        if (diag) {
            d.max_k_violation = diag->max_k_violation;
            d.k_clip_count = diag->k_clip_count;
            d.mass_fix_count = diag->mass_fix_count;
        }
        c->s = remap_single_axis(c->s, c->mats, c->lag, dt, axis_x ? Axis::X : Axis::Y, c->rc,
                                 remap_velocity != 0, diag ? &d : nullptr);
        if (diag) {
            diag->max_k_violation = d.max_k_violation;
            diag->k_clip_count = d.k_clip_count;
            diag->mass_fix_count = d.mass_fix_count;
        }
        c->have_lag = false;
    });
}

namespace {
void st3(const double* x, Stencil3x3& st) {
    for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) {
            st.a[p][q] = x[p * 3 + q];
            st.xl[p][q] = {x[9 + p * 3 + q], x[18 + p * 3 + q]};
        }
}
// one record of h2d_scalar_eval through the reference function; true = it threw
bool ref_scalar(int op, const double* x, double* o) {
    try {
        switch (op) {
        case H2D_SC_VAN_LEER: o[0] = van_leer(x[0]); break;
        case H2D_SC_LIMITED_GRADIENT: o[0] = limited_gradient_1d(x[0], x[1], x[2], x[3], x[4], x[5]); break;
        case H2D_SC_FACE_VALUE: {
            Stencil1D d{{x[1], x[2], x[3]}, {x[4], x[5], x[6]}};
            o[0] = face_value(static_cast<int>(x[0]), d, x[7], x[8], x[9]);
            break;
        }
        case H2D_SC_CORNER_VALUE: {
            Stencil3x3 st;
            st3(x + 1, st);
            const double* k = x + 28;
            CornerKin kin;
            kin.dxp = k[0];
            kin.dyp = k[1];
            kin.lag_wx = k[2];
            kin.lag_wy = k[3];
            kin.sgn_fx = k[4];
            kin.u_fx_dt = k[5];
            kin.sgn_fy = k[6];
            kin.u_fy_dt = k[7];
            kin.eval_rel = {k[8], k[9]};
            kin.dx = k[10];
            kin.dy = k[11];
            o[0] = corner_value(static_cast<CornerScheme>(static_cast<int>(x[0])), st, kin);
            break;
        }
        case H2D_SC_MULTID_PLANE: {
            Stencil3x3 st;
            st3(x, st);
            const PlaneRecon pl = multid_plane(st, x[27], x[28]);
            const double v[] = {pl.a0, pl.center.x, pl.center.y, pl.grad_raw.x, pl.grad_raw.y, pl.grad.x, pl.grad.y};
            std::memcpy(o, v, sizeof v);
            break;
        }
        case H2D_SC_CLIPPED_FRACTION: o[0] = clipped_fraction(x[0], x[1], {x[2], x[3]}, x[4]); break;
        case H2D_SC_PLACE_INTERFACE:
            o[0] = place_interface(x[0], {x[1], x[2]}, Rect{{x[3], x[4]}, {x[5], x[6]}}).d;
            break;
        case H2D_SC_YOUNGS_NORMAL: {
            Field<double> k1(3, 3);
            for (int di = -1; di <= 1; ++di)
                for (int dj = -1; dj <= 1; ++dj) k1(1 + di, 1 + dj) = x[(di + 1) * 3 + dj + 1];
            const Vec2 n = youngs_normal(k1, 1, 1, x[9], x[10]);
            o[0] = n.x;
            o[1] = n.y;
            break;
        }
        case H2D_SC_CELL_VOLUME:
            o[0] = cell_volume({x[0], x[1]}, {x[2], x[3]}, {x[4], x[5]}, {x[6], x[7]});
            break;
        case H2D_SC_CF_CORNER_FLUX: {
            const CornerFlux f = cf_corner_flux({x[0], x[1]}, x[2]);
            o[0] = f.dvol;
            o[1] = f.sx;
            o[2] = f.sy;
            break;
        }
        case H2D_SC_CF_FACE_FLUX_X:
        case H2D_SC_CF_FACE_FLUX_Y: {
            const CfFaceFlux f = op == H2D_SC_CF_FACE_FLUX_X ? cf_face_flux_x(x[0], x[1], {x[2], x[3]}, {x[4], x[5]})
                                                              : cf_face_flux_y(x[0], x[1], {x[2], x[3]}, {x[4], x[5]});
            o[0] = f.dvol;
            o[1] = f.wlo;
            o[2] = f.whi;
            break;
        }
        case H2D_SC_PSEUDO_VISCOSITY:
            o[0] = pseudo_viscosity(x[0], x[1], x[2], PseudoViscosityParams{x[3], x[4]}, x[5]);
            break;
        case H2D_SC_DIV_U_CELL: {
            Field<Vec2> u(1, 1);
            u(0, 0) = {x[0], x[1]};
            u(1, 0) = {x[2], x[3]};
            u(0, 1) = {x[4], x[5]};
            u(1, 1) = {x[6], x[7]};
            o[0] = div_u_cell(Mesh(3, 3, x[8], x[9]), u, 0, 0);
            break;
        }
        case H2D_SC_GRAD_PQ_NODE: {
            Field<double> p(3, 3), q(3, 3);
            const int ci[4] = {0, 1, 0, 1}, cj[4] = {0, 0, 1, 1};
            for (int r = 0; r < 4; ++r) {
                p(ci[r], cj[r]) = x[r];
                q(ci[r], cj[r]) = x[4 + r];
            }
            const Vec2 g = grad_pq_node(Mesh(3, 3, x[8], x[9]), p, q, 1, 1);
            o[0] = g.x;
            o[1] = g.y;
            break;
        }
        case H2D_SC_AD_FACE_FLUX: {
            // one X face of ad_face_fluxes on a 3 x 3 mesh whose dy and cv are the record's
            const double dy = x[3], dx = x[4] / x[3];
            Field<Vec2> uh(4, 4);  // the other faces of column 0 cancel: (0, 1), (0, 2) carry 0
            uh(0, 0) = {x[0], 0.0};
            uh(0, 1) = {x[1], 0.0};
            uh(0, 2) = {-x[1], 0.0};
            uh(0, 3) = {x[1], 0.0};
            o[0] = ad_face_fluxes(Axis::X, Mesh(3, 3, dx, dy), uh, x[2])(0, 0);
            break;
        }
        default: return true;
        }
    } catch (const std::exception&) {
        return true;
    }
    return false;
}
}  // namespace

int h2dr_scalar_eval(int op, int n, const double* in, double* out, int* flags) {
    for (int r = 0; r < n; ++r) {
        const bool bad = ref_scalar(op, in + (size_t)r * H2D_SC_IN, out + (size_t)r * H2D_SC_OUT);
        if (flags) flags[r] = bad ? 1 : 0;
    }
    return 0;
}

}  // extern "C"

// hydro_api.cpp — the C++ hydro:: drop-in (include/hydro/b200.hpp) over the
// C-ABI (include/h2d.h).  Value-semantics reference calls (cfl_dt,
// lagrange_step, remap_step, fill_ghosts, sync_derived, ...) upload the
// caller's State into a cached device context, run the CUDA kernels and read
// the result back in the reference Field layout; hydro::b200::Simulation keeps
// the State resident on the GPU for the run loop.  All step arithmetic runs on
// the device; the only host work is layout-preserving copies plus the
// reference's pure helpers make_state / nodal_mass / compute_totals.
#include "../../include/h2d.h"
#include "../../include/hydro/b200.hpp"
#include "h2d_io.h"

#include <cstring>
#include <memory>
#include <ostream>

namespace hydro {
namespace {

[[noreturn]] void throw_error(const h2d_error& e) {
    const std::string w(e.what);
    switch (e.kind) {
    case H2D_ERR_TANGLED: throw TangledCellError(SimError::Formatted{}, w, e.i, e.j, e.step);
    case H2D_ERR_UNPHYSICAL: throw UnphysicalStateError(SimError::Formatted{}, w, e.i, e.j, e.step);
    case H2D_ERR_NEGMASS: throw NegativeMassError(SimError::Formatted{}, w, e.i, e.j, e.step);
    case H2D_ERR_CFL: throw CflViolationError(SimError::Formatted{}, w, e.i, e.j, e.step);
    case H2D_ERR_ISOLATED: throw IsolatedMixedCellError(SimError::Formatted{}, w, e.i, e.j, e.step);
    case H2D_ERR_SIM: throw SimError(SimError::Formatted{}, w, e.i, e.j, e.step);
    default: throw std::runtime_error("hydro2d-b200 device error: " + w);
    }
}

h2d_config make_cfg(const Mesh& m, int nmat, const MaterialSet* mats, const PseudoViscosityParams& pv,
                    const ReconConfig& rc) {
    h2d_config c;
    std::memset(&c, 0, sizeof c);  // the cache compares raw bytes
    c.mesh.nx = m.nx;
    c.mesh.ny = m.ny;
    c.mesh.dx = m.dx;
    c.mesh.dy = m.dy;
    c.mesh.x0 = m.x0;
    c.mesh.y0 = m.y0;
    c.mesh.bc_x = m.periodic_x() ? H2D_BC_PERIODIC : H2D_BC_WALL;
    c.mesh.bc_y = m.periodic_y() ? H2D_BC_PERIODIC : H2D_BC_WALL;
    c.nmat = nmat;
    for (int a = 0; a < nmat; ++a) {
        const EosModel q = mats ? mats->mat[a].eos : EosModel::perfect(1.4);
        c.eos[a].kind = q.kind == EosModel::Kind::Stiffened ? H2D_EOS_STIFFENED : H2D_EOS_PERFECT;
        c.eos[a].gamma = q.gamma;
        c.eos[a].pi = q.pi;
    }
    c.pv_a1 = pv.a1;
    c.pv_a2 = pv.a2;
    c.face_order = rc.face_order;
    c.corner = static_cast<int>(rc.corner);
    c.interface_degrade = rc.interface_degrade ? 1 : 0;
    return c;
}

struct Ctx {
    h2d_config cfg{};
    h2d_ctx* h = nullptr;
    ~Ctx() {
        if (h) h2d_destroy(h);
    }
};
thread_local std::unique_ptr<Ctx> g_cache;

h2d_ctx* context(const h2d_config& cfg) {
    if (g_cache && std::memcmp(&g_cache->cfg, &cfg, sizeof cfg) == 0) return g_cache->h;
    g_cache.reset();
    auto c = std::make_unique<Ctx>();
    c->cfg = cfg;
    const int rc = h2d_create(&cfg, -1, &c->h);
    if (rc == H2D_ERR_SIM) throw SimError("mesh must be at least 3x3");
    if (rc) throw std::runtime_error("hydro2d-b200: cannot create a device context (error " + std::to_string(rc) + ")");
    g_cache = std::move(c);
    return g_cache->h;
}

void check(h2d_ctx* h, int rc) {
    if (!rc) return;
    h2d_error e{};
    h2d_last_error(h, &e);
    throw_error(e);
}

double* p(Field<double>& f) { return f.raw().empty() ? nullptr : f.raw().data(); }
double* p(const Field<double>& f) { return const_cast<Field<double>&>(f).raw().empty() ? nullptr : const_cast<double*>(f.raw().data()); }
double* pv(Field<Vec2>& f) { return f.raw().empty() ? nullptr : &f.raw().data()->x; }
double* pv(const Field<Vec2>& f) { return pv(const_cast<Field<Vec2>&>(f)); }

h2d_state view(const State& s, bool derived = true) {
    h2d_state v;
    std::memset(&v, 0, sizeof v);
    for (int a = 0; a < s.nmat; ++a) {
        v.m[a] = p(s.m[a]);
        v.e[a] = p(s.e[a]);
        v.k[a] = p(s.k[a]);
    }
    if (derived) {
        v.vol = p(s.vol);
        v.m_mix = p(s.m_mix);
        v.e_mix = p(s.e_mix);
        v.rho_mix = p(s.rho_mix);
        v.p_mix = p(s.p_mix);
    }
    v.iface_normal = pv(s.iface_normal);
    v.u = pv(s.u);
    v.step = s.step;
    v.time = s.time;
    return v;
}

h2d_ctx* load(const State& s, const MaterialSet* mats, const PseudoViscosityParams& pvp = {},
              const ReconConfig& rc = {}) {
    h2d_ctx* h = context(make_cfg(s.mesh, s.nmat, mats, pvp, rc));
    const h2d_state v = view(s);
    check(h, h2d_upload_state(h, &v));
    return h;
}

void store(h2d_ctx* h, State& s) {
    h2d_state v = view(s);
    check(h, h2d_download_state(h, &v));
    s.step = v.step;
    s.time = v.time;
}

}  // namespace

// ---- state helpers (state.cpp) ------------------------------------------------
State make_state(const Mesh& mesh, int nmat) {
    State s;
    s.mesh = mesh;
    s.nmat = nmat;
    for (int a = 0; a < kMaxMat; ++a) {
        s.m[a] = Field<double>(mesh.nx, mesh.ny);
        s.e[a] = Field<double>(mesh.nx, mesh.ny);
        s.k[a] = Field<double>(mesh.nx, mesh.ny, a == 0 ? 1.0 : 0.0);
    }
    s.vol = Field<double>(mesh.nx, mesh.ny, mesh.cell_volume());
    s.m_mix = Field<double>(mesh.nx, mesh.ny);
    s.e_mix = Field<double>(mesh.nx, mesh.ny);
    s.rho_mix = Field<double>(mesh.nx, mesh.ny);
    s.p_mix = Field<double>(mesh.nx, mesh.ny);
    s.iface_normal = Field<Vec2>(mesh.nx, mesh.ny, Vec2{1.0, 0.0});
    s.u = Field<Vec2>(mesh.nx + 1, mesh.ny + 1);
    return s;
}

double nodal_mass(const State& s, int i, int j) {
    return 0.25 * (s.m_mix(i - 1, j - 1) + s.m_mix(i, j - 1) + s.m_mix(i - 1, j) + s.m_mix(i, j));
}

Field<double> nodal_masses(const State& s) {
    Field<double> mp(s.mesh.nx + 1, s.mesh.ny + 1);
    for (int j = 0; j <= s.mesh.ny; ++j)
        for (int i = 0; i <= s.mesh.nx; ++i) mp(i, j) = nodal_mass(s, i, j);
    return mp;
}

void fill_ghosts(State& s) {
    h2d_ctx* h = load(s, nullptr);
    check(h, h2d_fill_ghosts(h));
    State t = s;
    store(h, t);
    for (int a = 0; a < s.nmat; ++a) {
        s.m[a] = t.m[a];
        s.e[a] = t.e[a];
        s.k[a] = t.k[a];
    }
    s.iface_normal = t.iface_normal;
    s.u = t.u;
}

namespace {
// one ghost fill through a scratch State slot
template <class F>
void ghost_fill_via(const Mesh& mesh, F&& place) {
    State s = make_state(mesh, 1);
    place(s, true);
    h2d_ctx* h = context(make_cfg(mesh, 1, nullptr, {}, {}));
    h2d_state v = view(s, false);
    check(h, h2d_upload_state(h, &v));
    check(h, h2d_fill_ghosts(h));
    v = view(s, false);
    check(h, h2d_download_state(h, &v));
    place(s, false);
}
}  // namespace

void fill_ghost_cells(const Mesh& mesh, Field<double>& f) {
    ghost_fill_via(mesh, [&](State& s, bool in) {
        if (in) s.m[0] = f; else f = s.m[0];
    });
}
void fill_ghost_cells(const Mesh& mesh, Field<Vec2>& f) {
    ghost_fill_via(mesh, [&](State& s, bool in) {
        if (in) s.iface_normal = f; else f = s.iface_normal;
    });
}
void fill_ghost_nodes(const Mesh& mesh, Field<Vec2>& u) {
    ghost_fill_via(mesh, [&](State& s, bool in) {
        if (in) s.u = u; else u = s.u;
    });
}

void sync_derived(State& s, const MaterialSet& mats) {
    h2d_ctx* h = load(s, &mats);
    check(h, h2d_sync_derived(h));
    store(h, s);
}

void update_interface_normals(State& s) {
    if (s.nmat != 2) return;
    h2d_ctx* h = load(s, nullptr);
    check(h, h2d_update_interface_normals(h));
    State t = s;
    store(h, t);
    s.iface_normal = t.iface_normal;
}

Totals compute_totals(const State& s) {
    Totals t;
    const int nx = s.mesh.nx, ny = s.mesh.ny;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            t.mass += s.m_mix(i, j);
            t.internal_energy += s.m_mix(i, j) * s.e_mix(i, j);
            for (int a = 0; a < s.nmat; ++a) t.mass_mat[a] += s.m[a](i, j);
        }
    const int ie = s.mesh.periodic_x() ? nx - 1 : nx, je = s.mesh.periodic_y() ? ny - 1 : ny;
    for (int j = 0; j <= je; ++j)
        for (int i = 0; i <= ie; ++i) t.momentum += nodal_mass(s, i, j) * s.u(i, j);
    return t;
}

// ---- the step ------------------------------------------------------------------
double cfl_dt(const State& s, const MaterialSet& mats, double cfl) {
    h2d_ctx* h = load(s, &mats);
    double dt = 0.0;
    check(h, h2d_cfl_dt(h, cfl, &dt));
    return dt;
}

LagrangeResult lagrange_step(const State& s, const MaterialSet& mats, double dt, const PseudoViscosityParams& prm) {
    h2d_ctx* h = load(s, &mats, prm);
    LagrangeResult r;
    const int nx = s.mesh.nx, ny = s.mesh.ny;
    r.u_half = Field<Vec2>(nx + 1, ny + 1);
    r.u_lag = Field<Vec2>(nx + 1, ny + 1);
    for (int a = 0; a < s.nmat; ++a) r.e_lag[a] = Field<double>(nx, ny);
    r.vol_lag = Field<double>(nx, ny);
    r.q = Field<double>(nx, ny);
    h2d_lagrange out;
    std::memset(&out, 0, sizeof out);
    out.u_half = pv(r.u_half);
    out.u_lag = pv(r.u_lag);
    for (int a = 0; a < s.nmat; ++a) out.e_lag[a] = p(r.e_lag[a]);
    out.vol_lag = p(r.vol_lag);
    out.q = p(r.q);
    check(h, h2d_lagrange_step(h, dt, &out));
    r.floor_count = out.floor_count;
    return r;
}

State remap_step(const State& s, const MaterialSet& mats, const LagrangeResult& lag, double dt, RemapKind kind,
                 const ReconConfig& rc, bool x_first, bool remap_velocity, RemapDiag* diag) {
    h2d_ctx* h = load(s, &mats, {}, rc);
    h2d_lagrange in;
    std::memset(&in, 0, sizeof in);
    in.u_half = pv(lag.u_half);
    in.u_lag = pv(lag.u_lag);
    for (int a = 0; a < s.nmat; ++a) in.e_lag[a] = p(lag.e_lag[a]);
    in.vol_lag = p(lag.vol_lag);
    in.q = p(lag.q);
    in.floor_count = lag.floor_count;
    check(h, h2d_set_lagrange(h, &in));
    h2d_remap_diag d{};
    if (diag) {
        d.max_k_violation = diag->max_k_violation;
        d.k_clip_count = diag->k_clip_count;
        d.mass_fix_count = diag->mass_fix_count;
    }
    const int hk = kind == RemapKind::AD ? H2D_REMAP_AD : kind == RemapKind::Direct ? H2D_REMAP_DIRECT : H2D_REMAP_DIRECTCF;
    check(h, h2d_remap_step(h, dt, hk, x_first ? 1 : 0,
                            remap_velocity ? 1 : 0,
                            diag ? &d : nullptr));
    if (diag) {
        diag->max_k_violation = d.max_k_violation;
        diag->k_clip_count = d.k_clip_count;
        diag->mass_fix_count = d.mass_fix_count;
    }
    State out = make_state(s.mesh, s.nmat);
    store(h, out);
    return out;
}

State remap_single_axis(const State& s, const MaterialSet& mats, const LagrangeResult& lag, double dt, Axis axis,
                        const ReconConfig& rc, bool remap_velocity, RemapDiag* diag) {
    h2d_ctx* h = load(s, &mats, {}, rc);
    h2d_lagrange in;
    std::memset(&in, 0, sizeof in);
    in.u_half = pv(lag.u_half);
    in.u_lag = pv(lag.u_lag);
    for (int a = 0; a < s.nmat; ++a) in.e_lag[a] = p(lag.e_lag[a]);
    in.vol_lag = p(lag.vol_lag);
    in.q = p(lag.q);
    check(h, h2d_set_lagrange(h, &in));
    h2d_remap_diag d{};
    if (diag) {
        d.max_k_violation = diag->max_k_violation;
        d.k_clip_count = diag->k_clip_count;
        d.mass_fix_count = diag->mass_fix_count;
    }
    check(h, h2d_remap_single_axis(h, dt, axis == Axis::X ? 1 : 0, remap_velocity ? 1 : 0, diag ? &d : nullptr));
    if (diag) {
        diag->max_k_violation = d.max_k_violation;
        diag->k_clip_count = d.k_clip_count;
        diag->mass_fix_count = d.mass_fix_count;
    }
    State out = make_state(s.mesh, s.nmat);
    store(h, out);
    return out;
}

// ---- predict / correct (lagrange.hpp:46-52) ---------------------------------------
HalfStepState predict(const State& s, const MaterialSet& mats, double dt, const PseudoViscosityParams& prm) {
    h2d_ctx* h = load(s, &mats, prm);
    const Mesh& m = s.mesh;
    const int nx = m.nx, ny = m.ny;
    HalfStepState r;
    r.u_half = Field<Vec2>(nx + 1, ny + 1);
    r.vol_half = Field<double>(nx, ny);
    for (int a = 0; a < s.nmat; ++a) {
        r.e_half[a] = Field<double>(nx, ny);
        r.p_half[a] = Field<double>(nx, ny);
    }
    r.p_mix_half = Field<double>(nx, ny);
    r.q = Field<double>(nx, ny);
    r.x_half = Field<Vec2>(nx + 1, ny + 1);
    h2d_half out;
    std::memset(&out, 0, sizeof out);
    out.x_half = pv(r.x_half);
    out.u_half = pv(r.u_half);
    out.vol_half = p(r.vol_half);
    for (int a = 0; a < s.nmat; ++a) {
        out.e_half[a] = p(r.e_half[a]);
        out.p_half[a] = p(r.p_half[a]);
    }
    out.p_mix_half = p(r.p_mix_half);
    out.q = p(r.q);
    check(h, h2d_predict(h, dt, &out));
    r.floor_count = out.floor_count;
    return r;
}

LagrangeResult correct(const State& s, const MaterialSet& mats, const HalfStepState& half, double dt) {
    h2d_ctx* h = load(s, &mats);
    const int nx = s.mesh.nx, ny = s.mesh.ny;
    h2d_half in;
    std::memset(&in, 0, sizeof in);
    in.u_half = pv(half.u_half);
    for (int a = 0; a < s.nmat; ++a) in.p_half[a] = p(half.p_half[a]);
    in.q = p(half.q);
    in.floor_count = half.floor_count;
    LagrangeResult r;
    r.u_half = Field<Vec2>(nx + 1, ny + 1);
    r.u_lag = Field<Vec2>(nx + 1, ny + 1);
    for (int a = 0; a < s.nmat; ++a) r.e_lag[a] = Field<double>(nx, ny);
    r.vol_lag = Field<double>(nx, ny);
    r.q = Field<double>(nx, ny);
    h2d_lagrange out;
    std::memset(&out, 0, sizeof out);
    out.u_half = pv(r.u_half);
    out.u_lag = pv(r.u_lag);
    for (int a = 0; a < s.nmat; ++a) out.e_lag[a] = p(r.e_lag[a]);
    out.vol_lag = p(r.vol_lag);
    out.q = p(r.q);
    check(h, h2d_correct(h, dt, &in, &out));
    r.floor_count = out.floor_count;
    return r;
}

Field<double> compute_q(const State& s, const MaterialSet& mats, const PseudoViscosityParams& prm) {
    // Q^n is predict's first product (lagrange.cpp:84); with dt = 0 the half
    // step cannot tangle, so the only error left is Q's own sound speed
    return predict(s, mats, 0.0, prm).q;
}

// ---- scalar kernels on the device (h2d_scalar_eval) --------------------------------
namespace {

struct Scalar {
    double in[H2D_SC_IN] = {};
    double out[H2D_SC_OUT] = {};
    int flag = 0;
    // evaluate one record; true when the reference call would throw
    bool eval(int op) {
        const int rc = h2d_scalar_eval(op, 1, in, out, &flag);
        if (rc) throw std::runtime_error("hydro2d-b200: the scalar kernels need a CUDA device (error " +
                                         std::to_string(rc) + ")");
        return flag != 0;
    }
};

void put_st3(double* x, const Stencil3x3& st) {
    for (int p = 0; p < 3; ++p)
        for (int q = 0; q < 3; ++q) {
            x[p * 3 + q] = st.a[p][q];
            x[9 + p * 3 + q] = st.xl[p][q].x;
            x[18 + p * 3 + q] = st.xl[p][q].y;
        }
}

[[noreturn]] void throw_centroids() { throw SimError("non-increasing centroid coordinates"); }

}  // namespace

double van_leer(double r) {
    Scalar k;
    k.in[0] = r;
    k.eval(H2D_SC_VAN_LEER);
    return k.out[0];
}

double limited_gradient_1d(double am, double ac, double ap, double xm, double xc, double xp) {
    Scalar k;
    const double v[] = {am, ac, ap, xm, xc, xp};
    std::memcpy(k.in, v, sizeof v);
    if (k.eval(H2D_SC_LIMITED_GRADIENT)) throw_centroids();
    return k.out[0];
}

double face_value(int order, const Stencil1D& d, double sgn_dvol, double lag_width, double u_face_dt) {
    Scalar k;
    const double v[] = {double(order), d.a[0], d.a[1], d.a[2], d.x[0], d.x[1], d.x[2], sgn_dvol, lag_width, u_face_dt};
    std::memcpy(k.in, v, sizeof v);
    if (k.eval(H2D_SC_FACE_VALUE)) throw_centroids();
    return k.out[0];
}

double corner_value(CornerScheme scheme, const Stencil3x3& st, const CornerKin& kin) {
    Scalar k;
    k.in[0] = double(static_cast<int>(scheme));
    put_st3(k.in + 1, st);
    const double v[] = {kin.dxp,     kin.dyp,    kin.lag_wx,  kin.lag_wy,     kin.sgn_fx, kin.u_fx_dt,
                        kin.sgn_fy,  kin.u_fy_dt, kin.eval_rel.x, kin.eval_rel.y, kin.dx,     kin.dy};
    std::memcpy(k.in + 28, v, sizeof v);
    if (k.eval(H2D_SC_CORNER_VALUE)) throw_centroids();
    return k.out[0];
}

PlaneRecon multid_plane(const Stencil3x3& st, double dx, double dy) {
    Scalar k;
    put_st3(k.in, st);
    k.in[27] = dx;
    k.in[28] = dy;
    if (k.eval(H2D_SC_MULTID_PLANE)) throw_centroids();
    PlaneRecon pl;
    pl.a0 = k.out[0];
    pl.center = {k.out[1], k.out[2]};
    pl.grad_raw = {k.out[3], k.out[4]};
    pl.grad = {k.out[5], k.out[6]};
    return pl;
}

Vec2 youngs_normal(const Field<double>& k1, int i, int j, double dx, double dy) {
    Scalar k;
    for (int di = -1; di <= 1; ++di)
        for (int dj = -1; dj <= 1; ++dj) k.in[(di + 1) * 3 + dj + 1] = k1(i + di, j + dj);
    k.in[9] = dx;
    k.in[10] = dy;
    if (k.eval(H2D_SC_YOUNGS_NORMAL))
        throw IsolatedMixedCellError("isolated mixed cell: zero fraction gradient", i, j);
    return {k.out[0], k.out[1]};
}

double clipped_fraction(double w, double h, const Vec2& n, double d) {
    Scalar k;
    const double v[] = {w, h, n.x, n.y, d};
    std::memcpy(k.in, v, sizeof v);
    k.eval(H2D_SC_CLIPPED_FRACTION);
    return k.out[0];
}

InterfaceLine place_interface(double frac, const Vec2& n, const Rect& proxy) {
    Scalar k;
    const double v[] = {frac, n.x, n.y, proxy.lo.x, proxy.lo.y, proxy.hi.x, proxy.hi.y};
    std::memcpy(k.in, v, sizeof v);
    k.eval(H2D_SC_PLACE_INTERFACE);
    return {n, k.out[0]};
}

double cell_volume(const Vec2& p00, const Vec2& p10, const Vec2& p11, const Vec2& p01) {
    Scalar k;
    const double v[] = {p00.x, p00.y, p10.x, p10.y, p11.x, p11.y, p01.x, p01.y};
    std::memcpy(k.in, v, sizeof v);
    if (k.eval(H2D_SC_CELL_VOLUME)) throw TangledCellError("tangled cell");
    return k.out[0];
}

CornerFlux cf_corner_flux(const Vec2& u_half, double dt) {
    Scalar k;
    k.in[0] = u_half.x;
    k.in[1] = u_half.y;
    k.in[2] = dt;
    k.eval(H2D_SC_CF_CORNER_FLUX);
    CornerFlux f;
    f.dvol = k.out[0];
    f.sx = static_cast<int>(k.out[1]);
    f.sy = static_cast<int>(k.out[2]);
    return f;
}

static CfFaceFlux face_flux(int op, double lo, double hi, const Vec2& dm, const Vec2& dp) {
    Scalar k;
    const double v[] = {lo, hi, dm.x, dm.y, dp.x, dp.y};
    std::memcpy(k.in, v, sizeof v);
    k.eval(op);
    CfFaceFlux f;
    f.dvol = k.out[0];
    f.wlo = k.out[1];
    f.whi = k.out[2];
    return f;
}
CfFaceFlux cf_face_flux_x(double ym, double yp, const Vec2& dm, const Vec2& dp) {
    return face_flux(H2D_SC_CF_FACE_FLUX_X, ym, yp, dm, dp);
}
CfFaceFlux cf_face_flux_y(double xm, double xp, const Vec2& dm, const Vec2& dp) {
    return face_flux(H2D_SC_CF_FACE_FLUX_Y, xm, xp, dm, dp);
}

Field<double> ad_face_fluxes(Axis axis, const Mesh& mesh, const Field<Vec2>& u_half, double dt) {
    // every face in one launch, records in the reference loop order (j outer,
    // i inner) so the first flagged record is the reference's first throw
    const bool x = axis == Axis::X;
    const int ni = x ? mesh.nx + 1 : mesh.nx, nj = x ? mesh.ny : mesh.ny + 1;
    const int n = ni * nj;
    std::vector<double> in(static_cast<size_t>(n) * H2D_SC_IN, 0.0), out(static_cast<size_t>(n) * H2D_SC_OUT);
    std::vector<int> flags(n);
    const double cv = mesh.cell_volume();
    for (int j = 0; j < nj; ++j)
        for (int i = 0; i < ni; ++i) {
            double* r = &in[static_cast<size_t>(j * ni + i) * H2D_SC_IN];
            r[0] = x ? u_half(i, j).x : u_half(i, j).y;
            r[1] = x ? u_half(i, j + 1).x : u_half(i + 1, j).y;
            r[2] = dt;
            r[3] = x ? mesh.dy : mesh.dx;
            r[4] = cv;
        }
    if (int rc = h2d_scalar_eval(H2D_SC_AD_FACE_FLUX, n, in.data(), out.data(), flags.data()))
        throw std::runtime_error("hydro2d-b200: the scalar kernels need a CUDA device (error " + std::to_string(rc) + ")");
    Field<double> f(ni, nj);
    for (int j = 0; j < nj; ++j)
        for (int i = 0; i < ni; ++i) {
            const int r = j * ni + i;
            f(i, j) = out[static_cast<size_t>(r) * H2D_SC_OUT];
            if (flags[r]) throw CflViolationError(x ? "CFL violation at X-face" : "CFL violation at Y-face", i, j);
        }
    return f;
}

double pseudo_viscosity(double rho, double c_sound, double div_u, const PseudoViscosityParams& prm, double L) {
    Scalar k;
    const double v[] = {rho, c_sound, div_u, prm.a1, prm.a2, L};
    std::memcpy(k.in, v, sizeof v);
    k.eval(H2D_SC_PSEUDO_VISCOSITY);
    return k.out[0];
}

double div_u_cell(const Mesh& mesh, const Field<Vec2>& u, int i, int j) {
    Scalar k;
    const Vec2 c[4] = {u(i, j), u(i + 1, j), u(i, j + 1), u(i + 1, j + 1)};
    for (int q = 0; q < 4; ++q) {
        k.in[2 * q] = c[q].x;
        k.in[2 * q + 1] = c[q].y;
    }
    k.in[8] = mesh.dx;
    k.in[9] = mesh.dy;
    k.eval(H2D_SC_DIV_U_CELL);
    return k.out[0];
}

Vec2 grad_pq_node(const Mesh& mesh, const Field<double>& pf, const Field<double>& qf, int i, int j) {
    Scalar k;
    const int ci[4] = {i - 1, i, i - 1, i}, cj[4] = {j - 1, j - 1, j, j};
    for (int q = 0; q < 4; ++q) {
        k.in[q] = pf(ci[q], cj[q]);
        k.in[4 + q] = qf(ci[q], cj[q]);
    }
    k.in[8] = mesh.dx;
    k.in[9] = mesh.dy;
    k.eval(H2D_SC_GRAD_PQ_NODE);
    return {k.out[0], k.out[1]};
}

// ---- io.hpp --------------------------------------------------------------------------
void write_fields(const State& s, std::ostream& out, DumpFormat fmt) {
    const h2d_config cfg = make_cfg(s.mesh, s.nmat, nullptr, {}, {});
    std::string text;
    h2d_io::format_fields(cfg, view(s), fmt == DumpFormat::Csv ? H2D_DUMP_CSV : H2D_DUMP_VTK, text);
    out << text;
}

void write_fields(const State& s, const std::string& path, DumpFormat fmt) {
    const h2d_config cfg = make_cfg(s.mesh, s.nmat, nullptr, {}, {});
    const h2d_state v = view(s);
    if (h2d_write_fields_host(&cfg, &v, path.c_str(), fmt == DumpFormat::Csv ? H2D_DUMP_CSV : H2D_DUMP_VTK))
        throw SimError("cannot write: " + path);
}

void append_diag_line(std::ostream& out, int step, double t, double dt, const Totals& totals, double min_rho,
                      double max_rho, double min_p, double max_p) {
    h2d_step_diag d{};
    d.step = step;
    d.t = t;
    d.dt = dt;
    d.mass = totals.mass;
    d.mass_mat[0] = totals.mass_mat[0];
    d.mass_mat[1] = totals.mass_mat[1];
    d.momentum_x = totals.momentum.x;
    d.momentum_y = totals.momentum.y;
    d.internal_energy = totals.internal_energy;
    d.min_rho = min_rho;
    d.max_rho = max_rho;
    d.min_p = min_p;
    d.max_p = max_p;
    out << h2d_io::diag_line(d);
}

// ---- device-resident run loop ------------------------------------------------------
namespace b200 {

static StepDiag from_c(const h2d_step_diag& c) {
    StepDiag d;
    d.step = c.step;
    d.t = c.t;
    d.dt = c.dt;
    d.totals.mass = c.mass;
    d.totals.mass_mat[0] = c.mass_mat[0];
    d.totals.mass_mat[1] = c.mass_mat[1];
    d.totals.momentum = Vec2{c.momentum_x, c.momentum_y};
    d.totals.internal_energy = c.internal_energy;
    d.min_rho = c.min_rho;
    d.max_rho = c.max_rho;
    d.min_p = c.min_p;
    d.max_p = c.max_p;
    return d;
}

Simulation::Simulation(const State& initial, const MaterialSet& mats, const PseudoViscosityParams& pvp,
                       const ReconConfig& rc, int device)
    : mesh_(initial.mesh), nmat_(initial.nmat) {
    const h2d_config cfg = make_cfg(initial.mesh, initial.nmat, &mats, pvp, rc);
    h2d_ctx* h = nullptr;
    const int code = h2d_create(&cfg, device, &h);
    if (code) throw std::runtime_error("hydro2d-b200: cannot create a device context (error " + std::to_string(code) + ")");
    ctx_ = h;
    upload(initial);
}

Simulation::~Simulation() {
    if (ctx_) h2d_destroy(static_cast<h2d_ctx*>(ctx_));
}

void Simulation::upload(const State& s) {
    h2d_ctx* h = static_cast<h2d_ctx*>(ctx_);
    const h2d_state v = view(s);
    check(h, h2d_upload_state(h, &v));
}

State Simulation::download() const {
    State s = make_state(mesh_, nmat_);
    store(static_cast<h2d_ctx*>(ctx_), s);
    return s;
}

StepDiag Simulation::diag_now(double dt) const {
    h2d_ctx* h = static_cast<h2d_ctx*>(ctx_);
    h2d_step_diag d;
    check(h, h2d_step_diag_now(h, dt, &d));
    return from_c(d);
}

void Simulation::write_fields(const std::string& path, DumpFormat fmt) const {
    h2d_ctx* h = static_cast<h2d_ctx*>(ctx_);
    check(h, h2d_write_fields(h, path.c_str(), fmt == DumpFormat::Csv ? H2D_DUMP_CSV : H2D_DUMP_VTK));
}

void Simulation::save(const std::string& path) const {
    h2d_ctx* h = static_cast<h2d_ctx*>(ctx_);
    check(h, h2d_save_state(h, path.c_str()));
}

void Simulation::load(const std::string& path) {
    h2d_ctx* h = static_cast<h2d_ctx*>(ctx_);
    check(h, h2d_load_state(h, path.c_str()));
}

StepInfo Simulation::run(int max_steps, double t_end, double cfl, RemapDiag* diag) {
    h2d_ctx* h = static_cast<h2d_ctx*>(ctx_);
    StepInfo info;
    info.dts.assign(max_steps > 0 ? max_steps : 65536, 0.0);
    h2d_run_args a;
    std::memset(&a, 0, sizeof a);
    a.max_steps = max_steps;
    a.t_end = t_end;
    a.cfl = cfl;
    a.remap_kind = H2D_REMAP_DIRECTCF;
    a.dt_log = info.dts.data();
    a.dt_log_cap = static_cast<int>(info.dts.size());
    std::vector<h2d_step_diag> ser(info.dts.size());
    a.series = ser.data();
    a.series_cap = static_cast<int>(ser.size());
    if (diag) {
        a.diag.max_k_violation = diag->max_k_violation;
        a.diag.k_clip_count = diag->k_clip_count;
        a.diag.mass_fix_count = diag->mass_fix_count;
    }
    const int rc = h2d_run(h, &a);
    info.steps_done = a.steps_done;
    info.floor_count = a.floor_count;
    info.dts.resize(std::min<size_t>(info.dts.size(), static_cast<size_t>(a.steps_done)));
    for (size_t q = 0; q < info.dts.size(); ++q) info.series.push_back(from_c(ser[q]));
    if (diag) {
        diag->max_k_violation = a.diag.max_k_violation;
        diag->k_clip_count = a.diag.k_clip_count;
        diag->mass_fix_count = a.diag.mass_fix_count;
    }
    check(h, rc);
    return info;
}

}  // namespace b200
}  // namespace hydro

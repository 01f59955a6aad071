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
    check(h, h2d_remap_step(h, dt, kind == RemapKind::AD ? H2D_REMAP_AD : H2D_REMAP_DIRECTCF, x_first ? 1 : 0,
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

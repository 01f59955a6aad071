// hydro_harness.cpp — the driver layer of the C++ drop-in (harness.hpp,
// config.hpp): the case catalogue, the initial-state painter, run() with the
// State resident on the device, the mesh-refinement study and the key = value
// run configuration.  The reference's callers (tools/main.cpp `hydro2d run`,
// src/bindings/module.cpp run_case, tests/acceptance.cpp) link against this
// unchanged (tests/cpp/Makefile).
//
// run() (harness.cpp:380-424): the dynamic branch is ONE h2d_run call (the
// device-resident CUDA-graph loop, dt / counters / StepDiag reduced on the
// device) when no hook is installed on a mesh above 2^20 cells; otherwise the
// loop advances one device step per call and records make_diag with the
// reference's serial sums (h2d_step_diag_now), handing a hook the downloaded
// State, so RunReport::series and a hook that writes the ledger
// (main.cpp:40-49) carry the reference's bytes.  The
// imposed-velocity branch (harness.cpp:391-402) drives h2d_remap_step with
// the kinematic LagrangeResult.
#include "../../include/h2d.h"
#include "../../include/hydro/b200.hpp"

#include <chrono>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>

namespace hydro {

Mesh CaseSpec::make_mesh() const { return Mesh(nx, ny, lx / nx, ly / ny, x0, y0, bc_x, bc_y); }

const char* scheme_name(RemapKind k) {
    return k == RemapKind::AD ? "AD" : k == RemapKind::Direct ? "Direct" : k == RemapKind::DirectCF ? "DirectCF" : "?";
}

// ---- case catalogue (harness.cpp:22-163) ----------------------------------------------
namespace {

using Shape = Region::Shape;

Material air() { return {"air", EosModel::perfect(1.4)}; }
Material water() { return {"water", EosModel::stiffened(7.0, 2.1e9)}; }

Region paint(Shape shape, int mat, double rho, double p, Vec2 u = {}) {
    Region r;
    r.shape = shape;
    r.mat = mat;
    r.rho = rho;
    r.p = p;
    r.u = u;
    return r;
}
Region box(double x0, double y0, double x1, double y1, int mat, double rho, double p, Vec2 u = {}) {
    Region r = paint(Shape::Rectangle, mat, rho, p, u);
    r.rect = Rect{{x0, y0}, {x1, y1}};
    return r;
}
Region disc(double cx, double cy, double radius, int mat, double rho, double p, Vec2 u = {}) {
    Region r = paint(Shape::Circle, mat, rho, p, u);
    r.center = {cx, cy};
    r.radius = radius;
    return r;
}

// a divisor shrinks a desk run's mesh, never below 8 cells
int mesh_n(int n, int divisor) {
    const int v = n / (divisor < 1 ? 1 : divisor);
    return v < 8 ? 8 : v;
}

constexpr double kTwoPi = 2.0 * 3.14159265358979323846;

}  // namespace

std::vector<std::string> case_list() {
    return {"uniform", "mono_advect", "mono_rotation", "multimat_advect", "water_air_rotation", "haas", "impact"};
}

CaseSpec build_case(const std::string& name, int divisor) {
    CaseSpec cs;
    cs.name = name;
    auto one_material = [&](int n) {
        cs.nx = cs.ny = mesh_n(n, divisor);
        cs.mats.n = 1;
        cs.mats.mat[0] = air();
    };
    if (name == "uniform") {  // free stream, harness.cpp:47-56
        one_material(50);
        cs.regions = {paint(Shape::All, 0, 1.0, 1e5, {5.0, 5.0})};
        cs.t_end = 1.0;
        cs.max_steps = 50;
    } else if (name == "mono_advect" || name == "multimat_advect") {  // :57-76
        const bool two = name == "multimat_advect";
        one_material(100);
        if (two) {
            cs.mats.n = 2;
            cs.mats.mat[1] = {"air2", EosModel::perfect(1.4)};
        }
        cs.regions = {paint(Shape::All, 0, two ? 1.29 : 0.1, 1e5),
                      box(0.2, 0.2, 0.4, 0.4, two ? 1 : 0, two ? 1.29 : 10.0, 1e5)};
        cs.imposed = ImposedVelocity::Constant;
        cs.u_const = {5.0, 5.0};
        cs.flip_time = 0.06;
        cs.t_end = 0.12;
    } else if (name == "mono_rotation") {  // :77-92
        one_material(100);
        cs.regions = {paint(Shape::All, 0, 0.1, 1e5), box(0.4, 0.65, 0.6, 0.85, 0, 10.0, 1e5)};
        cs.imposed = ImposedVelocity::Rotation;
        cs.rot_center = {0.5, 0.5};
        cs.rot_omega = kTwoPi;
        cs.t_end = 1.0;
    } else if (name == "water_air_rotation") {  // :93-110
        one_material(400);
        cs.lx = cs.ly = 4.0;
        cs.mats.n = 2;
        cs.mats.mat[1] = water();
        cs.regions = {paint(Shape::All, 0, 1.29, 1e5), box(1.6, 2.5, 2.4, 3.3, 1, 1000.0, 1e5)};
        cs.imposed = ImposedVelocity::Rotation;
        cs.rot_center = {2.0, 2.0};
        cs.rot_omega = kTwoPi * 1e3;
        cs.t_end = 1e-3;
    } else if (name == "haas") {  // shock / helium bubble, :111-134
        cs.nx = mesh_n(1000, divisor);
        cs.ny = mesh_n(90, divisor);
        cs.lx = 10.0;
        cs.ly = 0.09;
        cs.bc_x = cs.bc_y = BoundaryKind::Wall;
        cs.mats.n = 2;
        cs.mats.mat[0] = air();
        cs.mats.mat[1] = {"helium", EosModel::perfect(1.66)};
        Region shocked = paint(Shape::HalfPlaneX, 0, 1.376363, 1.5698e5, {124.824, 0.0});
        shocked.xsplit = 0.8;
        cs.regions = {paint(Shape::All, 0, 1.0, 1e5), shocked, disc(1.0, 0.045, 0.04, 1, 0.18187, 1e5)};
        cs.t_end = 1e-3;
    } else if (name == "impact") {  // water jet on a wall, :135-160
        cs.nx = mesh_n(320, divisor);
        cs.ny = mesh_n(160, divisor);
        cs.lx = 0.10;
        cs.ly = 0.05;
        cs.bc_x = cs.bc_y = BoundaryKind::Wall;
        cs.mats.n = 2;
        cs.mats.mat[0] = air();
        cs.mats.mat[1] = water();
        cs.regions = {paint(Shape::All, 0, 1.29, 1e5, {-1000.0, 0.0}), box(0.0, 0.0, 0.01, 0.05, 1, 1000.0, 1e5),
                      disc(0.03, 0.025, 0.01, 1, 1000.0, 1e5, {-1000.0, 0.0})};
        cs.t_end = 6e-3;
    } else {
        throw SimError("unknown case: " + name);
    }
    return cs;
}

// ---- initial state (harness.cpp:163-291) ------------------------------------------------
namespace {

double rmax(double a, double b) { return a < b ? b : a; }  // std::max
double rmin(double a, double b) { return b < a ? b : a; }  // std::min

bool inside(const Region& r, const Vec2& p) {
    switch (r.shape) {
    case Shape::All: return true;
    case Shape::HalfPlaneX: return p.x < r.xsplit;
    case Shape::Rectangle: return p.x >= r.rect.lo.x && p.x <= r.rect.hi.x && p.y >= r.rect.lo.y && p.y <= r.rect.hi.y;
    case Shape::Circle: {
        const double ex = p.x - r.center.x, ey = p.y - r.center.y;
        return ex * ex + ey * ey <= r.radius * r.radius;
    }
    }
    return false;
}

// covered share of the cell [lo, hi]: exact for the half plane and the
// rectangle, 16 x 16 sub-cell samples for a circle
double covered(const Region& r, const Mesh& m, const Vec2& lo, const Vec2& hi) {
    switch (r.shape) {
    case Shape::All: return 1.0;
    case Shape::HalfPlaneX: {
        const double v = (r.xsplit - lo.x) / m.dx;
        return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);  // std::clamp(v, 0, 1)
    }
    case Shape::Rectangle: {
        const double wx = rmax(0.0, rmin(hi.x, r.rect.hi.x) - rmax(lo.x, r.rect.lo.x));
        const double wy = rmax(0.0, rmin(hi.y, r.rect.hi.y) - rmax(lo.y, r.rect.lo.y));
        return (wx / m.dx) * (wy / m.dy);
    }
    case Shape::Circle: {
        int hits = 0;
        for (int sy = 0; sy < 16; ++sy)
            for (int sx = 0; sx < 16; ++sx) {
                const Vec2 q{lo.x + (sx + 0.5) / 16.0 * m.dx, lo.y + (sy + 0.5) / 16.0 * m.dy};
                hits += inside(r, q) ? 1 : 0;
            }
        return hits / 256.0;
    }
    }
    return 0.0;
}

double energy_of(const EosModel& eos, double rho, double p) {
    const double pi = eos.kind == EosModel::Kind::Stiffened ? eos.pi : 0.0;
    return (p + pi) / ((eos.gamma - 1.0) * rho);
}

// the per-cell material mixture a sequence of regions paints: a later region
// covering a share f scales what is there by (1 - f) and adds f of itself
struct Mixture {
    double k[kMaxMat] = {}, m[kMaxMat] = {}, me[kMaxMat] = {};
    void overlay(int nmat, int mat, double f, double rho, double e, double cv) {
        for (int a = 0; a < nmat; ++a) {
            k[a] *= (1.0 - f);
            m[a] *= (1.0 - f);
            me[a] *= (1.0 - f);
        }
        k[mat] += f;
        m[mat] += f * rho * cv;
        me[mat] += f * rho * e * cv;
    }
    // a trace fraction below kPureTol joins the other material
    void snap(int nmat) {
        for (int a = 0; a < nmat; ++a)
            if (k[a] < kPureTol) {
                const int b = 1 - a;
                k[b] += k[a];
                m[b] += m[a];
                me[b] += me[a];
                k[a] = m[a] = me[a] = 0.0;
            }
    }
};

void imposed_field(State& s, const CaseSpec& cs, double t) {
    const Mesh& m = s.mesh;
    const double sgn = (cs.flip_time > 0.0 && t >= cs.flip_time) ? -1.0 : 1.0;
    for (int j = 0; j <= m.ny; ++j)
        for (int i = 0; i <= m.nx; ++i) {
            if (cs.imposed == ImposedVelocity::Constant) {
                s.u(i, j) = sgn * cs.u_const;
            } else {
                const Vec2 p = m.node_pos(i, j);
                s.u(i, j) = cs.rot_omega * Vec2{-(p.y - cs.rot_center.y), p.x - cs.rot_center.x};
            }
        }
    fill_ghost_nodes(m, s.u);
}

}  // namespace

State init_case(const CaseSpec& cs) {
    const Mesh mesh = cs.make_mesh();
    const int nmat = cs.mats.n;
    State s = make_state(mesh, nmat);
    const double cv = mesh.cell_volume();
    std::vector<double> e_reg(cs.regions.size());
    for (size_t r = 0; r < cs.regions.size(); ++r)
        e_reg[r] = energy_of(cs.mats.mat[cs.regions[r].mat].eos, cs.regions[r].rho, cs.regions[r].p);
    for (int j = 0; j < mesh.ny; ++j)
        for (int i = 0; i < mesh.nx; ++i) {
            Mixture mx;
            const Vec2 lo = mesh.node_pos(i, j), hi = mesh.node_pos(i + 1, j + 1), c = mesh.cell_center(i, j);
            for (size_t r = 0; r < cs.regions.size(); ++r) {
                const Region& reg = cs.regions[r];
                // the first region fills the cell; later ones paint whole cells by
                // centroid unless they bring a second material into a cell not yet
                // full of it, which gets its covered share
                double f = 1.0;
                if (r > 0) f = (nmat == 2 && mx.k[reg.mat] < 1.0) ? covered(reg, mesh, lo, hi) : (inside(reg, c) ? 1.0 : 0.0);
                if (f <= 0.0) continue;
                mx.overlay(nmat, reg.mat, f, reg.rho, e_reg[r], cv);
            }
            mx.snap(nmat);
            for (int a = 0; a < nmat; ++a) {
                s.k[a](i, j) = mx.k[a];
                s.m[a](i, j) = mx.m[a];
                s.e[a](i, j) = mx.m[a] > 0.0 ? mx.me[a] / mx.m[a] : 0.0;
            }
        }
    for (int j = 0; j <= mesh.ny; ++j)
        for (int i = 0; i <= mesh.nx; ++i) {
            const Vec2 p = mesh.node_pos(i, j);
            Vec2 u;
            for (const Region& reg : cs.regions)
                if (inside(reg, p)) u = reg.u;
            s.u(i, j) = u;
        }
    // the init tail (harness.cpp:286-289) on the device
    fill_ghosts(s);
    sync_derived(s, cs.mats);
    update_interface_normals(s);
    if (cs.imposed != ImposedVelocity::None) imposed_field(s, cs, 0.0);
    return s;
}

double l2_error(const Field<double>& a, const Field<double>& b, const Mesh& mesh) {
    if (a.nx() != b.nx() || a.ny() != b.ny() || a.nx() != mesh.nx || a.ny() != mesh.ny)
        throw SimError("field/mesh size mismatch");
    double sum = 0.0;
    for (int j = 0; j < mesh.ny; ++j)
        for (int i = 0; i < mesh.nx; ++i) {
            const double d = a(i, j) - b(i, j);
            sum += d * d;
        }
    return std::sqrt(sum * mesh.dx * mesh.dy);
}

// ---- run (harness.cpp:380-424) ----------------------------------------------------------
namespace {

h2d_config config_of(const CaseSpec& cs, const Mesh& m) {
    h2d_config c;
    std::memset(&c, 0, sizeof c);
    c.mesh = {m.nx, m.ny, m.dx, m.dy, m.x0, m.y0, m.periodic_x() ? H2D_BC_PERIODIC : H2D_BC_WALL,
              m.periodic_y() ? H2D_BC_PERIODIC : H2D_BC_WALL};
    c.nmat = cs.mats.n;
    for (int a = 0; a < cs.mats.n; ++a) {
        const EosModel& q = cs.mats.mat[a].eos;
        c.eos[a] = {q.kind == EosModel::Kind::Stiffened ? H2D_EOS_STIFFENED : H2D_EOS_PERFECT, q.gamma, q.pi};
    }
    c.pv_a1 = cs.pv.a1;
    c.pv_a2 = cs.pv.a2;
    c.face_order = cs.recon.face_order;
    c.corner = static_cast<int>(cs.recon.corner);
    c.interface_degrade = cs.recon.interface_degrade ? 1 : 0;
    return c;
}

int remap_code(RemapKind k) {
    return k == RemapKind::AD ? H2D_REMAP_AD : k == RemapKind::Direct ? H2D_REMAP_DIRECT : H2D_REMAP_DIRECTCF;
}

// one device context holding the run's State (RAII)
struct Resident {
    h2d_ctx* h = nullptr;
    Mesh mesh;
    int nmat = 1;
    Resident(const CaseSpec& cs, const State& s) : mesh(s.mesh), nmat(s.nmat) {
        const h2d_config cfg = config_of(cs, s.mesh);
        const int rc = h2d_create(&cfg, -1, &h);
        if (rc) throw std::runtime_error("hydro2d-b200: cannot create a device context (error " + std::to_string(rc) + ")");
        upload(s);
    }
    ~Resident() {
        if (h) h2d_destroy(h);
    }
    Resident(const Resident&) = delete;
    Resident& operator=(const Resident&) = delete;

    h2d_error error() const {
        h2d_error e{};
        h2d_last_error(h, &e);
        return e;
    }
    void upload(const State& s) {
        h2d_state v = view(const_cast<State&>(s));
        ok(h2d_upload_state(h, &v));
    }
    static h2d_state view(State& s) {
        h2d_state v;
        std::memset(&v, 0, sizeof v);
        for (int a = 0; a < s.nmat; ++a) {
            v.m[a] = s.m[a].raw().data();
            v.e[a] = s.e[a].raw().data();
            v.k[a] = s.k[a].raw().data();
        }
        v.vol = s.vol.raw().data();
        v.m_mix = s.m_mix.raw().data();
        v.e_mix = s.e_mix.raw().data();
        v.rho_mix = s.rho_mix.raw().data();
        v.p_mix = s.p_mix.raw().data();
        v.iface_normal = &s.iface_normal.raw().data()->x;
        v.u = &s.u.raw().data()->x;
        v.step = s.step;
        v.time = s.time;
        return v;
    }
    State download() const {
        State s = make_state(mesh, nmat);
        h2d_state v = view(s);
        ok(h2d_download_state(h, &v));
        s.step = v.step;
        s.time = v.time;
        return s;
    }
    StepDiag diag_now(double dt) const {
        h2d_step_diag c{};
        ok(h2d_step_diag_now(h, dt, &c));
        return from_c(c);
    }
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
    void ok(int rc) const {
        if (rc) rethrow(error(), nullptr);
    }
    // the reference exception class; an error inside lagrange_step /
    // remap_step is re-thrown by run() as SimError with the case and step
    // appended (harness.cpp:404-407)
    [[noreturn]] static void rethrow(const h2d_error& e, const CaseSpec* cs) {
        if (cs && e.in_step)
            throw SimError(std::string(e.what) + " [" + cs->name + " step " + std::to_string(e.step) + "]");
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
};

struct Counters {
    int floors = 0, clips = 0, fixes = 0;
    double kviol = 0.0;
    void add(const h2d_run_args& a) {
        floors += a.floor_count;
        clips += a.diag.k_clip_count;
        fixes += a.diag.mass_fix_count;
        if (a.diag.max_k_violation > kviol) kviol = a.diag.max_k_violation;
    }
};

// the dynamic branch: cfl_dt -> lagrange_step -> remap_step -> nan_scan -> make_diag
void run_dynamic(const CaseSpec& cs, Resident& dev, const StepHook& hook, RunReport& rep, Counters& cnt) {
    constexpr int kChunk = 65536;  // the device run loop's dt / StepDiag log capacity per call
    std::vector<double> dts;
    std::vector<h2d_step_diag> ser;
    // one h2d_run call from the State's step `from` up to (absolute) step `to`
    auto call = [&](int from, int to, bool series) {
        h2d_run_args a;
        std::memset(&a, 0, sizeof a);
        a.max_steps = to;
        a.t_end = cs.t_end;
        a.cfl = cs.cfl;
        a.remap_kind = remap_code(cs.scheme);
        dts.assign(static_cast<size_t>(to - from), 0.0);
        a.dt_log = dts.data();
        a.dt_log_cap = static_cast<int>(dts.size());
        if (series) {
            ser.assign(dts.size(), h2d_step_diag{});
            a.series = ser.data();
            a.series_cap = static_cast<int>(ser.size());
        }
        const int rc = h2d_run(dev.h, &a);
        cnt.add(a);
        if (series)
            for (int q = 0; q < a.steps_done && q < a.series_cap; ++q) rep.series.push_back(Resident::from_c(ser[q]));
        if (rc) Resident::rethrow(dev.error(), &cs);
        return a.steps_done;
    };
    // the StepDiag sums: the device run loop reduces them as a fixed-order
    // tree (within n 2^-53 sum|x| of the reference's serial loop); a hook, or a
    // mesh up to kSerialDiagCells, gets the reference's serial sums bit for bit
    // (h2d_step_diag_now after every device step)
    constexpr long long kSerialDiagCells = 1LL << 20;
    const bool fast = !hook && static_cast<long long>(cs.nx) * cs.ny > kSerialDiagCells;
    for (int step = rep.initial_state.step;;) {
        if (cs.max_steps > 0 && step >= cs.max_steps) break;
        int to = fast ? step + kChunk : step + 1;
        if (cs.max_steps > 0 && to > cs.max_steps) to = cs.max_steps;
        const int done = call(step, to, fast);
        step += done;
        if (!fast && done == 1) {
            rep.series.push_back(dev.diag_now(dts[0]));
            if (hook) hook(dev.download(), rep.series.back());
        }
        if (done < to - (step - done)) break;  // t_end reached
    }
}

double kinematic_dt(const State& s, double cfl) {
    double umax = 0.0;
    for (int j = 0; j <= s.mesh.ny; ++j)
        for (int i = 0; i <= s.mesh.nx; ++i) umax = rmax(umax, norm(s.u(i, j)));
    if (!(umax > 0.0)) throw SimError("imposed velocity field is zero");
    return cfl * rmin(s.mesh.dx, s.mesh.dy) / umax;
}

void nan_check(const State& s) {
    for (int j = 0; j < s.mesh.ny; ++j)
        for (int i = 0; i < s.mesh.nx; ++i)
            if (!std::isfinite(s.m_mix(i, j)) || !std::isfinite(s.e_mix(i, j)) || !std::isfinite(s.p_mix(i, j)))
                throw SimError("non-finite cell state", i, j, s.step);
    for (int j = 0; j <= s.mesh.ny; ++j)
        for (int i = 0; i <= s.mesh.nx; ++i)
            if (!std::isfinite(s.u(i, j).x) || !std::isfinite(s.u(i, j).y))
                throw SimError("non-finite velocity", i, j, s.step);
}

// the imposed-velocity branch: kinematic_dt (flip-limited) -> kinematic
// LagrangeResult -> remap without velocity remap -> impose_velocity
void run_kinematic(const CaseSpec& cs, Resident& dev, const StepHook& hook, RunReport& rep, Counters& cnt) {
    State s = rep.initial_state;
    h2d_remap_diag rd{};
    const int nx = s.mesh.nx, ny = s.mesh.ny;
    while (s.time < cs.t_end - 1e-15 * rmax(1.0, cs.t_end)) {
        if (cs.max_steps > 0 && s.step >= cs.max_steps) break;
        double dt = kinematic_dt(s, cs.cfl);
        if (cs.flip_time > 0.0 && s.time < cs.flip_time) dt = rmin(dt, cs.flip_time - s.time);
        dt = rmin(dt, cs.t_end - s.time);
        Field<double> q(nx, ny);
        h2d_lagrange lag;
        std::memset(&lag, 0, sizeof lag);
        lag.u_half = &s.u.raw().data()->x;
        lag.u_lag = &s.u.raw().data()->x;
        for (int a = 0; a < s.nmat; ++a) lag.e_lag[a] = s.e[a].raw().data();
        lag.vol_lag = s.vol.raw().data();
        lag.q = q.raw().data();
        dev.ok(h2d_set_lagrange(dev.h, &lag));
        if (h2d_remap_step(dev.h, dt, remap_code(cs.scheme), s.step % 2 == 0 ? 1 : 0, 0, &rd)) {
            h2d_error e = dev.error();
            e.in_step = 1;
            e.step = s.step;
            Resident::rethrow(e, &cs);
        }
        s = dev.download();
        imposed_field(s, cs, s.time);
        dev.upload(s);
        nan_check(s);
        rep.series.push_back(dev.diag_now(dt));
        if (hook) hook(s, rep.series.back());
    }
    cnt.clips = rd.k_clip_count;
    cnt.fixes = rd.mass_fix_count;
    cnt.kviol = rd.max_k_violation;
}

}  // namespace

RunReport run(const CaseSpec& cs, const StepHook& hook) {
    const auto t0 = std::chrono::steady_clock::now();
    RunReport rep;
    rep.spec = cs;
    rep.initial_state = init_case(cs);
    Resident dev(cs, rep.initial_state);
    rep.series.push_back(dev.diag_now(0.0));
    Counters cnt;
    if (cs.imposed == ImposedVelocity::None)
        run_dynamic(cs, dev, hook, rep, cnt);
    else
        run_kinematic(cs, dev, hook, rep, cnt);
    rep.final_state = dev.download();
    rep.steps = rep.final_state.step;
    rep.max_k_violation = cnt.kviol;
    rep.k_clip_count = cnt.clips;
    rep.mass_fix_count = cnt.fixes;
    rep.energy_floor_count = cnt.floors;
    const Mesh& m = rep.final_state.mesh;
    rep.l2_rho_vs_initial = l2_error(rep.final_state.rho_mix, rep.initial_state.rho_mix, m);
    if (cs.mats.n == 2) rep.l2_k_vs_initial = l2_error(rep.final_state.k[1], rep.initial_state.k[1], m);
    rep.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rep;
}

std::vector<ConvergenceResult> convergence_study(const std::string& case_name, const std::vector<int>& meshes,
                                                 const std::vector<RemapKind>& schemes) {
    std::vector<ConvergenceResult> out;
    for (const RemapKind scheme : schemes) {
        ConvergenceResult res;
        res.scheme = scheme;
        for (const int n : meshes) {
            CaseSpec cs = build_case(case_name);
            cs.nx = cs.ny = n;
            cs.scheme = scheme;
            const RunReport rep = run(cs);
            res.rows.push_back({n, cs.mats.n == 2 ? rep.l2_k_vs_initial : rep.l2_rho_vs_initial});
        }
        // least-squares slope of log(err) against log(dx) (harness.cpp:445-457)
        double sx = 0.0, sy = 0.0, sxx = 0.0, sxy = 0.0;
        const int m = static_cast<int>(res.rows.size());
        for (const ConvergenceRow& row : res.rows) {
            const double lx = std::log(1.0 / row.n), ly = std::log(rmax(row.err, 1e-300));
            sx += lx;
            sy += ly;
            sxx += lx * lx;
            sxy += lx * ly;
        }
        res.slope = m > 1 ? (m * sxy - sx * sy) / (m * sxx - sx * sx) : 0.0;
        out.push_back(std::move(res));
    }
    return out;
}

// ---- run configuration (config.cpp) -------------------------------------------------------
namespace {

std::string strip(const std::string& s) {
    const char* ws = " \t\r";
    const size_t b = s.find_first_not_of(ws);
    if (b == std::string::npos) return "";
    return s.substr(b, s.find_last_not_of(ws) - b + 1);
}

[[noreturn]] void bad_line(int line, const std::string& msg) {
    throw SimError("config line " + std::to_string(line) + ": " + msg);
}

double number(const std::string& v, int line) {
    size_t used = 0;
    double x = 0.0;
    try {
        x = std::stod(v, &used);
    } catch (const std::exception&) {
        bad_line(line, "not a number: '" + v + "'");
    }
    // the reference's own throw of the trailing-characters case is caught by
    // its catch-all and reported as "not a number" (config.cpp:41-50)
    if (used != v.size()) bad_line(line, "not a number: '" + v + "'");
    return x;
}

}  // namespace

RunConfig parse_config(const std::string& text) {
    RunConfig rc;
    std::istringstream in(text);
    std::string raw;
    for (int line = 1; std::getline(in, raw); ++line) {
        const std::string body = strip(raw.substr(0, raw.find('#')));
        if (body.empty()) continue;
        const size_t eq = body.find('=');
        if (eq == std::string::npos) bad_line(line, "expected 'key = value'");
        const std::string key = strip(body.substr(0, eq)), val = strip(body.substr(eq + 1));
        if (key == "case") {
            rc.case_name = val;
        } else if (key == "scheme") {
            if (val == "AD") rc.scheme = RemapKind::AD;
            else if (val == "Direct") rc.scheme = RemapKind::Direct;
            else if (val == "DirectCF") rc.scheme = RemapKind::DirectCF;
            else bad_line(line, "invalid scheme '" + val + "' (valid: AD, Direct, DirectCF)");
        } else if (key == "face_order") {
            const int o = static_cast<int>(number(val, line));
            if (o != 1 && o != 2) bad_line(line, "face_order must be 1 or 2");
            rc.face_order = o;
        } else if (key == "corner_scheme") {
            static const char* names[] = {"upwind", "avg_min", "linear_xy", "linear_diag", "multid"};
            int found = -1;
            for (int q = 0; q < 5; ++q)
                if (val == names[q]) found = q;
            if (found < 0)
                bad_line(line, "invalid corner_scheme '" + val + "' (valid: upwind, avg_min, linear_xy, linear_diag, multid)");
            rc.corner = static_cast<CornerScheme>(found);
        } else if (key == "cfl") {
            rc.cfl = number(val, line);
        } else if (key == "divisor") {
            rc.divisor = static_cast<int>(number(val, line));
        } else if (key == "t_end") {
            rc.t_end = number(val, line);
        } else if (key == "max_steps") {
            rc.max_steps = static_cast<int>(number(val, line));
        } else if (key == "out_dir") {
            rc.out_dir = val;
        } else if (key == "output_every") {
            rc.output_every = static_cast<int>(number(val, line));
        } else if (key == "seed") {
            rc.seed = static_cast<unsigned long>(number(val, line));
        } else {
            bad_line(line, "unknown key '" + key + "'");
        }
    }
    return rc;
}

RunConfig load_config(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw SimError("cannot open config file: " + path);
    std::ostringstream all;
    all << f.rdbuf();
    return parse_config(all.str());
}

CaseSpec configure_case(const RunConfig& rc) {
    if (rc.case_name.empty()) throw SimError("config is missing 'case'");
    CaseSpec cs = build_case(rc.case_name, rc.divisor);
    cs.scheme = rc.scheme;
    cs.recon.face_order = rc.face_order;
    cs.recon.corner = rc.corner;
    cs.cfl = rc.cfl;
    if (rc.t_end >= 0.0) cs.t_end = rc.t_end;
    if (rc.max_steps > 0) cs.max_steps = rc.max_steps;
    return cs;
}

}  // namespace hydro

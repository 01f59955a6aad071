// hydro/b200.hpp — C++ drop-in of the reference solver interface
// (proj/include/hydro/*.hpp) for the hot path, implemented over the C-ABI of
// include/h2d.h (CUDA sm_100a).  Reference callers include the usual
// per-topic headers (hydro/state.hpp, hydro/lagrange.hpp, hydro/remap.hpp,
// hydro/harness.hpp, ...), which all forward here.  Types keep the reference
// names, members and byte layout (so State fields are passed to the device
// without repacking); functions keep the reference signatures and exceptions.
//
// Provided (reference file:line of the replaced declaration):
//   Vec2, Rect                          vec2.hpp:7-38
//   SimError + 5 subclasses             errors.hpp:11-34
//   Field<T>, kGhost                    field.hpp:11-44
//   Mesh, BoundaryKind                  mesh.hpp:8-40
//   EosModel, eos_pressure, sound_speed eos.hpp:11-34
//   kMaxMat, kPureTol, kThermoTol, Material, MaterialSet, State, make_state,
//   nodal_mass, fill_ghosts, sync_derived, Totals, compute_totals
//                                       state.hpp:13-100
//   PseudoViscosityParams, LagrangeResult, lagrange_step   lagrange.hpp:7-59
//   CornerScheme, ReconConfig           reconstruct.hpp:7-13
//   RemapKind, RemapDiag, remap_step, update_interface_normals  remap.hpp:9-64
//   cfl_dt                              harness.hpp:64
//   cell_volume                         state.hpp:70
//   pseudo_viscosity, div_u_cell, grad_pq_node, HalfStepState, compute_q,
//   predict, correct                    lagrange.hpp:12-52
//   van_leer, limited_gradient_1d, Stencil1D, face_value, Stencil3x3,
//   CornerKin, corner_value, PlaneRecon, multid_plane, plane_eval
//                                       reconstruct.hpp:15-69
//   CornerFlux, cf_corner_flux, CfFaceFlux, cf_face_flux_x/_y,
//   ad_face_fluxes, remap_single_axis   remap.hpp:15-57
//   InterfaceLine, youngs_normal, clipped_fraction, place_interface
//                                       vof.hpp:13-31
//   ImposedVelocity, Region, CaseSpec, build_case, case_list, init_case,
//   l2_error, StepDiag, RunReport, StepHook, run, ConvergenceRow,
//   ConvergenceResult, convergence_study, scheme_name   harness.hpp:13-113
//   RunConfig, parse_config, load_config, configure_case  config.hpp:9-28
//   DumpFormat, write_fields, append_diag_line            io.hpp:9-22
// plus hydro::b200::Simulation, the device-resident run loop
// (harness.cpp:390-412) that keeps the State on the GPU between steps.
// Scalar functions evaluate on the device through h2d_scalar_eval (the step
// kernels' own device functions); run() keeps the State resident and
// downloads it only when a StepHook is installed.
#pragma once

#include <array>
#include <cmath>
#include <functional>
#include <iosfwd>
#include <stdexcept>
#include <string>
#include <vector>

namespace hydro {

// ---- geometry -------------------------------------------------------------
struct Vec2 {
    double x = 0.0, y = 0.0;
    Vec2() = default;
    Vec2(double x_, double y_) : x(x_), y(y_) {}
    Vec2& operator+=(const Vec2& o) { x += o.x; y += o.y; return *this; }
    Vec2& operator-=(const Vec2& o) { x -= o.x; y -= o.y; return *this; }
    Vec2& operator*=(double s) { x *= s; y *= s; return *this; }
};
inline Vec2 operator+(Vec2 a, const Vec2& b) { return a += b; }
inline Vec2 operator-(Vec2 a, const Vec2& b) { return a -= b; }
inline Vec2 operator*(double s, Vec2 a) { return a *= s; }
inline Vec2 operator*(Vec2 a, double s) { return a *= s; }
inline double dot(const Vec2& a, const Vec2& b) { return a.x * b.x + a.y * b.y; }
inline double cross(const Vec2& a, const Vec2& b) { return a.x * b.y - a.y * b.x; }
inline double norm(const Vec2& a) { return std::sqrt(a.x * a.x + a.y * a.y); }

struct Rect {
    Vec2 lo, hi;
    double width() const { return hi.x - lo.x; }
    double height() const { return hi.y - lo.y; }
    double area() const { return width() * height(); }
    Vec2 center() const { return {0.5 * (lo.x + hi.x), 0.5 * (lo.y + hi.y)}; }
};

// ---- located exceptions ----------------------------------------------------
class SimError : public std::runtime_error {
public:
    SimError(std::string what, int i = -1, int j = -1, int step = -1)
        : std::runtime_error(located(what, i, j, step)), i_(i), j_(j), step_(step) {}
    int i() const { return i_; }
    int j() const { return j_; }
    int step() const { return step_; }

    // already-formatted message coming back from the device
    struct Formatted {};
    SimError(Formatted, const std::string& full, int i, int j, int step)
        : std::runtime_error(full), i_(i), j_(j), step_(step) {}

private:
    static std::string located(const std::string& w, int i, int j, int step) {
        std::string s = w;
        if (i >= 0 || j >= 0) s += " at cell (" + std::to_string(i) + "," + std::to_string(j) + ")";
        if (step >= 0) s += " step " + std::to_string(step);
        return s;
    }
    int i_, j_, step_;
};
struct TangledCellError : SimError { using SimError::SimError; };
struct UnphysicalStateError : SimError { using SimError::SimError; };
struct NegativeMassError : SimError { using SimError::SimError; };
struct CflViolationError : SimError { using SimError::SimError; };
struct IsolatedMixedCellError : SimError { using SimError::SimError; };

// ---- ghosted fields ----------------------------------------------------------
inline constexpr int kGhost = 2;

template <class T>
class Field {
public:
    Field() = default;
    Field(int nx, int ny, T init = T{})
        : nx_(nx), ny_(ny), pitch_(nx + 2 * kGhost), v_(std::size_t(pitch_) * (ny + 2 * kGhost), init) {}
    int nx() const { return nx_; }
    int ny() const { return ny_; }
    T& operator()(int i, int j) { return v_[at(i, j)]; }
    const T& operator()(int i, int j) const { return v_[at(i, j)]; }
    void fill(T v) { v_.assign(v_.size(), v); }
    std::vector<T>& raw() { return v_; }
    const std::vector<T>& raw() const { return v_; }

private:
    std::size_t at(int i, int j) const { return std::size_t(j + kGhost) * pitch_ + std::size_t(i + kGhost); }
    int nx_ = 0, ny_ = 0, pitch_ = 0;
    std::vector<T> v_;
};

// ---- mesh, EOS, materials ------------------------------------------------------
enum class BoundaryKind { Periodic, Wall };

struct Mesh {
    int nx = 0, ny = 0;
    double dx = 0.0, dy = 0.0, x0 = 0.0, y0 = 0.0;
    BoundaryKind bc_x = BoundaryKind::Periodic, bc_y = BoundaryKind::Periodic;
    Mesh() = default;
    Mesh(int nx_, int ny_, double dx_, double dy_, double x0_ = 0.0, double y0_ = 0.0,
         BoundaryKind bx = BoundaryKind::Periodic, BoundaryKind by = BoundaryKind::Periodic)
        : nx(nx_), ny(ny_), dx(dx_), dy(dy_), x0(x0_), y0(y0_), bc_x(bx), bc_y(by) {
        if (nx < 3 || ny < 3) throw SimError("mesh must be at least 3x3");
        if (dx <= 0.0 || dy <= 0.0) throw SimError("mesh spacing must be positive");
    }
    double cell_volume() const { return dx * dy; }
    Vec2 cell_center(int i, int j) const { return {x0 + (i + 0.5) * dx, y0 + (j + 0.5) * dy}; }
    Vec2 node_pos(int i, int j) const { return {x0 + i * dx, y0 + j * dy}; }
    bool periodic_x() const { return bc_x == BoundaryKind::Periodic; }
    bool periodic_y() const { return bc_y == BoundaryKind::Periodic; }
    double char_length() const { return std::sqrt(dx * dy); }
};

struct EosModel {
    enum class Kind { Perfect, Stiffened };
    Kind kind = Kind::Perfect;
    double gamma = 1.4;
    double pi = 0.0;
    static EosModel perfect(double g) { return {Kind::Perfect, g, 0.0}; }
    static EosModel stiffened(double g, double p) { return {Kind::Stiffened, g, p}; }
};
inline double eos_pressure(const EosModel& q, double rho, double e) {
    double p = (q.gamma - 1.0) * rho * e;
    if (q.kind == EosModel::Kind::Stiffened) p -= q.pi;
    return p;
}
inline double sound_speed(const EosModel& q, double rho, double p) {
    const double pi = q.kind == EosModel::Kind::Stiffened ? q.pi : 0.0;
    const double c2 = q.gamma * (p + pi) / rho;
    if (!(c2 >= 0.0)) throw UnphysicalStateError("unphysical state: gamma*(P+pi)/rho < 0");
    return std::sqrt(c2);
}

inline constexpr int kMaxMat = 2;
inline constexpr double kPureTol = 1e-10;
inline constexpr double kThermoTol = 1e-6;

struct Material {
    std::string name;
    EosModel eos;
};
struct MaterialSet {
    int n = 1;
    std::array<Material, kMaxMat> mat{};
};

struct State {
    Mesh mesh;
    int nmat = 1;
    std::array<Field<double>, kMaxMat> m, e, k;
    Field<double> vol, m_mix, e_mix, rho_mix, p_mix;
    Field<Vec2> iface_normal;
    Field<Vec2> u;
    int step = 0;
    double time = 0.0;
};

State make_state(const Mesh& mesh, int nmat);
// two-triangle quad area, throws TangledCellError (state.hpp:70)
double cell_volume(const Vec2& p00, const Vec2& p10, const Vec2& p11, const Vec2& p01);
double nodal_mass(const State& s, int i, int j);
Field<double> nodal_masses(const State& s);
void fill_ghost_cells(const Mesh& mesh, Field<double>& f);
void fill_ghost_cells(const Mesh& mesh, Field<Vec2>& f);
void fill_ghost_nodes(const Mesh& mesh, Field<Vec2>& u);
void fill_ghosts(State& s);
void sync_derived(State& s, const MaterialSet& mats);

struct Totals {
    double mass = 0.0;
    std::array<double, kMaxMat> mass_mat{};
    Vec2 momentum;
    double internal_energy = 0.0;
};
Totals compute_totals(const State& s);

// ---- Lagrangian phase -------------------------------------------------------------
struct PseudoViscosityParams {
    double a1 = 0.2;
    double a2 = 1.0;
};
struct LagrangeResult {
    Field<Vec2> u_half, u_lag;
    std::array<Field<double>, kMaxMat> e_lag;
    Field<double> vol_lag, q;
    int floor_count = 0;
};
double pseudo_viscosity(double rho, double c_sound, double div_u, const PseudoViscosityParams& prm, double L);
double div_u_cell(const Mesh& mesh, const Field<Vec2>& u, int i, int j);
Vec2 grad_pq_node(const Mesh& mesh, const Field<double>& p, const Field<double>& q, int i, int j);
struct HalfStepState {
    Field<Vec2> x_half;
    Field<Vec2> u_half;
    Field<double> vol_half;
    std::array<Field<double>, kMaxMat> e_half;
    std::array<Field<double>, kMaxMat> p_half;
    Field<double> p_mix_half;
    Field<double> q;
    int floor_count = 0;
};
Field<double> compute_q(const State& s, const MaterialSet& mats, const PseudoViscosityParams& prm);
HalfStepState predict(const State& s, const MaterialSet& mats, double dt, const PseudoViscosityParams& prm);
LagrangeResult correct(const State& s, const MaterialSet& mats, const HalfStepState& half, double dt);
// the reference inlines correct(predict(...)) (lagrange.hpp:56-59); the device
// runs the same arithmetic in two fused kernels
LagrangeResult lagrange_step(const State& s, const MaterialSet& mats, double dt, const PseudoViscosityParams& prm);

// ---- remap -------------------------------------------------------------------------
enum class CornerScheme { Upwind, AvgMin, LinearXY, LinearDiag, Multid };
struct ReconConfig {
    int face_order = 2;
    CornerScheme corner = CornerScheme::LinearDiag;
    bool interface_degrade = true;
};
double van_leer(double r);
double limited_gradient_1d(double am, double ac, double ap, double xm, double xc, double xp);
struct Stencil1D {
    double a[3];
    double x[3];
};
double face_value(int order, const Stencil1D& donor, double sgn_dvol, double lag_width, double u_face_dt);
struct Stencil3x3 {
    double a[3][3];
    Vec2 xl[3][3];
};
struct CornerKin {
    double dxp = 0.0, dyp = 0.0;
    double lag_wx = 0.0, lag_wy = 0.0;
    double sgn_fx = 0.0, u_fx_dt = 0.0;
    double sgn_fy = 0.0, u_fy_dt = 0.0;
    Vec2 eval_rel;
    double dx = 1.0, dy = 1.0;
};
double corner_value(CornerScheme scheme, const Stencil3x3& st, const CornerKin& kin);
struct PlaneRecon {
    double a0 = 0.0;
    Vec2 center;
    Vec2 grad_raw;
    Vec2 grad;
};
PlaneRecon multid_plane(const Stencil3x3& st, double dx, double dy);
inline double plane_eval(const PlaneRecon& pl, const Vec2& x) { return pl.a0 + dot(pl.grad, x - pl.center); }

// ---- vof.hpp (vof.hpp:13-31) -----------------------------------------------------
struct InterfaceLine {
    Vec2 normal;
    double d = 0.0;
};
Vec2 youngs_normal(const Field<double>& k1, int i, int j, double dx, double dy);
double clipped_fraction(double w, double h, const Vec2& n, double d);
InterfaceLine place_interface(double frac, const Vec2& n, const Rect& proxy);

enum class RemapKind { AD, Direct, DirectCF };
enum class Axis { X, Y };
struct CornerFlux {
    double dvol = 0.0;
    int sx = 0;
    int sy = 0;
};
CornerFlux cf_corner_flux(const Vec2& u_half, double dt);
struct CfFaceFlux {
    double dvol = 0.0;
    double wlo = 0.0;
    double whi = 0.0;
};
CfFaceFlux cf_face_flux_x(double ym, double yp, const Vec2& disp_m, const Vec2& disp_p);
CfFaceFlux cf_face_flux_y(double xm, double xp, const Vec2& disp_m, const Vec2& disp_p);
Field<double> ad_face_fluxes(Axis axis, const Mesh& mesh, const Field<Vec2>& u_half, double dt);
struct RemapDiag {
    double max_k_violation = 0.0;
    int k_clip_count = 0;
    int mass_fix_count = 0;
};
State remap_step(const State& s, const MaterialSet& mats, const LagrangeResult& lag, double dt, RemapKind kind,
                 const ReconConfig& rc, bool x_first = true, bool remap_velocity = true, RemapDiag* diag = nullptr);
State remap_single_axis(const State& s, const MaterialSet& mats, const LagrangeResult& lag, double dt, Axis axis,
                        const ReconConfig& rc, bool remap_velocity = true, RemapDiag* diag = nullptr);
void update_interface_normals(State& s);

// ---- harness -------------------------------------------------------------------------
enum class ImposedVelocity { None, Constant, Rotation };
struct Region {
    enum class Shape { All, HalfPlaneX, Rectangle, Circle };
    Shape shape = Shape::All;
    double xsplit = 0.0;
    Rect rect;
    Vec2 center;
    double radius = 0.0;
    int mat = 0;
    double rho = 1.0;
    double p = 1e5;
    Vec2 u;
};
struct CaseSpec {
    std::string name;
    int nx = 0, ny = 0;
    double x0 = 0.0, y0 = 0.0, lx = 1.0, ly = 1.0;
    BoundaryKind bc_x = BoundaryKind::Periodic;
    BoundaryKind bc_y = BoundaryKind::Periodic;
    MaterialSet mats;
    std::vector<Region> regions;
    double t_end = 0.0;
    double cfl = 0.3;
    int max_steps = 0;
    RemapKind scheme = RemapKind::DirectCF;
    ReconConfig recon;
    PseudoViscosityParams pv;
    ImposedVelocity imposed = ImposedVelocity::None;
    Vec2 u_const;
    double flip_time = -1.0;
    Vec2 rot_center;
    double rot_omega = 0.0;
    Mesh make_mesh() const;
};
CaseSpec build_case(const std::string& name, int divisor = 1);
std::vector<std::string> case_list();
State init_case(const CaseSpec& cs);
double cfl_dt(const State& s, const MaterialSet& mats, double cfl);
double l2_error(const Field<double>& a, const Field<double>& b, const Mesh& mesh);

// StepDiag, harness.hpp:66-72 (the record run() appends per step)
struct StepDiag {
    int step = 0;
    double t = 0.0, dt = 0.0;
    Totals totals;
    double min_rho = 0.0, max_rho = 0.0;
    double min_p = 0.0, max_p = 0.0;
};

struct RunReport {
    CaseSpec spec;
    std::vector<StepDiag> series;
    State initial_state;
    State final_state;
    int steps = 0;
    double wall_seconds = 0.0;
    double max_k_violation = 0.0;
    int k_clip_count = 0;
    int mass_fix_count = 0;
    int energy_floor_count = 0;
    double l2_rho_vs_initial = 0.0;
    double l2_k_vs_initial = 0.0;
};
using StepHook = std::function<void(const State&, const StepDiag&)>;
// the run loop (harness.cpp:380-424) with the State resident on the device;
// a hook receives the downloaded State after every step
RunReport run(const CaseSpec& cs, const StepHook& hook = {});
struct ConvergenceRow {
    int n = 0;
    double err = 0.0;
};
struct ConvergenceResult {
    RemapKind scheme{};
    std::vector<ConvergenceRow> rows;
    double slope = 0.0;
};
std::vector<ConvergenceResult> convergence_study(const std::string& case_name, const std::vector<int>& meshes,
                                                 const std::vector<RemapKind>& schemes);
const char* scheme_name(RemapKind k);

// ---- config.hpp (config.hpp:9-28) ------------------------------------------------------
struct RunConfig {
    std::string case_name;
    RemapKind scheme = RemapKind::DirectCF;
    int face_order = 2;
    CornerScheme corner = CornerScheme::LinearDiag;
    double cfl = 0.3;
    int divisor = 1;
    double t_end = -1.0;
    int max_steps = 0;
    std::string out_dir = "out";
    int output_every = 0;
    unsigned long seed = 0;
};
RunConfig parse_config(const std::string& text);
RunConfig load_config(const std::string& path);
CaseSpec configure_case(const RunConfig& rc);

// ---- io.hpp (io.hpp:9-22): the reference's CSV / legacy-VTK cell dump and
// the conservation-ledger line, byte-identical output
enum class DumpFormat { Csv, VtkLegacyAscii };
void write_fields(const State& s, const std::string& path, DumpFormat fmt);
void write_fields(const State& s, std::ostream& out, DumpFormat fmt);
void append_diag_line(std::ostream& out, int step, double t, double dt, const Totals& totals, double min_rho,
                      double max_rho, double min_p, double max_p);

namespace b200 {

struct StepInfo {
    int steps_done = 0;
    int floor_count = 0;
    std::vector<double> dts;
    // make_diag of every new State (RunReport::series[1:], harness.cpp:410),
    // reduced on the device inside the step (see h2d.h, h2d_step_diag)
    std::vector<StepDiag> series;
};

// Device-resident run loop: the State lives on the GPU between steps; only
// upload() / download() move it (harness.cpp:390-412 without the hook).
class Simulation {
public:
    Simulation(const State& initial, const MaterialSet& mats, const PseudoViscosityParams& pv = {},
               const ReconConfig& rc = {}, int device = 0);
    ~Simulation();
    Simulation(const Simulation&) = delete;
    Simulation& operator=(const Simulation&) = delete;

    void upload(const State& s);
    State download() const;
    // runs until s.step >= max_steps (if > 0) or time >= t_end; throws the
    // reference exception of the first failing step
    StepInfo run(int max_steps, double t_end, double cfl, RemapDiag* diag = nullptr);
    // make_diag(s, dt) of the resident State (harness.cpp:360-376), e.g. series[0]
    StepDiag diag_now(double dt = 0.0) const;
    // write_fields of the resident State (io.hpp:17) without a State copy in the caller
    void write_fields(const std::string& path, DumpFormat fmt) const;
    // binary checkpoint of the resident State; load() resumes bit-exactly
    void save(const std::string& path) const;
    void load(const std::string& path);

private:
    void* ctx_ = nullptr;
    Mesh mesh_;
    int nmat_ = 1;
};

}  // namespace b200
}  // namespace hydro

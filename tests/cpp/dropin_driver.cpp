// dropin_driver.cpp — ONE source compiled twice: against the reference
// (proj/include + the reference library, oracle/Makefile target `dropin`) and
// against the B200 drop-in (include/hydro + libh2d.so, tests/cpp/Makefile).
// It uses only the reference's public solver API the way reference callers do
// (harness.cpp:390-412 run loop; test_remap.cpp kinematic() remaps) and
// writes every dt, counter, caught exception and final State byte to argv[1].
// test_dropin.py requires the two output files to be identical.
#include "hydro/lagrange.hpp"
#include "hydro/remap.hpp"
#include "hydro/state.hpp"
#include "hydro/harness.hpp"
#include "hydro/io.hpp"

#include <cmath>
#include <cstdio>
#include <random>
#include <sstream>
#include <string>
#include <typeinfo>
#include <vector>

using namespace hydro;

static FILE* out;

static void put(const void* p, size_t n) { std::fwrite(p, 1, n, out); }
static void put_d(double v) { put(&v, sizeof v); }
static void put_i(int v) { put(&v, sizeof v); }
static void put_s(const std::string& s) {
    put_i(static_cast<int>(s.size()));
    put(s.data(), s.size());
}
static void put_field(const Field<double>& f) { put(f.raw().data(), f.raw().size() * sizeof(double)); }
static void put_vfield(const Field<Vec2>& f) { put(f.raw().data(), f.raw().size() * sizeof(Vec2)); }
static void put_state(const State& s) {
    for (int a = 0; a < s.nmat; ++a) {
        put_field(s.m[a]);
        put_field(s.e[a]);
        put_field(s.k[a]);
    }
    put_field(s.vol);
    put_field(s.m_mix);
    put_field(s.e_mix);
    put_field(s.rho_mix);
    put_field(s.p_mix);
    put_vfield(s.iface_normal);
    put_vfield(s.u);
    put_i(s.step);
    put_d(s.time);
}
template <class E>
static void put_error(const E& e) {
    put_s(e.what());
    put_i(e.i());
    put_i(e.j());
}

// run loop of harness.cpp:390-412 on a caller-built State
static void run_loop(State s, const MaterialSet& mats, double cfl, int steps, const char* tag,
                     RemapKind kind = RemapKind::DirectCF) {
    put_s(tag);
    RemapDiag diag;
    int floors = 0;
    try {
        for (int n = 0; n < steps; ++n) {
            const double dt = cfl_dt(s, mats, cfl);
            put_d(dt);
            LagrangeResult lag = lagrange_step(s, mats, dt, PseudoViscosityParams{});
            floors += lag.floor_count;
            s = remap_step(s, mats, lag, dt, kind, ReconConfig{}, s.step % 2 == 0, true, &diag);
        }
        put_s("ok");
    } catch (const UnphysicalStateError& e) {
        put_s("UnphysicalStateError");
        put_error(e);
    } catch (const SimError& e) {
        put_s("SimError");
        put_error(e);
    }
    put_i(floors);
    put_d(diag.max_k_violation);
    put_i(diag.k_clip_count);
    put_i(diag.mass_fix_count);
    put_state(s);
    const Totals t = compute_totals(s);
    put_d(t.mass);
    put_d(t.internal_energy);
    put_d(t.momentum.x);
    put_d(t.momentum.y);
    // io.hpp: the cell dumps and the ledger line of the final State
    std::ostringstream csv, vtk, line;
    write_fields(s, csv, DumpFormat::Csv);
    write_fields(s, vtk, DumpFormat::VtkLegacyAscii);
    append_diag_line(line, s.step, s.time, 0.5, t, 0.25, 4.0, 0.1, 9.0);
    put_s(csv.str().c_str());
    put_s(vtk.str().c_str());
    put_s(line.str().c_str());
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    out = std::fopen(argv[1], "wb");
    if (!out) return 3;

    // 1. two-state Riemann problem, one material, walls (config 1 at 64^2)
    {
        MaterialSet mats;
        mats.mat[0] = {"gas", EosModel::perfect(1.4)};
        Mesh mesh(64, 64, 1.0 / 64, 1.0 / 64, 0.0, 0.0, BoundaryKind::Wall, BoundaryKind::Wall);
        State s = make_state(mesh, 1);
        for (int j = 0; j < 64; ++j)
            for (int i = 0; i < 64; ++i) {
                const bool left = mesh.cell_center(i, j).x < 0.5;
                const double rho = left ? 1.0 : 0.125, p = left ? 1.0 : 0.1;
                s.m[0](i, j) = rho * mesh.cell_volume();
                s.e[0](i, j) = p / (0.4 * rho);
            }
        fill_ghosts(s);
        sync_derived(s, mats);
        run_loop(s, mats, 0.5, 60, "riemann");
        run_loop(s, mats, 0.5, 60, "riemann_ad", RemapKind::AD);
    }
    // 2. two materials: a disc of material 1 in a moving material-0 slab
    {
        MaterialSet mats;
        mats.n = 2;
        mats.mat[0] = {"A", EosModel::perfect(1.4)};
        mats.mat[1] = {"B", EosModel::stiffened(4.4, 0.6)};
        Mesh mesh(48, 40, 0.025, 0.025, 0.0, 0.0, BoundaryKind::Wall, BoundaryKind::Periodic);
        State s = make_state(mesh, 2);
        for (int j = 0; j < 40; ++j)
            for (int i = 0; i < 48; ++i) {
                int inside = 0;
                for (int q = 0; q < 8; ++q)
                    for (int p = 0; p < 8; ++p) {
                        const double x = (i + (p + 0.5) / 8.0) * 0.025 - 0.6, y = (j + (q + 0.5) / 8.0) * 0.025 - 0.5;
                        inside += x * x + y * y <= 0.04;
                    }
                const double k1 = inside / 64.0, k0 = 1.0 - k1;
                s.k[0](i, j) = k0;
                s.k[1](i, j) = k1;
                s.m[0](i, j) = k0 * 1.0 * mesh.cell_volume();
                s.m[1](i, j) = k1 * 3.0 * mesh.cell_volume();
                s.e[0](i, j) = k0 > 0.0 ? 2.5 : 0.0;
                s.e[1](i, j) = k1 > 0.0 ? 1.2 : 0.0;
            }
        for (int j = 0; j <= 40; ++j)
            for (int i = 0; i <= 48; ++i) s.u(i, j) = Vec2{i < 12 ? 0.4 : 0.0, 0.0};
        fill_ghosts(s);
        sync_derived(s, mats);
        update_interface_normals(s);
        run_loop(s, mats, 0.3, 40, "disc");
        run_loop(s, mats, 0.3, 40, "disc_ad", RemapKind::AD);
    }
    // 3. kinematic remaps on a periodic grid (test_remap.cpp:46-54 pattern)
    {
        MaterialSet mats;
        mats.mat[0] = {"air", EosModel::perfect(1.4)};
        Mesh mesh(12, 10, 1.0, 1.0);
        State s = make_state(mesh, 1);
        std::mt19937_64 rng(31);
        std::uniform_real_distribution<double> d(0.5, 2.0), vu(-0.2, 0.2);
        for (int j = 0; j < 10; ++j)
            for (int i = 0; i < 12; ++i) {
                s.m[0](i, j) = d(rng);
                s.e[0](i, j) = d(rng);
            }
        Field<Vec2> u(13, 11);
        for (int j = 0; j < 10; ++j)
            for (int i = 0; i < 12; ++i) u(i, j) = {vu(rng), vu(rng)};
        for (int j = 0; j <= 10; ++j) u(12, j) = u(0, j % 10);
        for (int i = 0; i <= 12; ++i) u(i, 10) = u(i % 12, 0);
        fill_ghosts(s);
        s.u = u;
        fill_ghost_nodes(s.mesh, s.u);
        sync_derived(s, mats);
        LagrangeResult lag;
        lag.u_half = s.u;
        lag.u_lag = s.u;
        lag.e_lag[0] = s.e[0];
        lag.vol_lag = s.vol;
        lag.q = Field<double>(12, 10);
        for (int order : {1, 2}) {
            ReconConfig rc;
            rc.face_order = order;
            rc.corner = order == 1 ? CornerScheme::Upwind : CornerScheme::LinearDiag;
            const State o = remap_step(s, mats, lag, 1.0, RemapKind::DirectCF, rc);
            put_s("kinematic");
            put_state(o);
            // the faces-only Direct engine (remap.cpp:593-724) and AD through
            // the same call: each RemapKind must reach its own engine
            const State od = remap_step(s, mats, lag, 1.0, RemapKind::Direct, rc);
            put_s("kinematic direct");
            put_state(od);
            const State oa = remap_step(s, mats, lag, 1.0, RemapKind::AD, rc, order == 1);
            put_s("kinematic ad");
            put_state(oa);
        }
        // CFL refusal with a located error (test_remap.cpp:505-513)
        Field<Vec2> fast(13, 11, Vec2{0.95, 0.0});
        lag.u_half = fast;
        lag.u_lag = fast;
        try {
            (void)remap_step(s, mats, lag, 1.0, RemapKind::DirectCF, ReconConfig{});
            put_s("no error");
        } catch (const CflViolationError& e) {
            put_s("CflViolationError");
            put_error(e);
        }
    }
    std::fclose(out);
    return 0;
}

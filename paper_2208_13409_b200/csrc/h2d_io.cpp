// h2d_io.cpp — field readback formats and State checkpoints (SURVEY.md 8f
// row 3), host side of libh2d.so.
//
// * write_fields (reference io.hpp:11-18, io.cpp:15-83): the CSV / legacy-VTK
//   cell dump, byte-identical to the reference's text ("%.17g" numbers, the
//   same column order, the same cell-mean velocity arithmetic).
// * append_diag_line (io.hpp:20-22, io.cpp:85-92): the conservation ledger.
// * A binary State checkpoint (no reference counterpart, SPEC non-goal): the
//   persistent State in the reference Field layout, so a run can stop and
//   resume bit-exactly.
//
// The device entry points download the resident State into pinned staging
// and format it on the host; nothing here runs a kernel of its own.
#include "h2d_io.h"

#include <cinttypes>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

constexpr int G = H2D_GHOST;

// fixed 17-significant-digit decimal text, locale-independent (io.cpp:15-19)
inline void num(std::string& o, double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    o += buf;
}
inline void inum(std::string& o, long long v) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "%lld", v);
    o += buf;
}

struct View {
    const h2d_mesh& m;
    int nmat;
    const h2d_state& s;
    size_t C(int i, int j) const { return (size_t)(j + G) * (m.nx + 2 * G) + (i + G); }
    size_t N(int i, int j) const { return (size_t)(j + G) * (m.nx + 1 + 2 * G) + (i + G); }
    double rho(int i, int j) const { return s.rho_mix[C(i, j)]; }
    double e(int i, int j) const { return s.e_mix[C(i, j)]; }
    double p(int i, int j) const { return s.p_mix[C(i, j)]; }
    double k0(int i, int j) const { return s.k[0][C(i, j)]; }
    // the reference format has k0 and k1 columns only; a three-material State
    // dumps its first two fractions
    double k1(int i, int j) const { return nmat >= 2 ? s.k[1][C(i, j)] : 0.0; }
    // cell_u_mean (io.cpp:21-23): 0.25 * (((u00 + u10) + u01) + u11), per component
    double um(int i, int j, int c) const {
        const double* u = s.u;
        return 0.25 * (((u[2 * N(i, j) + c] + u[2 * N(i + 1, j) + c]) + u[2 * N(i, j + 1) + c]) +
                       u[2 * N(i + 1, j + 1) + c]);
    }
};

bool check_view(const h2d_state* s, int nmat) {
    if (!s || !s->rho_mix || !s->e_mix || !s->p_mix || !s->k[0] || !s->u) return false;
    return !(nmat >= 2 && !s->k[1]);
}

// write_csv, io.cpp:25-39
void csv(const View& v, std::string& o) {
    o += "i,j,x,y,rho,e,p,k0,k1,ux_mean,uy_mean\n";
    const h2d_mesh& m = v.m;
    for (int j = 0; j < m.ny; ++j)
        for (int i = 0; i < m.nx; ++i) {
            inum(o, i);
            o += ',';
            inum(o, j);
            o += ',';
            num(o, m.x0 + (i + 0.5) * m.dx);  // Mesh::cell_center, mesh.hpp:32
            o += ',';
            num(o, m.y0 + (j + 0.5) * m.dy);
            o += ',';
            num(o, v.rho(i, j));
            o += ',';
            num(o, v.e(i, j));
            o += ',';
            num(o, v.p(i, j));
            o += ',';
            num(o, v.k0(i, j));
            o += ',';
            num(o, v.k1(i, j));
            o += ',';
            num(o, v.um(i, j, 0));
            o += ',';
            num(o, v.um(i, j, 1));
            o += '\n';
        }
}

// write_vtk + write_scalar_block, io.cpp:41-70
void vtk(const View& v, int step, double time, std::string& o) {
    const h2d_mesh& m = v.m;
    o += "# vtk DataFile Version 3.0\nhydro2d fields step ";
    inum(o, step);
    o += " time ";
    num(o, time);
    o += "\nASCII\nDATASET STRUCTURED_POINTS\nDIMENSIONS ";
    inum(o, m.nx + 1);
    o += ' ';
    inum(o, m.ny + 1);
    o += " 1\nORIGIN ";
    num(o, m.x0);
    o += ' ';
    num(o, m.y0);
    o += " 0\nSPACING ";
    num(o, m.dx);
    o += ' ';
    num(o, m.dy);
    o += " 1\nCELL_DATA ";
    inum(o, (long long)m.nx * m.ny);
    o += '\n';
    auto block = [&](const char* name, auto get) {
        o += "SCALARS ";
        o += name;
        o += " double 1\nLOOKUP_TABLE default\n";
        for (int j = 0; j < m.ny; ++j)
            for (int i = 0; i < m.nx; ++i) {
                num(o, get(i, j));
                o += '\n';
            }
    };
    block("rho", [&](int i, int j) { return v.rho(i, j); });
    block("e", [&](int i, int j) { return v.e(i, j); });
    block("p", [&](int i, int j) { return v.p(i, j); });
    block("k0", [&](int i, int j) { return v.k0(i, j); });
    block("k1", [&](int i, int j) { return v.k1(i, j); });
    block("ux_mean", [&](int i, int j) { return v.um(i, j, 0); });
    block("uy_mean", [&](int i, int j) { return v.um(i, j, 1); });
}

int write_file(const char* path, const std::string& text) {
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return H2D_ERR_SIM;  // SimError("cannot write: " + path), io.cpp:79
    const size_t n = std::fwrite(text.data(), 1, text.size(), f);
    const int bad = std::fclose(f) != 0 || n != text.size();
    return bad ? H2D_ERR_SIM : H2D_OK;  // SimError("write failed: " + path), io.cpp:81
}

// ---- checkpoint --------------------------------------------------------------
constexpr char kMagic[8] = {'H', '2', 'D', 'S', 'T', 'A', 'T', '1'};
struct CkptHeader {
    char magic[8];
    int32_t nx, ny, nmat, ghost, step, pad;
    double time, dx, dy, x0, y0;
    int32_t bc_x, bc_y;
};

size_t cell_count(const h2d_mesh& m) { return (size_t)(m.nx + 2 * G) * (m.ny + 2 * G); }
size_t node_count(const h2d_mesh& m) { return (size_t)(m.nx + 1 + 2 * G) * (m.ny + 1 + 2 * G); }

// the persistent State (state.hpp:43-62) in Field order: m, e, k per
// material, vol, m_mix, e_mix, rho_mix, p_mix, iface_normal, u
template <class F>
void for_fields(const h2d_mesh& m, int nmat, h2d_state& s, F f) {
    const size_t nc = cell_count(m), nn = node_count(m);
    for (int a = 0; a < nmat; ++a) f(s.m[a], nc);
    for (int a = 0; a < nmat; ++a) f(s.e[a], nc);
    for (int a = 0; a < nmat; ++a) f(s.k[a], nc);
    f(s.vol, nc);
    f(s.m_mix, nc);
    f(s.e_mix, nc);
    f(s.rho_mix, nc);
    f(s.p_mix, nc);
    f(s.iface_normal, 2 * nc);
    f(s.u, 2 * nn);
}

}  // namespace

namespace h2d_io {

bool format_fields(const h2d_config& cfg, const h2d_state& s, int fmt, std::string& text) {
    if (!check_view(&s, cfg.nmat) || (fmt != H2D_DUMP_CSV && fmt != H2D_DUMP_VTK)) return false;
    const View v{cfg.mesh, cfg.nmat, s};
    text.clear();
    text.reserve((size_t)cfg.mesh.nx * cfg.mesh.ny * (fmt == H2D_DUMP_CSV ? 200 : 170) + 512);
    if (fmt == H2D_DUMP_CSV)
        csv(v, text);
    else
        vtk(v, s.step, s.time, text);
    return true;
}

std::string diag_line(const h2d_step_diag& dd) {
    const h2d_step_diag* d = &dd;
    // append_diag_line, io.cpp:85-92
    std::string o;
    inum(o, d->step);
    o += ' ';
    num(o, d->t);
    o += ' ';
    num(o, d->dt);
    o += " mass=";
    num(o, d->mass);
    o += " mass0=";
    num(o, d->mass_mat[0]);
    o += " mass1=";
    num(o, d->mass_mat[1]);
    o += " momx=";
    num(o, d->momentum_x);
    o += " momy=";
    num(o, d->momentum_y);
    o += " eint=";
    num(o, d->internal_energy);
    o += " rho=[";
    num(o, d->min_rho);
    o += ',';
    num(o, d->max_rho);
    o += "] p=[";
    num(o, d->min_p);
    o += ',';
    num(o, d->max_p);
    o += "]\n";
    return o;
}

}  // namespace h2d_io

extern "C" {

int h2d_write_fields_host(const h2d_config* cfg, const h2d_state* s, const char* path, int fmt) {
    if (!cfg || !s || !path) return H2D_ERR_INVALID;
    std::string text;
    if (!h2d_io::format_fields(*cfg, *s, fmt, text)) return H2D_ERR_INVALID;
    return write_file(path, text);
}

int h2d_diag_line(const h2d_step_diag* d, char* buf, int cap) {
    if (!d || !buf || cap <= 0) return H2D_ERR_INVALID;
    const std::string o = h2d_io::diag_line(*d);
    if ((int)o.size() + 1 > cap) return H2D_ERR_INVALID;
    std::memcpy(buf, o.c_str(), o.size() + 1);
    return H2D_OK;
}

int h2d_save_state_host(const h2d_config* cfg, const h2d_state* s, const char* path) {
    if (!cfg || !s || !path) return H2D_ERR_INVALID;
    CkptHeader h{};
    std::memcpy(h.magic, kMagic, 8);
    const h2d_mesh& m = cfg->mesh;
    h.nx = m.nx;
    h.ny = m.ny;
    h.nmat = cfg->nmat;
    h.ghost = G;
    h.step = s->step;
    h.time = s->time;
    h.dx = m.dx;
    h.dy = m.dy;
    h.x0 = m.x0;
    h.y0 = m.y0;
    h.bc_x = m.bc_x;
    h.bc_y = m.bc_y;
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return H2D_ERR_SIM;
    bool ok = std::fwrite(&h, sizeof h, 1, f) == 1;
    h2d_state v = *s;
    for_fields(m, cfg->nmat, v, [&](double* p, size_t n) {
        if (!ok) return;
        if (!p) {
            ok = false;
            return;
        }
        ok = std::fwrite(p, sizeof(double), n, f) == n;
    });
    ok = (std::fclose(f) == 0) && ok;
    return ok ? H2D_OK : H2D_ERR_SIM;
}

int h2d_load_state_host(const h2d_config* cfg, h2d_state* s, const char* path) {
    if (!cfg || !s || !path) return H2D_ERR_INVALID;
    std::FILE* f = std::fopen(path, "rb");
    if (!f) return H2D_ERR_SIM;
    CkptHeader h{};
    const h2d_mesh& m = cfg->mesh;
    bool ok = std::fread(&h, sizeof h, 1, f) == 1 && std::memcmp(h.magic, kMagic, 8) == 0 && h.nx == m.nx &&
              h.ny == m.ny && h.nmat == cfg->nmat && h.ghost == G && h.dx == m.dx && h.dy == m.dy &&
              h.x0 == m.x0 && h.y0 == m.y0 && h.bc_x == m.bc_x && h.bc_y == m.bc_y;
    if (!ok) {
        std::fclose(f);
        return H2D_ERR_INVALID;  // not a checkpoint of this mesh / material count
    }
    for_fields(m, cfg->nmat, *s, [&](double* p, size_t n) {
        if (!ok) return;
        if (!p) {
            ok = false;
            return;
        }
        ok = std::fread(p, sizeof(double), n, f) == n;
    });
    std::fclose(f);
    if (!ok) return H2D_ERR_SIM;
    s->step = h.step;
    s->time = h.time;
    return H2D_OK;
}

}  // extern "C"

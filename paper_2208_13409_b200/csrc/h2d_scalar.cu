// h2d_scalar.cu — the reference's public scalar kernels evaluated on the
// device (h2d_scalar_eval, H2D_SC_* in include/h2d.h): one record per thread,
// each op calling the SAME device functions the step kernels use
// (h2d_device.cuh: van_leer, lim_grad, face_value2, corner_diag,
// corner_value_other, multid_plane, clipped_fraction, place_interface), so the
// C++ drop-in's scalar API (reconstruct.hpp, vof.hpp, remap.hpp,
// lagrange.hpp, state.hpp free functions) answers with the step's own
// arithmetic.  A record whose reference call would throw sets flags[r] (the
// host re-throws the reference exception class).
#include "../../include/h2d.h"
#include "h2d_launch.h"

namespace h2d {

namespace {

constexpr int IN = H2D_SC_IN, OUT = H2D_SC_OUT;

// quad_volume_disp (lagrange.cpp:36-46) is per mesh; cell_volume (state.cpp:25-32)
// is the same two-triangle split on absolute node positions
__device__ double cell_volume4(const double* p, bool& tangled) {
    const double p00x = p[0], p00y = p[1], p10x = p[2], p10y = p[3];
    const double p11x = p[4], p11y = p[5], p01x = p[6], p01y = p[7];
    const double ax = p10x - p00x, ay = p10y - p00y, bx = p01x - p00x, by = p01y - p00y;
    const double cx = p01x - p11x, cy = p01y - p11y, ex = p10x - p11x, ey = p10y - p11y;
    const double s1 = 0.5 * (ax * by - ay * bx);
    const double s2 = 0.5 * (cx * ey - cy * ex);
    if (s1 <= 0.0 || s2 <= 0.0) tangled = true;
    return s1 + s2;
}

// cf_face_flux_x (remap.cpp:27-47) on (ym, yp, dm, dp)
__device__ void cf_face_flux(double ym, double yp, double dmx, double dmy, double dpx, double dpy, double* o) {
    o[0] = o[1] = o[2] = 0.0;
    const double wlo = ym + rmax(0.0, dmy);
    const double whi = yp + rmin(0.0, dpy);
    if (whi <= wlo) return;
    o[1] = wlo;
    o[2] = whi;
    const double den = (yp + dpy) - (ym + dmy);
    double xlo, xhi;
    if (fabs(den) < 1e-300) {
        xlo = xhi = 0.5 * (dmx + dpx);
    } else {
        const double slope = (dpx - dmx) / den;
        xlo = dmx + slope * (wlo - (ym + dmy));
        xhi = dmx + slope * (whi - (ym + dmy));
    }
    o[0] = 0.5 * (xlo + xhi) * (whi - wlo);
}

__global__ void k_scalar(int op, int n, const double* __restrict__ in, double* __restrict__ out,
                         int* __restrict__ flags) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const double* x = in + (size_t)r * IN;
    double* o = out + (size_t)r * OUT;
#pragma unroll
    for (int q = 0; q < OUT; ++q) o[q] = 0.0;
    bool bad = false;
    switch (op) {
    case H2D_SC_VAN_LEER:
        o[0] = van_leer(x[0]);
        break;
    case H2D_SC_LIMITED_GRADIENT:
        o[0] = lim_grad(x[0], x[1], x[2], x[3], x[4], x[5], bad);
        break;
    case H2D_SC_FACE_VALUE:  // face_value (reconstruct.cpp:26-31)
        o[0] = x[0] <= 1.0 ? x[2] : face_value2(x[1], x[2], x[3], x[4], x[5], x[6], x[7], x[8], x[9], bad);
        break;
    case H2D_SC_CORNER_VALUE: {  // corner_value (reconstruct.cpp:116-152)
        const int scheme = (int)x[0];
        const double* a = x + 1;
        const double* xlx = x + 10;
        const double* xly = x + 19;
        const double* k = x + 28;  // dxp dyp lwx lwy sfx ufx sfy ufy erx ery dx dy
        const double kdx = k[10], kdy = k[11];
        const double diag = sqrt(kdx * kdx + kdy * kdy);
        Dev d{};
        d.dgx = kdx / diag;
        d.dgy = kdy / diag;
        if (scheme == CS_UPWIND) {
            o[0] = a[4];
        } else if (scheme == CS_LINEARDIAG) {
            o[0] = corner_diag(d, a, xlx, xly, k[0], k[1], k[2], k[3], bad);
        } else {
            const Kin kin{k[0], k[1], k[2], k[3], k[4], k[5], k[6], k[7], k[8], k[9]};
            o[0] = corner_value_other(scheme, d.dgx, d.dgy, a, xlx, xly, kin, &bad);
        }
        break;
    }
    case H2D_SC_MULTID_PLANE: {  // multid_plane (reconstruct.cpp:74-107)
        const double kdx = x[27], kdy = x[28];
        const double diag = sqrt(kdx * kdx + kdy * kdy);
        double a0, cx, cy, gx, gy, graw[2] = {0.0, 0.0};
        multid_plane(kdx / diag, kdy / diag, x, x + 9, x + 18, a0, cx, cy, gx, gy, bad, graw);
        o[0] = a0;
        o[1] = cx;
        o[2] = cy;
        o[3] = graw[0];
        o[4] = graw[1];
        o[5] = gx;
        o[6] = gy;
        break;
    }
    case H2D_SC_CLIPPED_FRACTION:
        o[0] = clipped_fraction(x[0], x[1], x[2], x[3], x[4]);
        break;
    case H2D_SC_PLACE_INTERFACE:
        o[0] = place_interface(x[0], x[1], x[2], x[3], x[4], x[5], x[6]);
        break;
    case H2D_SC_YOUNGS_NORMAL: {  // youngs_normal (vof.cpp:10-22); k at [(di+1)*3 + (dj+1)]
        const double* k = x;
        auto col = [&](int di) { return k[(di + 1) * 3 + 0] + 2.0 * k[(di + 1) * 3 + 1] + k[(di + 1) * 3 + 2]; };
        auto row = [&](int dj) { return k[0 * 3 + dj + 1] + 2.0 * k[1 * 3 + dj + 1] + k[2 * 3 + dj + 1]; };
        const double gx = (col(1) - col(-1)) / (8.0 * x[9]);
        const double gy = (row(1) - row(-1)) / (8.0 * x[10]);
        const double g = sqrt(gx * gx + gy * gy);
        if (g < 1e-300) {
            bad = true;
            o[0] = o[1] = 0.0;
        } else {
            o[0] = gx / g;
            o[1] = gy / g;
        }
        break;
    }
    case H2D_SC_CELL_VOLUME:
        o[0] = cell_volume4(x, bad);
        break;
    case H2D_SC_CF_CORNER_FLUX: {  // cf_corner_flux (remap.cpp:16-25)
        const double dx = x[0] * x[2], dy = x[1] * x[2];
        const double dv = fabs(dx * dy);
        o[0] = dv == 0.0 ? 0.0 : dv;
        o[1] = dv == 0.0 ? 0.0 : (dx > 0.0 ? 1.0 : -1.0);
        o[2] = dv == 0.0 ? 0.0 : (dy > 0.0 ? 1.0 : -1.0);
        break;
    }
    case H2D_SC_CF_FACE_FLUX_X:
        cf_face_flux(x[0], x[1], x[2], x[3], x[4], x[5], o);
        break;
    case H2D_SC_CF_FACE_FLUX_Y:  // cf_face_flux_x with swapped components (remap.cpp:49-51)
        cf_face_flux(x[0], x[1], x[3], x[2], x[5], x[4], o);
        break;
    case H2D_SC_PSEUDO_VISCOSITY: {  // pseudo_viscosity (lagrange.cpp:7-12)
        const double rho = x[0], c = x[1], div = x[2], a1 = x[3], a2 = x[4], L = x[5];
        if (div >= 0.0) {
            o[0] = 0.0;
        } else {
            const double du = L * fabs(div);
            o[0] = rho * a1 * du * c + a2 * rho * du * du;
        }
        break;
    }
    case H2D_SC_DIV_U_CELL: {  // div_u_cell (lagrange.cpp:14-20); u00 u10 u01 u11 as (x, y)
        const double ux_l = 0.5 * (x[0] + x[4]);
        const double ux_r = 0.5 * (x[2] + x[6]);
        const double uy_b = 0.5 * (x[1] + x[3]);
        const double uy_t = 0.5 * (x[5] + x[7]);
        o[0] = (ux_r - ux_l) / x[8] + (uy_t - uy_b) / x[9];
        break;
    }
    case H2D_SC_GRAD_PQ_NODE: {  // grad_pq_node (lagrange.cpp:22-30); p, q at (i-1,j-1) (i,j-1) (i-1,j) (i,j)
        const double pa = x[0] + x[4], pb = x[1] + x[5], pc = x[2] + x[6], pe = x[3] + x[7];
        o[0] = (pb + pe - pa - pc) / (2.0 * x[8]);
        o[1] = (pc + pe - pa - pb) / (2.0 * x[9]);
        break;
    }
    case H2D_SC_AD_FACE_FLUX: {  // one face of ad_face_fluxes (remap.cpp:53-73)
        const double f = 0.5 * (x[0] + x[1]) * x[2] * x[3];
        o[0] = f;
        if (fabs(f) > kCflFrac * x[4]) bad = true;
        break;
    }
    default:
        bad = true;
    }
    if (flags) flags[r] = bad ? 1 : 0;
}

}  // namespace

void launch_scalar(int op, int n, const double* in, double* out, int* flags, cudaStream_t s) {
    if (n <= 0) return;
    k_scalar<<<(n + 127) / 128, 128, 0, s>>>(op, n, in, out, flags);
    add_launches(1);
}

}  // namespace h2d

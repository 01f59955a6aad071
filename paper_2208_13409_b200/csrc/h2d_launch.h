// h2d_launch.h — host-callable launch wrappers of h2d_kernels.cu.
#pragma once
#include <cuda_runtime.h>

#include "h2d_device.cuh"

namespace h2d {

struct FieldList {
    double* f[16];
    int n;
    int respect_halt;
};

// Work planes between the two passes of the AD split remap (remap.cpp:87-97):
// pass 0 writes them, pass 1 reads them.
struct AdWork {
    double *m[kMatSlots], *me[kMatSlots], *e[kMatSlots], *k[kMatSlots], *nrx, *nry, *mcell, *ux, *uy;
};

// Work inputs of one AD directional pass: pass 0 reads the State and the
// LagrangeResult (make_work, remap.cpp:116-140), pass 1 the AdWork of pass 0.
struct AdIO {
    const double *m[kMatSlots], *me[kMatSlots], *e[kMatSlots], *k[kMatSlots], *nrx, *nry, *mcell, *ux, *uy;
    int me_from_e;  // pass 0: w.me = m * e_lag (remap.cpp:128); mcell == nullptr: sum of m
    int pass;       // 0 / 1 (error phases PH_AD_* + 5 pass)
    int axis_x;     // 1: X pass, 0: Y pass
};

// the halo rectangles of one block, one segment per neighbour direction
struct HaloPlan {
    int n;
    Rng rc[8], rn[8];
    long long off[9];
};

long long launch_count();
int remap_uses_classes(int nmat);  // the remap tile launches dispatch on per-tile material classes
int remap_tile_w();  // remap-tile shape (cells): the tile-class grid
int remap_tile_h();
int tma_node_box_w();  // remap-tile TMA box sizes (doubles)
int tma_node_box_h();
int tma_cell_box_w();
int tma_cell_box_h();
void add_launches(long long n);  // kernels replayed by a CUDA graph launch
void launch_begin(Ctl* c, int mode, double dt, cudaStream_t s);
void launch_cfl(const Dev& d, int run_loop, cudaStream_t s);
void launch_ghost_cells(const Dev& d, const FieldList& fl, cudaStream_t s);
void launch_ghost_nodes(const Dev& d, const FieldList& fl, cudaStream_t s);
void launch_sync(const Dev& d, int next, int respect_halt, cudaStream_t s);
void launch_lagrange(const Dev& d, int write_vol_lag, cudaStream_t s);
// mode 0 = lagrange_step, 1 = predict only, 2 = correct from the u_half / p_half / q planes
void launch_lagrange_mode(const Dev& d, int write_vol_lag, int mode, cudaStream_t s);
// one AD directional pass as remap_single_axis (remap.cpp:1098-1104)
void launch_remap_single_axis(const Dev& d, const AdWork& W, int axis_x, int remap_velocity, cudaStream_t s);
// the reference's scalar kernels over n records (h2d.h H2D_SC_*)
void launch_scalar(int op, int n, const double* in, double* out, int* flags, cudaStream_t s);
void launch_lagrange_run(const Dev& d, cudaStream_t s);
void launch_remap(const Dev& d, cudaStream_t s);
void launch_remap_core(const Dev& d, cudaStream_t s);  // = tile + slivers + dual
void launch_lag_fused(const Dev& d, cudaStream_t s);
void launch_lag_ghosts(const Dev& d, cudaStream_t s);
void launch_post(const Dev& d, int run_loop, cudaStream_t s);
long long diag_partials(const Dev& d, int which);
void launch_tail(const Dev& d, int start_next, cudaStream_t s);  // run-loop epilogue
void launch_post_ghosts(const Dev& d, cudaStream_t s);
void launch_remap_tile(const Dev& d, cudaStream_t s);
void launch_remap_slivers(const Dev& d, cudaStream_t s);
void launch_remap_dual(const Dev& d, cudaStream_t s);
void post_and_ghosts(const Dev& d, int run_loop, cudaStream_t s);
void launch_step(const Dev& d, int fused_start, cudaStream_t s);  // one run-loop step
// AD split remap: both directional passes of remap_step(AD) (remap.cpp:1110-1115)
// leaving the next State's Work in `d`'s next-state planes, then the post
// kernels (run_loop: also the NaN scan and the next wave speed)
void launch_remap_ad(const Dev& d, const AdWork& W, int x_first, int remap_velocity, int run_loop, cudaStream_t s);
void launch_step_ad(const Dev& d, const AdWork& W, int x_first, int fused_start, cudaStream_t s);  // one AD run-loop step
void launch_cfl_next(const Dev& d, cudaStream_t s);
void launch_cls_flags(const Dev& d, cudaStream_t s);  // Dev::pcls of the current State (start of a run)
void launch_step_start(const Dev& d, cudaStream_t s);
void launch_commit_finish(const Dev& d, cudaStream_t s);               // wave speed of the current State
void launch_commit(Ctl* c, int advance, cudaStream_t s);
void launch_normals_api(const Dev& d, cudaStream_t s);
void launch_rollback(Ctl* c, cudaStream_t s);
// block-mode data plane (h2d_blocks_run)
void launch_step_block_head(const Dev& d, int part, cudaStream_t s);  // part 1: start + inner tiles, 2: edge tiles
void launch_step_block_rest(const Dev& d, cudaStream_t s);
void launch_step_block_ad_mid(const Dev& d, const AdWork& W, int x_first, cudaStream_t s);   // lag ghosts + AD pass 0
void launch_step_block_ad_rest(const Dev& d, const AdWork& W, int x_first, cudaStream_t s);  // AD pass 1 + post + tail
void launch_xhalf(const Dev& d, double* xh, double* yh, cudaStream_t s);  // HalfStepState::x_half
int lag_tile_w();  // the fused Lagrange kernel's node tile
int lag_tile_h();
void launch_red_pack(const Ctl* c, unsigned long long* red, cudaStream_t s);
void launch_red_apply(Ctl* c, const unsigned long long* red, cudaStream_t s);
void launch_red_local(unsigned long long* const* red, int n, cudaStream_t s);
void launch_halo_multi(const Dev& d, const FieldList& cells, const FieldList& nodes, const HaloPlan& plan,
                       double* buf, int to_buf, cudaStream_t s);
void launch_rect_xfer(const Dev& d, const FieldList& cells, const FieldList& nodes, Rng rc, Rng rn, double* buf,
                      int to_buf, cudaStream_t s);
void launch_global_xfer(const Dev& d, double* buf, Rng r, double* px, double* py, int vec, int to_block,
                        cudaStream_t s);
void launch_deinterleave(const double* src, double* x, double* y, int W, int H, int P, cudaStream_t s);
void launch_interleave(double* dst, const double* x, const double* y, int W, int H, int P, cudaStream_t s);

}  // namespace h2d

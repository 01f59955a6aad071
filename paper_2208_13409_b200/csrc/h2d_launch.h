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

long long launch_count();
void add_launches(long long n);  // kernels replayed by a CUDA graph launch
void launch_begin(Ctl* c, int mode, double dt, cudaStream_t s);
void launch_cfl(const Dev& d, int run_loop, cudaStream_t s);
void launch_ghost_cells(const Dev& d, const FieldList& fl, cudaStream_t s);
void launch_ghost_nodes(const Dev& d, const FieldList& fl, cudaStream_t s);
void launch_sync(const Dev& d, int next, int respect_halt, cudaStream_t s);
void launch_lagrange(const Dev& d, int write_vol_lag, cudaStream_t s);
void launch_lagrange_run(const Dev& d, cudaStream_t s);
void launch_remap(const Dev& d, cudaStream_t s);
void launch_remap_core(const Dev& d, cudaStream_t s);  // = tile + slivers + dual
void launch_lag_fused(const Dev& d, cudaStream_t s);
void launch_lag_ghosts(const Dev& d, cudaStream_t s);
void launch_post(const Dev& d, int run_loop, cudaStream_t s);
void launch_post_ghosts(const Dev& d, cudaStream_t s);
void launch_remap_tile(const Dev& d, cudaStream_t s);
void launch_remap_slivers(const Dev& d, cudaStream_t s);
void launch_remap_dual(const Dev& d, cudaStream_t s);
void post_and_ghosts(const Dev& d, int run_loop, cudaStream_t s);
void launch_step(const Dev& d, cudaStream_t s);  // one run-loop step
void launch_cfl_next(const Dev& d, cudaStream_t s);
void launch_step_start(const Dev& d, cudaStream_t s);
void launch_commit_finish(const Dev& d, cudaStream_t s);               // wave speed of the current State
void launch_commit(Ctl* c, int advance, cudaStream_t s);
void launch_nan_finish(const Dev& d, cudaStream_t s);
void launch_normals_api(const Dev& d, cudaStream_t s);
void launch_rollback(Ctl* c, cudaStream_t s);
void launch_rect_xfer(const Dev& d, const FieldList& cells, const FieldList& nodes, Rng rc, Rng rn, double* buf,
                      int to_buf, cudaStream_t s);
void launch_global_xfer(const Dev& d, double* buf, Rng r, double* px, double* py, int vec, int to_block,
                        cudaStream_t s);
void launch_deinterleave(const double* src, double* x, double* y, int W, int H, int P, cudaStream_t s);
void launch_interleave(double* dst, const double* x, const double* y, int W, int H, int P, cudaStream_t s);

}  // namespace h2d

// f64 instantiations of the pass launchers (kernels_launch.cuh).
#include "kernels_launch.cuh"

namespace dfftb {

cudaError_t launch_pass_f64(int n, const PassParams& p, bool adj, cudaStream_t s) {
  return launch_prec<double>(n, p, adj, s);
}
cudaError_t launch_pass_tma_f64(int n, const PassParams& p, bool adj, const TmaPlan& tp, int grid_limit,
                                 cudaStream_t s) {
  return launch_tma_prec<double>(n, p, adj, tp, grid_limit, s);
}
int tma_tile_w_f64(int n) { return tma_w_prec<double>(n); }
int tma_tile_w_halfreal_f64(int n) { return tma_w_halfreal_prec<double>(n); }

}  // namespace dfftb

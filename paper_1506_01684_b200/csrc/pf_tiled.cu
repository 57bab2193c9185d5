// pf_tiled.cu — tiled z-marching sweeps (placeholder: forwards to the naive
// kernels until the tiled implementation lands).
#include "pf_kernels.cuh"
namespace pf {
void launch_phi_tiled(cudaStream_t s, const KParams &kp, const BlockView &b) { launch_phi_naive(s, kp, b); }
void launch_mu_tiled(cudaStream_t s, const KParams &kp, const BlockView &b) { launch_mu_naive(s, kp, b); }
}  // namespace pf

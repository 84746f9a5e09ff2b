// Per-cell finalisation: partial marginals -> moments -> relax / lift tables.
//
// One CTA per x cell.  The marginal partials of all tiles are summed in a fixed
// tile order (the same order for every marginal index and its mirror), then
// the moments follow ref/moments.py:100-113 operation for operation:
//   rho   = (sum_j m_x[j]) * dvol                          (:101)
//   rho_u = (sum_{j<n/2} (m[j] - m[n-1-j]) c[j]) * dvol     (:80-88, :106-107)
//   theta = (sum_a sum_j (c_a[j]-u_a)^2 m_a[j]) * dvol / (3 rho)   (:108-112)
// and the table row follows ref/lifting.py:44-57 + ref/kinetic.py:130-134:
//   g_a[j] = exp(-(c_a[j]-u_a)^2 / (2 theta)),  amp = rho / (2 pi theta)^1.5,
//   mass   = amp * sum gx * sum gy * sum gz * dvol  (separable form of sum f),
//   lam    = dt*tau/eps,  r = 1/(1+lam),  ls = lam*rho/mass.
// All reductions are fixed warp trees (lane-strided sequential + xor butterfly).
#include <cuda_runtime.h>

#include "common.cuh"
#include "finalize_impl.cuh"
#include "ptx.cuh"

namespace pbgk {

#ifndef PBGK_FIN_THREADS
#define PBGK_FIN_THREADS 128
#endif
#ifndef PBGK_FIN_MINB
#define PBGK_FIN_MINB 16
#endif
constexpr int kFinThreads = PBGK_FIN_THREADS;

// MINB: resident CTAs per SM the register budget targets -- 16 (32 registers)
// when there are enough cells to fill the GPU, 4 (no spills) for few cells.
template <int MINB>
__global__ void __launch_bounds__(kFinThreads, MINB) finalize_kernel(const FinalArgs a) {
  pdl_wait();  // the partials / moments come from the preceding kernel
  pdl_trigger();
  extern __shared__ double sm[];
  __shared__ double sh[16];
  finalize_cell(a, blockIdx.x, sm, sh);
}

// the same per-cell work for window blockIdx.y of a batch
template <int MINB>
__global__ void __launch_bounds__(kFinThreads, MINB)
    finalize_batch_kernel(const FinalArgs a0, const FinalBatch b) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double sm[];
  __shared__ double sh[16];
  FinalArgs a = a0;
  const long long w = blockIdx.y;
  if (a.part != nullptr) a.part += w * b.part_ws;
  if (a.mom_in != nullptr) a.mom_in += w * b.mom_in_ws;
  if (a.mom_out != nullptr) a.mom_out += w * b.mom_out_ws;
  if (a.tab != nullptr) a.tab += w * b.tab_ws;
  if (a.relax_tab != nullptr) a.relax_tab += w * b.tab_ws;
  if (b.errw != nullptr) a.err = b.errw + w;
  finalize_cell(a, blockIdx.x, sm, sh);
}

__global__ void set_key_kernel(ErrKey* p, ErrKey v) { *p = v; }

cudaError_t launch_finalize(const FinalArgs& a, cudaStream_t st) {
  size_t smem = (size_t)2 * (a.nvx + a.nvy + a.nvz) * sizeof(double);
  if (a.mom_in == nullptr && a.mode != kFinIdentity)
    smem += (size_t)chunk_scratch(a.t, a.nvx, a.nvy, a.nvz) * sizeof(double);
  int nsm = 148;
  {
    static int cached = 0;
    if (!cached) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    }
    if (cached > 0) nsm = cached;
  }
  // one wave at 4 CTAs/SM: registers; otherwise occupancy
  auto k = (a.nx > nsm * 4) ? finalize_kernel<PBGK_FIN_MINB> : finalize_kernel<4>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  return launch_pdl(k, a.nx, kFinThreads, smem, st, a);
}

cudaError_t launch_finalize_batch(const FinalArgs& a, const FinalBatch& b, int nwin, cudaStream_t st) {
  size_t smem = (size_t)2 * (a.nvx + a.nvy + a.nvz) * sizeof(double);
  if (a.mom_in == nullptr && a.mode != kFinIdentity)
    smem += (size_t)chunk_scratch(a.t, a.nvx, a.nvy, a.nvz) * sizeof(double);
  auto k = finalize_batch_kernel<4>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  return launch_pdl_grid(k, dim3(a.nx, nwin), kFinThreads, smem, st, a, b);
}

cudaError_t launch_set_key(ErrKey* p, ErrKey v, cudaStream_t st) {
  set_key_kernel<<<1, 1, 0, st>>>(p, v);
  return cudaGetLastError();
}

}  // namespace pbgk

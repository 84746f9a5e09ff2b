// Shared-memory load cost microbenchmark (development tool): cycles per warp
// instruction for LDS.64 / LDS.128 under different address patterns, with 16
// warps per SM, to size the table-slice layout of the multi-step pass kernel.
#include <cstdio>
#include <cuda_runtime.h>

template <int PAT>
__device__ __forceinline__ int addr_of(int lane, int it) {
  // byte offset within a 4 KB window; (it & 7) * 4096 moves the window
  switch (PAT) {
    case 0: return 0;                                   // LDS.64 uniform
    case 1: return (lane >> 2) * 8;                     // LDS.64 8 distinct contiguous
    case 2: return lane * 8;                            // LDS.64 32 distinct contiguous
    case 3: return (lane >> 4) * 8;                     // LDS.64 2 distinct (half warps)
    case 4: return 0;                                   // LDS.128 uniform
    case 5: return ((lane & 3) * 2 + ((lane >> 2) & 1)) * 16;  // LDS.128 8 distinct per quarter (same in all quarters)
    case 6: return lane * 16;                           // LDS.128 32 distinct contiguous
    case 7: return (lane >> 3) * 16;                    // LDS.128 uniform per quarter, 4 distinct
    case 8: return (lane >> 4) * 16;                    // LDS.128 2 distinct (half warps)
    case 9: return (lane & 3) * 16;                     // LDS.128 4 distinct contiguous
    case 10: return lane * 128 + ((lane & 7) ^ 0) * 16; // LDS.128 stride 128 + swizzle: conflict-free
    case 11: return lane * 128;                         // LDS.128 stride 128: 8-way conflicts
  }
  return 0;
}

template <int PAT, bool WIDE, int NF>
__global__ void __launch_bounds__(512, 1) k(double* out, long long* cyc, int iters) {
  extern __shared__ __align__(128) unsigned char sm[];
  for (int i = threadIdx.x; i < 40960 / 8; i += blockDim.x) reinterpret_cast<double*>(sm)[i] = 1.0 + i * 1e-9;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int base = addr_of<PAT>(lane, 0);
  double acc0 = 0.0, acc1 = 0.0, f0 = 1.0, f1 = 1.0, f2 = 1.0, f3 = 1.0;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const unsigned char* p = sm + ((it & 7) << 12) + base;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (WIDE) {
        double2 v;
        asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p + u * 16 * (PAT == 10 || PAT == 11 ? 0 : 1))));
        acc0 += v.x;
        acc1 += v.y;
      } else {
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p + u * 8)));
        acc0 += v;
      }
#pragma unroll
      for (int q = 0; q < NF; ++q) {
        f0 = fma(f0, 1.0000001, 1e-9);
        f1 = fma(f1, 1.0000001, 1e-9);
        f2 = fma(f2, 1.0000001, 1e-9);
        f3 = fma(f3, 1.0000001, 1e-9);
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + f0 + f1 + f2 + f3;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int PAT, bool WIDE, int NF>
void run(const char* name, double* out, long long* cyc) {
  const int iters = 4096;
  auto fn = k<PAT, WIDE, NF>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 40960);
  fn<<<148, 512, 40960>>>(out, cyc, 64);
  cudaDeviceSynchronize();
  fn<<<148, 512, 40960>>>(out, cyc, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  // per SM: 16 warps x iters x 8 loads
  const double ninst = 16.0 * iters * 8;
  printf("%-52s NF=%d  %.2f cycles per warp-LDS (SM-wide), %.2f cycles per warp-DFMA  [%s]\n", name, NF, c / ninst,
         NF ? c / (ninst * 4 * NF) : 0.0, cudaGetErrorString(e));
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * 8);
  cudaMalloc(&cyc, 148 * 8);
  run<0, false, 0>("LDS.64 uniform", out, cyc);
  run<1, false, 0>("LDS.64 8 distinct (lane>>2)", out, cyc);
  run<2, false, 0>("LDS.64 32 distinct contiguous", out, cyc);
  run<3, false, 0>("LDS.64 2 distinct (half warps)", out, cyc);
  run<4, true, 0>("LDS.128 uniform", out, cyc);
  run<5, true, 0>("LDS.128 8 distinct per quarter (gz pattern)", out, cyc);
  run<6, true, 0>("LDS.128 32 distinct contiguous", out, cyc);
  run<7, true, 0>("LDS.128 uniform per quarter, 4 distinct", out, cyc);
  run<8, true, 0>("LDS.128 2 distinct (half warps)", out, cyc);
  run<9, true, 0>("LDS.128 4 distinct (lane&3)", out, cyc);
  run<10, true, 0>("LDS.128 stride 128 B, no swizzle, same addr x8", out, cyc);
  run<11, true, 0>("LDS.128 stride 128 B, 8-way conflict", out, cyc);
  run<0, false, 1>("LDS.64 uniform + 4 DFMA", out, cyc);
  run<0, false, 2>("LDS.64 uniform + 8 DFMA", out, cyc);
  run<4, true, 2>("LDS.128 uniform + 8 DFMA", out, cyc);
  run<6, true, 2>("LDS.128 32 distinct + 8 DFMA", out, cyc);
  run<6, true, 4>("LDS.128 32 distinct + 16 DFMA", out, cyc);
  run<2, false, 4>("LDS.64 32 distinct + 16 DFMA", out, cyc);
  return 0;
}

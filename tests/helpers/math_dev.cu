// Device build of the product's lean FP64 math (paper_2402_06491_b200/csrc/
// rt_math.cuh) for tests/test_gpu_math.py: the same routines the tree walk
// inlines, evaluated on the GPU (MUFU seeds, FMA contraction as compiled).
#include <cstdint>

#include "rt_math.cuh"

using namespace rtk;

__global__ void math_kernel(int which, const double* x, long n, double* y, double* z) {
  long q = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (q >= n) return;
  switch (which) {
    case 0: y[q] = log_tab(x[q], kLogTable); break;
    case 1: sincospi2(x[q], y[q], z[q]); break;
    case 2: y[q] = cospi2(x[q]); break;
    case 3: y[q] = sqrt_nr(x[q]); break;
    case 4: y[q] = rcp_nr(x[q]); break;
    case 6: sincos2pi_u32(static_cast<uint32_t>(x[q]), y[q], z[q]); break;
    case 7: y[q] = cos2pi_u32(static_cast<uint32_t>(x[q])); break;
    case 8: y[q] = exp_neg_tab(x[q], kExpT32); break;
    case 9: y[q] = mul_exp_tab(z[q], x[q], kExpT32); break;   // z: the factor a
    default: y[q] = exp_neg(x[q]); break;
  }
}

extern "C" int math_dev(int which, const double* hx, long n, double* hy, double* hz) {
  double *x, *y, *z;
  if (cudaMalloc(&x, n * 8) || cudaMalloc(&y, n * 8) || cudaMalloc(&z, n * 8)) return 1;
  cudaMemcpy(x, hx, n * 8, cudaMemcpyHostToDevice);
  if (hz) cudaMemcpy(z, hz, n * 8, cudaMemcpyHostToDevice);   // (case 9: the factor a)
  math_kernel<<<(n + 255) / 256, 256>>>(which, x, n, y, z);
  cudaError_t e = cudaMemcpy(hy, y, n * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && hz) e = cudaMemcpy(hz, z, n * 8, cudaMemcpyDeviceToHost);
  cudaFree(x); cudaFree(y); cudaFree(z);
  return e == cudaSuccess ? 0 : 2;
}

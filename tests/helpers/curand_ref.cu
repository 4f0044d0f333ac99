// Library pin for Philox4x32-10 on the GPU: cuRAND's device API.
// curand_init(seed, subsequence = (c3 << 32) | c2, offset = 4 * ((c1 << 32) | c0))
// positions the generator at counter (c0, c1, c2, c3) with key = seed
// (curand_kernel.h: skipahead_sequence adds to ctr.z/w, skipahead adds n/4
// to ctr.x/y); curand4 then returns philox(key, ctr).  Valid for c1 < 2^30.
#include <cstdint>
#include <curand_kernel.h>

__global__ void ref_kernel(unsigned long long seed, const uint32_t* ctr, int n, uint32_t* out) {
  int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const uint32_t* c = ctr + 4 * q;
  curandStatePhilox4_32_10_t s;
  unsigned long long sub = (static_cast<unsigned long long>(c[3]) << 32) | c[2];
  unsigned long long off = 4ull * ((static_cast<unsigned long long>(c[1]) << 32) | c[0]);
  curand_init(seed, sub, off, &s);
  uint4 r = curand4(&s);
  out[4 * q] = r.x; out[4 * q + 1] = r.y; out[4 * q + 2] = r.z; out[4 * q + 3] = r.w;
}

extern "C" int curand_philox_ref(unsigned long long seed, const uint32_t* h_ctr, int n,
                                 uint32_t* h_out) {
  uint32_t *dc = nullptr, *dout = nullptr;
  if (cudaMalloc(&dc, 16ull * n) != cudaSuccess) return 1;
  if (cudaMalloc(&dout, 16ull * n) != cudaSuccess) return 1;
  cudaMemcpy(dc, h_ctr, 16ull * n, cudaMemcpyHostToDevice);
  ref_kernel<<<(n + 127) / 128, 128>>>(seed, dc, n, dout);
  cudaError_t e = cudaMemcpy(h_out, dout, 16ull * n, cudaMemcpyDeviceToHost);
  cudaFree(dc);
  cudaFree(dout);
  return e == cudaSuccess ? 0 : 2;
}

// derive_bench.cu -- device-side cost of derive_core (one thread), in cycles.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2604_25306_b200/csrc/qflash_params.cuh"

__global__ void k(float sq, float sk, int d, qf::IntParams* o, long long* cyc) {
  long long t0 = clock64();
  qf::IntParams p;
  int st = qf::derive_core(sq, sk, d, &p, nullptr);
  p.status = st;
  *o = p;
  long long t1 = clock64();
  *cyc = t1 - t0;
}
int main() {
  qf::IntParams* o; long long* c; cudaMalloc(&o, sizeof(qf::IntParams)); cudaMalloc(&c, 8);
  for (int rep = 0; rep < 3; ++rep) {
    k<<<1, 1>>>(0.055f + rep * 0.001f, 0.052f, 64, o, c);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("derive_core: %lld cycles (%s)\n", h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

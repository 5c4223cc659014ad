// udiv_check.cu -- exhaustive check of qf::udiv_small (qflash_params.cuh) against
// the plain 64-bit '/' and '%' over every divisor D in [1, 2^25] (s_inv <= 2^24 + 1),
// for the numerators derive_core divides: 2^32, 2^(32 + sh) for both shift rules, and
// r1 * 2^32 for r1 in {0, 1, D/3, D/2, D - 1, a hashed value < D}.  Runs the host
// build of the helper and the device build (fp64 RZ product of RN reciprocal).
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/udiv_check.cu -o tools/udiv_check
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2604_25306_b200/csrc/qflash_params.cuh"

__host__ __device__ inline int nums(uint64_t D, uint64_t* out) {
  const int L = qf::ceil_log2(D);
  int k = 0;
  out[k++] = uint64_t(1) << 32;
  out[k++] = uint64_t(1) << (32 + (L > 7 ? L - 7 : 0));
  out[k++] = uint64_t(1) << (32 + (L > 8 ? L - 8 : 0));
  const uint64_t h = (D * 0x9E3779B97F4A7C15ull) >> 40;
  const uint64_t r1s[6] = {0, 1 % D, D / 3, D / 2, D - 1, h % D};
  for (int i = 0; i < 6; ++i) out[k++] = r1s[i] << 32;
  return k;
}

__host__ __device__ inline unsigned long long check_one(uint64_t D) {
  uint64_t n[9];
  const int k = nums(D, n);
  unsigned long long bad = 0;
  for (int i = 0; i < k; ++i) {
    uint64_t r;
    const uint64_t q = qf::udiv_small(n[i], D, &r);
    if (q != n[i] / D || r != n[i] % D) ++bad;
  }
  return bad;
}

__global__ void kcheck(uint64_t lo, uint64_t hi, unsigned long long* bad) {
  unsigned long long b = 0;
  for (uint64_t D = lo + blockIdx.x * blockDim.x + threadIdx.x; D <= hi; D += gridDim.x * blockDim.x)
    b += check_one(D);
  if (b) atomicAdd(bad, b);
}

int main() {
  const uint64_t lo = 1, hi = uint64_t(1) << 25;
  unsigned long long hbad = 0;
  for (uint64_t D = lo; D <= hi; ++D) hbad += check_one(D);
  printf("host:   D in [1, 2^25], 9 numerators each: %llu mismatches\n", hbad);
  unsigned long long* dbad;
  if (cudaMalloc(&dbad, 8) != cudaSuccess) {
    printf("device: no GPU\n");
    return hbad != 0;
  }
  cudaMemset(dbad, 0, 8);
  kcheck<<<148 * 8, 256>>>(lo, hi, dbad);
  unsigned long long db = ~0ull;
  cudaMemcpy(&db, dbad, 8, cudaMemcpyDeviceToHost);
  printf("device: D in [1, 2^25], 9 numerators each: %llu mismatches (%s)\n", db,
         cudaGetErrorString(cudaGetLastError()));
  return (hbad != 0 || db != 0);
}

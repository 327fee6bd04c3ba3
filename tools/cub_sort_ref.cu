// Reference timing only (not part of the product): CUB's device radix sort
// of N u64 keys over the low `bits` bits, to calibrate what a library sort
// costs at the step path's sizes on this GPU.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cub_ref tools/cub_sort_ref.cu && /tmp/cub_ref
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>
#include <random>

int main() {
  for (size_t N : {65536ul, 1000000ul, 4194304ul, 16777216ul}) {
    std::vector<unsigned long long> h(N);
    std::mt19937_64 rng(1);
    for (auto& x : h) x = (rng() & ((1ull << 34) - 1)) << 30 | (rng() & ((1ull << 30) - 1));
    unsigned long long *a, *b;
    cudaMalloc(&a, N * 8); cudaMalloc(&b, N * 8);
    cudaMemcpy(a, h.data(), N * 8, cudaMemcpyHostToDevice);
    size_t tmp = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp, a, b, (int)N, 30, 64);
    void* t; cudaMalloc(&t, tmp);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) cub::DeviceRadixSort::SortKeys(t, tmp, a, b, (int)N, 30, 64);
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0);
      cub::DeviceRadixSort::SortKeys(t, tmp, a, b, (int)N, 30, 64);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    printf("cub SortKeys u64 bits[30,64) N=%zu : %.1f us\n", N, best * 1e3);
    cudaFree(a); cudaFree(b); cudaFree(t);
  }
  return 0;
}

// Microbenchmark: random-gather cost on B200 for the table-probe access
// pattern (one random aligned chunk per thread), by chunk size and load
// flavour.  Not part of the product; informs the bucket layout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o randread tools/randread.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t h) {
  h ^= h >> 16; h *= 0x85ebca6bu; h ^= h >> 13; h *= 0xc2b2ae35u; h ^= h >> 16; return h;
}

template <int BYTES>
__global__ void k_gather(const uint4* __restrict__ tab, uint64_t n_chunks, int64_t n, uint32_t seed,
                         uint32_t* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t c = mix((uint32_t)i * 2654435761u + seed) & (n_chunks - 1);
  const uint4* p = tab + c * (BYTES / 16);
  uint32_t acc = 0;
  if (BYTES == 16) {
    uint4 v = __ldg(p); acc = v.x ^ v.w;
  } else {
#pragma unroll
    for (int k = 0; k < BYTES / 32; ++k) {
      uint32_t r[8];
      asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "l"(p + 2 * k));
      acc ^= r[0] ^ r[7];
    }
  }
  out[i] = acc;
}

// 8 lanes cooperatively read one 128-byte line (16 B each)
__global__ void k_gather_coop128(const uint4* __restrict__ tab, uint64_t n_lines, int64_t n, uint32_t seed,
                                 uint32_t* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t i = t >> 3;
  int sub = t & 7;
  if (i >= n) return;
  uint64_t c = mix((uint32_t)i * 2654435761u + seed) & (n_lines - 1);
  uint4 v = __ldg(tab + c * 8 + sub);
  uint32_t acc = v.x ^ v.w;
  acc ^= __shfl_xor_sync(0xffffffff, acc, 1);
  acc ^= __shfl_xor_sync(0xffffffff, acc, 2);
  acc ^= __shfl_xor_sync(0xffffffff, acc, 4);
  if (sub == 0) out[i] = acc;
}

int main() {
  const size_t table_bytes = size_t(512) << 20;
  const int64_t n = 10000000;
  uint4* tab; uint32_t* out;
  cudaMalloc(&tab, table_bytes);
  cudaMalloc(&out, n * 4);
  cudaMemset(tab, 1, table_bytes);
  void* flush; size_t fb = size_t(256) << 20; cudaMalloc(&flush, fb);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  size_t lim = 0;
  cudaDeviceGetLimit(&lim, cudaLimitMaxL2FetchGranularity);
  printf("default MaxL2FetchGranularity = %zu\n", lim);
  for (int g : {0, 32, 64, 128}) {
    if (g) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
    cudaDeviceGetLimit(&lim, cudaLimitMaxL2FetchGranularity);
    for (int mode = 0; mode < 5; ++mode) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemsetAsync(flush, rep, fb);
        cudaEventRecord(a);
        uint32_t seed = 77 + rep;
        switch (mode) {
          case 0: k_gather<16><<<(n + 255) / 256, 256>>>(tab, table_bytes / 16, n, seed, out); break;
          case 1: k_gather<32><<<(n + 255) / 256, 256>>>(tab, table_bytes / 32, n, seed, out); break;
          case 2: k_gather<64><<<(n + 255) / 256, 256>>>(tab, table_bytes / 64, n, seed, out); break;
          case 3: k_gather<128><<<(n + 255) / 256, 256>>>(tab, table_bytes / 128, n, seed, out); break;
          case 4: k_gather_coop128<<<(n * 8 + 255) / 256, 256>>>(tab, table_bytes / 128, n, seed, out); break;
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      const int bytes[] = {16, 32, 64, 128, 128};
      printf("limit=%3zu chunk=%3dB%s  %.4f ms  %.1f Greads/s  useful %.0f GB/s\n", lim, bytes[mode],
             mode == 4 ? "(coop8)" : "       ", best, n / best / 1e6, n * (double)bytes[mode] / best / 1e6);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

// Microbenchmark: 10M random 32-byte bucket probes on a 240 MB table, by
// load flavour (L1 path / cache operator / width).  Run under ncu with
// lts__t_sectors_srcunit_tex_op_read.sum,dram__sectors_read.sum to see how
// many sectors each flavour pulls per probe.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probeload tools/probeload.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t h) {
  h ^= h >> 16; h *= 0x85ebca6bu; h ^= h >> 13; h *= 0xc2b2ae35u; h ^= h >> 16; return h;
}

#define LD8(OP)                                                                                          \
  asm volatile(OP " {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                                                  \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) \
               : "l"(p))
#define LD4(OP, Q, O)                                                                                    \
  asm volatile(OP " {%0,%1,%2,%3}, [%4];" : "=r"(r[O]), "=r"(r[O + 1]), "=r"(r[O + 2]), "=r"(r[O + 3]) : "l"(Q))

template <int MODE>
__global__ void k_probe(const uint4* __restrict__ tab, uint32_t n_buckets, int64_t n, uint32_t seed,
                        uint32_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t b = __umulhi(mix((uint32_t)i * 2654435761u + seed), n_buckets);
  const uint4* p = tab + 2 * (size_t)b;
  uint32_t r[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (MODE == 0) LD8("ld.global.nc.L1::no_allocate.v8.u32");
  if (MODE == 1) LD8("ld.global.cg.v8.u32");
  if (MODE == 2) LD8("ld.global.v8.u32");
  if (MODE == 3) LD8("ld.relaxed.gpu.global.v8.u32");
  if (MODE == 4) { LD4("ld.global.nc.L1::no_allocate.v4.u32", p, 0); LD4("ld.global.nc.L1::no_allocate.v4.u32", p + 1, 4); }
  if (MODE == 5) { LD4("ld.global.cg.v4.u32", p, 0); LD4("ld.global.cg.v4.u32", p + 1, 4); }
  if (MODE == 6) LD4("ld.global.cg.v4.u32", p, 0);
  if (MODE == 7) LD8("ld.global.cv.v8.u32");
  if (MODE == 8) LD8("ld.global.nc.L1::no_allocate.L2::64B.v8.u32");
  out[i] = r[0] ^ r[3] ^ r[4] ^ r[7];
}

// U independent probes per thread (memory-level parallelism per thread)
template <int U>
__global__ void k_probe_multi(const uint4* __restrict__ tab, uint32_t n_buckets, int64_t n, uint32_t seed,
                              uint32_t* __restrict__ out) {
  const int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * U;
  uint32_t r[U][8];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t i = i0 + u;
    const uint32_t b = __umulhi(mix((uint32_t)(i < n ? i : 0) * 2654435761u + seed), n_buckets);
    const uint4* p = tab + 2 * (size_t)b;
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[u][0]), "=r"(r[u][1]), "=r"(r[u][2]), "=r"(r[u][3]), "=r"(r[u][4]), "=r"(r[u][5]),
                   "=r"(r[u][6]), "=r"(r[u][7])
                 : "l"(p));
  }
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (i0 + u < n) out[i0 + u] = r[u][0] ^ r[u][3] ^ r[u][4] ^ r[u][7];
}

int main(int argc, char** argv) {
  // table size in MB (default 240; e.g. 9600 for the configs[4] table)
  const uint32_t n_buckets = (argc > 1 ? (uint32_t)(atof(argv[1]) * 1e6 / 32) : 7500000u);
  printf("table %.0f MB\n", n_buckets * 32.0 / 1e6);
  // optional second argument: cudaLimitMaxL2FetchGranularity in bytes
  if (argc > 2) {
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[2]));
    size_t v = 0;
    cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("L2 fetch granularity limit %zu\n", v);
  }
  const int64_t n = 10000000;
  uint4* tab; uint32_t* out;
  cudaMalloc(&tab, (size_t)n_buckets * 32);
  cudaMalloc(&out, n * 4);
  cudaMemset(tab, 1, (size_t)n_buckets * 32);
  void* flush; size_t fb = size_t(256) << 20; cudaMalloc(&flush, fb);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"nc.L1::no_allocate.v8", "cg.v8", "v8 (ca)", "relaxed.gpu.v8", "nc.v4 x2", "cg.v4 x2",
                         "cg.v4 (16B only)", "cv.v8", "nc.L2::64B.v8"};
  for (int mode = 0; mode < 9; ++mode) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemsetAsync(flush, rep, fb);
      cudaEventRecord(a);
      const unsigned g = (unsigned)((n + 255) / 256);
      switch (mode) {
        case 0: k_probe<0><<<g, 256>>>(tab, n_buckets, n, 77 + rep, out); break;
        case 1: k_probe<1><<<g, 256>>>(tab, n_buckets, n, 77 + rep, out); break;
        case 2: k_probe<2><<<g, 256>>>(tab, n_buckets, n, 77 + rep, out); break;
        case 3: k_probe<3><<<g, 256>>>(tab, n_buckets, n, 77 + rep, out); break;
        case 4: k_probe<4><<<g, 256>>>(tab, n_buckets, n, 77 + rep, out); break;
        case 5: k_probe<5><<<g, 256>>>(tab, n_buckets, n, 77 + rep, out); break;
        case 6: k_probe<6><<<g, 256>>>(tab, n_buckets, n, 77 + rep, out); break;
        case 7: k_probe<7><<<g, 256>>>(tab, n_buckets, n, 77 + rep, out); break;
        case 8: k_probe<8><<<g, 256>>>(tab, n_buckets, n, 77 + rep, out); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-22s %.4f ms  %.1f Gprobes/s\n", names[mode], best, n / best / 1e6);
  }
  for (int u : {1, 2, 4}) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemsetAsync(flush, rep, fb);
      cudaEventRecord(a);
      const unsigned g = (unsigned)((n / u + 255) / 256);
      if (u == 1) k_probe_multi<1><<<g, 256>>>(tab, n_buckets, n, 77 + rep, out);
      if (u == 2) k_probe_multi<2><<<g, 256>>>(tab, n_buckets, n, 77 + rep, out);
      if (u == 4) k_probe_multi<4><<<g, 256>>>(tab, n_buckets, n, 77 + rep, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%d probes/thread        %.4f ms  %.1f Gprobes/s\n", u, best, n / best / 1e6);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// Microbenchmark: cost of the claim pattern's memory ops on random 16-byte
// slots of a 240 MB table (10M ops): load only, load+CAS128, CAS128 only,
// load+CAS64, load+atomicCAS32, load+store.  Informs the claim design.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t mix(uint32_t h) { h ^= h >> 16; h *= 0x85ebca6bu; h ^= h >> 13; h *= 0xc2b2ae35u; h ^= h >> 16; return h; }
__device__ __forceinline__ bool cas128(uint4* addr, uint4 cmp, uint4 val) {
  unsigned long long clo = ((unsigned long long)cmp.y << 32) | cmp.x, chi = ((unsigned long long)cmp.w << 32) | cmp.z;
  unsigned long long vlo = ((unsigned long long)val.y << 32) | val.x, vhi = ((unsigned long long)val.w << 32) | val.z;
  unsigned long long olo, ohi;
  asm volatile("{\n\t.reg .b128 c, v, o;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 v, {%4, %5};\n\tatom.global.cas.b128 o, [%6], c, v;\n\tmov.b128 {%0, %1}, o;\n\t}"
               : "=l"(olo), "=l"(ohi) : "l"(clo), "l"(chi), "l"(vlo), "l"(vhi), "l"(addr) : "memory");
  return olo == clo && ohi == chi;
}
__device__ __forceinline__ uint4 ld128r(const uint4* p) { uint4 r; asm volatile("ld.relaxed.gpu.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory"); return r; }
template <int MODE>
__global__ void k(uint4* tab, uint32_t nslots, int64_t n, uint32_t seed, uint32_t* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t s = (uint32_t)(((uint64_t)mix((uint32_t)i * 2654435761u + seed) * nslots) >> 32);
  uint4* p = tab + s;
  uint32_t r = 0;
  if (MODE == 0) { uint4 v = ld128r(p); r = v.w; }
  if (MODE == 1) { uint4 v = ld128r(p); r = cas128(p, v, make_uint4(1, 2, 3, (uint32_t)i)); }
  if (MODE == 2) { r = cas128(p, make_uint4(~0u, ~0u, ~0u, ~0u), make_uint4(1, 2, 3, (uint32_t)i)); }
  if (MODE == 3) { uint4 v = ld128r(p); unsigned long long o = atomicCAS((unsigned long long*)p, ((unsigned long long)v.y << 32) | v.x, 5ull); r = (uint32_t)o; }
  if (MODE == 4) { uint4 v = ld128r(p); r = atomicCAS(&p->w, v.w, (uint32_t)i); }
  if (MODE == 5) { uint4 v = ld128r(p); p->w = v.w + 1; r = 1; }
  if (MODE == 6) { r = atomicMin(&p->w, (uint32_t)i); }
  out[i] = r;
}
int main() {
  const uint32_t nslots = 15000000; const int64_t n = 5000000;
  uint4* tab; uint32_t* out; cudaMalloc(&tab, (size_t)nslots * 16); cudaMalloc(&out, n * 4);
  void* flush; size_t fb = size_t(256) << 20; cudaMalloc(&flush, fb);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"ld128 only", "ld128+CAS128", "CAS128 only", "ld128+CAS64", "ld128+CAS32", "ld128+st32", "atomicMin32"};
  for (int mode = 0; mode < 7; ++mode) {
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(tab, 0xFF, (size_t)nslots * 16);
      cudaMemsetAsync(flush, rep, fb);
      cudaEventRecord(a);
      switch (mode) {
        case 0: k<0><<<(n + 255) / 256, 256>>>(tab, nslots, n, rep, out); break;
        case 1: k<1><<<(n + 255) / 256, 256>>>(tab, nslots, n, rep, out); break;
        case 2: k<2><<<(n + 255) / 256, 256>>>(tab, nslots, n, rep, out); break;
        case 3: k<3><<<(n + 255) / 256, 256>>>(tab, nslots, n, rep, out); break;
        case 4: k<4><<<(n + 255) / 256, 256>>>(tab, nslots, n, rep, out); break;
        case 5: k<5><<<(n + 255) / 256, 256>>>(tab, nslots, n, rep, out); break;
        case 6: k<6><<<(n + 255) / 256, 256>>>(tab, nslots, n, rep, out); break;
      }
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("%-14s %.4f ms  %.1f Gops/s\n", names[mode], best, n / best / 1e6);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

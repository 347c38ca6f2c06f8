// ash_route.cu — multi-GPU routing kernels for the hash-partitioned map.
//
// No reference counterpart (the reference has no distributed mode; SURVEY
// §8(e)).  owner(key) = mix64(key) mapped to [0, world) by multiply-shift;
// the mix is independent of the in-table bucket hash (ash_map.cu) so shards
// stay uniformly loaded.  The partition is STABLE: a rank's keys for one
// owner keep batch order, and NCCL all-to-all concatenates by source rank,
// so every owner sees its keys in global batch order and first-occurrence
// winners stay bit-exact (verified on the oracle in SURVEY §8(e)).
//
// One partition = three launches: count (owner per key -> uint8 + per-tile
// per-owner counts), a one-block scan, and a scatter that writes the send
// buffers directly (key rows + one payload row per key + the permutation),
// so no separate gather pass touches the batch again.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/ash.h"
#include "launch_count.h"

namespace {

constexpr int kBlock = 256;
constexpr int kItems = 8;
constexpr int kTile = kBlock * kItems;
constexpr int kMaxWorld = 64;

thread_local char g_route_err[256] = "";

// ASH_PUT_STAGED=0: the put stores each row straight to its owner instead of
// staging the tile's rows per owner (A/B runs); read at load time
int g_put_staged = [] {
  const char* e = getenv("ASH_PUT_STAGED");
  return e ? (e[0] != '0' ? 1 : 0) : 1;
}();

int rfail(const char* msg) {
  snprintf(g_route_err, sizeof(g_route_err), "%s", msg);
  return ASH_ERR_INVALID;
}

int rcheck(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_route_err, sizeof(g_route_err), "%s: %s", what, cudaGetErrorString(e));
    return ASH_ERR_CUDA;
  }
  return ASH_OK;
}

__device__ __forceinline__ uint64_t fmix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

// row: global key row (read-only path) or registers
template <typename Row>
__device__ __forceinline__ uint32_t owner_of(const Row& row, int arity, uint32_t world) {
  uint64_t x = 0x243F6A8885A308D3ull ^ static_cast<uint64_t>(arity);
  for (int d = 0; d < arity; ++d)
    x = fmix64(x ^ (static_cast<uint64_t>(static_cast<uint32_t>(row[d])) + 0x9E3779B97F4A7C15ull * (d + 1)));
  return static_cast<uint32_t>((static_cast<uint64_t>(static_cast<uint32_t>(x >> 32)) * world) >> 32);
}

// a key row in global memory (read-only path)
__device__ __forceinline__ uint32_t owner_of_global(const int32_t* row, int arity, uint32_t world) {
  struct Ldg {
    const int32_t* r;
    __device__ int32_t operator[](int d) const { return __ldg(r + d); }
  };
  return owner_of(Ldg{row}, arity, world);
}

// pass 1: owner of every key (uint8) and per-tile, per-owner counts ->
// cnt[owner * n_tiles + tile]
__global__ void __launch_bounds__(kBlock) k_route_count(const int32_t* __restrict__ keys, int64_t n, int arity,
                                                        uint32_t world, uint8_t* __restrict__ owners,
                                                        int32_t* __restrict__ cnt, int64_t n_tiles) {
  __shared__ int32_t s_cnt[kMaxWorld];
  for (int o = threadIdx.x; o < kMaxWorld; o += kBlock) s_cnt[o] = 0;
  __syncthreads();
  const int64_t base = blockIdx.x * static_cast<int64_t>(kTile);
  // every item's owner first (all key loads of the tile in flight), then the
  // warp-aggregated shared-memory counts
  uint32_t own[kItems];
  const int64_t p8 = base + threadIdx.x * kItems;  // 8 consecutive positions
  if (arity == 3 && base + kTile <= n && (reinterpret_cast<uintptr_t>(keys) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(owners) & 7) == 0) {  // block-uniform: full tile
    // int3 keys, full octet: the thread's 8 rows (96 bytes) as six 16-byte
    // loads, the 8 owner bytes as one 8-byte store; counts do not depend on
    // the item layout (the scatter recomputes its ranks from `owners`)
    int32_t kw[kItems * 3];
    const int4* src = reinterpret_cast<const int4*>(keys + p8 * 3);
#pragma unroll
    for (int v = 0; v < kItems * 3 / 4; ++v) {
      const int4 q = __ldg(src + v);
      kw[4 * v] = q.x, kw[4 * v + 1] = q.y, kw[4 * v + 2] = q.z, kw[4 * v + 3] = q.w;
    }
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int32_t row[3] = {kw[3 * it], kw[3 * it + 1], kw[3 * it + 2]};
      own[it] = owner_of(row, 3, world);
      if (it < 4) lo |= own[it] << (8 * it);
      else hi |= own[it] << (8 * (it - 4));
    }
    *reinterpret_cast<uint2*>(owners + p8) = make_uint2(lo, hi);
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const unsigned same = __match_any_sync(0xFFFFFFFFu, own[it]);
      if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&s_cnt[own[it]], __popc(same));
    }
    __syncthreads();
    for (int o = threadIdx.x; o < static_cast<int>(world); o += kBlock) cnt[o * n_tiles + blockIdx.x] = s_cnt[o];
    return;
  }
  if (arity == 3) {  // int3 keys: all 24 key words of the thread in flight first
    int32_t kw[kItems][3];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t p = base + it * kBlock + threadIdx.x;
#pragma unroll
      for (int d = 0; d < 3; ++d) kw[it][d] = p < n ? __ldg(keys + p * 3 + d) : 0;
    }
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t p = base + it * kBlock + threadIdx.x;
      own[it] = p < n ? owner_of(kw[it], 3, world) : 0xFFFFFFFFu;
    }
  } else {
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t p = base + it * kBlock + threadIdx.x;
      own[it] = p < n ? owner_of_global(keys + p * arity, arity, world) : 0xFFFFFFFFu;
    }
  }
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int64_t p = base + it * kBlock + threadIdx.x;
    if (p < n) owners[p] = static_cast<uint8_t>(own[it]);
    const unsigned same = __match_any_sync(0xFFFFFFFFu, own[it]);
    if (own[it] != 0xFFFFFFFFu && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&s_cnt[own[it]], __popc(same));
  }
  __syncthreads();
  for (int o = threadIdx.x; o < static_cast<int>(world); o += kBlock) cnt[o * n_tiles + blockIdx.x] = s_cnt[o];
}

// pass 2 (one block): exclusive scan over the owner-major count matrix;
// per-owner totals to counts[]
__global__ void __launch_bounds__(1024) k_route_scan(int32_t* cnt, int64_t len, int64_t n_tiles, uint32_t world,
                                                     int64_t* counts) {
  // 32 warps, each a contiguous segment of whole 32-entry chunks read
  // coalesced and 8 chunks in flight: segment sums, a scan of the 32 sums,
  // then each warp rescans its segment from its offset.  (A 1024-wide loop
  // with block barriers per chunk cost ~25 us at 8 owners x 4.9K tiles.)
  constexpr int kU = 8;
  __shared__ int32_t warp_off[32];
  __shared__ int32_t s_total;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t chunks = (len + 31) / 32;
  const int64_t per = (chunks + 31) / 32;  // chunks per warp
  const int64_t c0 = warp * per, c1 = c0 + per < chunks ? c0 + per : chunks;
  int32_t sum = 0;
  for (int64_t c = c0; c < c1; c += kU) {
    int32_t x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = (c + u) * 32 + lane;
      x[u] = (c + u < c1 && i < len) ? cnt[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) sum += x[u];
  }
  sum = __reduce_add_sync(0xFFFFFFFFu, sum);
  if (lane == 0) warp_off[warp] = sum;
  __syncthreads();
  if (warp == 0) {
    const int32_t w = warp_off[lane];
    int32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += y;
    }
    warp_off[lane] = wi - w;
    if (lane == 31) s_total = wi;
  }
  __syncthreads();
  int32_t carry = warp_off[warp];
  for (int64_t c = c0; c < c1; c += kU) {
    int32_t x[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = (c + u) * 32 + lane;
      x[u] = (c + u < c1 && i < len) ? cnt[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      int32_t incl = x[u];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
      }
      const int64_t i = (c + u) * 32 + lane;
      if (c + u < c1 && i < len) cnt[i] = carry + incl - x[u];
      carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
  }
  __syncthreads();
  for (uint32_t o = threadIdx.x; o < world; o += 1024) {
    const int64_t start = cnt[o * n_tiles];
    const int64_t end = (o + 1 < world) ? cnt[(o + 1) * n_tiles] : s_total;
    counts[o] = end - start;
  }
}

__device__ __forceinline__ void copy_row_words(uint8_t* dst, const uint8_t* src, int64_t rb) {
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | rb) & 3) == 0) {
    for (int64_t i = 0; i < rb; i += 4)
      *reinterpret_cast<uint32_t*>(dst + i) = __ldg(reinterpret_cast<const uint32_t*>(src + i));
  } else {
    for (int64_t i = 0; i < rb; ++i) dst[i] = src[i];
  }
}

// pass 3: stable scatter.  Destination of position p = offset(owner, tile) +
// rank of p among the tile's positions with that owner, in (item, warp,
// lane) = position order.  Writes perm[dst] = p, the key row and one payload
// row at dst.
__global__ void __launch_bounds__(kBlock) k_route_scatter(const int32_t* __restrict__ keys, int64_t n, int arity,
                                                          uint32_t world, const uint8_t* __restrict__ owners,
                                                          const int32_t* __restrict__ off, int64_t n_tiles,
                                                          int32_t* __restrict__ perm, int32_t* __restrict__ keys_out,
                                                          const uint8_t* __restrict__ pay, int64_t pay_rb,
                                                          uint8_t* __restrict__ pay_out) {
  constexpr int kW = kBlock / 32;
  __shared__ int32_t s_pre[kItems][kW][kMaxWorld];
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < kItems * kW * kMaxWorld; e += kBlock) (&s_pre[0][0][0])[e] = 0;
  __syncthreads();
  const int64_t base = blockIdx.x * static_cast<int64_t>(kTile);
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  uint32_t own[kItems], rank_in_warp[kItems];
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int64_t p = base + it * kBlock + threadIdx.x;
    own[it] = p < n ? owners[p] : 0xFFFFFFFFu;
    const unsigned same = __match_any_sync(0xFFFFFFFFu, own[it]);
    rank_in_warp[it] = __popc(same & lt);
    if (p < n && (same & lt) == 0) s_pre[it][warp][own[it]] = __popc(same);
  }
  __syncthreads();
  for (uint32_t o = threadIdx.x; o < world; o += kBlock) {
    int32_t run = off[o * n_tiles + blockIdx.x];
    for (int it = 0; it < kItems; ++it)
      for (int w = 0; w < kW; ++w) {
        const int32_t c = s_pre[it][w][o];
        s_pre[it][w][o] = run;
        run += c;
      }
  }
  __syncthreads();
  if (arity == 3 && keys_out &&
      (!pay_out || (pay_rb == 4 && ((reinterpret_cast<uintptr_t>(pay) | reinterpret_cast<uintptr_t>(pay_out)) & 3) == 0))) {
    // common case (int3 keys, one 4-byte payload word): every load of the
    // thread's items before any store
    uint32_t kw[kItems][3], pw[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t p = base + it * kBlock + threadIdx.x;
      if (p >= n) continue;
#pragma unroll
      for (int d = 0; d < 3; ++d) kw[it][d] = static_cast<uint32_t>(__ldg(keys + p * 3 + d));
      if (pay_out) pw[it] = __ldg(reinterpret_cast<const uint32_t*>(pay) + p);
    }
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t p = base + it * kBlock + threadIdx.x;
      if (p >= n) continue;
      const int64_t dst = s_pre[it][warp][own[it]] + rank_in_warp[it];
      perm[dst] = static_cast<int32_t>(p);
#pragma unroll
      for (int d = 0; d < 3; ++d) keys_out[dst * 3 + d] = static_cast<int32_t>(kw[it][d]);
      if (pay_out) reinterpret_cast<uint32_t*>(pay_out)[dst] = pw[it];
    }
    return;
  }
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int64_t p = base + it * kBlock + threadIdx.x;
    if (p >= n) continue;
    const int64_t dst = s_pre[it][warp][own[it]] + rank_in_warp[it];
    perm[dst] = static_cast<int32_t>(p);
    if (keys_out)
      for (int d = 0; d < arity; ++d) keys_out[dst * arity + d] = __ldg(keys + p * arity + d);
    if (pay_out) copy_row_words(pay_out + dst * pay_rb, pay + p * pay_rb, pay_rb);
  }
}

// ---------------------------------------------------------------------------
// Peer-memory dispatch / combine (the all-to-all fused into the partition).
//
// Every rank's receive buffers are symmetric allocations (torch symmetric
// memory: each rank maps every peer's buffer over NVLink).  The owner's
// receive buffer holds its sources' segments in source-rank order, so the
// shard sees its keys in global batch order (first-occurrence exactness).
// k_route_put computes the stable owner partition exactly like
// k_route_scatter and stores each key row (+ payload row) straight into the
// owner's buffer at row_off[owner] + j, j = the position's index within its
// owner segment (kept in jdx for the combine).  k_route_pull reads each
// position's result back from its owner's result buffer.  No staging copy,
// no NCCL payload collective: the only collective is the N x N count exchange.

struct PeerArgs {
  int64_t row_off[kMaxWorld];     // this rank's first row in owner o's receive buffers
  int32_t* keys[kMaxWorld];       // owner o's receive key rows
  uint8_t* pay[kMaxWorld];        // owner o's receive payload rows (or null)
  const int32_t* ret[kMaxWorld];  // owner o's result buffer
};

__global__ void __launch_bounds__(kBlock) k_route_put(const int32_t* __restrict__ keys, int64_t n, int arity,
                                                      uint32_t world, const uint8_t* __restrict__ owners,
                                                      const int32_t* __restrict__ off, int64_t n_tiles,
                                                      const uint8_t* __restrict__ pay, int64_t pay_rb, PeerArgs pa,
                                                      int32_t* __restrict__ jdx, const int64_t* __restrict__ cmat,
                                                      uint32_t rank, int64_t cap, int staged) {
  constexpr int kW = kBlock / 32;
  // per-(item, warp, owner) offsets first; the same memory then stages the
  // tile's rows owner by owner (key words, then 4-byte payload words), each
  // owner's run aligned like its destination
  constexpr int kPreWords = kItems * kW * kMaxWorld;
  constexpr int kStageKeyWords = kTile * 3 + 4 * kMaxWorld;
  constexpr int kStageWords = kStageKeyWords + kTile + 4 * kMaxWorld;
  static_assert(kStageKeyWords % 4 == 0, "payload stage 16-byte aligned");
  __shared__ __align__(16) int32_t s_raw[kStageWords > kPreWords ? kStageWords : kPreWords];
  auto s_pre = reinterpret_cast<int32_t(*)[kW][kMaxWorld]>(s_raw);
  __shared__ int64_t s_off[kMaxWorld];
  __shared__ int32_t s_t0[kMaxWorld], s_tc[kMaxWorld], s_kb[kMaxWorld], s_pb[kMaxWorld];
  __shared__ int32_t* s_run_dst[2 * kMaxWorld];  // staged runs: peer destination, stage offset, words
  __shared__ int32_t s_run_src[2 * kMaxWorld], s_run_n[2 * kMaxWorld], s_run_ch[2 * kMaxWorld + 1], s_runs;
  __shared__ int s_skip;
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < kPreWords; e += kBlock) s_raw[e] = 0;
  if (threadIdx.x == 0) s_skip = 0;
  __syncthreads();
  // row offsets: given, or from the exchanged count matrix cmat[src][owner]
  // (rows of earlier sources at each owner); an owner whose rows would pass
  // its receive capacity makes every rank skip the put (all see the same
  // matrix), and the host re-puts after growing the buffers
  for (uint32_t o = threadIdx.x; o < world; o += kBlock) {
    int64_t before = pa.row_off[o];
    if (cmat) {
      int64_t tot = 0;
      before = 0;
      for (uint32_t src = 0; src < world; ++src) {
        const int64_t c = cmat[src * world + o];
        if (src < rank) before += c;
        tot += c;
      }
      if (tot > cap) s_skip = 1;
    }
    s_off[o] = before;
  }
  __syncthreads();
  if (s_skip) return;
  const int64_t base = blockIdx.x * static_cast<int64_t>(kTile);
  uint32_t lt;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
  uint32_t own[kItems], rank_in_warp[kItems];
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int64_t p = base + it * kBlock + threadIdx.x;
    own[it] = p < n ? owners[p] : 0xFFFFFFFFu;
    const unsigned same = __match_any_sync(0xFFFFFFFFu, own[it]);
    rank_in_warp[it] = __popc(same & lt);
    if (p < n && (same & lt) == 0) s_pre[it][warp][own[it]] = __popc(same);
  }
  __syncthreads();
  // index within the owner's segment: global owner-major offset minus the
  // segment start off[o * n_tiles]
  for (uint32_t o = threadIdx.x; o < world; o += kBlock) {
    int32_t run = off[o * n_tiles + blockIdx.x] - off[o * n_tiles];
    s_t0[o] = run;  // the tile's rows for owner o: [run, run + count) of this source's segment
    for (int it = 0; it < kItems; ++it)
      for (int w = 0; w < kW; ++w) {
        const int32_t c = s_pre[it][w][o];
        s_pre[it][w][o] = run;
        run += c;
      }
    s_tc[o] = run - s_t0[o];
  }
  __syncthreads();
  if (arity == 3 && (pay_rb == 0 || (pay_rb == 4 && (reinterpret_cast<uintptr_t>(pay) & 3) == 0))) {
    // int3 keys + at most one 4-byte value: every load first, then the
    // (peer) stores
    uint32_t kw[kItems][3], pw[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t p = base + it * kBlock + threadIdx.x;
      if (p >= n) continue;
#pragma unroll
      for (int d = 0; d < 3; ++d) kw[it][d] = static_cast<uint32_t>(__ldg(keys + p * 3 + d));
      if (pay_rb) pw[it] = __ldg(reinterpret_cast<const uint32_t*>(pay) + p);
    }
    if (!staged) {  // direct stores (A/B: ASH_PUT_STAGED=0)
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int64_t p = base + it * kBlock + threadIdx.x;
        if (p >= n) continue;
        const uint32_t o = own[it];
        const int32_t j = s_pre[it][warp][o] + static_cast<int32_t>(rank_in_warp[it]);
        const int64_t row = s_off[o] + j;
        jdx[p] = j;
        int32_t* kd = pa.keys[o] + row * 3;
#pragma unroll
        for (int d = 0; d < 3; ++d) kd[d] = static_cast<int32_t>(kw[it][d]);
        if (pay_rb) reinterpret_cast<uint32_t*>(pa.pay[o])[row] = pw[it];
      }
      return;
    }
    // rows for this rank's own shard are local stores, coalesced by the L2;
    // rows for a peer are staged per owner and leave as 16-byte vectors (a
    // direct int3 row store from a warp whose rows spread over N owners
    // moves ~4-byte pieces of many sectors across NVLink)
    int32_t jr[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t p = base + it * kBlock + threadIdx.x;
      jr[it] = 0;
      if (p >= n) continue;
      const uint32_t o = own[it];
      jr[it] = s_pre[it][warp][o] + static_cast<int32_t>(rank_in_warp[it]);
      jdx[p] = jr[it];
      if (o == rank) {
        const int64_t row = s_off[o] + jr[it];
        int32_t* kd = pa.keys[o] + row * 3;
#pragma unroll
        for (int d = 0; d < 3; ++d) kd[d] = static_cast<int32_t>(kw[it][d]);
        if (pay_rb) reinterpret_cast<uint32_t*>(pa.pay[o])[row] = pw[it];
      }
    }
    if (world == 1) return;
    __syncthreads();  // s_pre is read: its memory becomes the stage
    constexpr int kChunk = 128;  // 16-byte vectors per warp task
    if (threadIdx.x == 0) {
      uint32_t kb = 0, pb = 0;
      int32_t runs = 0, chunks = 0;
      for (uint32_t o = 0; o < world; ++o) {
        const int32_t c = o == rank ? 0 : s_tc[o];
        const int64_t row0 = s_off[o] + s_t0[o];
        for (int part = 0; part < (pay_rb ? 2 : 1); ++part) {
          int32_t* dst = part == 0 ? pa.keys[o] + row0 * 3 : reinterpret_cast<int32_t*>(pa.pay[o]) + row0;
          const int32_t words = part == 0 ? 3 * c : c;
          uint32_t& b = part == 0 ? kb : pb;
          const uint32_t a = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(dst) >> 2) & 3);
          b += (a - b) & 3u;  // the run starts congruent with its destination mod 16 bytes
          if (part == 0) s_kb[o] = static_cast<int32_t>(b);
          else s_pb[o] = static_cast<int32_t>(b);
          if (words > 0) {
            const int32_t head = min(words, static_cast<int32_t>((4 - a) & 3));
            const int32_t nv = (words - head) >> 2;
            s_run_dst[runs] = dst;
            s_run_src[runs] = static_cast<int32_t>(b) + (part == 0 ? 0 : kStageKeyWords);
            s_run_n[runs] = words;
            s_run_ch[runs] = chunks;
            chunks += nv > 0 ? (nv + kChunk - 1) / kChunk : 1;
            ++runs;
          }
          b += static_cast<uint32_t>(words);
        }
      }
      s_run_ch[runs] = chunks;
      s_runs = runs;
    }
    __syncthreads();
    int32_t* sk = s_raw;
    int32_t* sp = s_raw + kStageKeyWords;
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int64_t p = base + it * kBlock + threadIdx.x;
      if (p >= n || own[it] == rank) continue;
      const uint32_t o = own[it];
      const int32_t l = jr[it] - s_t0[o];
#pragma unroll
      for (int d = 0; d < 3; ++d) sk[s_kb[o] + 3 * l + d] = static_cast<int32_t>(kw[it][d]);
      if (pay_rb) sp[s_pb[o] + l] = static_cast<int32_t>(pw[it]);
    }
    __syncthreads();
    // warp tasks: chunk k of run r = vectors [k * kChunk, (k + 1) * kChunk),
    // the first chunk adds the unaligned head words, the last the tail
    const int lane = threadIdx.x & 31;
    const int32_t runs = s_runs, total = s_run_ch[runs];
    int r = 0;
    for (int32_t c = warp; c < total; c += kW) {
      while (s_run_ch[r + 1] <= c) ++r;
      int32_t* dst = s_run_dst[r];
      const int32_t* src = s_raw + s_run_src[r];
      const int32_t words = s_run_n[r];
      const int32_t head = min(words, static_cast<int32_t>((4 - ((reinterpret_cast<uintptr_t>(dst) >> 2) & 3)) & 3));
      const int32_t nv = (words - head) >> 2;
      const int32_t k = c - s_run_ch[r], last = s_run_ch[r + 1] - s_run_ch[r] - 1;
      if (k == 0 && lane < head) dst[lane] = src[lane];
      const int4* s4 = reinterpret_cast<const int4*>(src + head);
      int4* d4 = reinterpret_cast<int4*>(dst + head);
      const int32_t v1 = min(nv, (k + 1) * kChunk);
      for (int32_t v = k * kChunk + lane; v < v1; v += 32) d4[v] = s4[v];
      const int32_t t0 = head + 4 * nv;
      if (k == last && lane < words - t0) dst[t0 + lane] = src[t0 + lane];
    }
    return;
  }
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const int64_t p = base + it * kBlock + threadIdx.x;
    if (p >= n) continue;
    const uint32_t o = own[it];
    const int32_t j = s_pre[it][warp][o] + static_cast<int32_t>(rank_in_warp[it]);
    const int64_t row = s_off[o] + j;
    jdx[p] = j;
    int32_t* kd = pa.keys[o] + row * arity;
    for (int d = 0; d < arity; ++d) kd[d] = __ldg(keys + p * arity + d);
    if (pay_rb) copy_row_words(pa.pay[o] + row * pay_rb, pay + p * pay_rb, pay_rb);
  }
}

// out[p] = the owner's result; out_mask[p] = (out[p] >= 0) when given (the
// partitioned result's mask, so no separate compare pass)
// 4 positions per thread (vector loads of owners / jdx, vector stores); the
// per-owner base pointers are staged in shared memory
__global__ void __launch_bounds__(kBlock) k_route_pull(const uint8_t* __restrict__ owners,
                                                       const int32_t* __restrict__ jdx, int64_t n, PeerArgs pa,
                                                       uint32_t world, int32_t* __restrict__ out,
                                                       uint8_t* __restrict__ out_mask,
                                                       const int64_t* __restrict__ cmat, uint32_t rank,
                                                       const int32_t* recv_status) {
  __shared__ const int32_t* s_base[kMaxWorld];
  // an overflowed exchange stored nothing (and left jdx unwritten): no results
  if (recv_status && recv_status[1]) return;
  for (uint32_t o = threadIdx.x; o < world; o += kBlock) {
    int64_t off = pa.row_off[o];
    if (cmat) {  // this rank's first row at owner o: rows of the sources before it
      off = 0;
      for (uint32_t src = 0; src < rank; ++src) off += cmat[src * world + o];
    }
    s_base[o] = pa.ret[o] + off;
  }
  __syncthreads();
  const int64_t p0 = (blockIdx.x * static_cast<int64_t>(kBlock) + threadIdx.x) * 4;
  if (p0 >= n) return;
  const bool vec = p0 + 4 <= n && ((reinterpret_cast<uintptr_t>(owners) | reinterpret_cast<uintptr_t>(jdx) |
                                    reinterpret_cast<uintptr_t>(out) |
                                    reinterpret_cast<uintptr_t>(out_mask)) & 15) == 0 && (p0 & 3) == 0;
  if (vec) {
    const uint32_t ow = *reinterpret_cast<const uint32_t*>(owners + p0);
    const int4 j = *reinterpret_cast<const int4*>(jdx + p0);
    const int32_t jj[4] = {j.x, j.y, j.z, j.w};
    int32_t v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = s_base[(ow >> (8 * i)) & 0xFF][jj[i]];
    *reinterpret_cast<int4*>(out + p0) = make_int4(v[0], v[1], v[2], v[3]);
    if (out_mask)
      *reinterpret_cast<uint32_t*>(out_mask + p0) =
          (v[0] >= 0) | ((v[1] >= 0) << 8) | ((v[2] >= 0) << 16) | ((v[3] >= 0) << 24);
    return;
  }
  for (int64_t p = p0; p < n && p < p0 + 4; ++p) {
    const int32_t v = s_base[owners[p]][jdx[p]];
    out[p] = v;
    if (out_mask) out_mask[p] = v >= 0;
  }
}

// The rows this rank receives (sum of its column of the exchanged count
// matrix) into status[0] for the device-sized shard op, 0 when some owner's
// rows pass the receive capacity (k_route_put then stores nothing, on every
// rank alike); status[1] = that overflow.
__global__ void k_route_recv_status(const int64_t* __restrict__ cmat, uint32_t world, uint32_t rank, int64_t cap,
                                    int32_t* status) {
  __shared__ int s_over;
  if (threadIdx.x == 0) s_over = 0;
  __syncthreads();
  for (uint32_t o = threadIdx.x; o < world; o += blockDim.x) {
    int64_t tot = 0;
    for (uint32_t src = 0; src < world; ++src) tot += cmat[src * world + o];
    if (tot > cap) s_over = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t m = 0;
    for (uint32_t src = 0; src < world; ++src) m += cmat[src * world + rank];
    status[0] = s_over ? 0 : static_cast<int32_t>(m);
    status[1] = s_over;
  }
}

// Count-matrix exchange over peer memory (replaces the all-gather of the
// per-owner counts and ash_route_recv_status): every rank's exchange buffer
// holds the world x world matrix followed by one epoch flag per source rank.
// Thread t stores this rank's count row into peer t's matrix (row `rank`),
// fences at system scope and release-stores the op's epoch into peer t's
// flag[rank]; then it acquire-spins on its own flag[t] until source t's row
// of this epoch has landed.  The matrix is copied out (the next op's rows may
// overwrite the exchange buffer only after this rank passed the op's
// post-put barrier, i.e. after this copy), and the receive status computed
// as k_route_recv_status does.  A source silent for timeout_ns sets
// status[1] = 2 (the put then stores nothing, the pull is a no-op).
struct XchgArgs {
  int64_t* x[kMaxWorld];
};

__device__ __forceinline__ void st_release_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int64_t ld_relaxed_sys_i64(const int64_t* p) {
  int64_t v;
  asm volatile("ld.relaxed.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kMaxWorld) k_route_exchange(const int64_t* __restrict__ counts, uint32_t world,
                                                              uint32_t rank, XchgArgs xa, uint64_t epoch,
                                                              int64_t cap, int64_t* __restrict__ mat,
                                                              int32_t* status, uint64_t timeout_ns) {
  __shared__ int s_over, s_late;
  const uint32_t t = threadIdx.x;
  if (t == 0) s_over = s_late = 0;
  const uint32_t ww = world * world;
  if (t < world) {
    int64_t* px = xa.x[t];
    for (uint32_t j = 0; j < world; ++j) px[rank * world + j] = counts[j];
    __threadfence_system();
    st_release_sys_u64(reinterpret_cast<uint64_t*>(px + ww + rank), epoch);
  }
  __syncthreads();
  const int64_t* lx = xa.x[rank];
  if (t < world) {
    const uint64_t* f = reinterpret_cast<const uint64_t*>(lx + ww + t);
    const uint64_t t0 = global_ns();
    while (static_cast<int64_t>(ld_acquire_sys_u64(f) - epoch) < 0) {
      if (global_ns() - t0 > timeout_ns) {
        s_late = 1;
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  for (uint32_t i = t; i < ww; i += blockDim.x) mat[i] = ld_relaxed_sys_i64(lx + i);
  __syncthreads();
  for (uint32_t o = t; o < world; o += blockDim.x) {
    int64_t tot = 0;
    for (uint32_t src = 0; src < world; ++src) tot += mat[src * world + o];
    if (tot > cap) s_over = 1;
  }
  __syncthreads();
  if (t == 0) {
    int64_t m = 0;
    for (uint32_t src = 0; src < world; ++src) m += mat[src * world + rank];
    const int bad = s_late ? 2 : s_over;
    status[0] = bad ? 0 : static_cast<int32_t>(m);
    status[1] = bad;
  }
}

// dst[i] = src[idx[i]] (gather) / dst[idx[i]] = src[i] (scatter): thread per row
__global__ void k_gather_rows(const uint8_t* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                              int64_t rb, uint8_t* __restrict__ dst) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) copy_row_words(dst + i * rb, src + static_cast<int64_t>(__ldg(idx + i)) * rb, rb);
}

__global__ void k_scatter_rows(const uint8_t* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                               int64_t rb, uint8_t* __restrict__ dst) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) copy_row_words(dst + static_cast<int64_t>(__ldg(idx + i)) * rb, src + i * rb, rb);
}

// 4-byte rows (the routed result indices): two independent loads per row
__global__ void k_scatter_words(const uint32_t* __restrict__ src, const int32_t* __restrict__ idx, int64_t n,
                                uint32_t* __restrict__ dst) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) dst[__ldg(idx + i)] = __ldg(src + i);
}

__global__ void k_owner_of(const int32_t* __restrict__ keys, int64_t n, int arity, uint32_t world,
                           int32_t* __restrict__ out) {
  const int64_t p = blockIdx.x * static_cast<int64_t>(kBlock) + threadIdx.x;
  if (p < n) out[p] = static_cast<int32_t>(owner_of_global(keys + p * arity, arity, world));
}

inline unsigned blocks(int64_t work, int per) {
  int64_t g = (work + per - 1) / per;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

const char* ash_route_last_error(void) { return g_route_err; }

int64_t ash_route_scratch_len(int64_t n, int32_t world) {
  return ((n + kTile - 1) / kTile) * static_cast<int64_t>(world);
}

int ash_route_owner(const int32_t* keys, int64_t n, int32_t arity, int32_t world, int32_t* out, void* stream) {
  if (n < 0 || arity < 1 || world < 1 || world > kMaxWorld) return rfail("bad routing arguments");
  if (n == 0) return ASH_OK;
  k_owner_of<<<blocks(n, kBlock), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(keys, n, arity,
                                                                                 static_cast<uint32_t>(world), out); note_launch();
  return rcheck("ash_route_owner");
}

int ash_route_partition(const int32_t* keys, int64_t n, int32_t arity, int32_t world, int32_t* perm,
                        int64_t* counts, uint8_t* owners, int32_t* keys_out, const void* payload,
                        int64_t payload_row_bytes, void* payload_out, int32_t* scratch, int64_t scratch_len,
                        void* stream) {
  if (n < 0 || arity < 1 || world < 1 || world > kMaxWorld) return rfail("bad routing arguments");
  if (n >= (int64_t(1) << 31)) return rfail("routing batch too long");
  if (!counts) return rfail("null routing output");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n == 0) {  // empty tensors may carry null pointers
    cudaMemsetAsync(counts, 0, sizeof(int64_t) * world, s);
    return rcheck("ash_route_partition");
  }
  if (!perm || !owners || !scratch) return rfail("null routing output");
  if ((payload == nullptr) != (payload_out == nullptr) || payload_row_bytes < 0)
    return rfail("payload and payload_out must both be given");
  const int64_t n_tiles = (n + kTile - 1) / kTile;
  if (scratch_len < n_tiles * world) return rfail("routing scratch too small");
  const uint32_t w = static_cast<uint32_t>(world);
  k_route_count<<<static_cast<unsigned>(n_tiles), kBlock, 0, s>>>(keys, n, arity, w, owners, scratch, n_tiles); note_launch();
  k_route_scan<<<1, 1024, 0, s>>>(scratch, n_tiles * world, n_tiles, w, counts); note_launch();
  k_route_scatter<<<static_cast<unsigned>(n_tiles), kBlock, 0, s>>>(
      keys, n, arity, w, owners, scratch, n_tiles, perm, keys_out, static_cast<const uint8_t*>(payload),
      payload_row_bytes, static_cast<uint8_t*>(payload_out)); note_launch();
  return rcheck("ash_route_partition");
}

int ash_route_count(const int32_t* keys, int64_t n, int32_t arity, int32_t world, int64_t* counts, uint8_t* owners,
                    int32_t* scratch, int64_t scratch_len, void* stream) {
  if (n < 0 || arity < 1 || world < 1 || world > kMaxWorld) return rfail("bad routing arguments");
  if (n >= (int64_t(1) << 31)) return rfail("routing batch too long");
  if (!counts) return rfail("null routing output");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n == 0) {
    cudaMemsetAsync(counts, 0, sizeof(int64_t) * world, s);
    return rcheck("ash_route_count");
  }
  if (!keys || !owners || !scratch) return rfail("null routing buffer");
  const int64_t n_tiles = (n + kTile - 1) / kTile;
  if (scratch_len < n_tiles * world) return rfail("routing scratch too small");
  const uint32_t w = static_cast<uint32_t>(world);
  k_route_count<<<static_cast<unsigned>(n_tiles), kBlock, 0, s>>>(keys, n, arity, w, owners, scratch, n_tiles); note_launch();
  k_route_scan<<<1, 1024, 0, s>>>(scratch, n_tiles * world, n_tiles, w, counts); note_launch();
  return rcheck("ash_route_count");
}

static int route_put(const int32_t* keys, int64_t n, int32_t arity, int32_t world, const uint8_t* owners,
                     const int32_t* scratch, int64_t scratch_len, const int64_t* row_off, const int64_t* cmat,
                     int32_t rank, int64_t cap, void* const* peer_keys, const void* payload,
                     int64_t payload_row_bytes, void* const* peer_payload, int32_t* jdx, void* stream) {
  if (n < 0 || arity < 1 || world < 1 || world > kMaxWorld) return rfail("bad routing arguments");
  if (n == 0) return ASH_OK;
  if (!keys || !owners || !scratch || !(row_off || cmat) || !peer_keys || !jdx) return rfail("null routing buffer");
  if (cmat && (rank < 0 || rank >= world || cap < 0)) return rfail("bad rank or receive capacity");
  if (payload_row_bytes < 0 || (payload_row_bytes && (!payload || !peer_payload)))
    return rfail("payload and peer payload buffers must both be given");
  const int64_t n_tiles = (n + kTile - 1) / kTile;
  if (scratch_len < n_tiles * world) return rfail("routing scratch too small");
  PeerArgs pa;
  memset(&pa, 0, sizeof(pa));
  for (int o = 0; o < world; ++o) {
    if (!peer_keys[o]) return rfail("null peer key buffer");
    pa.row_off[o] = row_off ? row_off[o] : 0;
    pa.keys[o] = static_cast<int32_t*>(peer_keys[o]);
    pa.pay[o] = payload_row_bytes ? static_cast<uint8_t*>(peer_payload[o]) : nullptr;
  }
  k_route_put<<<static_cast<unsigned>(n_tiles), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(
      keys, n, arity, static_cast<uint32_t>(world), owners, scratch, n_tiles,
      static_cast<const uint8_t*>(payload), payload_row_bytes, pa, jdx, cmat, static_cast<uint32_t>(rank),
      cap, g_put_staged); note_launch();
  return rcheck("ash_route_put");
}

int ash_route_put(const int32_t* keys, int64_t n, int32_t arity, int32_t world, const uint8_t* owners,
                  const int32_t* scratch, int64_t scratch_len, const int64_t* row_off, void* const* peer_keys,
                  const void* payload, int64_t payload_row_bytes, void* const* peer_payload, int32_t* jdx,
                  void* stream) {
  if (!row_off) return rfail("null routing buffer");
  return route_put(keys, n, arity, world, owners, scratch, scratch_len, row_off, nullptr, 0, 0, peer_keys,
                   payload, payload_row_bytes, peer_payload, jdx, stream);
}

int ash_route_put_counts(const int32_t* keys, int64_t n, int32_t arity, int32_t world, int32_t rank,
                         const uint8_t* owners, const int32_t* scratch, int64_t scratch_len,
                         const int64_t* count_matrix, int64_t recv_capacity, void* const* peer_keys,
                         const void* payload, int64_t payload_row_bytes, void* const* peer_payload, int32_t* jdx,
                         void* stream) {
  if (!count_matrix) return rfail("null count matrix");
  return route_put(keys, n, arity, world, owners, scratch, scratch_len, nullptr, count_matrix, rank,
                   recv_capacity, peer_keys, payload, payload_row_bytes, peer_payload, jdx, stream);
}

int ash_route_pull(const uint8_t* owners, const int32_t* jdx, int64_t n, int32_t world, const int64_t* row_off,
                   const void* const* peer_ret, int32_t* out, uint8_t* out_mask, void* stream) {
  if (n < 0 || world < 1 || world > kMaxWorld) return rfail("bad routing arguments");
  if (n == 0) return ASH_OK;
  if (!owners || !jdx || !row_off || !peer_ret || !out) return rfail("null routing buffer");
  PeerArgs pa;
  memset(&pa, 0, sizeof(pa));
  for (int o = 0; o < world; ++o) {
    if (!peer_ret[o]) return rfail("null peer result buffer");
    pa.row_off[o] = row_off[o];
    pa.ret[o] = static_cast<const int32_t*>(peer_ret[o]);
  }
  k_route_pull<<<blocks((n + 3) / 4, kBlock), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(
      owners, jdx, n, pa, static_cast<uint32_t>(world), out, out_mask, nullptr, 0, nullptr); note_launch();
  return rcheck("ash_route_pull");
}

int ash_route_recv_status(const int64_t* count_matrix, int32_t world, int32_t rank, int64_t recv_capacity,
                          int32_t* status, void* stream) {
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world || recv_capacity < 0)
    return rfail("bad routing arguments");
  if (!count_matrix || !status) return rfail("null routing buffer");
  k_route_recv_status<<<1, 64, 0, static_cast<cudaStream_t>(stream)>>>(count_matrix, static_cast<uint32_t>(world),
                                                                      static_cast<uint32_t>(rank), recv_capacity,
                                                                      status); note_launch();
  return rcheck("ash_route_recv_status");
}

int ash_route_exchange(const int64_t* counts, int32_t world, int32_t rank, void* const* peer_xchg, uint64_t epoch,
                       int64_t recv_capacity, int64_t* count_matrix, int32_t* status, uint64_t timeout_ns,
                       void* stream) {
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world || recv_capacity < 0 || epoch == 0)
    return rfail("bad routing arguments");
  if (!counts || !peer_xchg || !count_matrix || !status) return rfail("null routing buffer");
  XchgArgs xa;
  memset(&xa, 0, sizeof(xa));
  for (int o = 0; o < world; ++o) {
    if (!peer_xchg[o]) return rfail("null peer exchange buffer");
    xa.x[o] = static_cast<int64_t*>(peer_xchg[o]);
  }
  k_route_exchange<<<1, kMaxWorld, 0, static_cast<cudaStream_t>(stream)>>>(
      counts, static_cast<uint32_t>(world), static_cast<uint32_t>(rank), xa, epoch, recv_capacity, count_matrix,
      status, timeout_ns);
  note_launch();
  return rcheck("ash_route_exchange");
}

int ash_route_pull_counts(const uint8_t* owners, const int32_t* jdx, int64_t n, int32_t world, int32_t rank,
                          const int64_t* count_matrix, const int32_t* recv_status, const void* const* peer_ret,
                          int32_t* out, uint8_t* out_mask, void* stream) {
  if (n < 0 || world < 1 || world > kMaxWorld || rank < 0 || rank >= world) return rfail("bad routing arguments");
  if (n == 0) return ASH_OK;
  if (!owners || !jdx || !count_matrix || !peer_ret || !out) return rfail("null routing buffer");
  PeerArgs pa;
  memset(&pa, 0, sizeof(pa));
  for (int o = 0; o < world; ++o) {
    if (!peer_ret[o]) return rfail("null peer result buffer");
    pa.ret[o] = static_cast<const int32_t*>(peer_ret[o]);
  }
  k_route_pull<<<blocks((n + 3) / 4, kBlock), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(
      owners, jdx, n, pa, static_cast<uint32_t>(world), out, out_mask, count_matrix, static_cast<uint32_t>(rank),
      recv_status);
  note_launch();
  return rcheck("ash_route_pull_counts");
}

int ash_gather_rows(const void* src, const int32_t* idx, int64_t n, int64_t row_bytes, void* dst, void* stream) {
  if (n < 0 || row_bytes < 0) return rfail("bad gather arguments");
  if (n == 0 || row_bytes == 0) return ASH_OK;
  k_gather_rows<<<blocks(n, kBlock), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src), idx, n, row_bytes, static_cast<uint8_t*>(dst)); note_launch();
  return rcheck("ash_gather_rows");
}

int ash_scatter_rows(const void* src, const int32_t* idx, int64_t n, int64_t row_bytes, void* dst, void* stream) {
  if (n < 0 || row_bytes < 0) return rfail("bad scatter arguments");
  if (n == 0 || row_bytes == 0) return ASH_OK;
  if (row_bytes == 4 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 3) == 0) {
    k_scatter_words<<<blocks(n, kBlock), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint32_t*>(src), idx, n, static_cast<uint32_t*>(dst)); note_launch();
    return rcheck("ash_scatter_rows");
  }
  k_scatter_rows<<<blocks(n, kBlock), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src), idx, n, row_bytes, static_cast<uint8_t*>(dst)); note_launch();
  return rcheck("ash_scatter_rows");
}

}  // extern "C"

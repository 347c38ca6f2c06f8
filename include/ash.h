/*
 * ash.h — C ABI of the B200-native spatial hash map (libash.so).
 *
 * This is the drop-in boundary below the reference's Python map API
 * (/root/reference/pkg/src/spatialhash/hashmap.py:153-515).  The reference has
 * no FFI of its own — it is pure numpy — so each entry point below names the
 * reference method whose semantics it implements; INTEGRATION.md shows the
 * ctypes binding a maintainer would add on the reference side.
 *
 * Rules of the ABI
 *   - Stateless launchers.  All memory (table, buffers, heap, counters, scan
 *     workspace) is allocated by the caller and described by ash_map_t; no
 *     ownership crosses the boundary.
 *   - Every call is asynchronous on `stream` (a cudaStream_t passed as void*).
 *     Results that the host needs (sizes, counts, error flags) are written to
 *     device counters; the caller reads them when it must.
 *   - Return codes: ASH_OK, or an ASH_ERR_* code with a message retrievable
 *     through ash_last_error() (thread-local).
 *   - Plain pointers and sizes only: no torch or CUDA types in signatures.
 */
#ifndef ASH_H
#define ASH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASH_ABI_VERSION 7

#define ASH_OK 0
#define ASH_ERR_INVALID 1   /* bad argument (caller bug) -> ValueError        */
#define ASH_ERR_CAPACITY 2  /* batch needs more free indices -> CapacityError */
#define ASH_ERR_CUDA 3      /* launch / runtime failure -> RuntimeError       */

#define ASH_MAX_VALUE_BUFFERS 8

/* device counter slots (int32 each, ASH_N_COUNTERS of them) */
#define ASH_CTR_TOP 0      /* index-heap top; equals the map size          */
#define ASH_CTR_TOMBS 1    /* tombstone slots (erased / rolled-back claims) */
#define ASH_CTR_WINNERS 2  /* new keys of the last insert/activate         */
#define ASH_CTR_ERASED 3   /* keys removed by the last erase               */
#define ASH_CTR_FLAGS 4    /* sticky error bits, see ASH_FLAG_*            */
#define ASH_CTR_COUNT 5    /* result count of the last compaction/voxelize */
#define ASH_CTR_TOP_BASE 6 /* heap top at the start of the current commit   */
#define ASH_CTR_HEAP_DIRTY 7 /* heap[i] == i for every i >= this value     */
#define ASH_N_COUNTERS 8

#define ASH_FLAG_TABLE_FULL 1  /* a claim probe wrapped the table (or hit max_probe) */
#define ASH_FLAG_RANGE 2       /* quantized coordinate outside int32 */
#define ASH_FLAG_CAPACITY 4    /* a device-sized insert did not fit: nothing committed */
#define ASH_FLAG_SPEC 8        /* state, not an error: the last claim used top + pos pending states */

/*
 * Map state.  Table slots are 16 bytes {w0, w1, w2, state}: the first three
 * key words inline (zero-padded for arity < 3) and
 *   state = 0xFFFFFFFF EMPTY | 0xFFFFFFFE TOMBSTONE | [0, 2^31) buffer index
 *         | 0x80000000|pos  (PENDING, only inside one insert batch).
 * Slots are probed in 32-byte buckets (two slots, one DRAM sector).
 */
typedef struct ash_map {
  void* slots;              /* n_slots x 16 B                                  */
  int64_t n_slots;          /* even, 64 <= n_slots <= 2^30                     */
  int32_t* key_buf;         /* capacity x arity int32  (hashmap.py:203)        */
  int32_t arity;            /* >= 1                                            */
  int32_t n_values;         /* number of value buffers, <= 8                   */
  void* value_bufs[ASH_MAX_VALUE_BUFFERS];          /* capacity x row bytes    */
  int64_t value_row_bytes[ASH_MAX_VALUE_BUFFERS];   /* hashmap.py:204-206      */
  int32_t* heap;            /* capacity, index free list (index_heap.py:17-20) */
  uint8_t* active;          /* capacity, 0/1 (hashmap.py:207)                  */
  int32_t* erase_claim;     /* capacity, INT32_MAX between calls               */
  uint8_t* freed;           /* capacity, 0 between calls                       */
  int32_t* counters;        /* ASH_N_COUNTERS                                  */
  uint64_t* scan_status;    /* single-pass scan tile status, zeroed once       */
  int64_t scan_status_len;  /* >= ash_scan_tiles(max(n, capacity))             */
  int32_t* tile_counts;     /* per-2048-position winner counts, zero between   */
  int64_t tile_counts_len;  /* batches; >= ash_scan_tiles(n); with H =        */
                            /* (len-1)/2 >= tiles, inserts count in [0, H) and */
                            /* keep the tile prefixes in [H, 2H]               */
  int64_t capacity;         /* <= 2^31 - 1                                     */
  uint32_t epoch;           /* scan epoch; the library bumps it per launch     */
  uint32_t max_probe;       /* claim probe limit in buckets (0: whole table); */
                            /* a claim that hits it sets ASH_FLAG_TABLE_FULL */
  int32_t* rank_words;      /* optional: 2 x ceil(n / 32) int32, lets the     */
  int64_t rank_words_len;   /* table-sweep commit rank winners without tmp    */
} ash_map_t;

int ash_abi_version(void);
const char* ash_last_error(void);

/* Per-device setup for the random-access workload: caps the L2 fetch
 * granularity at `l2_fetch_bytes` (32 = one sector per random probe) on the
 * current device.  Call once per process and device. */
int ash_device_setup(int32_t l2_fetch_bytes);

/* Mark batch streams (keys, values, scratch, outputs) L2 evict-first so the
 * table keeps the L2 (default on; process-wide). */
int ash_set_stream_hints(int32_t on);

/* Kernels launched by this library so far (process-wide counter). */
int64_t ash_launch_count(void);

/* Insert commit strategy (process-wide; same results in every mode).
 *   bulk = 1: TMA-staged persistent commit where the batch qualifies (arity
 *             <= 3, one register-sized value buffer or none, 16-byte aligned
 *             streams, tile workspace >= 2 * tiles + 1); 0: plain commit.
 *   sweep_div > 0: batches with >= n_buckets / sweep_div winners commit the
 *             slot states in one sequential table pass instead of random
 *             stores; 0: never.  Defaults: 1, 5. */
int ash_set_commit_mode(int32_t bulk, int32_t sweep_div);
/* Tables of at most `bytes` (slots x 16) never take the table sweep: their
 * lines stay in the L2 between the claim and the commit, so the commit's
 * state stores are L2 hits.  < 0: the default, three quarters of the L2;
 * 0: every table may sweep (tests of the sweep on small maps). */
int ash_set_sweep_table_min(int64_t bytes);


/* Scan-status words needed for a single-pass scan over n items. */
int64_t ash_scan_tiles(int64_t n);

/* HashMap.__init__/_init_state (hashmap.py:200-210): all slots EMPTY,
 * heap = arange(capacity), counters 0, active 0; key/value rows zeroed when
 * zero_rows != 0. */
int ash_map_reset(ash_map_t* m, int32_t zero_rows, void* stream);

/* HashMap.find (hashmap.py:415-429): out_idx = buffer index or -1,
 * out_mask = 1 where present.  One fused hash+probe kernel. */
int ash_find(ash_map_t* m, const int32_t* keys, int64_t n, int32_t* out_idx,
             uint8_t* out_mask, void* stream);

/* radius_neighbors (geometry.py:87-99): for each of n int3 coordinates and
 * each of the (2r+1)^3 lattice offsets in lexicographic order (dx outer),
 * find(coords[i] + offset[j]) -> out_idx / out_mask [i * (2r+1)^3 + j].
 * The offset queries are generated in-kernel (no n x 27 key buffer).
 * Requires key arity 3 and 0 <= r <= 15. */
int ash_find_lattice(ash_map_t* m, const int32_t* coords, int64_t n, int32_t r,
                     int32_t* out_idx, uint8_t* out_mask, void* stream);

/* HashMap.insert / activate (hashmap.py:336-413), generic-backend semantics:
 * winners are first occurrences of absent keys, winner of rank r gets
 * heap[top + r].  `values` holds n_values device pointers (rows of
 * value_row_bytes each, batch order) or is NULL for activate/HashSet.
 * association != 0 gives activate masks (found OR winner).
 * Precondition: capacity - size >= n (the caller checks; otherwise use the
 * claim/count/commit|rollback sequence below).  ash_insert = claim + count +
 * commit. */
int ash_insert(ash_map_t* m, const int32_t* keys, int64_t n,
               const void* const* values, int32_t association,
               int32_t* out_idx, uint8_t* out_mask, void* stream);

/* Split form of ash_insert for the capacity-uncertain path
 * (hashmap.py:389-396 re-plan on growth, :317-324 CapacityError):
 *   claim -> count (counters[WINNERS]; scans the per-tile winner counts the
 *   claim kept) -> host reads the count -> commit when it fits, else
 *   rollback (map unchanged).  commit requires the preceding count. */
int ash_insert_claim(ash_map_t* m, const int32_t* keys, int64_t n,
                     int32_t* out_idx, uint8_t* out_mask, void* stream);
int ash_insert_count(ash_map_t* m, int64_t n, const int32_t* out_idx,
                     const uint8_t* out_mask, void* stream);
int ash_insert_commit(ash_map_t* m, const int32_t* keys, int64_t n,
                      const void* const* values, int32_t association,
                      int32_t* out_idx, uint8_t* out_mask, void* stream);
int ash_insert_rollback(ash_map_t* m, int64_t n, const int32_t* out_idx,
                        void* stream);

/* Deferred slot-state commit (same contract and results as ash_insert /
 * ash_insert_commit; needs m->rank_words).  When the batch is large enough
 * for the table-sweep commit, the sweep is not run: the table keeps the
 * batch's winners as PENDING|pos, which ash_find / ash_find_lattice resolve
 * on the fly from the rank words (index = top + rank(pos), or
 * heap[top + rank]).  The caller MUST call ash_settle before the next
 * mutating call on m (insert / activate / erase / rebuild / rehash / reset
 * excepted: a reset discards the table).  The sweep then runs once, or never
 * if the map is reset first.  Reference semantics are unchanged
 * (hashmap.py:397-413): only the moment the slot states are written moves. */
int ash_insert_lazy(ash_map_t* m, const int32_t* keys, int64_t n,
                    const void* const* values, int32_t association,
                    int32_t* out_idx, uint8_t* out_mask, void* stream);
int ash_insert_commit_lazy(ash_map_t* m, const int32_t* keys, int64_t n,
                           const void* const* values, int32_t association,
                           int32_t* out_idx, uint8_t* out_mask, void* stream);
int ash_settle(ash_map_t* m, void* stream);

/* HashMap.erase (hashmap.py:431-456): first found occurrence per key is
 * removed; freed indices return to the heap sorted (index_heap.py:38-47).
 * scratch: 2*n int32 device words. */
int ash_erase(ash_map_t* m, const int32_t* keys, int64_t n, uint8_t* out_mask,
              int32_t* scratch, void* stream);

/* HashMap.active_indices (hashmap.py:458-460): ascending; `out` must hold
 * size entries; the count is also written to counters[COUNT]. */
int ash_active_indices(ash_map_t* m, int32_t* out, void* stream);

/* HashMap._rehash_into (hashmap.py:326-332): dst is freshly reset; rows
 * act[0..n_act) of src (ascending) become rows 0..n_act-1 of dst. */
int ash_rehash_from(ash_map_t* dst, const ash_map_t* src, const int32_t* act,
                    int64_t n_act, void* stream);

/* Tombstone cleanup: rebuild the table into new_slots (same indices, no API
 * visible change).  The caller swaps m->slots afterwards. */
int ash_rebuild_table(ash_map_t* m, void* new_slots, int64_t new_n_slots,
                      void* stream);

/* Fill a table with EMPTY slots (workspace initialisation). */
int ash_table_clear(void* slots, int64_t n_slots, void* stream);

/* geometry.quantize (geometry.py:49-56): floor(p / cell) in float64;
 * out of int32 range sets ASH_FLAG_RANGE in flags[0]. */
int ash_quantize(const void* points, int32_t points_are_f64, int64_t n,
                 double cell, int32_t* out_coords, int32_t* flags, void* stream);

/* geometry.voxel_downsample (geometry.py:59-76), fused quantize + set insert
 * + first-occurrence select.  `ws` supplies an all-EMPTY workspace table,
 * counters and scan status; the slots claimed are left EMPTY again.  Writes
 * count voxels to out_coords (count x 3) / out_sel (int64) in ascending
 * point order; count in ws->counters[COUNT].  The table must hold every
 * distinct voxel: with n_slots >= 2n it always does; a smaller table (sized
 * from an estimate, ws->max_probe bounding the probes) may overflow, which
 * sets ASH_FLAG_TABLE_FULL: the results are then invalid, the table must be
 * refilled with EMPTY and the call repeated with a larger one.
 * scratch_idx: n int32 (>= ceil(n / 32) used: word prefixes); scratch_mask:
 * 8 * ceil(n / 32) bytes, 4-byte aligned (candidate / displaced bitmaps). */
int ash_voxelize(ash_map_t* ws, const void* points, int32_t points_are_f64,
                 int64_t n, double voxel, int32_t* out_coords, int64_t* out_sel,
                 int32_t* scratch_idx, uint8_t* scratch_mask, void* stream);

/* ---- hash-partitioned multi-GPU mode (no reference
 * counterpart): owner(key) = mix64(key) -> [0, world). ---------------------- */

const char* ash_route_last_error(void);

/* int32 scratch words ash_route_partition needs for n keys and world ranks. */
int64_t ash_route_scratch_len(int64_t n, int32_t world);

/* owner rank of every key (world <= 64). */
int ash_route_owner(const int32_t* keys, int64_t n, int32_t arity, int32_t world,
                    int32_t* out, void* stream);

/* Stable partition of a batch by owner: perm lists positions grouped by
 * owner rank, batch order kept inside each group; counts[world] (int64) are
 * the group sizes (the all-to-all send splits); owners[n] (uint8) the owner
 * of every key.  The send buffers are written in the same pass: keys_out
 * (n x arity, may be NULL) and one payload row per key (payload_row_bytes
 * each; payload/payload_out both NULL for none). */
int ash_route_partition(const int32_t* keys, int64_t n, int32_t arity, int32_t world,
                        int32_t* perm, int64_t* counts, uint8_t* owners, int32_t* keys_out,
                        const void* payload, int64_t payload_row_bytes, void* payload_out,
                        int32_t* scratch, int64_t scratch_len, void* stream);

/* dst[i] = src[idx[i]] and dst[idx[i]] = src[i] for rows of row_bytes. */
int ash_gather_rows(const void* src, const int32_t* idx, int64_t n, int64_t row_bytes,
                    void* dst, void* stream);
int ash_scatter_rows(const void* src, const int32_t* idx, int64_t n, int64_t row_bytes,
                     void* dst, void* stream);

/* Distinct int3 rows of a batch in first-occurrence order (the local
 * activate + survivor gather of tsdf/grid.py:140-142 without a local map):
 * out_keys[0 .. ws->counters[ASH_CTR_COUNT]) and, if out_first is given,
 * their first positions (int64).  Workspace rules as for ash_voxelize. */
int ash_unique_rows(ash_map_t* ws, const int32_t* keys, int64_t n, int32_t* out_keys,
                    int64_t* out_first, int32_t* scratch_idx, uint8_t* scratch_mask, void* stream);

/* Block candidates of one depth frame (tsdf/grid.py:98-125 _candidate_blocks
 * + block_of :24-27).  depth: height x width float64 (row-major, device);
 * cam = {fx, fy, cx, cy, depth_min, depth_max}; pose: 4x4 row-major float64
 * camera-to-world (host).  neighbor = 0: ray mode (samples at half-block
 * spacing within +-trunc of the surface), 1: surface block + 26 neighbours.
 * Virtual position p = pixel * per_pixel + sample, per_pixel =
 * ash_frame_positions(...) / (height * width).  Float64 arithmetic follows
 * the reference's operation order (FrameSrc in ash_map.cu). */
int64_t ash_frame_positions(int64_t height, int64_t width, double block_size, double trunc,
                            int32_t neighbor);

/* Every virtual position's candidate (out_coords: positions x 3) and
 * out_valid = 1 where its pixel is valid (Frame.valid_mask); the reference's
 * candidate list is out_coords[out_valid].  flags |= ASH_FLAG_RANGE when a
 * block coordinate leaves int32. */
int ash_frame_candidates(const double* depth, int64_t height, int64_t width, const double* cam,
                         const double* pose, double block_size, double trunc, int32_t neighbor,
                         int32_t* out_coords, uint8_t* out_valid, int32_t* flags, void* stream);

/* Fused candidates + dedup (the local activate of grid.py:140-142): the
 * frame's distinct block coordinates in first-occurrence order, written to
 * out_coords[0 .. ws->counters[ASH_CTR_COUNT]).  ws is an all-EMPTY workspace
 * table as for ash_voxelize (left EMPTY again); scratch_idx: positions int32,
 * scratch_mask: 8 * ceil(positions / 32) bytes. */
int ash_frame_blocks(ash_map_t* ws, const double* depth, int64_t height, int64_t width,
                     const double* cam, const double* pose, double block_size, double trunc,
                     int32_t neighbor, int32_t* out_coords, int32_t* scratch_idx,
                     uint8_t* scratch_mask, void* stream);

/* Device-sized batches: ash_find / ash_insert (claim + count + commit) on
 * keys[0 .. *d_n), the length read on the device when each kernel starts;
 * n_max >= *d_n bounds it (grids, scratch, tile workspace for n_max).  Lets
 * one stream chain an op whose result count stays on the device (a dedup,
 * a routed shard batch) into a map op with no host round trip.  The insert
 * clears counters[FLAGS] first and checks capacity on the device: when the
 * winners do not fit below capacity it commits nothing and sets
 * ASH_FLAG_CAPACITY; a claim that cannot place a key within 4096 buckets
 * sets ASH_FLAG_TABLE_FULL.  On either flag the caller runs
 * ash_insert_rollback(m, *d_n, out_idx) (which also clears the flags) and
 * redoes the batch on the host-checked path (growth / CapacityError,
 * hashmap.py:389-396). */
int ash_find_dn(ash_map_t* m, const int32_t* keys, int64_t n_max, const int32_t* d_n,
                int32_t* out_idx, uint8_t* out_mask, void* stream);
int ash_insert_dn(ash_map_t* m, const int32_t* keys, int64_t n_max, const int32_t* d_n,
                  const void* const* values, int32_t association, int32_t* out_idx,
                  uint8_t* out_mask, void* stream);

/* VoxelBlockGrid.allocate_blocks map calls (tsdf/grid.py:136-150) as one
 * stream-ordered sequence with no host round trip: the distinct rows of
 * coords[0..n) in first-occurrence order -> out_blocks (ash_unique_rows on
 * the workspace ws), then the global activate of those rows
 * (ash_insert_dn, association = 1) -> out_gi / out_gmask.  status (device,
 * int32[5]): [0] rows activated (0 when the workspace prefix overflowed:
 * refill it and repeat on a larger one), [1] distinct rows, [2] workspace
 * flags, [3] global flags (ASH_FLAG_CAPACITY / TABLE_FULL: roll back
 * [0] claims and redo the activate on the host path), [4] new blocks.
 * out_blocks: n x 3, out_gi / out_gmask: n entries; scratch as for
 * ash_unique_rows; global tile workspace for n positions.  small_activate:
 * run the activate in one block (up to 8192 distinct rows; more leave
 * status[0] = 0 and nothing claimed, for the host path): the caller's
 * choice from the previous frame's count. */
int ash_allocate_blocks(ash_map_t* global, ash_map_t* ws, const int32_t* coords, int64_t n,
                        int32_t* out_blocks, int32_t* out_gi, uint8_t* out_gmask,
                        int32_t* scratch_idx, uint8_t* scratch_mask, int32_t* status,
                        int32_t small_activate, void* stream);

/* Copy rows [0, min(*d_count, cap)) of two arrays (row sizes multiples of 4
 * bytes) in one launch: the caller's own copies of a fused allocate's
 * results (status + 1 = the distinct rows), enqueued before the count is
 * read on the host. */
int ash_copy_prefix2(const void* src0, void* dst0, int64_t row_bytes0, const void* src1, void* dst1,
                     int64_t row_bytes1, const int32_t* d_count, int64_t cap, void* stream);

/* The same from a depth frame (candidates generated in-kernel, as
 * ash_frame_blocks): VoxelBlockGrid.allocate_blocks(frame), grid.py:127-150. */
int ash_allocate_frame(ash_map_t* global, ash_map_t* ws, const double* depth, int64_t height,
                       int64_t width, const double* cam, const double* pose, double block_size,
                       double trunc, int32_t neighbor, int32_t* out_blocks, int32_t* out_gi,
                       uint8_t* out_gmask, int32_t* scratch_idx, uint8_t* scratch_mask,
                       int32_t* status, int32_t small_activate, void* stream);

/* Delegate-backend insert commit (hashmap.py:369-387), after
 * ash_insert_claim + ash_insert_count: position p owns heap[top + p]; every
 * key row is written there (losers' rows stay as stale data, as in the
 * reference); winner p keeps heap[top + p]; the other positions' indices are
 * written to loser_out[0 .. n - winners) in position order.  The caller
 * sorts them (fill the rest of loser_out with INT32_MAX first) and hands
 * them to ash_heap_put_losers.  Precondition: capacity - size >= n. */
int ash_insert_commit_delegate(ash_map_t* m, const int32_t* keys, int64_t n,
                               const void* const* values, int32_t association, int32_t* out_idx,
                               uint8_t* out_mask, int32_t* loser_out, void* stream);

/* heap[top_base + W + i] = sorted_losers[i] for i < n - W (the sorted free of
 * index_heap.py:38-47), W / top_base from the device counters. */
int ash_heap_put_losers(ash_map_t* m, const int32_t* sorted_losers, int64_t n, void* stream);

/* Peer-memory dispatch / combine for the hash-partitioned map (no NCCL
 * payload collective).  ash_route_count: owners + per-owner counts (device
 * int64[world]) with the tile offsets in scratch.  ash_route_put: the stable
 * owner partition stores every key row (and payload row) directly into owner
 * o's receive buffers peer_keys[o] / peer_payload[o] (symmetric allocations
 * mapped on this rank; host arrays of world device pointers) at row
 * row_off[o] + j, j = index within this rank's owner-o segment (-> jdx).
 * ash_route_pull: out[p] = peer_ret[owner(p)][row_off[owner(p)] + jdx[p]].
 * The caller orders put -> (peer barrier) -> shard op -> (peer barrier) -> pull. */
int ash_route_count(const int32_t* keys, int64_t n, int32_t arity, int32_t world, int64_t* counts,
                    uint8_t* owners, int32_t* scratch, int64_t scratch_len, void* stream);
int ash_route_put(const int32_t* keys, int64_t n, int32_t arity, int32_t world, const uint8_t* owners,
                  const int32_t* scratch, int64_t scratch_len, const int64_t* row_off,
                  void* const* peer_keys, const void* payload, int64_t payload_row_bytes,
                  void* const* peer_payload, int32_t* jdx, void* stream);
/* ash_route_put with the row offsets taken on the device from the exchanged
 * count matrix count_matrix[src * world + owner] (device int64, world x world):
 * row_off[o] = sum over src < rank of count_matrix[src][o].  The put is
 * launched before the host has read the matrix, so the host read overlaps
 * it.  If any owner's total rows exceed recv_capacity (rows of each receive
 * buffer) nothing is stored: every rank sees the same matrix and skips
 * alike, and the caller grows the buffers and puts again. */
int ash_route_put_counts(const int32_t* keys, int64_t n, int32_t arity, int32_t world, int32_t rank,
                         const uint8_t* owners, const int32_t* scratch, int64_t scratch_len,
                         const int64_t* count_matrix, int64_t recv_capacity, void* const* peer_keys,
                         const void* payload, int64_t payload_row_bytes, void* const* peer_payload,
                         int32_t* jdx, void* stream);
int ash_route_pull(const uint8_t* owners, const int32_t* jdx, int64_t n, int32_t world,
                   const int64_t* row_off, const void* const* peer_ret, int32_t* out,
                   uint8_t* out_mask /* optional: out >= 0 */, void* stream);

/* Sync-free routing (the peer transport's device-sized shard ops): the rows
 * this rank receives, sum of its column of the exchanged count matrix, into
 * status[0] (0 when any owner's rows pass recv_capacity: ash_route_put_counts
 * then stores nothing on every rank, status[1] = 1, and the caller redoes
 * the op with grown buffers); ash_route_pull with this rank's row offsets
 * taken from the count matrix on the device, a no-op when recv_status[1]
 * reports the overflow. */
int ash_route_recv_status(const int64_t* count_matrix, int32_t world, int32_t rank,
                          int64_t recv_capacity, int32_t* status, void* stream);
int ash_route_pull_counts(const uint8_t* owners, const int32_t* jdx, int64_t n, int32_t world,
                          int32_t rank, const int64_t* count_matrix, const int32_t* recv_status,
                          const void* const* peer_ret, int32_t* out, uint8_t* out_mask, void* stream);
/* Count-matrix exchange over peer memory, replacing the all-gather of the
 * per-owner counts and ash_route_recv_status in one kernel.  peer_xchg[r]:
 * rank r's exchange buffer (int64, world * world + world entries, mapped
 * here; its flag tail zeroed before the first op).  Stores this rank's
 * counts into row `rank` of every peer's matrix and release-stores `epoch`
 * (> 0, +1 per op, the same on every rank) into its flag; waits (device
 * side) for every source's flag of this epoch, then writes the matrix to
 * count_matrix (device, world x world) and status as ash_route_recv_status,
 * with status[1] = 2 when some source stayed silent for timeout_ns. */
int ash_route_exchange(const int64_t* counts, int32_t world, int32_t rank, void* const* peer_xchg,
                       uint64_t epoch, int64_t recv_capacity, int64_t* count_matrix, int32_t* status,
                       uint64_t timeout_ns, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ASH_H */

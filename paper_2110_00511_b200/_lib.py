"""ctypes binding of libash.so (include/ash.h).

There is no CPU fallback: importing this module without the built library
raises, and every launcher error surfaces as a Python exception.
"""
from __future__ import annotations

import ctypes
import os as _os
from ctypes import POINTER, c_char_p, c_double, c_int32, c_int64, c_uint32, c_void_p

from .build import LIB_PATH

ASH_OK, ASH_ERR_INVALID, ASH_ERR_CAPACITY, ASH_ERR_CUDA = 0, 1, 2, 3
MAX_VALUE_BUFFERS = 8
CTR_TOP, CTR_TOMBS, CTR_WINNERS, CTR_ERASED, CTR_FLAGS, CTR_COUNT, CTR_TOP_BASE = 0, 1, 2, 3, 4, 5, 6
CTR_HEAP_DIRTY = 7
N_COUNTERS = 8
FLAG_TABLE_FULL, FLAG_RANGE, FLAG_CAPACITY, FLAG_SPEC = 1, 2, 4, 8
TILE = 2048  # positions per scan tile (csrc kTile)


class AshMap(ctypes.Structure):
    """Mirror of ``ash_map_t``."""
    _fields_ = [
        ("slots", c_void_p), ("n_slots", c_int64),
        ("key_buf", c_void_p), ("arity", c_int32), ("n_values", c_int32),
        ("value_bufs", c_void_p * MAX_VALUE_BUFFERS),
        ("value_row_bytes", c_int64 * MAX_VALUE_BUFFERS),
        ("heap", c_void_p), ("active", c_void_p), ("erase_claim", c_void_p),
        ("freed", c_void_p), ("counters", c_void_p), ("scan_status", c_void_p),
        ("scan_status_len", c_int64), ("tile_counts", c_void_p), ("tile_counts_len", c_int64),
        ("capacity", c_int64),
        ("epoch", c_uint32), ("max_probe", c_uint32),
        ("rank_words", c_void_p), ("rank_words_len", c_int64),
    ]


_M = POINTER(AshMap)
_SIGNATURES = {
    "ash_abi_version": (c_int32, []),
    "ash_last_error": (c_char_p, []),
    "ash_device_setup": (c_int32, [c_int32]),
    "ash_set_stream_hints": (c_int32, [c_int32]),
    "ash_launch_count": (c_int64, []),
    "ash_set_commit_mode": (c_int32, [c_int32, c_int32]),
    "ash_set_sweep_table_min": (c_int32, [c_int64]),
    "ash_scan_tiles": (c_int64, [c_int64]),
    "ash_map_reset": (c_int32, [_M, c_int32, c_void_p]),
    "ash_find": (c_int32, [_M, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "ash_find_lattice": (c_int32, [_M, c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p]),
    "ash_insert": (c_int32, [_M, c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    "ash_insert_claim": (c_int32, [_M, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "ash_insert_count": (c_int32, [_M, c_int64, c_void_p, c_void_p, c_void_p]),
    "ash_insert_commit": (c_int32, [_M, c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    "ash_insert_rollback": (c_int32, [_M, c_int64, c_void_p, c_void_p]),
    "ash_insert_lazy": (c_int32, [_M, c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    "ash_insert_commit_lazy": (c_int32, [_M, c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                         c_void_p]),
    "ash_settle": (c_int32, [_M, c_void_p]),
    "ash_find_dn": (c_int32, [_M, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ash_insert_dn": (c_int32, [_M, c_void_p, c_int64, c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p]),
    "ash_copy_prefix2": (c_int32, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_int64,
                                   c_void_p]),
    "ash_allocate_blocks": (c_int32, [_M, _M, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_int32, c_void_p]),
    "ash_allocate_frame": (c_int32, [_M, _M, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_double, c_double,
                                     c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                     c_int32, c_void_p]),
    "ash_insert_commit_delegate": (c_int32, [_M, c_void_p, c_int64, c_void_p, c_int32, c_void_p, c_void_p,
                                             c_void_p, c_void_p]),
    "ash_heap_put_losers": (c_int32, [_M, c_void_p, c_int64, c_void_p]),
    "ash_erase": (c_int32, [_M, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "ash_active_indices": (c_int32, [_M, c_void_p, c_void_p]),
    "ash_rehash_from": (c_int32, [_M, _M, c_void_p, c_int64, c_void_p]),
    "ash_rebuild_table": (c_int32, [_M, c_void_p, c_int64, c_void_p]),
    "ash_table_clear": (c_int32, [c_void_p, c_int64, c_void_p]),
    "ash_quantize": (c_int32, [c_void_p, c_int32, c_int64, c_double, c_void_p, c_void_p, c_void_p]),
    "ash_voxelize": (c_int32, [_M, c_void_p, c_int32, c_int64, c_double, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_void_p]),
    "ash_unique_rows": (c_int32, [_M, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ash_frame_positions": (c_int64, [c_int64, c_int64, c_double, c_double, c_int32]),
    "ash_frame_candidates": (c_int32, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_double, c_double,
                                       c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ash_frame_blocks": (c_int32, [_M, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_double, c_double,
                                   c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ash_route_last_error": (c_char_p, []),
    "ash_route_scratch_len": (c_int64, [c_int64, c_int32]),
    "ash_route_owner": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p]),
    "ash_route_partition": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p,
                                      c_void_p, c_void_p, c_void_p, c_int64, c_void_p,
                                      c_void_p, c_int64, c_void_p]),
    "ash_route_count": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_int64,
                                  c_void_p]),
    "ash_route_put": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p, c_int64, c_void_p,
                                c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "ash_route_put_counts": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_int32, c_void_p, c_void_p,
                                       c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_void_p,
                                       c_void_p, c_void_p]),
    "ash_route_pull": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p]),
    "ash_route_recv_status": (c_int32, [c_void_p, c_int32, c_int32, c_int64, c_void_p, c_void_p]),
    "ash_route_pull_counts": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_void_p]),
    "ash_route_exchange": (c_int32, [c_void_p, c_int32, c_int32, c_void_p, ctypes.c_uint64, c_int64, c_void_p,
                                     c_void_p, ctypes.c_uint64, c_void_p]),
    "ash_gather_rows": (c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "ash_scatter_rows": (c_int32, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
}
_ROUTE_FUNCS = ("ash_route_owner", "ash_route_partition", "ash_gather_rows", "ash_scatter_rows",
                "ash_route_count", "ash_route_put", "ash_route_put_counts", "ash_route_pull",
                "ash_route_recv_status", "ash_route_pull_counts", "ash_route_exchange")

EXPORTED = tuple(_SIGNATURES)


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA library must be built first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ash_abi_version() != 7:
        raise ImportError("libash.so ABI version mismatch; rebuild")
    return lib


lib = _load()
lib.ash_set_stream_hints(int(_os.environ.get("ASH_STREAM_HINTS", "1")))
lib.ash_set_sweep_table_min(int(_os.environ.get("ASH_SWEEP_TABLE_MIN", "-1")))
lib.ash_set_commit_mode(int(_os.environ.get("ASH_COMMIT_BULK", "1")),
                        int(_os.environ.get("ASH_SWEEP_DIV", "5")))


class AshError(RuntimeError):
    pass


def call(name: str, *args) -> None:
    """Invoke an ABI entry point and map its status code to an exception."""
    rc = getattr(lib, name)(*args)
    if rc == ASH_OK:
        return
    err = lib.ash_route_last_error if name in _ROUTE_FUNCS else lib.ash_last_error
    msg = (err() or b"").decode(errors="replace")
    if rc == ASH_ERR_INVALID:
        raise ValueError(f"{name}: {msg}")
    raise AshError(f"{name} failed ({rc}): {msg}")


_setup_done = set()
# one DRAM sector per random probe (profiles/ r01 showed 64+ B over-fetch);
# ASH_L2_FETCH=0 leaves the driver default (for A/B measurements)
L2_FETCH_BYTES = int(_os.environ.get("ASH_L2_FETCH", "32"))


def device_setup(device) -> None:
    """Once per process and device: cap the L2 fetch granularity."""
    import torch
    key = (device.type, device.index)
    if key in _setup_done:
        return
    with torch.cuda.device(device):
        call("ash_device_setup", L2_FETCH_BYTES)
    _setup_done.add(key)


def scan_tiles(n: int) -> int:
    """ash_scan_tiles(n) (ceil(max(n, 1) / TILE)) without the foreign call;
    tests/test_abi_cpu.py checks the two agree."""
    return (max(int(n), 1) + TILE - 1) // TILE

"""ctypes binding of libhetm_b200.so (include/hetm_b200/capi.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  There is no CPU fallback: importing without the library raises,
and every device call on a machine without a CUDA device raises
``NoDeviceError`` (HETM_ERR_NO_DEVICE).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhetm_b200.so")

if not os.path.exists(LIB_PATH):  # fail loudly: the CUDA extension is the product
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
    )

lib = C.CDLL(LIB_PATH)

u8p = C.POINTER(C.c_uint64)


class DevConfig(C.Structure):
    _fields_ = [
        ("size_words", C.c_uint64),
        ("shard_base", C.c_uint64),
        ("rs_gran_bytes", C.c_uint64),
        ("chunk_bytes", C.c_uint64),
        ("log_capacity", C.c_uint64),
        ("max_attempts", C.c_uint32),
        ("device", C.c_int32),
        ("flags", C.c_uint32),
        ("reserved", C.c_uint32),
    ]


class DevInfo(C.Structure):
    _fields_ = [
        ("size_words", C.c_uint64),
        ("shard_base", C.c_uint64),
        ("rs_gran_bytes", C.c_uint64),
        ("chunk_bytes", C.c_uint64),
        ("cell_bytes", C.c_uint64),
        ("rs_bits", C.c_uint64),
        ("rs_words", C.c_uint64),
        ("chunk_bits", C.c_uint64),
        ("chunk_words", C.c_uint64),
        ("log_capacity", C.c_uint64),
        ("device_bytes", C.c_uint64),
        ("device", C.c_int32),
        ("sm_count", C.c_int32),
        ("l2_bytes", C.c_uint64),
        ("ticket_next", C.c_uint64),
    ]


class Delivery(C.Structure):  # hetm_delivery (bus.hpp:51-56 Delivery + completion handle)
    _fields_ = [
        ("seq", C.c_uint64),
        ("n_entries", C.c_uint64),
        ("bytes", C.c_uint64),
        ("handle", C.c_uint64),
        ("src_thread", C.c_int32),
        ("mode", C.c_int32),
    ]


class SourceStats(C.Structure):  # hetm_source_stats
    _fields_ = [("chunks", C.c_uint64), ("entries", C.c_uint64), ("last_seq", C.c_uint64),
                ("last_handle", C.c_uint64)]


class BatchStats(C.Structure):
    _fields_ = [
        ("n_tx", C.c_uint64),
        ("committed", C.c_uint64),
        ("aborts", C.c_uint64),
        ("livelocked", C.c_uint64),
        ("ticket_first", C.c_uint64),
        ("ticket_end", C.c_uint64),
        ("kernel_ms", C.c_double),
        ("retried", C.c_uint64),
    ]


class MergeStats(C.Structure):
    _fields_ = [
        ("dirty_chunks", C.c_uint64),
        ("transfers", C.c_uint64),
        ("bytes_d2h", C.c_uint64),
        ("bytes_h2d", C.c_uint64),
        ("bytes_d2d", C.c_uint64),
        ("ms", C.c_double),
    ]


class TransferRecord(C.Structure):
    _fields_ = [("dir", C.c_int32), ("tag", C.c_int32), ("bytes", C.c_uint64)]


_vp = C.c_void_p
_sigs = {
    "hetm_strerror": (C.c_char_p, [C.c_int]),
    "hetm_abi_version": (C.c_int, []),
    "hetm_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "hetm_dev_config_default": (None, [C.POINTER(DevConfig)]),
    "hetm_dev_open": (C.c_int, [C.POINTER(DevConfig), C.POINTER(_vp)]),
    "hetm_dev_close": (C.c_int, [_vp]),
    "hetm_dev_info_get": (C.c_int, [_vp, C.POINTER(DevInfo)]),
    "hetm_dev_last_error": (C.c_char_p, [_vp]),
    "hetm_dev_raw_write": (C.c_int, [_vp, C.c_int, C.c_uint64, C.c_uint64]),
    "hetm_dev_raw_read": (C.c_int, [_vp, C.c_int, C.c_uint64, u8p]),
    "hetm_dev_upload": (C.c_int, [_vp, C.c_int, C.c_uint64, _vp, C.c_uint64]),
    "hetm_dev_download": (C.c_int, [_vp, C.c_int, C.c_uint64, _vp, C.c_uint64]),
    "hetm_dev_register_kernel": (C.c_int, [_vp, C.c_int]),
    "hetm_dev_execute_batch": (C.c_int, [_vp, C.c_int, _vp, C.c_uint64, C.c_uint64, _vp, C.POINTER(BatchStats)]),
    "hetm_dev_bitmap_stats": (C.c_int, [_vp, u8p, u8p, u8p]),
    "hetm_dev_bitmap_words": (C.c_int, [_vp, C.c_int, u8p]),
    "hetm_dev_snapshot_bitmap": (C.c_int, [_vp, C.c_int, _vp, C.c_uint64]),
    "hetm_dev_or_bitmap": (C.c_int, [_vp, C.c_int, _vp, C.c_uint64]),
    "hetm_dev_open_intake": (C.c_int, [_vp]),
    "hetm_dev_close_intake": (C.c_int, [_vp]),
    "hetm_dev_stream_chunk": (C.c_int, [_vp, _vp, C.c_uint64, C.c_int, C.c_uint64, C.c_int]),
    "hetm_dev_stream_chunk_ex": (C.c_int, [_vp, _vp, C.c_uint64, C.c_int, C.c_uint64, C.c_int, C.POINTER(Delivery)]),
    "hetm_dev_delivery_done": (C.c_int, [_vp, C.c_uint64, C.POINTER(C.c_int)]),
    "hetm_dev_delivery_wait": (C.c_int, [_vp, C.c_uint64]),
    "hetm_dev_source_stats": (C.c_int, [_vp, C.c_int, C.POINTER(SourceStats)]),
    "hetm_dev_set_validation_period": (C.c_int, [_vp, C.c_uint32]),
    "hetm_dev_apply_log": (C.c_int, [_vp]),
    "hetm_dev_poll_conflict": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "hetm_dev_round_verdict": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "hetm_dev_sync": (C.c_int, [_vp]),
    "hetm_dev_merge_commit": (C.c_int, [_vp, _vp, C.POINTER(MergeStats)]),
    "hetm_dev_merge_abort_device": (C.c_int, [_vp, C.c_int, _vp, C.POINTER(MergeStats)]),
    "hetm_dev_merge_abort_host": (C.c_int, [_vp, _vp, _vp, C.POINTER(MergeStats)]),
    "hetm_dev_merge_wait": (C.c_int, [_vp]),
    "hetm_dev_clear_round": (C.c_int, [_vp, C.c_uint32]),
    "hetm_dev_transfer_count": (C.c_int, [_vp, u8p]),
    "hetm_dev_transfer_log": (C.c_int, [_vp, C.POINTER(TransferRecord), C.c_uint64, u8p]),
    "hetm_dev_clear_transfer_log": (C.c_int, [_vp]),
    "hetm_dev_execute_batch_dptr": (C.c_int, [_vp, C.c_int, _vp, C.c_uint64, _vp, _vp]),
    "hetm_dev_execute_batch_dptr_ex": (C.c_int, [_vp, C.c_int, _vp, C.c_uint64, _vp, _vp, _vp]),
    "hetm_dev_execute_batch_ex": (C.c_int, [_vp, C.c_int, _vp, C.c_uint64, C.c_uint64, _vp, _vp, C.c_uint64,
                                            C.POINTER(BatchStats)]),
    "hetm_dev_set_cache_geometry": (C.c_int, [_vp, C.c_uint64, C.c_uint64]),
    "hetm_cache_hash": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "hetm_cache_set_of": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
    "hetm_gen_cache_batch": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_uint32, C.c_int32,
                                       C.c_uint32, _vp]),
    "hetm_dev_validate_dptr": (C.c_int, [_vp, _vp, C.c_uint64, C.c_int, _vp]),
    "hetm_dev_read_counters": (C.c_int, [_vp, C.POINTER(C.c_int), C.POINTER(BatchStats)]),
    "hetm_dev_recv_arena": (C.c_int, [_vp, C.c_uint32, C.c_uint64, C.POINTER(_vp), C.POINTER(_vp)]),
    "hetm_dev_route_to_peers_dptr": (C.c_int, [_vp, _vp, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint64,
                                               C.c_uint32, _vp, _vp, _vp]),
    "hetm_dev_apply_received": (C.c_int, [_vp, C.c_uint32, C.c_int, u8p, _vp]),
    "hetm_ipc_get_handle": (C.c_int, [_vp, _vp]),
    "hetm_ipc_open_handle": (C.c_int, [_vp, C.POINTER(_vp)]),
    "hetm_ipc_close": (C.c_int, [_vp]),
    "hetm_enable_peer_access": (C.c_int, [C.c_int, C.c_int]),
    "hetm_dev_route_log_dptr": (C.c_int, [_vp, _vp, C.c_uint64, C.c_uint32, C.c_uint64, _vp, _vp, _vp]),
    "hetm_dev_stream_handle": (C.c_int, [_vp, C.c_int, C.POINTER(_vp)]),
    "hetm_dev_flush_l2": (C.c_int, [_vp, _vp]),
    "hetm_dev_set_timing": (C.c_int, [_vp, C.c_int]),
    "hetm_dev_debug_words": (C.c_int, [_vp, _vp, C.c_uint64]),
    "hetm_dev_trace_next_batch": (C.c_int, [_vp, _vp]),
    "hetm_dev_set_fault": (C.c_int, [_vp, C.c_uint32]),
    "hetm_dev_set_schedule": (C.c_int, [_vp, C.c_int]),
    "hetm_dev_merge_prepare": (C.c_int, [_vp, _vp]),
    "hetm_dev_merge_stage": (C.c_int, [_vp]),
    "hetm_dev_bitmap_dptr": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "hetm_dev_bitmap_or_peers": (C.c_int, [_vp, C.c_int, _vp, C.c_uint32, C.c_uint64, C.c_uint64, _vp]),
    "hetm_dev_timing": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_double), u8p]),
    "hetm_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(_vp)]),
    "hetm_host_free": (C.c_int, [_vp]),
    "hetm_host_register": (C.c_int, [_vp, C.c_uint64]),
    "hetm_host_unregister": (C.c_int, [_vp]),
    "hetm_gen_bank_batch": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _vp]),
    "hetm_gen_bank_batch_zipf": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, _vp]),
    "hetm_gen_host_log_zipf": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                                         C.c_uint64, C.c_double, _vp]),
    "hetm_gen_host_log": (
        C.c_int,
        [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, _vp],
    ),
}

EXPORTED = tuple(_sigs)

for _name, (_res, _args) in _sigs.items():
    _f = getattr(lib, _name)  # AttributeError here = the library does not export the header's symbol
    _f.restype = _res
    _f.argtypes = _args

"""ctypes binding of include/suco_b200.h (libsuco_b200.so, built in-tree).

The product path: every call lands in hand-written sm_100a kernels. There is
no CPU fallback — if the shared library is missing this module raises at
import, and on a host without a GPU every compute call raises Error.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SUCO_LIB") or os.path.join(HERE, "libsuco_b200.so")  # SUCO_LIB: tuning builds only

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library first "
        "(python -c 'import __graft_entry__ as g; g.build()')")

lib = C.CDLL(LIB_PATH)

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


class IndexParamsC(C.Structure):
    _fields_ = [("num_subspaces", C.c_uint32), ("k_half", C.c_uint32), ("iterations", C.c_uint32),
                ("mode", C.c_uint32), ("seed", C.c_uint64)]


class CollisionParamsC(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_double), ("k", C.c_uint32)]


def _sig(name, restype, *argtypes):
    try:
        f = getattr(lib, name)
    except AttributeError:
        if LIB_PATH == os.path.join(HERE, "libsuco_b200.so"):
            raise
        def missing(*_a, _n=name):  # an older SUCO_LIB build (A/B timing only)
            raise ImportError(f"{LIB_PATH} does not export {_n}")
        return missing
    f.restype = restype
    f.argtypes = list(argtypes)
    return f


last_error = _sig("suco_last_error", C.c_char_p)
device_count = _sig("suco_gpu_device_count", C.c_int, C.POINTER(C.c_int))
collision_count = _sig("suco_collision_count", C.c_uint64, C.c_double, C.c_uint64)
candidate_count = _sig("suco_candidate_count", C.c_uint64, C.c_double, C.c_uint64, C.c_uint64)
validate_collision_params = _sig("suco_validate_collision_params", C.c_int, C.POINTER(CollisionParamsC), C.c_uint64)
build_index = _sig("suco_gpu_build_index", C.c_int, f32p, C.c_uint64, C.c_uint32, C.POINTER(IndexParamsC), C.c_int,
                   C.POINTER(vp))
build_index_sampled = _sig("suco_gpu_build_index_sampled", C.c_int, f32p, C.c_uint64, C.c_uint32, C.POINTER(IndexParamsC),
                           u32p, C.c_uint64, C.c_int, C.POINTER(vp))
load_index = _sig("suco_gpu_load_index", C.c_int, u8p, C.c_uint64, f32p, C.c_uint64, C.c_uint32, C.c_int,
                  C.POINTER(vp))
serialize_index = _sig("suco_gpu_serialize_index", C.c_int, vp, u8p, C.c_uint64, u64p)
index_subspace = _sig("suco_gpu_index_subspace", C.c_int, vp, C.c_uint32, f32p, f32p, u64p, u32p)
index_info = _sig("suco_gpu_index_info", C.c_int, vp, u64p, u32p, C.POINTER(IndexParamsC), u32p, u32p, u32p)
free_index = _sig("suco_gpu_free_index", None, vp)
knn_query_batch = _sig("suco_gpu_knn_query_batch", C.c_int, vp, f32p, C.c_uint64, C.c_uint32,
                       C.POINTER(CollisionParamsC), u32p, f64p, vp)
knn_query_batch_device = _sig("suco_gpu_knn_query_batch_device", C.c_int, vp, vp, C.c_uint64, C.c_uint32,
                              C.POINTER(CollisionParamsC), vp, vp, vp, vp)
query_ctx_create = _sig("suco_gpu_query_ctx_create", C.c_int, vp, C.POINTER(vp))
query_ctx_free = _sig("suco_gpu_query_ctx_free", None, vp)
query_ctx_synchronize = _sig("suco_gpu_query_ctx_synchronize", C.c_int, vp)
query_ctx_set_profiling = _sig("suco_gpu_query_ctx_set_profiling", C.c_int, vp, C.c_int)
query_ctx_stage_times = _sig("suco_gpu_query_ctx_stage_times", C.c_int, vp, f64p, u64p)
query_ctx_last_launches = _sig("suco_gpu_query_ctx_last_launches", C.c_int, vp, u64p)
query_ctx_exchange_bytes = _sig("suco_gpu_query_ctx_exchange_bytes", C.c_int, vp, u64p)
exact_knn_batch = _sig("suco_gpu_exact_knn_batch", C.c_int, vp, f32p, C.c_uint64, C.c_uint32, C.c_uint32, u32p, f64p)
sc_scores = _sig("suco_gpu_sc_scores", C.c_int, vp, f32p, C.c_uint32, C.c_double, u32p)
sc_linear_batch = _sig("suco_gpu_sc_linear_batch", C.c_int, vp, f32p, C.c_uint64, C.c_uint32,
                       C.POINTER(CollisionParamsC), u32p, f64p)
read_vecs = _sig("suco_read_vecs", C.c_int, C.c_char_p, C.c_int, C.c_uint64, f32p, C.c_uint64, u64p, u32p)
write_vecs = _sig("suco_write_vecs", C.c_int, C.c_char_p, C.c_int, C.c_uint64, C.c_uint32, f32p)
build_index_from_vecs = _sig("suco_gpu_build_index_from_vecs", C.c_int, C.c_char_p, C.c_int, C.c_uint64,
                             C.POINTER(IndexParamsC), C.c_int, C.POINTER(vp))
load_index_from_vecs = _sig("suco_gpu_load_index_from_vecs", C.c_int, u8p, C.c_uint64, C.c_char_p, C.c_int, C.c_uint64,
                            C.c_int, C.POINTER(vp))
query_intermediates = _sig("suco_gpu_query_intermediates", C.c_int, vp, f32p, C.c_uint32,
                           C.POINTER(CollisionParamsC), u32p, u32p, u64p, u32p, u64p)
comm_nccl_id = _sig("suco_comm_nccl_id", C.c_int, u8p)
comm_nccl_create = _sig("suco_comm_nccl_create", C.c_int, u8p, C.c_int, C.c_int, C.c_int, C.POINTER(vp))
comm_local_create = _sig("suco_comm_local_create", C.c_int, C.c_int, C.POINTER(vp))
comm_info = _sig("suco_comm_info", C.c_int, vp, C.POINTER(C.c_int), C.POINTER(C.c_int), u64p)
comm_free = _sig("suco_comm_free", None, vp)
shard_block_hint = _sig("suco_gpu_shard_block_hint", C.c_int, C.c_uint64, C.c_uint32, u32p)
build_shard = _sig("suco_gpu_build_shard", C.c_int, vp, C.c_uint64, C.c_uint32, C.POINTER(IndexParamsC), C.c_uint32,
                   u32p, C.c_uint64, vp, C.c_int, C.POINTER(vp))
make_shard = _sig("suco_gpu_make_shard", C.c_int, vp, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(vp))
shard_info = _sig("suco_gpu_shard_info", C.c_int, vp, u64p, u64p, u32p, u32p, u32p)
shard_knn_query_batch = _sig("suco_gpu_shard_knn_query_batch", C.c_int, vp, vp, f32p, C.c_uint64, C.c_uint32,
                             C.POINTER(CollisionParamsC), u32p, f64p, vp)
shard_knn_query_batch_device = _sig("suco_gpu_shard_knn_query_batch_device", C.c_int, vp, vp, vp, C.c_uint64,
                                    C.c_uint32, C.POINTER(CollisionParamsC), vp, vp, vp, vp)
centroid_distances = _sig("suco_gpu_centroid_distances", C.c_int, f32p, C.c_uint32, f32p, C.c_uint32, f64p, u32p)
dynamic_activation = _sig("suco_gpu_dynamic_activation", C.c_int, C.c_double, C.c_uint64, f64p, u32p, f64p, u32p,
                          C.c_uint32, u64p, u32p, u32p, u64p, f64p, C.c_uint64, u64p)
rerank = _sig("suco_gpu_rerank", C.c_int, f32p, C.c_uint64, C.c_uint32, f32p, C.c_uint32, u32p, C.c_uint64,
              C.c_uint32, u32p, f64p)
kmeans = _sig("suco_gpu_kmeans", C.c_int, f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int,
              f32p, u32p, u32p, u32p)
build_imi = _sig("suco_gpu_build_imi", C.c_int, u32p, u32p, C.c_uint64, C.c_uint32, u64p, u32p)

# every entry point include/suco_b200.h declares (tests/test_capi.py checks the header agrees)
EXPORTED = [
    "suco_last_error", "suco_gpu_device_count", "suco_collision_count", "suco_candidate_count",
    "suco_validate_collision_params", "suco_gpu_build_index", "suco_gpu_build_index_sampled", "suco_gpu_load_index",
    "suco_gpu_serialize_index", "suco_gpu_index_subspace", "suco_gpu_index_info", "suco_gpu_free_index",
    "suco_gpu_knn_query_batch", "suco_gpu_knn_query_batch_device", "suco_gpu_query_ctx_create",
    "suco_gpu_query_ctx_free", "suco_gpu_query_ctx_synchronize", "suco_gpu_query_ctx_set_profiling",
    "suco_gpu_query_ctx_stage_times", "suco_gpu_query_ctx_last_launches", "suco_gpu_query_ctx_exchange_bytes",
    "suco_gpu_query_intermediates", "suco_comm_nccl_id", "suco_comm_nccl_create", "suco_comm_local_create",
    "suco_comm_info", "suco_comm_free", "suco_gpu_shard_block_hint", "suco_gpu_build_shard", "suco_gpu_make_shard",
    "suco_gpu_shard_info", "suco_gpu_shard_knn_query_batch", "suco_gpu_shard_knn_query_batch_device",
    "suco_gpu_exact_knn_batch", "suco_gpu_sc_scores", "suco_gpu_sc_linear_batch", "suco_read_vecs",
    "suco_write_vecs", "suco_gpu_build_index_from_vecs", "suco_gpu_load_index_from_vecs",
    "suco_gpu_centroid_distances", "suco_gpu_dynamic_activation", "suco_gpu_rerank", "suco_gpu_kmeans",
    "suco_gpu_build_imi",
]

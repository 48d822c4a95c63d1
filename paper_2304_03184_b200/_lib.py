"""ctypes binding of the C-ABI library (include/capfields_b200.h).

The library is the product: if it is missing or CUDA is unavailable, every
entry point raises — there is no CPU fallback on any path.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

from .errors import DegenerateWeightsError, OutOfSupportError, RecordFormatError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libcapfields_b200.so")

CF_OK = 0
CF_E_BAD_ARG = 1
CF_E_OUT_OF_SUPPORT = 2
CF_E_DUPLICATE_FRAME = 3
CF_E_DEGENERATE = 4
CF_E_CUDA = 5
CF_E_FORMAT = 6
CF_POOL_HUMAN = 0
CF_POOL_OBJECT = 1

CF_WARP_BACKWARD = 0
CF_WARP_FORWARD = 1
CF_BRUTE_QUERY = 2
CF_NEIGHBORS_ONLY = 3

CF_MAX_LEVELS = 16

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_f64 = ctypes.c_double


class HashGridDesc(ctypes.Structure):
    _fields_ = [
        ("n_levels", ctypes.c_int),
        ("n_features", ctypes.c_int),
        ("log2_table", ctypes.c_int),
        ("base_resolution", ctypes.c_int),
        ("max_resolution", ctypes.c_int),
        ("resolution", ctypes.c_int * CF_MAX_LEVELS),
        ("dense", ctypes.c_int * CF_MAX_LEVELS),
        ("offset", ctypes.c_int64 * (CF_MAX_LEVELS + 1)),
    ]


class Camera(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double), ("width", ctypes.c_int), ("height", ctypes.c_int),
                ("params", ctypes.c_void_p), ("row0", ctypes.c_int), ("row_stride", ctypes.c_int)]


class OccGrid(ctypes.Structure):
    _fields_ = [("min", ctypes.c_double * 3), ("cell", ctypes.c_double), ("res", ctypes.c_int)]


class MarchDesc(ctypes.Structure):
    _fields_ = [("origin", ctypes.c_double * 3), ("n_rays", ctypes.c_int64), ("n_samples", ctypes.c_int),
                ("t_near", ctypes.c_double), ("t_far", ctypes.c_double), ("dt", ctypes.c_double),
                ("human_grid", OccGrid), ("object_grid", OccGrid), ("obj_R", ctypes.c_double * 9),
                ("obj_t", ctypes.c_double * 3), ("obj_min", ctypes.c_double * 3), ("obj_inv_side", ctypes.c_double),
                ("human_cell_bbox", ctypes.c_void_p), ("sample_t", ctypes.c_void_p), ("frame", ctypes.c_void_p)]


class MarchOut(ctypes.Structure):
    _fields_ = [("records", ctypes.c_void_p), ("ray_offset", ctypes.c_void_p), ("ray_count", ctypes.c_void_p),
                ("counters", ctypes.c_void_p), ("capacity", ctypes.c_int64)]


class HumanWarp(ctypes.Structure):
    _fields_ = [("dqs", ctypes.c_void_p), ("k", ctypes.c_int), ("r2", ctypes.c_double),
                ("vert_Tinv", ctypes.c_void_p), ("lbs_max_d2", ctypes.c_double),
                ("canon_min", ctypes.c_double * 3), ("inv_side", ctypes.c_double),
                ("anchors", ctypes.c_void_p), ("n_nodes", ctypes.c_int), ("anchor_block", ctypes.c_void_p),
                ("cand_grid", ctypes.c_void_p)]


class FieldDesc(ctypes.Structure):
    _fields_ = [("has_deform", ctypes.c_int), ("dgrid", HashGridDesc), ("dtable", ctypes.c_void_p),
                ("cgrid", HashGridDesc), ("ctable", ctypes.c_void_p), ("wblob", ctypes.c_void_p),
                ("w_bytes", ctypes.c_int), ("dbias", ctypes.c_void_p), ("delta_scale", ctypes.c_float),
                ("inv_side", ctypes.c_float), ("save_h", ctypes.c_void_p), ("save_o", ctypes.c_void_p),
                ("save_mask", ctypes.c_void_p), ("precise", ctypes.c_int), ("wblob_lo", ctypes.c_void_p),
                ("train", ctypes.c_int), ("split_stages", ctypes.c_int), ("max_ctas", ctypes.c_int)]


class DwProblem(ctypes.Structure):
    _fields_ = [("A", ctypes.c_void_p), ("a_rows", ctypes.c_int64), ("m", ctypes.c_int),
                ("B", ctypes.c_void_p), ("b_rows", ctypes.c_int64), ("n", ctypes.c_int), ("C", ctypes.c_void_p), ("ldc", ctypes.c_int)]


class AdamTensor(ctypes.Structure):
    _fields_ = [("p", ctypes.c_void_p), ("g", ctypes.c_void_p), ("m", ctypes.c_void_p), ("v", ctypes.c_void_p),
                ("p16", ctypes.c_void_p), ("n", ctypes.c_int64), ("lr", ctypes.c_float), ("scale_idx", ctypes.c_int)]


class PackItem(ctypes.Structure):
    _fields_ = [("w", ctypes.c_void_p), ("blob", ctypes.c_void_p), ("blob_lo", ctypes.c_void_p), ("rows", ctypes.c_int),
                ("cols", ctypes.c_int), ("ldw", ctypes.c_int), ("col0", ctypes.c_int), ("transpose", ctypes.c_int)]


class MpInfo(ctypes.Structure):
    _fields_ = [("n_frames", ctypes.c_int64), ("n_nodes", ctypes.c_int32), ("n_theta", ctypes.c_int32),
                ("bytes", ctypes.c_int64)]


class VisCamera(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3), ("fx", ctypes.c_double),
                ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double)]


class PoolDesc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("count", ctypes.c_int), ("capacity", ctypes.c_int),
                ("n_theta", ctypes.c_int), ("vis_words", ctypes.c_int), ("theta", ctypes.c_void_p),
                ("vis", ctypes.c_void_p), ("t", ctypes.c_void_p), ("d", ctypes.c_void_p),
                ("beta_pose", ctypes.c_void_p), ("beta_vis", ctypes.c_double), ("beta_t", ctypes.c_double),
                ("beta_d", ctypes.c_double), ("gamma", ctypes.c_double)]


class PoolEntry(ctypes.Structure):
    _fields_ = [("theta", ctypes.c_void_p), ("vis", ctypes.c_void_p), ("t", ctypes.c_int64), ("d", ctypes.c_void_p)]


class PoolDecision(ctypes.Structure):
    _fields_ = [("insert", ctypes.c_int), ("evict", ctypes.c_int), ("nearest", ctypes.c_int), ("pad", ctypes.c_int),
                ("min_dissim", ctypes.c_double)]


class TsdfDesc(ctypes.Structure):
    _fields_ = [("tsdf", ctypes.c_void_p), ("weight", ctypes.c_void_p), ("resolution", ctypes.c_int),
                ("pad", ctypes.c_int), ("voxel", ctypes.c_double), ("origin", ctypes.c_double * 3),
                ("trunc", ctypes.c_double)]


class Rigid(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("t", ctypes.c_double * 3)]


class Pinhole(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double), ("cy", ctypes.c_double),
                ("width", ctypes.c_int), ("height", ctypes.c_int)]


class Csr(ctypes.Structure):
    _fields_ = [("val", ctypes.c_void_p), ("col", ctypes.c_void_p), ("rowptr", ctypes.c_void_p),
                ("rows", ctypes.c_int), ("cols", ctypes.c_int), ("nnz", ctypes.c_int64)]


class CopyList(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("src", ctypes.c_void_p * 8), ("dst", ctypes.c_void_p * 8),
                ("bytes", ctypes.c_int64 * 8)]


class NrSystem(ctypes.Structure):
    _p = ctypes.c_void_p
    _fields_ = [("dqs", _p), ("nodes", _p), ("n_nodes", ctypes.c_int), ("n_theta", ctypes.c_int),
                ("warped", _p), ("data_idx", _p), ("data_u", _p), ("data_n", _p), ("n_data", ctypes.c_int64),
                ("blend_idx", _p), ("blend_wn", _p), ("k", ctypes.c_int), ("w_data", ctypes.c_double),
                ("data_row0", ctypes.c_int64), ("data_entry0", ctypes.c_int64),
                ("do_bind", ctypes.c_int), ("node_lbs", _p), ("node_jth", _p), ("s_bind", ctypes.c_double),
                ("bind_row0", ctypes.c_int64), ("bind_entry0", ctypes.c_int64),
                ("edges", _p), ("n_edges", ctypes.c_int64), ("s_reg", ctypes.c_double),
                ("reg_row0", ctypes.c_int64), ("reg_entry0", ctypes.c_int64),
                ("pose_lbs", _p), ("pose_u", _p), ("pose_n", _p), ("pose_jth", _p), ("n_pose", ctypes.c_int64),
                ("w_pose", ctypes.c_double), ("pose_row0", ctypes.c_int64), ("pose_entry0", ctypes.c_int64),
                ("val", _p), ("col", _p), ("res", _p), ("energy", _p),
                ("jac_terms", ctypes.c_int)]


class DeformBwdIO(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("save_h", "save_o", "save_mask", "d_o", "dpre", "d_dfeat")]


class ColorBwdIO(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("h1", "cin", "c1", "c2", "d_o", "dc2", "dc1", "dg", "dh1", "dfeat")]


def byref(x):
    return ctypes.byref(x)


_P = ctypes.POINTER
# name -> argtypes (all return int status)
_SIGS = {
    "cf_device_sm_count": [],
    "cf_selftest_exact_div": [_i64, ctypes.c_uint64, ctypes.POINTER(_i64)],
    "cf_deform_nodes": [_p, _p, _i64, _p, _p],
    "cf_anchor_block_bytes": [_i64, _P(_i64)],
    "cf_cand_grid_bytes": [_i32, _i32, _P(_i64)],
    "cf_cand_grid_build": [_p, _i64, _i32, _f64, _i32, _i32, _p, _p],
    "cf_dq_blend": [_p, _p, _i64, _i32, _p, _p, _p],
    "cf_dq_status": [_p, _p],
    "cf_dq_apply": [_p, _i64, _p, _i64, _i64, _p, _p],
    "cf_deform_nodes_block": [_p, _p, _i64, _p, _p, _p],
    "cf_buckets_create": [_i64, _i32, ctypes.POINTER(_p)],
    "cf_buckets_destroy": [_p],
    "cf_buckets_destroy_async": [_p, _p],
    "cf_buckets_build": [_p, _p, _i64, _i32, _p],
    "cf_buckets_build_candidates": [_p, _i32, _p],
    "cf_knn_warp": [_p, _p, _p, _i64, _i32, _f64, _i32, _p, _i64, _p, _p, _p, _p, _p],
    "cf_knn_warp_cull": [_p, _p, _i64, _i32, _f64, _i32, _p, _p, _i64, _p, _p, _p, _p, _p],
    "cf_knnfield_build": [_p, _i64, _i32, _i32, _p, _f64, _f64, _p, _p],
    "cf_knnfield_update": [_p, _p, _i64, _p, _i32, _i32, _p, _f64, _f64, _p, _p, _p, _p],
    "cf_knnfield_query": [_p, _p, _p, _p, _i32, _i32, _p, _f64, _f64, _p, _i64, _p, _p, _p, _p, _p],
    "cf_knnfield_query_sparse": [_p, _p, _p, _p, _p, _i32, _i32, _p, _f64, _f64, _p, _i64, _p, _p, _p, _p, _p],
    "cf_knnfield_brick_count": [_i32, _P(_i64)],
    "cf_knnfield_brick_index": [_p, _i32, _p, _p, _p],
    "cf_knnfield_brick_pack": [_p, _i32, _p, _p, _p],
    "cf_knnfield_brick_unpack": [_p, _p, _i32, _p, _p],
    "cf_lbs_forward": [_p, _i32, _p, _p, _i64, _p, _p],
    "cf_lbs_vertex_transforms": [_p, _i32, _p, _i64, _p, _p, _p],
    "cf_lbs_setup": [_p, _i32, _p, _p, _i64, _p, _p, _p, _p, _p],
    "cf_lbs_backward": [_p, _p, _p, _i64, _f64, _p, _i64, _p, _p, _p, _p],
    "cf_hashgrid_init": [ctypes.POINTER(HashGridDesc), _i32, _i32, _i32, _i32, _i32],
    "cf_hashgrid_encode": [ctypes.POINTER(HashGridDesc), _p, _p, _i64, _p, _p],
    "cf_hashgrid_encode_bwd": [ctypes.POINTER(HashGridDesc), _p, _p, _i64, _p, _p],
    "cf_hashgrid_indices": [ctypes.POINTER(HashGridDesc), _p, _i64, _p, _p, _p],
    "cf_mlp_forward": [_i32, ctypes.POINTER(_i32), _p, _i32, _p, ctypes.POINTER(_i32), _p, _i64, _p, _p],
    "cf_camera_rays": [_P(Camera), _p, _p],
    "cf_occ_from_points": [_p, _P(OccGrid), _f64, _p, _p],
    "cf_occ_box_shell": [_P(OccGrid), _p, _f64, _p, _p],
    "cf_occ_splat": [_p, _P(OccGrid), _p, _p, _i32, _f64, _P(OccGrid), _p, _p],
    "cf_march": [_P(MarchDesc), _p, _p, _p, _P(MarchOut), _P(MarchOut), _p],
    "cf_rays_march": [_P(Camera), _P(MarchDesc), _p, _p, _p, _P(MarchOut), _P(MarchOut), _p],
    "cf_composite_final": [_P(MarchDesc), _P(MarchOut), _p, ctypes.c_float, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p],
    "cf_occ_bbox": [_p, _P(OccGrid), _p, _p],
    "cf_occ_cache": [_p, _P(OccGrid), _p, _i32, _f64, _i64, _p, _p, _p, _p, _p],
    "cf_occ_splat_cached": [_p, _p, _p, _p, _i64, _i32, _p, _P(OccGrid), _P(OccGrid), _p, _p, _p, _p],
    "cf_human_canon": [_P(MarchDesc), _p, _P(MarchOut), _P(HumanWarp), _p, _p, _p, _p],
    "cf_human_lbs_fallback": [_P(MarchDesc), _p, _P(MarchOut), _P(HumanWarp), _p, _i64, _p, _p, _p],
    "cf_object_canon": [_P(MarchDesc), _p, _P(MarchOut), _p, _p],
    "cf_composite": [_P(MarchDesc), _P(MarchOut), _p, ctypes.c_float, _p, _p, _p, _p],
    "cf_composite_layers": [_i64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p],
    "cf_field_forward": [_P(FieldDesc), _P(MarchOut), _p, _p, _p, _p, _p],
    "cf_field_scratch_bytes": [_P(FieldDesc), _i64, _P(_i64)],
    "cf_field_stage": [_P(FieldDesc), _P(MarchOut), _p, _p, _p, _p, _i32, _p],
    "cf_keyframe_rays": [_P(Camera), _p, _i64, _i64, ctypes.c_uint64, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p,
                         _p],
    "cf_train_sample": [_P(MarchDesc), _p, _p, _i32, _i32, _i32, _f64, ctypes.c_uint64, _p, _i64, _P(MarchOut), _p,
                        _p],
    "cf_loss_composite_bwd": [_P(MarchDesc), _P(MarchOut), _p, ctypes.c_float, _p, _p, _p, ctypes.c_float, _p, _p,
                              _p, _p],
    "cf_field_train_layout": [_i64, _p],
    "cf_compact_valid": [_P(MarchOut), _p, _P(MarchOut), _p, _p, _p, _p],
    "cf_scatter_rows": [_P(MarchOut), _p, _p, _p, _p],
    "cf_gather_rows": [_P(MarchOut), _p, _p, _p, _p],
    "cf_density_grid_update": [_P(HashGridDesc), _p, _p, _p, _i32, ctypes.c_float, ctypes.c_float, _i32, _p, _p, _p,
                               _p],
    "cf_dw_grouped": [_p, _i32, _p, _i64, _p],
    "cf_train_counts": [_p, _p, _p, _i64, _i32, _i64, _p, _p],
    "cf_train_norms": [_p, _i32, _p, _p, _p, _p, _p, _p],
    "cf_dw_pose_cols": [_p, _i32, _i32, _i32, _p, _i32, _p, _i32, _p],
    "cf_adam_multi": [_p, _i32, ctypes.c_float, ctypes.c_float, ctypes.c_float, _p, _p, _p],
    "cf_pack_multi": [_p, _i32, _p],
    "cf_color_backward": [_P(FieldDesc), _p, _P(MarchOut), _p, _p, _p, _p, _P(ColorBwdIO), _p],
    "cf_field_hash_backward": [_P(FieldDesc), _P(MarchOut), _p, _p, _p, _p, _p, _p],
    "cf_deform_backward": [_P(FieldDesc), _p, _P(MarchOut), _p, _p, _P(DeformBwdIO), _p],
    "cf_deform_hash_backward": [_P(FieldDesc), _P(MarchOut), _p, _p, _p, _p],
    "cf_adam": [_p, _p, _p, _p, _i64, ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float, _i32,
                ctypes.c_float, _p],
    "cf_pack_weight": [_p, _i32, _i32, _p, _p],
    "cf_pack_weight_split": [_p, _i32, _i32, _p, _p, _p],
    "cf_gemm_kmajor_f16": [_p, _i64, _p, _i64, _i32, _i64, _p, _i32, _p],
    "cf_store_to_host": [_p, _p, _i64, _i32, _p],
    "cf_load_from_host": [_p, _p, _i64, _p],
    "cf_copy_batch": [_P(CopyList), _p],
    "cf_mp_scan": [ctypes.c_char_p, _P(MpInfo)],
    "cf_mp_read": [ctypes.c_char_p, _i64, _i64, _p, _p, _p, _p, _p],
    "cf_mp_write": [ctypes.c_char_p, _i32, _i32, _i32, _i64, _p, _p, _p, _p, _p],
    "cf_skinning_transforms": [_p, _i64, _p, _p, _i32, _p, _p],
    "cf_pose_bias": [_p, _i32, _i32, _i32, _p, _i32, _p, _p],
    "cf_blur_score": [_p, _i32, _i32, _p, _p, _p],
    "cf_visibility_map": [_p, _i32, _p, _i32, _i32, _P(VisCamera), ctypes.c_double, _p, _p],
    "cf_pool_scan": [_P(PoolDesc), _P(PoolEntry), _p, _p, _p],
    "cf_tsdf_integrate": [_P(TsdfDesc), _p, _i32, _i32, _p, _P(Rigid), _P(Rigid), _P(Pinhole), _p],
    "cf_tsdf_sample": [_P(TsdfDesc), _p, _i64, _p, _p, _p, _p],
    "cf_tsdf_raycast": [_P(TsdfDesc), _P(Pinhole), _P(Rigid), _P(Rigid), _p, _i32, ctypes.c_double, ctypes.c_double,
                        ctypes.c_double, _p, _p, _p, _p],
    "cf_tsdf_crossings": [_P(TsdfDesc), _i32, _p, _p, _p],
    "cf_pcg_workspace_doubles": [_i32, _i32, _P(ctypes.c_int64)],
    "cf_depth_normals": [_p, _i32, _i32, _P(Pinhole), _P(Rigid), _p, _p],
    "cf_rigid_transform": [_p, _p, _i64, _P(Rigid), _p, _p, _p],
    "cf_lbs_theta_jacobian": [_p, _i32, _i32, _p, _p, _i64, ctypes.c_double, _p, _p],
    "cf_nr_warp": [_p, _p, _p, _i32, _p, _p, _i64, _p, _p, _p],
    "cf_nr_terms": [_P(NrSystem), _p],
    "cf_nr_step": [_p, _p, _i32, _p, _p],
    "cf_icp_residuals": [_p, _p, _p, _p, _i64, _p, _p],
    "cf_icp_normal_equations": [_p, _p, _p, _p, _i64, ctypes.c_double, _p, _p],
    "cf_find_correspondences": [_p, _p, _i64, _p, _i32, _i32, _p, _p, _P(Pinhole), _P(Rigid), _P(Rigid),
                                ctypes.c_double, ctypes.c_double, _p, _p, _p, _p],
    "cf_pcg_solve": [_P(Csr), _P(Csr), _p, ctypes.c_double, _i32, ctypes.c_double, _p, _p, _p, _p],
}

_lock = threading.Lock()
_lib = None


def lib():
    """Load the library (once). Raises if it was not built or CUDA is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"capfields_b200 CUDA library not built ({LIB_PATH}); run `python -m paper_2304_03184_b200.build`"
            )
        handle = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(handle, name, None)
            if fn is None:
                continue
            fn.argtypes = args
            fn.restype = ctypes.c_int
        handle.cf_last_error.restype = ctypes.c_char_p
        handle.cf_last_error.argtypes = []
        _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS.keys()) + ["cf_version", "cf_last_error"]


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("capfields_b200 needs a CUDA device (sm_100a); there is no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def check(rc: int, what: str = "") -> None:
    if rc == CF_OK:
        return
    msg = lib().cf_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == CF_E_OUT_OF_SUPPORT:
        raise OutOfSupportError(text)
    if rc == CF_E_DEGENERATE:
        raise DegenerateWeightsError(text)
    if rc == CF_E_FORMAT:
        raise RecordFormatError(msg)
    if rc in (CF_E_BAD_ARG, CF_E_DUPLICATE_FRAME):
        raise ValueError(msg)
    raise RuntimeError(text)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def ptr(t) -> int | None:
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()

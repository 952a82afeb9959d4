"""ctypes binding of include/latmap_b200.h (liblatmap_b200.so).

This is the reference-side FFI a Python caller binds; INTEGRATION.md shows the
equivalent C++ / ctypes stubs. Loading fails loudly when the library is missing:
there is no CPU fallback in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblatmap_b200.so")

OK, EINVAL, ESTALE, ECUDA, ENOMEM, EUNSUPPORTED = range(6)


class LatmapError(RuntimeError):
    pass


class InvalidArgument(LatmapError, ValueError):
    """std::invalid_argument in the reference."""


class StaleCache(LatmapError):
    """std::runtime_error for stale render / attention caches (render.cpp:256-260)."""


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32)]


class Pose(C.Structure):
    _fields_ = [("rotation", C.c_float * 4), ("translation", C.c_float * 3)]


class MapView(C.Structure):
    _fields_ = [("n", C.c_int64), ("query_dim", C.c_int32)] + [
        (f, C.c_void_p) for f in ("positions", "rotations", "colors", "log_scales", "opacity_logits", "features")]


class ProjectedSplat(C.Structure):
    _fields_ = [("mean2d", C.c_float * 2), ("cov_inv", C.c_float * 4), ("depth", C.c_float), ("alpha", C.c_float),
                ("source", C.c_int32), ("x0", C.c_int32), ("x1", C.c_int32), ("y0", C.c_int32), ("y1", C.c_int32)]


class LossBreakdown(C.Structure):
    _fields_ = [(f, C.c_float) for f in ("l_rgb", "l_ssim", "l_depth", "l_cos", "l_l2", "l_trust", "total")] + [
        ("supervised_rows", C.c_int64), ("depth_empty", C.c_int32), ("zero_norm_flagged", C.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


CONFIG_FLOATS = ("lambda_cos", "lambda_l2", "lambda_trust", "trust_delta", "lambda_i1", "lambda_i2", "lambda_rgb",
                 "lambda_depth", "lambda_feat", "lr_proj", "lr_dict", "lr_position", "lr_rotation", "lr_color",
                 "lr_log_scale", "lr_opacity", "lr_feature", "scene_extent", "softmax_temp")


class Config(C.Structure):
    _fields_ = [(f, C.c_float) for f in CONFIG_FLOATS] + [
        ("dict_learn", C.c_int32), ("segment_mode", C.c_int32), ("decoder_precision", C.c_int32)]


class Frame(C.Structure):
    _fields_ = [("pose", Pose), ("rgb", C.c_void_p), ("depth", C.c_void_p), ("assignment", C.c_void_p),
                ("features", C.c_void_p), ("n_set", C.c_int64)]


class PipelineConfig(C.Structure):
    """latmap_pipeline_config: the pipeline-level subset of latmap::Config (config.hpp:10-58)."""
    _fields_ = [("query_dim", C.c_int32), ("embed_dim", C.c_int32), ("dict_size", C.c_int32),
                ("stage1_iters", C.c_int32), ("stage2_iters", C.c_int32), ("history_sample", C.c_int32),
                ("history_capacity", C.c_int32), ("voxel_size", C.c_float), ("local_radius", C.c_float),
                ("sync_distance", C.c_float), ("hash_capacity", C.c_int64), ("local_mapping", C.c_int32),
                ("keyframe_stride", C.c_int32), ("seed", C.c_uint64), ("dict_init", C.c_int32),
                ("dict_decay", C.c_float), ("trust_anchor_persistent", C.c_int32)]


SYNC_FIELDS = ("written_back", "newborn_inserted", "newborn_rejected", "pruned", "fetched")


class KeyframeLog(C.Structure):
    """KeyframeLog (pipe/pipeline.hpp:70-80)."""
    _fields_ = [("frame_index", C.c_int32), ("loss", LossBreakdown), ("seeded", C.c_int64),
                ("active_count", C.c_int64), ("global_count", C.c_int64), ("dict_weight_mass", C.c_double),
                ("synced", C.c_int32), ("sync", C.c_int64 * 5), ("wall_ms", C.c_double)]

    def as_dict(self):
        return {"frame_index": self.frame_index, "loss": self.loss.as_dict(), "seeded": self.seeded,
                "active_count": self.active_count, "global_count": self.global_count,
                "dict_weight_mass": self.dict_weight_mass, "synced": bool(self.synced),
                "sync": dict(zip(SYNC_FIELDS, list(self.sync))), "wall_ms": self.wall_ms}


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() (no CPU fallback exists)")
        _lib = C.CDLL(os.environ.get("LATMAP_LIB", LIB_PATH))  # override: experiment builds only
        _declare(_lib)
    return _lib


def _declare(L):
    P = C.c_void_p
    st = C.c_int
    sig = {
        "latmap_ctx_create": [C.c_int32, P, C.POINTER(P)],
        "latmap_ctx_destroy": [P],
        "latmap_ctx_set_stream": [P, P],
        "latmap_ctx_synchronize": [P],
        "latmap_ctx_set_exact_blend": [P, C.c_int32],
        "latmap_ctx_set_decoder_path": [P, C.c_int32],
        "latmap_ctx_set_reconstruct_precision": [P, C.c_int32],
        "latmap_project_gaussian": [P, P, P, P, C.c_float, C.POINTER(Pose), C.POINTER(Intrinsics),
                                    C.POINTER(C.c_int32), P, P, P],
        "latmap_render_cache_create": [P, C.POINTER(P)],
        "latmap_render_cache_destroy": [P],
        "latmap_render": [P, C.POINTER(MapView), C.POINTER(Pose), C.POINTER(Intrinsics), P, P, P, P, P],
        "latmap_render_backward": [P, C.POINTER(MapView), C.POINTER(Pose), C.POINTER(Intrinsics), P, P, P, P,
                                   C.POINTER(MapView)],
        "latmap_render_cache_splats": [P, P, P, C.c_int64, C.POINTER(C.c_int64)],
        "latmap_render_cache_tiles": [P, P, P, P, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int64)],
        "latmap_reconstruct": [P, P, C.c_int64, C.c_int32, P, P, C.c_int64, C.c_int32, C.c_float, P, P],
        "latmap_reconstruct_backward": [P, P, P, C.c_int64, C.c_int32, P, P, C.c_int64, C.c_int32, C.c_float, P, P,
                                        P, P],
        "latmap_trust_region_penalty": [P, P, P, C.c_int64, C.c_int32, C.c_float, P, C.POINTER(C.c_float)],
        "latmap_ssim": [P, P, P, C.c_int32, C.c_int32, C.c_int32, P, C.POINTER(C.c_float)],
        "latmap_adam_step": [P, P, P, P, P, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_float,
                             C.POINTER(C.c_int32)],
        "latmap_session_create": [P, C.POINTER(Config), C.c_int64, C.c_int32, C.c_int64, C.c_int32,
                                  C.POINTER(Intrinsics), C.POINTER(P)],
        "latmap_session_destroy": [P],
        "latmap_session_set_map": [P, P, P, P, P, P, P],
        "latmap_session_get_map": [P, P, P, P, P, P, P],
        "latmap_session_set_dictionary": [P, P, P, P],
        "latmap_session_get_dictionary": [P, P, P],
        "latmap_session_get_anchor": [P, P],
        "latmap_session_set_frames": [P, C.c_int32, C.POINTER(Frame)],
        "latmap_session_set_batch": [P, C.c_int32, C.c_int32],
        "latmap_session_set_slot_offset": [P, C.c_int32],
        "latmap_session_objective": [P, C.c_int32, C.POINTER(LossBreakdown)],
        "latmap_session_apply": [P],
        "latmap_session_step": [P, C.POINTER(LossBreakdown)],
        "latmap_session_objective_ex": [P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(LossBreakdown)],
        "latmap_session_step_dict": [P, C.POINTER(LossBreakdown)],
        "latmap_session_set_graphs": [P, C.c_int32],
        "latmap_session_seed_candidates": [P, C.c_int32, P, C.c_int64, C.POINTER(C.c_int64)],
        "latmap_session_append_rows": [P, P, C.c_int64, P],
        "latmap_session_export_rows": [P, P],
        "latmap_session_import_rows": [P, P, C.c_int64, P, C.c_int64],
        "latmap_session_import_rows_device": [P, P, C.c_int64, P, C.c_int64],
        "latmap_session_read_loss_async": [P, P, C.c_int64, C.POINTER(C.c_int64)],
        "latmap_session_grad_buffer": [P, C.POINTER(P), C.POINTER(C.c_int64)],
        "latmap_session_loss_buffer": [P, C.POINTER(P), C.POINTER(C.c_int64)],
        "latmap_session_read_loss": [P, C.POINTER(LossBreakdown)],
        "latmap_session_frame_images": [P, C.c_int32, C.POINTER(P), C.POINTER(P), C.POINTER(P), C.POINTER(P)],
        "latmap_session_stats": [P, P, P],
        "latmap_session_profile": [P, C.c_int32],
        "latmap_session_set_parity_export": [P, C.c_int32],
        "latmap_session_decoder_export": [P, C.POINTER(C.c_int32), C.POINTER(C.c_int64), P, P],
        "latmap_selftest_umma": [P, P, P, P, C.c_int32, C.c_int32, C.c_int32, C.c_int32],
        "latmap_selftest_expf": [P, C.c_uint64, C.c_int64, P],
        "latmap_device_alloc": [P, C.c_int64, C.POINTER(P)],
        "latmap_device_free": [P, P],
        "latmap_copy": [P, P, P, C.c_int64, C.c_int32],
        "latmap_rgb_loss": [P, P, P, C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_float, P, P, P, P],
        "latmap_depth_loss": [P, P, P, P, C.c_int64, P, P, P],
        "latmap_feature_loss": [P, P, P, C.c_int64, C.c_int32, P, P, C.c_int64, C.c_float, C.c_float, C.c_float,
                                C.c_float, P, P, P, P],
        "latmap_weighted_kmeans": [P, P, P, C.c_int64, C.c_int32, C.c_int64, P, P, P, C.c_int64, C.c_int32, P, P,
                                   C.POINTER(C.c_int32)],
        "latmap_session_stream_kmeans": [P, P, C.c_int64, C.c_float, P, P],
        "latmap_session_get_dict_weights": [P, P],
        "latmap_gather_supervision": [P, P, C.c_int32, P, C.c_int64, P, C.c_int32, C.c_int32, P, P, P, C.c_int64,
                                      C.POINTER(C.c_int64)],
        "latmap_metric_cos": [P, P, P, C.c_int64, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int32)],
        "latmap_metric_miou": [P, P, P, C.c_int64, C.c_int32, P, C.c_int32, P, P, C.POINTER(C.c_double)],
        "latmap_metric_psnr": [P, P, P, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int32)],
        "latmap_query_map": [P, P, C.c_int64, C.c_int32, P, P, C.c_int64, C.c_int32, C.c_float, P, P],
        "latmap_session_set_dict_weights": [P, P],
        "latmap_store_create": [P, C.c_int64, C.c_int32, C.POINTER(P)],
        "latmap_store_destroy": [P],
        "latmap_store_get_records": [P, C.c_int64, C.c_int64, P, P],
        "latmap_store_insert_global": [P, P, C.c_int64, C.c_float, C.POINTER(C.c_int64)],
        "latmap_store_insert_keyed": [P, P, P, C.c_int64, C.POINTER(C.c_int64)],
        "latmap_comm_unique_id": [P, P],
        "latmap_comm_init": [P, C.c_int32, C.c_int32, P, C.POINTER(P)],
        "latmap_comm_destroy": [P],
        "latmap_comm_allreduce": [P, P, C.c_int64, C.c_int32],
        "latmap_session_allreduce": [P, P],
        "latmap_loss_assemble": [P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(Config), C.POINTER(LossBreakdown)],
        "latmap_session_check_overflow": [P, C.POINTER(C.c_int32)],
        "latmap_session_grad_layout": [P, P, P],
        "latmap_session_shard_range": [P, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
        "latmap_session_shard_check": [P, C.c_int64, C.c_int64],
        "latmap_session_apply_range": [P, C.c_int64, C.c_int64],
        "latmap_session_params_buffer": [P, C.POINTER(P), C.POINTER(C.c_int64)],
        "latmap_session_exchange_sharded": [P, P],
        "latmap_session_save_state": [P],
        "latmap_ctx_set_deterministic": [P, C.c_int32],
        "latmap_session_restore_state": [P],
        "latmap_pipeline_inject_fault": [P, C.c_int32],
        "latmap_session_overflow_steps": [P, C.POINTER(C.c_int64)],
        "latmap_pipeline_create": [P, C.POINTER(Config), C.POINTER(PipelineConfig), C.POINTER(Intrinsics),
                                   C.POINTER(P)],
        "latmap_pipeline_destroy": [P],
        "latmap_pipeline_process_keyframe": [P, C.POINTER(Frame), C.c_int32, C.POINTER(KeyframeLog)],
        "latmap_pipeline_flush": [P, P],
        "latmap_pipeline_state": [P, P],
        "latmap_pipeline_active_set": [P, P, P],
        "latmap_store_fetch_local": [P, P, C.c_float, P, C.c_int64, C.POINTER(C.c_int64), P],
        "latmap_store_sync": [P, P, P, P, C.c_int64, P, C.c_float, C.c_float, P, P, C.c_int64, P, P,
                              C.POINTER(C.c_int64)],
        "latmap_store_fetch_local_device": [P, P, C.c_float, P, C.c_int64, P, C.POINTER(C.c_int64)],
        "latmap_store_sync_device": [P, P, P, P, C.c_int64, P, C.c_float, C.c_float, P, P, C.c_int64, P, P,
                                     C.POINTER(C.c_int64)],
        "latmap_session_phase_times": [P, P, P],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = st
    L.latmap_ctx_last_error.argtypes = [P]
    L.latmap_ctx_last_error.restype = C.c_char_p
    L.latmap_ctx_launch_count.argtypes = [P]
    L.latmap_ctx_launch_count.restype = C.c_int64
    L.latmap_default_config.argtypes = [C.POINTER(Config)]
    L.latmap_default_config.restype = None
    L.latmap_ctx_stream.argtypes = [P]
    L.latmap_ctx_stream.restype = P
    L.latmap_voxel_of.argtypes = [P, C.c_float, P]
    L.latmap_voxel_of.restype = None
    L.latmap_hash_voxel.argtypes = [P, C.c_int64]
    L.latmap_hash_voxel.restype = C.c_int64
    L.latmap_store_size.argtypes = [P]
    L.latmap_store_size.restype = C.c_int64
    L.latmap_store_stats.argtypes = [P, P]
    L.latmap_store_stats.restype = None
    L.latmap_store_last_error.argtypes = [P]
    L.latmap_store_last_error.restype = C.c_char_p
    L.latmap_store_insert.argtypes = [P, P, P]
    L.latmap_store_insert.restype = C.c_int64
    L.latmap_store_update.argtypes = [P, P, P]
    L.latmap_store_update.restype = C.c_int32
    L.latmap_store_find.argtypes = [P, P]
    L.latmap_store_find.restype = C.c_int64
    L.latmap_session_size.argtypes = [P]
    L.latmap_session_size.restype = C.c_int64
    L.latmap_default_pipeline_config.argtypes = [C.POINTER(PipelineConfig)]
    L.latmap_default_pipeline_config.restype = None
    L.latmap_select_keyframe.argtypes = [C.c_int32, C.c_int32]
    L.latmap_select_keyframe.restype = C.c_int32
    L.latmap_pipeline_session.argtypes = [P]
    L.latmap_pipeline_session.restype = P
    L.latmap_pipeline_store.argtypes = [P]
    L.latmap_pipeline_store.restype = P
    L.latmap_pipeline_last_error.argtypes = [P]
    L.latmap_pipeline_last_error.restype = C.c_char_p


EXPORTED = ["latmap_ctx_create", "latmap_ctx_destroy", "latmap_ctx_set_stream", "latmap_ctx_synchronize",
            "latmap_ctx_set_exact_blend", "latmap_ctx_set_decoder_path", "latmap_ctx_set_reconstruct_precision",
            "latmap_ctx_last_error", "latmap_ctx_launch_count", "latmap_default_config", "latmap_project_gaussian",
            "latmap_render_cache_create", "latmap_render_cache_destroy", "latmap_render", "latmap_render_backward",
            "latmap_render_cache_splats", "latmap_render_cache_tiles", "latmap_reconstruct",
            "latmap_reconstruct_backward", "latmap_trust_region_penalty", "latmap_ssim", "latmap_adam_step",
            "latmap_session_create", "latmap_session_destroy", "latmap_session_set_map", "latmap_session_get_map",
            "latmap_session_set_dictionary", "latmap_session_get_dictionary", "latmap_session_get_anchor", "latmap_session_set_frames",
            "latmap_session_set_batch", "latmap_session_set_slot_offset", "latmap_session_objective",
            "latmap_session_apply", "latmap_session_step", "latmap_session_objective_ex", "latmap_session_step_dict",
            "latmap_session_export_rows", "latmap_session_import_rows", "latmap_session_import_rows_device", "latmap_session_read_loss_async",
            "latmap_session_size",
            "latmap_session_set_graphs", "latmap_session_seed_candidates", "latmap_session_append_rows",
            "latmap_session_grad_buffer", "latmap_session_loss_buffer",
            "latmap_session_read_loss", "latmap_session_frame_images", "latmap_session_stats",
            "latmap_session_profile", "latmap_session_phase_times", "latmap_session_set_parity_export",
            "latmap_session_decoder_export", "latmap_selftest_umma", "latmap_selftest_expf", "latmap_rgb_loss", "latmap_depth_loss", "latmap_device_alloc",
            "latmap_device_free", "latmap_copy",
            "latmap_feature_loss", "latmap_ctx_stream",
            "latmap_voxel_of", "latmap_hash_voxel", "latmap_store_create", "latmap_store_destroy", "latmap_store_size",
            "latmap_store_stats", "latmap_store_last_error", "latmap_store_insert", "latmap_store_update",
            "latmap_store_find", "latmap_store_get_records", "latmap_store_insert_global", "latmap_store_insert_keyed", "latmap_store_fetch_local",
            "latmap_store_sync", "latmap_store_sync_device", "latmap_store_fetch_local_device", "latmap_weighted_kmeans", "latmap_session_stream_kmeans",
            "latmap_session_get_dict_weights", "latmap_session_set_dict_weights", "latmap_gather_supervision",
            "latmap_metric_cos", "latmap_metric_miou", "latmap_metric_psnr", "latmap_query_map",
            "latmap_default_pipeline_config", "latmap_select_keyframe", "latmap_pipeline_create",
            "latmap_pipeline_destroy", "latmap_pipeline_process_keyframe", "latmap_pipeline_flush",
            "latmap_pipeline_session", "latmap_pipeline_store", "latmap_pipeline_state", "latmap_pipeline_active_set",
            "latmap_pipeline_last_error", "latmap_comm_unique_id", "latmap_comm_init",
            "latmap_comm_destroy", "latmap_comm_allreduce", "latmap_session_allreduce", "latmap_loss_assemble",
            "latmap_session_check_overflow", "latmap_session_overflow_steps", "latmap_session_grad_layout",
            "latmap_session_shard_range", "latmap_session_shard_check", "latmap_session_apply_range",
            "latmap_session_params_buffer", "latmap_session_exchange_sharded", "latmap_session_save_state",
            "latmap_session_restore_state", "latmap_pipeline_inject_fault", "latmap_ctx_set_deterministic"]


def check(ctx_handle, status):
    if status == OK:
        return
    msg = lib().latmap_ctx_last_error(ctx_handle)
    msg = msg.decode() if msg else ""
    if status == EINVAL:
        raise InvalidArgument(msg)
    if status == ESTALE:
        raise StaleCache(msg)
    raise LatmapError(f"latmap status {status}: {msg}")

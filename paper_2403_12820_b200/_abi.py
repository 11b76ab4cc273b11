"""ctypes view of the C-ABI in include/stencilcloth_b200.h.

The shared library ``libstencilcloth_b200.so`` (built in-tree by ``__graft_entry__.build()``
from ``paper_2403_12820_b200/csrc``) is the only compute path: there is no CPU fallback, and
loading fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SC_B200_LIB") or os.path.join(_HERE, "libstencilcloth_b200.so")

SC_OK, SC_ERR_CONFIG, SC_ERR_NUMERICS, SC_ERR_CUDA, SC_ERR_STATE = 0, 1, 2, 3, 4
SC_F32, SC_F64 = 0, 1
SC_MODE_PARITY, SC_MODE_FAST = 0, 1
CHANNELS = 12


class sc_params(C.Structure):
    _fields_ = [
        ("kernel_gain", C.c_double * CHANNELS),
        ("linear_w", C.c_double * CHANNELS),
        ("linear_b", C.c_double * 3),
        ("nonlinear_w", C.c_double * CHANNELS),
        ("deriv_w", C.c_double * CHANNELS),
        ("self_velocity_w", C.c_double),
        ("isru_alpha", C.c_double),
    ]


class sc_train_config(C.Structure):
    """TrainConfig (train.hpp:16-53) as the C-ABI carries it."""
    _fields_ = [
        ("alpha", C.c_double),
        ("batch_size", C.c_int32),
        ("epochs", C.c_int32),
        ("schedule_kind", C.c_int32),
        ("lr0", C.c_double),
        ("gamma", C.c_double),
        ("interval", C.c_int32),
        ("floor", C.c_double),
        ("period", C.c_int32),
        ("seed", C.c_uint64),
        ("de_population", C.c_int32),
        ("de_generations", C.c_int32),
        ("de_bound", C.c_double),
        ("de_cross_prob", C.c_double),
        ("de_diff_weight", C.c_double),
        ("de_probe_batch", C.c_int32),
        ("checkpoint_interval", C.c_int32),
        ("freeze_mask", C.c_uint32),
    ]


class sc_adam_state(C.Structure):
    _fields_ = [("m", C.c_double * 53), ("v", C.c_double * 53), ("step", C.c_int64)]


class sc_peer_export(C.Structure):
    """sc_peer_export: a strip context's IPC handles / pointers for a neighbour to link."""
    _fields_ = [
        ("state_handle", (C.c_ubyte * 64) * 2),
        ("flags_handle", C.c_ubyte * 64),
        ("state_ptr", C.c_void_p * 2),
        ("flags_ptr", C.c_void_p),
        ("plane_stride", C.c_int64),
        ("g0", C.c_int32), ("u0", C.c_int32), ("u1", C.c_int32), ("nx", C.c_int32),
        ("pitch", C.c_int32), ("batch", C.c_int32), ("cur", C.c_int32), ("device", C.c_int32),
    ]


class sc_sphere(C.Structure):
    _fields_ = [("center", C.c_double * 3), ("radius", C.c_double), ("friction", C.c_double)]


class sc_plane(C.Structure):
    _fields_ = [("height", C.c_double), ("friction", C.c_double)]


class sc_cloth_desc(C.Structure):
    _fields_ = [
        ("dt", C.c_double),
        ("mass", C.c_double),
        ("drag", C.c_double),
        ("pressure", C.c_double),
        ("gravity", C.c_double * 3),
        ("plug_pressure", C.c_int32),
        ("plug_gravity", C.c_int32),
        ("plug_drag", C.c_int32),
        ("n_pins", C.c_int32),
        ("pin_nodes", C.POINTER(C.c_int32)),
        ("pin_anchors", C.POINTER(C.c_double)),
        ("pin_velocity", C.c_double * 3),
        ("n_spheres", C.c_int32),
        ("spheres", C.POINTER(sc_sphere)),
        ("n_planes", C.c_int32),
        ("planes", C.POINTER(sc_plane)),
        ("stiffness", C.c_double),
        ("damping", C.c_double),
        ("spacing", C.c_double),
    ]


class sc_scene_desc(C.Structure):
    _fields_ = [
        ("nx", C.c_int32),
        ("ny", C.c_int32),
        ("batch", C.c_int32),
        ("cloths", C.POINTER(sc_cloth_desc)),
    ]


# name -> (restype, argtypes); exactly the entry points declared in include/stencilcloth_b200.h
_P = C.c_void_p
_I = C.c_int32
SIGNATURES = {
    "sc_abi_version": (C.c_int, []),
    "sc_last_error": (C.c_char_p, []),
    "sc_ctx_create": (C.c_int, [C.c_int, C.c_int, C.POINTER(_P)]),
    "sc_ctx_destroy": (None, [_P]),
    "sc_ctx_set_scene": (C.c_int, [_P, C.POINTER(sc_scene_desc)]),
    "sc_ctx_set_params": (C.c_int, [_P, C.POINTER(sc_params)]),
    "sc_ctx_set_state": (C.c_int, [_P, _P, _P]),
    "sc_ctx_get_state": (C.c_int, [_P, _P, _P]),
    "sc_ctx_advance": (C.c_int, [_P, _I, _I, C.c_int]),
    "sc_ctx_sync": (C.c_int, [_P]),
    "sc_ctx_set_health_checks": (C.c_int, [_P, _I]),
    "sc_ctx_set_persistent": (C.c_int, [_P, _I]),
    "sc_ctx_get_health": (C.c_int, [_P, _P, _P, _P]),
    "sc_rollout": (C.c_int, [_P, _P, _P, _I, _I, C.c_int, _P, _P, _P]),
    "sc_rollout_frames": (C.c_int, [_P, _P, _P, _I, _I, C.c_int, _P, _P]),
    "sc_forward_impulse": (C.c_int, [_P, _P, _P, _P]),
    "sc_plug_impulse": (C.c_int, [_P, _P, _P, _P]),
    "sc_advance_with_impulse": (C.c_int, [_P, _P, _P, _P, C.c_double, _P, _P, _P]),
    "sc_nn_step": (C.c_int, [_P, _P, _P, C.c_double, C.c_int, _P, _P, _P]),
    "sc_benchmark": (C.c_int, [_P, _I, _I, C.c_int, C.POINTER(C.c_double)]),
    "sc_total_impulse": (C.c_int, [_P, _P, _P, _P]),
    "sc_pbs_step": (C.c_int, [_P, _P, _P, C.c_double, _P, _P, _P]),
    "sc_simulate_frames": (C.c_int, [_P, _P, _P, _I, _I, _P, _P]),
    "sc_benchmark_sim": (C.c_int, [_P, _I, _I, C.POINTER(C.c_double)]),
    "sc_total_force": (C.c_int, [_P, _P, _P, _P]),
    "sc_evaluate_frames": (C.c_int, [C.c_int, _P, _P, _I, C.c_int64, _P]),
    "sc_eval_last_error": (C.c_char_p, []),
    "sc_trainer_create": (C.c_int, [C.c_int, _P, _I, _P, _P, C.POINTER(_P)]),
    "sc_trainer_destroy": (None, [_P]),
    "sc_trainer_sample_batch": (C.c_int, [_P, _I, C.c_uint64, _P, _P]),
    "sc_trainer_set_batch": (C.c_int, [_P, _P, _I]),
    "sc_sample_indices": (C.c_int, [_I, _I, C.c_uint64, _P]),
    "sc_trainer_compute_loss": (C.c_int, [_P, C.POINTER(sc_params), C.c_double, _P, _P]),
    "sc_trainer_run": (C.c_int, [_P, C.POINTER(sc_train_config), C.POINTER(sc_params), _P,
                                 C.POINTER(sc_adam_state), C.POINTER(sc_params), _P, _P, _P]),
    "sc_trainer_part_forward": (C.c_int, [_P, C.POINTER(sc_params), _I, _I, _P, _P]),
    "sc_trainer_part_chain": (C.c_int, [_P, _P, _P, _P]),
    "sc_trainer_part_backward": (C.c_int, [_P, C.POINTER(sc_params), C.c_double, C.c_uint64, _I,
                                           _P]),
    "sc_trainer_diagnose_forward": (C.c_int, [_P, C.POINTER(sc_params), _I, _I, C.c_char_p, _I]),
    "sc_backward_gradients": (C.c_int, [C.c_int, _I, _I, _P, _P, C.POINTER(sc_params), _P, _P]),
    "sc_benchmark_launches": (C.c_int, [_P, _I, _I, C.c_int, _P]),
    "sc_ctx_set_strip": (C.c_int, [_P, _I, _I]),
    "sc_ctx_halo_elems": (C.c_int64, [_P]),
    "sc_ctx_halo_pack": (C.c_int, [_P, _I, _P, _P]),
    "sc_ctx_halo_unpack": (C.c_int, [_P, _I, _P, _P]),
    "sc_ctx_strip_step": (C.c_int, [_P, _I, _I, _I, C.c_int, _P]),
    "sc_ctx_strip_commit": (C.c_int, [_P]),
    "sc_ctx_peer_export": (C.c_int, [_P, C.POINTER(sc_peer_export)]),
    "sc_ctx_set_peer": (C.c_int, [_P, _I, C.POINTER(sc_peer_export), _I]),
    "sc_ctx_peer_step": (C.c_int, [_P, _I, C.c_int, _P]),
    "sc_ctx_stream": (_P, [_P]),
    "sc_ctx_state_buffers": (
        C.c_int,
        [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(C.c_int64), C.POINTER(_I), C.POINTER(_I),
         C.POINTER(_I)],
    ),
    "sc_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(_P)]),
    "sc_host_free": (None, [_P]),
    "sc_ctx_launch_count": (C.c_int64, [_P]),
    # host-side seeded generators (csrc/host_gen.cpp)
    "sc_rng_mix": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "sc_mt64_fill": (None, [C.c_uint64, C.c_int64, _P]),
    "sc_rng_uniform01": (None, [C.c_uint64, C.c_int64, _P]),
    "sc_rng_normal": (None, [C.c_uint64, C.c_int64, C.c_double, _P]),
    "sc_gen_sheet": (
        None,
        [C.c_uint64, C.c_int64, _I, _I, _I, _I, C.c_double, C.c_double, _P, _P, _I],
    ),
}

_lib = None


def load(path: str | None = None) -> C.CDLL:
    """Load (once) and type the C-ABI library. Raises ImportError if it is not built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(
            f"{p} is missing: the CUDA extension is not built (run __graft_entry__.build()); "
            "there is no CPU fallback for this path"
        )
    lib = C.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib

"""B200-native network-cell rollout step of the arXiv 2403.12820 reference (`stencilcloth`).

Public surface mirrors the reference's Python binding for this path
(/root/reference/proj/python/stencilcloth/__init__.py:3-28, bindings.cpp:147-164):
Scene / NetworkParams / Trajectory types, parse_scene / load_scene, forward_impulse, rollout,
plus the other per-operator calls of the path and the batched f32 engine ClothBatch.
All compute runs in libstencilcloth_b200.so (sm_100a); importing fails loudly without it.
"""
from . import _abi

_abi.load()  # no CPU fallback: the CUDA extension must be present

from .scene import (BoundarySpec, ConfigError, GridPlane, IoError, MaterialParams,  # noqa: E402
                    NetworkParams, NumericsError, ParamGroup, PlaneCollider, PlugForce, Scene,
                    SphereCollider, Trajectory, build_grid, channel_order_hash, load_scene,
                    params_fingerprint, parse_scene)
from .api import (BenchResult, ClothBatch, Context, CudaError, advance_with_impulse,  # noqa: E402
                  apply_dirichlet, benchmark_net, benchmark_sim, forward_impulse, nn_step,
                  pinned_empty, plug_impulse, rollout, simulate, step_semi_implicit,
                  total_force, total_impulse)
from .training import (AdamState, DeConfig, LossRow, LossValue, ParamGradients,  # noqa: E402
                    ScheduleConfig, ScheduleKind, TrainConfig, Trainer, TrainResult,
                    backward_gradients, gradient_check, sample_indices, train,
                       train_loop)
from .dist_train import CudaPart, DistributedTrainer  # noqa: E402
from .trajio import (Checkpoint, EvalReport, evaluate, export_obj, load_checkpoint,  # noqa: E402
                     load_trajectory, save_checkpoint, save_trajectory, write_eval_csv,
                     write_loss_csv)

__all__ = [
    "BenchResult", "BoundarySpec", "ClothBatch", "ConfigError", "Context", "CudaError",
    "GridPlane", "IoError", "MaterialParams", "NetworkParams", "NumericsError", "ParamGroup",
    "PlaneCollider", "PlugForce", "Scene", "SphereCollider", "Trajectory", "advance_with_impulse",
    "apply_dirichlet", "benchmark_net", "build_grid", "channel_order_hash", "forward_impulse",
    "load_scene", "nn_step", "params_fingerprint", "parse_scene", "plug_impulse", "rollout",
    "benchmark_sim", "simulate", "step_semi_implicit", "total_force", "total_impulse",
    "EvalReport", "evaluate", "export_obj", "load_trajectory", "pinned_empty", "save_trajectory",
    "write_eval_csv", "Checkpoint", "load_checkpoint", "save_checkpoint", "write_loss_csv",
    "AdamState", "CudaPart", "DistributedTrainer", "DeConfig", "LossRow", "LossValue", "ParamGradients",
    "ScheduleConfig", "ScheduleKind", "TrainConfig", "Trainer", "TrainResult",
    "backward_gradients", "gradient_check", "sample_indices", "train", "train_loop",
]
__version__ = "0.1.0"

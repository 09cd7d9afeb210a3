"""B200-native FP64 matrix-free finite-element action (femgpu) — Python host binding."""
from .form import *  # noqa: F401,F403
from .action import (ExecutionOutcome, GpuInstance, TilingParams, device_count, emit_source, fp64_peak, fp64_peaks,  # noqa: F401
                     gpu_action, gpu_executor, jit_check, reference_counters)
from . import abi  # noqa: F401
from .mesh import CONFIGS, FUSED_PAIRS, color_cells, config_problem, fused_pair, mesh_problem, unit_mesh  # noqa: F401
from .io import load_instance, load_schedule, save_instance, save_schedule  # noqa: F401,E402
from .krylov import DeviceOperator, cg, symmetric_problem  # noqa: F401,E402
from .fuse import FusedOperator, fuse_problems, split_output  # noqa: F401,E402
from .reorder import inputs_to_new, output_to_original, reorder_problem  # noqa: F401,E402

"""B200-native CrossoverScheduler (arXiv 2103.07974).

Several data-parallel training apps share every GPU in a fixed rotation; one
app's fused-gradient synchronization (K1 pack -> bucket exchange over NVLink -- NCCL,
the fused P2P kernel, copy-engine pulls or NVSwitch multicast -> K2 fused average +
SGD update) runs on the comm stream while the next app's forward/backward occupies
the SMs.  The public API mirrors the reference
simulator (colosim, /root/reference/pkg/src/colosim/__init__.py:11-56): plans,
policies, traces, metrics -- backed by the device pipeline instead of a
discrete-event simulation.

Importing the package does not touch CUDA; the device pieces
(:mod:`.fusion`, :mod:`.scheduler`, :mod:`.equivalence`) load libcrossover.so
on first import and raise if it is missing (there is no CPU fallback).
"""

from .comm import (
    Architecture,
    ClusterSpec,
    SyncRequest,
    allreduce_bus_bytes,
    comm_comp_ratio,
    comm_time,
    comm_time_allreduce,
    comm_time_unfused,
)
from .engine import (
    EventKind,
    LaneKind,
    Phase,
    Span,
    Trace,
    schedule_key,
    trace_to_chrome_json,
    trace_to_json,
    validate_trace,
)
from .errors import ComparisonError, ConfigError, DeadlockError, InvalidTraceError
from .metrics import Metrics, compare, measure, metrics_from_json, report, samples_per_second
from .workload import (
    BucketLayout,
    FusedGradient,
    JobProfile,
    TensorSpec,
    comp_time,
    fuse_gradients,
    profile_from_module,
    tensor_specs_from_module,
    unfused_messages,
)

__version__ = "0.1.0"

_DEVICE_EXPORTS = {
    "Policy": "scheduler", "App": "scheduler", "SchedulePlan": "scheduler",
    "JobRuntimeState": "scheduler", "CrossoverScheduler": "scheduler",
    "simulate": "scheduler", "schedule_crossover": "scheduler",
    "schedule_sequential": "scheduler", "rotation_schedule": "scheduler",
    "steady_state_period": "scheduler", "predicted_speedup": "scheduler",
    "overlap_roofline": "scheduler",
    "SgdSettings": "fusion", "FusedGradientSync": "fusion", "flatten_parameters": "fusion",
    "NcclCommunicator": "comm", "PeerGroup": "comm",
    "RotationGraph": "graphs", "NvlsBuffer": "nvls",
}


def __getattr__(name):
    mod = _DEVICE_EXPORTS.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)

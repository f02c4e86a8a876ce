"""B200-native shared-prefix decode attention behind Parrot's engine API.

Drop-in for the data-parallel hot path of arXiv 2405.19888 (the reference
`semflow` package): `GpuEngine` mirrors `semflow.engine.Engine`; its block
table, forest and per-step work list live in libforkattn.so (C++), and its
decode step runs hand-written sm_100a kernels.
"""

from . import _lib
from .engine import (
    LLAMA_7B,
    LLAMA_13B,
    TINY,
    Context,
    ContextPlan,
    CostModel,
    Engine,
    FillTask,
    GenerationTask,
    GpuEngine,
    GpuKvStore,
    ModelGeometry,
    StepReport,
    SyntheticDecodeModel,
    TensorDecodeModel,
    engine_factory,
    format_ms,
    hash_token_ids,
)
from .errors import ContextBusy, KernelError, OutOfMemory, UnknownContext, UnknownParentContext

__all__ = [
    "GpuEngine", "Engine", "GpuKvStore", "CostModel", "Context", "ContextPlan", "FillTask",
    "GenerationTask", "StepReport", "ModelGeometry", "LLAMA_7B", "LLAMA_13B", "TINY",
    "SyntheticDecodeModel", "TensorDecodeModel", "engine_factory", "format_ms", "hash_token_ids",
    "OutOfMemory", "UnknownContext", "UnknownParentContext", "ContextBusy", "KernelError",
]

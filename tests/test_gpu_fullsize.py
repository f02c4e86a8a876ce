"""The benchmarked configurations, checked numerically at full depth.

bench.py times 40 (or 32) layers per step, replayed as one CUDA graph, with
partials double-buffered by launch parity, cross-layer PDL and decode growth
between steps.  These tests build the engine exactly as bench.py does
(bench.build_engine: synthetic prefill, model Q/K/V rows on the device,
reserved pages), run several real GpuEngine.step()s and compare sampled
layers of every recorded step against the fp64 oracle -- the synthetic
prefill rows plus the model rows each step appended (tests/gpu_check.py).
Steps after the first read the K/V rows the earlier steps appended.
"""

import os
import sys

import pytest

from gpu_check import check_history, tensor_model_oracle

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import bench  # noqa: E402


@pytest.mark.parametrize("name,steps", [("llama13b_p6000_b64", 6), ("llama7b_p6000_b64", 4),
                                        ("llama13b_p6000_b128", 4)])
def test_benchmarked_config_full_depth(cuda_device, name, steps):
    import torch

    cfg = bench.CONFIGS[name]
    L = cfg["L"]
    eng, rows = bench.build_engine(cfg, cuda_device, torch, out_len=64)
    eng.keep_history = True
    for i in range(steps):
        # the timed steps run without the fp32 capture (a different graph
        # argument only): the first steps check the bf16 output alone
        eng.capture_f32 = i >= steps - 2
        eng.step()
    eng.stream.synchronize()
    assert len(eng.history) == steps and eng.last_plan.num_rows == rows == cfg["B"]
    assert eng.last_plan.num_tc_items > 0  # the shared prefix ran on the tcgen05 kernel
    kv, queries = tensor_model_oracle(eng, eng.bench_leaf_n0)
    w = check_history(eng, steps=[0, steps // 2, steps - 1], layers=[0, L // 2 - 1, L - 1], kv=kv, queries=queries)
    assert w["pass"]
    print(name, w)
    eng.close()

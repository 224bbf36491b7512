"""The product's pipeline model (csrc/pipeline_model.cpp, afdk_simulate) vs the
reference's own simulate() (oracle/_ref, compiled from pipesim.cpp) — the
differential-oracle pattern of test_pipesim.cpp:146-157: identical tpot, tgs,
utilisation and bubbles (exact double equality) on random instances."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2507_19427_b200 import afdk


def rand_times(rng, L):
    return [rng.uniform(1e-6, 1e-4, L) for _ in range(4)]


@pytest.mark.parametrize("seed", range(40))
def test_simulate_matches_reference_exactly(seed):
    rng = np.random.default_rng(20250810 + seed)
    L = int(rng.integers(1, 62))
    n = int(rng.integers(1, 5))
    steps = int(rng.integers(2, 5))
    shared = bool(rng.integers(0, 2))
    t = rand_times(rng, L)
    if seed % 5 == 0:
        t[1][:] = 0.0  # zero-duration links
    mine = afdk.simulate(*t, n_micro=n, total_batch=1000 * n, total_gpus=8, token_steps=steps, shared_link=shared)
    ref = orc.ref_simulate(*t, n_micro=n, total_batch=1000 * n, total_gpus=8, token_steps=steps, shared_link=shared)
    assert mine["tpot"] == ref["tpot"]
    assert mine["tgs"] == ref["tgs"]
    assert mine["utilization"] == ref["utilization"]
    assert mine["bubble"] == ref["bubble"]


def test_simulate_balanced_toy_matches_reference():
    """Uniform stages (the balanced case of test_pipesim.cpp:125-137)."""
    L, n = 61, 3
    t = [np.full(L, 1e-4)] * 4
    mine = afdk.simulate(*t, n_micro=n, total_batch=6144, total_gpus=32)
    ref = orc.ref_simulate(*t, n_micro=n, total_batch=6144, total_gpus=32)
    assert mine == ref
    # 4 equal stages but only 3 micro-batches in flight: one slot per layer idles
    assert mine["tpot"] == pytest.approx(61 * 4e-4, rel=1e-9)


def test_simulate_rejects_bad_input():
    with pytest.raises(afdk.AfdkError):
        afdk.simulate([1e-4], [1e-4], [-1.0], [1e-4], n_micro=2, total_batch=2, total_gpus=2)


def test_reference_stage_times_feed_product_simulator():
    """derive_stage_times (reference, analytic) -> product simulate == reference simulate."""
    hw = dict(name="B200", f16=2.25e15, f8=4.5e15, bw=8e12, net=9e11, gps=1)
    st = orc.ref_derive_stage_times(hw, attn_inst=2, ffn_inst=6, micro_batch=256, n_micro=3, ctx=4096)
    mine = afdk.simulate(*st, n_micro=3, total_batch=768, total_gpus=8)
    ref = orc.ref_simulate(*st, n_micro=3, total_batch=768, total_gpus=8)
    assert mine == ref


@pytest.mark.parametrize("seed", range(6))
def test_trace_csv_matches_reference_bytes(seed):
    """The product's trace_csv (afdk_trace_csv) == the reference's trace_csv
    (pipesim.cpp:239-260) byte for byte on random stage times."""
    rng = np.random.default_rng(77 + seed)
    L, n = int(rng.integers(1, 20)), int(rng.integers(1, 4))
    t = rand_times(rng, L)
    mine = afdk.trace_csv(*t, n_micro=n, total_batch=100 * n, total_gpus=4)
    ref = orc.ref_trace_csv(*t, n_micro=n, total_batch=100 * n, total_gpus=4)
    assert mine == ref
    assert mine.splitlines()[0] == "time_s,resource,layer,micro_batch,stage,duration_s"


HW = dict(name="B200", f16=2.25e15, f8=4.5e15, bw=8e12, net=9e11, gps=1)


@pytest.mark.parametrize("plan", [(2, 6, 256, 3, 4096), (1, 1, 4096, 3, 4096), (2, 2, 2048, 3, 8192),
                                  (1, 3, 512, 2, 32768), (4, 4, 8192, 4, 4096)])
@pytest.mark.parametrize("tpot,stages", [(0.05, 3), (0.2, 3), (0.01, 3)])
def test_vet_stages_matches_reference_vet_plan(plan, tpot, stages):
    """stage_ok of the product's vet_stages == the reference's vet_plan
    stage_ok (planner.cpp:124-131) on the reference's own derived stage times:
    the same check can then run on MEASURED stage times."""
    na, nf, mb, nm, ctx = plan
    st = orc.ref_derive_stage_times(HW, attn_inst=na, ffn_inst=nf, micro_batch=mb, n_micro=nm, ctx=ctx)
    ref = orc.ref_vet_plan(HW, na, nf, mb, nm, ctx, tpot=tpot, stages=stages)
    mine = afdk.vet_stages(st[0], st[2], tpot_sla=tpot, pipeline_stages=stages, n_model_layers=61)
    assert mine["stage_ok"] == ref["stage_ok"], (mine, ref)
    assert mine["budget_s"] == orc.ref_stage_budget(tpot, stages, 61)

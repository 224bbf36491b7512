"""Measured provider (afdk_measure_stage_times / afd::measure_stage_times):
per-layer stage times come from running the kernels, have the reference's
StageTimes shape (61 layers, dense FFN on layers 0-3 and 60) and feed the
pipeline model."""
import json
import os
import subprocess

import pytest

from paper_2507_19427_b200 import afdk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_measured_stage_times_shape_and_simulate(ctx):
    st = ctx.measure_stage_times(attn_gpus=2, ffn_gpus=6, micro_batch=256, avg_ctx=4096)
    d = st["detail"]
    assert d["attn_batch"] == 128 and d["ffn_tokens"] == 256 and d["local_experts"] == 8
    assert all(len(st[k]) == 61 for k in ("attn", "comm_fwd", "ffn", "comm_bwd"))
    assert all(v > 0 for k in ("attn", "comm_fwd", "ffn", "comm_bwd") for v in st[k])
    dense = [0, 1, 2, 3, 60]
    assert all(st["ffn"][l] == d["dense_ffn_s"] for l in dense)
    assert all(st["ffn"][l] == d["moe_ffn_s"] for l in range(4, 60))
    # attention layer at 128 x 4K: KV 134 MB + 339 MB weights -> tens of us, far from ms
    assert 20e-6 < d["attn_s"] < 2e-3
    r = afdk.simulate(st["attn"], st["comm_fwd"], st["ffn"], st["comm_bwd"], n_micro=3, total_batch=768,
                      total_gpus=8)
    slowest = max(max(st[k]) for k in ("attn", "comm_fwd", "ffn", "comm_bwd"))
    assert r["tpot"] >= 61 * slowest * 0.999
    assert r["tgs"] == pytest.approx(768 / (r["tpot"] * 8))


@pytest.mark.gpu
def test_cpp_host_api_demo():
    exe = os.path.join(ROOT, "tests", "cpp", "stage_times_demo")
    out = subprocess.run([exe, "2", "6", "256", "4096", "3"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["plan"] == "2A6F" and d["tgs"] > 0 and d["attn_us"] > 0 and d["moe_ffn_us"] > 0


@pytest.mark.gpu
def test_reference_headers_build_drop_in():
    """The host API compiled against the reference's OWN headers and linked
    with the reference's own library (tests/cpp/stage_times_ref_demo, built by
    build() where /root/reference exists): the reference's catalog card feeds
    measure_stage_times, and the reference's own simulate() consumes the
    measured StageTimes — bit-identical to the product's pipeline model."""
    exe = os.path.join(ROOT, "tests", "cpp", "stage_times_ref_demo")
    if not os.path.exists(exe):
        pytest.skip("reference-headers demo not built (reference tree absent at build time)")
    out = subprocess.run([exe, "2", "6", "256", "4096", "3"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["model"] == "step3" and d["layers"] == 61
    assert d["ref_simulate_tpot_ms"] == d["product_simulate_tpot_ms"] > 0
    assert d["ref_simulate_tgs"] == d["product_simulate_tgs"]
    assert d["ref_tpot_bound_ms"] > 0  # the reference's analytic_tpot_bound on measured times (an estimate)
    assert d["attn_us"] > 0 and d["ffn_moe_us"] > 0 and d["ffn_dense_us"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("fmt,kv", [("fp8", "bf16"), ("mx", "e4m3"), ("bf16", "e4m3")])
def test_measured_provider_formats(ctx, fmt, kv):
    """Formats honoured: e4m3 KV makes the attention stage faster than bf16 KV
    (half the KV bytes), bf16 experts make the FFN stage slower than MXFP8
    (twice the weight bytes); the dense stage is this GPU's TP share."""
    st = ctx.measure_stage_times(attn_gpus=2, ffn_gpus=6, micro_batch=256, avg_ctx=4096, ffn_format=fmt, kv=kv)
    d = st["detail"]
    assert d["attn_s"] > 0 and d["moe_ffn_s"] > 0 and d["dense_ffn_s"] > 0
    base = ctx.measure_stage_times(attn_gpus=2, ffn_gpus=6, micro_batch=256, avg_ctx=4096, ffn_format="mx",
                                   kv="bf16")["detail"]
    if kv == "e4m3":
        assert d["attn_s"] < base["attn_s"]
    if fmt == "bf16":
        assert d["moe_ffn_s"] > base["moe_ffn_s"]

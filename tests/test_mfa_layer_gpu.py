"""Attention-side decode layer (K1 + K2/K3 + K4) vs the CPU oracle.

Tolerance (stated): bf16 storage at every stage against the oracle's bf16
rounding points: h_res/h_norm max|gpu-ref|/max|ref| <= 2e-2; appended K/V
(post-RoPE) <= 1e-2."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.golden import make_golden as mg
from tests.helpers import rel_err

STEP3 = dict(hidden=7168, q_lora=2048, n_heads=64, head_dim=256, page=64)


def run_layer(ctx, dims, seq_lens, seed):
    import torch

    x, w, kc, vc, bt, sl = mg.layer_inputs(dims, seq_lens, seed)
    dev = torch.device("cuda:0")
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(dev)
    wd = {k: bf(v) for k, v in w.items()}
    kd, vd = bf(kc), bf(vc)
    xd = bf(x)
    h_res = torch.empty_like(xd)
    h_norm = torch.empty_like(xd)
    ctx.mfa_layer(wd, xd, kd, vd, torch.from_numpy(bt).to(dev), torch.from_numpy(sl).to(dev), h_res, h_norm)
    torch.cuda.synchronize()
    k1, v1 = kc.copy(), vc.copy()
    r_res, r_norm = orc.mfa_layer(dims, x, w, k1, v1, bt, sl)
    return (h_res.float().cpu().numpy(), h_norm.float().cpu().numpy(), kd.float().cpu().numpy(),
            vd.float().cpu().numpy(), r_res, r_norm, k1, v1, bt, sl)


def check(res, page):
    g_res, g_norm, gk, gv, r_res, r_norm, rk, rv, bt, sl = res
    assert rel_err(g_res, r_res) <= 2e-2, rel_err(g_res, r_res)
    assert rel_err(g_norm, r_norm) <= 2e-2, rel_err(g_norm, r_norm)
    for b, L in enumerate(sl):
        pos = L - 1
        pg, s = bt[b, pos // page], pos % page
        assert rel_err(gk[pg, s], rk[pg, s]) <= 1e-2
        assert rel_err(gv[pg, s], rv[pg, s]) <= 1e-2  # bf16(v projection): ulp flips allowed
    # nothing else in the cache was touched
    mask = np.ones(gk.shape[:2], bool)
    for b, L in enumerate(sl):
        mask[bt[b, (L - 1) // page], (L - 1) % page] = False
    np.testing.assert_array_equal(gk[mask], rk[mask])


@pytest.mark.gpu
def test_mfa_layer_small_dims(ctx):
    check(run_layer(ctx, mg.SMALL, [70, 130, 1, 64], 12), 64)


@pytest.mark.gpu
def test_mfa_layer_step3_dims(ctx):
    check(run_layer(ctx, STEP3, [300, 4096, 65], 5), 64)


def run_layer_fp8(ctx, dims, seq_lens, seed):
    """Same layer over e4m3 KV caches with per-tensor scales."""
    import torch

    x, w, kc, vc, bt, sl = mg.layer_inputs(dims, seq_lens, seed)
    ks, vs = float(np.abs(kc).max()) / 448.0, float(np.abs(vc).max()) / 448.0
    kq = (torch.from_numpy(kc) / ks).to(torch.float8_e4m3fn).view(torch.uint8)
    vq = (torch.from_numpy(vc) / vs).to(torch.float8_e4m3fn).view(torch.uint8)
    dev = torch.device("cuda:0")
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(dev)
    wd = {k: bf(v) for k, v in w.items()}
    xd = bf(x)
    kd, vd = kq.to(dev), vq.to(dev)
    h_res, h_norm = torch.empty_like(xd), torch.empty_like(xd)
    ctx.mfa_layer(wd, xd, kd, vd, torch.from_numpy(bt).to(dev), torch.from_numpy(sl).to(dev), h_res, h_norm,
                  kv_scales=(ks, vs))
    torch.cuda.synchronize()
    k1 = orc.e4m3_to_f32(kq.numpy()) * np.float32(ks)
    v1 = orc.e4m3_to_f32(vq.numpy()) * np.float32(vs)
    r_res, r_norm = orc.mfa_layer(dict(dims, kv_k_scale=ks, kv_v_scale=vs), x, w, k1, v1, bt, sl)
    gk = orc.e4m3_to_f32(kd.cpu().numpy()) * np.float32(ks)
    gv = orc.e4m3_to_f32(vd.cpu().numpy()) * np.float32(vs)
    return h_res.float().cpu().numpy(), h_norm.float().cpu().numpy(), gk, gv, r_res, r_norm, k1, v1, bt, sl, (ks, vs)


@pytest.mark.gpu
@pytest.mark.parametrize("dims,seq_lens,seed", [(mg.SMALL, [70, 130, 1, 64], 12), (STEP3, [300, 4096, 65], 5)])
def test_mfa_layer_fp8_kv(ctx, dims, seq_lens, seed):
    """FP8 KV: appended token = e4m3(bf16(x)/scale) (one e4m3 ulp allowed where the
    bf16 projection itself differs by an ulp); h_res/h_norm within 3e-2 of the
    oracle (exact attention on the dequantised cache; the kernel rounds P to e4m3)."""
    g_res, g_norm, gk, gv, r_res, r_norm, rk, rv, bt, sl, (ks, vs) = run_layer_fp8(ctx, dims, seq_lens, seed)
    assert rel_err(g_res, r_res) <= 3e-2, rel_err(g_res, r_res)
    assert rel_err(g_norm, r_norm) <= 3e-2, rel_err(g_norm, r_norm)
    page = dims["page"]
    for b, L in enumerate(sl):
        pg, s = bt[b, (L - 1) // page], (L - 1) % page
        for g, r, sc in ((gk[pg, s], rk[pg, s], ks), (gv[pg, s], rv[pg, s], vs)):
            # one e4m3 step: 2^-3 of the binade (relative), 2^-9 * scale for subnormals
            close = np.abs(g - r) <= np.maximum(0.125 * np.abs(r), 2.0 ** -9 * sc) * 1.0001
            assert close.all() and np.mean(g != r) <= 0.05
    mask = np.ones(gk.shape[:2], bool)
    for b, L in enumerate(sl):
        mask[bt[b, (L - 1) // page], (L - 1) % page] = False
    np.testing.assert_array_equal(gk[mask], rk[mask])


@pytest.mark.gpu
@pytest.mark.parametrize("dims,seq_lens,seed", [(mg.SMALL, [70, 130, 2, 64, 65], 21), (STEP3, [300, 4096, 66], 8)])
def test_mfa_layer_mtp2(ctx, dims, seq_lens, seed):
    """MTP layer: 2 token rows per request, each appending its own K/V, causal
    attention among the new tokens.  The oracle runs the same rows as
    independent decode rows (seq_len L-1 and L, the request's pages)."""
    import torch

    x1, w, kc, vc, bt, sl = mg.layer_inputs(dims, seq_lens, seed)
    rng = np.random.default_rng(seed + 1)
    B = len(seq_lens)
    x = orc.bf16_round(rng.standard_normal((2 * B, dims["hidden"])).astype(np.float32))
    dev = torch.device("cuda:0")
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(dev)
    wd = {k: bf(v) for k, v in w.items()}
    kd, vd, xd = bf(kc), bf(vc), bf(x)
    h_res, h_norm = torch.empty_like(xd), torch.empty_like(xd)
    ctx.mfa_layer(wd, xd, kd, vd, torch.from_numpy(bt).to(dev), torch.from_numpy(sl).to(dev), h_res, h_norm, mtp=2)
    torch.cuda.synchronize()
    bt_rows = np.repeat(bt, 2, axis=0)
    sl_rows = np.stack([sl - 1, sl], axis=1).reshape(-1).astype(np.int32)
    k1, v1 = kc.copy(), vc.copy()
    r_res, r_norm = orc.mfa_layer(dims, x, w, k1, v1, bt_rows, sl_rows)
    assert rel_err(h_res.float().cpu().numpy(), r_res) <= 2e-2, rel_err(h_res.float().cpu().numpy(), r_res)
    assert rel_err(h_norm.float().cpu().numpy(), r_norm) <= 2e-2, rel_err(h_norm.float().cpu().numpy(), r_norm)
    gk = kd.float().cpu().numpy()
    page = dims["page"]
    for b, L in enumerate(sl):
        for j, pos in enumerate((L - 2, L - 1)):
            pg, s = bt[b, pos // page], pos % page
            assert rel_err(gk[pg, s], k1[pg, s]) <= 1e-2, (b, j)


@pytest.mark.gpu
@pytest.mark.parametrize("kv,batch", [("bf16", 256), ("e4m3", 256), ("bf16", 384), ("e4m3", 400)])
def test_mfa_layer_wide_batch(ctx, kv, batch):
    """256-400 requests (the AFD micro-batch): the 2-CTA-cluster row epilogues,
    the separate RoPE(q) row epilogue and the N=256 projections, or above 256
    rows the two-MMA (N/2 each) projections; ragged contexts."""
    rng = np.random.default_rng(77 + batch)
    seq_lens = rng.integers(1, 700, size=batch).tolist()
    if kv == "bf16":
        check(run_layer(ctx, STEP3, seq_lens, 31), 64)
    else:
        g_res, g_norm, gk, gv, r_res, r_norm, rk, rv, bt, sl, _ = run_layer_fp8(ctx, STEP3, seq_lens, 32)
        assert rel_err(g_res, r_res) <= 3e-2, rel_err(g_res, r_res)
        assert rel_err(g_norm, r_norm) <= 3e-2, rel_err(g_norm, r_norm)


@pytest.mark.gpu
@pytest.mark.parametrize("kv,batch", [("bf16", 64), ("e4m3", 64), ("e4m3", 320)])
def test_mfa_layer_mx_oproj(ctx, kv, batch):
    """o_proj as an MXFP8 GEMM (afdk_mfa_weights.w_o_mx / w_o_sf, afdk_linear_mx):
    the oracle quantises the attention output with the same MX rule (o_mx) and
    multiplies by the dequantised MX weights; bars as the bf16 / e4m3-KV layer."""
    import torch

    rng = np.random.default_rng(91 + batch)
    seq_lens = rng.integers(1, 700, size=batch).tolist()
    x, w, kc, vc, bt, sl = mg.layer_inputs(STEP3, seq_lens, 17)
    dev = torch.device("cuda:0")
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(dev)
    wd = {k: bf(v) for k, v in w.items()}
    n_out, nq = wd["o"].shape
    o_mx = torch.empty(n_out, nq, dtype=torch.uint8, device=dev)
    o_sf = torch.empty(n_out, nq // 32, dtype=torch.uint8, device=dev)
    ctx.quant_mx(wd["o"], o_mx, o_sf)
    wd["o_mx"], wd["o_sf"] = o_mx, o_sf
    w_or = dict(w)
    w_or["o"] = (orc.e4m3_to_f32(o_mx.cpu().numpy()) *
                 np.exp2(o_sf.cpu().numpy().astype(np.float32) - 127.0).repeat(32, axis=1)).astype(np.float32)
    dims = dict(STEP3, o_mx=1)
    xd = bf(x)
    h_res, h_norm = torch.empty_like(xd), torch.empty_like(xd)
    bt_d, sl_d = torch.from_numpy(bt).to(dev), torch.from_numpy(sl).to(dev)
    if kv == "e4m3":
        ks, vs = float(np.abs(kc).max()) / 448.0, float(np.abs(vc).max()) / 448.0
        kq = (torch.from_numpy(kc) / ks).to(torch.float8_e4m3fn).view(torch.uint8)
        vq = (torch.from_numpy(vc) / vs).to(torch.float8_e4m3fn).view(torch.uint8)
        ctx.mfa_layer(wd, xd, kq.to(dev), vq.to(dev), bt_d, sl_d, h_res, h_norm, kv_scales=(ks, vs))
        k1 = orc.e4m3_to_f32(kq.numpy()) * np.float32(ks)
        v1 = orc.e4m3_to_f32(vq.numpy()) * np.float32(vs)
        dims.update(kv_k_scale=ks, kv_v_scale=vs)
        bar = 3e-2
    else:
        ctx.mfa_layer(wd, xd, bf(kc), bf(vc), bt_d, sl_d, h_res, h_norm)
        k1, v1 = kc.copy(), vc.copy()
        bar = 2e-2
    torch.cuda.synchronize()
    r_res, r_norm = orc.mfa_layer(dims, x, w_or, k1, v1, bt, sl)
    e_res = rel_err(h_res.float().cpu().numpy(), r_res)
    e_norm = rel_err(h_norm.float().cpu().numpy(), r_norm)
    try:
        from tests.helpers import record
        record(f"mfa_layer_mx_oproj_{kv}_B{batch}", h_res=e_res, h_norm=e_norm)
    except Exception:  # noqa: BLE001
        pass
    assert e_res <= bar, e_res
    assert e_norm <= bar, e_norm


@pytest.mark.gpu
@pytest.mark.parametrize("kv,batch,o_mx", [("bf16", 64, False), ("e4m3", 64, True), ("e4m3", 352, True)])
def test_mfa_layer_mx_qup(ctx, kv, batch, o_mx):
    """q_up as an MXFP8 GEMM (afdk_mfa_weights.w_q_up_mx / w_q_up_sf): the
    oracle MX-quantises the q-RMSNorm output (qup_mx) and multiplies by the
    dequantised MX weights; alone and together with the MXFP8 o_proj (the AFD
    attention ranks' configuration).  Bars as the bf16 / e4m3-KV layer."""
    import torch

    rng = np.random.default_rng(7 + batch)
    seq_lens = rng.integers(1, 700, size=batch).tolist()
    x, w, kc, vc, bt, sl = mg.layer_inputs(STEP3, seq_lens, 23)
    dev = torch.device("cuda:0")
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).to(dev)
    wd = {k: bf(v) for k, v in w.items()}
    w_or = dict(w)
    dims = dict(STEP3, qup_mx=1, o_mx=int(o_mx))

    def mx(name):
        n, k = wd[name].shape
        q8 = torch.empty(n, k, dtype=torch.uint8, device=dev)
        sf = torch.empty(n, k // 32, dtype=torch.uint8, device=dev)
        ctx.quant_mx(wd[name], q8, sf)
        w_or[name] = (orc.e4m3_to_f32(q8.cpu().numpy()) *
                      np.exp2(sf.cpu().numpy().astype(np.float32) - 127.0).repeat(32, axis=1)).astype(np.float32)
        return q8, sf

    wd["q_up_mx"], wd["q_up_sf"] = mx("q_up")
    del wd["q_up"]  # the bf16 q_up must not be needed
    if o_mx:
        wd["o_mx"], wd["o_sf"] = mx("o")
    xd = bf(x)
    h_res, h_norm = torch.empty_like(xd), torch.empty_like(xd)
    bt_d, sl_d = torch.from_numpy(bt).to(dev), torch.from_numpy(sl).to(dev)
    if kv == "e4m3":
        ks, vs = float(np.abs(kc).max()) / 448.0, float(np.abs(vc).max()) / 448.0
        kq = (torch.from_numpy(kc) / ks).to(torch.float8_e4m3fn).view(torch.uint8)
        vq = (torch.from_numpy(vc) / vs).to(torch.float8_e4m3fn).view(torch.uint8)
        ctx.mfa_layer(wd, xd, kq.to(dev), vq.to(dev), bt_d, sl_d, h_res, h_norm, kv_scales=(ks, vs))
        k1 = orc.e4m3_to_f32(kq.numpy()) * np.float32(ks)
        v1 = orc.e4m3_to_f32(vq.numpy()) * np.float32(vs)
        dims.update(kv_k_scale=ks, kv_v_scale=vs)
        bar = 3e-2
    else:
        ctx.mfa_layer(wd, xd, bf(kc), bf(vc), bt_d, sl_d, h_res, h_norm)
        k1, v1 = kc.copy(), vc.copy()
        bar = 2e-2
    torch.cuda.synchronize()
    r_res, r_norm = orc.mfa_layer(dims, x, w_or, k1, v1, bt, sl)
    e_res = rel_err(h_res.float().cpu().numpy(), r_res)
    e_norm = rel_err(h_norm.float().cpu().numpy(), r_norm)
    try:
        from tests.helpers import record
        record(f"mfa_layer_mx_qup_{kv}_B{batch}{'_omx' if o_mx else ''}", h_res=e_res, h_norm=e_norm)
    except Exception:  # noqa: BLE001
        pass
    assert e_res <= bar, e_res
    assert e_norm <= bar, e_norm

"""Golden fixtures from the PUBLIC Step-3 decoder (vLLM), pinning the oracle's
numeric semantics to an implementation the builder did not write.

The reference (afdsim) has no numerics, so the oracle's choices
— RMSNorm eps and placement, NeoX RoPE and its theta, softmax scale, router
scoring / renormalisation, SiLU-and-mul experts, shared expert added with
weight 1 — are checked here against vLLM's Step-3 building blocks, run on
the CPU in fp32 (`forward_native` paths, no custom kernels):

  * configs/step3_vl.py Step3TextConfig defaults: rms_norm_eps, rope_theta,
    norm_expert_weight, moe_top_k / moe_num_experts, head_dim, share_q_dim,
    share_expert_dim;
  * models/step3_text.py Step3TextAttention.forward: qkv_proj -> split
    [q_size, kv, kv] -> inter_norm -> wq -> rotary_emb (get_rope(head_dim,
    rope_parameters), NeoX) -> attention with scaling = head_dim**-0.5 and one
    KV head -> o_proj; Step3TextDecoderLayer.forward: input_layernorm, then
    post_attention_layernorm(h, residual) -> (norm(h + x), h + x);
  * FusedMoEBlock: softmax top-k with renormalize = norm_expert_weight
    (layers/fused_moe/cpu_fused_moe.py select_experts, the torch router);
    Step3TextMLP: gate_up_proj -> SiluAndMul -> down_proj; the MoE output is
    share_output + moe_output.

The fixture stores inputs and outputs (tiny dims, float32).  It is
regenerated only here (vLLM is importable in the build container, not
needed on the GPU box):

    VLLM_TARGET_DEVICE=cpu python tests/golden/make_vllm_golden.py
"""
from __future__ import annotations

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "vllm_step3.npz")

# tiny geometry (the oracle takes any dims; 4 heads keep the fixture small)
HID, QL, NH, HD, PAGE = 256, 64, 4, 32, 16
SEQ = [5, 33, 17]
E, TOPK = 48, 3          # router at the Step-3 expert count
EM, HM, I = 8, 128, 32   # MoE layer fixture: 8 routed + shared, top-3


def main():
    os.environ.setdefault("VLLM_TARGET_DEVICE", "cpu")
    import torch
    from vllm.config import VllmConfig, set_current_vllm_config
    from vllm.config.device import DeviceConfig
    from vllm.transformers_utils.configs.step3_vl import Step3TextConfig

    torch.manual_seed(0)
    cfgd = Step3TextConfig()
    eps = float(cfgd.rms_norm_eps)
    theta = float(cfgd.rope_parameters["rope_theta"])
    renorm = bool(cfgd.norm_expert_weight)
    rng = np.random.default_rng(2507)
    f32 = lambda *s: rng.standard_normal(s).astype(np.float32)

    with set_current_vllm_config(VllmConfig(device_config=DeviceConfig(device="cpu"))):
        from vllm.model_executor.layers.activation import SiluAndMul
        from vllm.model_executor.layers.fused_moe.cpu_fused_moe import select_experts
        from vllm.model_executor.layers.layernorm import RMSNorm
        from vllm.model_executor.layers.rotary_embedding import get_rope

        # ------------------------------------------------ attention-side layer
        B = len(SEQ)
        w = {"in_norm": 1 + 0.1 * f32(HID), "qkv": f32(QL + 2 * HD, HID) / float(np.sqrt(HID)),
             "q_norm": 1 + 0.1 * f32(QL), "q_up": f32(NH * HD, QL) / float(np.sqrt(QL)),
             "o": f32(HID, NH * HD) / float(np.sqrt(NH * HD)), "post_norm": 1 + 0.1 * f32(HID)}
        w = {n: a.astype(np.float32) for n, a in w.items()}
        x = f32(B, HID)
        need = [(L + PAGE - 1) // PAGE for L in SEQ]
        num_pages = sum(need) + 2
        perm = rng.permutation(num_pages).astype(np.int32)
        bt = np.zeros((B, max(need)), np.int32)
        k0 = 0
        for b, n in enumerate(need):
            bt[b, :n] = perm[k0:k0 + n]
            k0 += n
        kc, vc = f32(num_pages, PAGE, HD), f32(num_pages, PAGE, HD)

        T = lambda a: torch.from_numpy(np.ascontiguousarray(a))
        in_ln = RMSNorm(HID, eps=eps)
        in_ln.weight.data = T(w["in_norm"])
        inter = RMSNorm(QL, eps=eps)
        inter.weight.data = T(w["q_norm"])
        post_ln = RMSNorm(HID, eps=eps)
        post_ln.weight.data = T(w["post_norm"])
        rope = get_rope(HD, max_position=65536, rope_parameters=dict(cfgd.rope_parameters))
        assert rope.is_neox_style and rope.rotary_dim == HD
        scaling = HD ** -0.5  # Step3TextAttention: scaling = self.head_dim**-0.5

        xt = T(x)
        hs = in_ln.forward_native(xt)
        qkv = hs @ T(w["qkv"]).T
        q, k, v = qkv.split([QL, HD, HD], dim=-1)
        q = inter.forward_native(q.contiguous())
        q = q @ T(w["q_up"]).T
        pos = torch.tensor([L - 1 for L in SEQ])
        q, k = rope.forward_native(pos, q.contiguous(), k.contiguous())
        kc_out, vc_out = kc.copy(), vc.copy()
        attn = torch.empty(B, NH * HD)
        for b, L in enumerate(SEQ):
            pg, sl = bt[b, (L - 1) // PAGE], (L - 1) % PAGE
            kc_out[pg, sl] = k[b].numpy()
            vc_out[pg, sl] = v[b].numpy()
            rows = [bt[b, p // PAGE] * PAGE + p % PAGE for p in range(L)]
            Kb = T(kc_out.reshape(-1, HD)[rows])
            Vb = T(vc_out.reshape(-1, HD)[rows])
            qb = q[b].view(NH, HD)
            ob = torch.nn.functional.scaled_dot_product_attention(
                qb[:, None, :], Kb.expand(NH, L, HD), Vb.expand(NH, L, HD), scale=scaling)
            attn[b] = ob.reshape(-1)
        o = attn @ T(w["o"]).T
        h_norm, h_res = post_ln.forward_native(o, xt.clone())

        # --------------------------------------------------------- router
        ntok = 9
        logits = f32(ntok, E)
        rw, rid = select_experts(None, T(logits), TOPK, False, renorm)

        # ---------------------------------------------- MoE layer (SwiGLU)
        mw, mid = select_experts(None, T(f32(ntok, EM)), TOPK, False, renorm)
        xm = f32(ntok, HM)
        w13 = (f32(EM + 1, 2 * I, HM) / float(np.sqrt(HM))).astype(np.float32)
        w2 = (f32(EM + 1, HM, I) / float(np.sqrt(I))).astype(np.float32)
        act = SiluAndMul()

        def mlp(e, xs):  # Step3TextMLP: gate_up_proj -> SiluAndMul -> down_proj
            return act.forward_native(xs @ T(w13[e]).T) @ T(w2[e]).T

        xmt = T(xm)
        moe = torch.zeros(ntok, HM)
        for t in range(ntok):
            for j in range(TOPK):
                moe[t] += mw[t, j] * mlp(int(mid[t, j]), xmt[t:t + 1])[0]
        share = mlp(EM, xmt)
        moe_out = share + moe

    np.savez_compressed(
        OUT, eps=eps, theta=theta, renorm=renorm, scaling=scaling, top_k=int(cfgd.moe_top_k),
        n_experts=int(cfgd.moe_num_experts), head_dim=int(cfgd.head_dim), share_q_dim=int(cfgd.share_q_dim),
        share_expert_dim=int(cfgd.share_expert_dim), moe_inter=int(cfgd.moe_intermediate_size),
        hidden=int(cfgd.hidden_size), dims=np.array([HID, QL, NH, HD, PAGE]), seq_lens=np.array(SEQ, np.int32),
        x=x, block_table=bt, k_cache=kc, v_cache=vc, **{"w_" + n: a for n, a in w.items()},
        h_res=h_res.numpy(), h_norm=h_norm.numpy(), k_cache_out=kc_out, v_cache_out=vc_out,
        logits=logits, topk_ids=rid.numpy(), topk_w=rw.numpy(),
        moe_x=xm, moe_ids=mid.numpy(), moe_wts=mw.numpy(), moe_w13=w13, moe_w2=w2, moe_out=moe_out.numpy())
    print("wrote", OUT)


if __name__ == "__main__":
    main()

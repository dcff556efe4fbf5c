"""Named ParamSet tables (tensor name, shape) in reference ParamSet order.

The reference trains toy models only; the hot path is exercised on synthetic
pseudo-gradients with the tensor shapes of real models.
Weights are stored [in, out] as in the reference (model.cpp:83).
"""
from __future__ import annotations


def opt(h: int, ffn: int, layers: int, vocab: int, pos: int):
    t = [("embed_tokens", (vocab, h)), ("embed_positions", (pos, h))]
    for i in range(layers):
        p = f"layers.{i}."
        for proj in ("q_proj", "k_proj", "v_proj", "out_proj"):
            t += [(p + f"self_attn.{proj}.weight", (h, h)), (p + f"self_attn.{proj}.bias", (h,))]
        t += [(p + "self_attn_layer_norm.weight", (h,)), (p + "self_attn_layer_norm.bias", (h,))]
        t += [(p + "fc1.weight", (h, ffn)), (p + "fc1.bias", (ffn,))]
        t += [(p + "fc2.weight", (ffn, h)), (p + "fc2.bias", (h,))]
        t += [(p + "final_layer_norm.weight", (h,)), (p + "final_layer_norm.bias", (h,))]
    t += [("final_layer_norm.weight", (h,)), ("final_layer_norm.bias", (h,))]
    return t


def mini_opt():
    """C1: ~10.76 M params (h=512, ffn=2048, L=2, vocab 8192, pos 514)."""
    return opt(512, 2048, 2, 8192, 514)


def opt_1_3b():
    """C2: OPT-1.3B, 1 315 758 080 params, 146 2-D + 242 1-D tensors."""
    return opt(2048, 8192, 24, 50272, 2050)


def opt_1_3b_layer():
    """One OPT-1.3B decoder layer (the bounded CPU-baseline sample unit)."""
    return [(n, s) for n, s in opt(2048, 8192, 1, 16, 16) if n.startswith("layers.")]


def llama7b_layer():
    """C3: one Llama-7B decoder layer, 202 383 360 params."""
    h, f = 4096, 11008
    return [("self_attn.q_proj.weight", (h, h)), ("self_attn.k_proj.weight", (h, h)),
            ("self_attn.v_proj.weight", (h, h)), ("self_attn.o_proj.weight", (h, h)),
            ("mlp.gate_proj.weight", (h, f)), ("mlp.up_proj.weight", (h, f)),
            ("mlp.down_proj.weight", (f, h)), ("input_layernorm.weight", (h,)),
            ("post_attention_layernorm.weight", (h,))]


def qwen107b_stage(layers: int = 2):
    """C4: a Qwen1.5-107B pipeline-stage shard (1 358 981 120 params per layer)."""
    h, kv, f = 8192, 1024, 49152
    t = []
    for i in range(layers):
        p = f"layers.{i}."
        t += [(p + "self_attn.q_proj.weight", (h, h)), (p + "self_attn.q_proj.bias", (h,)),
              (p + "self_attn.k_proj.weight", (h, kv)), (p + "self_attn.k_proj.bias", (kv,)),
              (p + "self_attn.v_proj.weight", (h, kv)), (p + "self_attn.v_proj.bias", (kv,)),
              (p + "self_attn.o_proj.weight", (h, h)),
              (p + "mlp.gate_proj.weight", (h, f)), (p + "mlp.up_proj.weight", (h, f)),
              (p + "mlp.down_proj.weight", (f, h)),
              (p + "input_layernorm.weight", (h,)), (p + "post_attention_layernorm.weight", (h,))]
    return t


CONFIGS = {
    "mini-opt": mini_opt,
    "opt-1.3b": opt_1_3b,
    "opt-1.3b-layer": opt_1_3b_layer,
    "llama7b-layer": llama7b_layer,
    "qwen107b-stage": qwen107b_stage,
}


def numel(table) -> int:
    n = 0
    for _, s in table:
        k = 1
        for d in s:
            k *= d
        n += k
    return n

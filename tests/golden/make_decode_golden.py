"""Generate tests/golden/decode_tiny.npz: Hugging Face transformers' Qwen2ForCausalLM
(fp32, eager attention) logits for the tiny geometry on the oracle's numpy weights.

This pins oracle/decoder_ref.py (fp32 mode) to an independent, public
implementation of the same decoder math; the reference itself has no decode
numerics (tpshift prices steps, it never computes them). Run in this container:

    python tests/golden/make_decode_golden.py

Needs transformers (present here); the test that consumes the fixture does not.
"""

import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

from oracle.decoder_ref import TINY, numpy_weights  # noqa: E402

SEED = 1234
PROMPTS = [[7, 99, 1024, 5, 4095, 17, 256, 3, 3, 3, 800, 12],
           [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12]]


def main():
    from transformers import Qwen2Config, Qwen2ForCausalLM

    g = TINY
    W = numpy_weights(g, SEED)
    cfg = Qwen2Config(vocab_size=g["vocab"], hidden_size=g["hidden"], intermediate_size=g["ffn"],
                      num_hidden_layers=g["num_layers"], num_attention_heads=g["n_q"],
                      num_key_value_heads=g["n_kv"], rms_norm_eps=g["rms_eps"],
                      rope_theta=g["rope_theta"], max_position_embeddings=4096,
                      tie_word_embeddings=False, attn_implementation="eager")
    m = Qwen2ForCausalLM(cfg).float().eval()
    D, nq, nkv, F = g["head_dim"], g["n_q"], g["n_kv"], g["ffn"]
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(W[(-1, "embed")])
        m.model.norm.weight.copy_(W[(-1, "ln_f")])
        m.lm_head.weight.copy_(W[(-1, "lm_head")])
        for l, layer in enumerate(m.model.layers):
            qkv, b = W[(l, "w_qkv")], W[(l, "b_qkv")]
            a = layer.self_attn
            a.q_proj.weight.copy_(qkv[:nq * D]); a.q_proj.bias.copy_(b[:nq * D])
            a.k_proj.weight.copy_(qkv[nq * D:(nq + nkv) * D]); a.k_proj.bias.copy_(b[nq * D:(nq + nkv) * D])
            a.v_proj.weight.copy_(qkv[(nq + nkv) * D:]); a.v_proj.bias.copy_(b[(nq + nkv) * D:])
            a.o_proj.weight.copy_(W[(l, "w_o")])
            gu = W[(l, "w_gu")]
            layer.mlp.gate_proj.weight.copy_(gu[:F]); layer.mlp.up_proj.weight.copy_(gu[F:])
            layer.mlp.down_proj.weight.copy_(W[(l, "w_d")])
            layer.input_layernorm.weight.copy_(W[(l, "ln1")])
            layer.post_attention_layernorm.weight.copy_(W[(l, "ln2")])
        ids = torch.tensor(PROMPTS)
        logits = m(input_ids=ids).logits.float().numpy()
    np.savez_compressed(os.path.join(HERE, "decode_tiny.npz"), logits=logits.astype(np.float32),
                        prompts=np.array(PROMPTS, dtype=np.int32), seed=np.int64(SEED))
    print("wrote decode_tiny.npz", logits.shape)


if __name__ == "__main__":
    main()

"""Config C4 high-priority workload (BASELINE.json configs[3]): Llama-2-7B
greedy decoding at batch 1 -- an unmodified inference application, run as
the serving engine would: a prefill CUDA graph and one decode-step CUDA
graph replayed once per generated token, each an exempt pipeline step of the
high-priority task (Tally never transforms high-priority kernels).

The decoder is plain PyTorch (cuBLAS GEMVs, bf16, static KV cache), written
graph-capturable: token, position and output buffers are device tensors the
graphs update in place.  Numerics follow HuggingFace ``LlamaForCausalLM``
(RMSNorm in fp32, rotate-half RoPE with bf16 cos/sin, SiLU-gated MLP); the
parity test compares per-step logits against it on a small config.  Random
init (no checkpoints offline): N(0, 0.02) weights generated on the device.
"""

from __future__ import annotations

import math

from . import kernels as K


class LlamaDecode:
    """One high-priority request = prefill a ``prompt``-token prompt, then
    ``gen`` decode steps; ``out`` [gen + 1] int64 receives the generated
    tokens.  ``prompt_ids`` [prompt] int64 is the request's input buffer."""

    def __init__(self, prompt=32, gen=16, model=None, seed=1, device="cuda", n_layer=None, config=None):
        import torch
        from transformers import LlamaConfig
        self.torch = torch
        if model is not None:
            cfg = model.config
            sd = {k: v.detach().to(device=device, dtype=torch.bfloat16) for k, v in model.state_dict().items()}
        else:
            cfg = config or LlamaConfig(**({"num_hidden_layers": n_layer} if n_layer else {}))
            sd = None
        self.cfg = cfg
        self.P, self.G, self.device = prompt, gen, device
        d, H = cfg.hidden_size, cfg.num_attention_heads
        self.d, self.H, self.D = d, H, d // H
        self.I, self.V, self.L = cfg.intermediate_size, cfg.vocab_size, cfg.num_hidden_layers
        if getattr(cfg, "num_key_value_heads", H) != H:
            raise ValueError("LlamaDecode: multi-head attention only (Llama-2-7B: 32 KV heads)")
        self.eps = cfg.rms_norm_eps
        rope = getattr(cfg, "rope_parameters", None) or {}
        theta = rope.get("rope_theta", getattr(cfg, "rope_theta", 10000.0))
        self.max_len = (prompt + gen + 1 + 7) // 8 * 8
        gen_ = torch.Generator(device=device).manual_seed(seed)

        def w(name, *shape):
            if sd is not None:
                return sd[name].contiguous()
            return (torch.randn(*shape, device=device, dtype=torch.bfloat16, generator=gen_) * 0.02)

        def ones(name, n):
            return sd[name].contiguous() if sd is not None else torch.ones(n, device=device, dtype=torch.bfloat16)

        self.embed = w("model.embed_tokens.weight", self.V, d)
        self.layers = []
        for i in range(self.L):
            p = f"model.layers.{i}."
            lay = {"ln1": ones(p + "input_layernorm.weight", d), "ln2": ones(p + "post_attention_layernorm.weight", d)}
            if sd is not None:
                lay["wqkv"] = torch.cat([sd[p + f"self_attn.{n}_proj.weight"] for n in "qkv"]).contiguous()
                lay["wgu"] = torch.cat([sd[p + "mlp.gate_proj.weight"], sd[p + "mlp.up_proj.weight"]]).contiguous()
            else:
                lay["wqkv"] = w(None, 3 * d, d)
                lay["wgu"] = w(None, 2 * self.I, d)
            lay["wo"] = w(p + "self_attn.o_proj.weight", d, d)
            lay["wd"] = w(p + "mlp.down_proj.weight", d, self.I)
            self.layers.append(lay)
        self.norm = ones("model.norm.weight", d)
        self.lm_head = w("lm_head.weight", self.V, d)
        # RoPE tables (HF: fp32 angles, cos/sin cast to the activation dtype)
        inv = 1.0 / (theta ** (torch.arange(0, self.D, 2, device=device, dtype=torch.float32) / self.D))
        ang = torch.arange(self.max_len, device=device, dtype=torch.float32)[:, None] * inv[None, :]
        emb = torch.cat([ang, ang], dim=-1)
        self.cos, self.sin = emb.cos().to(torch.bfloat16), emb.sin().to(torch.bfloat16)
        self.k_cache = torch.zeros(self.L, H, self.max_len, self.D, device=device, dtype=torch.bfloat16)
        self.v_cache = torch.zeros_like(self.k_cache)
        self.prompt_ids = torch.zeros(prompt, device=device, dtype=torch.int64)
        self.tok = torch.zeros(1, device=device, dtype=torch.int64)
        self.pos = torch.zeros(1, device=device, dtype=torch.int64)
        self.cur = torch.zeros(1, device=device, dtype=torch.int64)
        self.out = torch.zeros(gen + 1, device=device, dtype=torch.int64)
        self.logits = torch.zeros(1, self.V, device=device, dtype=torch.float32)
        self.keys = torch.arange(self.max_len, device=device)
        self._capture()

    # ---- the model -------------------------------------------------------------------
    def _rms(self, x, w):
        torch = self.torch
        xf = x.float()
        return w * (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + self.eps)).to(x.dtype)

    @staticmethod
    def _rot(x, cos, sin):
        torch = __import__("torch")
        h = x.shape[-1] // 2
        return x * cos + torch.cat([-x[..., h:], x[..., :h]], dim=-1) * sin

    def _forward(self, x, cos, sin, prefill):
        """x [T, d] hidden states of the new tokens -> [T, d]; writes the KV cache."""
        torch = self.torch
        F = torch.nn.functional
        T = x.shape[0]
        H, D, d = self.H, self.D, self.d
        for li, lay in enumerate(self.layers):
            h = self._rms(x, lay["ln1"])
            qkv = (h @ lay["wqkv"].t()).view(T, 3, H, D).permute(1, 2, 0, 3)    # [3, H, T, D]
            q = self._rot(qkv[0], cos, sin)
            k = self._rot(qkv[1], cos, sin)
            v = qkv[2]
            if prefill:
                self.k_cache[li, :, :T] = k
                self.v_cache[li, :, :T] = v
                a = F.scaled_dot_product_attention(q[None], k[None], v[None], is_causal=True)[0]
            else:
                self.k_cache[li].index_copy_(1, self.cur, k)
                self.v_cache[li].index_copy_(1, self.cur, v)
                s = (q @ self.k_cache[li].transpose(1, 2)).float() * (1.0 / math.sqrt(D))   # [H, 1, max_len]
                s = s.masked_fill((self.keys > self.cur)[None, None, :], float("-inf"))
                a = (s.softmax(-1).to(x.dtype) @ self.v_cache[li])                           # [H, 1, D]
            x = x + a.permute(1, 0, 2).reshape(T, d) @ lay["wo"].t()
            h2 = self._rms(x, lay["ln2"])
            g, u = (h2 @ lay["wgu"].t()).split(self.I, dim=-1)
            x = x + (F.silu(g) * u) @ lay["wd"].t()
        return x

    def _head(self, x_last):
        self.logits.copy_((self._rms(x_last, self.norm) @ self.lm_head.t()).float())
        return self.logits.argmax(-1)

    def _prefill(self):
        x = self.embed.index_select(0, self.prompt_ids)
        P = self.P
        x = self._forward(x, self.cos[:P], self.sin[:P], prefill=True)
        nt = self._head(x[-1:])
        self.tok.copy_(nt)
        self.out[0:1].copy_(nt)
        self.pos.fill_(P)

    def _decode(self):
        # the position saturates at the cache end: replaying the step graph on
        # its own (profiling, cost measurement) never indexes out of bounds;
        # a request (prefill first) never reaches it
        self.cur.copy_(self.pos.clamp(max=self.max_len - 1))
        x = self.embed.index_select(0, self.tok)
        cos = self.cos.index_select(0, self.cur)
        sin = self.sin.index_select(0, self.cur)
        x = self._forward(x, cos, sin, prefill=False)
        nt = self._head(x)
        self.out.index_copy_(0, (self.cur - (self.P - 1)).clamp(max=self.G), nt)
        self.tok.copy_(nt)
        self.pos.add_(1)

    def _capture(self):
        torch = self.torch
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.no_grad(), torch.cuda.stream(side):
            for _ in range(2):
                self._prefill()
                for _ in range(2):
                    self._decode()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        with torch.no_grad():
            self.g_prefill = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.g_prefill):
                self._prefill()
            self.g_decode = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.g_decode):
                self._decode()
        torch.cuda.synchronize()
        self.prefill_kernel = K.cuda_graph(self.g_prefill)
        self.decode_kernel = K.cuda_graph(self.g_decode)

    # ---- running it -------------------------------------------------------------------
    def pipeline(self):
        """The request's device steps: prefill, then ``gen`` decode steps."""
        return [self.prefill_kernel] + [self.decode_kernel] * self.G

    def generate(self, prompt_ids):
        """Eager convenience (tests): one request through the graphs."""
        self.prompt_ids.copy_(prompt_ids)
        self.g_prefill.replay()
        for _ in range(self.G):
            self.g_decode.replay()
        self.torch.cuda.synchronize()
        return self.out.clone()

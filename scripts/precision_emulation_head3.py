"""Variant of precision_emulation.py: hi + lo everywhere vs a three-term (hi + mid + lo)
split of the head input only / of every GEMM input / everywhere
(profiles/r02/parity/precision_emulation_c2_32layers_head3.txt).

CPU emulation of where the bf16 error comes from at full C2 depth.

    python scripts/precision_emulation.py [layers]   (default 32; ~6 GB RAM, minutes)

LLaDA-8B-shape model (2 distinct layers' bf16 weights cycled to `layers`), one
prefill forward of a C2 prompt in fp32, with the device's storage points
rounded to bf16 (`bf)`, kept as hi + lo pairs (`hilo`) or exact, separately for
the GEMM inputs (xn, act, head input), q/K/V and the attention output.  Prints
max |delta| of the normalised logits vs the exact forward for spike gain 0 and
33 (profiles/r02/parity/precision_emulation_c2_32layers.txt)."""
import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import bb_oracle as O
V = 126462; d = 4096; nh = 32; hd = 128; dff = 12288
LAY = int(sys.argv[1]) if len(sys.argv) > 1 else 32
P, G = 64, 256; L = P + G
arch = O.OArch(kind="llada", vocab_size=V, layers=2, d_model=d, n_heads=nh, n_kv_heads=nh, head_dim=hd, d_ff=dff,
               max_len=L, rope_theta=500000.0, norm_eps=1e-5, head_scale=0.4)
t = time.time()
W = O.hash_weights(arch, 0)
for k in list(W):
    if k not in ("ln1", "ln2", "lnf", "bqkv"):
        W[k] = O.bf16_round(W[k]).astype(np.float32)
print("weights", time.time() - t, flush=True)
bf = lambda x: O.bf16_round(x).astype(np.float32)
def hilo(x):
    h = bf(x); return h + bf(x - h)
ident = lambda x: np.asarray(x, np.float32)

def fwd(r_gemm, r_qkv, r_attn_out, tokens, lay=LAY, r_head=None):
    h = W["emb"][tokens].astype(np.float32)
    n = len(tokens); pos = np.arange(n)
    for l in range(lay):
        w = l % 2
        xn = r_gemm(O._rmsnorm(h, W["ln1"][w], 1e-5))
        qkv = xn @ W["wqkv"][w].T
        q = qkv[:, :nh*hd].reshape(n, nh, hd); k = qkv[:, nh*hd:2*nh*hd].reshape(n, nh, hd); v = qkv[:, 2*nh*hd:].reshape(n, nh, hd)
        q = r_qkv(O._rope(q, pos, 500000.0)); k = r_qkv(O._rope(k, pos, 500000.0)); v = r_qkv(v)
        s = np.einsum('qhd,khd->hqk', q, k) / np.sqrt(hd)
        s = s - s.max(-1, keepdims=True); p = np.exp(s); p /= p.sum(-1, keepdims=True)
        o = np.einsum('hqk,khd->qhd', p.astype(np.float32), v).reshape(n, nh*hd)
        h = h + r_attn_out(o) @ W["wo"][w].T
        x2 = r_gemm(O._rmsnorm(h, W["ln2"][w], 1e-5))
        g = x2 @ W["wg"][w].T; u = x2 @ W["wu"][w].T
        h = h + r_gemm(g / (1 + np.exp(-g)) * u) @ W["wd"][w].T
    hf = (r_head or r_gemm)(O._rmsnorm(h[P:], W["lnf"], 1e-5))
    raw = (hf @ W["head"].T) * 0.4
    return raw

task = O.make_task(0, P, G, V)
row = np.full(L, V + 1, dtype=np.int64); row[:P] = task.prompt
def stats(raw, gain):
    lg = raw + gain * np.maximum(0, raw - 0.72)
    m = lg.max(1, keepdims=True); ln = lg - m - np.log(np.exp(lg - m).sum(1, keepdims=True))
    return ln
t = time.time()
ref = fwd(ident, ident, ident, row); print("exact", time.time() - t, flush=True)
def three(x):
    h = bf(x); m = bf(x - h); return h + m + bf(x - h - m)
cfgs = {"all_hilo": (hilo, hilo, hilo, None), "all_hilo_head3": (hilo, hilo, hilo, three),
        "gemm3_rest_hilo": (three, hilo, hilo, three), "all3": (three, three, three, three)}
for name, (a, b, c, rh) in cfgs.items():
    raw = fwd(a, b, c, row, r_head=rh)
    for gain in (0.0, 33.0):
        la, lb = stats(raw, gain), stats(ref, gain)
        print(f"{name:26s} gain {gain:4.0f}: max|dlogn| {np.abs(la-lb).max():.3e}", flush=True)

"""Model-side types of the blockbatch API and the device-resident parameter set.

Mirrors ``blockbatch.model`` (reference ``model.py``) so callers switch
imports only.  The forward itself never runs here: ``ModelParams`` owns the
device weights (canonical (out, in) layout, fp32 or bf16) and the handle of
the C-ABI model (``bb_model_create``); every forward is a CUDA kernel
sequence launched by the session (``engine.py``).

Two weight initialisations:
  * ``init="philox"`` — exactly the reference's ``build_model`` draw
    (model.py:210-241: Philox(key=seed), N(0,1)/sqrt(d), fixed order), so
    the device model is the reference model (cast to fp32/bf16).
  * ``init="hash"``   — counter-based uniform init generated on the GPU
    (``bb_fill_hash_uniform``), used for the LLaDA-8B / Dream-7B shapes
    where host generation of 8B normals would dominate.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, ContractError, StateError

CATEGORY_COUNT = 4


def _default_categories(size: int) -> dict[int, str]:
    return {t: f"cat{t % CATEGORY_COUNT}" for t in range(size)}


@dataclass(frozen=True)
class Vocab:
    """Token layout (model.py:30-63): regular ids 0..size-1, eos = size, mask = size+1.
    ``category_of`` defaults to the reference's modular categories."""

    size: int = 32
    category_of: dict | None = field(default=None, compare=False, repr=False)

    def __post_init__(self):
        if self.size < 2:
            raise ConfigError("vocab needs at least 2 regular tokens")
        if self.category_of is None:
            object.__setattr__(self, "category_of", _default_categories(self.size))
        elif len(self.category_of) < self.size or any(t not in self.category_of for t in range(self.size)):
            missing = [t for t in range(self.size) if t not in self.category_of]
            raise ConfigError(f"category_of not total over regular tokens: {missing[:3]}")

    @property
    def eos_id(self) -> int:
        return self.size

    @property
    def mask_id(self) -> int:
        return self.size + 1

    @property
    def n_out(self) -> int:
        return self.size + 1

    @property
    def n_extended(self) -> int:
        return self.size + 2


@dataclass(frozen=True)
class ModelDims:
    """model.py:66-70 plus the LLaDA/Dream-shape fields (defaults = reference model)."""

    layers: int = 2
    d_model: int = 32
    max_len: int = 384
    arch: str = "ref"          # "ref" | "llada"
    n_heads: int = 1
    n_kv_heads: int = 1
    head_dim: int = 0          # 0 -> d_model (single-head reference attention)
    d_ff: int = 0
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    qkv_bias: bool = False

    @property
    def hd(self) -> int:
        return self.head_dim or self.d_model

    @property
    def qkv_out(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.hd


# public model shapes (LLaDA-8B: GSAI-ML config; Dream-7B = Qwen2.5-7B)
LLADA_8B = ModelDims(layers=32, d_model=4096, max_len=4096, arch="llada", n_heads=32, n_kv_heads=32,
                     head_dim=128, d_ff=12288, rope_theta=500000.0, norm_eps=1e-5)
LLADA_8B_VOCAB = 126462      # n_out = 126463, embedding rows 126464
DREAM_7B = ModelDims(layers=28, d_model=3584, max_len=4096, arch="llada", n_heads=28, n_kv_heads=4,
                     head_dim=128, d_ff=18944, rope_theta=1e6, norm_eps=1e-6, qkv_bias=True)
DREAM_7B_VOCAB = 152062


@dataclass(frozen=True)
class BlockWindow:
    """Half-open absolute position range [start, end) (model.py:73-89)."""

    start: int
    end: int

    def __post_init__(self):
        if self.start > self.end:
            raise ConfigError(f"window start {self.start} > end {self.end}")

    def positions(self) -> np.ndarray:
        return np.arange(self.start, self.end)

    @property
    def empty(self) -> bool:
        return self.start >= self.end


@dataclass
class SequenceRow:
    """One branch's token buffer (model.py:92-112)."""

    tokens: np.ndarray
    prompt_len: int

    def __len__(self) -> int:
        return len(self.tokens)

    def copy(self) -> "SequenceRow":
        return SequenceRow(self.tokens.copy(), self.prompt_len)

    def masked_positions(self, mask_id: int, window: BlockWindow | None = None) -> np.ndarray:
        pos = np.flatnonzero(self.tokens == mask_id)
        if window is not None:
            pos = pos[(pos >= window.start) & (pos < window.end)]
        return pos

    def generated(self, vocab: Vocab) -> np.ndarray:
        return self.tokens[self.prompt_len:]


@dataclass(frozen=True)
class DenoiseOutput:
    """Per-position logits/probabilities (model.py:160-180)."""

    positions: np.ndarray
    logits: np.ndarray
    probs: np.ndarray

    def restrict(self, positions: np.ndarray) -> "DenoiseOutput":
        index = {int(p): i for i, p in enumerate(self.positions)}
        try:
            rows = np.array([index[int(p)] for p in positions], dtype=int)
        except KeyError as exc:
            raise ContractError(f"position {exc} was not queried") from exc
        return DenoiseOutput(np.asarray(positions, dtype=int), self.logits[rows], self.probs[rows])


class KvCache:
    """Per-layer, per-position keys/values plus validity flags (model.py:136-157).

    ``keys`` / ``values`` are (layers, L, kv_dim) float64 arrays and ``valid``
    an (L,) bool array, as in the reference (kv_dim = d_model for the
    reference architecture).  Caches produced by the device seams
    (``full_forward`` / ``block_forward`` / forward observers) live on the GPU
    as one fp32 vector in ``kv_vectorize`` layout; the host arrays are
    materialised on first access.  Once a caller has touched the host arrays
    they are the source of truth (in-place edits are honoured)."""

    def __init__(self, keys=None, values=None, valid=None, *, vec=None, shape=None):
        if vec is not None:
            if shape is None or valid is None:
                raise ContractError("a device KvCache needs its shape and validity flags")
            self._vec, self._shape = vec, tuple(shape)
            self._keys = self._values = None
        else:
            if keys is None or values is None or valid is None:
                raise ContractError("KvCache needs keys, values and valid")
            self._keys, self._values = np.asarray(keys), np.asarray(values)
            self._vec, self._shape = None, tuple(self._keys.shape)
        self.valid = np.asarray(valid, dtype=bool)

    @classmethod
    def empty(cls, layers: int, length: int, d_model: int) -> "KvCache":
        return cls(np.zeros((layers, length, d_model)), np.zeros((layers, length, d_model)),
                   np.zeros(length, dtype=bool))

    def _host(self):
        if self._keys is None:
            layers, L, kvd = self._shape
            a = self._vec.view(layers, L, 2, kvd).double().cpu().numpy()
            self._keys, self._values = a[:, :, 0, :].copy(), a[:, :, 1, :].copy()
            self._vec = None  # host arrays are authoritative from now on
        return self._keys, self._values

    @property
    def keys(self) -> np.ndarray:
        return self._host()[0]

    @keys.setter
    def keys(self, v):
        self._host()
        self._keys = np.asarray(v)

    @property
    def values(self) -> np.ndarray:
        return self._host()[1]

    @values.setter
    def values(self, v):
        self._host()
        self._values = np.asarray(v)

    @property
    def length(self) -> int:
        return self._shape[1]

    @property
    def shape(self) -> tuple:
        return self._shape

    def device_vec(self):
        """The cache as a CUDA fp32 vector in kv_vectorize layout (uploaded if host-resident)."""
        if self._vec is None:
            import torch
            k, v = self._keys, self._values
            self._shape = tuple(k.shape)
            self._vec = torch.from_numpy(np.ascontiguousarray(np.stack([k, v], axis=2), dtype=np.float32)
                                         .reshape(-1)).to("cuda")
            return self._vec
        return self._vec

    def copy(self) -> "KvCache":
        if self._keys is not None:
            return KvCache(self._keys.copy(), self._values.copy(), self.valid.copy())
        return KvCache(vec=self._vec.clone(), shape=self._shape, valid=self.valid.copy())


def kv_vectorize(cache: KvCache) -> np.ndarray:
    """model.py:346-352: layer-major, position-minor, key before value."""
    if not np.asarray(cache.valid).all():
        raise StateError("cannot vectorize a cache with invalid positions")
    if cache._keys is None:
        return cache._vec.double().cpu().numpy()
    layers, length, d = cache.keys.shape
    return np.stack([cache.keys, cache.values], axis=2).reshape(layers * length * 2 * d).copy()


def full_forward(params: "ModelParams", row: SequenceRow, target) -> tuple:
    """model.py:322-328 on the device: the whole row from an empty cache;
    DenoiseOutput over every masked position plus the new KvCache."""
    from . import seams
    return seams.full_forward(params, row, target)


def block_forward(params: "ModelParams", row: SequenceRow, cache: KvCache, window: BlockWindow, target) -> tuple:
    """model.py:331-343 on the device: recompute the window's K/V only, attend
    to ``cache`` everywhere else; DenoiseOutput over the window's masked
    positions plus the new KvCache (copy-then-write: ``cache`` is unchanged)."""
    from . import seams
    return seams.block_forward(params, row, cache, window, target)


@dataclass(frozen=True)
class Task:
    """A seeded synthetic request (model.py:183-207)."""

    seed: int
    prompt: np.ndarray
    target: np.ndarray

    @property
    def prompt_len(self) -> int:
        return len(self.prompt)

    @property
    def gen_len(self) -> int:
        return len(self.target)

    def fresh_row(self, vocab: Vocab) -> SequenceRow:
        tokens = np.full(self.prompt_len + self.gen_len, vocab.mask_id, dtype=np.int64)
        tokens[:self.prompt_len] = self.prompt
        return SequenceRow(tokens, self.prompt_len)

    def effective_len(self, vocab: Vocab) -> int:
        eos = np.flatnonzero(self.target == vocab.eos_id)
        return int(eos[0]) + 1 if len(eos) else self.gen_len


def make_task(seed: int, prompt_len: int, gen_len: int, vocab: Vocab) -> Task:
    """model.py:363-374: Philox(key=(seed<<16)+0x7A5); eos planted w.p. 0.5 in [G/4, G)."""
    if prompt_len < 1 or gen_len < 1:
        raise ConfigError("prompt_len and gen_len must be positive")
    rng = np.random.Generator(np.random.Philox(key=(seed << 16) + 0x7A5))
    prompt = rng.integers(0, vocab.size, size=prompt_len, dtype=np.int64)
    target = rng.integers(0, vocab.size, size=gen_len, dtype=np.int64)
    if gen_len >= 4 and rng.random() < 0.5:
        eos_pos = int(rng.integers(gen_len // 4, gen_len))
        target[eos_pos] = vocab.eos_id
    return Task(seed=seed, prompt=prompt, target=target)


def exact_match(row: SequenceRow, task: Task, vocab: Vocab) -> bool:
    """model.py:377-381"""
    eff = task.effective_len(vocab)
    gen = row.tokens[row.prompt_len:row.prompt_len + eff]
    return bool(np.array_equal(gen, task.target[:eff]))


# --------------------------------------------------------------------------
# device parameters
# --------------------------------------------------------------------------

TID_EMB, TID_POS, TID_HEAD = 1, 2, 3
TID_WQKV, TID_BQKV, TID_WO, TID_WG, TID_WU, TID_WD = 16, 17, 18, 19, 20, 21


def _tid(base: int, layer: int) -> int:
    return base + 64 * (layer + 1)


@dataclass(frozen=True, eq=False)
class ModelParams:
    """Immutable seeded weights (model.py:115-133), resident on the GPU.

    ``weights`` holds torch CUDA tensors in the C-ABI layout (include/bb200.h
    bb_weights).  For ``init="philox"`` the reference's float64 matrices are
    kept on the host too (emb, pos, wq, wk, wv, wo, w_head) so
    ``serialize_params`` stays byte-compatible."""

    seed: int
    vocab: Vocab
    dims: ModelDims
    gamma: float
    radius: int
    head_scale: float
    spike_cut: float
    spike_gain: float
    dtype: str
    init: str
    weights: dict
    emb: np.ndarray | None = None
    pos: np.ndarray | None = None
    wq: tuple = ()
    wk: tuple = ()
    wv: tuple = ()
    wo: tuple = ()
    w_head: np.ndarray | None = None
    _handle: list = field(default_factory=lambda: [None], repr=False)
    _sessions: dict = field(default_factory=dict, repr=False)  # device sessions (scheduler.get_session)

    def clear_sessions(self) -> None:
        """Drop this model's cached device sessions (their workspaces free with them)."""
        self._sessions.clear()

    def desc(self) -> _lib.ModelDesc:
        d = self.dims
        return _lib.ModelDesc(
            arch=_lib.ARCH_REF if d.arch == "ref" else _lib.ARCH_LLADA, vocab_size=self.vocab.size,
            layers=d.layers, d_model=d.d_model, n_heads=d.n_heads, n_kv_heads=d.n_kv_heads, head_dim=d.hd,
            d_ff=d.d_ff, max_len=d.max_len, qkv_bias=int(d.qkv_bias),
            dtype={"f32": _lib.DTYPE_F32, "bf16": _lib.DTYPE_BF16, "bf16x2": _lib.DTYPE_BF16X2}[self.dtype],
            rope_theta=d.rope_theta,
            norm_eps=d.norm_eps, gamma=self.gamma, radius=self.radius, head_scale=self.head_scale,
            spike_cut=self.spike_cut, spike_gain=self.spike_gain)

    def handle(self):
        """The C-ABI model (bb_model_create), created on first use."""
        if self._handle[0] is None:
            w = self.weights

            def p(name):
                t = w.get(name)
                return None if t is None else C.c_void_p(t.data_ptr())
            cw = _lib.Weights(emb=p("emb"), pos=p("pos"), wqkv=p("wqkv"), bqkv=p("bqkv"), wo=p("wo"),
                              wgu=p("wgu"), wd=p("wd"), ln1=p("ln1"), ln2=p("ln2"), lnf=p("lnf"), head=p("head"))
            h = C.c_void_p()
            desc = self.desc()
            _lib.check(_lib.lib().bb_model_create(C.byref(desc), C.byref(cw), C.byref(h)), "bb_model_create")
            self._handle[0] = h
        return self._handle[0]

    def __del__(self):
        try:
            self._sessions.clear()
            if self._handle[0] is not None and _lib._lib is not None:
                _lib._lib.bb_model_destroy(self._handle[0])
        except Exception:
            pass

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.weights.values())


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise StateError("ModelParams live on the GPU: no CUDA device available")
    return torch


def build_model(seed: int, vocab: Vocab, dims: ModelDims = ModelDims(), gamma: float = 8.0, radius: int = 4,
                head_scale: float = 1.0, spike_cut: float = 0.72, spike_gain: float = 33.0,
                dtype: str = "f32", init: str | None = None) -> ModelParams:
    """model.py:210-241 on the device.  ``dtype``: "f32" (verification mode:
    fp32 weights / activations / KV, SIMT kernels), "bf16" (bf16 weights,
    activations and KV; tcgen05) or "bf16x2" (bf16 weights; every activation,
    q/K/V and head input kept as a bf16 hi + lo pair that the tcgen05 MMAs
    consume both halves of -- fp32-grade activations at bf16 weight traffic;
    LLaDA/Dream shape with head_dim 128).  ``init`` "philox" (reference draw,
    default for arch "ref") or "hash" (device counter hash, default for arch
    "llada")."""
    if dims.layers < 1 or dims.d_model < 1 or dims.max_len < 1:
        raise ConfigError(f"non-positive model dimensions: {dims}")
    if dtype not in ("f32", "bf16", "bf16x2"):
        raise ConfigError(f"unknown dtype {dtype!r}")
    if dtype == "bf16x2" and (dims.arch != "llada" or dims.hd != 128):
        raise ConfigError("bf16x2 needs the LLaDA/Dream architecture with head_dim 128")
    init = init or ("philox" if dims.arch == "ref" else "hash")
    if dims.arch == "ref" and (dims.n_heads != 1 or dims.hd != dims.d_model or dims.d_ff):
        raise ConfigError("the reference architecture is single-head, head_dim = d_model, no MLP")
    torch = _torch()
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    kw = dict(seed=seed, vocab=vocab, dims=dims, gamma=gamma, radius=radius, head_scale=head_scale,
              spike_cut=spike_cut, spike_gain=spike_gain, dtype=dtype, init=init)
    if init == "philox":
        if dims.arch != "ref":
            raise ConfigError("philox init is defined for the reference architecture only")
        rng = np.random.Generator(np.random.Philox(key=seed))
        scale = 1.0 / np.sqrt(dims.d_model)
        d = dims.d_model

        def mat(r, c):
            return rng.standard_normal((r, c)) * scale
        emb = mat(vocab.n_extended, d)
        pos = mat(dims.max_len, d)
        wq, wk, wv, wo = [], [], [], []
        for _ in range(dims.layers):
            wq.append(mat(d, d))
            wk.append(mat(d, d))
            wv.append(mat(d, d))
            wo.append(mat(d, d))
        w_head = mat(d, vocab.n_out)

        def dev(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to("cuda").to(tdt).contiguous()
        weights = {"emb": dev(emb), "pos": dev(pos),
                   "wqkv": dev(np.stack([np.concatenate([q.T, k.T, v.T], 0) for q, k, v in zip(wq, wk, wv)])),
                   "wo": dev(np.stack([o.T for o in wo])), "head": dev(w_head.T)}
        return ModelParams(weights=weights, emb=emb, pos=pos, wq=tuple(wq), wk=tuple(wk), wv=tuple(wv),
                           wo=tuple(wo), w_head=w_head, **kw)
    if init != "hash":
        raise ConfigError(f"unknown init {init!r}")
    weights = _hash_weights(torch, vocab, dims, seed, dtype)
    return ModelParams(weights=weights, **kw)


def verification_copy(params: ModelParams) -> ModelParams:
    """The same model in fp32 verification mode: every weight upcast exactly
    (a bf16 model's fp32 twin holds the identical bf16-rounded values), so a
    bf16 run and its verification run differ only in arithmetic."""
    if params.dtype == "f32":
        return params
    weights = {k: v.float() for k, v in params.weights.items()}
    from dataclasses import replace
    return replace(params, dtype="f32", weights=weights, _handle=[None], _sessions={})


def _hash_weights(torch, vocab: Vocab, dims: ModelDims, seed: int, dtype: str) -> dict:
    dtype = "bf16" if dtype == "bf16x2" else dtype  # bf16x2 keeps bf16 weights
    L = _lib.lib()
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    cdt = _lib.DTYPE_F32 if dtype == "f32" else _lib.DTYPE_BF16
    d, dff, hd = dims.d_model, dims.d_ff, dims.hd
    attn = dims.n_heads * hd
    sd = 1.0 / np.sqrt(d)
    s = torch.cuda.current_stream().cuda_stream

    def fill(t, tid, scale, mode=0, start=0, fdt=None):
        c = float(np.float32(np.sqrt(3.0) * scale))
        _lib.check(L.bb_fill_hash_uniform(C.c_void_p(t.data_ptr()), cdt if fdt is None else fdt, t.numel(), seed,
                                          tid, c, start, mode, d, C.c_void_p(s)), "bb_fill_hash_uniform")
        return t

    W = {"emb": fill(torch.empty(vocab.n_extended, d, dtype=tdt, device="cuda"), TID_EMB, sd),
         "head": fill(torch.empty(vocab.n_out, d, dtype=tdt, device="cuda"), TID_HEAD, sd)}
    if dims.arch == "ref":
        W["pos"] = fill(torch.empty(dims.max_len, d, dtype=tdt, device="cuda"), TID_POS, sd)
    W["wqkv"] = torch.empty(dims.layers, dims.qkv_out, d, dtype=tdt, device="cuda")
    W["wo"] = torch.empty(dims.layers, d, attn, dtype=tdt, device="cuda")
    if dims.qkv_bias:
        W["bqkv"] = torch.empty(dims.layers, dims.qkv_out, dtype=torch.float32, device="cuda")
    if dff:
        W["wgu"] = torch.empty(dims.layers, 2 * dff, d, dtype=tdt, device="cuda")
        W["wd"] = torch.empty(dims.layers, d, dff, dtype=tdt, device="cuda")
    for l in range(dims.layers):
        fill(W["wqkv"][l], _tid(TID_WQKV, l), sd)
        fill(W["wo"][l], _tid(TID_WO, l), 1.0 / np.sqrt(attn))
        if dims.qkv_bias:
            fill(W["bqkv"][l], _tid(TID_BQKV, l), sd, fdt=_lib.DTYPE_F32)
        if dff:
            fill(W["wgu"][l], _tid(TID_WG, l), sd, mode=1)
            fill(W["wd"][l], _tid(TID_WD, l), 1.0 / np.sqrt(dff))
    if dims.arch == "llada":
        W["ln1"] = torch.ones(dims.layers, d, dtype=torch.float32, device="cuda")
        W["ln2"] = torch.ones(dims.layers, d, dtype=torch.float32, device="cuda")
        W["lnf"] = torch.ones(d, dtype=torch.float32, device="cuda")
    return W


def serialize_params(params: ModelParams) -> bytes:
    """model.py:384-391 (reference-initialised models only)."""
    if params.emb is None:
        raise StateError("serialize_params needs host weights (init='philox')")
    parts = [params.emb, params.pos]
    for layer in range(params.dims.layers):
        parts.extend([params.wq[layer], params.wk[layer], params.wv[layer], params.wo[layer]])
    parts.append(params.w_head)
    return b"".join(np.ascontiguousarray(p, dtype="<f8").tobytes() for p in parts)

"""ORACLE — test infrastructure only (never imported by the product path).

CPU restatement (numpy, fp32 activations, bf16-rounded weights) of what the
B200 engine computes for the experience-collection path:

  * synthetic weights / prompts / forced responses from the same integer hash
    as csrc/kernels/philox.cuh (bit-identical bf16 weights);
  * Llama-style forward: RMSNorm (eps 1e-5, fp32 gain), rotate-half RoPE
    (theta 1e4), causal softmax attention with GQA, SwiGLU MLP, untied LM head
    (actor / reference) or a d -> 1 value head (critic / reward);
  * actor log-probs of the response tokens (teacher-forced: the full causal
    forward equals incremental decode), greedy incremental decode with a KV
    cache (for the token agreement rate), exact two-level inverse-CDF sampling
    (half-tile by mass, then inside it) replayed in the kernel's fp32 summation
    order with the same Philox4x32-10 streams as the GPU sampler;
  * reference log-probs, critic values at positions P-1 .. P+R-2, reward score
    at position P+R-1;
  * post-processing: KL, reward shaping, GAE (the recursion of
    proj/src/numerics.cpp:27-34 with the explicit V_R = 0 bootstrap), returns
    (oracle/post_oracle.c restates the same in C).

PPO/KL and transformer math do not exist in the reference (SPEC.md:512 — an
explicit non-goal), so for those quantities parity is pinned only by this
oracle ("parity unpinned by the reference"); the GAE part is pinned against
the reference's golden vectors and library (tests/test_oracle.py).
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
TAG_EMBED, TAG_WQKV, TAG_WO, TAG_WGU, TAG_WD, TAG_LN1, TAG_LN2, TAG_LNF, TAG_HEAD, TAG_VHEAD = range(1, 11)
TAG_PROMPT, TAG_RESPONSE = 0xF1, 0xF2
ACTOR, REF, CRITIC, REWARD = 0, 1, 2, 3


def weight_tag(model: int, layer: int, kind: int) -> int:
    return (model << 24) | (layer << 8) | kind


def hash3(seed: int, tag: int, idx: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser of (seed, tag, index) — philox.cuh:hash3."""
    z0 = (seed ^ ((tag * 0xD1B54A32D192ED03) & M64)) & M64
    z = np.uint64(z0) + (idx.astype(np.uint64) + np.uint64(1)) * np.uint64(GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def unit24(h: np.ndarray) -> np.ndarray:
    return (h >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)


def to_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as fp32 values."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32)


_CLIB = None


def _clib():
    """oracle/_ref/liboracle_c.so (oracle/weights_oracle.c): the same values, threaded."""
    global _CLIB
    if _CLIB is None:
        import ctypes
        import os
        from pathlib import Path
        p = Path(__file__).resolve().parent / "_ref" / "liboracle_c.so"
        _CLIB = False
        if p.exists() and not os.environ.get("FP_ORACLE_NUMPY_WEIGHTS"):
            lib = ctypes.CDLL(str(p))
            if hasattr(lib, "oracle_uniform_weight"):
                f = ctypes.POINTER(ctypes.c_float)
                lib.oracle_uniform_weight.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_float,
                                                      f, ctypes.c_int]
                lib.oracle_gain.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, f, ctypes.c_int]
                _CLIB = lib
    return _CLIB or None


def _threads() -> int:
    import os
    return max(1, min(32, len(os.sched_getaffinity(0))))


def uniform_weight_np(seed, tag, n, scale) -> np.ndarray:
    t = unit24(hash3(seed, tag, np.arange(n, dtype=np.uint64))) * np.float32(2.0) - np.float32(1.0)
    return to_bf16(t * np.float32(scale))


def gain_np(seed, tag, n) -> np.ndarray:
    t = unit24(hash3(seed, tag, np.arange(n, dtype=np.uint64))) * np.float32(2.0) - np.float32(1.0)
    return np.float32(1.0) + np.float32(0.1) * t


def uniform_weight(seed, tag, n, scale) -> np.ndarray:
    lib = _clib()
    if lib is None:
        return uniform_weight_np(seed, tag, n, scale)
    import ctypes
    out = np.empty(n, dtype=np.float32)
    lib.oracle_uniform_weight(seed, tag, n, float(np.float32(scale)), out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                              _threads())
    return out


def gain(seed, tag, n) -> np.ndarray:
    lib = _clib()
    if lib is None:
        return gain_np(seed, tag, n)
    import ctypes
    out = np.empty(n, dtype=np.float32)
    lib.oracle_gain(seed, tag, n, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), _threads())
    return out


def fsqrt(x) -> np.float32:
    return np.sqrt(np.float32(x))


def make_weights(dims, model: int, seed: int) -> dict:
    """Same tensors, same bits as Engine::init_model (engine.cpp)."""
    L, d, H, KVH, hd, F, V = (dims.num_layers, dims.hidden, dims.num_heads, dims.num_kv_heads, dims.head_dim,
                              dims.ffn, dims.vocab)
    qw, ao = (H + 2 * KVH) * hd, H * hd
    W = {"dims": dims, "embed": uniform_weight(seed, weight_tag(model, 0, TAG_EMBED), V * d, 1.0).reshape(V, d),
         "layers": []}
    for l in range(L):
        gu = uniform_weight(seed, weight_tag(model, l, TAG_WGU), 2 * F * d, fsqrt(np.float32(3.0) / np.float32(d)))
        gu = gu.reshape(2 * F, d)
        W["layers"].append({
            "wqkv": uniform_weight(seed, weight_tag(model, l, TAG_WQKV), qw * d,
                                   fsqrt(np.float32(3.0) / np.float32(d))).reshape(qw, d),
            "wo": uniform_weight(seed, weight_tag(model, l, TAG_WO), d * ao,
                                 fsqrt(np.float32(3.0) / np.float32(ao))).reshape(d, ao),
            "wg": gu[:F], "wu": gu[F:],
            "wd": uniform_weight(seed, weight_tag(model, l, TAG_WD), d * F,
                                 fsqrt(np.float32(3.0) / np.float32(F))).reshape(d, F),
            "ln1": gain(seed, weight_tag(model, l, TAG_LN1), d),
            "ln2": gain(seed, weight_tag(model, l, TAG_LN2), d),
        })
    W["lnf"] = gain(seed, weight_tag(model, 0, TAG_LNF), d)
    if model in (ACTOR, REF):
        W["head"] = uniform_weight(seed, weight_tag(model, 0, TAG_HEAD), V * d,
                                   fsqrt(np.float32(3.0) / np.float32(d))).reshape(V, d)
    else:
        W["vhead"] = uniform_weight(seed, weight_tag(model, 0, TAG_VHEAD), d, fsqrt(np.float32(3.0) / np.float32(d)))
    return W


def synthetic_prompts(n: int, max_prompt: int, vocab: int, token_seed: int) -> np.ndarray:
    h = hash3(token_seed, TAG_PROMPT, np.arange(n * max_prompt, dtype=np.uint64))
    return ((h >> np.uint64(32)) % np.uint64(vocab)).astype(np.int64).reshape(n, max_prompt)


def forced_response(sid: int, R: int, max_new: int, vocab: int, token_seed: int) -> np.ndarray:
    idx = np.uint64(sid * max_new) + np.arange(R, dtype=np.uint64)
    return ((hash3(token_seed, TAG_RESPONSE, idx) >> np.uint64(32)) % np.uint64(vocab)).astype(np.int64)


# ---------------------------------------------------------------------------
# forward pieces (fp32)

def rmsnorm(x, g):
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + np.float32(1e-5)) * g


def rope(x, pos, theta=10000.0):
    """x [T, heads, hd] fp32, pos [T]; rotate-half pairs (i, i + hd/2)."""
    hd = x.shape[-1]
    half = hd // 2
    i = np.arange(half, dtype=np.float32)
    inv = np.exp2(-(np.float32(2.0) * i / np.float32(hd)) * np.float32(math.log2(theta))).astype(np.float32)
    ang = pos.astype(np.float32)[:, None] * inv[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def silu(x):
    return x / (np.float32(1.0) + np.exp(-x))


def forward(W, tokens: np.ndarray) -> np.ndarray:
    """Full causal forward of one sequence; returns the final normed hidden [T, d]."""
    D = W["dims"]
    H, KVH, hd = D.num_heads, D.num_kv_heads, D.head_dim
    T = len(tokens)
    x = W["embed"][tokens].astype(np.float32)
    pos = np.arange(T)
    mask = np.triu(np.full((T, T), -np.inf, dtype=np.float32), 1)
    for Lw in W["layers"]:
        h = rmsnorm(x, Lw["ln1"])
        qkv = h @ Lw["wqkv"].T
        q = qkv[:, :H * hd].reshape(T, H, hd)
        k = qkv[:, H * hd:(H + KVH) * hd].reshape(T, KVH, hd)
        v = qkv[:, (H + KVH) * hd:].reshape(T, KVH, hd)
        q, k = rope(q, pos), rope(k, pos)
        g = H // KVH
        k = np.repeat(k, g, axis=1)
        v = np.repeat(v, g, axis=1)
        s = np.einsum("thd,shd->hts", q, k) / np.float32(math.sqrt(hd)) + mask[None]
        s = s - s.max(-1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(-1, keepdims=True)
        o = np.einsum("hts,shd->thd", p, v).reshape(T, H * hd)
        x = x + o @ Lw["wo"].T
        h = rmsnorm(x, Lw["ln2"])
        x = x + (silu(h @ Lw["wg"].T) * (h @ Lw["wu"].T)) @ Lw["wd"].T
    return rmsnorm(x, W["lnf"])


def log_softmax(z):
    m = z.max(-1, keepdims=True)
    return z - m - np.log(np.exp(z - m).sum(-1, keepdims=True))


# ---------------------------------------------------------------------------
# Philox4x32-10 + two-level inverse-CDF sampling (the GPU sampler's streams)

def philox4x32_10(ctr: np.ndarray, k0: int, k1: int) -> np.ndarray:
    """ctr uint32 [..., 4] -> uint32 [..., 4]."""
    c = ctr.astype(np.uint64)
    k0 = np.uint64(k0 & 0xFFFFFFFF)
    k1 = np.uint64(k1 & 0xFFFFFFFF)
    m32 = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = np.uint64(0xD2511F53) * c[..., 0]
        p1 = np.uint64(0xCD9E8D57) * c[..., 2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & m32
        hi1, lo1 = p1 >> np.uint64(32), p1 & m32
        c = np.stack([(hi1 ^ c[..., 1] ^ k0) & m32, lo1, (hi0 ^ c[..., 3] ^ k1) & m32, lo0], axis=-1)
        k0 = (k0 + np.uint64(0x9E3779B9)) & m32
        k1 = (k1 + np.uint64(0xBB67AE85)) & m32
    return c.astype(np.uint32)


def _unit(w) -> np.float32:
    return (np.float32(int(w) >> 8) + np.float32(0.5)) * np.float32(1.0 / 16777216.0)


def _philox1(seed: int, c0: int, step: int, sid: int) -> int:
    return int(philox4x32_10(np.array([[c0, step, sid, 0xF00D]], dtype=np.uint32), seed & 0xFFFFFFFF,
                             (seed >> 32) & 0xFFFFFFFF)[0, 0])


def vocab_partials(z: np.ndarray, inv_temp_is_applied: bool = True, c2: np.float32 | None = None):
    """Per (256-column tile, 128-column half) statistics of one row, in the GPU's
    column order (half h owns chunks c0 = 32h, 32h + 64, ...): (m2, s, columns)."""
    V = len(z)
    out = []
    for t in range((V + 255) // 256):
        for h in range(2):
            cols = [256 * t + c0 + j for c0 in range(32 * h, 256, 64) for j in range(32) if 256 * t + c0 + j < V]
            out.append(cols)
    return out


def sample_token(logits: np.ndarray, inv_temp: float, seed: int, sid: int, step: int):
    """Two-level exact sampling of csrc/kernels/vocab.cuh (half-tile by mass, then
    inverse CDF inside it), replayed in fp32 in the kernel's summation order."""
    c2 = np.float32(inv_temp) * np.float32(1.4426950408889634)
    z2 = logits.astype(np.float32) * c2
    parts = []
    for pi, cols in enumerate(vocab_partials(logits)):
        if not cols:
            parts.append((np.float32(-np.inf), np.float32(0), -1))
            continue
        m = np.float32(-np.inf)
        s = np.float32(0)
        for k in range(0, len(cols), 32):  # chunk-wise online max / sum, as the epilogue
            ch = z2[cols[k:k + 32]]
            nm = max(m, ch.max())
            acc = np.float32(0) if m == -np.inf else np.float32(s * np.exp2(np.float32(m - nm)))
            for x in ch:
                acc = np.float32(acc + np.exp2(np.float32(x - nm)))
            m, s = nm, acc
        thr = _unit(_philox1(seed, pi, step, sid)) * s
        acc = np.float32(0)
        pick = cols[-1]
        for c in cols:
            acc = np.float32(acc + np.exp2(np.float32(z2[c] - m)))
            pick = c
            if acc >= thr:
                break
        parts.append((m, s, pick))
    # finalize (gemm.cu vocab_finalize_kernel): lane l of a warp owns the
    # contiguous half-tiles [l*C, (l+1)*C); lane sums, then lanes in order
    M = max(p[0] for p in parts)
    n = len(parts)
    C = (n + 31) // 32
    chunks = [range(min(n, l * C), min(n, l * C + C)) for l in range(32)]

    def w(t):
        return np.float32(parts[t][1] * np.exp2(np.float32(parts[t][0] - M)))

    lane_sum = []
    for ch in chunks:
        c = np.float32(0)
        for t in ch:
            if parts[t][0] != -np.inf:
                c = np.float32(c + w(t))
        lane_sum.append(c)
    tot = np.float32(0)
    for c in lane_sum:
        tot = np.float32(tot + c)
    thr = np.float32(_unit(_philox1(seed, 0xFFFFFFFF, step, sid)) * tot)
    acc = base = np.float32(0)
    pl = -1
    for l, c in enumerate(lane_sum):
        base = acc
        acc = np.float32(acc + c)
        if acc >= thr and c > 0:
            pl = l
            break
    if pl < 0:
        pl = 31
    acc = base
    tok = -1
    for t in chunks[pl]:
        if parts[t][0] == -np.inf:
            continue
        acc = np.float32(acc + w(t))
        tok = parts[t][2]
        if acc >= thr:
            break
    return tok


def _order_key(z: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(z, dtype=np.float32).view(np.uint32).astype(np.uint64)
    neg = (b & np.uint64(0x80000000)) != 0
    return np.where(neg, (~b) & np.uint64(0xFFFFFFFF), b | np.uint64(0x80000000))


def filtered_sample(z: np.ndarray, top_k: int, top_p: float, seed: int, sid: int, step: int, k_max: int = 1024):
    """Top-k / top-p sampling of csrc/kernels/sampling.cu on one row of z = logit / T
    (fp32), in the kernel's order: candidates = every z >= the k-th largest
    (ties kept), sorted by (z desc, id asc); masses 2^((z - z_0) log2 e) summed
    in 32 lane-contiguous chunks; nucleus = the shortest prefix reaching
    top_p of the candidates' mass; inverse-CDF draw at u * mass(nucleus),
    u = Philox(seed; 0xFFFFFFFE, step, sid, 0xF00D). Returns (token, kept ids)."""
    z = np.asarray(z, dtype=np.float32)
    V = len(z)
    k = min(V, min(top_k, k_max) if top_k > 0 else k_max)
    key = _order_key(z)
    kth = np.sort(key)[::-1][k - 1]
    ids = np.flatnonzero(key >= kth)
    ids = ids[np.lexsort((ids, -key[ids].astype(np.int64)))]  # key desc, id asc
    n = len(ids)
    e = np.exp2((z[ids] - z[ids[0]]).astype(np.float32) * np.float32(1.4426950408889634)).astype(np.float32)
    chunk = (n + 31) // 32
    csum = np.zeros(n, dtype=np.float32)
    lane_sum = []
    for l in range(32):
        c0, c1 = min(n, l * chunk), min(n, l * chunk + chunk)
        run = np.float32(0)
        for i in range(c0, c1):
            run = np.float32(run + e[i])
            csum[i] = run
        lane_sum.append(run)
    base = np.float32(0)
    for l in range(32):
        c0, c1 = min(n, l * chunk), min(n, l * chunk + chunk)
        for i in range(c0, c1):
            csum[i] = np.float32(csum[i] + base)
        base = np.float32(base + lane_sum[l])
    cut = n - 1
    if top_p < 1.0:
        need = np.float32(np.float32(top_p) * csum[n - 1])
        hit = np.flatnonzero(csum >= need)
        cut = min(int(hit[0]) if len(hit) else n, n - 1)
    thr = np.float32(_unit(_philox1(seed, 0xFFFFFFFE, step, sid)) * csum[cut])
    hit = np.flatnonzero(csum[:cut + 1] >= thr)
    sel = min(int(hit[0]) if len(hit) else cut + 1, cut)
    return int(ids[sel]), set(int(i) for i in ids[:cut + 1])


# ---------------------------------------------------------------------------
# experience

def gae(rewards, values, gamma, lam):
    """gae_recursive of proj/src/numerics.cpp:11-34: values has T+1 entries."""
    r, v = np.asarray(rewards, dtype=np.float64), np.asarray(values, dtype=np.float64)
    if len(r) < 1 or len(v) != len(r) + 1 or not (0 <= gamma <= 1 and 0 <= lam <= 1):
        raise ValueError("GaeInputs: need T >= 1 rewards, T+1 values, gamma and lam in [0, 1]")
    adv = r + gamma * v[1:] - v[:-1]
    c = gamma * lam
    for t in range(len(r) - 2, -1, -1):
        adv[t] += c * adv[t + 1]
    return adv


def postprocess(logp_actor, logp_ref, values, score, beta, gamma, lam):
    """fp64 KL / reward / GAE (explicit V_R = 0 bootstrap) / returns of one sample."""
    la, lr, v = (np.asarray(a, dtype=np.float64) for a in (logp_actor, logp_ref, values))
    kl = la - lr
    rew = -beta * kl
    rew[-1] += score
    adv = gae(rew, np.append(v, 0.0), gamma, lam)
    return {"kl": kl, "reward": rew, "adv": adv, "ret": adv + v}


class Oracle:
    """The four synthetic models of one workload."""

    def __init__(self, workload, weight_seed: int = 1234):
        self.w = workload
        self.models = [make_weights(workload.actor, ACTOR, weight_seed), make_weights(workload.ref, REF, weight_seed),
                       make_weights(workload.critic, CRITIC, weight_seed),
                       make_weights(workload.reward, REWARD, weight_seed)]

    def score_sample(self, prompt: np.ndarray, response: np.ndarray, temperature: float = 1.0) -> dict:
        """Teacher-forced pass of one (prompt, response): every per-token quantity."""
        toks = np.concatenate([prompt, response])
        P, R = len(prompt), len(response)
        rows = np.arange(P - 1, P + R - 1)
        out = {}
        for name, m in (("logp_actor", ACTOR), ("logp_ref", REF)):
            h = forward(self.models[m], toks)[rows]
            z = (h @ self.models[m]["head"].T) / np.float32(temperature if name == "logp_actor" else 1.0)
            out[name] = log_softmax(z)[np.arange(R), response]
        hc = forward(self.models[CRITIC], toks)
        out["values"] = hc[rows] @ self.models[CRITIC]["vhead"]
        hr = forward(self.models[REWARD], toks)
        out["score"] = float(hr[-1] @ self.models[REWARD]["vhead"])
        return out

    def experience(self, prompt, response, beta, gamma, lam, temperature=1.0) -> dict:
        s = self.score_sample(prompt, response, temperature)
        s.update(postprocess(s["logp_actor"], s["logp_ref"], s["values"], s["score"], beta, gamma, lam))
        s["tokens"] = np.asarray(response)
        return s

    def decode(self, prompt: np.ndarray, R: int, mode: str = "greedy", sample_id: int = 0, seed: int = 11,
               temperature: float = 1.0) -> tuple:
        """Incremental decode of R tokens (KV cache); returns (tokens, logps)."""
        W = self.models[ACTOR]
        D = W["dims"]
        H, KVH, hd = D.num_heads, D.num_kv_heads, D.head_dim
        g = H // KVH
        toks = list(prompt)
        out_t, out_lp = [], []
        K = [np.zeros((0, KVH, hd), np.float32) for _ in W["layers"]]
        Vc = [np.zeros((0, KVH, hd), np.float32) for _ in W["layers"]]

        def step(tok_ids, pos0):
            T = len(tok_ids)
            x = W["embed"][np.asarray(tok_ids)].astype(np.float32)
            pos = np.arange(pos0, pos0 + T)
            for li, Lw in enumerate(W["layers"]):
                h = rmsnorm(x, Lw["ln1"])
                qkv = h @ Lw["wqkv"].T
                q = rope(qkv[:, :H * hd].reshape(T, H, hd), pos)
                k = rope(qkv[:, H * hd:(H + KVH) * hd].reshape(T, KVH, hd), pos)
                v = qkv[:, (H + KVH) * hd:].reshape(T, KVH, hd)
                K[li] = np.concatenate([K[li], k])
                Vc[li] = np.concatenate([Vc[li], v])
                kk, vv = np.repeat(K[li], g, axis=1), np.repeat(Vc[li], g, axis=1)
                S = K[li].shape[0]
                s = np.einsum("thd,shd->hts", q, kk) / np.float32(math.sqrt(hd))
                s = s + np.triu(np.full((T, S), -np.inf, np.float32), S - T + 1)[None]
                s = s - s.max(-1, keepdims=True)
                p = np.exp(s)
                p /= p.sum(-1, keepdims=True)
                o = np.einsum("hts,shd->thd", p, vv).reshape(T, H * hd)
                x = x + o @ Lw["wo"].T
                h = rmsnorm(x, Lw["ln2"])
                x = x + (silu(h @ Lw["wg"].T) * (h @ Lw["wu"].T)) @ Lw["wd"].T
            return rmsnorm(x[-1:], W["lnf"])[0]

        if len(toks) > 1:
            step(toks[:-1], 0)
        cur, pos = toks[-1], len(toks) - 1
        for k in range(R):
            h = step([cur], pos)
            z = (h @ W["head"].T) / np.float32(temperature)
            lp = log_softmax(z)
            if mode == "greedy":
                t = int(np.argmax(z))
            else:
                t = sample_token(h @ W["head"].T, 1.0 / temperature, seed, sample_id, k)
            out_t.append(t)
            out_lp.append(float(lp[t]))
            cur, pos = t, pos + 1
        return np.asarray(out_t), np.asarray(out_lp)


class CppOracle:
    """oracle/_ref/liboracle_cpu.so (oracle/cpu_oracle.cpp): the same experience in
    fp32 C++, std::thread over samples — the timed CPU path of bench.py."""

    def __init__(self, workload, weight_seed: int = 1234, threads: int | None = None):
        import ctypes as C
        import os
        from pathlib import Path
        p = Path(__file__).resolve().parent / "_ref" / "liboracle_cpu.so"
        if not p.exists():
            raise FileNotFoundError(f"{p} not built (make -C oracle liboracle)")
        self.lib = C.CDLL(str(p))
        self.lib.cpu_oracle_create.restype = C.c_void_p
        self.lib.cpu_oracle_create.argtypes = [C.POINTER(C.c_int32), C.c_uint64, C.c_int32]
        self.lib.cpu_oracle_destroy.argtypes = [C.c_void_p]
        i32 = C.POINTER(C.c_int32)
        f32 = C.POINTER(C.c_float)
        self.lib.cpu_oracle_experience.argtypes = [C.c_void_p, C.c_int32, C.c_int32, i32, i32, i32, i32, C.c_float,
                                                   C.c_float, C.c_float, C.c_int32, f32, f32]
        self.threads = threads or len(os.sched_getaffinity(0))
        dims = []
        for d in (workload.actor, workload.ref, workload.critic, workload.reward):
            dims += [d.num_layers, d.hidden, d.num_heads, d.num_kv_heads, d.head_dim, d.ffn, d.vocab]
        arr = (C.c_int32 * 28)(*dims)
        self.h = self.lib.cpu_oracle_create(arr, weight_seed, self.threads)
        self.C = C

    def close(self):
        if getattr(self, "h", None):
            self.lib.cpu_oracle_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def experience_batch(self, prompts, prompt_len, responses, beta, gamma, lam):
        """prompts [n][max_prompt], prompt_len [n], responses: list of arrays -> dict of packed arrays."""
        C = self.C
        prompts = np.ascontiguousarray(prompts, dtype=np.int32)
        n, maxp = prompts.shape
        pl = np.ascontiguousarray(prompt_len, dtype=np.int32)
        off = np.zeros(n + 1, dtype=np.int32)
        off[1:] = np.cumsum([len(r) for r in responses])
        resp = np.ascontiguousarray(np.concatenate(responses), dtype=np.int32)
        out = np.zeros(7 * int(off[-1]), dtype=np.float32)
        score = np.zeros(n, dtype=np.float32)
        ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
        fp = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))  # noqa: E731
        rc = self.lib.cpu_oracle_experience(self.h, n, maxp, ip(pl), ip(prompts), ip(off), ip(resp), beta, gamma, lam,
                                            self.threads, fp(out), fp(score))
        if rc != 0:
            raise ValueError(f"cpu_oracle_experience: status {rc}")
        T = int(off[-1])
        names = ("logp_actor", "logp_ref", "values", "kl", "reward", "adv", "ret")
        res = {k: out[i * T:(i + 1) * T] for i, k in enumerate(names)}
        res["score"] = score
        res["off"] = off
        return res

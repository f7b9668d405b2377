"""The CPU oracle is pinned before it is trusted (test infrastructure checks).

* GAE (oracle/model_oracle.py, oracle/post_oracle.c) against the reference's
  golden vectors and the reference library's gae_recursive;
* incremental KV-cached decode == full causal forward (the teacher-forcing
  identity the engine parity tests rely on);
* synthetic weights/prompts are bit-stable (hash + bf16 RNE);
* Zipf lengths: deterministic, bounded, heavy-tailed as SURVEY §8d states.
"""
import ctypes
import json
from pathlib import Path

import numpy as np
import pytest

from model_oracle import Oracle, forced_response, forward, hash3, log_softmax, synthetic_prompts, to_bf16

ROOT = Path(__file__).resolve().parent.parent
GOLD = json.loads((ROOT / "tests" / "golden" / "sched_golden.json").read_text())


def test_gae_oracle_on_reference_golden_vectors():
    from model_oracle import gae
    for g in GOLD["gae"]:
        got = gae(g["rewards"], g["values"], g["gamma"], g["lam"])
        assert list(got) == g["recursive"]  # same recursion, same association: bit-exact
    a = gae([1.0, 1.0], [0.0, 0.0, 0.0], 0.9, 0.95)  # test_numerics.cpp:35-49
    assert abs(a[0] - 1.855) <= 1e-12 and a[1] == 1.0
    assert list(gae([2.0], [1.0, 4.0], 0.5, 0.7)) == [2.0 + 0.5 * 4.0 - 1.0]  # :122-131
    with pytest.raises(ValueError):
        gae([1.0], [0.0], 0.9, 0.9)


def test_post_oracle_c_matches_reference_gae():
    lib = ROOT / "oracle" / "_ref" / "liboracle_c.so"
    if not lib.exists():
        pytest.skip("make -C oracle liboracle")
    o = ctypes.CDLL(str(lib))
    dp = ctypes.POINTER(ctypes.c_double)
    for g in GOLD["gae"]:
        r = np.array(g["rewards"], dtype=np.float64)
        v = np.array(g["values"], dtype=np.float64)
        out = np.zeros(len(r))
        assert o.oracle_gae(r.ctypes.data_as(dp), v.ctypes.data_as(dp), ctypes.c_int32(len(r)),
                            ctypes.c_double(g["gamma"]), ctypes.c_double(g["lam"]), out.ctypes.data_as(dp)) == 0
        assert list(out) == g["recursive"]  # same association order: bit-exact
    a = np.zeros(2)
    o.oracle_gae(np.array([1.0, 1.0]).ctypes.data_as(dp), np.zeros(3).ctypes.data_as(dp), ctypes.c_int32(2),
                 ctypes.c_double(0.9), ctypes.c_double(0.95), a.ctypes.data_as(dp))
    assert abs(a[0] - 1.855) < 1e-12 and a[1] == 1.0


def test_bf16_rounding_and_hash_are_stable():
    x = np.array([1.0, 1.00390625, 1.005859375, -3.14159, 65504.0, 1e-8], dtype=np.float32)
    b = to_bf16(x)
    assert b[0] == 1.0 and b[1] == 1.0 and b[2] == 1.0078125  # ties-to-even
    h = hash3(1234, 42, np.arange(4, dtype=np.uint64))
    assert list(h) == list(hash3(1234, 42, np.arange(4, dtype=np.uint64)))
    assert len(set(h.tolist())) == 4


def test_incremental_decode_equals_full_forward():
    from paper_2409_13221_b200.configs import TOY, Workload
    w = Workload("t", TOY, TOY, TOY, TOY, 2, 12, 16)
    orc = Oracle(w)
    prompt = synthetic_prompts(1, 12, TOY.vocab, 7)[0]
    toks, lps = orc.decode(prompt, 10, "greedy")
    full = forward(orc.models[0], np.concatenate([prompt, toks]))
    z = full[len(prompt) - 1:len(prompt) - 1 + 10] @ orc.models[0]["head"].T
    ref = log_softmax(z)[np.arange(10), toks]
    assert np.max(np.abs(ref - lps)) < 1e-4
    assert np.array_equal(np.argmax(z, -1), toks)


def test_zipf_lengths_shape():
    from paper_2409_13221_b200.configs import zipf_lengths
    a = zipf_lengths(4096, 1024, 1.0, 16, 7)
    assert a == zipf_lengths(4096, 1024, 1.0, 16, 7)
    assert min(a) >= 16 and max(a) <= 1024
    med = float(np.median(a))
    assert 100 <= med <= 160  # median ~126 at s=1, max 1024
    u = zipf_lengths(4096, 1024, 0.0, 16, 7)
    assert 450 <= float(np.median(u)) <= 590  # s = 0 is uniform on [16, 1024]


def test_forced_responses_deterministic():
    a = forced_response(3, 50, 512, 2048, 7)
    assert np.array_equal(a, forced_response(3, 50, 512, 2048, 7))
    assert a.min() >= 0 and a.max() < 2048


def test_c_weight_generator_matches_numpy_restatement():
    """oracle/weights_oracle.c (threaded, used for the bench-size oracle models)
    gives the numpy restatement's bits."""
    import model_oracle as mo
    if mo._clib() is None:
        pytest.skip("oracle C library not built (make -C oracle liboracle)")
    for n, scale, tag in [(1, 0.5, 3), (4099, mo.fsqrt(np.float32(3.0) / np.float32(768)), mo.weight_tag(2, 7, 4)),
                          (65536, mo.fsqrt(np.float32(3.0) / np.float32(14336)), mo.weight_tag(0, 31, 5))]:
        a, b = mo.uniform_weight(1234, tag, n, scale), mo.uniform_weight_np(1234, tag, n, scale)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        a, b = mo.gain(99, tag, n), mo.gain_np(99, tag, n)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_cpp_cpu_oracle_matches_numpy_oracle():
    """oracle/cpu_oracle.cpp (threaded fp32 C++, the timed CPU path) restates the numpy
    oracle: same experience within fp32 summation-order noise, on the toy config and an
    hd-128 GQA model."""
    import model_oracle as mo
    from paper_2409_13221_b200.configs import Dims, Workload, WORKLOADS, scaled
    if not (ROOT / "oracle" / "_ref" / "liboracle_cpu.so").exists():
        pytest.skip("oracle C++ library not built (make -C oracle liboracle)")
    gq = Dims(2, 256, 4, 2, 64, 512, 1024)
    for w in (scaled(WORKLOADS["toy"], n_prompts=4, max_new=40, prompt_len=16),
              Workload("gqa", gq, gq, gq, gq, 3, 12, 30)):
        cpp = mo.CppOracle(w, threads=4)
        py = mo.Oracle(w)
        prompts = mo.synthetic_prompts(w.n_prompts, w.prompt_len, w.actor.vocab, 7)
        plen = [w.prompt_len - i for i in range(w.n_prompts)]
        resp = [mo.forced_response(i, 10 + 7 * i, w.max_new, w.actor.vocab, 7) for i in range(w.n_prompts)]
        got = cpp.experience_batch(prompts, plen, resp, 0.05, 1.0, 0.95)
        for i in range(w.n_prompts):
            ref = py.experience(prompts[i, :plen[i]], resp[i], 0.05, 1.0, 0.95)
            b, e = got["off"][i], got["off"][i + 1]
            for k in ("logp_actor", "logp_ref", "values", "kl", "adv", "ret"):
                assert np.max(np.abs(got[k][b:e] - ref[k])) < 2e-3, (w.name, i, k)
            assert abs(got["score"][i] - ref["score"]) < 2e-3
        cpp.close()

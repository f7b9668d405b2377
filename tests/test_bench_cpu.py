"""bench.py workload selection (CPU): the bench lines are quoted on
BASELINE.json configs[1] (gpt2s, 512 prompts per GPU) and configs[2] shapes
(1.3b, 256 prompts per GPU = 2048 at 8 GPUs)."""
import importlib.util
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_default_workload_is_configs1():
    b = _bench()
    w = b.workload_for(1)
    assert (w.name, w.n_prompts, w.prompt_len, w.max_new) == ("gpt2s", 512, 128, 1024)
    assert (w.actor.num_layers, w.actor.hidden, w.actor.vocab) == (12, 768, 50257)
    assert b.workload_for(4).n_prompts == 2048  # weak scaling
    assert "512 prompts x 128 tokens per GPU" in b.workload_desc(b.workload_for(4), 4)


def test_13b_workload_is_configs2_at_8_gpus():
    b = _bench()
    w = b.workload_for(8, "1.3b")
    assert w.n_prompts == 2048 and w.max_new == 1024 and w.prompt_len == 256
    for d in (w.actor, w.ref, w.critic, w.reward):
        assert (d.num_layers, d.hidden, d.num_heads, d.ffn, d.vocab) == (24, 2048, 16, 5632, 32000)
    assert "L24 d2048" in b.workload_desc(w, 8)


def test_8b_workload_shapes():
    b = _bench()
    w = b.workload_for(4, "8b")
    assert w.n_prompts == 256 and w.max_new == 4096
    a = w.actor
    assert (a.num_layers, a.hidden, a.num_heads, a.num_kv_heads, a.head_dim, a.ffn, a.vocab) == \
        (32, 4096, 32, 8, 128, 14336, 128256)
    assert b.workload_for(2, "gpt2s", 0.0).zipf_s == 0.0

#!/usr/bin/env python
"""bench.py — RLHF experience samples/s of the gen+inf stage on B200s.

One step = one full experience collection over a prompt batch: prefill, the
actor's batched decode with retire-on-finish (sampled tokens, Zipf-skewed
lengths), Reference/Critic/Reward scoring of every finished sample and
per-token KL / reward / GAE / returns — through the C ABI (fp_execute).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

N = 1: BASELINE.json configs[1] (GPT-2-small shape, 512 prompts x 128 tokens,
<= 1024 new). N > 1: weak scaling, 512 prompts per GPU, fused schedule with
the one-shot long-tail migration at r_t = 20% of the batch.
--workload 1.3b: configs[2] shapes (all four models 1.3B), 256 prompts per GPU
(2048 at 8 GPUs), same schedule.

`value`  — samples/s with prompts resident and the experience left in HBM;
`e2e`    — the same through host buffers (prompt upload and experience
           download inside the timed region);
`stage_barrier` — the unfused schedule on the same GPUs (same K);
`roofline` — decode attention (the dominant kernel), algorithmic bytes per
           launch / CUDA-event duration, against MEASURED_PEAKS.json;
`cpu_baseline` — the CPU path (fp32 C++ oracle port, one std::thread per sample) on a bounded sample, rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
import uuid
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "RLHF experience samples/sec (gen+inference fused) at 1/2/4/8 B200; % HBM/tensor roofline"
UNIT = "samples/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1590.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = Path(f"/tmp/fp_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=open(self.path, "w"),
                stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(", ") for r in self.path.read_text().strip().splitlines() if r.strip()]
        except OSError:
            return None
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 3 + i and r[3 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(rows[0][1]),
                "samples": len(rows), "reasons": reasons}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    pg = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
        pg = dist
    return world, rank, local, pg


# prompts per GPU (weak scaling). gpt2s: configs[1] (512 prompts on one B200).
# 1.3b: configs[2] (2048 prompts at 8 GPUs = 256 per GPU; all four models 1.3B).
# 8b: configs[3] shapes (Llama-3-8B GQA 32/8 actor + 8B ref/critic/reward) at a
# REDUCED batch, 64 prompts per GPU: the config's 4096 prompts need 8 GPUs.
PER_GPU = {"gpt2s": 512, "1.3b": 256, "8b": 64}
DESC = {"gpt2s": "GPT-2-small-shape", "1.3b": "1.3B-shape (Llama-style)", "8b": "Llama-3-8B-shape (GQA 32/8)"}


def workload_for(n_gpus, name="gpt2s", zipf_s=None, per_gpu=None):
    from paper_2409_13221_b200.configs import WORKLOADS, scaled
    w = WORKLOADS[name]
    w = scaled(w, n_prompts=(per_gpu or PER_GPU[name]) * n_gpus)
    return w if zipf_s is None else scaled(w, zipf_s=zipf_s)


def workload_desc(w, G):
    a = w.actor
    return (f"{DESC[w.name]} actor/ref/critic/reward (L{a.num_layers} d{a.hidden} H{a.num_heads} ffn{a.ffn} "
            f"V{a.vocab}), {w.n_prompts // G} prompts x {w.prompt_len} tokens per GPU, <= {w.max_new} new")


_ORACLES = {}


def cpu_oracle_rate(w, batch, n_samples: int | None = None):
    """Samples/s of the CPU path — oracle/cpu_oracle.cpp, fp32 C++ with one std::thread per
    sample over all host cores — on the first n_samples samples of the batch
    (default: one per host thread), teacher-forced through actor / ref / critic / reward and
    post-processed. The oracle's weights are built once, outside the timed region.
    Returns (samples/s, samples, tokens, seconds, threads)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    from model_oracle import CppOracle, forced_response, synthetic_prompts
    if w.name not in _ORACLES:
        _ORACLES[w.name] = CppOracle(w)
    orc = _ORACLES[w.name]
    n = min(len(batch), n_samples or orc.threads)
    prompts = synthetic_prompts(n, w.prompt_len, w.actor.vocab, 7)
    resp = [forced_response(s.id, s.target_output_len, w.max_new, w.actor.vocab, 7) for s in batch[:n]]
    t0 = time.perf_counter()
    orc.experience_batch(prompts, [s.prompt_len for s in batch[:n]], resp, 0.05, 1.0, 0.95)
    dt = time.perf_counter() - t0
    tokens = sum(s.prompt_len + s.target_output_len for s in batch[:n])
    return n / dt, n, tokens, dt, orc.threads


def python_batch(w):
    """The batch the GPU arm runs, built without the product library: the
    reference's make_batch (genfuse.cpp:403-414) from oracle/_ref when it was
    built here, else the same arithmetic in Python (kv_bytes_per_token =
    4 L hidden, core.cpp:90-93)."""
    from paper_2409_13221_b200.configs import zipf_lengths
    lens = zipf_lengths(w.n_prompts, w.max_new, w.zipf_s, w.zipf_lo, w.length_seed)
    ref_lib = ROOT / "oracle" / "_ref" / "libfuseplan_ref.so"
    if ref_lib.exists():
        from paper_2409_13221_b200.configs import batch_for
        from paper_2409_13221_b200.sched import Sched
        return batch_for(w, Sched(str(ref_lib)), lengths=lens), "reference make_batch (oracle/_ref)"
    from paper_2409_13221_b200.sched import GenSample
    kv = 4.0 * w.actor.num_layers * w.actor.hidden
    return [GenSample(i, w.prompt_len, L, 0, (w.prompt_len + L) * kv) for i, L in enumerate(lens)], "python"


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path. The reference library only
    simulates this stage (cost formulas, no model math), so the
    CPU implementation of the path that produces experience is the oracle
    port (oracle/cpu_oracle.cpp: fp32 C++, one std::thread per sample); the simulator's own
    runtime is reported beside it. Nothing here loads the product library."""
    if rank != 0:
        return
    w = workload_for(args.gpus, args.workload, args.zipf_s, args.prompts_per_gpu)
    batch, batch_src = python_batch(w)
    n_sub = None if w.name in ("toy", "gpt2s") else 1  # one sample per host thread (toy: the first ones)
    rates, walls = [], []
    info = None
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r, done, toks, dt, cores = cpu_oracle_rate(w, batch, n_samples=n_sub)
        if step >= args.warmup:
            rates.append(r)
            walls.append(time.perf_counter() - t0)
            info = (done, toks, dt)
    value = statistics.median(rates)
    sim = None
    ref_lib = ROOT / "oracle" / "_ref" / "libfuseplan_ref.so"
    if ref_lib.exists():
        from paper_2409_13221_b200.configs import gen_config
        from paper_2409_13221_b200.sched import Sched
        rs = Sched(str(ref_lib))
        cfg = gen_config(w, args.gpus, calibrated=True)
        t0 = time.perf_counter()
        rs.simulate_fused(batch, cfg, round(0.2 * len(batch)))
        sim = time.perf_counter() - t0
    sample = (f"{info[0]} of {len(batch)} prompts ({info[1]} tokens) teacher-forced through actor/ref/critic/reward "
              f"+ KL/GAE post-processing, fp32 C++ (oracle/cpu_oracle.cpp), one std::thread per sample; "
              f"step = that subset")
    cfg_line = config_dict(w, args.gpus, args)
    cfg_line["cpu_subset"] = f"{info[0]} of {len(batch)} prompts per step (batch built by {batch_src})"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * statistics.median(walls),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": cfg_line,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_simulator_seconds": sim,
            "note": "reference path is a discrete-event simulator without model math; CPU arm = the oracle port "
                    "(fp32 C++, std::thread over samples); ms_per_step = measured wall time of the subset"}
    print(json.dumps(line), flush=True)


def chooser_ratio(w, G):
    """R_t / n picked by tools/rt_chooser.py (committed fit of measured B200 steps), else 0.2."""
    key = {"gpt2s": "gpt2s", "1.3b": "13b", "8b": "8b"}.get(w.name)
    p = ROOT / "profiles" / f"r02_rt_chooser_{key}.json"
    if key and p.exists():
        g = json.loads(p.read_text())["G"].get(str(G))
        if g:
            return float(g["best_ratio"])
    return 0.2


def config_dict(w, G, args, r_t=None, ratio=None):
    return {"workload": workload_desc(w, G), "prompts": w.n_prompts, "zipf_s": w.zipf_s, "schedule": "fused",
            "r_t": r_t, "r_ratio": ratio, "r_ratio_source": getattr(args, "r_ratio", None),
            "token_mode": args.token_mode, "claim_tokens": args.claim_tokens,
            "l2": "inputs larger than L2 (KV pool and weights >> 126 MB)",
            "kv_pool_gb": getattr(args, "kv_pool_gb", 0.0) or None,
            "parallelism": f"dp{G} (one engine per B200)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--r-ratio", default="chooser",
                    help="migration threshold R_t / n; 'chooser': the best ratio of tools/rt_chooser.py's "
                         "sharing-aware model for this workload and G (profiles/r02_rt_chooser_<w>.json; 0.2 "
                         "without one); 'auto': the best ratio of the reference's sweep_threshold under the "
                         "calibrated CostModel")
    ap.add_argument("--token-mode", default="sample", choices=["forced", "greedy", "sample"])
    ap.add_argument("--claim-tokens", type=int, default=12288)  # swept: 8192 580.2, 10240 581.6, 12288 584.1, 16384 570.2
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-barrier-arm", action="store_true")
    ap.add_argument("--workload", default="gpt2s", choices=sorted(PER_GPU),
                    help="gpt2s = BASELINE configs[1] (the default bench line); 1.3b = configs[2] shapes; "
                         "8b = configs[3] shapes at a reduced batch (64 prompts per GPU)")
    ap.add_argument("--zipf-s", type=float, default=None,
                    help="output-length skew (configs[4] sweep): 0 = uniform on [16, max_new]; default = the "
                         "workload's (1.0)")
    ap.add_argument("--quick", action="store_true", help="value pass only (for profiling)")
    ap.add_argument("--prompts-per-gpu", type=int, default=None,
                    help="override the workload's prompts per GPU (e.g. 512 for configs[3] at its stated batch)")
    ap.add_argument("--kv-pool-gb", type=float, default=0.0,
                    help="> 0: physical KV pool per GPU (GB); admission is then KV-gated: the decision clock's "
                         "capacity is the pool in the reference's MHA reservation units (core.cpp:90-93)")
    ap.add_argument("--no-e2e", action="store_true", help="skip the e2e pass (long configs)")
    args = ap.parse_args()
    world, rank, local, dist = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        if dist:
            dist.barrier()
        return

    import torch
    torch.cuda.set_device(local)
    from paper_2409_13221_b200.configs import batch_for, gen_config
    from paper_2409_13221_b200.engine import Engine

    G = world
    w = workload_for(G, args.workload, args.zipf_s, args.prompts_per_gpu)
    max_live = min(w.n_prompts, 2 * w.n_prompts // G)
    pool = int(args.kv_pool_gb * 1e9)
    eng = Engine(w, device=local, max_samples=w.n_prompts, max_live=max_live, kv_pool_bytes=pool)
    batch = batch_for(w, eng.sched)
    cfg = gen_config(w, G, calibrated=True)  # decision-clock constants fitted to measured B200 steps
    if pool > 0:
        # KV-gated admission (genfuse.cpp:226-236): the clock reserves (prompt + target) x the reference's
        # MHA bytes per token (core.cpp:90-93, 4 L hidden); the engine holds GQA pages of 64 tokens. Map the
        # physical pool into the clock's units, less one page per live slot for the page rounding.
        a = w.actor
        page = 64 * eng.kv_bytes_per_token()
        mha_over_phys = 4.0 * a.num_layers * a.hidden / eng.kv_bytes_per_token()
        cfg.cluster.kv_capacity_per_instance = (pool - max_live * page) * mha_over_phys
    if args.r_ratio == "auto" and G > 1:
        sw = eng.sched.sweep_threshold(batch, cfg)
        ratio = sw.curve[sw.best_index][0]
    elif args.r_ratio == "chooser":
        ratio = chooser_ratio(w, G)
    else:
        ratio = float(args.r_ratio)
    r_t = round(ratio * len(batch)) if G > 1 else 0
    shm = None
    if dist:
        obj = [f"/fp_bench_{uuid.uuid4().hex[:12]}" if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        shm = obj[0]
    prompts = eng.synthetic_prompts(len(batch), 7)

    def barrier():
        if dist:
            dist.barrier()

    def step(schedule, resident, probe=False):
        return eng.execute(batch, cfg, r_t, token_mode=args.token_mode, schedule=schedule,
                           claim_tokens=args.claim_tokens, rank=rank, world=G,
                           shm_name=(shm + f"_{step.k}") if shm else None, prompts=prompts, resident=resident,
                           probe_attention=probe)
    step.k = 0

    # ncu --profile-from-start off: profile only the first timed region
    prof_range = os.environ.get("FUSEPLAN_PROFILE_TIMED") == "1"

    def timed(schedule, resident, K, probe=False):
        nonlocal prof_range
        outs = []
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if prof_range:
            torch.cuda.profiler.start()
        e0.record()
        for _ in range(K):
            step.k += 1
            outs.append(step(schedule, resident, probe))
        if prof_range:
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
            prof_range = False
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, outs

    # warm-up (both schedules, both residency modes)
    for i in range(args.warmup):
        step.k += 1
        step("fused", i % 2 == 0)
    log(f"[bench] rank {rank}: warm-up done")

    with Clocks(local) as clk:
        ms_v, outs_v = timed("fused", True, args.steps)
    clocks = clk.summary()
    n_total = len(batch)
    value = n_total * args.steps / (ms_v / 1000.0)
    st = outs_v[-1].stats
    launches = sum(o.stats["gpu_launches"] for o in outs_v)
    # roofline probe: one more (untimed) step with CUDA events around every
    # decode-attention launch (eager: the probe disables the step graphs)
    ms_p, outs_p = timed("fused", True, 1, probe=True)
    probe_ms = sum(o.stats["attn_probe_ms"] for o in outs_p)
    probe_bytes = sum(o.stats["attn_probe_bytes"] for o in outs_p)
    probe_n = sum(o.stats["attn_probe_launches"] for o in outs_p)

    e2e = sb = None
    outs_s = None
    h2d = len(batch) * w.prompt_len * 4 + len(batch) * 4 * 6
    d2h = int(st["total_resp"]) * 4 * 8 + len(batch) * 4
    if not args.quick:
        if not args.no_e2e:
            ms_e, outs_e = timed("fused", False, args.steps)
            e2e = n_total * args.steps / (ms_e / 1000.0)
        if not args.no_barrier_arm:
            ms_s, outs_s = timed("stage_barrier", True, args.steps)
            sb = n_total * args.steps / (ms_s / 1000.0)

    cpu = None
    if rank == 0 and G == 1 and not args.no_cpu_baseline and not args.quick:
        r, done, toks, dt, cores = cpu_oracle_rate(w, batch)
        cpu = {"value": r, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{done} of {len(batch)} prompts ({toks} tokens) through the fp32 C++ oracle "
                         f"(oracle/cpu_oracle.cpp: teacher-forced actor/ref/critic/reward + post-processing, "
                         f"one std::thread per sample), {dt:.1f}s"}

    # per-rank decode / scoring totals of the value steps, summed over ranks
    # (every rank decodes its own shard; any rank may score any sample)
    mine = {"dec_s": sum(o.stats["decode_gpu_seconds"] for o in outs_v),
            "steps": sum(o.stats["decode_steps"] for o in outs_v),
            "rows": sum(o.stats["decode_rows"] for o in outs_v),
            "ctx": sum(o.stats["decode_ctx_tokens"] for o in outs_v),
            "inf_s": sum(o.stats["infer_busy_seconds"] for o in (outs_s or outs_v)),
            "inf_steps": len(outs_s or outs_v)}
    ranks = [mine]
    if dist:
        ranks = [None] * G
        dist.all_gather_object(ranks, mine)
    if rank != 0:
        eng.close()
        return
    hbm, tflops, src = peaks()
    a = w.actor
    embed_bytes = a.vocab * a.hidden * 2
    w_step = eng.model_size(0)[0] - embed_bytes  # weights streamed once per step; the embedding is gathered
    kvb = eng.kv_bytes_per_token()
    dec_s = sum(r["dec_s"] for r in ranks)
    dec_b = sum(r["steps"] * w_step + r["rows"] * (a.hidden * 2 + kvb) + r["ctx"] * kvb for r in ranks)
    decode_roofline = {"bound": "hbm", "bytes_per_step": dec_b / len(outs_v), "seconds_per_step": dec_s / len(outs_v),
                       "achieved": dec_b / dec_s / 1e9 if dec_s else None, "peak": hbm, "unit": "GB/s",
                       "frac": dec_b / dec_s / 1e9 / hbm if dec_s else None, "ranks": len(ranks),
                       "note": "all ranks: decode steps x actor weight bytes without the embedding table + per row "
                               "its gathered embedding row and K/V append + sum over rows of ctx x K/V bytes per "
                               "token, / the ranks' summed decode-step GPU time"}
    # scoring (Ref/Critic/Reward forward over prompt + response) against the
    # bf16 tensor peak: algorithmic flops = 2 x dense weights per token (ref
    # adds the vocab head for its log-probs) + causal attention 2 T^2 H hd L,
    # over the scoring streams' busy GPU time summed over ranks (stage-barrier
    # arm when run, so decode does not share the SMs); each sample is scored
    # exactly once, on whichever rank claimed it
    def fwd_flops(d, T, vocab_head):
        dense = d.param_count(lm_head=False) - d.vocab * d.hidden
        return 2 * T * (dense + (d.hidden * d.vocab if vocab_head else d.hidden)) + \
            2 * T * T * d.num_heads * d.head_dim * d.num_layers
    src_name = "stage_barrier" if outs_s else "fused (overlaps decode)"
    inf_flops = sum(fwd_flops(w.ref, s.prompt_len + s.target_output_len, True) +
                    fwd_flops(w.critic, s.prompt_len + s.target_output_len, False) +
                    fwd_flops(w.reward, s.prompt_len + s.target_output_len, False) for s in batch)
    inf_s = sum(r["inf_s"] for r in ranks) / ranks[0]["inf_steps"]
    inf_tf = inf_flops / inf_s / 1e12 if inf_s else None
    inference_roofline = {"bound": "tensor", "achieved": inf_tf, "peak": tflops, "unit": "TFLOP/s",
                          "frac": inf_tf / tflops if inf_tf else None, "flops_per_step": inf_flops,
                          "seconds_per_step": inf_s, "arm": src_name, "ranks": len(ranks),
                          "note": "ref/critic/reward forward over every sample (prompt + target response): "
                                  "2 x dense weights per token (+ vocab head for ref) + causal attention "
                                  "2 T^2 H hd L; / the scoring streams' busy GPU time summed over ranks"}
    achieved = (probe_bytes / (probe_ms / 1000.0)) / 1e9 if probe_ms > 0 else None
    # traffic: DRAM bytes per launch from the committed ncu --set full capture
    # of this kernel (profiles/attn_decode_traffic.json), as its DRAM /
    # algorithmic ratio applied to this run's mean launch
    traffic = traffic_src = None
    tp = ROOT / "profiles" / "attn_decode_traffic.json"
    if tp.exists() and probe_n:
        tj = json.loads(tp.read_text())
        traffic = tj["dram_over_algorithmic"] * probe_bytes / probe_n
        traffic_src = f"{tj['source']} on {tj['config']}: dram/algorithmic = {tj['dram_over_algorithmic']:.3f}"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_v / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic: hash-seeded random-init weights and prompts, "
                f"Zipf(s={w.zipf_s}) output lengths on [{w.zipf_lo}, {w.max_new}], "
                f"{args.token_mode} tokens",
        "config": config_dict(w, G, args, r_t, ratio if G > 1 else 0.0),
        "roofline": {"kernel": "attn_decode (paged KV flash-decoding)", "bound": "hbm", "achieved": achieved,
                     "peak": hbm, "unit": "GB/s", "frac": (achieved / hbm) if achieved else None,
                     "traffic": traffic, "traffic_source": traffic_src, "peak_source": src, "launches": probe_n,
                     "bytes_per_launch": probe_bytes / max(probe_n, 1),
                     "share_of_step": (probe_ms / ms_p) if ms_p else None},
        # the whole decode step against HBM — weights once per step
        # plus K/V of every visible token, over the decode GPU time of the value steps
        "decode_roofline": decode_roofline,
        "inference_roofline": inference_roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "stage_barrier": {"value": sb, "unit": UNIT, "speedup_fused": (value / sb) if sb else None},
        "clocks": clocks,
        "gpu_launches": launches,
        "stats": {k: st[k] for k in ("decode_steps", "decode_rows", "decode_ctx_tokens", "prefill_tokens",
                                     "infer_tokens", "gen_seconds", "decode_gpu_seconds", "infer_busy_seconds",
                                     "migrated_in", "migrated_bytes")},
    }
    print(json.dumps(line), flush=True)
    eng.close()


if __name__ == "__main__":
    main()

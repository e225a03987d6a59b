#!/usr/bin/env python
"""Benchmark: LoRA + LeMo fine-tuning step on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lemo|reference]
                    [--config llama2_7b_16k|llama2_7b_4k|tiny]

Workload (default): Llama2-7B geometry, LoRA r=8 on q/v, LeMo predicted
patterns (random predictors r1=r2=d_p=1024, attention retention 0.5 by the
quantile rule re-derived every 50 calls, MLP thresholds = pooled mean of a
profiling pass), one 16,384-token synthetic sequence per GPU per step,
random-init weights (bf16 GEMM operands, fp32 residual/LoRA/Adam), scorers in
the "refined" precision (the reference's masks: bf16 scores, then the token
rows that can decide an MLP block near its threshold re-scored fp32-faithfully;
`--scoring-precision bf16|fp32`).  A step
= forward_step + sparse backward + (N>1: NCCL all-reduce of LoRA grads) +
Adam.  N>1: one process per GPU under torchrun, each rank its own sequence
(weak scaling); time = max over ranks of CUDA-event time.

Prints ONE JSON line (rank 0).  `value` = tokens/s over all ranks with
inputs resident in HBM; `e2e` = same through the host API (tokens from host
memory each step, loss read back each step); `dense_lora` = the same kernels
at full retention (the reference's definition of dense LoRA, model.py:
300-302) for the ≥1.3× tokens/s and ≥1.5× activation targets; `roofline`
= the dominant kernel (the tcgen05 gate/up GEMM of MLP scoring) timed live
with CUDA events; `mask_flips` = an untimed audit of every MLP decision of one
step against the fp32-faithful parity scorers (audit.MaskAudit);
`cpu_baseline` = the UNMODIFIED reference (baseline/_ref, sparsetune) timed on
this host on a bounded full-width sample (baseline/run_reference.py).

`--impl reference` is the reference arm: the unmodified reference on the host
cores (rank 0), one full-width 16K layer sample per step, extrapolated to the
32-layer step; see run_reference().
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "llama2_7b_16k": dict(seq=16384, model="llama2_7b", name="Llama2-7B"),
    "llama2_7b_4k": dict(seq=4096, model="llama2_7b", name="Llama2-7B"),
    "llama2_7b_32k": dict(seq=32768, model="llama2_7b", name="Llama2-7B"),
    "llama3_8b_16k": dict(seq=16384, model="llama3_8b", name="Llama3-8B (GQA 32/8)"),
    "mistral_7b_32k": dict(seq=32768, model="mistral_7b", name="Mistral-7B (GQA 32/8, no SWA)"),
    "opt_6.7b_64k": dict(seq=65536, model="opt_6_7b", name="OPT-6.7B (reference family: "
                                                          "RMSNorm, no bias; ReLU, learned pos.)"),
    "tiny": dict(seq=2048, model="tiny_t", name="tiny T"),
}
METRIC = "fine-tune tokens/sec + peak activation GB at 16K ctx (1/2/4/8 B200) vs CPU ref"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lemo", choices=["lemo", "reference"])
    ap.add_argument("--config", default="llama2_7b_16k", choices=list(CONFIGS))
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-law", action="store_true")
    ap.add_argument("--no-audit", action="store_true",
                    help="skip the mask-flip audit (production vs parity-precision scorers)")
    ap.add_argument("--scoring-precision", default="refined", choices=["bf16", "fp32", "refined"],
                    help="precision of the scorers in the timed step: bf16 (production), fp32 "
                         "(the mask-exact parity precision) or refined (bf16 + parity re-scoring "
                         "of the token rows that decide MLP blocks near their threshold)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N>1 (gloo only to smoke-test several "
                         "ranks sharing one GPU)")
    ap.add_argument("--cpu-tokens", type=int, default=4096,
                    help="tokens of the bounded reference sample behind cpu_baseline")
    ap.add_argument("--ref-budget-s", type=float, default=150.0,
                    help="reference arm: time budget for the full-width layer samples")
    ap.add_argument("--profile-tag", default="")
    return ap.parse_args()


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:  # noqa: BLE001
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        time.sleep(0.1)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) < 9:
                continue
            for i, nm in enumerate(names):
                if r[5 + i].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm (oracle restatement) on host cores


def cpu_geometry(cfg) -> dict:
    """Oracle CpuSample geometry of a ModelConfig (same widths as the GPU run)."""
    return dict(hidden=cfg.hidden_dim, heads=cfg.n_heads, kv_heads=cfg.kv_heads,
                mlp=cfg.mlp_dim, vocab=cfg.vocab_size, n_layers_model=cfg.n_layers,
                block=cfg.block_size, lora_rank=cfg.lora_rank, mlp_variant=cfg.mlp_variant,
                positions=cfg.positions)


REF_DIR = ROOT / "baseline" / "_ref"


def reference_available() -> bool:
    return (REF_DIR / "sparsetune" / "__init__.py").exists()


def run_reference_process(args_list, cores: int, timeout_s: float = 1500.0) -> dict:
    """baseline/run_reference.py in a subprocess: the unmodified reference
    (sparsetune from baseline/_ref) with NumPy's BLAS pool sized to `cores`
    before NumPy loads (torchrun exports OMP_NUM_THREADS=1 to its workers)."""
    env = dict(os.environ)
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        env[k] = str(cores)
    env["PYTHONPATH"] = str(REF_DIR)
    r = subprocess.run([sys.executable, str(ROOT / "baseline" / "run_reference.py"), *args_list],
                       env=env, capture_output=True, text=True, timeout=timeout_s)
    if r.returncode != 0:
        raise RuntimeError(f"reference run failed ({r.returncode}): {r.stderr[-2000:]}")
    return json.loads(r.stdout.strip().splitlines()[-1])


def _ref_layer_seq(wl) -> int:
    # the reference's O(s^2) Python tile loops: full-width samples up to 16K
    # (32K / 64K are not run)
    return min(wl["seq"], 16384)


def run_reference(args):
    """The reference arm: the unmodified reference (baseline/_ref) on the host
    cores, rank 0 only.  A "step" is one bounded sample of the workload: the
    reference's own forward_step + backward on a 1-layer Llama2-7B-width model
    at the workload's sequence length (repeated while the time budget allows);
    `value` is the 32-layer step extrapolated from it (32·t_layer + t_head),
    `ms_per_step` the measured per-sample time, so ms_per_step x steps is the
    time actually spent.  Config T's full training step is measured too."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle.cpu_sample import host_cores

    wl = CONFIGS[args.config]
    cores = host_cores()
    if not reference_available():
        return run_reference_port(args, cores)
    tiny_only = args.config == "tiny"
    seq = _ref_layer_seq(wl)
    meas = run_reference_process(["--tiny-steps", str(max(args.steps, 5)), "--layer-seq",
                                  *([] if tiny_only else [str(seq)]),
                                  "--budget-s", str(args.ref_budget_s)], cores)
    tiny = meas["tiny"]
    if tiny_only:
        value, ms, n = tiny["tokens_per_s"], tiny["median_s"] * 1e3, tiny["steps"]
        sample = "config T full training step, median of the timed steps"
        per = {}
    else:
        lay = meas[f"layer_{seq}"]
        value, ms, n = lay["tokens_per_s"], lay["median_sample_s"] * 1e3, lay["samples"]
        sample = (f"unmodified reference (baseline/_ref sparsetune): 1-layer Llama2-7B-width model "
                  f"at {seq} tokens, forward_step + backward in LeMo predicted mode per step "
                  f"(t_sample {lay['median_sample_s']:.1f}s = t_layer {lay['layer_s']:.1f}s + "
                  f"LM head {lay['head_s']:.1f}s); value extrapolated to 32 layers "
                  f"({lay['extrapolated_step_s']:.0f}s per 32-layer step)")
        per = {"per_layer_s": lay["layer_s"], "head_s": lay["head_s"],
               "extrapolated_step_s": lay["extrapolated_step_s"], "sample_s": lay["sample_s"],
               "retained": lay["retained"], "setup_s": lay["setup_s"]}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": n, "warmup": 0 if not tiny_only else 1,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic tokens, reference init",
        "config": {"workload": f"{args.config}: {wl['name']} LoRA+LeMo predicted mode",
                   "seq_len": seq if not tiny_only else 2048, "parallelism": "cpu",
                   "same_config": wl["model"] in ("llama2_7b", "tiny_t") and seq == wl["seq"]},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_samples": {"tiny_full_step": tiny, **({"layer": per} if per else {})},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_reference_port(args, cores):
    """Fallback when baseline/_ref is absent: the oracle restatement."""
    from oracle.cpu_sample import CpuSample
    from paper_2501_09767_b200 import model as M

    wl = CONFIGS[args.config]
    os.environ["OMP_NUM_THREADS"] = str(cores)
    try:
        from threadpoolctl import threadpool_limits
        _pool = threadpool_limits(limits=cores)  # noqa: F841 (kept for the run)
    except Exception:  # noqa: BLE001
        pass
    mcfg = getattr(M, wl["model"])(max_seq_len=wl["seq"])
    sample = CpuSample(sample_tokens=min(args.cpu_tokens, wl["seq"]), **cpu_geometry(mcfg))
    t_head = sample.time_head()
    times = [sample.time_step()[0] for _ in range(2)]
    t_layer = max(float(np.median(times)) - t_head, 1e-9)
    per_step = mcfg.n_layers * t_layer + t_head
    value = sample.s / per_step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": len(times), "warmup": 0, "ms_per_step": np.median(times) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {wl['name']} LoRA+LeMo predicted mode",
                   "seq_len": sample.s, "parallelism": "cpu", "same_config": False},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port",
                         "sample": f"baseline/_ref missing: oracle restatement, 1 decoder layer "
                                   f"on {sample.s} tokens, extrapolated to {mcfg.n_layers} layers"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# B200 arm


def _mlp_only_profile(src, S):
    """ExactPatternSource restricted to MLP scoring (attention retained in the
    profile pass; its thresholds are set by the predicted calibration pass)."""
    orig = src.pattern

    def pattern(layer_id, component, x, n_valid):
        if component == S.ATTENTION:
            return src._note(layer_id, component, None)
        return orig(layer_id, component, x, n_valid)

    return pattern


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            # communicator set-up lines (ring / NVLS / transport) on stderr, so a
            # scaling run shows how the LoRA-gradient all-reduce is carried
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    from paper_2501_09767_b200 import _lib, model as M, parallel, predictor as P, sparsity as S
    from paper_2501_09767_b200.optim import Adam

    wl = CONFIGS[args.config]
    seq = wl["seq"]
    cfg = getattr(M, wl["model"])(max_seq_len=seq)
    torch.manual_seed(0)
    # parity_weights keeps the bf16 residuals of the scoring weights (parity
    # precision for the refined scorers and the untimed mask audit).  Default:
    # the "refined" precision -- bf16 scorers, then the token rows that can decide
    # an MLP block near its threshold re-scored in parity precision, i.e. the reference's masks; the
    # plain bf16 scorers are timed as well (`bf16_scoring`)
    model = M.DecoderModel(cfg, seed=0, device=dev, init="torch",
                           scoring_precision=args.scoring_precision,
                           parity_weights=(not args.no_audit) or args.scoring_precision != "bf16")
    h = cfg.hidden_dim
    rp = h // 4
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    pairs = {}
    for l in range(cfg.n_layers):
        mk = lambda: P.Predictor(torch.randn(h, rp, generator=gen, device=dev) / math.sqrt(h),  # noqa
                                 torch.randn(rp, rp, generator=gen, device=dev) / math.sqrt(rp),
                                 torch.randn(rp, rp, generator=gen, device=dev) / math.sqrt(rp),
                                 device=dev)
        pairs[l] = (mk(), mk())
    model.attach_predictors(pairs)
    rng = np.random.default_rng(1000 + rank)
    tokens = rng.integers(0, cfg.vocab_size, size=seq)
    segments = 8 if seq >= 1024 else 1

    # thresholds (the reference pipeline's order: profile -> init -> predicted init):
    #  pass 1  retain-all profile of exact MLP scores -> MLP thresholds = pooled
    #          mean (init_thresholds, sparsity.py:360-376)
    #  pass 2  with those MLP thresholds, attention thresholds re-derived at 50%
    #          retention from the predicted scores (model.py:545-563)
    retention = {l: 0.5 for l in range(cfg.n_layers)}
    prof = M.ExactPatternSource(model, None, record=True)
    prof.pattern = _mlp_only_profile(prof, S)
    with torch.no_grad():
        model.forward_step(tokens, pattern_source=prof, segments=segments)
    thr = S.init_thresholds(prof.recorded_vectors)
    model._mlp_scored.clear()
    for l in range(cfg.n_layers):
        thr.set(l, S.ATTENTION, 0.0)
    cal = M.PredictedPatternSource(model, thr.copy(), target_retention=retention,
                                   recalibrate_every=1)
    with torch.no_grad():
        model.forward_step(tokens, pattern_source=cal, segments=segments)
    model._mlp_scored.clear()
    source = M.PredictedPatternSource(model, cal.thresholds.copy(), target_retention=retention,
                                      recalibrate_every=50)
    del prof, cal
    opt = Adam(model.lora_param, lr=1e-4)

    if world > 1:  # the path's only exchange: per-layer LoRA-gradient buckets
        model.grad_reducer = parallel.BucketedGradReducer()  # overlapped with backward (§8e)

    def step(src, batch, read_loss=False):
        loss, _ = model.forward_step(batch, pattern_source=src, segments=segments)
        loss.backward()
        opt.step()
        opt.zero_grad()
        return float(loss.detach()) if read_loss else loss

    def timed(src, batch_fn, steps, read_loss=False, timed_names=()):
        ins = _lib.INSTRUMENT
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ins.reset(timed_names)
        ins.enabled = True
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(steps):
            step(src, batch_fn(), read_loss)
        b.record()
        torch.cuda.synchronize()
        ins.enabled = False
        ms = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t)
            dist.barrier()
        return ms

    wbytes = sum(t.numel() * t.element_size() for L in model.layers
                 for t in (L.w_qkv_t, L.w_gu_t, L.w_down_t, L.w_o_t))
    staged = model.stage_tokens(tokens)
    for _ in range(args.warmup):
        step(source, staged)
    torch.cuda.synchronize()
    base_mem = torch.cuda.memory_allocated(dev)
    torch.cuda.reset_peak_memory_stats(dev)
    clocks = Clocks(local)
    clocks.start()
    gemm_name, embed_name = "lemo_gemm_gateup", "lemo_block_embed"
    fa_f, fa_b = "lemo_flash_fwd_tc", "lemo_flash_bwd_tc"
    ms = timed(source, lambda: staged, args.steps,
               timed_names=(gemm_name, embed_name, fa_f, fa_b))
    ck = clocks.stop()
    ins = _lib.INSTRUMENT
    launches_per_step = ins.total_launches() / args.steps
    # the dominant launch: the bf16 scoring GEMM over all s rows (the refined
    # precision's small parity re-scoring GEMMs share the entry point; notes
    # carry each call's (M, N, K, exact) so they are kept out of the average)
    gemm_ms = [t for t, (mm, _n, kk, ex) in zip(ins.elapsed_ms(gemm_name), ins.notes[gemm_name])
               if mm == seq and kk == cfg.hidden_dim and not ex]
    embed_ms = ins.elapsed_ms(embed_name)
    # attention (causal, compact retained rows): fwd 2·n²·h, bwd 5·n²·h algorithmic flops
    attn = {}
    for nm, mult in ((fa_f, 2.0), (fa_b, 5.0)):
        tms, ns = ins.elapsed_ms(nm), ins.notes.get(nm, [])
        if tms and len(ns) == len(tms):
            fl = sum(mult * float(nn) * nn * cfg.hidden_dim for nn in ns)
            attn[nm] = {"tflops": fl / (sum(tms) / 1e3) / 1e12, "launches": len(tms),
                        "avg_ms": sum(tms) / len(tms), "avg_rows": sum(ns) / len(ns)}
    lemo_stats = dict(model.last_stats)
    refined_rows = (sum(source.refined_rows.values()) if model.scoring_precision == "refined"
                    else None)  # rows re-scored in the parity precision, last step
    peak_step = torch.cuda.max_memory_allocated(dev) - base_mem
    ms_step = ms / args.steps
    value = world * seq * args.steps / (ms / 1e3)

    # e2e through the host API: host tokens in, loss read back every step
    ms_e2e = timed(source, lambda: tokens, args.steps, read_loss=True)
    e2e_value = world * seq * args.steps / (ms_e2e / 1e3)

    # the same step with the plain bf16 scorers (no refinement: ~0.4 % of the
    # MLP decisions differ from the reference's), for comparison
    bf16_scoring = None
    if args.scoring_precision != "bf16":
        model.set_scoring_precision("bf16")
        for _ in range(2):
            step(source, staged)
        ms_b = timed(source, lambda: staged, args.steps)
        bf16_scoring = {"value": world * seq * args.steps / (ms_b / 1e3), "unit": "tokens/s",
                        "ms_per_step": ms_b / args.steps,
                        "note": "bf16 scorers without refinement: masks differ from the "
                                "reference's on ~0.4 % of the MLP blocks (see mask_flips of a "
                                "--scoring-precision bf16 run)"}
        model.set_scoring_precision(args.scoring_precision)

    # mask-flip audit (untimed): every MLP decision of one step re-scored in the
    # fp32-faithful parity precision under the same threshold (audit.MaskAudit)
    audit = None
    if not args.no_audit:
        from paper_2501_09767_b200.audit import MaskAudit
        aud = MaskAudit(source, model)
        with torch.no_grad():
            model.forward_step(staged, pattern_source=aud, segments=segments)
        audit = aud.summary()
        del aud
        torch.cuda.empty_cache()

    dense = None
    if not args.no_dense:
        try:
            for _ in range(2):
                step(None, staged)
            torch.cuda.synchronize()
            torch.cuda.reset_peak_memory_stats(dev)
            base_d = torch.cuda.memory_allocated(dev)
            ms_d = timed(None, lambda: staged, args.steps)
            dense_stats = dict(model.last_stats)
            dense = {
                "value": world * seq * args.steps / (ms_d / 1e3), "unit": "tokens/s",
                "ms_per_step": ms_d / args.steps,
                "activation_gb_post_forward": dense_stats["activation_bytes_post_forward"] / 1e9,
                "peak_step_gb": (torch.cuda.max_memory_allocated(dev) - base_d) / 1e9,
            }
        except torch.cuda.OutOfMemoryError:
            _lib.INSTRUMENT.enabled = False
            opt.zero_grad()
            torch.cuda.empty_cache()
            dense = {"value": None, "oom": True, "note": "dense LoRA (full retention) does not "
                     f"fit in {torch.cuda.get_device_properties(dev).total_memory / 1e9:.0f} GB "
                     f"at {seq} tokens on one GPU"}

    # memory law (acceptance criterion 9) at this workload: logical saved-for-
    # backward bytes of the attention/MLP blocks (ledger) at evenly spaced
    # retained fractions, next to the allocator's post-forward mark
    law = None
    if not args.no_law:
        from paper_2501_09767_b200 import ledger as L
        pts = []
        # evenly spaced fractions; when full retention does not fit (dense OOM
        # above) the law is measured on the halved grid instead
        fracs = (1.0, 0.5, 0.25) if not (dense and dense.get("oom")) else (0.5, 0.25, 0.125)
        for f in fracs:
            led = L.Ledger(keep_series=False)
            try:
                with L.use(led):
                    loss, _ = model.forward_step(staged, pattern_source=M.FractionSource(
                        f, cfg.block_size), segments=segments)
                    loss.backward()
            except torch.cuda.OutOfMemoryError:
                opt.zero_grad()
                torch.cuda.empty_cache()
                continue
            opt.zero_grad()
            rep = led.report()
            pts.append((f, rep.activation_bytes("layer") / 1e9,
                        model.last_stats["activation_bytes_post_forward"] / 1e9))
        if len(pts) >= 3:
            a, c, r2 = L.affine_fit([p[0] for p in pts], [p[1] for p in pts])
            law = {"retained_fraction": [p[0] for p in pts],
                   "block_activation_gb": [round(p[1], 4) for p in pts],
                   "allocator_gb_post_forward": [round(p[2], 4) for p in pts],
                   "fit_gb": {"slope": a, "intercept": c, "r2": r2},
                   "ratio_half": (pts[1][1] - c) / (pts[0][1] - c)}
        else:
            law = {"skipped": f"only {len(pts)} retained fractions fit in memory"}

    # roofline of the dominant kernel (MLP-scoring gate/up GEMM, all s rows)
    pk, pk_src = peaks()
    flops_gemm = (2.0 if cfg.mlp_variant == "relu" else 4.0) * seq * cfg.hidden_dim * cfg.mlp_dim
    avg_gemm_s = (sum(gemm_ms) / max(len(gemm_ms), 1)) / 1e3
    ach = flops_gemm / avg_gemm_s / 1e12 if gemm_ms else None
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        try:
            tj = json.loads(tfile.read_text())
            if tj.get("seq_len") == seq and tj.get("model") == wl["model"]:
                traffic = tj.get("gemm_gateup_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None
    # the kernel is timed inside a long step: the denominator is the measured
    # SUSTAINED bf16 figure (torch.matmul back to back); the burst figure is
    # reported beside it.  frac > 1 means the kernel beats the sustained matmul
    # (the step interleaves HBM-bound kernels, so the power cap bites less).
    peak_g = pk["bf16_tflops_sustained"]
    roofline = {"kernel": "gemm_tn_pair_kernel<EpiGateUp> (lemo_gemm_gateup, MLP scoring, "
                          "256x256 CTA-pair tiles)",
                "bound": "tensor", "achieved": ach, "peak": peak_g,
                "unit": "TFLOP/s", "frac": (ach / peak_g) if ach else None,
                "peak_burst": pk["bf16_tflops"],
                "frac_burst": (ach / pk["bf16_tflops"]) if ach else None,
                "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write)",
                "peak_source": f"{pk_src} bf16_tflops_sustained (kernel timed inside the step); "
                               f"frac_burst against {pk_src} bf16_tflops",
                "algorithmic_per_launch": flops_gemm, "launches_timed": len(gemm_ms),
                "avg_launch_ms": avg_gemm_s * 1e3}
    nb = seq // cfg.block_size
    bytes_embed = seq * cfg.hidden_dim * 4 + nb * cfg.hidden_dim * 4
    avg_embed_s = (sum(embed_ms) / max(len(embed_ms), 1)) / 1e3
    ach_e = bytes_embed / avg_embed_s / 1e9 if embed_ms else None
    roofline_scoring = {"kernel": "block_embed_kernel (lemo_block_embed, predictor pooling)",
                        "bound": "hbm", "achieved": ach_e, "peak": pk["hbm_gbs"], "unit": "GB/s",
                        "frac": ach_e / pk["hbm_gbs"] if ach_e else None,
                        "algorithmic_per_launch": bytes_embed,
                        "avg_launch_us": avg_embed_s * 1e6}
    step_flops = None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle.cpu_sample import host_cores
            cores = host_cores()
            if reference_available():
                ts = min(args.cpu_tokens, seq)
                tiny_only = args.config == "tiny"
                meas = run_reference_process(["--tiny-steps", "5" if tiny_only else "0",
                                              "--layer-seq", *([] if tiny_only else [str(ts)]),
                                              "--budget-s", "1"], cores)
                if tiny_only:
                    t = meas["tiny"]
                    cpu = {"value": t["tokens_per_s"], "unit": "tokens/s", "cores": cores,
                           "kind": "reference",
                           "sample": "unmodified reference (baseline/_ref): config T full "
                                     f"training step, median of {t['steps']} steps"}
                else:
                    lay = meas[f"layer_{ts}"]
                    cpu = {"value": lay["tokens_per_s"], "unit": "tokens/s", "cores": cores,
                           "kind": "reference",
                           "sample": f"unmodified reference (baseline/_ref): 1 {wl['name']}-width "
                                     f"layer at {ts} tokens fwd+bwd in LeMo predicted mode, LM "
                                     f"head timed alone, extrapolated to {cfg.n_layers} layers "
                                     f"(t_layer={lay['layer_s']:.2f}s, t_head={lay['head_s']:.2f}s)"
                                     + ("" if ts == seq else
                                        f"; a {ts}-token sample of the {seq}-token workload "
                                        "(attention is O(s^2): the 16K CPU rate is lower, see the "
                                        "reference arm)")}
            else:
                from oracle.cpu_sample import CpuSample
                cs = CpuSample(sample_tokens=min(args.cpu_tokens, seq), **cpu_geometry(cfg))
                m_ = cs.measure()
                cpu = {"value": m_["tokens_per_s"], "unit": "tokens/s", "cores": cores,
                       "kind": "port",
                       "sample": f"oracle restatement (baseline/_ref missing), 1 layer on {cs.s} "
                                 f"tokens extrapolated to {cfg.n_layers} layers"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "tokens/s", "cores": None, "kind": "reference",
                   "sample": f"failed: {e}"}

    retained = lemo_stats.get("retained", {})
    attn_f = [v for (l, c), v in retained.items() if c == S.ATTENTION]
    mlp_f = [v for (l, c), v in retained.items() if c == S.MLP]
    act_gb = lemo_stats["activation_bytes_post_forward"] / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic tokens, random-init weights",
        "config": {"workload": f"{args.config}: {wl['name']} LoRA(r=8,q/v)+LeMo predicted patterns",
                   "model": wl["model"], "global_batch": world, "seq_len": seq,
                   "parallelism": f"dp{world}",
                   "l2": "weights + activations far larger than the 126 MB L2 (no flush)"
                   if wbytes > 126e6 else "fits in L2 (tiny model: launch-bound, no flush)",
                   "segments": segments, "block_size": cfg.block_size,
                   "target_retention": 0.5,
                   "scoring_precision": model.scoring_precision},
        "activation_gb_post_forward": act_gb,
        "peak_step_gb": peak_step / 1e9,
        "retained_mean": {"attention": float(np.mean(attn_f)) if attn_f else None,
                          "mlp": float(np.mean(mlp_f)) if mlp_f else None},
        "dense_lora": dense,
        "bf16_scoring": bf16_scoring,
        "speedup_vs_dense": (value / dense["value"]) if dense and dense["value"] else None,
        "activation_reduction_vs_dense": (dense["activation_gb_post_forward"] / act_gb)
        if dense and dense["value"] else None,
        "memory_law": law,
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": 2 * seq * 4,
                "d2h_bytes_per_step": 4},
        "gpu_launches": int(round(launches_per_step * args.steps)),
        "roofline": roofline,
        "roofline_scoring": roofline_scoring,
        "attention": {k: dict(v, bound="tensor", peak=pk["bf16_tflops_sustained"],
                              frac=v["tflops"] / pk["bf16_tflops_sustained"],
                              frac_burst=v["tflops"] / pk["bf16_tflops"])
                      for k, v in attn.items()},
        "mask_flips": audit,
        "refined_rows_per_step": refined_rows,
        "cpu_baseline": cpu,
        "clocks": ck,
    }
    if world > 1:
        # per-rank view of the same run (each rank trains its own sequence)
        mine = {"rank": rank, "ms_per_step": ms_step, "activation_gb_post_forward": act_gb,
                "peak_step_gb": peak_step / 1e9,
                "retained_mean_attention": line["retained_mean"]["attention"]}
        ranks = [None] * world
        dist.all_gather_object(ranks, mine)
        line["per_rank"] = ranks
        line["collective"] = {"backend": args.backend,
                              "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))
                              if args.backend == "nccl" else None,
                              "what": "per-layer LoRA-gradient buckets all-reduced (AVG) inside "
                                      "the backward sweep (parallel.BucketedGradReducer); "
                                      "NCCL_DEBUG=INFO/INIT lines on stderr"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

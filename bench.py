"""Benchmark: fused LLaMA-style block forward + backward, tokens/s (BASELINE.json).

  python bench.py [--gpus N --steps K --warmup W] [--config c4|c3|c1] [--impl coda|reference]

One step = `layer_forward` + `layer_backward` of the reference's
reparameterized block (6 + 13 fused launches) over this rank's tokens, plus
the NCCL all-reduce of weight gradients when N > 1 (token-sharded data
parallelism).  Prints ONE JSON line on rank 0.

  value  — whole-job tokens/s with inputs resident in HBM (device-timed, max over ranks)
  e2e    — same metric through the public API from pinned HOST buffers: the H2D copy of
           each step's inputs and the D2H read of its results are inside the timed region
  roofline — the dominant GEMM launch's achieved TFLOP/s vs the measured bf16 peak
  cpu_baseline — the CPU oracle (reference algorithm, oracle/) on a bounded token sample

`--impl reference` times the reference's CPU algorithm (oracle port; the
Python reference cannot travel to the GPU box) on all host cores instead.
"""

from __future__ import annotations

import argparse
import contextlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (hidden d, LLaMA intermediate I, tokens per GPU (weak) / per job (strong), label)
    "c1": (256, 1024, 128, "tiny LLaMA-style block fp32 (d=256, ffn=1024, 128 tokens)"),
    "c3": (2048, 8192, 8192, "LLaMA-3-1B block shapes (d=2048, ffn=8192, 8192 tokens) bf16 fwd+bwd"),
    "c4": (4096, 14336, 16384, "LLaMA-3-8B block shapes (d=4096, ffn=14336, 16384 tokens) bf16 fwd+bwd"),
    "c5": (4096, 14336, 8192, "LLaMA-3-8B 4-block stack bf16 fwd+bwd, 8192 tokens/GPU/block (65536 over 8 GPUs)"),
    # GQA extension (not a BASELINE config): the real LLaMA-3-8B projection, 8 KV heads of 128
    "c4gqa": (4096, 14336, 16384, "LLaMA-3-8B block shapes with GQA q 4096 + k 1024 + v 1024 "
                                  "(d=4096, ffn=14336, 16384 tokens) bf16 fwd+bwd"),
}
KV = {"c4gqa": 1024}   # k / v span width (default: d, the reference's packed 3d)
BLOCKS = {"c5": 4}
# SMs reserved for the NCCL weight-gradient all-reduce while it overlaps the backward (N > 1).
# Measured cost on one GPU with the same caps: 8 SMs +4.5 % step, 16 SMs +9.4 %
# (profiles/r02_ab_fold_cap.json); NCCL is limited to the same number of CTAs.
DEFAULT_COMM_SMS = 8
FP32 = {"c1"}          # BASELINE config 0 is the fp32 (SIM32) path


def flops_per_token(d: int, inter: int, kv: int | None = None) -> float:
    """fwd+bwd = 3 x 2(d^2 + d*F + I*d + d*Q), F = 2I, Q = 3d; Q = d + 2kv with GQA."""
    f, q = 2 * inter, d + 2 * (d if kv is None else kv)
    return 3 * 2.0 * (d * d + d * f + inter * d + d * q)


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text())
    return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0, "fallback": True}


class NvmlClockSampler:
    """NVML clocks / throttle reasons sampled every 20 ms during the timed region."""

    # nvmlClocksEventReason bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        import pynvml

        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        nv = self.nv

        def run():
            while not self._stop.is_set():
                try:
                    sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                    reasons = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    try:
                        mem = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_MEM)
                        power = nv.nvmlDeviceGetPowerUsage(self.h) / 1e3
                    except Exception:
                        mem = power = None
                    self.samples.append((sm, reasons, mem, power))
                except Exception:
                    pass
                self._stop.wait(0.02)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=2)

    def summary(self) -> dict:
        nv = self.nv
        try:
            mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception:
            mx = None
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({name for _, r, *_ in self.samples for name, bit in self.BITS.items() if r & bit})
        out = {"sm_mhz": statistics.median(s[0] for s in self.samples), "sm_max_mhz": mx, "reasons": reasons,
               "samples": len(self.samples), "sm_mhz_min": min(s[0] for s in self.samples)}
        mem = [s[2] for s in self.samples if s[2] is not None]
        power = [s[3] for s in self.samples if s[3] is not None]
        if mem:
            out["mem_mhz"] = statistics.median(mem)
        if power:
            out["power_w"] = round(statistics.median(power), 1)
        return out


def clock_sampler(index: int):
    try:
        return NvmlClockSampler(index)
    except Exception:
        return ClockSampler(index)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (NVML fallback)."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    fields = [x.strip() for x in out.split(",")] if out else []
                    if len(fields) == 6:          # an error message is not a sample
                        self.samples.append(fields)
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=6)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and
                          s[2 + i].lower() in ("active", "1")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- workload


def make_workload(cd, d, inter, m, start, device, seed=0, blocks=1, fp32=False, kv=None):
    """Synthetic bf16 inputs and random-init weights (N(0, 0.02^2), gains 1 + 0.1 N).

    Weights are identical on every rank (same seed); activations differ per
    shard; RoPE tables start at the shard's first token position.
    """
    import torch

    P = cd.PrecisionMode.SIM32 if fp32 else cd.PrecisionMode.SIMBF16
    g = torch.Generator(device=device).manual_seed(seed)
    gr = torch.Generator(device=device).manual_seed(seed * 1000 + 17 + start)

    def w(*shape, scale=0.02, gen=g):
        t = cd.tensors.alloc_matrix(shape[0], shape[1], P.torch_dtype, device)
        t.copy_(torch.randn(shape, generator=gen, device=device) * scale)
        return cd.DenseMatrix.from_tensor(t, P)

    def gain(n):
        return cd.Vector.from_tensor(1.0 + 0.1 * torch.randn(n, generator=g, device=device), P)

    f = 2 * inter
    qw = d + 2 * (d if kv is None else kv)

    def block():
        return cd.LayerWeights(w_out=w(d, d), gamma_ffn=gain(d), w_gate_up=w(d, f), w_down=w(inter, d),
                               gamma_qkv=gain(d), w_qkv=w(d, qw))

    weights = block() if blocks == 1 else [block() for _ in range(blocks)]
    acts = {name: w(m, width, scale=1.0, gen=gr) for name, width in
            (("x", d), ("z", d), ("grad_qkv", qw), ("grad_residual", d))}
    cos, sin = cd.qkv_rope_tables(m, d, start=start, precision=P, kv_width=kv)
    return weights, acts, cos, sin


def run_step(cd, cfg, weights, acts, cos, sin, hook=None, before_backward=None, bwd_sms=0):
    """One fwd+bwd step: a single block, or a stack when `weights` is a list of blocks.

    `before_backward` (optional) runs after the forward is enqueued — the e2e loop
    uses it to make the backward wait for its own inputs' host-to-device copy.
    `bwd_sms` > 0 caps the backward's GEMM launches at that many SMs, leaving the rest to
    the weight-gradient all-reduce the hook runs on a side stream."""
    from paper_2605_19269_b200 import _native

    if isinstance(weights, (list, tuple)):
        from paper_2605_19269_b200 import stack

        fwd = stack.stack_forward(acts["x"], acts["z"], weights, cos, sin, config=cfg)
        if before_backward is not None:
            before_backward()
        with (_native.limit_sms(bwd_sms) if bwd_sms else contextlib.nullcontext()):
            grads = stack.stack_backward(acts["grad_qkv"], acts["grad_residual"], fwd, weights, config=cfg,
                                         wgrad_hook=hook)
        return fwd, grads[0]
    fwd = cd.layer_forward(acts["x"], acts["z"], weights, cos, sin, config=cfg)
    if before_backward is not None:
        before_backward()
    with (_native.limit_sms(bwd_sms) if bwd_sms else contextlib.nullcontext()):
        bwd = cd.layer_backward(acts["grad_qkv"], fwd.tape, weights, grad_residual=acts["grad_residual"],
                                config=cfg, wgrad_hook=hook)
    return fwd, bwd


class CpuOracle:
    """The reference algorithm on the host cores: the fused-order SIMBF16 oracle
    (oracle/coda_oracle.py, numpy/OpenBLAS using every core) on a token sample."""

    def __init__(self, d, inter, sample_tokens, seed=0, fp32=False, kv=None):
        import numpy as np

        from oracle import coda_oracle as O

        self.O = O
        rng = np.random.default_rng(seed)
        self.mode = O.SIM32 if fp32 else O.SIMBF16
        self.w = O.random_layer(rng, d, 2 * inter, self.mode, scale=0.02, kv_width=kv)
        self.m = sample_tokens
        self.x, self.z = (O.q(rng.standard_normal((self.m, d)), self.mode) for _ in range(2))
        self.cos, self.sin = O.qkv_rope_tables(self.m, d, self.mode, kv_width=kv)
        self.gq = O.q(rng.standard_normal((self.m, d + 2 * (d if kv is None else kv))), self.mode)
        self.gres = O.q(rng.standard_normal((self.m, d)), self.mode)

    def step(self) -> float:
        O = self.O
        t0 = time.perf_counter()
        f = O.layer_forward(self.x, self.z, self.w, self.cos, self.sin, self.mode)
        b = O.layer_backward(self.gq, f, self.w, self.mode, grad_residual=self.gres)
        dt = time.perf_counter() - t0
        self.last = (f, b)
        return dt

    def gpu_parity(self, cd, kv=None) -> dict:
        """The same sample through the CUDA path: worst relative (Frobenius) and max
        absolute error over qkv and the eight gradients vs this oracle's outputs."""
        import numpy as np

        O = self.O
        P = cd.PrecisionMode.SIM32 if self.mode == O.SIM32 else cd.PrecisionMode.SIMBF16
        d = self.x.shape[1]
        M = lambda a: cd.DenseMatrix.from_array(a, P)  # noqa: E731
        V = lambda a: cd.Vector.from_array(a, P)  # noqa: E731
        w = self.w
        weights = cd.LayerWeights(w_out=M(w["w_out"]), gamma_ffn=V(w["gamma_ffn"]), w_gate_up=M(w["w_gate_up"]),
                                  w_down=M(w["w_down"]), gamma_qkv=V(w["gamma_qkv"]), w_qkv=M(w["w_qkv"]))
        cfg = cd.PipelineConfig(hidden=d, ffn=w["w_gate_up"].shape[1], precision=P, kv_width=kv)
        fwd = cd.layer_forward(M(self.x), M(self.z), weights, M(self.cos), M(self.sin), config=cfg)
        bwd = cd.layer_backward(M(self.gq), fwd.tape, weights, grad_residual=M(self.gres), config=cfg)
        f, b = self.last
        pairs = [("qkv", fwd.qkv.data, f["qkv"])] + [(k, getattr(bwd, k).data, b[k]) for k in O.GRAD_KEYS]
        rel = {k: O.rel_error(g, r) for k, g, r in pairs}
        mx = max(float(np.max(np.abs(g - r))) for _, g, r in pairs)
        mref = max(float(np.max(np.abs(r))) for _, _, r in pairs)
        worst = max(rel, key=rel.get)
        return {"rel_err_max": rel[worst], "worst_output": worst, "max_abs_err": mx, "max_abs_ref": mref,
                "tol": 1e-5 if P is cd.PrecisionMode.SIM32 else 2e-2, "vs": "fused-order CPU oracle, same inputs",
                "sample_tokens": self.m}


def upload_bf16(cd, a, dev):
    import numpy as np
    import torch

    t = cd.tensors.alloc_matrix(a.shape[0], a.shape[1], torch.bfloat16, dev)
    t.copy_(torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev))
    return cd.DenseMatrix.from_tensor(t, cd.PrecisionMode.SIMBF16)


def upload_vec(cd, a, dev):
    import numpy as np
    import torch

    return cd.Vector.from_tensor(torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev),
                                 cd.PrecisionMode.SIMBF16)


class NullReduce:
    """World-size-1 stand-in for the data-parallel hook: exercises the unrounded f32
    weight-gradient outputs and their single rounding (kernels.layer_backward)."""

    def __init__(self):
        self.names = []

    def __call__(self, name, tensor):
        self.names.append(name)


def _fixture_weights(cd, w, dev):
    return cd.LayerWeights(w_out=upload_bf16(cd, w["w_out"], dev), gamma_ffn=upload_vec(cd, w["gamma_ffn"], dev),
                           w_gate_up=upload_bf16(cd, w["w_gate_up"], dev), w_down=upload_bf16(cd, w["w_down"], dev),
                           gamma_qkv=upload_vec(cd, w["gamma_qkv"], dev), w_qkv=upload_bf16(cd, w["w_qkv"], dev))


def _fixture_compare(z, got: dict, dev) -> dict:
    """Each output against the fixture: exact (small outputs) or sketch + norm + sampled rows."""
    import numpy as np
    import torch

    from oracle import fullsize as FS

    out = {}
    for k in got:
        t = got[k].tensor
        if f"{k}__full" in z.files:
            out[k] = FS.compare(k, t.double().cpu().numpy(), {"full": z[f"{k}__full"]})
            continue
        fp = {"sketch": z[f"{k}__sketch"].astype(np.float64), "rows": z[f"{k}__rows"].astype(np.float64),
              "row_idx": z[f"{k}__row_idx"]}
        S = torch.from_numpy(FS.sketch_matrix(k, t.shape[0], fp["sketch"].shape[0])).to(dev, torch.float64)
        gs = (S @ t.double()).cpu().numpy()
        gr = t[torch.from_numpy(fp["row_idx"]).to(dev)].double().cpu().numpy()
        out[k] = FS.compare(k, None, fp, got_sketch=gs, got_rows=gr)
        gnorm = float(torch.linalg.vector_norm(t.double()))
        out[k]["norm_ratio"] = gnorm / float(z[f"{k}__norm"])
    return out


def fullsize_parity(name: str, variant: str = "plain") -> dict:
    """Full-size parity of config `name` (c3 / c4, or the c5 4-block stack) on cuda:0 against the
    committed oracle fixture tests/golden/fullsize_<name>.npz (made by
    tests/golden/make_fullsize.py): the same bf16 inputs are regenerated from the fixture's seed,
    the whole block (stack) runs through the public API, and every output is compared by its
    sketch, norm and sampled rows (oracle/fullsize.compare).  The checker only; nothing here is
    timed.  variant: plain | f32_hook | fold."""
    import numpy as np
    import torch

    import paper_2605_19269_b200 as cd
    from oracle import coda_oracle as O
    from oracle import fullsize as FS

    z = np.load(ROOT / "tests" / "golden" / f"fullsize_{name}.npz")
    dev = torch.device("cuda", 0)
    P = cd.PrecisionMode.SIMBF16
    if name in FS.BLOCKS:
        ws_np, acts_np = FS.make_stack_inputs(name, seed=int(z["meta_seed"]))
        ws = [_fixture_weights(cd, w, dev) for w in ws_np]
    else:
        acts_np = FS.make_inputs(name, seed=int(z["meta_seed"]))
        ws = _fixture_weights(cd, FS.weights_of(acts_np), dev)
    acts = {k: upload_bf16(cd, acts_np[k], dev) for k in ("x", "z", "grad_qkv", "grad_residual")}
    del acts_np
    m, d = acts["x"].shape
    f = (ws[0] if isinstance(ws, list) else ws).w_gate_up.cols
    kv = FS.KV.get(name)
    cfg = cd.PipelineConfig(hidden=d, ffn=f, precision=P, fold_gamma=(variant == "fold"), kv_width=kv)
    cos, sin = cd.qkv_rope_tables(m, d, precision=P, kv_width=kv)
    hook = NullReduce() if variant == "f32_hook" else None
    got = {}
    if isinstance(ws, list):
        from paper_2605_19269_b200 import stack

        fwd = stack.stack_forward(acts["x"], acts["z"], ws, cos, sin, config=cfg)
        grads = stack.stack_backward(acts["grad_qkv"], acts["grad_residual"], fwd, ws, config=cfg, wgrad_hook=hook)
        got.update({"qkv": fwd.qkv, "residual": fwd.residual, "x": grads[0].x, "z": grads[0].z})
        for b, g in enumerate(grads):
            got.update({f"{k}.{b}": getattr(g, k) for k in FS.WGRADS + FS.GAINS})
    else:
        fwd = cd.layer_forward(acts["x"], acts["z"], ws, cos, sin, config=cfg)
        bwd = cd.layer_backward(acts["grad_qkv"], fwd.tape, ws, grad_residual=acts["grad_residual"], config=cfg,
                                wgrad_hook=hook)
        got = {"qkv": fwd.qkv, "residual": fwd.residual}
        got.update({k: getattr(bwd, k) for k in O.GRAD_KEYS})
    torch.cuda.synchronize()
    return _fixture_compare(z, got, dev)


def fullsize_parity_dp(name: str, hook, rank: int, world: int, device) -> dict:
    """Data-parallel full-size parity (c3 / c4): every rank runs its strong-scaling token shard
    of the fixture's inputs (RoPE tables at the shard's positions) through layer_forward /
    layer_backward with the bench's weight-gradient hook; after the cross-rank reduction
    the weight and gain gradients must equal the whole batch's, so they are compared with
    the single-GPU fixture.  Collective: every rank calls it."""
    import numpy as np
    import torch

    import paper_2605_19269_b200 as cd
    from oracle import fullsize as FS
    from paper_2605_19269_b200 import parallel

    z = np.load(ROOT / "tests" / "golden" / f"fullsize_{name}.npz")
    P = cd.PrecisionMode.SIMBF16
    acts_np = FS.make_inputs(name, seed=int(z["meta_seed"]))
    ws = _fixture_weights(cd, FS.weights_of(acts_np), device)
    sh = parallel.shard(acts_np["x"].shape[0], rank, world, "strong")
    acts = {k: upload_bf16(cd, np.ascontiguousarray(acts_np[k][sh.start:sh.stop]), device)
            for k in ("x", "z", "grad_qkv", "grad_residual")}
    del acts_np
    d = acts["x"].shape[1]
    kv = FS.KV.get(name)
    cfg = cd.PipelineConfig(hidden=d, ffn=ws.w_gate_up.cols, precision=P, kv_width=kv)
    cos, sin = cd.qkv_rope_tables(sh.rows, d, start=sh.start, precision=P, kv_width=kv)
    fwd = cd.layer_forward(acts["x"], acts["z"], ws, cos, sin, config=cfg)
    bwd = cd.layer_backward(acts["grad_qkv"], fwd.tape, ws, grad_residual=acts["grad_residual"], config=cfg,
                            wgrad_hook=hook)
    if hook is not None and hasattr(hook, "wait"):
        hook.wait()
    torch.cuda.synchronize()
    return _fixture_compare(z, {k: getattr(bwd, k) for k in parallel.REDUCED}, device)


def fullsize_summary(res: dict, tol: float = 2e-2) -> dict:
    worst = max(res, key=lambda k: res[k]["rel"])
    return {"rel_err_max": res[worst]["rel"], "worst_output": worst,
            "max_abs_err": max(r["max_abs"] for r in res.values()),
            "rows_rel_max": max(r.get("rows_rel", 0.0) for r in res.values()),
            "tol": tol, "pass": all(r["rel"] <= tol and r.get("rows_rel", 0.0) <= tol for r in res.values()),
            "outputs": len(res),
            "vs": "token-chunked fused-order CPU oracle over the full block (tests/golden/fullsize_*.npz): "
                  "sketch-estimated Frobenius rel error per output + exact sampled rows"}


def cpu_oracle_tokens_per_s(d, inter, sample_tokens, seconds_budget=20.0, max_reps=5, fp32=False, kv=None):
    runner = CpuOracle(d, inter, sample_tokens, fp32=fp32, kv=kv)
    times = []
    t_start = time.perf_counter()
    while True:
        times.append(runner.step())
        if time.perf_counter() - t_start > seconds_budget or len(times) >= max_reps:
            break
    best = min(times)
    return sample_tokens / best, best, len(times), runner


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------- arms


def reference_arm(args, rank, world):
    """--impl reference: the reference algorithm on the host cores (oracle port)."""
    d, inter, tokens, label = CONFIGS[args.config]
    if rank != 0:
        return
    sample = min(args.cpu_sample, tokens)
    runner = CpuOracle(d, inter, sample, fp32=args.config in FP32, kv=KV.get(args.config))
    for _ in range(max(1, args.warmup)):
        runner.step()
    per_step = [runner.step() for _ in range(args.steps)]
    t = statistics.median(per_step)
    value = sample / t
    cores = host_cores()
    line = {
        "impl": "reference", "metric": "block fwd+bwd tokens/s", "value": value, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32 (bf16 storage grid)",
        "data": "synthetic", "config": {"workload": label, "tokens_sampled_per_step": sample},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port",
                         "sample": f"{sample} tokens of the {args.config} block per step, numpy/OpenBLAS all cores"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def wgrad_shapes(d, inter, kv=None):
    """The all-reduced gradients of one block in production order (kernels.py:936-1001)."""
    q = d + 2 * (d if kv is None else kv)
    return [("w_qkv", (d, q)), ("gamma_qkv", (d,)), ("w_down", (inter, d)), ("w_gate_up", (d, 2 * inter)),
            ("gamma_ffn", (d,)), ("w_out", (d, d))]


def launcher_check(args, rank, world):
    """--launcher-check: gloo on CPU, no kernels.  Each step all-reduces zero-filled f32 buffers
    with the block's gradient shapes through the same hook class the GPU path uses."""
    import torch
    import torch.distributed as dist

    from paper_2605_19269_b200 import parallel

    dist.init_process_group("gloo")
    d, inter, tokens, label = CONFIGS[args.config]
    tokens = args.tokens or tokens
    sh = parallel.shard(tokens, rank, world, args.scaling)
    bufs = [torch.zeros(shape, dtype=torch.float32) for _, shape in wgrad_shapes(d, inter, KV.get(args.config))]
    hook = parallel.WgradReduceScatter(dist) if args.wgrad_reduce == "rsag" else parallel.WgradAllReduce(dist)

    def step():
        for (name, _), b in zip(wgrad_shapes(d, inter), bufs):
            hook(name, b)
        hook.wait()

    for _ in range(args.warmup):
        step()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dist.barrier()
    ms = (time.perf_counter() - t0) * 1e3
    t = torch.tensor([ms])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    total = torch.tensor([sh.rows])
    dist.all_reduce(total)
    nbytes = sum(b.numel() * 4 for b in bufs)
    if rank == 0:
        print(json.dumps({
            "metric": "block fwd+bwd tokens/s", "launcher_check": True, "value": None, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": args.scaling, "backend": "gloo (CPU, no kernels)",
            "config": {"workload": label, "tokens_per_rank": sh.rows, "global_tokens": int(total.item())},
            "allreduce_bytes_per_step": nbytes, "names": hook.names[:len(bufs)],
        }), flush=True)
    dist.destroy_process_group()


def coda_arm(args, rank, world, local_rank):
    import torch

    import paper_2605_19269_b200 as cd
    from paper_2605_19269_b200 import _native

    device = torch.device("cuda", 0 if args.share_gpu else local_rank)
    torch.cuda.set_device(device)
    dist = None
    if world > 1 and args.share_gpu:
        # test mode: every rank on cuda:0 over gloo (NCCL needs one GPU per rank); the
        # collectives stage through the host, so nothing here is a measurement
        import torch.distributed as dist  # noqa: F811

        dist.init_process_group("gloo")
    elif world > 1 or args.force_dist:
        import torch.distributed as dist  # noqa: F811

        comm = args.comm_sms if args.comm_sms is not None else (DEFAULT_COMM_SMS if world > 1 else 0)
        if comm > 0:
            # the all-reduce runs concurrently with the SM-capped backward GEMMs: keep NCCL
            # inside the SMs left to it
            os.environ.setdefault("NCCL_MAX_CTAS", str(comm))

        if world == 1:   # --force-dist: a 1-rank NCCL group, to exercise the collective path on one GPU
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            dist.init_process_group("nccl", device_id=device, rank=0, world_size=1)
        else:
            dist.init_process_group("nccl", device_id=device)
    from paper_2605_19269_b200 import parallel

    d, inter, tokens, label = CONFIGS[args.config]
    tokens = args.tokens or tokens
    sh = parallel.shard(tokens, rank, world, args.scaling)
    m = sh.rows
    P = cd.PrecisionMode.SIMBF16
    kv = KV.get(args.config)
    cfg = cd.PipelineConfig(hidden=d, ffn=2 * inter, precision=P, kv_width=kv, fold_gamma=args.fold_gamma)
    nblocks = BLOCKS.get(args.config, 1)
    fp32 = args.config in FP32
    if fp32:
        if args.fold_gamma:
            raise SystemExit("--fold-gamma is implemented for the bf16 path")
        P = cd.PrecisionMode.SIM32
        cfg = cd.PipelineConfig(hidden=d, ffn=2 * inter, precision=P)
    weights, acts, cos, sin = make_workload(cd, d, inter, m, sh.start, device, blocks=nblocks, fp32=fp32, kv=kv)
    # SMs left to the side-stream all-reduce while a reduction is in flight (the hook caps the
    # persistent GEMMs from the first weight gradient of the backward until wait())
    comm_sms = args.comm_sms if args.comm_sms is not None else (DEFAULT_COMM_SMS if world > 1 else 0)
    if dist is None:
        hook = None
    elif args.wgrad_reduce == "peer" and not fp32:
        # weight gradients summed across ranks inside their GEMM epilogue (peer memory);
        # only the gain vectors go through NCCL, so no SMs are held back for it
        comm_sms = 0
        hook = parallel.PeerWgradReduce(dist, device)
    elif args.wgrad_reduce == "rsag" and args.wgrad_dtype == "f32" and not fp32:
        hook = parallel.WgradReduceScatter(dist, device, reserve_sms=comm_sms)
    else:
        hook = parallel.WgradAllReduce(dist, device, f32=args.wgrad_dtype == "f32", reserve_sms=comm_sms)
    bwd_sms = 0

    def step():
        out = run_step(cd, cfg, weights, acts, cos, sin, hook, bwd_sms=bwd_sms)
        if hook is not None:
            hook.wait()
        return out

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    if args.ncu:
        # profiler pass: a few steps, nothing else (numbers printed under ncu are not bench values)
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("measure")   # ncu --nvtx --nvtx-include "measure/" = one step
        for _ in range(max(1, args.steps)):
            step()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        # launch tags of one step, in order (tools/traffic_json.py maps ncu rows onto them)
        rows = []
        _native.record_tags(rows)
        step()
        _native.record_tags(None)
        if rank == 0:
            out = ROOT / "gpurun_out"
            out.mkdir(exist_ok=True)
            (out / f"launch_tags_{args.config}.json").write_text(json.dumps(rows))
        if dist is not None:
            dist.destroy_process_group()
        return
    for _ in range(args.warmup):
        step()
    barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def capture(fn):
        """Capture one call of `fn` (a whole step: its launches, the hook's collectives on
        the side stream and the join) as a CUDA graph (cd.StepGraph); replaying it costs the
        host ~10 us instead of the step's Python enqueue (1.3 ms, 3-7 ms with the
        per-gradient collective calls), which a strong-scaled rank (~2.4 ms of device work
        at P = 8) cannot hide."""
        sg = cd.StepGraph(fn, device, warmup=0)
        return sg.graph, sg.launches, sg.outputs

    graph = None
    graph_error = None
    if args.graph:
        try:
            graph, per_step_launches, _ = capture(step)
            for _ in range(2):
                graph.replay()
        except RuntimeError as exc:   # e.g. a collective this NCCL / torch cannot capture: time it eagerly
            graph, graph_error = None, f"{type(exc).__name__}: {exc}"[:300]
            print(f"bench.py: CUDA graph capture failed, timing eager steps ({graph_error})", file=sys.stderr)
            torch.cuda.synchronize()
            step()
        barrier()
    launches0 = _native.launch_count()
    with clock_sampler(device.index) as clocks:
        barrier()
        h0 = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                step()
        e1.record(stream)
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
        barrier()
    launches = _native.launch_count() - launches0
    if graph is not None:
        launches = per_step_launches * args.steps   # replayed graph nodes (captured once)
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = world * m / (ms_step / 1e3)

    # ---- gamma folded into W (north_star), A/B against the reference schedule: the two step
    # variants interleaved on this GPU (same power state), median device time of each
    fold_ab = None
    if world == 1 and not fp32 and not args.fold_gamma and args.ab_rounds > 0:
        cfg_f = cd.PipelineConfig(hidden=d, ffn=2 * inter, precision=P, kv_width=kv, fold_gamma=True)
        variants = {"reference_schedule": cfg, "gamma_folded": cfg_f}
        times = {k: [] for k in variants}
        for k, c in variants.items():
            run_step(cd, c, weights, acts, cos, sin)
        for _ in range(args.ab_rounds):
            for k, c in variants.items():
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                run_step(cd, c, weights, acts, cos, sin)
                a1.record(stream)
                torch.cuda.synchronize()
                times[k].append(a0.elapsed_time(a1))
        med = {k: statistics.median(v) for k, v in times.items()}
        fold_ab = {"rounds": args.ab_rounds, "ms_reference_schedule": med["reference_schedule"],
                   "ms_gamma_folded": med["gamma_folded"],
                   "speedup": med["reference_schedule"] / med["gamma_folded"],
                   "note": "fold launches (W' = diag(gamma) W) inside every folded step"}

    # ---- the other reading of the config text: weak scaling (the config's tokens on EVERY rank),
    # reported beside the strong-scaled headline for N > 1
    weak = None
    # (also under --force-dist at world size 1, so the one-GPU tests exercise this path)
    if (world > 1 or args.force_dist) and args.scaling == "strong":
        ww, wa, wc, wsn = make_workload(cd, d, inter, tokens, rank * tokens, device, blocks=nblocks, fp32=fp32,
                                        kv=kv)

        def weak_step():
            run_step(cd, cfg, ww, wa, wc, wsn, hook, bwd_sms=bwd_sms)
            if hook is not None:
                hook.wait()

        for _ in range(2):
            weak_step()
        weak_graph = capture(weak_step)[0] if graph is not None else None
        run_weak = weak_graph.replay if weak_graph is not None else weak_step
        run_weak()
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            run_weak()
        e1.record(stream)
        barrier()
        t = torch.tensor([e0.elapsed_time(e1)], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wms = float(t.item()) / args.steps
        weak = {"tokens_per_gpu": tokens, "global_tokens": world * tokens, "ms_per_step": wms,
                "value": world * tokens / (wms / 1e3), "unit": "tokens/s", "cuda_graph": weak_graph is not None}
        del ww, wa, wc, wsn, weak_graph

    # ---- e2e through the public API from pinned host buffers.  Every step copies its
    # inputs H2D and reads its results D2H inside the timed region; the copies run on
    # their own streams (double-buffered inputs) so they overlap the previous/next step.
    host = [{k: (v.tensor * (1.0 + 0.01 * j)).to(v.tensor.dtype).cpu().pin_memory() for k, v in acts.items()}
            for j in range(2)]
    dev_in = [{k: torch.empty_like(v.tensor) for k, v in acts.items()} for _ in range(2)]
    h2d = sum(t.numel() * t.element_size() for t in host[0].values())
    out_host = [torch.empty((m, d), dtype=P.torch_dtype).pin_memory() for _ in range(2)]
    gam_host = [torch.empty((2, d), dtype=torch.float32).pin_memory() for _ in range(2)]
    d2h = out_host[0].numel() * out_host[0].element_size() + gam_host[0].numel() * 4
    h2d_stream, d2h_stream = torch.cuda.Stream(device), torch.cuda.Stream(device)

    # Forward inputs (x, z) are copied first with their own event, so a step's forward
    # starts after 268 MB rather than all 805 MB; the backward waits for grad_qkv /
    # grad_residual.  Results of step s are kept referenced until their D2H copy is
    # done (no record_stream: the allocator then reuses the same blocks every step).
    fwd_keys = ("x", "z")

    timeline = os.environ.get("CODA_E2E_TIMELINE") == "1"

    def mark(marks, what, st):
        if timeline:
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            marks.append((what, e))

    # with --graph, each input buffer's step is one captured graph (its launches and the
    # hook's collectives); the copies and the cross-stream events stay outside, so the copy
    # of step s+1 still overlaps step s.  The graph's step waits for all of its inputs.
    e2e_graphs = None
    if graph is not None:
        def graph_step(b):
            a = {k: cd.DenseMatrix.from_tensor(dev_in[b][k], P) for k in dev_in[b]}
            out = run_step(cd, cfg, weights, a, cos, sin, hook, bwd_sms=bwd_sms)
            if hook is not None:
                hook.wait()
            return out

        for b in range(2):
            graph_step(b)
        e2e_graphs = [capture(lambda b=b: graph_step(b)) for b in range(2)]

    def e2e_run(nsteps):
        marks = []
        mark(marks, "begin", stream)
        copied_f = [torch.cuda.Event() for _ in range(2)]
        copied_b = [torch.cuda.Event() for _ in range(2)]
        consumed = [torch.cuda.Event() for _ in range(2)]
        done = [torch.cuda.Event() for _ in range(2)]
        pending = [None, None]

        def issue_copy(s):
            b = s % 2
            with torch.cuda.stream(h2d_stream):
                if s >= 2:
                    h2d_stream.wait_event(consumed[b])
                mark(marks, f"copy{s} start", h2d_stream)
                for k in fwd_keys:
                    dev_in[b][k].copy_(host[b][k], non_blocking=True)
                copied_f[b].record(h2d_stream)
                for k in host[b]:
                    if k not in fwd_keys:
                        dev_in[b][k].copy_(host[b][k], non_blocking=True)
                copied_b[b].record(h2d_stream)
                mark(marks, f"copy{s} end", h2d_stream)

        h2d_stream.wait_stream(stream)
        issue_copy(0)
        for s in range(nsteps):
            b = s % 2
            if s + 1 < nsteps:
                issue_copy(s + 1)
            if pending[b] is not None:   # step s-2's results: D2H finished before their blocks are reused
                stream.wait_event(done[b])
                pending[b] = None
            if e2e_graphs is not None:
                stream.wait_event(copied_b[b])
                mark(marks, f"step{s} start", stream)
                g, _, (_, bwd) = e2e_graphs[b]
                g.replay()
            else:
                stream.wait_event(copied_f[b])
                mark(marks, f"step{s} start", stream)
                a = {k: cd.DenseMatrix.from_tensor(dev_in[b][k], P) for k in dev_in[b]}
                _, bwd = run_step(cd, cfg, weights, a, cos, sin, hook,
                                  before_backward=lambda: stream.wait_event(copied_b[b]), bwd_sms=bwd_sms)
                if hook is not None:
                    hook.wait()
            consumed[b].record(stream)
            mark(marks, f"step{s} end", stream)
            with torch.cuda.stream(d2h_stream):
                d2h_stream.wait_event(consumed[b])
                out_host[b].copy_(bwd.x.tensor, non_blocking=True)
                gam_host[b][0].copy_(bwd.gamma_ffn.tensor, non_blocking=True)
                gam_host[b][1].copy_(bwd.gamma_qkv.tensor, non_blocking=True)
                done[b].record(d2h_stream)
            pending[b] = bwd
        stream.wait_stream(d2h_stream)
        stream.wait_stream(h2d_stream)
        pending[0] = pending[1] = None   # later allocations on `stream` are ordered after the D2H
        if timeline:
            torch.cuda.synchronize()
            t0 = marks[0][1]
            for what, e in sorted(marks[1:], key=lambda x: t0.elapsed_time(x[1])):
                print(f"  e2e {what:14s} {t0.elapsed_time(e):9.2f} ms", file=sys.stderr)

    e2e_run(max(4, args.warmup))
    barrier()
    e0.record(stream)
    e2e_run(args.steps)
    e1.record(stream)
    barrier()
    ms_e2e = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms_e2e], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    e2e_value = world * m / (ms_e2e / args.steps / 1e3)

    # ---- roofline of the dominant launch: per-launch CUDA events over 2 profiled steps
    prof = _native.profile_launches(lambda: step(), reps=2)
    pk = peaks()
    roofline = None
    if prof:
        # the dominant tensor-core launch (HBM-bound helpers — rope, finalizers, the DP
        # slice rounding, the SIM32 operand split — are not what the tensor roofline bounds)
        gemms = [r for r in prof.values() if r["flops"] > 0] or list(prof.values())
        top = max(gemms, key=lambda r: r["total_ms"])
        achieved = top["flops"] / (top["avg_ms"] / 1e3) / 1e12
        # the sustained (power-capped) peak when the timed region ran under the power cap,
        # the burst peak when it did not (short steps, e.g. C3/C1, finish before the cap)
        capped = "sw_power_cap" in (clocks.summary() or {}).get("reasons", ["sw_power_cap"])
        peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) if capped else pk["bf16_tflops"]
        traffic, traffic_src = None, None
        tp = ROOT / "profiles" / "traffic.json"
        if tp.exists():
            tj = json.loads(tp.read_text())
            traffic = tj.get(f"{args.config}:{top['name']}")
            meta = tj.get("_meta", {}).get(args.config)
            if traffic is not None:
                traffic_src = ("profiles/traffic.json: " + (f"ncu DRAM bytes of build {meta['git']} ({meta['date']})"
                                                            if meta else "ncu DRAM bytes of a round-1 build"))
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src, "kernel": top["name"],
                    "peak_kind": ("measured sustained bf16 (MEASURED_PEAKS.json; sw_power_cap seen in the timed region)"
                                  if capped else "measured burst bf16 (MEASURED_PEAKS.json; no power cap in the timed region)"),
                    "share_of_step": top["total_ms"] / sum(r["total_ms"] for r in prof.values())}
    total_flops = flops_per_token(d, inter, kv) * m * nblocks
    block_tflops = total_flops / (ms_step / 1e3) / 1e12

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sample = min(args.cpu_sample, m)
        tps, secs, reps, runner = cpu_oracle_tokens_per_s(d, inter, sample, seconds_budget=20.0, max_reps=3,
                                                          fp32=fp32, kv=kv)
        parity = runner.gpu_parity(cd, kv=kv)
        cpu = {"value": tps, "unit": "tokens/s", "cores": host_cores(), "kind": "port",
               "sample": f"{sample} tokens of the {args.config} block, fused-order "
                         f"{'SIM32' if fp32 else 'SIMBF16'} oracle, "
                         f"best of {reps} ({secs:.2f} s each)"}

    fullsize = None
    have_fixture = (ROOT / "tests" / "golden" / f"fullsize_{args.config}.npz").exists()
    if dist is not None and hook is not None and not args.no_parity and args.tokens is None and \
            args.scaling == "strong" and not fp32 and not args.fold_gamma and args.config in ("c3", "c4", "c4gqa") and \
            have_fixture:
        # every rank runs its shard of the fixture's batch; the reduced weight and gain gradients
        # must equal the single-GPU oracle's (not timed; a collective, so all ranks take part)
        res = fullsize_parity_dp(args.config, hook, rank, world, device)
        if rank == 0:
            fullsize = fullsize_summary(res)
            fullsize["vs"] = (f"token-chunked fused-order CPU oracle of the whole block: the {len(res)} weight and "
                              f"gain gradients after the {world}-rank {type(hook).__name__} reduction of "
                              "token-sharded backward passes (sketch + sampled rows)")
    elif rank == 0 and world == 1 and not args.no_parity and args.tokens is None and have_fixture:
        # the measured configuration itself, every output, against the pinned oracle (not timed)
        fullsize = fullsize_summary(fullsize_parity(args.config, "fold" if args.fold_gamma else "plain"))

    if rank == 0:
        line = {
            "metric": "block fwd+bwd tokens/s", "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32" if fp32 else "bf16",
            "data": "synthetic (random-init weights, N(0,1) activations)",
            "config": {"workload": label, "blocks": nblocks, "tokens_per_gpu": m, "global_tokens": world * m,
                       "hidden": d,
                       "intermediate": inter, "ffn_interleaved": 2 * inter, "qkv": d + 2 * (d if kv is None else kv),
                       "parallelism": f"token-sharded dp{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (>=100 MB activations per launch)"},
            "block_tflops": block_tflops,
            "frac_of_bf16_peak": block_tflops / pk["bf16_tflops"],
            "clocks": clocks.summary(),
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "cuda_graph": e2e_graphs is not None},
            "gpu_launches": launches,
            "host_enqueue_ms_per_step": host_ms,
            "cuda_graph": graph is not None,
            "graph_error": graph_error,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "parity": parity,
            "parity_fullsize": fullsize,
            "weak_scaling": weak,
            "fold_gamma_ab": fold_ab,
            "comm_sms": comm_sms if dist is not None else 0,
            "wgrad_allreduce_dtype": args.wgrad_dtype if dist is not None else None,
            "wgrad_reduce": (type(hook).__name__ if hook is not None else None),
            "share_gpu": bool(args.share_gpu),
            "fold_gamma": bool(args.fold_gamma),
            "launch_breakdown_ms": {k: round(v["avg_ms"], 4) for k, v in (prof or {}).items()},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def free_port() -> int:
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def spawn(args, argv) -> int:
    """`--gpus N` without a torchrun environment: launch N ranks of this script through
    torch.distributed.run (one process per GPU, 127.0.0.1 rendezvous) and return its exit
    code.  Fails loudly when fewer than N CUDA devices are visible (unless --launcher-check,
    which runs the launch / rendezvous / all-reduce / max-over-ranks machinery on CPU)."""
    if not args.launcher_check and not args.share_gpu:
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) are visible",
                  file=sys.stderr, flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd, cwd=str(ROOT))


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("coda", "reference"), default="coda")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="c4")
    ap.add_argument("--scaling", choices=("strong", "weak"), default=None,
                    help="multi-GPU token sharding (default: strong for the 16384-token C4/C3 jobs, weak for "
                         "the per-GPU C5 stack)")
    ap.add_argument("--tokens", type=int, default=None,
                    help="override the config's token count (per-rank shape proxies at N=1)")
    ap.add_argument("--fold-gamma", action="store_true", help="gains folded into W (north_star variant)")
    ap.add_argument("--ab-rounds", type=int, default=8,
                    help="interleaved same-GPU A/B rounds of the reference schedule vs gamma folded (0 = skip)")
    ap.add_argument("--comm-sms", type=int, default=None,
                    help="SMs left to the NCCL all-reduce while it overlaps the backward (default 8 when N > 1)")
    ap.add_argument("--wgrad-dtype", choices=("f32", "bf16"), default="f32",
                    help="dtype of the data-parallel weight-gradient all-reduce (f32: single rounding, "
                         "the reference's; bf16 halves the bytes)")
    ap.add_argument("--wgrad-reduce", choices=("rsag", "allreduce", "peer"), default="rsag",
                    help="data-parallel weight gradients: NCCL reduce-scatter of the f32 sums, bf16 rounding of "
                         "each rank's slice, all-gather of the bf16 slices (default: the reference's single "
                         "rounding with 25%% fewer bytes than an f32 all-reduce); NCCL all-reduce; or the sum "
                         "fused into the weight-gradient GEMM epilogue over peer memory (coda_gemm_peer_reduce)")
    ap.add_argument("--cpu-sample", type=int, default=256)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the full-size oracle parity check (c3/c4)")
    ap.add_argument("--ncu", action="store_true", help="profiling pass only (no timing / JSON line)")
    ap.add_argument("--graph", action="store_true", default=None,
                    help="replay each step (device-timed, weak-scaling and e2e loops) as one captured CUDA graph "
                         "(default: on when N > 1 and for C1, where the host enqueue of a step would "
                         "otherwise exceed its device time)")
    ap.add_argument("--no-graph", dest="graph", action="store_false")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the NCCL wgrad all-reduce path even at world size 1 (collective overlap check)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="test mode: N ranks share cuda:0 over gloo (the multi-rank bench path on a one-GPU "
                         "box; no CUDA graphs, all-reduce hook; not a measurement)")
    ap.add_argument("--launcher-check", action="store_true",
                    help="CPU/gloo check of the multi-rank launch: rendezvous, the per-step weight-gradient "
                         "all-reduce of this config's shapes, max-over-ranks timing and the rank-0 JSON line "
                         "(no kernels; not a measurement)")
    args = ap.parse_args(argv)
    args.warmup = max(3, args.warmup)
    if args.scaling is None:
        args.scaling = "weak" if args.config == "c5" else "strong"
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args, argv)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr, flush=True)
        return 2
    if args.graph is None:   # host-enqueue-bound steps: the strong-scaled ranks and the tiny C1 block
        args.graph = (world > 1 or args.config == "c1") and not args.share_gpu
    if args.share_gpu:
        if args.graph:
            print("bench.py: --share-gpu runs gloo collectives, which CUDA graphs cannot capture", file=sys.stderr)
            return 2
        args.wgrad_reduce = "allreduce"
    if args.launcher_check:
        launcher_check(args, rank, world)
    elif args.impl == "reference":
        reference_arm(args, rank, world)
    else:
        coda_arm(args, rank, world, local_rank)
    return 0


if __name__ == "__main__":
    sys.exit(main())

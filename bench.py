#!/usr/bin/env python
"""bench.py -- dynamically scaled Float8Linear fwd+bwd step on B200 (TorchAO §2.1, Appendix A).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5|...] [--sub c2,c3,c5]
                    [--impl ours|reference]

One step = one pass of the whole hot path (plus a7 at N>1) over
one batch: amax -> scale -> cast (X, W, dY) -> Y = X W^T, dX = dY W, dW = dY^T X, all
in libfp8train.so through the C-ABI (fp8_linear_fwd / fp8_linear_bwd).
  N = 1 : headline c4 = BASELINE.json configs[3], the largest single-GPU config (Llama-3-70B
          MLP w1, M=16384 K=8192 N=28672, MXFP8 block-32 E8M0, bf16 in/out); the same run
          measures c2 (configs[1], tensorwise), c3 (configs[2], one layer's seven rowwise
          linears) and c5 through the FSDP gather path at one rank (configs[4]) under "sub".
  N > 1 : c5 (Llama-3.1-405B w1, K=16384 N=53248, 8192 tokens per rank), FSDP2-style weak
          scaling: each rank owns N/P weight rows; a step adds the FP8 weight gather (amax
          all-reduce MAX + FP8 all-gather) before the forward and the dW reduce-scatter.
Inputs come from synth.device (the parity tests' generator, run on the GPU; SHA-256 recorded).
Prints ONE JSON line on rank 0 (contract: DESIGN.md §8).  --impl reference times the
CPU oracle (oracle/) on a bounded sample of the same workload on the host cores.
"""

import argparse
import json
import os
import statistics
import sys
import threading
import time

# NCCL writes its debug/version banner to stdout by default; the contract wants exactly one JSON
# line on stdout, so route NCCL's log to stderr unless the caller chose a file (and main() points
# fd 1 at stderr for the whole run, writing only the JSON line to the original stdout).
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
_JSON_FD = None


def emit(line):
    """Write the one JSON result line to the original stdout."""
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP8 linear fwd+bwd TFLOPS/GPU vs FP8 peak & BF16; cast GB/s vs HBM; 1-8 GPU"

CONFIGS = {
    "c2": dict(M=16384, N=14336, K=4096, recipe="tensorwise", cfg="c2",
               workload="c2: Llama-3-8B MLP w1 linear fwd+bwd, M=16384 tokens, K=4096, N=14336, "
                        "tensorwise e4m3 fwd / e5m2 grad, bf16 in/out (BASELINE.json configs[1])"),
    "c4": dict(M=16384, N=28672, K=8192, recipe="mxfp8", cfg="c4",
               workload="c4: Llama-3-70B MLP w1 linear fwd+bwd, M=16384, K=8192, N=28672, "
                        "MXFP8 block-32 E8M0 FLOOR, bf16 in/out (BASELINE.json configs[3])"),
    "c3w1": dict(M=16384, N=14336, K=4096, recipe="rowwise", cfg="c3",
                 workload="c3 (w1 linear): Llama-3-8B MLP w1 fwd+bwd, rowwise scaling, bf16 in/out "
                          "(BASELINE.json configs[2])"),
    "c3w1hp": dict(M=16384, N=14336, K=4096, recipe="rowwise_gw_hp", cfg="c3",
                   workload="c3 (w1 linear), rowwise_gw_hp recipe (dW in bf16, PAPER.md:598)"),
    "c5": dict(M=8192, N=53248, K=16384, recipe="tensorwise", cfg="c5",
               workload="c5: Llama-3.1-405B w1 linear fwd+bwd, M=8192 tokens per GPU, K=16384, N=53248, "
                        "tensorwise (BASELINE.json configs[4]; FSDP2 FP8 all-gather at N>1)"),
    "c3": dict(M=16384, K=4096, N=14336, recipe="rowwise", cfg="c3", kind="layer",
               linears=[("wq", 4096, 4096), ("wk", 1024, 4096), ("wv", 1024, 4096), ("wo", 4096, 4096),
                        ("w1", 14336, 4096), ("w3", 14336, 4096), ("w2", 4096, 14336)],
               # linears that read the same input in a Llama layer (the attention norm's output, the MLP
               # norm's output): one X per group, cast once (fp8_linear_fwd_shared)
               shared=[("wq", "wk", "wv"), ("w1", "w3")],
               workload="c3: one Llama-3-8B layer's seven linears (attention wq/wk/wv/wo + MLP w1/w3/w2) fwd+bwd, "
                        "M=16384 tokens, rowwise scaling, bf16 in/out (BASELINE.json configs[2])"),
    "moe": dict(T=32768, E=8, N=14336, K=4096, recipe="rowwise", cfg="c3", kind="moe",
                workload="moe: Mixtral-8x7B-style expert w1 scaled grouped GEMM fwd+bwd (PAPER.md:739 "
                         "scaled_grouped_mm), E=8 experts, K=4096, N=14336, 16384 tokens x top-2 = 32768 routed "
                         "rows, seeded imbalanced routing (expert groups padded to 128 rows), rowwise e4m3/e5m2, "
                         "bf16 in/out"),
}
# oracle sample for the reference arm (per step, so the whole --steps/--warmup run stays within a
# few minutes) and for the cpu_baseline (one step of ~10-30 s of CPU work): same K and value
# recipe, fewer rows
CPU_SAMPLE = dict(M=128, N=2048)
CPU_BASELINE_M = 2560   # tokens of the cpu_baseline sample: ~10-30 s of oracle work on the box's host cores
# the MX oracle spends its time in the element codecs (decode / encode per element), so its sample keeps
# fewer weight rows for the same few seconds per step


def sample_n(cfg):
    return 768 if cfg["recipe"] == "mxfp8" else CPU_SAMPLE["N"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="headline workload; default c4 (the largest single-GPU config, BASELINE.json "
                         "configs[3]) at N=1 and c5 (the FSDP config, configs[4]) at N>1")
    ap.add_argument("--sub", default=None,
                    help="comma list of further configs measured in the same run and reported under 'sub' "
                         "(no e2e / cpu_baseline); default at N=1 with the default headline: c2,c3,c5,c3w1hp,moe "
                         "(c5 through the FSDP gather path, the same-config N=1 point of the N>1 runs; c3w1hp the "
                         "rowwise_gw_hp recipe; moe the scaled grouped GEMM)")
    ap.add_argument("--no-digest", dest="digest", action="store_false",
                    help="skip the SHA-256 of the timed inputs")
    ap.add_argument("--knob", action="append", default=[],
                    help="name=value: select a kernel variant via fp8_set_knob (A/B experiments; default = "
                         "the product path); recorded in the JSON line")
    ap.add_argument("--layer-separate", action="store_true",
                    help="c3 layer: every linear casts its own input (default: wq/wk/wv and w1/w3 read one X, "
                         "cast once through fp8_linear_fwd_shared)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # 24 streamed steps: the first input copy and the last output copy (not overlapped with any compute) are
    # inside the timed region, so fewer steps would mostly measure that pipeline fill and drain
    ap.add_argument("--e2e-steps", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bf16", action="store_true")
    ap.add_argument("--gather", default="auto", choices=["auto", "p2p", "nccl"],
                    help="tensorwise FSDP weight gather: p2p = fused cast-and-push over NVLink peer memory "
                         "(fp8_fsdp_allgather_p2p), nccl = cast + ncclAllGather; auto = p2p, falling back to "
                         "nccl if the peer windows cannot be created (auto uses nccl at N=1: no peers)")
    ap.add_argument("--fsdp", action="store_true",
                    help="use the FSDP path (fp8_fsdp_allgather + pre-cast weight) even at N=1")
    return ap.parse_args()


# ----------------------------------------------------------------------------- oracle arm

def _threads_used():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return int(max(n)) if n else 1
    except Exception:
        return os.cpu_count() or 1


def oracle_step_fn(cfg, Ms=CPU_SAMPLE["M"]):
    """One oracle fwd+bwd on the bounded sample (CPU).  Returns (fn, flops, sample_desc)."""
    import synth
    from oracle import linear as olin
    if cfg.get("kind") == "moe":
        from oracle import grouped as ogrp
        Ts, Es, Ns, K = max(Ms, 128), 2, CPU_SAMPLE["N"] // 2, cfg["K"]
        f = synth.RECIPES[cfg["cfg"]]
        x, w, dy = f("x", (Ts, K), 0, cfg["cfg"]), f("w", (Es * Ns, K), 0, cfg["cfg"]), f("dy", (Ts, Ns), 0, cfg["cfg"])
        offs = [0, Ts // 2 // 64 * 64, Ts]

        def mstep():
            ogrp.forward(x, w, offs, cfg["recipe"])
            ogrp.backward(x, w, dy, offs, cfg["recipe"])

        desc = (f"oracle/grouped forward+backward ({cfg['recipe']}) on a T={Ts}, E={Es}, N={Ns}, K={K} sample of "
                f"the moe workload (same K and value recipe); numpy fp64 GEMMs + fp32/numpy encodes")
        return mstep, 6.0 * Ts * Ns * K, desc
    Ns, K = sample_n(cfg), cfg["K"]
    f = synth.RECIPES[cfg["cfg"]]
    x, w, dy = f("x", (Ms, K), 0, cfg["cfg"]), f("w", (Ns, K), 0, cfg["cfg"]), f("dy", (Ms, Ns), 0, cfg["cfg"])
    recipe = cfg["recipe"]

    def step():
        olin.forward(x, w, recipe)
        olin.backward(x, w, dy, recipe)

    desc = (f"oracle/linear forward+backward ({recipe}) on a {Ms}x{Ns}x{K} (MxNxK) sample of the "
            f"{cfg['cfg']} workload (same K and value recipe, {Ms} of {cfg['M']} tokens, {Ns} of {cfg['N']} "
            f"weight rows); numpy fp64 GEMMs + fp32/numpy encodes")
    return step, 6.0 * Ms * Ns * K, desc


def cpu_baseline(cfg):
    oracle_step_fn(cfg)[0]()  # untimed warm run on the small sample (thread pools, page faults)
    step, flops, desc = oracle_step_fn(cfg, CPU_BASELINE_M)
    t0 = time.perf_counter()
    step()
    dt = time.perf_counter() - t0
    return {"value": flops / dt / 1e12, "unit": "TFLOP/s", "cores": _threads_used(), "kind": "oracle",
            "sample": desc, "seconds": dt}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # N > 1: rank 0 alone runs the oracle
    cfg = CONFIGS[a.config]
    step, flops, desc = oracle_step_fn(cfg)
    for _ in range(a.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(a.steps):
        step()
    dt = time.perf_counter() - t0
    v = flops * a.steps / dt / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt / a.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64 (oracle GEMMs) / fp32 casts", "data": "synthetic",
            "config": {"workload": cfg["workload"], "sample": f"{CPU_SAMPLE['M']}x{sample_n(cfg)}x{cfg['K']}"},
            "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": _threads_used(), "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """NVML sampling of SM clock + throttle reasons while the timed region runs."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.ok = False
        self.samples, self.reasons = [], set()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None
        self._stop = threading.Event()

    def _violation(self):
        """Cumulative power / thermal policy violation times (ns) -- they advance whenever the driver
        held clocks down for that reason, even between two samples."""
        out = {}
        for key, pol in (("sw_power_cap", "NVML_PERF_POLICY_POWER"), ("sw_thermal_slowdown", "NVML_PERF_POLICY_THERMAL")):
            try:
                out[key] = self.nv.nvmlDeviceGetViolationStatus(self.h, getattr(self.nv, pol)).violationTime
            except Exception:
                pass
        return out

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.v0 = self._violation()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()
            v1 = self._violation()
            self.violation_ns = {k: v1[k] - self.v0[k] for k in v1 if k in self.v0}
            for k, dv in self.violation_ns.items():
                if dv > 0:
                    self.reasons.add(k)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "violation_ns": getattr(self, "violation_ns", None)}


# ----------------------------------------------------------------------------- our arm

def _peaks():
    """Roofline denominators: driver-measured MEASURED_PEAKS.json, else the guide's fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm": d["hbm_gbs"], "bf16": d["bf16_tflops"], "bf16_sus": d.get("bf16_tflops_sustained",
                                                                              d["bf16_tflops"]),
                "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sus": 1400.0, "src": "fallback (B200_PROFILING.md)"}


def _traffic(workload_key):
    """Per-launch DRAM bytes of the GEMM from the committed ncu --set full capture (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(workload_key)
    return None


def make_inputs(cfg, M_local, N, K, rank, world, dev, seed=0):
    """Seeded synthetic inputs with the config's value recipe (SURVEY §8d / DESIGN.md "Input recipe"),
    generated on the device by synth.device -- the torch port of the synth generator the parity tests
    use, so at rank 0 these are the tensors tests/test_gpu_fullsize.py checks (same cfg, name, shape
    and seed; the port's agreement with synth is tests/test_gpu_synth.py).  X and dY are per-rank
    token streams (seed + 1000 * rank); W is the same full tensor on every rank, each rank taking its
    FSDP2 row shard [r*N/P, (r+1)*N/P)."""
    from synth import device as sd
    c = cfg["cfg"]
    x = sd.tensor(c, "x", (M_local, K), seed + 1000 * rank, dev)
    dy = sd.tensor(c, "dy", (M_local, N), seed + 1000 * rank, dev)
    w = sd.tensor(c, "w", (N, K), seed, dev, rows=(rank * N // world, (rank + 1) * N // world))
    return x, w, dy


def input_digest(dev_tensors, seeds):
    """SHA-256 of the exact bytes of every timed input tensor (copied to the host once, outside the
    timed region) plus the generator and seeds that made them."""
    import hashlib
    import torch
    out = {"generator": "synth.device (torch port of synth: splitmix64 -> Box-Muller fp64 -> recipe -> "
                        "RNE bf16), verified against synth by tests/test_gpu_synth.py", "seeds": seeds}
    for name, t in dev_tensors.items():
        out["sha256_" + name] = hashlib.sha256(t.contiguous().view(-1).view(torch.uint8).cpu().numpy()
                                               .tobytes()).hexdigest()
    return out


def run_ours(a):
    result = None
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    elif a.fsdp:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("gloo", rank=0, world_size=1)

    import paper_2507_16099_b200 as fp8t  # noqa: F401  (loads libfp8train.so; raises if missing)
    from paper_2507_16099_b200 import _lib as L, ops
    from paper_2507_16099_b200.fsdp import Comm

    cfg = CONFIGS[a.config]
    M, N, K = cfg["M"], cfg["N"], cfg["K"]
    fsdp = world > 1 or a.fsdp
    if fsdp and cfg["recipe"] not in ("tensorwise", "mxfp8"):
        raise SystemExit("low-precision weight all-gather: tensorwise (PAPER.md:596) or mxfp8 (SURVEY §8f.3)")
    mx_fsdp = fsdp and cfg["recipe"] == "mxfp8"
    x, w_shard, dy = make_inputs(cfg, M, N, K, rank, world, dev)
    digest = input_digest({"x": x, "w": w_shard, "dy": dy},
                          {"x": 1000 * rank, "dy": 1000 * rank, "w": 0, "w_rows": [rank * N // world,
                                                                                  (rank + 1) * N // world]}) \
        if a.digest else None
    plan = ops.LinearPlan(M, N, K, recipe=cfg["recipe"], out_dtype=torch.bfloat16, device=dev)
    saved = plan.new_saved(dev)
    y = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    dx = torch.empty((M, K), dtype=torch.bfloat16, device=dev)
    dw = torch.empty((N, K), dtype=torch.bfloat16, device=dev)
    comm = Comm() if fsdp else None
    if fsdp:
        w_full = torch.empty((N, K), dtype=torch.uint8, device=dev)
        w_scale = torch.empty(1, dtype=torch.float32, device=dev)
        w_amax = torch.empty(1, dtype=torch.float32, device=dev)
        dw_shard = torch.empty((N // world, K), dtype=torch.bfloat16, device=dev)
        p2p = None
        gather_impl = "nccl (fp8_fsdp_allgather_mx)" if mx_fsdp else "nccl (fp8_fsdp_allgather)"
        if not mx_fsdp and (a.gather == "p2p" or (a.gather == "auto" and world > 1)):
            from paper_2507_16099_b200.fsdp import P2PWindow
            try:
                p2p = P2PWindow(comm, N * K)
                w_full = p2p.buffer(N, K, dev)
                # pre-flight: the fused gather must reproduce the NCCL gather byte for byte on every rank
                ref_q, ref_s, _ = comm.allgather_fp8(w_shard, "e4m3")
                got_q, got_s, _ = p2p.allgather_fp8(w_shard, "e4m3")
                ok = torch.tensor([int(torch.equal(ref_q, got_q) and torch.equal(ref_s, got_s))], device=dev)
                dist.all_reduce(ok, op=dist.ReduceOp.MIN)
                del ref_q
                if not ok.item():
                    raise RuntimeError("p2p pre-flight: gathered bytes differ from the NCCL gather")
                gather_impl = "p2p (fp8_fsdp_allgather_p2p: cast pushes codes to every rank over NVLink)"
            except Exception as e:  # noqa: BLE001  (IPC / peer access unavailable, pre-flight mismatch)
                if a.gather == "p2p":
                    raise
                if p2p is not None:
                    p2p.close()
                    p2p = None
                w_full = torch.empty((N, K), dtype=torch.uint8, device=dev)
                gather_impl = f"nccl (p2p unavailable: {str(e)[:120]})"
        if mx_fsdp:   # MXFP8 gather (fp8_fsdp_allgather_mx): dim0 + dim1 codes and E8M0 scales
            mx_out = {"q": w_full, "scale": torch.empty(N * K // 32, dtype=torch.uint8, device=dev),
                      "q_t": torch.empty((N, K), dtype=torch.uint8, device=dev),
                      "scale_t": torch.empty(N * K // 32, dtype=torch.uint8, device=dev)}
            mx_ws = torch.empty(N * K // 32, dtype=torch.uint8, device=dev)

    def gather(ww):
        """FSDP weight gather of this step: the pre-cast weight the linear consumes."""
        if mx_fsdp:
            return comm.allgather_mx(ww, "e4m3", out=mx_out, ws=mx_ws)
        if p2p is not None:
            p2p.allgather_fp8(ww, "e4m3", scale=w_scale, amax=w_amax)
        else:
            comm.allgather_fp8(ww, "e4m3", out=w_full, scale=w_scale, amax=w_amax)
        return (w_full, w_scale)

    # dW reduce-scatter at N > 1: fused into the dW GEMM's epilogue over a P2P window
    # (fp8_linear_bwd_rs) unless --gather nccl, with a pre-flight against torch's NCCL reduce-scatter
    rs_win = None
    rs_impl = "torch NCCL reduce_scatter_tensor (bf16)" if world > 1 else None
    if world > 1 and a.gather != "nccl":
        from paper_2507_16099_b200.fsdp import P2PWindow
        try:
            rs_win = P2PWindow(comm, N * K * 2)
            wf0 = gather(w_shard)
            plan.forward(x, None, saved, y=y, w_fp8=wf0)
            plan.backward(dy, saved, dx=dx, dw=dw, w_fp8=wf0)
            ref = torch.empty_like(dw_shard)
            dist.reduce_scatter_tensor(ref, dw)
            ops.linear_backward_rs(plan, dy, saved, rs_win, dw_shard, dx=dx, w_fp8=wf0)
            err = (dw_shard.float() - ref.float()).norm() / ref.float().norm().clamp_min(1e-30)
            ok = torch.tensor([int(bool(err < 1e-2))], device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            del ref
            if not ok.item():
                raise RuntimeError(f"fused reduce-scatter pre-flight: rel err {float(err):.3g} vs NCCL")
            rs_impl = "fused (fp8_linear_bwd_rs: dW GEMM epilogue stores tiles into the owner's staging over NVLink)"
        except Exception as e:  # noqa: BLE001
            if rs_win is not None:
                rs_win.close()
                rs_win = None
            rs_impl = f"torch NCCL reduce_scatter_tensor (fused RS unavailable: {str(e)[:120]})"

    def step(xx=x, ww=w_shard, gg=dy):
        if fsdp:
            wf = gather(ww)
            plan.forward(xx, None, saved, y=y, w_fp8=wf)
            if rs_win is not None:
                ops.linear_backward_rs(plan, gg, saved, rs_win, dw_shard, dx=dx, w_fp8=wf)
            else:
                plan.backward(gg, saved, dx=dx, dw=dw, w_fp8=wf)
                if world > 1:
                    dist.reduce_scatter_tensor(dw_shard, dw)
        else:
            plan.forward(xx, ww, saved, y=y)
            plan.backward(gg, saved, dx=dx, dw=dw, x=xx)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(max(a.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---------------- timed region (device events, max over ranks) ----------------
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_steps = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]   # per-step boundaries
    L.lib.fp8_profile_collect(None, None, 0)
    L.lib.fp8_profile_enable(1)
    n0 = ops.launch_count()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i_ in range(a.steps):
            step()
            ev_steps[i_].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = ops.launch_count() - n0
    L.lib.fp8_profile_enable(0)
    import ctypes
    cap = launches + 16
    kinds = (ctypes.c_int * cap)()
    durs = (ctypes.c_float * cap)()
    nrec = L.lib.fp8_profile_collect(kinds, durs, cap)
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / a.steps
    step_pct = step_percentiles(ev0, ev_steps)

    gather_info = None
    if fsdp:
        # the weight gather alone (same calls as inside the step), device-timed, max over ranks
        for _ in range(3):
            gather(w_shard)
        torch.cuda.synchronize()
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(a.steps):
            gather(w_shard)
        g1.record(stream)
        torch.cuda.synchronize()
        gms = g0.elapsed_time(g1) / a.steps
        if world > 1:
            t = torch.tensor([gms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            gms = float(t.item())
        recv = N * K * (world - 1) // world * (2 + 2 / 32 if mx_fsdp else 1)   # bytes each rank receives
        gather_info = {"impl": gather_impl, "reduce_scatter": rs_impl, "ms": gms, "recv_bytes_per_rank": recv,
                       "busbw_GBps": recv / (gms / 1e3) / 1e9 if world > 1 else None,
                       "nvlink_peak_GBps": 900.0}
        if world > 1:
            # context: the BF16 all-gather of the same shard over NCCL, as FSDP2 without FP8 gathers
            try:
                full_bf16 = torch.empty((w_shard.shape[0] * world, w_shard.shape[1]), dtype=w_shard.dtype, device=dev)
                for _ in range(3):
                    dist.all_gather_into_tensor(full_bf16, w_shard)
                torch.cuda.synchronize()
                barrier()
                b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                b0.record(stream)
                for _ in range(a.steps):
                    dist.all_gather_into_tensor(full_bf16, w_shard)
                b1.record(stream)
                torch.cuda.synchronize()
                bms = b0.elapsed_time(b1) / a.steps
                t = torch.tensor([bms], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                bms = float(t.item())
                gather_info["bf16_allgather_ms"] = bms
                gather_info["fp8_vs_bf16_gather_speedup"] = bms / gms if gms > 0 else None
                del full_bf16
            except Exception as e:   # context only: never lose the line over it
                gather_info["bf16_allgather_error"] = str(e)[:200]

    flops_step = 6.0 * M * N * K            # three GEMMs of 2*M*N*K each (per rank)
    total_flops = flops_step * a.steps * world
    value = total_flops / (ms / 1e3) / 1e12

    # per-kernel durations from the live events
    by = {}
    for i in range(max(nrec, 0)):
        by.setdefault(kinds[i], []).append(durs[i])
    gemm_kind = 5 if cfg["recipe"] == "mxfp8" else 4   # (rowwise_gw_hp's BF16 dW GEMM is kind 6)
    gemm_ms = by.get(gemm_kind, [float("nan")])
    gemm_avg = sum(gemm_ms) / len(gemm_ms)
    # launches per step: forward (1 problem) + backward (dX and dW grouped in one launch);
    # algorithmic flops per launch differ, so achieved = GEMM flops per step / GEMM time per step
    gemm_launches_per_step = len(gemm_ms) / a.steps
    fp8_gemm_flops = (4.0 if cfg["recipe"] == "rowwise_gw_hp" else 6.0) * M * N * K   # gw_hp: dW is bf16
    gemm_tflops = fp8_gemm_flops / (sum(gemm_ms) / a.steps / 1e3) / 1e12
    peaks = _peaks()
    # dense FP8 peak = 2 x measured bf16 cuBLAS (the guide's nominal FP8/BF16 ratio).  The timed region
    # is well under a second, so the burst figure is the denominator; sustained is reported beside it.
    fp8_peak = 2.0 * peaks["bf16"]
    fp8_peak_sus = 2.0 * peaks["bf16_sus"]
    # algorithmic cast bytes per step: per hp element read by amax 2 B, by the cast 2 B,
    # plus 1 B per FP8 layout written (X, W, dY each written in 2 layouts)
    if cfg["recipe"] == "mxfp8":          # one fused dim0+dim1 read, 2 FP8 layouts + E8M0 scales
        cast_bytes = (M * K + (N // world) * K + M * N) * (2 + 2 + 2 / 32.0)
        cast_kinds = (2,)
    elif cfg["recipe"] == "rowwise":       # amax read 2 + cast read 2 + row- and column-scaled layouts 1 + 1
        cast_bytes = (M * K + N * K + M * N) * 6
        cast_kinds = (0, 1)
    elif cfg["recipe"] == "rowwise_gw_hp":  # X, dY: row-scaled layout only (5 B); W: both layouts (6 B)
        cast_bytes = (M * K + M * N) * 5 + N * K * 6
        cast_kinds = (0, 1)
    elif not fsdp:                         # tensorwise: amax 2 + cast 2 + one row-major layout 1 (the
        cast_bytes = (M * K + N * K + M * N) * 5   # backward GEMMs read it MN-major)
        cast_kinds = (0, 1)
    else:                                  # X, dY: amax 2 + cast 2 + one layout 1; W shard: 2 + 2 + 1
        cast_bytes = (M * K + M * N + (N // world) * K) * 5
        cast_kinds = (0, 1)
    cast_ms = sum(sum(by.get(k, [])) for k in cast_kinds) / a.steps
    cast_gbps = cast_bytes / (cast_ms / 1e3) / 1e9 if cast_ms > 0 else None
    step_gemm_share = sum(gemm_ms) / a.steps / ms_step if ms_step > 0 else None

    # ---------------- end-to-end through the public API with host buffers ----------------
    # Every step copies its inputs (X, W, dY) from pinned host memory and its outputs (Y, dX, dW)
    # back, inside the timed region.  Copies run on their own streams, double-buffered against the
    # compute stream (inputs of step i+1 and outputs of step i-1 move while step i computes), i.e.
    # the steady state of a training loop that streams its batches.
    e2e = None
    if a.e2e_steps > 0:
        xh = x.cpu().pin_memory()
        wh = w_shard.cpu().pin_memory()
        gh = dy.cpu().pin_memory()
        dw_out = dw if not fsdp else dw_shard
        yh = torch.empty_like(y, device="cpu").pin_memory()
        dxh = torch.empty_like(dx, device="cpu").pin_memory()
        dwh = torch.empty_like(dw_out, device="cpu").pin_memory()
        ins = [(torch.empty_like(x), torch.empty_like(w_shard), torch.empty_like(dy)) for _ in range(2)]
        outs = [(torch.empty_like(y), torch.empty_like(dx), torch.empty_like(dw_out)) for _ in range(2)]
        s_h2d, s_d2h = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_used = [torch.cuda.Event() for _ in range(2)]     # compute done with the set's inputs
        ev_out = [torch.cuda.Event() for _ in range(2)]
        ev_read = [torch.cuda.Event() for _ in range(2)]     # D2H done with the set's outputs

        def copy_in(i):
            b = i % 2
            with torch.cuda.stream(s_h2d):
                if i >= 2:
                    s_h2d.wait_event(ev_used[b])
                for d_, h_ in zip(ins[b], (xh, wh, gh)):
                    d_.copy_(h_, non_blocking=True)
                ev_in[b].record(s_h2d)

        def compute(i):
            b = i % 2
            stream.wait_event(ev_in[b])
            if i >= 2:
                stream.wait_event(ev_read[b])
            xd, wd, gd = ins[b]
            yo, dxo, dwo = outs[b]
            if fsdp:
                wf = gather(wd)
                plan.forward(xd, None, saved, y=yo, w_fp8=wf)
                if rs_win is not None:
                    ops.linear_backward_rs(plan, gd, saved, rs_win, dwo, dx=dxo, w_fp8=wf)
                elif world > 1:
                    plan.backward(gd, saved, dx=dxo, dw=dw, w_fp8=wf)
                    dist.reduce_scatter_tensor(dwo, dw)
                else:
                    plan.backward(gd, saved, dx=dxo, dw=dw, w_fp8=wf)
                    dwo.copy_(dw)
            else:
                plan.forward(xd, wd, saved, y=yo)
                plan.backward(gd, saved, dx=dxo, dw=dwo, x=xd)
            ev_used[b].record(stream)
            ev_out[b].record(stream)

        def copy_out(i):
            b = i % 2
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev_out[b])
                for h_, d_ in zip((yh, dxh, dwh), outs[b]):
                    h_.copy_(d_, non_blocking=True)
                ev_read[b].record(s_d2h)

        def run(n):
            copy_in(0)
            for i in range(n):
                if i + 1 < n:
                    copy_in(i + 1)
                compute(i)
                copy_out(i)
            ev_last = torch.cuda.Event()
            ev_last.record(s_d2h)
            stream.wait_event(ev_last)

        run(2)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s_h2d.wait_event(e0)
        run(a.e2e_steps)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        h2d = (x.numel() + w_shard.numel() + dy.numel()) * 2
        d2h = (y.numel() + dx.numel() + dw_out.numel()) * 2
        e2e = {"value": flops_step * a.e2e_steps * world / (ems / 1e3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ems / a.e2e_steps,
               "path": "pinned host -> device copies of X, W, dY + fp8_linear_fwd/bwd (C-ABI) + device -> host "
                       "copies of Y, dX, dW, every step; copies on separate streams, double-buffered"}

    # ---------------- cuBLAS BF16 linear of the same shape (context) ----------------
    bf16 = None
    if not a.no_bf16 and not fsdp:
        wb = w_shard

        def bstep():
            torch.matmul(x, wb.t(), out=y)
            torch.matmul(dy, wb, out=dx)
            torch.matmul(dy.t(), x, out=dw)

        for _ in range(3):
            bstep()
        torch.cuda.synchronize()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(a.steps):
            bstep()
        b1.record(stream)
        torch.cuda.synchronize()
        bms = b0.elapsed_time(b1) / a.steps
        bf16 = {"ms_per_step": bms, "tflops": flops_step / (bms / 1e3) / 1e12,
                "speedup_fp8_vs_bf16": bms / ms_step, "impl": "torch.matmul (cuBLAS) bf16, same 3 GEMMs"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
            "warmup": max(a.warmup, 3), "ms_per_step": ms_step, "step_ms_p10_p50_p90": step_pct, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp8 (e4m3 x e5m2 codes, fp32 accumulate, bf16 out)",
            "data": "synthetic (seeded synth generator run on the device, config value recipe; = the parity tests' inputs at rank 0)",
            "config": {"workload": cfg["workload"], "M_per_gpu": M, "N": N, "K": K, "recipe": cfg["recipe"],
                       "parallelism": (f"fsdp{world} (mxfp8 all-gather, shard-local E8M0 scales)" if mx_fsdp else
                                       f"fsdp{world} (fp8 all-gather + amax all-reduce)") if fsdp else "single GPU",
                       "l2": f"inputs larger than L2 (126 MB): X {M * K * 2 / 2**20:.0f} MiB, "
                             f"dY {M * N * 2 / 2**20:.0f} MiB, W {N * K * 2 / 2**20:.0f} MiB bf16; no flush"},
            "roofline": {"bound": "tensor", "kernel": "fp8_gemm_kernel (tcgen05 kind::%s)" %
                         ("mxf8f6f4.block_scale" if cfg["recipe"] == "mxfp8" else "f8f6f4"),
                         "achieved": gemm_tflops, "peak": fp8_peak, "unit": "TFLOP/s",
                         "frac": gemm_tflops / fp8_peak, "traffic": _traffic(a.config),
                         "peak_source": f"{peaks['src']}: bf16_tflops (burst) x 2 (dense FP8/BF16 ratio)",
                         "frac_of_sustained": gemm_tflops / fp8_peak_sus,
                         "algorithmic": f"2*M*N*K = {2.0 * M * N * K:.4g} flop per GEMM problem; the forward "
                                        f"launch has 1 problem, the backward launch 2 (dX, dW)",
                         "launches_per_step": gemm_launches_per_step,
                         "avg_launch_ms": gemm_avg, "share_of_step": step_gemm_share},
            "cast": {"gbps": cast_gbps, "peak_gbps": peaks["hbm"], "frac": (cast_gbps / peaks["hbm"])
                     if cast_gbps else None, "ms_per_step": cast_ms, "algorithmic_bytes_per_step": cast_bytes},
            "kernels_ms_per_step": {name: round(sum(by.get(k, [])) / a.steps, 4)
                                    for k, name in ((0, "amax"), (1, "cast"), (2, "mx_cast"), (3, "transpose_u8"),
                                                    (4, "gemm_fp8"), (5, "gemm_mxfp8"), (6, "gemm_bf16"),
                                                    (7, "p2p_sync"))},
            "bf16": bf16,
            "gather": gather_info,
            "inputs": digest,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        result = line
    if fsdp and p2p is not None:
        p2p.close()
    if fsdp and rs_win is not None:
        rs_win.close()
    if comm is not None:
        comm.close()
    if dist.is_initialized():
        dist.destroy_process_group()
    return result


def step_percentiles(ev0, ev_steps):
    """p10 / median / p90 of the per-step device times (this rank; events on the step stream)."""
    prev, t = ev0, []
    for e in ev_steps:
        t.append(prev.elapsed_time(e))
        prev = e
    if not t:
        return None
    t.sort()
    pick = lambda q: t[min(len(t) - 1, int(round(q * (len(t) - 1))))]  # noqa: E731
    return [round(pick(0.1), 4), round(pick(0.5), 4), round(pick(0.9), 4)]


def moe_offsets(T, E, seed=0):
    """Seeded imbalanced routing: expert loads ~ exp(N(0, 0.5^2)) normalised, rounded to multiples of
    128 rows with the total kept at T (MoE frameworks pad each expert's token group)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    p = np.exp(rng.normal(0.0, 0.5, E))
    p /= p.sum()
    units = T // 128
    c = np.floor(p * units).astype(np.int64)
    for i in np.argsort(-(p * units - c))[:units - int(c.sum())]:
        c[i] += 1
    return np.concatenate([[0], np.cumsum(c * 128)]).astype(np.int32)


def run_layer(a):
    """All linears of one transformer layer (BASELINE.json configs[2]), each a Float8Linear fwd+bwd
    through the C-ABI, back to back on one stream (replicas at N>1)."""
    import ctypes
    result = None
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2507_16099_b200 as fp8t  # noqa: F401  (loads libfp8train.so; raises if missing)
    from paper_2507_16099_b200 import _lib as L, ops
    cfg = CONFIGS[a.config]
    M = cfg["M"]
    units = []
    for i, (name, N, K) in enumerate(cfg["linears"]):
        x, w, dy = make_inputs(dict(cfg, N=N, K=K), M, N, K, rank, 1, dev, seed=i)
        units.append(dict(name=name, N=N, K=K, x=x, w=w, dy=dy,
                          y=torch.empty((M, N), dtype=torch.bfloat16, device=dev),
                          dx=torch.empty((M, K), dtype=torch.bfloat16, device=dev),
                          dw=torch.empty((N, K), dtype=torch.bfloat16, device=dev)))
    # groups of linears reading one X (the first member's); --layer-separate: every linear on its own
    byname = {u["name"]: u for u in units}
    groups = [] if a.layer_separate else [[byname[n] for n in g] for g in cfg.get("shared", [])]
    grouped = {id(u) for g in groups for u in g}
    groups += [[u] for u in units if id(u) not in grouped]
    groups.sort(key=lambda g: units.index(g[0]))
    for g in groups:
        for u in g[1:]:
            u["x"] = g[0]["x"]
        if len(g) == 1:
            u = g[0]
            u["plan"] = ops.LinearPlan(M, u["N"], u["K"], recipe=cfg["recipe"], out_dtype=torch.bfloat16, device=dev)
            u["saved"] = u["plan"].new_saved(dev)
        else:
            sp = ops.SharedInputPlan(M, [u["N"] for u in g], g[0]["K"], recipe=cfg["recipe"],
                                     out_dtype=torch.bfloat16, device=dev)
            sv = sp.new_saved(dev)
            for u, t in zip(g, sv):
                u["saved"] = t
            g[0]["group_plan"] = sp

    def run_group(g, xs, ws_, dys):
        if len(g) == 1:
            u = g[0]
            u["plan"].forward(xs[0], ws_[0], u["saved"], y=u["y"])
            u["plan"].backward(dys[0], u["saved"], dx=u["dx"], dw=u["dw"], x=xs[0])
        else:
            sp, sv = g[0]["group_plan"], [u["saved"] for u in g]
            sp.forward(xs[0], ws_, sv, ys=[u["y"] for u in g])
            sp.backward(dys, sv, dxs=[u["dx"] for u in g], dws=[u["dw"] for u in g], x=xs[0])

    def step():
        for g in groups:
            run_group(g, [g[0]["x"]], [u["w"] for u in g], [u["dy"] for u in g])

    for _ in range(max(a.warmup, 3)):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_steps = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]   # per-step boundaries
    L.lib.fp8_profile_collect(None, None, 0)
    L.lib.fp8_profile_enable(1)
    n0 = ops.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i_ in range(a.steps):
            step()
            ev_steps[i_].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = ops.launch_count() - n0
    L.lib.fp8_profile_enable(0)
    cap = launches + 16
    kinds, durs = (ctypes.c_int * cap)(), (ctypes.c_float * cap)()
    nrec = L.lib.fp8_profile_collect(kinds, durs, cap)
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / a.steps
    step_pct = step_percentiles(ev0, ev_steps)
    flops_step = sum(6.0 * M * u["N"] * u["K"] for u in units)
    value = flops_step * a.steps * world / (ms / 1e3) / 1e12
    by = {}
    for i in range(max(nrec, 0)):
        by.setdefault(kinds[i], []).append(durs[i])
    gemm_ms = by.get(4, [float("nan")])
    gemm_tflops = flops_step / (sum(gemm_ms) / a.steps / 1e3) / 1e12
    peaks = _peaks()
    fp8_peak = 2.0 * peaks["bf16"]
    # rowwise: 6 B / element (read for the amax, read for the cast, two 1-byte copies); X once per group
    cast_bytes = sum((u["N"] * u["K"] + M * u["N"]) * 6 for u in units) + sum(M * g[0]["K"] * 6 for g in groups)
    cast_ms = sum(sum(by.get(k, [])) for k in (0, 1)) / a.steps
    e2e = None
    if a.e2e_steps > 0:
        host = {id(u): dict(x=u["x"].cpu().pin_memory() if u is g[0] else None, w=u["w"].cpu().pin_memory(),
                            dy=u["dy"].cpu().pin_memory(), y=torch.empty_like(u["y"], device="cpu").pin_memory(),
                            dx=torch.empty_like(u["dx"], device="cpu").pin_memory(),
                            dw=torch.empty_like(u["dw"], device="cpu").pin_memory()) for g in groups for u in g}
        dbuf = {id(u): dict(x=torch.empty_like(u["x"]) if u is g[0] else None, w=torch.empty_like(u["w"]),
                            dy=torch.empty_like(u["dy"])) for g in groups for u in g}

        def e2e_step():
            for g in groups:
                for u in g:
                    for k in ("x", "w", "dy"):
                        if host[id(u)][k] is not None:
                            dbuf[id(u)][k].copy_(host[id(u)][k], non_blocking=True)
                run_group(g, [dbuf[id(g[0])]["x"]], [dbuf[id(u)]["w"] for u in g], [dbuf[id(u)]["dy"] for u in g])
                for u in g:
                    for k in ("y", "dx", "dw"):
                        host[id(u)][k].copy_(u[k], non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        e2e = {"value": flops_step * a.e2e_steps * world / (ems / 1e3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": sum((u["w"].numel() + u["dy"].numel()) * 2 for u in units)
                                     + sum(g[0]["x"].numel() * 2 for g in groups),
               "d2h_bytes_per_step": sum((u["y"].numel() + u["dx"].numel() + u["dw"].numel()) * 2 for u in units),
               "ms_per_step": ems / a.e2e_steps,
               "path": "per linear group: pinned host -> device X (once per group), W, dY + fp8_linear_fwd/bwd or "
                       "fp8_linear_fwd/bwd_shared (C-ABI) + device -> host Y, dX, dW, every step, on the compute stream"}
    bf16 = None
    if not a.no_bf16:
        def bstep():
            for u in units:
                torch.matmul(u["x"], u["w"].t(), out=u["y"])
                torch.matmul(u["dy"], u["w"], out=u["dx"])
                torch.matmul(u["dy"].t(), u["x"], out=u["dw"])
        for _ in range(3):
            bstep()
        torch.cuda.synchronize()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(a.steps):
            bstep()
        b1.record(stream)
        torch.cuda.synchronize()
        bms = b0.elapsed_time(b1) / a.steps
        bf16 = {"ms_per_step": bms, "tflops": flops_step / (bms / 1e3) / 1e12, "speedup_fp8_vs_bf16": bms / ms_step,
                "impl": "torch.matmul (cuBLAS) bf16, same 3 GEMMs per linear"}
    cpu = cpu_baseline(dict(cfg, N=14336)) if (rank == 0 and world == 1 and not a.no_cpu_baseline) else None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
            "warmup": max(a.warmup, 3), "ms_per_step": ms_step, "step_ms_p10_p50_p90": step_pct, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp8 (e4m3 x e5m2 codes, fp32 accumulate, bf16 out)",
            "data": "synthetic (seeded synth generator run on the device, config value recipe; = the parity tests' inputs at rank 0)",
            "config": {"workload": cfg["workload"], "M_per_gpu": M, "linears": cfg["linears"], "recipe": cfg["recipe"],
                       "shared_input_groups": [[u["name"] for u in g] for g in groups if len(g) > 1],
                       "parallelism": "single GPU" if world == 1 else f"{world} independent replicas",
                       "l2": "inputs larger than L2 (126 MB) for the MLP linears; no flush"},
            "roofline": {"bound": "tensor", "kernel": "fp8_gemm_kernel (tcgen05 kind::f8f6f4)",
                         "achieved": gemm_tflops, "peak": fp8_peak, "unit": "TFLOP/s", "frac": gemm_tflops / fp8_peak,
                         "traffic": None,
                         "peak_source": f"{peaks['src']}: bf16_tflops (burst) x 2 (dense FP8/BF16 ratio)",
                         "algorithmic": "2*M*N*K flop per GEMM problem, summed over the 7 linears x 3 GEMMs",
                         "launches_per_step": len(gemm_ms) / a.steps, "share_of_step": sum(gemm_ms) / a.steps / ms_step},
            "cast": {"gbps": cast_bytes / (cast_ms / 1e3) / 1e9 if cast_ms > 0 else None, "peak_gbps": peaks["hbm"],
                     "frac": cast_bytes / (cast_ms / 1e3) / 1e9 / peaks["hbm"] if cast_ms > 0 else None,
                     "ms_per_step": cast_ms, "algorithmic_bytes_per_step": cast_bytes},
            "kernels_ms_per_step": {name: round(sum(by.get(k, [])) / a.steps, 4)
                                    for k, name in ((0, "amax"), (1, "cast"), (4, "gemm_fp8"))},
            "bf16": bf16, "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
        }
        result = line
    if dist.is_initialized():
        dist.destroy_process_group()
    return result


def run_moe(a):
    """MoE scaled grouped GEMM fwd+bwd (fp8_grouped_linear_fwd/bwd) on one GPU (replicas at N>1:
    the grouped GEMM has no exchange step of its own; expert parallelism's all-to-all is out of scope)."""
    import ctypes
    result = None
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2507_16099_b200 as fp8t  # noqa: F401  (loads libfp8train.so; raises if missing)
    from paper_2507_16099_b200 import _lib as L, ops
    cfg = CONFIGS[a.config]
    T, E, N, K = cfg["T"], cfg["E"], cfg["N"], cfg["K"]
    offs_h = moe_offsets(T, E)
    offs = torch.from_numpy(offs_h).to(dev)
    # routed tokens and their output grads, E stacked expert weights [E*N, K]; c3 value recipe
    # (weights N(0, 0.02^2) x 2^U(-4,4) per row), synth.device like every bench input
    from synth import device as sd
    x = sd.tensor("c3", "x", (T, K), 1000 * rank, dev)
    dy = sd.tensor("c3", "dy", (T, N), 1000 * rank, dev)
    w = sd.tensor("c3", "w", (E * N, K), 0, dev)
    plan = ops.GroupedPlan(T, E, N, K, recipe=cfg["recipe"], out_dtype=torch.bfloat16, device=dev)
    saved = plan.new_saved(dev)
    y = torch.empty((T, N), dtype=torch.bfloat16, device=dev)
    dx = torch.empty((T, K), dtype=torch.bfloat16, device=dev)
    dw = torch.empty((E * N, K), dtype=torch.bfloat16, device=dev)

    def step(xx=x, ww=w, gg=dy, yy=y, dxx=dx, dww=dw):
        plan.forward(xx, ww, offs, saved, y=yy)
        plan.backward(gg, offs, saved, dx=dxx, dw=dww)

    for _ in range(max(a.warmup, 3)):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_steps = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]   # per-step boundaries
    L.lib.fp8_profile_collect(None, None, 0)
    L.lib.fp8_profile_enable(1)
    n0 = ops.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i_ in range(a.steps):
            step()
            ev_steps[i_].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = ops.launch_count() - n0
    L.lib.fp8_profile_enable(0)
    cap = launches + 16
    kinds, durs = (ctypes.c_int * cap)(), (ctypes.c_float * cap)()
    nrec = L.lib.fp8_profile_collect(kinds, durs, cap)
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / a.steps
    step_pct = step_percentiles(ev0, ev_steps)
    flops_step = 6.0 * T * N * K
    value = flops_step * a.steps * world / (ms / 1e3) / 1e12
    by = {}
    for i in range(max(nrec, 0)):
        by.setdefault(kinds[i], []).append(durs[i])
    gemm_ms = by.get(4, [float("nan")])
    gemm_tflops = flops_step / (sum(gemm_ms) / a.steps / 1e3) / 1e12
    peaks = _peaks()
    fp8_peak = 2.0 * peaks["bf16"]
    cast_bytes = (T * K + E * N * K + T * N) * 6
    cast_ms = sum(sum(by.get(k, [])) for k in (0, 1)) / a.steps
    # end to end through the public API: pinned host inputs (X, W, dY, offsets) in, Y, dX, dW out, every step
    e2e = None
    if a.e2e_steps > 0:
        hx, hw, hg = x.cpu().pin_memory(), w.cpu().pin_memory(), dy.cpu().pin_memory()
        ho = torch.from_numpy(offs_h).pin_memory()
        hy, hdx, hdw = (torch.empty_like(t_, device="cpu").pin_memory() for t_ in (y, dx, dw))
        dxi, dwi, dgi, doi = torch.empty_like(x), torch.empty_like(w), torch.empty_like(dy), torch.empty_like(offs)

        def e2e_step():
            for d_, h_ in ((dxi, hx), (dwi, hw), (dgi, hg), (doi, ho)):
                d_.copy_(h_, non_blocking=True)
            plan.forward(dxi, dwi, doi, saved, y=y)
            plan.backward(dgi, doi, saved, dx=dx, dw=dw)
            for h_, d_ in ((hy, y), (hdx, dx), (hdw, dw)):
                h_.copy_(d_, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1)
        e2e = {"value": flops_step * a.e2e_steps * world / (ems / 1e3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": (x.numel() + w.numel() + dy.numel()) * 2 + offs.numel() * 4,
               "d2h_bytes_per_step": (y.numel() + dx.numel() + dw.numel()) * 2, "ms_per_step": ems / a.e2e_steps,
               "path": "pinned host -> device X, W, dY, offsets + fp8_grouped_linear_fwd/bwd (C-ABI) + device -> "
                       "host Y, dX, dW, every step, on the compute stream"}
    bf16 = None
    if not a.no_bf16:
        def bstep():
            for g in range(E):
                r0, r1 = int(offs_h[g]), int(offs_h[g + 1])
                if r1 == r0:
                    continue
                wg = w[g * N:(g + 1) * N]
                torch.matmul(x[r0:r1], wg.t(), out=y[r0:r1])
                torch.matmul(dy[r0:r1], wg, out=dx[r0:r1])
                torch.matmul(dy[r0:r1].t(), x[r0:r1], out=dw[g * N:(g + 1) * N])
        for _ in range(3):
            bstep()
        torch.cuda.synchronize()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(a.steps):
            bstep()
        b1.record(stream)
        torch.cuda.synchronize()
        bms = b0.elapsed_time(b1) / a.steps
        bf16 = {"ms_per_step": bms, "tflops": flops_step / (bms / 1e3) / 1e12, "speedup_fp8_vs_bf16": bms / ms_step,
                "impl": "torch.matmul (cuBLAS) bf16, 3 GEMMs per expert"}
    cpu = cpu_baseline(cfg) if (rank == 0 and world == 1 and not a.no_cpu_baseline) else None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
            "warmup": max(a.warmup, 3), "ms_per_step": ms_step, "step_ms_p10_p50_p90": step_pct, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp8 (e4m3 x e5m2 codes, fp32 accumulate, bf16 out)",
            "data": "synthetic (seeded synth generator run on the device, c3 value recipe; seeded routing)",
            "config": {"workload": cfg["workload"], "T": T, "E": E, "N": N, "K": K, "recipe": cfg["recipe"],
                       "group_rows": [int(offs_h[i + 1] - offs_h[i]) for i in range(E)],
                       "parallelism": "single GPU" if world == 1 else f"{world} independent replicas",
                       "l2": "inputs larger than L2 (126 MB); no flush"},
            "roofline": {"bound": "tensor", "kernel": "fp8_gemm_kernel (tcgen05 kind::f8f6f4, grouped)",
                         "achieved": gemm_tflops, "peak": fp8_peak, "unit": "TFLOP/s", "frac": gemm_tflops / fp8_peak,
                         "traffic": None,
                         "peak_source": f"{peaks['src']}: bf16_tflops (burst) x 2 (dense FP8/BF16 ratio)",
                         "algorithmic": "2*T*N*K flop per grouped GEMM (sum over experts of 2*M_g*N*K); fwd launch "
                                        "1 grouped problem, bwd launch 2 (dX M-grouped, dW K-grouped)",
                         "launches_per_step": len(gemm_ms) / a.steps, "share_of_step": sum(gemm_ms) / a.steps / ms_step},
            "cast": {"gbps": cast_bytes / (cast_ms / 1e3) / 1e9 if cast_ms > 0 else None, "peak_gbps": peaks["hbm"],
                     "frac": cast_bytes / (cast_ms / 1e3) / 1e9 / peaks["hbm"] if cast_ms > 0 else None,
                     "ms_per_step": cast_ms, "algorithmic_bytes_per_step": cast_bytes},
            "kernels_ms_per_step": {name: round(sum(by.get(k, [])) / a.steps, 4)
                                    for k, name in ((0, "amax"), (1, "cast"), (4, "gemm_fp8_grouped"))},
            "bf16": bf16, "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": cpu,
        }
        result = line
    if dist.is_initialized():
        dist.destroy_process_group()
    return result


def host_info():
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count()}


PAPER_CONTEXT = ("paper (context, not a target): FP8 tensorwise training up to 1.5x the BF16 throughput on Llama "
                 "3.1 405B, 512 H100s, FSDP2 + torch.compile (PAPER.md:129-130, 292-294); 1.25x tensorwise + FP8 "
                 "all-gather / 1.10x rowwise on Llama3-8B, 8 H100s (PAPER.md:446-448).  End-to-end model "
                 "throughputs on other hardware; this line times the linear's hot path alone.")


def run_config(a, name, sub=False):
    import copy
    aa = copy.copy(a)
    aa.config = name
    if sub:
        aa.e2e_steps, aa.no_cpu_baseline, aa.digest = 0, True, False
        if name == "c5" and int(os.environ.get("WORLD_SIZE", "1")) == 1:
            aa.fsdp = True      # the same-config N=1 point of the FSDP runs
    kind = CONFIGS[name].get("kind")
    fn = run_moe if kind == "moe" else run_layer if kind == "layer" else run_ours
    line = fn(aa)
    import torch
    torch.cuda.empty_cache()
    return line


def main():
    global _JSON_FD
    a = parse()
    sys.stdout.flush()
    _JSON_FD = os.dup(1)    # keep the real stdout for the JSON line; everything else -> stderr
    os.dup2(2, 1)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    default_headline = a.config is None
    if default_headline:
        a.config = "c4" if world == 1 else "c5"
    if a.impl == "reference":
        run_reference(a)
        return
    subs = [c for c in (a.sub.split(",") if a.sub else (["c2", "c3", "c5", "c3w1hp", "moe"]
                                                          if default_headline and world == 1 else [])) if c]
    if a.knob:
        import paper_2507_16099_b200  # noqa: F401
        from paper_2507_16099_b200 import ops
        for kv in a.knob:
            k, v = kv.split("=")
            ops.set_knob(k, int(v))
    line = run_config(a, a.config)
    sub = {}
    for c in subs:
        sl = run_config(a, c, sub=True)
        if sl is not None:
            key = c + ("_fsdp1" if c == "c5" and world == 1 else "")
            sub[key] = {k: v for k, v in sl.items() if k not in ("metric", "unit", "e2e", "cpu_baseline", "steps",
                                                                  "warmup", "higher_is_better", "vs_baseline",
                                                                  "n_gpus", "scaling")}
    if line is not None:
        line["host"] = host_info()
        if a.knob:
            line["knobs"] = a.knob
        line["context"] = PAPER_CONTEXT
        if sub:
            line["sub"] = sub
        emit(line)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""EP-HDC client-side encrypted inference on B200: queries/s (BASELINE.json metric).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

A step = the whole hot path over one batch of nq synthetic queries with inputs and
the encrypted model resident in HBM: ephdc_encode_queries (HDC encoding + Q-bit
quantisation) + ephdc_infer_batch (per ciphertext batch: slot pack + INTT_t, lift +
NTT_q + ct x pt MAC over all D dims, finalize) -> nb scores ciphertexts.
Default workload: c4 (BASELINE.json configs[3], the largest single-GPU config; the
metric names no config).  Multi-GPU: one process per GPU, each rank a full replica
on its own nq queries (batches are independent: weak scaling, no data-path
collective); value = all ranks' queries / max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import ephdc_inputs as inp  # noqa: E402

METRIC = "encrypted-HDC queries/sec on 1 B200; NTT+MAC fraction of HBM/int roofline"
# Roofline of the dominant kernel.  FP64 path: the pipe is the
# FP64 unit, 64 DFMA-class lanes/clk/SM (profiles/r01/int_peak.jsonl measures 63.1);
# the algorithmic work of a launch is its butterflies and MAC products at the minimum
# instruction count of the exact double arithmetic (modf64.cuh): 8 per butterfly
# (one exact product = 6, plus the add and the subtract), 7 per MAC term (product +
# accumulate).  Integer path: 64 IMAD lanes/clk/SM, 10 multiply instructions per u64
# Shoup/Montgomery product.
FP64_PER_SM_CLK = 64
F64_OPS_PER_BFLY = 8
F64_OPS_PER_MAC = 7
IMAD_PER_SM_CLK = 64
IMAD_PER_MULMOD = 10


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=["c1q3", "c2", "c3", "c4"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="--impl reference: seconds of timed oracle steps (each step = one full batch)")
    ap.add_argument("--threads", type=int, default=0, help="oracle threads (OMP_NUM_THREADS; 0 = all host cores)")
    ap.add_argument("--plan", default="", help="A/B only: workspace launch-plan overrides, e.g. 'flags=2,bg=8'")
    return ap.parse_args()


def fp64_ceiling():
    """The FP64 butterfly mix's sustained rate measured on a B200 (tools/int_peak.cu
    `sustained`, profiles/r02/r19/fp64_ceiling.json) and this kernel's fraction of it is
    reported next to the nominal peak; None if the record is absent."""
    try:
        rec = json.loads(open(os.path.join(ROOT, "profiles", "r02", "r19", "fp64_ceiling.json")).readline())
        return {"value": rec["Gops"], "unit": "GFP64op/s", "source": "profiles/r02/r19/fp64_ceiling.json"}
    except Exception:
        return None


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- oracle
class OracleSample:
    """The oracle (plain CPU C + numpy, OpenMP over dims; TEST INFRASTRUCTURE, executed only
    by this leg) on the unit of the workload: encode + client evaluation of ONE full
    ciphertext batch (B queries) over ALL D_live dims against the stored model -- the
    same arithmetic the GPU does per batch, nothing extrapolated.  The model is
    encrypted once (untimed, like the resident GPU model)."""

    def __init__(self, cfg, data):
        from oracle import hdc, pipeline as opipe
        Xtr, ytr, Xq, P = data
        self.cfg, self.hdc, self.P = cfg, hdc, P
        self.om = opipe.build_model(cfg, P, Xtr, ytr)
        self.bfv = self.om.bfv
        self.B = self.bfv.B
        self.Xb = np.ascontiguousarray(Xq[: self.B])
        self.model = self.bfv.encrypt_dims(self.om.class_hv, self.om.enc_seed, 0, cfg.D_live)

    def step(self) -> float:
        """One batch; returns its wall time in seconds."""
        t0 = time.perf_counter()
        H = self.hdc.quantise_queries(self.hdc.encode_raw(self.P, self.Xb, self.cfg.D_live), self.om.qshift,
                                      self.om.Qbits)
        self.bfv.infer_batch(H, H.shape[1], 0, model=self.model)
        return time.perf_counter() - t0

    def describe(self, dt: float, threads: int) -> str:
        return (f"{self.cfg.name}: encode + evaluation of one full batch ({self.B} queries, all "
                f"{self.cfg.D_live} dims x {self.bfv.L} primes, model resident) in {dt:.1f} s on {threads} "
                f"thread(s); batches are identical units (one scores ciphertext each), no extrapolation")


def oracle_threads() -> int:
    return int(os.environ.get("OMP_NUM_THREADS") or os.cpu_count() or 1)


def cpu_baseline(cfg, data) -> dict:
    o = OracleSample(cfg, data)
    dt = o.step()
    return {"value": o.B / dt, "unit": "queries/s", "cores": oracle_threads(), "kind": "oracle",
            "sample": o.describe(dt, oracle_threads())}


# ----------------------------------------------------------------------------- main
def main():
    a = parse()
    if a.threads > 0:   # before the oracle's OpenMP runtime loads
        os.environ["OMP_NUM_THREADS"] = str(a.threads)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = inp.CONFIGS[a.config]

    if a.impl == "reference":
        # the oracle as it stands on the host cores (rank 0 only); a step = one full batch.
        # Steps are capped so the run ends within --ref-budget seconds; the line reports the
        # steps it actually timed.
        if rank != 0:
            return 0
        Xtr, ytr, Xq, _ = inp.gen_features(cfg)
        P = inp.gen_projection(cfg)
        o = OracleSample(cfg, (Xtr, ytr, Xq, P))
        t_first = o.step()                                        # warm-up step 1
        budget = max(a.ref_budget, 2 * t_first)
        warm = 1
        while warm < a.warmup and (warm + 1) * t_first < 0.25 * budget:
            o.step()
            warm += 1
        steps = max(1, min(a.steps, int((budget - warm * t_first) // max(t_first, 1e-3))))
        times = [o.step() for _ in range(steps)]
        ms = 1e3 * sum(times) / steps
        v = o.B / (ms / 1e3)
        threads = oracle_threads()
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "queries/s", "n_gpus": a.gpus,
                "steps": steps, "warmup": warm, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "u64 (exact modular integers, CPU)",
                "data": "synthetic",
                "config": {"workload": cfg.name, "queries_per_step": o.B, "N": cfg.N, "L": cfg.L, "D": cfg.D_live,
                           "k": cfg.k, "requested": {"steps": a.steps, "warmup": a.warmup},
                           "threads": threads},
                "cpu_baseline": {"value": v, "unit": "queries/s", "cores": threads, "kind": "oracle",
                                 "sample": o.describe(ms / 1e3, threads)},
                "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0

    import torch
    import torch.distributed as dist
    import paper_2511_00737_b200 as eph
    from paper_2511_00737_b200 import pipeline as ppipe
    from paper_2511_00737_b200 import dist as pdist

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    # every rank: the same model (replicated), its own query stream (weak scaling)
    Xtr, ytr, Xq, _ = inp.gen_features(cfg, stream=rank)
    P = inp.gen_projection(cfg)
    ps = ppipe.build(cfg, P, Xtr, ytr, device=local)
    ctx, model = ps.ctx, ps.model
    nq = cfg.nq
    nb = ctx.n_batches(nq)
    X_dev = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).to(dev)
    plan = {k: int(v, 0) for k, v in (kv.split("=") for kv in a.plan.split(",") if kv)} or None
    ws = eph.Workspace(ctx, nq, plan=plan)
    H = torch.empty((cfg.D_live, nq), dtype=torch.int8, device=dev)
    out = torch.empty(ctx.ct_shape(nq), dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        eph.encode_queries(ctx, X_dev, ps.P_dev, H)
        eph.infer_batch(ctx, model, ws, H, nq, out)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    ws.set_timing(True)
    ws.timing()                                  # reset
    n0 = eph.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    enc_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    e0.record(stream)
    for i in range(a.steps):
        enc_ev[i][0].record(stream)
        eph.encode_queries(ctx, X_dev, ps.P_dev, H)
        enc_ev[i][1].record(stream)
        eph.infer_batch(ctx, model, ws, H, nq, out)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    launches = eph.launch_count() - n0
    enc_ms = sum(x.elapsed_time(y) for x, y in enc_ev)
    kt = ws.timing()
    ws.set_timing(False)
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / a.steps
    ms_max = pdist.max_over_ranks(ms)
    value = world * nq / (ms_max / 1e3)

    # roofline of the dominant kernel: the fused lift + NTT_q + MAC (all batches per launch)
    mac_ms, mac_n = kt["ntt_mac"]
    mac_s = mac_ms / a.steps / 1e3                              # per step
    N, L, D = ctx.N, ctx.L, cfg.D_live
    bfly = nb * D * L * (N // 2) * cfg.log2N                    # butterflies per step
    macs = nb * D * L * 2 * N                                   # MAC products per step
    smax = measured_peaks().get("sm_max_mhz") or 1965.0
    if ctx.arith == "f64":
        achieved = (F64_OPS_PER_BFLY * bfly + F64_OPS_PER_MAC * macs) / mac_s / 1e9
        peak = 148 * FP64_PER_SM_CLK * smax * 1e6 / 1e9
        unit, kname = "GFP64op/s", "k_ntt_mac_f64"
        src = ("derived: 148 SMs x 64 FP64 lanes/clk x sm_max_mhz; work = 8 ops/butterfly + 7 ops/MAC "
               "term of the exact double arithmetic (DESIGN.md)")
    else:
        achieved = (bfly + macs) / mac_s / 1e9
        peak = 148 * IMAD_PER_SM_CLK * smax * 1e6 / IMAD_PER_MULMOD / 1e9
        unit, kname = "Gmulmod/s", "k_ntt_mac"
        src = "derived: 148 SMs x 64 IMAD/clk x sm_max_mhz / 10 IMAD per u64 mulmod (DESIGN.md)"
    kt["encode"] = (enc_ms, a.steps)
    total_ms = sum(v[0] for v in kt.values())
    traffic = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(cfg.name)
        if tr and tr.get("kernel") == kname:
            traffic = tr["bytes_per_step"]
    except Exception:
        pass
    roofline = {"bound": "alu", "kernel": kname, "achieved": round(achieved, 1), "peak": round(peak, 1),
                "unit": unit, "frac": round(achieved / peak, 4), "traffic": traffic,
                "algorithmic": {"butterflies_per_step": bfly, "mac_terms_per_step": macs,
                                "model_bytes": D * L * 2 * N * 8, "launches_per_step": mac_n / a.steps},
                "mulmod_rate_G_per_s": round((bfly + macs) / mac_s / 1e9, 1),
                "peak_source": src,
                "measured_ceiling": fp64_ceiling() if ctx.arith == "f64" else None,
                "frac_of_measured_ceiling": (round(achieved / fp64_ceiling()["value"], 4)
                                             if ctx.arith == "f64" and fp64_ceiling() else None),
                "share_of_step": round(mac_ms / max(total_ms, 1e-9), 4),
                "kernel_ms": {k: round(v[0] / a.steps, 3) for k, v in kt.items()}}

    # pipe / DRAM figures of the step's kernels from the committed ncu capture of this
    # config (profiles/ncu_metrics.json, written by tools/ncu_metrics.py from an
    # `ncu --set full` run of this bench command; ncu figures, not this run's)
    ncu = None
    try:
        nm = json.load(open(os.path.join(ROOT, "profiles", "ncu_metrics.json"))).get(cfg.name)
        if nm:
            ncu = dict(nm)
            ncu["hbm_peak_gbs"] = measured_peaks().get("hbm_gbs")
    except Exception:
        pass

    # e2e: the same step through the host-buffer C-ABI call (H2D + compute + D2H per step)
    e2e = None
    if not a.no_e2e:
        # the call a client makes: features from host memory in, the scores message it
        # sends to the server (bit-packed ciphertexts, ephdc_classify_host_packed) out
        Xh = torch.from_numpy(np.ascontiguousarray(Xq).view(np.int8)).pin_memory()
        oh = torch.empty(eph.scores_message_bytes(ctx, nb), dtype=torch.uint8, pin_memory=True)
        for _ in range(max(1, a.warmup)):
            eph.classify_host_packed(ctx, model, ws, Xh, ps.P_dev, oh)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(a.steps):
            eph.classify_host_packed(ctx, model, ws, Xh, ps.P_dev, oh)
        f1.record(stream)
        torch.cuda.synchronize(dev)
        ems = pdist.max_over_ranks(f0.elapsed_time(f1) / a.steps)
        e2e = {"value": world * nq / (ems / 1e3), "unit": "queries/s",
               "h2d_bytes_per_step": int(Xh.numel()), "d2h_bytes_per_step": int(oh.numel()),
               "call": "ephdc_classify_host_packed (features in, bit-packed scores message out)"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = cpu_baseline(cfg, (Xtr, ytr, Xq, P))

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": "queries/s", "n_gpus": world,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_max, 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": ("u64 residues, exact modular arithmetic on the FP64 pipe" if ctx.arith == "f64"
                          else "u64 residues, integer pipe"), "data": "synthetic",
                "config": {"workload": cfg.name, "nq_per_gpu": nq, "batches": nb, "N": N, "L": L, "D": D,
                           "k": cfg.k, "F": cfg.F, "t": ctx.t, "log2q": sum(int(q).bit_length() for q in ctx.q),
                           "parallelism": f"replica x{world} (independent query batches)",
                           "arith": ctx.arith,
                           "l2": "inputs larger than L2 (encrypted model %.1f GB in HBM)" % (D * L * 2 * N * 8 / 1e9)},
                "gpu_launches": int(launches), "clocks": clk, "roofline": roofline, "ncu": ncu, "cpu_baseline": cpu,
                "e2e": e2e}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

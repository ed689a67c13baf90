#!/usr/bin/env python
"""profiles/ncu_metrics.json entry for one config from an `ncu --set full` capture of the
bench command (kernels k_ntt_mac_f64 / k_ntt_mac, k_pack_intt32 / k_pack_intt_q, k_encode_tc):
  fused pass: DRAM bytes, duration, GB/s, FP64-pipe and integer-pipe utilisation;
  pack + INTT_t: integer-pipe (alu + fma) utilisation, duration;
  encoder: tensor-pipe utilisation, duration.
usage: ncu_metrics.py <rep> <config> [out.json]"""
import csv
import io
import json
import subprocess
import sys


def f(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, units = r[0], r[1]
    res = []
    for v in r[2:]:
        d = dict(zip(h, v))
        u = dict(zip(h, units)).get("gpu__time_duration.sum", "")
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(u.strip(), 1.0)
        d["_ms"] = f(d.get("gpu__time_duration.sum")) * scale
        b = dict(zip(h, units)).get("dram__bytes_read.sum", "")
        bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(b.strip(), 1)
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            d[key] = f(d.get(key)) * bscale
        res.append(d)
    return res


def main():
    rep, cfg = sys.argv[1], sys.argv[2]
    path = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_metrics.json"
    out = {"source": rep.split("/")[-1]}
    for k in rows(rep):
        name = k["Kernel Name"]
        ms = k["_ms"]
        if "k_ntt_mac" in name and "fused" not in out:
            rd, wr = f(k["dram__bytes_read.sum"]), f(k["dram__bytes_write.sum"])
            out["fused"] = {"kernel": name.split("(")[0], "duration_ms": ms, "dram_read_bytes": rd, "dram_write_bytes": wr,
                            "dram_GBps": (rd + wr) / (ms * 1e-3) / 1e9,
                            "fp64_pipe_pct": f(k["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]),
                            "alu_pipe_pct": f(k["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"]),
                            "dram_throughput_pct": f(k["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"])}
        elif "k_pack_intt" in name and "pack" not in out:
            out["pack"] = {"kernel": name.split("(")[0], "duration_ms": ms,
                           "alu_pipe_pct": f(k["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"]),
                           "fma_pipe_pct": f(k["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"]),
                           "fmaheavy_cycles_pct": f(k["sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"]),
                           "issue_active_pct": f(k["smsp__issue_active.avg.pct_of_peak_sustained_active"])}
        elif "k_encode_tc" in name and "encode" not in out:
            # tcgen05 MMAs: the realtime tensor-pipe counter (the plain sm__pipe_tensor_cycles_active
            # stays 0 for UTC*MMA on this ncu)
            tp = f(k.get("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"))
            out["encode"] = {"kernel": name.split("(")[0], "duration_ms": ms, "tensor_pipe_pct": tp}
    try:
        allm = json.load(open(path))
    except Exception:
        allm = {}
    allm[cfg] = out
    json.dump(allm, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""Summarise the ncu evidence of one round into profiles/ (run here, on the reports gpurun
brought back).

  python scripts/ncu_summary.py ROUND [gpurun_out]

Reads   <dir>/prof_gemm.ncu-rep, <dir>/prof_mem.ncu-rep  (ncu --set full, scripts/ncu_round.sh)
        <dir>/launches.csv                               (ncu --metrics gpu__time_duration.sum)
Writes  profiles/<ROUND>_ncu_full_summary.json  per-launch duration, DRAM bytes, tensor pipe %
        profiles/<ROUND>_launches.txt           per-kernel totals and shares of the launch list
        profiles/ncu_traffic.json               DRAM R+W bytes per launch, keyed by bench name
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# kernel-name fragment -> bench name, in the order the bench step launches them
GEMM_ORDER = ["ffn_gemm1", "ffn_gemm2", "wgrad_w2", "dgrad_dA", "wgrad_w1", "dgrad_dX"]
MEM_NAMES = [("gate_fwd", "gate_topk"), ("route_hist", "route_hist"), ("route_scan", "route_scan"),
             ("dispatch", "dispatch"), ("combine_fwd", "combine_fwd"),
             ("combine_bwd", "combine_bwd"), ("gate_dx", "gate_dx"), ("gate_dw", "gate_dw"),
             ("reduce_partials", "gate_dw_reduce"), ("colsum", "bias_grad"),
             ("bias_part", "bias_grad")]

COLS = {
    "dur_ns": "gpu__time_duration.sum",
    "rd": "dram__bytes_read.sum",
    "wr": "dram__bytes_write.sum",
    "clk": "sm__cycles_elapsed.avg.per_second",
    "regs": "launch__registers_per_thread",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "bf16_ops_pct": "sm__ops_path_tensor_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed",
    "dram_pct": "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6,
              "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "hz": 1, "Khz": 1e3, "Mhz": 1e6,
              "Ghz": 1e9, "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")], "grid": r[hdr.index("Grid Size")],
             "block": r[hdr.index("Block Size")]}
        for k, c in COLS.items():
            if c not in hdr:
                d[k] = None
                continue
            i = hdr.index(c)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                d[k] = None
                continue
            d[k] = v * UNIT_SCALE.get(units[i], 1)
        res.append(d)
    return res


def bench_name(kernel, gemm_idx):
    if "tc_gemm" in kernel:
        return GEMM_ORDER[gemm_idx % len(GEMM_ORDER)]
    for frag, name in MEM_NAMES:
        if frag in kernel:
            return name
    return kernel


def main():
    rnd = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    summary, traffic = [], OrderedDict()
    for rep in ("prof_gemm.ncu-rep", "prof_mem.ncu-rep"):
        path = os.path.join(src, rep)
        if not os.path.exists(path):
            continue
        gi = 0
        for d in raw_rows(path):
            name = bench_name(d["kernel"], gi)
            if "tc_gemm" in d["kernel"]:
                gi += 1
            rd, wr, dur = d["rd"] or 0, d["wr"] or 0, d["dur_ns"] or 0
            e = OrderedDict(bench=name, kernel=d["kernel"][:80], grid=d["grid"], block=d["block"],
                            dur_us=round(dur / 1e3, 2), dram_read_MB=round(rd / 1e6, 2),
                            dram_write_MB=round(wr / 1e6, 2),
                            dram_GBps=round((rd + wr) / dur, 1) if dur else None,
                            dram_pct=d["dram_pct"], tensor_pct=d["tensor_pct"],
                            bf16_ops_pct=d["bf16_ops_pct"],
                            sm_clock_GHz=round(d["clk"] / 1e9, 3) if d["clk"] else None,
                            regs=d["regs"])
            summary.append(e)
            traffic.setdefault(name, int(rd + wr))
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_full_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic["_source"] = (f"profiles/{rnd}_ncu_full_summary.json (ncu --set full, "
                          "dram__bytes_read.sum + dram__bytes_write.sum, first launch of each)")
    json.dump({"c3": traffic}, open(tp, "w"), indent=1)

    lp = os.path.join(src, "launches.csv")
    if os.path.exists(lp):
        txt = open(lp).read()
        txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
        rows = list(csv.DictReader(io.StringIO(txt)))
        tot = OrderedDict()
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(r["Metric Value"].replace(",", ""))
            unit = r.get("Metric Unit", "nsecond")
            v = v * UNIT_SCALE.get(unit, 1) / 1e3
            k = r["Kernel Name"][:60]
            n, s = tot.get(k, (0, 0.0))
            tot[k] = (n + 1, s + v)
        ours = {k: v for k, v in tot.items() if "moe::" in k or "tc_gemm" in k}
        total = sum(s for _, s in ours.values()) or 1.0
        with open(os.path.join(ROOT, "profiles", f"{rnd}_launches.txt"), "w") as f:
            f.write("# ncu --metrics gpu__time_duration.sum --clock-control none, "
                    "python bench.py --steps 2 --warmup 1\n# (cold-cache, serialised: compare "
                    "SHARES, not absolutes)\n# kernel | launches | total us | share of our kernels\n")
            for k, (n, s) in tot.items():
                share = f"{100 * s / total:6.2f}%" if k in ours else "   (not ours)"
                f.write(f"{k:<62}{n:>4} {s:>10.1f} {share}\n")
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()

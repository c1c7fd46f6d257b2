"""Summarises ncu captures into the JSON/markdown kept under profiles/.

usage: python profiles/summarize.py full <rep.ncu-rep> <out.json>        (one --set full capture)
       python profiles/summarize.py launches <launches.csv> <out.json>   (gpu__time_duration launch list)
"""
import csv
import collections
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "lts__t_sectors.avg.pct_of_peak_sustained_elapsed": "l2_sectors_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1tex_smem_pct",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_tc_wavefronts_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_active_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__cluster_dim_x": "cluster_x",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_mufu_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed": "sm_to_l2_request_path_pct",
    "dram__cycles_active.avg.pct_of_peak_sustained_elapsed": "dram_cycles_active_pct",
}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e-3, "msecond": 1e-3, "usecond": 1e-6,
         "us": 1e-6, "ns": 1e-9, "nsecond": 1e-9, "Ghz": 1e9, "Mhz": 1e6}


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = float(vals[i].replace(",", "")) if vals[i] not in ("", "n/a") else None
                u = units[i]
                if v is not None and u in SCALE:
                    v *= SCALE[u]
                    u = {"Gbyte": "B", "Mbyte": "B", "Kbyte": "B", "byte": "B", "msecond": "s", "ms": "s",
                         "usecond": "s", "us": "s", "ns": "s", "nsecond": "s", "Ghz": "Hz", "Mhz": "Hz"}[units[i]]
                d[name] = v
                d[name + "_unit"] = u
        if d.get("dram_read") is not None:
            d["dram_bytes_per_launch"] = d["dram_read"] + (d.get("dram_write") or 0.0)
            d["dram_gbs"] = d["dram_bytes_per_launch"] / d["duration"] / 1e9
        res.append(d)
    json.dump(res[0] if len(res) == 1 else res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


def launches(path, out):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    total = 0.0
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-9)
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
        total += v
    res = {"total_s": total, "kernels": [{"kernel": k, "launches": c, "total_s": t, "avg_s": t / c,
                                         "share": t / total} for k, (c, t) in
                                        sorted(agg.items(), key=lambda kv: -kv[1][1])]}
    json.dump(res, open(out, "w"), indent=1)
    for k in res["kernels"]:
        print(f"{k['kernel'][:60]:60s} {k['launches']:5d} {k['total_s']*1e3:10.2f} ms {100*k['share']:6.2f}%")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])

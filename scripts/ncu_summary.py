"""Summarise an `ncu --set full` report into a small JSON (committed under profiles/).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_ncu_summary.json profiles/attn_ncu_summary.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "l1tex__m_xbar2l1tex_read_bytes.sum": "l2_to_sm_bytes",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__registers_per_thread": "registers",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}
SCALE = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9,
         "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "Tbyte": 1e12, "Ghz": 1e9, "Mhz": 1e6,
         "cycle/nsecond": 1e9, "cycle/usecond": 1e6}


def summarise(rep):
    """Every captured launch: name + the METRICS above (one dict per launch, capture order)."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        res = {"kernel": row[hdr.index("Kernel Name")].split("(")[0]}
        for m, key in METRICS.items():
            cols = [j for j, h in enumerate(hdr) if h == m or h.endswith("." + m)]
            if not cols:
                continue
            i = cols[0]
            try:
                v = float(row[i].replace(",", ""))
            except ValueError:
                continue
            res[key] = v * SCALE.get(units[i], 1.0)
        if "dram_read" in res and "dram_write" in res:
            res["dram_bytes"] = res["dram_read"] + res["dram_write"]
        out.append(res)
    return out


def main(rep, out_all, out_attn):
    """out_all: every launch of the capture; out_attn: the attention call (K/V append + both
    k_attn_sm100 launches of one step) summed -- the traffic bench.py reports per call."""
    launches = summarise(rep)
    json.dump({"source": f"{rep} (ncu --set full --clock-control none, one steady-state step)",
               "launches": launches}, open(out_all, "w"), indent=1)
    parts = [x for x in launches if "k_attn_sm100" in x["kernel"] or "k_attn_p2" in x["kernel"]
             or "k_kv_append" in x["kernel"]]
    attn = {"source": f"{rep} (ncu --set full; k_attn_sm100 phase 2 + phase 1 of one step, + k_kv_append when the call appends)",
            "kernels": [x["kernel"] for x in parts],
            "duration": sum(x.get("duration", 0.0) for x in parts),
            "dram_read": sum(x.get("dram_read", 0.0) for x in parts),
            "dram_write": sum(x.get("dram_write", 0.0) for x in parts)}
    attn["dram_bytes_per_launch"] = attn["dram_read"] + attn["dram_write"]
    attn["per_kernel"] = parts
    json.dump(attn, open(out_attn, "w"), indent=1)
    for x in launches:
        print(f"{x['kernel'][:40]:40s} {x.get('duration', 0) * 1e6:9.1f} us  dram {x.get('dram_bytes', 0) / 1e6:9.1f} MB"
              f"  issue {x.get('issue_active_pct', 0):5.1f}%  tensor {x.get('tensor_pipe_active_pct', 0):5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:4])

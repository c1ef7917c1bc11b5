"""Summarise an `ncu --set full` report into a small JSON (committed under profiles/).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep k_attn_sm100 profiles/attn_ncu_summary.json
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


def main(rep, kernel, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {"source": f"{rep} (ncu --set full, kernel {kernel})", "launches": 0}
    for row in rows[2:]:
        name = row[hdr.index("Kernel Name")]
        if kernel not in name:
            continue
        res["launches"] += 1
        res["kernel"] = name.split("(")[0]
        for m, key in METRICS.items():
            cols = [j for j, h in enumerate(hdr) if h == m or h.endswith("." + m)]
            if not cols:
                continue
            i = cols[0]
            try:
                v = float(row[i].replace(",", ""))
            except ValueError:
                continue
            v *= SCALE.get(units[i], 1.0)
            res[key] = v
        break
    if "dram_read" in res and "dram_write" in res:
        res["dram_bytes_per_launch"] = res["dram_read"] + res["dram_write"]
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])

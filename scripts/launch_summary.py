"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) of bench.py steps:
per kernel the launch count, the median of its last 3 launches and its share of one step's
library-kernel time.  Cold-cache serialised replays: compare shares, not absolute times.

    python scripts/launch_summary.py gpurun_out/launches.csv > profiles/r01_launches_summary.txt
"""
import csv
import sys
from collections import OrderedDict

import numpy as np


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = OrderedDict()
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        per.setdefault(r[ik].split("(")[0], []).append(float(r[iv].replace(",", "")))
    unit = "ns" if max(max(v) for v in per.values()) > 1e5 else "us"
    sc = 1e3 if unit == "ns" else 1.0
    med = {k: float(np.median(v[-3:])) / sc for k, v in per.items()}
    own = {k: v for k, v in med.items() if "il::" in k or "sm100::" in k or "p2::" in k or k.startswith("k_")}
    # one step = each library kernel once (the attention: k_attn_sm100 = the dense pass over the
    # shared prefix, k_attn_p2 = each request's own part; IL_P2=0 runs k_attn_sm100 twice)
    step = sum(v for k, v in own.items() if len(per[k]) >= 2)
    print("# ncu launch list (gpu__time_duration.sum, --clock-control none), bench.py --steps 2 --warmup 3")
    print("# per kernel: launches, median of the last 3 launches (us), share of one step's own-kernel time")
    print("# cold-cache, serialised replays: compare SHARES, not absolute times")
    for k, v in sorted(med.items(), key=lambda kv: -kv[1]):
        share = f"{100 * v / step:5.1f}%" if k in own and len(per[k]) >= 2 else "  n/a"
        print(f"{k[:48]:48s} launches={len(per[k]):3d} median_us={v:9.1f} share={share}")


if __name__ == "__main__":
    main(sys.argv[1])

"""Profiling aid: build variants of the library with different compile-time attention knobs and
time the attention stage of the default bench workload with each (one GPU call).

    python scripts/attn_variants.py build NAME -DKNOB=VALUE ...   # here (nvcc cross-compiles)
    python scripts/attn_variants.py run NAME [NAME ...]            # on the GPU box
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    if sys.argv[1] == "build":
        sys.path.insert(0, os.path.join(ROOT, "paper_2507_08523_b200"))
        import build
        print(build.build(variant=sys.argv[2], defines=tuple(sys.argv[3:])))
        return
    for name in sys.argv[2:]:
        env = dict(os.environ)
        if name != "default":
            env["IL_LIB_VARIANT"] = name
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline", "--steps", "30"],
                             env=env, capture_output=True, text=True, timeout=600)
        try:
            d = json.loads(out.stdout.strip().split("\n")[-1])
            print(f"{name:16s} attn {d['stage_ms']['attn']:.4f} ms  total {d['ms_per_step']:.4f} ms  "
                  f"frac {d['roofline']['frac']:.3f}", flush=True)
        except Exception:
            print(name, "FAILED", out.stderr[-2000:], flush=True)


if __name__ == "__main__":
    main()

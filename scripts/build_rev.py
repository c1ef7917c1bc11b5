"""Profiling aid: build the library of a git revision as a variant
(paper_2507_08523_b200/variants/libinferlog_b200_NAME.so) for same-box A/B timing.

    python scripts/build_rev.py REV NAME [-DKNOB=VALUE ...]
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rev, name, defines = sys.argv[1], sys.argv[2], sys.argv[3:]
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run(f"git -C {ROOT} archive {rev} paper_2507_08523_b200 include | tar -x -C {tmp}", shell=True, check=True)
        sys.path.insert(0, os.path.join(tmp, "paper_2507_08523_b200"))
        import build
        out = build.build(variant=name, defines=tuple(defines))
        dst = os.path.join(ROOT, "paper_2507_08523_b200", "variants", os.path.basename(out))
        os.makedirs(os.path.dirname(dst), exist_ok=True)
        os.replace(out, dst)
        print(dst)


if __name__ == "__main__":
    main()

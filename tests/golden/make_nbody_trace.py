"""Generates tests/golden/nbody_trace/*: the reference n-body runner's instrumented reports
(fields_{update,move}.csv, heatmap_{update,move}.csv and its CSV rows) from oracle/_ref/ref_nbody,
the unmodified runner (proj/tools/nbody/runner.cpp:344-436) built from /root/reference.
Run in the build container:  python tests/golden/make_nbody_trace.py
"""
import json
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "nbody_trace")

# (layout, n, steps, f64, trace, heatmap granularity)
CASES = [
    ("aosoa:4", 64, 2, False, True, 64),
    ("soa-mb", 48, 3, True, True, 0),
    ("aos-packed", 32, 2, False, False, 1),
    ("bytesplit:soa-mb", 32, 2, False, True, 8),
    ("changetype:f32=f64:aosoa:8", 40, 2, False, True, 16),
    ("bitpack-float:8,23", 32, 2, False, True, 4),
    ("soa-sb", 37, 2, False, True, 32),
]


def case_dir(layout, n, steps, f64, trace, gran):
    tag = layout.replace(":", "_").replace(",", "_").replace("=", "_")
    return f"{tag}_{n}_{steps}_{'f64' if f64 else 'f32'}_t{int(trace)}_g{gran}"


def main():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_tool")
    shutil.rmtree(OUT, ignore_errors=True)
    index = []
    for layout, n, steps, f64, trace, gran in CASES:
        d = os.path.join(OUT, case_dir(layout, n, steps, f64, trace, gran))
        os.makedirs(d)
        r = subprocess.run([exe, "nbody", layout, str(n), str(steps), str(int(f64)), "42", str(int(trace)), str(gran), d],
                           check=True, capture_output=True, text=True)
        with open(os.path.join(d, "stdout.csv"), "w") as f:
            f.write(r.stdout)
        index.append({"dir": os.path.basename(d), "layout": layout, "n": n, "steps": steps, "f64": f64,
                      "trace": trace, "gran": gran})
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=1)
    print(f"wrote {len(index)} n-body trace fixtures")


if __name__ == "__main__":
    sys.exit(main())

"""Print the key fields of a bench.py JSON line."""
import json
import sys

d = json.load(open(sys.argv[1]))
print({k: d.get(k) for k in ["value", "ms_per_step", "gpu_launches", "clocks"]})
print("roofline", d.get("roofline"))
print("e2e", d.get("e2e"))
print("cpu_baseline", d.get("cpu_baseline"))
s = d.get("suite") or {}
if "C1_aos_to_soamb_1M" in s:
    print("C1", s["C1_aos_to_soamb_1M"])
for k, v in (s.get("C3_bitpack_2^28") or {}).items():
    print("C3", k, {a: round(b, 3) for a, b in v.items()})
if s.get("C5_shard_125M_R64_to_FAC_changetype_bytesplit"):
    print("C5", s["C5_shard_125M_R64_to_FAC_changetype_bytesplit"])
c4 = s.get("C4_nbody_128K_f32") or {}
for k, v in c4.items():
    if isinstance(v, dict) and "fast" in v:
        print("C4", k, {m: (round(x["interactions/s"] / 1e9, 1), round(x["frac_measured_fp32_peak"], 3))
                        for m, x in v.items() if isinstance(x, dict)})
print("C4 peak", c4.get("fp32_peak_measured_tflops"), c4.get("clocks_during_nbody"))
for k, v in (s.get("C6_other_compositions_2^26") or {}).items():
    print("C6", k, round(v["GB/s"]), round(v["frac"], 3))
if s.get("cpu_reference"):
    print("cpu_reference", json.dumps(s["cpu_reference"]))

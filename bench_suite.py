"""Secondary configs of BASELINE.json timed on one GPU (bench.py --suite).

C1  1M n-body records aos-packed -> soa-mb (fits in L2: reported, not a roofline number)
C3  BitpackIntSoA b in {3,7,12,16,24,31} and BitpackFloatSoA e8m10 / e5m10, pack and unpack, 2^28 values
C4  n-body 128K particles f32: update (exact and fast) over aos-packed / soa-mb / aosoa:8 / aosoa:32
C5  one GPU's shard of the 1e9-record copy: 125M R64 records aos-packed ->
    FieldAccessCount(changetype:f64=f32:bytesplit:soa-mb), 84 B/record
"""
from __future__ import annotations

R32 = "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}"
R64 = "Record{Pos:Record{x:f64,y:f64,z:f64},Vel:Record{x:f64,y:f64,z:f64},Mass:f64}"


def _time(fn, reps=5, warm=2):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for r in range(reps):
        ev[2 * r].record()
        fn()
        ev[2 * r + 1].record()
    torch.cuda.synchronize()
    ms = sorted(ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(reps))
    return ms[len(ms) // 2]


def _fill(L, view, seed):
    import torch
    lay = view.layout
    n = lay.element_count
    types = lay.leaf_types
    size = sum(lay.leaf(f)[1] for f in range(lay.leaf_count))
    g = torch.Generator(device="cuda").manual_seed(seed)
    raw = torch.randint(0, 2**31 - 1, ((n * size + 3) // 4,), device="cuda", dtype=torch.int32, generator=g)
    raw = raw.view(torch.uint8)[: n * size]
    if all(t == 8 for t in types):  # floats: keep them finite-ish so the minifloat paths see real values
        raw = (torch.randn(n * len(types), device="cuda", generator=g) * 100).to(torch.float32).view(torch.uint8)
    schema = view.layout.schema
    tmp = L.View(L.Layout(schema, f"i32:[{n}]", "aos-packed"), blobs=[raw.data_ptr()], blob_bytes=[n * size])
    L.copy_view(tmp, view)
    torch.cuda.synchronize()


OTHER_PAIRS = [  # compositions outside the BASELINE configs (informative)
    (R32, "aos-packed", "bytesplit:soa-mb", 0), (R32, "bytesplit:soa-mb", "aos-packed", 0),
    (R32, "aos-packed", "changetype:f32=f64:soa-mb", 0), (R32, "aos-packed", "split:Pos:soa-mb:aos-packed", 0),
    (R32, "aos-packed", "aosoa:3", 0), (R32, "aos-packed", "aos-aligned", 0), (R32, "soa-mb", "aos-packed", 1),
    (R32, "aos-packed", "soa-mb", 2), (R32, "aos-packed", "bitpack-float:5,10", 0),
    ("Record{a:f64,b:u16,c:i8,d:f32}", "aos-packed", "soa-mb", 0),
    (R64, "aos-packed", "bytesplit:soa-mb", 0), (R64, "changetype:f64=f32:bytesplit:soa-mb", "aos-packed", 0),
]


def cpu_reference(parts):
    """The reference's CPU path (oracle/_ref, the unmodified library) on bounded samples of each
    config, on 1 core (as shipped) and on every host core (the loop body over disjoint ranges,
    SURVEY 8(d) variant ii), timed on this box in the same run."""
    import os

    import numpy as np
    from oracle import ref
    if not ref.available():
        return {"unavailable": "oracle/_ref not built"}
    cores = os.cpu_count() or 1
    out = {"cores_all": cores}
    rng = np.random.default_rng(1)

    def copy_rate(schema, n, a, b, bytes_per, wrap=0, threads=1):
        ext = f"i32:[{n}]"
        src = [rng.integers(0, 256, sz, dtype=np.uint8) for sz in ref.layout_info(schema, ext, a)["blob_sizes"]]
        if "Record{v:f32}" in schema or schema == R64:
            # finite float values so the minifloat / conversion paths see real numbers
            vals = (rng.standard_normal(n * (7 if schema == R64 else 1)) * 100)
            src = ref.write_values(schema, ext, a, (vals.astype(np.float64 if schema == R64 else np.float32)
                                                    .view(np.uint64 if schema == R64 else np.uint32)
                                                    .astype(np.uint64).reshape(n, -1)))
        dst = ref.zero_blobs(schema, ext, b)
        r = ref.copy(schema, ext, a, src, b, dst, dst_wrap=wrap, nthreads=threads)
        return bytes_per * n / r["seconds"] / 1e9

    if "C3" in parts:
        c3 = {}
        for bits in (3, 12, 31):
            byt = 4 + bits / 8
            c3[f"int{bits}_pack_GB/s"] = {t: copy_rate("Record{v:u32}", 1 << 22, "soa-mb", f"bitpack-int:{bits}", byt,
                                                       threads=t) for t in (1, cores)}
        c3["e8m10_pack_GB/s"] = {t: copy_rate("Record{v:f32}", 1 << 21, "soa-mb", "bitpack-float:8,10", 4 + 19 / 8,
                                              threads=t) for t in (1, cores)}
        out["C3"] = dict(c3, sample="2^22 (int) / 2^21 (float) values per measurement")
    if "C4" in parts:
        c4 = {}
        for t in (1, cores):
            n = 16384 if t == 1 else 65536
            _, _, us, _ = ref.nbody("soa-mb", n, 1, seed=42, nthreads=t, with_blobs=False)
            c4[t] = n * n / us
        out["C4_interactions/s"] = dict(c4, sample="one update step, soa-mb, N=16384 (1 core) / 65536 (all cores)")
    if "C5" in parts:
        out["C5_GB/s"] = {t: copy_rate(R64, 1 << 20, "aos-packed", "changetype:f64=f32:bytesplit:soa-mb", 84, wrap=1,
                                       threads=t) for t in (1, cores)}
        out["C5_sample"] = "2^20 records per measurement"
    return out


def run_suite(L, device=0, peak_gbs=None, parts=("C1", "C3", "C4", "C5", "C6")):
    import torch
    if peak_gbs is None:
        from bench import peaks
        peak_gbs = peaks()[0]  # MEASURED_PEAKS.json hbm_gbs
    out = {}
    # ---- C1 ------------------------------------------------------------------------------
    if "C1" in parts:
        n = 1 << 20
        a = L.View(L.Layout(R32, f"i32:[{n}]", "aos-packed"))
        b = L.View(L.Layout(R32, f"i32:[{n}]", "soa-mb"))
        _fill(L, a, 1)
        ms = _time(lambda: L.copy_view(a, b))
        K = 50
        msk = _time(lambda: [L.copy_view(a, b) for _ in range(K)], reps=3, warm=1) / K
        out["C1_aos_to_soamb_1M"] = {
            "GB/s": 56 * n / msk / 1e6, "ms_per_copy": msk, "single_call_ms": ms,
            "note": "58.7 MB working set is L2-resident; GB/s over 50 back-to-back copies (device time per copy); "
                    "single_call_ms includes the ~6 us host dispatch of one call"}
        del a, b
    # ---- C3 ------------------------------------------------------------------------------
    if "C3" in parts:
        n = 1 << 28
        c3 = {}
        src = L.View(L.Layout("Record{v:u32}", f"i32:[{n}]", "soa-mb"))
        _fill(L, src, 3)
        back = L.View(L.Layout("Record{v:u32}", f"i32:[{n}]", "soa-mb"))
        for bits in (3, 7, 12, 16, 24, 31):
            pk = L.View(L.Layout("Record{v:u32}", f"i32:[{n}]", f"bitpack-int:{bits}"))
            byt = (4 + bits / 8) * n
            msp = _time(lambda: L.copy_view(src, pk), reps=3)
            msu = _time(lambda: L.copy_view(pk, back), reps=3)
            c3[f"int{bits}"] = {"pack_GB/s": byt / msp / 1e6, "unpack_GB/s": byt / msu / 1e6,
                                "pack_frac": byt / msp / 1e6 / peak_gbs, "unpack_frac": byt / msu / 1e6 / peak_gbs}
            del pk
        del src, back
        fsrc = L.View(L.Layout("Record{v:f32}", f"i32:[{n}]", "soa-mb"))
        _fill(L, fsrc, 4)
        fback = L.View(L.Layout("Record{v:f32}", f"i32:[{n}]", "soa-mb"))
        for e, m in ((8, 10), (5, 10)):
            pk = L.View(L.Layout("Record{v:f32}", f"i32:[{n}]", f"bitpack-float:{e},{m}"))
            byt = (4 + (1 + e + m) / 8) * n
            msp = _time(lambda: L.copy_view(fsrc, pk), reps=3)
            msu = _time(lambda: L.copy_view(pk, fback), reps=3)
            c3[f"e{e}m{m}"] = {"pack_GB/s": byt / msp / 1e6, "unpack_GB/s": byt / msu / 1e6,
                               "pack_frac": byt / msp / 1e6 / peak_gbs, "unpack_frac": byt / msu / 1e6 / peak_gbs}
            del pk
        del fsrc, fback
        out["C3_bitpack_2^28"] = c3
    # ---- C4 ------------------------------------------------------------------------------
    if "C4" in parts:
        n = 128 * 1024
        from bench import ClockSampler
        props = torch.cuda.get_device_properties(device)
        nominal = 2 * 128 * props.multi_processor_count * 1.965e9 / 1e12  # TFLOP/s at max SM clock
        with ClockSampler(device) as clk_peak:
            measured = L.fp32_peak_tflops(device, 2.0)  # sustained FFMA chains, same power regime
        c4 = {}
        with ClockSampler(device) as clk:
            for lay in ("aos-packed", "soa-mb", "aosoa:8", "aosoa:32"):
                v = L.View(L.Layout(R32, f"i64:[{n}]", lay))
                v.nbody_init(42)
                row = {}
                for mode, name in ((1, "fast"), (0, "exact")):
                    ms = _time(lambda: v.nbody_update(mode), reps=5, warm=2)
                    ips = n * n / (ms * 1e-3)
                    row[name] = {"ms_per_update": ms, "interactions/s": ips, "TFLOP/s@20": ips * 20 / 1e12,
                                 "frac_measured_fp32_peak": ips * 20 / 1e12 / measured,
                                 "frac_nominal_fp32_peak": ips * 20 / 1e12 / nominal}
                row["move_ms"] = _time(lambda: v.nbody_move(), reps=3)
                c4[lay] = row
                del v
            # the reference's hand-written baselines (steps.hpp:124-230) as plain device kernels:
            # library / hand-written = paper Fig. 3's ratio
            for kind, lib_lay in (("manual-aos", "aos-packed"), ("manual-soa", "soa-mb")):
                m = L.ManualNbody(kind, n, seed=42)
                row = {}
                for mode, name in ((1, "fast"), (0, "exact")):
                    ms = _time(lambda: m.update(mode), reps=5, warm=2)
                    ips = n * n / (ms * 1e-3)
                    row[name] = {"ms_per_update": ms, "interactions/s": ips,
                                 "frac_measured_fp32_peak": ips * 20 / 1e12 / measured,
                                 "library_over_handwritten": c4[lib_lay][name]["interactions/s"] / ips}
                row["move_ms"] = _time(lambda: m.move(), reps=3)
                c4[kind] = row
                del m
        out["C4_nbody_128K_f32"] = dict(
            c4, fp32_peak_measured_tflops=measured, fp32_peak_nominal_tflops=nominal,
            clocks_during_peak=clk_peak.summary(), clocks_during_nbody=clk.summary(),
            peak_note="measured: lam_bench_fma_peak (independent FFMA chains, 2 s sustained); "
                      "nominal: 2 x 128 lanes x SMs x 1.965 GHz; flop convention 20 per interaction")
    # ---- C5 ------------------------------------------------------------------------------
    if "C5" in parts:
        n = 125_000_000
        src = L.View(L.Layout(R64, f"i32:[{n}]", "aos-packed"))
        _fill(L, src, 5)
        dst = L.View(L.Layout(R64, f"i32:[{n}]", "changetype:f64=f32:bytesplit:soa-mb", wrap=1))
        ms = _time(lambda: L.copy_view(src, dst), reps=3)
        r, w = dst.counters()
        out["C5_shard_125M_R64_to_FAC_changetype_bytesplit"] = {
            "GB/s": 84 * n / ms / 1e6, "frac": 84 * n / ms / 1e6 / peak_gbs, "ms": ms,
            "writes_per_leaf_after_runs": [int(x) for x in w]}
        del src, dst
    # ---- C6 (not a BASELINE config): other compositions, 2^26 records ---------------------
    if "C6" in parts:
        n = 1 << 26
        c6 = {}
        for schema, a, b, wrap in OTHER_PAIRS:
            la = L.Layout(schema, f"i32:[{n}]", a)
            lb = L.Layout(schema, f"i32:[{n}]", b, wrap=wrap, granularity=64)
            s, d = L.View(la), L.View(lb)
            _fill(L, s, 6)
            ms = _time(lambda: L.copy_view(s, d), reps=3, warm=1)
            # algorithmic bytes: source storage read + destination storage written
            byt = sum(la.blob_sizes) + sum(lb.blob_sizes)
            tag = {0: "", 1: " +FieldAccessCount", 2: " +Heatmap(64)"}[wrap]
            c6[f"{a} -> {b}{tag}" + {R32: "", R64: " (R64)"}.get(schema, " (mixed record)")] = {
                "GB/s": byt / ms / 1e6, "frac": byt / ms / 1e6 / peak_gbs}
            del s, d
        out["C6_other_compositions_2^26"] = c6
    out["cpu_reference"] = cpu_reference(parts)
    return out


if __name__ == "__main__":
    import json
    import sys
    sys.path.insert(0, ".")
    from paper_2302_08251_b200 import lamina
    print(json.dumps(run_suite(lamina, 0, parts=tuple(sys.argv[1:]) or ("C1", "C3", "C4", "C5", "C6")), indent=1))

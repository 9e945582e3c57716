"""Parity at configuration scale (SURVEY 8(d) "Parity at scale ... chunk-wise").

Every BASELINE config is checked at the size its throughput is quoted on, against the
reference itself (oracle/_ref/libref.so, the unmodified lamina library):

  C2  all 25 ordered pairs of {aos-packed, soa-sb, soa-mb, aosoa:8, aosoa:32} at 2^26 R32
      records. The GPU copies the whole view; the reference copyView (view.cpp:168-189) runs
      on 2^22-record chunks [a, a+c) built from the same values, and each chunk's blobs must
      equal the GPU blob slices (aos/aosoa: bytes [28a, 28(a+c)); soa-mb: [4a, 4(a+c)) per
      blob; soa-sb: the same slice of every leaf subarray). Every byte is compared.
  C3  BitpackIntSoA b = 3..31 (u32 and i32) and BitpackFloatSoA e8m10 / e5m10 over 2^28
      values. Packed words equal the reference chunk-wise (chunks are multiples of 32
      values, so a chunk starts on a word: words [a*b/32, (a+c)*b/32)). For b >= 16 the bit
      offsets pass 2^32. Unpack equals the reference's read semantics (computed.cpp:101-122)
      on the full array and the reference itself on chunks incl. the last word.
  C4  n-body 128K f32, 5 steps, exact mode: final state and checksum bit-identical to the
      reference runner body (steps.hpp:13-118, 16 host threads over disjoint i-ranges, same
      j order) for four mappings; fast mode within FAST_TOL.
  C5  one 125M-record GPU shard of the 1e9-record C5 copy: R64 aos-packed ->
      FieldAccessCount(changetype:f64=f32:bytesplit:soa-mb), source = scalarSample(F64,
      i*7+f) (oracles.cpp:211-223). All 28 byte planes (3.5 GB) equal the reference's
      conversion of every value; chunks at the start, past the 4 GiB source byte offset and at
      the end equal the reference copyView; write counters = N per leaf.

Sizes are the configs' own; the whole module runs in a few minutes on a 16-core host.
"""
import os

import numpy as np
import pytest

from conftest import R32, R64

pytestmark = pytest.mark.gpu

THREADS = max(1, min(32, os.cpu_count() or 1))
C2_LAYOUTS = ["aos-packed", "soa-sb", "soa-mb", "aosoa:8", "aosoa:32"]
FAST_TOL = 2e-5  # |pos_fast - pos_exact| <= FAST_TOL * max(1, |pos_exact|) after 5 steps at 128K


def lm():
    from paper_2302_08251_b200 import lamina
    return lamina


def chunk_slices(layout, n, a, c, leaf_sizes):
    """(global blob, global lo, global hi, chunk blob, chunk lo, chunk hi) of the element range
    [a, a+c) of an n-element view vs the c-element chunk view (SURVEY 8(d) slice rules)."""
    rec = sum(leaf_sizes)
    if layout in ("aos-packed",) or layout.startswith("aosoa:"):
        return [(0, rec * a, rec * (a + c), 0, 0, rec * c)]
    if layout == "soa-mb":
        return [(f, s * a, s * (a + c), f, 0, s * c) for f, s in enumerate(leaf_sizes)]
    if layout == "soa-sb":
        out, base_g, base_c = [], 0, 0
        for s in leaf_sizes:
            out.append((0, base_g + s * a, base_g + s * (a + c), 0, base_c, base_c + s * c))
            base_g += s * n
            base_c += s * c
        return out
    raise ValueError(layout)


def assert_chunk_equal(tag, got_blobs, ref_blobs, slices):
    for g, lo, hi, cb, clo, chi in slices:
        x, y = got_blobs[g][lo:hi], ref_blobs[cb][clo:chi]
        if not np.array_equal(x, y):
            bad = np.flatnonzero(x != y)
            raise AssertionError(f"{tag}: blob {g} bytes [{lo},{hi}) differ at +{bad[:6]} (of {bad.size})")


# ----------------------------------------------------------------------------------------- C2
def c2_values(n, seed=2026):
    """[n, 7] u32 bit patterns: full range plus NaN / sNaN / +-0 / denormal / Inf patterns."""
    rng = np.random.default_rng(seed)
    v = rng.integers(0, 2**32, (n, 7), dtype=np.uint32)
    special = np.array([0x7FC00000, 0xFFC00000, 0x7F800001, 0xFFA00001, 0x7F800000, 0xFF800000, 0x00000001,
                        0x80000001, 0x007FFFFF, 0x80000000, 0x00000000], np.uint32)
    idx = rng.integers(0, n, n // 7)
    v[idx, rng.integers(0, 7, idx.size)] = special[rng.integers(0, special.size, idx.size)]
    return v


def test_c2_all_pairs_2p26_vs_reference(ref):
    L = lm()
    n, c = 1 << 26, 1 << 22
    ext = f"i32:[{n}]"
    vals = c2_values(n)
    aos_bytes = vals.reshape(-1).view(np.uint8)
    lays = {a: L.Layout(R32, ext, a) for a in C2_LAYOUTS}
    aos = L.View(lays["aos-packed"])
    aos.upload(0, aos_bytes)
    dst = {b: L.View(lays[b]) for b in C2_LAYOUTS}
    cext = f"i32:[{c}]"
    sizes = [4] * 7
    checked = 0
    for a in C2_LAYOUTS:
        if a == "aos-packed":
            src = aos
        else:  # the (aos-packed, a) pair has been verified below before it is used as a source
            src = L.View(lays[a])
            L.copy_view(aos, src)
        for b in C2_LAYOUTS:
            L.copy_view(src, dst[b])
            got = dst[b].download_all()
            for k in range(n // c):
                lo = k * c
                chunk_aos = [np.ascontiguousarray(aos_bytes[28 * lo:28 * (lo + c)])]
                if a == "aos-packed":
                    chunk_src = chunk_aos
                else:
                    chunk_src = ref.zero_blobs(R32, cext, a)
                    ref.copy(R32, cext, "aos-packed", chunk_aos, a, chunk_src, nthreads=THREADS)
                chunk_dst = ref.zero_blobs(R32, cext, b)
                ref.copy(R32, cext, a, chunk_src, b, chunk_dst, nthreads=THREADS)
                assert_chunk_equal(f"{a} -> {b} chunk {k}", got, chunk_dst, chunk_slices(b, n, lo, c, sizes))
                checked += sum(x.nbytes for x in chunk_dst)
            del got
        del src
    assert checked == 25 * 28 * n


# ----------------------------------------------------------------------------------------- C3
N3 = 1 << 28
C3 = 1 << 24  # chunk: multiple of 32 values, so a chunk begins on a 32-bit word of every width


@pytest.fixture(scope="module")
def c3_src():
    L = lm()
    rng = np.random.default_rng(3)
    vals = rng.integers(0, 2**32, N3, dtype=np.uint32)
    vals[: 1 << 20] &= np.uint32(0x7F)  # small magnitudes: round trips exercise the sign bit of b
    src = L.View(L.Layout("Record{v:u32}", f"i32:[{N3}]", "soa-mb"))
    src.upload(0, vals.view(np.uint8))
    ssrc = L.View(L.Layout("Record{v:i32}", f"i32:[{N3}]", "soa-mb"))  # the same bits as i32 values
    ssrc.upload(0, vals.view(np.uint8))
    yield vals, src, ssrc
    del src, ssrc


def ref_pack_chunks(ref, schema, layout, vals_u8, vsize, bits, chunks):
    """Reference copyView soa-mb -> layout over value chunks; yields (chunk index, packed words)."""
    ext = f"i32:[{C3}]"
    for k in chunks:
        lo = k * C3
        src = [np.ascontiguousarray(vals_u8[vsize * lo: vsize * (lo + C3)])]
        dst = ref.zero_blobs(schema, ext, layout)
        ref.copy(schema, ext, "soa-mb", src, layout, dst, nthreads=THREADS)
        yield k, dst[0]


def check_packed_vs_ref(ref, schema, layout, vals_u8, packed, bits, chunks):
    for k, words in ref_pack_chunks(ref, schema, layout, vals_u8, 4, bits, chunks):
        lo = k * C3 * bits // 8
        assert np.array_equal(packed[lo: lo + words.nbytes], words), f"{layout} chunk {k} (byte {lo})"


def check_unpacked_vs_ref(ref, schema, layout, packed, got_u8, bits, chunks):
    ext = f"i32:[{C3}]"
    for k in chunks:
        lo = k * C3 * bits // 8
        src = [np.ascontiguousarray(packed[lo: lo + C3 * bits // 8])]
        dst = ref.zero_blobs(schema, ext, "soa-mb")
        ref.copy(schema, ext, layout, src, "soa-mb", dst, nthreads=THREADS)
        assert np.array_equal(got_u8[4 * k * C3: 4 * (k + 1) * C3], dst[0]), f"unpack {layout} chunk {k}"


@pytest.mark.parametrize("bits", list(range(3, 32)))
def test_c3_bitpack_int_2p28_vs_reference(ref, c3_src, bits):
    L = lm()
    vals, src, ssrc = c3_src
    ext = f"i32:[{N3}]"
    nchunks = N3 // C3
    pk = L.View(L.Layout("Record{v:u32}", ext, f"bitpack-int:{bits}"))
    L.copy_view(src, pk)
    packed = pk.download(0)
    assert packed.nbytes == ((N3 * bits + 31) // 32) * 4
    # every word against the reference (the chunks tile the whole stream)
    check_packed_vs_ref(ref, "Record{v:u32}", f"bitpack-int:{bits}", vals.view(np.uint8), packed, bits, range(nchunks))
    # unpack u32: zero extension of the low b bits (computed.cpp:101-122), every value ...
    back = L.View(L.Layout("Record{v:u32}", ext, "soa-mb"))
    L.copy_view(pk, back)
    got = back.download(0).view(np.uint32)
    mask = np.uint32((1 << bits) - 1)
    assert np.array_equal(got, vals & mask)
    # ... and the reference itself on the first, the 2^32-bit-offset straddling and the last chunk
    straddle = min(nchunks - 1, (1 << 32) // bits // C3)
    check_unpacked_vs_ref(ref, "Record{v:u32}", f"bitpack-int:{bits}", packed, got.view(np.uint8), bits,
                          sorted({0, straddle, nchunks - 1}))
    del back, got
    # i32: the packed words are the same low bits; unpack sign-extends
    spk = L.View(L.Layout("Record{v:i32}", ext, f"bitpack-int:{bits}"))
    L.copy_view(ssrc, spk)
    assert np.array_equal(spk.download(0), packed)
    sback = L.View(L.Layout("Record{v:i32}", ext, "soa-mb"))
    L.copy_view(spk, sback)
    sgot = sback.download(0).view(np.int32)
    low = (vals & mask).astype(np.int64)
    sign = np.int64(1 << (bits - 1))
    assert np.array_equal(sgot, ((low ^ sign) - sign).astype(np.int32))
    check_unpacked_vs_ref(ref, "Record{v:i32}", f"bitpack-int:{bits}", packed, sgot.view(np.uint8), bits,
                          sorted({0, straddle, nchunks - 1}))


def c3_float_values(n, seed=4):
    """SURVEY 8(d) C3 float input: (u*2-1)*10^k, k uniform in [-6, 6], plus 1% specials (+-0,
    +-Inf, NaN with payloads, f32 subnormals, +-65520 (e5m10 overflow), 3.4e38 (e8 overflow))."""
    rng = np.random.default_rng(seed)
    out = np.empty(n, np.uint32)
    step = 1 << 24
    special = np.array([0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0xFFC00001, 0x7F800001,
                        0x7FA5A5A5, 0x00000001, 0x807FFFFF, 0x00400000, 0x477FF000, 0xC77FF000, 0x7F7FFFFF,
                        0x7F7FF000, 0x33800000, 0x33000000, 0x387FC000], np.uint32)
    for lo in range(0, n, step):
        m = min(step, n - lo)
        v = ((rng.random(m) * 2 - 1) * 10.0 ** rng.integers(-6, 7, m)).astype(np.float32).view(np.uint32)
        pick = rng.random(m) < 0.01
        v[pick] = special[rng.integers(0, special.size, int(pick.sum()))]
        out[lo:lo + m] = v
    return out


@pytest.mark.parametrize("fmt", [(8, 10), (5, 10)], ids=["e8m10", "e5m10"])
def test_c3_bitpack_float_2p28_vs_reference(ref, fmt):
    L = lm()
    e, m = fmt
    bits = 1 + e + m
    vals = c3_float_values(N3)
    ext = f"i32:[{N3}]"
    lay = f"bitpack-float:{e},{m}"
    src = L.View(L.Layout("Record{v:f32}", ext, "soa-mb"))
    src.upload(0, vals.view(np.uint8))
    pk = L.View(L.Layout("Record{v:f32}", ext, lay))
    L.copy_view(src, pk)
    del src
    packed = pk.download(0)
    nchunks = N3 // C3
    check_packed_vs_ref(ref, "Record{v:f32}", lay, vals.view(np.uint8), packed, bits, range(nchunks))
    back = L.View(L.Layout("Record{v:f32}", ext, "soa-mb"))
    L.copy_view(pk, back)
    got = back.download(0)
    check_unpacked_vs_ref(ref, "Record{v:f32}", lay, packed, got, bits, range(nchunks))


# ----------------------------------------------------------------------------------------- C4
N4 = 128 * 1024


@pytest.fixture(scope="module")
def c4_reference(ref):
    """The reference n-body body (ref_shim ref_nbody: drawInitValues + steps.hpp:13-118) at 128K,
    5 steps, i-range split over the host threads with the reference's j order per i."""
    cs, blobs, _, _ = ref.nbody("soa-mb", N4, 5, nthreads=THREADS)
    return cs, blobs


@pytest.mark.parametrize("layout", ["soa-mb", "aos-packed", "aosoa:8", "aosoa:32"])
def test_c4_nbody_128k_exact_vs_reference(c4_reference, layout):
    L = lm()
    cs, ref_blobs = c4_reference
    v = L.View(L.Layout(R32, f"i64:[{N4}]", layout))
    v.nbody_init(42)
    for _ in range(5):
        v.nbody_step(L.NBODY_EXACT)
    assert v.nbody_checksum() == cs
    as_soa = L.View(L.Layout(R32, f"i64:[{N4}]", "soa-mb"))
    L.copy_view(v, as_soa)
    for f, (x, y) in enumerate(zip(as_soa.download_all(), ref_blobs)):
        assert np.array_equal(x, y), f"leaf {f}: {np.flatnonzero(x != y)[:8]}"


def test_c4_nbody_128k_fast_within_tolerance(c4_reference):
    L = lm()
    _, ref_blobs = c4_reference
    v = L.View(L.Layout(R32, f"i64:[{N4}]", "soa-mb"))
    v.nbody_init(42)
    for _ in range(5):
        v.nbody_step(L.NBODY_FAST)
    got = v.download_all()
    for f in range(3):
        a = got[f].view(np.float32).astype(np.float64)
        b = ref_blobs[f].view(np.float32).astype(np.float64)
        err = np.abs(a - b) / np.maximum(1.0, np.abs(b))
        assert err.max() <= FAST_TOL, (f, err.max())


# ----------------------------------------------------------------------------------------- C5
N5 = 125_000_000
C5_LAYOUT = "changetype:f64=f32:bytesplit:soa-mb"


def scalar_sample_f64(idx_u64):
    """oracle::scalarSample(F64, salt) (tests/support/oracles.cpp:211-223), vectorised."""
    h = idx_u64 * np.uint64(0x9E3779B97F4A7C15) + np.uint64(0x2545F4914F6CDD1D)
    return (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 * 4.0 - 2.0


def test_c5_shard_125m_vs_reference(ref):
    import torch
    L = lm()
    n = N5
    ext = f"i32:[{n}]"
    # source: scalarSample(F64, i*7+f) generated on the device (torch int64 arithmetic wraps mod 2^64)
    src_t = torch.empty(n * 7, dtype=torch.float64, device="cuda")
    step = 1 << 26
    for lo in range(0, n * 7, step):
        hi = min(n * 7, lo + step)
        s = torch.arange(lo, hi, dtype=torch.int64, device="cuda")
        h = s * (0x9E3779B97F4A7C15 - 2**64) + 0x2545F4914F6CDD1D
        u = (h >> 11) & ((1 << 53) - 1)
        src_t[lo:hi] = u.to(torch.float64) * 2.0 ** -53 * 4.0 - 2.0
    torch.cuda.synchronize()
    src = L.View(L.Layout(R64, ext, "aos-packed"), blobs=[src_t.data_ptr()], blob_bytes=[n * 56])
    dst = L.View(L.Layout(R64, ext, C5_LAYOUT, wrap=1))
    L.copy_view(src, dst)
    reads, writes = dst.counters()
    assert list(writes) == [n] * 7 and list(reads) == [0] * 7
    planes = dst.download_all()
    assert len(planes) == 28 and all(p.nbytes == n for p in planes)
    # every value: x86 cvtsd2ss of the source (finite values in [-2, 2): numpy's RNE cast is it)
    step = 1 << 24
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        idx = np.arange(lo, hi, dtype=np.uint64)
        for f in range(7):
            f32 = scalar_sample_f64(idx * np.uint64(7) + np.uint64(f)).astype(np.float32).view(np.uint32)
            for k in range(4):
                want = ((f32 >> np.uint32(8 * k)) & np.uint32(0xFF)).astype(np.uint8)
                assert np.array_equal(planes[4 * f + k][lo:hi], want), f"leaf {f} byte {k} records [{lo},{hi})"
    # the reference copyView itself on chunks: start, past the 4 GiB source offset, the end
    c = 1 << 22
    host_src = None
    for a in (0, (1 << 32) // 56 // c * c + c, n - c):
        idx = (np.arange(a, a + c, dtype=np.uint64)[:, None] * np.uint64(7) + np.arange(7, dtype=np.uint64))
        host_src = [scalar_sample_f64(idx).reshape(-1).view(np.uint8)]
        assert np.array_equal(host_src[0], src_t[a * 7:(a + c) * 7].cpu().numpy().view(np.uint8))
        cext = f"i32:[{c}]"
        chunk = ref.zero_blobs(R64, cext, C5_LAYOUT)
        r = ref.copy(R64, cext, "aos-packed", host_src, C5_LAYOUT, chunk, dst_wrap=1, nthreads=THREADS)
        assert list(r["dst_fac"][7:]) == [c] * 7
        for p in range(28):
            assert np.array_equal(planes[p][a:a + c], chunk[p]), f"plane {p} chunk at {a}"
    del src, dst, src_t

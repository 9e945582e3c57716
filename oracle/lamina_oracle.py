"""TEST INFRASTRUCTURE ONLY — CPU restatement (numpy) of the reference's hot path.

This is the checker for the sm_100a kernels.  It is never imported by the product
package; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.

It restates, vectorised over the element index, the algorithm of the reference
library `lamina` (/root/reference/proj, paths relative to it):

  record schema + leaf table      core/src/record.cpp:86-158, grammar 364-479
  array extents                   core/src/extents.cpp:47-177
  AoS / SoA / AoSoA / One offsets core/src/mappings.cpp:23-175
  Split                           core/src/mappings.cpp:180-389
  BitpackIntSoA / BitpackFloatSoA core/src/computed.cpp:18-222
  ChangeType / Bytesplit / Null   core/src/computed.cpp:228-531
  readBits / writeBits / pack     core/src/bitpack.cpp:11-94
  floatEncode / floatDecode       core/src/bitpack.cpp:96-188
  ScalarValue conversions         core/include/lamina/scalar.hpp:112-356
  FieldAccessCount / Heatmap      core/src/instrument.cpp:24-229
  copyView                        core/src/view.cpp:168-189
  n-body kernel / steps / init    tools/nbody/kernel.hpp:15-41, steps.hpp:13-118,
                                  runner.cpp:30-72

Pinning: tests/test_oracle_*.py check this module against the reference's own
known-answer tests (test_bitpack.cpp, test_computed.cpp, test_mappings.cpp,
test_view.cpp, test_instrument.cpp, test_kernel.cpp, acceptance.cpp) and against
the compiled reference itself (oracle/_ref, fixtures in tests/golden/).

Values travel as the storage bits of their scalar kind in uint64 arrays
(ScalarValue::storageBits, scalar.hpp:231-246).  Since distinct (i, f) accesses
never share storage bits, copyView's i-outer/f-inner loop (view.cpp:186-188) is
evaluated leaf by leaf over all i at once with identical results.
"""
from __future__ import annotations

import re
from dataclasses import dataclass, field

import numpy as np

I8, I16, I32, I64, U8, U16, U32, U64, F32, F64, BOOL = range(11)
NAMES = ("i8", "i16", "i32", "i64", "u8", "u16", "u32", "u64", "f32", "f64", "bool")
SIZE = (1, 2, 4, 8, 1, 2, 4, 8, 4, 8, 1)

U = np.uint64


def _is_signed(t):
    return t in (I8, I16, I32, I64)


def _is_unsigned(t):
    return t in (U8, U16, U32, U64)


def _is_int(t):
    return _is_signed(t) or _is_unsigned(t)


def _is_float(t):
    return t in (F32, F64)


def _mask(bits):
    return U(0xFFFFFFFFFFFFFFFF) if bits >= 64 else U((1 << bits) - 1)


def _shl(x, s):
    """x << s for uint64 arrays, 0 when s >= 64 (numpy would wrap the count)."""
    s = int(s)
    if s >= 64:
        return np.zeros_like(x)
    return x << U(s)


def _shr(x, s):
    s = int(s)
    if s >= 64:
        return np.zeros_like(x)
    return x >> U(s)


# =============================================================================================
# schema — record.cpp:86-158 (leaf table), 364-479 (grammar)
# =============================================================================================
@dataclass
class Node:
    kind: str  # "leaf" | "record" | "array"
    scalar: int = F64
    count: int = 0
    element: "Node | None" = None
    fields: list = field(default_factory=list)  # [(tag, Node)]

    def children(self):
        if self.kind == "record":
            return [n for _, n in self.fields]
        if self.kind == "array":
            return [self.element] * self.count
        return []


@dataclass
class Leaf:
    coord: tuple
    path: str
    type: int
    size: int
    offset_packed: int = 0
    offset_aligned: int = 0


def _same(a: Node, b: Node) -> bool:
    if a.kind != b.kind:
        return False
    if a.kind == "leaf":
        return a.scalar == b.scalar
    if a.kind == "array":
        return a.count == b.count and _same(a.element, b.element)
    return len(a.fields) == len(b.fields) and all(
        ta == tb and _same(na, nb) for (ta, na), (tb, nb) in zip(a.fields, b.fields))


class Schema:
    def __init__(self, root: Node):
        self.root = root
        self.leaves: list[Leaf] = []

        def walk(n, coord, path):
            if n.kind == "leaf":
                self.leaves.append(Leaf(tuple(coord), path, n.scalar, SIZE[n.scalar]))
                return
            if n.kind == "record":
                for k, (tag, c) in enumerate(n.fields):
                    walk(c, coord + [k], f"{path}.{tag}" if path else tag)
            else:
                for k in range(n.count):
                    walk(n.element, coord + [k], f"{path}[{k}]")

        walk(root, [], "")
        packed = aligned = 0
        mx = 1
        for l in self.leaves:
            l.offset_packed = packed
            packed += l.size
            aligned = (aligned + l.size - 1) // l.size * l.size
            l.offset_aligned = aligned
            aligned += l.size
            mx = max(mx, l.size)
        self.size_packed = packed
        self.size_aligned = (aligned + mx - 1) // mx * mx

    @staticmethod
    def parse(text: str) -> "Schema":
        toks = re.findall(r"[A-Za-z_][A-Za-z0-9_]*|\d+|[{}\[\]:,]", text)
        pos = 0

        def take(expect=None):
            nonlocal pos
            if pos >= len(toks):
                raise ValueError("schema parse error: unexpected end")
            t = toks[pos]
            if expect is not None and t != expect:
                raise ValueError(f"schema parse error: expected '{expect}'")
            pos += 1
            return t

        def node():
            w = take()
            if w == "Record":
                take("{")
                fields = []
                if toks[pos] != "}":
                    while True:
                        tag = take()
                        take(":")
                        fields.append((tag, node()))
                        if toks[pos] == ",":
                            take(",")
                            continue
                        break
                take("}")
                base = Node("record", fields=fields)
            else:
                if w not in NAMES:
                    raise ValueError(f"unknown scalar type: '{w}'")
                base = Node("leaf", scalar=NAMES.index(w))
            counts = []
            while pos < len(toks) and toks[pos] == "[":
                take("[")
                counts.append(int(take()))
                take("]")
            for c in reversed(counts):
                base = Node("array", count=c, element=base)
            return base

        root = node()
        if pos != len(toks):
            raise ValueError("schema parse error: trailing characters")
        return Schema(root)

    def node_at(self, coord):
        n = self.root
        for i in coord:
            ch = n.children()
            if i >= len(ch):
                return None
            n = ch[i]
        return n

    def coord_of(self, dotted: str):
        """record.cpp:220-277"""
        path = []
        n = self.root
        for seg in [s for s in re.split(r"[.\[\]]", dotted) if s != ""]:
            if seg[0].isdigit():
                idx = int(seg)
                ch = n.children()
                if idx >= len(ch):
                    raise ValueError(f"no such field: index {seg}")
                path.append(idx)
                n = ch[idx]
                continue
            if n.kind != "record":
                raise ValueError(f"no such field: '{seg}'")
            for k, (tag, c) in enumerate(n.fields):
                if tag == seg:
                    path.append(k)
                    n = c
                    break
            else:
                raise ValueError(f"no such field: '{seg}'")
        return tuple(path)

    def path_of(self, coord):
        out = ""
        n = self.root
        for i in coord:
            if n.kind == "record":
                out += ("." if out else "") + n.fields[i][0]
                n = n.fields[i][1]
            else:
                out += f"[{i}]"
                n = n.element
        return out

    def leaf_range(self, coord):
        idx = [k for k, l in enumerate(self.leaves) if l.coord[: len(coord)] == tuple(coord)]
        return (idx[0], idx[-1] + 1) if idx else (0, 0)

    def __eq__(self, other):
        return _same(self.root, other.root)


# =============================================================================================
# extents — extents.cpp:47-177
# =============================================================================================
_IT_MAX = {"i16": 0x7FFF, "i32": 0x7FFFFFFF, "i64": 0x7FFFFFFFFFFFFFFF, "u16": 0xFFFF, "u32": 0xFFFFFFFF,
           "u64": 0xFFFFFFFFFFFFFFFF}


def parse_extents(text: str, dyn=()):
    it, rest = text.split(":", 1)
    dims = [d.strip() for d in rest.strip()[1:-1].split(",") if d.strip() != ""]
    vals = list(dyn)
    n = 1
    for d in dims:
        e = vals.pop(0) if d == "dyn" else int(d)
        if e > _IT_MAX[it]:
            raise OverflowError("index type overflow: extent")
        n *= e
        if n > _IT_MAX[it]:
            raise OverflowError("index type overflow: total element count")
    return n


# =============================================================================================
# scalar value conversions — scalar.hpp:295-306 with x86 SSE (cvtss2sd / cvtsd2ss) NaN rules
# =============================================================================================
def f32_to_f64(b32):
    b = np.asarray(b32, dtype=U) & U(0xFFFFFFFF)
    nan = ((b & U(0x7F800000)) == U(0x7F800000)) & ((b & U(0x7FFFFF)) != 0)
    with np.errstate(all="ignore"):
        conv = b.astype(np.uint32).view(np.float32).astype(np.float64).view(U)
    q = ((b >> U(31)) << U(63)) | U(0x7FF8000000000000) | ((b & U(0x7FFFFF)) << U(29))
    return np.where(nan, q, conv)


def f64_to_f32(b64):
    b = np.asarray(b64, dtype=U)
    nan = ((b & U(0x7FF0000000000000)) == U(0x7FF0000000000000)) & ((b & U(0xFFFFFFFFFFFFF)) != 0)
    with np.errstate(all="ignore"):
        conv = b.view(np.float64).astype(np.float32).view(np.uint32).astype(U)
    q = ((b >> U(63)) << U(31)) | U(0x7FC00000) | ((b >> U(29)) & U(0x3FFFFF))
    return np.where(nan, q, conv)


def convert(v, frm, to):
    """ScalarValue::convertTo on storage bits."""
    if frm == to:
        return v
    if frm == F32 and to == F64:
        return f32_to_f64(v)
    if frm == F64 and to == F32:
        return f64_to_f32(v)
    fw, tw = 8 * SIZE[frm], 8 * SIZE[to]
    v = np.asarray(v, dtype=U)
    if _is_signed(frm) and fw < 64:
        s = U(1 << (fw - 1))
        v = ((v & _mask(fw)) ^ s) - s
    return v & _mask(tw)


def canonical(v, t):
    """ScalarValue::fromStorageBits(kind, bits).storageBits() (scalar.hpp:251-271)."""
    v = np.asarray(v, dtype=U)
    if t == BOOL:
        return ((v & U(0xFF)) != 0).astype(U)
    return v & _mask(8 * SIZE[t])


# =============================================================================================
# bit primitives — bitpack.cpp:11-94
# =============================================================================================
def read_bits(blob: np.ndarray, bit_off, bits: int):
    """readBits over uint8 `blob` for every offset in `bit_off` (LSB-first)."""
    off = np.asarray(bit_off, dtype=U)
    pad = np.concatenate([blob, np.zeros(16, np.uint8)])
    idx = (off >> U(3)).astype(np.int64)
    sh = off & U(7)
    lo = np.zeros(off.shape, U)
    for k in range(8):
        lo |= pad[idx + k].astype(U) << U(8 * k)
    v = lo >> sh
    hi = pad[idx + 8].astype(U)
    need = sh + U(bits)
    extra = np.where(need > U(64), hi << (U(64) - np.where(sh == 0, U(1), sh)), U(0))
    v = v | np.where(sh == 0, U(0), extra)
    return v & _mask(bits)


def write_bits(blob: np.ndarray, bit_off, bits: int, values):
    """writeBits for every (offset, value); fields must not overlap (they never do in a copy)."""
    off = np.asarray(bit_off, dtype=U)
    val = np.asarray(values, dtype=U) & _mask(bits)
    n = blob.size
    maskacc = np.zeros(n + 16, np.uint8)
    valacc = np.zeros(n + 16, np.uint8)
    idx = (off >> U(3)).astype(np.int64)
    sh = (off & U(7)).astype(np.int64)
    fieldmask = np.full(off.shape, _mask(bits), U)
    for k in range(9):
        # bits [8k - sh, 8k - sh + 8) of the field land in byte idx + k
        s = 8 * k - sh
        part_v = np.where(s >= 0, _rshift_var(val, s), _lshift_var(val, -s)) & U(0xFF)
        part_m = np.where(s >= 0, _rshift_var(fieldmask, s), _lshift_var(fieldmask, -s)) & U(0xFF)
        live = part_m != 0
        if not live.any():
            continue
        np.bitwise_or.at(maskacc, idx[live] + k, part_m[live].astype(np.uint8))
        np.bitwise_or.at(valacc, idx[live] + k, part_v[live].astype(np.uint8))
    blob[:] = (blob & ~maskacc[:n]) | (valacc[:n] & maskacc[:n])


def _rshift_var(x, s):
    s = np.asarray(s, dtype=np.int64)
    return np.where(s >= 64, U(0), x >> np.minimum(s, 63).astype(U))


def _lshift_var(x, s):
    s = np.asarray(s, dtype=np.int64)
    return np.where(s >= 64, U(0), x << np.minimum(s, 63).astype(U))


# =============================================================================================
# minifloat codec — bitpack.cpp:51-188
# =============================================================================================
def _rne_shift(x, s):
    """round(x / 2^s), ties to even; s may be an array; s <= 0 shifts left exactly."""
    x = np.asarray(x, dtype=U)
    s = np.broadcast_to(np.asarray(s, dtype=np.int64), x.shape)
    left = _lshift_var(x, np.maximum(-s, 0))
    sc = np.clip(s, 1, 63).astype(U)
    q = x >> sc
    rem = x & ((U(1) << sc) - U(1))
    half = U(1) << (sc - U(1))
    up = (rem > half) | ((rem == half) & ((q & U(1)) != 0))
    right = q + up.astype(U)
    return np.where(s <= 0, left, np.where(s >= 64, U(0), right))


def float_encode(bits64, E: int, M: int):
    """floatEncode((double)bits, E, M) — bitpack.cpp:96-163."""
    b = np.asarray(bits64, dtype=U)
    sign_bit = _shl(b >> U(63), E + M)
    exp_mask = (1 << E) - 1
    inf = sign_bit | U(exp_mask << M)
    raw = ((b >> U(52)) & U(0x7FF)).astype(np.int64)
    frac = b & U((1 << 52) - 1)
    is_nan = (raw == 0x7FF) & (frac != 0)
    is_inf = (raw == 0x7FF) & (frac == 0)
    is_zero = (raw == 0) & (frac == 0)
    sub = (raw == 0) & (frac != 0)
    # bit length of subnormal fractions (exact: frac < 2^52)
    _, bl = np.frexp(np.where(sub, frac, U(1)).astype(np.float64))
    shift = (53 - bl).astype(np.int64)
    frac_n = np.where(sub, _lshift_var(frac, shift), frac | U(1 << 52))
    e2 = np.where(sub, 1 - 1023 - 52 - shift, raw - 1023 - 52)
    bias = (1 << (E - 1)) - 1
    biased = e2 + 52 + bias
    # normal candidate
    q = _rne_shift(frac_n, 52 - M)
    carry = _shr(q, M + 1) != 0
    q = np.where(carry, q >> U(1), q)
    be = biased + carry.astype(np.int64)
    normal = np.where(be >= exp_mask, inf,
                      sign_bit | (_lshift_var(np.maximum(be, 0).astype(U), M)) | (q - U(1 << M)))
    # subnormal candidate
    s = (1 - bias - M) - e2
    qs = _rne_shift(frac_n, s)
    rounded_up = _shr(qs, M) != 0
    smallest = inf if 1 >= exp_mask else sign_bit | U(1 << M)
    subn = np.where(rounded_up, smallest, sign_bit | qs)
    nan_pat = inf if M == 0 else inf | U(1 << (M - 1))
    out = np.where(biased >= 1, normal, subn)
    out = np.where(is_zero, sign_bit, out)
    out = np.where(is_inf, inf, out)
    out = np.where(is_nan, nan_pat, out)
    return out.astype(U)


def float_decode(pattern, E: int, M: int):
    """floatDecode -> double bits — bitpack.cpp:165-188."""
    p = np.asarray(pattern, dtype=U) & _mask(1 + E + M)
    sign = _shr(p, E + M) & U(1)
    expf = (p >> U(M)) & U((1 << E) - 1)
    man = p & _mask(M)
    bias = (1 << (E - 1)) - 1
    special = expf == U((1 << E) - 1)
    e_sub = int(np.clip(1 - bias - M, -5000, 5000))
    e_norm = np.clip(expf.astype(np.int64) - bias - M, -5000, 5000).astype(np.int32)
    with np.errstate(all="ignore"):
        sub_v = np.ldexp(man.astype(np.float64), e_sub)
        norm_v = np.ldexp((U(1 << M) + man).astype(np.float64), e_norm)
    mag = np.where(expf == 0, sub_v, norm_v).view(U)
    mag = np.where(special, np.where(man != 0, U(0x7FF8000000000000), U(0x7FF0000000000000)), mag)
    return mag | (sign << U(63))


# =============================================================================================
# mappings
# =============================================================================================
class Mapping:
    fac = False
    heat = 0

    def __init__(self, schema: Schema, n: int):
        self.schema = schema
        self.n = n

    def is_computed(self, f):
        return False

    def is_fully_physical(self):
        return not any(self.is_computed(f) for f in range(len(self.schema.leaves)))

    def has_mutable_state(self):
        return False

    def idx(self):
        return np.arange(self.n, dtype=U)


class Physical(Mapping):
    """Blob offsets (nr, off[i]) of a physical leaf; read/write move LE bytes."""

    def offsets(self, f):
        raise NotImplementedError

    def read(self, blobs, f):
        l = self.schema.leaves[f]
        nr, off = self.offsets(f)
        b = blobs[nr]
        v = np.zeros(self.n, U)
        o = off.astype(np.int64)
        for k in range(l.size):
            v |= b[o + k].astype(U) << U(8 * k)
        return canonical(v, l.type)  # Bool reads canonicalise (scalar.hpp:259-260)

    def write(self, blobs, f, v):
        l = self.schema.leaves[f]
        nr, off = self.offsets(f)
        o = off.astype(np.int64)
        v = np.asarray(v, dtype=U)
        for k in range(l.size):
            blobs[nr][o + k] = ((v >> U(8 * k)) & U(0xFF)).astype(np.uint8)

    def ranges(self, f):
        nr, off = self.offsets(f)
        return [(nr, off, off + U(self.schema.leaves[f].size))]


class AoS(Physical):  # mappings.cpp:23-50
    def __init__(self, schema, n, aligned):
        super().__init__(schema, n)
        self.aligned = aligned
        self.rec = schema.size_aligned if aligned else schema.size_packed

    def name(self):
        return "aos-aligned" if self.aligned else "aos-packed"

    def blob_sizes(self):
        return [self.n * self.rec]

    def offsets(self, f):
        l = self.schema.leaves[f]
        return 0, self.idx() * U(self.rec) + U(l.offset_aligned if self.aligned else l.offset_packed)


class SoA(Physical):  # mappings.cpp:56-101
    def __init__(self, schema, n, multi):
        super().__init__(schema, n)
        self.multi = multi
        self.base = []
        b = 0
        for l in schema.leaves:
            self.base.append(b)
            b += n * l.size

    def name(self):
        return "soa-mb" if self.multi else "soa-sb"

    def blob_sizes(self):
        if self.multi:
            return [self.n * l.size for l in self.schema.leaves]
        return [self.n * self.schema.size_packed]

    def offsets(self, f):
        s = self.schema.leaves[f].size
        if self.multi:
            return f, self.idx() * U(s)
        return 0, U(self.base[f]) + self.idx() * U(s)


class AoSoA(Physical):  # mappings.cpp:107-148
    def __init__(self, schema, n, lanes):
        super().__init__(schema, n)
        if lanes < 1:
            raise ValueError("lane count must be >= 1")
        self.L = lanes
        self.block = schema.size_packed * lanes

    def name(self):
        return f"aosoa:{self.L}"

    def blob_sizes(self):
        return [(self.n + self.L - 1) // self.L * self.block]

    def offsets(self, f):
        l = self.schema.leaves[f]
        i = self.idx()
        return 0, (i // U(self.L)) * U(self.block) + U(l.offset_packed * self.L) + (i % U(self.L)) * U(l.size)


class One(Physical):  # mappings.cpp:154-175
    def __init__(self, schema, n):
        super().__init__(schema, n)
        if n != 1:
            raise ValueError("one mapping requires a unit array extent")

    def name(self):
        return "one"

    def blob_sizes(self):
        return [self.schema.size_packed]

    def offsets(self, f):
        return 0, np.full(self.n, self.schema.leaves[f].offset_packed, U)


class Null(Mapping):  # computed.cpp:508-531
    def name(self):
        return "null"

    def blob_sizes(self):
        return []

    def is_computed(self, f):
        return True

    def read(self, blobs, f):
        return np.zeros(self.n, U)

    def write(self, blobs, f, v):
        pass

    def ranges(self, f):
        return []


class BitpackInt(Mapping):  # computed.cpp:48-127
    def __init__(self, schema, n, bits):
        super().__init__(schema, n)
        for l in schema.leaves:
            if not _is_int(l.type):
                raise ValueError(f"bitpack-int requires integer leaves, got {NAMES[l.type]}")
            if bits < 1 or bits > 8 * l.size:
                raise ValueError(f"bit count {bits} out of range for leaf")
        self.b = bits

    def name(self):
        return f"bitpack-int:{self.b}"

    def blob_sizes(self):
        return [(self.n * self.b + 31) // 32 * 4 for _ in self.schema.leaves]

    def is_computed(self, f):
        return True

    def read(self, blobs, f):
        t = self.schema.leaves[f].type
        p = read_bits(blobs[f], self.idx() * U(self.b), self.b)
        if _is_signed(t):
            s = U(1 << (self.b - 1))
            p = (p ^ s) - s
        return p & _mask(8 * SIZE[t])

    def write(self, blobs, f, v):
        write_bits(blobs[f], self.idx() * U(self.b), self.b, np.asarray(v, U) & _mask(self.b))

    def ranges(self, f):
        o = self.idx() * U(self.b)
        return [(f, o >> U(3), (o + U(self.b + 7)) >> U(3))]


class BitpackFloat(Mapping):  # computed.cpp:133-222
    def __init__(self, schema, n, E, M):
        super().__init__(schema, n)
        for l in schema.leaves:
            if not _is_float(l.type):
                raise ValueError(f"bitpack-float requires float leaves, got {NAMES[l.type]}")
        if E < 1 or 1 + E + M > 64:
            raise ValueError("float bit layout out of range")
        self.E, self.M = E, M
        self.w = 1 + E + M

    def name(self):
        return f"bitpack-float:{self.E},{self.M}"

    def blob_sizes(self):
        return [(self.n * self.w + 31) // 32 * 4 for _ in self.schema.leaves]

    def is_computed(self, f):
        return True

    def read(self, blobs, f):
        d = float_decode(read_bits(blobs[f], self.idx() * U(self.w), self.w), self.E, self.M)
        return f64_to_f32(d) if self.schema.leaves[f].type == F32 else d

    def write(self, blobs, f, v):
        d = f32_to_f64(v) if self.schema.leaves[f].type == F32 else np.asarray(v, U)
        write_bits(blobs[f], self.idx() * U(self.w), self.w, float_encode(d, self.E, self.M))

    def ranges(self, f):
        o = self.idx() * U(self.w)
        return [(f, o >> U(3), (o + U(self.w + 7)) >> U(3))]


def _rebuild(node, fn):
    if node.kind == "leaf":
        return fn(node)
    if node.kind == "record":
        return Node("record", fields=[(t, _rebuild(c, fn)) for t, c in node.fields])
    return None  # arrays handled by callers


class ChangeType(Mapping):  # computed.cpp:228-399
    def __init__(self, schema, n, changes, make_inner):
        super().__init__(schema, n)
        types = [l.type for l in schema.leaves]
        for sel, target in changes:
            if isinstance(sel, int):
                types = [target if schema.leaves[f].type == sel else t for f, t in enumerate(types)]
            else:
                a, b = schema.leaf_range(sel)
                for f in range(a, b):
                    types[f] = target
        for f, t in enumerate(types):
            lt = schema.leaves[f].type
            ok = lt == t or (_is_float(lt) and _is_float(t)) or (_is_signed(lt) and _is_signed(t)) or (
                _is_unsigned(lt) and _is_unsigned(t))
            if not ok:
                raise ValueError(f"unsupported type change: {NAMES[lt]} -> {NAMES[t]}")
        self.storage = types
        nxt = iter(types)

        def rb(nd):
            if nd.kind == "leaf":
                return Node("leaf", scalar=next(nxt))
            if nd.kind == "record":
                return Node("record", fields=[(t, rb(c)) for t, c in nd.fields])
            els = [rb(nd.element) for _ in range(nd.count)]
            if all(_same(e, els[0]) for e in els):
                return Node("array", count=nd.count, element=els[0])
            return Node("record", fields=[(f"e{k}", e) for k, e in enumerate(els)])

        self.changes = changes
        self.inner = make_inner(Schema(rb(schema.root)), n)

    def name(self):
        parts = []
        for sel, t in self.changes:
            parts.append(f"{NAMES[sel] if isinstance(sel, int) else self.schema.path_of(sel)}={NAMES[t]}")
        return "changetype:" + ",".join(parts) + ":" + self.inner.name()

    def blob_sizes(self):
        return self.inner.blob_sizes()

    def is_computed(self, f):
        return self.storage[f] != self.schema.leaves[f].type or self.inner.is_computed(f)

    def has_mutable_state(self):
        return self.inner.has_mutable_state()

    def read(self, blobs, f):
        return convert(self.inner.read(blobs, f), self.storage[f], self.schema.leaves[f].type)

    def write(self, blobs, f, v):
        self.inner.write(blobs, f, convert(v, self.schema.leaves[f].type, self.storage[f]))

    def ranges(self, f):
        return self.inner.ranges(f)


class Bytesplit(Mapping):  # computed.cpp:405-502
    def __init__(self, schema, n, make_inner):
        super().__init__(schema, n)

        def rb(nd):
            if nd.kind == "leaf":
                return Node("array", count=SIZE[nd.scalar], element=Node("leaf", scalar=U8))
            if nd.kind == "record":
                return Node("record", fields=[(t, rb(c)) for t, c in nd.fields])
            return Node("array", count=nd.count, element=rb(nd.element))

        self.inner = make_inner(Schema(rb(schema.root)), n)
        self.base = [l.offset_packed for l in schema.leaves]

    def name(self):
        return "bytesplit:" + self.inner.name()

    def blob_sizes(self):
        return self.inner.blob_sizes()

    def is_computed(self, f):
        return True

    def has_mutable_state(self):
        return self.inner.has_mutable_state()

    def read(self, blobs, f):
        l = self.schema.leaves[f]
        v = np.zeros(self.n, U)
        for k in range(l.size):
            v |= (self.inner.read(blobs, self.base[f] + k) & U(0xFF)) << U(8 * k)
        return canonical(v, l.type)

    def write(self, blobs, f, v):
        v = np.asarray(v, U)
        for k in range(self.schema.leaves[f].size):
            self.inner.write(blobs, self.base[f] + k, (v >> U(8 * k)) & U(0xFF))

    def ranges(self, f):
        out = []
        for k in range(self.schema.leaves[f].size):
            out += self.inner.ranges(self.base[f] + k)
        return out


class Split(Mapping):  # mappings.cpp:180-389
    def __init__(self, schema, n, selectors, make_a, make_b):
        super().__init__(schema, n)
        self.selectors = selectors

        def sel(coord):
            return any(coord[: len(s)] == tuple(s) for s in selectors)

        def filt(nd, coord, keep):
            if nd.kind == "leaf":
                return nd if sel(tuple(coord)) == keep else None
            if nd.kind == "record":
                fs = [(t, filt(c, coord + [k], keep)) for k, (t, c) in enumerate(nd.fields)]
                fs = [(t, c) for t, c in fs if c is not None]
                return Node("record", fields=fs) if fs else None
            kept = [filt(nd.element, coord + [k], keep) for k in range(nd.count)]
            if all(k is None for k in kept):
                return None
            if kept[0] is not None and all(k is not None and _same(k, kept[0]) for k in kept):
                return Node("array", count=nd.count, element=kept[0])
            return Node("record", fields=[(f"e{k}", c) for k, c in enumerate(kept) if c is not None])

        ra = filt(schema.root, [], True) or Node("record", fields=[])
        rb = filt(schema.root, [], False) or Node("record", fields=[])
        self.a = make_a(Schema(ra), n)
        self.b = make_b(Schema(rb), n)
        self.route = []
        na = nb = 0
        for l in schema.leaves:
            if sel(l.coord):
                self.route.append((True, na))
                na += 1
            else:
                self.route.append((False, nb))
                nb += 1

    def name(self):
        return "split:" + ",".join(self.schema.path_of(s) for s in self.selectors) + ":" + self.a.name() + ":" + \
            self.b.name()

    def blob_sizes(self):
        return self.a.blob_sizes() + self.b.blob_sizes()

    def is_computed(self, f):
        s, k = self.route[f]
        return (self.a if s else self.b).is_computed(k)

    def has_mutable_state(self):
        return self.a.has_mutable_state() or self.b.has_mutable_state()

    def _side(self, blobs, f):
        s, k = self.route[f]
        na = len(self.a.blob_sizes())
        return (self.a, blobs[:na], k, 0) if s else (self.b, blobs[na:], k, na)

    def read(self, blobs, f):
        m, bl, k, _ = self._side(blobs, f)
        return m.read(bl, k)

    def write(self, blobs, f, v):
        m, bl, k, _ = self._side(blobs, f)
        m.write(bl, k, v)

    def ranges(self, f):
        m, _, k, shift = self._side([None] * len(self.blob_sizes()), f)
        return [(nr + shift, lo, hi) for nr, lo, hi in m.ranges(k)]


class FieldAccessCount(Mapping):  # instrument.cpp:24-117
    fac = True

    def __init__(self, inner):
        super().__init__(inner.schema, inner.n)
        self.inner = inner
        L = len(inner.schema.leaves)
        self.reads = np.zeros(L, U)
        self.writes = np.zeros(L, U)

    def name(self):
        return f"field-access-count({self.inner.name()})"

    def blob_sizes(self):
        return self.inner.blob_sizes()

    def is_computed(self, f):
        return self.inner.is_computed(f)

    def has_mutable_state(self):
        return True

    def read(self, blobs, f):
        v = self.inner.read(blobs, f)
        self.reads[f] += U(self.n)
        return v

    def write(self, blobs, f, v):
        self.inner.write(blobs, f, v)
        self.writes[f] += U(self.n)

    def ranges(self, f):
        return self.inner.ranges(f)


class Heatmap(Mapping):  # instrument.cpp:123-229
    def __init__(self, inner, g):
        super().__init__(inner.schema, inner.n)
        if g < 1:
            raise ValueError("heatmap granularity must be >= 1")
        self.inner = inner
        self.g = g
        self.blocks = [np.zeros((s + g - 1) // g, U) for s in inner.blob_sizes()]

    def name(self):
        return f"heatmap:{self.g}({self.inner.name()})"

    def blob_sizes(self):
        return self.inner.blob_sizes()

    def is_computed(self, f):
        return self.inner.is_computed(f)

    def has_mutable_state(self):
        return True

    def _touch(self, f):
        for nr, lo, hi in self.inner.ranges(f):
            lo = np.asarray(lo, U)
            hi = np.asarray(hi, U)
            live = lo < hi
            first = (lo[live] // U(self.g)).astype(np.int64)
            last = ((hi[live] - U(1)) // U(self.g)).astype(np.int64)
            span = int((last - first).max()) + 1 if first.size else 0
            for d in range(span):
                m = first + d <= last
                np.add.at(self.blocks[nr], first[m] + d, U(1))

    def read(self, blobs, f):
        v = self.inner.read(blobs, f)
        self._touch(f)
        return v

    def write(self, blobs, f, v):
        self.inner.write(blobs, f, v)
        self._touch(f)

    def ranges(self, f):
        return self.inner.ranges(f)


# ---- layout grammar — layout_spec.cpp:37-167 --------------------------------------------------
def parse_layout(text: str, schema: Schema, n: int) -> Mapping:
    if text.startswith("field-access-count(") and text.endswith(")"):
        return FieldAccessCount(parse_layout(text[19:-1], schema, n))
    m = re.match(r"heatmap:(\d+)\((.*)\)$", text)
    if m:
        return Heatmap(parse_layout(m.group(2), schema, n), int(m.group(1)))
    toks = text.split(":")
    pos = 0

    def nxt():
        nonlocal pos
        if pos >= len(toks):
            raise ValueError("missing layout token")
        pos += 1
        return toks[pos - 1]

    def mapping(s, n):
        form = nxt()
        if form == "aos-packed":
            return AoS(s, n, False)
        if form == "aos-aligned":
            return AoS(s, n, True)
        if form == "soa-sb":
            return SoA(s, n, False)
        if form == "soa-mb":
            return SoA(s, n, True)
        if form == "one":
            return One(s, n)
        if form == "null":
            return Null(s, n)
        if form == "aosoa":
            return AoSoA(s, n, int(nxt()))
        if form == "split":
            sels = [s.coord_of(p) for p in nxt().split(",")]
            return Split(s, n, sels, mapping, mapping)
        if form == "bitpack-int":
            return BitpackInt(s, n, int(nxt()))
        if form == "bitpack-float":
            e, m_ = nxt().split(",")
            return BitpackFloat(s, n, int(e), int(m_))
        if form == "changetype":
            changes = []
            for entry in nxt().split(","):
                sel, tgt = entry.split("=")
                selector = NAMES.index(sel) if sel in NAMES else s.coord_of(sel)
                changes.append((selector, NAMES.index(tgt)))
            inner = mapping if pos < len(toks) else (lambda s2, n2: AoS(s2, n2, False))
            return ChangeType(s, n, changes, inner)
        if form == "bytesplit":
            if pos >= len(toks):
                raise ValueError("missing inner layout for bytesplit")
            return Bytesplit(s, n, mapping)
        raise ValueError(f"unknown layout: '{form}'")

    m = mapping(schema, n)
    if pos != len(toks):
        raise ValueError(f"trailing layout tokens: '{toks[pos]}'")
    return m


def make(schema_text: str, extents_text: str, layout: str, dyn=(), wrap=0, gran=0) -> Mapping:
    s = Schema.parse(schema_text)
    m = parse_layout(layout, s, parse_extents(extents_text, dyn))
    if wrap & 1:
        m = FieldAccessCount(m)
    if wrap & 2:
        m = Heatmap(m, gran)
    return m


def zero_blobs(m: Mapping):
    return [np.zeros(s, np.uint8) for s in m.blob_sizes()]


def write_all(m: Mapping, blobs, values):
    """View::write of values[i, f] (storage bits) for every (i, f)."""
    for f, l in enumerate(m.schema.leaves):
        m.write(blobs, f, canonical(values[:, f], l.type))


def read_all(m: Mapping, blobs):
    return np.stack([m.read(blobs, f) for f in range(len(m.schema.leaves))], axis=1) if m.schema.leaves else \
        np.zeros((m.n, 0), U)


def _fac_of(m):
    while m is not None:
        if isinstance(m, FieldAccessCount):
            return m
        m = getattr(m, "inner", None)
    return None


def _heat_of(m):
    while m is not None:
        if isinstance(m, Heatmap):
            return m
        m = getattr(m, "inner", None)
    return None


def copy_view(src: Mapping, src_blobs, dst: Mapping, dst_blobs):
    """copyView — view.cpp:168-189.  dst_blobs updated in place."""
    if not (src.schema == dst.schema) or src.n != dst.n:
        raise ValueError("incompatible views")
    same = src.name() == dst.name() and not src.has_mutable_state() and not dst.has_mutable_state() and \
        src.is_fully_physical() and dst.is_fully_physical()
    if same:
        for nr, b in enumerate(src_blobs):
            dst_blobs[nr][:] = b
        return
    for f in range(len(src.schema.leaves)):
        dst.write(dst_blobs, f, src.read(src_blobs, f))


def counters(m: Mapping):
    """[reads..., writes..., heat blocks...] in the layout of lam_copy_host's counter arrays."""
    out = []
    fac = _fac_of(m)
    h = _heat_of(m)
    if fac is None and h is None:
        return None
    if fac is not None:
        out += [fac.reads, fac.writes]
    if h is not None:
        out += h.blocks
    return np.concatenate(out) if out else np.zeros(0, U)


# =============================================================================================
# n-body — tools/nbody/kernel.hpp:15-41, steps.hpp:13-118, runner.cpp:30-72
# =============================================================================================
class MT19937_64:
    """std::mt19937_64 (the generator drawInitValues uses, runner.cpp:30-43)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def nbody_init_values(seed: int, n: int):
    """drawInitValues: (posX, posY, posZ, mass) doubles per particle, uniform in [0,1)."""
    g = MT19937_64(seed)
    raw = np.array([g() >> 11 for _ in range(4 * n)], dtype=np.float64) * 2.0 ** -53
    return raw.reshape(n, 4)


EPS2 = 0.01
DT = 0.0001


def nbody_update(pos, vel, mass, dtype=np.float32):
    """updateStep: per i, j = 0..n-1 in order, reference operation order, no FMA."""
    T = dtype
    px, py, pz = (pos[:, k].astype(T) for k in range(3))
    vx, vy, vz = (vel[:, k].astype(T).copy() for k in range(3))
    m = mass.astype(T)
    eps2, dt, one = T(EPS2), T(DT), T(1.0)
    with np.errstate(all="ignore"):
        for j in range(px.size):
            dx = px - px[j]
            dy = py - py[j]
            dz = pz - pz[j]
            d2 = ((eps2 + dx * dx) + dy * dy) + dz * dz
            d6 = (d2 * d2) * d2
            inv = one / np.sqrt(d6)
            sts = (m[j] * inv) * dt
            vx = vx + dx * sts
            vy = vy + dy * sts
            vz = vz + dz * sts
    return np.stack([vx, vy, vz], axis=1)


def nbody_move(pos, vel, dtype=np.float32):
    T = dtype
    return (pos.astype(T) + vel.astype(T) * T(DT)).astype(T)


def nbody_run(n, steps, seed=42, dtype=np.float32):
    """Whole benchmark body; returns (pos, vel, mass, checksum)."""
    init = nbody_init_values(seed, n)
    pos = init[:, :3].astype(dtype)
    mass = init[:, 3].astype(dtype)
    vel = np.zeros((n, 3), dtype)
    for _ in range(steps):
        vel = nbody_update(pos, vel, mass, dtype)
        pos = nbody_move(pos, vel, dtype)
    return pos, vel, mass, checksum(pos)


def checksum(pos):
    """checksumView: Σ x,y,z in double, index order (sequential accumulate, not pairwise)."""
    return float(np.cumsum(pos.astype(np.float64).reshape(-1))[-1]) if pos.size else 0.0


# ---- instrumented n-body: the runner's traced counters (runner.cpp:344-436) -------------------
NBODY_SCHEMA = {
    False: "Record{Pos:Record{x:f32,y:f32,z:f32},Vel:Record{x:f32,y:f32,z:f32},Mass:f32}",
    True: "Record{Pos:Record{x:f64,y:f64,z:f64},Vel:Record{x:f64,y:f64,z:f64},Mass:f64}",
}


def nbody_access_multiplicity(n: int, phase: str, ib: int = 0, ie: int | None = None):
    """Accesses per (element, leaf) of one step through the funnel accessor (steps.hpp:13-118).

    update, for i in [ib, ie): read the 7 leaves of i (loadLeafSimd), read Pos.{x,y,z} and Mass
    of every j (acc.get<>), write Vel.{x,y,z} of i (storeLeafSimd).  move, for i: read Pos and
    Vel, write Pos.  Returns (reads[7][n], writes[7][n]) as uint64 arrays.
    """
    ie = n if ie is None else ie
    own = np.zeros(n, U)
    own[ib:ie] = 1
    cnt = U(ie - ib)
    reads = np.zeros((7, n), U)
    writes = np.zeros((7, n), U)
    if phase == "update":
        for f in (0, 1, 2, 6):
            reads[f] = cnt + own
        for f in (3, 4, 5):
            reads[f] = own
            writes[f] = own
    else:
        for f in (0, 1, 2):
            reads[f] = own
            writes[f] = own
        for f in (3, 4, 5):
            reads[f] = own
    return reads, writes


def nbody_trace(layout: str, n: int, steps: int, f64: bool = False, gran: int = 0):
    """fields_{update,move} and heatmap_{update,move} of `lamina-nbody --trace-fields --heatmap g`.

    Counters are sums over accesses, so each phase is the per-(element, leaf) multiplicity of
    nbody_access_multiplicity times the leaf's access ranges (Mapping::accessRanges), summed
    over the steps.  Returns {"update": (reads[7], writes[7], blocks or None), "move": ...}.
    """
    base = parse_layout(layout, Schema.parse(NBODY_SCHEMA[f64]), n)
    out = {}
    for phase in ("update", "move"):
        reads, writes = nbody_access_multiplicity(n, phase)
        r = reads.sum(axis=1) * U(steps)
        w = writes.sum(axis=1) * U(steps)
        blocks = None
        if gran:
            blocks = [np.zeros((s + gran - 1) // gran, U) for s in base.blob_sizes()]
            for f in range(7):
                m = (reads[f] + writes[f]) * U(steps)
                for nr, lo, hi in base.ranges(f):
                    lo = np.asarray(lo, U)
                    hi = np.asarray(hi, U)
                    live = (lo < hi) & (m > 0)
                    first = (lo[live] // U(gran)).astype(np.int64)
                    last = ((hi[live] - U(1)) // U(gran)).astype(np.int64)
                    wt = m[live]
                    span = int((last - first).max()) + 1 if first.size else 0
                    for d in range(span):
                        k = first + d <= last
                        np.add.at(blocks[nr], first[k] + d, wt[k])
        out[phase] = (r, w, blocks)
    return out

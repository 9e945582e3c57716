// Device-side value semantics of the reference, restated for sm_100a:
//   * values travel as the storage bits of their scalar kind, zero-extended to 64 bits
//     (ScalarValue::storageBits, scalar.hpp:231-246);
//   * type conversion = ScalarValue::convertTo (scalar.hpp:295-306) with x86 SSE NaN rules
//     (cvtsd2ss / cvtss2sd keep sign and top payload bits and set the quiet bit) — the
//     reference is compiled for x86-64 without -march, so those are its semantics;
//   * minifloat codec = floatEncode / floatDecode (bitpack.cpp:96-188), integer-exact;
//   * bit streams = LSB-first little-endian u32 words (bitpack.cpp:11-47).
// All arithmetic is integer or correctly-rounded IEEE (no fast-math, no FTZ).
#pragma once

#include "lam_plan.h"

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define LAM_DEV __device__ __forceinline__

namespace lamd
{
    enum : int
    {
        I8 = 0,
        I16,
        I32,
        I64,
        U8,
        U16,
        U32,
        U64,
        F32,
        F64,
        BOOL
    };

    LAM_DEV uint32_t scalar_size(int t)
    {
        // i8 i16 i32 i64 u8 u16 u32 u64 f32 f64 bool
        return (0x18484218421ull >> (4 * t)) & 0xF;
    }
    LAM_DEV bool is_signed(int t)
    {
        return t <= I64;
    }
    LAM_DEV uint64_t low_mask(uint32_t bits)
    {
        return bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
    }

    // ---- conversions (ScalarValue::convertTo) -----------------------------------------
    LAM_DEV uint64_t f32_to_f64_bits(uint32_t b)
    {
        // branch-free: the NaN pattern (quiet bit set, payload kept) is selected, not branched to
        const uint64_t nan = (uint64_t(b >> 31) << 63) | 0x7FF8000000000000ull | (uint64_t(b & 0x007FFFFFu) << 29);
        const uint64_t cvt = static_cast<uint64_t>(__double_as_longlong(static_cast<double>(__uint_as_float(b))));
        return (b & 0x7FFFFFFFu) > 0x7F800000u ? nan : cvt;
    }
    LAM_DEV uint32_t f64_to_f32_bits(uint64_t b)
    {
        if((b & 0x7FF0000000000000ull) == 0x7FF0000000000000ull && (b & 0x000FFFFFFFFFFFFFull) != 0ull)
            return (uint32_t(b >> 63) << 31) | 0x7FC00000u | uint32_t((b >> 29) & 0x003FFFFFu);
        return __float_as_uint(__double2float_rn(__longlong_as_double(static_cast<long long>(b))));
    }

    LAM_DEV uint64_t convert_value(uint64_t v, int from, int to)
    {
        if(from == to)
            return v;
        if(from == F32 && to == F64)
            return f32_to_f64_bits(static_cast<uint32_t>(v));
        if(from == F64 && to == F32)
            return f64_to_f32_bits(v);
        const uint32_t fw = 8 * scalar_size(from);
        const uint32_t tw = 8 * scalar_size(to);
        if(is_signed(from) && fw < 64)
        {
            // sign-extend from the source width, keep the low bits of the target width
            const uint64_t s = 1ull << (fw - 1);
            v = ((v & low_mask(fw)) ^ s) - s;
        }
        return v & low_mask(tw);
    }

    // ---- minifloat codec (bitpack.cpp:51-188) ------------------------------------------
    LAM_DEV uint64_t rne_shift(uint64_t x, int s)
    {
        if(s <= 0)
            return x << static_cast<unsigned>(-s);
        if(s >= 64)
            return 0;
        const uint64_t q = x >> s;
        const uint64_t rem = x & low_mask(static_cast<uint32_t>(s));
        const uint64_t half = 1ull << (s - 1);
        return (rem > half || (rem == half && (q & 1ull))) ? q + 1 : q;
    }

    // floatEncode(value, E, M) on the double's bit pattern
    static __device__ __noinline__ uint64_t float_encode(uint64_t bits64, uint32_t E, uint32_t M)
    {
        const uint64_t signBit = (bits64 >> 63) << (E + M);
        const uint64_t expMask = low_mask(E);
        const uint64_t inf = signBit | (expMask << M);
        const uint32_t rawExp = static_cast<uint32_t>((bits64 >> 52) & 0x7FF);
        uint64_t frac = bits64 & low_mask(52);
        if(rawExp == 0x7FF)
        {
            if(frac == 0 || M == 0)
                return inf;
            return inf | (1ull << (M - 1));
        }
        if(rawExp == 0 && frac == 0)
            return signBit;
        int64_t e2;
        if(rawExp == 0)
        {
            const int shift = 52 - (63 - __clzll(static_cast<long long>(frac)));
            frac <<= shift;
            e2 = 1 - 1023 - 52 - shift;
        }
        else
        {
            frac |= 1ull << 52;
            e2 = static_cast<int64_t>(rawExp) - 1023 - 52;
        }
        const int64_t bias = (int64_t(1) << (E - 1)) - 1;
        int64_t biasedExp = e2 + 52 + bias;
        const int64_t maxExpField = static_cast<int64_t>(expMask);
        if(biasedExp >= 1)
        {
            uint64_t q = rne_shift(frac, 52 - static_cast<int>(M));
            if((q >> (M + 1)) != 0)
            {
                q >>= 1;
                ++biasedExp;
            }
            if(biasedExp >= maxExpField)
                return inf;
            return signBit | (static_cast<uint64_t>(biasedExp) << M) | (q - (1ull << M));
        }
        const int64_t shift = (1 - bias - static_cast<int64_t>(M)) - e2;
        const uint64_t q = rne_shift(frac, shift > 64 ? 64 : static_cast<int>(shift));
        if((q >> M) != 0)
        {
            if(1 >= maxExpField)
                return inf;
            return signBit | (1ull << M);
        }
        return signBit | q;
    }

    // floatDecode(pattern, E, M) -> double bit pattern
    static __device__ __noinline__ uint64_t float_decode(uint64_t p, uint32_t E, uint32_t M)
    {
        p &= low_mask(1 + E + M);
        const uint64_t sign = (p >> (E + M)) & 1ull;
        const uint64_t expField = (p >> M) & low_mask(E);
        const uint64_t man = p & low_mask(M);
        const int64_t bias = (int64_t(1) << (E - 1)) - 1;
        auto clampExp = [](int64_t e) { return static_cast<int>(e < -5000 ? -5000 : (e > 5000 ? 5000 : e)); };
        uint64_t mag;
        if(expField == low_mask(E))
            mag = man != 0 ? 0x7FF8000000000000ull : 0x7FF0000000000000ull;
        else if(expField == 0)
            mag = static_cast<uint64_t>(__double_as_longlong(
                ldexp(__ull2double_rn(man), clampExp(1 - bias - static_cast<int64_t>(M)))));
        else
            mag = static_cast<uint64_t>(__double_as_longlong(ldexp(
                __ull2double_rn((1ull << M) + man),
                clampExp(static_cast<int64_t>(expField) - bias - static_cast<int64_t>(M)))));
        return mag | (sign << 63);
    }

    // RNE of x / 2^s for 0 < s < 32 (rneShift, bitpack.cpp:57-69, on 32-bit significands)
    LAM_DEV uint32_t rne32(uint32_t x, uint32_t s)
    {
        const uint32_t q = x >> s;
        const uint32_t rem = x & ((1u << s) - 1u);
        const uint32_t half = 1u << (s - 1);
        return (rem > half || (rem == half && (q & 1u))) ? q + 1 : q;
    }

    // floatEncode((double)f, E, M) for an f32 input f, in 32-bit integer arithmetic.  The f32
    // significand has 24 bits, so the reference's RNE of the 53-bit double significand (whose
    // low 29 bits are zero) by 52 - M is the RNE of the 24-bit one by 23 - M; M > 23 shifts
    // left exactly.  Every E >= 1 and width 1 + E + M <= 64; checked against float_encode on
    // all 2^32 inputs for a set of formats (tests/test_gpu_codec.py).
    LAM_DEV uint32_t float_encode_f32_small(uint32_t b, uint32_t E, uint32_t M);
    LAM_DEV uint64_t float_encode_f32(uint32_t b, uint32_t E, uint32_t M)
    {
        if(E <= 8 && M <= 23)
            return float_encode_f32_small(b, E, M);
        const uint64_t signBit = uint64_t(b >> 31) << (E + M);
        const uint64_t expMask = low_mask(E);
        const uint64_t inf = signBit | (expMask << M);
        const uint32_t a = b & 0x7FFFFFFFu;
        if(a >= 0x7F800000u)
            return (a == 0x7F800000u || M == 0) ? inf : (inf | (1ull << (M - 1)));
        if(a == 0)
            return signBit;
        uint32_t frac = a & 0x7FFFFFu;
        int e2; // value = frac * 2^e2, frac in [2^23, 2^24)
        if((a >> 23) == 0)
        {
            const int sh = __clz(frac) - 8;
            frac <<= sh;
            e2 = 1 - 127 - 23 - sh;
        }
        else
        {
            frac |= 1u << 23;
            e2 = static_cast<int>(a >> 23) - 127 - 23;
        }
        const int64_t bias = (int64_t(1) << (E - 1)) - 1;
        int64_t biasedExp = e2 + 23 + bias;
        const int64_t maxExpField = static_cast<int64_t>(expMask);
        if(biasedExp >= 1)
        {
            uint64_t q = M <= 23 ? (M == 23 ? frac : rne32(frac, 23 - M)) : (uint64_t(frac) << (M - 23));
            if((q >> (M + 1)) != 0)
            {
                q >>= 1;
                ++biasedExp;
            }
            if(biasedExp >= maxExpField)
                return inf;
            return signBit | (static_cast<uint64_t>(biasedExp) << M) | (q - (1ull << M));
        }
        const int64_t shift = (1 - bias - static_cast<int64_t>(M)) - e2;
        const uint64_t q = shift <= 0 ? (uint64_t(frac) << (-shift)) : (shift >= 32 ? 0 : rne32(frac, uint32_t(shift)));
        if((q >> M) != 0)
        {
            if(1 >= maxExpField)
                return inf;
            return signBit | (1ull << M);
        }
        return signBit | q;
    }

    // The same for E <= 8, M <= 23 with the rounding done the hardware way: a normal result is
    // the f32 pattern rounded to M mantissa bits by the integer RNE (a + half - 1 + lsb) >> (23 - M)
    // (a carry moves into the exponent, as the reference's renormalisation), re-biased; a
    // subnormal result is RNE(|x| * 2^(bias - 1 + M)) by cvt.rni (the scaling by powers of two is
    // exact).  ~12 instructions on the normal path instead of the 24-bit normalise-and-shift.
    LAM_DEV uint32_t float_encode_f32_small(uint32_t b, uint32_t E, uint32_t M)
    {
        const uint32_t sign = (b >> 31) << (E + M);
        const uint32_t maxExp = (1u << E) - 1u;
        const uint32_t inf = sign | (maxExp << M);
        const uint32_t a = b & 0x7FFFFFFFu;
        if(a >= 0x7F800000u)
            return (a == 0x7F800000u || M == 0) ? inf : (inf | (1u << (M - 1)));
        const int bias = (1 << (E - 1)) - 1;
        if(static_cast<int>(a >> 23) - 127 + bias >= 1)
        {
            // the parity for ties-to-even is the LSB of the rounded significand: mantissa bit
            // 23 - M, or -- at M = 0, where only the implicit 1 remains -- always odd
            const uint32_t sh = 23 - M;
            const uint32_t lsb = M ? (a >> sh) & 1u : 1u;
            const uint32_t r = sh ? a + ((1u << (sh - 1)) - 1u) + lsb : a;
            const int e = static_cast<int>(r >> 23) - 127 + bias;
            if(e >= static_cast<int>(maxExp))
                return inf;
            return sign | (static_cast<uint32_t>(e) << M) | ((r >> sh) & ((1u << M) - 1u));
        }
        // |x| < 2^(1 - bias): scale by 2^M, then by 2^(bias - 1), round to an integer (only a
        // halving at E = 1 can round, and only far below 1/2, where q is 0 either way)
        const float t = __fmul_rn(__fmul_rn(__uint_as_float(a), __uint_as_float(static_cast<uint32_t>(M + 127) << 23)),
                                  __uint_as_float(static_cast<uint32_t>(bias - 1 + 127) << 23));
        const uint32_t q = __float2uint_rn(t);
        if(q >> M)
            return 1 >= maxExp ? inf : (sign | (1u << M));
        return sign | q;
    }

    // (float)floatDecode(p, E, M) (bitpack.cpp:165-188, scalar.hpp:151-152) for E <= 8, M <= 23:
    // every such minifloat is exactly an f32, so the bits are assembled directly; NaN -> the
    // f32 quiet NaN with the sign, as the double quiet_NaN converts
    LAM_DEV uint32_t float_decode_f32(uint32_t p, uint32_t E, uint32_t M)
    {
        const uint32_t sign = ((p >> (E + M)) & 1u) << 31;
        const uint32_t allOnes = (1u << E) - 1u;
        const uint32_t ef = (p >> M) & allOnes;
        const uint32_t man = p & ((1u << M) - 1u);
        const int bias = (1 << (E - 1)) - 1;
        if(ef == allOnes)
            return sign | (man ? 0x7FC00000u : 0x7F800000u);
        if(ef == 0)
        {
            if(man == 0)
                return sign;
            const int top = 31 - __clz(man);              // man in [2^top, 2^(top + 1))
            const int e = top + 1 - bias - static_cast<int>(M); // exponent of the leading bit
            if(e >= -126)
                return sign | (static_cast<uint32_t>(e + 127) << 23) | ((man << (23 - top)) & 0x7FFFFFu);
            return sign | (man << (1 - bias - static_cast<int>(M) + 149)); // f32 subnormal, units of 2^-149
        }
        return sign | (static_cast<uint32_t>(static_cast<int>(ef) - bias + 127) << 23) | (man << (23 - M));
    }

    // The two functions above without branches, for the bit-packing kernels' hot loops
    // (float_encode_f32_small took ~43 instructions per value with its BRA/BSSY pairs and
    // kept k_pack32<8,3> ALU-bound at 36% of HBM).  Per-format constants are built once per
    // thread by f32_codec; the results are bit-identical to the branchy functions (checked
    // exhaustively over all 2^32 f32 inputs, tests/test_gpu_codec.py).
    struct F32Codec
    {
        uint32_t sh, half, lsbAnd, odd, C1, minN, ovf, inf, nan, sgnSh, sgnBit; // encode
        float s1, s2;
        uint32_t mag, C2, subMax; // decode
        float ds, dsOff;
    };

    LAM_DEV F32Codec f32_codec(uint32_t E, uint32_t M)
    {
        F32Codec c;
        const int bias = (1 << (E - 1)) - 1;
        const uint32_t maxExp = (1u << E) - 1u;
        c.sh = 23 - M;
        c.half = c.sh ? (1u << (c.sh - 1)) - 1u : 0u;
        c.lsbAnd = (c.sh && M) ? 1u : 0u;
        c.odd = M == 0 ? 1u : 0u;
        c.C1 = static_cast<uint32_t>(bias - 127) << M;
        c.minN = static_cast<uint32_t>(127 - bias + 1) << 23;
        c.ovf = static_cast<uint32_t>(static_cast<int>(maxExp) - bias + 127) << 23;
        c.inf = maxExp << M;
        c.nan = M ? (c.inf | (1u << (M - 1))) : c.inf;
        c.sgnSh = 31 - (E + M);
        c.sgnBit = 1u << (E + M);
        c.s1 = __uint_as_float(static_cast<uint32_t>(M + 127) << 23);
        c.s2 = __uint_as_float(static_cast<uint32_t>(bias - 1 + 127) << 23);
        c.mag = (1u << (E + M)) - 1u;
        c.C2 = static_cast<uint32_t>(127 - bias) << 23;
        c.subMax = 1u << M; // magnitudes below: exponent field 0
        // subnormal: man * 2^(1 - bias - M) = (float(2^23 + man) - 2^23) * 2^(1 - bias - M), one FFMA
        const int k = 1 - bias - static_cast<int>(M);
        c.ds = k >= -126 ? __uint_as_float(static_cast<uint32_t>(k + 127) << 23) : __uint_as_float(1u << (k + 149));
        const int k2 = k + 23;
        c.dsOff = -(k2 >= -126 ? __uint_as_float(static_cast<uint32_t>(k2 + 127) << 23) : __uint_as_float(1u << (k2 + 149)));
        return c;
    }

    LAM_DEV uint32_t f32_encode_bf(const F32Codec& c, uint32_t b)
    {
        const uint32_t a = b & 0x7FFFFFFFu;
        const uint32_t r = a + c.half + (((a >> c.sh) & c.lsbAnd) | c.odd);
        const uint32_t nrm = (r >> c.sh) + c.C1;
        // |x| < 2^(1 - bias): RNE(|x| * 2^(M + bias - 1)) by the 2^23 magic add (the product is < 2^M <= 2^23)
        const float t = __fmul_rn(__uint_as_float(a), c.s1);
        const uint32_t q = __float_as_uint(__fmaf_rn(t, c.s2, 8388608.0f)) - 0x4B000000u;
        uint32_t res = a >= c.minN ? nrm : q;
        res = r >= c.ovf ? c.inf : res;
        res = a > 0x7F800000u ? c.nan : res;
        return res | ((b >> c.sgnSh) & c.sgnBit);
    }

    LAM_DEV uint32_t f32_decode_bf(const F32Codec& c, uint32_t p)
    {
        const uint32_t mag = p & c.mag;
        const uint32_t sign = (p << c.sgnSh) & 0x80000000u;
        const uint32_t nrm = (mag << c.sh) + c.C2;
        const uint32_t sub = __float_as_uint(__fmaf_rn(__uint_as_float(mag | 0x4B000000u), c.ds, c.dsOff));
        uint32_t res = mag < c.subMax ? sub : nrm;
        res = mag >= c.inf ? (mag > c.inf ? 0x7FC00000u : 0x7F800000u) : res;
        return sign | res;
    }

    // Fast f32 encoders, equal to floatEncode((double)f, E, M) on every f32 input
    // (checked exhaustively against the reference on the GPU, tests/test_gpu_codec.py).
    LAM_DEV uint32_t encode_e8m10_f32(uint32_t b)
    {
        const uint32_t s = (b >> 31) << 18;
        const uint32_t a = b & 0x7FFFFFFFu;
        // e8m10 is TF32: cvt.rn.tf32.f32 rounds to nearest-even into the top 19 bits, overflow
        // to Inf -- equal to the integer RNE (a + 0xFFF + lsb) >> 13 on every non-NaN input
        // (exhaustive, tools/scratch/tf32.cu); NaN keeps the reference's canonical quiet pattern
        uint32_t t;
        asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(t) : "f"(__uint_as_float(b)));
        return a > 0x7F800000u ? (s | 0x3FE00u) : (t >> 13); // NaN: exp all ones | quiet bit
    }

    LAM_DEV uint32_t encode_e5m10_f32(uint32_t b)
    {
        const uint32_t a = b & 0x7FFFFFFFu;
        if(a > 0x7F800000u)
            return ((b >> 31) << 15) | 0x7E00u;
        return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(__uint_as_float(b))));
    }

    // ---- raw byte access ----------------------------------------------------------------
    LAM_DEV uint64_t load_bytes(const uint8_t* p, uint32_t size, bool aligned)
    {
        if(aligned)
        {
            switch(size)
            {
            case 1:
                return *p;
            case 2:
                return *reinterpret_cast<const uint16_t*>(p);
            case 4:
                return *reinterpret_cast<const uint32_t*>(p);
            default:
                return *reinterpret_cast<const unsigned long long*>(p);
            }
        }
        uint64_t v = 0;
        for(uint32_t k = 0; k < size; ++k)
            v |= uint64_t(p[k]) << (8 * k);
        return v;
    }

    LAM_DEV void store_bytes(uint8_t* p, uint32_t size, bool aligned, uint64_t v)
    {
        if(aligned)
        {
            switch(size)
            {
            case 1:
                *p = static_cast<uint8_t>(v);
                return;
            case 2:
                *reinterpret_cast<uint16_t*>(p) = static_cast<uint16_t>(v);
                return;
            case 4:
                *reinterpret_cast<uint32_t*>(p) = static_cast<uint32_t>(v);
                return;
            default:
                *reinterpret_cast<unsigned long long*>(p) = v;
                return;
            }
        }
        for(uint32_t k = 0; k < size; ++k)
            p[k] = static_cast<uint8_t>(v >> (8 * k));
    }

    // ---- bit streams (readBits/writeBits, bitpack.cpp:11-47) -----------------------------
    LAM_DEV uint64_t read_bits(const uint32_t* w, uint64_t bitOff, uint32_t bits)
    {
        const uint64_t wi = bitOff >> 5;
        const uint32_t sh = static_cast<uint32_t>(bitOff & 31);
        const uint32_t need = sh + bits; // 1..95
        uint64_t lo = w[wi];
        if(need > 32)
            lo |= uint64_t(w[wi + 1]) << 32;
        uint64_t v = lo >> sh;
        if(need > 64)
            v |= uint64_t(w[wi + 2]) << (64 - sh);
        return v & low_mask(bits);
    }

    // race-free against other threads writing other fields of the same words
    LAM_DEV void write_bits_atomic(uint32_t* w, uint64_t bitOff, uint32_t bits, uint64_t v)
    {
        uint64_t wi = bitOff >> 5;
        uint32_t sh = static_cast<uint32_t>(bitOff & 31);
        uint32_t left = bits;
        v &= low_mask(bits);
        while(left > 0)
        {
            const uint32_t take = (32 - sh) < left ? (32 - sh) : left;
            const uint32_t mask = static_cast<uint32_t>(low_mask(take)) << sh;
            const uint32_t chunk = static_cast<uint32_t>(v & low_mask(take)) << sh;
            if(mask == 0xFFFFFFFFu)
                w[wi] = chunk;
            else
            {
                atomicAnd(&w[wi], ~mask);
                atomicOr(&w[wi], chunk);
            }
            v >>= take;
            left -= take;
            sh = 0;
            ++wi;
        }
    }

    // ---- plan interpreter ----------------------------------------------------------------
    struct ViewCtx
    {
        const lamp_node* nodes;
        const lamp_stream* streams;
        uint8_t* const* sptr;
        unsigned long long* heat;
        const uint64_t* heatOff;
        uint64_t gran;
        unsigned long long heatMul; // accesses one touch stands for (1 except in n-body accounting)
    };

    LAM_DEV ViewCtx make_ctx(const lamp_view* v)
    {
        ViewCtx c;
        c.nodes = v->nodes;
        c.streams = v->streams;
        c.sptr = v->stream_ptr;
        c.heat = v->heat ? v->heat_counters : nullptr;
        c.heatOff = v->heat_offset;
        c.gran = v->heat_gran;
        c.heatMul = 1;
        return c;
    }

    LAM_DEV uint64_t block_rel(const lamp_stream& st, uint64_t i, uint32_t inblock, uint32_t ls)
    {
        if(st.lanes == 1)
            return i * st.block_stride + inblock;
        uint64_t blk, lane;
        if(st.lane_shift != 0xFFFFFFFFu)
        {
            blk = i >> st.lane_shift;
            lane = i & (st.lanes - 1);
        }
        else
        {
            blk = i / st.lanes;
            lane = i - blk * st.lanes;
        }
        return blk * st.block_stride + inblock + lane * ls;
    }

    // Heatmap touch of byte range [begin, end) of blob nr (instrument.cpp:163-176).  Lanes that
    // hit the same first block (neighbouring elements of one leaf, g >= element stride) are
    // combined into one atomic by the lowest such lane (opportunistic warp aggregation).
    LAM_DEV void heat_touch(const ViewCtx& v, uint32_t nr, uint64_t begin, uint64_t end)
    {
        if(begin >= end)
            return;
        const uint64_t first = begin / v.gran, last = (end - 1) / v.gran;
        const unsigned long long idx = v.heatOff[nr] + first;
        const unsigned peers = __match_any_sync(__activemask(), idx);
        if((threadIdx.x & 31) == static_cast<unsigned>(__ffs(peers) - 1))
            atomicAdd(&v.heat[idx], v.heatMul * static_cast<unsigned long long>(__popc(peers)));
        for(uint64_t b = first + 1; b <= last; ++b)
            atomicAdd(&v.heat[v.heatOff[nr] + b], v.heatMul);
    }

    template<int D>
    __device__ __noinline__ uint64_t read_node(const ViewCtx& v, uint32_t n, uint64_t i)
    {
        const lamp_node nd = v.nodes[n];
        switch(nd.kind)
        {
        case LAMP_PHYS:
        {
            const lamp_stream st = v.streams[nd.stream];
            const uint64_t rel = block_rel(st, i, nd.a, nd.b);
            const uint32_t size = scalar_size(nd.type);
            uint64_t bits = load_bytes(v.sptr[nd.stream] + rel, size, nd.flags & LAMP_FLAG_ALIGNED);
            if(v.heat)
                heat_touch(v, st.nr, st.base0 + rel, st.base0 + rel + size);
            return nd.type == BOOL ? uint64_t(bits != 0) : bits;
        }
        case LAMP_BITS_INT:
        {
            const uint64_t off = i * nd.a;
            uint64_t p = read_bits(reinterpret_cast<const uint32_t*>(v.sptr[nd.stream]), off, nd.a);
            if(v.heat)
                heat_touch(v, v.streams[nd.stream].nr, off / 8, (off + nd.a + 7) / 8);
            if(nd.flags & LAMP_FLAG_SIGNED)
            {
                const uint64_t s = 1ull << (nd.a - 1);
                p = (p ^ s) - s;
            }
            return p & low_mask(8 * scalar_size(nd.type));
        }
        case LAMP_BITS_FLT:
        {
            const uint32_t w = 1 + nd.a + nd.b;
            const uint64_t off = i * w;
            const uint64_t p = read_bits(reinterpret_cast<const uint32_t*>(v.sptr[nd.stream]), off, w);
            if(v.heat)
                heat_touch(v, v.streams[nd.stream].nr, off / 8, (off + w + 7) / 8);
            const uint64_t d = float_decode(p, nd.a, nd.b);
            return nd.type == F32 ? f64_to_f32_bits(d) : d;
        }
        case LAMP_CONVERT:
            if constexpr(D > 1)
            {
                const uint64_t c = read_node<D - 1>(v, nd.child, i);
                return convert_value(c, v.nodes[nd.child].type, nd.type);
            }
            else
                __trap();
        case LAMP_SPLIT:
            if constexpr(D > 1)
            {
                uint64_t acc = 0;
                for(uint32_t k = 0; k < nd.nchild; ++k)
                    acc |= (read_node<D - 1>(v, nd.child + k, i) & 0xFFull) << (8 * k);
                return nd.type == BOOL ? uint64_t(acc != 0) : acc;
            }
            else
                __trap();
        default: // LAMP_NULL
            return 0;
        }
    }

    template<int D>
    __device__ __noinline__ void write_node(const ViewCtx& v, uint32_t n, uint64_t i, uint64_t bits)
    {
        const lamp_node nd = v.nodes[n];
        switch(nd.kind)
        {
        case LAMP_PHYS:
        {
            const lamp_stream st = v.streams[nd.stream];
            const uint64_t rel = block_rel(st, i, nd.a, nd.b);
            const uint32_t size = scalar_size(nd.type);
            store_bytes(v.sptr[nd.stream] + rel, size, nd.flags & LAMP_FLAG_ALIGNED, bits);
            if(v.heat)
                heat_touch(v, st.nr, st.base0 + rel, st.base0 + rel + size);
            return;
        }
        case LAMP_BITS_INT:
        {
            const uint64_t off = i * nd.a;
            write_bits_atomic(reinterpret_cast<uint32_t*>(v.sptr[nd.stream]), off, nd.a, bits);
            if(v.heat)
                heat_touch(v, v.streams[nd.stream].nr, off / 8, (off + nd.a + 7) / 8);
            return;
        }
        case LAMP_BITS_FLT:
        {
            const uint32_t w = 1 + nd.a + nd.b;
            const uint64_t off = i * w;
            const uint64_t d = nd.type == F32 ? f32_to_f64_bits(static_cast<uint32_t>(bits)) : bits;
            write_bits_atomic(reinterpret_cast<uint32_t*>(v.sptr[nd.stream]), off, w, float_encode(d, nd.a, nd.b));
            if(v.heat)
                heat_touch(v, v.streams[nd.stream].nr, off / 8, (off + w + 7) / 8);
            return;
        }
        case LAMP_CONVERT:
            if constexpr(D > 1)
                write_node<D - 1>(v, nd.child, i, convert_value(bits, nd.type, v.nodes[nd.child].type));
            else
                __trap();
            return;
        case LAMP_SPLIT:
            if constexpr(D > 1)
            {
                for(uint32_t k = 0; k < nd.nchild; ++k)
                    write_node<D - 1>(v, nd.child + k, i, (bits >> (8 * k)) & 0xFFull);
            }
            else
                __trap();
            return;
        default: // LAMP_NULL: discarded
            return;
        }
    }

    // The heatmap ranges of one access of node n at element i (Mapping::accessRanges: physical
    // = [off, off+size), bit fields = outward-rounded bytes, byte splits = their s bytes), without
    // touching the data: heat accounting for copies whose data moved through a fast kernel.
    template<int D>
    __device__ __noinline__ void touch_node(const ViewCtx& v, uint32_t n, uint64_t i)
    {
        const lamp_node nd = v.nodes[n];
        switch(nd.kind)
        {
        case LAMP_PHYS:
        {
            const lamp_stream st = v.streams[nd.stream];
            const uint64_t rel = block_rel(st, i, nd.a, nd.b);
            heat_touch(v, st.nr, st.base0 + rel, st.base0 + rel + scalar_size(nd.type));
            return;
        }
        case LAMP_BITS_INT:
        {
            const uint64_t off = i * nd.a;
            heat_touch(v, v.streams[nd.stream].nr, off / 8, (off + nd.a + 7) / 8);
            return;
        }
        case LAMP_BITS_FLT:
        {
            const uint32_t w = 1 + nd.a + nd.b;
            const uint64_t off = i * w;
            heat_touch(v, v.streams[nd.stream].nr, off / 8, (off + w + 7) / 8);
            return;
        }
        case LAMP_CONVERT:
            if constexpr(D > 1)
                touch_node<D - 1>(v, nd.child, i);
            return;
        case LAMP_SPLIT:
            if constexpr(D > 1)
                for(uint32_t k = 0; k < nd.nchild; ++k)
                    touch_node<D - 1>(v, nd.child + k, i);
            return;
        default:
            return;
        }
    }
} // namespace lamd

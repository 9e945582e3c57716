// Copy planning on the host.  makePlan lowers a (src, dst) layout pair into the tile-plan
// form (tile.h: streams, per-leaf terminals, conversions); launchTile then hands the plan to
// the first specialised kernel whose predicate holds -- register transpose (vec_transpose.cu),
// bit packing (pack.cu), record <-> byte planes (planes.cu), f32 <-> f64 transpose, direct L1
// gathers for the remaining uniform pairs, the general warp-tile engine (copy_tile.cu), and
// last the TMA tile engine -- adds FieldAccessCount in closed form and accounts a Heatmap in a
// separate range-only pass.  Pairs no plan can express run on the generic interpreter kernel
// (copy_generic.cu).
#include "capi_internal.hpp"
#include "tile.h"

#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace lamk
{
    cudaError_t tile_copy(const lamt_params& p, uint32_t smemBytes, uint32_t ctasPerSm, cudaStream_t s);
    cudaError_t uniform_direct(const lamt_params& p, uint64_t n, cudaStream_t s);
    cudaError_t uniform_warp(const lamt_params& p, uint32_t ntiles, cudaStream_t s);
    cudaError_t warp_tile(const lamt_params& p, uint32_t ntiles, cudaStream_t s);

    struct VecSide
    {
        unsigned long long leafBase[LAMT_UNI_LEAVES];
        unsigned long long recBase;
        uint32_t recordContig;
        uint32_t bs, lanes, lshift;
    };
    struct VecParams
    {
        VecSide s, d;
        unsigned long long begin;
        unsigned long long groups;
        unsigned long long facSrc, facDst;
        uint32_t nl, facS, facD;
        uint32_t sstage; // AoS source loaded warp-coalesced through the smem slice (k_vec_transpose)
    };
    bool vec_transpose(const VecParams& p, uint32_t leafSize, cudaStream_t s);
    bool vec_convert(const VecParams& p, uint32_t ss, uint32_t ds, cudaStream_t s);

    struct PackParams
    {
        unsigned long long vals, bits, begin, groups;
        uint32_t w, kind, sgn, E, M, valType;
        unsigned long long facSrc, facDst;
        uint32_t facS, facD, leaf, nleaves;
        uint32_t vbs, vl, vsh, vinb;
    };
    bool pack32(const PackParams& p, bool pack, cudaStream_t s);

    struct RecPackParams
    {
        unsigned long long rec;
        unsigned long long bits[8];
        unsigned long long begin, groups;
        uint32_t nl, lanes, lsh, sgnMask;
        uint32_t w, E, M;
        uint32_t gmag;
    };
    bool rec_pack(const RecPackParams& q, uint32_t kind, bool pack, cudaStream_t s);

    struct PlaneParams
    {
        unsigned long long rec;
        unsigned long long plane[8][8];
        unsigned long long begin, groups;
        uint32_t nl;
    };
    bool planes_copy(const PlaneParams& p, uint32_t sb, bool cvt, bool toPlanes, cudaStream_t s);
}

using namespace lamb;

namespace lamjit
{
    bool tryCopy(const lamt_params& p, uint64_t begin, uint64_t end, uint64_t* doneEnd, cudaStream_t s);
}

namespace lamhost
{
    namespace
    {
        uint64_t gcd64(uint64_t a, uint64_t b)
        {
            while(b)
            {
                const uint64_t t = a % b;
                a = b;
                b = t;
            }
            return a;
        }
        uint64_t lcm64(uint64_t a, uint64_t b)
        {
            return a / gcd64(a, b) * b;
        }

        // tuning knobs (defaults chosen from the B200 sweep in profiles/)
        double envNum(const char* name, double dflt)
        {
            const char* v = std::getenv(name);
            if(!v || !*v)
                return dflt;
            return std::atof(v);
        }

        struct Side
        {
            const Lowered* L;
            std::vector<int> map; // lowered stream -> tile stream (-1 unused)
        };

        struct Plan
        {
            bool ok = false;
            lamt_params p{};
            uint32_t smem = 0;
            uint32_t ctas = 1;
            std::vector<int> srcStreams, dstStreams; // tile stream order -> lowered stream
        };

        int useStream(Side& s, uint16_t lowered, std::vector<int>& order)
        {
            if(s.map[lowered] < 0)
            {
                s.map[lowered] = static_cast<int>(order.size());
                order.push_back(lowered);
            }
            return s.map[lowered];
        }

        // one side of a leaf: [CONVERT] -> PHYS | SPLIT(PHYS u8...) | BITS_INT | BITS_FLT | NULL
        bool parseSide(Side& side, uint16_t root, bool isDst, uint8_t& kind, uint8_t& stype, uint8_t& ltype,
                       lamt_term* terms, uint8_t& nterms, uint8_t& E, uint8_t& M, uint8_t& sgn,
                       std::vector<int>& order, int streamBase)
        {
            const auto& nodes = side.L->nodes;
            const auto& streams = side.L->streams;
            lamp_node nd = nodes[root];
            ltype = nd.type;
            if(nd.kind == LAMP_CONVERT)
            {
                nd = nodes[nd.child];
                if(nd.kind == LAMP_CONVERT)
                    return false;
            }
            stype = nd.type;
            auto physTerm = [&](const lamp_node& t, lamt_term& out) -> bool
            {
                const lamp_stream& st = streams[t.stream];
                const uint64_t size = scalarSize(t.type);
                if(st.kind != LAMS_PHYS || st.block_stride == 0)
                    return false;
                if(t.a + (st.lanes - 1) * uint64_t(t.b) + size > st.block_stride)
                    return false; // terminal straddles its block
                // a destination with padding is preloaded by the warp-tile engine (stream.preload);
                // no other tile kernel may take such a plan
                if(st.block_stride > 0xFFFFFFFFull || st.lanes > 0xFFFFFFFFull)
                    return false;
                out.stream = static_cast<uint16_t>(streamBase + useStream(side, t.stream, order));
                out.size = static_cast<uint8_t>(size);
                out.aligned = (t.a % size == 0 && st.block_stride % size == 0 && (st.lanes == 1 || t.b % size == 0));
                out.inblock = t.a;
                out.ls = t.b;
                return true;
            };
            switch(nd.kind)
            {
            case LAMP_PHYS:
                kind = LAMT_K_PHYS;
                nterms = 1;
                return physTerm(nd, terms[0]);
            case LAMP_SPLIT:
                kind = LAMT_K_SPLIT;
                if(nd.nchild > LAMT_MAX_TERMS)
                    return false;
                nterms = nd.nchild;
                for(uint32_t k = 0; k < nd.nchild; ++k)
                {
                    const lamp_node& c = nodes[nd.child + k];
                    if(c.kind != LAMP_PHYS || c.type != U8)
                        return false;
                    if(!physTerm(c, terms[k]))
                        return false;
                }
                return true;
            case LAMP_BITS_INT:
            case LAMP_BITS_FLT:
            {
                kind = nd.kind == LAMP_BITS_INT ? LAMT_K_BITS_INT : LAMT_K_BITS_FLT;
                nterms = 1;
                E = static_cast<uint8_t>(nd.a);
                M = static_cast<uint8_t>(nd.b);
                sgn = (nd.flags & LAMP_FLAG_SIGNED) ? 1 : 0;
                terms[0] = lamt_term{};
                terms[0].stream = static_cast<uint16_t>(streamBase + useStream(side, nd.stream, order));
                return true;
            }
            case LAMP_NULL:
                kind = LAMT_K_NULL;
                nterms = 0;
                return true;
            default:
                return false;
            }
        }

        Plan makePlan(const Lowered& S, const Lowered& D)
        {
            Plan pl; // heatmaps are accounted separately (launchTile -> heat_account)
            const size_t nleaves = S.roots.size();
            if(nleaves == 0 || nleaves > LAMT_MAX_LEAVES)
                return pl;
            Side ss{&S, std::vector<int>(S.streams.size(), -1)};
            Side ds{&D, std::vector<int>(D.streams.size(), -1)};
            // first pass: source streams, to know the destination base index
            std::vector<lamt_leaf> leaves(nleaves);
            for(size_t f = 0; f < nleaves; ++f)
            {
                lamt_leaf& L = leaves[f];
                uint8_t lt = 0;
                if(!parseSide(ss, S.roots[f], false, L.skind, L.stype, lt, L.s, L.sn, L.sE, L.sM, L.ssigned,
                              pl.srcStreams, 0))
                    return pl;
                L.ltype = lt;
            }
            const int nsrc = static_cast<int>(pl.srcStreams.size());
            for(size_t f = 0; f < nleaves; ++f)
            {
                lamt_leaf& L = leaves[f];
                uint8_t lt = 0, sg = 0;
                if(!parseSide(ds, D.roots[f], true, L.dkind, L.dtype, lt, L.d, L.dn, L.dE, L.dM, sg, pl.dstStreams,
                              nsrc))
                    return pl;
                if(lt != L.ltype)
                    return pl;
                L.pure = L.skind == LAMT_K_PHYS && L.dkind == LAMT_K_PHYS && L.stype == L.ltype && L.dtype == L.ltype;
            }
            const int ndst = static_cast<int>(pl.dstStreams.size());
            if(nsrc + ndst > LAMT_MAX_STREAMS)
                return pl;

            // tile size
            uint64_t unit = lcm64(lcm64(S.shardUnit, D.shardUnit), 32);
            double bpe = 0;
            auto perElem = [](const lamp_stream& st) {
                return st.kind == LAMS_BITS ? st.block_stride / 8.0 : double(st.block_stride) / double(st.lanes);
            };
            for(int k : pl.srcStreams)
                bpe += perElem(S.streams[k]);
            for(int k : pl.dstStreams)
            {
                bpe += perElem(D.streams[k]);
                if(D.streams[k].kind == LAMS_BITS)
                    bpe += D.streams[k].block_stride > 32 ? 8 : 4;
            }
            // CTA pipeline: `stages` source buffers + `dstages` destination buffers of one tile each
            const double stageTarget = envNum("LAMB_TILE_KB", 24.0) * 1024; // src+dst bytes of one tile
            const uint32_t stages = static_cast<uint32_t>(envNum("LAMB_TILE_STAGES", 3));
            const uint32_t dstages = static_cast<uint32_t>(envNum("LAMB_TILE_DSTAGES", 2));
            if(unit > (1u << 16) || bpe * unit > 100.0 * 1024 || stages < 1 || stages > LAMT_MAX_STAGES
               || dstages < 2 || dstages > 4)
                return pl;
            uint64_t T = static_cast<uint64_t>(stageTarget / (bpe > 0 ? bpe : 1) / unit) * unit;
            if(T < unit)
                T = unit;
            if(T > (1u << 16))
                T = (1u << 16) / unit * unit;

            lamt_params& p = pl.p;
            p.T = static_cast<uint32_t>(T);
            p.nleaves = static_cast<uint32_t>(nleaves);
            p.nsrc = static_cast<uint32_t>(nsrc);
            p.ndst = static_cast<uint32_t>(ndst);
            uint32_t off = 0;
            uint32_t tmaBytes = 0;
            auto fillStream = [&](lamt_stream& t, const lamp_stream& st)
            {
                t.kind = st.kind == LAMS_BITS ? 1 : 0;
                t.bs = static_cast<uint32_t>(st.block_stride);
                t.lanes = t.kind ? 1 : static_cast<uint32_t>(st.lanes);
                t.lshift = t.kind ? 0 : st.lane_shift;
                t.tile_bytes = t.kind ? static_cast<uint32_t>(T * st.block_stride / 8)
                                      : static_cast<uint32_t>(T / st.lanes * st.block_stride);
                t.smem_off = off;
                off += (t.tile_bytes + 127) & ~127u;
            };
            for(int k = 0; k < nsrc; ++k)
            {
                fillStream(p.st[k], S.streams[pl.srcStreams[k]]);
                tmaBytes += p.st[k].tile_bytes;
            }
            p.src_bytes = off;
            off = 0;
            for(int k = 0; k < ndst; ++k)
            {
                const lamp_stream& ls = D.streams[pl.dstStreams[k]];
                fillStream(p.st[nsrc + k], ls);
                p.st[nsrc + k].preload = ls.kind == LAMS_PHYS && !ls.holefree;
                p.dst_holes |= p.st[nsrc + k].preload;
            }
            for(int k = 0; k < ndst; ++k)
            {
                lamt_stream& t = p.st[nsrc + k];
                if(t.kind == 1)
                {
                    t.scratch64 = t.bs > 32;
                    t.scratch_off = off;
                    off += static_cast<uint32_t>(((T + 2) * (t.scratch64 ? 8 : 4) + 127) & ~uint64_t{127});
                }
            }
            p.dst_bytes = off;
            p.tma_bytes = tmaBytes; // adjusted per launch for non-TMA streams
            std::memcpy(p.leaf, leaves.data(), nleaves * sizeof(lamt_leaf));
            p.facS = S.fac;
            p.facD = D.fac;
            p.stages = stages;
            p.dstages = dstages;
            p.any_bits = 0;
            for(int k = 0; k < ndst; ++k)
                p.any_bits |= p.st[nsrc + k].kind == 1;
            p.threads = static_cast<uint32_t>(envNum("LAMB_TILE_THREADS", 256));
            p.stg = envNum("LAMB_TILE_STG", 1) != 0;
            p.lmode = static_cast<uint32_t>(envNum("LAMB_TILE_LMODE", 1));
            p.chunk = static_cast<uint32_t>(envNum("LAMB_TILE_CHUNK", 0)) & ~15u;
            if(p.lmode == 1 && stages < 2)
                return pl;
            pl.smem = stages * p.src_bytes + dstages * p.dst_bytes;
            const uint32_t smBudget = 226 * 1024;
            if(pl.smem > smBudget)
                return pl;
            pl.ctas = std::max<uint32_t>(1, std::min<uint32_t>(static_cast<uint32_t>(envNum("LAMB_TILE_CTAS", 4)),
                                                               smBudget / (pl.smem + 1024)));

            // uniform fast path: all leaves same-size aligned physical moves, one geometry per side
            bool uni = nleaves <= LAMT_UNI_LEAVES;
            const lamt_leaf& L0 = leaves[0];
            for(size_t f = 0; uni && f < nleaves; ++f)
            {
                const lamt_leaf& L = leaves[f];
                uni = L.pure && L.stype != Bool && (L.s[0].size == 4 || L.s[0].size == 8) && L.s[0].size == L0.s[0].size
                    && L.s[0].aligned && L.d[0].aligned;
                if(!uni)
                    break;
                const lamt_stream &a0 = p.st[L0.s[0].stream], &a = p.st[L.s[0].stream];
                const lamt_stream &b0 = p.st[L0.d[0].stream], &b = p.st[L.d[0].stream];
                uni = a.bs == a0.bs && a.lanes == a0.lanes && L.s[0].ls == L0.s[0].ls && b.bs == b0.bs
                    && b.lanes == b0.lanes && L.d[0].ls == L0.d[0].ls;
            }
            if(uni)
            {
                p.uni = 1;
                p.usize = L0.s[0].size;
                const lamt_stream &a = p.st[L0.s[0].stream], &b = p.st[L0.d[0].stream];
                p.ubs_s = a.bs;
                p.ul_s = a.lanes;
                p.ush_s = a.lshift;
                p.uls_s = L0.s[0].ls;
                p.ubs_d = b.bs;
                p.ul_d = b.lanes;
                p.ush_d = b.lshift;
                p.uls_d = L0.d[0].ls;
                for(size_t f = 0; f < nleaves; ++f)
                {
                    p.uoff_s[f] = p.st[leaves[f].s[0].stream].smem_off + leaves[f].s[0].inblock;
                    p.uoff_d[f] = p.st[leaves[f].d[0].stream].smem_off + leaves[f].d[0].inblock;
                }
            }
            pl.ok = true;
            return pl;
        }

        uint64_t tileOff(const lamt_stream& s, uint64_t t0)
        {
            if(s.kind == 1)
                return t0 * s.bs / 8;
            return t0 / s.lanes * s.bs;
        }
    } // namespace

    // General warp-tile engine (copy_tile.cu k_warp_tile): re-tile the plan for one warp per
    // tile of `wt` elements (about 6 KB of images + bit scratch per warp), every image 16-byte
    // aligned in global memory and a multiple of 16 bytes long.
    static bool tryWarpTile(const lamt_params& p, const Lowered& S, const Lowered& D, const DeviceImage& si,
                            DeviceImage& di, uint64_t begin, uint64_t end, cudaStream_t s);

    // FieldAccessCount under copyView (view.cpp:186-188): every element of the range reads each
    // source leaf once and writes each destination leaf once, so the specialised kernels add
    // the counts in closed form (one tiny launch) instead of atomics in the streaming loop
    static void addAccessCounts(const lamt_params& p, const Lowered& S, uint64_t count, cudaStream_t s)
    {
        if(!(p.facS || p.facD) || count == 0)
            return;
        lam_cuda_check(lamk::fac_add(p.facS ? reinterpret_cast<unsigned long long*>(p.facSrc) : nullptr,
                                     p.facD ? reinterpret_cast<unsigned long long*>(p.facDst) : nullptr,
                                     static_cast<uint32_t>(S.roots.size()), count, s),
                       "fac_add");
    }

    static bool tryWarpTile(const lamt_params& p, const Lowered& S, const Lowered& D, const DeviceImage& si,
                            DeviceImage& di, uint64_t begin, uint64_t end, cudaStream_t s)
    {
        if(p.nsrc + p.ndst > LAMT_WT_MAX_STREAMS)
            return false;
        const uint64_t unit = lcm64(lcm64(S.shardUnit, D.shardUnit), 32);
        double bpe = 0;
        for(uint32_t k = 0; k < p.nsrc + p.ndst; ++k)
        {
            const lamt_stream& t = p.st[k];
            bpe += t.kind ? t.bs / 8.0 : double(t.bs) / t.lanes;
            if(k >= p.nsrc && t.kind)
                bpe += t.bs > 32 ? 8 : 4;
        }
        const double target = envNum("LAMB_WARP_TILE_KB", 6.0) * 1024;
        uint64_t wt = static_cast<uint64_t>(target / (bpe > 0 ? bpe : 1) / unit) * unit;
        if(wt < unit)
            wt = unit;
        const uint64_t ntw = (end - begin) / wt;
        if(ntw == 0 || ntw > 0x7FFFFFFFull || wt > 4096 || p.nsrc + p.ndst > 255)
            return false;
        lamt_params q = p;
        q.T = static_cast<uint32_t>(wt);
        uint32_t off = 0, chunk = 0;
        for(uint32_t k = 0; k < q.nsrc + q.ndst; ++k)
        {
            lamt_stream& t = q.st[k];
            if(k == q.nsrc)
            {
                q.src_bytes = off;
                off = 0;
                chunk = 0;
            }
            const uint64_t bytes = t.kind ? wt * t.bs / 8 : wt / t.lanes * t.bs;
            if(bytes % 16 || (t.gptr + (t.kind ? (begin * t.bs) / 8 : begin / t.lanes * t.bs)) % 16)
                return false;
            t.tile_bytes = static_cast<uint32_t>(bytes);
            t.smem_off = off;
            t.pad = chunk;
            off += static_cast<uint32_t>(bytes);
            chunk += static_cast<uint32_t>(bytes / 16);
        }
        for(uint32_t k = q.nsrc; k < q.nsrc + q.ndst; ++k)
        {
            lamt_stream& t = q.st[k];
            if(t.kind == 1)
            {
                t.scratch64 = t.bs > 32;
                t.scratch_off = off;
                off += static_cast<uint32_t>(((wt + 2) * (t.scratch64 ? 8 : 4) + 15) & ~uint64_t{15});
            }
        }
        q.dst_bytes = off;
        const uint32_t chS = q.src_bytes / 16, chD = chunk;
        if(8ull * (q.src_bytes + q.dst_bytes) > 180 * 1024 || chS + chD > 1024)
            return false;
        q.wt_chs = chS;
        q.wt_chd = chD;
        for(uint32_t k = 0; k < q.nsrc + q.ndst; ++k)
        {
            const lamt_stream& t = q.st[k];
            for(uint32_t c = 0; c < t.tile_bytes / 16; ++c)
                q.wt_cst[(k < q.nsrc ? 0 : chS) + t.pad + c] = static_cast<uint8_t>(k);
        }
        q.facS = 0; // closed form below
        q.facD = 0;
        // per-leaf fast descriptors (terms on lanes == 1 streams: smem offset + element stride)
        for(uint32_t f = 0; f < q.nleaves; ++f)
        {
            const lamt_leaf& L = q.leaf[f];
            lamt_wfast& W = q.wf[f];
            W = lamt_wfast{};
            W.mode = LAMT_WF_GENERIC;
            if(L.dkind == LAMT_K_NULL)
            {
                W.mode = LAMT_WF_SKIP;
                continue;
            }
            const bool sPhys = L.skind == LAMT_K_PHYS, dPhys = L.dkind == LAMT_K_PHYS;
            const bool sSplit = L.skind == LAMT_K_SPLIT, dSplit = L.dkind == LAMT_K_SPLIT;
            if(!((sPhys || sSplit) && (dPhys || dSplit)) || (sSplit && dSplit))
                continue;
            W.sn = sPhys ? 1 : L.sn;
            W.dn = dPhys ? 1 : L.dn;
            bool ok = W.sn <= 8 && W.dn <= 8;
            bool planes = q.T % 4 == 0;
            bool unalignedS = false, unalignedD = false;
            W.sL = W.dL = 1;
            auto term = [&](const lamt_term& t, uint32_t& base, uint32_t& bs, bool split) -> bool
            {
                const lamt_stream& st = q.st[t.stream];
                if(st.kind != 0 || (split && !t.aligned))
                    return false;
                if(st.lanes != 1)
                {
                    // AoSoA: only as the single term of a PHYS -> PHYS leaf
                    if(split || !(sPhys && dPhys) || st.lanes >= (1u << 16) || q.T >= (1u << 16))
                        return false;
                    const bool isSrc = &t == &L.s[0];
                    (isSrc ? W.sL : W.dL) = st.lanes;
                    (isSrc ? W.sls : W.dls) = t.ls;
                    (isSrc ? W.smagic : W.dmagic) = static_cast<uint32_t>(((uint64_t{1} << 32) + st.lanes - 1) / st.lanes);
                }
                if(!t.aligned)
                    (&t == &L.s[0] ? unalignedS : unalignedD) = true;
                base = st.smem_off + t.inblock;
                bs = st.bs;
                if(split)
                    planes = planes && bs == 1 && (base & 3) == 0;
                return true;
            };
            for(uint32_t k = 0; ok && k < W.sn; ++k)
                ok = term(L.s[k], W.sbase[k], W.sbs[k], sSplit);
            for(uint32_t k = 0; ok && k < W.dn; ++k)
                ok = term(L.d[k], W.dbase[k], W.dbs[k], dSplit);
            if(!ok)
                continue;
            W.ssz = static_cast<uint8_t>((sPhys ? L.s[0].size : 1) | (unalignedS ? 0x80 : 0));
            W.dsz = static_cast<uint8_t>((dPhys ? L.d[0].size : 1) | (unalignedD ? 0x80 : 0));
            W.conv = !(L.stype == L.ltype && L.ltype == L.dtype);
            W.boolean = L.stype == Bool;
            W.mode = sPhys && dPhys ? LAMT_WF_PP
                   : dSplit       ? (planes ? LAMT_WF_PS_PLANES : LAMT_WF_PS_BYTES)
                                  : (planes ? LAMT_WF_SP_PLANES : LAMT_WF_SP_BYTES);
        }
        lam_cuda_check(lamk::warp_tile(q, static_cast<uint32_t>(ntw), s), "warp_tile");
        addAccessCounts(p, S, ntw * wt, s);
        const uint64_t doneEnd = begin + ntw * wt;
        if(doneEnd < end)
            lam_cuda_check(lamk::generic_copy(si.hdr, di.hdr, doneEnd, end, static_cast<uint32_t>(S.roots.size()), S.fac,
                                              D.fac, s, false),
                           "generic_copy(tail)");
        (void)D;
        return true;
    }

    // register-transpose path (vec_transpose.cu) for uniform 4/8-byte-leaf pairs whose sides are
    // leaf-contiguous in groups of V elements (SoA, AoSoA with V | L) or record-contiguous (AoS)
    static bool tryVec(const lamt_params& p, uint64_t begin, uint64_t end, const DeviceImage& si, DeviceImage& di,
                       const Lowered& S, const Lowered& D, cudaStream_t s)
    {
        if(p.usize != 4 && p.usize != 8)
            return false;
        const uint32_t V = 16 / p.usize;
        const uint32_t nl = p.nleaves;
        if(nl < 1 || nl > 8 || begin % V)
            return false;
        lamk::VecParams vp{};
        auto side = [&](bool src, lamk::VecSide& sd) -> bool
        {
            const uint32_t L = src ? p.ul_s : p.ul_d;
            const uint32_t bs = src ? p.ubs_s : p.ubs_d;
            const uint32_t ls = src ? p.uls_s : p.uls_d;
            const uint32_t sh = src ? p.ush_s : p.ush_d;
            const uint32_t S = p.usize;
            bool recordContig = L == 1 && bs == nl * S;
            bool leafContig = (L == 1 && bs == S) || (L > 1 && L % V == 0 && sh != 0xFFFFFFFFu && ls == S);
            if(recordContig)
            {
                // one stream, leaves packed in leaf order
                const lamt_leaf& L0 = p.leaf[0];
                const lamt_term& t0 = src ? L0.s[0] : L0.d[0];
                for(uint32_t f = 0; f < nl && recordContig; ++f)
                {
                    const lamt_term& t = src ? p.leaf[f].s[0] : p.leaf[f].d[0];
                    recordContig = t.stream == t0.stream && t.inblock == f * S;
                }
                if(recordContig)
                {
                    sd.recordContig = 1;
                    sd.recBase = p.st[t0.stream].gptr;
                    return (sd.recBase % 16) == 0;
                }
            }
            if(!leafContig)
                return false;
            if(!src && L == V && bs == nl * 16)
            {
                // AoSoA<V> destination: a thread's V elements are one whole block, leaf f's vector at
                // f * 16, so the warp's 32 blocks are contiguous and are staged like AoS records
                // (512-byte stores instead of 16-byte stores at the block stride)
                bool blockMajor = true;
                const lamt_term& t0 = p.leaf[0].d[0];
                for(uint32_t f = 0; f < nl && blockMajor; ++f)
                {
                    const lamt_term& t = p.leaf[f].d[0];
                    blockMajor = t.stream == t0.stream && t.inblock == f * 16;
                }
                if(blockMajor && p.st[t0.stream].gptr % 16 == 0 && envNum("LAMB_VEC_BLOCKSTAGE", 1) != 0)
                {
                    sd.recordContig = 2;
                    sd.recBase = p.st[t0.stream].gptr;
                    return true;
                }
            }
            sd.recordContig = 0;
            sd.bs = bs;
            sd.lanes = L;
            sd.lshift = L == 1 ? 0 : sh;
            for(uint32_t f = 0; f < nl; ++f)
            {
                const lamt_term& t = src ? p.leaf[f].s[0] : p.leaf[f].d[0];
                sd.leafBase[f] = p.st[t.stream].gptr + t.inblock;
                if(sd.leafBase[f] % 16)
                    return false;
            }
            return bs % 16 == 0 || L == 1;
        };
        if(!side(true, vp.s) || !side(false, vp.d))
            return false;
        vp.begin = begin;
        vp.groups = (end - begin) / V;
        vp.nl = nl;
        vp.facS = 0; // counted in closed form below (fac_add)
        vp.facD = 0;
        vp.facSrc = p.facSrc;
        vp.facDst = p.facDst;
        if(vp.groups == 0)
            return false;
        vp.sstage = vp.s.recordContig == 1 && envNum("LAMB_VEC_SSTAGE", 1) != 0;
        if(!vp.s.recordContig && vp.s.lanes > 1 && (32 * V) % vp.s.lanes == 0 && vp.s.bs == nl * vp.s.lanes * p.usize
           && envNum("LAMB_VEC_SSTAGE", 1) != 0)
        {
            // AoSoA<L> source, leaves in order, no padding: the warp's span is contiguous
            bool inOrder = true;
            const unsigned long long b0 = vp.s.leafBase[0];
            for(uint32_t f = 0; f < nl && inOrder; ++f)
                inOrder = vp.s.leafBase[f] == b0 + uint64_t(f) * vp.s.lanes * p.usize;
            if(inOrder && b0 % 16 == 0)
            {
                vp.s.recBase = b0;
                vp.sstage = 2;
            }
        }
        if(!lamk::vec_transpose(vp, p.usize, s))
            return false;
        addAccessCounts(p, S, vp.groups * V, s);
        const uint64_t doneEnd = begin + vp.groups * V;
        if(doneEnd < end)
            lam_cuda_check(lamk::generic_copy(si.hdr, di.hdr, doneEnd, end, static_cast<uint32_t>(S.roots.size()), S.fac,
                                              D.fac, s, false),
                           "generic_copy(tail)");
        (void)D;
        return true;
    }

    // Uniform physical pairs over multi-stream sides (Split mappings, vec_multi.cu k_vec_multi):
    // every leaf a same-size (4 or 8 byte) physical move without conversion; on each side a
    // leaf is either leaf-contiguous (SoA, AoSoA with V | L) or sits in a record stream
    // (L = 1) whose leaves cover the whole record.
    static bool tryVecMulti(const lamt_params& p, uint64_t begin, uint64_t end, const DeviceImage& si,
                            DeviceImage& di, const Lowered& S, const Lowered& D, cudaStream_t s)
    {
        const uint32_t nl = p.nleaves;
        if(nl < 1 || nl > 8 || envNum("LAMB_VEC_MULTI", 1) == 0)
            return false;
        const uint32_t sz = p.leaf[0].s[0].size;
        if(sz != 4 && sz != 8)
            return false;
        const uint32_t V = 16 / sz, WPE = sz / 4;
        if(begin % V)
            return false;
        for(uint32_t f = 0; f < nl; ++f)
        {
            const lamt_leaf& L = p.leaf[f];
            if(L.skind != LAMT_K_PHYS || L.dkind != LAMT_K_PHYS || L.s[0].size != sz || L.d[0].size != sz
               || L.stype != L.dtype || L.stype != L.ltype || L.ltype == Bool)
                return false;
        }
        lamk::VMParams vp{};
        uint32_t row = 0;
        auto side = [&](bool src, lamk::VMSide& sd) -> bool
        {
            uint32_t streams[8], nst = 0;
            for(uint32_t f = 0; f < nl; ++f)
            {
                const lamt_term& t = src ? p.leaf[f].s[0] : p.leaf[f].d[0];
                const lamt_stream& st = p.st[t.stream];
                const bool soa = st.lanes == 1 && st.bs == sz;
                const bool aosoa = st.lanes > 1 && st.lanes % V == 0 && st.lshift != 0xFFFFFFFFu && t.ls == sz;
                if(soa || aosoa)
                {
                    sd.mode[f] = 0;
                    sd.base[f] = st.gptr + t.inblock;
                    sd.bs[f] = soa ? sz * V : st.bs; // per group of V elements: (e0 >> lsh) * bs
                    sd.lsh[f] = soa ? 0 : st.lshift;
                    sd.lmask[f] = soa ? 0 : st.lanes - 1;
                    if(soa)
                    {
                        // e0 is a multiple of V: e0 * sz = (e0 >> 0) * bs with bs = sz, lmask 0
                        sd.bs[f] = sz;
                    }
                    if(sd.base[f] % 16 || (aosoa && st.bs % 16))
                        return false;
                    continue;
                }
                if(st.lanes != 1 || st.bs % sz || t.inblock % sz || st.bs > 8 * sz || st.gptr % 16)
                    return false;
                uint32_t r = 0;
                while(r < nst && streams[r] != t.stream)
                    ++r;
                if(r == nst)
                    streams[nst++] = t.stream;
                sd.mode[f] = 1;
            }
            // record streams: covered by their leaves (each record position once), V records =
            // bs * V / 16 vectors, laid out in the lane row
            for(uint32_t r = 0; r < nst; ++r)
            {
                const lamt_stream& st = p.st[streams[r]];
                const uint32_t rl = st.bs / sz;
                uint32_t seen = 0, cnt = 0;
                for(uint32_t f = 0; f < nl; ++f)
                {
                    const lamt_term& t = src ? p.leaf[f].s[0] : p.leaf[f].d[0];
                    if(sd.mode[f] != 1 || t.stream != streams[r])
                        continue;
                    const uint32_t q = t.inblock / sz;
                    if(q >= rl || (seen >> q) & 1u)
                        return false;
                    seen |= 1u << q;
                    ++cnt;
                    sd.wpos[f] = row + q * WPE;
                    sd.wstep[f] = rl * WPE;
                }
                if(cnt != rl)
                    return false;
                const uint32_t nv = st.bs * V / 16;
                for(uint32_t k = 0; k < nv; ++k)
                {
                    if(sd.nvec >= 8)
                        return false;
                    sd.vb[sd.nvec] = st.gptr + 16ull * k;
                    sd.vs[sd.nvec] = st.bs;
                    sd.vrow[sd.nvec] = row + 4 * k;
                    ++sd.nvec;
                }
                row += nv * 4;
            }
            // AoS: a single record stream with every leaf at inblock f * sz -> registers only
            sd.full = 0;
            if(nst == 1)
            {
                bool full = true;
                for(uint32_t f = 0; f < nl && full; ++f)
                {
                    const lamt_term& t = src ? p.leaf[f].s[0] : p.leaf[f].d[0];
                    full = sd.mode[f] == 1 && t.stream == streams[0] && t.inblock == f * sz;
                }
                if(full)
                {
                    sd.full = 1;
                    row -= sd.nvec * 4; // no row needed
                }
            }
            return true;
        };
        if(!side(true, vp.s) || !side(false, vp.d))
            return false;
        vp.rowWords = row | 1u;
        vp.begin = begin;
        vp.groups = (end - begin) / V;
        vp.nl = nl;
        if(vp.groups == 0 || !lamk::vec_multi(vp, sz, s))
            return false;
        addAccessCounts(p, S, vp.groups * V, s);
        const uint64_t doneEnd = begin + vp.groups * V;
        if(doneEnd < end)
            lam_cuda_check(lamk::generic_copy(si.hdr, di.hdr, doneEnd, end, static_cast<uint32_t>(S.roots.size()), S.fac,
                                              D.fac, s, false),
                           "generic_copy(tail)");
        return true;
    }

    // ChangeType f32 <-> f64 over uniform geometries (vec_transpose.cu k_vec_convert): every leaf
    // PHYS -> PHYS with source size SS and destination size DS (4 <-> 8), one conversion
    // f32 -> f64 or f64 -> f32 between them; each side record-contiguous or leaf-contiguous.
    static bool tryVecConvert(const lamt_params& p, uint64_t begin, uint64_t end, const DeviceImage& si,
                              DeviceImage& di, const Lowered& S, const Lowered& D, cudaStream_t s)
    {
        const uint32_t nl = p.nleaves;
        if(nl < 1 || nl > 8 || begin % 4 || envNum("LAMB_VEC_CONVERT", 1) == 0)
            return false;
        const uint32_t ss = p.leaf[0].s[0].size, ds = p.leaf[0].d[0].size;
        if(!((ss == 4 && ds == 8) || (ss == 8 && ds == 4)))
            return false;
        for(uint32_t f = 0; f < nl; ++f)
        {
            const lamt_leaf& L = p.leaf[f];
            if(L.skind != LAMT_K_PHYS || L.dkind != LAMT_K_PHYS || L.s[0].size != ss || L.d[0].size != ds)
                return false;
            // exactly one f32 <-> f64 conversion on the way (storage -> logical -> storage)
            const bool widen = ss == 4 && L.stype == F32 && L.dtype == F64 && (L.ltype == F32 || L.ltype == F64);
            const bool narrow = ss == 8 && L.stype == F64 && L.dtype == F32 && (L.ltype == F32 || L.ltype == F64);
            if(!(widen || narrow))
                return false;
        }
        lamk::VecParams vp{};
        auto side = [&](bool src, lamk::VecSide& sd) -> bool
        {
            const uint32_t S0 = src ? ss : ds;
            const lamt_term& t0 = src ? p.leaf[0].s[0] : p.leaf[0].d[0];
            const lamt_stream& st0 = p.st[t0.stream];
            bool rec = st0.lanes == 1 && st0.bs == nl * S0;
            for(uint32_t f = 0; f < nl && rec; ++f)
            {
                const lamt_term& t = src ? p.leaf[f].s[0] : p.leaf[f].d[0];
                rec = t.stream == t0.stream && t.inblock == f * S0;
            }
            if(rec)
            {
                sd.recordContig = 1;
                sd.recBase = st0.gptr;
                return (sd.recBase + begin * nl * S0) % 16 == 0;
            }
            sd.recordContig = 0;
            sd.bs = st0.bs;
            sd.lanes = st0.lanes;
            sd.lshift = st0.lanes == 1 ? 0 : st0.lshift;
            if(!((st0.lanes == 1 && st0.bs == S0)
                 || (st0.lanes > 1 && st0.lanes % 4 == 0 && st0.lshift != 0xFFFFFFFFu && st0.bs % 16 == 0)))
                return false;
            for(uint32_t f = 0; f < nl; ++f)
            {
                const lamt_term& t = src ? p.leaf[f].s[0] : p.leaf[f].d[0];
                const lamt_stream& st = p.st[t.stream];
                if(st.lanes != st0.lanes || st.bs != st0.bs || (st.lanes > 1 && t.ls != S0))
                    return false;
                sd.leafBase[f] = st.gptr + t.inblock;
                if((sd.leafBase[f] + (st.lanes == 1 ? begin * S0 : 0)) % 16)
                    return false;
            }
            return true;
        };
        if(!side(true, vp.s) || !side(false, vp.d))
            return false;
        vp.begin = begin;
        vp.groups = (end - begin) / 4;
        vp.nl = nl;
        if(vp.groups == 0 || !lamk::vec_convert(vp, ss, ds, s))
            return false;
        addAccessCounts(p, S, vp.groups * 4, s);
        const uint64_t doneEnd = begin + vp.groups * 4;
        if(doneEnd < end)
            lam_cuda_check(lamk::generic_copy(si.hdr, di.hdr, doneEnd, end, static_cast<uint32_t>(S.roots.size()), S.fac,
                                              D.fac, s, false),
                           "generic_copy(tail)");
        return true;
    }

    // K3/K4 record side: every leaf a 4-byte leaf of one record stream -- AoS packed, or AoSoA<L>
    // with L | 32 and L < 32 -- against bit streams of one width and format (pack.cu k_rec_pack /
    // k_rec_unpack, one pass instead of staging through an SoA scratch)
    static bool tryRecPack(const lamt_params& p, uint64_t begin, uint64_t groups, cudaStream_t s)
    {
        const uint32_t nl = p.nleaves;
        // one leaf: the record stream is an SoA array, which k_pack32 handles with every warp busy
        if(nl < 2 || nl > 8 || envNum("LAMB_RECPACK", 1) == 0)
            return false;
        lamk::RecPackParams q{};
        bool packDir = false;
        uint32_t kind = 0, stream0 = 0;
        for(uint32_t f = 0; f < nl; ++f)
        {
            const lamt_leaf& L = p.leaf[f];
            const bool pk = L.skind == LAMT_K_PHYS && (L.dkind == LAMT_K_BITS_INT || L.dkind == LAMT_K_BITS_FLT);
            const bool up = L.dkind == LAMT_K_PHYS && (L.skind == LAMT_K_BITS_INT || L.skind == LAMT_K_BITS_FLT);
            if(!(pk || up) || (f && pk != packDir))
                return false;
            packDir = pk;
            const lamt_term& vt = pk ? L.s[0] : L.d[0];
            const lamt_stream& vs = p.st[vt.stream];
            const lamt_stream& bs = p.st[pk ? L.d[0].stream : L.s[0].stream];
            if(vt.size != 4 || L.stype != L.ltype || L.dtype != L.ltype || L.ltype == Bool)
                return false;
            const uint8_t k = pk ? L.dkind : L.skind;
            const uint32_t kd = k == LAMT_K_BITS_FLT ? 1 : 0;
            const uint32_t E = pk ? L.dE : L.sE, M = pk ? L.dM : L.sM;
            const uint32_t w = kd ? 1 + E + M : E;
            if(f == 0)
            {
                stream0 = vt.stream;
                kind = kd;
                q.E = E;
                q.M = M;
                q.w = w;
                q.lanes = vs.lanes;
                if(vs.lanes == 1)
                {
                    if(vs.bs != nl * 4)
                        return false;
                }
                else if(vs.lanes >= 32 || 32 % vs.lanes || vs.lshift == 0xFFFFFFFFu || vs.bs != vs.lanes * nl * 4)
                    return false;
                q.lsh = vs.lanes == 1 ? 0 : vs.lshift;
                q.rec = vs.gptr;
            }
            if(vt.stream != stream0 || kd != kind || E != q.E || M != q.M || w < 1 || w > 32 || bs.bs != w)
                return false;
            if(vs.lanes == 1 ? vt.inblock != f * 4 : (vt.inblock != f * 4 * vs.lanes || vt.ls != 4))
                return false;
            if(kd == 1 && L.ltype != F32)
                return false;
            q.bits[f] = bs.gptr;
            if(bs.gptr % 4)
                return false;
            if(up && L.ssigned)
                q.sgnMask |= 1u << f;
        }
        if(begin % q.lanes || (q.rec + begin * nl * 4) % 16)
            return false;
        q.nl = nl;
        q.gmag = ((1u << 24) + 32 * nl - 1) / (32 * nl);
        q.begin = begin;
        q.groups = groups;
        return lamk::rec_pack(q, kind, packDir, s);
    }

    // bit stream -> bit stream for every leaf (4-byte leaf types, fields <= 32 bits, float formats
    // E <= 8, M <= 23): k_repack32, one launch per leaf
    static bool tryRepack(const lamt_params& p, uint64_t begin, uint64_t end, const DeviceImage& si, DeviceImage& di,
                          const Lowered& S, const Lowered& D, cudaStream_t s)
    {
        if(begin % 32 || envNum("LAMB_REPACK", 1) == 0)
            return false;
        const uint64_t groups = (end - begin) / 32;
        if(groups == 0)
            return false;
        std::vector<lamk::RepackParams> jobs;
        for(uint32_t f = 0; f < p.nleaves; ++f)
        {
            const lamt_leaf& L = p.leaf[f];
            const bool sb = L.skind == LAMT_K_BITS_INT || L.skind == LAMT_K_BITS_FLT;
            const bool db = L.dkind == LAMT_K_BITS_INT || L.dkind == LAMT_K_BITS_FLT;
            if(!sb || !db || L.skind != L.dkind || L.stype != L.ltype || L.dtype != L.ltype || scalarSize(L.ltype) != 4)
                return false;
            const bool flt = L.skind == LAMT_K_BITS_FLT;
            // minifloat -> minifloat: one pass when both formats have compile-time codecs (e8m10,
            // e5m10, e4m3, e5m2; k_repack_flt); other formats measured faster staged through the SoA
            // scratch (tools/repack_cmp.py), LAMB_REPACK=2 forces the runtime-format one-pass kernel
            auto fastFmt = [](uint32_t E, uint32_t M)
            { return (E == 8 && M == 10) || (E == 5 && M == 10) || (E == 4 && M == 3) || (E == 5 && M == 2); };
            if(flt && envNum("LAMB_REPACK", 1) != 2 && !(fastFmt(L.sE, L.sM) && fastFmt(L.dE, L.dM)))
                return false;
            if(flt && (L.ltype != F32 || L.sE > 8 || L.sM > 23 || L.dE > 8 || L.dM > 23 || L.sE < 1 || L.dE < 1))
                return false;
            lamk::RepackParams j{};
            j.kind = flt ? 1 : 0;
            j.ws = flt ? 1u + L.sE + L.sM : L.sE;
            j.wd = flt ? 1u + L.dE + L.dM : L.dE;
            j.sE = flt ? L.sE : 8;
            j.sM = flt ? L.sM : 23;
            j.dE = flt ? L.dE : 8;
            j.dM = flt ? L.dM : 23;
            j.ssgn = L.ssigned;
            const lamt_stream& ss = p.st[L.s[0].stream];
            const lamt_stream& ds = p.st[L.d[0].stream];
            if(j.ws < 1 || j.ws > 32 || j.wd < 1 || j.wd > 32 || ss.bs != j.ws || ds.bs != j.wd || ss.gptr % 4 || ds.gptr % 4)
                return false;
            j.src = ss.gptr;
            j.dst = ds.gptr;
            j.begin = begin;
            j.groups = groups;
            jobs.push_back(j);
        }
        for(const auto& j : jobs)
            if(!(j.kind == 1 && envNum("LAMB_REPACK", 1) != 2 ? lamk::repack_flt_fast(j, s) : lamk::repack32(j, s)))
                return false;
        addAccessCounts(p, S, groups * 32, s);
        const uint64_t doneEnd = begin + groups * 32;
        if(doneEnd < end)
            lam_cuda_check(lamk::generic_copy(si.hdr, di.hdr, doneEnd, end, static_cast<uint32_t>(S.roots.size()), S.fac,
                                              D.fac, s, false),
                           "generic_copy(tail)");
        return true;
    }

    // K3/K4: every leaf physical (SoA or AoSoA with 32 | L) <-> bit stream: 4-byte leaves with fields
    // <= 32 bits through k_pack32/k_unpack32, 1/2/8-byte leaves and wider fields through packv.cu
    static bool tryPack(const lamt_params& p, uint64_t begin, uint64_t end, const DeviceImage& si, DeviceImage& di,
                        const Lowered& S, const Lowered& D, cudaStream_t s)
    {
        if(begin % 32 || envNum("LAMB_PACK", 1) == 0)
            return false;
        const uint64_t groups = (end - begin) / 32;
        if(groups == 0)
            return false;
        if(tryRecPack(p, begin, groups, s))
        {
            addAccessCounts(p, S, groups * 32, s);
            const uint64_t doneEnd = begin + groups * 32;
            if(doneEnd < end)
                lam_cuda_check(lamk::generic_copy(si.hdr, di.hdr, doneEnd, end, static_cast<uint32_t>(S.roots.size()),
                                                  S.fac, D.fac, s, false),
                               "generic_copy(tail)");
            return true;
        }
        std::vector<lamk::PackParams> jobs;
        std::vector<std::pair<lamk::PackVParams, uint32_t>> vjobs; // other value sizes / wide fields
        bool packDir = false;
        for(uint32_t f = 0; f < p.nleaves; ++f)
        {
            const lamt_leaf& L = p.leaf[f];
            const bool pk = L.skind == LAMT_K_PHYS && (L.dkind == LAMT_K_BITS_INT || L.dkind == LAMT_K_BITS_FLT);
            const bool up = L.dkind == LAMT_K_PHYS && (L.skind == LAMT_K_BITS_INT || L.skind == LAMT_K_BITS_FLT);
            if(!(pk || up) || (f && pk != packDir))
                return false;
            packDir = pk;
            const lamt_term& vt = pk ? L.s[0] : L.d[0];
            const lamt_stream& vs = p.st[vt.stream];
            const lamt_stream& bs = p.st[pk ? L.d[0].stream : L.s[0].stream];
            const uint32_t vsz = vt.size;
            if((vsz != 1 && vsz != 2 && vsz != 4 && vsz != 8) || L.stype != L.ltype || L.dtype != L.ltype
               || L.ltype == Bool)
                return false;
            const bool soa = vs.lanes == 1 && vs.bs == vsz;
            const bool aosoa = vs.lanes % 32 == 0 && vs.lshift != 0xFFFFFFFFu && vt.ls == vsz;
            if(!(soa || aosoa))
                return false;
            const uint8_t kind = pk ? L.dkind : L.skind;
            const uint32_t kd = kind == LAMT_K_BITS_FLT ? 1 : 0;
            const uint32_t E = pk ? L.dE : L.sE, M = pk ? L.dM : L.sM;
            const uint32_t w = kd ? 1 + E + M : E;
            if(w < 1 || w > 64 || bs.bs != w || (kd == 0 && w > 8 * vsz))
                return false;
            if(kd == 1 && !((L.ltype == F32 && vsz == 4) || (L.ltype == F64 && vsz == 8)))
                return false;
            const uint64_t vals = vs.gptr + (soa ? vt.inblock : 0);
            if((vals + (soa ? 0 : vt.inblock)) % 16 || bs.gptr % 16)
                return false;
            if(vsz != 4 || w > 32)
            {
                lamk::PackVParams v{};
                v.vals = vals;
                v.bits = bs.gptr;
                v.begin = begin;
                v.groups = groups;
                v.w = w;
                v.kind = kd;
                v.sgn = pk ? 0 : L.ssigned;
                v.E = E;
                v.M = M;
                v.vbs = vs.bs;
                v.vl = vs.lanes;
                v.vsh = soa ? 0 : vs.lshift;
                v.vinb = soa ? 0 : vt.inblock;
                vjobs.emplace_back(v, vsz);
                continue;
            }
            lamk::PackParams j{};
            j.kind = kd;
            j.E = E;
            j.M = M;
            j.w = w;
            j.sgn = pk ? 0 : L.ssigned;
            j.valType = L.ltype;
            j.vals = vals;
            j.vinb = soa ? 0 : vt.inblock;
            j.vbs = vs.bs;
            j.vl = vs.lanes;
            j.vsh = soa ? 0 : vs.lshift;
            j.bits = bs.gptr;
            j.begin = begin;
            j.groups = groups;
            j.facS = 0; // counted in closed form below (fac_add)
            j.facD = 0;
            j.facSrc = p.facSrc;
            j.facDst = p.facDst;
            j.leaf = f;
            j.nleaves = p.nleaves;
            jobs.push_back(j);
        }
        for(size_t a = 0; a < vjobs.size();)
        {
            size_t b = a + 1;
            const lamk::PackVParams& v0 = vjobs[a].first;
            while(b < vjobs.size() && b - a < 8 && vjobs[b].second == vjobs[a].second && vjobs[b].first.w == v0.w
                  && vjobs[b].first.kind == v0.kind && vjobs[b].first.E == v0.E && vjobs[b].first.M == v0.M)
                ++b;
            std::vector<lamk::PackVParams> grp;
            for(size_t k = a; k < b; ++k)
                grp.push_back(vjobs[k].first);
            if(!lamk::packv(grp.data(), static_cast<uint32_t>(grp.size()), vjobs[a].second, packDir, s))
                throw std::runtime_error(std::string("packv launch failed: ") + cudaGetErrorString(cudaGetLastError()));
            a = b;
        }
        for(const auto& j : jobs)
            if(!lamk::pack32(j, packDir, s))
                throw std::runtime_error(std::string("pack32 launch failed: ") + cudaGetErrorString(cudaGetLastError()));
        addAccessCounts(p, S, groups * 32, s);
        const uint64_t doneEnd = begin + groups * 32;
        if(doneEnd < end)
            lam_cuda_check(lamk::generic_copy(si.hdr, di.hdr, doneEnd, end, static_cast<uint32_t>(S.roots.size()), S.fac,
                                              D.fac, s, false),
                           "generic_copy(tail)");
        return true;
    }

    // K5: record-contiguous f64 -> changetype f32 -> bytesplit into 1-byte SoA planes
    // Bytesplit against a record-contiguous side (planes.cu): every leaf an SB-byte physical leaf
    // of one packed record stream on one side, and byte planes (packed u8 arrays) on the other,
    // either the same type (plain bytesplit) or f64 records <-> f32 planes (ChangeType, C5).
    static bool trySplit(const lamt_params& p, uint64_t begin, uint64_t end, const DeviceImage& si, DeviceImage& di,
                         const Lowered& S, const Lowered& D, cudaStream_t s)
    {
        if(begin % 4 || p.nleaves > 8 || envNum("LAMB_SPLITK", 1) == 0)
            return false;
        const uint32_t nl = p.nleaves;
        const bool toPlanes = p.leaf[0].skind == LAMT_K_PHYS;
        lamk::PlaneParams pp{};
        const lamt_term& r0 = toPlanes ? p.leaf[0].s[0] : p.leaf[0].d[0];
        const uint32_t sb = r0.size;
        bool cvt = false;
        for(uint32_t f = 0; f < nl; ++f)
        {
            const lamt_leaf& L = p.leaf[f];
            const uint8_t recKind = toPlanes ? L.skind : L.dkind, plKind = toPlanes ? L.dkind : L.skind;
            const uint32_t pn = toPlanes ? L.dn : L.sn;
            if(recKind != LAMT_K_PHYS || plKind != LAMT_K_SPLIT)
                return false;
            const bool pure = L.stype == L.ltype && L.ltype == L.dtype && pn == sb;
            const bool conv = sb == 8 && pn == 4
                && (toPlanes ? (L.stype == F64 && L.ltype == F64 && L.dtype == F32)
                             : (L.stype == F32 && L.ltype == F64 && L.dtype == F64));
            if(!(pure || conv) || (f > 0 && conv != cvt))
                return false;
            cvt = conv;
            const lamt_term& t = toPlanes ? L.s[0] : L.d[0];
            const lamt_stream& st = p.st[t.stream];
            if(t.stream != r0.stream || t.size != sb || t.inblock != f * sb || st.lanes != 1 || st.bs != nl * sb)
                return false;
            for(uint32_t k = 0; k < pn; ++k)
            {
                const lamt_term& d = toPlanes ? L.d[k] : L.s[k];
                const lamt_stream& ds = p.st[d.stream];
                if(ds.lanes != 1 || ds.bs != 1)
                    return false;
                pp.plane[f][k] = ds.gptr + d.inblock;
                if((pp.plane[f][k] + begin) % 4)
                    return false;
            }
        }
        if(sb != 4 && sb != 8)
            return false;
        pp.rec = p.st[r0.stream].gptr;
        if((pp.rec + begin * nl * sb) % 16)
            return false;
        pp.begin = begin;
        pp.groups = (end - begin) / 4;
        pp.nl = nl;
        if(pp.groups == 0 || !lamk::planes_copy(pp, sb, cvt, toPlanes, s))
            return false;
        addAccessCounts(p, S, pp.groups * 4, s);
        const uint64_t doneEnd = begin + pp.groups * 4;
        if(doneEnd < end)
            lam_cuda_check(lamk::generic_copy(si.hdr, di.hdr, doneEnd, end, static_cast<uint32_t>(S.roots.size()), S.fac,
                                              D.fac, s, false),
                           "generic_copy(tail)");
        return true;
    }

    static bool launchTileData(const Lowered& S, const DeviceImage& si, const std::vector<uint8_t*>& sptr,
                               const Lowered& D, DeviceImage& di, const std::vector<uint8_t*>& dptr, uint64_t begin,
                               uint64_t end, cudaStream_t s);

    // Heatmap accounting when every terminal of the side is a physical byte range (PHYS leaves,
    // ChangeType over PHYS, byte splits): copy_generic.cu k_heat_phys.  False = not eligible.
    static bool heatPhys(const Lowered& L, const DeviceImage& img, uint64_t begin, uint64_t end, cudaStream_t s)
    {
        if(envNum("LAMB_HEAT_PHYS", 1) == 0 || !img.heat || L.heatGran == 0)
            return false;
        std::vector<std::vector<lamk::HeatTerm>> perStream(L.streams.size());
        std::vector<uint32_t> stack;
        for(uint16_t r : L.roots)
        {
            stack.assign(1, r);
            while(!stack.empty())
            {
                const lamp_node& nd = L.nodes[stack.back()];
                stack.pop_back();
                switch(nd.kind)
                {
                case LAMP_PHYS:
                    perStream[nd.stream].push_back({nd.a, nd.b, static_cast<uint32_t>(scalarSize(nd.type))});
                    break;
                case LAMP_CONVERT:
                    stack.push_back(nd.child);
                    break;
                case LAMP_SPLIT:
                    for(uint32_t k = 0; k < nd.nchild; ++k)
                        stack.push_back(nd.child + k);
                    break;
                case LAMP_NULL:
                    break;
                default:
                    return false; // bit streams: the generic range pass
                }
            }
        }
        lamk::HeatParams hp{};
        hp.heat = static_cast<unsigned long long*>(img.heat);
        hp.heatOff = reinterpret_cast<const uint64_t*>(static_cast<const uint8_t*>(img.mem) + img.offHeatOff);
        hp.begin = begin;
        hp.end = end;
        hp.gran = L.heatGran;
        hp.gshift = 64;
        if((L.heatGran & (L.heatGran - 1)) == 0)
            for(uint32_t k = 0; k < 64; ++k)
                if((uint64_t{1} << k) == L.heatGran)
                    hp.gshift = k;
        const uint32_t maxW = 6144;
        uint64_t E = 1u << 16, unit = 1;
        uint32_t nt = 0;
        for(size_t k = 0; k < L.streams.size(); ++k)
        {
            if(perStream[k].empty())
                continue;
            const lamp_stream& st = L.streams[k];
            if(st.kind != LAMS_PHYS || hp.nstreams >= 64 || nt + perStream[k].size() > 256)
                return false;
            lamk::HeatStream& h = hp.st[hp.nstreams++];
            h.base0 = st.base0;
            h.bs = st.block_stride;
            h.lanes = st.lanes;
            h.lshift = st.lane_shift;
            h.nr = st.nr;
            h.t0 = nt;
            for(const auto& t : perStream[k])
                hp.term[nt++] = t;
            h.t1 = nt;
            // elements per CTA such that the block window of this stream fits in maxW counters
            const uint64_t e = (maxW - 4) * L.heatGran * st.lanes / st.block_stride;
            E = std::min<uint64_t>(E, e);
            unit = lcm64(unit, st.lanes);
        }
        if(hp.nstreams == 0)
            return true; // nothing physical to touch (Null leaves only)
        // enough CTAs to fill the SMs (several per SM), each element run still long enough
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t fill = (end - begin) / (static_cast<uint64_t>(lamk::sm_count(dev)) * 8);
        if(fill >= 4096 && fill < E)
            E = fill;
        E = E / unit * unit;
        if(E < 64 || begin % unit)
            return false;
        hp.E = E;
        hp.maxWindow = maxW;
        lam_cuda_check(lamk::heat_phys(hp, s), "heat_phys");
        return true;
    }


    // LAMB_TRACE=1: the path each copy takes, on stderr (diagnostics only)
    static void trace(const char* what)
    {
        static const bool on = std::getenv("LAMB_TRACE") && std::getenv("LAMB_TRACE")[0] == '1';
        if(on)
            std::fprintf(stderr, "lamb path: %s\n", what);
    }

    // physical pairs no fixed kernel covers (mixed leaf sizes, unaligned packed records, lane
    // counts no vector group fits, padded destinations): a kernel generated for the exact pair
    // (jit.cpp); false when NVRTC is unavailable or the pair does not fit its 16-byte groups
    static bool tryJit(const lamt_params& p, uint64_t begin, uint64_t end, const DeviceImage& si, DeviceImage& di,
                       const Lowered& S, const Lowered& D, cudaStream_t s)
    {
        uint64_t doneEnd = begin;
        if(!lamjit::tryCopy(p, begin, end, &doneEnd, s))
            return false;
        addAccessCounts(p, S, doneEnd - begin, s);
        if(doneEnd < end)
            lam_cuda_check(lamk::generic_copy(si.hdr, di.hdr, doneEnd, end, static_cast<uint32_t>(S.roots.size()), S.fac,
                                              D.fac, s, false),
                           "generic_copy(tail)");
        return true;
    }

    // the data moves through the tile kernels (none of which counts heat); a Heatmap on either
    // side is then accounted over the whole range in one pass that touches ranges, not data
    static bool launchTile(const Lowered& S, const DeviceImage& si, const std::vector<uint8_t*>& sptr, const Lowered& D,
                           DeviceImage& di, const std::vector<uint8_t*>& dptr, uint64_t begin, uint64_t end,
                           cudaStream_t s)
    {
        if(!launchTileData(S, si, sptr, D, di, dptr, begin, end, s))
            return false;
        const uint32_t nl = static_cast<uint32_t>(S.roots.size());
        if(S.heat && !heatPhys(S, si, begin, end, s))
            lam_cuda_check(lamk::heat_account(si.hdr, begin, end, nl, s), "heat_account(src)");
        if(D.heat && !heatPhys(D, di, begin, end, s))
            lam_cuda_check(lamk::heat_account(di.hdr, begin, end, nl, s), "heat_account(dst)");
        return true;
    }

    static bool launchTileData(const Lowered& S, const DeviceImage& si, const std::vector<uint8_t*>& sptr,
                               const Lowered& D, DeviceImage& di, const std::vector<uint8_t*>& dptr, uint64_t begin,
                               uint64_t end, cudaStream_t s)
    {
        Plan pl = makePlan(S, D);
        if(!pl.ok)
            return trace("no tile plan"), false;
        lamt_params& p = pl.p;
        const uint64_t n = end - begin;
        const uint64_t ntiles = n / p.T;
        if(ntiles == 0 || ntiles > 0xFFFFFFFFull)
            return false;
        p.begin = begin;
        p.ntiles = static_cast<uint32_t>(ntiles);
        uint32_t tma = 0;
        for(uint32_t k = 0; k < p.nsrc + p.ndst; ++k)
        {
            lamt_stream& t = p.st[k];
            const bool isSrc = k < p.nsrc;
            uint8_t* g = isSrc ? sptr[pl.srcStreams[k]] : dptr[pl.dstStreams[k - p.nsrc]];
            t.gptr = reinterpret_cast<unsigned long long>(g);
            const uint64_t first = reinterpret_cast<uint64_t>(g) + tileOff(t, begin);
            t.tma = (first % 16 == 0) && (t.tile_bytes % 16 == 0);
            if(isSrc && t.tma)
                tma += t.tile_bytes;
        }
        p.tma_bytes = tma;
        p.any_coop = 0;
        for(uint32_t k = 0; k < p.nsrc + p.ndst; ++k)
            p.any_coop |= p.st[k].tile_bytes && !p.st[k].tma;
        p.facSrc = reinterpret_cast<unsigned long long>(si.facDev);
        p.facDst = reinterpret_cast<unsigned long long>(di.facDev);
        if(p.dst_holes)
        {
            if(tryJit(p, begin, end, si, di, S, D, s))
                return trace("jit (holes)"), true;
            trace("warp tile (holes)");
            return envNum("LAMB_WARP_TILE", 1) != 0 && tryWarpTile(p, S, D, si, di, begin, end, s);
        }
        if(p.uni && envNum("LAMB_VEC", 1) != 0 && tryVec(p, begin, end, si, di, S, D, s))
            return trace("vec"), true;
        if(!p.uni && tryRepack(p, begin, end, si, di, S, D, s))
            return trace("repack"), true;
        if(!p.uni && tryPack(p, begin, end, si, di, S, D, s))
            return trace("pack"), true;
        if(!p.uni && trySplit(p, begin, end, si, di, S, D, s))
            return trace("planes"), true;
        if(!p.uni && tryVecConvert(p, begin, end, si, di, S, D, s))
            return trace("vec convert"), true;
        if(!p.uni && tryVecMulti(p, begin, end, si, di, S, D, s))
            return trace("vec multi"), true;
        // uniform pairs get here when the register transpose cannot take them (AoSoA lanes that are not
        // a power of two or not a multiple of 16/size): the generated kernel measured 0.81-0.99 of HBM
        // on them against 0.59-0.71 for k_uniform_direct (profiles/r02/jit/jit_uni.log)
        if((!p.uni || envNum("LAMB_JIT_UNI", 1) != 0) && tryJit(p, begin, end, si, di, S, D, s))
            return trace("jit"), true;
        // uniform pairs the register transpose cannot take (AoSoA lanes not a multiple of 16/size,
        // non-power-of-two lanes): direct per-element moves through L1 (k_uniform_direct), block /
        // lane by a magic multiply -- measured 1.7x over the warp-tile transpose (aosoa:2, aosoa:3)
        const uint64_t maxL = std::max<uint64_t>(std::max<uint64_t>(p.ul_s, p.ul_d), 1);
        if(p.uni && envNum("LAMB_DIRECT", 1) != 0 && end < (uint64_t{1} << 32) / maxL)
        {
            lamt_params q = p;
            q.umag_s = q.ul_s > 1 ? static_cast<uint32_t>(((uint64_t{1} << 32) + q.ul_s - 1) / q.ul_s) : 0;
            q.umag_d = q.ul_d > 1 ? static_cast<uint32_t>(((uint64_t{1} << 32) + q.ul_d - 1) / q.ul_d) : 0;
            q.facS = q.facD = 0;
            trace("uniform direct");
            lam_cuda_check(lamk::uniform_direct(q, end - begin, s), "uniform_direct");
            addAccessCounts(p, S, end - begin, s);
            return true;
        }
        if(p.uni && !p.any_coop && envNum("LAMB_UNI_WARP", 1) != 0)
        {
            // warp-tile transpose: WT elements per warp tile, equal-size images per side
            const uint64_t unit = lcm64(lcm64(S.shardUnit, D.shardUnit), 32);
            uint64_t wt = static_cast<uint64_t>(envNum("LAMB_WT", 64));
            wt = std::max<uint64_t>(unit, wt / unit * unit);
            lamt_params q = p;
            q.T = static_cast<uint32_t>(wt);
            bool ok = true;
            uint32_t imgS = 0, imgD = 0;
            for(uint32_t k = 0; k < q.nsrc + q.ndst && ok; ++k)
            {
                lamt_stream& t = q.st[k];
                const uint64_t bytes = wt / t.lanes * t.bs;
                uint32_t& img = k < q.nsrc ? imgS : imgD;
                if(img == 0)
                    img = static_cast<uint32_t>(bytes);
                ok = bytes == img && bytes % 16 == 0 && bytes <= 16384;
                t.tile_bytes = static_cast<uint32_t>(bytes);
                t.smem_off = (k < q.nsrc ? k : k - q.nsrc) * img;
            }
            const uint64_t ntw = (end - begin) / wt;
            if(ok && ntw > 0 && ntw <= 0xFFFFFFFFull)
            {
                q.src_bytes = q.nsrc * imgS;
                q.dst_bytes = q.ndst * imgD;
                for(uint32_t f = 0; f < q.nleaves; ++f)
                {
                    q.uoff_s[f] = q.st[q.leaf[f].s[0].stream].smem_off + q.leaf[f].s[0].inblock;
                    q.uoff_d[f] = q.st[q.leaf[f].d[0].stream].smem_off + q.leaf[f].d[0].inblock;
                }
                if(8ull * (q.src_bytes + q.dst_bytes) <= 200 * 1024)
                {
                    trace("uniform warp");
                    lam_cuda_check(lamk::uniform_warp(q, static_cast<uint32_t>(ntw), s), "uniform_warp");
                    const uint64_t doneEnd = begin + ntw * wt;
                    if(doneEnd < end)
                        lam_cuda_check(lamk::generic_copy(si.hdr, di.hdr, doneEnd, end,
                                                          static_cast<uint32_t>(S.roots.size()), S.fac, D.fac, s, false),
                                       "generic_copy(tail)");
                    return true;
                }
            }
        }
        if(envNum("LAMB_WARP_TILE", 1) != 0 && tryWarpTile(p, S, D, si, di, begin, end, s))
            return trace("warp tile"), true;
        trace("tma tile");
        lam_cuda_check(lamk::tile_copy(p, pl.smem, pl.ctas, s), "tile_copy");
        const uint64_t doneEnd = begin + ntiles * p.T;
        if(doneEnd < end)
            lam_cuda_check(lamk::generic_copy(si.hdr, di.hdr, doneEnd, end, static_cast<uint32_t>(S.roots.size()),
                                              S.fac, D.fac, s, false),
                           "generic_copy(tail)");
        return true;
    }

    bool tileCopyImages(const Lowered& S, const DeviceImage& si, const Lowered& D, DeviceImage& di, uint64_t begin,
                        uint64_t end, cudaStream_t s)
    {
        std::vector<uint8_t*> sp(S.streams.size()), dp(D.streams.size());
        if(!S.streams.empty())
            std::memcpy(sp.data(), si.host.data() + si.offPtrs, sp.size() * sizeof(uint8_t*));
        if(!D.streams.empty())
            std::memcpy(dp.data(), di.host.data() + di.offPtrs, dp.size() * sizeof(uint8_t*));
        return launchTile(S, si, sp, D, di, dp, begin, end, s);
    }

    bool tileCopyPtrs(const Lowered& S, const DeviceImage& si, uint8_t* const* sptr, const Lowered& D, DeviceImage& di,
                      uint8_t* const* dptr, uint64_t begin, uint64_t end, cudaStream_t s)
    {
        std::vector<uint8_t*> sp(sptr, sptr + S.streams.size()), dp(dptr, dptr + D.streams.size());
        return launchTile(S, si, sp, D, di, dp, begin, end, s);
    }

    bool tileCopy(const lam_view& src, lam_view& dst, uint64_t begin, uint64_t end, cudaStream_t s)
    {
        return tileCopyImages(*src.L, src.img, *dst.L, dst.img, begin, end, s);
    }

    bool tileEligible(const Lowered& S, const Lowered& D)
    {
        return makePlan(S, D).ok;
    }
} // namespace lamhost

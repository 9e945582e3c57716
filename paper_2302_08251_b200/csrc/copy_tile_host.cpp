// Tile-engine planning on the host: decides whether a (src, dst) layout pair can run on
// the TMA-staged tile kernel, sizes the tile, places stream images in shared memory and
// fills the kernel parameter block.  Pairs it cannot express fall back to the generic
// interpreter kernel (copy_generic.cu).
#include "capi_internal.hpp"
#include "tile.h"

#include <cstring>

namespace lamk
{
    cudaError_t tile_copy(const lamt_params& p, uint32_t smemBytes, uint32_t ctasPerSm, cudaStream_t s);
}

using namespace lamb;

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
                if(isDst && !st.holefree)
                    return false; // whole-image stores would clobber bytes copyView never writes
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
            Plan pl;
            if(S.heat || D.heat)
                return pl;
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
            const double stageTarget = 48.0 * 1024;
            if(unit > (1u << 20) || bpe * unit > 100.0 * 1024)
                return pl;
            uint64_t T = static_cast<uint64_t>(stageTarget / (bpe > 0 ? bpe : 1) / unit) * unit;
            if(T < unit)
                T = unit;
            if(T > (1u << 20))
                T = (1u << 20) / unit * unit;

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
                fillStream(p.st[nsrc + k], D.streams[pl.dstStreams[k]]);
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
            pl.smem = 2 * (p.src_bytes + p.dst_bytes);
            if(pl.smem > 220 * 1024)
                return pl;
            pl.ctas = pl.smem <= 110 * 1024 ? 2 : 1;
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

    static bool launchTile(const Lowered& S, const DeviceImage& si, const std::vector<uint8_t*>& sptr, const Lowered& D,
                           DeviceImage& di, const std::vector<uint8_t*>& dptr, uint64_t begin, uint64_t end,
                           cudaStream_t s)
    {
        Plan pl = makePlan(S, D);
        if(!pl.ok)
            return false;
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
        p.facSrc = reinterpret_cast<unsigned long long>(si.facDev);
        p.facDst = reinterpret_cast<unsigned long long>(di.facDev);
        lam_cuda_check(lamk::tile_copy(p, pl.smem, pl.ctas, s), "tile_copy");
        const uint64_t doneEnd = begin + ntiles * p.T;
        if(doneEnd < end)
            lam_cuda_check(lamk::generic_copy(si.hdr, di.hdr, doneEnd, end, static_cast<uint32_t>(S.roots.size()),
                                              S.fac, D.fac, s),
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

// Tile-engine planning on the host: decides whether a (src, dst) layout pair can run on
// the TMA-staged tile kernel, sizes the tile, places stream images in shared memory and
// fills the kernel parameter block.  Pairs it cannot express fall back to the generic
// interpreter kernel (copy_generic.cu).
#include "capi_internal.hpp"
#include "tile.h"

#include <cstdlib>
#include <cstring>

namespace lamk
{
    cudaError_t tile_copy(const lamt_params& p, uint32_t smemBytes, uint32_t ctasPerSm, cudaStream_t s);
    cudaError_t uniform_direct(const lamt_params& p, uint64_t n, cudaStream_t s);
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
        p.any_coop = 0;
        for(uint32_t k = 0; k < p.nsrc + p.ndst; ++k)
            p.any_coop |= p.st[k].tile_bytes && !p.st[k].tma;
        p.facSrc = reinterpret_cast<unsigned long long>(si.facDev);
        p.facDst = reinterpret_cast<unsigned long long>(di.facDev);
        if(p.uni && !p.facS && !p.facD && envNum("LAMB_DIRECT", 0) != 0 && (p.ush_s != 0xFFFFFFFFu || p.ul_s == 1)
           && (p.ush_d != 0xFFFFFFFFu || p.ul_d == 1))
        {
            lam_cuda_check(lamk::uniform_direct(p, end - begin, s), "uniform_direct");
            return true;
        }
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

// Run-time specialised copy kernels for layout pairs (NVRTC).
//
// The reference's mappings are run-time objects (mapping.hpp:44-155). LLAMA, the library the
// paper describes, resolves them at compile time. For the pairs the fixed kernels do not cover,
// this path does what LLAMA's compile-time mappings do. Those pairs are records with mixed leaf
// sizes, padded destinations, byte planes against anything but a packed record, ChangeType
// leaves, and AoSoA lane counts no vector group fits. The path generates a kernel for the exact
// pair of lowered layouts, with every block stride, lane count and leaf offset a literal. It
// compiles the kernel with NVRTC for sm_100a, once per pair and cached, and launches it.
//
// The generated kernel:
// - A thread owns G consecutive elements. G is chosen so that, for every stream of both sides,
//   the bytes of those elements are whole 16-byte vectors: G/L whole blocks of a record or
//   AoSoA<L> stream ("block span"), or one run of G values of a leaf inside an AoSoA<L> block
//   ("run span"). A block span of exactly 8 bytes per group (a 1-byte SoA leaf or byte plane at
//   G = 8) is accessed with 8-byte vectors. A side is physical leaves or byte planes (Bytesplit
//   term k = byte k).
// - Every destination word is assembled from source words by PRMT byte permutes with
//   compile-time selectors. Bool bytes are canonicalised (__vcmpne4).
// - ChangeType leaves (f32 <-> f64, integer widen / narrow) are converted in registers with the
//   reference's rules (scalar.hpp:295-319).
// - Destination bytes copyView never writes (padding) come from the destination's own words,
//   read first.
// - A destination span that is byte for byte a source span is a warp-coalesced pass-through copy.
// - Block spans of more than one vector per thread can move through warp-private shared-memory
//   slabs (coalesced 16-byte accesses, odd lane stride).
// - The staging mode (destination slabs, source slabs, both, none) and a register cap are
//   autotuned on the first copy of a pair at >= 2^22 elements: eight variants, compiled in
//   parallel and timed on the copy itself. Smaller copies use a heuristic.
// The semantics are copyView's fieldwise loop (view.cpp:184-188).
//
// NVRTC is loaded with dlopen. When it is absent or a compile fails, the pair falls back to the
// warp-tile engine (never to the CPU).
//
// Knobs:
// - LAMB_JIT=0 disables this path.
// - LAMB_JIT_STAGE=1|s|d|0 forces a staging mode, and LAMB_JIT_MINB a register cap.
// - LAMB_JIT_TUNE=0 turns autotuning off.
// - LAMB_JIT_HALF=0 disables 8-byte spans (1-byte leaves at G = 8).
// - LAMB_JIT_DUMP=file appends the generated sources to that file; LAMB_JIT_LOG=1 prints compile errors.
#include "capi_internal.hpp"
#include "launch.h"
#include "tile.h"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

namespace lamjit
{
    namespace
    {
        typedef struct _nvrtcProgram* nvrtcProgram;
        struct Nvrtc
        {
            bool ok = false;
            int (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
            int (*compile)(nvrtcProgram, int, const char* const*) = nullptr;
            int (*cubinSize)(nvrtcProgram, size_t*) = nullptr;
            int (*cubin)(nvrtcProgram, char*) = nullptr;
            int (*logSize)(nvrtcProgram, size_t*) = nullptr;
            int (*log)(nvrtcProgram, char*) = nullptr;
            int (*destroy)(nvrtcProgram*) = nullptr;
        };

        Nvrtc& nvrtc()
        {
            static Nvrtc n;
            static std::once_flag once;
            std::call_once(
                once,
                [&]
                {
                    void* h = nullptr;
                    for(const char* name : {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"})
                        if((h = dlopen(name, RTLD_NOW | RTLD_LOCAL)))
                            break;
                    if(!h)
                        return;
                    n.create = reinterpret_cast<decltype(n.create)>(dlsym(h, "nvrtcCreateProgram"));
                    n.compile = reinterpret_cast<decltype(n.compile)>(dlsym(h, "nvrtcCompileProgram"));
                    n.cubinSize = reinterpret_cast<decltype(n.cubinSize)>(dlsym(h, "nvrtcGetCUBINSize"));
                    n.cubin = reinterpret_cast<decltype(n.cubin)>(dlsym(h, "nvrtcGetCUBIN"));
                    n.logSize = reinterpret_cast<decltype(n.logSize)>(dlsym(h, "nvrtcGetProgramLogSize"));
                    n.log = reinterpret_cast<decltype(n.log)>(dlsym(h, "nvrtcGetProgramLog"));
                    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "nvrtcDestroyProgram"));
                    n.ok = n.create && n.compile && n.cubinSize && n.cubin && n.logSize && n.log && n.destroy;
                });
            return n;
        }

        // compiled kernels by generated source (a failed compile is remembered as nullptr)
        std::mutex g_mu;
        std::map<std::string, cudaKernel_t> g_cache;
        std::map<std::string, cudaKernel_t> g_keyCache; // by plan key (jit.cpp tryCopy)
        std::map<std::string, std::pair<char, int>> g_modeCache; // autotuned (staging mode, minB) per pair

        cudaKernel_t compile(const std::string& src)
        {
            {
                std::lock_guard<std::mutex> lk(g_mu);
                auto it = g_cache.find(src);
                if(it != g_cache.end())
                    return it->second;
            }
            Nvrtc& n = nvrtc();
            cudaKernel_t kern = nullptr;
            if(n.ok)
            {
                nvrtcProgram prog = nullptr;
                if(n.create(&prog, src.c_str(), "lamjit.cu", 0, nullptr, nullptr) == 0)
                {
                    const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-default-device"};
                    const int rc = n.compile(prog, 3, opts);
                    if(rc != 0 && std::getenv("LAMB_JIT_LOG"))
                    {
                        size_t ls = 0;
                        n.logSize(prog, &ls);
                        std::string lg(ls, '\0');
                        n.log(prog, lg.data());
                        std::fprintf(stderr, "lamjit: compile failed (%d):\n%s\n%s\n", rc, lg.c_str(), src.c_str());
                    }
                    if(rc == 0)
                    {
                        size_t sz = 0;
                        n.cubinSize(prog, &sz);
                        std::vector<char> bin(sz);
                        n.cubin(prog, bin.data());
                        cudaLibrary_t lib = nullptr;
                        if(cudaLibraryLoadData(&lib, bin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) == cudaSuccess)
                        {
                            if(cudaLibraryGetKernel(&kern, lib, "lamjit_copy") != cudaSuccess)
                                kern = nullptr;
                        }
                        cudaGetLastError(); // a failed load must not poison later launches
                    }
                    n.destroy(&prog);
                }
            }
            std::lock_guard<std::mutex> lk(g_mu);
            g_cache[src] = kern;
            return kern;
        }
    } // namespace

    // one side of a pair, as 16-byte vectors of the G-element group
    struct Span
    {
        bool run = false;            // false: G/L whole blocks (address base + g * gstride)
        unsigned long long base = 0; // run: leaf-run base (stream + inblock); block: stream + (begin/L)*bs
        uint64_t gstride = 0;        // block: bytes per group
        uint32_t lsh = 0, bs = 0, lmask = 0, ls = 0; // run: base + (e0 >> lsh)*bs + (e0 & lmask)*ls
        uint32_t bytes = 0;          // multiple of 16 (a half span occupies 16 in the word space)
        uint32_t word0 = 0;          // first word of the span in the side's word space
        bool half = false;           // block span of 8 bytes per group (words 2, 3 are padding)
    };

    bool tryCopy(const lamt_params& p, uint64_t begin, uint64_t end, uint64_t* doneEnd, cudaStream_t s)
    {
        const char* env = std::getenv("LAMB_JIT");
        if(env && env[0] == '0')
            return false;
        const uint32_t nl = p.nleaves;
        if(nl < 1 || nl > LAMT_MAX_LEAVES)
            return false;
        // every leaf a byte move, or a ChangeType conversion (computed.cpp:228-404) between f32 and
        // f64 or between integer types; a side is one physical term of its stored size, or byte
        // planes (Bytesplit, computed.cpp:405-502: term k holds byte k)
        auto isInt = [](int t) { return t <= lamb::U64; };
        auto cvtOk = [&](int a, int b)
        {
            return a == b || ((a == lamb::F32 || a == lamb::F64) && (b == lamb::F32 || b == lamb::F64)) || (isInt(a) && isInt(b));
        };
        std::vector<uint32_t> ssz(nl), dsz(nl);
        std::vector<bool> conv(nl, false);
        for(uint32_t f = 0; f < nl; ++f)
        {
            const lamt_leaf& L = p.leaf[f];
            if(!cvtOk(L.stype, L.ltype) || !cvtOk(L.ltype, L.dtype))
                return false;
            conv[f] = L.stype != L.ltype || L.ltype != L.dtype;
            ssz[f] = static_cast<uint32_t>(lamb::scalarSize(L.stype));
            dsz[f] = static_cast<uint32_t>(lamb::scalarSize(L.dtype));
            for(int side = 0; side < 2; ++side)
            {
                const uint8_t kind = side ? L.dkind : L.skind;
                const uint8_t nt = side ? L.dn : L.sn;
                const lamt_term* t = side ? L.d : L.s;
                const uint32_t sz = side ? dsz[f] : ssz[f];
                if(kind == LAMT_K_PHYS)
                {
                    if(t[0].size != sz)
                        return false;
                }
                else if(kind == LAMT_K_SPLIT)
                {
                    if(nt != sz)
                        return false;
                    for(uint32_t k = 0; k < nt; ++k)
                        if(t[k].size != 1)
                            return false;
                }
                else
                    return false;
            }
        }
        // the smallest group size G for which every stream of both sides is whole vectors
        std::vector<uint32_t> candidates = {4, 8, 16, 32, 12, 24, 48};
        std::vector<Span> sv[2];
        std::vector<int> spanOfStream[2];
        // leaf f, element j, byte b -> (span word index, byte) on each side
        const char* envHalf = std::getenv("LAMB_JIT_HALF");
        const bool halfOk = !(envHalf && envHalf[0] == '0');
        auto build = [&](uint32_t G, bool src, std::vector<Span>& spans, std::vector<int>& sos,
                         std::vector<uint32_t>& wordOf) -> bool
        {
            spans.clear();
            sos.assign(LAMT_MAX_STREAMS, -1);
            uint32_t words = 0;
            wordOf.assign(size_t(nl) * G * 16, 0xFFFFFFFFu);
            for(uint32_t f = 0; f < nl; ++f)
            {
                const lamt_leaf& lf = p.leaf[f];
                const bool split = (src ? lf.skind : lf.dkind) == LAMT_K_SPLIT;
                const uint32_t vs = src ? ssz[f] : dsz[f];
                const uint32_t nt = split ? vs : 1;
                for(uint32_t k = 0; k < nt; ++k)
                {
                    const lamt_term& t = src ? lf.s[k] : lf.d[k];
                    const lamt_stream& st = p.st[t.stream];
                    const uint32_t L = st.lanes;
                    int run = -1;
                    if(G % L == 0)
                    {
                        if(sos[t.stream] < 0)
                        {
                            Span sp;
                            sp.run = false;
                            sp.base = st.gptr + (begin / L) * st.bs;
                            sp.gstride = uint64_t(G / L) * st.bs;
                            sp.bytes = static_cast<uint32_t>(sp.gstride);
                            if(sp.bytes == 8 && sp.base % 8 == 0 && halfOk)
                            {
                                // 8 bytes per group (a 1-byte SoA leaf at G = 8): one 8-byte access
                                sp.half = true;
                                sp.bytes = 16;
                            }
                            else if(sp.bytes % 16 || sp.base % 16 || sp.gstride % 16)
                                return false;
                            if(words + sp.bytes / 4 > 4096)
                                return false;
                            sp.word0 = words;
                            words += sp.bytes / 4;
                            sos[t.stream] = static_cast<int>(spans.size());
                            spans.push_back(sp);
                        }
                    }
                    else if(L % G == 0 && st.lshift != 0xFFFFFFFFu)
                    {
                        Span sp;
                        sp.run = true;
                        sp.base = st.gptr + t.inblock;
                        sp.lsh = st.lshift;
                        sp.bs = st.bs;
                        sp.lmask = L - 1;
                        sp.ls = t.ls;
                        sp.bytes = G * t.size;
                        if(t.ls == t.size && sp.bytes == 8 && sp.base % 8 == 0 && st.bs % 8 == 0 && halfOk)
                        {
                            sp.half = true; // 8 bytes per group: one 8-byte access
                            sp.bytes = 16;
                        }
                        else if(t.ls != t.size || sp.bytes % 16 || sp.base % 16 || st.bs % 16)
                            return false;
                        sp.word0 = words;
                        words += sp.bytes / 4;
                        run = static_cast<int>(spans.size());
                        spans.push_back(sp);
                    }
                    else
                        return false;
                    // value bytes this term holds: all of them (physical) or byte k (plane)
                    const uint32_t b0 = split ? k : 0, nb = split ? 1 : vs;
                    for(uint32_t j = 0; j < G; ++j)
                        for(uint32_t i = 0; i < nb; ++i)
                        {
                            uint32_t byteInSpan, w0;
                            if(run >= 0)
                            {
                                byteInSpan = j * t.size + i;
                                w0 = spans[run].word0;
                            }
                            else
                            {
                                byteInSpan = (j / L) * st.bs + t.inblock + (L > 1 ? (j % L) * t.ls : 0) + i;
                                w0 = spans[sos[t.stream]].word0;
                            }
                            // (word << 2) | byte
                            wordOf[(size_t(f) * G + j) * 16 + b0 + i] = ((w0 + byteInSpan / 4) << 2) | (byteInSpan & 3);
                        }
                }
            }
            return true;
        };
        uint32_t G = 0;
        std::vector<uint32_t> wS, wD;
        for(uint32_t c : candidates)
        {
            if(begin % c)
                continue;
            if(build(c, true, sv[0], spanOfStream[0], wS) && build(c, false, sv[1], spanOfStream[1], wD))
            {
                G = c;
                break;
            }
        }
        if(G == 0)
            return false;
        const uint64_t groups = (end - begin) / G;
        if(groups == 0)
            return false;
        // destination word -> its 4 source bytes (0xFFFFFFFF: a hole, keep the old byte)
        uint32_t dWords = 0;
        for(const Span& sp : sv[1])
            dWords += sp.bytes / 4;
        std::vector<uint32_t> srcOfDst(size_t(dWords) * 4, 0xFFFFFFFFu);
        // bytes of bool leaves: canonicalised to 0 / 1 (any non-zero byte reads as true, scalar.hpp)
        std::vector<uint32_t> boolMask(dWords, 0);
        // converted values are "virtual" source words after the real ones: value (f, j) converted
        // to the destination's stored type, ceil(dsz / 4) words
        uint32_t sWordsAll = 0;
        for(const Span& sp : sv[0])
            sWordsAll += sp.bytes / 4;
        struct Virt
        {
            uint32_t f, j, first;
        };
        std::vector<Virt> virt; // per virtual word
        for(uint32_t f = 0; f < nl; ++f)
            for(uint32_t j = 0; j < G; ++j)
            {
                uint32_t vid = 0;
                if(conv[f])
                {
                    vid = sWordsAll + static_cast<uint32_t>(virt.size());
                    for(uint32_t q = 0; q < (dsz[f] + 3) / 4; ++q)
                        virt.push_back({f, j, vid});
                }
                for(uint32_t b = 0; b < dsz[f]; ++b)
                {
                    const size_t k = (size_t(f) * G + j) * 16 + b;
                    const uint32_t d = wD[k];
                    srcOfDst[size_t(d >> 2) * 4 + (d & 3)] = conv[f] ? (((vid + b / 4) << 2) | (b & 3)) : wS[k];
                    if(!conv[f] && p.leaf[f].ltype == lamb::Bool)
                        boolMask[d >> 2] |= 0xFFu << (8 * (d & 3));
                }
            }
        // destination vectors with holes are preloaded
        // words 2, 3 of a half destination span are never stored: don't care, not holes
        constexpr uint32_t kDontCare = 0xFFFFFFFEu;
        for(const Span& sp : sv[1])
            if(sp.half)
                for(uint32_t b = 8; b < 16; ++b)
                    srcOfDst[size_t(sp.word0) * 4 + b] = kDontCare;
        std::vector<bool> holeVec(dWords / 4, false);
        for(uint32_t w = 0; w < dWords; ++w)
            for(uint32_t b = 0; b < 4; ++b)
                if(srcOfDst[size_t(w) * 4 + b] == 0xFFFFFFFFu)
                    holeVec[w / 4] = true;
        // pass-through spans: a destination block span that is byte for byte a source block span
        // (an SoA leaf or byte plane on both sides, AoSoA<L> to AoSoA<L>, ...) is copied by the warp
        // as one coalesced vector stream, without registers or slabs
        std::vector<int> passSrc(sv[1].size(), -1);
        std::vector<bool> srcPassed(sv[0].size(), false);
        for(size_t m = 0; m < sv[1].size(); ++m)
        {
            const Span& dm = sv[1][m];
            const uint32_t s0 = srcOfDst[size_t(dm.word0) * 4];
            if(s0 == 0xFFFFFFFFu || (s0 & 3))
                continue;
            for(size_t k = 0; k < sv[0].size(); ++k)
            {
                const Span& sk = sv[0][k];
                if(srcPassed[k] || sk.word0 != (s0 >> 2) || sk.bytes != dm.bytes || sk.half != dm.half)
                    continue;
                bool same = true;
                // half spans: only their first 8 bytes are real (words 2, 3 don't care)
                for(uint32_t w = 0; w < (dm.half ? 2u : dm.bytes / 4) && same; ++w)
                {
                    same = boolMask[dm.word0 + w] == 0;
                    for(uint32_t b = 0; b < 4 && same; ++b)
                        same = srcOfDst[size_t(dm.word0 + w) * 4 + b] == (((sk.word0 + w) << 2) | b);
                }
                if(same)
                {
                    passSrc[m] = static_cast<int>(k);
                    srcPassed[k] = true;
                }
                break;
            }
        }

        // ---- generate ----
        // A warp owns 32 consecutive groups.  A block span (G/L whole blocks) of K > 1 vectors per
        // group is one contiguous 32*K-vector region per warp: it moves between HBM and a
        // warp-private shared-memory slab with coalesced 16-byte accesses, slot t at t*KP with
        // KP = K | 1 so the per-thread 16-byte slab accesses are bank-conflict-free.  Leaf runs of
        // AoSoA blocks and one-vector spans are accessed by their own thread directly.
        struct Lay
        {
            bool staged;
            uint32_t K, KP, rb;
        };
        const char* envStage = std::getenv("LAMB_JIT_STAGE");
        // Which sides go through slabs (profiles/r02/jit/jit_variants.log, 21 pairs): by default the
        // destination only -- uncoalesced stores cost more than uncoalesced loads, and one staged side
        // keeps twice the warps resident (0.79-0.93 of HBM where staging both gave 0.44-0.83) --
        // unless the source's direct loads would not fit in registers; then the source only.
        // LAMB_JIT_STAGE = 1 (both), s, d, 0 (neither) overrides.
        uint32_t srcWords = 0;
        for(size_t k = 0; k < sv[0].size(); ++k)
            if(!srcPassed[k])
                srcWords += sv[0][k].bytes / 4;
        const char forcedMode = envStage && envStage[0] ? envStage[0] : 'a';
        const bool autoMode = forcedMode == 'a';
        // widest block span on each side (16-byte vectors per thread)
        uint32_t maxK[2] = {0, 0};
        for(int side = 0; side < 2; ++side)
            for(size_t k = 0; k < sv[side].size(); ++k)
                if(!sv[side][k].run && !(side ? passSrc[k] >= 0 : srcPassed[k]))
                    maxK[side] = std::max(maxK[side], sv[side][k].bytes / 16);
        const char heuristic = (srcWords <= 128 || maxK[1] >= maxK[0]) ? 'd' : 's';
        // uniform pairs whose sides are both wide blocks beyond the register budget (aosoa:8 <->
        // aosoa:3, R64 aos-packed -> aosoa:3) measured faster on k_uniform_direct
        if(autoMode && p.uni && srcWords > 128 && maxK[1] > 8)
            return false;
        // one generated kernel per staging mode; timedMs != nullptr times the launch (autotuning)
        const char* envMinB = std::getenv("LAMB_JIT_MINB");
        const int forcedMinB = envMinB ? std::atoi(envMinB) : 0;
        // minB: CTAs per SM the register allocation must allow (__launch_bounds__ second argument,
        // 0 = none); prepareOnly: generate and compile, do not launch
        auto attempt = [&](char mode, int minB, float* timedMs, bool prepareOnly) -> bool
        {
        const bool stageOn = mode != '0';
        const bool stageSide[2] = {mode != 'd', mode != 's'};
        std::vector<Lay> lay[2];
        uint32_t slab[2] = {0, 0}; // slab vectors per warp on each side
        uint32_t directWords = 0;
        for(int side = 0; side < 2; ++side)
            for(size_t k = 0; k < sv[side].size(); ++k)
            {
                const Span& sp = sv[side][k];
                const bool passed = side ? passSrc[k] >= 0 : srcPassed[k];
                Lay l;
                l.K = sp.bytes / 16;
                l.staged = stageOn && stageSide[side] && !sp.run && l.K > 1 && !passed;
                l.KP = l.K | 1u;
                l.rb = slab[side];
                if(l.staged)
                    slab[side] += 32 * l.KP;
                else if(side == 0 && !passed)
                    directWords += 4 * l.K;
                lay[side].push_back(l);
            }
        // a source too wide for registers and not staged: its vectors are loaded at first use
        const bool lazySrc = directWords > 128;
        const uint32_t warpBytes = (slab[0] + slab[1]) * 16;
        if(warpBytes > 100 * 1024)
            return false;
        bool anyHole = false;
        for(bool h : holeVec)
            anyHole |= h;
        if(autoMode && anyHole && mode == 's')
            return false; // padded destinations read back thread by thread: the warp-tile engine is faster
        const size_t nspan = sv[0].size() + sv[1].size();
        if(nspan > 96)
            return false;
        // cache key: everything the generated source depends on (not the base pointers, begin or
        // groups, which are kernel parameters), so a repeated pair skips generation entirely
        std::string key;
        auto put = [&](uint64_t x) { key.append(reinterpret_cast<const char*>(&x), sizeof x); };
        put(G);
        put(static_cast<uint64_t>(static_cast<unsigned char>(mode)));
        put(static_cast<uint64_t>(minB));
        put(lazySrc);
        put(slab[0]);
        put(slab[1]);
        for(int side = 0; side < 2; ++side)
        {
            put(sv[side].size());
            for(size_t k = 0; k < sv[side].size(); ++k)
            {
                const Span& sp = sv[side][k];
                const Lay& l = lay[side][k];
                put(sp.run | (uint64_t(sp.half) << 1));
                put(sp.gstride);
                put((uint64_t(sp.lsh) << 32) | sp.bs);
                put((uint64_t(sp.lmask) << 32) | sp.ls);
                put((uint64_t(sp.bytes) << 32) | sp.word0);
                put((uint64_t(l.staged) << 48) | (uint64_t(l.K) << 32) | (uint64_t(l.KP) << 16) | l.rb);
            }
        }
        for(int x : passSrc)
            put(static_cast<uint64_t>(static_cast<int64_t>(x)));
        for(uint32_t f = 0; f < nl; ++f)
            put((uint64_t(p.leaf[f].stype) << 16) | (uint64_t(p.leaf[f].ltype) << 8) | p.leaf[f].dtype);
        key.append(reinterpret_cast<const char*>(srcOfDst.data()), srcOfDst.size() * sizeof(uint32_t));
        key.append(reinterpret_cast<const char*>(boolMask.data()), boolMask.size() * sizeof(uint32_t));
        for(bool h : holeVec)
            key.push_back(h ? '1' : '0');
        cudaKernel_t kern = nullptr;
        bool known = false;
        {
            std::lock_guard<std::mutex> lk(g_mu);
            auto it = g_keyCache.find(key);
            if(it != g_keyCache.end())
            {
                known = true;
                kern = it->second;
            }
        }
        const char* dump = std::getenv("LAMB_JIT_DUMP");
        if(known && dump)
            if(FILE* fp = std::fopen(dump, "a"))
            {
                std::fprintf(fp, "// G=%u groups=%llu (cached)\n", G, static_cast<unsigned long long>(groups));
                std::fclose(fp);
            }
        if(!known)
        {
        std::ostringstream o;
        o << "struct LJP { unsigned long long base[" << nspan << "]; unsigned long long begin, groups; };\n"
          << "__device__ __forceinline__ unsigned prm(unsigned a, unsigned b, unsigned s) { unsigned r; "
             "asm(\"prmt.b32 %0, %1, %2, %3;\" : \"=r\"(r) : \"r\"(a), \"r\"(b), \"r\"(s)); return r; }\n"
          << "__device__ __forceinline__ unsigned bcn(unsigned w, unsigned m) { return (w & ~m) | (__vcmpne4(w & m, 0u) & m & "
             "0x01010101u); }\n"
          << "__device__ __forceinline__ void lj_cvt(unsigned lo, unsigned hi, int from, int to, unsigned& ol, unsigned& oh) {\n"
             " if(from == to) { ol = lo; oh = hi; return; }\n"
             " if(from == 8 && to == 9) { unsigned long long r;\n"
             "  if((lo & 0x7F800000u) == 0x7F800000u && (lo & 0x7FFFFFu)) r = ((unsigned long long)(lo >> 31) << 63) | "
             "0x7FF8000000000000ull | ((unsigned long long)(lo & 0x7FFFFFu) << 29);\n"
             "  else r = (unsigned long long)__double_as_longlong((double)__uint_as_float(lo));\n"
             "  ol = (unsigned)r; oh = (unsigned)(r >> 32); return; }\n"
             " if(from == 9 && to == 8) { const unsigned long long b = lo | ((unsigned long long)hi << 32); oh = 0u;\n"
             "  if((b & 0x7FF0000000000000ull) == 0x7FF0000000000000ull && (b & 0x000FFFFFFFFFFFFFull)) "
             "ol = ((hi >> 31) << 31) | 0x7FC00000u | (unsigned)((b >> 29) & 0x3FFFFFu);\n"
             "  else ol = __float_as_uint(__double2float_rn(__longlong_as_double((long long)b))); return; }\n"
             " const unsigned fw = 8u * ((0x18484218421ull >> (4 * from)) & 0xF), tw = 8u * ((0x18484218421ull >> (4 * to)) & 0xF);\n"
             " unsigned long long v = lo | ((unsigned long long)hi << 32);\n"
             " if(from <= 3 && fw < 64) { const unsigned long long sb = 1ull << (fw - 1); v = ((v & ((1ull << fw) - 1ull)) ^ sb) - sb; }\n"
             " if(tw < 64) v &= (1ull << tw) - 1ull;\n"
             " ol = (unsigned)v; oh = (unsigned)(v >> 32); }\n"
          << "__device__ __forceinline__ unsigned long long lj_run(unsigned long long base, unsigned long long e, unsigned sh, "
             "unsigned long long bs, unsigned long long mask, unsigned long long ls, unsigned v) { return base + (e >> sh) * bs + "
             "(e & mask) * ls + 16ull * v; }\n"
          << "__device__ __forceinline__ uint4 ldg(unsigned long long a) { uint4 v; asm volatile(\"ld.global.cs.v4.u32 "
             "{%0,%1,%2,%3}, [%4];\" : \"=r\"(v.x), \"=r\"(v.y), \"=r\"(v.z), \"=r\"(v.w) : \"l\"(a)); return v; }\n"
          << "__device__ __forceinline__ uint4 ldg8(unsigned long long a) { uint4 v; v.z = 0u; v.w = 0u; asm volatile(\"ld.global.cs.v2.u32 "
             "{%0,%1}, [%2];\" : \"=r\"(v.x), \"=r\"(v.y) : \"l\"(a)); return v; }\n"
          << "__device__ __forceinline__ uint4 ldo8(unsigned long long a) { uint4 v; v.z = 0u; v.w = 0u; asm volatile(\"ld.global.v2.u32 "
             "{%0,%1}, [%2];\" : \"=r\"(v.x), \"=r\"(v.y) : \"l\"(a)); return v; }\n"
          << "__device__ __forceinline__ void stg8(unsigned long long a, uint4 v) { asm volatile(\"st.global.cs.v2.u32 [%0], "
             "{%1,%2};\" :: \"l\"(a), \"r\"(v.x), \"r\"(v.y) : \"memory\"); }\n"
          << "__device__ __forceinline__ uint4 ldo(unsigned long long a) { uint4 v; asm volatile(\"ld.global.v4.u32 "
             "{%0,%1,%2,%3}, [%4];\" : \"=r\"(v.x), \"=r\"(v.y), \"=r\"(v.z), \"=r\"(v.w) : \"l\"(a)); return v; }\n"
          << "__device__ __forceinline__ void stg(unsigned long long a, uint4 v) { asm volatile(\"st.global.cs.v4.u32 [%0], "
             "{%1,%2,%3,%4};\" :: \"l\"(a), \"r\"(v.x), \"r\"(v.y), \"r\"(v.z), \"r\"(v.w) : \"memory\"); }\n"
          << "extern \"C\" __global__ void __launch_bounds__(128" << (minB ? ", " + std::to_string(minB) : std::string()) << ") lamjit_copy(const LJP P) {\n"
          << " extern __shared__ uint4 lj_sm[];\n"
          << " const unsigned lane = threadIdx.x & 31u;\n"
          << " uint4* ss = lj_sm + (threadIdx.x >> 5) * " << (slab[0] + slab[1]) << "u;\n"
          << " uint4* sd = ss + " << slab[0] << "u;\n (void)ss; (void)sd;\n"
          << " const unsigned long long wstride = (unsigned long long)gridDim.x * (blockDim.x >> 5) * 32ull;\n"
          << " for(unsigned long long gw = ((unsigned long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32ull; "
             "gw < P.groups; gw += wstride) {\n"
          << "  const unsigned cnt = (unsigned)min(32ull, P.groups - gw);\n"
          << "  const unsigned long long g = gw + lane;\n"
          << "  const bool act = lane < cnt;\n"
          << "  const unsigned long long e0 = P.begin + g * " << G << "ull;\n  (void)e0;\n";
        auto addr = [&](const Span& sp, size_t idx) -> std::string
        {
            std::ostringstream a;
            if(sp.run)
                a << "(P.base[" << idx << "] + (e0 >> " << sp.lsh << ") * " << sp.bs << "ull + (e0 & " << sp.lmask
                  << "ull) * " << sp.ls << "ull)";
            else
                a << "(P.base[" << idx << "] + g * " << sp.gstride << "ull)";
            return a.str();
        };
        auto slot = [&](const Lay& l, uint32_t v) -> std::string
        {
            std::ostringstream a;
            a << "[" << l.rb << "u + lane * " << l.KP << "u + " << v << "u]";
            return a.str();
        };
        // holeMask (destination preload): bit v set = vector v of a group has bytes copyView never
        // writes; only those are read back (all of them when K > 64)
        auto coop = [&](const Span& sp, const Lay& l, size_t idx, bool load, const char* slabName, const char* fn,
                        uint64_t holeMask = ~0ull)
        {
            o << "  { const unsigned long long a = P.base[" << idx << "] + gw * " << sp.gstride << "ull;\n"
              << "#pragma unroll\n   for(unsigned j = 0; j < " << l.K << "u; ++j) { const unsigned i = lane + 32u * j; "
              << "if(i < cnt * " << l.K << "u";
            if(holeMask != ~0ull)
                o << " && ((0x" << std::hex << holeMask << std::dec << "ull >> (i % " << l.K << "u)) & 1ull)";
            o << ") ";
            if(load)
                o << slabName << "[" << l.rb << "u + (i / " << l.K << "u) * " << l.KP << "u + i % " << l.K << "u] = " << fn
                  << "(a + 16ull * i); } }\n";
            else
                o << "stg(a + 16ull * i, " << slabName << "[" << l.rb << "u + (i / " << l.K << "u) * " << l.KP << "u + i % "
                  << l.K << "u]); } }\n";
        };
        // pass-through spans: warp-coalesced vector copies; the vectors of all such spans are
        // batched 16 per lane, every load of a batch issued before its first store.  Vector i of
        // the warp's region of span m is vector i % K of group gw + i / K: contiguous for a block
        // span, and for a leaf run the runs of consecutive groups are adjacent inside a block.
        {
            auto passAddr = [&](const Span& sp, size_t idx, const std::string& i, uint32_t K) -> std::string
            {
                std::ostringstream a;
                if(!sp.run)
                    a << "(pb" << idx << " + " << (sp.half ? 8 : 16) << "ull * " << i << ")";
                else
                    a << "lj_run(P.base[" << idx << "], P.begin + (gw + " << i << " / " << K << "u) * " << G << "ull, " << sp.lsh
                      << "u, " << sp.bs << "ull, " << sp.lmask << "ull, " << sp.ls << "ull, " << i << " % " << K << "u)";
                return a.str();
            };
            std::vector<std::pair<size_t, uint32_t>> pv; // (destination span, vector j)
            for(size_t m = 0; m < sv[1].size(); ++m)
                if(passSrc[m] >= 0)
                    for(uint32_t j = 0; j < lay[1][m].K; ++j)
                        pv.emplace_back(m, j);
            for(size_t m = 0; m < sv[1].size(); ++m)
                if(passSrc[m] >= 0)
                    for(int side = 0; side < 2; ++side)
                    {
                        const size_t k = side ? m : static_cast<size_t>(passSrc[m]);
                        const Span& sp = sv[side][k];
                        const size_t idx = side ? sv[0].size() + m : k;
                        if(!sp.run)
                            o << "  const unsigned long long pb" << idx << " = P.base[" << idx << "] + gw * " << sp.gstride << "ull;\n";
                    }
            for(size_t b0 = 0; b0 < pv.size(); b0 += 16)
            {
                const size_t b1 = std::min(pv.size(), b0 + 16);
                o << "  {\n";
                for(size_t q = b0; q < b1; ++q)
                {
                    const size_t m = pv[q].first, k = static_cast<size_t>(passSrc[m]);
                    const uint32_t j = pv[q].second, K = lay[1][m].K;
                    const std::string i = "i" + std::to_string(q - b0);
                    o << "   uint4 t" << q - b0 << "; const unsigned " << i << " = lane + " << 32 * j << "u; if(" << i << " < cnt * " << K
                      << "u) t" << q - b0 << " = " << (sv[0][k].half ? "ldg8" : "ldg") << "(" << passAddr(sv[0][k], k, i, K) << ");\n";
                }
                for(size_t q = b0; q < b1; ++q)
                {
                    const size_t m = pv[q].first;
                    const uint32_t K = lay[1][m].K;
                    const std::string i = "i" + std::to_string(q - b0);
                    o << "   if(" << i << " < cnt * " << K << "u) " << (sv[1][m].half ? "stg8" : "stg") << "("
                      << passAddr(sv[1][m], sv[0].size() + m, i, K) << ", t" << q - b0 << ");\n";
                }
                o << "  }\n";
            }
        }
        // direct source vectors first (most loads in flight), then the coalesced slab loads
        for(size_t k = 0; k < sv[0].size(); ++k)
            if(!lay[0][k].staged && !lazySrc && !srcPassed[k])
            {
                for(uint32_t v = 0; v < lay[0][k].K; ++v)
                    o << "  uint4 S" << k << "_" << v << " = make_uint4(0u, 0u, 0u, 0u);\n";
                o << "  if(act) { const unsigned long long a = " << addr(sv[0][k], k) << ";";
                for(uint32_t v = 0; v < lay[0][k].K; ++v)
                    o << " S" << k << "_" << v << " = " << (sv[0][k].half ? "ldg8" : "ldg") << "(a + " << 16 * v << "ull);";
                o << " }\n";
            }
        for(size_t k = 0; k < sv[0].size(); ++k)
            if(lay[0][k].staged)
                coop(sv[0][k], lay[0][k], k, true, "ss", "ldg");
        for(size_t k = 0; k < sv[1].size(); ++k)
        {
            bool holes = false;
            uint64_t mask = 0;
            for(uint32_t v = 0; v < lay[1][k].K; ++v)
            {
                const bool h = holeVec[sv[1][k].word0 / 4 + v];
                holes |= h;
                if(h && v < 64)
                    mask |= 1ull << v;
            }
            if(lay[1][k].staged && holes)
                coop(sv[1][k], lay[1][k], sv[0].size() + k, true, "sd", "ldo", lay[1][k].K <= 64 ? mask : ~0ull);
        }
        o << "  __syncwarp();\n  if(act) {\n";
        if(lazySrc)
            for(size_t k = 0; k < sv[0].size(); ++k)
                if(!lay[0][k].staged && !srcPassed[k])
                    o << "   const unsigned long long as" << k << " = " << addr(sv[0][k], k) << ";\n";
        // source word w -> "S<k>_<v>.<c>"; staged vectors are read from the slab at first use
        std::vector<int> spanOfWord;
        for(size_t k = 0; k < sv[0].size(); ++k)
            for(uint32_t w = 0; w < sv[0][k].bytes / 4; ++w)
                spanOfWord.push_back(static_cast<int>(k));
        std::vector<bool> emitted(spanOfWord.size() / 4, false);
        // a word from 4 (variable, byte) pairs: a PRMT chain whose first step takes the bytes of two
        // words and each further step adds one ("0u" supplies zero bytes)
        auto assemble = [&](const std::string* var, const uint32_t* byt) -> std::string
        {
            if(var[0] == var[1] && var[1] == var[2] && var[2] == var[3] && byt[0] == 0 && byt[1] == 1 && byt[2] == 2
               && byt[3] == 3)
                return var[0];
            std::string acc;
            bool placed[4] = {false, false, false, false};
            for(uint32_t b = 0; b < 4; ++b)
            {
                if(placed[b])
                    continue;
                const std::string x = var[b];
                uint32_t sel = 0;
                std::ostringstream e;
                if(acc.empty())
                {
                    std::string y;
                    for(uint32_t c2 = 0; c2 < 4; ++c2)
                        if(var[c2] != x && y.empty())
                            y = var[c2];
                    for(uint32_t c2 = 0; c2 < 4; ++c2)
                    {
                        uint32_t nib = 0;
                        if(var[c2] == x)
                        {
                            nib = byt[c2];
                            placed[c2] = true;
                        }
                        else if(!y.empty() && var[c2] == y)
                        {
                            nib = 4 + byt[c2];
                            placed[c2] = true;
                        }
                        sel |= nib << (4 * c2);
                    }
                    e << "prm(" << x << ", " << (y.empty() ? x : y) << ", 0x" << std::hex << sel << std::dec << "u)";
                }
                else
                {
                    for(uint32_t c2 = 0; c2 < 4; ++c2)
                    {
                        uint32_t nib = c2;
                        if(!placed[c2] && var[c2] == x)
                        {
                            nib = 4 + byt[c2];
                            placed[c2] = true;
                        }
                        sel |= nib << (4 * c2);
                    }
                    e << "prm(" << acc << ", " << x << ", 0x" << std::hex << sel << std::dec << "u)";
                }
                acc = e.str();
            }
            return acc;
        };
        std::vector<bool> vEmitted(virt.size(), false);
        std::function<std::string(uint32_t)> srcWord;
        srcWord = [&](uint32_t w) -> std::string
        {
            if(w >= sWordsAll)
            {
                // a converted value: gather its stored bytes, convert stype -> ltype -> dtype
                const Virt& vt = virt[w - sWordsAll];
                const uint32_t first = vt.first - sWordsAll;
                const std::string nm = "V" + std::to_string(first);
                if(!vEmitted[first])
                {
                    vEmitted[first] = true;
                    const lamt_leaf& lf = p.leaf[vt.f];
                    std::string half[2];
                    for(uint32_t h = 0; h < 2; ++h)
                    {
                        std::string var[4];
                        uint32_t byt[4];
                        for(uint32_t b = 0; b < 4; ++b)
                        {
                            const uint32_t vb = 4 * h + b;
                            if(vb < ssz[vt.f])
                            {
                                const uint32_t sw = wS[(size_t(vt.f) * G + vt.j) * 16 + vb];
                                var[b] = srcWord(sw >> 2);
                                byt[b] = sw & 3;
                            }
                            else
                            {
                                var[b] = "0u";
                                byt[b] = 0;
                            }
                        }
                        half[h] = (4 * h < ssz[vt.f]) ? assemble(var, byt) : "0u";
                    }
                    o << "   unsigned " << nm << "_0, " << nm << "_1;\n   { unsigned t0, t1; lj_cvt(" << half[0] << ", " << half[1]
                      << ", " << int(lf.stype) << ", " << int(lf.ltype) << ", t0, t1); lj_cvt(t0, t1, " << int(lf.ltype) << ", "
                      << int(lf.dtype) << ", " << nm << "_0, " << nm << "_1); }\n";
                }
                return nm + "_" + std::to_string(w - vt.first);
            }
            const int k = spanOfWord[w];
            const uint32_t v = (w - sv[0][k].word0) / 4;
            if(lay[0][k].staged && !emitted[w / 4])
            {
                o << "   const uint4 S" << k << "_" << v << " = ss" << slot(lay[0][k], v) << ";\n";
                emitted[w / 4] = true;
            }
            else if(lazySrc && !emitted[w / 4])
            {
                o << "   const uint4 S" << k << "_" << v << " = " << (sv[0][k].half ? "ldg8" : "ldg") << "(as" << k << " + " << 16 * v
                  << "ull);\n";
                emitted[w / 4] = true;
            }
            static const char* comp = "xyzw";
            return "S" + std::to_string(k) + "_" + std::to_string(v) + "." + comp[w & 3];
        };
        for(size_t k = 0; k < sv[1].size(); ++k)
        {
            if(passSrc[k] >= 0)
                continue; // copied above
            const Span& sp = sv[1][k];
            const Lay& l = lay[1][k];
            const size_t idx = sv[0].size() + k;
            const std::string ad = "ad" + std::to_string(k);
            if(!l.staged)
                o << "   const unsigned long long " << ad << " = " << addr(sp, idx) << ";\n";
            for(uint32_t v = 0; v < l.K; ++v)
            {
                const uint32_t w0 = sp.word0 + 4 * v;
                std::string oldName = "O" + std::to_string(k) + "_" + std::to_string(v);
                if(holeVec[w0 / 4])
                {
                    if(l.staged)
                        o << "   const uint4 " << oldName << " = sd" << slot(l, v) << ";\n";
                    else
                        o << "   const uint4 " << oldName << " = " << (sp.half ? "ldo8" : "ldo") << "(" << ad << " + " << 16 * v
                          << "ull);\n";
                }
                std::string dn[4];
                for(uint32_t c = 0; c < 4; ++c)
                {
                    const uint32_t w = w0 + c;
                    std::string var[4];
                    uint32_t byt[4];
                    for(uint32_t b = 0; b < 4; ++b)
                    {
                        const uint32_t sw = srcOfDst[size_t(w) * 4 + b];
                        if(sw == kDontCare)
                        {
                            var[b] = "0u";
                            byt[b] = 0;
                        }
                        else if(sw == 0xFFFFFFFFu)
                        {
                            var[b] = oldName + "." + "xyzw"[c];
                            byt[b] = b;
                        }
                        else
                        {
                            var[b] = srcWord(sw >> 2);
                            byt[b] = sw & 3;
                        }
                    }
                    dn[c] = assemble(var, byt);
                    if(boolMask[w])
                        dn[c] = "bcn(" + dn[c] + ", " + std::to_string(boolMask[w]) + "u)";
                }
                const std::string val = "make_uint4(" + dn[0] + ", " + dn[1] + ", " + dn[2] + ", " + dn[3] + ")";
                if(l.staged)
                    o << "   sd" << slot(l, v) << " = " << val << ";\n";
                else
                    o << "   " << (sp.half ? "stg8" : "stg") << "(" << ad << " + " << 16 * v << "ull, " << val << ");\n";
            }
        }
        o << "  }\n  __syncwarp();\n";
        for(size_t k = 0; k < sv[1].size(); ++k)
            if(lay[1][k].staged)
                coop(sv[1][k], lay[1][k], sv[0].size() + k, false, "sd", "");
        o << "  __syncwarp();\n }\n}\n";
        const std::string src = o.str();
        if(dump)
            if(FILE* fp = std::fopen(dump, "a"))
            {
                std::fprintf(fp, "// G=%u groups=%llu\n%s\n", G, static_cast<unsigned long long>(groups), src.c_str());
                std::fclose(fp);
            }
        kern = compile(src);
        std::lock_guard<std::mutex> lk(g_mu);
        g_keyCache[key] = kern;
        }
        if(!kern)
            return false;
        if(prepareOnly)
            return true;
        // warps per CTA: 4 while the slabs fit 100 KB per CTA
        const char* envCta = std::getenv("LAMB_JIT_CTA_KB");
        const uint32_t ctaBytes = (envCta ? static_cast<uint32_t>(std::atoi(envCta)) : 100) * 1024;
        const uint32_t wpc = warpBytes == 0 ? 4 : std::max<uint32_t>(1, std::min<uint32_t>(4, ctaBytes / warpBytes));
        const size_t smem = size_t(wpc) * warpBytes;
        if(smem > 48 * 1024
           && cudaFuncSetAttribute(reinterpret_cast<const void*>(kern), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem))
               != cudaSuccess)
        {
            cudaGetLastError();
            return false;
        }
        // parameters: the span bases (runtime pointers), begin, groups
        std::vector<unsigned long long> prm(nspan + 2);
        for(size_t k = 0; k < sv[0].size(); ++k)
            prm[k] = sv[0][k].base;
        for(size_t k = 0; k < sv[1].size(); ++k)
            prm[sv[0].size() + k] = sv[1][k].base;
        prm[nspan] = begin;
        prm[nspan + 1] = groups;
        void* args[] = {prm.data()};
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t warps = (groups + 31) / 32;
        const uint64_t want = (warps + wpc - 1) / wpc;
        const uint64_t cap = static_cast<uint64_t>(lamk::sm_count(dev)) * (64 / wpc);
        const unsigned grid = static_cast<unsigned>(want < cap ? want : cap);
        cudaEvent_t ev[2] = {nullptr, nullptr};
        if(timedMs)
        {
            cudaEventCreate(&ev[0]);
            cudaEventCreate(&ev[1]);
            cudaEventRecord(ev[0], s);
        }
        const cudaError_t e =
            cudaLaunchKernel(reinterpret_cast<const void*>(kern), dim3(grid), dim3(32 * wpc), args, smem, s);
        if(timedMs)
        {
            cudaEventRecord(ev[1], s);
            cudaEventSynchronize(ev[1]);
            cudaEventElapsedTime(timedMs, ev[0], ev[1]);
            cudaEventDestroy(ev[0]);
            cudaEventDestroy(ev[1]);
        }
        if(e != cudaSuccess)
        {
            cudaGetLastError();
            return false;
        }
        lamk::count_launch();
        *doneEnd = begin + groups * G;
        return true;
        };

        if(!autoMode)
            return attempt(forcedMode, forcedMinB, nullptr, false);
        // Staging mode: the heuristic above, or -- the first time a pair is copied at >= 2^22
        // elements outside stream capture -- the fastest of the four modes, each timed on the copy
        // itself (every mode writes the same bytes, so the last timed launch leaves the finished
        // copy), remembered per pair.  LAMB_JIT_TUNE=0 keeps the heuristic.
        std::string pairKey;
        {
            auto put = [&](uint64_t x) { pairKey.append(reinterpret_cast<const char*>(&x), sizeof x); };
            put(G);
            for(int side = 0; side < 2; ++side)
                for(const Span& sp : sv[side])
                {
                    put(sp.run | (uint64_t(sp.half) << 1));
                    put(sp.gstride);
                    put((uint64_t(sp.lsh) << 32) | sp.bs);
                    put((uint64_t(sp.lmask) << 32) | sp.ls);
                    put((uint64_t(sp.bytes) << 32) | sp.word0);
                }
            for(uint32_t f = 0; f < nl; ++f)
                put((uint64_t(p.leaf[f].stype) << 16) | (uint64_t(p.leaf[f].ltype) << 8) | p.leaf[f].dtype);
            pairKey.append(reinterpret_cast<const char*>(srcOfDst.data()), srcOfDst.size() * sizeof(uint32_t));
            pairKey.append(reinterpret_cast<const char*>(boolMask.data()), boolMask.size() * sizeof(uint32_t));
        }
        std::pair<char, int> chosen{heuristic, forcedMinB};
        bool decided = false;
        {
            std::lock_guard<std::mutex> lk(g_mu);
            auto it = g_modeCache.find(pairKey);
            if(it != g_modeCache.end())
            {
                chosen = it->second;
                decided = true;
            }
        }
        const char* tune = std::getenv("LAMB_JIT_TUNE");
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cap);
        if(!decided && !(tune && tune[0] == '0') && groups * G >= (uint64_t{1} << 22) && cap == cudaStreamCaptureStatusNone)
        {
            // candidates: 4 staging modes x (no register cap, 3 CTAs per SM); compiled in parallel
            std::vector<std::pair<char, int>> cand;
            for(char m : {'d', 's', '1', '0'})
                for(int mb : {0, 3})
                    cand.emplace_back(m, mb);
            int dev = 0;
            cudaGetDevice(&dev);
            std::vector<char> ready(cand.size(), 0);
            {
                std::vector<std::thread> th;
                for(size_t c = 0; c < cand.size(); ++c)
                    th.emplace_back(
                        [&, c]
                        {
                            cudaSetDevice(dev);
                            ready[c] = attempt(cand[c].first, cand[c].second, nullptr, true) ? 1 : 0;
                        });
                for(auto& t : th)
                    t.join();
            }
            float best = 0;
            int bestC = -1;
            for(size_t c = 0; c < cand.size(); ++c)
            {
                float ms = 0;
                if(!ready[c] || !attempt(cand[c].first, cand[c].second, nullptr, false)) // warm: module load
                    continue;
                if(attempt(cand[c].first, cand[c].second, &ms, false) && (bestC < 0 || ms < best))
                {
                    best = ms;
                    bestC = static_cast<int>(c);
                }
            }
            if(bestC < 0)
                return false;
            std::lock_guard<std::mutex> lk(g_mu);
            g_modeCache[pairKey] = cand[bestC];
            return true;
        }
        return attempt(chosen.first, chosen.second, nullptr, false);
    }
} // namespace lamjit

// Tile-plan parameter block (host <-> device), shared by the tile kernels (copy_tile.cu) and
// read by the specialised kernels' predicates (copy_tile_host.cpp).
//
// A tile is T consecutive elements (T a multiple of every AoSoA lane count, of 32 and of
// both layouts' shard units).  Each blob stream of the source and destination occupies
// one contiguous byte range per tile ("image"), moved between HBM and shared memory with
// 1-D TMA bulk copies (cp.async.bulk) when 16-byte aligned.  The transform step runs the
// per-leaf value pipeline (read terminal(s) -> convert -> write terminal(s)) entirely in
// shared memory; bit-packed destinations are assembled word by word by their owning
// thread (no read-modify-write anywhere, bitpack.hpp:16-17).
#pragma once

#include <stdint.h>

#define LAMT_MAX_LEAVES 32
#define LAMT_MAX_STREAMS 128   // plan streams (byte planes of wide records: 2 x 42 planes)
#define LAMT_WT_MAX_STREAMS 64 // streams the warp-tile engine (k_warp_tile) takes
#define LAMT_MAX_TERMS 8

#define LAMT_K_PHYS 0
#define LAMT_K_SPLIT 1
#define LAMT_K_BITS_INT 2
#define LAMT_K_BITS_FLT 3
#define LAMT_K_NULL 4

struct lamt_stream
{
    unsigned long long gptr; // stream pointer (blob + base0; virtual for chunk views)
    uint32_t smem_off;       // image offset inside a stage buffer
    uint32_t tile_bytes;     // image bytes per full tile
    uint32_t bs;             // PHYS: block stride bytes ; BITS: bits per element
    uint32_t lanes;          // PHYS: L ; BITS: 1
    uint32_t lshift;         // log2(L) or 0xFFFFFFFF
    uint32_t kind;           // 0 PHYS, 1 BITS
    uint32_t tma;            // image start is 16-byte aligned in global memory
    uint32_t scratch_off;    // BITS destination: per-element pattern scratch (stage-relative)
    uint32_t scratch64;      // scratch slots are 8 bytes (field width > 32)
    uint32_t pad;            // warp-tile engine: first 16-byte chunk of this image in its buffer
    uint32_t preload;        // destination with bytes copyView never writes (padding): the image is
                             // read before the transform so whole-image stores keep them
};

struct lamt_term
{
    uint16_t stream;
    uint8_t size;
    uint8_t aligned; // naturally aligned inside the smem image
    uint32_t inblock;
    uint32_t ls;
};

struct lamt_leaf
{
    uint8_t skind, stype, ltype, dkind, dtype, sn, dn, pure;
    uint8_t sE, sM, dE, dM; // BITS_INT: E = bits ; BITS_FLT: (E, M)
    uint8_t ssigned, pad0, pad1, pad2;
    lamt_term s[LAMT_MAX_TERMS];
    lamt_term d[LAMT_MAX_TERMS];
};

// warp-tile engine: a leaf's terminal addressing resolved on the host (k_warp_tile)
#define LAMT_WF_GENERIC 0
#define LAMT_WF_PP 1        // PHYS -> PHYS
#define LAMT_WF_PS_PLANES 2 // PHYS -> byte planes (packed u8 arrays): 4 elements per lane, u32 per plane
#define LAMT_WF_PS_BYTES 3  // PHYS -> byte terms
#define LAMT_WF_SP_PLANES 4 // byte planes -> PHYS
#define LAMT_WF_SP_BYTES 5  // byte terms -> PHYS
#define LAMT_WF_SKIP 6      // Null destination
struct lamt_wfast
{
    uint8_t mode, sn, dn, conv, boolean, ssz, dsz, pad;
    uint32_t sbase[8], sbs[8], dbase[8], dbs[8]; // smem image offset (incl. inblock) and element stride
    // PHYS terms on AoSoA streams (lanes L > 1): element e at base + (e / L) * bs + (e % L) * ls,
    // e / L = __umulhi(e, magic) with magic = ceil(2^32 / L) (exact for tile-local e < 2^16)
    uint32_t sL, sls, smagic, dL, dls, dmagic;
};

#define LAMT_MAX_WARPS 32
#define LAMT_MAX_STAGES 4
#define LAMT_UNI_LEAVES 16

struct lamt_params
{
    unsigned long long begin; // first element of tile 0
    uint32_t T;               // elements per tile (one warp owns one tile at a time)
    uint32_t ntiles;
    uint32_t nleaves;
    uint32_t nsrc, ndst; // streams [0, nsrc) source, [nsrc, nsrc+ndst) destination
    uint32_t src_bytes;  // stage bytes (source images)
    uint32_t dst_bytes;  // stage bytes (destination images + scratch)
    uint32_t tma_bytes;  // source bytes delivered by TMA per tile
    uint32_t stages;     // source stage buffers (loads in flight ahead of the transform)
    uint32_t dstages;    // destination buffers (stores draining behind it), >= 2
    uint32_t threads;    // threads per CTA
    uint32_t stg;        // destination images leave through 16-byte thread stores instead of TMA
    uint32_t lmode;      // 0: TMA bulk loads (mbarrier), 1: cp.async 16-byte loads (commit groups)
    uint32_t chunk;      // lmode 0: bytes per bulk op (0 = whole image)
    uint32_t any_bits;   // some destination stream is bit-packed
    uint32_t any_coop;   // some stream is not TMA-able
    uint32_t facS, facD;
    unsigned long long facSrc; // device counters (reads) or 0
    unsigned long long facDst; // device counters (writes) or 0
    // uniform fast path: every leaf a same-size physical move, one block geometry per side
    uint32_t uni, usize;
    uint32_t ubs_s, ul_s, ush_s, uls_s;
    uint32_t ubs_d, ul_d, ush_d, uls_d;
    uint32_t umag_s, umag_d; // ceil(2^32 / L) for non-power-of-two lanes (e / L = umulhi(e, mag), e < 2^32 / L)
    uint32_t uoff_s[LAMT_UNI_LEAVES], uoff_d[LAMT_UNI_LEAVES];
    lamt_stream st[LAMT_MAX_STREAMS];
    lamt_leaf leaf[LAMT_MAX_LEAVES];
    lamt_wfast wf[LAMT_MAX_LEAVES];
    // warp-tile engine: stream of each 16-byte image chunk, source chunks then destination
    // chunks (host-built, copied to shared memory by each CTA)
    uint32_t wt_chs, wt_chd;
    uint32_t dst_holes; // some destination stream has preload set (only k_warp_tile handles it)
    __align__(16) uint8_t wt_cst[1024];
};

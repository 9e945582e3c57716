// Lowered mapping ("plan"): the POD form in which a lamina mapping tree reaches the
// device.  Built on the host by host_layout.cpp; consumed by the kernels.
//
// A mapping tree (AoS/SoA/AoSoA/One/Split/Bitpack*/ChangeType/Bytesplit/Null, with the
// FieldAccessCount/Heatmap wrappers on top) is resolved per logical leaf into a small
// node tree:
//   PHYS      stored bytes at  stream_ptr + (i / L) * BS + inblock + (i % L) * LS
//             (AoS: L=1, BS=recordSize; SoA: L=1, BS=leafSize; AoSoA: L lanes,
//              BS=blockSize, LS=leafSize — mappings.hpp:54-57, 102-108, 151-159)
//   BITS_INT  b-bit field at bit i*b of a word stream   (computed.cpp:101-122)
//   BITS_FLT  (1,E,M) minifloat at bit i*(1+E+M)        (computed.cpp:192-217)
//   NULL      nothing stored, reads zero                (computed.cpp:508-531)
//   CONVERT   logical type <- -> child storage type     (computed.cpp:363-378)
//   SPLIT     s children, child k holds LE byte k       (computed.cpp:460-490)
// Streams group terminals that share a blob region advancing by BS bytes every L
// elements; a stream is the unit of tiling, chunking and sharding.
#pragma once

#include <stdint.h>

#define LAMP_PHYS 0
#define LAMP_BITS_INT 1
#define LAMP_BITS_FLT 2
#define LAMP_NULL 3
#define LAMP_CONVERT 4
#define LAMP_SPLIT 5

#define LAMP_FLAG_ALIGNED 1 // PHYS: every access is naturally aligned for its size
#define LAMP_FLAG_SIGNED 2  // BITS_INT: sign-extend on load

#define LAMS_PHYS 0
#define LAMS_BITS 1

#define LAMP_MAX_DEPTH 6

struct lamp_node
{
    uint8_t kind;
    uint8_t type; // scalar kind of the value at this node (LAM_I8 ... LAM_BOOL)
    uint8_t nchild;
    uint8_t flags;
    uint16_t child; // first child (children are contiguous)
    uint16_t stream;
    uint32_t a; // PHYS: inblock byte offset | BITS_INT: bits | BITS_FLT: expBits
    uint32_t b; // PHYS: lane stride         | BITS_FLT: manBits
};

struct lamp_stream
{
    uint64_t base0;        // blob byte offset of block 0
    uint64_t block_stride; // BS bytes per block of `lanes` elements (PHYS) ; bits per element (BITS)
    uint64_t lanes;        // L (PHYS), 1 (BITS)
    uint32_t nr;           // blob index
    uint32_t kind;         // LAMS_PHYS / LAMS_BITS
    uint32_t lane_shift;   // log2(L) when L is a power of two, else 0xFFFFFFFF
    uint32_t holefree;     // every byte of each block is some terminal's byte (safe to overwrite whole blocks)
};

// Device-resident view header.  Arrays follow the header in one allocation.
struct lamp_view
{
    uint64_t n;          // element count
    uint32_t nleaves;
    uint32_t nnodes;
    uint32_t nstreams;
    uint32_t nblobs;
    uint32_t fac;        // FieldAccessCount wrapper present
    uint32_t heat;       // Heatmap wrapper present
    uint64_t heat_gran;  // Heatmap granularity
    const uint16_t* roots;             // [nleaves]
    const lamp_node* nodes;            // [nnodes]
    const lamp_stream* streams;        // [nstreams]
    uint8_t* const* stream_ptr;        // [nstreams] blob_ptr[nr] + base0 (virtual when chunked)
    unsigned long long* fac_counters;  // [2 * nleaves] reads then writes
    unsigned long long* heat_counters; // [sum blocks]
    const uint64_t* heat_offset;       // [nblobs] first counter of blob nr
};

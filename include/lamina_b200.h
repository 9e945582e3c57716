/*
 * lamina_b200 — C ABI of the B200-native layout-copy / bit-pack / instrumentation /
 * n-body hot path of the LLAMA-paper reference library `lamina`
 * (/root/reference/proj, arXiv 2302.08251).
 *
 * Drop-in boundary: every entry point replaces one reference interface on the hot
 * path (file:line relative to /root/reference/proj).  Plain pointers and sizes only;
 * no torch or C++ types cross this line.  All device work is stream-ordered on the
 * cudaStream_t passed as `void* stream` (NULL = legacy default stream).
 *
 * Errors: every int-returning call returns LAM_OK (0) or one of the LAM_E* codes,
 * which map 1:1 onto the exception types the reference throws
 * (include/lamina_b200.hpp rethrows them):
 *   LAM_EINVAL    std::invalid_argument  ("incompatible views", "type mismatch",
 *                 "blob count mismatch", "blob size mismatch", "unknown layout", ...)
 *   LAM_ERANGE    std::out_of_range      ("index out of range")
 *   LAM_EOVERFLOW std::overflow_error    ("index type overflow")
 *   LAM_ELOGIC    std::logic_error       ("computed leaf has no physical offset")
 *   LAM_ERUNTIME  std::runtime_error
 *   LAM_ECUDA     CUDA runtime failure (no reference counterpart)
 * lam_last_error() returns the thread-local message of the last failing call.
 */
#ifndef LAMINA_B200_H
#define LAMINA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LAM_OK 0
#define LAM_EINVAL 1
#define LAM_ERANGE 2
#define LAM_EOVERFLOW 3
#define LAM_ELOGIC 4
#define LAM_ERUNTIME 5
#define LAM_ECUDA 6

/* Scalar kinds, same numbering as lamina::Scalar (core/include/lamina/scalar.hpp:16-29). */
#define LAM_I8 0
#define LAM_I16 1
#define LAM_I32 2
#define LAM_I64 3
#define LAM_U8 4
#define LAM_U16 5
#define LAM_U32 6
#define LAM_U64 7
#define LAM_F32 8
#define LAM_F64 9
#define LAM_BOOL 10

/* Instrumentation wrappers (lamina::FieldAccessCount / lamina::Heatmap,
 * core/include/lamina/instrument.hpp:27-127).  Heatmap is outermost when both. */
#define LAM_WRAP_FIELD_ACCESS_COUNT 1
#define LAM_WRAP_HEATMAP 2

/* n-body arithmetic modes (tools/nbody/kernel.hpp:15-41). */
#define LAM_NBODY_EXACT 0 /* IEEE add/mul/sqrt/div in the reference's order: bit-identical */
#define LAM_NBODY_FAST 1  /* FMA + rsqrt, j-tile reassociation: within stated tolerance */

typedef struct lam_layout lam_layout; /* lowered mapping (schema + extents + layout) */
typedef struct lam_view lam_view;     /* device blobs bound to a layout (+ device counters) */

/* ---- errors --------------------------------------------------------------------- */
const char* lam_last_error(void);
const char* lam_version(void);

/* ---- layouts ------------------------------------------------------------------------
 * Replaces lamina::parseLayout(text, schema, extents)  (core/include/lamina/layout_spec.hpp:19,
 * core/src/layout_spec.cpp:164-167) together with RecordSchema::parse (core/src/record.cpp:480)
 * and ArrayExtents::parse (core/src/extents.cpp:135).  `layout` is the reference grammar
 * (aos-packed, aos-aligned, soa-sb, soa-mb, aosoa:L, one, null, split:..., bitpack-int:b,
 * bitpack-float:E,M, changetype:..., bytesplit:...) and additionally accepts the names the
 * reference prints for its wrappers, "field-access-count(<inner>)" and "heatmap:<g>(<inner>)",
 * so Mapping::name() of any reference mapping round-trips. `wrap`/`granularity` add the
 * wrappers programmatically (FieldAccessCount(inner) / Heatmap(inner, g)). */
int lam_layout_create(const char* schema, const char* extents, const uint64_t* dyn_values, size_t n_dyn,
                      const char* layout, int wrap, uint64_t granularity, lam_layout** out);
void lam_layout_destroy(lam_layout* layout);
/* Mapping::name() (core/include/lamina/mapping.hpp:72); returns the length, copies up to cap-1. */
size_t lam_layout_name(const lam_layout* layout, char* buf, size_t cap);
/* RecordSchema::toString (core/src/record.cpp:472) / ArrayExtents::toString (core/src/extents.cpp:118). */
size_t lam_layout_schema(const lam_layout* layout, char* buf, size_t cap);
size_t lam_layout_extents(const lam_layout* layout, char* buf, size_t cap);
/* Mapping::blobCount/blobSize (mapping.hpp:74-75). */
size_t lam_layout_blob_count(const lam_layout* layout);
uint64_t lam_layout_blob_size(const lam_layout* layout, size_t nr);
uint64_t lam_layout_element_count(const lam_layout* layout);
size_t lam_layout_leaf_count(const lam_layout* layout);
/* Leaf table entry (RecordSchema::leaf, record.hpp:173): scalar kind, size, packed offset. */
int lam_layout_leaf(const lam_layout* layout, size_t flat_leaf, int* kind, size_t* size, size_t* offset_packed);
size_t lam_layout_leaf_path(const lam_layout* layout, size_t flat_leaf, char* buf, size_t cap);
/* Mapping::isComputed / isFullyPhysical / hasMutableState (mapping.hpp:86-105). */
int lam_layout_is_computed(const lam_layout* layout, size_t flat_leaf);
int lam_layout_is_fully_physical(const lam_layout* layout);
int lam_layout_has_mutable_state(const lam_layout* layout);
/* ArrayExtents::isFullyStatic (extents.hpp:127-130) and Mapping::runtimeStateBytes
 * (mapping.hpp:145-148; wrappers add inner mappings and counters, instrument.cpp:79-82,197-200). */
int lam_layout_is_fully_static(const lam_layout* layout);
uint64_t lam_layout_runtime_state_bytes(const lam_layout* layout);
/* Mapping::physicalOffset (mapping.hpp:109); LAM_ELOGIC for computed leaves. */
int lam_layout_physical_offset(const lam_layout* layout, uint64_t linear, size_t flat_leaf, size_t* nr,
                               uint64_t* offset);
/* Heatmap::blockCount summed over blobs (instrument.hpp:107); 0 when not wrapped. */
uint64_t lam_layout_heatmap_blocks(const lam_layout* layout, size_t nr);
/* Mapping::contiguousRun (core/include/lamina/mapping.hpp:122-135, mappings.cpp:44-50,96-101,
 * 140-148, computed.cpp:386-394): *has_run = 1 and (nr, offset) of element `linear` when the n
 * values of leaf `flat_leaf` starting there are contiguous with stride = leaf size; 0 otherwise
 * (computed leaves, counting wrappers, strided AoS runs, runs crossing an AoSoA block). */
int lam_layout_contiguous_run(const lam_layout* layout, uint64_t linear, size_t flat_leaf, uint64_t n, int* has_run,
                              size_t* nr, uint64_t* offset);
/* Element alignment unit for sharding/chunking: every multiple of it starts every blob
 * stream on a 16-byte boundary (AoSoA lanes, bit-stream words). */
uint64_t lam_layout_shard_unit(const lam_layout* layout);
/* Blob streams (disjoint blob regions advancing by a fixed stride per element block) and the
 * byte range [lo, hi) of blob *nr that elements [begin, end) occupy in stream s: what a shard
 * of a multi-GPU run owns and exchanges (e.g. the n-body all-gather of positions). */
size_t lam_layout_stream_count(const lam_layout* layout);
int lam_layout_stream_region(const lam_layout* layout, size_t stream, uint64_t begin, uint64_t end, size_t* nr,
                             uint64_t* lo, uint64_t* hi);

/* ---- device views ---------------------------------------------------------------------
 * Replaces lamina::View(MappingPtr) (core/src/view.cpp:97-103): allocates blobCount()
 * device blobs of exactly blobSize(nr) bytes, zero-filled (parity with Blob,
 * core/include/lamina/blob.hpp:22-29).  Counters (FieldAccessCount / Heatmap) live in
 * device memory and start at zero. */
int lam_view_alloc(const lam_layout* layout, int device, void* stream, lam_view** out);
/* Replaces lamina::View(MappingPtr, std::vector<Blob>) (core/src/view.cpp:105-118): adopts
 * caller-owned device blobs (not freed by lam_view_free).  `blob_bytes` (required: a Blob
 * always knows its size) is checked like the reference ("blob count mismatch" / "blob size
 * mismatch"); NULL fails with "blob size mismatch".  Blob pointers must be 16-byte aligned. */
int lam_view_wrap(const lam_layout* layout, int device, void* const* device_blobs, const uint64_t* blob_bytes,
                  size_t n_blobs, lam_view** out);
void lam_view_free(lam_view* view);
/* View::isTriviallyRelocatable / blobBytes / stateBytes (core/src/view.cpp:145-162):
 * relocatable = fully static extents, no mutable state, no runtime state; state = blob bytes
 * + runtime state bytes (acceptance criterion 10, acceptance.cpp:772-790). */
int lam_view_is_trivially_relocatable(const lam_view* view);
uint64_t lam_view_blob_bytes(const lam_view* view);
uint64_t lam_view_state_bytes(const lam_view* view);
const lam_layout* lam_view_layout(const lam_view* view);
void* lam_view_blob(const lam_view* view, size_t nr);
/* Device pointer to the view's lowered plan (struct lamp_view): the argument user kernels pass
 * to lamina_b200::DeviceView (include/lamina_b200_device.cuh) to read / write the view through
 * its mapping from their own kernels (View::read/write/load/store, view.hpp:144-181). */
const void* lam_view_device_plan(const lam_view* view);
/* Stream-ordered host<->device blob transfer (pinned host memory makes them async). */
int lam_view_upload(lam_view* view, size_t nr, const void* host, void* stream);
int lam_view_download(const lam_view* view, size_t nr, void* host, void* stream);
/* Byte sub-range [offset, offset + nbytes) of blob nr (the reference exposes blobs as spans,
 * View::blobs(), view.hpp:133-141); out-of-bounds ranges fail with "index out of range". */
int lam_view_upload_range(lam_view* view, size_t nr, uint64_t offset, uint64_t nbytes, const void* host,
                          void* stream);
int lam_view_download_range(const lam_view* view, size_t nr, uint64_t offset, uint64_t nbytes, void* host,
                            void* stream);

/* ---- view dump / restore (core/include/lamina/view_io.hpp; core/src/view_io.cpp:28-129) ----
 * The reference's on-disk format: <stem>.meta (schema=, extents=, extent-values=, mapping=,
 * blobs=, blob<nr>-size=) and <stem>.blob<nr>.bin.  lam_view_dump = writeViewDump (blobs are
 * read back from the device), lam_view_restore = readViewDump (a new layout + device view;
 * the caller frees both), with readViewDump's error messages ("cannot read", "malformed
 * sidecar line", "sidecar missing field", "blob count mismatch", "blob size mismatch",
 * "blob file truncated") as LAM_ERUNTIME.  lam_layout_dump_meta returns the .meta text. */
size_t lam_layout_dump_meta(const lam_layout* layout, char* buf, size_t cap);
int lam_view_dump(const lam_view* view, const char* stem);
int lam_view_restore(const char* stem, int device, void* stream, lam_layout** layout_out, lam_view** view_out);

/* ---- the hot path: layout-aware copy ---------------------------------------------------
 * Replaces lamina::copyView(const View& src, View& dst)  (core/include/lamina/view.hpp:285,
 * core/src/view.cpp:168-189).  Same contract: schema and extents must be equal
 * ("incompatible views"); equal fully-physical, uninstrumented layouts copy blob-wise
 * (view.cpp:175-181); everything else copies fieldwise with dst's projection applied
 * (truncation, type change, byte split, bit packing, counting).  Bit-exact to the
 * reference, including bytes it never writes (padding, AoSoA tail lanes, bit-stream tail). */
int lam_copy(const lam_view* src, lam_view* dst, void* stream);
/* Same, over the element range [begin, end) only (both multiples of lam_layout_shard_unit
 * of src and dst, or end == element count): the per-shard call of a multi-GPU copy. */
int lam_copy_range(const lam_view* src, lam_view* dst, uint64_t begin, uint64_t end, void* stream);
/* lam_copy for n (src[k], dst[k]) pairs, each on its own device (SURVEY 8(b) lam_copy_sharded):
 * all copies in flight at once on per-device streams, returns when all are done. */
int lam_copy_sharded(const lam_view* const* src, lam_view* const* dst, size_t n);
/* copyView over HOST views: host blobs in, host blobs out (dst blobs are in/out so that
 * bytes the copy never writes keep their values).  Streams chunks through the GPU with
 * overlapped H2D / kernel / D2H.  Synchronous.  Host memory should be pinned.  The counter
 * outputs (optional) receive per side the FieldAccessCount deltas reads[leaves], writes[leaves]
 * (if the side counts) followed by the Heatmap block counters of every blob (if it has one). */
int lam_copy_host(const lam_layout* src_layout, const void* const* src_host_blobs, const lam_layout* dst_layout,
                  void* const* dst_host_blobs, int device, uint64_t* src_counters, uint64_t* dst_counters);

/* ---- instrumentation ---------------------------------------------------------------------
 * FieldAccessCount::counters()/reset() (instrument.hpp:56-58): reads[leaves], writes[leaves]. */
int lam_counters_read(const lam_view* view, uint64_t* reads, uint64_t* writes);
int lam_counters_reset(lam_view* view, void* stream);
/* Heatmap::blockCounter over blob nr (instrument.hpp:112): out[blocks(nr)]. */
int lam_heatmap_read(const lam_view* view, size_t nr, uint64_t* out);

/* ---- scalar access (host-side convenience; generic funnel View::read/write, view.cpp:120-128)
 * Values are storage bits of the leaf's logical type (ScalarValue::storageBits, scalar.hpp:231).
 * Runs one tiny device launch per call batch: n (linear, leaf) pairs. */
int lam_view_read_values(const lam_view* view, const uint64_t* linear, const uint32_t* leaf, uint64_t* bits_out,
                         size_t n, void* stream);
int lam_view_write_values(lam_view* view, const uint64_t* linear, const uint32_t* leaf, const uint64_t* bits,
                          size_t n, void* stream);

/* ---- n-body (tools/nbody) ------------------------------------------------------------------
 * The paper's all-pairs benchmark over any mapping of
 * Record{Pos:{x,y,z},Vel:{x,y,z},Mass} (f32 or f64 leaves).
 * lam_nbody_init   = drawInitValues(seed) + initView  (tools/nbody/runner.cpp:30-58)
 * lam_nbody_update = updateStep   (tools/nbody/steps.hpp:13-42, kernel.hpp:15-41); updates
 *                    Vel of elements [i_begin, i_end) against ALL j in index order.
 * lam_nbody_move   = moveStep     (tools/nbody/steps.hpp:97-118) over [i_begin, i_end).
 * lam_nbody_checksum = checksumView (runner.cpp:62-72): Σ pos in double, index order.
 * On an instrumented view (FieldAccessCount and/or Heatmap) update and move also add the
 * counts the reference runner's funnel accessor produces (runner.cpp:344-436): update reads
 * Pos/Mass of every j once per i in the range and reads 7 / writes 3 leaves of each i; move
 * reads Pos+Vel and writes Pos of each i.  Counts are exact (not sampled). */
int lam_nbody_init(lam_view* view, uint64_t seed, void* stream);
int lam_nbody_update(lam_view* view, int mode, uint64_t i_begin, uint64_t i_end, void* stream);
int lam_nbody_move(lam_view* view, uint64_t i_begin, uint64_t i_end, void* stream);
/* One runner step (runner.cpp:387-421): lam_nbody_update then lam_nbody_move over [i_begin, i_end). */
int lam_nbody_step(lam_view* view, int mode, uint64_t i_begin, uint64_t i_end, void* stream);
int lam_nbody_checksum(const lam_view* view, double* out);

/* The reference's hand-written baselines (tools/nbody/steps.hpp:124-230, runner.cpp:239-323:
 * layouts "manual-aos" = ManualParticle[], "manual-soa" = ManualSoA) as plain device kernels
 * without mappings: state drawn by drawInitValues(seed), update (mode EXACT | FAST), move,
 * checksum as runManual.  They measure the library-vs-hand-written ratio (paper Fig. 3). */
typedef struct lam_nbody_manual lam_nbody_manual;
int lam_nbody_manual_create(const char* kind, uint64_t n, int f64, uint64_t seed, int device, void* stream,
                            lam_nbody_manual** out);
int lam_nbody_manual_update(lam_nbody_manual* m, int mode, void* stream);
int lam_nbody_manual_move(lam_nbody_manual* m, void* stream);
int lam_nbody_manual_checksum(const lam_nbody_manual* m, double* out);
void lam_nbody_manual_free(lam_nbody_manual* m);
/* The fused multi-GPU update step: elements [i_begin, i_end) of `view` against j-sources read
 * directly from other views -- view k supplies particles [j_begin[k], j_end[k]) (global indices,
 * visited in the given order, so exact mode matches the single-view update when the ranges tile
 * [0, n) in order).  Peer GPUs' shards are mapped with lam_ipc_open and wrapped as views
 * (lam_view_wrap) on the updating device: the all-gather of the reference's one-process loop
 * (steps.hpp:13-42) becomes NVLink loads inside the update kernel.  Up to 64 sources. */
int lam_nbody_update_multi(lam_view* view, const lam_view* const* j_views, const uint64_t* j_begin,
                           const uint64_t* j_end, size_t n_sources, int mode, uint64_t i_begin, uint64_t i_end,
                           void* stream);
/* CUDA IPC of device allocations (64-byte handles) for the fused multi-GPU step. */
/* Positions-only exchange of the multi-GPU step: particles [i_begin, i_end) of the
 * view packed into `out` (device) as SoA x[cnt], y[cnt], z[cnt] (and m[cnt] with with_mass),
 * cnt = i_end - i_begin, in the view's float type; read through the view's mapping. */
int lam_nbody_pack_positions(const lam_view* view, uint64_t i_begin, uint64_t i_end, int with_mass, void* out,
                             void* stream);
int lam_ipc_get_handle(const void* device_ptr, void* handle64_out);
int lam_ipc_open(const void* handle64, int device, void** device_ptr);
int lam_ipc_close(void* device_ptr);

/* ---- misc ------------------------------------------------------------------------------- */
/* Number of kernels this library launched on the calling process (all devices). */
uint64_t lam_launch_count(void);
/* Measurement helper (n-body roofline denominator): sustained FP32 FFMA throughput of the
 * device over about `seconds`, in TFLOP/s (2 flops per FMA). */
int lam_bench_fma_peak(int device, double seconds, double* tflops);
int lam_device_sync(int device);

#ifdef __cplusplus
}
#endif

#endif /* LAMINA_B200_H */

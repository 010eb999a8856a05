/*
 * sentinel_b200 -- C ABI of the B200 hashing engine.
 *
 * The reference (`sentinel`, /root/reference/pkg/src/sentinel) is pure Python
 * and has no FFI seam of its own; its drop-in boundary is the function API
 * re-exported in __init__.py:3-43. Each entry point below is what a binding
 * for one of those functions calls. All pointers named d_* are DEVICE
 * pointers; everything else is host memory. Every launch goes to the
 * caller's stream and nothing synchronises unless stated. The library never
 * owns caller memory and keeps no mutable global state.
 *
 * Return value: 0 on success, a negative snt_status otherwise. No C++
 * exception crosses this boundary. The Python package maps the codes onto the
 * reference's exception classes (errors.py:4-33).
 */
#ifndef SENTINEL_B200_H
#define SENTINEL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* cudaStream_t without pulling in the CUDA headers. */
typedef void* snt_stream_t;

typedef enum snt_status {
    SNT_OK = 0,
    SNT_ERR_INVALID_INPUT = -1, /* errors.py:8  InvalidInput  (empty model, zero blocks) */
    SNT_ERR_INVALID_STATE = -2, /* errors.py:12 InvalidState  (reduce_level on < 2 digests) */
    SNT_ERR_CONFIG = -3,        /* errors.py:16 ConfigError   (bad block size / algorithm) */
    SNT_ERR_VALIDATION = -4,    /* errors.py:24 ValidationError */
    SNT_ERR_RESOURCE = -5       /* errors.py:28 ResourceError (CUDA failure, workspace too small) */
} snt_status;

/* compression.py:19-22 CompressionAlg; digest lengths compression.py:39-43. */
typedef enum snt_alg { SNT_SHA256 = 0, SNT_BLAKE2B = 1, SNT_SHA3_256 = 2 } snt_alg;

#define SNT_LEVELS_TO_ROOT 0xffffffffu

const char* snt_strerror(int status);
/* Last CUDA error string seen by this thread's failing call (diagnostics). */
const char* snt_last_cuda_error(void);
uint32_t snt_abi_version(void);
/* Diagnostic: kernels launched by this library in this process so far. */
uint64_t snt_debug_launch_count(void);
/* How snt_merkle_inplace / snt_merkle_leaves / snt_lthash_* schedule their work (process-wide; returns the previous
 * setting, an unknown value changes nothing). All three give bit-identical results.
 *   SNT_SCHEDULE_PERSISTENT (default): one persistent CTA per SM, leaves hashed in warp-wide chains with a
 *       time-sliced tail (csrc/merkle_fused.cuh), then the level-reducer launches. Fastest on every measured
 *       configuration.
 *   SNT_SCHEDULE_FUSED: the same leaf scheduling with the tree folded into the SAME launch through
 *       completion counters -- one launch per hash (needs >= 5 levels and an initialised workspace,
 *       otherwise falls back to PERSISTENT).
 *   SNT_SCHEDULE_GRID: one thread per leaf (or sample) on a plain grid, then the level reducer (round 1's
 *       path).
 * The LtHash entry points pick between their plain grid and their persistent chain kernel by item length
 * and launch size under PERSISTENT; FUSED forces the chain kernel, GRID the grid. */
typedef enum snt_schedule { SNT_SCHEDULE_PERSISTENT = 0, SNT_SCHEDULE_FUSED = 1, SNT_SCHEDULE_GRID = 2 } snt_schedule;
int snt_merkle_schedule(int schedule);
/* Diagnostic: a device buffer of 6 x u64 per SM (zeroed by the caller) into which every persistent CTA of
 * the fused kernel writes {start ns, last warp exit ns, group reductions done, chain slices run, last
 * chain finished ns, unused}; NULL (the default) turns tracing off. */
void snt_debug_fused_trace(void* d_trace);
/* 32, 64, 32 -- or 0 for an unknown algorithm. */
uint32_t snt_digest_len(int alg);

/* ---- model block table ---------------------------------------------------
 * Replaces BlockTable.build (model.py:137-146): a per-tensor table
 * (address, byte length, first leaf index) kept on the device, searched by
 * the kernels. Empty tensors own no leaves; the last leaf of a tensor is
 * hashed at its true length. Creating a plan allocates one small device
 * buffer with the stream-ordered allocator and fills it with an asynchronous
 * copy on `stream`; use the plan on that stream (or order other streams after
 * it). Destroying it frees the buffer in stream order. Hashing calls never
 * allocate and nothing here synchronises the device.
 */
typedef struct snt_model_plan snt_model_plan;

int snt_model_plan_create(const void* const* d_tensor_ptrs, const uint64_t* tensor_nbytes,
                          uint32_t n_tensors, uint32_t block_size, snt_stream_t stream,
                          snt_model_plan** out_plan);
void snt_model_plan_destroy(snt_model_plan* plan);
uint64_t snt_model_plan_leaf_count(const snt_model_plan* plan);
uint64_t snt_model_plan_total_bytes(const snt_model_plan* plan);

/* Bytes of scratch snt_merkle_inplace / snt_merkle_root / snt_merkle_reduce_levels need for
 * `count` leaves or input digests of `alg` (0 for an unknown algorithm). The workspace holds the
 * reducer's ping-pong levels and, behind them, the state of the fused single-launch kernel
 * (completion counters, stage nodes, parked chain states). A workspace belongs to one
 * (alg, count) and to one call at a time. */
size_t snt_merkle_work_bytes(int alg, uint64_t count);

/* Zero a fresh workspace (asynchronous memset on `stream`). Required once before the first
 * snt_merkle_inplace that uses it; every call hands the workspace back ready for the next one
 * (the kernel returns each counter to zero as it consumes it), so launches need no memset. */
int snt_merkle_work_init(void* d_work, size_t work_bytes, snt_stream_t stream);

/* Leaf stage alone: hash_blocks over the in-place block table (model.py:300-305,
 * merkle.py:93-114). Leaf k of [leaf_begin, leaf_end) is written at
 * d_leaves + (k - leaf_begin) * digest_len. */
int snt_merkle_leaves(const snt_model_plan* plan, int alg, uint64_t leaf_begin, uint64_t leaf_end,
                      void* d_leaves, snt_stream_t stream);

/* inplace_hash, MERKLE construction (model.py:298-310): hash leaves
 * [leaf_begin, leaf_end) of the plan and reduce them `levels` tree levels.
 *   levels = SNT_LEVELS_TO_ROOT with the full range: d_out receives the root
 *   (for a one-leaf model, the leaf itself -- merkle.py:159-160).
 *   levels = k with leaf_begin a multiple of 2^k and leaf_end a multiple of
 *   2^k or the leaf count: d_out receives the ceil((end-begin)/2^k) level-k
 *   nodes of that range (multi-GPU sharding; nodes combine with
 *   snt_merkle_root / snt_merkle_reduce_levels into the reference root).
 * d_leaves (may not be NULL) receives every leaf digest of the range.
 * The workspace must hold snt_merkle_work_bytes(alg, leaf_end - leaf_begin) bytes prepared by
 * snt_merkle_work_init. Launches: one for the leaves plus one to three for the levels, or a single
 * one under SNT_SCHEDULE_FUSED (see snt_merkle_schedule).
 */
int snt_merkle_inplace(const snt_model_plan* plan, int alg, uint64_t leaf_begin,
                       uint64_t leaf_end, uint32_t levels, void* d_leaves, void* d_work,
                       size_t work_bytes, void* d_out, snt_stream_t stream);

/* hash_blocks (merkle.py:93-114): d_out[i] = H(d_base[d_off[i] .. +d_len[i]]).
 * Blocks may be empty, ragged and unaligned. n == 0 -> SNT_ERR_INVALID_INPUT. */
int snt_hash_blocks(int alg, const void* d_base, const uint64_t* d_off, const uint64_t* d_len,
                    uint64_t n, void* d_out, snt_stream_t stream);

/* reduce_level (merkle.py:117-149) generalised to `levels` consecutive
 * levels over the node range [first, first + n_in) of a level that has
 * `level_count` nodes in the whole tree. first must be a multiple of
 * 2^levels; first + n_in must be level_count or a multiple of 2^levels.
 * Writes ceil(n_in / 2^levels) nodes. An odd level pairs its last node with
 * zero bytes; levels are never skipped (a lone node is paired with zeros: the
 * shard rule), so the reference's "fewer than two digests" InvalidState
 * (merkle.py:125-126) is raised by the Python reduce_level wrapper, not here.
 * d_out must not alias d_in. */
int snt_merkle_reduce_levels(int alg, const void* d_in, uint64_t first, uint64_t n_in,
                             uint64_t level_count, uint32_t levels, void* d_work,
                             size_t work_bytes, void* d_out, snt_stream_t stream);

/* merkle_root (merkle.py:152-165): count == 1 copies the leaf;
 * count == 0 -> SNT_ERR_INVALID_INPUT. d_nodes is not modified. */
int snt_merkle_root(int alg, const void* d_nodes, uint64_t count, void* d_work, size_t work_bytes,
                    void* d_root, snt_stream_t stream);

/* ---- LtHash ------------------------------------------------------------------
 * Accumulators are n_sources x 32 u64 lanes (sums modulo 2^64 of the u16
 * lanes; exact modulo 2^16 after snt_lt_finalize), n_sources u64 counts and a
 * u64 status word. Calls ADD into them (zero them first for a fresh digest), so
 * batches stream through the same accumulators (SourceAccumulator,
 * dataset.py:52-71). Everything is u64 so that a caller can keep lanes, counts
 * and status in ONE array and combine the partial accumulators of several GPUs
 * with a single 64-bit sum all-reduce, nothing packed or unpacked.
 */

/* process_batch / hash_sample (dataset.py:41-49, :74-86): sample i is
 * d_shard[d_off[i] .. +d_len[i]], digest BLAKE2b-512(LE64(d_ids[i]) || sample),
 * added into source slot d_slot[i]. A sample whose slot is >= n_sources is
 * skipped and counted in *d_status (if not NULL): non-zero = undeclared source.
 * d_digests, if not NULL, receives the n x 64 per-sample digests. */
int snt_lthash_samples(const void* d_shard, const uint64_t* d_off, const uint64_t* d_len,
                       const uint64_t* d_ids, const uint32_t* d_slot, uint64_t n,
                       uint32_t n_sources, uint64_t* d_acc, uint64_t* d_counts, void* d_digests,
                       uint64_t* d_status, snt_stream_t stream);

/* The same with what the caller knows about the sample lengths (it built d_len). Results never depend on
 * it; the launch does: SNT_SAMPLES_UNKNOWN / _RAGGED take the persistent-lane kernel (every lane of a warp
 * fetches its next sample the moment it finishes one, so ragged samples need no sorting), _UNIFORM -- all
 * n lengths equal -- the one-thread-per-sample grid. snt_lthash_samples == shape SNT_SAMPLES_UNKNOWN. */
typedef enum snt_samples_shape { SNT_SAMPLES_UNKNOWN = 0, SNT_SAMPLES_UNIFORM = 1, SNT_SAMPLES_RAGGED = 2 } snt_samples_shape;
int snt_lthash_samples_shaped(const void* d_shard, const uint64_t* d_off, const uint64_t* d_len,
                              const uint64_t* d_ids, const uint32_t* d_slot, uint64_t n,
                              uint32_t n_sources, uint64_t* d_acc, uint64_t* d_counts, void* d_digests,
                              uint64_t* d_status, uint32_t shape, snt_stream_t stream);

/* The loader-side form of process_batch (dataset.py:74-86; the on-the-fly use of the paper): a batch as a GPU data
 * loader holds it -- n rows of row_bytes bytes each in one device tensor -- with the raw source id of every row.
 * The slot of a row is found inside the kernel by binary search of d_src_ids[i] in d_table, the n_sources declared
 * source ids in ascending order; an id that is not in the table is skipped and counted in *d_status. One launch
 * per batch, nothing else. */
int snt_lthash_rows(const void* d_rows, uint64_t row_bytes, uint64_t n, const uint64_t* d_ids,
                    const int64_t* d_src_ids, const int64_t* d_table, uint32_t n_sources, uint64_t* d_acc,
                    uint64_t* d_counts, void* d_digests, uint64_t* d_status, snt_stream_t stream);

/* inplace_hash, LATTICE construction (model.py:312-315): leaves
 * [leaf_begin, leaf_end) tagged LE64(k), summed into d_acc[32] / d_counts[1]. */
int snt_lthash_model(const snt_model_plan* plan, uint64_t leaf_begin, uint64_t leaf_end,
                     uint64_t* d_acc, uint64_t* d_counts, void* d_digests, snt_stream_t stream);

/* per_layer_hash, LATTICE construction (model.py:255-262): block j of tensor i is
 * tagged LE64(i) || LE64(j) and added into slot i of d_acc[n_tensors x 32] /
 * d_counts[n_tensors]; an empty tensor keeps the zero digest. */
int snt_lthash_model_layers(const snt_model_plan* plan, uint64_t leaf_begin, uint64_t leaf_end,
                            uint64_t* d_acc, uint64_t* d_counts, void* d_digests,
                            snt_stream_t stream);

/* per_layer_hash, MERKLE construction (model.py:245-253): one tree per segment.
 * Segment t owns digests [seg_first[t], seg_first[t+1]) of d_digests (seg_first is a
 * HOST array of n_segments + 1 entries); its root (merkle_root rule) goes to
 * d_out + t * digest_len. An empty segment receives d_empty_digest (the digest of
 * the empty message, model.py:247-248). */
int snt_merkle_roots_segmented(int alg, const void* d_digests, const uint64_t* seg_first,
                               uint32_t n_segments, const void* d_empty_digest, void* d_work,
                               size_t work_bytes, void* d_out, snt_stream_t stream);

/* Staging of host-resident models (the reference-shaped call, hash_model on host buffers): n asynchronous
 * host-to-device copies h_src[i] -> d_dst[i] of nbytes[i] bytes on `stream`, issued back to back from C. A state
 * dict has hundreds of small tensors (biases, norms) whose DMA takes a microsecond; issuing their copies one
 * Python call at a time leaves the link idle between them (5 ms of a 123 ms GPT2-XL transfer). Page-locked
 * sources copy asynchronously; pageable ones are staged by the driver. Zero-length entries are skipped. */
int snt_memcpy_h2d_batch(void* const* d_dst, const void* const* h_src, const uint64_t* nbytes, uint32_t n,
                         snt_stream_t stream);

/* 1 when kernels of the current device can read page-locked host memory through the host pointer itself (unified
 * addressing, and registered memory usable under its host address): then snt_gather_spans may be given page-locked
 * HOST source addresses, which is how hash_model fetches the many small tensors of a pinned state dict with one
 * launch instead of one copy-engine transfer (~3.7 us) each. 0: the caller keeps to snt_memcpy_h2d_batch. */
int snt_device_reads_pinned_host(void);

/* Data movement of the strategies that copy before hashing: span i =
 * d_len[i] bytes at device address d_src_addr[i] goes to d_dst + d_dst_off[i];
 * with pad_block != 0 the span is zero-filled up to the next multiple of
 * pad_block. coalesce_hash (model.py:203-228) packs every tensor this way
 * (pad_block = 0); per_layer_hash (model.py:245-253) zero-pads the ragged last
 * block of each tensor (pad_block = block size, spans = the tails only).
 * d_chunk_first[n_spans + 1] is the running count of 32 KiB chunks
 * (snt_gather_chunk_bytes) of the padded spans; n_chunks = its last entry.
 * All four arrays are DEVICE pointers. Destination ranges must not overlap. */
uint32_t snt_gather_chunk_bytes(void);
int snt_gather_spans(const uint64_t* d_src_addr, const uint64_t* d_len, const uint64_t* d_dst_off,
                     const uint64_t* d_chunk_first, uint32_t n_spans, uint64_t n_chunks,
                     uint32_t pad_block, void* d_dst, snt_stream_t stream);

/* lt_reduce (lattice.py:104-119): add n 64-byte digests into d_acc[32]. */
int snt_lt_reduce(const void* d_digests, uint64_t n, uint64_t* d_acc, snt_stream_t stream);

/* Mask to 16 bits and pack: d_out receives n_sources x 64 bytes
 * (LatticeDigest layout, lattice.py:37-58). */
int snt_lt_finalize(const uint64_t* d_acc, uint32_t n_sources, void* d_out, snt_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SENTINEL_B200_H */

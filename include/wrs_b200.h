/*
 * include/wrs_b200.h -- B200 extensions to the wrs.h ABI (libwrs_b200.so).
 *
 * Everything here is additive: a reference client never needs it.  It exposes
 * what a GPU caller wants beyond the reference surface -- device-resident
 * input and output (so a 4 GB draw need not round-trip through the host), an
 * explicit PSA job count, asynchronous rebuild/draw on a caller stream for
 * timing, the sharded multi-GPU pieces, and read-back of the table and of the
 * build's intermediate arrays for parity tests.  Plain pointers and sizes
 * only; streams are passed as void* (a cudaStream_t, NULL = the handle's own).
 */
#ifndef WRS_B200_H
#define WRS_B200_H

#include "wrs.h"

#ifdef __cplusplus
extern "C" {
#endif

/* PSA job count "psa" uses for n items.  The table depends on it
 * (alias.hpp:211-213 keeps only masses invariant), so parity tests run the
 * reference at this same count. */
WRS_API uint64_t wrs_b200_default_jobs(uint64_t n);

/* The library keeps freed device buffers for reuse (at most WRS_B200_CACHE_MB,
 * default 8192 MB, per process).  Returns every cached buffer to the driver
 * and the number of bytes released. */
WRS_API uint64_t wrs_b200_release_cache(void);

/* Checked builds (make -C paper_1903_00227_b200/csrc checked ->
 * libwrs_b200_checked.so): the number of device-side index-check violations
 * so far, the first offending source line in *first_line.  -1 in the normal
 * build (no checks compiled in). */
WRS_API int64_t wrs_b200_check_failures(unsigned* first_line);

/* Weights already in device memory of the current CUDA device.  copy != 0
 * duplicates them; copy == 0 borrows d_w (caller keeps it alive and
 * unchanged until every handle built from it is freed). */
WRS_API wrs_status wrs_b200_weights_from_device(const double* d_w, uint64_t n, int copy,
                                                wrs_weights** out);
/* Items [lo, hi) of the global vector wrs_weights_generate(dist, param,
 * n_total, seed) would produce, generated on the device (a shard's slice):
 * "uniform" is counter-based (only the slice is generated); "powerlaw" deals
 * all n_total items (its Fisher-Yates is global, resolved in parallel on the
 * device, generate_kernels.cu) and keeps the slice.  wrs_weights_generate
 * ("powerlaw") uses the same device deal. */
WRS_API wrs_status wrs_b200_weights_generate_range(const char* dist, double param,
                                                   uint64_t n_total, uint64_t lo, uint64_t hi,
                                                   uint64_t seed, wrs_weights** out);
/* Pairwise total W (weights.hpp:19-28, bit-exact) and the device pointer. */
WRS_API double wrs_b200_weights_total(const wrs_weights* w);
WRS_API const double* wrs_b200_weights_device(const wrs_weights* w);

/* Build flags. */
#define WRS_B200_KEEP_WORKSPACE 1u /* keep intermediates for wrs_b200_sampler_stage */

/* PSA build with an explicit job count (0 = wrs_b200_default_jobs(n)). */
WRS_API wrs_status wrs_b200_sampler_build_psa(const wrs_weights* w, uint64_t jobs,
                                              unsigned flags, wrs_sampler** out);
WRS_API uint64_t wrs_b200_sampler_jobs(const wrs_sampler* s);
WRS_API uint64_t wrs_b200_sampler_size(const wrs_sampler* s);
WRS_API double wrs_b200_sampler_bucket_mean(const wrs_sampler* s);
WRS_API double wrs_b200_sampler_total(const wrs_sampler* s);
/* Table as 16-byte {double share; uint32 item; uint32 alias} records
 * (alias.hpp:26-33 byte layout). */
WRS_API const void* wrs_b200_sampler_device_buckets(const wrs_sampler* s);
WRS_API wrs_status wrs_b200_sampler_copy_buckets(const wrs_sampler* s, void* host_out);

/* Re-run the build (K1..K4b; W comes from the weights handle, as the
 * reference's AliasTable takes it from its WeightTable) in place,
 * asynchronously on `stream`; no host synchronisation.  Plan errors are
 * latched on the device and reported by wrs_b200_sampler_check. */
WRS_API wrs_status wrs_b200_sampler_rebuild_async(wrs_sampler* s, void* stream);
/* Give the sampler a second table: from then on a rebuild writes the table
 * the draws are not reading (after the draws that last read it finish) and
 * does not hold up `stream`; draws issued after it read the new table (they
 * wait for it on their own stream).  Lets a rebuild on one stream overlap the
 * draws of the previous table on another.  Table pointers / IPC handles then
 * refer to the table current at the time of the call. */
WRS_API wrs_status wrs_b200_sampler_double_buffer(wrs_sampler* s);
WRS_API wrs_status wrs_b200_sampler_check(const wrs_sampler* s);

/* Draw into device memory, asynchronously on `stream`.  Same values as
 * wrs_sampler_draw(s, seed, count, workers, ...). */
WRS_API wrs_status wrs_b200_sampler_draw_device(const wrs_sampler* s, uint64_t seed,
                                                uint64_t count, unsigned workers,
                                                uint32_t* d_out, void* stream);

/* Philox draw mode (north star: counter-based Philox uniforms): draw q of
 * the call is Philox4x32-10(counter (q_lo, q_hi, 0, 0), key (seed_lo,
 * seed_hi)) -> words o0..o3; bucket = ((o1:o0) * n) >> 64, coin = ((o3:o2)
 * >> 11) * 2^-53 * bucket_mean, answer ia[coin >= share] (alias.hpp:265-269).
 * Not the reference's stream (wrs_sampler_draw is); checked by replaying the
 * same uniforms on the table.  Device output, asynchronous on `stream`. */
WRS_API wrs_status wrs_b200_sampler_draw_philox_device(const wrs_sampler* s, uint64_t seed,
                                                       uint64_t count, uint32_t* d_out,
                                                       void* stream);

/* Aggregated draws: the distinct items of
 * wrs_sampler_draw(s, seed, k, workers, ...) with their multiplicities,
 * items ascending.  items / counts hold min(k, n) entries; *n_unique gets
 * the number written; the counts sum to k.  The draws are the same as the
 * plain draw's, so the pairs are exactly the histogram of that output.
 * _device: device outputs (n_unique too), asynchronous on `stream`. */
WRS_API wrs_status wrs_b200_sampler_draw_counts(const wrs_sampler* s, uint64_t seed, uint64_t k,
                                                unsigned workers, uint32_t* items,
                                                uint64_t* counts, uint64_t* n_unique);
WRS_API wrs_status wrs_b200_sampler_draw_counts_device(const wrs_sampler* s, uint64_t seed,
                                                       uint64_t k, unsigned workers,
                                                       uint32_t* d_items, uint64_t* d_counts,
                                                       uint64_t* d_n_unique, void* stream);

/* implied_masses (verify.hpp:43-54) of the sampler's table into out[0..n)
 * (host or device) and, if worst is not NULL, max_relative_mass_error
 * (verify.hpp:92-98) against the weights -- on the device, bit for bit.
 * wrs_sampler_verify_masses uses the same computation.  n < 2^31. */
WRS_API wrs_status wrs_b200_sampler_implied_masses(const wrs_sampler* s, double* out,
                                                   double* worst);

/* Copy a named intermediate of the last build (needs WRS_B200_KEEP_WORKSPACE):
 * "counts" (u64 nl, nh), "heavy" (u32 heavy ids), "light_w", "heavy_w" (f64),
 * "light_prefix", "heavy_prefix" (f64, n_x + 1 entries; builds of large
 * tables keep instead "light_ckpt", "heavy_ckpt": f64 (hi, lo) pairs, the
 * prefix chain's state before every 16th element), "block_totals",
 * "carries" (f64, light blocks then heavy blocks), "split_light",
 * "split_heavy" (u32, P + 1), "split_spill" (f64, P + 1), "light_rank"
 * (u32, nl: the heavy rank j each light was paired with; its alias is
 * heavy[min(j, nh-1)]), "heavy_share" (f64, nh).  *bytes
 * receives the size; host_out may be NULL to query it. */
WRS_API wrs_status wrs_b200_sampler_stage(const wrs_sampler* s, const char* name,
                                          void* host_out, uint64_t capacity,
                                          uint64_t* bytes);

/* Device time of each build stage of the last wrs_b200_sampler_rebuild_async
 * made with timing on (wrs_b200_set_timing(1)), in milliseconds:
 * [K1 partition, K2a block totals, K2b carries, K2c prefixes, K3 splits,
 *  K4a pack, K4b assemble].  Returns the number written. */
WRS_API int wrs_b200_set_timing(int on);
WRS_API int wrs_b200_sampler_stage_times(const wrs_sampler* s, float* ms, int max);

/* ---------------------------------------------------- sharded (multi-GPU)
 * Contiguous shards of ceil(n/G) items (two_level.hpp:33-41).  Each rank
 * builds its shard with "psa" and contributes the shard total; the top table
 * over the G totals is built redundantly on every rank (two_level.hpp:56-57)
 * and k is split across shards by a binomial descent that every rank
 * reproduces from the seed (no communication).  The exchange of the G totals
 * is done by the caller's collective (NCCL allgather of G doubles). */
WRS_API void wrs_b200_shard_range(uint64_t n, uint64_t groups, uint64_t g,
                                  uint64_t* lo, uint64_t* hi);
/* counts[0..G) summing to k: sample counts per shard for (seed, k).  Pure
 * host arithmetic, identical on every rank (binomial.hpp:161-170). */
WRS_API wrs_status wrs_b200_shard_counts(const double* totals, uint64_t groups,
                                         uint64_t seed, uint64_t k, uint64_t* counts);
/* Seed shard g draws with: RngStream(seed, 'sdrw').derive(g) key. */
WRS_API uint64_t wrs_b200_shard_seed(uint64_t seed, uint64_t shard);
/* Draw `count` samples from shard `shard`'s table -- exactly
 * AliasTable(shard).sample_many(wrs_b200_shard_seed(seed, shard), count, 1)
 * -- and add `base` (the shard's first global id) to every index, into device
 * memory, asynchronously on `stream`. */
WRS_API wrs_status wrs_b200_sampler_draw_shard_device(const wrs_sampler* s, uint64_t seed,
                                                      uint64_t shard, uint64_t count,
                                                      uint64_t base, uint32_t* d_out,
                                                      void* stream);

/* -------------------------------------------- multi-GPU sampler (NCCL)
 * One rank per GPU (one process each, or G handles in one process): rank g
 * owns the contiguous shard [g*ceil(n/G), min(n, (g+1)*ceil(n/G))) of the
 * global weight vector (two_level.hpp:33-41), builds its PSA table, and the
 * ranks all-gather their shard totals (each the shard's bit-exact pairwise
 * sum, two_level.hpp:49-51) with one ncclAllGather of G doubles, device to
 * device, over NVLink.  Every rank then builds the same top table over the
 * totals (two_level.hpp:56-57) and derives the same per-rank draw counts for
 * (seed, k) with the communication-free binomial descent
 * (wrs_b200_shard_counts); each rank draws its count from its own table and
 * writes global ids.  The library owns the NCCL communicator; NCCL itself
 * (libnccl.so.2) is loaded at the first multi call, so single-GPU users never
 * need it. */
typedef struct wrs_b200_multi wrs_b200_multi;
/* 1 if libnccl.so.2 can be loaded (its version in *version, may be NULL). */
WRS_API int wrs_b200_nccl_available(int* version);
/* A new NCCL unique id (128 bytes) for one job: rank 0 creates it, the
 * caller hands it to every rank. */
WRS_API wrs_status wrs_b200_nccl_unique_id(void* id128);
/* Rank `rank` of `ranks`: `shard` holds this rank's items (on the current
 * device).  With nccl_id != NULL the communicator is created
 * (ncclCommInitRank, collective over all ranks) and the totals exchanged;
 * with nccl_id == NULL the caller supplies the gathered totals with
 * wrs_b200_multi_set_totals (its own collective). */
WRS_API wrs_status wrs_b200_multi_create(const wrs_weights* shard, uint64_t n_total,
                                         uint32_t rank, uint32_t ranks, const void* nccl_id,
                                         wrs_b200_multi** out);
/* All G ranks in this process, shards[g] on its own device (distinct
 * devices): one ncclCommInitAll, then every rank's exchange in one group. */
WRS_API wrs_status wrs_b200_multi_create_local(const wrs_weights* const* shards, uint32_t ranks,
                                               uint64_t n_total, wrs_b200_multi** out);
WRS_API wrs_status wrs_b200_multi_set_totals(wrs_b200_multi* m, const double* totals);
/* Re-exchange the totals (ncclAllGather on `stream`, device to device; the
 * host copy is read back before returning).  Collective. */
WRS_API wrs_status wrs_b200_multi_exchange(wrs_b200_multi* m, void* stream);
/* Rebuild this rank's shard table on `stream` (wrs_b200_sampler_rebuild_async). */
WRS_API wrs_status wrs_b200_multi_rebuild_async(wrs_b200_multi* m, void* stream);
WRS_API wrs_status wrs_b200_multi_totals(const wrs_b200_multi* m, double* totals);
/* counts[0..ranks) for (seed, k), identical on every rank. */
WRS_API wrs_status wrs_b200_multi_counts(const wrs_b200_multi* m, uint64_t seed, uint64_t k,
                                         uint64_t* counts);
/* This rank's draws of the k-draw job (global ids) into d_out, asynchronous
 * on `stream`; *count gets how many (counts[rank]).  The same values as
 * wrs_b200_sampler_draw_shard_device(shard table, seed, rank, count, lo). */
WRS_API wrs_status wrs_b200_multi_draw_device(const wrs_b200_multi* m, uint64_t seed,
                                              uint64_t k, uint32_t* d_out, void* stream,
                                              uint64_t* count);
/* The top table over the gathered totals (ranks 16-B buckets) and its mean. */
WRS_API wrs_status wrs_b200_multi_top_buckets(const wrs_b200_multi* m, void* host_out,
                                              double* bucket_mean);
/* This rank's shard sampler (owned by the handle; do not free). */
WRS_API const wrs_sampler* wrs_b200_multi_shard(const wrs_b200_multi* m);
WRS_API void wrs_b200_multi_free(wrs_b200_multi* m);

/* ------------------------------------------ routed two-level draws (§8f 2)
 * TwoLevelTable::sample_many(seed, k, workers) (two_level.hpp:66-81),
 * outputs [q_begin, q_end) into d_out[0 .. q_end - q_begin): per query the
 * top table (groups buckets, mean top_mean) picks group g, then g's table
 * (d_tables[g]: sizes[g] buckets of 16 B, mean bucket_means[g]) the local
 * item; the answer is bases[g] + item.  Tables may be peer-GPU memory (e.g.
 * opened with wrs_b200_ipc_open): each query then gathers its bucket over
 * NVLink.  groups <= 256.  Asynchronous on `stream`. */
WRS_API wrs_status wrs_b200_two_level_draw_device(const void* const* d_tables,
                                                  const uint64_t* sizes,
                                                  const double* bucket_means,
                                                  const uint64_t* bases, uint64_t groups,
                                                  const void* d_top, double top_mean,
                                                  uint64_t seed, uint64_t q_begin,
                                                  uint64_t q_end, uint64_t k, unsigned workers,
                                                  uint32_t* d_out, void* stream);
/* CUDA IPC of a sampler's table (handle: 64 bytes), for peer processes. */
WRS_API wrs_status wrs_b200_sampler_ipc_handle(const wrs_sampler* s, void* handle);
WRS_API wrs_status wrs_b200_ipc_open(const void* handle, void** d_ptr);
WRS_API wrs_status wrs_b200_ipc_close(void* d_ptr);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* WRS_B200_H */

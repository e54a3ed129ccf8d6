/*
 * semisort_b200 — C ABI of the B200-native semisort / collect-reduce /
 * histogram hot path (arXiv 2304.10078).
 *
 * Every export is extern "C", takes plain pointers and sizes (device
 * pointers as void*, sizes as uint64_t, the CUDA stream as void*), returns
 * an int status and never throws.  Status codes map to the reference's
 * exception types (semisort/errors.py:4-13):
 *   SS_OK             0
 *   SS_ERR_CONFIG     1   -> ConfigurationError (ValueError)
 *   SS_ERR_CONTRACT   2   -> ContractError (TypeError)
 *   SS_ERR_RESOURCE   3   -> MemoryError / RuntimeError (CUDA failure)
 *   SS_ERR_COMM       4   -> RuntimeError (collective failure)
 * ss_last_error() returns a thread-local message for the last failure.
 *
 * Buffers are SoA exactly like the reference RecordArray (records.py:34-132):
 * keys are uint32 or uint64 (key_bytes 4 / 8), and for ss_semisort also
 * 128-bit (key_bytes 16: (lo, hi) uint64 rows, records.py:8-10); values are optional
 * (value_bytes 0 / 4 / 8 / 16).  All work is stream-ordered on `stream`.
 * Callers own every buffer; scratch comes from a caller-provided workspace
 * (size queries below), so the library never allocates on the hot path.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/semisort):
 *   ss_semisort            core.py:566-598      semisort(data, adapter, mode, params)
 *   ss_local_refine        core.py:533-563      local_refine(buffers, plan, ...)
 *   ss_collect_reduce      aggregate.py:267-290 collect_reduce(..., ReduceSpec.summing64())
 *   ss_histogram           aggregate.py:293-299 histogram(data, adapter, params)
 *   ss_sample_heavy        core.py:221-260      sample_and_bucket(data, adapter, params, depth, rng)
 *   ss_assign_bucket_ids   core.py:169-190      assign_bucket_ids(...)
 *   ss_count_matrix        core.py:294-299      count_into_matrix(...) / _counts_from_ids (:268-291)
 *   ss_column_scan         core.py:302-318      column_major_exclusive_scan(counts)
 *   ss_distribute          core.py:339-380      distribute(...) / _distribute_ids(...)
 *   ss_base_case           core.py:404-429      base_case_eq / base_case_lt
 *   ss_partition           (new, multi-GPU)     stable hash partition before the exchange
 *   ss_partition_pairs     (new, multi-GPU)     the same, packed records for ONE exchange
 *   ss_semisort_pairs      core.py:566-598      semisort of received packed records, in place
 *   ss_dist_semisort       (new, multi-GPU)     one rank of the sharded semisort over NCCL
 *   ss_params_for_input    params.py:64-86      TuningParams.for_input for a rank's size
 */
#ifndef SEMISORT_B200_H
#define SEMISORT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_OK 0
#define SS_ERR_CONFIG 1
#define SS_ERR_CONTRACT 2
#define SS_ERR_RESOURCE 3
#define SS_ERR_COMM 4

#define SS_MODE_EQ 0
#define SS_MODE_LT 1

#define SS_AGG_COUNT 0
#define SS_AGG_SUM64 1

/* TuningParams (params.py:38-47) plus the integer heavy threshold
 * ceil(heavy_threshold) computed by the caller from the same float. */
typedef struct ss_params {
  uint64_t input_size;
  uint32_t light_buckets;
  uint32_t light_bits;
  uint64_t subarray_len;
  uint64_t base_case_cutoff;
  uint32_t max_heavy;
  uint32_t sample_factor;
  uint64_t seed;
  uint64_t sample_count;
  uint64_t heavy_threshold_int;
  double heavy_threshold;
} ss_params;

/* Telemetry (core.py:42-61): same counter semantics.  matrix_cells_by_level
 * is indexed by level (1..64).  `timing` (input) != 0 records per-phase
 * device time into phase_ms (sample, count, scan, distribute, copy_back,
 * children, leaves, other). */
typedef struct ss_telemetry {
  uint64_t max_depth;
  uint64_t nodes;
  uint64_t scratch_allocations;
  uint64_t scratch_moves;
  uint64_t bucket_assignments;
  uint64_t matrix_cells_by_level[65];
  uint64_t kernel_launches;
  uint64_t levels;
  uint64_t leaves_smem;
  uint64_t leaves_global;
  uint64_t nodes_folded;   /* aggregation nodes reduced in one pass (node_fold.cuh) */
  uint64_t fold_records;   /* records of those nodes (read once by the fold) */
  int32_t timing;
  int32_t reserved;
  double phase_ms[8];
} ss_telemetry;

const char* ss_last_error(void);
int ss_version(void);

/* ---- whole-path entry points ------------------------------------------- */

uint64_t ss_semisort_workspace_bytes(uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                                     const ss_params* params);

/* In place on (keys, values); mode SS_MODE_EQ / SS_MODE_LT; identity != 0
 * selects the identity hash (adapters.py:112-119).  key_bytes 16 runs the
 * UInt128KeyAdapter semantics (adapters.py:147-198): hash mix64(mix64(hi) ^ lo)
 * (identity: lo), equality on both words, SS_MODE_LT order by (hi, lo);
 * keys must be 16-byte aligned. */
int ss_semisort(void* keys, void* values, uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                int mode, int identity, const ss_params* params, void* workspace,
                uint64_t workspace_bytes, ss_telemetry* telemetry, void* stream);

/* Refine a node already distributed by ss_distribute (core.py:533-563).
 * `offsets` is the host copy of the bucket offsets (n_buckets + 1 entries),
 * live_in_primary says which buffer holds the distributed records. */
int ss_local_refine(void* keys, void* values, void* scratch_keys, void* scratch_values, uint64_t n,
                    uint32_t key_bytes, uint32_t value_bytes, int mode, int identity,
                    const ss_params* params, const int64_t* offsets, uint32_t n_buckets,
                    int live_in_primary, uint32_t depth, void* workspace, uint64_t workspace_bytes,
                    ss_telemetry* telemetry, void* stream);

uint64_t ss_aggregate_workspace_bytes(uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                                      const ss_params* params);

/* Per-key count (SS_AGG_COUNT) or wrapping uint64 sum of the first value
 * word (SS_AGG_SUM64).  The input is not modified.  The distinct-key pairs
 * stay in the workspace: *out_count receives their number, then
 * ss_result_copy moves them to caller buffers (keys as key_bytes, aggregates
 * as uint64). */
int ss_collect_reduce(const void* keys, const void* values, uint64_t n, uint32_t key_bytes,
                      uint32_t value_bytes, int kind, int identity, const ss_params* params,
                      void* workspace, uint64_t workspace_bytes, uint64_t* out_count,
                      ss_telemetry* telemetry, void* stream);
int ss_histogram(const void* keys, uint64_t n, uint32_t key_bytes, int identity,
                 const ss_params* params, void* workspace, uint64_t workspace_bytes,
                 uint64_t* out_count, ss_telemetry* telemetry, void* stream);
int ss_result_copy(const void* workspace, uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                   const ss_params* params, void* out_keys, void* out_aggs, uint64_t count,
                   void* stream);

/* ---- phase-level entry points (the reference's exported phases) ------- */

uint64_t ss_phase_workspace_bytes(uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                                  const ss_params* params);

/* Heavy keys of keys[0..n) sampled from Philox(key=rng_key); written to
 * out_heavy (device, >= max_heavy uint64) in discovery order. */
int ss_sample_heavy(const void* keys, uint64_t n, uint32_t key_bytes, const ss_params* params,
                    uint64_t rng_key, void* out_heavy, uint32_t* out_n_heavy, void* workspace,
                    uint64_t workspace_bytes, void* stream);

int ss_assign_bucket_ids(const void* keys, uint64_t n, uint32_t key_bytes, int identity,
                         const ss_params* params, uint32_t depth, const void* heavy_keys,
                         uint32_t n_heavy, void* out_ids, void* workspace, uint64_t workspace_bytes,
                         void* stream);

/* counts: int64 [ceil(n / subarray_len) x n_buckets].  If ids != NULL the
 * bucket of record i is ids[i] (int32), else it is derived from the key. */
int ss_count_matrix(const void* keys, const void* ids, uint64_t n, uint32_t key_bytes, int identity,
                    const ss_params* params, uint32_t depth, const void* heavy_keys, uint32_t n_heavy,
                    uint32_t n_buckets, void* out_counts, void* workspace, uint64_t workspace_bytes,
                    void* stream);

int ss_column_scan(const void* counts, uint64_t rows, uint32_t n_buckets, void* out_prefix,
                   void* out_offsets, void* workspace, uint64_t workspace_bytes, void* stream);

/* prefix: int64 [ceil(n / subarray_len) x n_buckets] destination cursors. */
int ss_distribute(const void* src_keys, const void* src_values, void* dst_keys, void* dst_values,
                  const void* ids, uint64_t n, uint32_t key_bytes, uint32_t value_bytes, int identity,
                  const ss_params* params, uint32_t depth, const void* heavy_keys, uint32_t n_heavy,
                  uint32_t n_buckets, const void* prefix, void* workspace, uint64_t workspace_bytes,
                  void* stream);

int ss_base_case(void* keys, void* values, uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                 int mode, int identity, void* workspace, uint64_t workspace_bytes, void* stream);
uint64_t ss_base_case_workspace_bytes(uint64_t n, uint32_t key_bytes, uint32_t value_bytes);

/* ---- multi-GPU partition (hash-partition by the top bits of mix64) ----- */

/* Stable partition of (keys, values) into `parts` (a power of two) groups by
 * dest = mix64(key) >> (64 - log2 parts); writes the grouped records to
 * dst_* and the per-group counts (uint64, host) to out_counts. */
int ss_partition(const void* keys, const void* values, uint64_t n, uint32_t key_bytes,
                 uint32_t value_bytes, uint32_t parts, void* dst_keys, void* dst_values,
                 uint64_t* out_counts, void* workspace, uint64_t workspace_bytes, void* stream);
uint64_t ss_partition_workspace_bytes(uint64_t n, uint32_t parts);

/* Packed variant (one exchange instead of one per column): keys and values
 * of the key width (4 or 8 bytes) are written to dst_pairs as (key, value)
 * records, 2n words, grouped by part in stable order. */
int ss_partition_pairs(const void* keys, const void* values, uint64_t n, uint32_t key_bytes,
                       uint32_t parts, void* dst_pairs, uint64_t* out_counts, void* workspace,
                       uint64_t workspace_bytes, void* stream);
uint64_t ss_partition_pairs_workspace_bytes(uint64_t n, uint32_t parts);

/* Semisort of n packed (key, value) records (what a rank receives from the
 * exchange).  The result is left as SoA columns in the SAME memory:
 * keys = words [0, n), values = words [n, 2n) of `pairs`.  scratch: 2n
 * words (e.g. the partition's send buffer, free after the exchange), or
 * NULL to carve it from the workspace (ss_semisort_pairs_workspace_bytes
 * with_scratch = 1).  Otherwise as ss_semisort (core.py:566-598). */
int ss_semisort_pairs(void* pairs, uint64_t n, uint32_t key_bytes, int mode, int identity,
                      const ss_params* params, void* scratch, void* workspace, uint64_t workspace_bytes,
                      ss_telemetry* telemetry, void* stream);
uint64_t ss_semisort_pairs_workspace_bytes(uint64_t n, uint32_t key_bytes, const ss_params* params,
                                           int with_scratch);

/* TuningParams.for_input(n, ...) (params.py:64-86) with the tunables of
 * `tmpl`: subarray_len, sample_count and the heavy threshold re-derived
 * for n (a rank's received size is known only after the count exchange). */
int ss_params_for_input(uint64_t n, const ss_params* tmpl, ss_params* out);

/* ---- multi-GPU over NCCL (new, the reference has no
 * distributed path).  NCCL is loaded at run time (libnccl.so.2).  One
 * process per GPU; the caller sets the device before ss_nccl_comm_init.
 * ss_dist_semisort runs one rank's whole pipeline on `stream`:
 *   1. stable packed partition by dest = top log2(world) bits of mix64(key)
 *      into `scratch` (2 * capacity words),
 *   2. per-peer counts exchanged (grouped ncclSend / ncclRecv),
 *   3. ONE all-to-allv of packed records into `recv_block` (2 * capacity
 *      words), in source-rank order,
 *   4. ss_semisort_pairs of what arrived (params re-derived for that size
 *      from `params`' tunables), scratch reused.
 * Output: *out_n records, keys = recv_block words [0, *out_n), values =
 * words [*out_n, 2 * *out_n).  recv_block may alias the input columns
 * (the partition has consumed them before anything is received), which is
 * what lets strong scaling keep two buffers per rank.  If more than
 * `capacity` records would arrive the call fails with SS_ERR_RESOURCE
 * before the payload exchange (the input is intact, *out_n says how many).
 * The rank-ordered concatenation of every rank's output is a stable
 * global semisort. */
int ss_nccl_unique_id(unsigned char* out128);
int ss_nccl_comm_init(const unsigned char* id128, int world, int rank, void** out_comm);
int ss_nccl_comm_destroy(void* comm);
int ss_dist_semisort(void* comm, uint32_t world, uint32_t rank, const void* keys, const void* values,
                     uint64_t n_local, uint32_t key_bytes, int mode, int identity, const ss_params* params,
                     void* recv_block, void* scratch, uint64_t capacity, void* workspace,
                     uint64_t workspace_bytes, uint64_t* out_n, ss_telemetry* telemetry, void* stream);
uint64_t ss_dist_semisort_workspace_bytes(uint64_t capacity, uint32_t key_bytes, uint32_t world,
                                          const ss_params* params);

/* ---- device utilities (bench / validation) ----------------------------- */

/* Seeded synthetic keys with the reference generator families
 * (datagen.py): family 0 uniform[0, param), 1 floor(exponential(1/param)),
 * 2 zipf(s=param) ranks over [1, universe], 3 uniform 64-bit, 4 the config-5
 * 50/50 mix (uniform 64-bit / zipf(param) over [1, universe]).  hash_ranks
 * != 0 stores mix64(rank - 1) instead of the rank.  values_mode: 0 none,
 * 1 index (value = first_index + i), 2 uniform bits >> value_shift. */
int ss_generate(int family, double param, uint64_t universe, uint64_t n, uint64_t first_index,
                uint32_t key_bytes, uint64_t seed, int hash_ranks, void* out_keys,
                void* out_values, uint32_t value_bytes, int values_mode, uint32_t value_shift,
                void* stream);

/* O(n) semisort validity for inputs whose values are 0..n-1 (SURVEY.md
 * §8(c)): out_flags[0..3] = permutation, records intact, contiguous (run
 * count == distinct count, given), stable. */
int ss_validate_indexed(const void* keys_in, const void* keys_out, const void* values_out,
                        uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                        uint64_t distinct_keys, void* workspace, uint64_t workspace_bytes,
                        int32_t* out_flags, void* stream);
uint64_t ss_validate_workspace_bytes(uint64_t n);

/* Validation of one output shard of a generated input (ss_generate family,
 * param, universe, seed, hash_ranks) whose values are the global record
 * indices: out[0] records whose key differs from the generator's key for
 * their value, out[1] runs (key changes + 1), out[2] stability violations
 * inside runs, out[3] keys whose dest (top log2(parts) bits of mix64) is not
 * `rank`, out[4..6] sum of v, v^2, mix64(v) (mod 2^64) -- the ranks add the
 * fingerprints and compare with ss_index_fingerprint over [0, N). */
int ss_validate_shard(int family, double param, uint64_t universe, uint64_t seed, int hash_ranks,
                      const void* keys_out, const void* values_out, uint64_t m, uint32_t key_bytes,
                      uint32_t parts, uint32_t rank, void* workspace, uint64_t workspace_bytes,
                      uint64_t* out7, void* stream);
int ss_index_fingerprint(uint64_t lo, uint64_t hi, void* workspace, uint64_t workspace_bytes, uint64_t* out3,
                         void* stream);

/* Number of distinct keys (GPU hash set; the contiguity reference count). */
int ss_count_distinct(const void* keys, uint64_t n, uint32_t key_bytes, void* workspace,
                      uint64_t workspace_bytes, uint64_t* out_count, void* stream);
uint64_t ss_count_distinct_workspace_bytes(uint64_t n);

/* ---- graph applications -------------------------
 * CSR graphs: offsets u64[n_vertices + 1], targets u32[m] (device).
 *
 * ss_graph_transpose replaces graphs.transpose (graphs.py:77-105): every
 * edge (u, v) becomes (v, u); the (target, source) records are semisorted
 * with the identity hash and the CSR rebuilt from the runs, so each
 * transposed adjacency list is in ascending source order.  Outputs:
 * out_offsets u64[n_vertices + 1], out_targets u32[m].
 *
 * ss_csr_from_edges replaces graphs.from_edges (graphs.py:59-71): CSR by
 * source, adjacency lists in edge input order (the stable semisort by
 * source).  Inputs sources/targets u32[m] must be < n_vertices (the Python
 * layer validates, as the reference does, before calling).
 *
 * params: TuningParams bound to m (params.py:64-86).  Workspace:
 * ss_csr_workspace_bytes (the same for both). */
uint64_t ss_csr_workspace_bytes(uint64_t n_vertices, uint64_t m, const ss_params* params);
int ss_graph_transpose(uint64_t n_vertices, uint64_t m, const uint64_t* offsets, const uint32_t* targets,
                       uint64_t* out_offsets, uint32_t* out_targets, const ss_params* params,
                       void* workspace, uint64_t workspace_bytes, ss_telemetry* telemetry, void* stream);
int ss_csr_from_edges(uint64_t n_vertices, uint64_t m, const uint32_t* sources, const uint32_t* targets,
                      uint64_t* out_offsets, uint32_t* out_targets, const ss_params* params,
                      void* workspace, uint64_t workspace_bytes, ss_telemetry* telemetry, void* stream);

/* ---- record-dump rows (records.py:149-202) --------------------------------
 * A record dump ("SSR1" header, then n packed little-endian rows of
 * key_bytes + value_bytes, key first) is split into / packed from SoA device
 * columns.  rows, keys, values are device buffers, 4-byte aligned; key_bytes
 * 4 / 8 / 16, value_bytes a multiple of 4 (0 = no values).  The header itself
 * is parsed by the caller (write_records / read_records). */
int ss_records_unpack(const void* rows, uint64_t n, uint32_t key_bytes, uint32_t value_bytes, void* keys,
                      void* values, void* stream);
int ss_records_pack(const void* keys, const void* values, uint64_t n, uint32_t key_bytes, uint32_t value_bytes,
                    void* rows, void* stream);

/* ---- byte-view keys (adapters.py:200-275, hashing.py:56-106, ngrams.py) --
 * Keys are (offset, length) u64 rows (views, device) into a device byte
 * arena of arena_len bytes.  The Python layer (bytes_keys.py) turns them into
 * 128-bit identity keys (lo = content hash, hi = length for semisort= /
 * aggregation, = exact lexicographic content rank for semisort<) and runs
 * ss_semisort / ss_collect_reduce on those; these calls supply the pieces.
 * counter: one u64 of device scratch.
 *
 * ss_bytes_hash: out_hash[i] = mix64(poly(bytes) ^ mix64(len)), poly the
 *   wrapping polynomial with multiplier 0x100000001B3 (hashing.py:56-66 /
 *   BytePrefixHasher.hash_views :98-106).  SS_ERR_CONFIG when a view leaves
 *   the arena.
 * ss_bytes_chunk: out[i] = bytes [7c, 7c+7) of view i as 9-bit digits
 *   (byte + 1, 0 past the end), int64: lexicographic order chunk by chunk.
 * ss_bytes_equal: *out_mismatches = #{i : content(a[i]) != content(b[i])}. */
int ss_bytes_hash(const void* arena, uint64_t arena_len, const void* views, uint64_t n, void* out_hash,
                  void* counter, void* stream);
int ss_bytes_chunk(const void* arena, const void* views, uint64_t n, uint64_t chunk, void* out, void* stream);
int ss_bytes_equal(const void* arena, const void* views_a, const void* views_b, uint64_t n, void* counter,
                   uint64_t* out_mismatches, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SEMISORT_B200_H */

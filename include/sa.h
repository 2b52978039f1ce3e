/*
 * sa.h -- C ABI of libsa: batched exact matching of short reads against one
 * reference genome by binary search over its suffix array, on NVIDIA B200
 * (sm_100a).  The data-parallel hot path of arXiv 1303.3692 (PAPER.md,
 * cited "P:L<line>"), re-designed for B200.
 *
 * Conventions for every entry point
 * ---------------------------------
 *  - Return codes only; no exceptions cross the ABI.  On failure a one-line
 *    detail (e.g. the symbol and its position) is available from
 *    sa_last_error() on the calling thread.
 *  - "dev" pointers are CUDA device pointers on the index's device (e.g.
 *    torch.Tensor.data_ptr()); "host" pointers are CPU memory (page-locked
 *    memory is recommended where stated).  The caller owns every buffer it
 *    passes; the library never frees them and keeps no reference after the
 *    call's stream work completes.
 *  - `stream` is a cudaStream_t passed as void* (NULL = the legacy default
 *    stream).  Device-side calls are stream-ordered and asynchronous: results
 *    are valid after the stream is synchronised.
 *  - The index is immutable after sa_index_create; concurrent sa_match_batch /
 *    sa_locate calls on different streams are safe.  sa_match_batch_host
 *    serialises on an internal per-index lock.
 *
 * Alphabet and packing
 * --------------------
 *  Sigma = {a,c,g,t} ordered a<c<g<t (Sec. III), codes A=0 C=1 G=2
 *  T=3.  A query of m bases is packed 2 bits per base, MSB-first, into uint64
 *  words: base j of query q is at word q*stride_words + j/32, bits
 *  [63-2(j%32) .. 62-2(j%32)].  Bits past m are ignored.
 *  Dense layout (stride_words = 0, fixed-length reads only: q_len = NULL,
 *  fixed_len = m > 0): the reads are one continuous 2-bit stream, base j of
 *  query q is stream base q*m + j (word (q*m+j)/32, same bit order); the buffer
 *  holds ceil(Q*m/32) words.  25 bytes per 100-bp read instead of 32.
 *
 * What a match computes (Sec. IV; Alg. 1)
 * ----------------------------------------------------------------
 *  With SA the suffix array of S (Table I: all suffix starts in
 *  lexicographic order, a proper prefix sorting first, no sentinel) and
 *  t_i = S[i .. min(i+m, n)) the m-truncated suffix,
 *      lo = #{ i : t_i <  P },   hi = #{ i : t_i <= P }.
 *  [lo, hi) is the paper's [LB, RB] as a half-open interval: count = hi-lo,
 *  positions = SA[lo..hi) in SA order ("namely 9, 0, 5").  A query that
 *  does not occur ("(LB,RB) is NULL") yields lo == hi == its insertion
 *  point.  m = 0 yields [0, n).  Results are unique, hence bit-exact.
 */
#ifndef SA_H
#define SA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sa_index sa_index; /* opaque; owns all index memory on its device */

typedef enum {
    SA_OK = 0,
    SA_EINVAL = -1,   /* bad argument: NULL pointer with Q > 0, stride < ceil(m/32), k out of range, ... */
    SA_ESYMBOL = -2,  /* reference byte not in {A,C,G,T,a,c,g,t}; position in sa_last_error() */
    SA_ETOOLONG = -3, /* n > 2^32 - 1 (the suffix array holds uint32 positions) */
    SA_ENOMEM = -4,   /* device allocation failed */
    SA_ECUDA = -5,    /* any other CUDA error, including "no device" */
    SA_EEMPTY = -6    /* n == 0 */
} sa_status;

typedef struct {
    int32_t device;    /* CUDA device ordinal; -1 = the calling thread's current device */
    uint32_t kmer_k;   /* k of the k-mer bracket table, 1..16; 0 = auto (min(16, floor(log4 n) + 1)) */
    uint32_t flags;    /* 0, SA_INDEX_PLAIN or SA_INDEX_REC32, optionally | SA_INDEX_BUILD_DC3 */
    uint32_t reserved; /* must be 0 */
} sa_index_opts;

/* sa_index_opts.flags: the layout of the suffix array in HBM.  Default: 16-byte records
 * {SA[r], the 48 bases of suffix SA[r] that follow its first k bases} -- one 32-byte sector per
 * search step decides most comparisons (16 B x n).  SA_INDEX_REC32: 32-byte records caching 112
 * bases (32 B x n; reads up to k+112 bases never touch the text).  SA_INDEX_PLAIN: a plain uint32
 * SA (4 B x n); every step also reads the packed text. */
#define SA_INDEX_PLAIN 1u
#define SA_INDEX_REC32 2u
/* sa_index_opts.flags: build the suffix array with the paper's DC3 / skew algorithm (P:L105-150,
 * Sec. III; on the GPU: radix-sorted sample triples, recursion on the reduced string, merge-path
 * merge) instead of the default prefix doubling.  Same SA (it is unique); a different build cost. */
#define SA_INDEX_BUILD_DC3 4u
/* sa_index_opts.flags: k-mer buckets holding more than 32 suffixes (repeats) get a second-level
 * bracket table over the next 4 bases (257 SA ranks each, found through a hash of the k-mer), so
 * reads of >= k+4 bases in such a bucket start from a bracket ~256x smaller. */
#define SA_INDEX_SUBTABLE 8u
/* sa_index_opts.flags (with SA_INDEX_REC32, not with SA_INDEX_SUBTABLE): every k-mer bucket of >= 32
 * suffixes (repeats) also gets the records of the top levels of its binary search laid out two levels
 * per 128-byte line (a pivot and both its children), found through a hash of the k-mer: a read in a
 * large bucket makes the same probes, with about half as many DRAM lines.  Same results. */
#define SA_INDEX_BUCKET_TREE 16u

/* sa_match_batch flags. */
#define SA_MATCH_STATS 1u  /* also write per-query search statistics into the workspace (the
                              workspace must then hold >= 8*Q bytes): uint32 [0, Q) = steps |
                              (text windows fetched << 16); uint32 [Q, 2Q) = the query's algorithmic
                              bytes (SURVEY.md Sec. 8(d) "useful bytes": the packed read, the table
                              entries, 4 B per probed SA entry plus the 2-bit bases from the known
                              common prefix to the first difference, the 8-byte result) */
#define SA_MATCH_PRESORT 4u /* order the batch by the reads' first 12 bases (CUB radix sort in the
                               workspace) before the search, so that neighbouring threads walk the
                               same region of the suffix array; results still land at the reads'
                               original positions.  Requires Q < 2^32. */
#define SA_MATCH_ROWS_ORDERED 8u /* q_words / q_len are already in `order` order (sa_match_order's
                                    ordered_words / ordered_len): thread slot t reads row t and
                                    writes its interval to out_lohi at read order[t] */
#define SA_MATCH_COOPERATIVE 32u /* reads of more than 4 words (m > 128 bases) are searched by groups
                                    of 8 / 16 / 32 lanes, one word per lane, compared with
                                    __ballot_sync / __shfl_sync (the warp-cooperative compare of
                                    north_star); default: one thread per read.  Same results. */

#define SA_MATCH_SMEM_TREE 64u /* the shared-memory top tree: with an `order`
                                   from sa_match_order, each CTA of 256 reads stages the records of the
                                   first L levels of the binary search over its reads' SA range into
                                   shared memory (one TMA bulk copy per record) and every read walks them
                                   before its own probes.  L = SA_MATCH_TREE_LEVELS (1..12, 0 = 8); the
                                   key length of the order = SA_MATCH_TREE_KEY_BASES (0 = 12).  Record
                                   layouts, reads of <= 128 bases, no sub-tables.  Same results. */
/* sa_match_batch flag: reads of <= 128 bases in two passes -- every read whose k-mer bracket holds at
 * most 2^SA_MATCH_DEFER_LOG2 (default 8) suffixes first, the others (repeats) deferred to a second pass
 * that searches them with full warps -- so a warp's lanes are not held by one slow repeat read.  Same
 * results.  Workspace: sa_match_workspace_size with this flag (12 B per query more).  Not with
 * SA_MATCH_ROWS_ORDERED, SA_MATCH_STATS or SA_MATCH_SMEM_TREE. */
#define SA_MATCH_DEFER (1u << 17)
/* sa_match_batch flag: the large-batch load hints (a 64-byte L2 fetch for the read row and the bracket
 * table pair; automatic from 2^20 reads per call) at any batch size.  Same results. */
#define SA_MATCH_WIDE (1u << 24)
#define SA_MATCH_DEFER_LOG2(b) (((uint32_t)(b) & 15u) << 18)
#define SA_MATCH_TREE_LEVELS(l) (((uint32_t)(l) & 15u) << 8)
#define SA_MATCH_TREE_KEY_BASES(b) (((uint32_t)(b) & 31u) << 12)

/* Build the index of ref_ascii[0..n) (host memory, case-insensitive ACGT) on
 * the device: validate + pack to 2 bits/base, build the suffix array on the
 * GPU (radix sort + prefix doubling), build the k-mer bracket table.
 * The index build is P:L105-150 (Sec. III) re-designed; it is not
 * on the timed path.  opts may be NULL (defaults).  Synchronous.
 * Errors: SA_EINVAL (ref_ascii or out NULL, bad opts), SA_EEMPTY (n == 0),
 * SA_ETOOLONG, SA_ESYMBOL (first bad position reported), SA_ENOMEM, SA_ECUDA.
 * On error *out is set to NULL and nothing is leaked. */
sa_status sa_index_create(const char *ref_ascii, uint64_t n, const sa_index_opts *opts, sa_index **out);

/* Free all device memory of the index.  NULL-safe.  Synchronises its device. */
void sa_index_destroy(sa_index *idx);

/* Any output pointer may be NULL.  device_bytes = resident index bytes. */
sa_status sa_index_info(const sa_index *idx, uint64_t *n, uint32_t *kmer_k, uint64_t *device_bytes, int32_t *device);

/* Copy the suffix array (n uint32, host) -- for checking it against the oracle. */
sa_status sa_index_export_sa(const sa_index *idx, uint32_t *host_out);

/* Copy the k-mer bracket table T (4^k + 1 uint32, host):
 * T[x] = #{ i : trunc_k(S_i) < x } for x in [0, 4^k], x read as a k-mer. */
sa_status sa_index_export_table(const sa_index *idx, uint32_t *host_out);

/* Copy the packed text (ceil(n/32) words, host, same packing as queries). */
sa_status sa_index_export_text(const sa_index *idx, uint64_t *host_out);

/* Match Q packed queries (the hot path).
 *   q_words   dev, Q*stride_words uint64, layout above.
 *   q_len     dev, Q uint32 lengths, or NULL: every query has fixed_len bases.
 *   order     dev, Q uint32 permutation (from sa_match_order) or NULL: the order in which thread
 *             slots take reads.  It never changes a result, only which reads run side by side.
 *   out_lohi  dev, 2Q uint32: out_lohi[2q] = lo, out_lohi[2q+1] = hi
 *             (Alg. 1 lines 44-45, res[thd<<1] = LB, res[(thd<<1)+1] = RB, reading A8).
 *   workspace dev scratch of sa_match_workspace_size(..., flags, ...) bytes (may be NULL if
 *             that is 0).  With SA_MATCH_STATS its first 4*Q bytes receive the statistics.
 *   flags     0, or SA_MATCH_STATS / SA_MATCH_PRESORT / SA_MATCH_ROWS_ORDERED / SA_MATCH_COOPERATIVE /
 *             SA_MATCH_SMEM_TREE (| SA_MATCH_TREE_LEVELS(l) | SA_MATCH_TREE_KEY_BASES(b)).
 * Requirements: every length m <= 32*stride_words (longer lengths are clamped) and
 * m <= 65535; stride_words = 0 selects the dense layout (above).  Q == 0 is a no-op.
 * Errors: SA_EINVAL.  Asynchronous on `stream`. */
sa_status sa_match_workspace_size(const sa_index *idx, uint64_t Q, uint32_t stride_words, uint32_t flags,
                                  size_t *bytes);
sa_status sa_match_batch(const sa_index *idx, const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len,
                         uint32_t stride_words, uint64_t Q, const uint32_t *order, uint32_t *out_lohi,
                         void *workspace, size_t ws_bytes, uint32_t flags, void *stream);

/* The read ordering of SA_MATCH_PRESORT as its own step: order (dev, Q uint32) receives a
 * permutation of [0, Q) that sorts the reads by their first key_bases bases (1..16, 0 = 12;
 * stable; SA_MATCH_PRESORT uses 12).  Passing it as
 * sa_match_batch's `order` makes thread slot t search read order[t]; results are still written at
 * each read's own index.  The SURVEY.md Sec. 8(a) a5 row ("query ordering"), the B200 reading of the
 * paper's "coalesced binary search".  Requires Q < 2^32.
 * ordered_words (dev, Q*stride_words, nullable) / ordered_len (dev, Q, nullable): if given, also
 * receive the reads' rows / lengths in that order (row t = read order[t]), for SA_MATCH_ROWS_ORDERED. */
/* key_bases flag: order by bucket placement instead of the stable radix sort -- one count pass,
 * one scan over 4^key_bases counters, one placement pass (an atomic slot claim per bucket).  The
 * buckets come out in the same key order; reads with EQUAL keys are in no fixed order (not stable,
 * not reproducible between calls).  Results of sa_match_batch never depend on the order.  Meant for
 * batches whose permutation and counters fit the 126 MB L2 (e.g. Q <= 16 M at key_bases = 12);
 * key_bases <= 13.  Workspace: sa_match_order_workspace_size_ex(Q, key_bases | SA_ORDER_BUCKETS). */
#define SA_ORDER_BUCKETS 0x100u
sa_status sa_match_order_workspace_size(uint64_t Q, size_t *bytes);
/* The workspace of sa_match_order for these key_bases (with or without SA_ORDER_BUCKETS). */
sa_status sa_match_order_workspace_size_ex(uint64_t Q, uint32_t key_bases, size_t *bytes);
sa_status sa_match_order(const sa_index *idx, const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len,
                         uint32_t stride_words, uint64_t Q, uint32_t key_bases, uint32_t *order,
                         uint64_t *ordered_words, uint32_t *ordered_len, void *workspace, size_t ws_bytes,
                         void *stream);

/* The same match with HOST buffers (page-locked recommended): the queries are
 * streamed host->device in chunks of chunk_Q queries (0 = auto), each chunk ordered
 * (as sa_match_order, 12 bases) and matched, and the intervals streamed back, with
 * copies and kernels overlapped on two internal streams.  Synchronous: out_lohi
 * (host, 2Q uint32) is complete on return, and on an error return no copy into or
 * out of the caller's buffers is still in flight. */
sa_status sa_match_batch_host(sa_index *idx, const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len,
                              uint32_t stride_words, uint64_t Q, uint32_t *out_lohi, uint64_t chunk_Q);

/* Locate (positions SA[lo..hi) per query, in SA order):
 *   sa_locate_offsets: offsets (dev, Q+1 uint64) = exclusive prefix sum of hi-lo;
 *                      offsets[Q] = total number of positions.
 *   sa_locate:         positions (dev, offsets[Q] uint32): positions[offsets[q] + j] = SA[lo_q + j]. */
sa_status sa_locate_workspace_size(uint64_t Q, size_t *bytes);
sa_status sa_locate_offsets(const sa_index *idx, const uint32_t *out_lohi, uint64_t Q, uint64_t *offsets,
                            void *workspace, size_t ws_bytes, void *stream);
sa_status sa_locate(const sa_index *idx, const uint32_t *out_lohi, const uint64_t *offsets, uint64_t Q,
                    uint32_t *positions, void *stream);

/* Measurement tool (not on the path): random-access gather rate of the
 * device's memory.  Allocates buffer_bytes, then every thread issues `loads`
 * independent (dependent=0) or pointer-chased (dependent=1) loads -- or, with dependent=2,
 * independent stores; 10..13: independent loads with the PTX cache operator .nc / .cg / .cv /
 * .nc.L1::no_allocate (access_bytes 8 or 32); 20..22 (access_bytes 32): TMA bulk copies into
 * shared memory, cp.async.cg (LDGSTS), ld.global.nc.L2::64B -- of
 * access_bytes (4, 8, 16 or 32) at hashed, access_bytes-aligned offsets.
 * *ms = device time of one launch of n_threads threads (CUDA events). */
sa_status sa_tool_random_gather(int32_t device, uint64_t buffer_bytes, uint32_t access_bytes, uint64_t n_threads,
                                uint32_t loads, int32_t dependent, float *ms);

/* Partitioned index (not in the paper): for references whose index exceeds one
 * GPU.  Part `part` of `nparts` (>= 2) holds the suffixes whose route key -- their first route_bases
 * (1..12, < k) bases, a suffix shorter than that padded with 'a' and placed like the k-mer table does --
 * lies in [part_keys[part], part_keys[part+1]): a contiguous range of SA ranks [rank_lo, rank_hi).
 * Boundaries balance the ranks over the parts.  sa_index_create_part builds ONLY that slice of the suffix
 * array (MSD refinement of the part's suffixes on the packed text), of the k-mer table (entries
 * [part_keys[part], part_keys[part+1]] x 4^(k-route_bases), clamped to the slice's ranks) and of the
 * records, plus the whole packed text and the route-level table (4^route_bases + 1 uint32); opts.flags may
 * only choose the layout.  Every answer of a part is clamped to its ranks: [clamp(lo), clamp(hi)] with
 * clamp(v) = min(max(v, rank_lo), rank_hi) -- the global interval for a read routed to the part (route
 * key inside its range), and for a read shorter than route_bases (sent to every part) a term of
 * lo = sum over parts of (clamp(lo) - rank_lo) (sa_part_collect).  sa_index_export_sa / _table copy the
 * slice (rank_hi - rank_lo SA entries; the table entries of the part's route keys).
 *   sa_index_part_info: part_keys / part_ranks (nullable) receive nparts+1 route-key / rank boundaries.
 *   sa_match_route:     orders a batch by route key, reads shorter than route_bases last (order, as
 *                       sa_match_order), gathers the rows in that order (ordered_words/_len) and writes
 *                       dest_offsets (dev, nparts+1 uint64): ordered rows [dest_offsets[g], dest_offsets[g+1])
 *                       are routed to part g; rows [dest_offsets[nparts], Q) are the short reads.
 *                       Workspace: sa_match_order_workspace_size.
 *   sa_part_pack:       the send buffer (dev, send_rows = dest_offsets[nparts] + nparts * n_short rows):
 *                       block g = the rows routed to part g followed by all short rows.
 *   sa_part_collect:    back_lohi (dev) = the parts' answers to the blocks, in the same layout (after the
 *                       all-to-all back); writes every read's global interval to out_lohi at read order[t].
 *   sa_scatter_results: out_lohi[order[t]] = in_lohi[t] (results back in the batch's own order).
 * The exchange itself (all-to-all of the rows and of the intervals) is the caller's collective
 * (paper_1303_3692_b200/shard.py: torch.distributed all_to_all_single over NCCL). */
sa_status sa_index_create_part(const char *ref_ascii, uint64_t n, const sa_index_opts *opts, uint32_t part,
                               uint32_t nparts, uint32_t route_bases, sa_index **out);
sa_status sa_index_part_info(const sa_index *idx, uint32_t *part, uint32_t *nparts, uint32_t *route_bases,
                             uint64_t *rank_lo, uint64_t *rank_hi, uint32_t *part_keys, uint64_t *part_ranks);
sa_status sa_match_route(const sa_index *idx, const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len,
                         uint32_t stride_words, uint64_t Q, uint32_t *order, uint64_t *ordered_words,
                         uint32_t *ordered_len, uint64_t *dest_offsets, void *workspace, size_t ws_bytes, void *stream);
sa_status sa_part_pack(const sa_index *idx, const uint64_t *ordered_words, const uint32_t *ordered_len,
                       uint32_t stride_words, const uint64_t *dest_offsets, uint64_t Q, uint64_t send_rows,
                       uint64_t *send_words, uint32_t *send_len, void *stream);
sa_status sa_part_collect(const sa_index *idx, const uint32_t *back_lohi, const uint64_t *dest_offsets, uint64_t Q,
                          const uint32_t *order, uint32_t *out_lohi, void *stream);
sa_status sa_scatter_results(const uint32_t *order, const uint32_t *in_lohi, uint64_t Q, uint32_t *out_lohi,
                             void *stream);

/* Flattened suffix tree ("flatten tree consisting of an
 * array of edges", Table V STK): built from an index's suffix array (LCP on the GPU, the
 * lcp-interval tree on the host), 32-byte nodes {lb, rb, string depth, SA[lb], child[a,c,g,t]} in
 * HBM.  The tree BORROWS the index (destroy the tree first).  Requires n < 2^31.
 * sa_tree_match walks it from the root, one node and one edge-label compare per branching level,
 * and writes the same half-open SA intervals as sa_match_batch (out_lohi, 2Q uint32), misses at their
 * insertion point.  Strided reads only (stride_words >= 1); order as for sa_match_batch (nullable).
 * Asynchronous on `stream`. */
typedef struct sa_tree sa_tree;
sa_status sa_tree_create(const sa_index *idx, sa_tree **out);
void sa_tree_destroy(sa_tree *tree);
sa_status sa_tree_info(const sa_tree *tree, uint64_t *nodes, uint64_t *device_bytes);
sa_status sa_tree_match(const sa_tree *tree, const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len,
                        uint32_t stride_words, uint64_t Q, const uint32_t *order, uint32_t *out_lohi, void *stream);

/* DC3 trace for checking the build against the paper's worked example (Tables II-III,
 * P:L112-128): runs DC3 on ref_ascii[0..n) on the current device and returns, on the host,
 * sample_rank[i] = the 1-based rank of S_i among the sample suffixes (i mod 3 != 0; 0 for i mod 3 = 0)
 * and nonsample[0..ceil(n/3)) = the B_0 positions in suffix order (DC3 step 2).  Either may be NULL. */
sa_status sa_dc3_trace(const char *ref_ascii, uint64_t n, uint32_t *sample_rank, uint32_t *nonsample);

/* Thread-local detail of the last failure on this thread ("" if none). */
const char *sa_last_error(void);

/* Library version (major*10000 + minor*100 + patch). */
int32_t sa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SA_H */

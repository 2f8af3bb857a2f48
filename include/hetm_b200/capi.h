/*
 * hetm_b200 — C-ABI into the B200 (sm_100a) device side of Speculative HeTM.
 *
 * This header is the ONLY door from host code into CUDA.  Every entry point
 * takes plain pointers and sizes (no C++ / torch types) and returns an `int`
 * status (HETM_OK == 0).  There is no CPU fallback: without a usable CUDA
 * device every call that needs one returns HETM_ERR_NO_DEVICE.
 *
 * Reference interfaces each group replaces (paths relative to the reference
 * tree, /root/reference):
 *
 *   stmr module           SPEC.md:29-70   Stmr/create/rawWrite/rawRead/copyChunks
 *   guest-stm-batch       SPEC.md:196-229 BatchSpec/executeBatch/clearRound/bitmapStats
 *   bitmaps               proj/include/hetm/bitmap.hpp:15-158 (BitmapSnapshot word layout)
 *   interconnect          proj/include/hetm/bus.hpp:43-91, SPEC.md:270-307 (streamChunk,
 *                         copyDeviceToHost, copyDeviceToDevice, transferLog)
 *   engine                SPEC.md:319-389 (TsArray, validateChunk, earlyValidate,
 *                         mergeCommit, mergeAbortDevice, mergeAbortHost)
 *   write log wire format proj/include/hetm/write_log.hpp:16-25 (24-byte <addr,value,ts>)
 *   errors                proj/include/hetm/types.hpp:35-49 (one status per HetmError subclass)
 *
 * Threading: all hetm_dev_* calls come from one
 * controller thread, except hetm_dev_stream_chunk which is safe to call from
 * any host worker thread (chunks are serialised per device in call order,
 * which preserves the per-source-thread FIFO of SPEC.md:300).
 */
#ifndef HETM_B200_CAPI_H
#define HETM_B200_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HETM_B200_ABI_VERSION 3  /* 3: hetm_batch_stats.retried */

/* ---------------------------------------------------------------- status --
 * One code per hetm::HetmError subclass (types.hpp:38-48) plus device codes. */
enum hetm_status {
    HETM_OK = 0,
    HETM_ERR_INVALID_SIZE = 1,          /* InvalidSizeError          types.hpp:38 */
    HETM_ERR_OUT_OF_BOUNDS = 2,         /* OutOfBoundsError          types.hpp:39 */
    HETM_ERR_ROUND_CLOSED = 3,          /* RoundClosedError          types.hpp:40 */
    HETM_ERR_KERNEL_NOT_REGISTERED = 4, /* KernelNotRegisteredError  types.hpp:41 */
    HETM_ERR_LIVELOCK = 5,              /* LivelockError             types.hpp:42 */
    HETM_ERR_NO_IMPLEMENTATION = 6,     /* NoImplementationError     types.hpp:43 */
    HETM_ERR_BAD_AFFINITY = 7,          /* BadAffinityError          types.hpp:44 */
    HETM_ERR_INCOMPLETE_TRACE = 8,      /* IncompleteTraceError      types.hpp:45 */
    HETM_ERR_NONDETERMINISTIC = 9,      /* NondeterministicInputError types.hpp:46 */
    HETM_ERR_CONFIG = 10,               /* ConfigError               types.hpp:47 */
    HETM_ERR_IO = 11,                   /* IoError                   types.hpp:48 */
    HETM_ERR_INVALID_ARG = 100,         /* null handle / bad enum value */
    HETM_ERR_CUDA = 101,                /* a CUDA runtime call failed */
    HETM_ERR_NO_DEVICE = 102,           /* no CUDA device: there is no CPU fallback */
    HETM_ERR_NONMONOTONE_TS = 103,      /* log ts not above the previous round's max (TS array not reset) */
    HETM_ERR_STATE = 104                /* call not valid in the current round phase */
};

/* Buffers addressable by raw region ops — hetm::Replica (types.hpp:21). */
enum hetm_replica {
    HETM_REPLICA_HOST = 0,          /* host-owned; not addressable through this ABI */
    HETM_REPLICA_DEV = 1,
    HETM_REPLICA_DEV_SHADOW = 2,
    HETM_REPLICA_HOST_SNAPSHOT = 3  /* host-owned; not addressable through this ABI */
};

/* Which device bitmap (bitmap.hpp:94-158). */
enum hetm_bitmap_kind { HETM_BMP_RS = 0, HETM_BMP_WS = 1, HETM_BMP_CHUNK = 2 };

/* validateChunk applyMode. */
enum hetm_validate_mode { HETM_APPLY = 0, HETM_VALIDATE_ONLY = 1 };
/* hetm_dev_validate_dptr mode flag: the entries are also copied (D2D) into the
 * round's log arena, so the incremental shadow refresh and the optimized
 * rollback cover them (without it the next shadow refresh is a full copy). */
#define HETM_RETAIN 0x100

/* Built-in transactional kernels (kernels are registered by id). */
enum hetm_kernel_id {
    HETM_KERNEL_BANK = 1, /* hetm_bank_tx: read 4 accounts, move amount acct0 -> acct1 */
    HETM_KERNEL_RW = 2,   /* hetm_rw_tx: generic <=4 reads / <=2 read-modify-writes   */
    HETM_KERNEL_CACHE = 3 /* hetm_cache_tx: MemcachedGPU-style GET/SET (below)         */
};

/* hetm_dev_clear_round flags. */
#define HETM_CLEAR_RESET_TS 1u /* also zero the TS array (SPEC.md:421 literal reset) */
#define HETM_CLEAR_ASYNC 2u    /* enqueue the reset (bitmaps, round flags, counter roll) behind
                                  the round's work without a host sync (pipelined rounds); the
                                  device state after it equals the synchronous clear's */

/* hetm_dev_config.flags */
#define HETM_CFG_NO_SHADOW 1u /* do not allocate devShadow (validation-only sweeps) */
#define HETM_CFG_L2_FETCH_32 2u /* cudaLimitMaxL2FetchGranularity = 32 B (random 8-B word access) */
#define HETM_CFG_DETERMINISTIC 8u /* deterministic single-worker batches: transactions
                                     commit one at a time in input order, ticket i = first + i
                                     (reproducible runs; orders of magnitude slower) */
#define HETM_CFG_MERGE_DELTA 4u /* mergeCommit ships the device write set as {word, value} records
                                   (16 B per written word) when that is smaller than the dirty
                                   chunks; recorded as HETM_TAG_MERGE_DELTA.  Off: the SPEC.md:
                                   363-371 chunk copy (16 KiB per dirty chunk) */

/* ------------------------------------------------------------ wire types -- */

/* One committed host write: layout-identical to hetm::WriteLogEntry
 * (write_log.hpp:16-22), 24 bytes on the wire (write_log.hpp:25). `addr` is a
 * GLOBAL word index; ts >= 1. */
typedef struct hetm_log_entry {
    uint64_t addr;
    uint64_t value;
    uint64_t ts;
} hetm_log_entry;

/* Bank transfer input record (24 B): read acct[0..3], then
 * acct[0] -= amount, acct[1] += amount (uint64 wrap-around).  Accounts are
 * GLOBAL word indices < 2^32. */
typedef struct hetm_bank_tx {
    uint32_t acct[4];
    uint64_t amount;
} hetm_bank_tx;

/* Generic read/modify transaction (72 B): reads r_addr[0..nr), then for each
 * j < nw: stmr[w_addr[j]] = stmr[w_addr[j]] + add[j] + sum(reads).  Writes
 * imply reads (no blind writes). */
typedef struct hetm_rw_tx {
    uint32_t nr;
    uint32_t nw;
    uint64_t r_addr[4];
    uint64_t w_addr[2];
    uint64_t add[2];
} hetm_rw_tx;

/* MemcachedGPU-style set-associative cache in the STMR (BASELINE configs[3];
 * PAPER.md:480-508).  A set holds HETM_CACHE_WAYS ways of
 * HETM_CACHE_WAY_WORDS words {key0, key1, value0..3, lru, flags}; set s
 * occupies words [base + 64 s, base + 64 s + 64).  Keys route by their last
 * bit: part p = key[0] & 1 owns sets [p n/2, (p+1) n/2), and
 * set = p n/2 + (hetm_cache_hash(key) mod n/2), so the CPU (part 0) and GPU
 * (part 1) halves of the cache never share a set or a 1 KiB RS granule.
 *   GET: hit -> value, the way's lru := ticket+1 (LRU touch); miss -> nothing.
 *   SET: hit -> value and lru rewritten; miss -> the first invalid way, else
 *        the least-recently-used way (lowest index on ties) takes key, value,
 *        lru := ticket+1, flags := 1.
 * Every written word is read first (no blind writes). */
#define HETM_CACHE_WAYS 8
#define HETM_CACHE_WAY_WORDS 8
#define HETM_CACHE_SET_WORDS 64
enum hetm_cache_op { HETM_CACHE_GET = 0, HETM_CACHE_SET = 1 };
typedef struct hetm_cache_tx {
    uint32_t op; /* hetm_cache_op */
    uint32_t reserved;
    uint64_t key[2];
    uint64_t value[4]; /* SET only */
} hetm_cache_tx;
enum hetm_cache_status {
    HETM_CACHE_MISS = 0,     /* GET: key absent */
    HETM_CACHE_HIT = 1,      /* GET: value returned */
    HETM_CACHE_UPDATED = 2,  /* SET: key present, value replaced */
    HETM_CACHE_INSERTED = 3, /* SET: stored in an invalid way */
    HETM_CACHE_EVICTED = 4   /* SET: stored over the LRU way */
};
typedef struct hetm_cache_result {
    uint64_t value[4]; /* GET hit: the value; SET: the value stored */
    uint32_t status;   /* hetm_cache_status */
    uint32_t way;      /* way used (HETM_CACHE_WAYS on a miss) */
} hetm_cache_result;

typedef struct hetm_dev_config {
    uint64_t size_words;    /* STMR words held by this device (its shard)           */
    uint64_t shard_base;    /* first global word index held (0 on a single GPU)      */
    uint64_t rs_gran_bytes; /* RS/WS granularity: pow2 multiple of 8 (default 1024)  */
    uint64_t chunk_bytes;   /* ChunkMap granularity: pow2 multiple of 8 (16384)      */
    uint64_t log_capacity;  /* initial round-log arena (entries); 0 = auto; grows    */
    uint32_t max_attempts;  /* livelock budget per transaction; 0 = default (1<<24)  */
    int32_t device;         /* CUDA device ordinal                                   */
    uint32_t flags;         /* HETM_CFG_*                                            */
    uint32_t reserved;
} hetm_dev_config;

typedef struct hetm_dev_info {
    uint64_t size_words, shard_base, rs_gran_bytes, chunk_bytes, cell_bytes;
    uint64_t rs_bits, rs_words, chunk_bits, chunk_words;
    uint64_t log_capacity;
    uint64_t device_bytes; /* HBM allocated by this handle */
    int32_t device, sm_count;
    uint64_t l2_bytes;
    uint64_t ticket_next;  /* next commit ticket to be handed out */
} hetm_dev_info;

typedef struct hetm_batch_stats {
    uint64_t n_tx;
    uint64_t committed;
    uint64_t aborts;       /* intra-device aborted attempts (retried) */
    uint64_t livelocked;   /* transactions that exhausted the budget */
    uint64_t ticket_first; /* tickets of this batch lie in [ticket_first, ticket_end) */
    uint64_t ticket_end;
    double kernel_ms;      /* device time of the batch kernel (CUDA events) */
    uint64_t retried;      /* transactions that committed only after >= 2 aborted attempts */
} hetm_batch_stats;

typedef struct hetm_merge_stats {
    uint64_t dirty_chunks;
    uint64_t transfers;      /* coalesced copy descriptors issued */
    uint64_t bytes_d2h;
    uint64_t bytes_h2d;
    uint64_t bytes_d2d;
    double ms;               /* host wall time of the call */
} hetm_merge_stats;

/* Interconnect transferLog record (bus.hpp:27-32, BusDir bus.hpp:16). */
enum hetm_bus_dir { HETM_H2D = 0, HETM_D2H = 1, HETM_D2D = 2 };
typedef struct hetm_transfer_record {
    int32_t dir;
    int32_t tag;   /* HETM_TAG_* */
    uint64_t bytes;
} hetm_transfer_record;
enum hetm_transfer_tag {
    HETM_TAG_LOG = 0, HETM_TAG_MERGE = 1, HETM_TAG_SHADOW = 2, HETM_TAG_ROLLBACK = 3,
    HETM_TAG_INPUT = 4, HETM_TAG_OUTPUT = 5, HETM_TAG_RAW = 6, HETM_TAG_MERGE_DELTA = 7
};

typedef struct hetm_dev hetm_dev;

/* ------------------------------------------------------------ lifecycle -- */
const char* hetm_strerror(int status);
int hetm_abi_version(void);
int hetm_device_count(int* n);
void hetm_dev_config_default(hetm_dev_config* cfg);
/* Stmr create: all device replicas zero-filled. */
int hetm_dev_open(const hetm_dev_config* cfg, hetm_dev** out);
int hetm_dev_close(hetm_dev* dev);
int hetm_dev_info_get(hetm_dev* dev, hetm_dev_info* out);
/* Last CUDA error string seen by this handle (diagnostics). */
const char* hetm_dev_last_error(hetm_dev* dev);

/* ----------------------------------------------- raw region ops (stmr) --
 * SPEC.md:53-61; caller-enforced quiescence.  Addresses are
 * GLOBAL word indices; out-of-shard -> HETM_ERR_OUT_OF_BOUNDS. */
int hetm_dev_raw_write(hetm_dev* dev, int replica, uint64_t addr, uint64_t value);
int hetm_dev_raw_read(hetm_dev* dev, int replica, uint64_t addr, uint64_t* value);
int hetm_dev_upload(hetm_dev* dev, int replica, uint64_t addr, const uint64_t* src, uint64_t n);
int hetm_dev_download(hetm_dev* dev, int replica, uint64_t addr, uint64_t* dst, uint64_t n);

/* --------------------------------------------- guest-stm-batch (device) -- */
/* registerTxType's device half: unknown id -> NO_IMPLEMENTATION. */
int hetm_dev_register_kernel(hetm_dev* dev, int kernel_id);
/* executeBatch.  `inputs` is HOST memory (n_tx records of
 * rec_bytes, which must equal the kernel's record size).  Every transaction
 * eventually commits or the call fails with HETM_ERR_LIVELOCK.  tickets_out
 * (nullable, n_tx entries) receives each transaction's commit ticket: replaying
 * the batch in ascending ticket order reproduces devReplica.
 * UINT64_MAX marks a transaction that exhausted the livelock budget. */
int hetm_dev_execute_batch(hetm_dev* dev, int kernel_id, const void* inputs, uint64_t rec_bytes,
                           uint64_t n_tx, uint64_t* tickets_out, hetm_batch_stats* stats);
/* executeBatch with per-transaction results (HETM_KERNEL_CACHE: one
 * hetm_cache_result per transaction; res_bytes must equal its size). */
int hetm_dev_execute_batch_ex(hetm_dev* dev, int kernel_id, const void* inputs, uint64_t rec_bytes,
                              uint64_t n_tx, uint64_t* tickets_out, void* results_out, uint64_t res_bytes,
                              hetm_batch_stats* stats);
/* Cache region of HETM_KERNEL_CACHE: n_sets (power of two >= 2) sets from
 * GLOBAL word base_word.  Default: the largest power-of-two set count that
 * fits the shard, from its first word. */
int hetm_dev_set_cache_geometry(hetm_dev* dev, uint64_t base_word, uint64_t n_sets);
/* The key hash and set routing used by the device (for host-side tooling). */
uint64_t hetm_cache_hash(uint64_t key0, uint64_t key1);
uint64_t hetm_cache_set_of(uint64_t key0, uint64_t key1, uint64_t n_sets);
/* bitmapStats. */
int hetm_dev_bitmap_stats(hetm_dev* dev, uint64_t* rs_bits, uint64_t* ws_bits, uint64_t* chunks);
int hetm_dev_bitmap_words(hetm_dev* dev, int which, uint64_t* n_words);
/* BitmapSnapshot::words (bitmap.hpp:15-23): bit b <-> words[b>>6] >> (b&63). */
int hetm_dev_snapshot_bitmap(hetm_dev* dev, int which, uint64_t* out_words, uint64_t n_words);
/* OR `words` into a device bitmap (seeding RS for validation sweeps, tests). */
int hetm_dev_or_bitmap(hetm_dev* dev, int which, const uint64_t* words, uint64_t n_words);

/* ------------------------------------------- interconnect + validation -- */
/* Log intake (bus.hpp:72-76): open at round start; merge closes it. */
int hetm_dev_open_intake(hetm_dev* dev);
int hetm_dev_close_intake(hetm_dev* dev);
/* streamChunk + validateChunk.  `entries` is a
 * HOST buffer borrowed until the chunk is delivered (hetm_dev_stream_chunk_ex
 * handle; at the latest, the next hetm_dev_round_verdict / hetm_dev_sync;
 * pinned memory gives an asynchronous DMA).  The chunk is appended to the
 * round's device log arena.  APPLY: validate + TS-guarded apply, ordered after
 * the device's in-flight batch.  VALIDATE_ONLY: early validation (SPEC.md:
 * 354-362), runs concurrently with execution; its apply is deferred to
 * hetm_dev_apply_log.  After close_intake -> HETM_ERR_ROUND_CLOSED. */
int hetm_dev_stream_chunk(hetm_dev* dev, const hetm_log_entry* entries, uint64_t n,
                          int src_thread, uint64_t seq, int mode);
/* Delivery handle of one streamed chunk (bus.hpp:51-56 `Delivery`, returned by
 * Bus::streamChunk, bus.hpp:80; "completion observable via the
 * handle").  `handle` orders every chunk of the device; the chunk is delivered
 * when its H2D copy into the device log arena has completed, and from then on
 * its host buffer belongs to the caller again (a producer can recycle a small
 * pinned staging ring instead of pinning the whole round's log). */
typedef struct hetm_delivery {
    uint64_t seq;        /* LogChunk::seq (bus.hpp:47) */
    uint64_t n_entries;  /* Delivery::nEntries (bus.hpp:53) */
    uint64_t bytes;      /* wire bytes, 24 per entry (write_log.hpp:25) */
    uint64_t handle;     /* completion id: hetm_dev_delivery_done / _wait */
    int32_t src_thread;  /* LogChunk::sourceThread (bus.hpp:46) */
    int32_t mode;        /* HETM_APPLY / HETM_VALIDATE_ONLY */
} hetm_delivery;
/* streamChunk with its delivery handle (out may be NULL).  `entries` is
 * borrowed until the handle reports delivered.  Chunks of one src_thread are
 * copied, validated and applied in call order (per-source FIFO). */
int hetm_dev_stream_chunk_ex(hetm_dev* dev, const hetm_log_entry* entries, uint64_t n,
                             int src_thread, uint64_t seq, int mode, hetm_delivery* out);
/* Non-blocking: *done = 1 once the chunk's H2D copy has completed. */
int hetm_dev_delivery_done(hetm_dev* dev, uint64_t handle, int* done);
/* Blocks until the chunk's H2D copy has completed. */
int hetm_dev_delivery_wait(hetm_dev* dev, uint64_t handle);
/* Per-source accounting of the round's streamed chunks. */
typedef struct hetm_source_stats {
    uint64_t chunks, entries;
    uint64_t last_seq, last_handle;
} hetm_source_stats;
int hetm_dev_source_stats(hetm_dev* dev, int src_thread, hetm_source_stats* out);
/* Early-validation period (default k = 8): VALIDATE_ONLY chunks
 * are validated in one launch every k chunks; an APPLY chunk, apply_log and the
 * verdict validate the pending ones first.  k = 1 validates every chunk. */
int hetm_dev_set_validation_period(hetm_dev* dev, uint32_t k);
/* Apply every arena entry streamed VALIDATE_ONLY this round (final validation
 * phase re-validates them). */
int hetm_dev_apply_log(hetm_dev* dev);
/* Non-blocking: conflict flag as of the last completed validation work. */
int hetm_dev_poll_conflict(hetm_dev* dev, int* conflict);
/* Blocking: waits for all streamed chunks; returns the round conflictFlag
 * (monotone within a round). */
int hetm_dev_round_verdict(hetm_dev* dev, int* conflict);
/* Waits for all work on all device streams. */
int hetm_dev_sync(hetm_dev* dev);

/* ---------------------------------------------------------------- merge --
 * host_replica: HOST array of size_words words (this shard's slice), ideally
 * pinned (hetm_host_alloc / hetm_host_register). */
/* mergeCommit: devShadow := devReplica; dirty chunks are
 * copied shadow -> host_replica in coalesced transfers.  Asynchronous w.r.t.
 * the next round's execution: call hetm_dev_merge_wait before touching
 * host_replica. */
int hetm_dev_merge_commit(hetm_dev* dev, uint64_t* host_replica, hetm_merge_stats* st);
/* mergeAbortDevice.  optimized=0: host_replica copied over
 * the device's dirty chunks.  optimized=1: round-start shadow + the round's
 * host log in ts order, swapped in.  Both end with devReplica == host_replica. */
int hetm_dev_merge_abort_device(hetm_dev* dev, int optimized, const uint64_t* host_replica,
                                hetm_merge_stats* st);
/* mergeAbortHost: host_replica := host_snapshot, then the
 * device's dirty chunks are copied device -> host.  The round's log must not
 * have been applied (validate-only rounds). */
int hetm_dev_merge_abort_host(hetm_dev* dev, uint64_t* host_replica, const uint64_t* host_snapshot,
                              hetm_merge_stats* st);
int hetm_dev_merge_wait(hetm_dev* dev);
/* clearRound: RS/WS/ChunkMap zeroed, arena emptied,
 * conflict flag cleared, intake reopened.  The TS array is NOT reset unless
 * HETM_CLEAR_RESET_TS is given: with a monotone GlobalClock
 * stale TS values are always older than the next round's ts, so the apply
 * outcome is identical; a log ts not above the previous round's maximum is
 * reported as HETM_ERR_NONMONOTONE_TS by the next verdict. */
int hetm_dev_clear_round(hetm_dev* dev, uint32_t flags);

/* ------------------------------------------------ interconnect accounting --
 * transferLog (bus.hpp:84-91). */
int hetm_dev_transfer_count(hetm_dev* dev, uint64_t* n);
int hetm_dev_transfer_log(hetm_dev* dev, hetm_transfer_record* out, uint64_t max, uint64_t* n);
int hetm_dev_clear_transfer_log(hetm_dev* dev);

/* ------------------------------------------------ device-resident entries --
 * The same kernels on DEVICE pointers, enqueued on `stream` (a cudaStream_t;
 * NULL = the handle's execution stream) without synchronising.  Used by the
 * benchmark (inputs resident in HBM) and by the multi-GPU shard router.
 * Batches of one handle must not run concurrently (executeBatch is
 * externally single-caller): a caller passing its own streams
 * orders successive batches itself — the bank kernel locks words through the
 * handle's stripe table, the rw and cache kernels through the cells. */
int hetm_dev_execute_batch_dptr(hetm_dev* dev, int kernel_id, const void* d_inputs, uint64_t n_tx,
                                uint64_t* d_tickets, void* stream);
/* ... with a device results array (HETM_KERNEL_CACHE). */
int hetm_dev_execute_batch_dptr_ex(hetm_dev* dev, int kernel_id, const void* d_inputs, uint64_t n_tx,
                                   uint64_t* d_tickets, void* d_results, void* stream);
int hetm_dev_validate_dptr(hetm_dev* dev, const hetm_log_entry* d_entries, uint64_t n, int mode,
                           void* stream);
/* Read back (synchronously) the device conflict / stats counters. */
int hetm_dev_read_counters(hetm_dev* dev, int* conflict, hetm_batch_stats* last_batch);
/* Shard router for address-range sharding (G GPUs, shard s owns global words
 * [s*shard_words, (s+1)*shard_words)).  Stable-partitions d_in into d_out by
 * owner shard; d_counts[s] receives the bucket sizes (device array of
 * n_shards uint64).  d_out must hold n entries. */
int hetm_dev_route_log_dptr(hetm_dev* dev, const hetm_log_entry* d_in, uint64_t n, uint32_t n_shards,
                            uint64_t shard_words, hetm_log_entry* d_out, uint64_t* d_counts,
                            void* stream);
/* Fused route + delivery over NVLink (no NCCL on the data path).
 * Every shard exposes two receive arenas (round parity) of n_shards regions of
 * `cap` entries and two bucket-count blocks of 64 (hetm_dev_recv_arena returns
 * their bases); the sender's router writes its bucket for owner s straight
 * into s's arena[parity] region [my_shard] and the bucket size into s's
 * counts[parity][my_shard] — peer pointers (hetm_enable_peer_access, one
 * process) or IPC-opened pointers (hetm_ipc_*, one process per GPU).  Every
 * sender writes every owner's count (0 included) every round.  After all
 * senders of a round have completed (stream sync + a barrier among ranks),
 * hetm_dev_apply_received validates/applies arena[parity] (mode as in
 * stream_chunk) in ONE launch that reads the counts on the device — no host
 * round trip, so the ranks can order it behind a device-side barrier (e.g. a
 * 1-element NCCL all-reduce on the same stream).  n_out (nullable) costs a
 * sync: entries applied.  Alternating the parity per round lets a sender
 * route round r+1 while an owner still applies round r. */
int hetm_dev_recv_arena(hetm_dev* dev, uint32_t n_shards, uint64_t cap, void** d_entries, void** d_counts);
int hetm_dev_route_to_peers_dptr(hetm_dev* dev, const hetm_log_entry* d_in, uint64_t n, uint32_t n_shards,
                                 uint64_t shard_words, uint32_t my_shard, uint64_t cap, uint32_t parity,
                                 void* const* peer_entries, void* const* peer_counts, void* stream);
int hetm_dev_apply_received(hetm_dev* dev, uint32_t parity, int mode, uint64_t* n_out, void* stream);
/* Bitmap OR-reduce over NVLink (NCCL has no bitwise OR):
 * hetm_dev_bitmap_dptr exposes a bitmap (HETM_BMP_RS / WS / CHUNK) for CUDA IPC
 * export; hetm_dev_bitmap_or_peers ORs words [word_lo, word_hi) (word_hi == 0:
 * all) of n_peers peer bitmaps of the same geometry — device pointers usable
 * from this GPU (IPC-opened, or other handles in the process) — into this
 * handle's bitmap, ordered after its batches, on `stream` (NULL: the handle's
 * validation stream).  Every rank ORing all words is the all-reduce; each
 * rank ORing only its own slice [lo, hi) is the reduce-scatter.  The caller
 * orders the peers' bitmaps before the call (a barrier). */
int hetm_dev_bitmap_dptr(hetm_dev* dev, int which, void** dptr, uint64_t* n_words);
int hetm_dev_bitmap_or_peers(hetm_dev* dev, int which, const void* const* peer_words, uint32_t n_peers,
                             uint64_t word_lo, uint64_t word_hi, void* stream);
/* CUDA IPC of device buffers between the ranks of one node (64-byte handles). */
int hetm_ipc_get_handle(void* dptr, void* handle64);
int hetm_ipc_open_handle(const void* handle64, void** dptr);
int hetm_ipc_close(void* dptr);
int hetm_enable_peer_access(int device, int peer_device);
/* Streams owned by the handle: 0 = execution, 1 = log copy, 2 = validation, 3 = merge. */
int hetm_dev_stream_handle(hetm_dev* dev, int which, void** stream);
/* Per-kernel device timing (CUDA events around every batch / validation
 * launch of this handle).  which: 0 = batch kernels, 1 = validation kernels,
 * 2 = the device half of mergeCommit (hetm_dev_merge_stage: claim, emit,
 * shadow refresh).
 * hetm_dev_timing waits for the recorded launches, returns their summed
 * duration and count, and resets the accumulator. */
int hetm_dev_set_timing(hetm_dev* dev, int on);
int hetm_dev_timing(hetm_dev* dev, int which, double* total_ms, uint64_t* count);
/* Diagnostic counter words (phase clocks of instrumented builds); n <= 20. */
int hetm_dev_debug_words(hetm_dev* dev, uint64_t* out, uint64_t n);
/* Flush L2 (writes a buffer larger than L2) on `stream` — benchmark hygiene. */
int hetm_dev_flush_l2(hetm_dev* dev, void* stream);

/* Bank batch schedule.  OPTIMISTIC: the PR-STM-style
 * phased kernel (lock / ticket / validate / write-back, retries on conflict).
 * SCAN: an abort-free execution of the batch in input order (ticket = first +
 * input index): a radix sort of the written accounts + a segmented sum of
 * the transfers' deltas per account (applied with commutative adds; a traced
 * batch runs a segmented scan for every access's pre-value); its cost does not
 * grow with skew, while the optimistic kernel serializes every commit on a hot
 * account.  AUTO (default):
 * host-buffer batches take SCAN when a sample of the inputs predicts a chain
 * of >= 768 conflicting commits on one account (HETM_SCHED_CHAIN); device-
 * pointer batches follow the same estimate of an EARLIER device batch of the
 * handle (a one-CTA kernel samples each batch on a side stream into mapped
 * host memory, read by the next call without a sync), so a steady hot
 * workload switches after its first batch; they also take SCAN for the 15
 * batches after an optimistic one aborted > 1/128 of its transactions (judged
 * at the caller's next counters read / verdict), then retry optimistic.  The deterministic mode (HETM_CFG_DETERMINISTIC) always
 * runs bank batches as SCAN: the same input-order serialization, in parallel.
 * Cache batches have a SCAN schedule too (a stable sort by set, then one
 * thread per set runs that set's transactions in input order with the set in
 * registers); AUTO uses it for batches of >= 8192 transactions.
 * Both schedules give serializable batches whose replay in ticket order is
 * bit-exact (RS/WS/ChunkMap, write-set log, results and tickets included). */
enum { HETM_SCHED_OPTIMISTIC = 0, HETM_SCHED_SCAN = 1, HETM_SCHED_AUTO = 2 };
int hetm_dev_set_schedule(hetm_dev* dev, int mode);

/* Early merge (PAPER.md:355 double buffering, pushed one phase earlier): the
 * execution phase of the round is over (no executeBatch until its merge), so
 * the device write set is sorted, gathered and copied to the host now —
 * overlapping the log streaming and validation — instead of after the
 * verdict.  With host_replica != NULL the worker pool also writes it into the
 * host replica speculatively, each record keeping the value it replaced; the
 * round's mergeCommit then only refreshes devShadow, while mergeAbortDevice /
 * mergeAbortHost (or a new batch, or clearRound) first put the host replica
 * back.  Between this call and the round's merge call no host transaction may
 * touch host_replica (the host cut-off precedes validation).
 * A no-op without HETM_CFG_MERGE_DELTA or when the write-set log overflowed. */
int hetm_dev_merge_prepare(hetm_dev* dev, uint64_t* host_replica);
/* The device half of mergeCommit (HETM_CFG_MERGE_DELTA), fully
 * asynchronous on the merge stream and without a host round trip: the round's
 * device write set becomes one {word, value} record per written word in HBM
 * (claim + emit kernels over the write-set log) and devShadow := devReplica
 * (the records plus the winners of the round's host log).  The kernels read
 * the round's verdict themselves: on a conflict (or a write-set log overflow)
 * they do nothing, so mergeAbortDevice stays exact.  Closes the log intake and
 * ends the round's execution (later batches: HETM_ERR_STATE).  A following
 * hetm_dev_merge_commit only ships the staged records to the host replica. */
int hetm_dev_merge_stage(hetm_dev* dev);

/* ---------------------------------------------------- checker support -- *
 * Traces for the P1 / P2-dagger consistency checker (the
 * `checker` module).  Recording is toggleable and lossless:
 * events carry values, not just addresses.
 *
 * hetm_dev_trace_next_batch arms the NEXT hetm_dev_execute_batch /
 * hetm_dev_execute_batch_ex call of the handle (host-buffer form, bank and rw
 * kernels): out_records must hold n_tx * HETM_TRACE_TX_WORDS words and
 * receives, per input transaction i, {ticket, the values it read in program
 * order (bank: acct0..3; rw: r_addr[0..nr)), the values its read-modify-writes
 * read (rw: w_addr[0..nw); bank: acct0, acct1), the values it wrote, and 3
 * reserved words};
 * ticket = ~0 when it did not commit.  The batch runs the traced kernel
 * instantiation; untraced batches are unaffected. */
#define HETM_TRACE_TX_WORDS 12
int hetm_dev_trace_next_batch(hetm_dev* dev, uint64_t* out_records);

/* Fault injection for the checker's mutation suite ("rejects
 * every seeded mutation"): each flag disables one step of the protocol so the
 * tests can show the checker catches it.  Never set outside tests. */
#define HETM_FAULT_SKIP_RS 1u       /* validation never tests the RS bitmap (no conflicts) */
#define HETM_FAULT_SKIP_TS 2u       /* APPLY stores entries in arrival order, no TS freshness */
#define HETM_FAULT_SKIP_ROLLBACK 4u /* mergeAbortDevice leaves 1/8 of the write set un-restored */
#define HETM_FAULT_ALL 7u
int hetm_dev_set_fault(hetm_dev* dev, uint32_t flags);

/* One recorded event (40 B).  device: 0 host, 1 device.  kind: HETM_EV_*.
 * tx: host (thread << 40 | per-thread attempt number), device
 * (1 << 63 | batch number << 32 | input index).  value: read/write value,
 * SPEC_COMMIT ts (host) or commit ticket (device), FINAL_COMMIT round id,
 * ABORT reason.  seq: global append order (the real-time order key of host
 * events; device events are appended when the batch returns). */
enum {
    HETM_EV_BEGIN = 0,
    HETM_EV_READ = 1,
    HETM_EV_WRITE = 2,
    HETM_EV_SPEC_COMMIT = 3,
    HETM_EV_FINAL_COMMIT = 4,
    HETM_EV_ABORT = 5,
    HETM_EV_ROUND = 6 /* round boundary marker: value = round id */
};
enum { HETM_ABORT_CONFLICT = 1, HETM_ABORT_ROUND = 2 };
typedef struct hetm_trace_event {
    uint64_t seq;
    uint64_t tx;
    uint64_t addr;
    uint64_t value;
    uint32_t round;
    uint8_t device;
    uint8_t kind;
    uint16_t pad;
} hetm_trace_event;

/* ------------------------------------------------------------ host side -- */
int hetm_host_alloc(uint64_t bytes, void** p); /* pinned, portable */
int hetm_host_free(void* p);
int hetm_host_register(void* p, uint64_t bytes);
int hetm_host_unregister(void* p);
/* Seeded bank batch generator (DetRng, det_rng.hpp:19-42): for each tx, 4
 * distinct accounts uniform in [lo, lo+span) drawn by below(span) with
 * rejection on repeats, then amount = below(100)+1. */
int hetm_gen_bank_batch(uint64_t seed, uint64_t n, uint64_t lo, uint64_t span, hetm_bank_tx* out);
/* Seeded host write log: n_tx host transactions, each writing `writes_per_tx`
 * distinct words uniform in [lo, lo+span) with value = DetRng draw and one
 * shared ts (ts_base+1, ts_base+2, ... in commit order).  The
 * transactions are dealt round-robin to n_threads per-thread logs
 * (ts-ordered within a thread, write_log.hpp:27-28) and concatenated in
 * thread order like WriteLog::allEntries (write_log.hpp:74-82). */
int hetm_gen_host_log(uint64_t seed, uint64_t n_tx, uint32_t writes_per_tx, uint32_t n_threads,
                      uint64_t lo, uint64_t span, uint64_t ts_base, hetm_log_entry* out);
/* Zipf-skewed variants (BASELINE configs[2]): every account /
 * word is drawn as lo + rank - 1 with rank ~ Zipf(alpha) over [1, span] (rank 1
 * hottest; rejection-inversion sampler over DetRng uniform(), det_rng.hpp:36).
 * alpha == 0 is the uniform generator above. */
/* Seeded cache transactions (BASELINE configs[3]): key rank ~ Zipf(alpha)
 * over [1, key_space] (uniform when alpha == 0); key = {splitmix64(rank) with
 * its last bit set to the part, rank}; part = `part` (0 or 1) or, when part <
 * 0, part 1 except with probability steal_permille/1000 part 0; op GET with
 * probability get_permille/1000, else SET of 4 DetRng value words. */
int hetm_gen_cache_batch(uint64_t seed, uint64_t n, uint64_t key_space, double alpha, uint32_t get_permille,
                         int32_t part, uint32_t steal_permille, hetm_cache_tx* out);
int hetm_gen_bank_batch_zipf(uint64_t seed, uint64_t n, uint64_t lo, uint64_t span, double alpha, hetm_bank_tx* out);
int hetm_gen_host_log_zipf(uint64_t seed, uint64_t n_tx, uint32_t writes_per_tx, uint32_t n_threads, uint64_t lo,
                           uint64_t span, uint64_t ts_base, double alpha, hetm_log_entry* out);

#ifdef __cplusplus
}
#endif

#endif /* HETM_B200_CAPI_H */

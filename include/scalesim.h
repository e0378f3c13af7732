/*
 * scalesim.h — C ABI (v1) of the B200-native ScaleSim invocation-distance memory planner.
 *
 * The operation (arXiv 2601.21473, /root/reference/PAPER.md = P:<line>, SPEC.md = S:<line>):
 * every simulation step, (1) score every agent's invocation distance (§3.2, P:197-229,
 * Eq. 1, Eq. 2), (2) rank agents by (distance, agent id), (3) keep the
 * longest prefix of that order that fits the GPU memory budget, which yields the evict
 * list (Table 1 Evict; §3.3) and the prefetch list (Table 1
 * DispatchLoadTasks; §3.3), and (4) move the agents' memory blocks
 * between pinned host memory and HBM (Table 1 Load).  The readings the paper
 * leaves open are DESIGN.md §3 (R1..R17).
 *
 * Mapping of the paper's interface (Table 1) onto this ABI:
 *   agent distances from the frontend -> scalesim_score (computed here from agent state)
 *   Evict + DispatchLoadTasks         -> scalesim_plan  (one stateless plan per step)
 *   Load                              -> scalesim_transfer
 *   HandleReq                         -> stays with the caller: it marks requesting agents
 *                                        WAITING (distance 0) in their record.
 *
 * Conventions (all calls):
 *   - Every entry point returns scalesim_status and never throws or aborts.
 *   - Ownership: the caller owns every buffer (typically torch tensors) and keeps them alive
 *     until scalesim_destroy.  The device entry points never allocate memory after init; all
 *     scratch lives in the caller's workspace (size from scalesim_workspace_bytes).  The host
 *     entry points (scalesim_step_host, _stage_host, _stage_updates, _step_updates,
 *     _submit_updates, _collect) allocate, on first use, library-owned staging: three device
 *     input buffers of max(16 (n_local + n_kin), 20 n_local) bytes, three host-mapped pinned
 *     read-back slots of 256 + 8 n_local bytes, and one input stream; freed by scalesim_destroy.
 *   - Asynchrony: score/plan/transfer/step enqueue work on the caller's CUDA streams and
 *     return without a host synchronisation (graph-capturable).  Device-detected conditions
 *     (budget too small for the active agents, malformed records) are reported in the
 *     device status word and surface at scalesim_sync.  Sticky CUDA/NCCL errors surface at
 *     the next call as SCALESIM_E_CUDA / SCALESIM_E_NCCL.
 *   - Threading: one context per host thread.  Not re-entrant on one context.
 *   - Determinism: outputs are a pure function of (records, kinematics, residency, config),
 *     independent of launch configuration and of the number of ranks.
 */
#ifndef SCALESIM_H
#define SCALESIM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCALESIM_ABI_VERSION 1u

typedef struct scalesim_ctx scalesim_ctx;

typedef enum {
  SCALESIM_OK = 0,
  SCALESIM_E_INVALID = 1,        /* bad argument: null/misaligned pointer, size mismatch, block size
                                    not a page multiple, arena smaller than the budget, ... (S:487 exit 2) */
  SCALESIM_E_INSUFFICIENT = 2,   /* the active (distance 0) agents do not fit the budget; the plan is
                                    still produced and keeps the longest fitting prefix (R11) */
  SCALESIM_E_NOT_RESTORABLE = 3, /* reserved: a planned block without host backing */
  SCALESIM_E_ORDER = 4,          /* calls out of order: plan before score, transfer of a stale plan */
  SCALESIM_E_CUDA = 5,
  SCALESIM_E_NCCL = 6,
  SCALESIM_E_INVARIANT = 7,      /* device self-check failed (S:487 exit 3) */
  SCALESIM_E_BAD_INPUT = 8       /* malformed agent record or non-finite kinematics (status word) */
} scalesim_status;

/* Bits of the device status word (plan header field SCALESIM_H_STATUS). */
#define SCALESIM_ST_INSUFFICIENT 1u /* a distance-0 agent is outside the kept set */
#define SCALESIM_ST_BAD_RECORD 2u   /* class 3, or an INT agent whose kin index >= n_kin */
#define SCALESIM_ST_BAD_KIN 4u      /* ACTING INT agent with non-finite kinematics (excluded) */
#define SCALESIM_ST_NO_PAGES 8u     /* free page pool exhausted (cannot happen for a valid config) */
#define SCALESIM_ST_SYNC 16u        /* internal: a fused-kernel CTA timed out waiting for another
                                       CTA's published offsets (cannot happen: grid co-resident) */
#define SCALESIM_ST_LIMIT 32u       /* a large context (more than 12288 agents per SM, integer
                                       distances: the streaming single-kernel plan) met a step
                                       outside its scope: D* >= 2048 ticks, or more than 4096
                                       eligible agents at finite distances >= 2048 ticks (128
                                       per SM); the step's plan is not produced (create the
                                       context with SCALESIM_F_MULTI_KERNEL for such workloads).
                                       Not detected, also outside that kernel's scope: more than
                                       65535 eligible agents of one SM's id range (one CTA tile:
                                       contexts above ~9.7M agents) at the same distance value
                                       (its per-CTA bucket counters are 32-bit sums of 16-bit
                                       parts) */

/* Config flags. */
#define SCALESIM_F_NO_TRANSFER 1u   /* plan + byte accounting only: no arena, no pages, no copies
                                       (logical sizes, BASELINE configs 4 and 5) */
#define SCALESIM_F_KEEP_DIST 2u     /* keep per-agent distances readable after plan (dist view); the
                                       single-kernel path skips writing them otherwise */
#define SCALESIM_F_MULTI_KERNEL 4u  /* force the multi-kernel plan path (otherwise, at world == 1 and
                                       <= 16384 agents per SM, one persistent cooperative kernel
                                       scores and plans the step; both paths give identical plans) */
#define SCALESIM_F_EXPLICIT_DIST 8u /* records carry their distance (reading R19): word [0] = f32 bits
                                       of d >= 0 or +inf (NaN / negative: ST_BAD_RECORD, d = +inf;
                                       -0 -> +0); phase, class and kinematics are not used, every
                                       record is eligible below theta[0].  Plans shared memory
                                       objects from scalesim_object_min.  Requires
                                       n_kin == 0. */
#define SCALESIM_F_EXCLUSIVE 16u    /* the caller dedicates the device to this library's plans while
                                       they run: every SM usable (no MPS / green-context partition)
                                       and no other kernel concurrent with a plan launch.  The
                                       single-kernel plan is then launched without the cooperative
                                       attribute, so its prologue overlaps the previous kernel's tail
                                       (~2 us per step, profiles/r02_*); co-residency of its CTAs
                                       (one per SM) is checked at init, and the library orders the
                                       single-kernel plans of its exclusive contexts on one device
                                       one after another (event chain across their streams).
                                       Without the flag the launch is cooperative: the grid is
                                       scheduled as a whole and cannot deadlock against other work
                                       holding SMs (the kernel's grid barrier needs every CTA). */
#define SCALESIM_F_LOOPBACK 32u     /* world > 1 without NCCL: this context is rank `rank` of a world
                                       whose ranks all live on this device (one process) and are
                                       stepped together by scalesim_step_group: one launch of the
                                       single-kernel plan, floor(SMs / world) CTAs per rank, the
                                       exchange of the global cut through the ranks' workspaces
                                       after a world-wide barrier.  Shards must be
                                       contiguous, in rank order and cover [0, n_agents).
                                       Interaction agents (n_kin > 0) are allowed: each rank's
                                       pair scan runs over the world's participants, gathered
                                       from every rank's kinematics through device memory
                                       (SURVEY §8(e) "all-gather of kin for active INT agents";
                                       exact all-pairs, Eq. 2).  The ranks of
                                       one world must agree on n_kin > 0 (the distance class mix
                                       decides the histogram layout). */
#define SCALESIM_F_THREADS 128u     /* world > 1 on one device without NCCL, multi-kernel path: rank
                                       `rank` of a world whose ranks are contexts of this process on
                                       one device, each driven by its own host thread calling the
                                       same sequence of score / plan / step (a host barrier per
                                       collective).  The collectives the NCCL path calls (DESIGN §8:
                                       sums of the byte histograms, min of the bucket min keys,
                                       the all-gather of the ranks' bytes at D*, the kept tie bytes)
                                       run as reductions over the ranks' device buffers.  The
                                       group is the contexts created with the same 128-byte
                                       nccl_unique_id (any bytes).  Not with SCALESIM_F_LOOPBACK.
                                       Like NCCL ranks, a rank that stops calling (an error
                                       before a collective) leaves the others waiting in theirs;
                                       shards that are not contiguous in rank order fail the
                                       first collective with SCALESIM_E_INVALID on every rank. */
#define SCALESIM_F_TP_SLICED 64u    /* with SCALESIM_F_LOOPBACK and transfers: tensor-parallel
                                       agent memory (§4.2: "All multi-GPU setups
                                       use tensor parallelism"; reading R16).  Every rank holds
                                       slice `rank` (bytes [rank * page_bytes / world, +
                                       page_bytes / world)) of every resident page, so the block
                                       tables of every rank cover ALL n_agents agents (blk_ptr has
                                       n_agents + 1 entries) and a device page slot is
                                       page_bytes / world bytes (dev_bytes / slot slots, at least
                                       ceil(budget / page_bytes)).  Per step the ranks' lists are
                                       merged into the world's lists in every rank (SURVEY §8(e)
                                       step 4, the all-gather of per-rank lists), every rank
                                       assigns the pages of the whole plan (the same FIFO pool
                                       evolution on every rank) and copies its slice of each
                                       listed page.  Requires page_bytes % (16 * world) == 0 and
                                       no resident_init.  The merged lists and their transfer
                                       header: scalesim_world_view. */

/* Agent record: 4 x uint32 per agent, 16-byte aligned, one 128-bit load.
 *   [0] t_next : action-end tick (ACTING independent / interaction agents), or remaining hop
 *                count to the diffusion wave (ACTING diffusion agents; 0xFFFFFFFF = unreachable)
 *   [1] footprint bytes of the agent (must equal the sum of its block sizes)
 *   [2] flags  : bits 0-1 phase {0 ACTING, 1 WAITING, 2 GENERATING, 3 IDLE}
 *                bits 2-3 class {0 independent, 1 interaction, 2 diffusion}
 *                bit 4    dirty (KV / history written since last write-back, R13)
 *   [3] index into the kinematics array (interaction agents)
 * Kinematics: 4 x float per entry = {x, y, vx, vy} (Eq. 2).
 * Block kinds: 0 LORA (never written back), 1 KV page, 2 HIST (written back when dirty). */

typedef struct {
  uint32_t abi_version;   /* SCALESIM_ABI_VERSION */
  uint32_t flags;         /* SCALESIM_F_* */
  uint64_t n_agents;      /* global number of agents N (ids 0..N-1) */
  uint64_t shard_begin;   /* this rank's contiguous id range [shard_begin, shard_end) */
  uint64_t shard_end;
  uint64_t n_kin;         /* entries in the kinematics array (0 if no interaction agents) */
  uint64_t budget_bytes;  /* global GPU memory budget B for agent memory */
  float theta[3];         /* prefetch thresholds per class (R4); +inf allowed, >= 0 */
  float hop_scale;        /* ticks per hop for diffusion distances (R5), > 0, finite */
  uint64_t page_bytes;    /* device arena page size; every block size is a multiple; 4096-aligned */
  int32_t device;         /* CUDA device ordinal */
  int32_t rank, world;    /* world > 1: NCCL exchange for the global cut, or
                             SCALESIM_F_LOOPBACK (scalesim_step_group) */
  const void *nccl_unique_id; /* 128 bytes from scalesim_nccl_unique_id on rank 0, broadcast by the
                                 caller (e.g. torch.distributed); ignored when world == 1 */
  void *stream;           /* cudaStream_t for score/plan (0 = legacy default stream) */
  void *copy_stream;      /* cudaStream_t for the block transfers (must differ from stream to overlap) */
} scalesim_config;

typedef struct {
  /* device, read each step: the caller writes them before scalesim_score / scalesim_step */
  const uint32_t *agent_rec;    /* 4 * n_local uint32, n_local = shard_end - shard_begin, 16-B aligned */
  const float *agent_kin;       /* 4 * n_kin float, 16-B aligned; may be NULL when n_kin == 0 */
  /* device, read-only after init: CSR agent -> memory blocks (local agents) */
  const uint64_t *blk_ptr;      /* n_local + 1 (SCALESIM_F_TP_SLICED: n_agents + 1, every agent) */
  const uint32_t *blk_size;     /* n_blocks, multiples of page_bytes */
  const uint64_t *blk_host_off; /* n_blocks, byte offset of the block in host_arena (page aligned) */
  const uint8_t *blk_kind;      /* n_blocks, 0 LORA / 1 KV / 2 HIST */
  uint64_t n_blocks;
  uint64_t n_block_pages;       /* sum over blocks of blk_size / page_bytes */
  /* arenas (ignored with SCALESIM_F_NO_TRANSFER) */
  void *host_arena;             /* pinned, device-mapped (cudaHostAlloc / torch pin_memory) */
  uint64_t host_bytes;
  void *dev_arena;              /* HBM; dev_bytes / page_bytes pages, >= ceil(budget / page_bytes) */
  uint64_t dev_bytes;
  /* scratch: device, >= scalesim_workspace_bytes(), 256-B aligned, owned by the library until destroy */
  void *workspace;
  uint64_t workspace_bytes;
  /* optional device bitmap (n_local bits, 32-agent words) of agents resident at init; their
     blocks receive pages in id order and (unless NO_TRANSFER) are loaded at init */
  const uint32_t *resident_init;
} scalesim_tables;

/* Header fields of a plan (uint64 each), device: scalesim_plan_view.header, host: scalesim_plan_host. */
enum {
  SCALESIM_H_N_PREFETCH = 0, /* entries of prefetch_ids */
  SCALESIM_H_N_EVICT = 1,    /* entries of evict_ids */
  SCALESIM_H_BYTES_H2D = 2,  /* sum of footprints of prefetched agents */
  SCALESIM_H_BYTES_D2H = 3,  /* sum of KV+HIST block bytes of evicted dirty agents (R13) */
  SCALESIM_H_CUT_BITS = 4,   /* f32 bits of the boundary distance D*; 0xFFFFFFFF if all fit */
  SCALESIM_H_CUT_REM = 5,    /* B - bytes(eligible agents with distance < D*) */
  SCALESIM_H_STATUS = 6,     /* SCALESIM_ST_* bits */
  SCALESIM_H_N_D2H = 7,      /* page descriptors in d2h_desc */
  SCALESIM_H_N_H2D = 8,      /* page descriptors in h2d_desc */
  SCALESIM_H_KEPT_BYTES = 9, /* bytes of the kept (resident) set, global */
  SCALESIM_H_N_ELIGIBLE = 10,/* eligible agents on this rank */
  SCALESIM_H_POOL_HEAD = 11, /* free-page FIFO counters after this plan */
  SCALESIM_H_POOL_TAIL = 12,
  SCALESIM_H_SEQ = 13,       /* plans completed on the device so far (integrity check for graphs) */
  SCALESIM_H_FIELDS = 16
};

typedef struct {
  /* device views into the workspace; valid until the next scalesim_plan / scalesim_step */
  const uint32_t *prefetch_ids;    /* global agent ids, ascending (distance, id): most urgent first */
  const uint32_t *evict_ids;       /* global agent ids, descending (distance, id): largest first */
  const uint32_t *resident_bitmap; /* kept set after this plan, n_local bits */
  const float *dist;               /* per local agent distance (valid with SCALESIM_F_KEEP_DIST) */
  const uint32_t *page_table;      /* per block page: device page index, 0xFFFFFFFF = not resident */
  const uint64_t *d2h_desc;        /* pairs {host byte offset, device page}, n_d2h entries */
  const uint64_t *h2d_desc;        /* pairs {host byte offset, device page}, n_h2d entries */
  const uint64_t *header;          /* SCALESIM_H_FIELDS uint64 */
  void *done_event;                /* cudaEvent_t recorded on copy_stream after this plan's transfer */
} scalesim_plan_view;

typedef struct {
  uint64_t f[SCALESIM_H_FIELDS];   /* host copy of the header, indexed by SCALESIM_H_* */
} scalesim_plan_host;

/* Bytes of workspace the context needs (0 on invalid config).  Pure host function. */
uint64_t scalesim_workspace_bytes(const scalesim_config *cfg, const scalesim_tables *tables);

/* Validate cfg/tables, take the workspace, build the page pool from resident_init, create the
 * NCCL communicator when world > 1.  Synchronous.  *out is NULL on error. */
scalesim_status scalesim_init(const scalesim_config *cfg, const scalesim_tables *tables, scalesim_ctx **out);

/* (1) Score: invocation distance of every local agent at tick now_tick (Eq. 1-2),
 * eligibility (R4) and the byte-weighted distance histogram.  If dist_out (device, n_local
 * floats) is non-NULL the distances are also written there.  Async on cfg.stream. */
scalesim_status scalesim_score(scalesim_ctx *ctx, int64_t now_tick, float *dist_out);

/* (2)+(3) Plan: rank by (distance, id), cut the longest prefix within the budget, emit the
 * evict/prefetch lists, the new residency, byte totals and (unless NO_TRANSFER) the page
 * assignment and copy descriptors.  Requires a preceding scalesim_score.  With world > 1
 * the NCCL exchange for the global cut runs inside, on cfg.stream.  out may be NULL. */
scalesim_status scalesim_plan(scalesim_ctx *ctx, scalesim_plan_view *out);

/* (4) Transfer: write back the dirty evicted blocks, then load the prefetched blocks
 * (device page <-> pinned host), on copy_stream, after the plan's event; records the plan's
 * done_event.  Requires the most recent plan. */
scalesim_status scalesim_transfer(scalesim_ctx *ctx, const scalesim_plan_view *plan);

/* Fill *out with the views of the context's latest plan (e.g. after scalesim_step_batch). */
scalesim_status scalesim_view(scalesim_ctx *ctx, scalesim_plan_view *out);

/* score + plan + transfer of one step. */
scalesim_status scalesim_step(scalesim_ctx *ctx, int64_t now_tick, scalesim_plan_view *out);

/* One step of several independent contexts (simulation replicas / parameter sweeps, C5,
 * BASELINE configs[4]) in as few launches as possible: each context is planned by its
 * own group of floor(SMs / k) CTAs of one persistent kernel (k <= SMs contexts per launch; a
 * group of one CTA orders its lists in shared memory instead of the multi-CTA slot pass).
 * All contexts must use the single-kernel plan path (scalesim_fused == 1) on the same device
 * and the same cfg.stream; each context's inputs are its own tables; all share now_tick.
 * Equivalent to scalesim_step on every context in turn (same plans, tests/test_gpu_parity.py).
 * Errors: SCALESIM_E_INVALID for a NULL / non-fused / mixed-stream context or a context too
 * large for its group's tile; otherwise the first failing context's status. */
scalesim_status scalesim_step_batch(scalesim_ctx *const *ctxs, uint32_t n, int64_t now_tick);

/* One step of a world of `world` ranks on one device (contexts created with
 * SCALESIM_F_LOOPBACK, ctxs[r] = rank r, all on the same device and cfg.stream, same n_agents,
 * budget and thresholds, contiguous shards in rank order covering [0, n_agents), equal step
 * counts): score + plan + transfer of every rank, the global cut exchanged inside one launch.
 * Each rank's plan holds its own shard's lists (global ids, list order of the world) and
 * residency; cut_bits, cut_rem, kept_bytes, n_eligible and the INSUFFICIENT bit are
 * world-wide, the other header fields the rank's.  plan(world) == plan(1) restricted to the
 * shard (tests/test_gpu_world.py).  Errors: SCALESIM_E_INVALID for a malformed world. */
scalesim_status scalesim_step_group(scalesim_ctx *const *ctxs, uint32_t world, int64_t now_tick);

/* The world's merged plan of a SCALESIM_F_TP_SLICED rank after its last step (device views into
 * the workspace, overwritten by the next step): prefetch_ids (ascending (distance, id)) and
 * evict_ids (descending), identical in every rank and equal to the world-1 plan's lists
 * (Table 1 Evict / DispatchLoadTasks); header: SCALESIM_H_N_PREFETCH /
 * _N_EVICT (the world's counts), SCALESIM_H_N_D2H / _N_H2D (pages of the whole plan; this rank
 * moves its slice of each), SCALESIM_H_BYTES_D2H (the world's write-back bytes, R13).  The
 * rank's own header (scalesim_view) keeps its shard's plan and carries the page counts.
 * Errors: SCALESIM_E_INVALID (NULL, not TP-sliced), SCALESIM_E_ORDER (before the first step). */
typedef struct {
  const uint32_t *prefetch_ids;
  const uint32_t *evict_ids;
  const uint64_t *header;  /* SCALESIM_H_* fields as above */
} scalesim_world_view_t;
scalesim_status scalesim_world_view(scalesim_ctx *ctx, scalesim_world_view_t *out);

/* ---- NEXT #2: the preemptive priority load scheduler (App. A "Load task scheduler"
 * and "Preemption support"; SPEC.md S:291-293, S:324-327, S:348-356, S:366-374;
 * readings R21-R23).  One channel moves one task's chunk per slot from
 * the pinned host arena to the device arena; at every chunk boundary the boundary's events are
 * admitted, then the most urgent waiting task runs, preempting the executing task when it is
 * strictly more urgent (the preempted task resumes later with its completed chunks kept). */
#define SCALESIM_LOAD_SUBMIT 0u   /* a load task for `agent` (coalesced into the agent's live task:
                                     the smaller priority wins, no new task) */
#define SCALESIM_LOAD_REFRESH 1u  /* the agent's refreshed distance: its waiting (queued or
                                     preempted) task is cancelled when priority >= threshold; the
                                     executing task never is */
typedef struct {
  uint32_t slot;      /* admitted at the boundary before chunk slot `slot`; events sorted by slot,
                         same-slot events applied in array order */
  uint32_t kind;      /* SCALESIM_LOAD_* */
  uint32_t agent;     /* < n_agents */
  float priority;     /* SUBMIT: invocation distance (>= 0, lower = more urgent, ties by task id);
                         REFRESH: the agent's new distance */
  uint64_t host_off;  /* SUBMIT: source bytes in the host arena (16-byte aligned) ... */
  uint64_t dev_off;   /* ... destination in the device arena (16-byte aligned) */
  uint64_t bytes;     /* ... length (chunks = ceil(bytes / chunk_bytes), at least 1) */
} scalesim_load_event;
typedef struct {
  uint32_t task, chunk; /* what moved in a slot; task 0xFFFFFFFF = idle channel */
} scalesim_load_slot;
typedef struct {
  uint32_t agent, chunks, done, state; /* state: 0 queued, 1 executing, 2 preempted, 3 done, 4 cancelled */
  float priority;                      /* after coalescing */
  uint32_t preemptions, finish_slot, pad;
} scalesim_load_task;                  /* task ids = creation order (non-coalesced submissions) */

uint64_t scalesim_sched_scratch_bytes(uint32_t n_events, uint32_t n_agents);
/* Run a whole schedule on `stream` (asynchronous, one persistent launch): events (device,
 * n_events), the prefetch threshold of REFRESH events, chunk_bytes (multiple of 16; the SPEC's
 * default is 16 MB), host_arena (pinned, device-mapped) and dev_arena.  Outputs (device): trace
 * (max_slots entries), tasks (n_events entries), counts[0] = slots run (the schedule stops when
 * no task is live and no event is left, or at max_slots), counts[1] = tasks created.  scratch:
 * 256-byte aligned device memory of scalesim_sched_scratch_bytes.  Errors: SCALESIM_E_INVALID
 * for NULL / misaligned arguments or chunk_bytes % 16 != 0; SCALESIM_E_CUDA. */
scalesim_status scalesim_sched_run(const scalesim_load_event *events, uint32_t n_events, uint32_t n_agents,
                                   float threshold, uint64_t chunk_bytes, const void *host_arena, void *dev_arena,
                                   uint32_t max_slots, scalesim_load_slot *trace, scalesim_load_task *tasks,
                                   uint32_t *counts, void *scratch, uint64_t scratch_bytes, void *stream);

/* End-to-end step from HOST buffers: copies host_rec (4*n_local uint32) and host_kin
 * (4*n_kin float, may be NULL) to the device, runs scalesim_step, waits, and copies the
 * plan header and lists back (prefetch_out/evict_out: host, n_local capacity each, may be
 * NULL).  Synchronous.  Returns SCALESIM_E_INSUFFICIENT / _BAD_INPUT per the status word. */
scalesim_status scalesim_step_host(scalesim_ctx *ctx, int64_t now_tick, const uint32_t *host_rec,
                                   const float *host_kin, scalesim_plan_host *out,
                                   uint32_t *prefetch_out, uint32_t *evict_out);

/* Pipelined end-to-end steps (the host side of P:242's overlap: a later step's inputs cross
 * the host link while this step plans).  Starts the host->device copy of a LATER step's
 * inputs — host_rec (4*n_local uint32) and host_kin (4*n_kin float; may be NULL when
 * n_kin == 0), ideally pinned — into one of two library-owned device buffers on a
 * library-owned stream, and returns at once.  The host buffers must stay unchanged until the
 * scalesim_step_host call that consumes them returns.  A later scalesim_step_host(ctx, now,
 * host_rec, host_kin, ...) with the SAME pointers plans from the staged copy (its plan waits
 * for that copy on the device, not on the host) instead of copying synchronously; the
 * context's own input buffers (init / scalesim_set_inputs) are left untouched.  Usage:
 * stage(in[0]); for t: { stage(in[t+1]); step_host(in[t]); }.  At most three staged steps
 * may be outstanding.  Errors: SCALESIM_E_INVALID (NULL ctx / host_rec, or host_kin NULL with
 * n_kin > 0), SCALESIM_E_ORDER (three staged steps not yet consumed), SCALESIM_E_CUDA. */
scalesim_status scalesim_stage_host(scalesim_ctx *ctx, const uint32_t *host_rec, const float *host_kin);

/* Incremental end-to-end steps.  Agent state changes only where the simulation acted (P:197-205:
 * an invocation starts or ends an action; ~5% of AgentSociety's agents per step), so the
 * step's inputs are the CHANGED records: host_ids (n_upd global agent ids of this shard,
 * distinct — with a repeated id, which of its records lands is unspecified) and host_rec
 * (4*n_upd uint32, the new 16-byte records in the layout of scalesim_init's agent_rec).  The
 * records are written into the context's current record buffer (scalesim_init /
 * scalesim_set_inputs, device, caller-owned: it must hold the previous step's records, e.g.
 * after one scalesim_step_host), then the step runs and its header and lists come back as in
 * scalesim_step_host.  scalesim_stage_updates starts the host->device copy of a LATER step's
 * updates (library-owned staging shared with scalesim_stage_host: at most three staged steps)
 * and returns at once; scalesim_step_updates with the same (host_ids, host_rec, n_upd) uses
 * that copy (the scatter waits for it on the device), otherwise it copies synchronously.  The
 * scatter runs on the plan stream after the previous step's plan, so staging never races a
 * plan still reading the records.  Contexts with kinematics (n_kin > 0) use
 * scalesim_step_host.  Errors: SCALESIM_E_INVALID (NULL ctx, NULL arrays with n_upd > 0,
 * n_upd > n_local, n_kin > 0), SCALESIM_E_ORDER (three staged steps not yet consumed),
 * SCALESIM_E_BAD_INPUT (ids outside the shard: skipped, the step still runs on the others),
 * else as scalesim_step_host. */
scalesim_status scalesim_stage_updates(scalesim_ctx *ctx, const uint32_t *host_ids, const uint32_t *host_rec,
                                       uint32_t n_upd);
scalesim_status scalesim_step_updates(scalesim_ctx *ctx, int64_t now_tick, const uint32_t *host_ids,
                                      const uint32_t *host_rec, uint32_t n_upd, scalesim_plan_host *out,
                                      uint32_t *prefetch_out, uint32_t *evict_out);

/* Asynchronous form of scalesim_step_updates: submit enqueues the step (its updates' copy on
 * the library's input stream, the scatter, the plan, and the read-back of header and lists
 * into library-owned host-mapped memory) and returns at once; collect waits for the OLDEST
 * submitted step and copies its header and lists out (prefetch_out / evict_out: host,
 * n_local capacity each, may be NULL).  Steps run in submission order on the device; while
 * the host collects step t, steps t+1 and t+2 already copy and plan.  Usage: submit(0);
 * submit(1); for t: { submit(t+2); collect(t); }.  At most three submitted steps may be
 * uncollected (SCALESIM_E_ORDER), and
 * scalesim_step_host / scalesim_step_updates refuse to run (SCALESIM_E_ORDER) until all are
 * collected.  The host arrays must stay unchanged until their step is collected.  Errors of
 * submit: as scalesim_stage_updates; of collect: SCALESIM_E_ORDER (nothing submitted),
 * SCALESIM_E_BAD_INPUT (that step had ids outside the shard), SCALESIM_E_INSUFFICIENT /
 * SCALESIM_E_INVARIANT per its status word, SCALESIM_E_CUDA. */
scalesim_status scalesim_submit_updates(scalesim_ctx *ctx, int64_t now_tick, const uint32_t *host_ids,
                                        const uint32_t *host_rec, uint32_t n_upd);
scalesim_status scalesim_collect(scalesim_ctx *ctx, scalesim_plan_host *out, uint32_t *prefetch_out,
                                 uint32_t *evict_out);

/* Point the context at another record / kinematics buffer (same sizes; device). */
scalesim_status scalesim_set_inputs(scalesim_ctx *ctx, const uint32_t *agent_rec, const float *agent_kin);

/* Wait for the last plan (and its transfer) and copy its header to the host.  Returns
 * SCALESIM_E_INSUFFICIENT / SCALESIM_E_BAD_INPUT according to the status word. */
scalesim_status scalesim_sync(scalesim_ctx *ctx, scalesim_plan_host *out);

/* NCCL unique id (128 bytes) for rank 0 to broadcast. */
scalesim_status scalesim_nccl_unique_id(void *out128);

/* Make cfg.stream wait for the last plan's transfer (joins copy_stream back into the
 * caller's stream: required before reading arena pages on cfg.stream, and before ending a
 * CUDA-graph capture that contains scalesim_transfer). */
scalesim_status scalesim_join(scalesim_ctx *ctx);

/* 1 if this context plans each step with the single persistent kernel, 2 with its streaming
 * variant (integer distances, more than 12288 agents per SM: fused_big.cu), 0 with the
 * multi-kernel path (world > 1 over NCCL, SCALESIM_F_MULTI_KERNEL, or large non-integer
 * contexts), -1 on NULL. */
int scalesim_fused(const scalesim_ctx *ctx);

/* Device pointer to 64 uint64 %globaltimer stamps (ns) written by the fused plan kernel:
 * [0] earliest CTA start past the dependency wait (atomicMin), [1] latest CTA end
 * (atomicMax), [2..10] and [32..35] phase boundaries seen by CTA 0, [11..31] latest CTA per
 * phase (atomicMax) and per-slot section times (tools/timing_probe.py names them).  The caller
 * resets [0] to UINT64_MAX and the rest to 0 between launches it wants to time.  Profiling
 * aid; NULL for a NULL context. */
const uint64_t *scalesim_profile_stamps(const scalesim_ctx *ctx);

/* Fine-grained distance assignment for shared memory objects ("the invocation
 * distance of a memory object as the minimum invocation distance among all agents that
 * currently reference it"; S:263-271 recompute_object_distances; reading R19):
 *   dist(o) = min { agent_dist[a] : a in ref_agent[ref_ptr[o] .. ref_ptr[o+1]) },  +inf if empty.
 * Writes one record per object for a context created with SCALESIM_F_EXPLICIT_DIST
 * (word [0] = f32 bits of dist(o), [1] = obj_bytes[o], [2] = obj_flags[o] (0 if NULL), [3] = 0),
 * so the objects are ranked, cut and transferred by the same planner.
 *   agent_dist   device f32 [n_agents], >= 0 or +inf (e.g. the dist view of an agent context
 *                created with SCALESIM_F_KEEP_DIST, after its plan)
 *   ref_ptr      device u64 [n_objects + 1], non-decreasing CSR offsets into ref_agent
 *   ref_agent    device u32 [ref_ptr[n_objects]], agent indices; an index >= n_agents is skipped
 *                and sets SCALESIM_ST_BAD_RECORD in *status_out
 *   obj_bytes    device u32 [n_objects]; obj_flags device u32 [n_objects] or NULL
 *   obj_rec_out  device, 16-byte aligned, 4 x u32 per object; obj_dist_out device f32 [n_objects]
 *                or NULL; status_out device u32 (ORed) or NULL
 *   stream       cudaStream_t (NULL: legacy default stream)
 * Asynchronous (stream-ordered, graph-capturable).  Returns SCALESIM_E_INVALID for NULL or
 * misaligned required pointers, SCALESIM_E_CUDA on a launch error.  n_objects == 0 is a no-op. */
scalesim_status scalesim_object_min(const float *agent_dist, uint64_t n_agents, const uint64_t *ref_ptr,
                                    const uint32_t *ref_agent, uint64_t n_objects, const uint32_t *obj_bytes,
                                    const uint32_t *obj_flags, void *obj_rec_out, float *obj_dist_out,
                                    uint32_t *status_out, void *stream);

/* Reactive LRU baseline (the paper's SGLang-style comparison policy; S:330-338;
 * reading R20), as explicit-distance records for a context created with
 * SCALESIM_F_EXPLICIT_DIST and planned with theta = 0: an agent in an LLM phase (WAITING /
 * GENERATING) gets distance 0 and last_use[i] = now_tick; any other agent gets
 * now_tick - last_use[i] (+inf while last_use[i] == 0xFFFFFFFF, never used).  Record word
 * [1] = the agent's footprint, [2] = its dirty bit.
 *   agent_rec   device, 16-byte aligned, 4 x u32 per agent (the planner's record layout)
 *   last_use    device u32 [n_agents], caller-initialised to 0xFFFFFFFF; updated in place
 *   rec_out     device, 16-byte aligned, 4 x u32 per agent
 *   now_tick    0 <= now_tick < 2^32 - 1, non-decreasing across calls
 * Asynchronous on `stream`.  Returns SCALESIM_E_INVALID for NULL / misaligned pointers or a
 * tick out of range. */
scalesim_status scalesim_lru_records(const uint32_t *agent_rec, uint64_t n_agents, int64_t now_tick,
                                     uint32_t *last_use, void *rec_out, void *stream);

/* Hop counts for the diffusion class ("hop count from the information source", R9):
 * breadth-first levels from a source set over a CSR graph, on the GPU (an initialisation-time
 * computation: the caller turns them into the records' remaining-hop words).
 *   row_ptr   device u64 [n_vertices + 1], col device u32 [row_ptr[n_vertices]] (neighbours;
 *             indices >= n_vertices are ignored)
 *   sources   device u32 [n_sources] (out-of-range entries ignored, duplicates allowed)
 *   hops_out  device u32 [n_vertices]: BFS level, 0xFFFFFFFF where unreachable
 *   scratch   device, 16-byte aligned, >= scalesim_bfs_scratch_bytes(n_vertices) bytes
 * Synchronous on `stream` (the host reads each level's frontier size).  Returns
 * SCALESIM_E_INVALID for NULL / misaligned / undersized arguments or n_vertices >= 2^32 - 1. */
uint64_t scalesim_bfs_scratch_bytes(uint64_t n_vertices);
scalesim_status scalesim_bfs_hops(const uint64_t *row_ptr, const uint32_t *col, uint64_t n_vertices,
                                  const uint32_t *sources, uint64_t n_sources, uint32_t *hops_out, void *scratch,
                                  uint64_t scratch_bytes, void *stream);

/* Launches of library kernels enqueued so far (for the bench's gpu_launches). */
uint64_t scalesim_launch_count(const scalesim_ctx *ctx);

/* Destroy the context (synchronises its streams).  NULL is a no-op. */
void scalesim_destroy(scalesim_ctx *ctx);

const char *scalesim_strerror(scalesim_status s);

#ifdef __cplusplus
}
#endif
#endif /* SCALESIM_H */

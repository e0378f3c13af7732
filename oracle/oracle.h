/*
 * oracle.h — CPU oracle for the ScaleSim invocation-distance memory planner.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2601_21473_b200/, include/scalesim.h) never links, includes or calls it,
 * and this tree includes nothing from the product.
 *
 * It is a plain, slow, single-threaded implementation of the definitions in
 * /root/reference/PAPER.md (cited P:<line>) and SPEC.md (S:<line>), with the
 * readings listed in DESIGN.md §3.  No blocking, no fusion, no radix select: it
 * scores every agent by the formula, sorts the eligible agents with std::sort on
 * the (distance, agent id) key and walks the sorted order.
 *
 * Record layout (shared *input format*, not shared code):
 *   rec[4*i+0] t_next   action-end tick (ACTING IND/INT) or remaining hop count (ACTING DIFF;
 *                       0xFFFFFFFF = unreachable)
 *   rec[4*i+1] footprint bytes of agent i (sum of its block sizes)
 *   rec[4*i+2] flags: bits0-1 phase {0 ACTING,1 WAITING,2 GENERATING,3 IDLE},
 *                     bits2-3 class {0 IND,1 INT,2 DIFF}, bit4 dirty
 *   rec[4*i+3] index into kin (INT agents)
 *   kin[4*k+0..3] = x, y, vx, vy (float)
 *
 * Parity pins for every function are in tests/test_oracle_*.py.
 */
#ifndef SCALESIM_ORACLE_H
#define SCALESIM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* status bits (same meaning as the product's device status word; defined independently) */
#define ORACLE_ST_INSUFFICIENT 1u /* some d==0 agent is outside the kept set */
#define ORACLE_ST_BAD_RECORD   2u /* class 3, or INT agent whose kin index >= n_kin */
#define ORACLE_ST_BAD_KIN      4u /* ACTING INT agent with a non-finite kinematic value */
#define ORACLE_ST_NO_PAGES     8u /* free page pool exhausted (cannot happen when dev pages >= budget) */

/* Score every agent: §3.2, Eq. 1, Eq. 2.
 * d_out[i] receives the invocation distance of agent i (float, >= +0, +inf allowed).
 * *status receives ORACLE_ST_BAD_RECORD / ORACLE_ST_BAD_KIN bits. */
void oracle_score(uint64_t n, const uint32_t *rec, const float *kin, uint64_t n_kin,
                  int64_t now, float hop_scale, float *d_out, uint32_t *status);

/* Fine-grained distance assignment for shared memory objects ("the invocation
 * distance of a memory object as the minimum invocation distance among all agents that
 * currently reference it"; reading R19):
 *   d_obj[o] = min { agent_dist[a] : a in ref_agent[ref_ptr[o] .. ref_ptr[o+1]) },  +inf if none.
 * An agent index >= n_agents is skipped and a NaN / negative agent distance is read as +inf
 * (*status |= ORACLE_ST_BAD_RECORD for either); -0 reads as +0. */
void oracle_object_min(uint64_t n_agents, const float *agent_dist, uint64_t n_obj, const uint64_t *ref_ptr,
                       const uint32_t *ref_agent, float *d_obj, uint32_t *status);

/* Explicit distances (reading R19): d_out[i] = the float whose bits are rec word 0 of record i;
 * NaN or negative -> +inf and ORACLE_ST_BAD_RECORD; -0 -> +0. */
void oracle_explicit_dist(uint64_t n, const uint32_t *rec, float *d_out, uint32_t *status);

/* Reactive LRU baseline as explicit distances (P:303 SGLang-style on-demand loading with LRU
 * eviction; reading R20): agent i in WAITING or GENERATING gets distance 0 and
 * last_use[i] = now; any other agent gets now - last_use[i], or +inf while last_use[i] is
 * 0xFFFFFFFF (never used).  rec_out[i] = {f32 bits of the distance, footprint, dirty bit, 0}. */
void oracle_lru_records(uint64_t n, const uint32_t *rec, int64_t now, uint32_t *last_use, uint32_t *rec_out);

/* Diffusion hop counts ("hop count from the information source", R9): breadth-first
 * levels from the source set over a CSR graph (row_ptr [n+1], col); 0xFFFFFFFF unreachable.
 * Out-of-range neighbour / source indices are ignored. */
void oracle_bfs_hops(uint64_t n, const uint64_t *row_ptr, const uint32_t *col, const uint32_t *sources,
                     uint64_t n_sources, uint32_t *hops);

/* Interaction component only (Eq. 2): dint[k] = min over other ACTING INT agents j of
 * (r.r)/(-r.w) for approaching pairs, +inf otherwise; indexed by kin index.  Exposed so
 * the tests can pin Eq. 2 separately.  Entries of kin not owned by an ACTING INT agent
 * get +inf. */
/* oracle_score's distances for a sample of agents only (agents[0..n_sample)): the same
 * definitions, the Eq. 2 scan restricted to the sampled rows (full-size parity of the spatial
 * grid at 10^6 interaction agents, where the full O(n^2) scan is out of reach). */
void oracle_score_sampled(uint64_t n, const uint32_t *rec, const float *kin, uint64_t n_kin, int64_t now,
                          float hop_scale, const uint64_t *agents, uint64_t n_sample, float *d_out,
                          uint32_t *status);

void oracle_interaction(uint64_t n, const uint32_t *rec, const float *kin, uint64_t n_kin,
                        float *dint, uint32_t *status);

/* Plan one step: §3.3, Table 1 Evict / DispatchLoadTasks.
 *   resident_in/out: one byte per agent (0/1).
 *   theta[3]: prefetch thresholds per class (IND, INT, DIFF).
 *   prefetch/evict: capacity n each; filled in list order (prefetch ascending key,
 *   evict descending key).
 *   out[0]=bytes_h2d (sum footprint of prefetched), out[1]=cut_bits (f32 bits of D*,
 *   0xFFFFFFFF if every eligible agent fits), out[2]=cut_rem (B - bytes(elig, d<D*)),
 *   out[3]=kept bytes, out[4]=n eligible.
 *   *status |= ORACLE_ST_INSUFFICIENT when a d==0 agent is not kept. */
void oracle_plan(uint64_t n, const uint32_t *rec, const float *d, const uint8_t *resident_in,
                 const float *theta, uint64_t budget, uint8_t *resident_out,
                 uint32_t *prefetch, uint64_t *n_prefetch, uint32_t *evict, uint64_t *n_evict,
                 uint64_t *out, uint32_t *status);

/* Paged device arena: blocks are runs of page_bytes pages; a FIFO
 * pool of free device pages; deterministic assignment. */
typedef struct oracle_mem oracle_mem;
oracle_mem *oracle_mem_create(uint64_t n_agents, const uint64_t *blk_ptr, const uint32_t *blk_size,
                              const uint64_t *blk_host_off, const uint8_t *blk_kind,
                              uint64_t page_bytes, uint64_t n_pages, const uint8_t *resident_init);
void oracle_mem_destroy(oracle_mem *m);
/* Apply a plan: releases the evicted agents' pages (evict-list order, block order, page
 * order) to the tail of the pool, then assigns pool-head pages to the prefetched agents
 * (prefetch-list order, block order, page order).  Emits page-granular copy descriptors:
 *   d2h: (host byte offset, device page) for every page of a non-LORA block of an evicted
 *        agent whose dirty bit is set, in release order;  h2d: for every page of every
 *        block of a prefetched agent, in assignment order.
 * out[0] = bytes_d2h, out[1] = bytes_h2d, out[2] = n_d2h descriptors, out[3] = n_h2d. */
void oracle_mem_apply(oracle_mem *m, const uint32_t *rec, const uint32_t *prefetch, uint64_t n_prefetch,
                      const uint32_t *evict, uint64_t n_evict,
                      uint64_t *d2h_host, uint32_t *d2h_page, uint64_t *h2d_host, uint32_t *h2d_page,
                      uint64_t *out, uint32_t *status);
/* page_table: one u32 per block page (0xFFFFFFFF = not resident), in block order. */
uint64_t oracle_mem_total_pages(const oracle_mem *m);
void oracle_mem_page_table(const oracle_mem *m, uint32_t *page_table);
void oracle_mem_pool(const oracle_mem *m, uint64_t *head, uint64_t *tail, uint32_t *ring);

#ifdef __cplusplus
}
#endif
#endif

// internal.h — shared between api.cpp (host, C ABI) and kernels.cu (device).  Not installed.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ss {

constexpr int NT = 256;                   // threads per block of the agent-scan kernels
constexpr uint32_t TILE = 2048;           // agents per tile (id-ordered kernels); multiple of 32
constexpr uint32_t SORT_CH = 8192;        // list elements per sort chunk
constexpr uint32_t EXP_CH = 256;          // list entries per expansion chunk
constexpr uint32_t KEY_NONE = 0xFFFFFFFFu;
constexpr int DESC_HDR = 4;  // descriptor buffer: n_d2h, n_h2d, n_h2d_independent, 0, then pairs
constexpr uint32_t PAGE_NONE = 0xFFFFFFFFu;
constexpr int L1_BITS = 11, L2_BITS = 10, L3_BITS = 10;  // distance-bit digits [30:20] [19:10] [9:0]
constexpr uint32_t GRID_MAX_SIDE = 128;   // a1' spatial grid: at most 128 x 128 cells
constexpr uint64_t GRID_MIN_PARTICIPANTS = 2048;  // below: tiled all-pairs scan
constexpr int FUSED_MAX_CTAS = 160;       // fused path: one CTA per SM (B200: 148)
constexpr int COPY_CTAS = 8;              // a6: CTAs per page-copy launch (two run at once: write-backs and
                                          // independent loads); the single-kernel plan of a transfer
                                          // context leaves 2 * COPY_CTAS SMs to them, so the plan of step
                                          // t+1 runs beside the copies of step t
constexpr uint32_t FUSED_MAX_TILE = 12288;  // fused path: agents per CTA held in shared memory
constexpr uint32_t FUSED_OVF_CAP = 256;     // fused fast lists: agents in multi-valued level-1 buckets
constexpr uint32_t BIG_OVF_CAP = 4096;      // ... in the streaming kernel of large contexts (sorted, not counted)
constexpr uint32_t FUSED_MAX_WORLD = 8;     // ranks of one world planned in one launch (SCALESIM_F_LOOPBACK)

// status bits (mirror include/scalesim.h)
constexpr uint32_t ST_INSUFFICIENT = 1u, ST_BAD_RECORD = 2u, ST_BAD_KIN = 4u, ST_NO_PAGES = 8u, ST_SYNC = 16u,
                   ST_LIMIT = 32u;

// header fields (mirror SCALESIM_H_*)
enum { H_N_PF = 0, H_N_EV, H_H2D, H_D2H, H_CUT_BITS, H_CUT_REM, H_STATUS, H_N_D2H, H_N_H2D,
       H_KEPT, H_N_ELIG, H_POOL_HEAD, H_POOL_TAIL, H_SEQ, H_FIELDS = 16 };

// Device-side selection state of one plan (radix select of the boundary distance).
struct SelState {
  unsigned long long below;      // bytes of eligible agents with key < prefix range (global)
  unsigned long long rem;        // B - bytes(d < D*)
  unsigned long long total;      // total eligible bytes (global)
  unsigned long long tie_local;  // this rank's bytes at d == D*
  unsigned long long tie_kept;   // this rank's kept bytes at d == D*
  unsigned long long zero_bytes; // bytes of d == 0 agents (global after exchange)
  unsigned int prefix;           // distance bits fixed so far
  unsigned int level;            // next histogram level to build (1..3), 4 = resolved
  unsigned int done;             // D* resolved
  unsigned int all_fit;          // every eligible agent fits
  unsigned int dstar;            // boundary distance bits
  unsigned int status;           // SCALESIM_ST_* of this plan
  unsigned int int_count;        // interaction participants
  unsigned int sort_or[2], sort_and[2];  // varying-bit analysis of the two lists
  unsigned int pad[3];
};

// a1' spatial grid header (workspace, interaction.cu).  The bounding-box / speed accumulators
// are filled by k_int_compact with atomics and reset by k_grid_setup for the next step.
struct GridHdr {
  double xmin, ymin, h, vmax;
  uint32_t ncx, ncy, count, n_heavy;
  int32_t acc_x0, acc_y0, acc_x1, acc_y1;  // order-preserving integer keys of the coordinates
  uint32_t acc_vmax;                        // float bits of the largest speed (non-negative)
  uint32_t pad[3];
};

// Workspace carve-up (byte offsets from the workspace base, 256-B aligned).
struct Layout {
  uint64_t n_local, n_words, n_kin, n_tiles, n_blocks, n_block_pages, n_dev_pages, desc_cap, world;
  uint64_t max_sort_chunks, max_exp_chunks;
  uint64_t keys, elig, bm[2], dint, ilist_kin, ilist_idx, ilist_dact, grid_hdr, heavy, cell_cnt, cell_start, g_cell, g_kin, g_ent;
  uint64_t hist1, mm1, hist2, mm2, hist3, state, header, gather;
  uint64_t tile_tie, tile_tie_excl, tile_pf, tile_ev, tile_pf_excl, tile_ev_excl, tile_h2d, tile_tiekept, tile_elig;
  uint64_t pf_ids, ev_ids, sort_ka, sort_va, sort_kb, sort_vb, sort_cnt, pfa_key, pfa_val;
  uint64_t exp_sum, exp_excl;
  uint64_t page_first, page_table, ring, pool, desc[2];
  // fused path (double-buffered by fused-step parity where noted)
  uint64_t f_hist1, f_mm1, f_hist2, f_mm2, f_hist3, f_cta_cpf, f_cta_cev, f_tot, f_acc;
  uint64_t f_rows1, f_rows2, f_rows3, f_cta_lmm;
  uint64_t f_sk2, f_sv2, f_sk3, f_sv3, f_bar, f_prof, wb_bytes, params_dev;
  uint64_t f_pos, f_rt, f_crow, f_ovf, big_codes;
  // world > 1 on one device (SCALESIM_F_LOOPBACK): the gathered interaction participants of the
  // world, and (SCALESIM_F_TP_SLICED) the world's merged lists and their transfer header
  uint64_t wkin, wcnt, tp_pf, tp_ev, tp_dirty, tp_hdr, tp_kpf, tp_kev, xscratch;
  uint64_t total;
};

// n_tab: agents the block tables cover (n_local, or n_agents when TP-sliced); n_wkin: capacity of
// the world's gathered interaction list (0 unless a loopback world has interaction agents)
Layout make_layout(uint64_t n_local, uint64_t n_kin, uint64_t n_blocks, uint64_t n_block_pages,
                   uint64_t n_dev_pages, uint64_t world, bool transfer, uint64_t n_tab = 0, uint64_t n_wkin = 0,
                   bool tp = false);

// Pointers derived from the layout.
struct Dev {
  uint8_t *base;
  uint32_t *keys, *elig, *bm[2];
  float *dint;
  float4 *ilist_kin;
  uint32_t *ilist_idx;
  float *ilist_dact;                 // D_action of each participant (a1' pruning bound)
  uint8_t *grid_hdr;                 // a1' grid: GridHdr
  uint32_t *heavy;                   // [n_kin] participants whose search continues warp-wide
  uint32_t *cell_cnt, *cell_start;   // [GRID_MAX_SIDE^2 (+1)]
  uint32_t *g_cell, *g_ent;          // [n_kin] cell of each participant; participant of each sorted slot
  float4 *g_kin;                     // [n_kin] kinematics in cell order
  unsigned long long *hist1, *hist2, *hist3;
  uint32_t *mm1, *mm2;  // [0, 2^w) min of bits, [2^w, 2^(w+1)) min of ~bits (= ~max)
  SelState *state;
  unsigned long long *header, *gather;
  unsigned long long *tile_tie, *tile_tie_excl, *tile_h2d, *tile_tiekept;
  uint32_t *tile_pf, *tile_ev, *tile_pf_excl, *tile_ev_excl, *tile_elig;
  uint32_t *pf_ids, *ev_ids;
  uint32_t *sort_ka, *sort_va, *sort_kb, *sort_vb, *sort_cnt, *pfa_key, *pfa_val;
  unsigned long long *exp_sum, *exp_excl;
  unsigned long long *page_first;
  uint32_t *page_table, *ring;
  unsigned long long *pool;  // [0] head, [1] tail
  unsigned long long *desc[2];  // each: d2h [desc_cap pairs] then h2d [desc_cap pairs]
  // fused path (parity = launch number & 1)
  unsigned long long *f_hist1;  // [2][4096] level-1 byte histogram, then [2][64] coarse sums
  uint32_t *f_mm1;              // [2][2][4096] per-bucket min key, min complemented key
  unsigned long long *f_hist2;  // [2][1024]
  uint32_t *f_mm2;              // [2][2][1024]
  unsigned long long *f_hist3;  // [2][1024]
  uint32_t *f_cta_cpf, *f_cta_cev;                      // [CTAS][1024] (offset << 16) | count of the CTA's
                                                        // list members per bucket (staged bucket-major)
  uint32_t *f_tot;                                      // [2][2][1024] list bucket totals
  unsigned long long *f_acc;                            // [2][8]
  unsigned long long *f_rows1, *f_rows2, *f_rows3;      // [CTAS][4096] / [CTAS][1024] per-CTA histogram rows
  uint32_t *f_cta_lmm;                                  // [CTAS][2 lists][3][1024] the CTA's list members per
                                                        // bucket: min key, ~max key, OR of key bits [20:0]
                                                        // (valid where the row count is nonzero)
  uint32_t *wb_bytes;                                   // [n_local] KV+HIST bytes per agent (R13)
  uint8_t *params_dev;                                  // device copy of the context's Params (fused path)
  uint32_t *f_sk2, *f_sv2, *f_sk3, *f_sv3;              // [n_local] evict-segment sort scratch
  unsigned int *f_bar;                                  // [2] grid-barrier counters
  unsigned long long *f_prof;                           // [16] globaltimer stamps of the last fused launch
  // fused fast list placement (integer-distance contexts):
  uint32_t *f_crow;            // [2][G][4096] per-CTA eligible counts per level-1 bucket (non-resident | resident << 16)
  unsigned long long *f_pos;   // [2][4096][FUSED_MAX_CTAS] bucket owners' list offsets per (bucket, CTA), epoch-tagged
  unsigned long long *f_rt;    // [2][FUSED_MAX_CTAS] bucket owners' range totals, epoch-tagged
  uint4 *f_ovf;                // [2][BIG_OVF_CAP] eligible agents in multi-valued buckets: {key, id, resident, 0}
  uint16_t *big_codes;         // [n_words * 32] large contexts (fused_big.cu): bucket | eligible << 12 | dirty << 13 per agent (lanes of a word permuted)
  // loopback worlds
  float4 *wkin;                // [n_agents] the world's interaction participants, rank-major (kin all-gather)
  uint32_t *wcnt;              // [FUSED_MAX_WORLD + 1] rank offsets into wkin, then the world's count
  uint32_t *tp_pf, *tp_ev;     // [n_agents] the world's merged lists (TP-sliced transfers)
  uint8_t *tp_dirty;           // [n_agents] dirty bit of each merged evict entry
  unsigned long long *tp_hdr;  // [H_FIELDS] list counts and transfer fields of the merged plan
  uint32_t *tp_kpf, *tp_kev;   // [n_local] distance bits of this rank's list entries (merge keys)
  uint8_t *xscratch;           // [32 KB] result of a thread-exchange collective before it lands
};

Dev make_dev(void *ws, const Layout &L);

struct Params {
  // sizes
  uint64_t n_local, n_words, n_kin, n_tiles, shard_begin, budget, page_bytes, n_dev_pages, desc_cap;
  uint64_t n_agents;
  // a6 page slots: slot_bytes per device page slot, slice_off = this rank's byte offset within a
  // page (TP-sliced: page_bytes / world and rank * slot_bytes; otherwise page_bytes and 0)
  uint64_t slot_bytes, slice_off;
  const uint8_t *ev_dirty;  // expansion of merged lists: dirty bit per evict entry (else from rec)
  float theta[3];
  float hop_scale;
  int rank, world;
  // inputs
  const uint4 *rec;
  const float4 *kin;
  const unsigned long long *blk_ptr;
  const uint32_t *blk_size;
  const unsigned long long *blk_host_off;
  const uint8_t *blk_kind;
  uint8_t *host_arena, *dev_arena;
  // state
  int keep_dist;  // fused path: also write the distances to the workspace (dist view)
  int int_mode;   // every distance is an integer or +inf (no interaction class, integral hop_scale)
  int explicit_dist;  // SCALESIM_F_EXPLICIT_DIST: record word 0 holds the distance bits (R19)
  int loopback;       // SCALESIM_F_LOOPBACK: a rank of a world planned in one launch (step_group)
  int tp;             // SCALESIM_F_TP_SLICED: every rank holds slice `rank` of every resident page
  int cur;  // index of the residency bitmap holding the residency before this plan
  int desc_buf;
  Dev d;
};

// Launchers (kernels.cu).  Each returns the number of kernels it enqueued.
int launch_plan_init(const Params &p, cudaStream_t s);
int launch_score(const Params &p, int64_t now, float *dist_out, cudaStream_t s, int grid);
int launch_interaction(const Params &p, int64_t now, cudaStream_t s, int grid);
int launch_grid_pairmin(const Params &p, cudaStream_t s, int grid);
int launch_select(const Params &p, int level, cudaStream_t s);
int launch_hist(const Params &p, int level, cudaStream_t s, int grid);
int launch_tie(const Params &p, cudaStream_t s);
int launch_emit(const Params &p, cudaStream_t s);
int launch_lists(const Params &p, cudaStream_t s);
int launch_expand(const Params &p, cudaStream_t s);
int launch_transfer(const Params &p, cudaStream_t s, int ctas);
int launch_transfer_split(const Params &p, cudaStream_t s, cudaStream_t s2, int ctas);
int launch_init_pages(const Params &p, const uint32_t *resident_init, cudaStream_t s);
int launch_copy_dist(const Params &p, float *dist_out, cudaStream_t s);
// loopback worlds (kernels.cu): ps[r] = rank r's (host) parameters; the world kernels read the
// ranks' static fields from their device copies (d.params_dev) and the per-step inputs from ps
int launch_world_interaction(const Params *const *ps, uint32_t G, int64_t now, cudaStream_t s);
int launch_tp_merge(const Params *const *ps, uint32_t G, int64_t now, cudaStream_t s);
int launch_tp_finish(const Params &rank_p, cudaStream_t s);
// collectives between same-device ranks driven by host threads (SCALESIM_F_THREADS)
int launch_xreduce(void *out, const void *const *ins, uint32_t G, uint64_t n, int kind, cudaStream_t s);
int launch_xgather(unsigned long long *out, const void *const *ins, uint32_t G, cudaStream_t s);
bool fused_supported(const Params &p, int grid, uint32_t *tile_out);
// one instance of a fused launch (see fused.cu)
struct FusedInst {
  const Params *params;  // device copy of the context's Params (static fields)
  const uint4 *rec;
  const float4 *kin;
  int64_t now;
  uint64_t n_local;  // agents of the instance (the kernel prefetches its records before reading params)
  const uint32_t *bm_old;  // residency bitmap before this plan (prefetched likewise)
  uint32_t cur, parity, epoch, tile;
};
constexpr int FUSED_MAX_BATCH = 160;
int launch_fused_batch(const FusedInst *insts, uint32_t n, uint32_t gsize, cudaStream_t s, bool coop,
                       uint32_t wsize = 1);
bool fused_prepare(int grid, uint32_t tile, uint32_t gsize);
// large integer-distance contexts (fused_big.cu): tiles beyond shared memory, up to 2^19 per CTA
constexpr uint32_t FUSED_BIG_MAX_TILE = 1u << 19;
bool fused_big_prepare(uint32_t gsize);
int launch_fused_big(const FusedInst &inst, uint32_t gsize, cudaStream_t s, bool coop);
size_t fused_smem_bytes(uint32_t tile);
int launch_readback(const unsigned long long *hdr, const uint32_t *pf, const uint32_t *ev, unsigned long long *out_hdr,
                    uint32_t *out_pf, uint32_t *out_ev, unsigned long long *done_word, unsigned long long seq,
                    unsigned int *tickets, cudaStream_t s);
int launch_apply_updates(uint4 *rec, const uint32_t *ids, const uint4 *upd, uint32_t n, uint64_t shard_begin,
                         uint64_t n_local, uint32_t *err, cudaStream_t s);

}  // namespace ss

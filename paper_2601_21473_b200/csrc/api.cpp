// api.cpp — the C ABI of include/scalesim.h: validation, workspace carve-up, the step
// sequence of launches (kernels.cu), and the NCCL exchange of the global cut (world > 1).
#include "../../include/scalesim.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "internal.h"

namespace ss {

static uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

Layout make_layout(uint64_t n_local, uint64_t n_kin, uint64_t n_blocks, uint64_t n_block_pages,
                   uint64_t n_dev_pages, uint64_t world, bool transfer, uint64_t n_tab, uint64_t n_wkin, bool tp) {
  if (n_tab < n_local) n_tab = n_local;
  Layout L = {};
  L.n_local = n_local;
  L.n_words = (n_local + 31) / 32;
  L.n_kin = n_kin;
  L.n_tiles = (n_local + TILE - 1) / TILE;
  L.n_blocks = n_blocks;
  L.n_block_pages = transfer ? n_block_pages : 0;
  L.n_dev_pages = transfer ? n_dev_pages : 0;
  L.desc_cap = transfer ? (n_block_pages < n_dev_pages ? n_block_pages : n_dev_pages) : 0;
  L.world = world;
  L.max_sort_chunks = (n_local + SORT_CH - 1) / SORT_CH + 1;
  L.max_exp_chunks = ((tp ? n_tab : n_local) + EXP_CH - 1) / EXP_CH + 1;  // (TP: the merged lists)
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) {
    uint64_t o = off;
    off = align_up(off + (bytes ? bytes : 1), 256);
    return o;
  };
  const uint64_t n1 = n_local ? n_local : 1, w1 = L.n_words ? L.n_words : 1, k1 = n_kin ? n_kin : 1;
  const uint64_t t1 = L.n_tiles ? L.n_tiles : 1;
  L.keys = take(4 * n1);
  L.elig = take(4 * (w1 + 1));
  L.bm[0] = take(4 * (w1 + 1));
  L.bm[1] = take(4 * (w1 + 1));
  L.dint = take(4 * k1);
  L.ilist_kin = take(16 * k1);
  L.ilist_idx = take(4 * k1);
  L.ilist_dact = take(4 * k1);
  L.grid_hdr = take(sizeof(GridHdr));
  L.heavy = take(4 * k1);
  L.cell_cnt = take(4 * (n_kin ? (uint64_t)GRID_MAX_SIDE * GRID_MAX_SIDE : 1));
  L.cell_start = take(4 * (n_kin ? (uint64_t)GRID_MAX_SIDE * GRID_MAX_SIDE + 1 : 1));
  L.g_cell = take(4 * k1);
  L.g_kin = take(16 * k1);
  L.g_ent = take(4 * k1);
  L.hist1 = take(8 * 4096);
  L.mm1 = take(4 * 4096);
  L.hist2 = take(8 * 1024);
  L.mm2 = take(4 * 2048);
  L.hist3 = take(8 * 1024);
  L.state = take(sizeof(SelState));
  L.header = take(8 * H_FIELDS);
  L.gather = take(8 * (world + 8));
  L.tile_tie = take(8 * t1);
  L.tile_tie_excl = take(8 * t1);
  L.tile_pf = take(4 * t1);
  L.tile_ev = take(4 * t1);
  L.tile_pf_excl = take(4 * t1);
  L.tile_ev_excl = take(4 * t1);
  L.tile_h2d = take(8 * t1);
  L.tile_tiekept = take(8 * t1);
  L.tile_elig = take(4 * t1);
  L.pf_ids = take(4 * n1);
  L.ev_ids = take(4 * n1);
  L.sort_ka = take(4 * n1);
  L.sort_va = take(4 * n1);
  L.sort_kb = take(4 * n1);
  L.sort_vb = take(4 * n1);
  L.pfa_key = take(4 * n1);
  L.pfa_val = take(4 * n1);
  L.sort_cnt = take(4 * 2048 * L.max_sort_chunks);
  L.exp_sum = take(8 * 4 * L.max_exp_chunks);
  L.exp_excl = take(8 * 4 * L.max_exp_chunks);
  L.page_first = take(8 * (n_blocks + 1));
  L.page_table = take(4 * (L.n_block_pages ? L.n_block_pages : 1));
  L.ring = take(4 * (L.n_dev_pages ? L.n_dev_pages : 1));
  L.pool = take(16);
  L.desc[0] = take(8 * DESC_HDR + 32 * (L.desc_cap ? L.desc_cap : 1));
  L.desc[1] = take(8 * DESC_HDR + 32 * (L.desc_cap ? L.desc_cap : 1));
  L.f_hist1 = take(8 * 2 * (4096 + 64));  // + [2][64] coarse sums
  L.f_mm1 = take(4 * 2 * 2 * 4096);
  L.f_hist2 = take(8 * 2 * 1024);
  L.f_mm2 = take(4 * 2 * 2 * 1024);
  L.f_hist3 = take(8 * 2 * 1024);
  L.f_cta_cpf = take(4 * (uint64_t)FUSED_MAX_CTAS * 1024);
  L.f_cta_cev = take(4 * (uint64_t)FUSED_MAX_CTAS * 1024);
  L.f_tot = take(4 * 2 * 2 * 1024);
  L.f_acc = take(8 * 2 * 8);
  L.f_rows1 = take(8 * (uint64_t)FUSED_MAX_CTAS * 4096);
  L.f_rows2 = take(8 * (uint64_t)FUSED_MAX_CTAS * 1024);
  L.f_rows3 = take(8 * (uint64_t)FUSED_MAX_CTAS * 1024);
  L.f_cta_lmm = take(4 * (uint64_t)FUSED_MAX_CTAS * 6 * 1024);
  L.wb_bytes = take(4 * n1);
  L.params_dev = take(sizeof(Params));
  L.f_sk2 = take(4 * n1);
  L.f_sv2 = take(4 * n1);
  L.f_sk3 = take(4 * n1);
  L.f_sv3 = take(4 * n1);
  L.f_bar = take(64);
  L.f_prof = take(512);
  L.f_pos = take(8 * 2 * 4096 * (uint64_t)FUSED_MAX_CTAS);
  L.f_rt = take(8 * 2 * (uint64_t)FUSED_MAX_CTAS);
  L.f_crow = take(4 * 2 * 4096 * (uint64_t)FUSED_MAX_CTAS);
  L.f_ovf = take(16 * 2 * (uint64_t)BIG_OVF_CAP);
  L.big_codes = take(2 * 32 * ((n1 + 31) / 32) + 64);  // (whole words; the stash copies 16-byte units)
  L.wkin = take(16 * (n_wkin ? n_wkin : 1));
  L.wcnt = take(4 * (FUSED_MAX_WORLD + 1));
  const uint64_t tn = tp ? n_tab : 1, tl = tp ? n1 : 1;
  L.tp_pf = take(4 * tn);
  L.tp_ev = take(4 * tn);
  L.tp_dirty = take(tn);
  L.tp_hdr = take(8 * H_FIELDS);
  L.tp_kpf = take(4 * tl);
  L.tp_kev = take(4 * tl);
  L.xscratch = take(world > 1 ? 32768 : 1);
  L.total = off;
  return L;
}

Dev make_dev(void *ws, const Layout &L) {
  Dev d = {};
  uint8_t *b = static_cast<uint8_t *>(ws);
  d.base = b;
  d.keys = (uint32_t *)(b + L.keys);
  d.elig = (uint32_t *)(b + L.elig);
  d.bm[0] = (uint32_t *)(b + L.bm[0]);
  d.bm[1] = (uint32_t *)(b + L.bm[1]);
  d.dint = (float *)(b + L.dint);
  d.ilist_kin = (float4 *)(b + L.ilist_kin);
  d.ilist_idx = (uint32_t *)(b + L.ilist_idx);
  d.ilist_dact = (float *)(b + L.ilist_dact);
  d.grid_hdr = (uint8_t *)(b + L.grid_hdr);
  d.heavy = (uint32_t *)(b + L.heavy);
  d.cell_cnt = (uint32_t *)(b + L.cell_cnt);
  d.cell_start = (uint32_t *)(b + L.cell_start);
  d.g_cell = (uint32_t *)(b + L.g_cell);
  d.g_kin = (float4 *)(b + L.g_kin);
  d.g_ent = (uint32_t *)(b + L.g_ent);
  d.hist1 = (unsigned long long *)(b + L.hist1);
  d.mm1 = (uint32_t *)(b + L.mm1);
  d.hist2 = (unsigned long long *)(b + L.hist2);
  d.mm2 = (uint32_t *)(b + L.mm2);
  d.hist3 = (unsigned long long *)(b + L.hist3);
  d.state = (SelState *)(b + L.state);
  d.header = (unsigned long long *)(b + L.header);
  d.gather = (unsigned long long *)(b + L.gather);
  d.tile_tie = (unsigned long long *)(b + L.tile_tie);
  d.tile_tie_excl = (unsigned long long *)(b + L.tile_tie_excl);
  d.tile_pf = (uint32_t *)(b + L.tile_pf);
  d.tile_ev = (uint32_t *)(b + L.tile_ev);
  d.tile_pf_excl = (uint32_t *)(b + L.tile_pf_excl);
  d.tile_ev_excl = (uint32_t *)(b + L.tile_ev_excl);
  d.tile_h2d = (unsigned long long *)(b + L.tile_h2d);
  d.tile_tiekept = (unsigned long long *)(b + L.tile_tiekept);
  d.tile_elig = (uint32_t *)(b + L.tile_elig);
  d.pf_ids = (uint32_t *)(b + L.pf_ids);
  d.ev_ids = (uint32_t *)(b + L.ev_ids);
  d.sort_ka = (uint32_t *)(b + L.sort_ka);
  d.sort_va = (uint32_t *)(b + L.sort_va);
  d.sort_kb = (uint32_t *)(b + L.sort_kb);
  d.sort_vb = (uint32_t *)(b + L.sort_vb);
  d.pfa_key = (uint32_t *)(b + L.pfa_key);
  d.pfa_val = (uint32_t *)(b + L.pfa_val);
  d.sort_cnt = (uint32_t *)(b + L.sort_cnt);
  d.exp_sum = (unsigned long long *)(b + L.exp_sum);
  d.exp_excl = (unsigned long long *)(b + L.exp_excl);
  d.page_first = (unsigned long long *)(b + L.page_first);
  d.page_table = (uint32_t *)(b + L.page_table);
  d.ring = (uint32_t *)(b + L.ring);
  d.pool = (unsigned long long *)(b + L.pool);
  d.desc[0] = (unsigned long long *)(b + L.desc[0]);
  d.desc[1] = (unsigned long long *)(b + L.desc[1]);
  d.f_hist1 = (unsigned long long *)(b + L.f_hist1);
  d.f_mm1 = (uint32_t *)(b + L.f_mm1);
  d.f_hist2 = (unsigned long long *)(b + L.f_hist2);
  d.f_mm2 = (uint32_t *)(b + L.f_mm2);
  d.f_hist3 = (unsigned long long *)(b + L.f_hist3);
  d.f_cta_cpf = (uint32_t *)(b + L.f_cta_cpf);
  d.f_cta_cev = (uint32_t *)(b + L.f_cta_cev);
  d.f_tot = (uint32_t *)(b + L.f_tot);
  d.f_acc = (unsigned long long *)(b + L.f_acc);
  d.f_rows1 = (unsigned long long *)(b + L.f_rows1);
  d.f_rows2 = (unsigned long long *)(b + L.f_rows2);
  d.f_rows3 = (unsigned long long *)(b + L.f_rows3);
  d.f_cta_lmm = (uint32_t *)(b + L.f_cta_lmm);
  d.wb_bytes = (uint32_t *)(b + L.wb_bytes);
  d.params_dev = (uint8_t *)(b + L.params_dev);
  d.f_sk2 = (uint32_t *)(b + L.f_sk2);
  d.f_sv2 = (uint32_t *)(b + L.f_sv2);
  d.f_sk3 = (uint32_t *)(b + L.f_sk3);
  d.f_sv3 = (uint32_t *)(b + L.f_sv3);
  d.f_bar = (unsigned int *)(b + L.f_bar);
  d.f_prof = (unsigned long long *)(b + L.f_prof);
  d.f_pos = (unsigned long long *)(b + L.f_pos);
  d.f_rt = (unsigned long long *)(b + L.f_rt);
  d.f_crow = (uint32_t *)(b + L.f_crow);
  d.f_ovf = (uint4 *)(b + L.f_ovf);
  d.big_codes = (uint16_t *)(b + L.big_codes);
  d.wkin = (float4 *)(b + L.wkin);
  d.wcnt = (uint32_t *)(b + L.wcnt);
  d.tp_pf = (uint32_t *)(b + L.tp_pf);
  d.tp_ev = (uint32_t *)(b + L.tp_ev);
  d.tp_dirty = (uint8_t *)(b + L.tp_dirty);
  d.tp_hdr = (unsigned long long *)(b + L.tp_hdr);
  d.tp_kpf = (uint32_t *)(b + L.tp_kpf);
  d.tp_kev = (uint32_t *)(b + L.tp_kev);
  d.xscratch = (uint8_t *)(b + L.xscratch);
  return d;
}

void launch_init_page_table(const Params &p, uint64_t n_block_pages, const uint32_t *res, uint64_t *cnt_dev,
                            cudaStream_t s);
int launch_fix_kept(const Params &p, cudaStream_t s);
int launch_mask_tail(const Params &p, cudaStream_t s);

// ---- NCCL, loaded lazily so the library has no link-time NCCL dependency ----
struct Nccl {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  bool load() {
    if (h) return true;
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
    CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
    AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
    AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
    return GetUniqueId && CommInitRank && CommDestroy && AllReduce && AllGather;
  }
};
static Nccl g_nccl;

// ---- SCALESIM_F_THREADS: the world > 1 collectives between ranks on one device, each rank
// driven by its own host thread (the exchange the NCCL calls perform, through device memory;
// DESIGN §8).  A group = the contexts created with the same 128-byte id.  Each collective:
// every rank records its input's readiness and publishes the pointer (host barrier); every rank
// waits for all inputs on its stream and reduces them into its scratch (host barrier: every
// wait is enqueued before any input is reused); the result lands in the rank's buffer.
struct ThreadGroup {
  int world = 0, joined = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  uint64_t shard[FUSED_MAX_WORLD][2] = {};  // the ranks' id ranges (checked at the first collective)
  const void *in[FUSED_MAX_WORLD] = {};
  cudaEvent_t ev_in[FUSED_MAX_WORLD] = {}, ev_red[FUSED_MAX_WORLD] = {};
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
static std::mutex g_groups_mu;
static std::vector<std::pair<std::vector<uint8_t>, ThreadGroup *>> g_groups;

static ThreadGroup *join_group(const void *id, int world) {
  std::vector<uint8_t> key(static_cast<const uint8_t *>(id), static_cast<const uint8_t *>(id) + 128);
  std::lock_guard<std::mutex> lk(g_groups_mu);
  for (auto &e : g_groups)
    if (e.first == key) {
      if (e.second->world != world) return nullptr;
      e.second->joined++;
      return e.second;
    }
  ThreadGroup *g = new (std::nothrow) ThreadGroup();
  if (!g) return nullptr;
  g->world = world;
  g->joined = 1;
  g_groups.emplace_back(key, g);
  return g;
}

static void leave_group(ThreadGroup *g) {
  std::lock_guard<std::mutex> lk(g_groups_mu);
  if (--g->joined > 0) return;
  for (size_t i = 0; i < g_groups.size(); ++i)
    if (g_groups[i].second == g) {
      g_groups.erase(g_groups.begin() + (long)i);
      break;
    }
  delete g;
}

// SCALESIM_F_EXCLUSIVE: the single-kernel plans of the exclusive contexts of a device run one
// after another (their grid barriers need every SM): the last launch's stream and event per
// device, and the number of such contexts (with one, nothing is recorded: consecutive launches
// on its stream stay directly linked for the programmatic launch overlap).
struct ExclusiveChain {
  cudaStream_t stream = nullptr;
  cudaEvent_t event = nullptr;
  int contexts = 0;
};
static std::mutex g_excl_mu;
static ExclusiveChain g_excl[64];

}  // namespace ss

using namespace ss;

// staging / read-back slots of the host entry points: host steps in flight
constexpr int NSLOT = 3;

struct scalesim_ctx {
  scalesim_config cfg;
  scalesim_tables tab;
  Layout L;
  Params p;
  cudaStream_t stream = nullptr, copy_stream = nullptr;
  cudaEvent_t ev_plan = nullptr, ev_xfer[2] = {nullptr, nullptr}, ev_side = nullptr;
  cudaStream_t copy_stream2 = nullptr;  // library-owned: loads that do not wait for write-backs
  bool transfer = false;
  int grid = 592;
  int copy_ctas = 64;
  uint64_t step = 0;        // plans made
  bool scored = false, planned = false, transferred = true;
  uint64_t launches = 0;
  ncclComm_t comm = nullptr;
  ThreadGroup *tgroup = nullptr;  // SCALESIM_F_THREADS
  cudaEvent_t ev_xin = nullptr, ev_xred = nullptr;
  int last_buf = 0;
  bool xfer_pending = false;
  bool xfer_recorded[2] = {false, false};  // ev_xfer[b] has been recorded at least once
  bool exclusive = false;                  // SCALESIM_F_EXCLUSIVE
  bool big = false;                        // large context: the streaming single-kernel plan
  cudaEvent_t ev_fused = nullptr;          // after this context's last single-kernel plan
  // fused single-kernel plan (world == 1)
  bool fused = false;
  uint32_t fused_tile = 0;
  int fused_grid = 0;
  uint64_t fused_steps = 0;
  bool deferred = false;  // score deferred into the fused plan kernel
  bool last_fused = false;
  int sms = 148;
  int64_t deferred_now = 0;
  // pipelined host inputs (scalesim_stage_host): two library-owned device buffers, each the
  // records (16 n_local B) followed by the kinematics (16 n_kin B), filled on in_stream
  cudaStream_t in_stream = nullptr;
  uint8_t *sbuf[NSLOT] = {};
  cudaEvent_t ev_in[NSLOT] = {}, ev_used[NSLOT] = {};
  const void *staged_rec[NSLOT] = {}, *staged_kin[NSLOT] = {};
  bool staged[NSLOT] = {}, sbuf_used[NSLOT] = {};
  bool staged_upd[NSLOT] = {};  // the slot holds (ids, records) updates, not whole inputs
  uint32_t staged_n[NSLOT] = {};
  int stage_next = 0;
  uint32_t *upd_err_h = nullptr, *upd_err_d = nullptr;  // host-mapped count of out-of-shard ids
  // host read-back (read_back): host-mapped pinned [done word | header | prefetch | evict]
  uint8_t *rb_h = nullptr, *rb_d = nullptr;
  unsigned int *rb_tickets = nullptr;
  unsigned long long rb_seq = 0;          // read-backs enqueued (slot = seq % 2)
  unsigned long long rb_pending[NSLOT] = {};  // submitted steps not yet collected, oldest first
  int n_pending = 0;
};

static scalesim_status cuda_status(cudaError_t e) { return e == cudaSuccess ? SCALESIM_OK : SCALESIM_E_CUDA; }

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t _e = (x);                                                           \
    if (_e != cudaSuccess) {                                                        \
      if (getenv("SCALESIM_VERBOSE")) fprintf(stderr, "scalesim: %s: %s\n", #x, cudaGetErrorString(_e)); \
      return SCALESIM_E_CUDA;                                                       \
    }                                                                               \
  } while (0)

#define NK(x)                                  \
  do {                                         \
    if ((x) != ncclSuccess) return SCALESIM_E_NCCL; \
  } while (0)

static bool aligned(const void *p, uint64_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

static scalesim_status validate_config(const scalesim_config *c) {
  if (!c || c->abi_version != SCALESIM_ABI_VERSION) return SCALESIM_E_INVALID;
  if (c->shard_begin > c->shard_end || c->shard_end > c->n_agents) return SCALESIM_E_INVALID;
  if (c->n_agents > 0xFFFFFFFFull) return SCALESIM_E_INVALID;  // ids are uint32
  if (c->world < 1 || c->rank < 0 || c->rank >= c->world) return SCALESIM_E_INVALID;
  if (c->world == 1 && (c->shard_begin != 0 || c->shard_end != c->n_agents)) return SCALESIM_E_INVALID;
  // interaction agents at world > 1: the kinematics all-gather of a loopback world
  if (c->world > 1 && c->n_kin > 0 && !(c->flags & SCALESIM_F_LOOPBACK)) return SCALESIM_E_INVALID;
  if ((c->flags & SCALESIM_F_LOOPBACK) && (c->world < 2 || c->world > (int)FUSED_MAX_WORLD)) return SCALESIM_E_INVALID;
  if ((c->flags & SCALESIM_F_THREADS) &&
      (c->world < 2 || c->world > (int)FUSED_MAX_WORLD || (c->flags & SCALESIM_F_LOOPBACK) || !c->nccl_unique_id))
    return SCALESIM_E_INVALID;
  if ((c->flags & SCALESIM_F_TP_SLICED) &&
      (!(c->flags & SCALESIM_F_LOOPBACK) || (c->flags & SCALESIM_F_NO_TRANSFER) || c->page_bytes % (16ull * c->world) != 0))
    return SCALESIM_E_INVALID;
  if ((c->flags & SCALESIM_F_EXPLICIT_DIST) && c->n_kin > 0) return SCALESIM_E_INVALID;
  if (c->flags & ~(uint32_t)(SCALESIM_F_NO_TRANSFER | SCALESIM_F_KEEP_DIST | SCALESIM_F_MULTI_KERNEL |
                             SCALESIM_F_EXPLICIT_DIST | SCALESIM_F_EXCLUSIVE | SCALESIM_F_LOOPBACK |
                             SCALESIM_F_TP_SLICED | SCALESIM_F_THREADS))
    return SCALESIM_E_INVALID;
  for (int k = 0; k < 3; ++k)
    if (std::isnan(c->theta[k]) || c->theta[k] < 0.0f) return SCALESIM_E_INVALID;
  if (!(c->hop_scale > 0.0f) || std::isinf(c->hop_scale)) return SCALESIM_E_INVALID;
  if (!(c->flags & SCALESIM_F_NO_TRANSFER)) {
    if (c->page_bytes == 0 || c->page_bytes % 4096 != 0) return SCALESIM_E_INVALID;
  }
  return SCALESIM_OK;
}

// the context's layout: block tables over the shard (or, TP-sliced, over every agent), device
// page slots of page_bytes (TP-sliced: page_bytes / world, every rank holding one slice)
static Layout layout_of(const scalesim_config *cfg, const scalesim_tables *t) {
  const bool transfer = !(cfg->flags & SCALESIM_F_NO_TRANSFER), tp = (cfg->flags & SCALESIM_F_TP_SLICED) != 0;
  const uint64_t n_local = cfg->shard_end - cfg->shard_begin;
  const uint64_t slot = tp ? cfg->page_bytes / cfg->world : cfg->page_bytes;
  const uint64_t n_dev_pages = transfer ? t->dev_bytes / slot : 0;
  const uint64_t n_wkin = (cfg->world > 1 && cfg->n_kin > 0) ? cfg->n_agents : 0;
  return make_layout(n_local, cfg->n_kin, t->n_blocks, t->n_block_pages, n_dev_pages, cfg->world, transfer,
                     tp ? cfg->n_agents : n_local, n_wkin, tp);
}

extern "C" uint64_t scalesim_workspace_bytes(const scalesim_config *cfg, const scalesim_tables *t) {
  if (validate_config(cfg) != SCALESIM_OK || !t) return 0;
  return layout_of(cfg, t).total;
}

extern "C" const char *scalesim_strerror(scalesim_status s) {
  switch (s) {
    case SCALESIM_OK: return "ok";
    case SCALESIM_E_INVALID: return "invalid argument";
    case SCALESIM_E_INSUFFICIENT: return "insufficient memory: active agents exceed the budget";
    case SCALESIM_E_NOT_RESTORABLE: return "block not restorable (no host backing)";
    case SCALESIM_E_ORDER: return "calls out of order";
    case SCALESIM_E_CUDA: return "CUDA error";
    case SCALESIM_E_NCCL: return "NCCL error";
    case SCALESIM_E_INVARIANT: return "invariant violation";
    case SCALESIM_E_BAD_INPUT: return "malformed agent record or kinematics";
  }
  return "unknown status";
}

extern "C" scalesim_status scalesim_nccl_unique_id(void *out128) {
  if (!out128) return SCALESIM_E_INVALID;
  if (!g_nccl.load()) return SCALESIM_E_NCCL;
  ncclUniqueId id;
  NK(g_nccl.GetUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
  return SCALESIM_OK;
}

extern "C" uint64_t scalesim_launch_count(const scalesim_ctx *ctx) { return ctx ? ctx->launches : 0; }

extern "C" int scalesim_fused(const scalesim_ctx *ctx) { return ctx ? (ctx->big ? 2 : (ctx->fused ? 1 : 0)) : -1; }

extern "C" const uint64_t *scalesim_profile_stamps(const scalesim_ctx *ctx) {
  return ctx ? reinterpret_cast<const uint64_t *>(ctx->p.d.f_prof) : nullptr;
}

extern "C" scalesim_status scalesim_init(const scalesim_config *cfg, const scalesim_tables *t, scalesim_ctx **out) {
  if (!out) return SCALESIM_E_INVALID;
  *out = nullptr;
  scalesim_status st = validate_config(cfg);
  if (st != SCALESIM_OK || !t) return SCALESIM_E_INVALID;
  const bool transfer = !(cfg->flags & SCALESIM_F_NO_TRANSFER);
  const uint64_t n_local = cfg->shard_end - cfg->shard_begin;
  if (n_local > 0 && (!t->agent_rec || !aligned(t->agent_rec, 16))) return SCALESIM_E_INVALID;
  if (cfg->n_kin > 0 && (!t->agent_kin || !aligned(t->agent_kin, 16))) return SCALESIM_E_INVALID;
  if (!t->blk_ptr || (t->n_blocks > 0 && (!t->blk_size || !t->blk_kind || !t->blk_host_off))) return SCALESIM_E_INVALID;
  if (!t->workspace || !aligned(t->workspace, 256)) return SCALESIM_E_INVALID;
  const bool tp = (cfg->flags & SCALESIM_F_TP_SLICED) != 0;
  const uint64_t slot = tp ? cfg->page_bytes / cfg->world : cfg->page_bytes;
  const uint64_t n_tab = tp ? cfg->n_agents : n_local;  // agents the block tables cover
  if (tp && t->resident_init) return SCALESIM_E_INVALID;  // (TP-sliced worlds start empty)
  uint64_t n_dev_pages = 0;
  if (transfer) {
    if (!t->dev_arena || !t->host_arena) return SCALESIM_E_INVALID;
    if (!aligned(t->dev_arena, 16) || !aligned(t->host_arena, 16)) return SCALESIM_E_INVALID;
    n_dev_pages = t->dev_bytes / slot;
    const uint64_t need = (cfg->budget_bytes + cfg->page_bytes - 1) / cfg->page_bytes;
    if (n_dev_pages < need || n_dev_pages > 0xFFFFFFFFull) return SCALESIM_E_INVALID;
  }
  Layout L = layout_of(cfg, t);
  if (t->workspace_bytes < L.total) return SCALESIM_E_INVALID;

  CK(cudaSetDevice(cfg->device));
  scalesim_ctx *c = new (std::nothrow) scalesim_ctx();
  if (!c) return SCALESIM_E_INVALID;
  c->cfg = *cfg;
  c->tab = *t;
  c->L = L;
  c->transfer = transfer;
  c->stream = static_cast<cudaStream_t>(cfg->stream);
  c->copy_stream = cfg->copy_stream ? static_cast<cudaStream_t>(cfg->copy_stream) : c->stream;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device);
  c->grid = sms * 4;
  c->copy_ctas = COPY_CTAS;
  auto fail = [&](scalesim_status s) {
    scalesim_destroy(c);
    return s;
  };
  if (cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->copy_stream2, cudaStreamNonBlocking) != cudaSuccess)
    return fail(SCALESIM_E_CUDA);
  if (cudaEventCreateWithFlags(&c->ev_plan, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_xfer[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_xfer[1], cudaEventDisableTiming) != cudaSuccess)
    return fail(SCALESIM_E_CUDA);

  Params &p = c->p;
  p.n_local = n_local;
  p.n_agents = cfg->n_agents;
  p.slot_bytes = slot;
  p.slice_off = tp ? (uint64_t)cfg->rank * slot : 0;
  p.tp = tp ? 1 : 0;
  p.ev_dirty = nullptr;
  p.n_words = L.n_words;
  p.n_kin = cfg->n_kin;
  p.n_tiles = L.n_tiles;
  p.shard_begin = cfg->shard_begin;
  p.budget = cfg->budget_bytes;
  p.page_bytes = cfg->page_bytes;
  p.n_dev_pages = n_dev_pages;
  p.desc_cap = L.desc_cap;
  for (int k = 0; k < 3; ++k) p.theta[k] = cfg->theta[k];
  p.hop_scale = cfg->hop_scale;
  p.explicit_dist = (cfg->flags & SCALESIM_F_EXPLICIT_DIST) ? 1 : 0;
  p.loopback = (cfg->flags & SCALESIM_F_LOOPBACK) ? 1 : 0;
  p.int_mode = (!p.explicit_dist && cfg->n_kin == 0 && cfg->hop_scale == std::floor(cfg->hop_scale)) ? 1 : 0;
  p.rank = cfg->rank;
  p.world = cfg->world;
  p.rec = reinterpret_cast<const uint4 *>(t->agent_rec);
  p.kin = reinterpret_cast<const float4 *>(t->agent_kin);
  p.blk_ptr = reinterpret_cast<const unsigned long long *>(t->blk_ptr);
  p.blk_size = t->blk_size;
  p.blk_host_off = reinterpret_cast<const unsigned long long *>(t->blk_host_off);
  p.blk_kind = t->blk_kind;
  p.host_arena = static_cast<uint8_t *>(t->host_arena);
  p.dev_arena = static_cast<uint8_t *>(t->dev_arena);
  p.cur = 0;
  p.desc_buf = 0;
  p.keep_dist = (cfg->flags & SCALESIM_F_KEEP_DIST) ? 1 : 0;
  p.d = make_dev(t->workspace, L);

  // Host-side validation of the block table: sizes are page multiples, CSR is monotone,
  // n_block_pages matches; page_first (prefix of pages per block) goes to the workspace.
  std::vector<uint64_t> bp(n_tab + 1);
  if (cudaMemcpy(bp.data(), t->blk_ptr, 8 * (n_tab + 1), cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(SCALESIM_E_CUDA);
  if (bp[0] != 0 || bp[n_tab] != t->n_blocks) return fail(SCALESIM_E_INVALID);
  for (uint64_t a = 0; a < n_tab; ++a)
    if (bp[a + 1] < bp[a]) return fail(SCALESIM_E_INVALID);
  std::vector<uint64_t> pf(t->n_blocks + 1, 0);
  if (t->n_blocks > 0) {
    std::vector<uint32_t> bs(t->n_blocks);
    std::vector<uint8_t> bk(t->n_blocks);
    std::vector<uint64_t> bo(t->n_blocks);
    if (cudaMemcpy(bs.data(), t->blk_size, 4 * t->n_blocks, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(bk.data(), t->blk_kind, t->n_blocks, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(bo.data(), t->blk_host_off, 8 * t->n_blocks, cudaMemcpyDeviceToHost) != cudaSuccess)
      return fail(SCALESIM_E_CUDA);
    const uint64_t pb = transfer ? cfg->page_bytes : 0;
    for (uint64_t b = 0; b < t->n_blocks; ++b) {
      if (bk[b] > 2) return fail(SCALESIM_E_INVALID);
      if (transfer) {
        if (bs[b] % pb != 0 || bo[b] % 16 != 0 || bo[b] + bs[b] > t->host_bytes) return fail(SCALESIM_E_INVALID);
        pf[b + 1] = pf[b] + bs[b] / pb;
      }
    }
  }
  if (transfer && pf[t->n_blocks] != t->n_block_pages) return fail(SCALESIM_E_INVALID);
  // per-agent write-back bytes (KV + HIST blocks, R13) for the fused path's d2h accounting
  std::vector<uint32_t> wb(n_local ? n_local : 1, 0);
  if (t->n_blocks > 0) {
    std::vector<uint32_t> bs(t->n_blocks);
    std::vector<uint8_t> bk(t->n_blocks);
    if (cudaMemcpy(bs.data(), t->blk_size, 4 * t->n_blocks, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(bk.data(), t->blk_kind, t->n_blocks, cudaMemcpyDeviceToHost) != cudaSuccess)
      return fail(SCALESIM_E_CUDA);
    const uint64_t a0 = tp ? cfg->shard_begin : 0;  // (TP-sliced: global tables)
    for (uint64_t a = 0; a < n_local; ++a) {
      uint64_t s = 0;
      for (uint64_t b = bp[a0 + a]; b < bp[a0 + a + 1]; ++b)
        if (bk[b] != 0) s += bs[b];
      if (s > 0xFFFFFFFFull) return fail(SCALESIM_E_INVALID);
      wb[a] = (uint32_t)s;
    }
  }
  if (cudaMemsetAsync(t->workspace, 0, L.total, c->stream) != cudaSuccess) return fail(SCALESIM_E_CUDA);
  GridHdr gh = {};  // a1' grid accumulators start empty (k_grid_setup re-arms them every step)
  gh.acc_x0 = gh.acc_y0 = 0x7FFFFFFF;
  gh.acc_x1 = gh.acc_y1 = (int32_t)0x80000000;
  if (cfg->n_kin > 0 &&
      cudaMemcpyAsync(p.d.grid_hdr, &gh, sizeof(gh), cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
    return fail(SCALESIM_E_CUDA);
  if (cudaMemcpyAsync(p.d.page_first, pf.data(), 8 * (t->n_blocks + 1), cudaMemcpyHostToDevice, c->stream) !=
      cudaSuccess)
    return fail(SCALESIM_E_CUDA);
  if (cudaMemcpyAsync(p.d.wb_bytes, wb.data(), 4 * wb.size(), cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
    return fail(SCALESIM_E_CUDA);
  c->launches += launch_init_pages(p, t->resident_init, c->stream);
  c->launches += launch_mask_tail(p, c->stream);
  if (transfer) {
    uint64_t *cnt = reinterpret_cast<uint64_t *>(p.d.gather);
    launch_init_page_table(p, L.n_block_pages, t->resident_init, cnt, c->stream);
    c->launches += 2;
    if (t->resident_init) {
      // load the initially resident blocks (synchronous, init time)
      std::vector<uint32_t> pt(L.n_block_pages ? L.n_block_pages : 1);
      if (cudaStreamSynchronize(c->stream) != cudaSuccess) return fail(SCALESIM_E_CUDA);
      if (L.n_block_pages &&
          cudaMemcpy(pt.data(), p.d.page_table, 4 * L.n_block_pages, cudaMemcpyDeviceToHost) != cudaSuccess)
        return fail(SCALESIM_E_CUDA);
      std::vector<uint64_t> bo(t->n_blocks ? t->n_blocks : 1);
      if (t->n_blocks && cudaMemcpy(bo.data(), t->blk_host_off, 8 * t->n_blocks, cudaMemcpyDeviceToHost) != cudaSuccess)
        return fail(SCALESIM_E_CUDA);
      std::vector<uint64_t> desc(2);
      uint64_t nh = 0;
      for (uint64_t b = 0; b < t->n_blocks; ++b)
        for (uint64_t q = pf[b]; q < pf[b + 1]; ++q)
          if (pt[q] != PAGE_NONE) {
            desc.push_back(bo[b] + (q - pf[b]) * cfg->page_bytes);
            desc.push_back(pt[q]);
            ++nh;
          }
      // layout of a descriptor buffer: [n_d2h, n_h2d, d2h pairs (desc_cap), h2d pairs]
      std::vector<uint64_t> buf(DESC_HDR + 4 * (L.desc_cap ? L.desc_cap : 1), 0);
      buf[0] = 0;
      buf[1] = nh;
      buf[2] = nh;  // every initial load is independent
      if (nh > L.desc_cap) return fail(SCALESIM_E_INVALID);
      for (uint64_t k = 0; k < 2 * nh; ++k) buf[DESC_HDR + 2 * L.desc_cap + k] = desc[2 + k];
      if (cudaMemcpy(p.d.desc[0], buf.data(), 8 * buf.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return fail(SCALESIM_E_CUDA);
      p.desc_buf = 0;
      c->launches += launch_transfer(p, c->stream, c->copy_ctas);
    }
  }
  c->launches += launch_plan_init(p, c->stream);
  // fused path: one CTA per SM, co-resident (cooperative launch); a loopback rank gets its
  // share of the SMs (its world is planned by one launch)
  if ((cfg->world == 1 || p.loopback) && !(cfg->flags & SCALESIM_F_MULTI_KERNEL)) {
    uint32_t tile = 0;
    // a transfer context leaves SMs to its page copies (they overlap the next plan)
    const int g = (p.loopback ? sms / cfg->world : sms) - (transfer && !p.loopback ? 2 * COPY_CTAS : 0);
    if (fused_supported(p, g, &tile) && fused_prepare(g * (p.loopback ? cfg->world : 1), tile, (uint32_t)g)) {
      c->fused = true;
      c->fused_tile = tile;
      c->fused_grid = g;
      c->sms = sms;
    } else if (cfg->world == 1 && p.int_mode) {
      // more agents per CTA than shared memory holds: the streaming kernel (fused_big.cu)
      uint64_t t = (p.n_local + g - 1) / g;
      t = (t + 31) / 32 * 32;
      if (t > FUSED_MAX_TILE && t <= FUSED_BIG_MAX_TILE && g <= FUSED_MAX_CTAS && fused_big_prepare((uint32_t)g)) {
        c->fused = true;
        c->big = true;
        c->fused_tile = (uint32_t)t;
        c->fused_grid = g;
        c->sms = sms;
      }
      if (cudaMemsetAsync(p.d.f_mm1, 0xFF, 4 * 2 * 2 * 4096, c->stream) != cudaSuccess ||
          cudaMemsetAsync(p.d.f_mm2, 0xFF, 4 * 2 * 2 * 1024, c->stream) != cudaSuccess)
        return fail(SCALESIM_E_CUDA);
    }
  }
  if (c->fused && (cfg->flags & SCALESIM_F_EXCLUSIVE)) {
    if (cfg->device < 0 || cfg->device >= 64 || cudaEventCreateWithFlags(&c->ev_fused, cudaEventDisableTiming) != cudaSuccess)
      return fail(SCALESIM_E_INVALID);
    std::lock_guard<std::mutex> g(g_excl_mu);
    c->exclusive = true;
    g_excl[cfg->device].contexts++;
  }
  // device copy of the parameters for the fused kernel (per-launch fields are overridden)
  if (cudaMemcpyAsync(p.d.params_dev, &p, sizeof(Params), cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
    return fail(SCALESIM_E_CUDA);
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return fail(SCALESIM_E_CUDA);
  if (p.loopback && !c->fused) return fail(SCALESIM_E_INVALID);  // (shard too large for its CTAs)
  if (cfg->flags & SCALESIM_F_THREADS) {
    if (cudaEventCreateWithFlags(&c->ev_xin, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_xred, cudaEventDisableTiming) != cudaSuccess)
      return fail(SCALESIM_E_CUDA);
    if (!(c->tgroup = join_group(cfg->nccl_unique_id, cfg->world))) return fail(SCALESIM_E_INVALID);
  } else if (cfg->world > 1 && !p.loopback) {
    if (!cfg->nccl_unique_id || !g_nccl.load()) return fail(SCALESIM_E_NCCL);
    ncclUniqueId id;
    memcpy(&id, cfg->nccl_unique_id, sizeof(id));
    if (g_nccl.CommInitRank(&c->comm, cfg->world, id, cfg->rank) != ncclSuccess) return fail(SCALESIM_E_NCCL);
    // the ranks' shards must be contiguous, in rank order and cover [0, n_agents) (the tie prefix
    // over lower ranks assumes it): all-gather (shard_begin, shard_end) once
    uint64_t *g = reinterpret_cast<uint64_t *>(p.d.xscratch);
    const uint64_t mine[2] = {cfg->shard_begin, cfg->shard_end};
    std::vector<uint64_t> all(2 * cfg->world);
    if (cudaMemcpyAsync(g, mine, 16, cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
        g_nccl.AllGather(g, g + 2, 2, ncclUint64, c->comm, c->stream) != ncclSuccess ||
        cudaMemcpyAsync(all.data(), g + 2, 16 * cfg->world, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess)
      return fail(SCALESIM_E_NCCL);
    for (int r = 0; r < cfg->world; ++r)
      if (all[2 * r] != (r == 0 ? 0 : all[2 * r - 1]) || (r == cfg->world - 1 && all[2 * r + 1] != cfg->n_agents))
        return fail(SCALESIM_E_INVALID);
  }
  *out = c;
  return SCALESIM_OK;
}

extern "C" scalesim_status scalesim_set_inputs(scalesim_ctx *c, const uint32_t *rec, const float *kin) {
  if (!c) return SCALESIM_E_INVALID;
  if (c->p.n_local > 0 && (!rec || !aligned(rec, 16))) return SCALESIM_E_INVALID;
  if (c->p.n_kin > 0 && (!kin || !aligned(kin, 16))) return SCALESIM_E_INVALID;
  c->p.rec = reinterpret_cast<const uint4 *>(rec);
  c->p.kin = reinterpret_cast<const float4 *>(kin);
  c->tab.agent_rec = rec;
  c->tab.agent_kin = kin;
  return SCALESIM_OK;
}

extern "C" scalesim_status scalesim_score(scalesim_ctx *c, int64_t now, float *dist_out) {
  if (!c) return SCALESIM_E_INVALID;
  CK(cudaGetLastError());
  // the accumulators were cleared at the end of the previous plan (or at init); a repeated
  // score without a plan clears them again
  if (c->scored) c->launches += launch_plan_init(c->p, c->stream);
  if (c->fused && !dist_out) {
    // the fused plan kernel scores the agents itself (phase P1); only the interaction
    // pair scan (which needs every participant before any agent is scored) runs here
    c->launches += launch_interaction(c->p, now, c->stream, c->grid);
    c->deferred = true;
    c->deferred_now = now;
  } else {
    c->launches += launch_score(c->p, now, dist_out, c->stream, c->grid);
    c->deferred = false;
  }
  CK(cudaGetLastError());
  c->scored = true;
  return SCALESIM_OK;
}

// in-place all-reduce (sum of u64 or min of u32) over the world's ranks: NCCL, or the thread
// group's device-memory exchange
static scalesim_status allreduce(scalesim_ctx *c, void *buf, size_t n, ncclDataType_t t, ncclRedOp_t op) {
  if (!c->tgroup) {
    NK(g_nccl.AllReduce(buf, buf, n, t, op, c->comm, c->stream));
    return SCALESIM_OK;
  }
  ThreadGroup &g = *c->tgroup;
  const int r = c->cfg.rank, G = c->cfg.world;
  const size_t bytes = n * (t == ncclUint64 ? 8 : 4);
  if (bytes > 32768) return SCALESIM_E_INVALID;
  CK(cudaEventRecord(c->ev_xin, c->stream));
  g.in[r] = buf;
  g.ev_in[r] = c->ev_xin;
  g.shard[r][0] = c->cfg.shard_begin;
  g.shard[r][1] = c->cfg.shard_end;
  g.barrier();
  // (every rank sees the same shards: all fail together, before the next barrier)
  for (int q = 0; q < G; ++q)
    if (g.shard[q][0] != (q == 0 ? 0 : g.shard[q - 1][1]) || (q == G - 1 && g.shard[q][1] != c->cfg.n_agents))
      return SCALESIM_E_INVALID;
  for (int q = 0; q < G; ++q)
    if (q != r) CK(cudaStreamWaitEvent(c->stream, g.ev_in[q], 0));
  c->launches += launch_xreduce(c->p.d.xscratch, g.in, (uint32_t)G, n, t == ncclUint64 ? 0 : 1, c->stream);
  CK(cudaEventRecord(c->ev_xred, c->stream));
  g.ev_red[r] = c->ev_xred;
  g.barrier();  // (every rank's waits on the inputs are enqueued)
  for (int q = 0; q < G; ++q)
    if (q != r) CK(cudaStreamWaitEvent(c->stream, g.ev_red[q], 0));  // (nobody still reads this input)
  CK(cudaMemcpyAsync(buf, c->p.d.xscratch, bytes, cudaMemcpyDeviceToDevice, c->stream));
  g.barrier();  // (every wait on this collective's events is enqueued before they are re-recorded)
  (void)op;
  return SCALESIM_OK;
}

// all-gather of one u64 per rank into recv[0, world)
static scalesim_status allgather_u64(scalesim_ctx *c, const unsigned long long *send, unsigned long long *recv) {
  if (!c->tgroup) {
    NK(g_nccl.AllGather(send, recv, 1, ncclUint64, c->comm, c->stream));
    return SCALESIM_OK;
  }
  ThreadGroup &g = *c->tgroup;
  const int r = c->cfg.rank, G = c->cfg.world;
  CK(cudaEventRecord(c->ev_xin, c->stream));
  g.in[r] = send;
  g.ev_in[r] = c->ev_xin;
  g.barrier();
  for (int q = 0; q < G; ++q)
    if (q != r) CK(cudaStreamWaitEvent(c->stream, g.ev_in[q], 0));
  c->launches += launch_xgather(recv, g.in, (uint32_t)G, c->stream);
  CK(cudaEventRecord(c->ev_xred, c->stream));
  g.ev_red[r] = c->ev_xred;
  g.barrier();
  for (int q = 0; q < G; ++q)
    if (q != r) CK(cudaStreamWaitEvent(c->stream, g.ev_red[q], 0));
  g.barrier();
  return SCALESIM_OK;
}

static void fill_plan(scalesim_ctx *c, scalesim_plan_view *out) {
  if (!out) return;
  const Params &p = c->p;
  out->prefetch_ids = p.d.pf_ids;
  out->evict_ids = p.d.ev_ids;
  out->resident_bitmap = p.d.bm[p.cur];  // after the flip: the new residency
  out->dist = reinterpret_cast<const float *>(p.d.keys);
  out->page_table = p.d.page_table;
  out->d2h_desc = reinterpret_cast<const uint64_t *>(p.d.desc[c->last_buf] + DESC_HDR);
  out->h2d_desc = reinterpret_cast<const uint64_t *>(p.d.desc[c->last_buf] + DESC_HDR + 2 * p.desc_cap);
  out->header = reinterpret_cast<const uint64_t *>(p.d.header);
  out->done_event = c->ev_xfer[c->last_buf];
}

static scalesim_status finish_plan(scalesim_ctx *c, scalesim_plan_view *out);

// One single-kernel plan launch (n instances on c's stream): cooperative unless c is an
// exclusive context; exclusive launches of different contexts of a device are chained.
static int launch_fused(scalesim_ctx *c, const FusedInst *insts, uint32_t n, uint32_t gsize, uint32_t wsize = 1) {
  if (c->big) {  // (single instance)
    if (!c->exclusive) return launch_fused_big(insts[0], gsize, c->stream, true);
    std::lock_guard<std::mutex> g(g_excl_mu);
    ExclusiveChain &x = g_excl[c->cfg.device];
    if (x.contexts > 1 && x.stream && x.stream != c->stream) cudaStreamWaitEvent(c->stream, x.event, 0);
    const int k = launch_fused_big(insts[0], gsize, c->stream, false);
    if (x.contexts > 1) {
      cudaEventRecord(c->ev_fused, c->stream);
      x.stream = c->stream;
      x.event = c->ev_fused;
    }
    return k;
  }
  if (!c->exclusive) return launch_fused_batch(insts, n, gsize, c->stream, true, wsize);
  std::lock_guard<std::mutex> g(g_excl_mu);
  ExclusiveChain &x = g_excl[c->cfg.device];
  if (x.contexts > 1 && x.stream && x.stream != c->stream) cudaStreamWaitEvent(c->stream, x.event, 0);
  const int k = launch_fused_batch(insts, n, gsize, c->stream, false, wsize);
  if (x.contexts > 1) {
    cudaEventRecord(c->ev_fused, c->stream);
    x.stream = c->stream;
    x.event = c->ev_fused;
  }
  return k;
}

static FusedInst fused_inst(const scalesim_ctx *c, uint32_t tile) {
  FusedInst f;
  f.params = reinterpret_cast<const Params *>(c->p.d.params_dev);
  f.rec = c->p.rec;
  f.kin = c->p.kin;
  f.now = c->deferred_now;
  f.n_local = c->p.n_local;
  f.bm_old = c->p.d.bm[c->p.cur];
  f.cur = (uint32_t)c->p.cur;
  f.parity = (uint32_t)(c->fused_steps & 1);
  f.epoch = (uint32_t)(c->fused_steps + 1);
  f.tile = tile;
  return f;
}

extern "C" scalesim_status scalesim_plan(scalesim_ctx *c, scalesim_plan_view *out) {
  if (!c) return SCALESIM_E_INVALID;
  if (c->p.loopback) return SCALESIM_E_INVALID;  // a loopback rank is planned with its world (scalesim_step_group)
  if (!c->scored) return SCALESIM_E_ORDER;
  Params &p = c->p;
  const bool multi = c->cfg.world > 1;
  if (c->deferred) {
    const FusedInst inst = fused_inst(c, c->fused_tile);
    c->launches += launch_fused(c, &inst, 1, (uint32_t)c->fused_grid);
    CK(cudaGetLastError());
    c->fused_steps++;
    c->deferred = false;
    c->last_fused = true;
    return finish_plan(c, out);
  }
  if (multi) {
    scalesim_status s;
    if ((s = allreduce(c, p.d.hist1, 2049, ncclUint64, ncclSum)) != SCALESIM_OK) return s;
    if ((s = allreduce(c, p.d.mm1, 4096, ncclUint32, ncclMin)) != SCALESIM_OK) return s;
  }
  c->launches += launch_select(p, 1, c->stream);
  c->launches += launch_hist(p, 2, c->stream, c->grid);
  if (multi) {
    scalesim_status s;
    if ((s = allreduce(c, p.d.hist2, 1024, ncclUint64, ncclSum)) != SCALESIM_OK) return s;
    if ((s = allreduce(c, p.d.mm2, 2048, ncclUint32, ncclMin)) != SCALESIM_OK) return s;
  }
  c->launches += launch_select(p, 2, c->stream);
  c->launches += launch_hist(p, 3, c->stream, c->grid);
  if (multi) {
    scalesim_status s;
    if ((s = allreduce(c, p.d.hist3, 1024, ncclUint64, ncclSum)) != SCALESIM_OK) return s;
  }
  c->launches += launch_select(p, 3, c->stream);
  c->launches += launch_tie(p, c->stream);
  if (multi) {
    scalesim_status s;
    if ((s = allgather_u64(c, &p.d.state->tie_local, p.d.gather)) != SCALESIM_OK) return s;
  }
  c->launches += launch_emit(p, c->stream);
  if (multi) {
    scalesim_status s;
    if ((s = allreduce(c, &p.d.state->tie_kept, 1, ncclUint64, ncclSum)) != SCALESIM_OK) return s;
    c->launches += launch_fix_kept(p, c->stream);
  }
  c->launches += launch_lists(p, c->stream);
  c->last_fused = false;
  return finish_plan(c, out);
}

static scalesim_status finish_plan(scalesim_ctx *c, scalesim_plan_view *out) {
  Params &p = c->p;
  const int buf = (int)(c->step & 1);
  p.desc_buf = buf;
  if (c->transfer) {
    // the descriptor buffer `buf` was last read by the transfer of plan step-2
    CK(cudaStreamWaitEvent(c->stream, c->ev_xfer[buf], 0));
    if (buf == c->last_buf) c->xfer_pending = false;
  }
  // byte accounting (multi-kernel path) and page assignment (transfers); the fused kernel
  // accounts the write-back bytes itself
  // (TP-sliced ranks: the expansion of the world's merged lists ran in scalesim_step_group)
  if ((c->transfer && !p.tp) || !c->last_fused) c->launches += launch_expand(p, c->stream);
  // the transfer's copy streams wait on this event (plan-only contexts record nothing: in a
  // captured graph consecutive plan kernels then stay directly linked, so their programmatic
  // launch overlap is kept)
  if (c->transfer) CK(cudaEventRecord(c->ev_plan, c->stream));
  if (!c->fused || p.n_kin > 0 || c->cfg.world > 1)
    c->launches += launch_plan_init(p, c->stream);  // clear the multi-kernel accumulators for the next step
  CK(cudaGetLastError());
  c->last_buf = buf;
  p.cur ^= 1;  // the new residency becomes current
  c->step++;
  c->scored = false;
  c->planned = true;
  c->transferred = false;
  fill_plan(c, out);
  return SCALESIM_OK;
}

extern "C" scalesim_status scalesim_view(scalesim_ctx *c, scalesim_plan_view *out) {
  if (!c || !out) return SCALESIM_E_INVALID;
  if (!c->planned) return SCALESIM_E_ORDER;
  fill_plan(c, out);
  return SCALESIM_OK;
}

extern "C" scalesim_status scalesim_transfer(scalesim_ctx *c, const scalesim_plan_view *plan) {
  if (!c) return SCALESIM_E_INVALID;
  if (!c->planned || c->transferred) return SCALESIM_E_ORDER;
  if (plan && plan->header != reinterpret_cast<const uint64_t *>(c->p.d.header)) return SCALESIM_E_ORDER;
  const int buf = c->last_buf;
  if (c->transfer) {
    CK(cudaStreamWaitEvent(c->copy_stream, c->ev_plan, 0));
    CK(cudaStreamWaitEvent(c->copy_stream2, c->ev_plan, 0));
    // the independent loads may reuse pages the previous step released: they must not
    // overtake that step's write-backs (still running on copy_stream when plans run ahead)
    if (c->xfer_recorded[buf ^ 1]) CK(cudaStreamWaitEvent(c->copy_stream2, c->ev_xfer[buf ^ 1], 0));
    Params q = c->p;
    q.desc_buf = buf;
    c->launches += launch_transfer_split(q, c->copy_stream, c->copy_stream2, c->copy_ctas);
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev_side, c->copy_stream2));
    CK(cudaStreamWaitEvent(c->copy_stream, c->ev_side, 0));
    CK(cudaEventRecord(c->ev_xfer[buf], c->copy_stream));
    c->xfer_recorded[buf] = true;
    c->xfer_pending = true;
  }
  c->transferred = true;
  return SCALESIM_OK;
}

extern "C" scalesim_status scalesim_join(scalesim_ctx *c) {
  if (!c) return SCALESIM_E_INVALID;
  if (c->xfer_pending) {
    CK(cudaStreamWaitEvent(c->stream, c->ev_xfer[c->last_buf], 0));
    c->xfer_pending = false;
  }
  return SCALESIM_OK;
}

extern "C" scalesim_status scalesim_step(scalesim_ctx *c, int64_t now, scalesim_plan_view *out) {
  scalesim_status s = scalesim_score(c, now, nullptr);
  if (s != SCALESIM_OK) return s;
  scalesim_plan_view pl;
  if ((s = scalesim_plan(c, &pl)) != SCALESIM_OK) return s;
  if ((s = scalesim_transfer(c, &pl)) != SCALESIM_OK) return s;
  if (out) *out = pl;
  return SCALESIM_OK;
}

// Instances per launch and CTAs per instance for a batch chunk starting at i0 (sms CTAs in
// all: one CTA per SM); false when a context's tile cannot fit shared memory.
static bool batch_chunk(scalesim_ctx *const *ctxs, uint32_t n, uint32_t i0, uint32_t sms, uint32_t *k_out,
                        uint32_t *gsize_out, uint32_t *tile_out) {
  uint32_t k = n - i0 < sms ? n - i0 : sms;
  if (k > (uint32_t)FUSED_MAX_BATCH) k = FUSED_MAX_BATCH;
  uint32_t gsize, tile;
  while (true) {
    gsize = sms / k;
    uint64_t nm = 0;
    for (uint32_t i = i0; i < i0 + k; ++i) nm = ctxs[i]->p.n_local > nm ? ctxs[i]->p.n_local : nm;
    uint64_t t = (nm + gsize - 1) / gsize;
    t = (t + 31) / 32 * 32;
    tile = (uint32_t)(t ? t : 32);
    if (tile <= FUSED_MAX_TILE || k == 1) break;
    k = k / 2;  // fewer instances per launch, more CTAs each
  }
  *k_out = k;
  *gsize_out = gsize;
  *tile_out = tile;
  return tile <= FUSED_MAX_TILE && fused_prepare((int)(k * gsize), tile, gsize);
}

extern "C" scalesim_status scalesim_step_batch(scalesim_ctx *const *ctxs, uint32_t n, int64_t now) {
  if (!ctxs || n == 0) return SCALESIM_E_INVALID;
  scalesim_ctx *c0 = ctxs[0];
  if (!c0) return SCALESIM_E_INVALID;
  for (uint32_t i = 0; i < n; ++i) {
    scalesim_ctx *c = ctxs[i];
    if (!c || !c->fused || c->big || c->stream != c0->stream || c->cfg.device != c0->cfg.device ||
        c->exclusive != c0->exclusive)
      return SCALESIM_E_INVALID;
    for (uint32_t j = 0; j < i; ++j)
      if (ctxs[j] == c) return SCALESIM_E_INVALID;  // a context at most once per batch
  }
  // validate every launch before enqueueing anything: an error leaves every context unchanged
  const uint32_t sms = (uint32_t)c0->sms;
  for (uint32_t i0 = 0; i0 < n;) {
    uint32_t k, gsize, tile;
    if (!batch_chunk(ctxs, n, i0, sms, &k, &gsize, &tile)) return SCALESIM_E_INVALID;
    i0 += k;
  }
  CK(cudaGetLastError());
  // (1) score: interaction pair scans (if any) and the deferred score of every instance
  for (uint32_t i = 0; i < n; ++i) {
    scalesim_status s = scalesim_score(ctxs[i], now, nullptr);
    if (s != SCALESIM_OK) return s;
  }
  // (2) plan: chunks of instances, each instance on its own group of CTAs, one launch each
  for (uint32_t i0 = 0; i0 < n;) {
    uint32_t k, gsize, tile;
    batch_chunk(ctxs, n, i0, sms, &k, &gsize, &tile);
    FusedInst insts[FUSED_MAX_BATCH];
    for (uint32_t i = 0; i < k; ++i) insts[i] = fused_inst(ctxs[i0 + i], tile);
    c0->launches += launch_fused(c0, insts, k, gsize);
    CK(cudaGetLastError());
    for (uint32_t i = i0; i < i0 + k; ++i) {
      scalesim_ctx *c = ctxs[i];
      c->fused_steps++;
      c->deferred = false;
      c->last_fused = true;
      scalesim_status s = finish_plan(c, nullptr);
      if (s != SCALESIM_OK) return s;
      if ((s = scalesim_transfer(c, nullptr)) != SCALESIM_OK) return s;
    }
    i0 += k;
  }
  return SCALESIM_OK;
}

extern "C" scalesim_status scalesim_step_group(scalesim_ctx *const *ctxs, uint32_t world, int64_t now) {
  if (!ctxs || world < 2 || world > FUSED_MAX_WORLD) return SCALESIM_E_INVALID;
  scalesim_ctx *c0 = ctxs[0];
  if (!c0) return SCALESIM_E_INVALID;
  uint64_t next = 0;  // shards: contiguous, in rank order, covering [0, n_agents)
  for (uint32_t r = 0; r < world; ++r) {
    const scalesim_ctx *c = ctxs[r];
    if (!c || !c->p.loopback || !c->fused || c->cfg.world != (int)world || c->cfg.rank != (int)r) return SCALESIM_E_INVALID;
    if (c->stream != c0->stream || c->cfg.device != c0->cfg.device || c->exclusive != c0->exclusive ||
        c->cfg.n_agents != c0->cfg.n_agents || c->cfg.budget_bytes != c0->cfg.budget_bytes ||
        c->cfg.hop_scale != c0->cfg.hop_scale || c->fused_steps != c0->fused_steps ||
        c->fused_grid != c0->fused_grid || c->p.int_mode != c0->p.int_mode || c->p.tp != c0->p.tp ||
        c->transfer != c0->transfer || c->p.explicit_dist != c0->p.explicit_dist)
      return SCALESIM_E_INVALID;
    for (int k = 0; k < 3; ++k)
      if (c->cfg.theta[k] != c0->cfg.theta[k]) return SCALESIM_E_INVALID;
    if (c->cfg.shard_begin != next) return SCALESIM_E_INVALID;
    next = c->cfg.shard_end;
  }
  if (next != c0->cfg.n_agents) return SCALESIM_E_INVALID;
  CK(cudaGetLastError());
  const Params *ps[FUSED_MAX_WORLD];
  bool kin = false;
  for (uint32_t r = 0; r < world; ++r) {
    ps[r] = &ctxs[r]->p;
    kin = kin || ctxs[r]->p.n_kin > 0;
  }
  // score: every agent is scored inside the plan kernel; the interaction pair scan first needs
  // the world's participants (§8(e): the all-gather of their kinematics, through device memory)
  for (uint32_t r = 0; r < world; ++r) {
    scalesim_ctx *c = ctxs[r];
    if (c->scored) c->launches += launch_plan_init(c->p, c->stream);
    c->deferred = true;
    c->deferred_now = now;
    c->scored = true;
  }
  if (kin) c0->launches += launch_world_interaction(ps, world, now, c0->stream);
  FusedInst insts[FUSED_MAX_WORLD];
  for (uint32_t r = 0; r < world; ++r) insts[r] = fused_inst(ctxs[r], ctxs[r]->fused_tile);
  c0->launches += launch_fused(c0, insts, world, (uint32_t)c0->fused_grid, world);
  CK(cudaGetLastError());
  if (c0->p.tp && c0->transfer) {
    // §8(e) step 4: the ranks' lists merged into the world's lists in every rank (all-gather
    // over device memory), then every rank assigns the pages of the whole plan (the same FIFO
    // on every rank) and moves its slice of each page
    c0->launches += launch_tp_merge(ps, world, now, c0->stream);
    for (uint32_t r = 0; r < world; ++r) {
      scalesim_ctx *c = ctxs[r];
      const int buf = (int)(c->step & 1);
      CK(cudaStreamWaitEvent(c->stream, c->ev_xfer[buf], 0));  // (its descriptor buffer's last reader)
      Params q = c->p;
      q.desc_buf = buf;
      q.shard_begin = 0;
      q.n_local = c->p.n_agents;
      q.d.pf_ids = c->p.d.tp_pf;
      q.d.ev_ids = c->p.d.tp_ev;
      q.d.header = c->p.d.tp_hdr;
      q.ev_dirty = c->p.d.tp_dirty;
      c->launches += launch_expand(q, c->stream);
      c->launches += launch_tp_finish(c->p, c->stream);
    }
    CK(cudaGetLastError());
  }
  for (uint32_t r = 0; r < world; ++r) {
    scalesim_ctx *c = ctxs[r];
    c->fused_steps++;
    c->deferred = false;
    c->last_fused = true;
    scalesim_status s = finish_plan(c, nullptr);
    if (s != SCALESIM_OK) return s;
    if ((s = scalesim_transfer(c, nullptr)) != SCALESIM_OK) return s;
  }
  return SCALESIM_OK;
}

extern "C" scalesim_status scalesim_world_view(scalesim_ctx *c, scalesim_world_view_t *out) {
  if (!c || !out) return SCALESIM_E_INVALID;
  if (!c->p.tp) return SCALESIM_E_INVALID;
  if (!c->planned) return SCALESIM_E_ORDER;
  out->prefetch_ids = c->p.d.tp_pf;
  out->evict_ids = c->p.d.tp_ev;
  out->header = reinterpret_cast<const uint64_t *>(c->p.d.tp_hdr);
  return SCALESIM_OK;
}

static scalesim_status status_of_header(uint64_t st) {
  if (st & (SCALESIM_ST_BAD_RECORD | SCALESIM_ST_BAD_KIN)) return SCALESIM_E_BAD_INPUT;
  if (st & (SCALESIM_ST_NO_PAGES | SCALESIM_ST_SYNC | SCALESIM_ST_LIMIT)) return SCALESIM_E_INVARIANT;
  if (st & SCALESIM_ST_INSUFFICIENT) return SCALESIM_E_INSUFFICIENT;
  return SCALESIM_OK;
}

extern "C" scalesim_status scalesim_sync(scalesim_ctx *c, scalesim_plan_host *out) {
  if (!c) return SCALESIM_E_INVALID;
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaStreamSynchronize(c->copy_stream));
  scalesim_plan_host h;
  CK(cudaMemcpy(h.f, c->p.d.header, sizeof(h.f), cudaMemcpyDeviceToHost));
  if (out) *out = h;
  return c->planned ? status_of_header(h.f[SCALESIM_H_STATUS]) : SCALESIM_OK;
}

// The step's header and lists to the host: k_readback writes them into host-mapped pinned
// memory (two slots, seq % 2: [done word | header @128 | prefetch @256 | evict]) and then the
// slot's completion word, which the host polls (one kernel instead of three copies and two
// stream synchronisations); the stream is queried now and then so that a failed launch returns
// instead of spinning.
static size_t rb_list_bytes(const scalesim_ctx *c) { return ((size_t)4 * c->p.n_local + 15) / 16 * 16; }
static size_t rb_slot_bytes(const scalesim_ctx *c) { return 256 + 2 * rb_list_bytes(c); }

static scalesim_status enqueue_readback(scalesim_ctx *c, unsigned long long *seq_out) {
  if (!c->rb_h) {
    CK(cudaHostAlloc(reinterpret_cast<void **>(&c->rb_h), NSLOT * rb_slot_bytes(c), cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->rb_d), c->rb_h, 0));
    CK(cudaMalloc(&c->rb_tickets, 16));
    CK(cudaMemset(c->rb_tickets, 0, 16));
    for (int k = 0; k < NSLOT; ++k) *reinterpret_cast<volatile unsigned long long *>(c->rb_h + k * rb_slot_bytes(c)) = 0ull;
  }
  const unsigned long long seq = ++c->rb_seq;
  uint8_t *d = c->rb_d + (seq % NSLOT) * rb_slot_bytes(c);
  auto *wd = reinterpret_cast<unsigned long long *>(d);
  c->launches += launch_readback(reinterpret_cast<const unsigned long long *>(c->p.d.header), c->p.d.pf_ids,
                                 c->p.d.ev_ids, wd + 16, reinterpret_cast<uint32_t *>(d + 256),
                                 reinterpret_cast<uint32_t *>(d + 256 + rb_list_bytes(c)), wd, seq,
                                 c->rb_tickets + (seq % NSLOT), c->stream);
  CK(cudaGetLastError());
  *seq_out = seq;
  return SCALESIM_OK;
}

static scalesim_status wait_readback(scalesim_ctx *c, unsigned long long seq, scalesim_plan_host *out,
                                     uint32_t *pf_out, uint32_t *ev_out) {
  const uint8_t *hb = c->rb_h + (seq % NSLOT) * rb_slot_bytes(c);
  volatile const unsigned long long *word = reinterpret_cast<volatile const unsigned long long *>(hb);
  for (uint64_t spin = 1; *word != seq; ++spin) {
    if ((spin & 1023) == 0) {
      const cudaError_t e = cudaStreamQuery(c->stream);
      if (e == cudaSuccess && *word != seq) return SCALESIM_E_CUDA;  // (done without the word: cannot happen)
      if (e != cudaSuccess && e != cudaErrorNotReady) return cuda_status(e);
    }
  }
  scalesim_plan_host h;
  memcpy(h.f, hb + 128, sizeof(h.f));
  if (pf_out && h.f[SCALESIM_H_N_PREFETCH]) memcpy(pf_out, hb + 256, 4 * h.f[SCALESIM_H_N_PREFETCH]);
  if (ev_out && h.f[SCALESIM_H_N_EVICT]) memcpy(ev_out, hb + 256 + rb_list_bytes(c), 4 * h.f[SCALESIM_H_N_EVICT]);
  if (c->transfer) CK(cudaStreamSynchronize(c->copy_stream));
  if (out) *out = h;
  return status_of_header(h.f[SCALESIM_H_STATUS]);
}

// (waits for the plan and its transfer)
static scalesim_status read_back(scalesim_ctx *c, scalesim_plan_host *out, uint32_t *pf_out, uint32_t *ev_out) {
  if (c->n_pending) return SCALESIM_E_ORDER;  // submitted steps not collected (their slots)
  unsigned long long seq;
  scalesim_status s = enqueue_readback(c, &seq);
  return s != SCALESIM_OK ? s : wait_readback(c, seq, out, pf_out, ev_out);
}

extern "C" scalesim_status scalesim_step_host(scalesim_ctx *c, int64_t now, const uint32_t *host_rec,
                                              const float *host_kin, scalesim_plan_host *out, uint32_t *pf_out,
                                              uint32_t *ev_out) {
  if (!c || !host_rec) return SCALESIM_E_INVALID;
  if (c->p.n_kin > 0 && !host_kin) return SCALESIM_E_INVALID;
  if (c->n_pending) return SCALESIM_E_ORDER;  // submitted steps not collected
  int si = -1;  // inputs staged by scalesim_stage_host (their copy may still be in flight)
  for (int i = 0; i < NSLOT; ++i)
    if (c->staged[i] && !c->staged_upd[i] && c->staged_rec[i] == host_rec &&
        (c->p.n_kin == 0 || c->staged_kin[i] == host_kin))
      si = i;
  scalesim_status s;
  if (si >= 0) {
    const uint4 *rec0 = c->p.rec;
    const float4 *kin0 = c->p.kin;
    CK(cudaStreamWaitEvent(c->stream, c->ev_in[si], 0));
    c->p.rec = reinterpret_cast<const uint4 *>(c->sbuf[si]);
    c->p.kin = reinterpret_cast<const float4 *>(c->sbuf[si] + 16 * c->p.n_local);
    s = scalesim_step(c, now, nullptr);  // (the launches capture the input pointers)
    c->p.rec = rec0;
    c->p.kin = kin0;
    c->staged[si] = false;
    c->sbuf_used[si] = true;
    CK(cudaEventRecord(c->ev_used[si], c->stream));  // the next copy into sbuf[si] waits for it
  } else {
    CK(cudaMemcpyAsync(const_cast<uint4 *>(c->p.rec), host_rec, 16 * c->p.n_local, cudaMemcpyHostToDevice, c->stream));
    if (c->p.n_kin > 0)
      CK(cudaMemcpyAsync(const_cast<float4 *>(c->p.kin), host_kin, 16 * c->p.n_kin, cudaMemcpyHostToDevice, c->stream));
    s = scalesim_step(c, now, nullptr);
  }
  if (s != SCALESIM_OK) return s;
  return read_back(c, out, pf_out, ev_out);
}

// A free staging slot (two per context), its buffer allocated and its last reader waited for
// on in_stream; -1 when both slots hold staged steps.
static int stage_slot(scalesim_ctx *c, scalesim_status *err) {
  *err = SCALESIM_OK;
  int i = c->stage_next;
  for (int k = 0; k < NSLOT && c->staged[i]; ++k) i = (i + 1) % NSLOT;
  if (c->staged[i]) {
    *err = SCALESIM_E_ORDER;  // two staged steps not yet run
    return -1;
  }
  auto fail = [&](cudaError_t e) { return e != cudaSuccess ? (*err = SCALESIM_E_CUDA, true) : false; };
  if (!c->in_stream) {
    if (fail(cudaStreamCreateWithFlags(&c->in_stream, cudaStreamNonBlocking))) return -1;
    for (int k = 0; k < NSLOT; ++k)
      if (fail(cudaEventCreateWithFlags(&c->ev_in[k], cudaEventDisableTiming)) ||
          fail(cudaEventCreateWithFlags(&c->ev_used[k], cudaEventDisableTiming)))
        return -1;
  }
  // whole inputs (records + kinematics) or up to n_local (id, record) updates
  const size_t full = 16 * (size_t)c->p.n_local + 16 * (size_t)c->p.n_kin, upd = 20 * (size_t)c->p.n_local + 16;
  if (!c->sbuf[i] && fail(cudaMalloc(&c->sbuf[i], (full > upd ? full : upd) + 16))) return -1;
  if (c->sbuf_used[i] && fail(cudaStreamWaitEvent(c->in_stream, c->ev_used[i], 0))) return -1;  // its last step read it
  return i;
}

static void stage_commit(scalesim_ctx *c, int i, const void *key0, const void *key1, bool upd, uint32_t n) {
  c->staged[i] = true;
  c->staged_upd[i] = upd;
  c->staged_rec[i] = key0;
  c->staged_kin[i] = key1;
  c->staged_n[i] = n;
  c->stage_next = (i + 1) % NSLOT;
}

extern "C" scalesim_status scalesim_stage_host(scalesim_ctx *c, const uint32_t *host_rec, const float *host_kin) {
  if (!c || !host_rec) return SCALESIM_E_INVALID;
  if (c->p.n_kin > 0 && !host_kin) return SCALESIM_E_INVALID;
  scalesim_status err;
  const int i = stage_slot(c, &err);
  if (i < 0) return err;
  const size_t rb = 16 * (size_t)c->p.n_local, kb = 16 * (size_t)c->p.n_kin;
  if (rb) CK(cudaMemcpyAsync(c->sbuf[i], host_rec, rb, cudaMemcpyHostToDevice, c->in_stream));
  if (kb) CK(cudaMemcpyAsync(c->sbuf[i] + rb, host_kin, kb, cudaMemcpyHostToDevice, c->in_stream));
  CK(cudaEventRecord(c->ev_in[i], c->in_stream));
  stage_commit(c, i, host_rec, host_kin, false, 0);
  return SCALESIM_OK;
}

// staged (ids, records) of n updates in slot i: ids at offset 0, records at the next 16-byte
// boundary
static size_t upd_rec_off(uint32_t n) { return ((size_t)4 * n + 15) / 16 * 16; }

extern "C" scalesim_status scalesim_stage_updates(scalesim_ctx *c, const uint32_t *host_ids,
                                                  const uint32_t *host_rec, uint32_t n_upd) {
  if (!c || (n_upd > 0 && (!host_ids || !host_rec)) || n_upd > c->p.n_local || c->p.n_kin > 0)
    return SCALESIM_E_INVALID;
  scalesim_status err;
  const int i = stage_slot(c, &err);
  if (i < 0) return err;
  if (n_upd) {
    CK(cudaMemcpyAsync(c->sbuf[i], host_ids, 4 * (size_t)n_upd, cudaMemcpyHostToDevice, c->in_stream));
    CK(cudaMemcpyAsync(c->sbuf[i] + upd_rec_off(n_upd), host_rec, 16 * (size_t)n_upd, cudaMemcpyHostToDevice,
                       c->in_stream));
  }
  CK(cudaEventRecord(c->ev_in[i], c->in_stream));
  stage_commit(c, i, host_ids, host_rec, true, n_upd);
  return SCALESIM_OK;
}

// Scatter of one step's updates (staged or copied now on in_stream) and the step, enqueued;
// the step's out-of-shard count goes to the host-mapped word of read-back slot `slot`.
static scalesim_status enqueue_updates_step(scalesim_ctx *c, int64_t now, const uint32_t *host_ids,
                                            const uint32_t *host_rec, uint32_t n_upd, int slot) {
  if (!c || (n_upd > 0 && (!host_ids || !host_rec)) || n_upd > c->p.n_local || c->p.n_kin > 0)
    return SCALESIM_E_INVALID;
  int si = -1;
  for (int i = 0; i < NSLOT; ++i)
    if (c->staged[i] && c->staged_upd[i] && c->staged_rec[i] == host_ids && c->staged_kin[i] == host_rec &&
        c->staged_n[i] == n_upd)
      si = i;
  scalesim_status s;
  if (si < 0) {  // not staged: the copy goes out now
    if ((s = scalesim_stage_updates(c, host_ids, host_rec, n_upd)) != SCALESIM_OK) return s;
    si = (c->stage_next + NSLOT - 1) % NSLOT;
  }
  if (!c->upd_err_h) {
    CK(cudaHostAlloc(reinterpret_cast<void **>(&c->upd_err_h), 16, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void **>(&c->upd_err_d), c->upd_err_h, 0));
  }
  // (the slot's previous step has been collected: its kernels are done)
  reinterpret_cast<volatile uint32_t *>(c->upd_err_h)[slot] = 0u;
  CK(cudaStreamWaitEvent(c->stream, c->ev_in[si], 0));
  const uint8_t *b = c->sbuf[si];
  c->launches += launch_apply_updates(const_cast<uint4 *>(c->p.rec), reinterpret_cast<const uint32_t *>(b),
                                      reinterpret_cast<const uint4 *>(b + upd_rec_off(n_upd)), n_upd,
                                      c->p.shard_begin, c->p.n_local, c->upd_err_d + slot, c->stream);
  CK(cudaGetLastError());
  c->staged[si] = false;
  c->sbuf_used[si] = true;
  CK(cudaEventRecord(c->ev_used[si], c->stream));  // the next copy into sbuf[si] waits for the scatter
  return scalesim_step(c, now, nullptr);
}

extern "C" scalesim_status scalesim_step_updates(scalesim_ctx *c, int64_t now, const uint32_t *host_ids,
                                                 const uint32_t *host_rec, uint32_t n_upd, scalesim_plan_host *out,
                                                 uint32_t *pf_out, uint32_t *ev_out) {
  if (!c) return SCALESIM_E_INVALID;
  if (c->n_pending) return SCALESIM_E_ORDER;
  const int slot = (int)((c->rb_seq + 1) % NSLOT);
  scalesim_status s = enqueue_updates_step(c, now, host_ids, host_rec, n_upd, slot);
  if (s != SCALESIM_OK) return s;
  s = read_back(c, out, pf_out, ev_out);
  if (s == SCALESIM_OK && reinterpret_cast<volatile uint32_t *>(c->upd_err_h)[slot]) return SCALESIM_E_BAD_INPUT;
  return s;
}

extern "C" scalesim_status scalesim_submit_updates(scalesim_ctx *c, int64_t now, const uint32_t *host_ids,
                                                   const uint32_t *host_rec, uint32_t n_upd) {
  if (!c) return SCALESIM_E_INVALID;
  if (c->n_pending >= NSLOT) return SCALESIM_E_ORDER;  // every read-back slot holds an uncollected step
  const int slot = (int)((c->rb_seq + 1) % NSLOT);
  scalesim_status s = enqueue_updates_step(c, now, host_ids, host_rec, n_upd, slot);
  if (s != SCALESIM_OK) return s;
  unsigned long long seq;
  if ((s = enqueue_readback(c, &seq)) != SCALESIM_OK) return s;
  c->rb_pending[c->n_pending++] = seq;
  return SCALESIM_OK;
}

extern "C" scalesim_status scalesim_collect(scalesim_ctx *c, scalesim_plan_host *out, uint32_t *pf_out,
                                            uint32_t *ev_out) {
  if (!c) return SCALESIM_E_INVALID;
  if (c->n_pending == 0) return SCALESIM_E_ORDER;
  const unsigned long long seq = c->rb_pending[0];
  for (int k = 1; k < NSLOT; ++k) c->rb_pending[k - 1] = c->rb_pending[k];
  c->n_pending--;
  scalesim_status s = wait_readback(c, seq, out, pf_out, ev_out);
  if (s == SCALESIM_OK && reinterpret_cast<volatile uint32_t *>(c->upd_err_h)[seq % NSLOT]) return SCALESIM_E_BAD_INPUT;
  return s;
}

extern "C" void scalesim_destroy(scalesim_ctx *c) {
  if (!c) return;
  if (c->in_stream) {
    cudaStreamSynchronize(c->in_stream);
    cudaStreamDestroy(c->in_stream);
  }
  for (int k = 0; k < NSLOT; ++k) {
    if (c->ev_in[k]) cudaEventDestroy(c->ev_in[k]);
    if (c->ev_used[k]) cudaEventDestroy(c->ev_used[k]);
  }
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (int k = 0; k < NSLOT; ++k)
    if (c->sbuf[k]) cudaFree(c->sbuf[k]);
  if (c->upd_err_h) cudaFreeHost(c->upd_err_h);
  if (c->rb_h) cudaFreeHost(c->rb_h);
  if (c->rb_tickets) cudaFree(c->rb_tickets);
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  if (c->tgroup) leave_group(c->tgroup);
  if (c->ev_xin) cudaEventDestroy(c->ev_xin);
  if (c->ev_xred) cudaEventDestroy(c->ev_xred);
  if (c->exclusive) {
    std::lock_guard<std::mutex> g(g_excl_mu);
    ExclusiveChain &x = g_excl[c->cfg.device];
    x.contexts--;
    if (x.event == c->ev_fused) {
      x.stream = nullptr;
      x.event = nullptr;
    }
  }
  if (c->ev_fused) cudaEventDestroy(c->ev_fused);
  if (c->copy_stream2) {
    cudaStreamSynchronize(c->copy_stream2);
    cudaStreamDestroy(c->copy_stream2);
  }
  if (c->ev_side) cudaEventDestroy(c->ev_side);
  if (c->ev_plan) cudaEventDestroy(c->ev_plan);
  for (int k = 0; k < 2; ++k)
    if (c->ev_xfer[k]) cudaEventDestroy(c->ev_xfer[k]);
  delete c;
}

/*
 * oracle.cpp — plain CPU oracle of the ScaleSim planner.  TEST INFRASTRUCTURE ONLY
 * (see oracle.h).  Compiled: g++ -std=c++17 -O2 -ffp-contract=off -fno-fast-math,
 * x86-64 SSE scalar float (no x87 excess precision, no FMA contraction).
 *
 * Every function follows the paper's definition step by step; the readings the paper
 * leaves open are DESIGN.md §3 R1..R17 and are cited where used.
 */
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <utility>
#include <vector>

namespace {

const uint32_t PH_ACTING = 0, PH_WAITING = 1, PH_GENERATING = 2, PH_IDLE = 3;
const uint32_t CL_IND = 0, CL_INT = 1, CL_DIFF = 2;
const uint8_t KIND_LORA = 0;
const float INF = std::numeric_limits<float>::infinity();

inline uint32_t phase_of(const uint32_t *rec, uint64_t i) { return rec[4 * i + 2] & 3u; }
inline uint32_t class_of(const uint32_t *rec, uint64_t i) { return (rec[4 * i + 2] >> 2) & 3u; }
inline bool dirty_of(const uint32_t *rec, uint64_t i) { return (rec[4 * i + 2] >> 4) & 1u; }
inline uint32_t footprint_of(const uint32_t *rec, uint64_t i) { return rec[4 * i + 1]; }

inline uint32_t f32_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}

/* An ACTING INT agent takes part in the pair scan iff its kin index is valid and its
 * kinematics are finite (R8). */
bool int_participant(const uint32_t *rec, const float *kin, uint64_t n_kin, uint64_t i,
                     uint32_t *status) {
  if (phase_of(rec, i) != PH_ACTING || class_of(rec, i) != CL_INT) return false;
  uint32_t k = rec[4 * i + 3];
  if (k >= n_kin) {
    *status |= ORACLE_ST_BAD_RECORD;
    return false;
  }
  for (int c = 0; c < 4; ++c)
    if (!std::isfinite(kin[4 * (uint64_t)k + c])) {
      *status |= ORACLE_ST_BAD_KIN;
      return false;
    }
  return true;
}

/* Eq. 2 with R6/R7: time to interaction of agents i and j moving toward each
 * other = |r| / closing speed = (r.r)/(-r.w) with r = p_j - p_i, w = v_j - v_i, and +inf
 * when they are not approaching (r.w >= 0).  Fixed op order, each op rounded to nearest. */
float pair_time(const float *ki, const float *kj) {
  float dx = kj[0] - ki[0];
  float dy = kj[1] - ki[1];
  float dvx = kj[2] - ki[2];
  float dvy = kj[3] - ki[3];
  float g2a = dx * dx;
  float g2b = dy * dy;
  float g2 = g2a + g2b;
  float rwa = dx * dvx;
  float rwb = dy * dvy;
  float rw = rwa + rwb;
  if (rw < 0.0f) {
    float den = -rw;
    return g2 / den;
  }
  return INF;
}

}  // namespace

extern "C" void oracle_interaction(uint64_t n, const uint32_t *rec, const float *kin, uint64_t n_kin,
                                   float *dint, uint32_t *status) {
  for (uint64_t k = 0; k < n_kin; ++k) dint[k] = INF;
  std::vector<uint64_t> part;
  for (uint64_t i = 0; i < n; ++i)
    if (int_participant(rec, kin, n_kin, i, status)) part.push_back(i);
  /* "min over other Acting agents of gap/closing-speed". */
  for (uint64_t a = 0; a < part.size(); ++a) {
    const float *ki = kin + 4 * (uint64_t)rec[4 * part[a] + 3];
    float best = INF;
    for (uint64_t b = 0; b < part.size(); ++b) {
      if (b == a) continue;
      const float *kj = kin + 4 * (uint64_t)rec[4 * part[b] + 3];
      float t = pair_time(ki, kj);
      if (t < best) best = t;
    }
    dint[rec[4 * part[a] + 3]] = best;
  }
}

/* Distance of agent i given the interaction times dint (indexed by kin index). */
static float agent_distance(const uint32_t *rec, uint64_t i, uint64_t n_kin, int64_t now, float hop_scale,
                            const float *dint, uint32_t *status) {
  uint32_t ph = phase_of(rec, i), cl = class_of(rec, i);
  if (cl == 3) *status |= ORACLE_ST_BAD_RECORD;
  float d;
  if (ph == PH_WAITING || ph == PH_GENERATING) {
    d = 0.0f; /* S:170 "any agent in WaitingForMemory or Generating -> 0" */
  } else if (ph == PH_IDLE) {
    d = INF; /* S:124 "+infinity for agents that will never activate again" */
  } else if (cl == CL_IND || cl == CL_INT) {
    /* D_action: remaining duration of the current action, R8 clamp */
    int64_t remain = (int64_t)rec[4 * i + 0] - now;
    float d_action = remain <= 0 ? 0.0f : (float)remain;
    d = d_action;
    if (cl == CL_INT) {
      /* Eq. 1: D = min(D_action, D_interaction) */
      uint32_t k = rec[4 * i + 3];
      float d_int = (k < n_kin) ? dint[k] : INF;
      if (k >= n_kin) *status |= ORACLE_ST_BAD_RECORD;
      if (d_int < d_action) d = d_int;
    }
  } else if (cl == CL_DIFF) {
    /* hop count from the information source, R5/R9: hop * hop_scale */
    uint32_t hop = rec[4 * i + 0];
    if (hop == 0xFFFFFFFFu)
      d = INF;
    else
      d = (float)hop * hop_scale;
  } else {
    d = INF; /* class 3: invalid record */
  }
  if (d == 0.0f) d = 0.0f; /* canonical +0 (R8) */
  return d;
}

extern "C" void oracle_score(uint64_t n, const uint32_t *rec, const float *kin, uint64_t n_kin,
                             int64_t now, float hop_scale, float *d_out, uint32_t *status) {
  std::vector<float> dint(n_kin > 0 ? n_kin : 1, INF);
  if (n_kin > 0) oracle_interaction(n, rec, kin, n_kin, dint.data(), status);
  for (uint64_t i = 0; i < n; ++i) d_out[i] = agent_distance(rec, i, n_kin, now, hop_scale, dint.data(), status);
}

extern "C" void oracle_score_sampled(uint64_t n, const uint32_t *rec, const float *kin, uint64_t n_kin, int64_t now,
                                     float hop_scale, const uint64_t *agents, uint64_t n_sample, float *d_out,
                                     uint32_t *status) {
  /* the same definitions for a sample of agents: the Eq. 2 minimum of each sampled
   * interaction participant over every other participant (the O(n^2) scan restricted to the
   * sampled rows) */
  std::vector<float> dint(n_kin > 0 ? n_kin : 1, INF);
  std::vector<uint64_t> part;
  for (uint64_t i = 0; i < n; ++i)
    if (int_participant(rec, kin, n_kin, i, status)) part.push_back(i);
  for (uint64_t s = 0; s < n_sample; ++s) {
    const uint64_t i = agents[s];
    if (!(i < n) || !int_participant(rec, kin, n_kin, i, status)) continue;
    const float *ki = kin + 4 * (uint64_t)rec[4 * i + 3];
    float best = INF;
    for (uint64_t b = 0; b < part.size(); ++b) {
      if (part[b] == i) continue;
      const float *kj = kin + 4 * (uint64_t)rec[4 * part[b] + 3];
      float t = pair_time(ki, kj);
      if (t < best) best = t;
    }
    dint[rec[4 * i + 3]] = best;
  }
  for (uint64_t s = 0; s < n_sample; ++s)
    d_out[s] = agents[s] < n ? agent_distance(rec, agents[s], n_kin, now, hop_scale, dint.data(), status) : INF;
}

extern "C" void oracle_plan(uint64_t n, const uint32_t *rec, const float *d, const uint8_t *resident_in,
                            const float *theta, uint64_t budget, uint8_t *resident_out,
                            uint32_t *prefetch, uint64_t *n_prefetch, uint32_t *evict, uint64_t *n_evict,
                            uint64_t *out, uint32_t *status) {
  /* 1. eligible agents (R4): resident, or d == 0 (on-demand), or d < theta_class
   *    ("invocation distance below a predefined threshold"). */
  std::vector<std::pair<uint64_t, uint64_t>> order; /* (key, id) */
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t cl = class_of(rec, i);
    float th = (cl < 3) ? theta[cl] : 0.0f;
    bool elig = resident_in[i] != 0 || d[i] == 0.0f || d[i] < th;
    if (!elig) continue;
    /* R1: one total order, key (d, id) ascending; d >= +0 so its bit pattern is monotone */
    uint64_t key = ((uint64_t)f32_bits(d[i]) << 32) | (uint64_t)i;
    order.push_back({key, i});
  }
  std::sort(order.begin(), order.end());

  /* 2. R3: keep the maximal prefix of that order whose bytes fit in the budget; stop at
   *    the first agent that does not fit. */
  for (uint64_t i = 0; i < n; ++i) resident_out[i] = 0;
  uint64_t used = 0, cut_bits = 0xFFFFFFFFull, cut_rem = 0;
  uint64_t bytes_before_cut_value = 0; /* bytes of eligible agents with d < D* */
  bool stopped = false;
  for (size_t k = 0; k < order.size(); ++k) {
    uint64_t i = order[k].second;
    uint64_t fp = footprint_of(rec, i);
    if (used + fp > budget) {
      stopped = true;
      cut_bits = order[k].first >> 32;
      break;
    }
    used += fp;
    resident_out[i] = 1;
  }
  if (stopped) {
    for (size_t k = 0; k < order.size(); ++k)
      if ((order[k].first >> 32) < cut_bits) bytes_before_cut_value += footprint_of(rec, order[k].second);
    cut_rem = budget - bytes_before_cut_value;
  } else {
    cut_rem = budget - used;
  }

  /* 3. Lists (R14): prefetch = kept and not resident, ascending key (most urgent first);
   *    evict = resident and not kept, descending key (largest distance first). */
  uint64_t np = 0, ne = 0, h2d = 0;
  for (size_t k = 0; k < order.size(); ++k) {
    uint64_t i = order[k].second;
    if (resident_out[i] && !resident_in[i]) {
      prefetch[np++] = (uint32_t)i;
      h2d += footprint_of(rec, i);
    }
  }
  for (size_t k = order.size(); k-- > 0;) {
    uint64_t i = order[k].second;
    if (resident_in[i] && !resident_out[i]) evict[ne++] = (uint32_t)i;
  }
  /* Residents are always eligible, so every resident agent appears in `order`. */

  /* 4. R11: INSUFFICIENT when an agent with d == 0 (active, pinned) is not kept. */
  for (uint64_t i = 0; i < n; ++i)
    if (d[i] == 0.0f && !resident_out[i]) *status |= ORACLE_ST_INSUFFICIENT;

  *n_prefetch = np;
  *n_evict = ne;
  out[0] = h2d;
  out[1] = cut_bits;
  out[2] = cut_rem;
  out[3] = used;
  out[4] = order.size();
}

/* ---------------------------------------------------------------------------------- */
/* Paged device arena: DESIGN.md §4.3 (blocks = runs of fixed-size pages, FIFO free pool) */

struct oracle_mem {
  uint64_t n_agents = 0, page_bytes = 0, n_pages = 0;
  std::vector<uint64_t> blk_ptr, blk_host_off, page_first;
  std::vector<uint32_t> blk_size;
  std::vector<uint8_t> blk_kind;
  std::vector<uint32_t> page_table; /* per block page: device page or 0xFFFFFFFF */
  std::vector<uint32_t> ring;       /* free device pages, FIFO */
  uint64_t head = 0, tail = 0;      /* pop at head, push at tail; free = tail - head */
};

static bool pool_pop(oracle_mem *m, uint32_t *pg) {
  if (m->head == m->tail) return false;
  *pg = m->ring[m->head % m->n_pages];
  m->head++;
  return true;
}
static void pool_push(oracle_mem *m, uint32_t pg) {
  m->ring[m->tail % m->n_pages] = pg;
  m->tail++;
}

extern "C" oracle_mem *oracle_mem_create(uint64_t n_agents, const uint64_t *blk_ptr, const uint32_t *blk_size,
                                         const uint64_t *blk_host_off, const uint8_t *blk_kind,
                                         uint64_t page_bytes, uint64_t n_pages, const uint8_t *resident_init) {
  oracle_mem *m = new oracle_mem();
  m->n_agents = n_agents;
  m->page_bytes = page_bytes;
  m->n_pages = n_pages;
  uint64_t nb = blk_ptr[n_agents];
  m->blk_ptr.assign(blk_ptr, blk_ptr + n_agents + 1);
  m->blk_size.assign(blk_size, blk_size + nb);
  m->blk_host_off.assign(blk_host_off, blk_host_off + nb);
  m->blk_kind.assign(blk_kind, blk_kind + nb);
  m->page_first.resize(nb + 1);
  m->page_first[0] = 0;
  for (uint64_t b = 0; b < nb; ++b) m->page_first[b + 1] = m->page_first[b] + blk_size[b] / page_bytes;
  m->page_table.assign(m->page_first[nb], 0xFFFFFFFFu);
  m->ring.resize(n_pages);
  for (uint64_t p = 0; p < n_pages; ++p) m->ring[p] = (uint32_t)p;
  m->head = 0;
  m->tail = n_pages;
  /* initially resident agents take pages in id order, block order, page order */
  if (resident_init)
    for (uint64_t a = 0; a < n_agents; ++a)
      if (resident_init[a])
        for (uint64_t b = blk_ptr[a]; b < blk_ptr[a + 1]; ++b)
          for (uint64_t p = m->page_first[b]; p < m->page_first[b + 1]; ++p) {
            uint32_t pg = 0xFFFFFFFFu;
            pool_pop(m, &pg);
            m->page_table[p] = pg;
          }
  return m;
}

extern "C" void oracle_mem_destroy(oracle_mem *m) { delete m; }

extern "C" void oracle_mem_apply(oracle_mem *m, const uint32_t *rec, const uint32_t *prefetch, uint64_t n_prefetch,
                                 const uint32_t *evict, uint64_t n_evict, uint64_t *d2h_host, uint32_t *d2h_page,
                                 uint64_t *h2d_host, uint32_t *h2d_page, uint64_t *out, uint32_t *status) {
  uint64_t bytes_d2h = 0, bytes_h2d = 0, nd = 0, nh = 0;
  /* Evict (Table 1 Evict): write back dirty non-LoRA blocks (R13; LoRA adapters are
   * read-only and host-backed), release every page to the pool. */
  for (uint64_t e = 0; e < n_evict; ++e) {
    uint64_t a = evict[e];
    bool dirty = dirty_of(rec, a);
    for (uint64_t b = m->blk_ptr[a]; b < m->blk_ptr[a + 1]; ++b) {
      bool wb = dirty && m->blk_kind[b] != KIND_LORA;
      if (wb) bytes_d2h += m->blk_size[b];
      for (uint64_t p = m->page_first[b]; p < m->page_first[b + 1]; ++p) {
        uint32_t pg = m->page_table[p];
        if (wb) {
          d2h_host[nd] = m->blk_host_off[b] + (p - m->page_first[b]) * m->page_bytes;
          d2h_page[nd] = pg;
          nd++;
        }
        pool_push(m, pg);
        m->page_table[p] = 0xFFFFFFFFu;
      }
    }
  }
  /* Load (Table 1 Load): every block of every prefetched agent, most urgent first. */
  for (uint64_t f = 0; f < n_prefetch; ++f) {
    uint64_t a = prefetch[f];
    for (uint64_t b = m->blk_ptr[a]; b < m->blk_ptr[a + 1]; ++b) {
      bytes_h2d += m->blk_size[b];
      for (uint64_t p = m->page_first[b]; p < m->page_first[b + 1]; ++p) {
        uint32_t pg = 0xFFFFFFFFu;
        if (!pool_pop(m, &pg)) *status |= ORACLE_ST_NO_PAGES;
        m->page_table[p] = pg;
        h2d_host[nh] = m->blk_host_off[b] + (p - m->page_first[b]) * m->page_bytes;
        h2d_page[nh] = pg;
        nh++;
      }
    }
  }
  out[0] = bytes_d2h;
  out[1] = bytes_h2d;
  out[2] = nd;
  out[3] = nh;
}

extern "C" uint64_t oracle_mem_total_pages(const oracle_mem *m) { return m->page_table.size(); }

extern "C" void oracle_mem_page_table(const oracle_mem *m, uint32_t *page_table) {
  std::copy(m->page_table.begin(), m->page_table.end(), page_table);
}

extern "C" void oracle_mem_pool(const oracle_mem *m, uint64_t *head, uint64_t *tail, uint32_t *ring) {
  *head = m->head;
  *tail = m->tail;
  if (ring) std::copy(m->ring.begin(), m->ring.end(), ring);
}

// ---------------------------------------------------------------------------------------
// Shared memory objects: P:459-463 (fine-grained distance assignment), R19.

void oracle_object_min(uint64_t n_agents, const float *agent_dist, uint64_t n_obj, const uint64_t *ref_ptr,
                       const uint32_t *ref_agent, float *d_obj, uint32_t *status) {
  uint32_t st = 0;
  for (uint64_t o = 0; o < n_obj; ++o) {
    // "the minimum invocation distance among all agents that currently reference it"
    float m = std::numeric_limits<float>::infinity();  // no referrer: +inf
    for (uint64_t k = ref_ptr[o]; k < ref_ptr[o + 1]; ++k) {
      const uint32_t a = ref_agent[k];
      if (a >= n_agents) {
        st |= ORACLE_ST_BAD_RECORD;
        continue;
      }
      float x = agent_dist[a];
      if (std::isnan(x) || x < 0.0f) {
        st |= ORACLE_ST_BAD_RECORD;
        x = std::numeric_limits<float>::infinity();
      }
      if (x < m) m = x;
    }
    if (m == 0.0f) m = 0.0f;  // -0 -> +0
    d_obj[o] = m;
  }
  *status |= st;
}

void oracle_explicit_dist(uint64_t n, const uint32_t *rec, float *d_out, uint32_t *status) {
  uint32_t st = 0;
  for (uint64_t i = 0; i < n; ++i) {
    float x;
    std::memcpy(&x, &rec[4 * i], sizeof(float));
    if (std::isnan(x) || x < 0.0f) {
      st |= ORACLE_ST_BAD_RECORD;
      x = std::numeric_limits<float>::infinity();
    }
    if (x == 0.0f) x = 0.0f;
    d_out[i] = x;
  }
  *status |= st;
}

// ---------------------------------------------------------------------------------------
// LRU baseline (R20): recency as a distance.

void oracle_lru_records(uint64_t n, const uint32_t *rec, int64_t now, uint32_t *last_use, uint32_t *rec_out) {
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t phase = rec[4 * i + 2] & 3u;
    float d;
    if (phase == PH_WAITING || phase == PH_GENERATING) {  // the agent's memory is in use now
      last_use[i] = (uint32_t)now;
      d = 0.0f;
    } else if (last_use[i] == 0xFFFFFFFFu) {
      d = std::numeric_limits<float>::infinity();  // never used
    } else {
      d = (float)(uint32_t)((uint32_t)now - last_use[i]);  // steps since the last use
    }
    uint32_t bits;
    std::memcpy(&bits, &d, sizeof(bits));
    rec_out[4 * i + 0] = bits;
    rec_out[4 * i + 1] = rec[4 * i + 1];
    rec_out[4 * i + 2] = rec[4 * i + 2] & 0x10u;
    rec_out[4 * i + 3] = 0;
  }
}

// ---------------------------------------------------------------------------------------
// Diffusion hop counts: P:229, R9 (plain FIFO breadth-first search).

void oracle_bfs_hops(uint64_t n, const uint64_t *row_ptr, const uint32_t *col, const uint32_t *sources,
                     uint64_t n_sources, uint32_t *hops) {
  for (uint64_t v = 0; v < n; ++v) hops[v] = 0xFFFFFFFFu;
  std::vector<uint32_t> queue;
  for (uint64_t k = 0; k < n_sources; ++k) {
    const uint32_t s = sources[k];
    if (s < n && hops[s] == 0xFFFFFFFFu) {
      hops[s] = 0;
      queue.push_back(s);
    }
  }
  for (size_t head = 0; head < queue.size(); ++head) {
    const uint32_t u = queue[head];
    for (uint64_t k = row_ptr[u]; k < row_ptr[u + 1]; ++k) {
      const uint32_t w = col[k];
      if (w < n && hops[w] == 0xFFFFFFFFu) {
        hops[w] = hops[u] + 1;
        queue.push_back(w);
      }
    }
  }
}

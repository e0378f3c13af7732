"""GPU parity of the shared-object path (NEXT #1: P:459-463, reading R19):
scalesim_object_min against the oracle bit for bit, and the whole pipeline (agent plan ->
object distances -> object plan with explicit distances) against the oracle."""
import numpy as np
import pytest
import torch

import oracle
import tracegen as tg
from helpers import rec_of

pytestmark = pytest.mark.gpu

PATHS = [pytest.param(False, id="fused"), pytest.param(True, id="multikernel")]


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2601_21473_b200 import build
    build.build()


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_object_min_edge_cases():
    from paper_2601_21473_b200.planner import object_min
    rng = np.random.default_rng(11)
    n = 5000
    dist = rng.integers(0, 300, n).astype(np.float32)
    dist[rng.random(n) < 0.1] = np.inf
    dist[3] = -0.0
    lists = [list(rng.integers(0, n, int(k))) for k in rng.integers(0, 12, 3000)]
    lists[5] = []                                   # no referrer
    lists[7] = list(rng.integers(0, n, 20000))      # one long segment
    lists[9] = [n + 4, 1]                           # out-of-range agent index
    lists[11] = [3]                                 # -0 reads as +0
    ptr = np.zeros(len(lists) + 1, np.uint64)
    ptr[1:] = np.cumsum([len(x) for x in lists])
    ag = np.array([a for x in lists for a in x], np.uint32)
    d_or, st_or = oracle.object_min(dist, ptr, ag)
    n_obj = len(lists)
    nbytes = rng.integers(1, 100, n_obj).astype(np.uint32) * tg.PAGE_BYTES
    flags = (rng.random(n_obj) < 0.5).astype(np.uint32) << 4
    rec = torch.zeros(16 * n_obj, dtype=torch.uint8, device="cuda")
    dout = torch.zeros(n_obj, dtype=torch.float32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    object_min(_dev(dist), _dev(ptr), _dev(ag), _dev(nbytes), rec, obj_flags=_dev(flags), dist_out=dout, status=st)
    torch.cuda.synchronize()
    got = dout.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), d_or.view(np.uint32))
    r = rec.cpu().numpy().view(np.uint32).reshape(-1, 4)
    assert np.array_equal(r[:, 0], d_or.view(np.uint32)) and np.array_equal(r[:, 1], nbytes)
    assert np.array_equal(r[:, 2], flags) and not r[:, 3].any()
    assert int(st.item()) == st_or == oracle.ST_BAD_RECORD


@pytest.mark.parametrize("mk", PATHS)
def test_object_pipeline_vs_oracle(mk):
    """Agents (C2 shape, 3000 agents) -> object distances (prompt shared by all, 30 persona
    adapters, private KV pages) -> object plan, every step element by element."""
    from paper_2601_21473_b200.planner import Planner, object_min
    w = tg.config_c2(seed=3, steps=10, n=3000)
    ob = tg.gen_objects(w.n, seed=3, personas=30)
    stream = torch.cuda.Stream()
    b = w.blocks
    agents = Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta, transfer=False,
                     keep_dist=True, multi_kernel=mk, stream=stream)
    ob_budget = int(ob.obj_bytes.astype(np.int64).sum()) // 4
    bo = ob.blocks
    objs = Planner(ob.n, bo.blk_ptr, bo.blk_size, bo.blk_host_off, bo.blk_kind, ob_budget, w.theta, transfer=False,
                   keep_dist=True, multi_kernel=mk, stream=stream, explicit_dist=True)
    assert agents.fused == (not mk) and objs.fused == (not mk)
    ptr_t, ag_t, by_t = _dev(ob.ref_ptr), _dev(ob.ref_agent), _dev(ob.obj_bytes)
    dobj = torch.zeros(ob.n, dtype=torch.float32, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    res = np.zeros(ob.n, np.uint8)
    for s in range(w.steps):
        agents.set_records(w.rec[s])
        agents.step(int(w.now[s]))
        flags = ob.flags(w.rec[s])
        with torch.cuda.stream(stream):
            fl_t = _dev(flags)
            object_min(agents.dist_tensor(), ptr_t, ag_t, by_t, objs.rec, obj_flags=fl_t, dist_out=dobj, status=st,
                       stream=stream)
        objs.step(int(w.now[s]))
        hdr = objs.sync()
        # oracle
        d_ag, _ = oracle.score(w.rec[s], None, int(w.now[s]))
        d_ob, st_or = oracle.object_min(d_ag, ob.ref_ptr, ob.ref_agent)
        orec = tg.object_records(d_ob.view(np.uint32), ob, flags)
        dx, _ = oracle.explicit_dist(orec)
        p = oracle.plan(orec, dx, res, w.theta, ob_budget)
        assert np.array_equal(dobj.cpu().numpy().view(np.uint32), d_ob.view(np.uint32)), s
        assert np.array_equal(objs.distances().view(np.uint32), dx.view(np.uint32)), s
        pf, ev = objs.lists(hdr)
        assert np.array_equal(pf, p["prefetch"]) and np.array_equal(ev, p["evict"]), s
        assert np.array_equal(objs.resident(), p["resident"])
        assert hdr["cut_bits"] == p["cut_bits"] and hdr["cut_rem"] == p["cut_rem"]
        assert hdr["bytes_h2d"] == p["bytes_h2d"] and hdr["kept_bytes"] == p["kept_bytes"]
        assert (hdr["status"] & ~oracle.ST_NO_PAGES) == (p["status"] & oracle.ST_INSUFFICIENT)
        res = p["resident"]
    # the shared prompt is resident whenever any active agent needs it
    assert res[0] == 1
    agents.close()
    objs.close()


def test_explicit_records_with_transfers():
    """Explicit-distance planning with physical page copies (harness: content, pages,
    descriptors), including malformed distance words."""
    from gpu_harness import run_parity
    rng = np.random.default_rng(4)
    n, steps = 1500, 5
    fp = rng.choice([1, 2, 3], n) * tg.PAGE_BYTES
    blocks = tg.make_blocks([[tg.KIND_KV]] * n, [[int(f)] for f in fp])
    recs = []
    for s in range(steps):
        d = rng.choice([0.0, 1.0, 2.5, 3.0, 9.75, 40.0, np.inf], n).astype(np.float32)
        r = np.zeros((n, 4), np.uint32)
        r[:, 0] = d.view(np.uint32)
        r[:, 1] = fp
        r[:, 2] = (rng.random(n) < 0.3).astype(np.uint32) << 4
        if s == 2:
            r[5, 0] = 0x7FC00000   # NaN
            r[6, 0] = np.float32(-1.0).view(np.uint32)
            r[7, 0] = 0x80000000   # -0
        recs.append(r)
    w = tg.Workload("explicit", n, np.zeros(steps, np.int64), np.stack(recs), None, blocks,
                    int(fp.sum() * 0.3), np.full(3, 5.0, np.float32))
    run_parity(w, explicit=True)
    run_parity(w, explicit=True, multi_kernel=True)


def test_bfs_hops_vs_oracle():
    """scalesim_bfs_hops (R9, NEXT #4): BFS levels on a 100k-vertex Barabasi-Albert graph
    (C3's diffusion graph shape) from 8 sources, plus a graph with unreachable parts, equal
    the oracle's FIFO BFS."""
    from paper_2601_21473_b200.planner import bfs_hops
    for n, m, extra in ((100_000, 4, 0), (5000, 2, 300)):
        adj = tg.ba_graph(n, m, seed=n)
        adj = adj + [[] for _ in range(extra)]  # isolated vertices
        ptr = np.zeros(len(adj) + 1, np.uint64)
        ptr[1:] = np.cumsum([len(a) for a in adj])
        col = np.array([w for a in adj for w in a], np.uint32)
        src = np.random.default_rng(n).choice(n, 8, replace=False).astype(np.uint32)
        exp = oracle.bfs_hops(ptr, col, src)
        got = bfs_hops(_dev(ptr), _dev(col), _dev(src)).cpu().numpy().view(np.uint32)
        assert np.array_equal(got, exp)
        assert np.array_equal(exp.astype(np.int64), np.where(tg.bfs_hops(adj, src) == tg.UNREACHABLE, 0xFFFFFFFF,
                                                             tg.bfs_hops(adj, src)))

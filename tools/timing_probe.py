"""Compare eager (spin-prefilled) vs CUDA-graph timing of the same steps, and their results."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import tracegen as tg
from paper_2601_21473_b200.planner import Planner

K = int(os.environ.get("K", "16"))
w = tg.config_c4(seed=1, steps=16 + K)
dev = torch.device("cuda", 0)
recs = torch.from_numpy(np.ascontiguousarray(w.rec).view(np.uint8).reshape(w.steps, -1)).to(dev)
ptr = [recs[s].data_ptr() for s in range(w.steps)]
b = w.blocks
res = {}
for mode in ("eager", "graph", "eager_sync"):
    pl = Planner(w.n, b.blk_ptr, b.blk_size, b.blk_host_off, b.blk_kind, w.budget, w.theta, transfer=False,
                 keep_dist=False)
    for s in range(16):
        pl.set_inputs_ptr(ptr[s]); pl.step(int(w.now[s]))
    pl.sync()
    def steps():
        for k in range(K):
            s = 16 + k
            pl.set_inputs_ptr(ptr[s]); pl.score(int(w.now[s])); pl.plan(); pl.transfer()
        pl.join()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    if mode == "graph":
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=pl.stream):
            steps()
        torch.cuda.synchronize()
        pl.stamps(reset=True)
        with torch.cuda.stream(pl.stream):
            t0.record(pl.stream); g.replay(); t1.record(pl.stream)
        torch.cuda.synchronize()
        st = pl.stamps().astype(np.int64)
        print("graph stamps: span of all launches (us)", (st[1]-st[0])/1e3, "last launch cta0 phases",
              [(st[i]-st[2])/1e3 if st[i] else None for i in range(3, 11)])
    elif mode == "eager":
        with torch.cuda.stream(pl.stream):
            torch.cuda._sleep(int(1e8))
        t0.record(pl.stream); steps(); t1.record(pl.stream)
    else:
        torch.cuda.synchronize()
        ts = []
        for k in range(K):
            s = 16 + k
            pl.set_inputs_ptr(ptr[s])
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            pl.stamps(reset=True)
            torch.cuda.synchronize()
            e0.record(pl.stream); pl.score(int(w.now[s])); pl.plan(); e1.record(pl.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            st = pl.stamps().astype(np.int64)
            if k < 4:
                r = lambda q: round((int(st[q]) - int(st[0])) / 1e3, 2) if st[q] else None
                print("us: cta0 P1end", r(3), "B1", r(4), "sel", r(9), "P3", r(10), "P4end", r(5), "B4", r(6),
                      "P5tab", r(7), "| max over CTAs: P1end", r(11), "P3end", r(14), "P4loop", r(27), "P4lists", r(17), "P4ranks", r(19), "P4rows", r(28),
                      "P4end", r(12), "B4max", r(30), "P5tot", r(31), "P5tables", r(13), "end", r(1), "| slots", int(st[16]), "max_sorted_seg", int(st[18]),
                      "slot_loop_ns_max", int(st[21]), "sections(seg+col, gather, scan, place) ns max", [int(st[q]) for q in (22, 23, 24, 29)],
                      "| fast: owner landed", r(40), "o.pass1", r(46), "o.scan", r(47), "owner done", r(41), "need", r(42), "positions", r(17), "members", r(38), "pf placed", r(43), "ev placed", r(44), "placed", r(39), "paths", (int(st[48]), int(st[49])), "| P1loop", r(25), "P1pub", r(26), "| last CTA start", r(15), "| cta0 select: cleared", r(32), "coarse", r(33), "fine", r(34), "barrier", r(35), "| members sub: sums", r(50), "pre-scan", r(51), "scan", r(52), "lists+sync", r(53), "positions", r(54))
        print("eager_sync per-step ms", np.round(ts, 4))
        t0.record(pl.stream); t1.record(pl.stream)
    torch.cuda.synchronize()
    h = pl.sync()
    pf, ev = pl.lists(h)
    res[mode] = (pl.resident(), pf, ev, h)
    print(mode, "ms/step", t0.elapsed_time(t1) / K, "seq", h["seq"], "npf", h["n_prefetch"], "nev", h["n_evict"], flush=True)
    pl.close()
for m in ("graph", "eager_sync"):
    same = all(np.array_equal(a, c) for a, c in zip(res["eager"][:3], res[m][:3]))
    print("eager vs", m, "identical:", same)

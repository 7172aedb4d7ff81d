#!/usr/bin/env python3
"""Pipeline timeline of the tcgen05 search (diagnostics): builds libfic_trace.so with
-DFIC_TC_TRACE, runs one level search of C3 per B (every range of the level, its entropy pool)
and prints, for CTA 0, the median cycles between the pipeline events (fic_tc.cu TC_TR):

  copy->full   bulk copy issued -> MMA warp sees the stage      (feed latency)
  copy gap     between consecutive copy issues                  (feed throughput)
  tfull wait   epilogue warp 2: previous tile done -> sees next tile
  ld           sees tile -> its TMEM loads done
  compute      loads done -> tile done
  tile         between consecutive tiles (epilogue warp 2)

  python scripts/tc_trace.py [B ...]
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SO = os.path.join(ROOT, "paper_1501_04140_b200", "libfic_trace.so")


def main():
    from paper_1501_04140_b200 import build as b
    if not os.path.exists(SO) or os.environ.get("FIC_TRACE_REBUILD"):
        b.build_variant(SO, defines=["FIC_TC_TRACE"] + os.environ.get("FIC_TRACE_DEFS", "").split())
    os.environ["FIC_SO"] = SO
    import torch
    from paper_1501_04140_b200 import fic
    from fic_inputs import config, image_for
    lib = fic.load(SO)
    lib.fic_debug_tc_trace.argtypes = [C.c_void_p]
    cfg = config("C3")
    img_np = image_for(cfg)
    img = torch.from_numpy(img_np).cuda()
    ctx = fic.Context(0)
    Bs = [int(x) for x in sys.argv[1:]] or [16, 8, 4]
    for B in Bs:
        li = [16, 8, 4, 2].index(B)
        pool = ctx.build_domain_pool(img, B, cfg["L"], cfg["tau"][li])
        N = cfg["N"]
        ranges = np.array([(u * B, v * B) for v in range(N // B) for u in range(N // B)], np.int32)
        dr = torch.from_numpy(ranges).cuda()
        tr = np.zeros((32, 4096), np.int64)
        for rep in range(3):
            tr[:] = 0
            ctx.encode_level(img, pool, dr, cfg["s"][li], 8.0, False)
            torch.cuda.synchronize()
            lib.fic_debug_tc_trace(tr.ctypes.data_as(C.c_void_p))
        st, en = tr[30][:4096], tr[31][:4096]
        live = en > 0
        if live.any():
            t0 = st[live].min()
            dur = (en[live] - st[live]) / 1e3
            fin = (en[live] - t0) / 1e3
            print(f"B={B}: {int(live.sum())} CTAs: duration us min {dur.min():.1f} med {np.median(dur):.1f} max {dur.max():.1f};"
                  f" finish us med {np.median(fin):.1f} max {fin.max():.1f}; start spread {(st[live].max() - t0) / 1e3:.1f}")
            nit, nsg = tr[28][:4096][live], tr[27][:4096][live]
            order = np.argsort(-dur)[:6]
            print("   slowest CTAs: dur us", np.round(dur[order], 1), "items", nit[order], "segments", nsg[order])
            print("   items per CTA med", np.median(nit), "max", nit.max(), "; segments med", np.median(nsg), "max", nsg.max())
            if os.environ.get("FIC_TRACE_SEG"):
                cids = np.nonzero(live)[0][order[:3]]
                for c in cids:
                    row = lambda kd: tr[kd][c * 8: c * 8 + 8]  # noqa: E731
                    s23, s24, s25, s26 = row(23), row(24), row(25), row(26)
                    for kk in range(int(tr[27][c])):
                        s20, s21, s22 = row(20), row(21), row(22)
                        print(f"   CTA {c} seg {kk}: start {(s23[kk] - st[c]) / 1e3:.1f} us, setup {(s20[kk] - s23[kk]) / 1e3:.2f}"
                              f" seed wait {(s21[kk] - s20[kk]) / 1e3:.2f} own seed {(s22[kk] - s21[kk]) / 1e3:.2f} wg bar {(s24[kk] - s22[kk]) / 1e3:.2f},"
                              f" tiles {(s25[kk] - s24[kk]) / 1e3:.1f}, drain {(s26[kk] - s25[kk]) / 1e3:.1f}")
                    print(f"   CTA {c} end {(en[c] - st[c]) / 1e3:.1f} us")
        wb = tr[29][0:64:2]; ww = tr[29][1:64:2]
        live_w = np.nonzero(wb > 0)[0]
        if len(live_w):
            print("   per epilogue warp (warp: SMSP busy/wait kcycles):",
                  " ".join(f"w{w}:{w % 4} {wb[w] / 1e3:.0f}/{ww[w] / 1e3:.0f}" for w in live_w))
            pc, pn = tr[29][64:128:2], tr[29][65:128:2]
            print("   push blocks per warp (kcycles / count / cycles each):",
                  " ".join(f"w{w} {pc[w] / 1e3:.0f}/{pn[w]}/{pc[w] / max(pn[w], 1):.0f}" for w in live_w))
        n_t = int((tr[6] > 0).sum())
        n_i = int((tr[0] > 0).sum())
        med = lambda a: float(np.median(a)) if len(a) else float("nan")  # noqa: E731
        c0, c1 = tr[0][:n_i], tr[1][:n_i]
        t4, t5, t6, t7 = tr[4][:n_t], tr[5][:n_t], tr[6][:n_t], tr[7][:n_t]
        t2, t3 = tr[2][:n_t], tr[3][:n_t]
        span = (t6[-1] - t4[0]) if n_t > 1 else 0
        print(f"B={B}: CTA 0 ran {n_t} tiles ({n_i} stages) in {span} cycles = {span / max(n_t, 1):.0f}/tile")
        print(f"  copy->full {med(c1 - c0):.0f}  copy gap {med(np.diff(c0)):.0f}  "
              f"mma: free->commit {med(t3 - t2):.0f}  commit gap {med(np.diff(t3)):.0f}")
        print(f"  epi2: tfull wait {med(t4[1:] - t6[:-1]):.0f}  ld {med(t5 - t4):.0f}  compute {med(t6 - t5):.0f}  "
              f"tile {med(np.diff(t6)):.0f}  last warp lag {med(t7 - t6):.0f}  commit->seen {med(t4 - t3):.0f}")
        nw = int((tr[8:20, 100] > 0).sum()) if n_t > 100 else 0
        if nw:
            ld = tr[8:8 + nw, :n_t].astype(np.float64)  # per epilogue warp, per tile: loads done
            lag = ld - np.median(ld, axis=0)
            last = np.argmax(ld, axis=0)
            print("   per warp (w:SMSP): mean lag vs median warp (cycles) / share of tiles it loads last:")
            print("   " + " ".join(f"w{w + 2}:{(w + 2) % 4} {lag[w].mean():.0f}/{(last == w).mean():.2f}" for w in range(nw)))
            spread = ld.max(axis=0) - ld.min(axis=0)
            print(f"   load spread across warps per tile: p10 {np.percentile(spread, 10):.0f} p50 {np.median(spread):.0f} p90 {np.percentile(spread, 90):.0f}")
        if os.environ.get("FIC_TRACE_DUMP") and n_t > 110 and n_i == n_t:
            base = t4[100]
            print("  tile  copy  full  free  commit  seen  loaded  done  lastdone   (cycles from tile 100 seen)")
            nw = int((tr[8:, 100] > 0).sum())
            for t in range(98, 108):
                print("  %4d %6d %6d %6d %6d %6d %6d %6d %6d" % (t, c0[t] - base, c1[t] - base, t2[t] - base, t3[t] - base,
                                                             t4[t] - base, t5[t] - base, t6[t] - base, t7[t] - base))
                print("        per-warp loaded:", " ".join("%d" % (tr[8 + w][t] - base) for w in range(nw)))
        for q in (10, 50, 90):
            print(f"  p{q}: compute {np.percentile(t6 - t5, q):.0f}  tfull wait {np.percentile(t4[1:] - t6[:-1], q):.0f}"
                  f"  copy->full {np.percentile(c1 - c0, q):.0f}")


if __name__ == "__main__":
    main()

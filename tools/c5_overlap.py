#!/usr/bin/env python
"""C5 overlap experiment: tet + prism launches back to back vs concurrent on two streams,
with static round-robin tiles or the dynamic tile queue (fek_batch_desc.scheduler)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from bench import Launcher, c5_parts
    from paper_1504_01023_b200 import mesh

    parts = c5_parts(1, 0)
    data = [(desc, lo) + mesh.device_config(cfg, lo, n) for cfg, desc, lo, n in parts]
    LS = [Launcher(desc, g, c, base_index=lo, dynamic=False) for desc, lo, g, c in data]
    LD = [Launcher(desc, g, c, base_index=lo, dynamic=True) for desc, lo, g, c in data]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=7):
        fn()
        torch.cuda.synchronize()
        out = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1))
        return sorted(out)[len(out) // 2]

    def conc(L, cap_t, cap_p, first):
        cur = torch.cuda.current_stream()

        def run():
            L[0].dd.ctas_per_sm, L[1].dd.ctas_per_sm = cap_t, cap_p
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            order = [(0, s1), (1, s2)] if first == "tet" else [(1, s2), (0, s1)]
            for idx, st in order:
                L[idx].stream = st.cuda_stream
                L[idx]()
            cur.wait_stream(s1)
            cur.wait_stream(s2)
        return run

    def reset(L):
        for x in L:
            x.stream = torch.cuda.current_stream().cuda_stream
            x.dd.ctas_per_sm = 0

    for name, L in (("static", LS), ("dynamic", LD)):
        print(name, "tet alone", timed(lambda: L[0]()), "prism alone", timed(lambda: L[1]()))
        print(name, "sequential ms", timed(lambda: (L[0](), L[1]())))
        for cap_t, cap_p, first in ((1, 0, "tet"), (1, 1, "tet"), (0, 0, "tet"), (0, 0, "prism"), (1, 0, "prism")):
            print(f"{name} concurrent tet_cap={cap_t} prism_cap={cap_p} first={first} ms",
                  timed(conc(L, cap_t, cap_p, first)))
            reset(L)
    # mixed: static tets pinned to 1 CTA/SM, prisms on the dynamic queue fill the rest
    M = [LS[0], LD[1]]
    for cap_t in (1, 2):
        print(f"mixed tet static cap={cap_t} + prism dynamic ms", timed(conc(M, cap_t, 0, "tet")))
        reset(M)
    # bitwise check: dynamic == static results
    for a, b in zip(LS, LD):
        a(); b()
        torch.cuda.synchronize()
        print("bitwise equal", torch.equal(a.A, b.A) and torch.equal(a.b, b.b), "sched words", b.sched.tolist())


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""C5 overlap experiment: tet + prism launches back to back vs concurrent on two streams."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

def main():
    import torch
    from bench import Launcher, c5_parts
    from paper_1504_01023_b200 import mesh
    parts = c5_parts(1, 0)
    L = []
    for cfg, desc, lo, n in parts:
        g, c = mesh.device_config(cfg, lo, n)
        L.append(Launcher(desc, g, c, base_index=lo))
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        fn(); torch.cuda.synchronize()
        out = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1))
        return sorted(out)[len(out) // 2]

    def seq():
        L[0](); L[1]()

    def conc(cap_t, cap_p, first):
        L[0].dd.ctas_per_sm, L[1].dd.ctas_per_sm = cap_t, cap_p
        cur = torch.cuda.current_stream()
        def run():
            s1.wait_stream(cur); s2.wait_stream(cur)
            order = [(0, s1), (1, s2)] if first == "tet" else [(1, s2), (0, s1)]
            for idx, st in order:
                L[idx].stream = st.cuda_stream
                L[idx]()
            cur.wait_stream(s1); cur.wait_stream(s2)
        return run
    print("sequential ms", timed(seq))
    for cap_t, cap_p, first in ((1, 0, "tet"), (1, 1, "tet"), (0, 0, "tet"), (0, 1, "prism"), (1, 0, "prism")):
        print(f"concurrent tet_cap={cap_t} prism_cap={cap_p} first={first} ms", timed(conc(cap_t, cap_p, first)))
        L[0].stream = L[1].stream = torch.cuda.current_stream().cuda_stream
        L[0].dd.ctas_per_sm = L[1].dd.ctas_per_sm = 0
    print("tet alone", timed(lambda: L[0]()), "prism alone", timed(lambda: L[1]()))

if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py -- elements integrated per second on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...           (N > 1; plain `python bench.py
                                                                --gpus N` starts torchrun itself)

Headline workload (N=1, BASELINE.json configs[1] -> SURVEY config C2):
generalized convection-diffusion-reaction on 4,088,832 linear tetrahedra
(88^3 Kuhn cells), per-element coefficients, fp64, natural QSS geo_linear
descriptor.  One step = one ``fek_integrate`` launch over the whole batch.
Scaling is weak: every rank integrates its own C2-sized range of a
(rank-seeded) mesh, base_index = rank*n, no collective on the hot path.

Printed JSON (rank 0, one line):
  value      whole-job elements/s, inputs already in HBM (device events, max
             over ranks; 1.7 GB of traffic per step >> 126 MB L2);
  e2e        same metric through the public API ``integrate_batch(desc,
             host_batch)`` with page-locked host buffers: H2D + kernel + D2H
             inside the timed region;
  roofline   of the integration kernel (algorithmic bytes / launch time vs the
             measured HBM copy peak);
  cpu_baseline  the reference algorithm (oracle port) on all host cores;
  cases      C1/C3/C4 (fp64, C4 also fp32) kernel timings + rooflines;
  parity     GPU vs CPU oracle on the full C2 batch and on case samples.

``--impl reference`` times the reference's CPU algorithm (oracle port) on the
same workload, on rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "elements integrated/sec (fp64) at 1/2/4/8 B200; % of HBM/FP64 roofline"
UNIT = "elements/s"
L2_BYTES = 126 * 2 ** 20


def parse(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[1])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--cases", default="C1,C3,C4,C4f32,C5,C2packed",
                    help="extra per-config kernel timings (N=1 only)")
    ap.add_argument("--no-cases", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-processes", type=int, default=None)
    ap.add_argument("--variant", default="qss", choices=("qss", "sqs", "ssq"))
    return ap.parse_args(argv)


def launched_by_torchrun() -> bool:
    """Under torchrun (any N, including 1) the NCCL process group is initialised."""
    return "WORLD_SIZE" in os.environ and "MASTER_ADDR" in os.environ


def _config_record(cfg, n_per_rank, world, desc, extra=None):
    rec = {
        "workload": f"{cfg.key}: {cfg.text}",
        "mesh": f"{cfg.spec.nx}x{cfg.spec.ny}x{cfg.spec.nz} {cfg.spec.element_type.value}",
        "elements_per_gpu": n_per_rank,
        "elements_total": n_per_rank * world,
        "descriptor": desc.short_name(),
        "layout": "element-major",
        "parallelism": f"element-range shards x{world} (no collective on the hot path)",
        "l2": f"per-step traffic {n_per_rank * 416 / 1e9:.2f} GB > {L2_BYTES / 2**20:.0f} MiB L2 (no reuse)",
    }
    if extra:
        rec.update(extra)
    return rec


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args) -> int:
    from oracle.cpu_baseline import PortPool, cpu_cores
    from paper_1504_01023_b200 import KernelDescriptor, mesh, natural_path
    from paper_1504_01023_b200.distributed import env_rank
    from paper_1504_01023_b200.problems import Variant

    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    cores = cpu_cores()
    procs = args.cpu_processes or cores["logical"] or 1
    keys = ("C5T", "C5P") if args.config == "C5" else (args.config,)
    sample_each = (1 << 19) // len(keys)
    sec, sample = 0.0, 0
    for key in keys:
        cfg = mesh.bench_configs()[key]
        et, pb = cfg.spec.element_type, cfg.problem
        desc = KernelDescriptor(Variant(args.variant), natural_path(et), pb, et)
        # host rows of a contiguous sample window only (the reference generator
        # is sequential; C5 is 64M elements): first `window` elements
        window = min(cfg.spec.n_elements, 4 * sample_each)
        if cfg.spec.n_elements <= (1 << 23):
            geo, cof = mesh.config_rows(cfg)
        else:
            import torch

            g, c = mesh.device_config(cfg, 0, window) if torch.cuda.is_available() else (None, None)
            if g is None:
                geo, cof = mesh.config_rows(cfg)
            else:
                geo = g.cpu().numpy().reshape(window, -1)
                cof = c.cpu().numpy().reshape(window, -1)
        n = geo.shape[0]
        part = min(n, sample_each)
        times = []
        with PortPool(desc.variant.value, desc.geometry_path.value, pb.value, et.value, geo, cof, procs) as pool:
            warm_until = time.perf_counter() + 1.0  # >= 1 s: worker heaps, page tables, CPU clocks settle
            done = 0
            while done < max(args.warmup, 1) or time.perf_counter() < warm_until:
                pool.run(0, part)
                done += 1
            for _ in range(args.steps):  # same window every step, as the reference's bench repeats its batch
                times.append(pool.run(0, part))
        sec += float(np.mean(times))
        sample += part
    cfg = mesh.bench_configs()[keys[0]]
    desc = KernelDescriptor(Variant(args.variant), natural_path(cfg.spec.element_type), cfg.problem,
                            cfg.spec.element_type)
    n = sum(mesh.bench_configs()[k].spec.n_elements for k in keys)
    value = sample / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference mesh generator, seeded coefficients)",
        "config": _config_record(cfg, n, 1, desc, {"sample_elements_per_step": sample,
                                                   "workload_parts": list(keys)}),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                         "sample": f"{sample} contiguous elements of {cfg.key} per step (oracle port of "
                                   f"feklab integrate_batch, {procs} processes)", "host_cores": cores},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

class Launcher:
    """Prepared fek_integrate call on device tensors (no Python work per launch but ctypes)."""

    def __init__(self, desc, geo, cof, base_index=0, layout=None, packed_layout=None, dynamic=True):
        import torch

        from paper_1504_01023_b200 import ELEMENT_MAJOR, _native
        from paper_1504_01023_b200.kernels.batched import _desc_struct

        self.lib = _native.load()
        et = desc.element
        ns = et.n_shape
        n = geo.numel() // et.geometry_size
        self.n = n
        self.err = torch.full((1,), -1, dtype=torch.int64, device=geo.device)
        self.keep = (geo, cof)
        code = _native.DTYPE["float64" if geo.dtype == torch.float64 else "float32"]
        if packed_layout is None:
            self.A = torch.empty((n, ns, ns), dtype=geo.dtype, device=geo.device)
            self.b = torch.empty((n, ns), dtype=geo.dtype, device=geo.device)
            ptrs = (self.A.data_ptr(), self.b.data_ptr())
        else:  # kernel writes flat_output() rows [A | b] directly
            from paper_1504_01023_b200 import flat_length

            self.flat = torch.empty(flat_length(n, ns * ns + ns, packed_layout), dtype=geo.dtype, device=geo.device)
            rows = self.flat.view(-1, ns * ns + ns)[:n] if packed_layout.lane_width == 1 else None
            self.A = rows[:, : ns * ns].unflatten(1, (ns, ns)) if rows is not None else None
            self.b = rows[:, ns * ns:] if rows is not None else None
            ptrs = (self.flat.data_ptr(), 0)
        self.dd = _desc_struct(desc, layout or ELEMENT_MAJOR, n, base_index, code, geo.data_ptr(), cof.data_ptr(),
                               ptrs[0], ptrs[1], self.err.data_ptr(), out_layout=packed_layout)
        # dynamic tile queue: two zeroed words, reset by the kernel's last CTA
        self.sched = torch.zeros(2, dtype=torch.int64, device=geo.device) if dynamic else None
        self.dd.scheduler = self.sched.data_ptr() if dynamic else None
        self.ref = ctypes.byref(self.dd)
        self.stream = torch.cuda.current_stream().cuda_stream

    def clone(self, *, dynamic, ctas_per_sm=0, stream=None):
        """Same inputs and outputs, another schedule: tile queue on/off, CTA cap, stream."""
        import copy

        import torch

        c = copy.copy(self)
        c.dd = type(self.dd).from_buffer_copy(self.dd)
        c.sched = torch.zeros(2, dtype=torch.int64, device=self.err.device) if dynamic else None
        c.dd.scheduler = c.sched.data_ptr() if dynamic else None
        c.dd.ctas_per_sm = ctas_per_sm
        c.ref = ctypes.byref(c.dd)
        c.stream = stream if stream is not None else self.stream
        return c

    def __call__(self):
        rc = self.lib.fek_integrate(self.ref, self.stream)
        if rc:
            from paper_1504_01023_b200 import _native

            _native.check(rc, "fek_integrate")

    def error_key(self) -> int:
        return int(self.err.item()) & 0xFFFFFFFFFFFFFFFF


def time_launches(launchers, steps, warmup, sampler=None):
    """Per-launch device times (ms) over `steps` launches cycling through `launchers`."""
    import torch

    for k in range(warmup):
        launchers[k % len(launchers)]()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t_all = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ctx = sampler if sampler is not None else _Null()
    with ctx:
        t_all[0].record()
        for k in range(steps):
            evs[k][0].record()
            launchers[k % len(launchers)]()
            evs[k][1].record()
        t_all[1].record()
        torch.cuda.synchronize()
    per = [a.elapsed_time(b) for a, b in evs]
    return per, t_all[0].elapsed_time(t_all[1])


def time_graph(launchers, steps, warmup, sampler=None, barrier=None):
    """Device time (ms) of `steps` launches cycling through `launchers`, replayed as one CUDA graph.

    `warmup` eager launches, then the `steps` launches are captured on a side
    stream into one graph, replayed once untimed, and replayed once between two
    CUDA events on that stream.  The graph takes the host launch path and the
    event records out of the timed region, so back-to-back steps are separated
    only by the GPU's own kernel-to-kernel gap (per-launch events on an eager
    stream add 3-5 us per launch: C1 53.7 vs 48.6 us).  `launchers` are
    Launcher objects or callables whose Launchers are listed in `.launchers`.
    `barrier` (multi-rank runs) is called right before the timed replay.
    """
    import torch

    for k in range(warmup):
        launchers[k % len(launchers)]()
    torch.cuda.synchronize()
    objs = []
    for L in launchers:
        objs.extend(getattr(L, "launchers", None) or [L])
    saved = [o.stream for o in objs]
    st = torch.cuda.Stream()
    for o in objs:
        o.stream = st.cuda_stream
    try:
        g = torch.cuda.CUDAGraph()
        # thread_local: other threads (the NCCL watchdog under torchrun) may query events meanwhile
        with torch.cuda.graph(g, stream=st, capture_error_mode="thread_local"):
            for k in range(steps):
                launchers[k % len(launchers)]()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):  # replay() launches on the current stream
            g.replay()
            st.synchronize()
            if barrier is not None:
                barrier()
                torch.cuda.synchronize()
            with (sampler if sampler is not None else _Null()):
                s.record(st)
                g.replay()
                e.record(st)
                st.synchronize()
        ms = s.elapsed_time(e)
        del g
        return ms
    finally:
        for o, v in zip(objs, saved):
            o.stream = v


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def sample_parity(desc, geo_rows, cof_rows, A_dev, b_dev, count=8192, seed=0):
    """Max relative Frobenius error of GPU outputs vs the oracle on `count` sampled elements.

    geo_rows / cof_rows: (n, DS) numpy arrays, or flat CUDA tensors (device-generated inputs).
    """
    import torch

    from oracle import numpy_oracle as O

    n = A_dev.shape[0]
    idx = np.unique(np.random.default_rng(seed).integers(0, n, size=min(count, n)))
    it = torch.from_numpy(idx).to(A_dev.device)
    if isinstance(geo_rows, torch.Tensor):
        g = geo_rows.view(n, -1).index_select(0, it).double().cpu().numpy()
        c = cof_rows.view(n, -1).index_select(0, it).double().cpu().numpy()
    else:
        g, c = geo_rows[idx], cof_rows[idx]
    A = A_dev.index_select(0, it).double().cpu().numpy()
    b = b_dev.index_select(0, it).double().cpu().numpy()
    Ao, bo = O.integrate(desc.variant.value, desc.geometry_path.value, desc.problem.value, desc.element.value, g, c)
    return float(max(O.rel_frobenius(A, Ao).max(), O.rel_frobenius(b, bo).max())), int(idx.size)


def measure_case(key, steps, warmup, variant="qss"):
    import torch

    from paper_1504_01023_b200 import KernelDescriptor, mesh, natural_path
    from paper_1504_01023_b200.measure import case_roofline
    from paper_1504_01023_b200.problems import Variant

    static = key.endswith("static")   # static round-robin tiles instead of the dynamic tile queue
    dynamic = not static
    base_key = key[:-6] if static else key
    fp32 = base_key.endswith("f32")
    packed = base_key.endswith("packed")
    cfg = mesh.bench_configs()[base_key.replace("f32", "").replace("packed", "")]
    et, pb = cfg.spec.element_type, cfg.problem
    desc = KernelDescriptor(Variant(variant), natural_path(et), pb, et)
    n = cfg.spec.n_elements
    dt = torch.float32 if fp32 else torch.float64
    geo64, cof64 = mesh.device_config(cfg)      # generated in HBM, bit-identical to the host mesh
    geo, cof = (geo64.float(), cof64.float()) if fp32 else (geo64, cof64)
    geo_rows, cof_rows = geo64, cof64
    rb = 4 if fp32 else 8
    per_set = n * (et.geometry_size + pb.coefficient_size(et) + et.n_shape * (et.n_shape + 1)) * rb
    sets = 1 if per_set > 3 * L2_BYTES else 3  # rotate buffer sets when one set is near L2 size
    from paper_1504_01023_b200 import ELEMENT_MAJOR

    pk = ELEMENT_MAJOR if packed else None
    launchers = [Launcher(desc, geo, cof, packed_layout=pk, dynamic=dynamic)]
    for _ in range(sets - 1):
        launchers.append(Launcher(desc, geo.clone(), cof.clone(), packed_layout=pk, dynamic=dynamic))
    from paper_1504_01023_b200.measure import ClockSampler

    sampler = ClockSampler(torch.cuda.current_device(), period=0.0005)
    ms_graph = time_graph(launchers, steps, warmup, sampler) / steps
    per, _ = time_launches(launchers, steps, warmup)       # eager stream, events around each launch
    for L in launchers:
        if L.error_key() != 0xFFFFFFFFFFFFFFFF:
            raise RuntimeError(f"{key}: unexpected geometry error key {L.error_key():#x}")
    ms = ms_graph
    err, cnt = sample_parity(desc, geo_rows, cof_rows, launchers[0].A, launchers[0].b)
    tol = 1e-3 if fp32 else 1e-12
    rec = {
        "workload": cfg.text + (" (fp32)" if fp32 else " (fp64)") +
                    (", kernel-packed flat_output rows" if packed else "") +
                    (", static round-robin tiles" if static else ""),
        "elements": n, "descriptor": desc.short_name(), "dtype": "f32" if fp32 else "f64",
        "value": n / (ms / 1e3), "unit": UNIT, "ms_per_launch": ms, "timing": "CUDA graph of the timed launches",
        "eager": {"ms_per_launch_mean": float(np.mean(per)), "ms_per_launch_min": float(np.min(per)),
                  "timing": "eager stream, CUDA events around each launch"},
        "buffer_sets": sets, "clocks": sampler.summary(),
        "roofline": dict(case_roofline(et, pb, n, ms / 1e3, rb),
                         traffic=load_profile_traffic(f"{desc.short_name()}_{'f32' if fp32 else 'f64'}")),
        "parity": {"max_rel_frobenius": err, "elements_checked": cnt, "tolerance": tol, "pass": err <= tol,
                   "against": "numpy oracle (bitwise-pinned restatement of the reference)"},
    }
    del launchers, geo, cof, geo64, cof64, geo_rows, cof_rows
    torch.cuda.empty_cache()
    return rec


def c5_parts(world: int, rank: int):
    """(cfg, desc, first, n) of this rank's contiguous shards of the two C5 batches."""
    from paper_1504_01023_b200 import KernelDescriptor, mesh, natural_path
    from paper_1504_01023_b200.distributed import shard_bounds
    from paper_1504_01023_b200.problems import Variant

    parts = []
    for key in ("C5T", "C5P"):
        cfg = mesh.bench_configs()[key]
        et = cfg.spec.element_type
        lo, hi = shard_bounds(cfg.spec.n_elements, world, rank)
        parts.append((cfg, KernelDescriptor(Variant.QSS, natural_path(et), cfg.problem, et), lo, hi - lo))
    return parts


def measure_c5(steps, warmup, world=1, rank=0, sampler=None, barrier=None):
    """C5: 64M-element mixed CDR mesh = one tet batch + one prism batch, range-sharded.

    A step integrates this rank's shard of both batches.  Inputs are generated
    in HBM by the device mesh generator.  Schedules timed:
    * serial  -- tet launch then prism launch on one stream, the K steps
      replayed as one CUDA graph (`serial_eager`: the same on an eager stream);
    * overlap_eager -- the memory-bound tet launch capped at 1 CTA per SM on a
      side stream with static tiles, the FP64-bound prism launch concurrently
      on the main stream taking the remaining slots from the dynamic tile queue.
    The record's headline is the fastest.
    """
    import torch

    from paper_1504_01023_b200 import mesh
    from paper_1504_01023_b200.kernels.counts import algorithmic_bytes, algorithmic_flops
    from paper_1504_01023_b200.measure import flop_peak, hbm_peak

    if sampler is None:
        from paper_1504_01023_b200.measure import ClockSampler

        sampler = ClockSampler(torch.cuda.current_device(), period=0.0005)
    launchers, parts = [], c5_parts(world, rank)
    for cfg, desc, lo, n in parts:
        geo, cof = mesh.device_config(cfg, lo, n)
        launchers.append((Launcher(desc, geo, cof, base_index=lo), desc, geo, cof))

    def serial():
        for L, *_ in launchers:
            L()

    serial.launchers = [L for L, *_ in launchers]

    side = torch.cuda.Stream()
    (LT, *_), (LP, *_) = launchers
    overlap_tet = LT.clone(dynamic=False, ctas_per_sm=1, stream=side.cuda_stream)

    def overlap():
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        overlap_tet()
        LP()
        cur.wait_stream(side)

    modes = {"serial": time_graph([serial], steps, warmup, sampler, barrier) / steps,
             "serial_eager": time_launches([serial], steps, warmup)[1] / steps,
             "overlap_eager": time_launches([overlap], steps, warmup)[1] / steps}
    if barrier is not None:  # multi-rank: every rank picks the same schedule (slowest rank per schedule)
        import torch.distributed as dist

        t = torch.tensor(list(modes.values()), dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        modes = dict(zip(modes, t.tolist()))
    best = min(modes, key=modes.get)
    if best != "serial" and sampler is not None:  # re-time the winner under the clock sampler
        modes[best] = time_launches([serial if best == "serial_eager" else overlap], steps, warmup, sampler)[1] / steps
    total_ms = modes[best] * steps
    for L, *_ in launchers:
        if L.error_key() != 0xFFFFFFFFFFFFFFFF:
            raise RuntimeError(f"C5: unexpected geometry error key {L.error_key():#x}")
    ms = total_ms / steps
    n_local = sum(n for *_, n in parts)
    hbm, _ = hbm_peak()
    fp, _ = flop_peak(8)
    by = sum(algorithmic_bytes(d.element, d.problem) * n for _, d, _, n in parts)
    fl = sum(algorithmic_flops(d.element, d.problem) * n for _, d, _, n in parts)
    t_roof = max(by / (hbm * 1e9), fl / (fp * 1e12))
    serial = sum(max(algorithmic_bytes(d.element, d.problem) * n / (hbm * 1e9),
                     algorithmic_flops(d.element, d.problem) * n / (fp * 1e12)) for _, d, _, n in parts)
    parity = {}
    for (L, desc, geo, cof), (cfg, *_) in zip(launchers, parts):
        err, cnt = sample_parity(desc, geo, cof, L.A, L.b, count=4096)
        parity[cfg.key] = {"max_rel_frobenius": err, "elements_checked": cnt, "pass": err <= 1e-12}
    rec = {"workload": "C5: 64,156,250-element mixed CDR mesh (175^3x6 tets + 4000^2x2 jittered prisms)",
           "elements_this_rank": n_local, "ms_per_step": ms, "value_this_rank": n_local / (ms / 1e3),
           "schedule": best, "ms_per_step_by_schedule": modes, "clocks": sampler.summary(),
           "roofline": {"bound": "concurrent max(sum bytes/HBM, sum flops/FP64)", "roof_ms": t_roof * 1e3,
                        "frac": t_roof / (ms / 1e3), "serialized_by_type_roof_ms": serial * 1e3,
                        "frac_of_serialized": serial / (ms / 1e3)},
           "parity": parity}
    del launchers
    torch.cuda.empty_cache()
    return rec


def load_profile_traffic(kernel_tag: str):
    """Per-launch dram bytes from the committed ncu summary, if present."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            data = json.load(fh)
        return data.get(kernel_tag, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def run_ours(args) -> int:
    import torch
    import torch.distributed as dist

    from oracle import numpy_oracle as O
    from paper_1504_01023_b200 import (DeviceBatch, ElementBatch, KernelDescriptor, integrate_batch, launch_config,
                                       mesh, natural_path)
    from paper_1504_01023_b200.distributed import env_rank
    from paper_1504_01023_b200.measure import ClockSampler, case_roofline, clocks_rejected
    from paper_1504_01023_b200.problems import Variant

    rank, world, local = env_rank()
    if not torch.cuda.is_available():
        print(json.dumps({"metric": METRIC, "error": "no CUDA device"}))
        return 1
    torch.cuda.set_device(local)
    distributed = launched_by_torchrun()
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    cfg = mesh.bench_configs()[args.config]
    et, pb = cfg.spec.element_type, cfg.problem
    desc = KernelDescriptor(Variant(args.variant), natural_path(et), pb, et)
    geo_rows = mesh.geometry_rows(cfg.spec)
    cof_rows = mesh.coefficient_rows(cfg.spec.n_elements, pb, et, cfg.coeff_seed + rank)
    n = geo_rows.shape[0]
    host_batch = ElementBatch.from_arrays(et, pb, geo_rows, cof_rows)      # page-locked flat arrays
    dev_batch = DeviceBatch.from_host(host_batch)
    launcher = Launcher(desc, dev_batch.geometry_data, dev_batch.coefficient_data, base_index=rank * n)

    # ---- device-resident timing (the `value`) ----
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local, period=0.0005)
    total_ms = time_graph([launcher], args.steps, args.warmup, sampler, barrier=dist.barrier if distributed else None)
    per, eager_ms = time_launches([launcher], args.steps, args.warmup)   # eager stream, for reference
    key = launcher.error_key()
    if key != 0xFFFFFFFFFFFFFFFF:
        raise RuntimeError(f"geometry error key {key:#x} in the benchmark mesh")
    step_ms = total_ms / args.steps
    launch_ms = step_ms  # one launch per step, back to back in the graph
    t = torch.tensor([step_ms, eager_ms / args.steps, float(np.mean(per))], dtype=torch.float64, device="cuda")
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms, eager_step_ms, eager_launch_ms = t.tolist()
    launch_ms = step_ms
    value = world * n / (step_ms / 1e3)
    clocks = sampler.summary()
    # the timed region is only a few ms: also sample a ~1 s sustained run of
    # the same launches so the clock record has enough samples under load
    sustained = ClockSampler(local, period=0.005)
    with sustained:
        t_end = time.time() + 1.0
        while time.time() < t_end:
            for _ in range(20):
                launcher()
            torch.cuda.synchronize()
    clocks["sustained_1s"] = sustained.summary()
    reject = clocks_rejected(clocks) or clocks_rejected(clocks["sustained_1s"])

    # ---- end-to-end through the public API on host buffers ----
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(1, min(args.steps, 10))
        # warm exactly like the timed loop: two results alive at once, so the
        # caching pinned-host allocator holds both result blocks before timing
        res = integrate_batch(desc, host_batch, base_index=rank * n)
        res = integrate_batch(desc, host_batch, base_index=rank * n)
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(e2e_steps):
            res = integrate_batch(desc, host_batch, base_index=rank * n)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / e2e_steps
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        if distributed:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        h2d = host_batch.geometry_data.nbytes + host_batch.coefficient_data.nbytes
        d2h = res.stiffness.nbytes + res.load.nbytes
        host_equal = bool(np.array_equal(res.stiffness, launcher.A.cpu().numpy()))
        e2e = {"value": world * n / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": ms, "steps": e2e_steps,
               "api": "paper_1504_01023_b200.integrate_batch(desc, ElementBatch) -> BatchResult (numpy)",
               "bitwise_equal_to_device_path": host_equal}

    out = None
    if rank == 0:
        cfgd = launch_config(desc, host_batch.layout, n)
        roof = case_roofline(et, pb, n, launch_ms / 1e3)
        kernel_tag = f"{desc.short_name()}_f64"
        roof_line = {"bound": roof["bound"], "achieved": roof["achieved"], "peak": roof["peak"],
                     "unit": roof["unit"], "frac": roof["frac"], "traffic": load_profile_traffic(kernel_tag),
                     "algorithmic_bytes_per_launch": roof["bytes_per_launch"],
                     "peak_source": roof["peak_source"], "kernel": f"fek::integrate_kernel<{kernel_tag}>",
                     "launch_ms": launch_ms, **cfgd}
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "f64",
               "data": "synthetic: reference unit-cube Kuhn mesh, numpy default_rng(seed+rank) U(-1,1) coefficients",
               "config": _config_record(cfg, n, world, desc), "clocks": clocks, "e2e": e2e,
               "gpu_launches": args.steps, "roofline": roof_line,
               "timing": "K launches captured as one CUDA graph, one timed replay between CUDA events on its stream",
               "eager": {"ms_per_step": eager_step_ms, "launch_ms_mean": eager_launch_ms,
                         "launch_ms_min": float(np.min(per)),
                         "timing": "same launches on an eager stream, CUDA events around each launch"}}
        if reject:
            out["clocks_warning"] = reject

    # ---- CPU baseline + full-size parity (rank 0, N=1) ----
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle.cpu_baseline import PortPool, cpu_cores

        cores = cpu_cores()
        procs = args.cpu_processes or cores["logical"] or 1
        with PortPool(desc.variant.value, desc.geometry_path.value, pb.value, et.value, geo_rows, cof_rows,
                      procs) as pool:
            warm_until = time.perf_counter() + 1.0  # >= 1 s of full-size runs before timing
            pool.run(0, n)
            while time.perf_counter() < warm_until:
                pool.run(0, n)
            sec = min(pool.run(0, n) for _ in range(2))
            A_cpu, b_cpu = pool.A, pool.b
            A_gpu = launcher.A.cpu().numpy()
            b_gpu = launcher.b.cpu().numpy()
            errA = float(O.rel_frobenius(A_gpu, A_cpu).max())
            errb = float(O.rel_frobenius(b_gpu, b_cpu).max())
        out["cpu_baseline"] = {"value": n / sec, "unit": UNIT, "cores": procs, "kind": "port",
                               "sample": f"full {cfg.key} batch ({n} elements) once, oracle port of feklab "
                                         f"integrate_batch on {procs} processes", "seconds": sec,
                               "host_cores": cores}
        out["parity"] = {"workload": cfg.key, "elements_checked": n, "max_rel_frobenius_A": errA,
                         "max_rel_frobenius_b": errb, "tolerance": 1e-12, "pass": max(errA, errb) <= 1e-12,
                         "against": "numpy oracle, bitwise-pinned to the reference (tests/golden)"}

    # ---- other configurations (N=1) ----
    if rank == 0 and world == 1 and not args.no_cases:
        del dev_batch
        cases = {}
        for key in [c for c in args.cases.split(",") if c]:
            try:
                cases[key] = measure_c5(args.steps, args.warmup) if key == "C5" else \
                    measure_case(key, args.steps, args.warmup)
            except Exception as exc:  # keep the headline line even if a case fails
                cases[key] = {"error": f"{type(exc).__name__}: {exc}"}
        out["cases"] = cases

    if distributed:
        # verification after timing: every rank's error word must be clear;
        # bit-pattern sums of all shards reduced over NCCL (reported, not timed)
        from paper_1504_01023_b200.distributed import allreduce_error_key, allreduce_sums, device_checksum
        from paper_1504_01023_b200.kernels.batched import BatchResult, _traffic

        key_all = allreduce_error_key(launcher.error_key())
        res = BatchResult(desc, n, launcher.A, launcher.b, _traffic(desc, n))
        f, u = allreduce_sums(*device_checksum(res, base_index=rank * n))
        if rank == 0:
            out["verification"] = {"error_key_all_ranks": "none" if key_all == 0xFFFFFFFFFFFFFFFF else hex(key_all),
                                   "sum_A": float(f[0]), "sum_abs_A": float(f[2]),
                                   "bitsum_A": int(u[0].item()) & 0xFFFFFFFFFFFFFFFF,
                                   "collectives": "NCCL all_reduce(MIN error key, SUM checksums) after timing"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_c5(args) -> int:
    """--config C5: the 64M mixed mesh, strong scaling (each rank generates and integrates its shard)."""
    import torch
    import torch.distributed as dist

    from paper_1504_01023_b200.distributed import env_rank
    from paper_1504_01023_b200.measure import ClockSampler, clocks_rejected

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    distributed = launched_by_torchrun()
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
    sampler = ClockSampler(local, period=0.0005)
    rec = measure_c5(args.steps, args.warmup, world, rank, sampler, barrier=dist.barrier if distributed else None)
    t = torch.tensor([rec["ms_per_step"]], dtype=torch.float64, device="cuda")
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    total = 64_156_250
    if rank == 0:
        clocks = sampler.summary()
        line = {"metric": METRIC, "value": total / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic: reference meshes generated in HBM (device PCG64, bit-identical to numpy)",
                "config": {"workload": rec["workload"], "elements_total": total,
                           "parallelism": f"element-range shards x{world} of both batches, no collective"},
                "clocks": clocks, "e2e": None, "gpu_launches": 2 * args.steps,
                "roofline": rec["roofline"], "parity_rank0": rec["parity"]}
        if clocks_rejected(clocks):
            line["clocks_warning"] = clocks_rejected(clocks)
        print(json.dumps(line), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _relaunch_under_torchrun(args, argv) -> int:
    """`python bench.py --gpus N` (N > 1) without torchrun: start N ranks on this node."""
    import socket
    import subprocess

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)]
    return subprocess.call(cmd + list(sys.argv[1:] if argv is None else argv))


def main(argv=None) -> int:
    args = parse(argv)
    if args.gpus > 1 and not launched_by_torchrun():
        return _relaunch_under_torchrun(args, argv)
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "C5":
        return run_c5(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

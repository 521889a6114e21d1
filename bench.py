#!/usr/bin/env python
"""Benchmark of the M-ABD step on B200 (BASELINE.json metric: body-steps/s, fp64, device-timed; % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Default workload: BASELINE.json configs[1] (config 2): 4096 independent chains × 256 links = 1,048,576
bodies, h = 1e-2, one Newton iteration per step. For N > 1 (torchrun) the 4096 chains are split into N
contiguous blocks, one per rank (independent assemblies, no collective in the step; strong
scaling); configs 3 and 4 split one chain / one tree with one NCCL all-gather per step.

Timed region: W untimed warm-up steps, then barrier + cuda.synchronize, CUDA events on the library's stream
around the enqueued steps (mabd_step_async; one CUDA graph per step), barrier + synchronize; the max over
ranks is reported. A rank whose state is smaller than the 126 MB L2 flushes L2 (256 MiB memset) before every
timed step, outside the event intervals; at N = 1 the config-2 state (192 MiB + 8 MiB of per-body mass
scales) is larger than L2 and streams from HBM.

``--impl reference`` times the CPU oracle (oracle/, as it stands, single-threaded) on a bounded sample of the
same workload; it is the reference arm of this tier (the paper has no code to install).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "body-steps/sec (fp64, device-timed) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "body-steps/s"

# algorithmic bytes per body-step of the fused chain kernel: read qⁿ, q̇ⁿ, write qⁿ⁺¹, q̇ⁿ⁺¹
# (4 × 96 B) + the per-body parameter the config carries (cfg 2: one fp64 mass scale; cfg 4: dims)
BYTES_PER_BODY = {1: 384, 2: 392, 3: 384, 4: 408, 5: 384}

CFG_TEXT = {
    1: "cfg1: chain of 8 unit cubes, ball joints, top pinned, h=1e-2",
    2: "cfg2: 4096 independent chains x 256 links (0.1x0.02x0.02 m boxes, rho~U[500,2000]), ball joints, "
       "first link pinned, twist U[-0.2,0.2] rad, h=1e-2, 1 Newton iteration",
    3: "cfg3: one chain of 1,048,576 cubes (0.05 m), ball joints, both ends pinned 10 m apart, h=1e-2",
    4: "cfg4: complete binary tree depth 16 (65,535 boxes), linear 6-row hinges, root pinned, h=1e-2",
    5: "cfg5: 512x512 net of 0.02 m cubes + 5% long-range links, corners pinned, h=1e-2",
}


def make_scene(cfg: int, rank: int = 0, world: int = 1):
    from mabd_scenes import generators as G
    if cfg == 2:
        return G.cfg2_batched_chains(4096, 256)
    return G.make_scene(cfg)


def fp64_peak():
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["tflops"]), "measured: " + d["source"]
    return 37.2, "nominal (64 FMA/clk/SM x 148 SMs x 1.965 GHz)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- clocks (NVML, sampled live)
class ClockSampler:
    """Samples SM clock and throttle reasons every ~10 ms on a thread while the timed region runs."""

    def __init__(self, device: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:  # the NVML handle is resolved from the torch device's UUID (CUDA_VISIBLE_DEVICES may hold UUIDs)
            import pynvml
            import torch
            pynvml.nvmlInit()
            self._nv = pynvml
            uuid = str(torch.cuda.get_device_properties(device).uuid)
            uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
            self._h = pynvml.nvmlDeviceGetHandleByUUID(uuid)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self._nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.002)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._ok:
            self._t.join()

    def summary(self):
        if not self._ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- CPU oracle sample
ORACLE_SAMPLE = {2: dict(n_chains=64, n_links=256), 1: {}, 3: dict(col_len=4096, n_cols=4, tail=0),
                 4: dict(depth=12), 5: dict(side=96)}


def oracle_sample_run(cfg: int, steps: int, warmup: int = 0) -> dict:
    """Run the oracle single-threaded in a subprocess on a bounded sample of the workload."""
    code = f"""
import json, time, sys
sys.path.insert(0, {ROOT!r})
import oracle as O
from mabd_scenes import generators as G
kw = {ORACLE_SAMPLE.get(cfg, {})!r}
sc = G.cfg2_batched_chains(**kw) if {cfg} == 2 else G.make_scene({cfg}, **kw)
q, qd = sc.q0, sc.qd0
for _ in range({warmup}):
    q, qd = O.step(sc, q, qd, sc.h)
t = time.perf_counter()
for _ in range({steps}):
    q, qd = O.step(sc, q, qd, sc.h)
dt = time.perf_counter() - t
print(json.dumps(dict(n=sc.n, steps={steps}, seconds=dt, name=sc.name)))
"""
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1",
               CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def cpu_baseline(cfg: int, steps: int = 10) -> dict:
    r = oracle_sample_run(cfg, steps)
    v = r["n"] * r["steps"] / r["seconds"]
    return {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{r['name']} ({r['n']} bodies, the same recipe), {r['steps']} steps, "
                      f"{r['seconds']:.1f} s, 1 thread (OMP/OPENBLAS_NUM_THREADS=1), host of the GPU box"}


# ----------------------------------------------------------------------------- arms
def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    r = oracle_sample_run(args.config, args.steps, args.warmup)
    v = r["n"] * r["steps"] / r["seconds"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * r["seconds"] / r["steps"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CFG_TEXT[args.config], "sample": r["name"], "bodies": r["n"]},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{r['name']} ({r['n']} bodies), one oracle KKT step per step"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


L2_BYTES = 126 * 2 ** 20


def state_bytes_per_rank(cfg: int, n: int, world: int, split: bool) -> int:
    return (BYTES_PER_BODY[cfg] // 2) * (n // world if split else n)   # q, q̇ (+ per-body params) of one rank


PARALLELISM = {
    2: "chains split over {w} ranks: contiguous blocks of 4096/{w} independent chains (no collective in the step)",
    3: "chain split over {w} ranks (NCCL all-gather of per-rank top systems, solved redundantly)",
    4: "tree split over {w} ranks (subtrees per rank, NCCL all-gather of the roots' condensed blocks, top levels "
       "replicated)",
}


def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2603_08079_b200 import Simulator

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    sc = make_scene(args.config, rank, world)
    n = sc.n
    h = sc.h
    stream = torch.cuda.Stream(device=dev)
    # configs 2 (4096 independent chains), 3 (one chain) and 4 (one tree) are split across the ranks (strong
    # scaling): config 2 by blocks of chains with no collective, config 3 with one all-gather of the
    # per-rank top systems per step, config 4 with one all-gather of the subtree roots' condensed blocks. Configs 1
    # and 5 run one independent assembly per rank (replicas, weak scaling).
    split = world > 1 and args.config in (2, 3, 4)
    if split:
        from paper_2603_08079_b200.binding import nccl_unique_id
        blob = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            blob.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(blob, src=0)
        sim = Simulator.from_scene(sc, device=local_rank, stream=stream, world=world, rank=rank,
                                   nccl_id=bytes(blob.cpu().tolist()), rotation=args.rotation)
    else:
        sim = Simulator.from_scene(sc, device=local_rank, stream=stream, rotation=args.rotation)
    sim.prefactor(h)
    q0 = sc.q0.copy()
    qd0 = sc.qd0.copy()
    info = sim.query()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # The configured workload is an episode of sc.nsteps steps (100 for configs 2-4) from the initial state; the
    # per-step cost depends on the state (the polar decomposition iterates more on strained links), so K timed
    # steps are run as episodes of ≤ nsteps steps, each from the initial state. The reset (a device copy of
    # q⁰, q̇⁰) happens between episodes, outside the timed intervals.
    episode = max(1, int(getattr(sc, "nsteps", 100) or 100))
    q0_dev = torch.as_tensor(q0, device=dev)
    qd0_dev = torch.as_tensor(qd0, device=dev)

    def reset():
        with torch.cuda.stream(stream):
            sim.set_state(q0_dev, qd0_dev)

    # L2 rule: a rank whose state is smaller than the 126 MB L2 gets an L2 flush (a 256 MiB memset) before every
    # timed step, outside the CUDA-event interval; a larger state streams from HBM anyway and is timed in one call.
    state_b = state_bytes_per_rank(args.config, n, world, split)
    flush = state_b < L2_BYTES
    l2buf = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev) if flush else None

    if args.warmup:
        sim.step(h, min(args.warmup, episode))
    reset()
    barrier()
    sampler = ClockSampler(local_rank)
    ms = 0.0
    # K < episode: the K timed steps are spread evenly over one episode (the steps between them run untimed), so the
    # number is the configured workload's average, not its cheapest first K steps (the polar decomposition's cost
    # grows with the strain the episode builds up, DESIGN R4). K ≥ episode: whole episodes.
    spread = args.steps < episode
    # config 1 (a one-warp chain scene): the library runs all steps of one mabd_step call in one launch, the state
    # in registers, so a timed interval is one call of a whole episode, with the L2 flush before it
    whole_calls = args.config == 1 and not spread
    with sampler:
        left = args.steps
        while left > 0:
            kk = min(episode, left)
            if flush and whole_calls:  # one mabd_step(h, kk) call per timed interval, L2 flushed before each
                with torch.cuda.stream(stream):
                    l2buf.zero_()
                ev0 = torch.cuda.Event(enable_timing=True)
                ev1 = torch.cuda.Event(enable_timing=True)
                ev0.record(stream)
                sim.step_async(h, kk)
                ev1.record(stream)
                sim.check()
                barrier()
                ms += ev0.elapsed_time(ev1)
            elif flush or spread:  # per-step intervals; the steps are enqueued without host waits
                stride = episode // kk if spread else 1
                evs = []
                for i in range(kk):
                    if stride > 1:
                        sim.step_async(h, stride - 1)      # untimed steps between the timed ones
                    if flush:
                        with torch.cuda.stream(stream):
                            l2buf.zero_()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    sim.step_async(h, 1)
                    e1.record(stream)
                    evs.append((e0, e1))
                sim.check()
                barrier()
                ms += sum(a.elapsed_time(b) for a, b in evs)
            else:
                ev0 = torch.cuda.Event(enable_timing=True)
                ev1 = torch.cuda.Event(enable_timing=True)
                ev0.record(stream)
                sim.step_async(h, kk)
                ev1.record(stream)
                sim.check()
                barrier()
                ms += ev0.elapsed_time(ev1)
            left -= kk
            if left > 0:
                reset()
                barrier()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    bodies_total = n if split else world * n
    value = bodies_total * args.steps / (ms * 1e-3)
    launches = info["launches_per_step"] * args.steps   # solver launches + the step_end node, per step
    if whole_calls:  # one launch per timed call
        launches = -(-args.steps // episode)

    # e2e through the public API with pinned host buffers: every step is H2D (q, q̇) → step → D2H (q, q̇). Two
    # independent problems are kept in flight (two handles, two streams, one host thread each: the binding's
    # set_state / get_state block on their own stream, ctypes releases the GIL), so one problem's H2D overlaps the
    # other's D2H on the two copy engines, as a serving loop would. Split configurations (one problem spread over
    # the ranks) keep a single pipeline. CUDA events bracket both streams.
    ke = max(1, min(args.steps, args.e2e_steps))
    n_pipe = 1 if split else 2
    sims = [sim]
    streams = [stream]
    for _ in range(n_pipe - 1):
        s2 = torch.cuda.Stream(device=dev)
        sims.append(Simulator.from_scene(sc, device=local_rank, stream=s2, rotation=args.rotation))
        sims[-1].prefactor(h)
        streams.append(s2)
    bufs = []
    for _ in range(n_pipe):
        hq = torch.empty((n, 12), dtype=torch.float64, pin_memory=True).numpy()
        hqd = torch.empty((n, 12), dtype=torch.float64, pin_memory=True).numpy()
        hq[:] = q0
        hqd[:] = qd0
        bufs.append((hq, hqd))

    def pipeline(i):
        s_, (hq_, hqd_) = sims[i], bufs[i]
        with torch.cuda.device(dev):
            for _ in range(ke):
                s_.set_state(hq_, hqd_)
                s_.step(h, 1)
                s_.get_state(hq_, hqd_)

    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for s2 in streams[1:]:
        s2.wait_event(e0)
    ths = [threading.Thread(target=pipeline, args=(i,)) for i in range(n_pipe)]
    for t_ in ths:
        t_.start()
    for t_ in ths:
        t_.join()
    for s2 in streams[1:]:
        ev = torch.cuda.Event()
        ev.record(s2)
        streams[0].wait_event(ev)
    e1.record(streams[0])
    barrier()
    ems = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ems], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
    ke = ke * n_pipe
    for s_ in sims[1:]:
        s_.close()
    e2e_value = bodies_total * ke / (ems * 1e-3)

    if rank == 0:
        peak, peak_src = peaks()
        bpb = BYTES_PER_BODY[args.config]
        n_rank = n // world if split else n          # bodies this rank advances per step
        achieved = bpb * n_rank / (ms_step * 1e-3) / 1e9
        lps = info["launches_per_step"]
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(prof):
            try:
                with open(prof) as fh:
                    traffic = json.load(fh).get(str(args.config))
            except Exception:
                traffic = None
        roof = None
        if info["solver"] == "sparse":  # fp64-bound: the dual's Cholesky, algorithmic flops / step time
            from paper_2603_08079_b200.binding import sparse_plan_stats
            st = sparse_plan_stats(sc)
            fp = fp64_peak()
            ach = st["flops"] / (ms_step * 1e-3) / 1e12
            roof = {"bound": "fp64", "achieved": ach, "peak": fp[0], "unit": "TFLOP/s", "frac": ach / fp[0],
                    "traffic": None, "kernel": f"sparse solver, step level ({info['launches_per_step']} launches)",
                    "flops_per_step": st["flops"],
                    "flops_source": "algorithmic Cholesky count of the plan (mabd_sparse_plan_stats)",
                    "peak_source": fp[1],
                    "duration": "CUDA-event time per step (all launches, incl. the per-body stages and solves)"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if split else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CFG_TEXT[args.config] + ("" if args.rotation == "polar" else
                                                              ", polar-free variant (Alg. 1, DESIGN R9)"),
                       "bodies": n, "bodies_per_gpu": n_rank,
                       "solver": info["solver"], "episode_steps": episode,
                       "timing": (f"{args.steps} timed steps spread evenly over one {episode}-step episode from the "
                                  f"initial state (every {episode // args.steps}th step timed, the others run "
                                  "untimed)" if spread else
                                  f"{args.steps} steps as episodes of <= {episode} steps from the initial state "
                                  "(reset between episodes, outside the CUDA-event intervals)") +
                                 ("; one launch per mabd_step call (all of its steps in one one-warp kernel)"
                                  if whole_calls else "; each step replays one CUDA graph"),
                       "dual_rows": info["n_dual_rows"],
                       "l2": (f"flushed before every timed {'call (one mabd_step of a whole episode)' if whole_calls else 'step'}"
                              f" (256 MiB memset outside the event interval): "
                              f"per-rank state {state_b / 2**20:.1f} MiB < 126 MB L2") if flush else
                             f"no flush: per-rank state {state_b / 2**20:.0f} MiB > 126 MB L2",
                       "parallelism": PARALLELISM[args.config].format(w=world) if split
                       else f"dp{world} (independent assemblies per rank)"},
            "roofline": roof or {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": traffic,
                         "traffic_source": "profiles/ncu_traffic.json (ncu --set full DRAM bytes per launch of the "
                                           "fused kernel, 1 GPU; not measured by this run)",
                         "kernel": "chain_kernel (fused stages 1-4)" if info["solver"] == "chain" and lps == 2
                         else "small_chain_kernel (one warp: stages 1-4 and the step bookkeeping)" if lps == 1
                         else f"{info['solver']} solver, step level ({lps} launches per step)",
                         "bytes_per_body_step": bpb, "peak_source": peak_src,
                         "duration": "CUDA-event time per step on the library's stream (" +
                                     ("the fused chain kernel + the 1-thread step_end node)" if lps == 2 else
                                      "one kernel)" if lps == 1 else
                                      f"{lps} launches: a step-level roofline)")},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * 96 * n * world,
                    "d2h_bytes_per_step": 2 * 96 * n * world, "steps": ke,
                    "path": "Simulator.set_state(pinned host) -> step(h,1) -> get_state(pinned host), "
                            f"{'one pipeline' if split else 'two independent problems in flight (two handles and streams)'}"},
            "gpu_launches": launches,
            "clocks": sampler.summary(),
        }
        if not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline(args.config, steps=args.cpu_steps)
            except Exception as e:  # report, never fake
                line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
        print(json.dumps(line), flush=True)
    sim.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--rotation", default="polar", choices=["polar", "length_preserving"],
                    help="length_preserving: the polar-free variant (P:283-310, DESIGN R9); not the default workload")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # communicator lines name the rank count (stderr)
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

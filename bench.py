#!/usr/bin/env python
"""Benchmark: gates/s of the 30-qubit random layered circuit (BASELINE.json
metric "gates/sec and circuit wall time (30q random, 34q QFT) vs HBM roofline")
on complex128 state vectors in HBM.

One step = one full circuit execution from |0...0>: reset the state, run every
planned pass (gen_random_circuit(30, 20, 424242): 1200 gates), reduce the
probability checksum (bench.hpp:141-148).  The reset is fused into the first
tile pass (qs_plan_enqueue_from_basis: that pass writes the state without
reading it).  `value` is original (unfused)
gates per second of device time with the circuit plan already resident;
`e2e` is the same metric through the public API (qs_apply_circuit with the
host gate array: planning + upload + execution + checksum read-back).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload random30|random28|qft30|hea24|ghz20] [--plan tiled|dense|unfused]

Under torchrun (N > 1, a power of two) the same circuit runs on ONE state
sharded over the N GPUs (top log2 N qubits = rank bits, half-shard exchanges
over NCCL; strong scaling); `--replicas` runs independent copies instead.  The
time is the max over ranks.  `--local-shards G` (N = 1) runs the sharded plan
with 2^G shards on one GPU (diagnostic).  `--impl reference` times the
reference CPU simulator (oracle/_ref/ref_driver, the unmodified qforge
headers) on rank 0.
"""
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

WORKLOADS = {
    # name: (generator, args, n)
    "random30": ("random", (30, 20, 424242), 30),
    "random28": ("random", (28, 20, 424242), 28),
    "qft30": ("qft", (30, 0x2AAAAAAA), 30),
    "hea24": ("hea", (24, 10, 2024), 24),
    "ghz20": ("ghz", (20,), 20),
    "qft34": ("qft", (34, 0x2AAAAAAAA), 34),  # sharded over >= 2 GPUs (256 GiB state)
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(workload, plan):
    """dram__bytes_read.sum + dram__bytes_write.sum of one tile pass from the
    committed ncu --set full capture (profiles/), per launch; None if absent."""
    if workload != "random30" or plan != "tiled":
        return None
    try:  # passes 0-3 of the current (13-qubit tile) plan, one `ncu --set full` capture; average per launch
        with open(os.path.join(ROOT, "profiles", "r1", "ncu_full_random30_m13_passes0-3.json")) as f:
            rows = json.load(f)
        scale = {"Gbyte": 1e9, "Mbyte": 1e6}
        tot = [float(d["dram__bytes_read.sum"][0]) * scale[d["dram__bytes_read.sum"][1]] +
               float(d["dram__bytes_write.sum"][0]) * scale[d["dram__bytes_write.sum"][1]] for d in rows]
        return sum(tot) / len(tot)
    except Exception:
        return None


def build_program(workload):
    from paper_2212_14201_b200 import qforge as Q
    gen, args, n = WORKLOADS[workload]
    p = {"random": Q.gen_random_circuit, "qft": Q.gen_qft, "hea": Q.gen_hea, "ghz": Q.gen_ghz}[gen](*args)
    return p, n


def cpu_baseline_reference(workload, layers, reps, threads=None):
    """Times the reference (oracle/_ref/ref_driver: unmodified qforge run()) on
    a bounded sample: the first `layers` layers of the workload, fusion on."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    if not os.path.exists(exe):
        return None, "oracle/_ref/ref_driver not built"
    gen, args, n = WORKLOADS[workload]
    if gen != "random":
        return None, "cpu baseline implemented for the random workloads"
    env = dict(os.environ)
    if threads:
        env["OMP_NUM_THREADS"] = str(threads)
    out = subprocess.run([exe, "bench", "random", str(args[0]), str(args[1]), str(args[2]), str(layers), "1",
                          str(reps)], capture_output=True, text=True, env=env, timeout=3600)
    if out.returncode != 0:
        return None, out.stderr.strip()[-200:]
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    return rows, None


class SingleRunner:
    """Whole state on one GPU (qs_state_t + qs_plan_t)."""

    sharded = False

    def __init__(self, n, gates, device, plan_mode):
        from paper_2212_14201_b200 import _native as N
        from paper_2212_14201_b200 import qforge as Q
        self.N, self.L = N, N.lib()
        t0 = time.time()
        self.cc = Q.CompiledCircuit(n, gates, plan=plan_mode, max_fused_qubits=3)
        self.plan_s = time.time() - t0
        self.stats = self.cc.stats()
        self.sv = Q.StateVector(n, device=device)
        self.shard_amps = 1 << n
        self.plan_mode = plan_mode
        self.arr, self.keep = N.gate_array(gates)
        self.G = len(gates)
        self.cs = N.C.c_double()
        self.e2e_path = "qs_run_circuit_checksum(|0..0>, host qs_gate array; checksum fused into the last pass)"

    def parallelism(self, world):
        return "replicas" if world > 1 else "single"

    def stream(self):
        return self.L.qs_stream(self.sv.handle())

    def reset(self):
        self.N.check(self.L.qs_reset(self.sv.handle()))

    def enqueue(self):
        self.N.check(self.L.qs_plan_enqueue(self.sv.handle(), self.cc._h))

    def run_from_zero(self):  # reset to |0...0> fused into the first pass, checksum into the last
        self.N.check(self.L.qs_plan_execute_from_basis_checksum(self.sv.handle(), self.cc._h, 0,
                                                                self.N.C.byref(self.cs)))

    def checksum(self):  # the step's result (already computed by its last pass)
        return self.cs.value

    def apply_host(self):  # run(): reset to |0...0> (fused) + the host gate list + checksum (fused)
        self.N.check(self.L.qs_run_circuit_checksum(self.sv.handle(), 0, self.arr, self.G, self.plan_mode, 3,
                                                    self.N.C.byref(self.cs)))

    def step_kinds(self):
        return [1] * self.stats["launches"]

    def timed(self):
        buf = (self.N.C.c_float * max(1, self.stats["launches"]))()
        self.N.check(self.L.qs_plan_execute_timed(self.sv.handle(), self.cc._h, buf))
        return list(buf)[:self.stats["launches"]]


class ShardedRunner:
    """Amplitude-sharded state: one shard per rank over NCCL (dist_world > 1), or
    2^local_g shards on this GPU (diagnostic: same plan, device-local exchanges)."""

    sharded = True

    def __init__(self, n, gates, device, dist_world=0, local_g=0):
        from paper_2212_14201_b200 import _native as N
        from paper_2212_14201_b200.sharded import DistComm, ShardedCircuit, ShardedState
        self.N, self.L = N, N.lib()
        self.g = (dist_world.bit_length() - 1) if dist_world else local_g
        self.dist = bool(dist_world)
        t0 = time.time()
        self.sc = ShardedCircuit(n, self.g, gates)
        self.plan_s = time.time() - t0
        self.stats = self.sc.stats()
        if self.dist:
            self.comm = DistComm.from_torch(device)
            self.st = ShardedState.distributed(n, self.comm)
        else:
            self.st = ShardedState.local(n, self.g, device)
        # amplitudes one step sweeps on this GPU (all local shards)
        self.shard_amps = 1 << (n - self.g) if self.dist else 1 << n
        self.arr, self.keep = N.gate_array(gates)
        self.G = len(gates)
        self.kinds = [k for k, _, _ in self.sc.steps()]
        self.e2e_path = "qs_shards_run_circuit(|0..0>, host qs_gate array) + qs_shards_checksum"

    def parallelism(self, world):
        if self.dist:
            return "amplitude-sharded over %d GPUs (%d rank qubits, NCCL exchanges)" % (world, self.g)
        return "%d local shards on 1 GPU (diagnostic)" % (1 << self.g)

    def stream(self):
        return self.st.stream()

    def reset(self):
        self.st.reset(0)

    def enqueue(self):
        self.st.execute(self.sc, sync=False)

    def run_from_zero(self):
        self.st.execute(self.sc, sync=False, from_basis=0)

    def checksum(self):
        return self.st.checksum()

    def apply_host(self):  # run(): reset to |0...0> (fused) + the host gate list
        self.N.check(self.L.qs_shards_run_circuit(self.st.handle(), 0, self.arr, self.G))

    def step_kinds(self):
        return self.kinds

    def timed(self):
        return self.st.execute_timed(self.sc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="random30", choices=sorted(WORKLOADS))
    ap.add_argument("--plan", default="tiled", choices=["tiled", "dense", "unfused"])
    ap.add_argument("--cpu-layers", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent replicas instead of one sharded state")
    ap.add_argument("--local-shards", type=int, default=0, metavar="G",
                    help="N=1 diagnostic: split the state into 2^G shards on this GPU")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the distributed (NCCL) code path even at N=1 (smoke test of the N>1 path)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return 0
        return run_reference(args)

    import torch
    import torch.distributed as dist
    if world > 1 or args.force_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)

    from paper_2212_14201_b200 import _native as N

    plan_mode = {"tiled": N.QS_PLAN_TILED, "dense": N.QS_PLAN_DENSE_FUSION, "unfused": N.QS_PLAN_UNFUSED}[args.plan]
    p, n = build_program(args.workload)
    gates = p.gates()
    G = len(gates)
    sharded = (world > 1 or args.force_dist) and not args.replicas
    if sharded and (world & (world - 1)):
        sharded = False  # amplitude sharding needs a power-of-two world
    if sharded:
        runner = ShardedRunner(n, gates, local, dist_world=world)
    elif args.local_shards:
        runner = ShardedRunner(n, gates, local, local_g=args.local_shards)
    else:
        runner = SingleRunner(n, gates, local, plan_mode)
    plan_s = runner.plan_s
    stats = runner.stats
    L = N.lib()
    stream = torch.cuda.ExternalStream(runner.stream(), device=torch.device("cuda", local))
    # replicas: every rank runs the whole circuit; sharded: the ranks share one state
    units = G * world if (world > 1 and not sharded) else G

    def step():  # reset to |0...0> + every pass (the reset fused into the first pass)
        runner.run_from_zero()

    for _ in range(args.warmup):
        step()
        runner.checksum()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = L.qs_kernel_launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        step()
        checksum = runner.checksum()  # device reduction + 8-byte read (rank-ordered sum when sharded)
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    launches = L.qs_kernel_launches() - launches0
    ms_total = ev0.elapsed_time(ev1)

    # per-step device times (CUDA events between steps, same stream)
    prof_runs = 2
    per, kinds = None, runner.step_kinds()
    for _ in range(prof_runs):
        runner.reset()
        t = runner.timed()
        per = t if per is None else [a + b for a, b in zip(per, t)]
    per = [x / prof_runs for x in per]
    clk = clocks.stop()

    ms_max = ms_total
    if world > 1:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    value = units / (ms_per_step / 1e3)

    # e2e through the public API with host buffers (planning + upload + run + checksum read)
    e2e = None
    if not args.no_e2e:
        h2d = N.C.sizeof(N.QsGate) * G
        for _ in range(2):
            runner.apply_host()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e_steps = max(2, min(args.steps, 5))
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e_steps):
            runner.apply_host()
            runner.checksum()
        e1.record(stream)
        e1.synchronize()
        wall = (time.perf_counter() - t0) * 1e3 / e_steps
        dev = e0.elapsed_time(e1) / e_steps
        e_ms = max(wall, dev)
        if world > 1:
            t = torch.tensor([e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": units / (e_ms / 1e3), "unit": "gates/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8, "path": runner.e2e_path}

    peak, peak_kind = peaks()
    state_bytes = 16 * runner.shard_amps  # bytes of the state (or shard) one pass sweeps
    # dominant kernel: the tile pass (or the per-gate kernel in other plans)
    pass_ms = [x for x, k in zip(per, kinds) if k != 2 and x > 0]
    xchg_ms = [x for x, k in zip(per, kinds) if k == 2]
    avg_pass_ms = sum(pass_ms) / len(pass_ms) if pass_ms else 0.0
    achieved = (2 * state_bytes) / (avg_pass_ms / 1e3) / 1e9 if avg_pass_ms else 0.0
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4),
                "traffic": ncu_traffic(args.workload, args.plan) if not runner.sharded else None,
                "kernel": "qsb_tile_* (per-pass NVRTC sm_100a)" if args.plan == "tiled" else "per-gate kernels",
                "algorithmic_bytes_per_launch": 2 * state_bytes, "launches_per_step": stats["launches"],
                "avg_launch_ms": round(avg_pass_ms, 4), "peak_kind": peak_kind,
                # tile passes' share of the per-step-timed run (full passes, not started
                # from a basis state, so its total exceeds the timed step's)
                "pass_time_share": round(sum(pass_ms) / sum(per), 4) if per and sum(per) else None}
    if xchg_ms:
        roofline["exchanges_per_step"] = len(xchg_ms)
        roofline["exchange_ms_total"] = round(sum(xchg_ms), 3)
    if pass_ms:
        srt = sorted(pass_ms)
        roofline["launch_ms_min_median_max"] = [round(srt[0], 3), round(srt[len(srt) // 2], 3), round(srt[-1], 3)]
        if os.environ.get("QSB_BENCH_PASSES"):
            roofline["launch_ms"] = [round(x, 3) for x in per]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.local_shards:
        rows, err = cpu_baseline_reference(args.workload, args.cpu_layers, 1)
        if rows:
            r = rows[-1]
            cpu = {"value": r["gates"] / r["seconds"], "unit": "gates/s", "cores": r["threads"], "kind": "reference",
                   "sample": "first %d layer(s) (%d gates) of the workload through qforge::run() with fusion "
                             "(k=3), incl. its 2^%d-state allocation and final-state copy" % (args.cpu_layers,
                                                                                               r["gates"], n),
                   "seconds": r["seconds"]}
        else:
            cpu = {"value": None, "unit": "gates/s", "cores": None, "kind": "reference", "sample": err}

    if rank == 0:
        line = {
            "metric": "gates/sec (30q random layered circuit, d=20, complex128) vs HBM roofline",
            "value": round(value, 2), "unit": "gates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "strong" if runner.sharded else "weak", "vs_baseline": None, "dtype": "complex128 (f64)",
            "data": "synthetic",
            "config": {"workload": "%s: %s%s" % (args.workload, WORKLOADS[args.workload][0], WORKLOADS[args.workload][1]),
                       "qubits": n, "gates": G, "plan": args.plan, "passes": stats["passes"],
                       "plan_seconds": round(plan_s, 3), "parallelism": runner.parallelism(world),
                       "l2": "inputs larger than L2 (%s %.1f GiB)" % ("shard" if runner.sharded else "state",
                                                                    state_bytes / 2 ** 30),
                       "checksum": checksum},
            "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline, "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line))
    if dist.is_initialized():
        del runner  # shards and their communicator go before the process group
        dist.destroy_process_group()
    return 0


def run_reference(args):
    """--impl reference: the reference CPU simulator on this host's cores."""
    gen, wargs, n = WORKLOADS[args.workload]
    if gen != "random":
        print(json.dumps({"impl": "reference", "unavailable": "reference arm implemented for random workloads"}))
        return 0
    reps = args.warmup + args.steps
    rows, err = cpu_baseline_reference(args.workload, args.cpu_layers, reps)
    if not rows:
        print(json.dumps({"impl": "reference", "unavailable": err}))
        return 0
    timed = rows[args.warmup:]
    sec = sum(r["seconds"] for r in timed) / len(timed)
    gates = timed[0]["gates"]
    value = gates / sec
    line = {
        "impl": "reference",
        "metric": "gates/sec (30q random layered circuit, d=20, complex128) vs HBM roofline",
        "value": round(value, 4), "unit": "gates/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 1), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "complex128 (f64)", "data": "synthetic",
        "config": {"workload": "%s: %s%s" % (args.workload, gen, wargs), "qubits": n,
                   "sample_gates": gates, "fusion": "reference fuse_circuit k=3"},
        "cpu_baseline": {"value": round(value, 4), "unit": "gates/s", "cores": timed[0]["threads"],
                         "kind": "reference",
                         "sample": "first %d layer(s) (%d gates) per step through qforge::run()" % (args.cpu_layers,
                                                                                                    gates)},
        "e2e": {"value": round(value, 4), "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())

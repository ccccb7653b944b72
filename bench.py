"""Benchmark: M elements/s for energy + gradient + Hessian + BSR assembly (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1|c2|c3|c4|c5] [--mode deterministic|atomic|ordered]

One step = one Assembler::assemble() of the whole configuration on device-resident inputs
(activation refresh, element kernels, SPD projection where the config asks for it, gradient +
BSR assembly, energy and finiteness reduction). The atomic assembly mode is timed right after
and reported in the same line ("atomic"); "e2e" adds the host copies (x in, E + gradient out),
"e2e_host_hessian" also copies the whole BCRS Hessian back every step.

Multi-GPU: one process per GPU. `--gpus N` outside torchrun re-launches itself as N ranks
(torch.distributed.run, 127.0.0.1). Config 2 shards into slabs (owner computes, E all-reduce);
other configs run replicas ("scaling": "weak"); max-over-ranks device time.

`--impl reference` runs the unmodified reference (oracle/_ref/ref_driver: reference headers
compiled in place, `source` backend, all host threads) through Assembler::assemble() on the
same config at FULL size (config 5: a bounded sample unless --ref-n is given); the
`cpu_baseline` key of our arm is the same reference on a bounded sample (n=40 for config 2).
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic FP64 flops per element: tape plan ops + (n_qp-1)*outputs for
# quadrature accumulation + outputs for the global accumulation.
FLOPS = {"tet4": 4406 + 157, "tet10": 4 * 23164 + 3 * 931 + 931, "membrane": 5622 + 91, "bending": 1009 + 157,
         "contact": 2811 + 157, "inertia": 23 + 13}
# compulsory bytes per element: unique inputs once + unique outputs once
# (tets and tet10: connectivity, x, X, their share of the BSR values and the gradient)
BYTES = {"tet4_c1": 223.0, "tet4": 211.0, "tet10": 2941.0,
         "membrane": 12 + 40,      # connectivity + Dm2inv / area (x, BSR, g counted once below)
         "bending": 16 + 1152,     # connectivity + the 144-double Q of the flap
         "contact": 16 + 96 + 16 * 72,  # connectivity + per-pair offsets + its 16 scattered blocks
         "inertia": 56 + 72}       # x_prev, v, m + the diagonal block


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2")
    p.add_argument("--mode", default="deterministic", choices=["deterministic", "atomic", "ordered"])
    p.add_argument("--no-spd", action="store_true", help="disable the config's SPD projection")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--ref-n", type=int, default=0, help="reference sample grid size (default per config)")
    return p.parse_args()


def make_case(cfg: str):
    from paper_2303_02156_b200 import configs as C
    return {"c1": C.config1, "c2": C.config2, "c3": C.config3, "c4": C.config4, "c5": C.config5}[cfg]()


def config_meta(cfg: str):
    return {
        "c1": dict(workload="config1: linear-tet Stable NH, 20^3 Kuhn grid, 48,000 tets", spd=False),
        "c2": dict(workload="config2: linear-tet Stable NH, 100^3 Kuhn grid, 6,000,000 tets, SPD projection", spd=True),
        "c3": dict(workload="config3: quadratic tet10 Stable NH, 40^3 grid, 384,000 elements, 4-pt rule", spd=False),
        "c4": dict(workload="config4: cloth 1000x1000, StVK membrane + hinge bending", spd=False),
        "c5": dict(workload="config5: config2 tets + inertia + 4,000,000 point-triangle barrier pairs, SPD", spd=True),
    }[cfg]


# SPD projection flops per projected element (SURVEY 8(d) "P_spd"): the standard count of the
# symmetric eigen-decomposition with vectors of the full n x n element Hessian (Golub & Van Loan:
# tridiagonalisation + explicit Q + implicit QR with vectors ~ 9 n^3) plus the rebuild
# V max(L, 0) V^T (~ n^3), n = 12. The fused kernel does less (9 x 9 reduced form, codegen.cpp).
SPD_N = 12
P_SPD = 10 * SPD_N ** 3


def spd_elements(cfg: str, case) -> int:
    if cfg == "c2":
        return case.conn.shape[0]
    if cfg == "c5":
        return case.conn.shape[0] + case.extra["pairs"].shape[0]
    return 0


def flops_per_step(cfg: str, case) -> float:
    if case.kind == "tet4":
        return FLOPS["tet4"] * case.conn.shape[0]
    if case.kind == "tet10":
        return FLOPS["tet10"] * case.conn.shape[0]
    if case.kind == "cloth":
        return FLOPS["membrane"] * case.conn.shape[0] + FLOPS["bending"] * case.extra["flaps"].shape[0]
    return (FLOPS["tet4"] * case.conn.shape[0] + FLOPS["contact"] * case.extra["pairs"].shape[0]
            + FLOPS["inertia"] * case.n_nodes)


def hbm_peak_gbs() -> float:
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written); else the profiling
    recipe's fallback (6.65 TB/s)."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def bytes_per_step(cfg: str, case) -> float:
    """Compulsory HBM bytes of one assemble: unique inputs read once + unique
    outputs written once; the static pattern and the tile plan (as-implemented extras) excluded."""
    if case.kind == "tet4":
        return BYTES["tet4_c1" if cfg == "c1" else "tet4"] * case.conn.shape[0]
    if case.kind == "tet10":
        return BYTES["tet10"] * case.conn.shape[0]
    if case.kind == "cloth":
        shared = 72.0 * 10_984_004 * case.n_nodes / 1_000_000 + 2 * 24.0 * case.n_nodes  # BSR + g + x
        return (BYTES["membrane"] * case.conn.shape[0] + BYTES["bending"] * case.extra["flaps"].shape[0] + shared)
    return (BYTES["tet4"] * case.conn.shape[0] + BYTES["contact"] * case.extra["pairs"].shape[0]
            + BYTES["inertia"] * case.n_nodes)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits", "-lms", "100"],
                                     stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait(timeout=5)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


REF_SAMPLE_N = {"c1": 20, "c2": 40, "c3": 16, "c4": 300, "c5": 30}   # bounded cpu_baseline samples
REF_FULL_N = {"c1": 20, "c2": 100, "c3": 40, "c4": 1000}              # the configs at full size


def ref_case(cfg: str, n: int):
    from paper_2303_02156_b200 import configs as C
    if cfg == "c5":
        return C.config5(n, 4 * (n + 1) ** 3)
    return {"c1": C.config1, "c2": C.config2, "c3": C.config3, "c4": C.config4}[cfg](n)


def cpu_reference(cfg: str, steps: int, warmup: int, n: int, threads: int = 0, spd_sample: bool = True):
    """The unmodified reference (oracle/_ref/ref_driver: reference headers compiled in place,
    `source` backend = the paper's compiled kernels, all host threads, lanes 8) running
    Assembler::assemble() on the same seeded generator at grid size n."""
    from oracle import oracle as O
    if not os.path.exists(O.REF_DRIVER):
        return None, "oracle/_ref/ref_driver not built"
    case = ref_case(cfg, n)
    d = tempfile.mkdtemp(prefix="symel_refbench_")
    try:
        case.write_case_dir(d)
        threads = threads or os.cpu_count() or 1
        info = O.run_ref_driver(d, backend="source", threads=threads, lanes=8, repeat=max(1, steps), dump=False,
                                cache=os.path.join(d, "kcache"), warmup=max(1, warmup))
    finally:
        shutil.rmtree(d, ignore_errors=True)
    melem = info["n_elements"] / (info["mean_ms"] * 1e-3) / 1e6
    sample = (f"{cfg} generator at n={n}: {info['n_elements']} elements; reference Assembler::assemble "
              f"(source backend, lanes 8, {threads} threads), mean of {steps} steady-state calls after "
              f"{max(1, warmup)} warm-up call(s) (first call {info['first_ms']:.0f} ms incl. kernel compile + "
              f"pattern build); no SPD projection (the reference has none)")
    out = {"value": melem, "unit": "M elements/s", "cores": threads, "kind": "reference", "sample": sample,
           "ms_per_assemble": info["mean_ms"], "eval_ms": info["eval_ms"], "assemble_ms": info["assemble_ms"],
           "first_ms": info["first_ms"], "n_elements": info["n_elements"], "n": n}
    if cfg in ("c2", "c5") and spd_sample:
        out["spd_projection"] = cpu_spd_projection(ref_case(cfg, min(n, 40)))
    return out, None


def cpu_spd_projection(case, count: int = 20000) -> dict:
    """The SPD oracle (numpy float64 eigh of each 12x12 element Hessian, V max(L,0) V^T) timed on
    host cores over a sample of the config's element Hessians -- the reference has no SPD
    projection, so this is reported as its own line."""
    from oracle import oracle as O
    from paper_2303_02156_b200.systems import golden_tape
    sysm = O.system_for_case(case, golden_tape)
    count = min(count, case.conn.shape[0])
    H = sysm.element_outputs(0, 0, count)[:, 13:].reshape(-1, 12, 12)
    O.spd_project(H[:100])
    t0 = time.perf_counter()
    O.spd_project(H)
    dt = time.perf_counter() - t0
    return {"value": count / dt / 1e6, "unit": "M elements/s", "cores": 1, "kind": "port",
            "sample": f"numpy.linalg.eigh projection of {count} tet element Hessians (12x12) of the sample"}


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` (N > 1) outside torchrun: re-exec as N ranks on this node."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def config_dict(cfg: str, n_elements: int, spd: bool, mode: str) -> dict:
    """The workload both arms report (identical keys and values)."""
    meta = config_meta(cfg)
    return {"workload": meta["workload"], "elements": int(n_elements), "spd": bool(spd), "mode": mode}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch_under_torchrun(args)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    meta = config_meta(args.config)
    spd = meta["spd"] and not args.no_spd
    metric = "M elements/s for energy+grad+Hessian+BSR assembly"

    if args.impl == "reference":
        if rank != 0:
            return 0
        n = args.ref_n or REF_FULL_N.get(args.config, REF_SAMPLE_N[args.config])
        base, why = cpu_reference(args.config, args.steps, args.warmup, n)
        if base is None:
            print(json.dumps({"impl": "reference", "unavailable": why}))
            return 0
        full = n == REF_FULL_N.get(args.config)
        ref_cfg = config_dict(args.config, base["n_elements"], spd, args.mode) if full else \
            {"workload": meta["workload"] + f" (bounded sample n={n})", "elements": base["n_elements"]}
        line = {"impl": "reference", "metric": metric, "value": base["value"], "unit": "M elements/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": base["ms_per_assemble"], "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded generator, BASELINE shapes)" if full else
                        "synthetic (seeded generator, bounded sample)",
                "config": ref_cfg,
                "reference_notes": {"sample": base["sample"], "first_call_ms": base["first_ms"],
                                    "eval_ms": base["eval_ms"], "assemble_ms": base["assemble_ms"],
                                    "spd_projection": "not part of the reference (SURVEY 8(c)); this arm's time "
                                                      "excludes it" if spd else "off"},
                "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": base["value"], "unit": "M elements/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        if "spd_projection" in base:
            line["reference_notes"]["spd_projection_oracle"] = base["spd_projection"]
        print(json.dumps(line))
        return 0

    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)

    from paper_2303_02156_b200.parallel import ShardedTetSystem, max_over_ranks, sum_over_ranks
    from paper_2303_02156_b200.systems import DeviceSystem

    if (world > 1 or os.environ.get("BENCH_FORCE_SLABS")) and args.config == "c2":
        # sharded, weak scaling: rank r owns a config-2-sized slab (100 x 100 x 100 hexes) of a
        # world*100 x 100 x 100 grid plus one ghost hex plane; the data-path collective is the
        # all-reduce of the owned energy (parallel.py)
        from paper_2303_02156_b200 import configs as C
        slab = C.tet4_slab_case(100, world, rank)
        shard = ShardedTetSystem(slab.case.x, slab.case.X, slab.case.conn, slab.n_own, slab.case.params,
                                 slab.row_lo, slab.row_hi, slab.global_ids, spd=spd, device=local)
        ds, case, n_elem = shard.ds, slab.case, slab.n_own
        parallelism = f"dp{world} slabs, owner computes (1 ghost hex plane), E all-reduce over NCCL"

        def step(mode=args.mode):
            return sum_over_ranks(shard.assemble(mode), device="cuda")
    else:
        case = make_case(args.config)
        ds = DeviceSystem(case, spd=spd, device=local)
        n_elem = case.n_elements()
        parallelism = f"replicas{world}" if world > 1 else "single GPU"

        def step(mode=args.mode):
            return ds.asm.assemble(mode)
    A = ds.asm
    stream = torch.cuda.ExternalStream(A.stream(), device=local)
    t_setup = time.time()
    for _ in range(max(3, args.warmup)):
        step()
    setup_s = time.time() - t_setup
    tm = A.timings()
    plan = A.plan_info()
    einfo = {n: A.energy_info(e) for n, e in ds.energies.items()}

    def timed(mode, steps):
        """K steps of `mode` between barriers, CUDA events on the library's stream; returns
        (ms per step, mean element-kernel ms, launches per step)."""
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = A.launch_count()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        kms = []
        for _ in range(steps):
            step(mode)
            kms.append(A.timings().eval_ms)
        e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize()
        launches = (A.launch_count() - l0) // max(1, steps)
        return max_over_ranks(e0.elapsed_time(e1) / steps, device="cuda"), float(np.mean(kms)), launches

    # ---- device-resident timed region (the headline mode)
    clocks = ClockSampler(local)
    clocks.start()
    ms, k_ms, launches = timed(args.mode, args.steps)
    clk = clocks.stop()
    value = world * n_elem / (ms * 1e-3) / 1e6

    # ---- the atomic path, reported alongside (north star)
    alt = None
    if args.mode == "deterministic":
        for _ in range(max(3, args.warmup)):
            step("atomic")
        ams, akms, alaunch = timed("atomic", args.steps)
        alt = {"mode": "atomic", "value": world * n_elem / (ams * 1e-3) / 1e6, "unit": "M elements/s",
               "ms_per_step": ams, "kernel_ms": akms, "gpu_launches": int(alaunch)}
        for _ in range(max(3, args.warmup)):
            step(args.mode)

    # ---- roofline of the dominant kernel (element eval + fused assembly)
    fl = flops_per_step(args.config, case)
    fl_spd = P_SPD * spd_elements(args.config, case) if spd else 0
    peak = A.fp64_peak_tflops()
    achieved = (fl + fl_spd) / (k_ms * 1e-3) / 1e12
    achieved_nospd = fl / (k_ms * 1e-3) / 1e12
    roof = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": None, "kernel_ms": k_ms, "kernel_share_of_step": k_ms / ms,
            "peak_source": "measured DFMA probe on this GPU (symel_cuda_fp64_peak), FMA = 2 flops",
            "algorithmic_flops_per_step": fl + fl_spd,
            "flops_definition": "reference tape plan ops + accumulation (SURVEY 8(d))"
                                + (f" + P_spd = 10*{SPD_N}^3 = {P_SPD} per projected element (standard symmetric "
                                   "eigen-decomposition with vectors + rebuild)" if spd else ""),
            "achieved_without_spd": achieved_nospd, "frac_without_spd": achieved_nospd / peak}
    # the element roofline is the slower of its flops at the FP64 peak and its compulsory bytes at
    # the HBM bandwidth (north star); config 4 (the 1152-byte bending Q per flap) is HBM-bound
    by = bytes_per_step(args.config, case)
    bw = hbm_peak_gbs()
    roof["algorithmic_bytes_per_step"] = by
    roof["hbm_achieved_gbs"] = by / (k_ms * 1e-3) / 1e9
    roof["hbm_frac"] = roof["hbm_achieved_gbs"] / bw
    if by / (bw * 1e9) > (fl + fl_spd) / (peak * 1e12):
        roof.update({"bound": "hbm", "achieved": roof["hbm_achieved_gbs"], "peak": bw, "unit": "GB/s",
                     "frac": roof["hbm_frac"], "fp64_frac": achieved / peak,
                     "peak_source": "HBM copy bandwidth of measured (MEASURED_PEAKS.json hbm_gbs)"})
    facts_path = os.path.join(ROOT, "profiles", "kernel_facts.json")
    if os.path.exists(facts_path):
        key = args.config if (spd or args.config != "c2") else "c2_nospd"
        facts = json.load(open(facts_path)).get(key)
        if facts:
            roof["traffic"] = facts["traffic_bytes"]
            roof["ncu"] = {k: v for k, v in facts.items() if k != "traffic_bytes"}

    # ---- end to end through the C ABI with host buffers: H2D x, assemble, D2H E + gradient
    # (+ the whole BCRS Hessian in the host-Hessian variant: the reference's hessian() contract)
    import ctypes
    lib = A.lib
    x_host = torch.empty(case.x.size, dtype=torch.float64, pin_memory=True)
    x_host.numpy()[:] = case.x.ravel()
    g_host = torch.empty(case.x.size, dtype=torch.float64, pin_memory=True)
    pb, _, pnb, _ = A.pattern_info()
    nvals = int(pnb) * int(pb) * int(pb)

    def e2e_run(with_h):
        h_host = torch.empty(max(1, nvals), dtype=torch.float64, pin_memory=True) if with_h else None
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e2 = torch.cuda.Event(enable_timing=True)
        e3 = torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        for _ in range(args.steps):
            lib.symel_cuda_set_array(A.h, ds.x, ctypes.c_void_p(x_host.data_ptr()), case.x.size)
            step()
            lib.symel_cuda_copy_gradient(A.h, ctypes.c_void_p(g_host.data_ptr()))
            if with_h:
                lib.symel_cuda_copy_hessian(A.h, ctypes.c_void_p(h_host.data_ptr()))
        e3.record(stream)
        e3.synchronize()
        t = max_over_ranks(e2.elapsed_time(e3) / args.steps, device="cuda")
        return {"value": world * n_elem / (t * 1e-3) / 1e6, "unit": "M elements/s",
                "h2d_bytes_per_step": int(case.x.size * 8),
                "d2h_bytes_per_step": int(case.x.size * 8 + 8 + (nvals * 8 if with_h else 0)), "ms_per_step": t}

    e2e = e2e_run(False)
    e2e["note"] = "x in, E + gradient out; BSR values stay device-resident for the device PCG consumer"
    e2e_h = e2e_run(True)
    e2e_h["note"] = ("x in, E + gradient + all BCRS values out every step (the reference's host "
                     "BcrsMatrix hessian() contract, assembly.hpp:177)")

    line = {"metric": metric, "value": value, "unit": "M elements/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, BASELINE shapes)",
            "config": config_dict(args.config, world * n_elem, spd, args.mode),
            "details": {"parallelism": parallelism, "elements_per_rank": n_elem,
                        "l2": "working set (BSR values + slot maps + connectivity) >> 126 MB L2; no flush needed",
                        "pattern_ms": tm.pattern_ms, "compile_ms": tm.compile_ms, "setup_s": setup_s,
                        "tile_plan": plan,
                        "kernel_ops": {n: {"tape": v["tape_ops"], "executed": v["fast_ops"],
                                           "frontier": v["frontier"]} for n, v in einfo.items()}},
            "roofline": roof, "clocks": clk, "e2e": e2e, "e2e_host_hessian": e2e_h, "gpu_launches": int(launches)}
    if alt:
        line["atomic"] = alt
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base, why = cpu_reference(args.config, 3, 1, args.ref_n or REF_SAMPLE_N[args.config])
        line["cpu_baseline"] = base if base else {"unavailable": why}
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

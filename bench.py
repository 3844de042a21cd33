"""Benchmark: BASELINE config 2 training step (3D SDF, hash L=16 F=2 T=2^19,
N_max=2048, 2x64 MLP -> 1 linear, MAPE, lr 1e-4, batch 2^18 per GPU) plus
config-5 inference queries/s, on N GPUs (one process per GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0. ``value`` is whole-job training samples/s with
inputs resident in HBM; ``e2e`` is the same metric through the public API
(FieldModel.train_step on pinned host buffers: H2D of X and target, the step,
D2H of the loss every step). ``--impl reference`` times the CPU restatement of
the reference (the Eigen-based reference cannot be built here).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG2 = dict(dims=3, levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048)
B_TRAIN = 1 << 18
LR = 1e-4
N_RESIDENT = 8          # distinct resident batches cycled through the timed steps
B_INFER = 1 << 24       # config-5 inference point for the headline queries/s
METRIC = "training samples/sec at batch 2^18 (enc+MLP fwd/bwd+Adam); inference queries/s"
WORKLOAD = "config2: 3D SDF hash L16 F2 T2^19 Nmin16 Nmax2048, MLP 32-64-64-1 ReLU/linear, MAPE, Adam lr1e-4"

# algorithmic work per unit
ADAM_BYTES_PER_PARAM = 34          # r: p g m v; w: p m v g(=0) + fp16 shadow
ENC_FWD_L2_BYTES_PER_SAMPLE = 2304  # 72 sectors x 32 B (3D, fp16 rows)
ENC_BWD_L2_BYTES_PER_SAMPLE = 2560  # 80 sectors x 32 B (fp32 F=2 rows, RED)
MLP_TRAIN_FLOP_PER_SAMPLE = 37248


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--infer-b", type=int, default=B_INFER)
    ap.add_argument("--no-nerf", action="store_true")
    ap.add_argument("--mlp-engine", type=int, default=0, choices=[0, 1, 2],
                    help="nfg_options.mlp_engine: 0 measured default, 1 mma.sync, 2 tcgen05 (A/B runs)")
    ap.add_argument("--launcher-selftest", action="store_true",
                    help="spawn/rendezvous check only (gloo, no GPU work): rank 0 prints the ranks it saw")
    return ap.parse_args()


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(args):
    """``--gpus N`` (N > 1) outside torchrun: re-exec this script under
    torch.distributed.run with N ranks on this node, so a plain
    ``python bench.py --gpus 8`` cannot silently measure one GPU. Returns the
    child's exit code, or None when this process already is a rank."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def launcher_selftest(rank, world):
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        seen = int(t.item())
        dist.destroy_process_group()
    else:
        seen = 1
    if rank == 0:
        print(json.dumps({"launcher_selftest": True, "n_gpus": world, "ranks_seen": seen, "pid": os.getpid()}),
              flush=True)


def peaks():
    """(HBM GB/s, dense bf16 TFLOP/s, source) from the driver-written
    MEASURED_PEAKS.json (key names matched loosely, nested dicts searched; a
    'sustained' HBM figure is preferred for kernels timed inside a long step),
    else B200_PROFILING.md's fallback (6.65 TB/s, 1.59 PFLOP/s)."""
    def flat(d, pre=""):
        for k, v in (d.items() if isinstance(d, dict) else []):
            key = f"{pre}.{k}".lower()
            if isinstance(v, dict):
                yield from flat(v, key)
            elif isinstance(v, (int, float)) and not isinstance(v, bool):
                yield key, float(v)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            items = list(flat(json.load(f)))
        hbm = [(k, v) for k, v in items if ("hbm" in k or "dram" in k or "copy" in k) and "lat" not in k]
        mma = [(k, v) for k, v in items if ("bf16" in k or "tflop" in k or "gemm" in k)]
        if not hbm or not mma:
            raise ValueError("no peaks")
        pick = lambda xs: sorted(xs, key=lambda kv: ("sustain" not in kv[0], kv[0]))[0][1]   # noqa: E731
        h, t = pick(hbm), pick(mma)
        h = h * 1000.0 if h < 100.0 else h          # TB/s -> GB/s
        t = t / 1000.0 if t > 100000.0 else t       # GFLOP/s -> TFLOP/s
        return h, t, "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class Clocks:
    """SM clocks and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line). NVML is polled in-process every ~2 ms, so
    even a few-millisecond timed region gets samples; nvidia-smi -lms is the
    fallback when NVML cannot be loaded."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, index):
        self.index = index
        self.rows = []          # (sm_mhz, max_mhz, reasons bitmask, util %)
        self._stop = threading.Event()
        self._proc = None
        self._nv = None

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self._max = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._poll_nvml, daemon=True)
            self._t.start()
            return self
        except Exception:
            self._nv = None
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,utilization.gpu")
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                           "--format=csv,noheader,nounits", "-lms", "50"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read_smi, daemon=True)
            self._t.start()
        except Exception:
            self._proc = None
        return self

    def _poll_nvml(self):
        nv, h = self._nv, self._h
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                ut = nv.nvmlDeviceGetUtilizationRates(h).gpu
                self.rows.append((float(sm), float(self._max), int(rs), int(ut)))
            except Exception:
                pass
            time.sleep(0.002)

    def _read_smi(self):
        for line in self._proc.stdout:
            p = [x.strip() for x in line.split(",")]
            try:
                self.rows.append((float(p[0]), float(p[1]), int(p[2], 16), int(p[3])))
            except Exception:
                pass

    def stop(self):
        self._stop.set()
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except Exception:
                self._proc.kill()
        if self._nv is not None:
            self._t.join(timeout=1)

    def mark(self):
        return len(self.rows)

    def summary(self, since=0):
        rows = self.rows[since:] or self.rows[-8:]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"], "samples": 0}
        sm = sorted(r[0] for r in rows)
        reasons = sorted({n for r in rows for n, bit in self.REASONS if r[2] & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_min_mhz": sm[0], "sm_max_mhz": rows[0][1], "reasons": reasons,
                "samples": len(rows), "source": "nvml" if self._nv is not None else "nvidia-smi"}


def ncu_traffic():
    """DRAM bytes per launch (dram__bytes_read + write) from the committed ncu capture."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "ncu_r*.json")))
    if not files:
        return {}
    with open(files[-1]) as f:
        d = json.load(f)
    out = {"_src": os.path.relpath(files[-1], ROOT)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for k, m in d.get("kernels", {}).items():
        try:
            tot = sum(float(m[n]["value"]) * scale[m[n]["unit"]] for n in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            out[k] = tot
        except Exception:
            pass
    return out


def image_target_torch(X):
    """The procedural test image (helpers.hpp:99-125) evaluated at continuous (u, v):
    the "16k x 16k" gigapixel target of config 3 without materialising it."""
    import torch
    u, v = X[:, 0].double(), X[:, 1].double()
    r = 0.35 + 0.3 * u + 0.15 * torch.sin(6.0 * u + 2.0 * v)
    g = 0.45 + 0.25 * v + 0.12 * torch.sin(9.0 * v - 3.0 * u + 1.3)
    b = 0.5 + 0.2 * torch.sin(4.0 * (u + v))
    for o in range(1, 4):
        f, a = 12.0 * o, 0.08 / o
        r = r + a * torch.sin(f * u + 0.7 * o) * torch.cos(f * 0.8 * v)
        g = g + a * torch.cos(f * v + 1.9 * o) * torch.sin(f * 0.6 * u)
        b = b + a * torch.sin(f * (u - v) + 0.4 * o)
    return torch.stack([r, g, b], 1).clamp(0.0, 1.0).float().contiguous()


def bench_gigapixel(nf, ctx, steps, warmup, T_log2=24, n_max=8192, batch=None, metric=None, config=None):
    """BASELINE config 3 on one GPU: 2D hash L16 F2 T=2^24, N_max 8192, 2x64 MLP
    -> RGB sigmoid, L2, batch 2^18 of random points on the procedural image. The
    fp16 tables (1 GB) exceed L2: the HBM-bound gather regime; Adam runs its
    sparse (skip-zero) pass since 2^18 x 4 corners touch ~6% of each level.
    With T_log2=14, n_max=1024, batch 2^16 the same harness times config 1."""
    import torch
    B_TRAIN = batch or globals()["B_TRAIN"]
    m = nf.FieldModel(ctx)
    m.hash_cfg = nf.HashEncodingConfig(levels=16, table_size=1 << T_log2, features=2, n_min=16, n_max=n_max, dims=2)
    m.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=3,
                             output_activation=nf.OutputActivation.Sigmoid)
    m.hyper = nf.AdamHyper(lr=1e-2)
    m.init(1337)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    Xs = [torch.rand(B_TRAIN, 2, device="cuda", generator=gen) for _ in range(4)]
    Ts = [image_target_torch(x) for x in Xs]
    stream = torch.cuda.ExternalStream(ctx.stream)
    for i in range(warmup):
        m.train_step_device(Xs[i % 4], Ts[i % 4], B_TRAIN, B_TRAIN, nf.LossKind.L2, i + 1)
    m.check()
    torch.cuda.synchronize()
    ctx.synchronize()
    import ctypes as C
    prof = (C.c_double * 4)()
    nst = C.c_int64()
    ctx.lib.nfg_ctx_set_profiling(ctx.h, 1)
    ctx.lib.nfg_ctx_read_profile(ctx.h, prof, C.byref(nst))   # reset
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        m.train_step_device(Xs[i % 4], Ts[i % 4], B_TRAIN, B_TRAIN, nf.LossKind.L2, warmup + i + 1)
    e1.record(stream)
    ctx.synchronize()
    torch.cuda.synchronize()
    ctx.lib.nfg_ctx_read_profile(ctx.h, prof, C.byref(nst))
    ctx.lib.nfg_ctx_set_profiling(ctx.h, 0)
    m.check()
    ms = e0.elapsed_time(e1) / steps
    n = m.parameter_count()
    m.close()
    return {"metric": metric or "gigapixel-image training samples/s (config 3, one GPU)",
            "value": B_TRAIN / (ms / 1000.0),
            "unit": "samples/s", "ms_per_step": ms, "params": n, "steps": steps, "warmup": warmup,
            "phases_ms_per_step": {"train_kernel": prof[0] / steps, "adam": prof[1] / steps},
            "config": config or (f"2D hash L16 F2 T2^{T_log2} Nmin16 Nmax{n_max}, MLP 32-64-64-3 sigmoid, L2, batch "
                                 f"2^{B_TRAIN.bit_length() - 1} random points of the procedural image "
                                 "(helpers.hpp:99-125) evaluated on the fly")}


def bench_nerf(nf, ctx, steps, warmup, W=128, views=16, samples=1 << 18):
    """BASELINE config 4 on one GPU: hash NeRF (T=2^19, density 1x64->16, color
    2x64->3) on the synthetic procedural scene, 2^18 compacted samples per step.
    Each step syncs once (sample count), so it is timed on the host clock."""
    cams, focal = nf.orbit_cameras(views, width=W)
    images = nf.nerf_scene_render(cams, W, W, focal, ctx=ctx)
    nerf = nf.NeRF(lr=1e-2, target_samples=samples, seed=1337, ctx=ctx)
    nerf.set_dataset(cams, images, W, W, focal)
    for s in range(1, warmup + 1):
        nerf.train_step(s)
    ctx.synchronize()
    t0 = time.perf_counter()
    tot_s = tot_r = tot_b = 0
    loss = 0.0
    for s in range(warmup + 1, warmup + steps + 1):
        loss, nr, ns = nerf.train_step(s)
        tot_s += ns
        tot_r += nr
        tot_b += nerf.last_backward_samples
    nerf.sync()   # the last step's deferred Adam belongs in the region
    ctx.synchronize()
    dt = time.perf_counter() - t0
    nerf.close()
    return {"metric": "NeRF training samples/s (config 4, synthetic scene)", "value": tot_s / dt, "unit": "samples/s",
            "rays_per_s": tot_r / dt, "ms_per_step": 1000.0 * dt / steps, "samples_per_step": tot_s / steps,
            "rays_per_step": tot_r / steps, "backward_samples_per_step": tot_b / steps, "steps": steps,
            "warmup": warmup, "loss": loss,
            "config": f"{views} views {W}x{W}, hash L16 F2 T2^19 Nmin16 Nmax2048, occupancy 128^3, "
                      f"dt sqrt(3)/1024, target 2^18 samples/step; timed on the host clock (one sync per step)"}


def sdf_torch(X):
    """Analytic CSG target of config 2 (sphere r=.3 U torus R=.25 r=.08 at the cube centre)."""
    import torch
    c = X - 0.5
    sphere = torch.sqrt((c * c).sum(1)) - 0.3
    q = torch.sqrt(c[:, 0] ** 2 + c[:, 2] ** 2) - 0.25
    torus = torch.sqrt(q * q + c[:, 1] ** 2) - 0.08
    return torch.minimum(sphere, torus).unsqueeze(1).contiguous()


def cpu_reference(steps, warmup, seconds_cap, native=True, batch=B_TRAIN):
    """Times the CPU restatement (oracle) of the reference on this host's cores."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import oracle as O
    if native:
        try:
            O.build(native=True)
        except Exception:
            native = False
    f = O.Field(O.GridCfg(**{"levels": 16, "table_size": 1 << 19, "features": 2, "n_min": 16, "n_max": 2048,
                             "dims": 3}), O.MlpCfg(hidden_layers=2, hidden_width=64, output_width=1),
                O.Hyper(lr=LR), native=native)
    f.init(1337)
    # The reference's MLP runs on Eigen GEMMs (mlp.hpp:114,147-149); time the
    # port with blocked FMA GEMMs in their place (nf_oracle.hpp fast::), not the
    # parity oracle's fixed-order loops, so the baseline is not understated.
    f.set_fast_mlp(True)
    rng = O.Pcg32(1337, 2)
    X = rng.floats(batch * 3).reshape(batch, 3)
    T = O.csg_sdf(X).reshape(batch, 1)
    for s in range(warmup):
        f.train_step(X, T, O.LOSS_MAPE, s + 1)
    f.reset_times()
    t0 = time.perf_counter()
    done = 0
    for s in range(steps):
        f.train_step(X, T, O.LOSS_MAPE, warmup + s + 1)
        done += 1
        if time.perf_counter() - t0 > seconds_cap:
            break
    dt = time.perf_counter() - t0
    threads = O.lib(native).orc_max_threads()
    # inference on the same host (queries/s at 2^20 queries; evaluate_chunked's
    # 2^16-column chunks, tasks.cpp:34-45)
    Q = O.Pcg32(7, 7).floats(3 * (1 << 20)).reshape(-1, 3)
    f.evaluate(Q[:1 << 16])
    t1 = time.perf_counter()
    for c0 in range(0, 1 << 20, 1 << 16):
        f.evaluate(Q[c0:c0 + (1 << 16)])
    qps = (1 << 20) / (time.perf_counter() - t1)
    # one thread (the reference's deterministic single-thread mode, acceptance.cpp:675;
    # SURVEY §8d): two steps, capped at a few seconds
    lib = O.lib(native)
    lib.orc_set_threads(1)
    t2 = time.perf_counter()
    one = 0
    while one < 2 and time.perf_counter() - t2 < 8.0:
        f.train_step(X, T, O.LOSS_MAPE, warmup + done + one + 1)
        one += 1
    v1 = one * batch / (time.perf_counter() - t2)
    lib.orc_set_threads(threads)
    return {"value": done * batch / dt, "steps": done, "seconds": dt, "threads": threads,
            "phases_s_per_step": {k: v / done for k, v in f.phase_times().items()}, "native": native,
            "inference_queries_per_s": qps, "value_1_thread": v1}


def run_reference(args, rank, world):
    if rank != 0:
        return
    r = cpu_reference(args.steps, args.warmup, seconds_cap=150.0)
    sample = (f"config2 full batch 2^18 per step, {r['steps']} timed steps after {args.warmup} warm-up, "
              f"CPU restatement of the reference (oracle/nf_oracle.hpp, -O2 -march=native, OpenMP "
              f"{r['threads']} threads; MLP on blocked FMA GEMMs standing in for Eigen; "
              f"encode_backward/Adam single-threaded as in the reference)")
    line = {"metric": METRIC, "value": r["value"], "unit": "samples/s", "n_gpus": world, "steps": r["steps"],
            "warmup": args.warmup, "ms_per_step": 1000.0 * r["seconds"] / max(r["steps"], 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOAD, "global_batch": B_TRAIN, "parallelism": "cpu"},
            "cpu_baseline": {"value": r["value"], "unit": "samples/s", "cores": r["threads"], "kind": "port",
                             "sample": sample, "phases_s_per_step": r["phases_s_per_step"],
                             "inference_queries_per_s": r["inference_queries_per_s"],
                             "value_1_thread": r["value_1_thread"]},
            "e2e": {"value": r["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl != "reference":
        rc = launch_ranks(args)
        if rc is not None:
            sys.exit(rc)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but this job has WORLD_SIZE={world} ranks; refusing to report "
                 "a number for a GPU count that is not the one measured")
    if args.launcher_selftest:
        return launcher_selftest(rank, world)

    import numpy as np
    import torch
    import torch.distributed as dist
    if torch.cuda.device_count() < world:
        sys.exit(f"bench.py: {world} ranks requested but only {torch.cuda.device_count()} GPUs are visible")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2201_05989_b200 import nf

    ctx = nf.Context(local)
    if world > 1:
        uid = [nf.Context.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.attach_comm(uid[0], rank, world)
        comm_rank, comm_size = ctx.comm_info()
        assert (comm_rank, comm_size) == (rank, world), (
            f"NCCL communicator reports rank {comm_rank} of {comm_size}, expected {rank} of {world}")
    model = nf.FieldModel(ctx, options=nf.Options(mlp_engine=args.mlp_engine))
    model.hash_cfg = nf.HashEncodingConfig(**CFG2)
    model.mlp_cfg = nf.MlpConfig(hidden_layers=2, hidden_width=64, output_width=1)
    model.hyper = nf.AdamHyper(lr=LR)
    model.init(1337)
    n_params = model.parameter_count()

    # resident synthetic batches (distinct per rank: data-parallel shards)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1337 + rank)
    Xs = [torch.rand(B_TRAIN, 3, device="cuda", generator=gen) for _ in range(N_RESIDENT)]
    Ts = [sdf_torch(x) for x in Xs]
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ctx.synchronize()

    step = 0

    def one(i):
        nonlocal step
        step += 1
        model.train_step_device(Xs[i % N_RESIDENT], Ts[i % N_RESIDENT], B_TRAIN, B_TRAIN * world,
                                nf.LossKind.Mape, step)

    clk = Clocks(local).start()
    t_wait = time.perf_counter()
    while not clk.rows and time.perf_counter() - t_wait < 3.0:   # first sample before timing
        time.sleep(0.01)
    for i in range(args.warmup):
        one(i)
    model.check()
    barrier()
    launches0 = ctx.launch_count
    lib = ctx.lib
    import ctypes as C
    lib.nfg_ctx_set_profiling(ctx.h, 1)
    ms = (C.c_double * 4)()
    nst = C.c_int64()
    lib.nfg_ctx_read_profile(ctx.h, ms, C.byref(nst))   # reset
    barrier()
    mark0 = clk.mark()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for i in range(args.steps):
        one(args.warmup + i)
    ev1.record(stream)
    barrier()
    mark1 = clk.mark()
    launches = ctx.launch_count - launches0
    t_ms = ev0.elapsed_time(ev1)
    lib.nfg_ctx_read_profile(ctx.h, ms, C.byref(nst))
    lib.nfg_ctx_set_profiling(ctx.h, 0)
    model.check()
    t_max = t_ms
    if world > 1:
        tt = torch.tensor([t_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    value = world * B_TRAIN * args.steps / (t_max / 1000.0)
    phase_ms = [ms[i] / max(args.steps, 1) for i in range(4)]

    # ---- strong scaling: global batch 2^18 split over the ranks ----
    strong = None
    if world > 1:
        try:
            b_loc = B_TRAIN // world
            barrier()
            ev0.record(stream)
            for i in range(args.steps):
                step += 1
                model.train_step_device(Xs[i % N_RESIDENT][:b_loc], Ts[i % N_RESIDENT][:b_loc], b_loc, B_TRAIN,
                                        nf.LossKind.Mape, step)
            ev1.record(stream)
            barrier()
            tt = torch.tensor([ev0.elapsed_time(ev1)], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_s = float(tt.item())
            strong = {"value": B_TRAIN * args.steps / (t_s / 1000.0), "unit": "samples/s", "global_batch": B_TRAIN,
                      "batch_per_gpu": b_loc, "ms_per_step": t_s / args.steps}
            model.check()
        except Exception as e:   # secondary number: never lose the headline line
            strong = {"error": str(e)[:200]}

    # ---- e2e: public API on pinned host buffers ----------------------------
    Xh = nf.PinnedBuffer((B_TRAIN, 3))
    Th = nf.PinnedBuffer((B_TRAIN, 1))
    Xh.array[:] = Xs[0].cpu().numpy()
    Th.array[:] = Ts[0].cpu().numpy()
    for i in range(2):
        step += 1
        model.train_step_host_ptr(Xh.ptr, Th.ptr, B_TRAIN, nf.LossKind.Mape, step)
    barrier()
    e2e_steps = max(10, args.steps)
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        step += 1
        loss = model.train_step_host_ptr(Xh.ptr, Th.ptr, B_TRAIN, nf.LossKind.Mape, step)
    ctx.synchronize()   # train_step returns once its loss is known; the last Adam belongs in the region
    t_e2e = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([t_e2e], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e_value = world * B_TRAIN * e2e_steps / t_e2e
    # the same call on PAGEABLE host memory (a reference caller's Eigen::MatrixXf
    # or a plain numpy array handed to the C ABI)
    Xp = np.array(Xh.array, copy=True)
    Tp = np.array(Th.array, copy=True)
    Xh.free()
    Th.free()
    for i in range(2):
        step += 1
        model.train_step_host_ptr(Xp.ctypes.data, Tp.ctypes.data, B_TRAIN, nf.LossKind.Mape, step)
    barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        step += 1
        loss = model.train_step_host_ptr(Xp.ctypes.data, Tp.ctypes.data, B_TRAIN, nf.LossKind.Mape, step)
    ctx.synchronize()
    t_pg = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([t_pg], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_pg = float(tt.item())
    e2e_pageable = world * B_TRAIN * e2e_steps / t_pg
    del Xp, Tp

    # ---- inference queries/s (config 5, queries sharded, no communication) ----
    Bq = args.infer_b
    Xq = torch.rand(Bq, 3, device="cuda", generator=gen)
    out = torch.empty(Bq, 1, device="cuda")
    for _ in range(3):
        model.evaluate_device(Xq, Bq, out)
    barrier()
    iters = 10
    ev0.record(stream)
    for _ in range(iters):
        model.evaluate_device(Xq, Bq, out)
    ev1.record(stream)
    barrier()
    t_inf = ev0.elapsed_time(ev1) / iters
    if world > 1:
        tt = torch.tensor([t_inf], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_inf = float(tt.item())
    qps = world * Bq / (t_inf / 1000.0)

    # config-5 sweep 2^16 .. 2^26 queries per GPU (same model, device-resident queries)
    sweep = []
    if rank == 0 and not args.no_nerf:
        for lg in (16, 18, 20, 22, 24, 26):
            nq = 1 << lg
            Xs_ = Xq[:nq] if nq <= Bq else torch.rand(nq, 3, device="cuda", generator=gen)
            o_ = torch.empty(nq, 1, device="cuda")
            for _ in range(2):
                model.evaluate_device(Xs_, nq, o_)
            ctx.synchronize()
            reps = max(3, min(50, (1 << 24) // nq))
            ev0.record(stream)
            for _ in range(reps):
                model.evaluate_device(Xs_, nq, o_)
            ev1.record(stream)
            ctx.synchronize()
            ms_ = ev0.elapsed_time(ev1) / reps
            sweep.append({"queries": nq, "queries_per_s": nq / (ms_ / 1000.0), "ms_per_call": ms_})
            del Xs_, o_

    # ---- config 3: gigapixel image, tables beyond L2 (one GPU) ----------------------
    # Secondary single-GPU numbers run on rank 0 only, on a context WITHOUT the
    # communicator: a field on the data-parallel context would issue collectives
    # the other ranks never join.
    sctx = nf.Context(local) if world > 1 and rank == 0 and not args.no_nerf else ctx
    giga_line = None
    if rank == 0 and not args.no_nerf:   # secondary, single-GPU numbers: rank 0 only
        try:
            giga_line = bench_gigapixel(nf, sctx, steps=max(5, args.steps // 2), warmup=3)
        except Exception as e:
            giga_line = {"error": str(e)[:200]}

    # ---- config 1: 2D image regression (the reference's CPU-runnable case) ----------
    c1_line = None
    if rank == 0 and not args.no_nerf:
        try:
            c1_line = bench_gigapixel(nf, sctx, steps=max(10, args.steps), warmup=5, T_log2=14, n_max=1024,
                                      batch=1 << 16, metric="image training samples/s (config 1, one GPU)",
                                      config="2D hash L16 F2 T2^14 Nmin16 Nmax1024, MLP 32-64-64-3 sigmoid, L2, "
                                             "lr 1e-2, batch 2^16 random points of the procedural image "
                                             "(helpers.hpp:99-125)")
        except Exception as e:
            c1_line = {"error": str(e)[:200]}

    # ---- config 4: NeRF training (occupancy-grid marching, compacted samples) ----
    nerf_line = None
    if rank == 0 and not args.no_nerf:
        try:
            nerf_line = bench_nerf(nf, sctx, steps=max(10, args.steps), warmup=40)
        except Exception as e:   # secondary number: never lose the headline line
            nerf_line = {"error": str(e)[:200]}

    clk.stop()
    clocks = clk.summary(mark0 if mark1 > mark0 else 0)
    if mark1 <= mark0:
        clocks["note"] = "no sample inside the training timed region; summary over the whole measurement"
    clocks["train_region_samples"] = mark1 - mark0

    # ---- roofline of the dominant kernel --------------------------------------
    # k_train and k_infer are L2-level bound (tables and gradients stay in the
    # 126 MB L2: ncu DRAM traffic is ~6% of their algorithmic bytes), so their
    # denominator is the L2-level rate of exactly their access kinds, measured
    # live on this GPU (csrc/diag.cu): random 4 B cp.async sector gathers,
    # random red.global.add.v2.f32 sector reductions, random 4 B ld.global.nc
    # gathers. Adam streams p/m/v from HBM: its denominator is the HBM peak.
    hbm_peak, tflops_peak, peak_src = peaks()
    l2 = {}
    try:
        for name, op in (("gather_cp_async", 1), ("red_v2_f32", 2), ("gather_ld_nc", 4), ("gather_ld_cg", 0),
                         ("stream_read", 3)):
            l2[name] = ctx.l2_peak(op)
    except Exception as e:   # never lose the headline line
        l2 = {"error": str(e)[:200]}
    train_ms, adam_ms = phase_ms[0], phase_ms[1]
    adam_gbs = n_params * ADAM_BYTES_PER_PARAM / (adam_ms / 1000.0) / 1e9 if adam_ms > 0 else None
    enc_bytes = B_TRAIN * (ENC_FWD_L2_BYTES_PER_SAMPLE + ENC_BWD_L2_BYTES_PER_SAMPLE)
    train_l2_gbs = enc_bytes / (train_ms / 1000.0) / 1e9 if train_ms > 0 else None
    train_tflops = B_TRAIN * MLP_TRAIN_FLOP_PER_SAMPLE / (train_ms / 1000.0) / 1e12 if train_ms > 0 else None
    ncu = ncu_traffic()
    fwd_sec, bwd_sec = ENC_FWD_L2_BYTES_PER_SAMPLE / 32, ENC_BWD_L2_BYTES_PER_SAMPLE / 32
    roof_train = roof_infer = None
    if "error" not in l2 and train_ms > 0:
        # time the kernel's sector mix needs at the measured per-kind rates
        t_bound = B_TRAIN * (fwd_sec / l2["gather_cp_async"] + bwd_sec / l2["red_v2_f32"])
        peak_mix = enc_bytes / t_bound / 1e9
        dram = ncu.get("k_train")
        roof_train = {
            "bound": "l2", "kernel": "k_train (fused encode+MLP+loss+backward)", "achieved": train_l2_gbs,
            "peak": peak_mix, "unit": "GB/s", "frac": train_l2_gbs / peak_mix, "traffic": dram,
            "peak_source": "measured live (csrc/diag.cu: random 4 B cp.async gathers and red.global.add.v2.f32, "
                           "L2-resident 96 MB footprint, full occupancy), weighted by the kernel's 72 gather + 80 "
                           "reduction sectors per sample",
            "algorithmic_bytes_per_launch": enc_bytes, "kernel_us": train_ms * 1000.0, "bound_us": t_bound * 1e6,
            "mlp_tflops": train_tflops, "mlp_tensor_frac": train_tflops / tflops_peak if train_tflops else None,
            "dram_gbs": dram / (train_ms / 1000.0) / 1e9 if dram else None,
            "dram_frac_of_hbm": dram / (train_ms / 1000.0) / 1e9 / hbm_peak if dram else None,
            "ncu": ncu.get("_src")}
        if t_inf > 0:
            inf_bytes = Bq * ENC_FWD_L2_BYTES_PER_SAMPLE
            t_b = Bq * fwd_sec / l2["gather_ld_nc"]
            ach = inf_bytes / (t_inf / 1000.0) / 1e9
            roof_infer = {
                "bound": "l2", "kernel": "k_infer (fused encode+MLP inference)", "achieved": ach,
                "peak": inf_bytes / t_b / 1e9, "unit": "GB/s", "frac": t_b / (t_inf / 1000.0),
                "traffic": ncu.get("k_infer"), "algorithmic_bytes_per_launch": inf_bytes,
                "kernel_us": t_inf * 1000.0, "bound_us": t_b * 1e6,
                "peak_source": "measured live (csrc/diag.cu: random 4 B ld.global.nc gathers), 72 sectors/query"}
    # legacy view kept for comparison with round 1: L2-level bytes over the HBM peak
    hbm_view = {"achieved": train_l2_gbs, "peak": hbm_peak, "frac": train_l2_gbs / hbm_peak if train_l2_gbs else None,
                "peak_source": peak_src, "note": "L2-level bytes over the HBM copy peak (round-1 convention; not "
                                                 "the binding resource)"}
    roof_adam = {"bound": "hbm", "kernel": "k_adam", "achieved": adam_gbs, "peak": hbm_peak, "unit": "GB/s",
                 "frac": adam_gbs / hbm_peak if adam_gbs else None, "traffic": ncu.get("k_adam"),
                 "algorithmic_bytes": n_params * ADAM_BYTES_PER_PARAM, "peak_source": peak_src}
    roof = roof_train if (roof_train and train_ms >= adam_ms) else roof_adam

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference(steps=100, warmup=1, seconds_cap=args.cpu_seconds, batch=1 << 16)
        cpu = {"value": r["value"], "unit": "samples/s", "cores": r["threads"], "kind": "port",
               "sample": f"config2 at batch 2^16 (a quarter of the 2^18 workload), {r['steps']} steps in "
                         f"{r['seconds']:.1f} s, CPU restatement of the reference (-O2 -march=native, OpenMP)",
               "phases_s_per_step": r["phases_s_per_step"],
               "inference_queries_per_s": r["inference_queries_per_s"], "value_1_thread": r["value_1_thread"]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f16-mma/f32-accum, f32 Adam",
                "data": "synthetic (U[0,1]^3 points, analytic CSG SDF targets; random-init weights)",
                "config": {"workload": WORKLOAD, "global_batch": B_TRAIN * world, "batch_per_gpu": B_TRAIN,
                           "parallelism": f"dp{world}" if world > 1 else "single",
                           "l2": "not flushed: each step streams ~0.42 GB of Adam state (> 126 MB L2); "
                                 f"inputs cycle over {N_RESIDENT} resident batches"},
                "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": B_TRAIN * 16,
                        "d2h_bytes_per_step": 32, "steps": e2e_steps, "host_memory": "pinned (cudaHostAlloc)"},
                "e2e_pageable": {"value": e2e_pageable, "unit": "samples/s", "h2d_bytes_per_step": B_TRAIN * 16,
                                 "d2h_bytes_per_step": 32, "steps": e2e_steps,
                                 "host_memory": "pageable (numpy arrays through the C ABI train_step)"},
                "inference": {"value": qps, "unit": "queries/s", "queries": Bq * world,
                              "ms_per_call": t_inf, "sweep_one_gpu": sweep},
                "strong_scaling": strong,
                "gigapixel": giga_line,
                "config1": c1_line,
                "nerf": nerf_line,
                "phases_ms_per_step": ({"train_kernel": phase_ms[0], "adam": phase_ms[1]} if world == 1 else
                                       {"train_kernel": phase_ms[0],
                                        "allreduce_pipelined_with_adam": phase_ms[2]}),
                "roofline": roof, "roofline_infer": roof_infer, "roofline_adam": roof_adam,
                "roofline_train_hbm_view": hbm_view, "l2_peaks_measured": l2,
                "secondary_rates": {"adam_gbs": adam_gbs, "train_l2_gbs": train_l2_gbs,
                                    "train_mlp_tflops": train_tflops},
                "gpu_launches": launches, "clocks": clocks, "cpu_baseline": cpu,
                "params": n_params}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()   # the other ranks wait for rank 0's single-GPU secondaries
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

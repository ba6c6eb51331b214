#!/usr/bin/env python
"""CBP decryption benchmark on B200 (BASELINE.json metric: frames/sec @1080p).

Workload (BASELINE.json configs[2], the 1080p config the metric is quoted on):
1920x1080 RGB latents, coprime 11x11 kernel pairs, kernel re-estimated every 30 frames.
One *step* = one 30-frame kernel epoch: decode_frame on frame 0 (luma width search
9..25, tau 1e-6, default epsilon, validation on: the reference decoder defaults,
decoder.hpp:10-20) followed by spectral_deblur of all 3 planes of frames 1..29 with the
recovered kernel, which stays on the device (cbp_kernel_slot).

Inputs: synthetic U[0,1) latents generated on the device, blurred on the device by
cbp_encode_frames with pairs from cbp_generate_coprime_pair (reference-exact host
draw). A pool of --pool epochs (default 5: 150 frames, 3.8 GB of public frames) is cycled, so every
step reads inputs far larger than the 126 MB L2.

Arms:
  default          the B200 path (libcbp_cuda.so via the C ABI), device-resident inputs
                   (`value`), plus the same metric through the host-buffer C ABI call
                   cbp_decode_run_host with pinned host memory (`e2e`).
  --impl reference the reference's CPU implementation of the path: the FP64 oracle
                   restatement (oracle/, the reference itself cannot be built here:
                   Eigen3/FFTW3 absent) on all host threads, frames in parallel like
                   `cbp decode` (tools/cbp.cpp:141-164).

Multi-GPU (torchrun): each rank decodes its own epochs (frames/streams are independent,
no collective on the data path); value = all frames / max-over-ranks time.
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

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "CBP decrypt frames/sec @1080p (1/2/4/8 B200); HBM GB/s % of peak; vs CPU ref"
ROWS, COLS, CH, T = 1080, 1920, 3, 11
EPOCH = 30


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--pool", type=int, default=5, help="distinct epochs cycled by the steps (>= recovery streams + 2)")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--profile-steps", type=int, default=3)
    p.add_argument("--cpu-threads", type=int, default=0)
    return p.parse_args()


# ------------------------------------------------------------------ helpers
def peaks():
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the GPU is busy."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
                for n, v in zip(names, r[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend, init_method="env://")
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def streams_for_rank(n_streams: int, world: int, rank: int) -> list:
    """Stream s of a multi-camera run goes to GPU s mod G;
    frames of different streams are independent, so there is no data-path collective."""
    return [s for s in range(n_streams) if s % world == rank]


def epoch_seed(e: int, rank: int) -> int:
    """Per-rank kernel epochs for the weak-scaling run: rank r decodes its own epochs."""
    return e + 1000 * rank


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------- CPU baseline
def cpu_reference_sample(pub32: np.ndarray, prv32: np.ndarray, kernel: np.ndarray, eps: float, threads: int,
                         n_frames: int):
    """Times the FP64 oracle (the reference restatement) on n_frames of one epoch with
    `threads` workers: frame 0 recovers the kernel (decode_frame), the rest reuse it
    (spectral_deblur of every plane). Returns frames/second."""
    from oracle import oracle as O
    rec = np.zeros(n_frames, np.int32)
    rec[0] = 1
    cfg = O.make_cfg(9, 25, 1e-6, validate=True)
    secs = O.bench_frames(pub32[:n_frames], prv32[:n_frames], rec, kernel, eps, cfg, threads)
    return n_frames / secs, secs


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path (oracle port) on the box's host cores."""
    if rank != 0:
        return
    from oracle import oracle as O
    threads = args.cpu_threads or os.cpu_count() or 1
    n = EPOCH  # one step = one whole epoch, the same frame mix as the GPU arm's step
    # identical synthetic workload shape: 1080p RGB, t = 11, epoch of 30 frames
    pair = O.generate_coprime_pair(T, O.frame_seed(2, 0))
    lat = np.stack([O.random_frame(ROWS, COLS, CH, O.frame_seed(1, i)) for i in range(n)])
    pub = np.empty((n, CH, ROWS + T - 1, COLS + T - 1), np.float32)
    prv = np.empty_like(pub)
    for i in range(n):
        a, b = O.encode_frame(lat[i], pair.k1, pair.k2)
        pub[i], prv[i] = a, b
    for _ in range(args.warmup):
        cpu_reference_sample(pub, prv, pair.k1, 1e-8, threads, n)
    times = []
    for _ in range(args.steps):
        fps, secs = cpu_reference_sample(pub, prv, pair.k1, 1e-8, threads, n)
        times.append(secs)
    value = n * len(times) / sum(times)
    line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "c3: 1920x1080 RGB, t=11, kernel re-estimated every 30 frames",
                       "rows": ROWS, "cols": COLS, "channels": CH, "kernel_width": T,
                       "parallelism": f"{threads} host threads, frames in parallel (tools/cbp.cpp:141-164)"},
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "port",
                             "sample": f"{n} frames of one epoch per step (1 decode_frame + {n - 1} spectral_deblur)"},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- B200 arm
SM_RESERVE = int(os.environ.get("CBP_BENCH_SM_RESERVE", "12"))
REC_STREAMS = int(os.environ.get("CBP_BENCH_REC_STREAMS", "3"))  # recoveries in flight


def run_b200(args, world, rank, local):
    import torch
    from paper_1203_4874_b200 import api

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    Mb, Nb = ROWS + T - 1, COLS + T - 1
    M, Nn = ROWS, COLS
    E = max(1, args.pool)
    # ---- inputs: device-generated latents, device encode (untimed)
    # device frames use a 16-byte row pitch (like cudaMallocPitch): vector copies in pass A
    NbP = (Nb + 3) // 4 * 4
    pub = torch.empty((E, EPOCH, CH, Mb, NbP), dtype=torch.float32, device=dev)[..., :Nb]
    prv = torch.empty((E, 1, CH, Mb, NbP), dtype=torch.float32, device=dev)[..., :Nb]
    pairs = []
    for e in range(E):
        pair = api.generate_coprime_pair(T, api.frame_seed(2, epoch_seed(e, rank)))
        pairs.append(pair)
        lat = api.synth_frames(EPOCH * CH, ROWS, COLS, seed=api.frame_seed(1, epoch_seed(e, rank)))
        lat = lat.view(EPOCH, CH, ROWS, COLS)
        p, q = api.encode_frame(lat, pair.k1, pair.k2)
        pub[e].copy_(p)
        prv[e, 0].copy_(q[0])
        del lat, p, q
    out = torch.empty((E, EPOCH, CH, Mb, NbP), dtype=torch.float32, device=dev)[..., :Nb]
    slots = torch.zeros((E, api.SLOT_BYTES), dtype=torch.uint8, device=dev)
    cfg = api.make_cfg(9, 25, 1e-6, validate=True)
    torch.cuda.synchronize(dev)

    # Recovery (decode_frame on frame 0) of the next epochs runs on recovery streams (one
    # context each: separate workspaces) while epoch s deconvolves: the recovery kernels are
    # latency bound on few SMs, the deconvolution passes fill the GPU. Epochs are
    # independent (slots/outputs are per epoch). An epoch's buffers are reused only after
    # its previous deconvolution finished (deb_ev).
    from paper_1203_4874_b200 import _native
    # The recovery chains have the higher priority and the deconvolution's persistent
    # grids leave them SM_RESERVE SMs' worth of slots.
    ctx_rec = [_native.Context(local) for _ in range(REC_STREAMS)]
    s_rec = [torch.cuda.Stream(dev, priority=-1) for _ in range(REC_STREAMS)]
    api.set_sm_reserve(SM_RESERVE, device=local)
    s_deb = torch.cuda.current_stream(dev)
    dec_ev = [torch.cuda.Event() for _ in range(E)]
    deb_ev = [torch.cuda.Event() for _ in range(E)]
    if E < REC_STREAMS + 2:
        raise ValueError(f"--pool must be >= {REC_STREAMS + 2} for the pipelined step")

    def issue_decode(s):
        # dec_ev[e] after the whole recovery frame (validation included): measured on B200,
        # releasing the deconvolution at slot-ready (decode_frames_async(slot_ready=...))
        # overlaps the FP64 validation with it and costs ~13% of throughput
        e, r = s % E, s % REC_STREAMS
        s_rec[r].wait_event(deb_ev[e])  # the epoch's previous deconvolution read its slot
        api.decode_frames_async(pub[e, 0:1], prv[e], cfg, out[e, 0:1], slots[e], ctx=ctx_rec[r], stream=s_rec[r])
        dec_ev[e].record(s_rec[r])

    def issue_deblur(s):
        e = s % E
        s_deb.wait_event(dec_ev[e])
        api.spectral_deblur_slot(pub[e, 1:], slots[e].data_ptr(), out[e, 1:], stream=s_deb)
        deb_ev[e].record(s_deb)

    def run_steps(n, start=0):
        """n pipelined steps: recoveries run REC_STREAMS epochs ahead of the deconvolution."""
        for s in range(start, start + min(REC_STREAMS, n)):
            issue_decode(s)
        for s in range(start, start + n):
            if s + REC_STREAMS < start + n:
                issue_decode(s + REC_STREAMS)
            issue_deblur(s)
        for st in s_rec:
            done = torch.cuda.Event()
            done.record(st)
            s_deb.wait_event(done)

    def step(s):
        run_steps(1, s)

    def count_launches():
        return api.launch_count(local) + sum(int(_native.lib().cbp_launch_count(c.ptr)) for c in ctx_rec)

    def run_steady(n, start=0):
        """n steps of the running pipeline: the recoveries of epochs start..start+REC_STREAMS-1
        are issued and finished BEFORE the timed region (pipeline pre-roll, untimed); inside it
        every step issues one recovery (REC_STREAMS epochs ahead) and one deconvolution batch,
        so the region holds exactly n recoveries + n x 29 deblurs, in steady state (no fill
        stall while the first recovery runs alone). Returns (ev0, ev1) around the region."""
        for s in range(start, start + REC_STREAMS):
            issue_decode(s)
        torch.cuda.synchronize(dev)
        barrier(world)
        torch.cuda.synchronize(dev)
        l0 = count_launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for st in s_rec:
            st.wait_event(e0)
        for s in range(start, start + n):
            issue_decode(s + REC_STREAMS)
            issue_deblur(s)
        for st in s_rec:
            done = torch.cuda.Event()
            done.record(st)
            s_deb.wait_event(done)
        e1.record(stream)
        return e0, e1, count_launches() - l0

    # ---- correctness guard on the pool (every epoch recovers its own kernel)
    for s in range(E):
        step(s)
    torch.cuda.synchronize(dev)
    for e, sl in enumerate(api.read_slots(slots, E)):
        if sl.status != 0 or sl.width != T:
            raise RuntimeError(f"epoch {e}: recovery failed (status {sl.status}, width {sl.width})")
        k = np.array(sl.weights[: T * T]).reshape(T, T)
        err = np.linalg.norm(k - pairs[e].k1) / np.linalg.norm(pairs[e].k1)
        if err > 1e-4:
            raise RuntimeError(f"epoch {e}: kernel error {err:.2e}")

    sampler = ClockSampler(local)
    sampler.start()
    for s in range(args.warmup):
        step(s)
    # keep the GPU busy >= 0.3 s before the timed region so clocks are sampled under load
    t_end = time.time() + 0.3
    s = 0
    while time.time() < t_end:
        step(s)
        s += 1
        if s % 8 == 0:
            torch.cuda.synchronize(dev)
    torch.cuda.synchronize(dev)
    ev0, ev1, launches = run_steady(args.steps)
    torch.cuda.synchronize(dev)
    barrier(world)
    ms_rank = ev0.elapsed_time(ev1)
    clocks = sampler.stop()
    ms = max_over_ranks(ms_rank, world)
    frames = EPOCH * args.steps * world
    value = frames / (ms / 1000.0)

    # ---- roofline of the dominant kernel group (deconvolution passes A+B+C)
    api.profile(True, local)
    torch.cuda.synchronize(dev)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    for st in s_rec:
        st.wait_event(pe0)
    run_steps(args.profile_steps)
    pe1.record(stream)
    torch.cuda.synchronize(dev)
    pass_ms, planes, groups = api.profile_read(local)
    api.profile(False, local)
    prof_step_ms = pe0.elapsed_time(pe1) / max(args.profile_steps, 1)
    deblur_ms = sum(pass_ms)
    bytes_per_plane = (Mb * Nb + M * Nn) * 4  # compulsory: blurred plane in, latent plane out
    achieved = bytes_per_plane * planes / (deblur_ms / 1000.0) / 1e9
    peak, peak_kind = peaks()
    traffic = None
    tp = os.path.join(HERE, "profiles", "deblur_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_plane")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_kind": peak_kind,
                "kernel": "deconvolution passes A+B+C (k_rows_forward, k_cols_filter, k_rows_inverse)",
                "algorithmic_bytes_per_plane": bytes_per_plane, "planes": planes,
                "pass_ms_per_plane": [m / max(planes, 1) for m in pass_ms],
                "share_of_step": deblur_ms / max(args.profile_steps, 1) / prof_step_ms}

    # ---- end-to-end through the host-buffer C ABI call (pinned host memory)
    e2e = None
    if not args.no_e2e:
        # one host-buffer run of e2e_steps epochs (distinct pool epochs), like the reference CLI
        # decoding a video run (tools/cbp.cpp:130-207): the pipeline streams across the epoch
        # boundaries (recovery frames at 0, 30, 60, ...) instead of refilling per epoch
        nE = args.e2e_steps
        hpub = torch.cat([pub[e % E].contiguous().cpu() for e in range(nE)]).pin_memory()
        hprv = torch.zeros_like(hpub).pin_memory()
        rec = np.zeros(EPOCH * nE, np.int32)
        for e in range(nE):
            hprv[EPOCH * e].copy_(prv[e % E, 0].cpu())
            rec[EPOCH * e] = 1
        hout = torch.empty_like(hpub).pin_memory()
        api.decode_run_host(hpub[:EPOCH], hprv[:EPOCH], rec[:EPOCH], cfg, out=hout[:EPOCH], device=local)  # warm-up
        barrier(world)
        t0 = time.perf_counter()
        _, sl = api.decode_run_host(hpub, hprv, rec, cfg, out=hout, device=local)
        t1 = time.perf_counter()
        barrier(world)
        e2e_s = max_over_ranks(t1 - t0, world)
        frame_bytes = CH * Mb * Nb * 4
        e2e = {"value": EPOCH * nE * world / e2e_s, "unit": "frames/s",
               "h2d_bytes_per_step": (EPOCH + 1) * frame_bytes, "d2h_bytes_per_step": EPOCH * frame_bytes,
               "steps": nE, "host_memory": "pinned",
               "api": f"cbp_decode_run_host (C ABI, host buffers, H2D/compute/D2H overlapped): one run of "
                      f"{nE} epochs = {EPOCH * nE} frames, a recovery frame every {EPOCH}"}
        if any(x.status != 0 or x.width != T for x in sl):
            raise RuntimeError("e2e recovery failed")
        del hpub, hprv, hout

    # ---- CPU baseline (rank 0, N = 1 only): bounded sample of the same workload
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = args.cpu_threads or os.cpu_count() or 1
        # one whole epoch (the step's own frame mix: 1 decode_frame + 29 spectral_deblur),
        # repeated until >= 10 s of CPU work (bounded at 6 repetitions)
        n = EPOCH
        pub_h = pub[0, :n].contiguous().cpu().numpy()
        prv_h = np.zeros_like(pub_h)
        prv_h[0] = prv[0, 0].cpu().numpy()
        reps, secs = 0, 0.0
        while reps < 6 and (reps == 0 or secs < 10.0):
            secs += cpu_reference_sample(pub_h, prv_h, pairs[0].k1, 1e-8, threads, n)[1]
            reps += 1
        fps = reps * n / secs
        cpu = {"value": fps, "unit": "frames/s", "cores": threads, "kind": "port",
               "sample": f"{reps} x one 1080p RGB epoch of {n} frames (1 decode_frame + {n - 1} spectral_deblur), "
                         f"{secs:.1f} s, FP64 oracle restatement (Eigen/FFTW reference unbuildable here)"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": "c3: 1920x1080 RGB, t=11, kernel re-estimated every 30 frames "
                                       "(1 decode_frame + 29 spectral_deblur per step)",
                           "rows": ROWS, "cols": COLS, "channels": CH, "kernel_width": T,
                           "frames_per_step": EPOCH, "pool_epochs": E,
                           "schedule": f"recoveries of epochs s+1..s+{REC_STREAMS} overlapped with deconvolution of epoch s "
                                       f"({REC_STREAMS} high-priority recovery streams + 1 deconvolution stream; "
                                       f"deconvolution leaves {SM_RESERVE} SMs); steady state: the recoveries of "
                                       f"the first {REC_STREAMS} epochs run before the timed region, each timed step "
                                       f"issues 1 recovery ({REC_STREAMS} epochs ahead) + 29 deblurs",
                           "l2": "inputs larger than L2 (each step reads 0.76 GB of distinct frames)",
                           "decode_cfg": "search 9..25, tau 1e-6, default epsilon, validate=true",
                           "parallelism": f"{world} independent GPU(s), no data-path collective"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "precision": "FP32 storage and deconvolution FFT; FP64 sampling and solves"}
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_b200(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

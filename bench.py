#!/usr/bin/env python
"""Benchmark of the encrypted-LR fast matmul hot path (arXiv 2204.05496).

Workload (default, BASELINE.json configs[3] = "C4"): 256 individuals x 40,000
features x 11 classes, N = 8192, production twin moduli (t0 = 1073872897,
t1 = 114689; 6 + 4 31-bit primes). One step = one matmul over the whole batch
(every (individual, class) pair: chunk products, 13 keyed rotations, mask,
packed accumulation, bias).

Arms:
  ours (default)      CUDA path, value = device-resident inputs (u32 in HBM),
                      e2e = C-ABI call with host u64 buffers (H2D + D2H timed).
  --impl reference    the reference's own CPU implementation (oracle/_ref,
                      compiled from /root/reference in the build container)
                      on the host cores, bounded sample per step.

Multi-GPU (torchrun): individuals shard across ranks (weak scaling, no
data-path collective; the packed partials would be combined by a mod-q add
of ~0.65 MB per rank). Rank 0 prints one JSON line.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

T0, T1, T1_16K = 1073872897, 114689, 163841
CONFIGS = {
    # name: (R, f, cols, N, p_feat, w_sigma)
    "c1": (1, 1000, 11, 8192, 0.05, 0.1),
    "c2": (1, 10000, 11, 8192, 0.05, 0.1),
    "c3": (1, 40000, 11, 8192, 0.03, 0.05),
    "c4": (256, 40000, 11, 8192, 0.03, 0.05),
    "c5": (4096, 40000, 33, 16384, 0.03, 0.05),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--rows", type=int, default=0, help="override individuals per rank")
    ap.add_argument("--batch-pairs", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-wire", dest="wire", action="store_false", help="skip the HECT wire-path e2e timing")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--latency", action="store_true", default=True, help="also time a single-individual (C3) call")
    ap.add_argument("--no-latency", dest="latency", action="store_false")
    ap.add_argument("--baseline", action="store_true", default=True, help="also time the standard algorithm at C3")
    ap.add_argument("--no-baseline", dest="baseline", action="store_false")
    return ap.parse_args()


def q_chain(n: int, t: int):
    """bfv::default_q_primes (params.cpp:84-104) for n >= 4096."""
    count = 6 if t >= (1 << 25) else 4
    two_n = 2 * n
    c = ((((1 << 31) - 2) // two_n) * two_n) + 1
    out = []
    while len(out) < count:
        if c != t and _is_prime(c):
            out.append(c)
        c -= two_n
    return out


def _is_prime(v: int) -> bool:
    if v < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if v % p == 0:
            return v == p
    d, r = v - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        x = pow(a, d, v)
        if x in (1, v - 1):
            continue
        for _ in range(r - 1):
            x = x * x % v
            if x == v - 1:
                break
        else:
            return False
    return True


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        cmd = ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
               "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the sampler is live (first line read) before the timed region starts
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 8:
                for k, nm in enumerate(names):
                    if r[4 + k].lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ reference
def reference_sample(cfg_name: str, rows: int | None = None, threads: int = 0):
    """Time the reference CPU path (oracle/_ref) on a bounded sample of the
    workload. Returns (inferences/s, sample description, threads, seconds)."""
    from oracle.oracle import Reference, TwinParams, ref_available
    from tests.helpers import synthetic

    R, f, cols, n, pf, ws = CONFIGS[cfg_name]
    if not ref_available():
        return None
    nthreads = threads or os.cpu_count() or 1
    r = rows or max(1, min(R, nthreads))
    p = TwinParams(n=n, t0=T0, t1=T1 if n < 16384 else T1_16K, sec=128)
    ref = Reference(p, key_seed=1, enc_seed=2)
    x, w, b = synthetic(r, f, cols, pf, ws)
    ref.encode_inputs(x)
    ref.set_weights(w)
    ref.set_bias(b)
    _, _, secs = ref.matmul(r, cols, threads=nthreads, export=False)
    return r / secs, f"{r} individuals x {f} features x {cols} classes (N={n}) per step", nthreads, secs, ref


def run_reference(args, world, rank):
    if rank != 0:
        return
    R, f, cols, n, _, _ = CONFIGS[args.config]
    res = reference_sample(args.config)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libheiref.so not built (needs /root/reference at build time)"}))
        return
    rate, sample, threads, _, ref = res
    r = max(1, min(R, threads))
    times = []
    for s in range(args.warmup + args.steps):
        _, _, secs = ref.matmul(r, cols, threads=threads, export=False)
        if s >= args.warmup:
            times.append(secs)
    v = r * len(times) / sum(times)
    line = {"metric": "encrypted LR inferences/sec at 40k features", "value": v, "unit": "inferences/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config}: {R}x{f}x{cols} N={n}", "sample_rows_per_step": r},
            "cpu_baseline": {"value": v, "unit": "inferences/s", "cores": threads, "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": "inferences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------ ours
def make_server(n, device, seed=1):
    """Twin context with real keys: TwinContext::keygen from util::Prng(1) run
    on the device (SURVEY §8d seeds), installed for both roles (server Galois
    keys, client public/secret keys). Returns (server, q0, q1, keygen_ms)."""
    from paper_2204_05496_b200 import GpuTwinServer, Prng, ScalingConfig

    t1 = T1 if n < 16384 else T1_16K
    q0, q1 = q_chain(n, T0), q_chain(n, t1)
    L = [len(q0), len(q1)]
    q = np.array(q0 + q1, dtype=np.uint64)
    srv = GpuTwinServer(n, (T0, t1), L, q, [], None, ScalingConfig(), device=device)
    srv.keygen(Prng(seed), install=True)  # warm (first-call allocations)
    t0 = time.perf_counter()
    srv.keygen(Prng(seed), install=True)
    kg_ms = (time.perf_counter() - t0) * 1000.0
    return srv, q0, q1, kg_ms


def wire_e2e(srv, ew, b, h_np, R, kc, n, L0, L1, world, steps):
    """Time hei_gpu_matmul_wire on the same residues laid out as the
    request's HECT blobs (serialize.cpp:63-78; treated as coeff form)."""
    import torch

    from paper_2204_05496_b200 import matmul_wire

    b0, b1 = srv.hect_bytes(0), srv.hect_bytes(1)
    hdr = [np.frombuffer(b"HECT\x01\x00" + srv.params_hash(k).to_bytes(8, "little") + b"\x02\x00\x00\x00\x05", np.uint8)
           for k in range(2)]
    buf = torch.empty(R * kc * (b0 + b1), dtype=torch.uint8, pin_memory=True)
    a = buf.numpy().reshape(R * kc, b0 + b1)
    src = h_np.reshape(R * kc, -1)
    off = 0
    for k, L in enumerate((L0, L1)):
        a[:, off:off + 19] = hdr[k]
        polys = a[:, off + 19: off + 19 + 2 * L * (1 + 8 * n)].reshape(R * kc, 2 * L, 1 + 8 * n)
        polys[:, :, 0] = 0
        w0 = (2 * L0 * n) if k else 0
        slab = np.ascontiguousarray(src[:, w0: w0 + 2 * L * n]).reshape(R * kc, 2 * L, n)
        polys[:, :, 1:] = slab.view(np.uint8).reshape(R * kc, 2 * L, 8 * n)
        off += (b0 if k == 0 else b1)
    outs, _ = matmul_wire(srv, ew, a, R, b)  # warm
    t0 = time.perf_counter()
    for _ in range(steps):
        outs, _ = matmul_wire(srv, ew, a, R, b)
    sec = (time.perf_counter() - t0) / steps
    res = {"value": world * R / sec, "unit": "inferences/s", "h2d_bytes_per_step": int(a.nbytes),
           "d2h_bytes_per_step": int(sum(len(o) for o in outs)), "ms_per_step": 1000 * sec,
           "format": "HECT coeff-form blobs [row][chunk][branch] in, HECT blobs out (server.cpp:112-172)"}
    del buf, a
    return res


def run_ours(args, world, rank, local):
    import torch

    from paper_2204_05496_b200 import encode_weights, matmul, matmul_device, native
    from tests.helpers import synthetic

    R_total, f, cols, n, pf, ws = CONFIGS[args.config]
    R = args.rows or R_total  # per rank (weak scaling: every rank gets the full per-GPU batch)
    # one process per GPU; the modulo only matters for the plumbing check below
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        # HEI_DIST_BACKEND=gloo: host-side exchange, used only to check the
        # multi-rank plumbing on a single-GPU box (never for numbers)
        backend = os.environ.get("HEI_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_2204_05496_b200 import Prng, encode_inputs_device

    srv, q0, q1, keygen_ms = make_server(n, local)
    if args.batch_pairs:
        srv.set_batch_pairs(args.batch_pairs)
    kc = (f + n - 1) // n
    P = len(q0) + len(q1)
    ctw = 2 * P * n
    # seeded synthetic individuals (rank r holds its own rows), weights, bias
    x, _, _ = synthetic(R, f, cols, pf, ws, seed=7 + rank)
    _, w, b = synthetic(1, f, cols, pf, ws)  # one model, shared by every rank
    ew = encode_weights(srv, w)
    # device-resident inputs: the client's real encryptions of x
    # (encode_inputs, matmul.cpp:201-223; Prng seeds 2, 3 as client_backend(keys, 2))
    d_in = torch.empty((R * kc, ctw), dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    for _ in range(2):  # first call also builds the cached mt19937_64 jump polynomial
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        encode_inputs_device(srv, x, Prng(2 + 2 * rank), Prng(3 + 2 * rank), d_in.data_ptr(), stream.cuda_stream)
        enc_ms = (time.perf_counter() - t0) * 1000.0
    C_ = (R * cols + n - 1) // n
    d_out = torch.empty((C_, ctw), dtype=torch.int32, device=dev)
    d_one = torch.empty((C_, ctw), dtype=torch.int32, device=dev)  # rank-local result (roofline step)

    if world == 1:
        def step():
            matmul_device(srv, d_in.data_ptr(), R, ew, b, d_out.data_ptr(), stream.cuda_stream)
    else:
        # individual sharding: rank r holds rows [r*R, (r+1)*R) of a world*R
        # batch; one int64 all-reduce of the packed partials (NCCL/NVLink),
        # then the mod-q reduction + bias add on every rank.
        from paper_2204_05496_b200.sharding import finish_packed_device, matmul_partial_device, packed_count

        total_rows = world * R
        Ct = packed_count(total_rows, cols, n)
        d_out = torch.empty((Ct, ctw), dtype=torch.int32, device=dev)
        exchange = os.environ.get("HEI_EXCHANGE", "p2p")
        acc = torch.zeros((Ct, ctw), dtype=torch.int64, device=dev)
        gather = None
        if exchange == "p2p":
            # each rank writes its packed accumulator into its slot of rank
            # 0's receive buffer through a CUDA IPC mapping (an NVLink peer
            # write); rank 0 sums the slots and finishes — no collective
            from paper_2204_05496_b200.sharding import PeerGather

            ok = 1
            try:
                gather = PeerGather(Ct * ctw * 8, local)
            except Exception as e:  # no peer access on this rank
                print(f"[bench] rank {rank}: p2p exchange unavailable ({e})", file=sys.stderr)
                ok = 0
            flag = torch.tensor([ok], dtype=torch.int32, device=dev)
            torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)  # every rank agrees
            if int(flag.item()) == 0:
                exchange = "nccl"
        if exchange == "p2p":
            def step():
                with torch.cuda.stream(stream):
                    acc.zero_()
                matmul_partial_device(srv, ew, d_in.data_ptr(), R, rank * R, total_rows, acc.data_ptr(),
                                      stream.cuda_stream)
                stream.synchronize()
                torch.distributed.barrier()  # the owner's previous reduce/finish is done with the slots
                gather.push(acc.data_ptr(), stream.cuda_stream)
                stream.synchronize()
                torch.distributed.barrier()  # every slot written
                if rank == 0:
                    gather.reduce(stream.cuda_stream)
                    finish_packed_device(srv, ew, gather.total_ptr, b, total_rows, d_out.data_ptr(),
                                         stream.cuda_stream)
        else:
            def step():
                with torch.cuda.stream(stream):
                    acc.zero_()
                matmul_partial_device(srv, ew, d_in.data_ptr(), R, rank * R, total_rows, acc.data_ptr(),
                                      stream.cuda_stream)
                with torch.cuda.stream(stream):
                    torch.distributed.all_reduce(acc)
                finish_packed_device(srv, ew, acc.data_ptr(), b, total_rows, d_out.data_ptr(), stream.cuda_stream)

    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    native.reset_launch_count()
    prof = os.environ.get("HEI_PROFILE_STEPS") == "1"  # ncu --profile-from-start off: timed steps only
    if prof:
        torch.cuda.cudart().cudaProfilerStart()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = native.launch_count()
    if prof:
        torch.cuda.cudart().cudaProfilerStop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = world * R / (ms / 1000.0)

    # e2e: host u64 (pinned) inputs through the C ABI, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        h_in = torch.empty((R, kc, ctw), dtype=torch.int64, pin_memory=True)
        h_in.copy_(d_in.view(R, kc, ctw).to(torch.int64).cpu())
        h_np = h_in.numpy().view(np.uint64)
        matmul(srv, h_np, ew, b)  # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_steps = max(1, min(args.steps, 3))
        for _ in range(e2e_steps):
            out, _ = matmul(srv, h_np, ew, b)
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        e2e = {"value": world * R / e2e_s, "unit": "inferences/s", "h2d_bytes_per_step": int(h_np.nbytes),
               "d2h_bytes_per_step": int(out.nbytes), "ms_per_step": 1000 * e2e_s}
        # the server's wire path (server.cpp:112-172): HECT coeff-form blobs
        # in, HECT blobs out, parse/NTT/INTT/serialize on the device
        if args.wire and world == 1:  # the wire copy doubles pinned host memory; one rank only
            e2e["wire"] = wire_e2e(srv, ew, b, h_np, R, kc, n, len(q0), len(q1), world, e2e_steps)
        del h_in, h_np

    # ---- roofline of the dominant kernel (key switch), timed live with CUDA
    # events on the launch stream inside the C ABI over one extra step.
    roof = int_roof = None
    if rank == 0:
        native.kernel_timing(srv.handle, True)
        # the rank's own fold work only: no collective, so rank 0 can time it alone
        matmul_device(srv, d_in.data_ptr(), R, ew, b, d_one.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        ks_n, ks_ms = native.kernel_stats(srv.handle, 0)
        dg_n, dg_ms = native.kernel_stats(srv.handle, 1)
        native.kernel_timing(srv.handle, False)
        L0, L1 = len(q0), len(q1)
        S = int(np.log2(n))  # fold steps per batch
        batches = ks_n // S
        # algorithmic bytes of one key-switch launch over P pairs: per pair
        # and output prime, c0/c1 read + out0/out1 written (4 polys of 4N B)
        # and L-1 digit polys read; the step's Galois key (2L polys of 8N B
        # per prime) once per launch.
        per_pair = sum(16 * n + 4 * n * (Lb - 1) for Lb in (L0, L1) for _ in range(Lb))
        keys = sum(16 * Lb * n * Lb for Lb in (L0, L1))
        tot_bytes = S * R * cols * per_pair + ks_n * keys
        avg_s = ks_ms / ks_n / 1000.0
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        hbm = float(peaks.get("hbm_gbs", 6650.0))
        traffic = None
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "keyswitch_traffic.json")))
            traffic = prof.get("dram_bytes_per_pair") * R * cols / batches
        except Exception:
            pass
        ach = tot_bytes / (ks_ms / 1000.0) / 1e9
        logn = n.bit_length() - 1
        blocks = R / batches * cols * (L0 + L1)  # (pair, prime) blocks per timed key-switch launch
        if blocks <= 148:
            ks_name = f"k_rot_keyswitch_w2<{logn}> (latency path: 2-group CTA, fused next digit)"
        elif logn == 14 and os.environ.get("HEI_KS14_TMEM", "1") != "0":
            ks_name = "k_rot_keyswitch_t<14> (TMEM accumulators, 1 CTA of 1024 threads/SM)"
        elif blocks < 296 or logn != 13 or os.environ.get("HEI_KS_TMEM", "4") == "0":
            ks_name = f"k_rot_keyswitch_s<{logn}> (shared-memory accumulators)"
        else:
            ks_name = "k_rot_keyswitch_t<13> (TMEM accumulators, 3 CTAs/SM)"
        roof = {"kernel": ks_name, "bound": "hbm", "achieved": ach, "peak": hbm,
                "unit": "GB/s", "frac": ach / hbm, "traffic": traffic,
                "algorithmic_bytes_per_launch": tot_bytes / ks_n, "avg_launch_ms": avg_s * 1e3, "launches": ks_n,
                "batches": batches, "peak_source": "MEASURED_PEAKS.json" if peaks else "fallback",
                "share_of_fold": ks_ms / (ks_ms + dg_ms), "digits_avg_launch_ms": dg_ms / max(1, dg_n)}
        bfly_pair = sum(((Lb - 1) * (n // 2) * S + 2 * Lb * n) for Lb in (L0, L1) for _ in range(Lb))
        tot_bfly = S * R * cols * bfly_pair
        peak_b = native.butterfly_peak(local)
        int_roof = {"kernel": ks_name, "bound": "int32 pipes (CT butterfly = Shoup mulmod + add + sub)",
                    "achieved": tot_bfly / (ks_ms / 1000.0) / 1e9, "peak": peak_b / 1e9, "unit": "Gbutterfly/s",
                    "frac": tot_bfly / (ks_ms / 1000.0) / peak_b,
                    "peak_source": "k_bfly_peak register microbenchmark, this run",
                    "butterfly_equivalents_per_launch": tot_bfly / ks_n}

    base = None
    if args.baseline and rank == 0:
        from paper_2204_05496_b200 import Prng, baseline_matmul

        R3, f3, c3, _, pf3, ws3 = CONFIGS["c3"]
        x3, w3, b3 = synthetic(R3, f3, c3, pf3, ws3)
        baseline_matmul(srv, x3, w3, b3, Prng(2), Prng(3))  # warm (incl. the cached jump polynomial)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, bc = baseline_matmul(srv, x3, w3, b3, Prng(2), Prng(3))
        bs = time.perf_counter() - t0
        base = {"algorithm": "standard (sample-batched, baseline_matmul)", "config": f"c3: {R3}x{f3}x{c3} N={n}",
                "ms": bs * 1000.0, "mul_plain": int(bc.mul_plain_count), "note": "host call incl. H2D of x, w and D2H"}
        base["client_encrypt"] = {"config": f"{R} individuals x {f} features ({R * kc} twin encryptions)",
                                  "ms": enc_ms, "individuals_per_s": R / (enc_ms / 1000.0)}

    lat = None
    if args.latency and rank == 0:
        # single individual, 40k features x 11 classes (C3 shape), device-resident
        d1 = d_in[:kc].contiguous()
        o1 = torch.empty((1, ctw), dtype=torch.int32, device=dev)
        for _ in range(3):
            matmul_device(srv, d1.data_ptr(), 1, ew, b, o1.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(10):
            matmul_device(srv, d1.data_ptr(), 1, ew, b, o1.data_ptr(), stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        lat = e0.elapsed_time(e1) / 10

    # client side of the result: decrypt + CRT unpack on the device
    # (unpack_results, matmul.cpp:257-271), checked against the exact product
    check = None
    if rank == 0:
        # world > 1: d_out is the all-reduced result of every rank's rows
        # (rank r encrypted synthetic(seed = 7 + r)); rank 0 regenerates them
        rows_all = world * R
        packed = d_out.cpu().numpy().view(np.uint32).astype(np.uint64)
        srv.unpack_results(packed, rows_all, cols)  # warm
        t0 = time.perf_counter()
        got = srv.unpack_results(packed, rows_all, cols)
        dec_ms = (time.perf_counter() - t0) * 1000.0
        x_all = x if world == 1 else np.concatenate(
            [synthetic(R, f, cols, pf, ws, seed=7 + r)[0] for r in range(world)], axis=0)
        want = np.rint(x_all.astype(np.float64) @ w.astype(np.float64)).astype(np.int64) + b  # exact: |sums| < 2^53
        check = {"decrypted_equals_integer_product": bool(np.array_equal(got, want)), "client_decrypt_ms": dec_ms,
                 "keygen_ms": keygen_ms, "client_encrypt_ms": enc_ms}

    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            res = reference_sample(args.config)
            if res:
                rate, sample, threads, secs, _ = res
                cpu = {"value": rate, "unit": "inferences/s", "cores": threads, "kind": "reference", "sample": sample,
                       "seconds": secs}
        except Exception as e:  # report, never fail the bench on the CPU leg
            cpu = {"error": str(e)}
    line = {
        "metric": "encrypted LR inferences/sec at 40k features",
        "value": value, "unit": "inferences/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {R} individuals/rank x {f} features x {cols} classes, N={n}, "
                               f"twin t=({T0},{T1 if n < 16384 else T1_16K}), L=({len(q0)},{len(q1)})",
                   "inputs": "real encryptions (device keygen from Prng(1), client encryption with Prng(2),(3)) of "
                             "seeded Bernoulli features, resident in HBM; inputs > L2 (no flush needed)",
                   "parallelism": f"dp{world} (individual sharding)" + (
                       f", exchange={exchange}" if world > 1 else "")},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    line["roofline"] = roof
    line["int_roofline"] = int_roof
    if lat is not None:
        line["latency_ms_single_individual"] = lat
    if base is not None:
        line["standard_algorithm"] = base
    if check is not None:
        line["client_roundtrip"] = check
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

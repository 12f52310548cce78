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
GOLDEN = os.path.join(ROOT, "tests", "golden", "configs")


def _configs():
    from paper_2204_05496_b200.workload import CONFIGS  # (R, f, cols, N, p_feat, w_sigma)

    return CONFIGS


def golden(case: str):
    """Reference-written digests (tests/golden/make_golden_configs.py)."""
    try:
        return json.load(open(os.path.join(GOLDEN, case + ".json")))
    except Exception:
        return None


def sha(a) -> str:
    import hashlib

    if isinstance(a, (bytes, bytearray)):
        return hashlib.sha256(a).hexdigest()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--rows", type=int, default=0, help="override individuals per rank")
    ap.add_argument("--batch-pairs", type=int, default=0)
    ap.add_argument("--shard", default="rows", choices=["rows", "features"],
                    help="N > 1: shard individuals (weak scaling) or feature blocks (strong scaling, C5's second mode)")
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
        pw = []
        for r in self.rows:
            try:
                pw.append(float(r[2]))
            except (IndexError, ValueError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w": statistics.median(pw) if pw else None}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ roofline model
def algorithmic_counts(R: int, f: int, cols: int, n: int, L=(6, 4)):
    """algorithmic HBM bytes and modular multiplies per
    inference of the fast algorithm (one HBM pass per HE op, u32 residues,
    the reference's pass structure; weights, keys and packed output amortised
    over the batch)."""
    P = 4 * n
    k = (f + n - 1) // n
    S = n.bit_length() - 1
    Cb = [2 * Lb * P for Lb in L]
    per = sum(k * Cb[i] + cols * (2 * S + 2) * Cb[i] + cols * L[i] * P for i in range(2))
    shared = sum(cols * k * L[i] * P + S * 2 * L[i] ** 2 * P + ((R * cols + n - 1) // n) * Cb[i] for i in range(2))
    bytes_inf = per + shared / R
    M = cols * S * sum(Lb ** 2 for Lb in L) * n * (S / 2 + 2) + cols * (k + 1) * sum(2 * Lb * n for Lb in L)
    return bytes_inf, M


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "MEASURED_PEAKS.json"
    except Exception:
        return {"hbm_gbs": 7672.0}, "B200_PROFILING.md fallback"


# ------------------------------------------------------------------ reference
def _ref_session(cfg: str, rows: int | None = None):
    from oracle.oracle import Reference, production_params
    from paper_2204_05496_b200.workload import config_workload

    R, f, cols, n, pf, ws = _configs()[cfg]
    r = rows or R
    x, w, b = config_workload(cfg, rows=r)
    ref = Reference(production_params(n), key_seed=1, enc_seed=2)
    return ref, x, w, b, r, f, cols, n


def reference_sample(cfg_name: str, rows: int | None = None, threads: int = 0):
    """The reference CPU path (oracle/_ref = the unmodified reference compiled
    in place) on `rows` individuals of the workload, all host threads.
    Returns (inferences/s, sample description, threads, seconds, session)."""
    from oracle.oracle import ref_available

    if not ref_available():
        return None
    ref, x, w, b, r, f, cols, n = _ref_session(cfg_name, rows)
    nthreads = threads or os.cpu_count() or 1
    ref.encode_inputs(x)
    ref.set_weights(w)
    ref.set_bias(b)
    _, _, secs = ref.matmul(r, cols, threads=nthreads, export=False)
    return r / secs, f"{r} individuals x {f} features x {cols} classes (N={n}) per step", nthreads, secs, ref


def reference_latency(threads: int = 0):
    """Reference single-individual latency at C3 (matmul.cpp:239-255: rows are
    the only parallel axis, so R = 1 runs on one thread whatever `threads`)."""
    res = reference_sample("c3", threads=threads)
    if res is None:
        return None
    _, _, nthreads, secs, ref = res
    ref.close()
    return {"value_ms": secs * 1000.0, "cores": 1, "threads_offered": nthreads, "kind": "reference",
            "sample": "c3: 1 individual x 40000 features x 11 classes (N=8192), one full call"}


def reference_standard(prefix: int = 400):
    """Reference baseline_matmul (matmul.cpp:273-344, single-threaded, constant
    cost per feature: 1 encryption + |Y| ct x pt per feature) timed on the
    first `prefix` features of C3 and extrapolated to 40,000."""
    from oracle.oracle import ref_available

    if not ref_available():
        return None
    ref, x, w, b, r, f, cols, n = _ref_session("c3")
    _, _, secs = ref.baseline_matmul(x[:, :prefix], w[:prefix], b, export=False)
    ref.close()
    return {"value_ms": secs / prefix * f * 1000.0, "cores": 1, "kind": "reference",
            "sample": f"c3 baseline_matmul on the first {prefix} of {f} features ({secs:.2f} s), "
                      f"extrapolated linearly (constant per-feature cost, matmul.cpp:301-320)"}


def run_reference(args, world, rank):
    if rank != 0:
        return
    R, f, cols, n, _, _ = _configs()[args.config]
    res = reference_sample(args.config, rows=R)  # the full batch: same config as our arm
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libheiref.so not built (needs /root/reference at build time)"}))
        return
    _, sample, threads, first, ref = res
    times = []
    for s in range(args.warmup + args.steps):
        _, _, secs = ref.matmul(R, cols, threads=threads, export=False)
        if s >= args.warmup:
            times.append(secs)
    v = R * len(times) / sum(times)
    line = {"metric": "encrypted LR inferences/sec at 40k features", "value": v, "unit": "inferences/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config}: {R} individuals x {f} features x {cols} classes, N={n}",
                       "rows_per_step": R, "same_config_as_ours": True},
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


def wire_e2e(srv, ew, b, h_np, R, world, steps, g):
    """Time hei_gpu_matmul_wire on the client's request: the same ciphertexts
    serialised as HECT coeff-form blobs (save_ciphertext, serialize.cpp:63-78),
    and compare the response bytes with the reference server's."""
    from paper_2204_05496_b200 import matmul_wire, save_ciphertexts

    import torch

    raw = save_ciphertexts(srv, h_np)
    pinned = torch.empty(len(raw), dtype=torch.uint8, pin_memory=True)  # as the e2e path's inputs
    blobs = pinned.numpy()
    blobs[:] = np.frombuffer(raw, np.uint8)
    del raw
    outs, _ = matmul_wire(srv, ew, blobs, R, b)  # warm
    t0 = time.perf_counter()
    for _ in range(steps):
        outs, _ = matmul_wire(srv, ew, blobs, R, b)
    sec = (time.perf_counter() - t0) / steps
    resp = b"".join(outs)
    res = {"value": world * R / sec, "unit": "inferences/s", "h2d_bytes_per_step": int(blobs.nbytes),
           "d2h_bytes_per_step": len(resp), "ms_per_step": 1000 * sec,
           "format": "HECT coeff-form blobs [row][chunk][branch] in, HECT blobs out (server.cpp:112-172)"}
    if g and "wire_request_sha256" in g:
        res["request_equals_reference_client"] = sha(blobs) == g["wire_request_sha256"]
        res["response_equals_reference_server"] = sha(resp) == g["wire_response_sha256"]
    return res


def standard_algorithm(srv, bfly_peak):
    """The standard algorithm (baseline_matmul, matmul.cpp:273-344) at C3:
    40,000 column encryptions from the reference's Prng stream, summed over
    features for 11 classes. Checked against the reference's bytes
    (tests/golden/configs/base_c3.json) and decrypted."""
    from paper_2204_05496_b200 import Prng, baseline_matmul
    from paper_2204_05496_b200.workload import config_workload

    R3, f3, c3, n3, _, _ = _configs()["c3"]
    x3, w3, b3 = config_workload("c3")
    baseline_matmul(srv, x3, w3, b3, Prng(2), Prng(3))  # warm (incl. the cached jump polynomial)
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        blocks, bc = baseline_matmul(srv, x3, w3, b3, Prng(2), Prng(3))
        times.append(time.perf_counter() - t0)
    ms = 1000 * statistics.median(times)
    g = golden("base_c3")
    dec = srv.unpack_baseline(blocks, R3, c3)
    # the reference algorithm's own work: per feature one twin
    # encryption (3 sum(L) NTTs + 2 sum(L) N products) and |Y| ct x pt
    # products over 2 sum(L) N residues, at the measured butterfly peak
    L = (6, 4)
    S = n3.bit_length() - 1
    per_feat = 3 * sum(L) * (n3 // 2) * S + 2 * sum(L) * n3 + c3 * 2 * sum(L) * n3
    floor_ms = per_feat * f3 / bfly_peak * 1000.0
    return {"algorithm": "standard (sample-batched, baseline_matmul)", "config": f"c3: {R3}x{f3}x{c3} N={n3}",
            "ms": ms, "mul_plain": int(bc.mul_plain_count), "note": "host call incl. H2D of x, w and D2H of the blocks",
            "bit_exact_vs_reference": bool(g is not None and sha(blocks) == g["blocks_sha256"]),
            "decrypted_equals_integer_product": bool(np.array_equal(dec, x3 @ w3 + b3)),
            "reference_algorithm_int_floor_ms": floor_ms,
            "reference_algorithm_int_floor_note": "the reference's per-feature transform + product count at the "
                                                  "measured butterfly peak; the device computes the same residues by "
                                                  "linearity (coefficient-domain sums, DESIGN.md §4), so it can run "
                                                  "below this floor"}


def run_ours(args, world, rank, local):
    import torch

    from paper_2204_05496_b200 import encode_weights, matmul, matmul_device, native
    from paper_2204_05496_b200.workload import workload

    R_total, f, cols, n, pf, ws = _configs()[args.config]
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
    # seeded workload from util::Prng(7): one X of world*R rows
    # (rank r holds rows [rR, (r+1)R)), then the shared model W, bias
    feat = args.shard == "features" and world > 1
    rows_all = R if feat else world * R
    x, w, b = workload(rows_all, f, cols, pf, ws, row_lo=0 if feat else rank * R, row_hi=R if feat else (rank + 1) * R)
    ew = encode_weights(srv, w)
    # device-resident inputs: the client's real encryptions of x
    # (encode_inputs, matmul.cpp:59-81; Prng seeds 2, 3 as client_backend(keys, 2))
    d_in = torch.empty((R * kc, ctw), dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    seed_r = 0 if feat else rank  # feature sharding: every rank encrypts the same rows, then keeps its block
    for _ in range(2):  # first call also builds the cached mt19937_64 jump polynomial
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        encode_inputs_device(srv, x, Prng(2 + 2 * seed_r), Prng(3 + 2 * seed_r), d_in.data_ptr(), stream.cuda_stream)
        enc_ms = (time.perf_counter() - t0) * 1000.0
    C_ = (R * cols + n - 1) // n
    d_out = torch.empty((C_, ctw), dtype=torch.int32, device=dev)
    d_one = torch.empty((C_, ctw), dtype=torch.int32, device=dev)  # rank-local result (roofline step)
    exchange = None

    if world == 1:
        def step():
            matmul_device(srv, d_in.data_ptr(), R, ew, b, d_out.data_ptr(), stream.cuda_stream)
    elif args.shard == "rows":
        # individual sharding: rank r holds rows [r*R, (r+1)*R) of a world*R
        # batch. Each rank's packed partial is reduced mod q to u32 and the
        # partials are all-gathered with NCCL on the compute stream; rank 0
        # sums them mod q and adds the bias (no host barrier in the step).
        from paper_2204_05496_b200.sharding import (exchange_partials, finish_parts_device, matmul_partial_device,
                                                    packed_count, reduce_packed_device)

        total_rows = world * R
        Ct = packed_count(total_rows, cols, n)
        d_out = torch.empty((Ct, ctw), dtype=torch.int32, device=dev)
        exchange = "nccl all-gather of u32 partials" if os.environ.get("HEI_DIST_BACKEND", "nccl") == "nccl" else "gloo"
        acc = torch.zeros((Ct, ctw), dtype=torch.int64, device=dev)
        part = torch.empty((Ct, ctw), dtype=torch.int32, device=dev)

        def step():
            with torch.cuda.stream(stream):
                acc.zero_()
            matmul_partial_device(srv, ew, d_in.data_ptr(), R, rank * R, total_rows, acc.data_ptr(), stream.cuda_stream)
            reduce_packed_device(srv, acc.data_ptr(), Ct, part.data_ptr(), stream.cuda_stream)
            with torch.cuda.stream(stream):
                gathered = exchange_partials(part)
            if rank == 0:
                finish_parts_device(srv, ew, gathered.data_ptr(), world, b, total_rows, d_out.data_ptr(),
                                    stream.cuda_stream)
    else:
        # feature-block sharding (C5's second mode): every rank
        # holds chunk block shard_chunks(kc) of all rows_all rows; per row
        # batch the chunk-product partials are reduce-scattered by rows (exact
        # integer sums), each rank folds and masks its row block, and the
        # packed partials are exchanged as in row sharding. Strong scaling
        # over a fixed batch of R rows.
        from paper_2204_05496_b200.sharding import (chunk_dot_partial_device, exchange_partials, finish_parts_device,
                                                    fold_pack_device, packed_count, reduce_packed_device,
                                                    reduce_scatter_dots, shard_chunks, shard_rows)

        klo, kn = shard_chunks(kc, world, rank)
        if kn == 0:
            raise SystemExit(f"--shard features needs world <= chunks per row ({kc})")
        total_rows = R
        torch.cuda.synchronize()
        d_in = d_in.view(R, kc, ctw)[:, klo:klo + kn].contiguous().view(R * kn, ctw)  # this rank's feature block only
        Ct = packed_count(total_rows, cols, n)
        d_out = torch.empty((Ct, ctw), dtype=torch.int32, device=dev)
        exchange = ("nccl reduce-scatter of chunk-product partials + all-gather of u32 packed partials"
                    if os.environ.get("HEI_DIST_BACKEND", "nccl") == "nccl" else "gloo")
        acc = torch.zeros((Ct, ctw), dtype=torch.int64, device=dev)
        part = torch.empty((Ct, ctw), dtype=torch.int32, device=dev)
        RB = max(world, min(R, 4 * world))  # rows per exchange batch (bounds the u64 dot buffer)
        dot = torch.empty((RB * cols, ctw), dtype=torch.int64, device=dev)

        def step():
            with torch.cuda.stream(stream):
                acc.zero_()
            for r0 in range(0, R, RB):
                nr = min(RB, R - r0)
                with torch.cuda.stream(stream):
                    dot[: nr * cols].zero_()
                chunk_dot_partial_device(srv, ew, d_in[r0 * kn:(r0 + nr) * kn].data_ptr(), nr, klo, kn, dot.data_ptr(),
                                         stream.cuda_stream)
                with torch.cuda.stream(stream):
                    mine = reduce_scatter_dots(dot[: nr * cols], nr)
                lo, cnt = shard_rows(nr, world, rank)
                if cnt:
                    fold_pack_device(srv, ew, mine.data_ptr(), r0 + lo, cnt, total_rows, acc.data_ptr(),
                                     stream.cuda_stream)
            reduce_packed_device(srv, acc.data_ptr(), Ct, part.data_ptr(), stream.cuda_stream)
            with torch.cuda.stream(stream):
                gathered = exchange_partials(part)
            if rank == 0:
                finish_parts_device(srv, ew, gathered.data_ptr(), world, b, total_rows, d_out.data_ptr(),
                                    stream.cuda_stream)

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
    value = rows_all / (ms / 1000.0)

    # bit-exactness of the timed path against the reference (single rank:
    # the golden digests cover exactly this workload, keys and encryption)
    g = None
    if world == 1 and rank == 0:
        g = golden("stream_c5") if args.config == "c5" else golden(f"fast_{args.config}")
        if g is not None and g.get("rows") != R:
            g = None
    packed_dev = d_out.cpu().numpy().view(np.uint32).astype(np.uint64) if rank == 0 else None
    parity = None
    if g is not None:
        parity = {"golden": os.path.relpath(os.path.join(GOLDEN, g["case"] + ".json"), ROOT),
                  "device_packed_equals_reference": sha(packed_dev) == g["packed_sha256"]}

    # e2e: host u64 (pinned) inputs through the C ABI, copies inside the timed region
    e2e = None
    if not args.no_e2e and not feat:
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
        if parity is not None:
            if "inputs_sha256" in g:  # (the streamed C5 golden has no input digest: 32 GB of ciphertexts)
                parity["inputs_equal_reference_client"] = sha(h_np) == g["inputs_sha256"]
            parity["e2e_packed_equals_reference"] = sha(out) == g["packed_sha256"]
        # the server's wire path (server.cpp:112-172): HECT coeff-form blobs
        # in, HECT blobs out, parse/NTT/INTT/serialize on the device
        if args.wire and world == 1:  # the wire copy doubles pinned host memory; one rank only
            e2e["wire"] = wire_e2e(srv, ew, b, h_np, R, world, e2e_steps, g)
            if parity is not None and "response_equals_reference_server" in e2e["wire"]:
                parity["wire_response_equals_reference"] = e2e["wire"]["response_equals_reference_server"]
        del h_in, h_np

    # ---- rooflines, timed live with CUDA events on the launch stream inside
    # the C ABI over one extra (serialised) step
    roof = int_roof = step_roof = None
    peaks, peak_src = _peaks()
    hbm = float(peaks.get("hbm_gbs", 7672.0))
    bfly_peak = native.butterfly_peak(local) if rank == 0 else None
    if feat:
        d_in = None  # the sliced block is not a full-row input for the single-GPU legs below
    L0, L1 = len(q0), len(q1)
    if rank == 0 and not feat:
        native.kernel_timing(srv.handle, True)
        # the rank's own fold work only: no collective, so rank 0 can time it alone
        matmul_device(srv, d_in.data_ptr(), R, ew, b, d_one.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        ks_n, ks_ms = native.kernel_stats(srv.handle, 0)
        dg_n, dg_ms = native.kernel_stats(srv.handle, 1)
        native.kernel_timing(srv.handle, False)
        S = int(np.log2(n))  # fold steps per batch
        batches = ks_n // S
        pairs_per_launch = R * cols / batches
        # per pair-rotation the twin ciphertext is read and
        # written once (2 sum_b C_b, C_b = 2 L_b 4N bytes); the step's Galois
        # key (2 L_b^2 polys of value + Shoup u32 per branch) once per launch
        pair_bytes = 2 * sum(2 * Lb * 4 * n for Lb in (L0, L1))
        key_bytes = sum(2 * Lb * Lb * 4 * n * 2 for Lb in (L0, L1))
        launch_bytes = pairs_per_launch * pair_bytes + key_bytes
        avg_s = ks_ms / ks_n / 1000.0
        traffic = None
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "keyswitch_traffic.json")))
            traffic = prof.get("dram_bytes_per_pair") * pairs_per_launch
        except Exception:
            pass
        logn = n.bit_length() - 1
        blocks = pairs_per_launch * (L0 + L1)  # (pair, prime) blocks per timed key-switch launch
        if blocks <= 148:
            ks_name = f"k_rot_keyswitch_w2<{logn}> (latency path)"
        elif logn == 14:
            ks_name = "k_rot_keyswitch_h (half-ring blocks, TMEM accumulators)"
        elif blocks < 296:
            ks_name = f"k_rot_keyswitch_s<{logn}> (shared-memory accumulators)"
        else:
            ks_name = "k_rot_keyswitch_t<13> (TMEM accumulators, 3 CTAs/SM)"
        ach = launch_bytes / avg_s / 1e9
        roof = {"kernel": ks_name, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": traffic, "binding": "int32 pipes (see int_roofline)",
                "algorithmic_bytes_per_launch": launch_bytes, "bytes_model": "SURVEY 8(d): pairs x 2 sum_b C_b + key",
                "avg_launch_ms": avg_s * 1e3, "launches": ks_n, "pairs_per_launch": pairs_per_launch,
                "peak_source": peak_src, "share_of_fold": ks_ms / (ks_ms + dg_ms),
                "digits_avg_launch_ms": dg_ms / max(1, dg_n)}
        bfly_pair = sum(((Lb - 1) * (n // 2) * S + 2 * Lb * n) for Lb in (L0, L1) for _ in range(Lb))
        tot_bfly = pairs_per_launch * bfly_pair
        int_roof = {"kernel": ks_name, "bound": "int32 pipes (CT butterfly = Shoup mulmod + add + sub)",
                    "achieved": tot_bfly / avg_s / 1e9, "peak": bfly_peak / 1e9, "unit": "Gbutterfly/s",
                    "frac": tot_bfly / avg_s / bfly_peak, "binding": True,
                    "peak_source": "k_bfly_peak register microbenchmark, this run",
                    "butterfly_equivalents_per_launch": tot_bfly}
        bi, M = algorithmic_counts(R, f, cols, n, (L0, L1))
        t_int = R * M / bfly_peak
        t_hbm = R * bi / (hbm * 1e9)
        step_roof = {"model": "SURVEY 8(d) per inference: bytes and modular multiplies of the fast algorithm",
                     "bytes_per_inference": bi, "modmul_per_inference": M,
                     "hbm_frac": t_hbm / (ms / 1000.0), "int_frac": t_int / (ms / 1000.0),
                     "binding": "int" if t_int > t_hbm else "hbm",
                     "roofline_inferences_per_s": world * R / max(t_int, t_hbm)}

    base = None
    if args.baseline and rank == 0:
        base = standard_algorithm(srv, bfly_peak)
        base["client_encrypt"] = {"config": f"{R} individuals x {f} features ({R * kc} twin encryptions)",
                                  "ms": enc_ms, "individuals_per_s": R / (enc_ms / 1000.0)}

    lat = None
    if args.latency and rank == 0:
        # single individual, C3 (40,000 features x 11 classes): its own seeded
        # workload, encrypted with Prng(2)/(3), device-resident; the output is
        # compared with the reference's (tests/golden/configs/fast_c3.json)
        from paper_2204_05496_b200.workload import config_workload

        x3, w3, b3 = config_workload("c3")
        ew3 = encode_weights(srv, w3)
        kc3 = (x3.shape[1] + n - 1) // n  # the C3 row's chunks (not this config's)
        d1 = torch.empty((kc3, ctw), dtype=torch.int32, device=dev)
        encode_inputs_device(srv, x3, Prng(2), Prng(3), d1.data_ptr(), stream.cuda_stream)
        o1 = torch.empty((1, ctw), dtype=torch.int32, device=dev)
        for _ in range(3):
            matmul_device(srv, d1.data_ptr(), 1, ew3, b3, o1.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(20):
            matmul_device(srv, d1.data_ptr(), 1, ew3, b3, o1.data_ptr(), stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        lat_ms = e0.elapsed_time(e1) / 20
        g3 = golden("fast_c3")
        bi3, M3 = algorithmic_counts(1, 40000, 11, n, (L0, L1))
        lat = {"ms": lat_ms, "config": "c3: 1 individual x 40000 features x 11 classes, device-resident",
               "bit_exact_vs_reference": bool(g3 is not None and n == 8192 and
                                              sha(o1.cpu().numpy().view(np.uint32).astype(np.uint64)) == g3["packed_sha256"]),
               "roofline": {"int_frac": M3 / bfly_peak * 1000.0 / lat_ms, "hbm_frac": bi3 / (hbm * 1e9) * 1000.0 / lat_ms,
                            "model": "SURVEY 8(d) per-inference bytes and modmuls at R = 1"}}
        del d1, ew3

    # client side of the result: decrypt + CRT unpack on the device
    # (unpack_results, matmul.cpp:257-271), checked against the exact product
    check = None
    if rank == 0:
        # world > 1: d_out is the reduced result of every rank's rows
        srv.unpack_results(packed_dev, rows_all, cols)  # warm
        t0 = time.perf_counter()
        got = srv.unpack_results(packed_dev, rows_all, cols)
        dec_ms = (time.perf_counter() - t0) * 1000.0
        x_all = x if (world == 1 or feat) else workload(rows_all, f, cols, pf, ws)[0]
        want = np.rint(x_all.astype(np.float64) @ w.astype(np.float64)).astype(np.int64) + b  # exact: |sums| < 2^53
        check = {"decrypted_equals_integer_product": bool(np.array_equal(got, want)), "client_decrypt_ms": dec_ms,
                 "keygen_ms": keygen_ms, "client_encrypt_ms": enc_ms}

    if rank != 0:
        return
    cpu = cpu_lat = cpu_std = None
    if not args.no_cpu_baseline and world == 1:
        try:
            res = reference_sample(args.config, rows=min(R, 32))
            if res:
                rate, sample, threads, secs, ref = res
                ref.close()
                cpu = {"value": rate, "unit": "inferences/s", "cores": threads, "kind": "reference", "sample": sample,
                       "seconds": secs}
            if args.latency:
                cpu_lat = reference_latency()
            if args.baseline:
                cpu_std = reference_standard()
        except Exception as e:  # report, never fail the bench on the CPU leg
            cpu = {"error": str(e)}
    line = {
        "metric": "encrypted LR inferences/sec at 40k features",
        "value": value, "unit": "inferences/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if feat else "weak",
        "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {R} individuals/rank x {f} features x {cols} classes, N={n}, "
                               f"twin t=({T0},{T1 if n < 16384 else T1_16K}), L=({len(q0)},{len(q1)})",
                   "inputs": "seeded util::Prng(7) workload (SURVEY 8d), real encryptions (device keygen from "
                             "Prng(1), client encryption with Prng(2),(3)), resident in HBM; inputs > L2 (no flush "
                             "needed)",
                   "parallelism": f"dp{world} ({'feature-block' if feat else 'individual'} sharding)" + (
                       f", exchange={exchange}" if world > 1 else "")},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cpu,
        "bit_exact_vs_reference": None if parity is None else all(v for k, v in parity.items() if k != "golden"),
        "parity": parity,
    }
    line["roofline"] = roof
    line["int_roofline"] = int_roof
    line["step_roofline"] = step_roof
    if lat is not None:
        line["latency_single_individual"] = lat
        line["latency_ms_single_individual"] = lat["ms"]
        if cpu_lat is not None:
            lat["cpu_baseline"] = cpu_lat
    if base is not None:
        line["standard_algorithm"] = base
        if cpu_std is not None:
            base["cpu_baseline"] = cpu_std
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

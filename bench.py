#!/usr/bin/env python
"""bench.py -- decode-step retrieve+attend latency and frame-ingest rate (BASELINE.json metric).

Workload (config 2): LLaVA-OneVision-7B-shaped KV -- 28 layers x 4 KV heads =
112 clustering domains, d = 128, bf16, a 128K-token stream (669 frames x 196 tokens = 131,124
tokens per domain) held as 256 clusters per domain, top-16 cluster retrieval (k_v = 1) plus the
4-frame local window. Synthetic data generated on the GPU (paper_2604_10060_b200/workload.py);
the pre-clustered state is installed through the bulk add_cluster path, then `--frames` new
frames are ingested online (timed: frames/s) and `--steps` decode steps are timed.

One JSON line on rank 0. `value` = decode µs/step (lower is better) measured with CUDA events on
the context stream, inputs resident in HBM; `e2e` = the same through the public API with host
query / host output (H2D + D2H inside the timed region). Per-step working set (~530 MB of
selected K/V) exceeds the 126 MB L2 and every step uses a different query (different clusters),
so no L2 flush is needed ("inputs larger than L2").

--gpus N (torchrun): the 112 domains are sharded across ranks by (layer, KV head); each step ends
with an NCCL all-gather of the per-domain outputs; time = max over ranks (strong scaling).
--impl reference: the reference's own CPU path (oracle/_ref, compiled from the unmodified
reference sources) on the host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import gc
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

METRIC = "decode-step retrieve+attend µs @128K-token KV; frame ingest frames/s"
D_TOTAL, HEAD_DIM, N_TOK, N_CLUST, T_FRAME, TOP_K, WINDOW = 112, 128, 669 * 196, 256, 196, 16, 4
CPU_DOMS = 8  # domains of host input kept for the CPU baselines (replicated across threads)


RESOLVE_KERNEL = "seq" if os.environ.get("KVC_RESOLVE") == "seq" else "spec"
RESOLVE_PHASES = {  # clock64 phases of the resolve kernel (kvc_debug_resolve_profile), domain mean
    "seq": ["argmax", "hot", "update", "build", "chain", "decide", "commit", "keyring"],
    "spec": ["setup", "slot_table", "rep_chains", "exact_sums", "bound_max", "var_chain", "decisions",
             "buffers", "verify", "commit", "rounds", "setup_keys", "setup_topm"],
}

def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--frames", type=int, default=0, help="timed ingest frames (default = steps)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-offload", action="store_true", help="skip the config-3 host-tier measurement")
    p.add_argument("--no-streams", action="store_true", help="skip the config-5 streams + token-ablation measurement")
    p.add_argument("--no-config4", action="store_true", help="skip the config-4 (Qwen2-VL-72B head shard) measurement")
    p.add_argument("--exchange", default="fused", choices=["fused", "nccl"], help="multi-GPU output exchange")
    p.add_argument("--domains", type=int, default=D_TOTAL)
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.sampler = "nvidia-smi"
        self._stop = threading.Event()
        self._t = None

    def _nvml_row(self, h):
        """The same fields as the nvidia-smi query, in process through NVML (no fork/exec of
        nvidia-smi inside the timed region)."""
        import pynvml as N

        sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        pw = N.nvmlDeviceGetPowerUsage(h) / 1000.0
        r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
        act = lambda bit: "Active" if r & bit else "Not Active"
        return [str(self.index), str(sm), str(mx), f"{pw:.1f}", hex(r), act(N.nvmlClocksEventReasonHwSlowdown),
                act(N.nvmlClocksEventReasonHwThermalSlowdown), act(N.nvmlClocksEventReasonSwThermalSlowdown),
                act(N.nvmlClocksEventReasonSwPowerCap)]

    def _run(self):
        h = None
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.sampler = "nvml (in process; nvidia-smi's fields)"
        except Exception:
            h = None
        while not self._stop.is_set():
            try:
                if h is not None:
                    self.rows.append(self._nvml_row(h))
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        # Python's cyclic garbage collector is paused inside timed regions (as timeit does): a
        # collection pause of the harness would otherwise land on a random step
        self._gc = gc.isenabled()
        gc.disable()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)
        if self._gc:
            gc.enable()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "sampler": self.sampler}


def traffic_from_profiles():
    """dram bytes per attention launch from the committed `ncu --set full` capture
    (profiles/ncu_attend_summary.json, written by scripts/summarize_profiles.py) and where it came
    from: the profile round, the commit it was captured at, the command. ncu cannot run inside the
    timed bench, so the number is stamped rather than silently reused."""
    path = os.path.join(ROOT, "profiles", "ncu_attend_summary.json")
    try:
        with open(path) as f:
            j = json.load(f)
        return j.get("dram_bytes_per_launch"), {k: j.get(k) for k in ("round", "head", "captured", "command", "source")}
    except Exception:
        return None, None


# --------------------------------------------------------------------------- reference arm

def run_reference(args, rank: int):
    if rank != 0:
        return
    from oracle import pyoracle as po

    if po.reference() is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libkvclust_ref.so not built"}))
        return
    threads = os.cpu_count() or 1
    dom, scale = _ref_plan(threads)
    st = _host_sample(dom)
    q = _host_queries(st, args.warmup + args.steps)
    us, mean = po.time_reference(0, threads, st["keys"], st["values"], st["assign"], N_CLUST,
                                 args.warmup, args.steps, TOP_K, WINDOW * T_FRAME, queries=q)
    per_step = us * scale
    sample = (f"{threads} concurrent reference instances x {dom} domains = {threads * dom} domain-steps per step "
              f"(x{scale:.3f} to the 112 domains; N={N_TOK}, C={N_CLUST}, top-{TOP_K} + {WINDOW}-frame window): "
              f"retrieve() + fp64 attention over the attended set, wall us/step (max over instances)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(per_step, 3), "unit": "us/step",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step / 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(args, 1),
        "cpu_baseline": {"value": round(per_step, 3), "unit": "us/step", "cores": threads,
                         "kind": "reference", "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": round(per_step, 3), "unit": "us/step", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    # the ingest half of the metric: place_frame + on_insert on drift-regime frames (the same
    # generator and regime as our arm's headline ingest number)
    try:
        from paper_2604_10060_b200 import workload

        nfr = max(2, min(args.steps, 10))
        fk, fv, fvis, _ = workload.frames_drift(st["state"], nfr + 1, N_TOK // T_FRAME + 1, seed=7)
        us_i, _ = po.time_reference(1, threads, st["keys"], st["values"], st["assign"], N_CLUST, 1, nfr, TOP_K,
                                    WINDOW * T_FRAME, fvis=fvis, fkeys=fk.float().cpu().numpy(),
                                    fvals=fv.float().cpu().numpy())
        line["ingest"] = {"value": round(1e6 / (us_i * scale), 2), "unit": "frames/s",
                          "us_per_frame": round(us_i * scale, 1),
                          "sample": f"{threads} instances x {dom} domains, {nfr} timed drift-regime frames"}
    except Exception as e:
        line["ingest"] = {"value": None, "error": f"{type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)


def _host_sample(dom: int, seed: int = 42):
    """A bounded host copy of the workload: `dom` domains of the config-2 state (f32)."""
    import torch
    from paper_2604_10060_b200 import workload

    dev = "cuda" if torch.cuda.is_available() else "cpu"
    st = workload.clustered_state(dom, N_TOK, N_CLUST, HEAD_DIM, T_FRAME, seed=seed, device=dev)
    return {"keys": st.keys.float().cpu().numpy(), "values": st.values.float().cpu().numpy(),
            "assign": st.assign, "state": st}


def _host_queries(h, n):
    from paper_2604_10060_b200 import workload

    return workload.queries_near(h["state"], n).cpu().numpy()


def _config(args, world):
    return {"workload": "config2: LLaVA-OV-7B KV (28 layers x 4 KV heads = 112 domains), d=128, bf16, "
                        "131,124-token stream/domain, 256 clusters/domain, top-16 + 4-frame window",
            "domains": D_TOTAL, "tokens_per_domain": N_TOK, "clusters_per_domain": N_CLUST,
            "top_k": TOP_K, "window_frames": WINDOW, "head_dim": HEAD_DIM, "kv_dtype": "bf16",
            "parallelism": f"domain-shard{world}" if world > 1 else "single",
            "l2": "per-step working set > L2 (no flush)"}


def self_launch(args) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1 and return rank 0's exit code. Fails loudly when fewer than
    N GPUs are visible (KVC_BENCH_ONE_GPU=1: every rank on cuda:0, development only)."""
    import socket

    import torch

    n_vis = torch.cuda.device_count()
    if n_vis < args.gpus and os.environ.get("KVC_BENCH_ONE_GPU") != "1":
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {n_vis}", file=sys.stderr)
        return 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# --------------------------------------------------------------------------- our arm

def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)  # rank 0 alone (host cores); other ranks exit without work
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines on stderr (rank / device evidence)

    import torch
    import torch.distributed as dist

    from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload

    # KVC_BENCH_ONE_GPU=1 (development only): every rank on cuda:0 with gloo, to exercise the
    # multi-rank path (sharding, fused exchange through CUDA IPC) on a single-GPU box
    one_gpu = os.environ.get("KVC_BENCH_ONE_GPU") == "1"
    torch.cuda.set_device(0 if one_gpu else local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2604_10060_b200.sharding import FusedExchange, gather_domain_outputs, shard_domains

    d0, d1 = shard_domains(args.domains, world, rank)  # strong scaling over (layer, head) domains
    D = d1 - d0
    frames_t = args.frames or args.steps

    cfg = Config.make(kv_dtype=DTYPE_BF16, k_v=1, k_s=TOP_K, window_frames=WINDOW, build_batch_frames=1,
                      offload_horizon_frames=1 << 30, device_capacity_entries=1 << 40,
                      pool_bytes=int(1.25 * D * (N_TOK + 64 * N_CLUST + 400 * T_FRAME) * HEAD_DIM * 4),
                      max_slots=max(4096, 4 * D * N_CLUST), max_cluster_pages=512, max_tokens=T_FRAME)
    kv = ClusterKVCache(cfg, HEAD_DIM, D)
    st = workload.clustered_state(D, N_TOK, N_CLUST, HEAD_DIM, T_FRAME, seed=42 + rank)
    t0 = time.time()
    kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, N_CLUST)
    load_s = time.time() - t0
    nd_cpu = min(CPU_DOMS, D)
    host_state = None
    if world == 1 and not args.no_cpu_baseline:  # the CPU baselines' input: the first domains, f32
        host_state = {"keys": st.keys[:nd_cpu].float().cpu().numpy(), "values": st.values[:nd_cpu].float().cpu().numpy(),
                      "assign": np.ascontiguousarray(st.assign[:nd_cpu]), "visual": st.visual}
    del st.keys, st.values
    torch.cuda.empty_cache()
    stream = torch.cuda.ExternalStream(kv.stream)

    # ------------------------------------------------------------------ ingest (frames/s)
    # two regimes, timed the same way: the reference stream's dynamics (gen_stream: noise 0.02,
    # center drift 0.01/frame -> the Eq. 5 threshold is crossed, clusters split) -- the headline
    # ingest number -- and an absorb-only regime (frames near existing centres, noise 0.015).
    first = N_TOK // T_FRAME + 1
    absorb = ingest_regime(kv, stream, args, world, local, frames_t,
                           lambda n, f0, seed: workload.frames_near(st, n, f0, seed=seed), first, "absorb")
    absorb.pop("_clocks")
    absorb_ms, absorb_e2e_ms = absorb.pop("_ms"), absorb.pop("_e2e_ms")
    absorb.pop("_frames_f32")

    # ------------------------------------------------------------------ decode (us/step)
    nq = args.warmup + args.steps
    q_dev = workload.queries_near(st, nq, seed=11 + rank)
    out_dev = torch.zeros(D, HEAD_DIM, device="cuda")
    # multi-GPU output exchange: fused into the attention kernel (peer-memory row stores through
    # CUDA IPC mappings + a per-step signal/wait), or NCCL all-gather (--exchange nccl / fallback)
    exchange = "none"
    ex = None
    full_out = torch.zeros(args.domains, HEAD_DIM, device="cuda")
    if world > 1:
        exchange = "nccl"
        if args.exchange == "fused":
            try:
                ex = FusedExchange(kv, args.domains)
                exchange = "fused"
            except Exception as e:  # e.g. no peer access: the collective still works
                print(f"fused exchange unavailable ({e}); using NCCL all-gather", file=sys.stderr)

    def exchange_step():
        if ex is not None:
            ex.gathered(full_out)
        elif world > 1:
            gather_domain_outputs(out_dev, args.domains)
    for i in range(args.warmup):
        kv.query(i, q_dev[i], out=out_dev)
        exchange_step()
    launches0 = kv.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # timed region: no per-kernel instrumentation (events / phase clocks are a separate pass below)
    with Clocks(local) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            h0 = time.perf_counter()
            step_ev = []
            for i in range(args.warmup, nq):
                kv.query(i, q_dev[i], out=out_dev)
                exchange_step()  # per-domain outputs to every rank
                e = torch.cuda.Event(enable_timing=True)  # step boundary (after K6, before the next K4)
                e.record(stream)
                step_ev.append(e)
            host_issue_us = (time.perf_counter() - h0) * 1e6 / args.steps
            ev1.record(stream)
        torch.cuda.synchronize()
    decode_ms = ev0.elapsed_time(ev1)
    periods = [step_ev[i].elapsed_time(step_ev[i + 1]) * 1e3 for i in range(len(step_ev) - 1)]
    decode_launches = kv.launch_count() - launches0
    # instrumented pass over the same queries: per-kernel CUDA events on the context stream
    # (K4 and K6 durations, attended bytes per K6 launch) and host phases
    kv.set_timing(True)
    att_us, k4_us, att_bytes_l, host_ph, span_us = [], [], [], [], []
    with torch.cuda.stream(stream):
        for i in range(args.warmup, nq):
            kv.query(i, q_dev[i], out=out_dev)
            tm = kv.step_timing()
            k4_us.append(tm[0])
            span_us.append(tm[3])
            att_us.append(tm[1])
            att_bytes_l.append(tm[4])
            host_ph.append(tm[5:9].copy())
    torch.cuda.synchronize()
    k4_cycles = kv.resolve_profile(decode=True)
    kv.set_timing(False)
    # e2e decode: host query in, host output out, through the public API
    q_pin = q_dev.cpu().pin_memory()  # pinned host buffers: the contract's e2e copies
    out_pin = torch.zeros(D, HEAD_DIM, dtype=torch.float32).pin_memory()
    q_host, out_host = q_pin.numpy(), out_pin.numpy()
    torch.cuda.synchronize()
    e0.record(stream)
    h0 = time.perf_counter()
    for i in range(args.warmup, nq):
        kv.query(i, q_host[i], out=out_host)
    e2e_host_us = (time.perf_counter() - h0) * 1e6 / args.steps
    e1.record(stream)
    torch.cuda.synchronize()
    decode_e2e_ms = e0.elapsed_time(e1)

    # the drift regime last (its splits grow the index past config 2's 256 clusters per domain, so
    # the decode measurement above runs on the config-2 state)
    drift = ingest_regime(kv, stream, args, world, local, frames_t,
                          lambda n, f0, seed: workload.frames_drift(st, n, f0, seed=seed), first + 100000, "drift")
    ingest_launches = absorb.pop("_launches") + drift.pop("_launches")
    clk_ingest = drift.pop("_clocks")
    ingest_ms, ingest_e2e_ms = drift.pop("_ms"), drift.pop("_e2e_ms")
    drift_frames_f32 = drift.pop("_frames_f32")

    # max over ranks
    vals = torch.tensor([decode_ms, decode_e2e_ms, ingest_ms, ingest_e2e_ms, absorb_ms, absorb_e2e_ms], device="cuda",
                        dtype=torch.float64)
    if world > 1:
        if one_gpu:
            vc = vals.cpu()
            dist.all_reduce(vc, op=dist.ReduceOp.MAX)
            vals = vc
        else:
            dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    decode_ms, decode_e2e_ms, ingest_ms, ingest_e2e_ms, absorb_ms, absorb_e2e_ms = vals.tolist()
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    us_step = decode_ms * 1e3 / args.steps
    hbm, src = peaks()
    # algorithmic bytes of the attention launch: attended tokens x (K + V) x bf16
    att_bytes = float(np.mean(att_bytes_l))
    att_time = float(np.mean(att_us)) * 1e-6
    achieved = att_bytes / att_time / 1e9
    step_bytes = att_bytes + D * N_CLUST * HEAD_DIM * 8 + D * HEAD_DIM * 8  # + fp64 centroids + q/out
    traffic, traffic_src = traffic_from_profiles()
    line = {
        "metric": METRIC, "value": round(us_step, 3), "unit": "us/step", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": us_step / 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (GPU generator, reference distributions)", "config": _config(args, world),
        "e2e": {"value": round(decode_e2e_ms * 1e3 / args.steps, 3), "unit": "us/step",
                "h2d_bytes_per_step": D * world * HEAD_DIM * 4, "d2h_bytes_per_step": D * world * HEAD_DIM * 4},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "traffic_source": traffic_src,
                     "kernel": "k_attend (split-KV attention over selected clusters + window)",
                     "peak_source": src, "algorithmic_bytes_per_launch": att_bytes,
                     "kernel_us": round(att_time * 1e6, 2),
                     "step_bytes": step_bytes, "step_frac": round(step_bytes / (us_step * 1e-6) / 1e9 / hbm, 4),
                     "score_select_us": round(float(np.mean(k4_us)), 2)},
        "gpu_launches": int(decode_launches),
        "phases_us": {"score_select": round(float(np.mean(k4_us)), 2), "attend": round(att_time * 1e6, 2),
                      "host_issue_per_step": round(host_issue_us, 2),
                      "e2e_host_per_step": round(e2e_host_us, 2),
                      "step_period_us": {"min": round(min(periods), 2) if periods else None,
                                         "median": round(float(np.median(periods)), 2) if periods else None,
                                         "max": round(max(periods), 2) if periods else None},
                      "host_wait_device": round(float(np.mean([h[0] for h in host_ph])), 2),
                      "host_replay": round(float(np.mean([h[1] for h in host_ph])), 2),
                      "host_repin": round(float(np.mean([h[2] for h in host_ph])), 2),
                      "device_span": round(float(np.mean(span_us)), 2),
                      "host_layer_loop": round(float(np.mean([h[3] for h in host_ph])), 2),
                      "k4_cycles": dict(zip(["query_visual", "candidates", "approx", "boundary_exact", "verified", "ring",
                                             "descriptors", "boundary_set", "-", "-", "-", "-", "tail_after_marks",
                                             "block_start_skew_ns", "span_ns", "mean_block_ns"],
                                            k4_cycles.round(0).tolist()))},
        "clocks": clk.summary(),
        "ingest": ingest_line(frames_t, D, world, ingest_ms, ingest_e2e_ms, drift, clk_ingest, ingest_launches,
                              absorb_ms, absorb_e2e_ms, absorb, hbm, src),
        "bulk_load_s": round(load_s, 2),
    }
    if world > 1:
        line["config"]["output_exchange"] = ("fused: K6 stores output rows into every rank's buffer over peer memory, "
                                             "per-step signal/wait" if exchange == "fused" else "NCCL all-gather")
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, host_state, q_dev[:, :nd_cpu].cpu().numpy())
        line["ingest"]["cpu_baseline"] = cpu_baseline_ingest(args, host_state, drift_frames_f32)
    if world == 1 and not args.no_streams:
        try:
            line["streams"] = streams_phase(args)
        except Exception as e:
            line["streams"] = {"error": f"{type(e).__name__}: {e}"}
    if world == 1 and not args.no_config4:
        kv.close()
        torch.cuda.empty_cache()
        try:
            line["config4_shard"] = config4_phase(args)
        except Exception as e:
            line["config4_shard"] = {"error": f"{type(e).__name__}: {e}"}
    if world == 1 and not args.no_offload:
        kv.close()
        del kv, q_dev, out_dev
        torch.cuda.empty_cache()
        try:
            line["offload"] = offload_phase(args)
        except Exception as e:  # the host tier needs pinned host RAM; never lose the main line
            line["offload"] = {"error": f"{type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def ingest_regime(kv, stream, args, world, local, frames_t, gen, first, name):
    """Times `frames_t` frames of one ingest regime (after `args.warmup` untimed ones): CUDA events
    on the context stream around the public ingest call with the frames resident in HBM; then an
    instrumented pass over 3 more frames (per-kernel events, touched clusters) and the e2e pass
    from pinned host frames. gen(n, first_frame, seed) -> (keys, values, visual, frame_ids)."""
    import torch
    import torch.distributed as dist

    nf = args.warmup + frames_t
    fk, fv, fvis, fids = gen(nf, first, 7)
    for i in range(args.warmup):
        kv.process_frame(int(fids[i]), fvis[i], fk[i], fv[i], want_assigned=False)
    s0 = kv.maint_stats()
    kv.wave_profile(reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = kv.launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with Clocks(local) as clk:
        ev0.record(stream)
        h0 = time.perf_counter()
        for i in range(args.warmup, nf):
            kv.process_frame(int(fids[i]), fvis[i], fk[i], fv[i], want_assigned=False)
        host_us = (time.perf_counter() - h0) * 1e6 / frames_t
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches = kv.launch_count() - launches0
    maint = (kv.maint_stats() - s0).tolist()
    waves = kv.wave_profile(reset=True)
    n_clusters = len(kv.cluster_ids())
    # instrumented pass (outside the timed region): kernel phases and touched clusters |U|
    kv.set_timing(True)
    xk, xv, xvis, xids = gen(3, first + nf + 10, 123)
    ph, touched = [], []
    for i in range(3):
        _, asg = kv.process_frame(int(xids[i]), xvis[i], xk[i], xv[i], want_assigned=True)
        ph.append(kv.ingest_timing())
        touched.append(float(np.mean([len(np.unique(asg[l])) for l in range(asg.shape[0])])))
    prof = kv.resolve_profile()
    kv.set_timing(False)
    phases = dict(zip(["cands", "assign", "topm", "resolve", "store_rows", "host_wait", "host_insert_loop",
                       "host_replay", "host_relaunch_issue", "host_events"], np.mean(ph, axis=0).round(2).tolist()))
    phases["host_per_frame_timed_loop"] = round(host_us, 2)
    # e2e: frames from pinned host memory through the public API
    mk, mv, mvis, mids = gen(frames_t, first + nf + 50, 99)
    mk_h = mk.view(torch.int16).cpu().pin_memory().numpy()
    mv_h = mv.view(torch.int16).cpu().pin_memory().numpy()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(frames_t):
        kv.process_frame(int(mids[i]), mvis[i], mk_h[i], mv_h[i], want_assigned=False)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    # CPU-baseline input: the timed frames of the first domains, f32 (bf16 values)
    nd = min(CPU_DOMS, fk.shape[1])
    frames_f32 = (fvis[args.warmup:], fk[args.warmup:, :nd].float().cpu().numpy(),
                  fv[args.warmup:, :nd].float().cpu().numpy())
    return {"_ms": ms, "_e2e_ms": e2e_ms, "_launches": launches, "_clocks": clk, "_frames_f32": frames_f32,
            "phases_us": phases, "maint_delta": dict(zip(MAINT_KEYS, maint)), "wave_engine": waves,
            "resolve_cycles_per_frame": dict(zip(RESOLVE_PHASES[RESOLVE_KERNEL], prof.round(1).tolist())),
            "touched_clusters_per_domain_frame": round(float(np.mean(touched)), 2),
            "clusters_per_domain": round(n_clusters / kv.L, 1)}


MAINT_KEYS = ["inserts", "absorbed", "immediate_splits", "deferred_marks", "settled_splits", "split_ops", "host_over",
              "maint_fetches", "partitions_opened"]


def chain_latencies():
    """Measured fp64 dependency latencies (scripts/fp64_latency.cu on a B200, profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_latency.json")) as f:
            return json.load(f)
    except Exception:
        return None


def ingest_line(frames_t, D, world, ms, e2e_ms, r, clk, launches, a_ms, a_e2e_ms, a, hbm, src):
    """Frame-ingest JSON block: the gen_stream (drift) regime is the headline, absorb-only beside
    it; roofline = SURVEY §8(d) algorithmic bytes per frame (read K/V, write K/V into the store,
    the partition's fp32 centroid mirror, fp64 master r/w of the touched clusters) over the
    measured frame time; chain bound = the per-domain dependent Eq. 3/4 chain (196 inserts); tensor
    pipe = the distance tile's flops (bf16 hi + lo) over its measured kernel time."""
    us = ms * 1e3 / frames_t
    Dall = D * world
    T, d = T_FRAME, HEAD_DIM

    def roof(res, us_frame):
        Cp = res["clusters_per_domain"]
        U = res["touched_clusters_per_domain_frame"]
        b = D * (4 * T * d * 2 + Cp * d * 4 + 2 * U * d * 8)
        ach = b / (us_frame * 1e-6) / 1e9
        flops = D * 2 * 2 * T * Cp * d  # tcgen05 tile: hi and lo halves of the fp64 centroids
        tile_us = res["phases_us"]["assign"]
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 5),
                "algorithmic_bytes_per_frame": int(b), "peak_source": src,
                "tensor_tile": {"kernel": "k_assign_tc", "flops_per_frame": int(flops), "kernel_us": tile_us,
                                "achieved_tflops": round(flops / (tile_us * 1e-6) / 1e12, 2) if tile_us else None,
                                "peak_tflops": tensor_peak()}}

    line = {"value": round(frames_t / (ms * 1e-3), 1), "unit": "frames/s",
            "regime": "gen_stream dynamics (workload.cpp:110-135): keys normalize(center + 0.02 N(0,1)), center drift "
                      "0.01/frame -> clusters cross the Eq. 5 threshold and split",
            "us_per_frame": round(us, 2), "frames": frames_t, "domains_per_frame": Dall, "tokens_per_frame": T,
            "e2e": {"value": round(frames_t / (e2e_ms * 1e-3), 1), "unit": "frames/s",
                    "h2d_bytes_per_step": D * T * d * 2 * 2, "d2h_bytes_per_step": 0},
            "gpu_launches": int(launches), "roofline": roof(r, us), **{k: v for k, v in r.items()},
            "resolve_kernel": RESOLVE_KERNEL, "clocks": clk.summary()}
    lat = chain_latencies()
    if lat:
        ghz = (clk.summary().get("sm_mhz") or 1965.0) / 1e3
        lo = T * lat["eq34_element_chain_cycles"] / ghz / 1e3
        hi = T * (d * lat["reg_dot_cycles_per_elem"] + lat["ddiv_chain_cycles"]) / ghz / 1e3
        line["chain_bound_us"] = {"state_chain": round(lo, 2), "sequential_rescore": round(hi, 2),
                                  "definition": "per domain (domains run in parallel): 196 dependent Eq. 3/4 element "
                                                "updates (DMUL+DADD+DDIV) = the floor; 196 x a d-long sequential fp64 dot "
                                                "+ division = every routing decision waiting for the previous update",
                                  "latencies": lat}
    us_a = a_ms * 1e3 / frames_t
    line["absorb_only"] = {"value": round(frames_t / (a_ms * 1e-3), 1), "unit": "frames/s", "us_per_frame": round(us_a, 2),
                           "regime": "frames near existing centres (noise 0.015): every insert absorbs",
                           "e2e": {"value": round(frames_t / (a_e2e_ms * 1e-3), 1), "unit": "frames/s"},
                           "roofline": roof(a, us_a), **{k: v for k, v in a.items()}}
    return line


def tensor_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        for k in ("bf16_tflops", "bf16_dense_tflops", "tensor_bf16_tflops"):
            if k in m:
                return float(m[k])
    except Exception:
        pass
    return None


def config4_phase(args):
    """Config 4 per-GPU shard (BASELINE.json configs[3]): Qwen2-VL-72B KV is 80
    layers x 8 KV heads = 640 domains at 256K tokens, head-sharded over 8 GPUs -> one GPU owns 80
    domains (1 KV head x 80 layers) x 262,248 tokens (1,338 frames x 196), C = 512 clusters per
    domain (~512 tokens each), top-16 + 4-frame window, bf16, d = 128: ~10.7 GB of K/V. Decode
    steps timed like the headline (CUDA events on the context stream, inputs in HBM, a different
    query per step); K6's roofline from the instrumented pass against its attended bytes (SURVEY
    §8(d): 80 x ~8,976 x 512 B + 80 x 512 x 128 x 4 B = 388.6 MB -> 59 us at peak)."""
    import torch

    from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload

    D4, N4, C4 = 80, 1338 * T_FRAME, 512
    kv_bytes = D4 * (N4 + 64 * C4 + WINDOW * T_FRAME) * HEAD_DIM * 2 * 2
    cfg = Config.make(kv_dtype=DTYPE_BF16, k_v=1, k_s=TOP_K, window_frames=WINDOW, build_batch_frames=1,
                      offload_horizon_frames=1 << 30, device_capacity_entries=1 << 40,
                      pool_bytes=int(1.2 * kv_bytes), max_slots=max(4096, 3 * D4 * C4), max_cluster_pages=512,
                      max_tokens=T_FRAME, host_pool_bytes=0, max_candidates=1024)
    t0 = time.time()
    kv = ClusterKVCache(cfg, HEAD_DIM, D4)
    st = workload.clustered_state(D4, N4, C4, HEAD_DIM, T_FRAME, seed=4040)
    kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C4)
    del st.keys, st.values
    torch.cuda.empty_cache()
    # fill the local window with 4 new frames (window pages are attended too)
    fk, fv, fvis, fids = workload.frames_near(st, WINDOW, N4 // T_FRAME + 1)
    for i in range(WINDOW):
        kv.process_frame(int(fids[i]), fvis[i], fk[i], fv[i], want_assigned=False)
    del fk, fv
    setup_s = time.time() - t0
    stream = torch.cuda.ExternalStream(kv.stream)
    nq = args.warmup + args.steps
    q_dev = workload.queries_near(st, nq, seed=404)
    out_dev = torch.zeros(D4, HEAD_DIM, device="cuda")
    for i in range(args.warmup):
        kv.query(i, q_dev[i], out=out_dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with Clocks(0) as clk:
        with torch.cuda.stream(stream):
            ev0.record(stream)
            for i in range(args.warmup, nq):
                kv.query(i, q_dev[i], out=out_dev)
            ev1.record(stream)
        torch.cuda.synchronize()
    us_step = ev0.elapsed_time(ev1) * 1e3 / args.steps
    kv.set_timing(True)
    att_us, att_b, k4_us = [], [], []
    with torch.cuda.stream(stream):
        for i in range(args.warmup, nq):
            kv.query(i, q_dev[i], out=out_dev)
            tm = kv.step_timing()
            k4_us.append(tm[0])
            att_us.append(tm[1])
            att_b.append(tm[4])
    torch.cuda.synchronize()
    kv.set_timing(False)
    hbm, src = peaks()
    ab, au = float(np.mean(att_b)), float(np.mean(att_us))
    ach = ab / (au * 1e-6) / 1e9
    step_bytes = ab + D4 * C4 * HEAD_DIM * 4 + D4 * HEAD_DIM * 8
    res = {"workload": "config4 per-GPU shard: Qwen2-VL-72B KV head shard, 80 domains (80 layers x 1 KV head) x 262,248 "
                       "tokens, 512 clusters/domain, top-16 + 4-frame window, bf16, d=128",
           "us_per_step": round(us_step, 2), "unit": "us/step", "steps": args.steps,
           "attended_tokens_per_domain": round(ab / (D4 * 2 * HEAD_DIM * 2), 1),
           "roofline": {"bound": "hbm", "kernel": "k_attend", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(ach / hbm, 4), "algorithmic_bytes_per_launch": ab, "kernel_us": round(au, 2),
                        "peak_source": src, "step_bytes": step_bytes,
                        "step_frac": round(step_bytes / (us_step * 1e-6) / 1e9 / hbm, 4)},
           "score_select_us": round(float(np.mean(k4_us)), 2), "clocks": clk.summary(), "setup_s": round(setup_s, 1),
           "kv_bytes": kv_bytes}
    kv.close()
    del kv
    torch.cuda.empty_cache()
    return res


def offload_phase(args):
    """Config 3 per-GPU shard (14 of 112 domains, as one rank of 8 holds), 1-hour 1 fps stream:
    705,600 tokens/domain in 1,378 clusters of 512, cold clusters offloaded to pinned host memory
    by the reference cadence policy (engine.cpp:95-132; horizon 16 frames). Measures decode steps
    whose selected clusters are cold (K6 attends them in the host tier through the mapping while
    their fetches migrate on the copy engines), the same steps hot, and host-link GB/s of batched
    per-cluster migrations (wall clock of kvc_tier_sync, host bookkeeping included)."""
    import torch

    from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload

    D3, N3, C3 = 14, 3600 * T_FRAME, 1378
    kv_bytes = D3 * (N3 + 64 * C3) * HEAD_DIM * 2 * 2
    cfg = Config.make(kv_dtype=DTYPE_BF16, k_v=1, k_s=TOP_K, window_frames=WINDOW, build_batch_frames=1,
                      offload_horizon_frames=16, device_capacity_entries=1 << 40,
                      pool_bytes=int(1.3 * kv_bytes), host_pool_bytes=int(1.1 * kv_bytes), tier_stage_pages=16384,
                      max_slots=max(4096, 4 * D3 * C3), max_cluster_pages=512, max_tokens=T_FRAME,
                      max_candidates=2048)
    t0 = time.time()
    kv = ClusterKVCache(cfg, HEAD_DIM, D3)
    st = workload.clustered_state(D3, N3, C3, HEAD_DIM, T_FRAME, seed=4242)
    kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C3)
    del st.keys, st.values
    torch.cuda.empty_cache()
    setup_s = time.time() - t0
    # a new frame far past the loaded ones: the cadence offloads every stale cluster
    fk, fv, fvis, fids = workload.frames_near(st, 1, N3 // T_FRAME + 100)
    t0 = time.time()
    kv.process_frame(int(fids[0]), fvis[0], fk[0], fv[0], want_assigned=False)
    kv.tier_sync()
    offload_s = time.time() - t0
    s0 = kv.tier_stats()
    stream = torch.cuda.ExternalStream(kv.stream)
    nq = args.warmup + args.steps
    q_dev = workload.queries_near(st, nq, seed=77)
    out_dev = torch.zeros(D3, HEAD_DIM, device="cuda")

    def timed():
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record(stream)
        for i in range(args.warmup, nq):
            kv.query(i, q_dev[i], out=out_dev)
        ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) * 1e3 / args.steps

    for i in range(args.warmup):  # warm-up queries (their clusters become hot; not re-timed cold)
        kv.query(i, q_dev[i], out=out_dev)
    kv.tier_sync()
    s1 = kv.tier_stats()
    cold_us = timed()
    s2 = kv.tier_stats()
    kv.tier_sync()
    s3 = kv.tier_stats()
    hot_us = timed()  # the same queries: their clusters now sit in HBM
    # host-link bandwidth of batched migrations: the clusters the timed steps fetched go out and back
    ids = kv.cluster_ids()
    moved = [c for c in ids if kv.cluster(c)[0][6] == 0][:2048]
    t0 = time.time()
    for c in moved:
        kv.offload(c)
    kv.tier_sync()
    d2h_s = time.time() - t0
    s4 = kv.tier_stats()
    t0 = time.time()
    for c in moved:
        kv.fetch(c, 1)
    kv.tier_sync()
    h2d_s = time.time() - t0
    s5 = kv.tier_stats()
    # the reference's cross-layer prefetch (retrieval.cpp:117-128: layer l's query ranks layer
    # l+1's clusters, which are fetched with cause Prefetch) turned on: its fetches are real H2D
    # migrations on the transfer stream, issued after each step's replay while the next steps run.
    # Measured on fresh cold queries with every resident cluster offloaded again first.
    pf = {}
    try:
        kv.set_retrieval(prefetch_enabled=1, prefetch_k=TOP_K)
        for c in [c for c in kv.cluster_ids() if kv.cluster(c)[0][6] == 0]:
            kv.offload(c)
        kv.tier_sync()
        q2 = workload.queries_near(st, nq, seed=991)
        l0, p0 = kv.ledger(), kv.tier_stats()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record(stream)
        for i in range(nq):
            kv.query(100000 + i, q2[i], out=out_dev)
        ev1.record(stream)
        torch.cuda.synchronize()
        l1, p1 = kv.ledger(), kv.tier_stats()
        causes = ("retrieval", "maintenance", "prefetch", "completion", "offload")
        pf = {"cold_us_per_step_with_prefetch": round(ev0.elapsed_time(ev1) * 1e3 / nq, 2),
              "ledger_h2d_bytes_per_step_by_cause": {causes[k]: int((l1[1][k] - l0[1][k]) / nq) for k in (0, 2, 3)},
              "physical_h2d_bytes_per_step": int((p1["bytes_h2d"] - p0["bytes_h2d"]) / nq),
              "migrations_in_flight_at_end": p1["in_flight"] + p1["queued"],
              "note": "one step covers every layer at once, so a layer's prediction for layer l+1 is "
                      "issued with (not ahead of) that layer's own selection: the side-stream fetches "
                      "help the following steps only"}
    except Exception as e:  # never lose the main line
        pf = {"error": f"{type(e).__name__}: {e}"}
    # the host link's own copy-engine bandwidth (pinned 256 MiB, best of 5): the roofline of a cold step
    link = {}
    try:
        hb = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
        db = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        for name, (dst, src) in (("h2d", (db, hb)), ("d2h", (hb, db))):
            best = 1e30
            for _ in range(6):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                dst.copy_(src, non_blocking=True)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1))
            link[name + "_gbs"] = round(hb.numel() / (best * 1e-3) / 1e9, 2)
        del hb, db
    except Exception as e:
        link = {"error": f"{type(e).__name__}: {e}"}
    fr_bytes = (s3["read_fetch_bytes"] - s1["read_fetch_bytes"]) / args.steps
    return {
        "workload": "config3 per-GPU shard: 14 domains x 705,600 tokens (3600 frames x 196), 1,378 clusters/domain, "
                    "top-16 + 4-frame window, bf16; cold clusters in pinned host memory (cadence horizon 16)",
        "cold_us_per_step": round(cold_us, 2), "hot_us_per_step": round(hot_us, 2),
        "cold_fetches_per_step": round((s3["fetches"] - s1["fetches"]) / args.steps, 1),
        # fetch-on-read: the step copies its selected Host clusters into HBM between K4 and K6
        # (select.cu R6 + tiers.cu k_fetch_read) instead of K6 reading them in place and the queued
        # fetch migration reading them again
        "fetch_on_read": {
            "clusters_per_step": round((s3["read_fetches"] - s1["read_fetches"]) / args.steps, 1),
            "h2d_bytes_per_step": int((s3["read_fetch_bytes"] - s1["read_fetch_bytes"]) / args.steps),
            "link_gbs_over_cold_step": round(fr_bytes / max(cold_us, 1e-9) / 1e3, 2),
            # the copies' share of the step: cold minus hot time (K4 / K6 / launches as in a hot step)
            "link_gbs_over_copy_time": round(fr_bytes / max(cold_us - hot_us, 1e-9) / 1e3, 2),
            "link_frac": round(fr_bytes / max(cold_us - hot_us, 1e-9) / 1e3 / link["h2d_gbs"], 3)
            if "h2d_gbs" in link else None},
        "host_link_copy_engine": dict(link, how="pinned 256 MiB tensor copy, best of 6, CUDA events"),
        "host_pages_after_cadence": s0["host_pages"], "host_bytes_after_cadence": s0["host_pages"] * 2 * 64 * HEAD_DIM * 2,
        "offload_wall_s": round(offload_s, 3), "setup_s": round(setup_s, 2),
        "d2h_gbs_wall": round((s4["bytes_d2h"] - s3["bytes_d2h"]) / max(d2h_s, 1e-9) / 1e9, 2),
        "h2d_gbs_wall": round((s5["bytes_h2d"] - s4["bytes_h2d"]) / max(h2d_s, 1e-9) / 1e9, 2),
        "migrated_clusters": len(moved), "in_flight_at_end_of_cold_steps": s2["in_flight"] + s2["queued"],
        "dma_copies": {"offload_batch": s4["copies"] - s3["copies"], "fetch_batch": s5["copies"] - s4["copies"]},
        "prefetch": pf,
    }


def streams_phase(args):
    """Config 5 per-GPU share: 4 of 32 independent streams (32 streams partitioned by stream over 8
    GPUs, no collective), each LLaVA-shaped (112 domains) with 65,464 tokens (334 frames x 196) in
    128 clusters of ~512, top-16 + 4-frame window; all 4 contexts decode concurrently (one CUDA
    stream each). Ablation: the token-level top-k baseline (retrieval.cpp:166-254) on the same rows
    at the same budget (16 x 512 tokens), also 4 concurrent contexts."""
    import torch

    from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload

    S_, D5, T5 = 4, D_TOTAL, T_FRAME
    NF = 334
    N5, C5, BUDGET = NF * T5, 128, 16 * 512
    clu, tok, qs = [], [], []
    t0 = time.time()
    for si in range(S_):
        st = workload.clustered_state(D5, N5, C5, HEAD_DIM, T5, seed=500 + si)
        kv_bytes = D5 * (N5 + 64 * C5 + WINDOW * T5) * HEAD_DIM * 2 * 2
        ccfg = Config.make(kv_dtype=DTYPE_BF16, k_v=1, k_s=TOP_K, window_frames=WINDOW, build_batch_frames=1,
                           offload_horizon_frames=1 << 30, device_capacity_entries=1 << 40,
                           pool_bytes=int(1.3 * kv_bytes), max_slots=max(4096, 4 * D5 * C5), max_cluster_pages=512,
                           max_tokens=T5, host_pool_bytes=0)
        kc = ClusterKVCache(ccfg, HEAD_DIM, D5)
        kc.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C5)
        tcfg = Config.make(kv_dtype=DTYPE_BF16, token_mode=1, token_budget=BUDGET, window_frames=WINDOW,
                           pool_bytes=D5 * N5 * HEAD_DIM * 2 * 2, max_tokens=T5)
        kt = ClusterKVCache(tcfg, HEAD_DIM, D5)
        for f in range(NF):  # the same rows, frame by frame, from HBM
            kt.process_frame(f, st.visual, st.keys[:, f * T5:(f + 1) * T5].contiguous(),
                             st.values[:, f * T5:(f + 1) * T5].contiguous(), want_assigned=False)
        qs.append(workload.queries_near(st, args.warmup + args.steps, seed=900 + si))
        del st
        clu.append(kc)
        tok.append(kt)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    outs = [torch.zeros(D5, HEAD_DIM, device="cuda") for _ in range(S_)]

    def run(ctxs, host_sync):
        for i in range(args.warmup):
            for s_, c in enumerate(ctxs):
                c.query(i, qs[s_][i], out=outs[s_])
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        for i in range(args.warmup, args.warmup + args.steps):
            for s_, c in enumerate(ctxs):
                c.query(i, qs[s_][i], out=outs[s_])
        torch.cuda.synchronize()
        return (time.perf_counter() - h0) * 1e6 / args.steps

    clu_us = run(clu, False)
    tok_us = run(tok, True)
    att_c = float(np.mean([clu[0].layer_meta(l).attended_count for l in range(D5)]))
    att_t = float(np.mean([tok[0].layer_meta(l).attended_count for l in range(D5)]))
    return {
        "workload": "config5 per-GPU share: 4 of 32 streams, each 112 domains x 65,464 tokens (334 frames x 196), "
                    "128 clusters/domain, top-16 + 4-frame window, bf16; token ablation at budget 8,192",
        "cluster_us_per_step_all_streams": round(clu_us, 1),
        "cluster_stream_steps_per_s": round(S_ * 1e6 / clu_us, 1),
        "token_us_per_step_all_streams": round(tok_us, 1),
        "token_stream_steps_per_s": round(S_ * 1e6 / tok_us, 1),
        "token_over_cluster_time": round(tok_us / clu_us, 2),
        "attended_per_domain": {"cluster": round(att_c, 1), "token": round(att_t, 1)},
        "timing": "wall clock over all streams' steps (host bookkeeping included), torch.cuda.synchronize on both sides",
        "setup_s": round(setup_s, 1),
    }


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _ref_plan(threads):
    """Domains per reference instance so that `threads` concurrent instances cover all 112
    domains of a step (no extrapolation beyond the 112/(threads x dom) <= 1 correction)."""
    dom = min(CPU_DOMS, -(-D_TOTAL // threads))
    return dom, D_TOTAL / (threads * dom)


def _ref_timed(mode, threads, hs, dom, warmup, steps, queries=None, frames=None):
    from oracle import pyoracle as po

    k, v, a = hs["keys"][:dom], hs["values"][:dom], hs["assign"][:dom]
    if mode == 0:
        return po.time_reference(0, threads, k, v, a, N_CLUST, warmup, steps, TOP_K, WINDOW * T_FRAME,
                                 queries=np.ascontiguousarray(queries[:, :dom]))
    fvis, fk, fv = frames
    return po.time_reference(1, threads, k, v, a, N_CLUST, warmup, steps, TOP_K, WINDOW * T_FRAME,
                             fvis=fvis, fkeys=np.ascontiguousarray(fk[:, :dom]), fvals=np.ascontiguousarray(fv[:, :dom]))


def cpu_baseline(args, hs, queries):
    """The reference decode path (retrieve() + fp64 attention over its attended set) on ALL host
    cores: one reference instance per thread, each over `dom` domains of the same state, so the
    concurrent instances cover the 112 domains of a step."""
    try:
        from oracle import pyoracle as po

        if po.reference() is None:
            return {"value": None, "unit": "us/step", "cores": 0, "kind": "reference", "sample": "oracle/_ref not built"}
        threads = os.cpu_count() or 1
        dom, scale = _ref_plan(threads)
        t0 = time.time()
        us, _ = _ref_timed(0, threads, hs, dom, 1, 3, queries=queries)
        return {"value": round(us * scale, 1), "unit": "us/step", "cores": threads, "kind": "reference",
                "cpu_model": cpu_model(),
                "sample": f"{threads} concurrent reference instances x {dom} domains (N={N_TOK}, C={N_CLUST}, top-{TOP_K} "
                          f"+ window) = {threads * dom} domain-steps per step (x{scale:.3f} to 112), 3 timed steps of "
                          f"retrieve() + fp64 attention; {time.time() - t0:.1f} s wall incl. state build"}
    except Exception as e:  # the baseline must not break the GPU line
        return {"value": None, "unit": "us/step", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}


def cpu_baseline_ingest(args, hs, frames):
    """The reference ingest path (Maintainer::place_frame + on_insert of every (domain, token),
    maintainer.cpp:37-176, as StreamEngine::ingest_frame does) on the same drift-regime frames, ALL
    host cores, instances covering the 112 domains of a frame."""
    try:
        from oracle import pyoracle as po

        if po.reference() is None or hs is None:
            return {"value": None, "unit": "frames/s", "cores": 0, "kind": "reference", "sample": "unavailable"}
        threads = os.cpu_count() or 1
        dom, scale = _ref_plan(threads)
        nfr = frames[1].shape[0]
        t0 = time.time()
        us, _ = _ref_timed(1, threads, hs, dom, 1, nfr - 1, frames=frames)
        us_frame = us * scale
        return {"value": round(1e6 / us_frame, 2), "unit": "frames/s", "us_per_frame": round(us_frame, 1),
                "cores": threads, "kind": "reference", "cpu_model": cpu_model(),
                "sample": f"{threads} concurrent reference instances x {dom} domains, {nfr - 1} timed drift-regime frames "
                          f"(1 warm-up) of place_frame + 196 x {dom} on_insert, x{scale:.3f} to 112 domains; "
                          f"{time.time() - t0:.1f} s wall incl. state build"}
    except Exception as e:
        return {"value": None, "unit": "frames/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}


if __name__ == "__main__":
    main()

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
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def traffic_from_profiles():
    """dram bytes per attention launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_attend_summary.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


# --------------------------------------------------------------------------- reference arm

def run_reference(args, rank: int):
    if rank != 0:
        return
    from oracle import pyoracle as po

    if po.reference() is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libkvclust_ref.so not built"}))
        return
    threads = os.cpu_count() or 1
    dom_sample = 2  # domains per reference instance (each instance ~300 MB of KVEntry)
    st = _host_sample(dom_sample)
    q = _host_queries(st, args.warmup + args.steps)
    us, mean = po.time_reference(0, threads, st["keys"], st["values"], st["assign"], N_CLUST,
                                 args.warmup, args.steps, TOP_K, WINDOW * T_FRAME, queries=q)
    # `threads` instances ran concurrently, each over dom_sample domains
    scale = D_TOTAL / (dom_sample * threads)
    per_step = us * scale
    sample = (f"{threads} concurrent reference instances x {dom_sample} domains (N={N_TOK}, C={N_CLUST}, "
              f"top-{TOP_K} + {WINDOW}-frame window): retrieve() + fp64 attention over the attended set; "
              f"wall us/step scaled by {D_TOTAL}/({dom_sample}x{threads})")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(per_step, 3), "unit": "us/step",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step / 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": _config(args, 1),
        "cpu_baseline": {"value": round(per_step, 3), "unit": "us/step", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(per_step, 3), "unit": "us/step", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
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


# --------------------------------------------------------------------------- our arm

def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

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
    del st.keys, st.values
    torch.cuda.empty_cache()
    stream = torch.cuda.ExternalStream(kv.stream)

    # ------------------------------------------------------------------ ingest (frames/s)
    nf = args.warmup + frames_t
    fk, fv, fvis, fids = workload.frames_near(st, nf, N_TOK // T_FRAME + 1)
    for i in range(args.warmup):
        kv.process_frame(int(fids[i]), fvis[i], fk[i], fv[i])
    splits0 = kv.maint_stats()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = kv.launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with Clocks(local) as clk_ingest:
        ev0.record(stream)
        h0 = time.perf_counter()
        for i in range(args.warmup, nf):
            kv.process_frame(int(fids[i]), fvis[i], fk[i], fv[i], want_assigned=False)
        ingest_host_us = (time.perf_counter() - h0) * 1e6 / frames_t
        ev1.record(stream)
        torch.cuda.synchronize()
    # phase breakdown on a few extra frames (CUDA events add records; kept out of the timed loop)
    kv.set_timing(True)
    ph = []
    xk, xv, xvis, xids = workload.frames_near(st, 3, int(fids[-1]) + 10000, seed=123)
    for i in range(3):
        kv.process_frame(int(xids[i]), xvis[i], xk[i], xv[i], want_assigned=False)
        ph.append(kv.ingest_timing())
    prof_cycles = kv.resolve_profile()
    kv.set_timing(False)
    ingest_phases = dict(zip(["cands", "assign", "topm", "resolve", "store_rows", "host_wait",
                              "host_insert_loop", "host_replay", "host_relaunch_issue", "host_events"],
                             np.mean(ph, axis=0).round(2).tolist()))
    ingest_phases["host_per_frame_timed_loop"] = round(ingest_host_us, 2)
    ingest_ms = ev0.elapsed_time(ev1)
    ingest_launches = kv.launch_count() - launches0
    splits = (kv.maint_stats() - splits0).tolist()
    # e2e ingest: frames from pinned host memory through the public API
    more_k, more_v, more_vis, more_ids = workload.frames_near(st, frames_t, int(fids[-1]) + 20000, seed=99)
    mk_t = more_k.view(torch.int16).cpu().pin_memory()
    mv_t = more_v.view(torch.int16).cpu().pin_memory()
    mk_h, mv_h = mk_t.numpy(), mv_t.numpy()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(frames_t):
        kv.process_frame(int(more_ids[i]), more_vis[i], mk_h[i], mv_h[i], want_assigned=False)
    e1.record(stream)
    torch.cuda.synchronize()
    ingest_e2e_ms = e0.elapsed_time(e1)
    del fk, fv, more_k, more_v

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

    # max over ranks
    vals = torch.tensor([decode_ms, decode_e2e_ms, ingest_ms, ingest_e2e_ms], device="cuda", dtype=torch.float64)
    if world > 1:
        if one_gpu:
            vc = vals.cpu()
            dist.all_reduce(vc, op=dist.ReduceOp.MAX)
            vals = vc
        else:
            dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    decode_ms, decode_e2e_ms, ingest_ms, ingest_e2e_ms = vals.tolist()
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
    line = {
        "metric": METRIC, "value": round(us_step, 3), "unit": "us/step", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": us_step / 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (GPU generator, reference distributions)", "config": _config(args, world),
        "e2e": {"value": round(decode_e2e_ms * 1e3 / args.steps, 3), "unit": "us/step",
                "h2d_bytes_per_step": D * world * HEAD_DIM * 4, "d2h_bytes_per_step": D * world * HEAD_DIM * 4},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic_from_profiles(),
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
        "ingest": {"value": round(frames_t / (ingest_ms * 1e-3), 1), "unit": "frames/s",
                   "frames": frames_t, "domains_per_frame": D * world, "tokens_per_frame": T_FRAME,
                   "e2e": {"value": round(frames_t / (ingest_e2e_ms * 1e-3), 1), "unit": "frames/s",
                           "h2d_bytes_per_step": D * T_FRAME * HEAD_DIM * 2 * 2, "d2h_bytes_per_step": 0},
                   "gpu_launches": int(ingest_launches),
                   "phases_us": ingest_phases,
                   "resolve_kernel": RESOLVE_KERNEL,
                   "resolve_cycles_per_frame": dict(zip(RESOLVE_PHASES[RESOLVE_KERNEL], prof_cycles.round(1).tolist())),
                   "maint_delta": dict(zip(["inserts", "absorbed", "immediate_splits", "deferred_marks",
                                            "settled_splits", "split_ops", "host_over", "maint_fetches",
                                            "partitions_opened"], splits)),
                   "clocks": clk_ingest.summary()},
        "bulk_load_s": round(load_s, 2),
    }
    if world > 1:
        line["config"]["output_exchange"] = ("fused: K6 stores output rows into every rank's buffer over peer memory, "
                                             "per-step signal/wait" if exchange == "fused" else "NCCL all-gather")
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    if world == 1 and not args.no_streams:
        try:
            line["streams"] = streams_phase(args)
        except Exception as e:
            line["streams"] = {"error": f"{type(e).__name__}: {e}"}
    if world == 1 and not args.no_offload:
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
    return {
        "workload": "config3 per-GPU shard: 14 domains x 705,600 tokens (3600 frames x 196), 1,378 clusters/domain, "
                    "top-16 + 4-frame window, bf16; cold clusters in pinned host memory (cadence horizon 16)",
        "cold_us_per_step": round(cold_us, 2), "hot_us_per_step": round(hot_us, 2),
        "cold_fetches_per_step": round((s3["fetches"] - s1["fetches"]) / args.steps, 1),
        "host_pages_after_cadence": s0["host_pages"], "host_bytes_after_cadence": s0["host_pages"] * 2 * 64 * HEAD_DIM * 2,
        "offload_wall_s": round(offload_s, 3), "setup_s": round(setup_s, 2),
        "d2h_gbs_wall": round((s4["bytes_d2h"] - s3["bytes_d2h"]) / max(d2h_s, 1e-9) / 1e9, 2),
        "h2d_gbs_wall": round((s5["bytes_h2d"] - s4["bytes_h2d"]) / max(h2d_s, 1e-9) / 1e9, 2),
        "migrated_clusters": len(moved), "in_flight_at_end_of_cold_steps": s2["in_flight"] + s2["queued"],
        "dma_copies": {"offload_batch": s4["copies"] - s3["copies"], "fetch_batch": s5["copies"] - s4["copies"]},
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


def cpu_baseline(args):
    """The reference hot path on the host, single thread, bounded sample (1 domain)."""
    try:
        from oracle import pyoracle as po

        if po.reference() is None:
            return {"value": None, "unit": "us/step", "cores": 0, "kind": "reference",
                    "sample": "oracle/_ref not built"}
        dom = 1
        h = _host_sample(dom, seed=7)
        q = _host_queries(h, 3)
        us, _ = po.time_reference(0, 1, h["keys"], h["values"], h["assign"], N_CLUST, 1, 2, TOP_K,
                                  WINDOW * T_FRAME, queries=q)
        return {"value": round(us * D_TOTAL / dom, 1), "unit": "us/step", "cores": 1, "kind": "reference",
                "sample": f"1 domain (N={N_TOK}, C={N_CLUST}, top-{TOP_K}+window), 2 timed steps of retrieve() + "
                          f"fp64 attention, single thread, scaled x{D_TOTAL}"}
    except Exception as e:  # the baseline must not break the GPU line
        return {"value": None, "unit": "us/step", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}


if __name__ == "__main__":
    main()

"""bench.py -- one hybrid serving iteration's attention on B200 (HyGen hot path).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-extra]

A "step" is one pass of the whole hot path over one batch:
host plan (validation, indices, prefix tile map) + one descriptor H2D + KV append
+ hybrid attention, through the C ABI's fused entry point hg_hybrid_step.
The workload at EVERY N is BASELINE.json configs[3] ("c3": Llama-3-70B GQA
attention shape, 64 q / 8 KV heads, one 512-token online prefill chunk + 256
decodes at ctx 1-8K, half of them offline in 4 groups sharing 1024-token
prefixes) -- the north_star's head-sharded scaling case, so the N = 1 line and
the N = 1 point of the scaling run are the same measurement.  With --gpus N > 1
KV heads are sharded across N ranks (one process per GPU; bench.py re-launches
itself under torch.distributed.run when WORLD_SIZE is unset) and the outputs
are all-gathered by the attention epilogues themselves, storing into every
rank's peer window over NVLink (hg_hybrid_step_tp with an open window; NCCL is
only the fallback): total work fixed -> "strong".  c1 (configs[1]) and the
other configs are reported under "extra".

--impl reference times the fp64 CPU oracle (oracle/, the only reference this
paper-only task has) on the host cores, on a bounded sample of the same
workload, and prints the same JSON line with "impl": "reference".
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
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "mixed-batch attention tokens/s"
UNIT = "tokens/s"
WORKLOAD = "c3"
WORKLOAD_DESC = ("Llama-3-70B GQA attention shape (64 q / 8 KV heads, head_dim 128, KV block 16): one online "
                 "512-token prefill chunk at c=0 + 128 online decodes + 128 offline decodes (4 groups x 32 sharing "
                 "a 1024-token prefix), ctx U[1024,8192], bf16")


def config_dict(spec, world):
    """The line's `config` (identical in both arms, so the driver can pair them)."""
    return {"workload": WORKLOAD, "desc": WORKLOAD_DESC, "tokens_per_step": spec.T,
            "parallelism": "single GPU" if world == 1 else
            f"kv-head tp{world} (H_kv/{world} KV heads per rank), all-gather fused into the epilogues (peer window)",
            "l2": L2_FLUSH}


_T0 = time.perf_counter()


def progress(msg):
    """Section timestamps on stderr (the JSON line alone goes to stdout): a stalled
    section shows up in the log instead of as a silent timeout."""
    print(f"[bench +{time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi style clock / throttle sampling through NVML during the timed region."""

    def __init__(self, device_index: int, period_s: float = 0.001):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.power, self.mem = [], []
        self.dev, self.period = device_index, period_s
        self._stop = threading.Event()
        self._t = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                    self.mem.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_MEM))
                except Exception:
                    pass
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
            t0 = time.perf_counter()   # the thread is sampling before the timed region starts
            while len(self.samples) < 2 and time.perf_counter() - t0 < 1.0:
                time.sleep(0.0005)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "sm_mhz_min": min(self.samples), "reasons": sorted(self.reasons), "samples": len(self.samples),
                "mem_mhz": statistics.median(self.mem) if self.mem else None,
                "power_w_median": statistics.median(self.power) if self.power else None,
                "power_w_max": max(self.power) if self.power else None,
                "source": "NVML (nvmlDeviceGetClockInfo SM + clocks-event reasons), sampled every 1 ms "
                          "in a thread during the timed region"}


def timed_loop(step, steps, flush, stream, kernel_events):
    """K back-to-back steps, L2 flushed before each outside its events; returns the
    per-step device times (ms), the per-kernel events (if requested) and the host
    time of each step call."""
    import torch
    import paper_2501_14808_b200 as hg
    kev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(steps)] if kernel_events else None
    kopts = [hg.make_opts(events=e) for e in kev] if kernel_events else [None] * steps   # (records the events once)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    host_s = []
    torch.cuda.synchronize()
    for k in range(steps):
        flush_l2(flush)                     # L2 flushed between steps, outside the timed events
        starts[k].record(stream)
        h0 = time.perf_counter()
        step(kopts[k])
        host_s.append(time.perf_counter() - h0)
        ends[k].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in zip(starts, ends)], kev, host_s


def alg_bytes_splitk(spec, hbm_route=False):
    """Algorithmic bytes of the split-K kernel per launch.  HBM route (no tcgen05
    tiles: prefill rows and shared-prefix nodes run in split-K too): the whole
    step's unique KV bytes plus Q and O (alg_bytes_total).  tcgen05 route: the
    unique KV tokens read by decode rows (4*d*H_kv per token: K+V bf16; a shared
    prefix handled by the tcgen05 prefix pass is excluded) plus Q read and O
    written (2*d*H_q each per decode row).  SURVEY.md §8(d) per-unit figures."""
    if hbm_route:
        return alg_bytes_total(spec)
    d, Hk, Hq, B = spec.d, spec.H_kv, spec.H_q, spec.B
    kv_tok, rows = 0, 0
    groups = {}
    for i, r in enumerate(spec.requests):
        if r.n != 1:
            continue
        rows += 1
        s = spec.shared_blocks(i)
        if s:
            groups.setdefault(r.group, 0)
            groups[r.group] += 1
    for i, r in enumerate(spec.requests):
        if r.n != 1:
            continue
        s = spec.shared_blocks(i)
        pre = s * B if (s and groups.get(r.group, 0) >= 2) else 0
        kv_tok += r.c + 1 - pre
    return 4 * d * Hk * kv_tok + 4 * d * Hq * rows


def alg_bytes_total(spec):
    d, Hk, Hq, B = spec.d, spec.H_kv, spec.H_q, spec.B
    U = sum(r.c + r.n for r in spec.requests)
    seen = set()
    for i, r in enumerate(spec.requests):
        s = spec.shared_blocks(i)
        if s:
            if r.group in seen:
                U -= s * B
            seen.add(r.group)
    return 4 * d * Hk * U + 4 * d * Hq * spec.T


def alg_flops(spec):
    return sum(4 * spec.d * spec.H_q * (r.n * r.c + r.n * (r.n + 1) // 2) for r in spec.requests)


L2_FLUSH = ("flushed before every timed step, outside the events: 256 MB written, then another 256 MB read, "
            "so L2 (126 MB) holds clean unrelated lines and no dirty write-back of the flush lands in the step; "
            "KV working set > L2 as well")


def flush_buffer(dev):
    import torch
    return torch.zeros(512 << 20, dtype=torch.uint8, device=dev)


def flush_l2(buf):
    """Evict L2: write 256 MB, then read the other 256 MB (the reads push the dirty
    lines out during the flush, not during the timed step that follows)."""
    import torch
    half = buf.numel() // 2
    buf[:half].zero_()
    buf[half:].view(torch.int32).amax()


def run_ours(args):
    import torch
    import paper_2501_14808_b200 as hg
    from paper_2501_14808_b200.harness import Workload
    from synth.configs import make_config

    rank, world, local = env_rank()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # HG_BENCH_SAME_GPU=1 is a functional test of the multi-rank path on a one-GPU box:
    # every rank on device 0, gloo for the bench's own collectives, no NCCL
    # communicator (the peer window carries the gather).  Its timings are not a
    # scaling measurement (the ranks time-slice one GPU).
    same_gpu = os.environ.get("HG_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    peaks, peak_kind = load_peaks()
    spec = make_config(WORKLOAD, 0)

    if world > 1:
        return run_tp(args, spec, rank, world, dev, peaks, peak_kind)

    progress(f"workload {WORKLOAD}")
    wl = Workload(spec, device=dev)
    stream = torch.cuda.current_stream(dev)
    flush = flush_buffer(dev)
    for _ in range(args.warmup):
        wl.step()
    torch.cuda.synchronize()
    # Two passes of K timed steps: the headline pass with only the step events (so
    # the combine runs as a programmatic dependent launch right behind split-K),
    # then a pass with the library's per-kernel events around every kernel (the
    # dominant kernel's roofline; an event between two kernels breaks that PDL
    # pairing, so this pass is a little slower).  Steps are issued back to back:
    # the host plans step k+1 while the GPU runs step k (the serving-engine overlap).
    progress("warm-up done; timed steps")
    with ClockSampler(local) as clk:
        step_ms, _, host_s = timed_loop(lambda o: wl.step(o), args.steps, flush, stream, False)
    step_ms_ev, kev, _ = timed_loop(lambda o: wl.step(o), args.steps, flush, stream, True)
    # host cost of one call with the GPU idle (no staging-ring backpressure): validation,
    # plan, descriptor image, launches -- what a serving loop pays per step on the CPU
    host_idle = []
    for _ in range(5):
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        wl.step()
        host_idle.append(time.perf_counter() - h0)
    torch.cuda.synchronize()
    st = hg.hg_last_plan_stats(wl.pool)
    sk_ms = [e[2].elapsed_time(e[3]) for e in kev] if st["splitk_items"] else []
    tc_ms = [e[0].elapsed_time(e[1]) for e in kev] if st["tc_tiles"] else []
    cb_ms = [e[4].elapsed_time(e[5]) for e in kev] if st["combine_rows"] else []
    total_ms = sum(step_ms)
    ms = total_ms / args.steps
    stats = hg.hg_last_plan_stats(wl.pool)
    launches_per_step = stats["kernels"]        # fused step: append + tcgen05 + split-K + combine
    T = spec.T
    value = T * args.steps / (total_ms / 1e3)

    # roofline of the dominant kernel (split-K decode: HBM-bound)
    sk_avg = statistics.mean(sk_ms) if sk_ms else None
    bytes_sk = alg_bytes_splitk(spec, hbm_route=not st["tc_tiles"])
    achieved = bytes_sk / (sk_avg / 1e3) / 1e9 if sk_avg else None
    traffic = load_traffic(f"splitk_kernel@{WORKLOAD}", bytes_sk)
    roofline = {"bound": "hbm", "kernel": "splitk_kernel<128>", "achieved": achieved, "peak": peaks["hbm_gbs"],
                "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, copy)" if peak_kind == "measured" else "fallback",
                "unit": "GB/s", "frac": (achieved / peaks["hbm_gbs"]) if achieved else None,
                "traffic": traffic["bytes"] if traffic else None,   # DRAM read+write bytes per launch (ncu)
                "traffic_detail": traffic, "alg_bytes_per_launch": bytes_sk, "avg_launch_ms": sk_avg,
                "share_of_step": (sk_avg / (sum(step_ms_ev) / args.steps)) if sk_avg else None,
                "timing": "split-K events over a second pass of the same K timed steps (per-kernel events on)",
                "ms_per_step_with_kernel_events": sum(step_ms_ev) / args.steps}
    # whole-step roofline (all kernels): t_roof = max(bytes/BW, flops/TC)
    bt, fl = alg_bytes_total(spec), alg_flops(spec)
    t_roof = max(bt / (peaks["hbm_gbs"] * 1e9), fl / (peaks["bf16_tflops"] * 1e12))
    progress("timed steps done; e2e")
    e2e = None if args.profile else measure_e2e(wl, spec, args, stream)
    split_calls = None if args.profile else measure_append_attention(wl, flush, stream)
    progress("extra configs")
    extra = extra_configs(args, peaks, dev) if args.extra else None
    if extra:   # the tensor-bound (prefill-heavy) configs' rooflines, kept inside the roofline dict
        roofline["prefill_heavy"] = {k: v["roofline"] for k, v in extra.items() if k in ("p1", "p2")}
        roofline["other_configs"] = {k: v["roofline"] for k, v in extra.items() if k not in ("p1", "p2")}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (seeded counter-based N(0,1)-scale bf16 Q/K/V; fragmented block tables)",
        "config": config_dict(spec, 1),
        "roofline": roofline,
        "step_roofline": {"alg_bytes": bt, "alg_flops": fl, "t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / ms},
        "kernel_ms": {"splitk": sk_avg, "tc": statistics.mean(tc_ms) if tc_ms else None,
                      "combine": statistics.mean(cb_ms) if cb_ms else None},
        "host_call_ms": {"in_loop": statistics.median(host_s) * 1e3,
                         "gpu_idle": statistics.median(host_idle) * 1e3,
                         "note": "in_loop includes waiting for a free pinned staging slot (8-deep ring) "
                                 "while the GPU runs earlier steps; gpu_idle is the call's own CPU cost"},
        "kernel_ms_median": {"splitk": statistics.median(sk_ms) if sk_ms else None,
                             "tc": statistics.median(tc_ms) if tc_ms else None,
                             "combine": statistics.median(cb_ms) if cb_ms else None},
        "plan": stats,
        "append_and_attention_ms": split_calls,
        "gpu_launches": launches_per_step * args.steps,
        "e2e": e2e,
        "clocks": clk.summary(),
    }
    if extra:
        line["extra"] = extra
    if not args.profile and not args.no_predictor:
        progress("predictor sweeps")
        pred = predictor_sweep(dev, iters=args.sweep_iters)
        model = pred.pop("_model")
        line["predictor"] = pred
        pred2 = predictor_sweep(dev, iters=args.sweep_iters, shape="llama2-7b")   # C4's second shape
        pred2.pop("_model")
        line["predictor_llama2_7b"] = pred2
        progress("slo loops")
        line["slo_loop"] = slo_loop(dev, model)
        # the same loop with an online profiler refitting on its own observations
        line["slo_loop_online_refit"] = slo_loop(dev, model, refit_every=25)
        progress("psm vs fcfs")
        line["psm_vs_fcfs"] = psm_vs_fcfs(dev)
    if args.extra:
        progress("next4")
        line["next4"] = next4(dev, peaks)
        # the north_star's multi-GPU config (this line's workload): per-rank sharded step at G = 2/4/8
        progress("shard projections")
        line["shard_projection_c3"] = shard_projection(spec, dev, ms, peaks)
        line["shard_projection_c1"] = shard_projection(make_config("c1", 0), dev, extra["c1"]["ms_per_step"], peaks)
    progress("cpu baseline")
    line["cpu_baseline"] = None if args.profile else cpu_baseline(spec, wl)
    progress("done")
    wl.close()
    print(json.dumps(line))


def load_traffic(kernel, alg_bytes):
    """dram__bytes_read+write per launch for `kernel` from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        k = d["kernels"][kernel]
        return {"bytes": k["dram_bytes"], "over_alg": k["dram_bytes"] / alg_bytes, "source": d.get("source", p)}
    except Exception:
        return None


def shard_projection(spec, dev, ms_step, peaks, reps=50):
    """One GPU timing the per-rank work of KV-head sharding at G = 1, 2, 4, 8: rank
    0's slice (H_kv/G KV heads, H_q/G q heads) through the SHARDED entry point
    hg_hybrid_step_tp on a 1-rank peer-window communicator -- the fused append
    with the window entry barrier, the epilogues storing into the window, the
    exit flag barrier -- L2 flushed, device time (the GPU is kept busy while the
    host plans).  What a 1-GPU box cannot show: the other G-1 destinations of each
    epilogue store (T*H_q*d*2*(G-1)/G bytes per rank over NVLink, ~11 MB at G = 8 on
    C3 = ~12 us at 900 GB/s if none of it overlapped the kernels) and the wait for
    the slowest peer at the barriers."""
    import torch
    import paper_2501_14808_b200 as hg
    from paper_2501_14808_b200.harness import Workload
    from synth.configs import shard_slice
    out = {}
    flush = flush_buffer(dev)
    base = None
    for G in (1, 2, 4, 8):
        if spec.H_kv % G:
            continue
        local = shard_slice(spec, G)
        wl = Workload(local, device=dev)
        comm = hg.Comm(None, 0, 1, dev.index)
        h = comm.hg_comm_window_create(local.T * local.H_q * local.d * 2)
        comm.hg_comm_window_open([h])
        win = comm.window((local.T, local.H_q, local.d))
        ws = torch.empty(hg.hg_hybrid_attention_tp_workspace_size(wl.pool, comm, wl.batch, local.H_q),
                         dtype=torch.uint8, device=dev)
        step = lambda: hg.hg_hybrid_step_tp(wl.pool, comm, wl.batch, local.H_q, wl.q, wl.k_new, wl.v_new, win, ws)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush_l2(flush)
            torch.cuda._sleep(1_000_000)   # GPU busy while the host plans and enqueues: device time only
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        comm.close()
        wl.close()
        m = statistics.median(ts)
        base = m if G == 1 else base
        t_roof = alg_bytes_total(local) / (peaks["hbm_gbs"] * 1e9) * 1e3
        out[f"G={G}"] = {"per_rank_ms": m, "projected_speedup": base / m, "per_rank_t_roof_ms": t_roof,
                         "per_rank_roof_frac": t_roof / m}
    out["workload"] = spec.name
    out["note"] = ("rank 0's slice through hg_hybrid_step_tp on a 1-rank peer window (append + entry barrier, "
                   "epilogue window stores, exit barrier), each call alone, median of %d, L2 flushed, device time; "
                   "speedup against G = 1 timed the same way; the NVLink copies to the other G-1 ranks and "
                   "waiting for peers are not in it -- a projection, not a multi-GPU measurement (the bench "
                   "loop's own step at G = 1: %.4f ms)" % (reps, ms_step))
    return out


def measure_append_attention(wl, flush, stream, reps=30):
    """append timed separately and as append+attention -- the unfused
    calls (hg_kv_append, then hg_hybrid_attention), device time of each, L2 flushed."""
    import torch
    res = {}
    for name, fn in (("append", lambda: wl.append(stream)), ("attention", lambda: wl.attention(stream=stream)),
                     ("append_then_attention", lambda: (wl.append(stream), wl.attention(stream=stream))),
                     ("fused_step", lambda: wl.step(stream=stream))):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush_l2(flush)
            torch.cuda._sleep(1_000_000)   # GPU busy while the host plans and enqueues: device time only
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[name] = statistics.median(ts)
    res["note"] = ("each call alone (GPU kept busy while the host plans it, so device time only), median of "
                   "%d, L2 flushed; the timed steps above run back to back with per-kernel events" % reps)
    return res


def measure_e2e(wl, spec, args, stream):
    """Same metric through hg_hybrid_step_host: pinned host q/k/v in, host O out, copies timed."""
    import torch
    import paper_2501_14808_b200 as hg
    qh = wl.q.cpu().pin_memory()
    kh = wl.k_new.cpu().pin_memory()
    vh = wl.v_new.cpu().pin_memory()
    oh = torch.empty(wl.out.shape, dtype=torch.bfloat16).pin_memory()
    ws = torch.empty(hg.hg_hybrid_step_host_workspace_size(wl.pool, wl.batch, spec.H_q), dtype=torch.uint8,
                     device=wl.device)
    # warm-up: at least W steps and 0.5 s -- the host step's wall time settles only
    # after ~100 synchronised steps on these boxes (0.94 -> 0.61 ms, tools/prof_e2e.py)
    w, t0 = 0, time.perf_counter()
    while w < args.warmup or time.perf_counter() - t0 < 0.5:
        hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws, stream)
        w += 1
    torch.cuda.synchronize()
    steps = max(args.steps, 50)
    t0 = time.perf_counter()
    for _ in range(steps):
        hg.hg_hybrid_step_host(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws, stream)
    dt = time.perf_counter() - t0
    h2d = (qh.numel() + kh.numel() + vh.numel()) * 2
    # the serving-loop form: the next step is validated and planned while the GPU runs
    # this one (hg_hybrid_step_host_plan), each step still uploads its inputs only after
    # the previous step's result is back (synchronise, then the next call)
    sync = stream.synchronize if stream is not None else torch.cuda.synchronize
    for _ in range(max(args.warmup, 20)):
        hg.hg_hybrid_step_host_async(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws, stream)
        hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)
        sync()
    t1 = time.perf_counter()
    for _ in range(steps):
        hg.hg_hybrid_step_host_async(wl.pool, wl.batch, spec.H_q, qh, kh, vh, oh, ws, stream)
        hg.hg_hybrid_step_host_plan(wl.pool, wl.batch, spec.H_q)   # step k+1's plan beside step k
        sync()
    dt_pipe = time.perf_counter() - t1
    return {"value": spec.T * steps / dt, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": oh.numel() * 2, "ms_per_step": dt / steps * 1e3, "steps": steps,
            "warmup_steps": w,
            "api": "hg_hybrid_step_host (C ABI, host buffers; two pipelined input waves; synchronises each step)",
            "plan_ahead": {"value": spec.T * steps / dt_pipe, "ms_per_step": dt_pipe / steps * 1e3,
                           "api": "hg_hybrid_step_host_async + hg_hybrid_step_host_plan of the next step while the "
                                  "GPU runs, then synchronise (inputs of step k+1 still go up after step k's result)"}}


def cpu_baseline(spec, wl=None, sample_reqs=None, min_s=10.0):
    """The fp64 oracle (as it stands) on the host cores, on a bounded sample of the
    workload: the prefill request plus every 8th decode request; tokens/s is
    extrapolated by the sample's share of the attention work (key-rows x heads)."""
    import numpy as np
    import oracle
    from oracle.run import fill_pool
    from synth.layout import make_layout
    from synth.values import q_values
    lay = wl.lay if wl is not None else make_layout(spec)
    if sample_reqs is None:
        dec = [i for i, r in enumerate(spec.requests) if r.n == 1]
        pre = [i for i, r in enumerate(spec.requests) if r.n > 1]
        sample_reqs = sorted(pre + dec[::8])
    work = lambda idx: sum(r.n * r.c + r.n * (r.n + 1) // 2 for k, r in enumerate(spec.requests) if k in idx)
    frac = work(set(sample_reqs)) / work(set(range(len(spec.requests))))
    pool = fill_pool(spec, lay, req_sel=sample_reqs, device="cuda" if wl is not None else "cpu")
    c = np.array([r.c for r in spec.requests], np.int32)
    n = np.array([r.n for r in spec.requests], np.int32)
    q = q_values(spec)
    passes, t0 = 0, time.perf_counter()
    while True:       # repeat the sample for ~min_s of CPU work (bounded: a few minutes at most)
        pool.attention(lay.block_table, c, n, q, spec.H_q, req_sel=sample_reqs)
        passes += 1
        if time.perf_counter() - t0 >= min_s:
            break
    dt = (time.perf_counter() - t0) / passes
    t_full = dt / frac
    return {"value": spec.T / t_full, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{len(sample_reqs)} of {len(spec.requests)} requests ({frac:.1%} of the attention work) x "
                      f"{passes} passes, {dt:.3f} s per pass; full-batch time extrapolated by work share",
            "oracle_s_per_pass": dt}


def extra_configs(args, peaks, dev):
    """Other BASELINE.json configs (context; not the headline line)."""
    import torch
    import paper_2501_14808_b200 as hg
    from paper_2501_14808_b200.harness import Workload
    from synth.configs import make_config
    out = {}
    for name in ("c1", "c2", "p1", "p2"):
        progress(f"extra {name}")
        spec = make_config(name, 0)
        wl = Workload(spec, device=dev)
        flush = flush_buffer(dev)
        for _ in range(3):
            wl.step()
        n = 10
        kev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(n)]
        kopts = [hg.make_opts(events=e) for e in kev]
        se = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        torch.cuda.synchronize()
        for k in range(n):
            flush_l2(flush)
            se[k][0].record()
            wl.step(kopts[k])
            se[k][1].record()
        torch.cuda.synchronize()
        ms = [s.elapsed_time(e) for s, e in se]
        host_idle = []
        for _ in range(3):
            torch.cuda.synchronize()
            h0 = time.perf_counter()
            wl.step()
            host_idle.append(time.perf_counter() - h0)
        torch.cuda.synchronize()
        st = hg.hg_last_plan_stats(wl.pool)
        ker = {"tc": [e[0].elapsed_time(e[1]) for e in kev] if st["tc_tiles"] else [],
               "splitk": [e[2].elapsed_time(e[3]) for e in kev] if st["splitk_items"] else [],
               "combine": [e[4].elapsed_time(e[5]) for e in kev] if st["combine_rows"] else []}
        m = statistics.median(ms)
        bt, fl = alg_bytes_total(spec), alg_flops(spec)
        t_roof = max(bt / (peaks["hbm_gbs"] * 1e9), fl / (peaks["bf16_tflops"] * 1e12))
        kms = {k: (statistics.median(v) if v else None) for k, v in ker.items()}
        out[name] = {"tokens_per_s": spec.T / (m / 1e3), "ms_per_step": m, "t_roof_ms": t_roof * 1e3,
                     "step_roof_frac": t_roof * 1e3 / m, "alg_bytes": bt, "alg_flops": fl,
                     "kernel_ms": kms, "plan": hg.hg_last_plan_stats(wl.pool),
                     "host_call_ms_gpu_idle": statistics.median(host_idle) * 1e3}
        if name.startswith("p") and kms["tc"]:
            # tensor-bound: the tcgen05 kernel does all the work; algorithmic (causal) FLOPs
            ach = fl / (kms["tc"] / 1e3) / 1e12
            out[name]["roofline"] = {"bound": "tensor", "kernel": "tc_attn_kernel<128>", "achieved": ach,
                                     "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                                     "frac": ach / peaks["bf16_tflops"],
                                     "peak_kind": "measured burst (MEASURED_PEAKS.json bf16_tflops, cuBLAS)",
                                     # for a long prefill-heavy run: the part sits at its 1 kW power cap
                                     # (tools/clock_probe.py), where cuBLAS itself sustains this figure
                                     "frac_vs_sustained": ach / peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]),
                                     "alg_flops_per_launch": fl, "avg_launch_ms": kms["tc"], "step_ms": m,
                                     "share_of_step": kms["tc"] / m}
        elif kms["splitk"]:
            b_sk = alg_bytes_splitk(spec, hbm_route=not st["tc_tiles"])
            ach = b_sk / (kms["splitk"] / 1e3) / 1e9
            out[name]["roofline"] = {"bound": "hbm", "kernel": "splitk_kernel<128>", "achieved": ach,
                                     "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": ach / peaks["hbm_gbs"],
                                     "alg_bytes_per_launch": b_sk, "avg_launch_ms": kms["splitk"], "step_ms": m,
                                     "share_of_step": kms["splitk"] / m}
        wl.close()
        del wl
        torch.cuda.empty_cache()
    return out


def predictor_sweep(dev, iters=64, reps=5, shape="llama3-8b", seed=0):
    """C4: time hg_hybrid_attention on the bursty-trace batches, fit the paper's
    linear-regression predictor on a random 80%, report held-out MAPE.

    Target y = GPU time of the call's kernels (first kernel start -> last
    kernel end, library-recorded events), median of `reps`, L2 flushed before
    each rep.  K/V content is random (timing does not depend on values)."""
    import numpy as np
    import torch
    import paper_2501_14808_b200 as hg
    from synth.layout import make_layout
    from synth.trace import sweep
    H = {"llama3-8b": (32, 8, 128), "llama2-7b": (32, 32, 128)}[shape]
    t0 = time.perf_counter()
    specs = sweep(seed=seed, iters=iters, H_q=H[0], H_kv=H[1], d=H[2])
    need = max(sum(-(-(r.c + r.n) // 16) for r in s.requests) for s in specs)
    N = int(need * 1.25) + 64
    kc = torch.randn((N, H[1], 16, H[2]), device=dev).to(torch.bfloat16)
    vc = torch.randn((N, H[1], 16, H[2]), device=dev).to(torch.bfloat16)
    pool = hg.KVPool(kc, vc, N, 16, H[1], H[2], dev.index)
    maxT = max(s.T for s in specs)
    q = torch.randn((maxT, H[0], H[2]), device=dev).to(torch.bfloat16)
    kn = torch.randn((maxT, H[1], H[2]), device=dev).to(torch.bfloat16)
    vn = torch.randn((maxT, H[1], H[2]), device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    flush = flush_buffer(dev)
    ws = None
    X, y, T, pre, stats = [], [], [], [], []
    for k, spec in enumerate(specs):
        lay = make_layout(spec, seed=k, num_blocks=N)
        b = hg.Batch(lay.block_table, [r.c for r in spec.requests], [r.n for r in spec.requests],
                     [int(r.offline) for r in spec.requests], lay.shared)
        need_ws = hg.hg_hybrid_attention_workspace_size(pool, b, H[0])
        if ws is None or ws.numel() < need_ws:
            ws = torch.empty(need_ws * 2, dtype=torch.uint8, device=dev)
        hg.hg_kv_append(pool, b, kn, vn)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(reps)]
        ops = [hg.make_opts(events=e) for e in evs]
        for r in range(reps):
            flush_l2(flush)
            hg.hg_hybrid_attention(pool, b, H[0], q, out, None, ws, None, ops[r])
        torch.cuda.synchronize()
        st = hg.hg_last_plan_stats(pool)
        stats.append([st[k] for k in ("tc_tiles", "prefix_tiles", "splitk_items", "combine_rows", "kernels")])
        first = 0 if st["tc_tiles"] else 2 if st["splitk_items"] else 4
        last = 5 if st["combine_rows"] else 3 if st["splitk_items"] else 1
        y.append(statistics.median(e[first].elapsed_time(e[last]) for e in evs))
        X.append(hg.hg_batch_features(b).as_array())
        T.append(spec.T)
        sp = sum(r.n for r in spec.requests if not (r.n == 1 and r.c >= 1))
        pre.append(sp / spec.T)
    pool.close()
    X, y = np.array(X), np.array(y)
    if os.environ.get("HG_SAVE_SWEEP"):   # raw sweep for offline residual analysis
        np.savez(os.path.join(os.environ["HG_SAVE_SWEEP"], f"sweep_{shape}.npz"), X=X, y=y, T=np.array(T),
                 stats=np.array(stats))
    rng = np.random.default_rng(1)
    perm = rng.permutation(len(y))
    ntr = int(0.8 * len(y))
    tr, te = perm[:ntr], perm[ntr:]
    res = {"batches": len(y), "shape": shape, "reps": reps, "target": "GPU ms of the call's kernels (median)",
           "sweep_s": time.perf_counter() - t0}
    fits = (("attn (S_p, P2, D_ctx, N_d, N_p)", hg.HG_MASK_ATTN),
            ("attn, relative-error LS", hg.HG_MASK_ATTN | hg.HG_FIT_RELATIVE),
            ("paper Eq.2 (S_p, S_p^2, N_p, N_d)", hg.HG_MASK_EQ2),
            ("paper Eq.2, relative-error LS", hg.HG_MASK_EQ2 | hg.HG_FIT_RELATIVE),
            ("paper Eq.1 (S_p, S_p^2, S_d^2, N_p, N_d)", hg.HG_MASK_EQ1))
    best = None
    for name, mask in fits:
        t1 = time.perf_counter()
        m = hg.hg_predictor_fit(X[tr], y[tr], mask)
        fit_ms = (time.perf_counter() - t1) * 1e3
        yh = np.array([hg.hg_predictor_predict(m, hg.features_from_array(x)) for x in X[te]])
        t2 = time.perf_counter()
        for x in X[te]:
            hg.hg_predictor_predict(m, hg.features_from_array(x))
        pred_us = (time.perf_counter() - t2) / len(te) * 1e6
        res[name] = {"mape_heldout": float(np.mean(np.abs(yh - y[te]) / y[te])), "train_mape": m.train_mape,
                     "fit_ms": fit_ms, "predict_us_python": pred_us, "w": list(m.w)}
        if mask & 0xFF == hg.HG_MASK_ATTN and (best is None or m.train_mape < best[0]):
            best = (m.train_mape, m, name)   # chosen on the TRAINING split only
    res["_model"] = best[1]
    res["selected_for_slo_loop"] = best[2]
    # tokens/s versus mix (share of prefill tokens in the batch)
    pre = np.array(pre)
    mix = {}
    for lo, hi in ((0, 0.05), (0.05, 0.5), (0.5, 0.9), (0.9, 1.01)):
        sel = (pre >= lo) & (pre < hi)
        if sel.any():
            mix[f"prefill_share[{lo},{hi})"] = {"batches": int(sel.sum()),
                                                 "tokens_per_s": float(np.sum(np.array(T)[sel]) / (np.sum(y[sel]) / 1e3))}
    res["tokens_per_s_vs_mix"] = mix
    return res


def slo_loop(dev, model, budget_ms=0.25, chunk=512, iters=300, seed=0, H=(32, 8, 128), refit_every=0):
    """NEXT-1 closed loop: HyGen's two-phase scheduling (Alg. 2 calls Alg. 1 for the
    online then the offline phase) with hg_slo_aware_schedule over the
    fitted predictor, on a bursty online trace + offline backlog (synth.trace
    shapes); every composed batch runs through hg_hybrid_attention and its
    measured kernel time is compared with the latency budget and the prediction."""
    import math
    import numpy as np
    import torch
    import paper_2501_14808_b200 as hg
    from synth.configs import BatchSpec, Request
    from synth.layout import make_layout
    from synth.trace import BASE_QPS, ITER_S, PERIOD_S, _lognormal
    rng = np.random.default_rng(seed)
    B = 16
    N = 40000
    kc = torch.randn((N, H[1], B, H[2]), device=dev).to(torch.bfloat16)
    vc = torch.randn((N, H[1], B, H[2]), device=dev).to(torch.bfloat16)
    pool = hg.KVPool(kc, vc, N, B, H[1], H[2], dev.index)
    q = torch.randn((4096, H[0], H[2]), device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    flush = flush_buffer(dev)
    ws = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    online, offline = [], []   # [prompt, output, done_prompt, done_out, group, prefix]
    obs_x, obs_y, refits, first_refit = [], [], 0, None
    t_sim, gid = rng.uniform(0, PERIOD_S), 0
    rows = []
    tok_on = tok_off = 0
    for it in range(iters):
        rate = 2.0 * BASE_QPS * (2.0 + math.sin(2 * math.pi * t_sim / PERIOD_S)) / 2.0
        for _ in range(rng.poisson(rate * ITER_S)):
            online.append([_lognormal(rng, 1024, 0.8, 32, 8192), _lognormal(rng, 128, 0.8, 1, 512), 0, 0, -1, 0])
        while len(offline) < 64:
            if rng.random() < 0.5:
                for _ in range(32):
                    offline.append([1024 + _lognormal(rng, 256, 0.8, 16, 2048), _lognormal(rng, 256, 0.8, 1, 512),
                                    0, 0, gid, 1024])
                gid += 1
            else:
                offline.append([_lognormal(rng, 6144, 0.5, 1024, 16384), _lognormal(rng, 256, 0.8, 1, 512), 0, 0, -1, 0])

        def split(reqs):
            run = [r for r in reqs if r[2] > 0]
            que = [r for r in reqs if r[2] == 0]
            f = lambda r: (r[2] + r[3], r[0] - r[2], r[5] if (r[4] >= 0 and r[2] >= r[5]) else 0, r[4])
            return run, que, [f(r) for r in run], [f(r) for r in que]
        entries = []
        t, c, m = budget_ms, chunk, N // 2
        state = hg.hg_sched_state()   # one batch: the offline phase continues the online one
        for phase, reqs in ((True, online), (False, offline)):
            run, que, rs, qs = split(reqs)
            sched, t, c, m = hg.hg_slo_aware_schedule(model, rs, qs, t, c, m, phase, state=state)
            for idx, l, tr in sched:
                r = run[idx] if idx < len(run) else que[idx - len(run)]
                entries.append((r, l, tr, phase))
        if not entries:
            t_sim += ITER_S
            continue
        reqs = []
        for r, l, tr, phase in entries:
            cached = r[2] + r[3]
            share = r[4] >= 0 and r[2] >= r[5]
            reqs.append(Request(cached, 1 if l == 0 else l, not phase, r[4], r[5], share=share))
        spec = BatchSpec("slo", H[0], H[1], H[2], B, 0, reqs)
        if spec.T > q.shape[0]:
            continue
        lay = make_layout(spec, seed=it, num_blocks=N)
        b = hg.Batch(lay.block_table, [x.c for x in reqs], [x.n for x in reqs], None, lay.shared)
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(5)]
        for ev in evs:   # median of 5 L2-flushed runs of the composed batch (as the C4 sweep's target)
            flush_l2(flush)
            hg.hg_hybrid_attention(pool, b, H[0], q, out, None, ws, None, hg.make_opts(events=ev))
        torch.cuda.synchronize()
        st = hg.hg_last_plan_stats(pool)
        first = 0 if st["tc_tiles"] else 2
        last = 5 if st["combine_rows"] else 3 if st["splitk_items"] else 1
        meas = statistics.median(ev[first].elapsed_time(ev[last]) for ev in evs)
        pred = model.w[0] + sum(tr for _, _, tr, _ in entries)
        feats = hg.hg_batch_features(b)
        whole = hg.hg_predictor_predict(model, feats)   # the model on the batch itself
        rows.append((meas, pred, whole))
        if refit_every:
            # online profiler: refit the predictor on the loop's own (batch, measured time)
            # pairs every `refit_every` iterations (same features, relative-error LS)
            obs_x.append(feats.as_array())
            obs_y.append(meas)
            if len(obs_y) >= 30 and len(obs_y) % refit_every == 0:
                ox = np.array(obs_x)
                mask = model.feature_mask
                for k in range(8):   # a feature constant over the loop's batches is collinear with the intercept
                    if mask >> k & 1 and np.ptp(ox[:, k]) == 0:
                        mask &= ~(1 << k)
                try:
                    model = hg.hg_predictor_fit(ox, np.array(obs_y), mask)
                    refits += 1
                    if first_refit is None:
                        first_refit = len(rows)
                except hg.HgError:
                    pass
        for r, l, tr, phase in entries:
            if l == 0:
                r[3] += 1
                if phase:
                    tok_on += 1
                else:
                    tok_off += 1
            else:
                r[2] += l
                if phase:
                    tok_on += l
                else:
                    tok_off += l
        online[:] = [r for r in online if r[3] < r[1]]
        offline[:] = [r for r in offline if r[3] < r[1]]
        t_sim += ITER_S
    pool.close()
    meas = np.array([r[0] for r in rows])
    pred = np.array([r[1] for r in rows])
    whole = np.array([r[2] for r in rows])
    return {"iterations": len(rows), "budget_ms": budget_ms, "chunk_budget": chunk, "reps_per_batch": 5,
            "within_budget_frac": float(np.mean(meas <= budget_ms)),
            "p99_ms": float(np.percentile(meas, 99)), "mean_ms": float(meas.mean()),
            "mape_pred_vs_measured": float(np.mean(np.abs(pred - meas) / meas)),
            "bias_pred_vs_measured": float(np.mean((pred - meas) / meas)),
            "mape_batch_predict_vs_measured": float(np.mean(np.abs(whole - meas) / meas)),
            "online_tokens": tok_on, "offline_tokens": tok_off,
            "refit_every": refit_every, "refits": refits,
            "mape_after_first_refit": (float(np.mean(np.abs(pred[first_refit:] - meas[first_refit:]) / meas[first_refit:]))
                                       if first_refit is not None and first_refit < len(rows) else None),
            "note": "kernel-level analogue of the paper's SLO loop: budget = attention GPU time per iteration"}


def next4(dev, peaks, reps=20):
    """NEXT-4 on one GPU: (a) the rope prologue's cost on the c1 step (hg_hybrid_step with
    and without hg_rope), (b) the output-projection GEMM of hg_out_proj_rs (G = 1: its
    epilogue stores straight into Y) at the Llama-3-70B shapes of c3 (hidden 8192; K =
    64 heads x 128 on one GPU, 8 heads x 128 per rank at TP-8), against its tensor roofline."""
    import torch
    import paper_2501_14808_b200 as hg
    from paper_2501_14808_b200.harness import Workload
    from synth.configs import make_config
    from synth.values import KIND_O, KIND_W, matrix
    res = {}
    spec = make_config("c1", 0)
    for name, sp in (("c1", spec), ("c1_rope", spec.with_(rope=(1e4, 0)))):
        wl = Workload(sp, device=dev)
        for _ in range(3):
            wl.step()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            wl.step()
        e.record()
        torch.cuda.synchronize()
        res[name + "_ms_per_step"] = s.elapsed_time(e) / reps
        wl.close()
    comm = hg.Comm(None, 0, 1, dev.index)
    peak = peaks["bf16_tflops"]
    for T, K, N in ((768, 8192, 8192), (768, 1024, 8192)):
        O = matrix(1, KIND_O, 0, T, K, device=dev)
        W = matrix(1, KIND_W, 0, K, N, scale=K ** -0.5, device=dev)
        y = torch.empty((T, N), dtype=torch.bfloat16, device=dev)
        for _ in range(3):
            hg.hg_out_proj_rs(comm, T, K, N, O, W, y)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            hg.hg_out_proj_rs(comm, T, K, N, O, W, y)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        tf = 2.0 * T * K * N / ms / 1e9
        res[f"out_proj_{T}x{K}x{N}"] = {"ms": ms, "tflops": tf, "roofline_frac": tf / peak, "peak": peak}
    comm.close()
    return res


def psm_vs_fcfs(dev, groups=64, per_group=32, batch=128, H=(32, 8, 128), seed=0):
    """NEXT-2 measured: MMLU-like offline backlog (groups of 32 sharing a 1024-token
    prefix) admitted in arrival (FCFS) order vs the PSM prefix tree's DFS
    order (hg_psm_dfs_order); consecutive batches of decodes run through
    hg_hybrid_attention.  Reports unique KV bytes and attention tokens/s."""
    import numpy as np
    import torch
    import paper_2501_14808_b200 as hg
    from synth.configs import BatchSpec, Request
    from synth.layout import make_layout
    rng = np.random.default_rng(seed)
    reqs = []   # (group, cached context, prompt tokens)
    for g in range(groups):
        prefix = list(rng.integers(0, 32000, 1024))
        for _ in range(per_group):
            suf = int(rng.integers(64, 512))
            reqs.append((g, 1024 + suf + int(rng.integers(1, 256)), prefix + list(rng.integers(0, 32000, suf))))
    arrival = list(rng.permutation(len(reqs)))
    tree = hg.PrefixTree()
    for rid in arrival:
        tree.hg_psm_insert(int(rid), reqs[rid][2])
    psm_order, _ = tree.hg_psm_dfs_order()
    tree.close()
    B = 16
    need = max(sum(-(-(reqs[i][1] + 1) // B) for i in order[k:k + batch])
               for order in (arrival, psm_order) for k in range(0, len(reqs), batch))
    N = need + 64
    kc = torch.randn((N, H[1], B, H[2]), device=dev).to(torch.bfloat16)
    vc = torch.randn((N, H[1], B, H[2]), device=dev).to(torch.bfloat16)
    pool = hg.KVPool(kc, vc, N, B, H[1], H[2], dev.index)
    q = torch.randn((batch, H[0], H[2]), device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush = flush_buffer(dev)
    res = {}
    for name, order in (("fcfs", arrival), ("psm", psm_order)):
        tot_ms, tot_tok, uniq = 0.0, 0, 0
        for k in range(0, len(order), batch):
            ids = order[k:k + batch]
            cnt = {}
            for i in ids:
                cnt[reqs[i][0]] = cnt.get(reqs[i][0], 0) + 1
            rr = [Request(reqs[i][1], 1, True, reqs[i][0], 1024, share=cnt[reqs[i][0]] > 1) for i in ids]
            spec = BatchSpec(name, H[0], H[1], H[2], B, 0, rr)
            lay = make_layout(spec, seed=k, num_blocks=N)
            b = hg.Batch(lay.block_table, [r.c for r in rr], [1] * len(rr), None, lay.shared)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            times = []
            for rep in range(3):
                flush_l2(flush)
                hg.hg_hybrid_attention(pool, b, H[0], q, out, None, ws, None, hg.make_opts(events=ev))
                torch.cuda.synchronize()
                st = hg.hg_last_plan_stats(pool)
                first = 0 if st["tc_tiles"] else 2
                last = 5 if st["combine_rows"] else 3
                times.append(ev[first].elapsed_time(ev[last]))
            tot_ms += min(times)
            tot_tok += len(rr)
            uniq += st["kv_bytes_unique"]
        res[name] = {"tokens_per_s": tot_tok / (tot_ms / 1e3), "attention_ms": tot_ms, "kv_bytes_unique": uniq}
    pool.close()
    res["speedup_psm_over_fcfs"] = res["psm"]["tokens_per_s"] / res["fcfs"]["tokens_per_s"]
    res["kv_bytes_saved_frac"] = 1 - res["psm"]["kv_bytes_unique"] / res["fcfs"]["kv_bytes_unique"]
    res["workload"] = f"{groups} groups x {per_group} decodes sharing 1024-token prefixes, batches of {batch}"
    return res


def run_tp(args, spec, rank, world, dev, peaks, peak_kind):
    """KV-head sharded attention on `world` GPUs, all-gather fused via peer windows
    (strong scaling): the same timing rules as N = 1 -- L2 flushed before every
    timed step, per-step CUDA events on the launching stream, the sum of the step
    times on each rank, MAX over ranks."""
    import torch
    import torch.distributed as dist
    import paper_2501_14808_b200 as hg
    from paper_2501_14808_b200.harness import Workload
    from synth.configs import shard_slice
    local = shard_slice(spec, world)
    # each rank's slice is generated as its own (smaller-head) workload; values are synthetic
    wl = Workload(local, device=dev)
    same_gpu = os.environ.get("HG_BENCH_SAME_GPU") == "1"
    # the timed path is the peer window (the epilogues store into every rank's window);
    # the library's NCCL communicator is only its fallback for calls larger than the
    # window, so a failing NCCL bootstrap degrades to a peer-only communicator
    comm_kind = "nccl + peer window"
    try:
        uid = [hg.hg_comm_unique_id() if rank == 0 and not same_gpu else None]
    except Exception:
        uid = [None]
    dist.broadcast_object_list(uid, src=0)
    try:
        comm = hg.Comm(uid[0], rank, world, dev.index)
    except hg.HgError as e:
        print(f"[bench rank {rank}] NCCL communicator unavailable ({e}); peer-window only", file=sys.stderr)
        comm = None
    ok = torch.tensor([1 if comm is not None else 0], device="cpu" if same_gpu else dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if ok.item() == 0 or uid[0] is None:
        if comm is not None:
            comm.close()
        comm = hg.Comm(None, rank, world, dev.index)
        comm_kind = "peer window only"
    # v2: a peer window per rank, mapped by every other rank (CUDA IPC over NVLink);
    # the attention epilogues store straight into all ranks' windows
    handles = [None] * world
    dist.all_gather_object(handles, comm.hg_comm_window_create(spec.T * spec.H_q * spec.d * 2))
    comm.hg_comm_window_open(handles)
    out = comm.window((spec.T, spec.H_q, spec.d))
    ws = torch.empty(hg.hg_hybrid_attention_tp_workspace_size(wl.pool, comm, wl.batch, spec.H_q), dtype=torch.uint8,
                     device=dev)
    stream = torch.cuda.current_stream(dev)
    flush = flush_buffer(dev)

    def step(opts=None):   # the sharded serving step: append of this rank's K/V slice fused with the attention
        hg.hg_hybrid_step_tp(wl.pool, comm, wl.batch, spec.H_q, wl.q, wl.k_new, wl.v_new, out, ws, stream, opts)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    with ClockSampler(dev.index) as clk:
        step_ms, _, _ = timed_loop(step, args.steps, flush, stream, False)
    dist.barrier()
    _, kev, _ = timed_loop(step, args.steps, flush, stream, True)   # per-kernel events (roofline)
    dist.barrier()
    st = hg.hg_last_plan_stats(wl.pool)
    sk_ms = [e[2].elapsed_time(e[3]) for e in kev] if st["splitk_items"] else []
    cdev = "cpu" if same_gpu else dev   # gloo (same-GPU functional test) reduces host tensors
    t = torch.tensor([sum(step_ms)], device=cdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = t.item()
    # per-rank rooflines: this rank's split-K kernel and its whole step
    sk_avg = statistics.mean(sk_ms) if sk_ms else None
    b_sk = alg_bytes_splitk(local, hbm_route=not st["tc_tiles"])
    ach = b_sk / (sk_avg / 1e3) / 1e9 if sk_avg else None
    t_roof_rank = alg_bytes_total(local) / (peaks["hbm_gbs"] * 1e9) * 1e3
    mine = torch.tensor([ach or 0.0, sum(step_ms) / args.steps], device=cdev, dtype=torch.float64)
    allr = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allr, mine)
    # e2e through the public API with host buffers: each rank's pinned q / k_new / v_new
    # slices in; out, the gathered O [T][H_q][d] read back once per job -- rank r copies
    # token rows [r T/N, (r+1) T/N) of it (every head: rows other ranks computed too);
    # slowest rank's wall time
    qh, kh, vh = wl.q.cpu().pin_memory(), wl.k_new.cpu().pin_memory(), wl.v_new.cpu().pin_memory()
    r0, r1 = spec.T * rank // world, spec.T * (rank + 1) // world
    oh = torch.empty(out[r0:r1].shape, dtype=torch.bfloat16).pin_memory()

    def step_host():
        wl.q.copy_(qh, non_blocking=True)
        wl.k_new.copy_(kh, non_blocking=True)
        wl.v_new.copy_(vh, non_blocking=True)
        step()
        oh.copy_(out[r0:r1], non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()

    for _ in range(max(args.warmup, 150)):   # the same count on every rank (peer barriers); see measure_e2e
        step_host()
    dist.barrier()
    e2e_steps = max(args.steps, 50)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_host()
    te = torch.tensor([time.perf_counter() - t0], device=cdev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = te.item() * args.steps / e2e_steps   # per args.steps steps, as below
    if rank == 0:
        ms = total_ms / args.steps
        per_rank = [{"rank": r, "ms_per_step": float(x[1]), "splitk_gbs": float(x[0]),
                     "step_roof_frac": t_roof_rank / float(x[1])} for r, x in enumerate(allr)]
        roofline = {"bound": "hbm", "kernel": "splitk_kernel<128> (per rank)", "achieved": ach,
                    "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": (ach / peaks["hbm_gbs"]) if ach else None,
                    "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, copy)", "traffic": None,
                    "alg_bytes_per_launch": b_sk, "avg_launch_ms": sk_avg,
                    "share_of_step": (sk_avg / ms) if sk_avg else None,
                    "per_rank_step": {"alg_bytes": alg_bytes_total(local), "t_roof_ms": t_roof_rank,
                                      "frac_slowest_rank": t_roof_rank / ms},
                    "ranks": per_rank}
        print(json.dumps({
            "metric": METRIC, "value": spec.T * args.steps / (total_ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded counter-based N(0,1)-scale bf16 Q/K/V; fragmented block tables)",
            "config": config_dict(spec, world),
            "roofline": roofline,
            "plan": st,
            "communicator": comm_kind,
            # the plan's kernels (append + split-K on the HBM route, whose first / last CTA run
            # the entry / exit barriers); the tcgen05 route adds the exit barrier kernel
            "gpu_launches": (st["kernels"] + (1 if st["tc_tiles"] else 0)) * args.steps,
            "e2e": {"value": spec.T * args.steps / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": (qh.numel() + kh.numel() + vh.numel()) * 2 * world,
                    "d2h_bytes_per_step": spec.T * spec.H_q * spec.d * 2, "ms_per_step": e2e_s / args.steps * 1e3,
                    "api": "per rank: pinned H2D of its q / k_new / v_new slices, hg_hybrid_step_tp "
                           "(append fused), D2H of its 1/N token rows of the gathered O; slowest rank"},
            "clocks": clk.summary(),
            **({"note": "HG_BENCH_SAME_GPU functional test: all ranks on one GPU, not a scaling number"}
               if same_gpu else {}),
        }))
    comm.close()
    dist.destroy_process_group()


def run_reference(args):
    """The fp64 CPU oracle timed as the reference arm (rank 0 only)."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from synth.configs import make_config
    spec = make_config(WORKLOAD, 0)
    base = None
    times = []
    for k in range(args.warmup + args.steps):
        # each step: a bounded sample (the prefill request + 4 decodes, rotating)
        dec = [i for i, r in enumerate(spec.requests) if r.n == 1]
        sel = sorted([0] + dec[(4 * k) % len(dec):(4 * k) % len(dec) + 4])
        cb = cpu_baseline(spec, None, sample_reqs=sel, min_s=0.0)
        if k >= args.warmup:
            times.append(spec.T / cb["value"])
            base = cb
    t = sum(times)
    val = spec.T * len(times) / t
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t / len(times) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(spec, world),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": base["cores"], "kind": "oracle",
                         "sample": "per step: the prefill request + 4 rotating decodes; " + base["sample"]},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)   # ~0.1 s timed: enough NVML clock samples
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", dest="extra", action="store_false",
                    help="skip the other configs (c2, c3, p1, p2) reported beside the headline")
    ap.add_argument("--profile", action="store_true", help="timed steps only (no e2e / cpu baseline): for ncu")
    ap.add_argument("--no-predictor", action="store_true", help="skip the C4 sweep + predictor fit")
    ap.add_argument("--sweep-iters", type=int, default=64, help="C4 iterations per (rho, chunk) point")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torch.distributed.run
        port = os.environ.get("MASTER_PORT", "29533")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

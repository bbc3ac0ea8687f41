"""Benchmark of the hot path: the cosine-threshold tensor join.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg1|cfg2|cfg3|cfg4|cfg5] [--theta T] [--sims exact|tensor]

Default workload: BASELINE.json configs[1] (cfg2, fits one B200): |R| =
100,000 x |S| = 1,000,000, d = 100, clustered generator (10,000 centroids,
sigma 0.5, seed 0), theta = 0.8; bf16 tensor-core filter with the provable
band, canonical fp32 recheck.  --config cfg5 (200k x 200k, 500 centroids,
the output-heavy theta sweep: --theta 0.95/0.8/0.6/0.4) and --config cfg3
(200k + 200k strings, FastText-style subword embedding from a 2M x 100 bucket
table, theta 0.85) print the same line for those workloads.

One step (N = 1) = prepare(R) + prepare(S) + fused join -> canonical device
MatchSet (cfg3: subword embed + normalise both relations, then the join).
N > 1: R is sharded over the ranks (strong scaling: total work fixed); each
rank holds its own pieces of S, prepares them once, and the prepared pieces
are all-gathered round by round while every rank filters the rounds that
have landed (multigpu.sharded_join_owned).  With --gpus N > 1 and no
WORLD_SIZE in the environment, bench.py re-launches itself under
torch.distributed.run with N ranks.

Prints ONE JSON line on rank 0.  ``value`` is device-resident throughput
(inputs in HBM), ``e2e`` the same metric through the public API with pinned
host buffers (H2D of the inputs and D2H of the MatchSet inside the timed
region); ``e2e_pageable`` / ``e2e_operator`` time pageable numpy inputs and
the drop-in tensor_join(RawRelation, RawRelation, LookupModel) beside it.
``--impl reference`` runs the UNMODIFIED reference package (baseline/_ref,
compiled backend, all host threads) on the same workload: full joins, one
per step.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "similarity-join pair evals/sec and % of bf16 tensor-core roofline, 1/2/4/8 B200"
UNIT = "pair evals/s"
BUDGET = 64 * 1024 * 1024          # the reference CLI's default budget (cli.py:31)

WORKLOADS = {
    "cfg1": dict(kind="vectors", n_left=10_000, n_right=10_000, dim=100, n_centroids=1_000,
                 sigma=0.5, theta=0.8, seed=0),
    "cfg2": dict(kind="vectors", n_left=100_000, n_right=1_000_000, dim=100,
                 n_centroids=10_000, sigma=0.5, theta=0.8, seed=0),
    "cfg5": dict(kind="vectors", n_left=200_000, n_right=200_000, dim=100, n_centroids=500,
                 sigma=0.5, theta=0.8, seed=0),
    "cfg3": dict(kind="strings", n_left=200_000, n_right=200_000, dim=100,
                 n_buckets=2_000_000, shared=0.3, theta=0.85, seed=0),
    # d = 768 bf16, R sharded over 8 GPUs: each rank joins 1/8 of R against all
    # of S; with fewer ranks the first N eighths run (per-GPU work fixed)
    "cfg4": dict(kind="wide", n_left=1_000_000, n_right=4_000_000, dim=768, n_centroids=50_000,
                 sigma=0.6, zipf=1.1, theta=0.75, seed=0, share=8),
}


def workload(args) -> dict:
    c = dict(WORKLOADS[args.config])
    if args.theta is not None:
        c["theta"] = float(args.theta)
    c["name"] = args.config
    if c["kind"] == "vectors":
        c["desc"] = (f"{args.config}: |R|={c['n_left']:,} x |S|={c['n_right']:,}, d={c['dim']}, "
                     f"theta={c['theta']}, clustered ({c['n_centroids']:,} centroids, sigma "
                     f"{c['sigma']}), seed {c['seed']}")
    elif c["kind"] == "wide":
        c["sims"] = args.sims
        c["desc"] = (f"{args.config}: |R|={c['n_left']:,} x |S|={c['n_right']:,}, d={c['dim']} "
                     f"bf16, theta={c['theta']}, clustered ({c['n_centroids']:,} centroids, "
                     f"sigma {c['sigma']}, Zipf({c['zipf']}) sizes), seed {c['seed']}; R in "
                     f"{c['share']} shares, one per rank (this run: the first N shares); raw bf16 "
                     f"operands, sims={args.sims}")
    else:
        c["desc"] = (f"{args.config}: {c['n_left']:,} x {c['n_right']:,} strings a-z len 3-12, "
                     f"{int(c['shared'] * 100)}% shared with 1-2 edits; subword model "
                     f"(word + char 3-6-grams, FNV-1a mod {c['n_buckets']:,}, table "
                     f"{c['n_buckets']:,}x{c['dim']} ~N(0,1/d)), theta={c['theta']}")
    return c


def make_vectors(c):
    from paper_2312_01476_b200 import datagen
    L, S = datagen.clustered_pair(c["n_left"], c["n_right"], c["dim"], c["n_centroids"],
                                  c["sigma"], c["seed"], zipf=c.get("zipf"))
    if c["kind"] == "wide":                     # cfg4 relations are bf16
        L, S = datagen.round_bf16(L), datagen.round_bf16(S)
    return L, S


def bf16_tensor(x: np.ndarray):
    """A bf16-exact fp32 array as a (host) torch bfloat16 tensor."""
    import torch
    from paper_2312_01476_b200 import datagen
    return torch.from_numpy(datagen.bf16_bits(x).view(np.int16)).view(torch.bfloat16)


def make_strings(c):
    from paper_2312_01476_b200 import datagen
    return datagen.strings(c["n_left"], c["n_right"], c["shared"], seed=c["seed"])


def host_table(c) -> np.ndarray:
    """cfg3 bucket table (host copy; seeded)."""
    from paper_2312_01476_b200 import datagen
    return datagen.bucket_table(c["n_buckets"], c["dim"], seed=c["seed"])


def set_digest(lo, ro, so, sims: bool = True) -> str:
    """Order-independent exact checksum of a match set: sum mod 2^64 of a
    mixed 64-bit hash of (left, right, sim bits).  Rank-local sums add up
    to the whole job's, so both arms (and any rank count) print the same
    digest for the same MatchSet.  sims=False: of the pairs only."""
    total = np.uint64(0)
    with np.errstate(over="ignore"):
        for s in range(0, len(lo), 1 << 24):
            l = np.asarray(lo[s:s + (1 << 24)], dtype=np.uint64)
            r = np.asarray(ro[s:s + (1 << 24)], dtype=np.uint64)
            b = np.asarray(so[s:s + (1 << 24)], dtype=np.float32).view(np.uint32).astype(np.uint64)
            if not sims:
                b = np.zeros_like(b)
            x = (l * np.uint64(0x9E3779B97F4A7C15)) ^ \
                ((r + np.uint64(0x632BE59BD9B4E019)) * np.uint64(0xC2B2AE3D27D4EB4F)) ^ \
                (b * np.uint64(0x165667B19E3779F9))
            x ^= x >> np.uint64(31)
            x *= np.uint64(0xBF58476D1CE4E5B9)
            x ^= x >> np.uint64(29)
            total = total + x.sum(dtype=np.uint64)
    return f"{int(total):016x}"


def _peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return (float(p["bf16_tflops"]), float(p["bf16_tflops_sustained"]),
                float(p.get("hbm_gbs", 0)) or None, "measured")
    except Exception:
        return 1590.0, 1400.0, 6500.0, "fallback"


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML during a region."""

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thr = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        names = {
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.01)

    def __enter__(self):
        if self._nv is not None:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._thr:
            self._thr.join()

    def summary(self):
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# CPU baseline leg of our arm: the reference's own C kernels (oracle/_ref) on a
# bounded sample, and a bitwise comparison of the sampled rows.

def cpu_reference_sample(L, S, theta, budget_s, threads, n_left_full):
    """The reference's kernels (oracle/_ref: _kernelcore.c built from the
    reference sources; orchestration restated from join.py) on the first r
    rows of R x all of S, r sized to ~budget_s.  Fixed per-join costs
    (normalize_rows(S), pack_transpose(S), join.py:337,342) are timed once.
    Returns (pairs/s of the full job, info, sample columns)."""
    sys.path.insert(0, os.path.join(HERE, "oracle"))
    import refkern
    if not refkern.available():
        raise RuntimeError("oracle/_ref not built")
    t0 = time.perf_counter()
    Sn, _ = refkern.normalize_rows(S)
    t_norm_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    packed = refkern.pack_transpose(Sn)
    t_pack = time.perf_counter() - t0
    r_cal = 128
    t0 = time.perf_counter()
    Ln, _ = refkern.normalize_rows(L[:r_cal])
    refkern.tensor_join_normalized(Ln, Sn, theta, threads=threads, packed=packed,
                                   plan_rows=n_left_full)
    t_cal = time.perf_counter() - t0
    rows = int(max(r_cal, min(L.shape[0], r_cal * budget_s / max(t_cal, 1e-6))))
    rows = max(r_cal, rows // 128 * 128)
    t0 = time.perf_counter()
    Ln, _ = refkern.normalize_rows(L[:rows])
    lo, ro, so, _ = refkern.tensor_join_normalized(Ln, Sn, theta, threads=threads, packed=packed,
                                                   plan_rows=n_left_full)
    t_rows = time.perf_counter() - t0
    full_time = t_norm_s + t_pack + t_rows * (n_left_full / rows)
    pairs = n_left_full * S.shape[0]
    return pairs / full_time, {
        "kind": "reference", "variant": refkern.variant(), "cores": threads,
        "sample": f"first {rows} of {n_left_full} R rows x all {S.shape[0]} S rows "
                  f"(reference kernels _kernelcore.c, tile plan of the full job, 64 MiB "
                  f"budget, {threads} threads); full job = normalize(S) {t_norm_s:.2f}s + "
                  f"pack_transpose(S) {t_pack:.2f}s + sample x {n_left_full / rows:.1f}",
        "sample_seconds": round(t_rows, 3), "sample_rows": rows}, (lo, ro, so)


def sample_parity(ref_cols, ours, rows, left_base=0, sims_tol=False):
    """Comparison of the reference sample (left rows < rows of this rank's
    share) with the same rows of our full result: bitwise, or (sims_tol:
    tensor similarities) the same pair set and the largest |sim| gap."""
    lo, ro, so = ours
    k = int(np.searchsorted(lo, np.uint64(left_base + rows), side="left"))
    rl, rr, rs = ref_cols
    rl = rl + np.uint64(left_base)
    same_pairs = len(rl) == k and np.array_equal(rl, lo[:k]) and np.array_equal(rr, ro[:k])
    out = {"sample_rows": rows, "reference_matches": int(len(rl)), "ours_matches": k}
    if sims_tol:
        gap = float(np.abs(rs.astype(np.float64) - so[:k].astype(np.float64)).max()) \
            if same_pairs and k else None
        out.update({"pair_set_equal": bool(same_pairs), "max_sim_gap": gap,
                    "within_1e-5": bool(same_pairs and (gap is None or gap <= 1e-5))})
    else:
        out["bitwise_equal"] = bool(same_pairs and np.array_equal(rs.view(np.uint32),
                                                                  so[:k].view(np.uint32)))
    return out


# ---------------------------------------------------------------------------
# Reference arm: the unmodified reference package, full joins.

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(HERE, "oracle"))
    import simjoin_ref
    c = workload(args)
    thr = host_threads()
    sj = simjoin_ref.load()
    if sj is None:
        print(json.dumps({"impl": "reference", "unavailable": simjoin_ref.error()}), flush=True)
        return
    steps = max(1, min(args.steps, args.ref_steps))
    warmup = min(args.warmup, args.ref_warmup)
    if c["kind"] == "wide":
        # a full cfg4 share is ~5e11 pairs at d = 768 (hours on the CPU):
        # every step times the reference kernels on a bounded row sample of
        # the rank-0 share against all of S
        L, S = make_vectors(c)
        share = max(world, c["share"])
        r0, r1 = 0, c["n_left"] // share
        rows_total = r1 * world
        vals, info, cols = [], None, None
        for i in range(warmup + steps):
            v, info, cols = cpu_reference_sample(L[r0:r1], S, c["theta"], args.ref_step_seconds,
                                                 thr, r1 - r0)
            if i >= warmup:
                vals.append(v)
        value = float(statistics.median(vals))
        pairs = rows_total * c["n_right"]
        lo, ro, so = cols
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": steps, "warmup": warmup, "steps_requested": args.steps,
                "warmup_requested": args.warmup, "ms_per_step": 1e3 * pairs / value,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "fp32", "data": "synthetic (seeded)", "impl": "reference",
                "config": {"workload": c["desc"], "global_batch": pairs},
                "cpu_baseline": dict(info, value=value, unit=UNIT),
                "parity": {"sample_matches": int(len(lo)),
                           "digest": set_digest(lo, ro, so),
                           "pairs_digest": set_digest(lo, ro, so, sims=False)},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    if c["kind"] == "vectors":
        L, S = make_vectors(c)
        ltok = [f"l{i}" for i in range(len(L))]
        rtok = [f"r{i}" for i in range(len(S))]
        table = dict(zip(ltok, L))
        table.update(zip(rtok, S))
        model = sj.LookupModel(table, c["dim"])
        model_desc = "LookupModel over the generated vectors"
    else:
        left, right = make_strings(c)
        import oracle as O
        tab = host_table(c)
        t0 = time.perf_counter()
        EL = O.subword_embed(left, tab)
        ER = O.subword_embed(right, tab)
        t_sub = time.perf_counter() - t0
        ltok, rtok = left, right
        table = dict(zip(ltok, EL))
        table.update(zip(rtok, ER))
        model = sj.LookupModel(table, c["dim"])
        model_desc = (f"LookupModel over subword vectors (the reference has no subword model, "
                      f"SPEC.md:175; oracle/sj_oracle.c embedded both relations in "
                      f"{t_sub:.2f} s, 1 thread)")
    left_r = sj.RawRelation("left", ltok)
    right_r = sj.RawRelation("right", rtok)
    pairs = len(ltok) * len(rtok)
    walls, ms = [], None
    for i in range(warmup + steps):
        ms, st = sj.tensor_join(left_r, right_r, model, c["theta"], BUDGET, threads=thr)
        if i >= warmup:
            walls.append(st.wall_nanos / 1e9)
    t0 = time.perf_counter()
    sj.embed_relation(model, left_r)
    sj.embed_relation(model, right_r)
    t_embed = time.perf_counter() - t0
    wall = statistics.median(walls)
    join_only = max(wall - t_embed, 1e-9)
    value = pairs / join_only
    lo = np.asarray(ms.lefts, dtype=np.uint64)
    ro = np.asarray(ms.rights, dtype=np.uint64)
    so = np.asarray(ms.sims, dtype=np.float32)
    # nlj_prefetch once, for context, on a bounded sample
    m_rows = max(1, min(len(ltok), int(args.nlj_pairs // max(1, len(rtok)))))
    t0 = time.perf_counter()
    _, nst = sj.nlj_prefetch(sj.RawRelation("left", ltok[:m_rows]), right_r, model,
                             c["theta"], threads=thr, inner="right")
    nlj_wall = time.perf_counter() - t0
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": steps, "warmup": warmup, "steps_requested": args.steps,
            "warmup_requested": args.warmup,
            "ms_per_step": 1e3 * join_only, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp32", "data": "synthetic (seeded)",
            "impl": "reference",
            "config": {"workload": c["desc"], "global_batch": pairs},
            "cpu_baseline": {
                "value": value, "unit": UNIT, "cores": thr, "kind": "reference",
                "sample": f"none: every step is one full reference tensor_join "
                          f"({len(ltok):,} x {len(rtok):,}; {model_desc}, budget 64 MiB, "
                          f"threads={thr}, backend {sj.kernels.active_backend()}); value uses "
                          f"the join-only time = JoinStats.wall_nanos - embed_relation(L, S)",
                "full_wall_s": wall, "embed_s": t_embed, "join_only_s": join_only,
                "full_wall_pairs_per_s": pairs / wall,
                "step_walls_s": walls},
            "nlj_prefetch": {"pairs_per_s": m_rows * len(rtok) / nlj_wall,
                             "wall_s": nlj_wall, "sample": f"first {m_rows} left tuples x all "
                                                          f"{len(rtok):,} right",
                             "matches": int(nst.matches)},
            "parity": {"matches": int(len(lo)), "digest": set_digest(lo, ro, so),
                       "pairs_digest": set_digest(lo, ro, so, sims=False)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Our arm.

def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2312_01476_b200 import build
    build.build()
    from paper_2312_01476_b200 import device as D
    from paper_2312_01476_b200 import multigpu as MG

    c = workload(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"rank {rank} needs GPU {local}; {torch.cuda.device_count()} visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def reduce(x: float, op) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max_over_ranks(x):
        return reduce(x, dist.ReduceOp.MAX if world > 1 else None)

    def sum_over_ranks(x):
        return reduce(x, dist.ReduceOp.SUM if world > 1 else None)

    theta, dim = c["theta"], c["dim"]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in ev:
        e.record()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)     # 256 MiB > 126 MB L2
    if c["kind"] == "wide":
        # rank r joins share r of `share` R shares (strong within the share
        # count, i.e. per-GPU work fixed as N grows up to `share`)
        share = max(world, c["share"])
        r0, r1 = MG.shard_range(c["n_left"], rank, share)
        rows_total = sum(MG.shard_range(c["n_left"], k, share)[1] -
                         MG.shard_range(c["n_left"], k, share)[0] for k in range(world))
    else:
        r0, r1 = MG.shard_range(c["n_left"], rank, world)
        rows_total = c["n_left"]
    n_shard, n_right = r1 - r0, c["n_right"]
    pairs_total = rows_total * n_right
    PR_last = {}

    if c["kind"] == "wide":
        L, S = make_vectors(c)
        R_dev = bf16_tensor(L[r0:r1]).to(dev)
        if world == 1:
            S_bf = bf16_tensor(S).to(dev)
        else:
            lay = MG.piece_layout(n_right, world)
            S_loc = bf16_tensor(MG.local_pieces(S, lay, rank)).to(dev)

        def step(events=None):
            Sx = S_bf if world == 1 else MG.gather_right_raw(S_loc, lay)
            PR_last["p"] = None
            PR_last["p"] = pr = D.prepare_bf16(Sx)
            return D.join_prepared(D.prepare_bf16(R_dev), pr, theta, left_base=r0,
                                   filter_events=events, sims=args.sims)
    elif c["kind"] == "vectors":
        L, S = make_vectors(c)
        R_dev = torch.from_numpy(L[r0:r1]).to(dev)
        if world == 1:
            S_dev = torch.from_numpy(S).to(dev)

            def step(events=None):
                return D.join_prepared(D.prepare(R_dev), D.prepare(S_dev), theta,
                                       left_base=r0, filter_events=events)
        else:
            lay = MG.piece_layout(n_right, world)
            S_loc = torch.from_numpy(MG.local_pieces(S, lay, rank)).to(dev)

            def step(events=None):
                m, PR_last["p"] = MG.sharded_join_owned(R_dev, S_loc, lay, theta, r0)
                return m
    else:
        left, right = make_strings(c)
        g = torch.Generator(device=dev).manual_seed(c["seed"])
        table = torch.randn((c["n_buckets"], dim), generator=g, device=dev) * (1.0 / dim ** 0.5)
        Lb, Lo = D.pack_tokens(left[r0:r1], dev)
        Sb, So = D.pack_tokens(right, dev)
        import ctypes
        from paper_2312_01476_b200 import _lib

        def embed(b, o, n):
            f32 = torch.empty((n, dim), dtype=torch.float32, device=dev)
            op = D.op_empty(n, dim, dev)
            rep = torch.zeros(1, dtype=torch.int64, device=dev)
            re, te = D._err_buffers(n, dev)
            _lib.check(_lib.lib().sjb_subword_embed(
                D._vp(b), D._vp(o), n, D._vp(table), table.shape[0], dim, 3, 6, 1, D._vp(f32),
                D._vp(op), D._vp(rep), D._vp(re), D._vp(te), D._stream(dev)), "subword_embed")
            return D.PreparedRelation(f32, op, n, dim, "", rep, re, te)

        def step(events=None):
            return D.join_prepared(embed(Lb, Lo, n_shard), embed(Sb, So, n_right), theta,
                                   left_base=r0, filter_events=events)

    m = None
    for _ in range(args.warmup):
        m = None                           # free the previous result before the next
        m = step()
    torch.cuda.synchronize()
    # cold call: a warm process meets a shape it has no capacity / recheck
    # placement history for (the sampled pre-pass sizes it); wall clock
    # around the whole call
    D._cap_cache.clear()
    m = None
    torch.cuda.synchronize()
    barrier()
    t_cold = time.perf_counter()
    m = step()
    torch.cuda.synchronize()
    cold_ms = max_over_ranks((time.perf_counter() - t_cold) * 1e3)
    cold_retries = int(getattr(m, "retries", 0))
    m = step()                             # warm again: the timed steps below
    torch.cuda.synchronize()
    barrier()

    step_ms, filt_ms = [], []
    launches0 = D.launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)                       # L2 flush between timed steps
            torch.cuda.synchronize()
            barrier()
            m = None
            ev[0].record()
            m = step((ev[2], ev[3]) if world == 1 else None)
            ev[1].record()
            torch.cuda.synchronize()
            step_ms.append(ev[0].elapsed_time(ev[1]))
            if world == 1:
                filt_ms.append(ev[2].elapsed_time(ev[3]))
        barrier()
    launches = D.launch_count() - launches0
    total_ms = max_over_ranks(sum(step_ms))
    ms_per_step = total_ms / args.steps
    value = pairs_total / (ms_per_step / 1e3)
    n_matches = int(sum_over_ranks(m.n_matches))
    n_cand = int(sum_over_ranks(m.n_candidates))
    ours_cols = m.to_host()
    digest_part = int(set_digest(*ours_cols), 16)
    pairs_part = int(set_digest(*ours_cols, sims=False), 16)

    # combine the rank-local digests (sum mod 2^64) without moving match data
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, (digest_part, pairs_part))
        digest = f"{sum(p[0] for p in parts) % (1 << 64):016x}"
        pairs_digest = f"{sum(p[1] for p in parts) % (1 << 64):016x}"
    else:
        digest, pairs_digest = f"{digest_part:016x}", f"{pairs_part:016x}"

    # ---- filter kernel alone (N > 1: the steps filter round by round) ------
    def filter_only_ms():
        if c["kind"] == "wide":
            pl, pr = D.prepare_bf16(R_dev), PR_last["p"]
        elif c["kind"] == "vectors":
            pl = D.prepare(R_dev)
            pr = PR_last["p"] if world > 1 else D.prepare(S_dev)
        else:
            pl, pr = embed(Lb, Lo, n_shard), embed(Sb, So, n_right)
        D.join_prepared(pl, pr, theta, left_base=r0, filter_events=(ev[2], ev[3]),
                        sims=args.sims if c["kind"] == "wide" else "exact")
        torch.cuda.synchronize()
        return ev[2].elapsed_time(ev[3])

    if not filt_ms:
        filt_ms = [filter_only_ms() for _ in range(3)]
    # free the last step's device result and prepared S before the e2e joins
    # (a cfg4 share's result alone is ~40 GB)
    m = None
    PR_last.clear()
    torch.cuda.empty_cache()

    # ---- end to end through the public API with host buffers ----------------
    from paper_2312_01476_b200.join import tensor_join, tensor_join_vectors
    from paper_2312_01476_b200.core import RawRelation
    e2e_extra = {}
    if c["kind"] == "wide":
        L_pin = bf16_tensor(L[r0:r1]).pin_memory()
        if world == 1:
            S_pin = bf16_tensor(S).pin_memory()
        else:
            S_pin = bf16_tensor(MG.local_pieces(S, lay, rank)).pin_memory()
        h2d = L_pin.numel() * 2 + S_pin.numel() * 2

        def e2e_step():
            if world == 1:
                ms, _ = tensor_join_vectors(L_pin, S_pin, theta, device=dev, sims=args.sims)
                return len(ms)
            Rd = L_pin.to(dev, non_blocking=True)
            Sd = MG.gather_right_raw(S_pin.to(dev, non_blocking=True), lay)
            mm = D.join_prepared(D.prepare_bf16(Rd), D.prepare_bf16(Sd), theta, left_base=r0,
                                 sims=args.sims)
            return len(mm.to_host()[0])
    elif c["kind"] == "vectors":
        L_pin = torch.from_numpy(L[r0:r1]).pin_memory()
        if world == 1:
            S_pin = torch.from_numpy(S).pin_memory()
            h2d = L_pin.numel() * 4 + S_pin.numel() * 4

            def e2e_step():
                ms, _ = tensor_join_vectors(L_pin, S_pin, theta, device=dev)
                return len(ms)
        else:
            S_loc_pin = torch.from_numpy(MG.local_pieces(S, lay, rank)).pin_memory()
            h2d = L_pin.numel() * 4 + S_loc_pin.numel() * 4

            def e2e_step():
                Rd = L_pin.to(dev, non_blocking=True)
                Sd = S_loc_pin.to(dev, non_blocking=True)
                mm, _ = MG.sharded_join_owned(Rd, Sd, lay, theta, r0)
                lo, ro, so = mm.to_host()            # rank-local result, pinned host
                return len(lo)
    else:
        model = None
        from paper_2312_01476_b200.embedding import SubwordModel
        model = SubwordModel(table)
        Lrel = RawRelation("left", left[r0:r1])
        Rrel = RawRelation("right", right)
        h2d = sum(len(s) for s in left[r0:r1]) + sum(len(s) for s in right) + \
            8 * (n_shard + n_right + 2)

        def e2e_step():
            ms, _ = tensor_join(Lrel, Rrel, model, theta, BUDGET, device=dev)
            return len(ms)

    def timed(fn, reps):
        for _ in range(min(2, args.warmup)):
            fn()
        torch.cuda.synchronize()
        barrier()
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            k = fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return max_over_ranks(statistics.median(ts)), k

    e2e_steps = max(1, min(args.steps, 5))
    e2e_time, k = timed(e2e_step, e2e_steps)
    h2d = int(sum_over_ranks(h2d))
    d2h = int(sum_over_ranks(k * 20))

    if world == 1 and c["kind"] == "vectors" and not args.no_extra_e2e:
        # pageable numpy inputs (what reference callers hold)
        t_pg, _ = timed(lambda: len(tensor_join_vectors(L, S, theta, device=dev)[0]), 3)
        e2e_extra["e2e_pageable"] = {"value": pairs_total / t_pg, "unit": UNIT,
                                     "seconds_per_step": t_pg,
                                     "inputs": "pageable numpy (tensor_join_vectors)"}
        # the drop-in operator: tensor_join(RawRelation, RawRelation, LookupModel)
        from paper_2312_01476_b200.embedding import LookupModel
        ltok = [f"l{i}" for i in range(len(L))]
        rtok = [f"r{i}" for i in range(len(S))]
        lm = LookupModel.from_matrix(ltok + rtok, np.concatenate([L, S]))
        Lr, Rr = RawRelation("left", ltok), RawRelation("right", rtok)
        t_op, _ = timed(lambda: len(tensor_join(Lr, Rr, lm, theta, BUDGET, device=dev)[0]), 3)
        e2e_extra["e2e_operator"] = {
            "value": pairs_total / t_op, "unit": UNIT, "seconds_per_step": t_op,
            "inputs": "tensor_join(RawRelation, RawRelation, LookupModel) with 1.1M string "
                      "tokens (token -> row lookup on the host, table resident on the device)"}

    # ---- roofline of the dominant kernel (the fused filter) -----------------
    burst, sustained, hbm, src = _peaks()
    filt_avg = statistics.mean(filt_ms) / 1e3
    flops = 2.0 * n_shard * n_right * dim                 # algorithmic, unpadded d
    achieved = flops / filt_avg / 1e12
    long_run = sum(step_ms) / 1e3 > 1.0
    peak = sustained if long_run else burst
    traffic = None
    tpath = os.path.join(HERE, "profiles", f"filter_traffic_{c['name']}.json")
    if not os.path.exists(tpath) and c["name"] == "cfg2":
        tpath = os.path.join(HERE, "profiles", "filter_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")

    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            if c["kind"] in ("vectors", "wide"):
                Lc, Sc = L[r0:r1], S
                emb = None
            else:
                sys.path.insert(0, os.path.join(HERE, "oracle"))
                import oracle as O
                tab = table.cpu().numpy()
                t0 = time.perf_counter()
                Lc = O.subword_embed(left, tab)
                t_l = time.perf_counter() - t0
                Sc = O.subword_embed(right, tab)
                emb = {"kind": "port", "cores": 1, "seconds": time.perf_counter() - t0,
                       "strings_per_s": (len(left) + len(right)) /
                       (time.perf_counter() - t0),
                       "what": "oracle/sj_oracle.c subword embedding of both relations "
                               f"(left {t_l:.2f} s)"}
            v, info, ref_cols = cpu_reference_sample(Lc, Sc, theta, args.cpu_seconds,
                                                     host_threads(), len(Lc))
            cpu = dict(info, value=v, unit=UNIT)
            if emb:
                cpu["embedding"] = emb
            parity = sample_parity(ref_cols, ours_cols, info["sample_rows"], left_base=r0,
                                   sims_tol=c["kind"] == "wide" and args.sims == "tensor")
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "error": f"{type(exc).__name__}: {exc}"}
    if parity is None:
        parity = {}
    parity.update({"matches": n_matches, "digest": digest, "pairs_digest": pairs_digest})

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16+fp32", "data": "synthetic (seeded generator)",
            "config": {"workload": c["desc"], "global_batch": pairs_total,
                       "parallelism": f"R-shard x{world}" + (
                           ", S owner-prepared + all-gathered per round" if world > 1 else ""),
                       "band": D.raw_band(dim) if c["kind"] == "wide" else D.default_band(dim),
                       "l2": "flushed (256 MiB write) between "
                                                         "timed steps",
                       "matches": n_matches, "candidates": n_cand,
                       "output_pairs_per_s": n_matches / (ms_per_step / 1e3),
                       "cold_first_call_ms": cold_ms, "cold_first_call_retries": cold_retries,
                       "launches_per_step": launches / args.steps},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                         "kernel": "join_filter_kernel", "filter_ms": filt_avg * 1e3,
                         "filter_share_of_step": filt_avg * 1e3 / ms_per_step,
                         "peak_source": f"{src} {'sustained' if long_run else 'burst'}",
                         "frac_burst": achieved / burst,
                         "k_pad_cap": dim / D.kpad(dim)},
            "e2e": {"value": pairs_total / e2e_time, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "seconds_per_step": e2e_time,
                    "inputs": {"vectors": "pinned host",
                               "wide": "pinned host bf16 rows (tensor_join_vectors), MatchSet "
                                       "columns copied back per left-row part"}.get(
                        c["kind"], "host strings through tensor_join(RawRelation, "
                                   "SubwordModel)")},
            **e2e_extra,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch(args) -> int:
    """--gpus N > 1 without a torchrun environment: run this script under
    torch.distributed.run with N ranks (one per GPU, NCCL), NCCL's
    communicator log on so the rank count is visible."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_MAX_CTAS", "16")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="cfg2",
                    help="cfg1 is the reference's own CPU-sized case (parity, launch tests)")
    ap.add_argument("--theta", type=float, default=None)
    ap.add_argument("--sims", choices=["exact", "tensor"], default="exact",
                    help="cfg4: canonical similarities (bitwise) or the epilogue's "
                         "(within 1e-5; pair set exact)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-steps", type=int, default=2,
                    help="reference arm: full joins timed (each is a whole 1e11-pair join)")
    ap.add_argument("--ref-warmup", type=int, default=1)
    ap.add_argument("--ref-step-seconds", type=float, default=20.0,
                    help="reference arm, cfg4: CPU seconds per sampled step")
    ap.add_argument("--nlj-pairs", type=float, default=2e9,
                    help="reference arm: pairs in the one nlj_prefetch sample")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch(args))
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_MAX_CTAS", "16")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

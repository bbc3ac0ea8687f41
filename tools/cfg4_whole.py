"""The WHOLE BASELINE cfg4 job (|R| = 1M x |S| = 4M, d = 768 bf16, theta 0.75:
4e12 pairs) on one GPU, as the 8 rank shares of the multi-GPU design run one
after the other: S is prepared once (what every rank does with the gathered
raw bf16 pieces), then each share's R rows are prepared and joined.  Prints
per share: device time (CUDA events), matches, candidates and the
order-independent digest of the share's MatchSet (bench.set_digest's formula
evaluated on the device), and the job totals -- the sum of the digests is the
digest an 8-rank run prints.  Share 0 is the bench line's workload
(`bench.py --config cfg4`), so its count and digest must equal that line's.
Usage: python tools/cfg4_whole.py [tensor|exact] [shares=8]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2312_01476_b200 import build  # noqa: E402
build.build()
from paper_2312_01476_b200 import device as D  # noqa: E402
from paper_2312_01476_b200 import multigpu as MG  # noqa: E402

M64 = (1 << 64) - 1


def _i64(x: int) -> int:
    x &= M64
    return x - (1 << 64) if x >> 63 else x


def _lsr(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical shift right of int64 bit patterns."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def device_digest(lo: torch.Tensor, ro: torch.Tensor, so: torch.Tensor, sims: bool = True) -> int:
    """bench.set_digest on the device: int64 arithmetic wraps mod 2^64 like uint64."""
    total = 0
    step = 1 << 26
    for s in range(0, lo.numel(), step):
        l, r = lo[s:s + step], ro[s:s + step]
        b = so[s:s + step].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        if not sims:
            b = torch.zeros_like(b)
        x = (l * _i64(0x9E3779B97F4A7C15)) ^ ((r + _i64(0x632BE59BD9B4E019)) * _i64(0xC2B2AE3D27D4EB4F)) \
            ^ (b * _i64(0x165667B19E3779F9))
        x = x ^ _lsr(x, 31)
        x = x * _i64(0xBF58476D1CE4E5B9)
        x = x ^ _lsr(x, 29)
        total = (total + int(x.sum().item())) & M64   # torch's int64 sum wraps too
    return total


def main() -> None:
    sims = sys.argv[1] if len(sys.argv) > 1 else "tensor"
    shares = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    c = dict(bench.WORKLOADS["cfg4"], name="cfg4")
    dev = torch.device("cuda", 0)
    t0 = time.perf_counter()
    L, S = bench.make_vectors(c)
    print(f"generated {L.shape} x {S.shape} in {time.perf_counter() - t0:.0f} s", flush=True)
    theta = c["theta"]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    S_dev = bench.bf16_tensor(S).to(dev)
    torch.cuda.synchronize()
    ev[0].record()
    pr = D.prepare_bf16(S_dev)
    ev[1].record()
    torch.cuda.synchronize()
    prep_s_ms = ev[0].elapsed_time(ev[1])
    del S, S_dev
    tot_ms = tot_matches = tot_cand = 0
    dig = pdig = 0
    for k in range(shares):
        r0, r1 = MG.shard_range(c["n_left"], k, c["share"])
        Rk = bench.bf16_tensor(L[r0:r1]).to(dev)
        torch.cuda.synchronize()
        ev[0].record()
        pl = D.prepare_bf16(Rk)
        m = D.join_prepared(pl, pr, theta, sims=sims, left_base=r0)
        ev[1].record()
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1])
        d = device_digest(m.lefts, m.rights, m.sims)
        pd = device_digest(m.lefts, m.rights, m.sims, sims=False)
        print(f"share {k}: R rows [{r0}, {r1}): {ms:.1f} ms, matches {m.n_matches}, candidates "
              f"{m.n_candidates}, retries {m.retries}, digest {d:016x}, pairs_digest {pd:016x}", flush=True)
        tot_ms += ms
        tot_matches += m.n_matches
        tot_cand += m.n_candidates
        dig = (dig + d) & M64
        pdig = (pdig + pd) & M64
        del m, pl, Rk
        torch.cuda.empty_cache()
    pairs = float(MG.shard_range(c["n_left"], shares - 1, c["share"])[1]) * c["n_right"]
    print(f"whole job ({shares} of {c['share']} shares, sims={sims}): {tot_ms / 1e3:.2f} s of joins + "
          f"{prep_s_ms:.0f} ms preparing S once; {pairs:.3g} pairs -> {pairs / (tot_ms / 1e3):.3e} pair "
          f"evals/s on one GPU; matches {tot_matches}, candidates {tot_cand}, digest {dig:016x}, "
          f"pairs_digest {pdig:016x}", flush=True)


if __name__ == "__main__":
    main()

"""Swap kernel sweep on one GPU: variant x CTAs, D2H and H2D GB/s for a 1 GiB batch of 64
tensors (and a mixed-size batch), against per-tensor cudaMemcpyAsync on the copy engines.
Byte-exactness of every variant is checked on the first run.  Writes gpurun_out/swap_sweep.json."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import chm  # noqa: E402


def run(ctx, descs, flags, reps=3):
    comp, sw = torch.cuda.current_stream(), torch.cuda.Stream()
    out, inn = [], []
    for _ in range(reps + 1):
        b = ctx.swap_out(descs, comp, sw, flags)
        ctx.batch_wait(b, comp)
        b2 = ctx.swap_in(descs, comp, sw, flags)
        ctx.batch_wait(b2, comp)
        torch.cuda.synchronize()
        out.append(ctx.batch_elapsed_ms(b))
        inn.append(ctx.batch_elapsed_ms(b2))
    nbytes = sum(d[2] for d in descs)
    return nbytes / (np.median(out[1:]) * 1e-3) / 1e9, nbytes / (np.median(inn[1:]) * 1e-3) / 1e9


def main():
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(0)
    nb = 16 << 20
    bufs = [torch.randint(0, 256, (nb,), dtype=torch.uint8, device=dev, generator=g) for _ in range(64)]
    ref = [b.clone() for b in bufs]
    descs = [(b.data_ptr(), j * nb, nb) for j, b in enumerate(bufs)]
    rng = np.random.default_rng(1)
    mixed_sizes = [int(512 * max(1, int(2 ** rng.uniform(3, 15)))) for _ in range(200)]
    mbufs = [torch.empty(s, dtype=torch.uint8, device=dev) for s in mixed_sizes]
    mdescs, off = [], 0
    for b in mbufs:
        mdescs.append((b.data_ptr(), off, b.numel()))
        off += b.numel()
    results = []
    for variant in (0, 1, 2):
        for ctas in ((2, 4, 8, 16, 32, 148) if "--quick" not in sys.argv else (16,)):
            ctx = chm.Context(device=0, host_arena_bytes=2 << 30, swap_ctas=ctas, time_batches=True,
                              swap_variant=variant)
            if ctas == 16:  # byte-exact check of this variant
                for b in bufs:
                    b.zero_()
                comp, sw = torch.cuda.current_stream(), torch.cuda.Stream()
                for b, r in zip(bufs, ref):
                    b.copy_(r)
                ctx.batch_wait(ctx.swap_out(descs, comp, sw), comp)
                for b in bufs:
                    b.zero_()
                ctx.batch_wait(ctx.swap_in(descs, comp, sw), comp)
                torch.cuda.synchronize()
                ok = all(torch.equal(b, r) for b, r in zip(bufs, ref))
            else:
                ok = None
            d2h, h2d = run(ctx, descs, chm.SWAP_KERNEL)
            md2h, mh2d = run(ctx, mdescs, chm.SWAP_KERNEL)
            results.append(dict(variant=variant, ctas=ctas, d2h=d2h, h2d=h2d, mixed_d2h=md2h, mixed_h2d=mh2d,
                                exact=ok))
            print(f"variant {variant} ctas {ctas:3d}: 1GiB d2h {d2h:5.1f} h2d {h2d:5.1f} | mixed d2h {md2h:5.1f} "
                  f"h2d {mh2d:5.1f} | exact {ok}", flush=True)
            ctx.close()
    ctx = chm.Context(device=0, host_arena_bytes=2 << 30, time_batches=True)
    curve = []
    for sz in (64 << 10, 256 << 10, 1 << 20, 2 << 20, 4 << 20, 8 << 20, 16 << 20, 64 << 20):
        cnt = max(1, min(256, (512 << 20) // sz))
        sb = [torch.empty(sz, dtype=torch.uint8, device=dev) for _ in range(cnt)]
        sd = [(b.data_ptr(), j * sz, sz) for j, b in enumerate(sb)]
        k = run(ctx, sd, chm.SWAP_KERNEL)
        e = run(ctx, sd, chm.SWAP_CE)
        curve.append(dict(size=sz, count=cnt, kernel_d2h=k[0], kernel_h2d=k[1], ce_d2h=e[0], ce_h2d=e[1]))
        print(f"size {sz >> 10:6d} KiB x {cnt:3d}: kernel d2h {k[0]:5.1f} h2d {k[1]:5.1f} | ce d2h {e[0]:5.1f} h2d {e[1]:5.1f}",
              flush=True)
        del sb
    ce = run(ctx, descs, chm.SWAP_CE)
    mce = run(ctx, mdescs, chm.SWAP_CE)
    print(f"copy engines: 1GiB d2h {ce[0]:5.1f} h2d {ce[1]:5.1f} | mixed d2h {mce[0]:5.1f} h2d {mce[1]:5.1f}")
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(dict(kernel=results, size_curve=curve, ce=dict(d2h=ce[0], h2d=ce[1], mixed_d2h=mce[0], mixed_h2d=mce[1]),
                   mixed_bytes=sum(mixed_sizes)), open("gpurun_out/swap_sweep.json", "w"), indent=1)


if __name__ == "__main__":
    main()

"""GPU policy execution: byte-exact swap round trips through the C-ABI (kernel and copy-engine
paths), descriptor validation, stream-ordering hazard test with a sabotage control, and an
executor replay of an installed policy on real device buffers."""
import ctypes

import numpy as np
import pytest

import oracle as O
from workloads import traces as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_11076_b200 import chm  # noqa: E402

ARENA = 512 << 20


@pytest.fixture(scope="module")
def ctx():
    c = chm.Context(device=0, host_arena_bytes=ARENA, swap_ctas=16)
    yield c
    c.close()


def arena_view(ctx):
    base, n = ctx.host_arena()
    return np.ctypeslib.as_array((ctypes.c_uint8 * n).from_address(base))


def rand_bytes(n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda", generator=g)


@pytest.mark.parametrize("flags", [chm.SWAP_KERNEL, chm.SWAP_CE, chm.SWAP_AUTO])
def test_round_trip_sizes_and_alignments(ctx, flags):
    sizes = [1, 15, 16, 17, 511, 4096, 65535, 65536, 65537, (4 << 20) + 3, (33 << 20) + 7]
    dev_offs = [0, 1, 16, 3, 0, 8, 0, 5, 16, 0, 2]
    host_offs = []
    off = 0
    bufs, descs, srcs = [], [], []
    for j, (n, do) in enumerate(zip(sizes, dev_offs)):
        b = rand_bytes(n + 32, 100 + j)
        bufs.append(b)
        src = b[do:do + n]
        srcs.append(src)
        ho = off + (j % 3)  # some host offsets misaligned
        host_offs.append(ho)
        descs.append((src.data_ptr(), ho, n))
        off = ho + n + 64
    s = torch.cuda.Stream()
    comp = torch.cuda.current_stream()
    b_out = ctx.swap_out(descs, comp, s, flags)
    ctx.batch_wait(b_out, comp)
    torch.cuda.synchronize()
    host = arena_view(ctx)
    for src, ho in zip(srcs, host_offs):
        assert np.array_equal(host[ho:ho + src.numel()], src.cpu().numpy())
    # the whole written arena range against the oracle's swap definition (memcpy per descriptor)
    exp = np.zeros(off, np.uint8)
    exp[:] = host[:off]  # bytes between descriptors are not written by either side
    src_host = [src.cpu().numpy() for src in srcs]
    O.swap_execute([exp.ctypes.data + ho for ho in host_offs], [a.ctypes.data for a in src_host], sizes)
    assert np.array_equal(host[:off], exp)
    dst = [torch.zeros(n + 32, dtype=torch.uint8, device="cuda") for n in sizes]
    in_descs = [(d[do:do + n].data_ptr(), ho, n) for d, n, do, ho in zip(dst, sizes, dev_offs, host_offs)]
    b_in = ctx.swap_in(in_descs, comp, s, flags)
    ctx.batch_wait(b_in, comp)
    torch.cuda.synchronize()
    assert ctx.batch_query(b_in)
    for d, src, n, do in zip(dst, srcs, sizes, dev_offs):
        assert torch.equal(d[do:do + n], src)
        assert int(d[:do].sum()) == 0 and int(d[do + n:].sum()) == 0  # nothing outside the block


def test_many_descriptors_multi_launch(ctx):
    n = 150  # > 64 descriptors per launch
    bufs = [rand_bytes(4096 + 512 * (j % 7), j) for j in range(n)]
    descs, off = [], 0
    for b in bufs:
        descs.append((b.data_ptr(), off, b.numel()))
        off += b.numel()
    comp = torch.cuda.current_stream()
    s = torch.cuda.Stream()
    ctx.batch_wait(ctx.swap_out(descs, comp, s), comp)
    torch.cuda.synchronize()
    host = arena_view(ctx)
    for (p, o, nb), b in zip(descs, bufs):
        assert np.array_equal(host[o:o + nb], b.cpu().numpy())
    out = [torch.empty_like(b) for b in bufs]
    ctx.batch_wait(ctx.swap_in([(o_.data_ptr(), d[1], d[2]) for o_, d in zip(out, descs)], comp, s), comp)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(out, bufs))
    # conservation: bytes out == bytes in
    assert sum(d[2] for d in descs) == sum(o_.numel() for o_ in out)


def test_validation_errors(ctx):
    b = rand_bytes(1024, 1)
    comp = torch.cuda.current_stream()
    bad = [
        [(b.data_ptr(), 0, 0)],                      # nbytes == 0
        [(0, 0, 16)],                                # dev == 0
        [(b.data_ptr(), ARENA - 8, 16)],             # past the arena
        [(b.data_ptr(), 0, 512), (b.data_ptr(), 256, 512)],  # overlapping host ranges
    ]
    for j, descs in enumerate(bad):
        with pytest.raises(chm.ChmError) as e:
            ctx.swap_out(descs, comp, comp)
        assert e.value.code == chm.CHM_E_INVAL
        assert e.value.index == (1 if j == 3 else 0)


@pytest.mark.parametrize("direction", ["out", "in"])
def test_misalignment_matrix(ctx, direction):
    """every (device, host) misalignment pair mod 16 through the kernel: same misalignment takes
    the shifted vector body, different misalignment the funnel-shift body; sizes span a head, a
    tail and more than one 64 KiB chunk.  Byte-exact against the oracle's swap definition."""
    comp = torch.cuda.current_stream()
    s = torch.cuda.Stream()
    host = arena_view(ctx)
    size_cycle = [1, 17, 4095, 65536 + 33, 3 * 65536 + 5, 200_003]
    for dev_mis in range(16):
        descs, srcs, dsts, off = [], [], [], 0
        for host_mis in range(16):
            n = size_cycle[(dev_mis + host_mis) % len(size_cycle)]
            base = rand_bytes(n + 64, 1000 + 16 * dev_mis + host_mis)
            ho = off + host_mis
            off = (ho + n + 64 + 15) // 16 * 16
            if direction == "out":
                src = base[dev_mis:dev_mis + n]
                descs.append((src.data_ptr(), ho, n))
                srcs.append(src)
            else:
                host[ho:ho + n] = base[:n].cpu().numpy()
                d = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
                descs.append((d[dev_mis:dev_mis + n].data_ptr(), ho, n))
                srcs.append(base[:n])
                dsts.append((d, dev_mis, n))
        if direction == "out":
            ctx.batch_wait(ctx.swap_out(descs, comp, s, chm.SWAP_KERNEL), comp)
            torch.cuda.synchronize()
            exp = np.zeros(off, np.uint8)
            exp[:] = host[:off]
            src_host = [x.cpu().numpy() for x in srcs]
            O.swap_execute([exp.ctypes.data + d[1] for d in descs], [a.ctypes.data for a in src_host],
                           [d[2] for d in descs])
            for (p_, ho, n), a in zip(descs, src_host):
                assert np.array_equal(host[ho:ho + n], a), (dev_mis, ho % 16, n)
            assert np.array_equal(host[:off], exp)
        else:
            ctx.batch_wait(ctx.swap_in(descs, comp, s, chm.SWAP_KERNEL), comp)
            torch.cuda.synchronize()
            for (d, do, n), src in zip(dsts, srcs):
                assert torch.equal(d[do:do + n], src), (dev_mis, n)
                assert int(d[:do].sum()) == 0 and int(d[do + n:].sum()) == 0


@pytest.mark.parametrize("sabotage", [False, True])
def test_swap_in_hazard(ctx, sabotage):
    """The wait before b_t (a swapped-in tensor must be on the device before its first
    backward use): the compute stream reads the destination right after the swap-in is issued.
    With the wait it reads the swapped-in bytes; sabotage (no wait) must be caught reading stale
    ones on a 256 MiB block."""
    n = 256 << 20
    src = rand_bytes(n, 91)
    comp = torch.cuda.current_stream()
    s = torch.cuda.Stream()
    ctx.batch_wait(ctx.swap_out([(src.data_ptr(), 0, n)], comp, s), comp)
    dst = torch.full((n,), 0x5A, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    b = ctx.swap_in([(dst.data_ptr(), 0, n)], comp, s)
    if not sabotage:
        ctx.batch_wait(b, comp)  # the executor's wait before b_t
    seen = dst.clone()  # the first use, on the compute stream
    torch.cuda.synchronize()
    fresh = torch.equal(seen, src)
    if sabotage:
        assert not fresh and int((seen == 0x5A).sum()) > 0, "sabotage run read fresh bytes: test is not sensitive"
    else:
        assert fresh


@pytest.mark.parametrize("sabotage", [False, True])
def test_release_hazard(ctx, sabotage):
    """Custom recordStream: after the stream-ordered release the compute stream reuses the
    block; the host copy must be intact.  Sabotage (no wait) must be detected on a big block."""
    n = 256 << 20
    src = rand_bytes(n, 77)
    ref = src.cpu().numpy()
    comp = torch.cuda.current_stream()
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    b = ctx.swap_out([(src.data_ptr(), 0, n)], comp, s)
    if not sabotage:
        ctx.batch_wait(b, comp)  # release: compute waits for the swap-out batch, no host sync
    src.fill_(0xAB)  # the reclaimed block is overwritten by the next compute op
    torch.cuda.synchronize()
    host = arena_view(ctx)[:n]
    intact = np.array_equal(host, ref)
    if sabotage:
        assert not intact, "sabotage run did not corrupt: hazard test is not sensitive"
    else:
        assert intact


def test_executor_swaps_real_buffers(ctx):
    """Drive the executor's issue calls with real storage: swap-out after a_t, stream-ordered
    release, swap-in into fresh blocks, wait before b_t; data must round-trip byte-exact."""
    tr = W.tiny()
    ctx.set_detailed(True)
    chm.record_iteration(ctx, tr)
    ctx.detect_seq_change(tr.t_iter)
    ctx.set_detailed(False)
    pt = ctx.trace_build(tr.budget, tr.static_bytes, tr.bw, tr.groups_fwd, tr.groups_bwd, t_iter=tr.t_iter)
    words = pt.candidate_mask(chm.EXHAUSTIVE, (1 << pt.K) - 1)  # swap every swappable tensor
    ctx.policy_install(pt, words)
    # real storage: device tensors whose data_ptr becomes the op records' ids
    storage = {t: rand_bytes(int(tr.nbytes[t]), 5000 + t) for t in range(tr.n_produced)}
    ref = {t: storage[t].clone() for t in storage}
    by_ptr_static = {}
    comp = torch.cuda.current_stream()
    s_out, s_in = torch.cuda.Stream(), torch.cuda.Stream()
    item_tensor = {}
    tok = [ctx.tokenize(nm) for nm in tr.op_names]

    def ref_of(t):
        if t < tr.n_produced:
            return (storage[t].data_ptr(), int(tr.nbytes[t]), int(tr.dtype[t]))
        if t not in by_ptr_static:
            by_ptr_static[t] = torch.empty(int(tr.nbytes[t]), dtype=torch.uint8, device="cuda")
        return (by_ptr_static[t].data_ptr(), int(tr.nbytes[t]), int(tr.dtype[t]))

    n_out = n_in = 0
    for i in range(tr.n_ops):
        ins = [ref_of(t) for t in tr.ins(i)]
        outs = [ref_of(t) for t in tr.outs(i)]
        freed = [ref_of(t)[0] for t in tr.frees(i)]
        act = ctx.record_op(tok[i], int(tr.phase[i]), ins, outs, freed)
        av = chm.actions_view(act)
        if av["swap_out"]:
            for (dev, off, nb), it in zip(av["swap_out"], av["swap_out_item"]):
                item_tensor[it] = next(t for t in storage if storage[t] is not None and storage[t].data_ptr() == dev)
            ctx.issue_swap_out(comp, s_out)
            n_out += len(av["swap_out"])
        for it in av["release"]:
            ctx.item_wait(it, False, comp)
            t = item_tensor[it]
            storage[t].fill_(0xEE)  # reclaimed block reused by compute after the wait
            storage[t] = None
        if av["swap_in"]:
            dev = []
            for (d, off, nb), it in zip(av["swap_in"], av["swap_in_item"]):
                t = item_tensor[it]
                storage[t] = torch.empty(int(nb), dtype=torch.uint8, device="cuda")
                dev.append(storage[t].data_ptr())
            ctx.issue_swap_in(dev, comp, s_in)
            n_in += len(av["swap_in"])
        for it in av["wait"]:
            ctx.item_wait(it, True, comp)
            t = item_tensor[it]
            assert torch.equal(storage[t], ref[t])  # after the wait, before op b_t reads it
    ctx.detect_seq_change(tr.t_iter)
    st = ctx.exec_stats()
    assert n_out == n_in == pt.K == st["n_matched"]
    assert st["bytes_out"] == st["bytes_in"] == int(sum(tr.nbytes[t] for t in item_tensor.values()))


@pytest.mark.parametrize("variant", [1, 2])
def test_round_trip_kernel_variants(variant):
    """L2::256B-prefetch and TMA bulk-copy variants: byte-exact, incl. a misaligned descriptor
    (the bulk variant falls back to the 16 B path for a batch that is not 16 B aligned)."""
    c = chm.Context(device=0, host_arena_bytes=64 << 20, swap_ctas=8, swap_variant=variant)
    comp, s = torch.cuda.current_stream(), torch.cuda.Stream()
    for sizes, offs in (([1 << 20, 3 << 20, 48 << 10], [0, 0, 0]), ([1 << 20, (3 << 20) + 5], [0, 3])):
        bufs = [rand_bytes(n + 16, 7 + j) for j, n in enumerate(sizes)]
        src = [b[o:o + n] for b, n, o in zip(bufs, sizes, offs)]
        descs, off = [], 0
        for x in src:
            descs.append((x.data_ptr(), off, x.numel()))
            off += (x.numel() + 511) // 512 * 512
        c.batch_wait(c.swap_out(descs, comp, s), comp)
        dst = [torch.zeros_like(x) for x in src]
        c.batch_wait(c.swap_in([(d.data_ptr(), o, n) for d, (_, o, n) in zip(dst, descs)], comp, s), comp)
        torch.cuda.synchronize()
        assert all(torch.equal(a, b) for a, b in zip(dst, src))
    c.close()


@pytest.mark.parametrize("flags", [chm.SWAP_KERNEL, chm.SWAP_CE])
def test_config_sized_tensor_round_trip(flags):
    """the largest activation of the configs (C3: [18, 4096, 11008] bf16 = 1.51 GiB), plus 7 bytes
    so the tail is not a multiple of 16, out and back byte-exact; the arena holds the same bytes"""
    n = 18 * 4096 * 11008 * 2 + 7
    c = chm.Context(device=0, host_arena_bytes=n + 4096)
    src = rand_bytes(n, 7)
    comp, s = torch.cuda.current_stream(), torch.cuda.Stream()
    c.batch_wait(c.swap_out([(src.data_ptr(), 0, n)], comp, s, flags), comp)
    torch.cuda.synchronize()
    host = arena_view(c)
    assert np.array_equal(host[:n], src.cpu().numpy())
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda")
    c.batch_wait(c.swap_in([(dst.data_ptr(), 0, n)], comp, s, flags), comp)
    torch.cuda.synchronize()
    assert torch.equal(dst, src)
    c.close()


@pytest.mark.parametrize("mode,numa", [(chm.ARENA_HOSTALLOC, -1), (chm.ARENA_REGISTER, -1), (chm.ARENA_REGISTER, -2),
                                       (chm.ARENA_REGISTER, 0)])
def test_arena_modes_round_trip(mode, numa):
    """both arena allocations (cudaHostAlloc; mmap + mbind + THP + pre-fault + cudaHostRegister) are
    UVA-mapped and swap byte-exact on the kernel and copy-engine paths, also after a regrow;
    placement reports the binding (node 0 is online on every host)"""
    c = chm.Context(device=0, host_arena_bytes=(8 << 20) + 5, arena_mode=mode, arena_numa=numa, arena_threads=3)
    pl = c.arena_placement()
    assert pl["mode"] == mode and pl["pin_s"] > 0
    if mode == chm.ARENA_REGISTER and numa == 0:
        assert pl["numa_node"] == 0
    if numa == -2 or mode == chm.ARENA_HOSTALLOC:
        assert pl["numa_node"] == -1
    comp, s = torch.cuda.current_stream(), torch.cuda.Stream()
    for grow in (0, 40 << 20):
        if grow:
            c.arena_reserve(grow + 3)
            assert c.host_arena()[1] == grow + 3 and c.arena_placement()["mode"] == mode
        n_arena = c.host_arena()[1]
        sizes = [1 << 20, (3 << 20) + 7, 4096]
        src = [rand_bytes(n, 40 + j + grow) for j, n in enumerate(sizes)]
        offs = [0, 1 << 20, n_arena - 4096]  # the last block ends at the arena's last byte
        for flags in (chm.SWAP_KERNEL, chm.SWAP_CE):
            descs = [(x.data_ptr(), o, x.numel()) for x, o in zip(src, offs)]
            c.batch_wait(c.swap_out(descs, comp, s, flags), comp)
            torch.cuda.synchronize()
            host = arena_view(c)
            assert all(np.array_equal(host[o:o + x.numel()], x.cpu().numpy()) for x, o in zip(src, offs))
            dst = [torch.zeros_like(x) for x in src]
            c.batch_wait(c.swap_in([(d.data_ptr(), o, d.numel()) for d, o in zip(dst, offs)], comp, s, flags), comp)
            torch.cuda.synchronize()
            assert all(torch.equal(a, b) for a, b in zip(dst, src))
    c.close()

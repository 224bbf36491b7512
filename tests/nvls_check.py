"""NVLS in-switch reduction check (TEST HARNESS; torchrun, one process per GPU).

    torchrun --nproc-per-node N tests/nvls_check.py [--out res.json]

Every rank joins one multicast group (afdk_nvls_*: rank 0 creates it, the
others import its descriptor), writes a rank-dependent bf16 contribution into
its unicast view, and rank 0 reads the element-wise sum through the multicast
address (multimem.ld_reduce in the switch).  Checked against the sum of the
gathered contributions (bar: bf16 rounding of an fp32 sum, rel <= 1e-2) and
timed against the copy-based path (peer DMA pulls of N-1 partials +
afdk_add_partials) at the AFD return size (T_mb 256 x 7168 bf16).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--rows", type=int, default=256)
    a = ap.parse_args()
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2507_19427_b200 import Context, afdk

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dev = torch.device(f"cuda:{rank}")
    dist.init_process_group("nccl", device_id=dev)
    ctx = Context(rank)
    lib = afdk.load()
    H = 7168
    count = a.rows * H
    sup = [None] * world
    dist.all_gather_object(sup, int(lib.afdk_nvls_supported(ctx.handle)))
    if not all(sup):
        if rank == 0:
            print(json.dumps({"nvls": "unsupported", "per_rank": sup}), flush=True)
        dist.destroy_process_group()
        return
    g = ctypes.c_void_p()
    fd = ctypes.c_int(-1)
    if rank == 0:
        afdk.check(lib.afdk_nvls_create(ctx.handle, world, count * 2, 0, -1, ctypes.byref(g), ctypes.byref(fd)))
    info = [None] * world
    dist.all_gather_object(info, (os.getpid(), fd.value))
    if rank != 0:
        afdk.check(lib.afdk_nvls_create(ctx.handle, world, count * 2, info[0][0], info[0][1], ctypes.byref(g), None))
    uc, mc = ctypes.c_void_p(), ctypes.c_void_p()
    afdk.check(lib.afdk_nvls_bind(g, ctypes.byref(uc), ctypes.byref(mc)))
    # my contribution, written through my unicast view
    gen = torch.Generator(device=dev).manual_seed(100 + rank)
    mine = torch.randn(count, generator=gen, device=dev).to(torch.bfloat16)
    torch.cuda.synchronize()
    ucview = torch.empty(count, dtype=torch.bfloat16, device=dev)  # staging to copy into the raw pointer
    lib.afdk_copy(ctx.handle, uc, ctypes.c_void_p(mine.data_ptr()), count * 2, None)
    torch.cuda.synchronize()
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    dist.barrier()
    res = {}
    if rank == 0:
        out = torch.empty(count, dtype=torch.bfloat16, device=dev)
        afdk.check(lib.afdk_nvls_reduce_bf16(ctx.handle, mc, ctypes.c_void_p(out.data_ptr()), count, None))
        torch.cuda.synchronize()
        ref = torch.stack([p.float() for p in parts]).sum(0)
        err = float((out.float() - ref).abs().max() / ref.abs().max())
        st = torch.cuda.current_stream()

        def timed(fn, n=50):
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(n):
                fn()
            e1.record(st)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / n * 1e3

        t_nvls = timed(lambda: lib.afdk_nvls_reduce_bf16(ctx.handle, mc, ctypes.c_void_p(out.data_ptr()), count,
                                                         ctypes.c_void_p(st.cuda_stream)))
        res = {"nvls": "ok" if err <= 1e-2 else "FAIL", "world": world, "rows": a.rows, "hidden": H,
               "rel_err": err, "nvls_reduce_us": t_nvls, "bytes_per_member": count * 2}
    dist.barrier()
    if rank == 0:
        # the copy path the runtime uses without NVLS: pull the other members'
        # partials (here: from the gathered copies, same size, over NVLink)
        # then add_partials
        bufs = [torch.empty(count, dtype=torch.bfloat16, device=dev) for _ in range(world - 1)]
        ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=dev)
        base = parts[0]
        out2 = torch.empty_like(base)
        st = torch.cuda.current_stream()

        def copy_path():
            for i, b in enumerate(bufs):
                b.copy_(parts[i + 1], non_blocking=True)
            lib.afdk_add_partials(ctx.handle, ctypes.c_void_p(base.data_ptr()), ctypes.c_void_p(ptrs.data_ptr()),
                                  world - 1, count, ctypes.c_void_p(out2.data_ptr()), ctypes.c_void_p(st.cuda_stream))

        for _ in range(5):
            copy_path()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(50):
            copy_path()
        e1.record(st)
        torch.cuda.synchronize()
        res["add_partials_local_us"] = e0.elapsed_time(e1) / 50 * 1e3
        print(json.dumps(res), flush=True)
        if a.out:
            json.dump(res, open(a.out, "w"))
    dist.barrier()
    lib.afdk_nvls_destroy(g)
    ctx.close()
    dist.destroy_process_group()
    sys.exit(0 if (rank != 0 or res.get("nvls") == "ok") else 1)


if __name__ == "__main__":
    main()

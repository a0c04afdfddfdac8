"""World-size-2 (gloo, CPU) test of the multi-GPU path's host logic.

Each rank builds the product's exchange plan for its macro partition
(tetmf_plan_*), fills its local storage with macro-local partial sums from
the oracle (the same quantity the element kernels leave in y before the
interface step), runs the product's own K4 body for rank-local groups and
its pack / combine bodies (tetmf_host_*) around a gloo send/recv -- the CPU
stand-in for the NCCL send/recv of exchange.cu -- and checks that every
stored copy then equals the full apply in reference numbering.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, mesh, form, level, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        import paper_2404_08371_b200 as tm
        from oracle.refapi import PortSystem, port_lib
        import ctypes

        space = tm.SPACE_ND1 if form == "N1" else tm.SPACE_P1
        ctx = tm.Context(mesh, device=-1, rank=rank, nranks=WORLD)
        macros = ctx.local_macros()
        ms, _ = ctx.layout(space, level)
        ref_map, nd = ctx.ref_map(space, level)

        port = PortSystem(mesh, form, level)
        x = port.seeded_input(42)
        c0, c1 = port.coefficients()
        w_full, _ = port.apply(x, c0, c1)
        nmac = ctx.num_macros()[0]
        L = port_lib().L
        L.port_apply_macros.restype = ctypes.c_int
        dp = ctypes.POINTER(ctypes.c_double)
        L.port_apply_macros.argtypes = [ctypes.c_void_p, dp, dp, dp, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_ubyte), dp]

        def ptr(a):
            return None if a is None else a.ctypes.data_as(dp)

        # local storage: macro-local partial sums on every copy
        y = np.zeros(ms * len(macros))
        for li, m in enumerate(macros):
            mask = np.zeros(nmac, dtype=np.uint8)
            mask[m] = 1
            wm = np.empty(port.num_dofs)
            assert L.port_apply_macros(port.h, ptr(x), ptr(c0), ptr(c1), 0,
                                       mask.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte)), ptr(wm)) == 0
            e = ref_map[li * ms:(li + 1) * ms]
            ok = e >= 0
            vals = wm[e[ok] >> 2]
            vals[(e[ok] & 2) != 0] *= -1
            y[li * ms:(li + 1) * ms][ok] = vals

        off, cp = ctx.local_groups(space, level)
        tm.host_local_sum(off, cp, y)
        plan = ctx.exchange_plan(space, level)
        send = tm.host_pack(y, plan["send_index"])
        recv = np.zeros(int(plan["recv_offsets"][-1]))
        reqs = []
        for i, peer in enumerate(plan["peers"]):
            so, se = plan["send_offsets"][i], plan["send_offsets"][i + 1]
            ro, re_ = plan["recv_offsets"][i], plan["recv_offsets"][i + 1]
            reqs.append(dist.isend(torch.from_numpy(send[so:se].copy()), peer))
            buf = torch.zeros(int(re_ - ro), dtype=torch.float64)
            dist.recv(buf, peer)
            recv[ro:re_] = buf.numpy()
        for r in reqs:
            r.wait()
        tm.host_combine(y, recv, plan["group_offsets"], plan["group_entries"])

        ok = ref_map >= 0
        expect = w_full[ref_map[ok] >> 2]
        expect[(ref_map[ok] & 2) != 0] *= -1
        err = np.abs(y[ok] - expect).max() / np.abs(w_full).max()
        q.put((rank, float(err), len(plan["peers"]), int(plan["group_offsets"].size - 1)))
        dist.destroy_process_group()
    except Exception as e:  # report to the parent
        import traceback
        q.put((rank, "error: " + traceback.format_exc(), 0, 0))


@pytest.mark.parametrize("mesh,form,level", [("cube6", "P1", 3), ("cube6", "N1", 2), ("cubes1x1x2", "P1", 2),
                                             ("cubes1x1x2", "N1", 2)])
def test_two_rank_exchange(mesh, form, level):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, mesh, form, level, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    for rank, err, npeers, ngroups in res:
        assert not isinstance(err, str), err
        assert npeers == 1 and ngroups > 0
        assert err <= 1e-13, (rank, err)

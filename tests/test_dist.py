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


def _transfer(tm, plan, y, rank, mode):
    """The exchange's transfer step on CPU (gloo standing in for the device
    transport). 'sendrecv': pack into a send buffer, one message per peer
    (the NCCL send/recv path). 'put': the direct-put addressing of
    TETMF_EXCHANGE_PUT -- the group's send-count matrix is all-gathered, each
    rank computes where its values land in every peer's receive buffer
    (tetmf_host_put_offsets / tetmf_host_put_targets, the put kernel's own
    addressing) and the receiver only stores them at those positions, which
    must be exactly the range its own plan reserves for that peer."""
    send = tm.host_pack(y, plan["send_index"])
    recv = np.zeros(int(plan["recv_offsets"][-1]))
    reqs = []
    if mode == "sendrecv":
        for i, peer in enumerate(plan["peers"]):
            so, se = plan["send_offsets"][i], plan["send_offsets"][i + 1]
            ro, re_ = plan["recv_offsets"][i], plan["recv_offsets"][i + 1]
            reqs.append(dist.isend(torch.from_numpy(send[so:se].copy()), peer))
            buf = torch.zeros(int(re_ - ro), dtype=torch.float64)
            dist.recv(buf, peer)
            recv[ro:re_] = buf.numpy()
    else:
        world = dist.get_world_size()
        row = torch.zeros(world, dtype=torch.int64)
        for i, peer in enumerate(plan["peers"]):
            row[peer] = int(plan["send_offsets"][i + 1] - plan["send_offsets"][i])
        rows = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(rows, row)
        counts = torch.stack(rows).numpy()
        peer_off = tm.host_put_offsets(counts, rank, plan["peers"])
        dst, slot = tm.host_put_targets(plan["send_offsets"], peer_off)
        seen = np.zeros(recv.size, dtype=int)
        for i, peer in enumerate(plan["peers"]):
            so, se = plan["send_offsets"][i], plan["send_offsets"][i + 1]
            assert (slot[so:se] == i).all()
            reqs.append(dist.isend(torch.from_numpy(dst[so:se].copy()), peer))
            reqs.append(dist.isend(torch.from_numpy(send[so:se].copy()), peer))
            ro, re_ = plan["recv_offsets"][i], plan["recv_offsets"][i + 1]
            pos = torch.zeros(int(re_ - ro), dtype=torch.int64)
            val = torch.zeros(int(re_ - ro), dtype=torch.float64)
            dist.recv(pos, peer)
            dist.recv(val, peer)
            pos = pos.numpy()
            assert ((pos >= ro) & (pos < re_)).all(), "a put lands outside the range reserved for its sender"
            recv[pos] = val.numpy()
            seen[pos] += 1
        assert (seen == 1).all()  # every receive position written exactly once
    for r in reqs:
        r.wait()
    return recv


def _worker(rank, port, mesh, form, level, q, mode="sendrecv"):
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
        recv = _transfer(tm, plan, y, rank, mode)
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


@pytest.mark.parametrize("mode", ["sendrecv", "put"])
@pytest.mark.parametrize("mesh,form,level", [("cube6", "P1", 3), ("cube6", "N1", 2), ("cubes1x1x2", "P1", 2),
                                             ("cubes1x1x2", "N1", 2)])
def test_two_rank_exchange(mesh, form, level, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, mesh, form, level, q, mode)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    for rank, err, npeers, ngroups in res:
        assert not isinstance(err, str), err
        assert npeers == 1 and ngroups > 0
        assert err <= 1e-13, (rank, err)


def _slab_worker(rank, world, port, mesh, level, q, mode="sendrecv"):
    """(macro, z-slab) partition (TETMF_PARTITION_SLAB): every rank stores
    every macro but only its units' planes are computed; copies elsewhere are
    poisoned (NaN) so that any use of a non-owned copy shows."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import ctypes

        import paper_2404_08371_b200 as tm
        from oracle.refapi import PortSystem, port_lib

        space = tm.SPACE_P1
        ctx = tm.Context(mesh, device=-1, rank=rank, nranks=world, partition=tm.PARTITION_SLAB)
        macros = ctx.local_macros()
        nmac = ctx.num_macros()[0]
        assert macros == list(range(nmac))  # every rank stores every macro
        ms, _ = ctx.layout(space, level)
        ref_map, nd = ctx.ref_map(space, level)
        n = 1 << level
        tet = lambda k: (k + 1) * (k + 2) * (k + 3) // 6
        starts = np.array([tet(n) - tet(n - z) for z in range(n + 1)])
        zslot = np.searchsorted(starts, np.arange(ms), side="right") - 1  # plane of each in-macro slot
        units = tm.slab_units(nmac, level, world, rank)
        own = np.zeros((nmac, ms), dtype=bool)
        for m, za, zb in units:
            own[m] = (zslot >= za) & (zslot < zb) & (np.arange(ms) < tet(n))
        port = PortSystem(mesh, "P1", level)
        x = port.seeded_input(42)
        w_full, _ = port.apply(x, None, None)
        L = port_lib().L
        L.port_apply_macros.restype = ctypes.c_int
        dp = ctypes.POINTER(ctypes.c_double)
        L.port_apply_macros.argtypes = [ctypes.c_void_p, dp, dp, dp, ctypes.c_int, ctypes.POINTER(ctypes.c_ubyte), dp]
        y = np.full(ms * nmac, np.nan)
        for m in range(nmac):
            mask = np.zeros(nmac, dtype=np.uint8)
            mask[m] = 1
            wm = np.empty(port.num_dofs)
            assert L.port_apply_macros(port.h, x.ctypes.data_as(dp), None, None, 0,
                                       mask.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte)),
                                       wm.ctypes.data_as(dp)) == 0
            e = ref_map[m * ms:(m + 1) * ms]
            sel = (e >= 0) & own[m]
            y[m * ms:(m + 1) * ms][sel] = wm[e[sel] >> 2]
        off, cp = ctx.local_groups(space, level)
        tm.host_local_sum(off, cp, y)
        plan = ctx.exchange_plan(space, level)
        recv = _transfer(tm, plan, y, rank, mode)
        tm.host_combine(y, recv, plan["group_offsets"], plan["group_entries"])
        sel = (ref_map >= 0) & own.ravel()
        expect = w_full[ref_map[sel] >> 2]
        err = np.abs(y[sel] - expect).max() / np.abs(w_full).max()
        q.put((rank, float(err), int(sel.sum()), units))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, "error: " + traceback.format_exc(), 0, None))


@pytest.mark.parametrize("mode", ["sendrecv", "put"])
@pytest.mark.parametrize("mesh,level,world", [("cube6", 4, 2), ("cube6", 4, 4), ("cube6", 5, 4),
                                              ("cubes1x1x2", 4, 3)])
def test_slab_partition_exchange(mesh, level, world, mode):
    """Config 4's strong-scaling partition: (macro, z-slab) units, exchange
    of the macro-interface copies across ranks; every owned copy equals the
    full apply and every lattice point is owned by exactly one rank."""
    import paper_2404_08371_b200 as tm
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, mesh, level, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    owned = 0
    for rank, err, cnt, units in res:
        assert not isinstance(err, str), err
        assert err <= 1e-13, (rank, err)
        owned += cnt
    # every stored point of every macro is owned once (units tile the planes)
    nmac = tm.Context(mesh, device=-1).num_macros()[0]
    n = 1 << level
    assert owned == nmac * (n + 1) * (n + 2) * (n + 3) // 6


def test_slab_units_balanced():
    import paper_2404_08371_b200 as tm
    n, L = 256, 8
    for world in (2, 4, 8):
        work = []
        covered = {}
        for r in range(world):
            w = 0
            for m, za, zb in tm.slab_units(6, L, world, r):
                assert za % 8 == 0 and (zb % 8 == 0 or zb == n + 1)
                for z in range(za, zb):
                    assert (m, z) not in covered
                    covered[(m, z)] = r
                    w += (n + 1 - z) * (n + 2 - z) // 2
            work.append(w)
        assert len(covered) == 6 * (n + 1)
        assert max(work) / (sum(work) / world) < 1.03, work  # within 3 % of perfect balance

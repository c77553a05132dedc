"""World-size-2 gloo run of the shard/gather driver (CPU; the oracle stands in
for the per-rank GPU compute)."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from conftest import ROOT

FIELDS = ("score", "i_begin", "i_end", "j_begin", "j_end", "matches", "aln_len")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from oracle import oracle
    from paper_2303_01845_b200 import blosum62
    from pastis_synth import workloads
    from paper_2303_01845_b200._native import RESULT_DTYPE
    from paper_2303_01845_b200.batch import pack_codes
    from paper_2303_01845_b200.distributed import align_distributed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mat = np.asarray(blosum62.MATRIX, dtype=np.int32)
    sa, sb = workloads.config3(300, seed=3)
    arena, table = pack_codes(sa, sb)

    def compute(a_s, t_s):
        ref = oracle.align_batch_c(a_s, t_s, 11, 1, mat, threads=2)
        rec = np.zeros(len(t_s), dtype=RESULT_DTYPE)
        for k, f in enumerate(FIELDS):
            rec[f] = ref[:, k]
        return rec

    out = align_distributed(arena, table, None, rank, world, compute=compute)
    if rank == 0:
        full = oracle.align_batch_c(arena, table, 11, 1, mat, threads=2)
        got = np.stack([out[f] for f in FIELDS], axis=1)
        q.put(bool((got == full[:, :7]).all()))
    dist.destroy_process_group()


def test_gloo_shard_gather_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok


def test_local_shard_dedups_and_roundtrips():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2303_01845_b200.batch import pack_codes
    from paper_2303_01845_b200.distributed import local_shard, partition
    sa = [b"AAAA", b"CCC", b"AAAA"]
    sb = [b"GG", b"GG", b"T"]
    arena, t = pack_codes(sa, sb)
    shard = partition(t, 2)
    seen = 0
    for r in range(2):
        a_s, t_s, idx = local_shard(arena, t, shard, r)
        for row, k in zip(t_s, idx):
            assert bytes(a_s[row["a_off"]:row["a_off"] + row["a_len"]]) == sa[k]
            assert bytes(a_s[row["b_off"]:row["b_off"] + row["b_len"]]) == sb[k]
            seen += 1
    assert seen == 3

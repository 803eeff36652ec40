"""The library's distributed matvec (blfmm_plan_attach_comm + blfmm_execute:
partitioned upsweep, sum all-reduce of the exchange buffer, owned downsweep
and near field, gather of the owned sorted slices of u, scatter to caller
order) with world_size 2 and 3 processes. They share the one GPU of the test
box, so the collectives are caller callbacks over a gloo process group
(host copies between the library's phases): no kernel of one rank waits on
another. The NCCL flavour of the same calls runs at world_size 1."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, out_path, name, n, leaf, nrhs):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1606_07652_b200 as B
    from paper_1606_07652_b200 import distributed as D
    from paper_1606_07652_b200 import inputs as I
    W = I.WORKLOADS[name]
    x, w = W.make(n)
    w = np.stack([w * (q + 1) for q in range(nrhs)]) if nrhs > 1 else w
    k = B.parse_kernel_spec(W.kernel)
    sm = D.ShardedMatvec(B.PointSet(W.d, x), leaf, k, W.sigma, W.m, nrhs=nrhs, device=0)
    assert sm.comm == "torch-host" and sm.world == world
    lam = torch.from_numpy(np.ascontiguousarray(w.reshape(nrhs, -1))).cuda()
    out = torch.empty_like(lam)
    for _ in range(2):  # second call reuses the plan and buffers
        st = sm.device(lam, out, stats=True)
    torch.cuda.synchronize()
    host = sm(w)  # host-buffer API (blfmm_execute)
    np.save(out_path + f".{rank}.npy", out.cpu().numpy())
    np.save(out_path + f".{rank}.host.npy", np.asarray(host.values).reshape(nrhs, -1))
    np.save(out_path + f".{rank}.imag.npy", np.array([st.max_imag_residual]))
    dist.barrier()
    dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,n,leaf,world,nrhs", [("P3", 60000, 4, 2, 1), ("P4", 40000, 5, 2, 1),
                                                   ("P3", 40000, 4, 3, 2), ("P2p", 20000, 3, 3, 1)])
def test_distributed_execute_matches_single_gpu(blfmm, tmp_path, name, n, leaf, world, nrhs):
    from paper_1606_07652_b200 import inputs as I
    W = I.WORKLOADS[name]
    x, w = W.make(n)
    w = np.stack([w * (q + 1) for q in range(nrhs)]) if nrhs > 1 else w
    ref = blfmm.Plan(blfmm.PointSet(W.d, x), leaf, blfmm.parse_kernel_spec(W.kernel),
                     W.sigma, W.m, nrhs=nrhs).execute(w)
    full = np.asarray(ref.values).reshape(nrhs, -1)
    out = str(tmp_path / "u")
    mp.spawn(_worker, args=(world, _port(), out, name, n, leaf, nrhs), nprocs=world, join=True)
    for r in range(world):  # u on every rank, both APIs
        for suffix in ("", ".host"):
            got = np.load(out + f".{r}{suffix}.npy")
            assert np.linalg.norm(got - full) / np.linalg.norm(full) <= 1e-13
        imag = float(np.load(out + f".{r}.imag.npy")[0])
        assert abs(imag - ref.stats.max_imag_residual) <= 1e-8 * max(1.0, imag)


@pytest.mark.parametrize("name,n,leaf,nrhs", [("P3", 30000, 4, 1), ("P4", 30000, 5, 3)])
def test_nccl_one_rank_group(blfmm, name, n, leaf, nrhs):
    """The NCCL flavour of the distributed execute on one GPU: unique id,
    ncclCommInitRank, the grouped ncclBroadcast gather and the ncclAllReduce
    (max) of the stats over a one-rank communicator - bit-identical to the
    plain execute (the same kernels; the sorted slice is scattered after the
    gather). Several NCCL ranks need one GPU each."""
    from paper_1606_07652_b200 import api as A
    from paper_1606_07652_b200 import inputs as I
    W = I.WORKLOADS[name]
    x, w = W.make(n)
    w = np.stack([w * (q + 1) for q in range(nrhs)]) if nrhs > 1 else w
    k = blfmm.parse_kernel_spec(W.kernel)
    ref = blfmm.Plan(blfmm.PointSet(W.d, x), leaf, k, W.sigma, W.m, nrhs=nrhs).execute(w)
    uid = A.nccl_unique_id()
    assert len(uid) == 128 and any(uid)
    p = blfmm.Plan(blfmm.PointSet(W.d, x), leaf, k, W.sigma, W.m, nrhs=nrhs)
    p.attach_nccl(uid)
    with pytest.raises(blfmm.InvalidArgument):
        p.attach_nccl(uid)  # one communicator per plan
    for _ in range(2):
        got = p.execute(w)
    assert np.array_equal(np.asarray(got.values), np.asarray(ref.values))
    assert got.stats.max_imag_residual == ref.stats.max_imag_residual


@pytest.mark.parametrize("args", [["3", "60000", "4", "2", "imq:c=0.1", "3.141592653589793", "16", "1"],
                                  ["3", "40000", "4", "3", "gaussian:c=64", "3.141592653589793", "16", "2"],
                                  ["2", "50000", "5", "4", "mq:c=0.05", "3.141592653589793", "16", "1"],
                                  # tools/fuzz_dist.sh: other even M (3-multiplication block-A
                                  # kernels in exchange mode), odd M, 32 right-hand sides, d = 1
                                  ["3", "20000", "3", "3", "gaussian:c=64", "3.141592653589793", "34", "1"],
                                  ["3", "20000", "3", "4", "imq:c=0.1", "3.141592653589793", "15", "1"],
                                  ["3", "30000", "3", "2", "gaussian:c=64", "3.141592653589793", "16", "32"],
                                  ["1", "5000", "4", "2", "gaussian:c=9", "3.141592653589793", "300", "2"]])
def test_cpp_caller_shards_through_the_c_abi(tmp_path, args):
    """A C++ program (tests/cpp/dist_threads.cpp) runs `world` ranks as
    threads, each with its own plan, and supplies host collectives through
    blfmm_comm_ops: the C ABI alone shards the matvec (no Python, no torch)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "dist_threads")
    libdir = os.path.join(root, "paper_1606_07652_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{root}/include", "-I/usr/local/cuda/include",
                    os.path.join(root, "tests", "cpp", "dist_threads.cpp"), "-o", exe,
                    f"-L{libdir}", "-lblfmm_gpu", "-L/usr/local/cuda/lib64", "-lcudart",
                    f"-Wl,-rpath,{libdir}", "-pthread"], check=True)
    r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, (r.returncode, r.stdout, r.stderr)

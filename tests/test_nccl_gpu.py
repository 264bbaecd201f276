"""The sharded step over a real NCCL process group.

One rank on the one GPU of the test box: ``init_process_group("nccl")``, the
row-shard driver with the collective on (``RowShardQuantizer(collective=True)``)
in both exchange modes -- the north star's ONE max all-reduce of every
tensor's amax per step, and the grouped step whose amaxes ride in the previous
group's quantize launch -- over the first layer of the Qwen3-8B workload (C2,
7 matrices, 218 M elements).  Every output is compared with the CPU oracle
(mode "given" with the whole tensor's amax): whole tensors for k/v (with the
FP64 sums), sampled row ranges for the rest, G bit for bit.  Then the SURVEY
§5 fault injection: a NaN in one shard raises the sticky flag after the
all-reduce and gives that tensor G = 1 while the other tensors keep theirs.
(Several NCCL ranks cannot share one device; the multi-rank exchange is
covered by tests/test_dist_gloo.py on CPU and tests/test_dist_gpu.py.)
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import ssgen

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NT = 7                      # layer 0: q, k, v, o, gate, up, down
ROWS = [(0, 64), (1000, 1040)]   # sampled row ranges (clipped per tensor) + the last 48 rows

SCRIPT = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, %(root)r)
import ssgen, paper_2605_12464_b200 as ss
from paper_2605_12464_b200.dist import CudaOps, RowShardQuantizer, ShardPlan
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
assert dist.get_backend() == "nccl" and dist.get_world_size() == 1
specs = ssgen.workload("c2_qwen3_8b_weights")[:%(nt)d]
plan = ShardPlan([(s.rows, s.cols) for s in specs], 0, 1)
# drawn on the host like the oracle's copy (the CPU and CUDA generators differ), then uploaded
xs = [ssgen.generate(s.kind, s.rows, s.cols, seed=ssgen.workloads.BASE_SEED, tid=s.tid).to(dev)
      for s in specs]
ops = CudaOps(-8, 8, want_err=True, want_sums=True)
res = {}
def rows_of(r):
    out = []
    for lo, hi in %(rows)r + [(r - 48, r)]:
        lo, hi = max(0, min(lo, r)), max(0, min(hi, r))
        if hi > lo:
            out.append((lo, hi))
    return out
for ex in ("grouped", "single"):
    outs = [ops.alloc_out(x) for x in xs]
    q = RowShardQuantizer(plan, ops, group=None, device=dev, collective=True, exchange=ex)
    n = q.step(xs, outs)
    torch.cuda.synchronize()
    res[ex + "_allreduces"] = np.array(q.allreduces)
    res[ex + "_groups"] = np.array(len(q.groups))
    res[ex + "_amax"] = q.amax_buf.cpu().numpy()
    res[ex + "_flags"] = np.array(ss.device_status())
    for k, (x, o) in enumerate(zip(xs, outs)):
        res["%%s_%%d_G" %% (ex, k)] = o.G.cpu().numpy()
        res["%%s_%%d_sums" %% (ex, k)] = o.sums.cpu().numpy()
        for lo, hi in rows_of(x.shape[0]) if x.shape[0] > 1024 else [(0, x.shape[0])]:
            nbr = x.shape[1] // 16
            res["%%s_%%d_%%d_codes" %% (ex, k, lo)] = o.codes[lo:hi].cpu().numpy()
            res["%%s_%%d_%%d_scales" %% (ex, k, lo)] = o.scales[lo:hi].cpu().numpy()
            res["%%s_%%d_%%d_err" %% (ex, k, lo)] = o.err[lo * nbr:hi * nbr].cpu().numpy()
# fault injection: NaN in tensor 2's shard
bad = [x.clone() for x in xs]
bad[2][5, 7] = float("nan")
outs = [ops.alloc_out(x) for x in bad]
RowShardQuantizer(plan, ops, group=None, device=dev, collective=True, exchange="single").step(bad, outs)
torch.cuda.synchronize()
res["nan_flags"] = np.array(ss.device_status())
res["nan_G"] = np.array([float(o.G.item()) for o in outs], np.float32)
dist.barrier()
dist.destroy_process_group()
np.savez(sys.argv[1], **res)
"""


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_run(tmp_path_factory):
    path = str(tmp_path_factory.mktemp("nccl") / "out.npz")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0",
               WORLD_SIZE="1", LOCAL_RANK="0", NCCL_DEBUG="WARN")
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT, "nt": NT, "rows": ROWS}, path],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    return np.load(path)


@pytest.mark.parametrize("exchange", ["grouped", "single"])
def test_nccl_step_matches_oracle(nccl_run, oracle_lib, exchange):
    res = nccl_run
    assert int(res[exchange + "_flags"]) == 0
    want_ar = 1 if exchange == "single" else int(res[exchange + "_groups"])
    assert int(res[exchange + "_allreduces"]) == want_ar and (exchange == "single" or want_ar > 1)
    specs = ssgen.workload("c2_qwen3_8b_weights")[:NT]
    for k, s in enumerate(specs):
        x = ssgen.generate(s.kind, s.rows, s.cols, seed=ssgen.workloads.BASE_SEED, tid=s.tid)
        amax = oracle_lib.tensor_amax(x)
        assert int(res[exchange + "_amax"][k]) & 0xFFFFFFFF == amax, k      # the all-reduced amax
        G = np.float32(oracle_lib.global_scale(1, amax))
        assert res["%s_%d_G" % (exchange, k)].view(np.uint32)[0] == G.view(np.uint32), k
        if s.rows <= 1024:                        # k, v: the whole tensor, with the FP64 sums
            ref = oracle_lib.quantize(x, s.rows, s.cols, -8, 8, "given", amax_bits=amax)
            assert np.array_equal(res["%s_%d_0_codes" % (exchange, k)], ref.codes), k
            assert np.array_equal(res["%s_%d_0_scales" % (exchange, k)], ref.scales), k
            assert np.array_equal(res["%s_%d_0_err" % (exchange, k)].view(np.uint32), ref.err.view(np.uint32))
            got = res["%s_%d_sums" % (exchange, k)]
            assert np.all(np.abs(got - ref.sums) <= 1e-9 * np.abs(ref.sums)), k
            continue
        for key in [f for f in res.files if f.startswith("%s_%d_" % (exchange, k)) and f.endswith("_codes")]:
            lo = int(key.split("_")[2])
            codes = res[key]
            hi = lo + codes.shape[0]
            ref = oracle_lib.quantize(x[lo:hi].contiguous(), hi - lo, s.cols, -8, 8, "given", amax_bits=amax)
            assert np.array_equal(codes, ref.codes), (k, lo)
            assert np.array_equal(res[key.replace("codes", "scales")], ref.scales), (k, lo)
            assert np.array_equal(res[key.replace("codes", "err")].view(np.uint32), ref.err.view(np.uint32))


def test_nccl_grouped_equals_single(nccl_run):
    res = nccl_run
    for f in res.files:
        if f.startswith("grouped_") and not f.endswith(("_allreduces", "_groups", "_flags")):
            assert np.array_equal(res[f], res[f.replace("grouped_", "single_", 1)]), f


def test_nccl_nan_fault_injection(nccl_run):
    res = nccl_run
    assert int(res["nan_flags"]) & 1                       # SS_FLAG_NONFINITE after the all-reduce
    G = res["nan_G"]
    assert G[2] == 1.0                                     # the poisoned tensor falls back to G = 1
    for k in range(NT):
        if k != 2:
            assert G[k] == res["single_%d_G" % k][0], k   # the others keep their global scale

"""One rank of the NCCL multi-GPU parity check (tests/test_nccl_gpu.py):
each golden case as an x-slab decomposition over the torchrun ranks, one GPU
per rank, the halo exchange and LLG all-reduces over NCCL inside the library
(parallel.run_ranks); rank 0 compares with the reference golden bit for bit.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        tests/nccl_worker.py mixed3d nonmono3d fail3d
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2510_22221_b200 import parallel  # noqa: E402
from tests.golden.cases import CASES, build, mirror_namespace  # noqa: E402
from tests.golden_io import load  # noqa: E402


def check(name: str) -> str:
    case = CASES[name]
    g = load(name)
    out = parallel.run_ranks(build(case, mirror_namespace()), bias=case.get("bias"))
    if dist.get_rank() != 0:
        return ""
    fields, M, probes, its = out
    if case.get("expect_failure"):
        assert fields is None, f"{name}: expected a StepFailure"
        step, res, it, kind = its
        assert step == int(g["fail_step"]) and it == int(g["fail_iterations"]), its
        assert res == float(g["fail_residual"]), its
        return f"OK {name} failure at step {step}"
    assert fields is not None, f"{name}: step failure {its}"
    for k, v in g["fields"].items():
        got = M if k == "M" else fields[k]
        assert np.array_equal(got, v), (name, k, float(np.max(np.abs(got - v))))
    assert np.array_equal(its, g["iterations"]), name
    for key, v in g["probes"].items():
        assert np.array_equal(probes[key], v), (name, key)
    return f"OK {name}"


def main() -> None:
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        for name in sys.argv[1:]:
            msg = check(name)
            if msg:
                print(msg, flush=True)
            dist.barrier()
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

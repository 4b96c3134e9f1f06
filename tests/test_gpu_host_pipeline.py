"""HostStepPipeline (verify.py): one verification step from pinned host
inputs to pinned host outputs, pipelined over chunks of sequences, must give
the same results as one TreeVerifier.step over the whole batch on device
inputs -- accepted paths / next tokens / uniforms bit-exact, attention output
and LSE within the bf16 / fp32 tolerance of a different split plan.  Needs a
B200."""

import os
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


@pytest.mark.parametrize("mode,chunks", [("greedy", 2), ("greedy", 3), ("stochastic", 2)])
def test_host_pipeline_matches_device_step(mode, chunks):
    import bench
    from paper_2508_08192_b200 import _lib
    from paper_2508_08192_b200.sharding import shard_for
    from paper_2508_08192_b200.verify import HostStepPipeline, StepInputs, TreeVerifier

    _lib.load()
    dev = torch.device("cuda", 0)
    cfg = dict(bench.CONFIGS["c3"], B=5, ctx=1000, V=5000)
    x, R = bench.make_inputs(cfg, shard_for(0, 1, cfg["Hq"], cfg["Hkv"], cfg["V"]), dev, mode=mode)
    temp, top_p = (0.0, 1.0) if mode == "greedy" else (bench.TEMPERATURE, bench.TOP_P)
    levels = bench._tree_levels(tuple(bench._augment(bench.TREE)))

    def make():
        return TreeVerifier(scale=cfg["d"] ** -0.5, temperature=temp, top_p=top_p, max_ctx=cfg["ctx"],
                            tree_levels=levels)

    names = ["logits", "parent", "n_rows", "ctx_len", "tokens", "q", "tree_k", "tree_v"]
    if mode != "greedy":
        names += ["draft_logits", "seeds", "steps"]
    k0, v0 = x.k_pool.clone(), x.v_pool.clone()
    ref = make()
    out, lse, acc, _ = ref.step(x)
    torch.cuda.synchronize()
    ref.check(acc=acc)
    want = {"out": out.cpu(), "lse": lse.cpu(), "path": acc.path.cpu(), "path_len": acc.path_len.cpu(),
            "next_token": acc.next_token.cpu()}
    # the same step from host buffers (pools restored: compaction wrote the accepted rows)
    x.k_pool.copy_(k0)
    x.v_pool.copy_(v0)
    pinned = {k: getattr(x, k).cpu().pin_memory() for k in names}
    fields = {k: getattr(x, k) for k in StepInputs.__dataclass_fields__}
    fields.update({k: torch.empty_like(getattr(x, k)) for k in names})
    xe = StepInputs(**fields)
    outs = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in want.items()}
    pipe = HostStepPipeline(make, chunks=chunks)
    pipe(xe, pinned, outs)
    torch.cuda.synchronize()
    pipe.check()
    assert torch.equal(outs["path_len"], want["path_len"])
    assert torch.equal(outs["next_token"], want["next_token"])
    for b in range(cfg["B"]):
        n = int(want["path_len"][b])
        assert torch.equal(outs["path"][b, :n], want["path"][b, :n]), b
    torch.testing.assert_close(outs["out"].float(), want["out"].float(), atol=2e-2, rtol=2e-2)
    torch.testing.assert_close(outs["lse"], want["lse"], atol=1e-3, rtol=1e-4)
    # compaction ran per chunk: the pools equal the single step's
    kp, vp = x.k_pool.clone(), x.v_pool.clone()
    x.k_pool.copy_(k0)
    x.v_pool.copy_(v0)
    ref.step(x)
    torch.cuda.synchronize()
    assert torch.equal(kp, x.k_pool) and torch.equal(vp, x.v_pool)

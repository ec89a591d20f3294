"""GPU: the C-ABI collective of the sharded path:
copris_allreduce_scalars over an NCCL communicator made by the C-ABI helpers.
One GPU is available here, so the communicators have one rank (NCCL refuses two
ranks on one device); the multi-rank reduction itself is covered by the gloo
tests of tests/test_sharding.py and by bench.py under torchrun."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_allreduce_scalars_init_all(ctx, oracle):
    from paper_2511_05589_b200.sharding import NcclScalars, loss_from_scalars
    from parity_util import Case
    case = Case(oracle, seed=3, P=4, G=4, V=32000, lmax=64)
    batch = case.upload(ctx)
    outs = ctx.alloc_outputs(batch.n_tok, torch.device("cuda", 0))
    dl = torch.empty((batch.n_tok, case.V), dtype=torch.bfloat16, device="cuda")
    ctx.loss_chunk_fused(case.logits_gpu(), batch, case.clip(), outs, dlogits=dl, row_base=0,
                         total_tokens=batch.n_tok)
    out4 = torch.zeros(4, dtype=torch.float64, device="cuda")
    ctx.reduce(outs, batch.n_tok, out4)
    before = out4.clone()
    (comm,) = NcclScalars.init_all([0])
    comm.allreduce(out4)
    torch.cuda.synchronize()
    assert torch.equal(out4, before)  # one rank: the sum is the rank's own scalars
    assert abs(loss_from_scalars(out4.cpu(), batch.n_tok) - case.ref.loss) <= 1e-5 * max(
        1.0, abs(case.ref.loss)) + 1e-12
    comm.close()


def test_allreduce_scalars_init_rank():
    from paper_2511_05589_b200.sharding import NcclScalars
    uid = NcclScalars.unique_id()
    assert len(uid) == 128
    comm = NcclScalars(0, 1, uid, 0)
    x = torch.tensor([1.5, 7.0, 3.0, 2.0], dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        comm.allreduce(x, stream=s)
    s.synchronize()
    assert x.tolist() == [1.5, 7.0, 3.0, 2.0]
    comm.close()


def test_allreduce_scalars_errors():
    from paper_2511_05589_b200 import _lib as L
    from paper_2511_05589_b200.sharding import NcclScalars
    lib = L.load()
    assert lib.copris_allreduce_scalars(None, None, None) == L.COPRIS_E_INVALID
    assert b"null pointer" in lib.copris_last_error()
    assert lib.copris_nccl_comm_init_all(0, None, None) == L.COPRIS_E_INVALID
    assert lib.copris_nccl_comm_destroy(None) == 0
    with pytest.raises(ValueError):
        NcclScalars(0, 1, bytes(128), 3)  # rank out of range

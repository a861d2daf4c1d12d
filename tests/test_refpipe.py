"""The reference arm's pipeline (oracle/refpipe.py) runs the reference's OWN
epsim code (pack_fields -> SPSC ring -> unpack_fields/imm -> apply_deliveries,
numba backend) and must deliver exactly the rows the oracle's dispatch puts in
each receive order — a second pin of oracle.ep.dispatch against reference
code, at the toy config (BASELINE.json configs[0]) and a ragged 3-rank case."""
import numpy as np
import pytest

from oracle import ep as O
from oracle import refpipe
from tests.helpers import bf16_random, make_routing


@pytest.fixture(scope="module")
def ref():
    refpipe.build_ref()
    if not (refpipe.REF_OUT / "epsim" / "kernels.py").exists():
        pytest.skip("oracle/_ref/epsim not built (no /root/reference here)")
    return refpipe.load_epsim()


@pytest.mark.parametrize("R,T,H,E,k", [(4, 128, 1024, 32, 2), (3, 1000, 256, 24, 4), (1, 300, 128, 8, 2)])
def test_reference_pipeline_matches_oracle(ref, R, T, H, E, k):
    g = np.random.default_rng(R * 100 + T)
    xs = [bf16_random(g, (T, H)) for _ in range(R)]
    idxs = [make_routing(g, T, E, k, mask_frac=0.1)[0] for _ in range(R)]
    in_ranks = [O.get_dispatch_layout(i, E, R)[2] for i in idxs]
    step = refpipe.HTDispatchStep(xs, in_ranks, seed=7)
    recv, comb = step.run()
    out, heads = O.dispatch(xs, in_ranks)
    ref_comb = O.combine([o["recv_x"] for o in out], in_ranks, heads, out[0]["rank_prefix_matrix"])
    for d in range(R):
        assert np.array_equal(recv[d], out[d]["recv_x"]), d
        assert np.array_equal(comb[d], ref_comb[d][0]), d
    step.pool.shutdown()

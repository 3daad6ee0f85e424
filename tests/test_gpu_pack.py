"""GPU parity for Tree Packing (tt_pack): bit-exact against the oracle's recursive DFS and the
brute-force tile classification."""
import numpy as np
import pytest

import oracle
from workloads import trees

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tt():
    import paper_2511_00413_b200 as P
    P.lib()
    return P


def _check_pack(tt, t, tiles=True):
    import torch
    pk = tt.tt_pack(t.parent, t.length, t.term)
    torch.cuda.synchronize()
    a = {k: (v.cpu().numpy() if v is not None else None) for k, v in pk.arrays().items()}
    o = oracle.pack(t.parent, t.length, t.term)
    for k in ("pos", "w", "E", "node"):
        assert np.array_equal(a[k], o[k]), k
    assert np.array_equal(a["node_start"], o["node_start"])
    assert np.array_equal(a["node_sub_end"], o["node_sub_end"])
    assert np.array_equal(a["node_depth"], o["node_depth"])
    assert np.array_equal(a["node_leaves"], o["node_leaves"])
    if tiles:
        cls, mn, mx = oracle.tiles(o, 128)
        assert np.array_equal(a["kblk_minE"], mn)
        assert np.array_equal(a["kblk_maxE"], mx)
        nb = cls.shape[0]
        for qb in range(nb):
            cnt = a["fwd_cnt"][qb]
            ent = a["fwd_list"][qb * (qb + 1) // 2: qb * (qb + 1) // 2 + cnt]
            kbs = ent & ((1 << 28) - 1)
            cl = ent >> 28
            exp_kb = np.flatnonzero(cls[qb])
            assert kbs.tolist() == exp_kb.tolist(), qb
            assert cl.tolist() == cls[qb, exp_kb].tolist(), qb
    return pk, o


@pytest.mark.parametrize("seed", range(30))
def test_pack_random_forests(tt, seed):
    rng = np.random.default_rng(seed)
    t = trees.gen_random_forest(rng, max_nodes=40, max_len=90, with_term=(seed % 3 == 0))
    _check_pack(tt, t)


@pytest.mark.parametrize("name,seed", [("tiny", None), ("agentic8k", 0), ("agentic8k", 1), ("agentic8k", 2),
                                       ("wide", None), ("wide_aligned", None)])
def test_pack_configs(tt, name, seed):
    _check_pack(tt, trees.config_tree(name, seed))


def test_pack_deep32k(tt):
    _check_pack(tt, trees.config_tree("deep32k", 1), tiles=False)


def test_pack_chain_10k_nodes(tt):
    _check_pack(tt, trees.chain(10000, seg=1), tiles=False)


def test_pack_star_and_zero_length(tt):
    _check_pack(tt, trees.Tree([-1, 0, 0, 2, -1, 4, 4], [0, 200, 0, 77, 130, 0, 5]))
    _check_pack(tt, trees.star(300, [1] * 200))


def test_pack_successor_lists(tt):
    """Continuation lists (loss targets at a node's last token) vs the oracle's branch paths."""
    t = trees.Tree([-1, 0, 0, 2, 2, 0], [3, 2, 0, 1, 4, 0], [0, 1, 0, 1, 1, 1])
    pk, o = _check_pack(tt, t, tiles=False)
    a = pk.arrays()
    sp = a["succ_ptr"].cpu().numpy()
    st = a["succ_tok"].cpu().numpy()
    # oracle: the set of next packed indices after the root's last token over all branches
    nxt = set()
    for idx in oracle.paths(o):
        if len(idx) > 3:
            nxt.add(int(idx[3]))
    assert sorted(st[sp[0]:sp[1]].tolist()) == sorted(nxt)


def test_pack_refuses_graph_capture_and_explicit_stream():
    """tt_pack stages its node tables through pinned host buffers: inside a CUDA-graph capture it
    returns TT_ERR_INVALID_ARGUMENT instead of recording a host copy; on an explicit side stream it
    packs exactly what the default stream does."""
    import numpy as np
    import torch
    import paper_2511_00413_b200 as tt
    from workloads import trees
    t = trees.gen_agentic(2000, root_len=300, seed=2)
    ref = tt.tt_pack(t.parent, t.length)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pk = tt.tt_pack(t.parent, t.length, stream=s)
    s.synchronize()
    for key in ("pos", "w", "E", "node", "fwd_cnt"):
        assert torch.equal(pk.arrays()[key], ref.arrays()[key]), key
    g = torch.cuda.CUDAGraph()
    with pytest.raises(tt.TTError) as ei:
        with torch.cuda.graph(g, stream=s):
            tt.tt_pack(t.parent, t.length, stream=s)
    assert ei.value.code == 1
    # many packs in a row reuse the 4 staging slots (each waits only for its slot's previous copy)
    outs = [tt.tt_pack(t.parent, t.length) for _ in range(9)]
    torch.cuda.synchronize()
    assert all(torch.equal(o.arrays()["E"], ref.arrays()["E"]) for o in outs)


@pytest.mark.parametrize("name", ["agentic8k", "deep32k", "wide"])
def test_schedule_statistics(tt, name):
    """tt_pack's host-side CTA-order statistics (include/tt.h: the backward's per-key-block query-tile
    counts nq_kb = ceil(maxE_kb / 64) - 2 kb, their sum and maximum) equal the definition applied to the
    oracle's subtree ends E."""
    t = trees.config_tree(name)
    pk = tt.tt_pack(t.parent, t.length, t.term)
    E = oracle.pack(t.parent, t.length, t.term)["E"].astype(np.int64)
    nb = (len(E) + 127) // 128
    nq = np.array([(int(E[128 * b:128 * b + 128].max()) + 63) // 64 - 2 * b for b in range(nb)])
    assert int(pk.c.sched_sum_nq) == int(nq.sum())
    assert int(pk.c.sched_max_nq) == int(nq.max())
    assert int(pk.c.wr_negative) == 0
    tt.tt_pack_weights(pk, np.full(pk.info["n_traj"], -0.5, np.float32))
    assert int(pk.c.wr_negative) == 1

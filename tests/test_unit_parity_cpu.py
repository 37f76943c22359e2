"""CPU checks of the scale-parity checker (oracle/unit_parity.py) itself:
fed a "device" trajectory that the oracle produced, it must report full
parity, and the real reference (when importable here) must agree with the
oracle step by step; a perturbed trajectory must be flagged."""

import copy

import numpy as np

from oracle import ctkv_oracle as O
from oracle import unit_parity as UP


def _fake_run(seed=5, b=1, h=8, g=2, d=64, s=1536, T=6, C=64, rho=96, cp=4, rp=32):
    q, k, v = O.generate(O.Drift(seed=seed, s=s, decode_steps=T), b, h, g, d)
    q, k, v = O.bf16_round(q), O.bf16_round(k), O.bf16_round(v)
    init, local = 32, 128
    st, ix = O.prefill(q[:, :, :s].copy(), k[:, :, :s].copy(), v[:, :, :s].copy(), init, local, C, rho)
    sn = dict(layer=0, seq=0, total=s, init_len=init, local_len=local,
              keys=st.keys[:, :, :s].copy(), values=st.values[:, :, :s].copy(),
              cent=ix.centroids.copy(), lists=ix.lists.copy(), fifo=ix.fifo_head.copy(), steps=[])
    for t in range(T):
        st.append(k[:, :, s + t], v[:, :, s + t])
        r = O.decode_step(st, ix, q[:, :, s + t], cp, rp)
        sn["steps"].append(dict(q=q[:, :, s + t].copy(), k=k[:, :, s + t].copy(),
                                v=v[:, :, s + t].copy(), out=r.out[0].copy(),
                                selected=r.selected[0].copy(), recall_len=np.array([len(x) for x in r.recalled[0]]),
                                sparse=[np.asarray(x) for x in r.sparse[0]]))
    sn["cent_final"] = ix.centroids.copy()
    sn["lists_final"] = ix.lists.copy()
    sn["fifo_final"] = ix.fifo_head.copy()
    return sn, cp, rp


def test_checker_accepts_identical_trajectory():
    sn, cp, rp = _fake_run()
    res = UP.check([sn], cp, rp)
    assert res["ok"], res
    assert res["recall"] == 1.0 and res["exact_steps"] == res["steps"] == 6
    assert res["dcu_rows"] == 6 * 2 and res["dcu_rows_exact"] == res["dcu_rows"]
    if res["reference"] is not None:           # the real package agrees with the oracle
        assert res["ref_vs_oracle_digest_mismatch"] == 0
        assert res["ref_vs_oracle_out_nrel_max"] < 1e-6
        assert len(res["ref_times"]) == 4


def test_checker_flags_a_wrong_sparse_set_and_dcu_row():
    sn, cp, rp = _fake_run(seed=6)
    bad = copy.deepcopy(sn)
    sp = bad["steps"][3]["sparse"][1]
    sp[-1] = -7                                  # an id the reference never selected
    bad["lists_final"][0, 0, int(sn["fifo"][0] % 64)][:5] = 1   # corrupt a DCU row
    res = UP.check([bad], cp, rp, use_reference=False)
    assert not res["ok"]
    assert res["hard_mismatches"] >= 1 and res["dcu_hard"] >= 1

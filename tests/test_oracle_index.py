"""Pins for the oracle's canonical join index (O1) -- CPU only.

The oracle sorts (key,row) pairs and binary-searches them; these tests compare it with an
independent brute-force nested-loop natural join (sec 2.2 "pairing tuples
... that agree on all shared attributes") followed by a dictionary group-by
(PAPER.md:332-340), i.e. the plain relational definitions, on many random tiny databases
that include dangling keys, negative keys, repeated E tuples, empty relations and hubs.
"""
import numpy as np
import pytest

import synth


def brute_force_index(e_src, e_dst, s_key, t_key, by_src_key=False):
    n_e = len(e_dst)
    rows = []
    for j in range(n_e):                       # nested-loop natural join
        s_row = -1
        if s_key is not None:
            hits = [i for i in range(len(s_key)) if s_key[i] == e_src[j]]
            if not hits:
                continue
            s_row = hits[0]
        if t_key is not None and not any(t_key[i] == e_dst[j] for i in range(len(t_key))):
            continue
        rows.append((int(e_dst[j]), j, s_row))
    groups = {}
    for t, j, s_row in rows:                   # group by t
        groups.setdefault(t, []).append((j, s_row))
    group_key, group_ptr, src_row, edge_row, group_dst_row = [], [0], [], [], []
    for t in sorted(groups):
        members = groups[t]
        if by_src_key:
            members = sorted(members, key=lambda m: (int(e_src[m[0]]), m[0]))
        else:
            members = sorted(members)
        for j, s_row in members:
            edge_row.append(j)
            src_row.append(s_row)
        group_key.append(t)
        group_ptr.append(len(edge_row))
        if t_key is not None:
            group_dst_row.append([i for i in range(len(t_key)) if t_key[i] == t][0])
        else:
            group_dst_row.append(-1)
    out = {"group_key": group_key, "group_ptr": group_ptr, "src_row": src_row,
           "edge_row": edge_row, "group_dst_row": group_dst_row}
    if s_key is not None:
        src_pos, src_ptr = [], [0]
        for i in range(len(s_key)):
            src_pos += [p for p in range(len(src_row)) if src_row[p] == i]
            src_ptr.append(len(src_pos))
        out["src_pos"], out["src_ptr"] = src_pos, src_ptr
    return out


def assert_same(idx, bf):
    for k, v in bf.items():
        got = idx[k]
        assert list(np.asarray(got).tolist()) == list(v), k


@pytest.mark.parametrize("seed", range(300))
def test_index_matches_nested_loop_join(ora, seed):
    rng = np.random.default_rng(seed)
    n_s, n_t, n_e = (int(x) for x in rng.integers(0, 12, size=3))
    n_e = int(rng.integers(0, 40))
    db = synth.random_db(rng, n_s, n_t, n_e, key_space=int(rng.integers(8, 40)))
    use_s = seed % 5 != 1
    use_t = seed % 3 != 2
    by_key = seed % 7 == 3
    s_key = db["s_key"] if use_s else None
    t_key = db["t_key"] if use_t else None
    idx = ora.build_join_index(db["e_src"], db["e_dst"], s_key, t_key, within_by_src_key=by_key)
    bf = brute_force_index(db["e_src"], db["e_dst"], s_key, t_key, by_key)
    assert_same(idx, bf)
    # invariants (SURVEY sec 8c pins (iii))
    gp = idx["group_ptr"]
    assert gp[0] == 0 and gp[-1] == idx["n_join_rows"] and np.all(np.diff(gp) > 0)
    assert np.all(np.diff(idx["group_key"]) > 0)
    if use_s:
        assert sorted(idx["src_pos"].tolist()) == list(range(idx["n_join_rows"]))
        for i in range(len(db["s_key"])):
            for q in range(idx["src_ptr"][i], idx["src_ptr"][i + 1]):
                assert idx["src_row"][idx["src_pos"][q]] == i


def test_duplicate_key_is_an_error(ora):
    with pytest.raises(ora.OracleError, match="duplicate"):
        ora.build_join_index([1, 2], [3, 3], s_key=[1, 2, 1], t_key=[3])
    with pytest.raises(ora.OracleError, match="duplicate"):
        ora.build_join_index([1, 2], [3, 3], s_key=[1, 2], t_key=[3, 3])


def test_empty_relations(ora):
    idx = ora.build_join_index(np.zeros(0, np.int64), np.zeros(0, np.int64), [1, 2], [3])
    assert idx["n_join_rows"] == 0 and idx["n_groups"] == 0 and idx["group_ptr"].tolist() == [0]
    assert idx["src_ptr"].tolist() == [0, 0, 0]
    idx = ora.build_join_index([5, 6], [7, 8], np.zeros(0, np.int64), [7, 8])
    assert idx["n_join_rows"] == 0


def test_permutation_of_edge_rows(ora):
    """Permuting E's rows permutes edge_row consistently and leaves group_key unchanged."""
    rng = np.random.default_rng(7)
    db = synth.random_db(rng, 30, 20, 200)
    a = ora.build_join_index(db["e_src"], db["e_dst"], db["s_key"], db["t_key"])
    perm = rng.permutation(200)
    b = ora.build_join_index(db["e_src"][perm], db["e_dst"][perm], db["s_key"], db["t_key"])
    assert a["group_key"].tolist() == b["group_key"].tolist()
    assert a["group_ptr"].tolist() == b["group_ptr"].tolist()
    for g in range(a["n_groups"]):
        lo, hi = a["group_ptr"][g], a["group_ptr"][g + 1]
        assert sorted(a["edge_row"][lo:hi].tolist()) == sorted(perm[b["edge_row"][lo:hi]].tolist())


def test_hub_and_sparse_63bit_keys(ora):
    rng = np.random.default_rng(3)
    s_key = rng.choice(2 ** 62, size=50, replace=False).astype(np.int64) - 2 ** 61
    t_key = np.array([-(2 ** 63), 2 ** 63 - 1, 0], np.int64)
    e_src = s_key[rng.integers(0, 50, 500)]
    e_dst = t_key[np.minimum(rng.integers(0, 4, 500), 2)]   # one hub group
    idx = ora.build_join_index(e_src, e_dst, s_key, t_key)
    bf = brute_force_index(e_src, e_dst, s_key, t_key)
    assert_same(idx, bf)
    assert idx["group_key"].tolist() == [-(2 ** 63), 0, 2 ** 63 - 1]

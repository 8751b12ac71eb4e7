"""Textual / structured layout surface (exported through the
C-ABI): parse / format of the paper's matrix notation, JSON, and canonical
equivalence -- checked against the paper's printed layouts and, on random
layouts, against brute-force set comparison of the induced maps by the
independent oracle (no GPU)."""
import numpy as np
import pytest

import oracle
from synth import layout

import paper_2601_19092_b200 as axe

TC_TEXT = "(8,2,4,2):(4@lane,1@warp,1@lane,1@reg) + [(2):(4@warp)] + 5@warp"


def spec_of(L):
    return layout(L.iters(0), L.iters(1), L.offset())


def same_map(a, b):
    """Oracle brute force: equal domains and f_a(x) == f_b(x) as sets for every x."""
    ea, eb = oracle.sizes(a)[0], oracle.sizes(b)[0]
    return ea == eb and all(oracle.eval_set(a, x) == oracle.eval_set(b, x) for x in range(ea))


def test_parse_paper_layouts():
    """§2.2 tensor-core tile and the §3.3 tile result in the paper's notation."""
    L = axe.Layout.parse(TC_TEXT)
    assert L.iters(0) == [(8, 4, "lane"), (2, 1, "warp"), (4, 1, "lane"), (2, 1, "reg")]
    assert L.iters(1) == [(2, 4, "warp")] and L.offset() == {"warp": 5}
    assert {c["warp"] for c in L.eval(0)} == {5, 9}
    T = axe.Layout.parse("(2, 8, 3, 8) : (192, 8, 64, 1)")          # whitespace is insignificant
    assert T.iters(0) == [(2, 192, "m"), (8, 8, "m"), (3, 64, "m"), (8, 1, "m")]
    S = axe.Layout.parse("(1,8,2,8):(192,8,64,1) + 64@m")             # the slice example
    assert S.offset() == {"m": 64}
    assert axe.Layout.parse("(4):(1) + 3@m + 5@m").offset() == {"m": 8}  # repeated offsets add
    assert axe.Layout.parse("(3):(-2)").iters(0) == [(3, -2, "m")]


@pytest.mark.parametrize("text,pos", [("(2,3):(3,0)", -1), ("(0):(1)", -1), ("(2,3):(3)", None), ("(2):(1) +", None),
                                      ("(2):(1) junk", None), ("(2):(1@9x)", None), ("(2):(1) + 4", None),
                                      ("(2):(1) + 1@m + [(2):(1)]", None), ("", None)])
def test_parse_errors(text, pos):
    with pytest.raises(axe.AxeError) as e:
        axe.Layout.parse(text)
    assert e.value.name == "AXE_ERR_INVALID_ARG"
    if pos is not None:
        assert e.value.pos == pos
    else:
        assert 0 <= e.value.pos <= len(text)


def rand_layout(rng, axes=("m", "lane", "warp")):
    nd, nr = int(rng.integers(1, 5)), int(rng.integers(0, 3))
    it = lambda: (int(rng.integers(1, 6)), int(rng.choice([-1, 1]) * rng.integers(1, 33)), str(rng.choice(axes)))
    O = {str(a): int(rng.integers(-9, 10)) for a in rng.choice(axes, size=int(rng.integers(0, 3)))}
    return layout([it() for _ in range(nd)], [it() for _ in range(nr)], {a: v for a, v in O.items() if v})


def test_format_parse_round_trip_random():
    rng = np.random.default_rng(1)
    for _ in range(300):
        spec = rand_layout(rng)
        L = axe.Layout(spec["D"], spec["R"], spec["O"])
        P = axe.Layout.parse(L.format())
        assert P.iters(0) == L.iters(0) and P.iters(1) == L.iters(1) and P.offset() == L.offset()
        j = L.to_json()
        assert j["schema_version"] == 1 and j["text"] == L.format()
        assert [tuple(x) for x in j["shard"]] == L.iters(0) and [tuple(x) for x in j["replica"]] == L.iters(1)
        assert j["offset"] == L.offset() and j["E_D"] == L.E_D and j["E_R"] == L.E_R


def test_equivalence_spec_examples():
    """SPEC canonicalizer examples: (2,8):(8,1) = (16):(1); (2,2):(4,1) != (4):(1) (images {0,1,4,5} vs
    {0,1,2,3}); App. F: the direct sum (2,2):(8,2) (+) (2,2):(4,1) is the contiguous (16):(1)."""
    eq = lambda a, b: axe.Layout.parse(a).equivalent(axe.Layout.parse(b))
    assert eq("(2,8):(8,1)", "(16):(1)") is True
    assert eq("(2,2):(4,1)", "(4):(1)") is False
    S = axe.Layout([(2, 8), (2, 2)]).direct_sum([2, 2], axe.Layout([(2, 4), (2, 1)]), [2, 2])
    assert S.equivalent(axe.Layout.parse("(16):(1)")) is True
    assert eq("(4):(1)", "(2):(1)") is False                        # different domains
    assert eq("(3):(-2)", "(3):(-2)") is True
    assert eq(TC_TEXT, "(8,2,4,2):(4@lane,1@warp,1@lane,1@reg) + [(2):(4@warp)] + 5@warp") is True
    assert eq(TC_TEXT, "(8,2,4,2):(4@lane,1@warp,1@lane,1@reg) + [(2):(4@warp)] + 6@warp") is False


def perturb(rng, spec):
    """Semantics-preserving rewrites (SPEC canonicalizer property suite): split a shard iter (Lemma split,
    P:1016-1026), flip a replica stride with offset compensation (rule C1), split a replica iter into two
    whose C2 merge reproduces it (rule C2, q = E1)."""
    D, R, O = list(spec["D"]), list(spec["R"]), dict(spec["O"])
    for _ in range(int(rng.integers(1, 6))):
        k = int(rng.integers(0, 3))
        if k == 0:
            i = int(rng.integers(0, len(D)))
            e, s, a = D[i]
            divs = [d for d in range(2, e) if e % d == 0]
            if divs:
                d = int(rng.choice(divs))
                D[i:i + 1] = [(e // d, s * d, a), (d, s, a)]
        elif k == 1 and R:
            i = int(rng.integers(0, len(R)))
            e, s, a = R[i]
            R[i] = (e, -s, a)
            O[a] = O.get(a, 0) + (e - 1) * s
        elif k == 2 and R:
            i = int(rng.integers(0, len(R)))
            e, s, a = R[i]
            divs = [d for d in range(2, e) if e % d == 0]
            if divs:
                d = int(rng.choice(divs))               # (d, s) + (e/d, d s) covers {0..e-1} s
                R[i:i + 1] = [(d, s, a), (e // d, d * s, a)]
    return layout(D, R, {a: v for a, v in O.items() if v})


def test_equivalence_under_perturbation_random():
    rng = np.random.default_rng(2)
    for _ in range(300):
        spec = rand_layout(rng)
        L = axe.Layout(spec["D"], spec["R"], spec["O"])
        Q = perturb(rng, spec)
        got = L.equivalent(axe.Layout(Q["D"], Q["R"], Q["O"]))
        assert got is True, (spec, Q)
        C = L.canonicalize()[0]
        assert L.equivalent(C) is True


def test_equivalence_decision_matches_brute_force():
    """Random pairs that differ in one stride / extent / offset: the library's decision (structural or
    enumerated) equals the oracle's pointwise set comparison."""
    rng = np.random.default_rng(3)
    n_true = n_false = 0
    for _ in range(400):
        a = rand_layout(rng, axes=("m", "lane"))
        b = {"D": list(a["D"]), "R": list(a["R"]), "O": dict(a["O"])}
        k = int(rng.integers(0, 4))
        if k == 0:
            i = int(rng.integers(0, len(b["D"])))
            e, s, ax = b["D"][i]
            b["D"][i] = (e, s + int(rng.choice([-1, 1])) or 1, ax)
        elif k == 1:
            b = perturb(rng, a)
        elif k == 2:
            b["O"] = {**b["O"], "m": b["O"].get("m", 0) + 1}
        else:
            i = int(rng.integers(0, len(b["D"])))
            e, s, ax = b["D"][i]
            j = int(rng.integers(0, len(b["D"])))
            b["D"][i], b["D"][j] = b["D"][j], b["D"][i]
        A, B = axe.Layout(a["D"], a["R"], a["O"]), axe.Layout(b["D"], b["R"], b["O"])
        got = A.equivalent(B)
        exp = same_map(a, layout(B.iters(0), B.iters(1), B.offset()))
        assert got == exp, (a, b)
        n_true += exp
        n_false += not exp
    assert n_true > 50 and n_false > 50


def test_equivalence_undecidable_without_gap_condition():
    """R = [(2,2),(2,3)] fails the gap condition (3 > 2*2 is false) and C2 cannot absorb it (3 is not a
    multiple of 2): above the enumeration threshold the answer is 'undecidable' (None), below it the
    pointwise comparison decides -- here between two orders of the same replica multiset and a
    different one."""
    a = axe.Layout.parse("(64):(8) + [(2,2):(2,3)]")
    b = axe.Layout.parse("(64):(8) + [(2,2):(3,2)]")
    c = axe.Layout.parse("(64):(8) + [(2,2):(3,1)]")
    assert a.canonicalize()[1] is False
    assert a.equivalent(b, threshold=10) is None
    assert a.equivalent(b) is True and a.equivalent(c) is False

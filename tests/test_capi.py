"""Host-side tests of libwino.so (no GPU): the library loads, exports every
symbol include/wino.h declares, and its exact C++ generator produces the same
rationals as the independent oracle (and bit-identical fp32 lowerings)."""
import ctypes
import os
import re
from fractions import Fraction as Fr

import numpy as np
import pytest

import paper_1905_05233_b200 as W
from paper_1905_05233_b200._lib import LIB_PATH, WinoError
from oracle import precision as P
from oracle import transforms as T

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "wino.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wino_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_symbol():
    assert os.path.exists(LIB_PATH)
    L = ctypes.CDLL(LIB_PATH)
    syms = _declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(L, s), s


CONFIGS = [("0,1,-1,inf", 2), ("0,-1,1,-1/2,1/2,inf", 4), ("0,1,-1,2,-2,inf", 4), ("0,a^2+1,inf", 2),
           ("0,-1,a^2+1,inf", 3), ("0,-1,1,a^2+1,inf", 4), ("a^2+1,a^2-2", 2), ("a^3-2,inf", 2), ("a^4+1", 2),
           ("0,a^2+a+1,inf", 2), ("0,-1,1,a^2-a+1,inf", 4), ("0,-1,1,a^2+1,a^2-2,inf", 6),
           ("0,1,a^3+a+1,inf", 4), ("0,a^4+1,inf", 4), ("a^3+2,a^2+1,inf", 4)]
CANON = ["lin2", "lin3", "lin4", "lin5", "lin6", "lin7", "lin8", "sup1_2", "sup1_3", "sup1_4", "sup1_5", "sup1_6",
         "sup1_7", "sup1_8", "sup2_2", "sup2_4", "sup2_6", "sup2_8", "lin10", "sup1_10", "sup1_12", "sup2_12"]


def _cases():
    out = list(CONFIGS)
    for name in CANON:
        mods, m = T.canonical(name)
        out.append((T.moduli_spec(mods), m))
    return out


def _fr(M):
    return [[Fr(v) for v in r] for r in M]


@pytest.mark.parametrize("spec,m", _cases())
def test_generator_matches_oracle_subsolver(spec, m):
    a = W.WinoAlgo(spec, m)
    ts = T.make_transforms(spec, m)
    assert a.mu == ts.mu == a.domain and a.units == ts.mu ** 2
    assert a.ratio_2d == pytest.approx(float(T.ratio(ts.moduli, m)))
    for which, ref in (("G", ts.G), ("B", ts.B), ("A", ts.A)):
        exact, f32 = a.matrix(which)
        assert exact == _fr(ref), which
        assert np.array_equal(f32.view(np.uint32), P.lower_f32(ref).view(np.uint32)), which


@pytest.mark.parametrize("name", ["lin4", "sup1_2", "sup1_4", "sup1_6", "sup1_8", "sup2_4", "sup2_6"])
def test_generator_matches_oracle_residue(name):
    mods, m = T.canonical(name)
    a = W.WinoAlgo(T.moduli_spec(mods), m, lowering="residue")
    rb = T.residue_blocks(mods, m)
    assert a.domain == rb.D == m + 2 or not any(x.is_inf for x in mods)
    assert a.units == rb.units_1d ** 2
    for which, ref in (("G", rb.GP), ("B", rb.BP), ("A", rb.AP)):
        exact, f32 = a.matrix(which)
        assert exact == _fr(ref), which
        assert np.array_equal(f32.view(np.uint32), P.lower_f32(ref).view(np.uint32)), which
    out_pt, in_pt, nterm, ta, coef = a.unit_table()
    units = P.residue_slabs(rb)
    assert len(units) == a.units
    for u, (po, pi, (sI, nI, phI), (sJ, nJ, phJ), (k, l, kk, ll)) in enumerate(units):
        assert out_pt[u] == po and in_pt[u] == pi
        terms = []
        for aa in range(nI):
            for bb in range(nJ):
                cf = phI[aa][kk][k] * phJ[bb][ll][l]
                if cf != 0:
                    terms.append(((sI + aa) * rb.D + (sJ + bb), float(cf)))
        assert nterm[u] == len(terms)
        assert [(int(ta[u][j]), coef[u][j]) for j in range(nterm[u])] == terms


def test_worked_example_sub_points():
    a = W.WinoAlgo("0,a^2+1,inf", 2, sub_points="0,1,inf")
    ts = T.make_transforms("0,a^2+1,inf", 2, 3, T.parse_points("0,1,inf"))
    assert a.matrix("B")[0] == _fr(ts.B) and a.matrix("G")[0] == _fr(ts.G)


def test_parse_moduli():
    mods = W.wino_parse_moduli("0, -1, 1/2, a^2+1, a+1, inf, 2*a^2-1")
    assert [m.degree for m in mods] == [1, 1, 1, 2, 1, 0, 2]
    assert (mods[2].num[0], mods[2].den[0]) == (1, 2)
    assert (mods[4].num[0], mods[4].den[0]) == (-1, 1)          # a + 1 -> point -1
    assert [(mods[6].num[k], mods[6].den[k]) for k in range(3)] == [(-1, 2), (0, 1), (1, 1)]   # monic


@pytest.mark.parametrize("spec,m,status,needle", [
    ("0,a^2+a,inf", 2, 2, "reducible"),
    ("1,1,-1,inf", 2, 2, "coprime"),
    ("0,-1,inf", 2, 2, "degree budget"),
    ("0,inf,-1,1", 2, 2, "last"),
    ("0,-1,1,inf", 13, 4, "2 <= m <= 12"),
    ("0,-1,1,-1/2,1/2,2,-2,-1/4,4,1/4,-4,a^2+1,inf", 8, 2, "budget"),
])
def test_config_errors(spec, m, status, needle):
    with pytest.raises(WinoError) as ei:
        W.WinoAlgo(spec, m)
    assert ei.value.status == status and needle in str(ei.value)


def test_mu_limit_and_residue_degree_limit():
    with pytest.raises(WinoError) as ei:
        W.WinoAlgo("a^3-2,inf", 2, lowering="residue")
    assert ei.value.status == 2
    # r != 3 unsupported
    mods, n = W.api._moduli_array("0,1,-1,inf")
    h = ctypes.c_void_p()
    assert W.lib().wino_make_transforms(mods, n, 2, 5, None, 0, 0, ctypes.byref(h)) == 4


def test_workspace_geometry():
    a = W.WinoAlgo("0,-1,1,-1/2,1/2,inf", 4)
    nb = W.wino_conv2d_workspace(a, 256, 512, 28, 28, 512, 1, "bf16")
    g = W.geometry(a, 256, 512, 28, 28, 512, 1, "bf16")
    assert g["T"] == 12544 and g["Q"] == 36 and g["Cp"] == 512
    expect = 36 * 512 * 512 * 2 + 36 * 12544 * 512 * 2 + 36 * 512 * 12544 * 4
    assert expect <= nb <= expect + 3 * 1024
    with pytest.raises(WinoError):
        W.wino_conv2d_workspace(a, 1, 8, 16, 16, 8, 2, "bf16")      # pad must be 0 or 1


def test_named_sets_match_oracle_canonical():
    from paper_1905_05233_b200.algos import canonical_spec
    for name in CANON:
        spec, m = canonical_spec(name)
        mods, m2 = T.canonical(name)
        assert m == m2 and [str(x) for x in T.parse_moduli(spec)] == [str(x) for x in mods]


@pytest.mark.parametrize("name", ["lin2", "lin4", "lin6", "lin8", "sup1_4", "sup1_6", "sup1_8", "sup2_6", "sup2_8"])
def test_scaled_generator_matches_oracle(name):
    """wino_scale_transforms (C++) and oracle.transforms.scale_pow2_balance
    (Python) apply the same exact power-of-two balancing independently."""
    from oracle.transforms import canonical, make_transforms, moduli_spec, scale_pow2_balance
    mods, m = canonical(name)
    a = W.WinoAlgo(moduli_spec(mods), m).scale("pow2")
    tss = scale_pow2_balance(make_transforms(mods, m))
    for which, ref in (("G", tss.G), ("B", tss.B), ("A", tss.A)):
        exact, f32 = a.matrix(which)
        assert exact == _fr(ref), which
        assert np.array_equal(f32.view(np.uint32), P.lower_f32(ref).view(np.uint32)), which


def test_scale_errors():
    a = W.WinoAlgo("0,-1,1,inf", 2)
    a.scale("none")
    a.scale("pow2")
    with pytest.raises(W.WinoError) as e:
        a.scale("pow2")
    assert e.value.status == 1
    r = W.WinoAlgo("0,a^2+1,inf", 2, lowering="residue")
    with pytest.raises(W.WinoError) as e:
        r.scale("pow2")
    assert e.value.status == 4


def test_bt_masks_header_in_sync():
    """csrc/bt_masks.hpp (B^T zero patterns and +-row pairs baked into K1) equals what
    scripts/gen_bt_masks.py derives from the generator now; a stale header would only
    cost speed (the runtime key would not match), this keeps it honest."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "gen_bt_masks.py"), "--check"], cwd=root)
    assert r.returncode == 0

"""Named polynomial sets (canonical sets) as moduli strings for
wino_make_transforms.  Points: PAPER.md P:533 ("0, -1, 1, -1/2, 2, 1/2, -2,
-1/4, 4"), reordered so the first five are BASELINE cfg3's {0, +-1, +-1/2}.

  lin(m)  = P[:m+1] + {inf}                 mu = m + 2   (Toom-Cook)
  sup1(m) = P[:m-1] + {a^2+1, inf}           mu = m + 3
  sup2(m) = P[:m-3] + {a^2+1, a^2-2, inf}    mu = m + 4   (m = 2: {a^2+1, a^2-2})
"""
import re

POINTS = ["0", "-1", "1", "-1/2", "1/2", "2", "-2", "-1/4", "4", "1/4", "-4"]   # + 1/4, -4: reading A21


def canonical_spec(name):
    mt = re.fullmatch(r"(lin|sup1|sup2)_?(\d+)", name)
    if not mt:
        raise ValueError(f"unknown algorithm name {name!r} (lin<m>, sup1_<m>, sup2_<m>)")
    fam, m = mt.group(1), int(mt.group(2))
    if fam == "lin":
        mods = POINTS[:m + 1] + ["inf"]
    elif fam == "sup1":
        mods = POINTS[:m - 1] + ["a^2+1", "inf"]
    else:
        mods = ["a^2+1", "a^2-2"] if m == 2 else POINTS[:m - 3] + ["a^2+1", "a^2-2", "inf"]
    return ",".join(mods), m

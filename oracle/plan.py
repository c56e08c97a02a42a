"""oracle/plan.py -- TEST INFRASTRUCTURE ONLY (never imported by the product path).

Plain-Python statement of the integer steps of the method, written out in the paper's order
and notation, used to check the C++ planner element by element:

  a1 classify()        index bundles I (A∩C), J (B∩C), P (A∩B)           P:262-298 §4
  a2 normalize()       the five-step heuristic of §7.3
  a3 scatter()         scatter vectors rscat/cscat                        P:528-580 §6.1
  a4 block_scatter()   block-scatter vectors rbs/cbs                      P:678-683 §6.2

Readings where the paper is silent (DESIGN.md §Readings R3, R4, R6, R9, R10, R11) are marked
inline. Nothing here is blocked, vectorised or reordered beyond what the paper states.
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple


class LabelError(ValueError):
    pass


class ShapeError(ValueError):
    pass


Dim = Dict[str, object]   # {"labels": str, "len": int, "stride": {"A": s, "B": s, "C": s}}


def classify(lab_a: str, lens_a: Sequence[int], str_a: Sequence[int],
             lab_b: str, lens_b: Sequence[int], str_b: Sequence[int],
             lab_c: str, lens_c: Sequence[int], str_c: Sequence[int]):
    """Step a1: I = labels in A and C, J = labels in B and C,
    P = labels in A and B. Every label must appear in exactly two tensors, once each (R6);
    lengths of a shared label must agree. Bundle order: I and P in A's label
    order, J in B's label order (the order is a choice the paper leaves open, P:265-275;
    the heuristic below reorders anyway)."""
    for lab in (lab_a, lab_b, lab_c):
        if len(set(lab)) != len(lab):
            raise LabelError(f"repeated label in {lab!r}")
    la = {x: (int(n), int(s)) for x, n, s in zip(lab_a, lens_a, str_a)}
    lb = {x: (int(n), int(s)) for x, n, s in zip(lab_b, lens_b, str_b)}
    lc = {x: (int(n), int(s)) for x, n, s in zip(lab_c, lens_c, str_c)}
    for x in set(lab_a) | set(lab_b) | set(lab_c):
        count = (x in la) + (x in lb) + (x in lc)
        if count != 2:
            raise LabelError(f"label {x!r} appears in {count} tensor(s), must be 2")
    I, J, P = [], [], []
    for x in lab_a:
        if x in lc:
            if la[x][0] != lc[x][0]:
                raise ShapeError(f"length mismatch for {x!r}")
            I.append({"labels": x, "len": la[x][0], "stride": {"A": la[x][1], "C": lc[x][1]}})
        else:
            if la[x][0] != lb[x][0]:
                raise ShapeError(f"length mismatch for {x!r}")
            P.append({"labels": x, "len": la[x][0], "stride": {"A": la[x][1], "B": lb[x][1]}})
    for x in lab_b:
        if x in lc:
            if lb[x][0] != lc[x][0]:
                raise ShapeError(f"length mismatch for {x!r}")
            J.append({"labels": x, "len": lb[x][0], "stride": {"B": lb[x][1], "C": lc[x][1]}})
    return I, J, P


def _fold(bundle: List[Dim]) -> List[Dim]:
    """Step 2: fold dimensions that are sequentially contiguous in all tensors.
    Reading R9: dims u, v fold (v after u) iff stride_v(T) == stride_u(T) * n_u for every
    tensor T carrying the bundle (the definition of sequential contiguity); the
    folded dim keeps u's strides and has length n_u * n_v. Pairs are searched u-major in the
    bundle's current order and the search repeats until no pair folds."""
    dims = [dict(d, stride=dict(d["stride"])) for d in bundle]
    changed = True
    while changed:
        changed = False
        for iu, u in enumerate(dims):
            for iv, v in enumerate(dims):
                if iu == iv:
                    continue
                if all(v["stride"][t] == u["stride"][t] * u["len"] for t in u["stride"]):
                    u["labels"] = u["labels"] + v["labels"]
                    u["len"] = u["len"] * v["len"]
                    del dims[iv]
                    changed = True
                    break
            if changed:
                break
    return dims


def normalize(I: List[Dim], J: List[Dim], P: List[Dim]):
    """The heuristic of P:926-934, steps in the paper's order:
      1. remove dimensions of length one;
      2. fold sequentially contiguous dimensions (R9, see _fold);
      3. sort I and J by increasing stride in C (R10: key |stride|, stable);
      4. if s_{j0}(C) = 1, swap A with B and I with J;
      5. sort P by increasing stride in A (R10: key |stride|, stable; A after the swap).
    Returns (I, J, P, swapped). After a swap the per-dim stride dicts are relabelled so that
    "A" always names the operand that carries the (new) I bundle."""
    I = [d for d in I if d["len"] != 1]
    J = [d for d in J if d["len"] != 1]
    P = [d for d in P if d["len"] != 1]
    I, J, P = _fold(I), _fold(J), _fold(P)
    I = sorted(I, key=lambda d: abs(d["stride"]["C"]))
    J = sorted(J, key=lambda d: abs(d["stride"]["C"]))
    swapped = False
    if J and J[0]["stride"]["C"] == 1:
        swapped = True
        I, J = J, I
        ren = {"A": "B", "B": "A", "C": "C"}
        I = [dict(d, stride={ren[t]: s for t, s in d["stride"].items()}) for d in I]
        J = [dict(d, stride={ren[t]: s for t, s in d["stride"].items()}) for d in J]
        P = [dict(d, stride={ren[t]: s for t, s in d["stride"].items()}) for d in P]
    P = sorted(P, key=lambda d: abs(d["stride"]["A"]))
    return I, J, P, swapped


def scatter(dims: Sequence[Tuple[int, int]]) -> List[int]:
    """Step a3 (generic form P:577-579 read as R3): for a bundle with ordered dims
    (n_0, s_0), (n_1, s_1), ..., scat_k = sum_d digit_d(k) * s_d where the digits decode k
    colexicographically (first dim fastest). An empty bundle has one entry, 0."""
    total = 1
    for n, _ in dims:
        total *= n
    out = []
    for k in range(total):
        off, q = 0, k
        for n, s in dims:
            off += (q % n) * s
            q //= n
        out.append(off)
    return out


def block_scatter(scat: Sequence[int], b: int) -> List[int]:
    """Step a4: entry i is s > 0 if scat_j - scat_{j-1} = s for all
    i*b < j < min(l, (i+1)*b), else 0. Reading R11: a block holding a single entry has no
    difference to test and gets s = 1; zero or negative common differences
    are not "s > 0" and give 0."""
    l = len(scat)
    out = []
    for i in range((l + b - 1) // b):
        lo, hi = i * b, min(l, (i + 1) * b)
        if hi - lo == 1:
            out.append(1)
            continue
        s = scat[lo + 1] - scat[lo]
        ok = s > 0 and all(scat[j] - scat[j - 1] == s for j in range(lo + 1, hi))
        out.append(s if ok else 0)
    return out


def plan_tables(lab_a, lens_a, str_a, lab_b, lens_b, str_b, lab_c, lens_c, str_c):
    """a1 -> a2 -> a3: the six scatter vectors of the normalised plan, in the roles after the
    swap: rscat_A, cscat_A, rscat_B, cscat_B, rscat_C, cscat_C."""
    I, J, P = classify(lab_a, lens_a, str_a, lab_b, lens_b, str_b, lab_c, lens_c, str_c)
    I, J, P, swapped = normalize(I, J, P)
    t = lambda bundle, who: scatter([(d["len"], d["stride"][who]) for d in bundle])  # noqa: E731
    return {
        "I": I, "J": J, "P": P, "swapped": swapped,
        "rscat_A": t(I, "A"), "cscat_A": t(P, "A"),
        "rscat_B": t(P, "B"), "cscat_B": t(J, "B"),
        "rscat_C": t(I, "C"), "cscat_C": t(J, "C"),
    }

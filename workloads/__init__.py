"""Seeded synthetic inputs for the BASELINE.json configs — shared by the oracle side and the
CUDA side, and holding none of the contraction's arithmetic (no bundle classification, no
folding, no scatter tables, no products).

Every tensor is stored in *general column-major order* over its own label order: the first
label is the fastest-varying dimension (§5). Values are drawn in storage
order from a seeded `torch.Generator`, A first, then B, then C
(seed = 1607000 + 100*config + case).

Configs (BASELINE.json `configs`, in order):
  cfg1  tiny rank-4            C_abcd = A_aebf * B_dfce, all lengths 8, U[-1,1], a=1, b=0 (C = NaN)
  cfg2  GEMM sanity            C_mn = A_mk * B_kn (and A_km, B_nk storage), 2048^3, a=1, b=0.5
  cfg3  CC ladder              C_abij += A_abef * B_efij, a..f=128, i,j=32, N(0,1), a=0.5, b=1
                               (variant: C stored as C_aibj)
  cfg4  20 random contractions (P:1159-1165 generator; reading in DESIGN.md), fp64 and fp32
  cfg5  rank-6                 C_abcijk = A_abdilm * B_dclmjk, a-d=48, i-m=24, N(0,1), b=0
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

SEED_BASE = 1607000


@dataclasses.dataclass
class Case:
    """One contraction instance: labels (storage order) + lengths + scalars + distributions."""
    name: str
    lab_c: str
    lab_a: str
    lab_b: str
    lens: Dict[str, int]
    dtype: torch.dtype = torch.float64
    dist: str = "uniform"          # 'uniform' (U[-1,1]) | 'normal' (N(0,1)) | 'int' (integers in [-4,4])
    alpha: float = 1.0
    beta: float = 0.0
    c_init: str = "nan"            # 'nan' | 'dist' (same distribution as A/B) | 'zero'
    seed: int = SEED_BASE

    @property
    def spec(self) -> str:
        """Index string in the paper's C-A-B order."""
        return f"{self.lab_c}-{self.lab_a}-{self.lab_b}"

    def shape(self, labels: str) -> List[int]:
        return [self.lens[x] for x in labels]

    def mnk(self):
        """Products of the free/bound extents (for flop counting only)."""
        m = math.prod(self.lens[x] for x in self.lab_a if x in self.lab_c)
        n = math.prod(self.lens[x] for x in self.lab_b if x in self.lab_c)
        k = math.prod(self.lens[x] for x in self.lab_a if x in self.lab_b)
        return m, n, k

    def flops(self) -> int:
        m, n, k = self.mnk()
        return 2 * m * n * k

    def scaled(self, new_lens: Dict[str, int], name: Optional[str] = None) -> "Case":
        return dataclasses.replace(self, lens=dict(new_lens), name=name or self.name + "_scaled")


def colmajor_strides(lens: Sequence[int]) -> List[int]:
    """General column-major strides: s_0 = 1, s_k = prod_{j<k} n_j."""
    s, out = 1, []
    for n in lens:
        out.append(s)
        s *= max(int(n), 1)
    return out


def colmajor_view(flat: torch.Tensor, lens: Sequence[int]) -> torch.Tensor:
    """View a flat buffer as a tensor of shape `lens` with column-major strides."""
    return flat.as_strided(tuple(int(x) for x in lens), tuple(colmajor_strides(lens)))


def _draw(n: int, dist: str, dtype: torch.dtype, gen: torch.Generator, device) -> torch.Tensor:
    if dist == "uniform":
        t = torch.rand(n, generator=gen, dtype=torch.float64, device=device).mul_(2.0).sub_(1.0)
    elif dist == "normal":
        t = torch.randn(n, generator=gen, dtype=torch.float64, device=device)
    elif dist == "int":
        t = torch.randint(-4, 5, (n,), generator=gen, device=device).to(torch.float64)
    else:
        raise ValueError(dist)
    return t.to(dtype)


def make_tensors(case: Case, device="cpu", gen_device: Optional[str] = None):
    """Materialise A, B, C (column-major over their label orders) for `case`.

    Values are drawn in float64 (fp32 cases round the same draws) on `gen_device`
    (default: `device`), A then B then C, from one generator seeded with `case.seed`.
    Returns (A, B, C) torch tensors (strided views over flat buffers)."""
    gen_device = gen_device or (device if str(device).startswith("cuda") else "cpu")
    gen = torch.Generator(device=gen_device)
    gen.manual_seed(case.seed)
    out = []
    for labels in (case.lab_a, case.lab_b):
        lens = case.shape(labels)
        flat = _draw(math.prod(lens), case.dist, case.dtype, gen, gen_device).to(device)
        out.append(colmajor_view(flat, lens))
    lens_c = case.shape(case.lab_c)
    nc = math.prod(lens_c)
    if case.c_init == "dist":
        flat = _draw(nc, case.dist, case.dtype, gen, gen_device).to(device)
    elif case.c_init == "nan":
        flat = torch.full((nc,), float("nan"), dtype=case.dtype, device=device)
    else:
        flat = torch.zeros(nc, dtype=case.dtype, device=device)
    out.append(colmajor_view(flat, lens_c))
    return tuple(out)


# ---------------------------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------------------------

def cfg1() -> Case:
    return Case("cfg1_abcd-aebf-dfce", "abcd", "aebf", "dfce", {x: 8 for x in "abcdef"},
                dist="uniform", alpha=1.0, beta=0.0, c_init="nan", seed=SEED_BASE + 100)


def cfg2(transposed: bool = False, n: int = 2048) -> Case:
    if transposed:
        return Case("cfg2T_mn-km-nk", "mn", "km", "nk", {"m": n, "n": n, "k": n}, dist="uniform",
                    alpha=1.0, beta=0.5, c_init="dist", seed=SEED_BASE + 201)
    return Case("cfg2_mn-mk-kn", "mn", "mk", "kn", {"m": n, "n": n, "k": n}, dist="uniform",
                alpha=1.0, beta=0.5, c_init="dist", seed=SEED_BASE + 200)


def cfg3(variant: bool = False, v: int = 128, o: int = 32) -> Case:
    lens = {"a": v, "b": v, "e": v, "f": v, "i": o, "j": o}
    if variant:
        return Case("cfg3v_aibj-abef-efij", "aibj", "abef", "efij", lens, dist="normal",
                    alpha=0.5, beta=1.0, c_init="dist", seed=SEED_BASE + 301)
    return Case("cfg3_abij-abef-efij", "abij", "abef", "efij", lens, dist="normal",
                alpha=0.5, beta=1.0, c_init="dist", seed=SEED_BASE + 300)


def cfg5(big: int = 48, small: int = 24) -> Case:
    lens = {x: big for x in "abcd"}
    lens.update({x: small for x in "ijklm"})
    return Case("cfg5_abcijk-abdilm-dclmjk", "abcijk", "abdilm", "dclmjk", lens, dist="normal",
                alpha=1.0, beta=0.0, c_init="nan", seed=SEED_BASE + 500)


def _group_lengths(rs: np.random.RandomState, g: int, target: int) -> List[int]:
    """Lengths of a g-index group whose product is within +-25% of `target`.
    A single-index group takes the target itself (reading R-cfg4 in DESIGN.md); a multi-index
    group takes lengths in [8, 64]."""
    if g == 1:
        return [int(target)]
    for _ in range(100000):
        first = [int(rs.randint(8, 65)) for _ in range(g - 1)]
        last = int(round(target / math.prod(first)))
        if 8 <= last <= 64:
            lens = first + [last]
            p = math.prod(lens)
            if 0.75 * target <= p <= 1.25 * target:
                rs.shuffle(lens)
                return lens
    raise RuntimeError("group length draw failed")


def cfg4(case: int, dtype: torch.dtype = torch.float64, alpha: float = 1.0, beta: float = 0.0,
         c_init: str = "nan") -> Case:
    """Random permuted contraction `case` in [0, 20) (SURVEY.md §8(d) generator)."""
    rs = np.random.RandomState(SEED_BASE + 400 + case)
    while True:
        gm, gn, gk = (int(rs.randint(1, 4)) for _ in range(3))
        if all(3 <= r <= 6 for r in (gm + gk, gk + gn, gm + gn)):
            break
    tm, tn, tk = (int(rs.randint(1000, 4001)) for _ in range(3))
    pool = list("abcdefghijklmnopqr")
    rs.shuffle(pool)
    li, lj, lp = pool[:gm], pool[gm:gm + gn], pool[gm + gn:gm + gn + gk]
    lens = {}
    for labs, t in ((li, tm), (lj, tn), (lp, tk)):
        for x, n in zip(labs, _group_lengths(rs, len(labs), t)):
            lens[x] = n
    perm = lambda labs: "".join(rs.permutation(labs))  # noqa: E731
    lab_a, lab_b, lab_c = perm(li + lp), perm(lp + lj), perm(li + lj)
    tag = "f64" if dtype == torch.float64 else "f32"
    return Case(f"cfg4_{case:02d}_{tag}_{lab_c}-{lab_a}-{lab_b}", lab_c, lab_a, lab_b, lens,
                dtype=dtype, dist="uniform", alpha=alpha, beta=beta, c_init=c_init,
                seed=SEED_BASE + 400 + case)


def all_parity_cases() -> List[Case]:
    out = [cfg1(), cfg2(False), cfg2(True), cfg3(False), cfg3(True)]
    out += [cfg4(i) for i in range(20)]
    out += [cfg4(i, torch.float32) for i in range(20)]
    out.append(cfg5())
    return out


# The 24 index strings of the paper's fig:bench, in the paper's order. Sizes are not in
# the paper, so any use assigns synthetic lengths.
FIG_BENCH_SPECS = [
    "abcde-efbad-cf", "abcde-efcad-bf", "abcd-dbea-ec", "abcde-ecbfa-fd", "abcd-deca-be",
    "abc-bda-dc", "abcd-ebad-ce", "abcdef-dega-gfbc", "abcdef-dfgb-geac", "abcdef-degb-gfac",
    "abcdef-degc-gfab", "abc-dca-bd", "abcd-ea-ebcd", "abcd-eb-aecd", "abcd-ec-abed",
    "abc-adec-ebd", "ab-cad-dcb", "ab-acd-dbc", "abc-acd-db", "abc-adc-bd", "ab-ac-cb",
    "abcd-aebf-fdec", "abcd-eafd-fbec", "abcd-aebf-dfce",
]


def random_tiny_case(seed: int, max_rank: int = 6, max_len: int = 5, dist: str = "uniform",
                     dtype: torch.dtype = torch.float64) -> Case:
    """Small random contraction for brute-force pins (orders <= 6, lengths <= 8,
    random label permutations, alpha/beta in {0, 0.5, 1, -1})."""
    rs = np.random.RandomState(seed)
    while True:
        gm, gn, gk = (int(rs.randint(0, 4)) for _ in range(3))
        if max(gm + gk, gk + gn, gm + gn) <= max_rank:
            break
    pool = list("abcdefghijklmnopqrstuvwxyz")
    rs.shuffle(pool)
    li, lj, lp = pool[:gm], pool[gm:gm + gn], pool[gm + gn:gm + gn + gk]
    lens = {x: int(rs.randint(1, max_len + 1)) for x in li + lj + lp}
    perm = lambda labs: "".join(rs.permutation(labs)) if labs else ""  # noqa: E731
    ab = [0.0, 0.5, 1.0, -1.0]
    return Case(f"tiny_{seed}", perm(li + lj), perm(li + lp), perm(lp + lj), lens, dtype=dtype,
                dist=dist, alpha=ab[int(rs.randint(1, 4))], beta=ab[int(rs.randint(0, 4))],
                c_init="dist", seed=SEED_BASE + 900000 + seed)


# ---------------------------------------------------------------------------------------------
# §8(f) follow-on families
# ---------------------------------------------------------------------------------------------

def fig_bench(idx: int, elems: int = 2 ** 25, dtype: torch.dtype = torch.float64) -> Case:
    """f2: entry `idx` of the paper's fig:bench (C-A-B order P:1327-1329) with synthetic
    sizes (the paper does not give them): every index has the same length
    L = round(elems ** (1 / r_max)), r_max the largest operand rank, so the largest operand holds
    about `elems` elements. Contractions whose bound bundle is a single short index stay
    bandwidth-bound and GEMM-like ones compute-bound, as in the paper's left-to-right order."""
    spec = FIG_BENCH_SPECS[idx]
    lab_c, lab_a, lab_b = spec.split("-")
    r_max = max(len(lab_a), len(lab_b), len(lab_c))
    L = int(round(elems ** (1.0 / r_max)))
    lens = {x: L for x in set(lab_a + lab_b + lab_c)}
    return Case(f"f2_{idx:02d}_{spec}", lab_c, lab_a, lab_b, lens, dtype=dtype, dist="uniform",
                alpha=1.0, beta=0.0, c_init="nan", seed=SEED_BASE + 600 + idx)


RANKK_K = [5, 16, 32, 64, 128, 256, 500]


def _factor(rs: np.random.RandomState, g: int, target: int) -> List[int]:
    if g == 1:
        return [int(target)]
    for _ in range(100000):
        base = target ** (1.0 / g)
        first = [max(2, int(round(base * rs.uniform(0.8, 1.25)))) for _ in range(g - 1)]
        last = max(2, int(round(target / math.prod(first))))
        lens = first + [last]
        if 0.75 * target <= math.prod(lens) <= 1.25 * target:
            rs.shuffle(lens)
            return lens
    raise RuntimeError("factor draw failed")


def rankk(i: int, mn: int = 16000, dtype: torch.dtype = torch.float64) -> Case:
    """f1: rank-k update family: m = n = 16000 (the paper's 12-core size),
    k = RANKK_K[i % 7] (5-500), each bundle split into 1-3 indices with product within +-25%
    of its target (bound bundles with k < 64 keep one index), operand index orders randomly
    permuted. alpha = 1, beta = 0."""
    k = RANKK_K[i % len(RANKK_K)]
    rs = np.random.RandomState(SEED_BASE + 700 + i)
    gm, gn = int(rs.randint(1, 4)), int(rs.randint(1, 4))
    gk = 1 if k < 64 else int(rs.randint(1, 3))
    pool = list("abcdefghijklmnopqr")
    rs.shuffle(pool)
    li, lj, lp = pool[:gm], pool[gm:gm + gn], pool[gm + gn:gm + gn + gk]
    lens = {}
    for labs, t in ((li, mn), (lj, mn), (lp, k)):
        for x, n in zip(labs, _factor(rs, len(labs), t)):
            lens[x] = n
    perm = lambda labs: "".join(rs.permutation(labs))  # noqa: E731
    lab_a, lab_b, lab_c = perm(li + lp), perm(lp + lj), perm(li + lj)
    return Case(f"f1_k{k}_{i:02d}_{lab_c}-{lab_a}-{lab_b}", lab_c, lab_a, lab_b, lens,
                dtype=dtype, dist="uniform", alpha=1.0, beta=0.0, c_init="nan",
                seed=SEED_BASE + 700 + i)

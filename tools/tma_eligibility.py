"""How many cfg4 operands could be loaded with TMA tiled copies under the kernels' tiling: every
128-row x BK tile of the operand (rows along its traversal bundle, BK along P) must be a box of the
operand viewed as a <= 5-D tensor (the tile may run past the end of the last dimension, which TMA
zero-fills, but must not cross any other dimension boundary), with 16-byte-multiple strides.
Host-only (the planner's folded, traversal-ordered dimensions through the C ABI).

    python tools/tma_eligibility.py > profiles/r02/tma_eligibility.txt
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1607_00291_b200 as tc  # noqa: E402
import workloads as W  # noqa: E402


def boxable(lens, tile):
    rem = tile
    for idx, n in enumerate(lens):
        if rem == 1 or n % rem == 0 or idx == len(lens) - 1:
            return True
        if rem % n == 0:
            rem //= n
            continue
        return False
    return True


def main():
    for dt in (torch.float32, torch.float64):
        e, bk = (4, 32) if dt == torch.float32 else (8, 16)
        ok = tot = 0
        for i in range(20):
            case = W.cfg4(i, dt)
            shapes = [case.shape(x) for x in (case.lab_a, case.lab_b, case.lab_c)]
            p = tc.Plan(case.spec, dt, shapes, [W.colmajor_strides(s) for s in shapes])
            I, J, P = p.dims(0), p.dims(1), p.dims(2)

            def strides_ok(dims, which):
                return all((d[2 + which] * e) % 16 == 0 or d[2 + which] == 1 for d in dims)
            a = (boxable([d[1] for d in I], 128) and boxable([d[1] for d in P], bk)
                 and strides_ok(I, 0) and strides_ok(P, 0))
            b = (boxable([d[1] for d in J], 128) and boxable([d[1] for d in P], bk)
                 and strides_ok(J, 0) and strides_ok(P, 1))
            print(f"{case.name[:40]:40s} I {[d[1] for d in I]} J {[d[1] for d in J]} "
                  f"P {[d[1] for d in P]}  A {'box' if a else '-'}  B {'box' if b else '-'}")
            ok += a + b
            tot += 2
        print(f"# {dt}: {ok} of {tot} operands have every tile a TMA box")


if __name__ == "__main__":
    main()

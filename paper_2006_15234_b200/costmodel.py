"""Algorithmic cost model of the reference's einsumsvd path (host side).

Reproduces the reference's own flop counter ``instr::flops``
(proj/include/peps/instrument.hpp:19-65): every pairwise contraction adds
2 * prod(extents of both reduced operands) (einsum.cpp:227), single-tensor
label sums add kept*summed (einsum.cpp:153), eigh adds 9 n^3 (linalg.cpp:188),
svd adds 14 mn^2 mx + 8 mn^3 (linalg.cpp:177-181).  The contraction order is
the reference's exact subset DP (einsum.cpp:244-313).  A complex multiply-add
counts 2 in this convention, so REAL FP64 flops = 4 x these counts.

bench.py reports einsumsvd throughput as 4 x (this count) / time, i.e. the
reference algorithm's work, independent of the extra CholeskyQR passes the
device implementation chooses to run.
"""
from __future__ import annotations

import math
from typing import Dict, List, Sequence, Tuple


def _result_of(mask: int, labels: Sequence[str], ext: Sequence[Dict[str, int]], output: str) -> Dict[str, int]:
    n = len(labels)
    inside: Dict[str, int] = {}
    for t in range(n):
        if mask & (1 << t):
            inside.update(ext[t])
    res = {}
    for c, e in inside.items():
        needed = c in output or any(c in labels[t] for t in range(n) if not mask & (1 << t))
        if needed:
            res[c] = e
    return res


def network_flops(shapes: Sequence[Sequence[int]], labels: Sequence[str], output: str,
                  real: Sequence[bool] | None = None):
    """instr::flops added by detail::contract_network (einsum.cpp:340-406).

    With ``real`` (one flag per tensor) the count is real-aware:
    a pairwise product with one real operand costs half the complex one (2 real
    flops per MAC instead of 4 x 2), with two real operands a quarter; the
    contraction order is the reference's either way.  Returns a float then."""
    n = len(labels)
    ext = [dict(zip(l, s)) for l, s in zip(labels, shapes)]
    if n == 1:
        f = _reduce_flops(ext[0], labels[0], output)
        return f * (0.5 if real and real[0] else 1.0) if real is not None else f
    if n > 10:
        raise NotImplementedError("greedy fallback not modelled")
    sub = [None] * (1 << n)
    for mask in range(1, 1 << n):
        sub[mask] = _result_of(mask, labels, ext, output)
    best = [None] * (1 << n)
    for mask in range(1, 1 << n):
        if bin(mask).count("1") == 1:
            continue
        b = None
        left = (mask - 1) & mask
        while left:
            right = mask ^ left
            if left <= right:
                uni = dict(sub[left])
                uni.update(sub[right])
                step, out_size = 2, 1
                for c, e in sorted(uni.items()):
                    step *= e
                    if c in sub[mask]:
                        out_size *= e
                fl, pk = step, out_size
                if bin(left).count("1") > 1:
                    fl += best[left][0]
                    pk = max(pk, best[left][1])
                if bin(right).count("1") > 1:
                    fl += best[right][0]
                    pk = max(pk, best[right][1])
                if b is None or fl < b[0] or (fl == b[0] and pk < b[1]):
                    b = (fl, pk, left, right)
            left = (left - 1) & mask
        best[mask] = b

    # walk the tree adding the leaf pre-reductions the reference performs
    total = 0
    flags = list(real) if real is not None else [False] * n

    def walk(mask) -> Tuple[str, Dict[str, int], bool]:
        nonlocal total
        if bin(mask).count("1") == 1:
            t = mask.bit_length() - 1
            return labels[t], ext[t], flags[t]
        _, _, l, r = best[mask]
        ll, le, lr = walk(l)
        rl, re_, rr = walk(r)
        keep = output + "".join(labels[t] for t in range(n) if not mask & (1 << t))
        # pre-reduce labels present on one side only and not kept (einsum.cpp:182-194)
        wa = {c: le[c] for c in le if c in rl or c in keep}
        wb = {c: re_[c] for c in re_ if c in ll or c in keep}
        if len(wa) != len(set(ll)):
            total += _sum_flops(le, wa) * (0.5 if lr else 1)
        if len(wb) != len(set(rl)):
            total += _sum_flops(re_, wb) * (0.5 if rr else 1)
        uni = dict(wa)
        uni.update(wb)
        total += 2 * math.prod(uni.values()) * (0.5 if lr else 1) * (0.5 if rr else 1)
        res = {c: e for c, e in uni.items() if c in sub[mask]}
        return "".join(res), res, lr and rr

    walk((1 << n) - 1)
    return total if real is not None else int(total)


def _sum_flops(ext: Dict[str, int], kept: Dict[str, int]) -> int:
    return math.prod(kept.values()) * math.prod(e for c, e in ext.items() if c not in kept)


def _reduce_flops(ext: Dict[str, int], labels: str, output: str) -> int:
    kept = {c: e for c, e in ext.items() if c in output}
    if len(kept) == len(ext):
        return 0
    return _sum_flops(ext, kept)


def svd_flops(rows: int, cols: int) -> int:
    mn, mx = min(rows, cols), max(rows, cols)
    return 14 * mn * mn * mx + 8 * mn ** 3


def gram_orth_flops(rows: int, k: int) -> int:
    """gram_orthogonalize (decomposition.cpp:160-193): G, eigh, Q."""
    return 2 * rows * k * k + 9 * k ** 3 + 2 * rows * k * k


def effective_oversample(oversample: int, target: int) -> int:
    return oversample if oversample >= 0 else max(5, math.ceil(0.1 * target))


def rsvd_flops(shapes, labels, rows: str, cols: str, max_rank: int, power_iters: int, oversample: int,
               real: Sequence[bool] | None = None):
    """randomized_svd (decomposition.cpp:259-306) with the reference's counters
    (real-aware for the operator applications when ``real`` flags are given)."""
    ext = {}
    for l, s in zip(labels, shapes):
        ext.update(dict(zip(l, s)))
    R = math.prod(ext[c] for c in rows)
    Cx = math.prod(ext[c] for c in cols)
    mindim = min(R, Cx)
    target = min(max_rank, mindim)
    k = min(target + effective_oversample(oversample, target), mindim)
    free = next(c for c in "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz"
                if c not in rows + cols + "".join(labels))
    rf = list(real) + [False] if real is not None else None  # the probe is complex
    ap = network_flops(list(shapes) + [[ext[c] for c in cols] + [k]], list(labels) + [cols + free], rows + free, rf)
    ad = network_flops(list(shapes) + [[ext[c] for c in rows] + [k]], list(labels) + [rows + free], cols + free, rf)
    total = (power_iters + 1) * ap + (power_iters + 1) * ad
    total += (power_iters + 1) * gram_orth_flops(R, k) + power_iters * gram_orth_flops(Cx, k)
    total += svd_flops(k, Cx) + 2 * R * k * k
    return total


def two_layer_row_flops(length: int, bond: int, m: int, power_iters: int, oversample: int, d: int = 2,
                        top_bonds: Sequence[int] | None = None, interior: bool = True,
                        real_sites: bool = False):
    """instr::flops of one two_layer_apply_row (contraction.cpp:269-311) on an
    interior row whose top boundary has bonds `m` (edges 1) and whose pending
    bond saturates at min(m, ...) as the reference's truncation dictates.

    ``real_sites``: the real-aware count of SURVEY §8(d) -- the bra/ket PEPS
    sites of the BASELINE configs are real, so their products are counted at 2
    real flops per MAC (the top boundary and pending tensor stay complex)."""
    r = bond
    dn = r if interior else 1
    tb = list(top_bonds) if top_bonds is not None else [1] + [m] * (length - 1) + [1]
    # column 0: contract_network({s0s (u,v,l,s), bra (d,u,m,b,e), ket (d,v,n,c,f)}) -> bcsef
    rl = [False, True, True] if real_sites else None
    total = network_flops([[r, r, 1, tb[1]], [d, r, 1, dn, r], [d, r, 1, dn, r]], ["uvls", "dumbe", "dvncf"],
                          "bcsef", rl)
    a = 1
    for c in range(1, length):
        right = r if c < length - 1 else 1
        shapes = [[a, dn, dn, tb[c], r, r], [r, r, tb[c], tb[c + 1]], [d, r, r, dn, right], [d, r, r, dn, right]]
        labels = ["apqsmn", "uvst", "dumbe", "dvncf"]
        total += rsvd_flops(shapes, labels, "apq", "bctef", m, power_iters, oversample,
                            [False, False, True, True] if real_sites else None)
        R = a * dn * dn
        Cx = right * right * tb[c + 1] * dn * dn
        k_max = min(R, Cx)
        a = min(m, k_max)
    return total

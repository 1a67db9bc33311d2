"""CPU restatement of the reference's ranking metric -- TEST INFRASTRUCTURE.

Checker for csrc/evaluate.cu. Restates hetsched/predictor.py:
  ref_count_inversions   _count_inversions   predictor.py:132-160 (bottom-up
                         merge sort, strict inversions)
  ref_tie_pairs          _tie_pairs          predictor.py:163-173
  ref_kendall_counts     kendall_tau_distance predictor.py:182-214, returning
                         the four integer counts and the distance
Pinned against tests/golden/kendall.npz (tests/test_evaluate.py).
"""

from __future__ import annotations


def ref_count_inversions(values):
    buf = list(values)
    n = len(buf)
    tmp = [0.0] * n
    count = 0
    width = 1
    while width < n:
        for lo in range(0, n, 2 * width):
            mid, hi = min(lo + width, n), min(lo + 2 * width, n)
            i, j, k = lo, mid, lo
            while i < mid and j < hi:
                if buf[j] < buf[i]:
                    tmp[k] = buf[j]
                    count += mid - i
                    j += 1
                else:
                    tmp[k] = buf[i]
                    i += 1
                k += 1
            tmp[k:hi] = buf[i:mid] if i < mid else buf[j:hi]
            buf[lo:hi] = tmp[lo:hi]
        width *= 2
    return count


def ref_tie_pairs(values):
    pairs, run = 0, 1
    for prev, cur in zip(values, values[1:]):
        if cur == prev:
            run += 1
        else:
            pairs += run * (run - 1) // 2
            run = 1
    return pairs + run * (run - 1) // 2


def ref_kendall_counts(predicted, truth):
    n = len(predicted)
    order = sorted(range(n), key=lambda i: (predicted[i], truth[i]))
    p_sorted = [predicted[i] for i in order]
    t_sorted = [truth[i] for i in order]
    disc = ref_count_inversions(t_sorted)
    ties_p = ref_tie_pairs(p_sorted)
    ties_t = ref_tie_pairs(sorted(truth))
    runs, rid = [], 0
    for i in range(n):
        if i > 0 and not (p_sorted[i] == p_sorted[i - 1] and t_sorted[i] == t_sorted[i - 1]):
            rid += 1
        runs.append(float(rid))
    ties_b = ref_tie_pairs(runs)
    half = (ties_p - ties_b) + (ties_t - ties_b)
    total = n * (n - 1) // 2
    return [disc, ties_p, ties_t, ties_b], (disc + 0.5 * half) / total

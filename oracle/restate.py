"""Independent numpy/Python restatement of the integer core of the hot path
(TEST INFRASTRUCTURE ONLY; pinned against oracle/_ref by tests/test_oracle.py).

Each function cites the reference lines it restates. It exists so the
integer stages have a second, implementation-independent oracle whose
correctness does not rest on the Eigen shim:
  - sgm_single_path: the SGM recurrence walk_line (sgm.cpp:91-196) for the
    Plane variant, written as the naive chain DP of tests/oracles.hpp:50-91
  - wta: sgm.cpp:333-349
  - census_cost: matching.cpp:249-260 given warped samples
  - median_5x5: pipeline.cpp:175-198
"""
from __future__ import annotations

import math

import numpy as np


def adaptive_phi2(phi1: float, alpha: float, beta: float, di: float) -> float:
    """sgm.cpp:22-24."""
    return phi1 * (1.0 + alpha * math.exp(-di / beta))


def _round_half_away(x: float) -> int:
    """std::llround: halfway cases away from zero."""
    a = abs(x)
    q = math.floor(a)
    r = q + 1 if a - q >= 0.5 else q  # a - floor(a) is exact for |a| < 2^52
    return int(r) if x >= 0 else -int(r)


def chain_dp(chain, phi1: int):
    """Naive O(L^2) single-chain DP with min-normalisation (oracles.hpp:50-91).

    chain: list of (first, costs (list[int]), shift, phi2) per pixel; empty
    costs break the path."""
    out = []
    prev = None
    prev_first = 0
    for first, costs, shift, phi2 in chain:
        if len(costs) == 0:
            prev = None
            out.append([])
            continue
        if prev is None:
            cur = [int(c) for c in costs]
        else:
            pmin = min(prev)
            cur = []
            for i, c in enumerate(costs):
                target = first + i + shift
                best = pmin + phi2
                for j, pv in enumerate(prev):
                    diff = abs(target - (prev_first + j))
                    best = min(best, pv + (0 if diff == 0 else phi1 if diff == 1 else phi2))
                cur.append(int(c) + best - pmin)
        out.append(cur)
        prev = cur
        prev_first = first
    return out


def sgm_single_path(first, count, offset, costs, image, width, height, dx, dy, phi1, phi2_fixed,
                    phi2_adaptive, alpha, beta, penalty_scale):
    """aggregate_single_path (sgm.cpp:301-315) for the Plane variant."""
    phi1_eff = _round_half_away(phi1 * penalty_scale)
    out = np.zeros(len(costs), np.uint64)
    for sy in range(height):
        for sx in range(width):
            if 0 <= sx - dx < width and 0 <= sy - dy < height:
                continue  # not a start pixel (sgm.cpp:215-219)
            chain, pos = [], []
            x, y = sx, sy
            prev_valid = False
            px = py = 0
            while 0 <= x < width and 0 <= y < height:
                p = y * width + x
                c = costs[int(offset[p]):int(offset[p]) + int(count[p])]
                if prev_valid and phi2_adaptive:
                    di = abs(float(image[y, x]) - float(image[py, px]))
                    phi2 = _round_half_away(adaptive_phi2(phi1, alpha, beta, di) * penalty_scale)
                else:
                    phi2 = _round_half_away(phi2_fixed * penalty_scale)
                chain.append((int(first[p]), list(c), 0, phi2))
                pos.append(p)
                prev_valid = len(c) > 0
                px, py = x, y
                x += dx
                y += dy
            for p, vals in zip(pos, chain_dp(chain, phi1_eff)):
                o = int(offset[p])
                for i, v in enumerate(vals):
                    out[o + i] = v
    return out.astype(np.uint32)


def wta(first, count, offset, values, width, height):
    """sgm.cpp:333-349: argmin, ties to the lowest index, -1 when empty."""
    out = np.full(width * height, -1, np.int32)
    for p in range(width * height):
        c = int(count[p])
        if c == 0:
            continue
        v = values[int(offset[p]):int(offset[p]) + c]
        out[p] = int(first[p]) + int(np.argmin(v))  # argmin returns the first minimum
    return out.reshape(height, width)


def census_cost(warped, ref_bits: int, bits: int) -> int:
    """matching.cpp:249-260 on one warped window (row-major samples)."""
    n = len(warped)
    wc = warped[n // 2]
    code = 0
    for i, v in enumerate(warped):
        if i == n // 2:
            continue
        code = (code << 1) | (1 if v < wc else 0)
    ham = bin(code ^ ref_bits).count("1")
    return _round_half_away(255.0 * ham / bits)


def median_5x5(depth: np.ndarray) -> np.ndarray:
    """pipeline.cpp:175-198."""
    h, w = depth.shape
    out = np.zeros_like(depth)
    for y in range(h):
        for x in range(w):
            win = depth[max(0, y - 2):y + 3, max(0, x - 2):x + 3].ravel()
            valid = np.sort(win[(win > 0) & np.isfinite(win)])
            if 2 * len(valid) < len(win):
                continue
            out[y, x] = valid[len(valid) // 2]
    return out

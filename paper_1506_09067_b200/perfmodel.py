"""The paper's theoretical analysis and performance model (§III-B/C), host only,
calibrated on the B200.

Formulas, written as the paper states them:

* speed-up (§III-B)::

      S_p = T_1 / T_p = [(a i + b it + c) + (d + e i + f i + g it) ep]
                      / [(a i + b it + c) + (d + e i / p_i + f i / p_i + g it / p_it) ep]

  with p_i = min(p, i), p_it = min(p, it).

* execution time (§III-C)::

      T(i, it, ep, p, s) = T_comp + T_mem                                       (1)
      T_comp = ( (Prep + 4 i + 2 it + 10 ep) / s                                (2)
               + ((FProp + BProp) / s) (i / p_i) ep                             (3)
               + (FProp / s) (i / p_i) ep                                       (4)
               + (FProp / s) (it / p_it) ep ) * CPI * OperationFactor           (5), (6)
      T_mem(ep, i, p) = MemoryContention * i * ep / p

  Rows (3)/(4)/(5) are Training, Validation (on the training set) and Testing.

* accuracy of a prediction: alpha = |mu - psi| / psi * 100 %, mu the
  measured and psi the predicted time.

B200 reading: a processing unit is one image in flight (a CTA worker holds G
of them), s is the SM clock in cycles per second, FProp/BProp are the algorithmic FLOP per
image of SURVEY §8(d) D-3.  CPI * OperationFactor (cycles per FLOP per unit) and Prep are fitted
(T is linear in CPI*OF and CPI*OF*Prep: ordinary least squares); MemoryContention is measured
separately, as in the paper, from the hogwild time minus the time of the same work publishing
into private slots (sync mode).  No constant comes from the paper (its Phi constants are not
printed).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def p_clamp(p: int, n: int) -> int:
    """p_i = min(p, i): one processing unit cannot process less than one image."""
    return max(1, min(int(p), int(n)))


def speedup(a, b, c, d, e, f, g, i, it, ep, p):
    """S_p of §III-B."""
    pi, pit = p_clamp(p, i), p_clamp(p, it)
    seq = a * i + b * it + c
    t1 = seq + (d + e * i + f * i + g * it) * ep
    tp = seq + (d + e * i / pi + f * i / pi + g * it / pit) * ep
    return t1 / tp


def t_mem(ep, i, p, contention):
    """T_mem(ep, i, p) = MemoryContention * i * ep / p."""
    return contention * i * ep / p


def t_comp_terms(i, it, ep, p, s, prep, fprop, bprop):
    """The bracket of rows (2)-(5) before the CPI * OperationFactor penalty, per row."""
    pi, pit = p_clamp(p, i), p_clamp(p, it)
    return {
        "prep": (prep + 4 * i + 2 * it + 10 * ep) / s,          # (2)
        "train": (fprop + bprop) / s * (i / pi) * ep,           # (3)
        "validation": fprop / s * (i / pi) * ep,                 # (4)
        "test": fprop / s * (it / pit) * ep,                     # (5)
    }


def predict_time(i, it, ep, p, s, prep, fprop, bprop, cpi_opf, contention, parts=("prep", "train", "validation", "test")):
    """T(i, it, ep, p, s) of (1)-(6); cpi_opf = CPI * OperationFactor.  `parts` selects rows
    (e.g. ("train",) for the Training phase alone)."""
    terms = t_comp_terms(i, it, ep, p, s, prep, fprop, bprop)
    comp = sum(terms[k] for k in parts) * cpi_opf
    mem = t_mem(ep, i, p, contention) if "train" in parts else 0.0
    return comp + mem


def alpha(measured, predicted):
    """Prediction accuracy alpha = |mu - psi| / psi * 100."""
    return abs(measured - predicted) / predicted * 100.0


@dataclass
class Calibration:
    cpi_opf: float      # cycles-per-FLOP penalty per unit (CPI * OperationFactor)
    prep: float         # sequential work per epoch run, in the units of row (2) (cycles)
    contention: float   # seconds per image per unit (MemoryContention), measured, not fitted
    residual: float     # rms relative residual of the fit


def calibrate(points, i, it, ep, s, fprop, bprop, contention, parts=("prep", "train")):
    """Least-squares fit of CPI*OperationFactor and Prep to measured times, MemoryContention
    given (the paper measures it separately; a fit could not tell it from the
    1/p compute rows).  points: iterable of (p, measured_seconds).  With u = CPI*OF and
    v = CPI*OF*Prep/s, T(p) - T_mem(p) = u * X(p) + v, X = the selected rows' bracket with
    Prep = 0 -- linear in (u, v); fitted in relative terms so every p weighs the same."""
    rows, rhs = [], []
    for p, t in points:
        x = sum(t_comp_terms(i, it, ep, p, s, 0.0, fprop, bprop)[k] for k in parts)
        tm = t_mem(ep, i, p, contention) if "train" in parts else 0.0
        rows.append([x / t, (1.0 if "prep" in parts else 0.0) / t])
        rhs.append((t - tm) / t)
    A = np.asarray(rows)
    sol, *_ = np.linalg.lstsq(A, np.asarray(rhs), rcond=None)
    u, v = float(sol[0]), float(sol[1])
    pred = A @ sol
    res = float(np.sqrt(np.mean((pred - np.asarray(rhs)) ** 2)))
    return Calibration(u, v * s / u if u else 0.0, float(contention), res)


def what_if(cal: Calibration, s, fprop, bprop, grid, parts=("prep", "train", "validation", "test")):
    """Table III analogue: predicted times over (p, i, it, ep) combinations."""
    return [{"p": p, "i": i, "it": it, "ep": ep,
             "seconds": predict_time(i, it, ep, p, s, cal.prep, fprop, bprop, cal.cpi_opf, cal.contention, parts)}
            for (p, i, it, ep) in grid]

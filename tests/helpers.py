"""Shared test helpers: the parity tolerance of DESIGN.md (reading R9 / SURVEY C-15)."""
import numpy as np


def split_blocks(vec, blocks):
    """Split a normative flat vector into per-tensor pieces [W0, b0, W1, b1, ...]."""
    out = []
    off = 0
    for _, nw, nb in blocks:
        out.append(vec[off:off + nw])
        out.append(vec[off + nw:off + nw + nb])
        off += nw + nb
    return out


def parity_report(got, ref, blocks, rel=1e-4, floor=1e-2, norm_rel=1e-5):
    """Per tensor T: |got-ref| <= rel*max(|ref|, floor*||ref||_inf) element-wise and
    ||got-ref||_2 <= norm_rel*||ref||_2.  Returns (ok, worst_ratio, worst_norm_ratio, details)."""
    ok = True
    worst = 0.0
    worst_norm = 0.0
    details = []
    for k, (g, r) in enumerate(zip(split_blocks(np.asarray(got, np.float64), blocks),
                                   split_blocks(np.asarray(ref, np.float64), blocks))):
        rmax = np.abs(r).max() if r.size else 0.0
        if rmax == 0.0:
            bad = np.abs(g).max() if g.size else 0.0
            ratio = 0.0 if bad == 0.0 else np.inf
            nr = 0.0 if bad == 0.0 else np.inf
        else:
            tol = rel * np.maximum(np.abs(r), floor * rmax)
            ratio = float(np.max(np.abs(g - r) / tol))
            nr = float(np.linalg.norm(g - r) / np.linalg.norm(r)) / norm_rel
        worst = max(worst, ratio)
        worst_norm = max(worst_norm, nr)
        details.append((k, ratio, nr))
        if ratio > 1.0 or nr > 1.0:
            ok = False
    return ok, worst, worst_norm, details


def assert_parity(got, ref, blocks, **kw):
    ok, w, wn, det = parity_report(got, ref, blocks, **kw)
    assert ok, f"parity failed: worst elementwise {w:.3g} x tol, worst norm {wn:.3g} x tol; per tensor {det}"
    return w, wn

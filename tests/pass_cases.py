"""Loader for tests/golden/pass_cases.npz (made by make_pass_golden.py):
groups of pass-formation problems sharing (cap, max_pass_ns, cost table)."""

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
K = 3


def groups():
    d = np.load(GOLDEN / "pass_cases.npz")
    out = []
    for g in range(int(d["n_groups"])):
        p = f"g{g}_"
        out.append({k[len(p):]: d[k] for k in d.files if k.startswith(p)})
    return out


def problem_jobs(g, i):
    """Problem i of group g as the oracle's job list."""
    j0, q = int(g["job_off"][i]), int(g["n_jobs"][i])
    coff = np.concatenate([[0], np.cumsum(g["n_cand"])])
    moff = np.concatenate([[0], np.cumsum(g["n_cand"].astype(np.int64) * g["size"])])
    jobs = []
    for j in range(j0, j0 + q):
        s, nc = int(g["size"][j]), int(g["n_cand"][j])
        jobs.append((s, int(g["deadline"][j]), g["cand_counts"][coff[j]:coff[j] + nc],
                     g["req_masks"][moff[j]:moff[j] + nc * s].reshape(nc, s)))
    return jobs


def expected(g, i):
    """(members, choices[members], est_ns, counts, masks) recorded for problem i."""
    j0 = int(g["job_off"][i])
    m = int(g["res_members"][i])
    roff = np.concatenate([[0], np.cumsum(g["res_requests"])])
    return (m, g["res_choice"][j0:j0 + m].tolist(), int(g["res_est"][i]), g["res_counts"][i].tolist(),
            g["res_mask"][roff[i]:roff[i + 1]].tolist())

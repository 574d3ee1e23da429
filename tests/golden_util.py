"""Helpers to turn the committed golden fixtures (tests/golden/*.npz, made by
tests/golden/make_golden.py from the reference itself) into configs + frames."""

from __future__ import annotations

from pathlib import Path

import numpy as np

from paper_2002_00250_b200.config import GmmParams, PbasParams, PipelineConfig

GOLDEN = Path(__file__).resolve().parent / "golden"

GMM_KEYS = ("rgb_w", "rgb_mu", "rgb_var", "d_w", "d_mu", "d_var")
PBAS_KEYS = ("samples", "dmin_rgb", "dmin_d", "len_rgb", "pos_rgb", "len_d", "pos_d",
             "r_rgb", "r_d", "t")


def load(name: str) -> dict:
    with np.load(GOLDEN / name) as z:
        return {k: z[k] for k in z.files}


def gmm_cases():
    return sorted(p.name for p in GOLDEN.glob("gmm_*.npz"))


def pbas_cases():
    return sorted(p.name for p in GOLDEN.glob("pbas_*.npz"))


def gmm_config(fx: dict, name: str) -> PipelineConfig:
    if name.startswith("gmm_equiv_"):
        mode = name[len("gmm_equiv_"):-4]
        params = GmmParams(k_rgb=int(fx["k_rgb"]), k_d=int(fx["k_d"]))
    else:
        mode = str(fx["mode"])
        a, s, tau, lam, var_init, w_init = (float(v) for v in fx["params"])
        params = GmmParams(k_rgb=int(fx["k_rgb"]), k_d=int(fx["k_d"]), alpha=a, s=s, tau=tau,
                           match_lambda=lam, var_init=var_init, w_init=w_init)
    return PipelineConfig(algorithm="gmm", mode=mode, gmm=params)


def pbas_config(fx: dict, name: str) -> PipelineConfig:
    if name.startswith("pbas_equiv_"):
        mode = name[len("pbas_equiv_"):-4]
        params = PbasParams(n=int(fx["n"]), min_matches=int(fx["min_matches"]))
    else:
        mode = str(fx["mode"])
        (r_init, r_lower, r_scale, r_inc_dec, t_init, t_lower, t_upper, t_inc,
         t_dec) = (float(v) for v in fx["params"])
        params = PbasParams(n=int(fx["n"]), min_matches=int(fx["min_matches"]), r_init=r_init,
                            r_lower=r_lower, r_scale=r_scale, r_inc_dec=r_inc_dec, t_init=t_init,
                            t_lower=t_lower, t_upper=t_upper, t_inc=t_inc, t_dec=t_dec)
    return PipelineConfig(algorithm="pbas", mode=mode, pbas=params, seed=int(fx["seed"]))

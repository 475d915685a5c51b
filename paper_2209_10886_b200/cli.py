"""Command-line front end of the SPEC over the GPU driver.

    python -m paper_2209_10886_b200.cli --n1 5 --n2 5 --cells 20 --precond sp --out runs/a
    python -m paper_2209_10886_b200.cli --config run.cfg --table 5x5,5x10 --out runs/t

Flags: --n1 --n2 --cells --kappa --side --precond {none,sp,bsp}
--bsp-seam {dedup,literal} --bsp-no-intermediate-residual --tol --maxit
--workers --mono-check --out --config, plus --scatterer cx,cy,r|none,
--direction, --blocks (BSP window count) and --table.  A config
file holds one `key = value` per line (`#` comments; keys are the flag names
without dashes, `-` or `_`); flags override the file.  Exit status: 0
converged, 2 not converged, 1 configuration error (message names the key).

The mono-domain check (`--mono-check`) needs a reference field: the mono solve
is a CPU oracle kept out of the product, so pass it as `--mono-field file.npy`.
"""

from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np

from . import artifacts
from .discretization import ProblemSpec, Scatterer
from .indexing import Partition
from .interface_system import GmresOptions, SweepConfig


class ConfigError(ValueError):
    def __init__(self, key, msg):
        super().__init__(f"{key}: {msg}")
        self.key = key


# key -> (type, default)
_KEYS = {
    "n1": (int, 2), "n2": (int, 2), "cells": (int, 20), "kappa": (float, 2 * math.pi),
    "side": (float, 2.5), "scatterer": (str, "0,0,1"), "direction": (float, 0.0),
    "precond": (str, "bsp"), "bsp_seam": (str, "dedup"), "bsp_no_intermediate_residual": (bool, False),
    "blocks": (int, None), "tol": (float, 1e-6), "maxit": (int, 200), "workers": (int, 1),
    "mono_check": (bool, False), "mono_field": (str, None), "out": (str, "helmsweep_out"),
    "table": (str, None), "timings": (bool, False), "device": (int, 0),
}


def _norm(key: str) -> str:
    return key.strip().lower().replace("-", "_")


def _convert(key, typ, raw):
    if raw is None:
        return None
    if typ is bool:
        if isinstance(raw, bool):
            return raw
        s = str(raw).strip().lower()
        if s in ("1", "true", "yes", "on"):
            return True
        if s in ("0", "false", "no", "off"):
            return False
        raise ConfigError(key, f"expected a boolean, got {raw!r}")
    try:
        return typ(raw)
    except (TypeError, ValueError):
        raise ConfigError(key, f"expected {typ.__name__}, got {raw!r}") from None


def parse_config_file(path) -> dict:
    """`key = value` lines, `#` comments."""
    out = {}
    with open(path) as f:
        for ln, line in enumerate(f, 1):
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise ConfigError(f"line {ln}", f"expected 'key = value', got {line!r}")
            k, v = (s.strip() for s in line.split("=", 1))
            k = _norm(k)
            if k not in _KEYS:
                raise ConfigError(k, "unknown key")
            out[k] = _convert(k, _KEYS[k][0], v)
    return out


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="helmsweep-b200", description=__doc__.split("\n\n")[0])
    for k, (typ, _) in _KEYS.items():
        flag = "--" + k.replace("_", "-")
        if typ is bool:
            p.add_argument(flag, dest=k, action="store_const", const=True, default=None)
        else:
            p.add_argument(flag, dest=k, default=None)
    p.add_argument("--config", dest="config", default=None)
    return p


def resolve(argv) -> dict:
    """Defaults <- config file <- flags, converted and validated."""
    ns = build_parser().parse_args(argv)
    cfg = {k: d for k, (_, d) in _KEYS.items()}
    if ns.config is not None:
        if not os.path.exists(ns.config):
            raise ConfigError("config", f"no such file {ns.config!r}")
        cfg.update(parse_config_file(ns.config))
    for k, (typ, _) in _KEYS.items():
        v = getattr(ns, k)
        if v is not None:
            cfg[k] = _convert(k, typ, v)
    for k in ("n1", "n2"):
        if cfg[k] < 1:
            raise ConfigError(k, f"must be >= 1, got {cfg[k]}")
    if cfg["cells"] < 4:
        raise ConfigError("cells", f"must be >= 4, got {cfg['cells']}")
    for k in ("kappa", "side", "tol"):
        if not cfg[k] > 0:
            raise ConfigError(k, f"must be positive, got {cfg[k]}")
    if cfg["maxit"] < 0:
        raise ConfigError("maxit", f"must be >= 0, got {cfg['maxit']}")
    if cfg["workers"] < 1:
        raise ConfigError("workers", f"must be >= 1, got {cfg['workers']}")
    if cfg["precond"] not in ("none", "sp", "bsp"):
        raise ConfigError("precond", f"must be none, sp or bsp, got {cfg['precond']!r}")
    if cfg["bsp_seam"] not in ("dedup", "literal"):
        raise ConfigError("bsp_seam", f"must be dedup or literal, got {cfg['bsp_seam']!r}")
    if cfg["blocks"] is not None and cfg["blocks"] < 1:
        raise ConfigError("blocks", f"must be >= 1, got {cfg['blocks']}")
    if cfg["mono_check"] and cfg["mono_field"] is None:
        raise ConfigError("mono_check", "needs --mono-field <file.npy> (the mono solve is a CPU oracle, not part of the product)")
    sc = str(cfg["scatterer"]).strip().lower()
    if sc == "none":
        cfg["scatterer_obj"] = None
    else:
        try:
            cx, cy, r = (float(t) for t in sc.split(","))
        except ValueError:
            raise ConfigError("scatterer", f"expected 'cx,cy,r' or 'none', got {cfg['scatterer']!r}") from None
        if r <= 0:
            raise ConfigError("scatterer", f"radius must be positive, got {r}")
        cfg["scatterer_obj"] = Scatterer((cx, cy), r)
    if cfg["table"] is not None:
        try:
            cfg["table_parts"] = [tuple(int(v) for v in t.lower().split("x")) for t in cfg["table"].split(",") if t.strip()]
        except ValueError:
            raise ConfigError("table", f"expected 'N1xN2,N1xN2,...', got {cfg['table']!r}") from None
    return cfg


def make_problem(cfg, n1=None, n2=None):
    d = cfg["direction"]
    try:
        spec = ProblemSpec(kappa=cfg["kappa"], cells_per_side=cfg["cells"], subdomain_side=cfg["side"],
                           scatterer=cfg["scatterer_obj"], incident_direction=(math.cos(d), math.sin(d)))
    except ValueError as e:
        raise ConfigError("problem", str(e)) from None
    return spec, Partition(n1 or cfg["n1"], n2 or cfg["n2"])


def sweep_of(cfg, kind=None) -> SweepConfig:
    return SweepConfig(kind=kind or cfg["precond"], bsp_seam=cfg["bsp_seam"],
                       bsp_intermediate_residual=not cfg["bsp_no_intermediate_residual"],
                       blocks=cfg["blocks"])


def run(cfg) -> int:
    """One experiment: solve, write the artefacts, exit 0/2."""
    from .driver import solve_problem
    spec, part = make_problem(cfg)
    mono = None
    if cfg["mono_field"] is not None:
        mono = np.load(cfg["mono_field"])
    rep = solve_problem(spec, part, sweep_of(cfg), GmresOptions(tol=cfg["tol"], maxit=cfg["maxit"]),
                        run_mono_check=cfg["mono_check"], mono=mono, device=cfg["device"])
    artifacts.write_artifacts(cfg["out"], rep, spec, part, cfg["precond"], timings=cfg["timings"])
    return 0 if rep.converged else 2


def experiment_table(cfg, partitions, path) -> int:
    """Table-1 sweep: one row per (partition, preconditioner)
    with ni, ns, t; a failing row records its error and the sweep continues."""
    from .driver import solve_problem
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    rows = [artifacts.TABLE_HEADER]
    for n1, n2 in partitions:
        for kind in ("sp", "bsp"):
            try:
                spec, part = make_problem(cfg, n1, n2)
                rep = solve_problem(spec, part, sweep_of(cfg, kind),
                                    GmresOptions(tol=cfg["tol"], maxit=cfg["maxit"]),
                                    device=cfg["device"], reconstruct=False)
                rows.append(artifacts.table_row(n1, n2, kind, rep))
            except (ValueError, RuntimeError) as e:
                rows.append(artifacts.table_row(n1, n2, kind, error=str(e)))
    with open(path, "w", newline="\n") as f:
        f.write("".join(rows))
    return 0


def main(argv=None) -> int:
    try:
        cfg = resolve(sys.argv[1:] if argv is None else argv)
        if cfg["table"] is not None:
            return experiment_table(cfg, cfg["table_parts"], os.path.join(cfg["out"], "table.csv"))
        return run(cfg)
    except ValueError as e:  # ConfigError, or a problem the system rejects (e.g. scatterer placement)
        print(f"configuration error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())

"""bench.py's multi-GPU launch contract on CPU: ``--gpus N`` without a
launcher really starts N ranks (one per GPU), and a rank count that does not
match --gpus is refused instead of producing a mislabelled line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=e, timeout=300)


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_n_spawns_n_ranks(n):
    r = _run(["--gpus", str(n), "--dry-run"])
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == n and lines[0]["ranks_joined"] == n


def test_mismatched_world_size_is_refused():
    r = _run(["--gpus", "4", "--dry-run"], env={"WORLD_SIZE": "2", "RANK": "0"})
    assert r.returncode == 2
    assert "refusing" in r.stderr


def test_reference_arm_line_contract():
    """The reference arm on CPU (C1, one bounded sample): the contract keys,
    an extrapolated full-step time, and the same config dict our arm emits
    (bench.workload_config) so the driver can compare like with like."""
    r = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert d["impl"] == "reference" and d["metric"].startswith("cell-updates/sec")
    assert d["cpu_baseline"]["extrapolated"] is True and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    cfg = d["config"]
    for k in ("workload", "config", "grid", "cells", "fields", "scheme", "outer_dt_over_dtE", "operators",
              "cell_updates_per_step", "decomposition", "l2", "parallelism"):
        assert k in cfg, k
    assert cfg["grid"] == [48, 48, 96] and cfg["operators"][0]["stages_or_iters"] == 962
    # the extrapolated step time is the step's cell-updates over the line's rate
    assert abs(d["ms_per_step"] / 1e3 - cfg["cell_updates_per_step"] / d["value"]) <= 1e-6 * d["ms_per_step"] / 1e3


def test_vector_march_label_and_radial_bytes():
    """bench.py names the kernel that runs the 3-component launches
    (k_vec_march under capi_ops.cuh vmarch_ok's grid conditions) and counts
    no rho stream when C5 / C5v's radial density is read per plane."""
    import types
    sys.path.insert(0, ROOT)
    import bench
    sph = types.SimpleNamespace(w=types.SimpleNamespace(grid=types.SimpleNamespace(metric="spherical")),
                                dg=types.SimpleNamespace(global_shape=(128, 128, 256)))
    args = types.SimpleNamespace(decomp=None)
    old = os.environ.pop("PC_NO_VMARCH", None)
    try:
        assert bench._vmarch_applies(sph, args)
        assert not bench._vmarch_applies(sph, types.SimpleNamespace(decomp="phi"))
        ragged = types.SimpleNamespace(w=sph.w, dg=types.SimpleNamespace(global_shape=(48, 48, 96 + 8)))
        assert not bench._vmarch_applies(ragged, args)
        cart = types.SimpleNamespace(w=types.SimpleNamespace(grid=types.SimpleNamespace(metric="cartesian")),
                                     dg=sph.dg)
        assert not bench._vmarch_applies(cart, args)
        os.environ["PC_NO_VMARCH"] = "1"
        assert not bench._vmarch_applies(sph, args)
    finally:
        os.environ.pop("PC_NO_VMARCH", None)
        if old is not None:
            os.environ["PC_NO_VMARCH"] = old
    # the radial-rho stage / fused launch move the vector's bytes, the field path 8 B more
    assert bench.BYTES[("vector_rho", "rkl2")] - bench.BYTES[("vector", "rkl2")] == 8
    assert bench.BYTES_F12[("vector_rho", "f12")] - bench.BYTES_F12[("vector", "f12")] == 4

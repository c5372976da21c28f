"""C-ABI library checks that need no GPU: it builds for sm_100a, loads, exports every function
include/hydro.h declares, and its structs have the C layout (gcc-compiled sizeof/offsetof)."""
import ctypes
import os
import re
import shutil
import subprocess

import pytest
import torch

from paper_2403_14902_b200 import build as B
from paper_2403_14902_b200 import hydro as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hydro.h")


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hydro_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ("hydro_create", "hydro_add_predicate", "hydro_submit_batch", "hydro_collect_results",
              "hydro_get_stats", "hydro_destroy"):
        assert f in fns


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(H.LIB_PATH)
    for f in declared_functions():
        assert hasattr(lib, f), f
    assert set(declared_functions()) == set(H.EXPORTS)


def test_sass_is_sm100a_with_tcgen05():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-sass", H.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for mnem in ("UTCHMMA", "LDTM", "UBLKCP", "UTCBAR"):
        assert mnem in out, mnem
    assert "HMMA" not in out.replace("UTCHMMA", "")  # no legacy mma.sync path


_LAYOUT_C = r"""
#include <stdio.h>
#include <stddef.h>
#include "hydro.h"
#define O(t, f) printf(#t "." #f " %zu\n", offsetof(t, f))
int main(void) {
  printf("hydro_config %zu\nhydro_predicate_desc %zu\nhydro_tuples %zu\nhydro_pred_stats %zu\nhydro_batch_report %zu\n",
         sizeof(hydro_config), sizeof(hydro_predicate_desc), sizeof(hydro_tuples), sizeof(hydro_pred_stats),
         sizeof(hydro_batch_report));
  O(hydro_config, frames); O(hydro_config, frame_w); O(hydro_config, nccl_unique_id);
  O(hydro_predicate_desc, threshold); O(hydro_predicate_desc, weight_bf16); O(hydro_predicate_desc, declared_selectivity);
  O(hydro_predicate_desc, hidden); O(hydro_predicate_desc, weight2_bf16); O(hydro_predicate_desc, bias2);
  O(hydro_tuples, on_device); O(hydro_pred_stats, cost_raw_total); O(hydro_batch_report, cost_raw);
  O(hydro_pred_stats, tuples_computed); O(hydro_pred_stats, cache_hit_rate); O(hydro_batch_report, tuples_computed);
  O(hydro_batch_report, n_pred);
  return 0;
}
"""


def test_ctypes_layout_matches_c(tmp_path):
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    c = tmp_path / "lay.c"
    c.write_text(_LAYOUT_C)
    exe = tmp_path / "lay"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)], check=True)
    got = dict(line.rsplit(" ", 1) for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n") if line)
    for name, st in (("hydro_config", H.hydro_config), ("hydro_predicate_desc", H.hydro_predicate_desc),
                     ("hydro_tuples", H.hydro_tuples), ("hydro_pred_stats", H.hydro_pred_stats),
                     ("hydro_batch_report", H.hydro_batch_report)):
        assert int(got[name]) == ctypes.sizeof(st), name
    for key, val in got.items():
        if "." in key:
            t, f = key.split(".")
            assert getattr(getattr(H, t), f).offset == int(val), key


def test_config_defaults_and_argument_errors():
    cfg = H.hydro_config_default()
    assert (cfg.policy, cfg.decay_gamma, cfg.prior_selectivity, cfg.warmup_tuples, cfg.world) == (0, 0.5, 0.5, 65536, 1)
    lib = H.lib()
    assert lib.hydro_create(None, None) == H.HYDRO_EINVAL
    bad = H.hydro_config_default()
    bad.decay_gamma = 0.0
    h = ctypes.c_void_p()
    assert lib.hydro_create(ctypes.byref(bad), ctypes.byref(h)) == H.HYDRO_EINVAL
    assert b"decay_gamma" in lib.hydro_last_error()
    bad = H.hydro_config_default()
    bad.world = 2  # no unique id
    assert lib.hydro_create(ctypes.byref(bad), ctypes.byref(h)) == H.HYDRO_EINVAL
    assert lib.hydro_destroy(None) == H.HYDRO_OK


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_no_gpu_fails_loudly():
    cfg = H.hydro_config_default()
    with pytest.raises(H.HydroError) as e:
        H.hydro_create(cfg)
    assert e.value.status == H.HYDRO_ECUDA


def test_crop_k_orders_are_row_permutations(tmp_path):
    """The three crop-row K orders of hydro_internal.cuh (K4, K4-T, K4's AREA converter; the weight
    tiling applies the same maps) are permutations of each crop row's 192 features, and the AREA
    order matches its converter's lane mapping (lane q -> pixels q, q + 32)."""
    import shutil
    import subprocess
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    src = os.path.join(ROOT, "tools", "check_k_orders.cu")
    exe = str(tmp_path / "check_k_orders")
    subprocess.run([nvcc, "-std=c++17", "-o", exe, src], check=True, capture_output=True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stdout

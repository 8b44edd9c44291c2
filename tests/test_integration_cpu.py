"""The reference-side binding (integration/allpairs_b200.py) against the reference's
own Application contract.  Runs only where the reference package is importable
(this container); the GPU box has no /root/reference and skips it."""

import ctypes as C
import importlib.util
import os
import sys

import pytest

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _binding():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present")
    sys.dont_write_bytecode = True      # never write into the (read-only) reference tree
    sys.path.insert(0, REF)
    spec = importlib.util.spec_from_file_location("allpairs_b200", os.path.join(HERE, "integration",
                                                                                  "allpairs_b200.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_binding_is_a_reference_application_with_matching_abi():
    mod = _binding()
    from allpairs.apps import Application
    from paper_2009_04755_b200 import _lib
    assert issubclass(mod.B200PCEApp, Application)
    for name in ("preprocess", "compare", "postprocess", "stage_cost"):
        assert getattr(mod.B200PCEApp, name) is not getattr(Application, name)
    # the binding's structs are the header's (same layout as the package's own ctypes mirror)
    assert C.sizeof(mod.RkAppParams) == C.sizeof(_lib.AppParams)
    assert [f[0] for f in mod.RkAppParams._fields_] == [f[0] for f in _lib.AppParams._fields_]
    assert C.sizeof(mod.RkPair) == C.sizeof(_lib.Pair) == 16
    assert mod.lib.rk_pair_id(5, 1, 3) == 1 * (2 * 5 - 1 - 1) // 2 + (3 - 1 - 1)


def test_binding_fails_loudly_without_a_device():
    mod = _binding()
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from allpairs.errors import AppError
    with pytest.raises((AppError, RuntimeError)):
        mod.B200PCEApp(4, side=256)

"""The reference-side binding (integration/allpairs_b200.py) against the reference's
own Application contract.  Uses the reference package staged in oracle/_ref
(oracle/Makefile) or /root/reference; runs the compare path in
tests/test_dropin_gpu.py."""

import ctypes as C
import importlib.util
import os
import sys

import pytest

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = next((p for p in (os.path.join(HERE, "oracle", "_ref"), "/root/reference/pkg/src")
            if os.path.isdir(os.path.join(p, "allpairs"))), None)


def _binding():
    if REF is None:
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
    from allpairs.apps import CompositionVectorApp
    assert issubclass(mod.B200PCEApp, Application)
    for name in ("preprocess", "compare", "postprocess", "stage_cost"):
        assert getattr(mod.B200PCEApp, name) is not getattr(Application, name)
    # the CV drop-in keeps the reference's corpus I/O and parse, replaces preprocess/compare
    assert issubclass(mod.B200CompositionVectorApp, CompositionVectorApp)
    for name in ("path_for_key", "fetch_raw", "parse", "postprocess"):
        assert getattr(mod.B200CompositionVectorApp, name) is getattr(CompositionVectorApp, name)
    for name in ("preprocess", "compare"):
        assert getattr(mod.B200CompositionVectorApp, name) is not getattr(CompositionVectorApp, name)
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

"""A short run of the randomised parity sweep (tests/fuzz_parity.py): random m, n, d, input kinds
and launch options; the dense and CSR sketches bit-exact against the oracle and the solve in
lockstep with it, in both stop modes.  The full sweeps are in profiles/r01_fuzz_parity.txt."""
import importlib.util
import os
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [20261019, 7])
def test_random_cases(seed, monkeypatch, capsys):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "fuzz_parity.py")
    spec = importlib.util.spec_from_file_location("fuzz_parity", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    monkeypatch.setattr(sys, "argv", ["fuzz_parity.py", "12", str(seed)])
    mod.main()  # exits 1 (SystemExit) or raises on the first mismatch
    assert "all 12 cases passed" in capsys.readouterr().out

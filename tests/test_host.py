"""CPU-side checks: the C-ABI library loads and exports its header, and the
host logic (selectors, family encoding, preconditions) mirrors the reference."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO


def _header_symbols():
    src = open(os.path.join(REPO, "include", "meshfree_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*|long long)\s+(mf_\w+)\s*\(", src, re.M)))


def test_library_builds_and_exports_every_header_symbol():
    from paper_1912_13282_b200 import _lib, build

    path = build.build()
    lib = ctypes.CDLL(path)
    syms = _header_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
    assert set(syms) == set(_lib.EXPORTS)
    assert _lib.load().mf_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    from paper_1912_13282_b200 import build

    out = subprocess.run(["cuobjdump", "--list-elf", build.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_expand_families_matches_reference_rules():
    from paper_1912_13282_b200 import FirstDerivative, StorageError, expand_families

    assert list(expand_families(["laplacian", "gradient"], 2)) == ["laplacian", "d1_0", "d1_1"]
    assert list(expand_families(["hessian"], 2)) == ["d2_0_0", "d2_0_1", "d2_1_1"]
    assert list(expand_families([("conv", FirstDerivative(0))], 2)) == ["conv"]
    for bad in (["laplacian", "laplacian"], ["d1_5"], [], ["d2_1_0"], ["curl"]):
        with pytest.raises(StorageError):
            expand_families(bad, 2)


def test_family_encoding_matches_oracle():
    import oracle

    from paper_1912_13282_b200.storage import encode_families, expand_families

    for dim, deg, fams in ((2, 2, ["laplacian", "gradient", "hessian", "identity"]),
                           (3, 4, ["laplacian", "gradient"]), (1, 3, ["d2_0_0"]), (3, 2, ["d2_0_2"])):
        kinds, ax_a, ax_b, orders, expos, base_bot = encode_families(expand_families(fams, dim), dim, deg)
        keys, codes, oexpos, obase = oracle.encode(fams, dim, deg)
        assert np.array_equal(np.stack([kinds, ax_a, ax_b, orders], 1), codes)
        assert np.array_equal(expos, oexpos)
        assert np.array_equal(base_bot, obase)


def test_graded_lex_order():
    from paper_1912_13282_b200 import graded_lex_exponents, monomial_count

    assert graded_lex_exponents(2, 2) == [(0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2)]
    assert len(graded_lex_exponents(3, 4)) == monomial_count(4, 3) == 35


def test_nodeset_selectors_and_errors():
    from paper_1912_13282_b200 import GeometryError, NodeSet, StencilError

    types = np.array([1, -1, 2, -2, 0, 1])
    ns = NodeSet(np.zeros((6, 2)), types)
    assert ns.select(None).tolist() == list(range(6))
    assert ns.select("interior").tolist() == [0, 2, 5]
    assert ns.select("boundary").tolist() == [1, 3]
    assert ns.select(-2).tolist() == [3]
    assert ns.select([1, 0]).tolist() == [0, 4, 5]
    assert ns.select(np.array([5, 1])).tolist() == [5, 1]
    assert ns.select(types > 0).tolist() == [0, 2, 5]
    for bad in ("nope", np.array([7]), np.ones(3, dtype=bool)):
        with pytest.raises(GeometryError):
            ns.select(bad)
    with pytest.raises(GeometryError):
        NodeSet(np.zeros(3), [1, 1, 1])
    with pytest.raises(StencilError):
        ns.stencil(0)
    ns2 = ns.with_stencils([0, 2], [np.array([0, 1, 2]), np.array([2, 0, 1])])
    assert ns2.has_stencil(2) and not ns2.has_stencil(1)
    assert ns2.stencil_matrix(np.array([0, 2])).tolist() == [[0, 1, 2], [2, 0, 1]]
    assert ns2.stencils[1] is None and ns2.stencils[2].tolist() == [2, 0, 1]
    ns3 = ns2.with_stencils([5], [np.array([5, 0])])
    with pytest.raises(StencilError, match="differ"):
        ns3.stencil_matrix(np.array([0, 5]))
    with pytest.raises(StencilError, match="node 1 has no stencil"):
        ns3.stencil_matrix(np.array([0, 1]))
    big = ns2.append([[1.0, 1.0]], -3)
    assert len(big) == 7 and big.has_stencil(0) and not big.has_stencil(6)
    with pytest.raises(GeometryError):
        ns.normal(0)


def test_stencil_preconditions_without_gpu():
    from paper_1912_13282_b200 import NodeSet, StencilError, find_closest_stencils

    ns = NodeSet(np.random.default_rng(0).uniform(size=(10, 2)), np.ones(10, dtype=np.int64))
    with pytest.raises(StencilError, match="exceeds search pool of 10"):
        find_closest_stencils(ns, 11)
    with pytest.raises(StencilError, match="at least 1"):
        find_closest_stencils(ns, 0)
    assert find_closest_stencils(ns, 3, for_which=np.array([], dtype=np.int64)) is ns


def test_compute_weights_preconditions_without_gpu():
    from paper_1912_13282_b200 import (ConfigError, NodeSet, Polyharmonic, RbfFd, StencilError,
                                       StorageError, compute_weights)

    ns = NodeSet(np.zeros((4, 2)), np.ones(4, dtype=np.int64))
    eng = RbfFd(Polyharmonic(3), degree=1, scale="support", solver="lu")
    with pytest.raises(StencilError, match="no node has a stencil"):
        compute_weights(ns, eng, ["laplacian"])
    ns = ns.with_stencils([0, 1], [np.array([0, 1, 2]), np.array([1, 0, 2])])
    with pytest.raises(StencilError, match="node 2 has no stencil"):
        compute_weights(ns, eng, ["laplacian"], for_which=np.array([0, 2]))
    # qr / svd, r^1, unknown scale rules run in the general engine kernel (GPU);
    # Python-defined kernels / weights / engines cannot run there at all
    with pytest.raises(ConfigError):
        compute_weights(ns, RbfFd(object(), degree=1), ["laplacian"])
    with pytest.raises(ConfigError):
        from paper_1912_13282_b200 import WeightedLeastSquares
        compute_weights(ns, WeightedLeastSquares(1, weight=lambda x: 1.0), ["laplacian"])
    with pytest.raises(ConfigError):
        compute_weights(ns, object(), ["laplacian"])
    with pytest.raises(StorageError, match="no engine given"):
        compute_weights(ns, {"laplacian": eng}, ["laplacian", "gradient"])
    with pytest.raises(StorageError, match="two engines"):
        compute_weights(ns, {"gradient": eng, "d1_0": eng}, ["gradient"])


def test_heat_argument_checks_without_gpu():
    from paper_1912_13282_b200 import ConfigError, NodeSet, run_heat_explicit

    ns = NodeSet(np.zeros((4, 2)), np.ones(4, dtype=np.int64))
    with pytest.raises(ConfigError):
        run_heat_explicit(ns, None, dt=0.0, steps=1)
    with pytest.raises(ConfigError):
        run_heat_explicit(ns, None, dt=1.0, steps=-1)


def test_gpu_entry_points_fail_loudly_without_device():
    import torch

    from paper_1912_13282_b200 import NodeSet, find_closest_stencils
    from paper_1912_13282_b200._lib import LibraryError

    if torch.cuda.is_available():
        pytest.skip("device present")
    ns = NodeSet(np.random.default_rng(0).uniform(size=(10, 2)), np.ones(10, dtype=np.int64))
    with pytest.raises(LibraryError, match="no CPU fallback"):
        find_closest_stencils(ns, 3)


def test_workloads_match_survey_inputs():
    from paper_1912_13282_b200 import workloads

    c2 = workloads.c2()
    assert c2.N == 200_023
    assert np.allclose(c2.extra["centres"][0], [0.164, -0.276], atol=1e-3)
    c4 = workloads.c4(1_000_000)
    assert int((c4.types < 0).sum()) == 3946

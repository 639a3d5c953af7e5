"""CPU-side checks of the product: the C ABI loads and exports every symbol the
header declares, the host table builder and the restated libm are bit-exact
with the reference / host glibc, and the API surface mirrors the reference.
No GPU compute here."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from oracle import gz_oracle as O

import paper_2405_19493_b200 as gz
from paper_2405_19493_b200 import _lib


def header_symbols():
    text = open(os.path.join(ROOT, "include", "gz_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gz_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.load(require_device=False)
    syms = header_symbols()
    assert len(syms) >= 18
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing
    assert set(syms) == set(_lib.EXPORTS)
    assert L.gz_version() >= 100


def test_no_device_means_loud_failure():
    L = _lib.load(require_device=False)
    if L.gz_device_count() > 0:
        pytest.skip("a CUDA device is visible")
    with pytest.raises(gz.EngineUnavailable):
        _lib.load()
    assert not gz.engine.available()
    assert not gz.engine.supports(gz.make_source("lcg48", 1))
    with pytest.raises(gz.EngineUnavailable):
        gz.engine.fill_gaussians(gz.make_sampler("polar"), gz.make_source("lcg48", 1), np.empty(4))


@pytest.mark.parametrize("n", [8, 16, 32, 64, 128, 256, 512, 1024])
def test_host_table_builder_is_bit_exact(n, golden):
    assert gz.tables_to_json(gz.build_ziggurat_tables(n)) == golden["tables"][str(n)]


def test_tables_json_round_trip_and_pins():
    t = gz.build_ziggurat_tables(128)
    assert gz.tables_from_json(gz.tables_to_json(t)) == t
    assert "3.4426198558966377" in gz.tables_to_json(t)           # test_tables.py:89-91
    assert (t.index_bits, t.mantissa_bits) == (7, 56)
    assert t.ktab[-1] == 0                                        # test_tables.py:71-72
    t2 = gz.build_ziggurat_tables(256)
    assert (t2.index_bits, t2.mantissa_bits) == (8, 55)
    assert abs(t.r - 3.442619855899) < 1e-9 and abs(t2.r - 3.654152885361) < 1e-9


def test_tables_reject_bad_layer_counts_and_corruption():
    for n in (0, 7, 100, 129, -8):
        with pytest.raises(ValueError):
            gz.build_ziggurat_tables(n)
    doc = json.loads(gz.tables_to_json(gz.build_ziggurat_tables(128)))
    doc["x"][3], doc["x"][4] = doc["x"][4], doc["x"][3]
    with pytest.raises(Exception):
        gz.tables_from_json(json.dumps(doc))


@pytest.mark.parametrize("fn", [0, 1])
def test_restated_libm_matches_host_glibc(fn):
    """The exp/log the kernels use, compiled for the host, vs the host glibc."""
    L = _lib.load(require_device=False)
    f = L.gz_libm_exp if fn == 0 else L.gz_libm_log
    xs = O.sweep_inputs(fn, 1 << 17, 100 + fn)
    got = np.array([f(float(v)) for v in xs])
    bad, first = O.libm_mismatches(fn, xs, got)
    assert bad == 0, xs[first]


def test_sources_known_answers():
    s = gz.Lcg48(0)
    v = s.next_bits(32)
    assert v - (1 << 32) == -1155484576                           # test_sources.py:24-27
    assert gz.SplitMix64(0).next_u64() == 0xE220A8397B1DCDAF      # test_sources.py:93-102
    for src, digest in (("lcg48", 0x425FE4E2A7905F40), ("splitmix", 0x399AC485230C35E0)):
        s, acc = gz.make_source(src, 12345), 0
        for _ in range(10_000):
            acc ^= s.next_u64()
        assert acc == digest                                      # test_sources.py:9-10
    assert gz.SplitMix64(3, gamma=0x1234567890ABCDE0).gamma & 1 == 1
    with pytest.raises(ValueError):
        gz.make_source("nope", 1)
    with pytest.raises(gz.ScriptExhausted):
        gz.ScriptedSource([]).next_u64()


def test_sampler_registry_and_pairing_gate():
    assert isinstance(gz.make_sampler("polar"), gz.PolarSampler)
    assert gz.make_sampler("ziggurat").tables.n == 128
    assert gz.make_sampler("modified-ziggurat").tables.n == 256
    assert gz.make_sampler("ziggurat", layers=64).tables.n == 64
    with pytest.raises(ValueError):
        gz.make_sampler("polar", layers=128)
    with pytest.raises(ValueError):
        gz.make_sampler("box-muller")
    assert not gz.is_sanctioned("lcg48", "modified-ziggurat")
    with pytest.raises(gz.UnsanctionedPairing):
        gz.require_sanctioned("lcg48", "modified-ziggurat")
    gz.require_sanctioned("splitmix", "modified-ziggurat")
    with pytest.raises(ValueError):
        gz.gaussian_affine(gz.make_source("lcg48", 1), gz.make_sampler("polar"), 0.0, -1.0)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2405_19493_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "gz_oracle" not in text and "libgzoracle" not in text, f

"""CPU checks of the boundary: the C-ABI library loads and exports every symbol the header
declares; host-only queries work without a GPU (no kernel is launched here)."""
import ctypes
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sntrup_gpu.h")


def _build_mod():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_sntrup_build", os.path.join(ROOT, "paper_2106_08759_b200", "_build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.fixture(scope="module")
def lib():
    b = _build_mod()
    b.build()
    return ctypes.CDLL(b.LIB)


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b([a-z_][a-z0-9_]*)\s*\(", txt, flags=re.M)
    return sorted(set(n for n in names if n not in ("defined",)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("sntrup_batch_keygen", "rq_mul_batch", "rq_recip_batch", "r3_recip_batch"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _build_mod().LIB], capture_output=True, text=True).stdout
    exported = set(l.split()[-1] for l in out.splitlines() if l.strip())
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_params_host_query(lib):
    import paper_2106_08759_b200 as S
    assert S.params(761) == dict(p=761, q=4591, w=286, p16=768, p8=768, pk_bytes=1158, sk_bytes=382)
    exp = {653: (994, 328), 857: (1322, 430), 953: (1505, 478), 1013: (1623, 508), 1277: (2067, 640)}
    for ps, (pk, sk) in exp.items():
        P = S.params(ps)
        assert (P["pk_bytes"], P["sk_bytes"]) == (pk, sk)
    with pytest.raises(S.SntrupError) as e:
        S.params(512)
    assert e.value.code == S.SNTRUP_E_PARAM


def test_argument_errors_without_gpu(lib):
    # n == 0 and unknown parameter sets are rejected before any device work
    import paper_2106_08759_b200 as S
    assert S._lib.sntrup_batch_keygen(761, 0, 1, None, None) == S.SNTRUP_E_ARG
    assert S._lib.sntrup_batch_keygen(700, 5, 1, None, None) == S.SNTRUP_E_PARAM
    assert S._lib.rq_mul_batch(761, 0, None, None, None, None) == S.SNTRUP_E_ARG
    assert S._lib.sntrup_strerror(S.SNTRUP_E_NOT_INVERTIBLE) == b"element not invertible"
    assert S._lib.sntrup_set_mul_impl(17) == S.SNTRUP_E_ARG
    assert S._lib.sntrup_set_mul_impl(12) == S.SNTRUP_OK
    assert S._lib.sntrup_set_mul_impl(11) == S.SNTRUP_OK
    assert S._lib.sntrup_set_mul_impl(10) == S.SNTRUP_OK
    assert S._lib.sntrup_set_mul_impl(9) == S.SNTRUP_OK
    assert S._lib.sntrup_set_mul_impl(8) == S.SNTRUP_OK
    assert S._lib.sntrup_set_mul_impl(7) == S.SNTRUP_OK
    assert S._lib.sntrup_set_mul_impl(6) == S.SNTRUP_OK
    assert S._lib.sntrup_set_mul_impl(2) == S.SNTRUP_OK
    with pytest.raises(S.SntrupError):
        S.set_mul_impl(-1)
    S.set_mul_impl(S.MUL_SCHOOLBOOK)
    S.set_mul_impl(S.MUL_TENSOR_CORE)


def test_root_impl_knob_without_gpu(lib):
    # sntrup_set_root_impl: 0 automatic, 1 one divstep at a time, 2 jump-divsteps, + 4 shared SMs
    import paper_2106_08759_b200 as S
    for v in (S.ROOT_AUTO, S.ROOT_STEP, S.ROOT_JUMP, S.ROOT_AUTO | S.ROOT_SHARED_SM,
              S.ROOT_JUMP | S.ROOT_SHARED_SM, S.ROOT_STEP | S.ROOT_SHARED_SM):
        assert S._lib.sntrup_set_root_impl(v) == S.SNTRUP_OK, v
    for v in (-1, 3, 7, 8):
        assert S._lib.sntrup_set_root_impl(v) == S.SNTRUP_E_ARG, v
    with pytest.raises(S.SntrupError):
        S.set_root_impl(3)
    S.set_root_impl(S.ROOT_AUTO)
    # sntrup_set_sched: tree-top routing threshold and items-per-CTA cap, both >= 0
    assert S._lib.sntrup_set_sched(1024, 4) == S.SNTRUP_OK
    assert S._lib.sntrup_set_sched(-1, 0) == S.SNTRUP_E_ARG
    assert S._lib.sntrup_set_sched(0, -2) == S.SNTRUP_E_ARG
    S.set_sched(0, 0)


def test_graph_flag_value():
    # SNTRUP_OPT_GRAPH in the binding matches the header
    import paper_2106_08759_b200 as S
    txt = open(HEADER).read()
    m = re.search(r"#define SNTRUP_OPT_GRAPH\s+(\d+)u", txt)
    assert m and int(m.group(1)) == S.OPT_GRAPH == 512


def test_full_sk_sizes_host_query(lib):
    import paper_2106_08759_b200 as S
    # App. D key-pair storage: pk + full sk = 2512 / 2921 / 3321
    for param, pair in ((653, 2512), (761, 2921), (857, 3321)):
        assert S.params(param)["pk_bytes"] + S.full_sk_bytes(param) == pair
    assert S._lib.sntrup_full_sk_bytes(700) == 0
    assert S._lib.sntrup_full_sk_batch(761, 0, 1, 0, None, None, None, None) == S.SNTRUP_E_ARG
    assert S._lib.sntrup_full_sk_batch(700, 5, 1, 0, None, None, None, None) == S.SNTRUP_E_PARAM


def irreducible_gf3(f):
    """Rabin's test over GF(3): x^(3^d) = x mod f and gcd(x^(3^(d/r)) - x, f) = 1, r | d prime."""
    import numpy as np
    import polytools as PT
    d = len(f) - 1

    def frob_pow(k):                       # x^(3^k) mod f
        h = np.array([0, 1])
        for _ in range(k):
            h = PT.gf_divmod(np.mod(PT.gf_mul(PT.gf_mul(h, h, 3), h, 3), 3), f, 3)[1]
        return h

    def minus_x(h):
        h = np.concatenate([h, np.zeros(max(0, 2 - len(h)), np.int64)])
        h[1] = (h[1] - 1) % 3
        return PT.trim(h)

    if len(minus_x(frob_pow(d))):
        return False
    for r in [r for r in range(2, d + 1) if d % r == 0 and all(r % s for s in range(2, r))]:
        if len(PT.gf_gcd(f, minus_x(frob_pow(d // r)), 3)) > 1:
            return False
    return True


def test_factor_tables_are_factors():
    # the generated small-factor tables divide x^p - x - 1 over GF(3) and are irreducible of
    # the stated degree (checked with the tests' own polynomial code)
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import numpy as np
    import polytools as PT
    src = open(os.path.join(ROOT, "paper_2106_08759_b200", "csrc", "factor_tables.h")).read()
    rows = re.findall(r"\{(\d+), (\d+), \{([\d, ]+)\}, \{([^}]*)\}\}", src)
    assert len(rows) == 6
    for p, cnt, degs, coefs in rows:
        p = int(p)
        degs = [int(d) for d in degs.split(",")]
        coefs = re.findall(r'"(\d+)"', coefs)
        assert len(coefs) == int(cnt) == len(degs)
        for d, cs in zip(degs, coefs):
            f = np.array([int(c) for c in cs])
            assert len(f) == d + 1 and f[-1] == 1
            _, r = PT.gf_divmod(PT.modulus(p, 3), f, 3)
            assert len(r) == 0
            assert irreducible_gf3(f)
    # 761: f1 digits match SURVEY C16's golden table check
    assert '"22022212120211112011"' in src


def test_missing_library_fails_loudly(tmp_path):
    # no CPU fallback: without the CUDA library the package refuses to import
    env = dict(os.environ, SNTRUP_GPU_LIB=str(tmp_path / "absent.so"))
    r = subprocess.run([sys.executable, "-c", "import paper_2106_08759_b200"], cwd=ROOT, env=env,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "no CPU fallback" in r.stderr


def test_product_code_never_touches_the_oracle():
    # the oracle is test infrastructure: nothing in the package (Python or CUDA/C) names it
    pkg = os.path.join(ROOT, "paper_2106_08759_b200")
    offenders = []
    for d, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp", ".c")):
                src = open(os.path.join(d, f), encoding="utf-8", errors="replace").read()
                for pat in (r"^\s*(import|from)\s+oracle\b", r"#include\s+[\"<][^\">]*oracle",
                            r"sntrup_oracle|liboracle|oracle\.so|oracle\.py", r"\bor_keygen\b"):
                    if re.search(pat, src, re.M):
                        offenders.append((f, pat))
    assert not offenders, offenders


def test_compute_calls_reject_host_tensors(lib):
    # the Python binding only marshals device tensors; host tensors are an error, not a fallback
    import torch
    import paper_2106_08759_b200 as S
    a = torch.zeros((4, 768), dtype=torch.int16)
    with pytest.raises((ValueError, RuntimeError, AssertionError)):
        S.rq_mul_batch(761, a, a.clone())


def test_workspace_query_host_only(lib):
    import paper_2106_08759_b200 as S
    L = S._lib
    assert L.sntrup_keygen_workspace_bytes(700, 10, 32) == 0
    assert L.sntrup_keygen_workspace_bytes(761, 0, 32) == 0
    assert L.sntrup_keygen_workspace_bytes_ex(761, 100, 3, 0, 0) == 0          # B not a power of two
    a = S.keygen_workspace_bytes(761, 65536, 1024, 0, 32768)
    b = S.keygen_workspace_bytes(761, 65536, 1024, S.OPT_LANES4, 16384)
    assert a > 0 and b > 0
    # one lane per chunk up to the lane count: 2 lanes of 32768 keys vs 4 lanes of 16384 keys
    # hold the same number of keys' buffers (+ per-level rounding)
    assert abs(a - b) < 0.01 * a
    # the plain query is the _ex query with default options
    assert L.sntrup_keygen_workspace_bytes(761, 5000, 64) == S.keygen_workspace_bytes(761, 5000, 64)
    # host outputs do not enlarge the workspace (staging is a separate allocation)
    assert S.keygen_workspace_bytes(761, 65536, 1024, S.OPT_HOST_OUTPUT, 32768) == a


def test_binding_checks_caller_outputs_without_gpu(lib):
    # outputs supplied by the caller are checked (shape, dtype, placement) before any
    # library call; host-output keygen wants host tensors
    import torch
    import paper_2106_08759_b200 as S
    bad = torch.zeros((4, 100), dtype=torch.uint8)
    sk = torch.zeros((4, 382), dtype=torch.uint8)
    with pytest.raises(ValueError):
        S.batch_keygen(761, 4, 1, flags=S.OPT_HOST_OUTPUT, pk_out=bad, sk_out=sk)
    with pytest.raises(ValueError):
        S.batch_keygen(761, 4, 1, flags=S.OPT_HOST_OUTPUT, pk_out=torch.zeros((4, 1158), dtype=torch.int16),
                       sk_out=sk)

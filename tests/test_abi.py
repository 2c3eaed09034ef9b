"""CPU-side checks of the C ABI: the library builds, loads, exports every
symbol include/embrace.h declares, validates configs on the host, and its
dense-queue issue rule equals the oracle's (pure host logic, no GPU)."""

import os
import random
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def E():
    from paper_2110_09132_b200.build import build
    build()
    from paper_2110_09132_b200 import embrace
    embrace.lib()
    return embrace


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "embrace.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(\w+)\s*\(", src, flags=re.M)))


def test_exports_every_declared_symbol(E):
    declared = _declared_functions()
    assert len(declared) >= 17
    L = E.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(E.EXPORTED) == declared


def test_status_strings(E):
    for code, name in E.STATUS.items():
        assert E.emb_status_str(code) == name


def test_host_validation(E):
    ok = E.make_config(1000, 16, world=2, rank=0)
    sym, loc = E.emb_workspace_bytes(ok)
    assert sym > 1000 * 8 * 4 and loc > 0
    bad = [
        (E.make_config(1000, 16, world=3), "EMB_ERR_SHAPE"),       # D % N != 0
        (E.make_config(1000, 16, world=8), "EMB_ERR_SHAPE"),       # d*e = 8 B, not a 16 B multiple
        (E.make_config(1000, 4, world=8), "EMB_ERR_SHAPE"),        # N > D... and N > 8 rejected below
        (E.make_config(1000, 16, world=2, rank=2), "EMB_ERR_INVALID_ARG"),
        (E.make_config(1000, 16, max_tokens=0), "EMB_ERR_CAPACITY"),
        (E.make_config(1000, 16, max_tokens=40000), "EMB_ERR_CAPACITY"),  # cap 32768 (16-CTA sort)
        (E.make_config(0, 16), "EMB_ERR_INVALID_ARG"),
    ]
    for cfg, want in bad:
        with pytest.raises(E.EmbError) as ei:
            E.emb_workspace_bytes(cfg)
        assert ei.value.name == want
    c = E.make_config(1000, 64, world=9)
    with pytest.raises(E.EmbError):
        E.emb_workspace_bytes(c)


def test_issue_rule_matches_oracle(E):
    from oracle.schedule import issue_order
    rng = random.Random(3)
    for _ in range(500):
        n = rng.randint(0, 30)
        pr = [rng.randint(-5, 5) for _ in range(n)]
        for W in (1, 2, 3, 8, 64):
            assert E.emb_queue_issue_order(pr, W) == issue_order(pr, W)

"""Checkpoint / resume on the host: the saved state round-trips exactly, the
RNG streams continue where they left off, and bad files are refused."""
import os

import pytest
import torch

from paper_2510_14564_b200 import checkpoint


def state(n=37, seed=0):
    g = torch.Generator().manual_seed(seed)
    return [torch.randn(59 * n, generator=g) for _ in range(3)]


def test_roundtrip_and_rng_continuation(tmp_path):
    n = 37
    th, m, v = state(n)
    gen = torch.Generator().manual_seed(5)
    torch.manual_seed(11)
    torch.rand(3)
    torch.randn(2, generator=gen)
    path = str(tmp_path / "a.pt")
    checkpoint.save(path, th, m, v, step=123, n=n, sh_degree=3, generators={"density": gen},
                    extra={"camera_cursor": 9, "hint0": torch.arange(5, dtype=torch.int32)})
    want_host = torch.rand(4)
    want_gen = torch.randn(4, generator=gen)
    torch.manual_seed(999)  # disturb both streams
    gen.manual_seed(1)
    st = checkpoint.load(path, generators={"density": gen})
    assert st["step"] == 123 and st["n"] == n and st["sh_degree"] == 3
    assert torch.equal(st["theta"], th) and torch.equal(st["exp_avg"], m) and torch.equal(st["exp_avg_sq"], v)
    assert st["extra"]["camera_cursor"] == 9 and torch.equal(st["extra"]["hint0"], torch.arange(5, dtype=torch.int32))
    assert torch.equal(torch.rand(4), want_host)
    assert torch.equal(torch.randn(4, generator=gen), want_gen)


def test_bad_shapes_are_refused_before_writing(tmp_path):
    th, m, v = state(10)
    path = str(tmp_path / "b.pt")
    checkpoint.save(path, th, m, v, step=1, n=10, sh_degree=3)
    before = open(path, "rb").read()
    with pytest.raises(ValueError):
        checkpoint.save(path, th[:-1], m, v, step=2, n=10, sh_degree=3)
    assert open(path, "rb").read() == before  # the previous checkpoint is intact
    assert not [f for f in os.listdir(tmp_path) if ".tmp" in f]


def test_truncated_and_foreign_files_are_refused(tmp_path):
    th, m, v = state(10)
    path = str(tmp_path / "c.pt")
    checkpoint.save(path, th, m, v, step=1, n=10, sh_degree=3)
    data = open(path, "rb").read()
    bad = str(tmp_path / "trunc.pt")
    with open(bad, "wb") as f:
        f.write(data[: len(data) // 2])
    with pytest.raises(ValueError):
        checkpoint.load(bad)
    other = str(tmp_path / "other.pt")
    torch.save({"format": 99}, other)
    with pytest.raises(ValueError):
        checkpoint.load(other)
    inconsistent = str(tmp_path / "inc.pt")
    st = torch.load(path, weights_only=False)
    st["n"] = 11
    torch.save(st, inconsistent)
    with pytest.raises(ValueError):
        checkpoint.load(inconsistent)
    with pytest.raises(ValueError):
        checkpoint.load(path, generators={"missing": torch.Generator()})

"""CLI parity with the reference's test_cli.py (gen hex/json/raw, jump).
hex/json/jump run on the host (CPU); raw output goes through the GPU."""

import io
import json
import sys

import numpy as np
import pytest

import paper_1805_01407_b200 as P
from paper_1805_01407_b200 import cli


def run_cli(capsys, *argv):
    code = cli.main(list(argv))
    out = capsys.readouterr()
    return code, out.out, out.err


def test_hex_matches_golden(capsys, G):
    code, out, _ = run_cli(capsys, "gen", "--algo", "xoshiro256starstar", "--seed", "42", "--values", "8",
                           "--format", "hex")
    assert code == 0
    want = G("generators")["xoshiro256starstar"]["first_outputs_seed42"][:8]
    assert ["0x" + t.lstrip("0") for t in out.split()] == want


def test_zero_values_and_unknown(capsys):
    code, out, _ = run_cli(capsys, "gen", "--algo", "xoroshiro128plus", "--seed", "1", "--values", "0",
                           "--format", "hex")
    assert code == 0 and out == ""
    code, _, err = run_cli(capsys, "gen", "--algo", "nope", "--values", "1", "--format", "hex")
    assert code == 2 and "unknown algorithm" in err


def test_state_escape_hatch_and_json(capsys):
    code, out, _ = run_cli(capsys, "gen", "--algo", "xoroshiro128plus", "--state", "1,2", "--values", "1",
                           "--format", "hex")
    assert code == 0 and out.strip() == f"{3:016x}"
    code, out, _ = run_cli(capsys, "gen", "--algo", "xoroshiro64star", "--seed", "3", "--values", "5",
                           "--format", "json")
    doc = json.loads(out)
    g = P.Generator.from_seed(P.get_spec("xoroshiro64star"), 3)
    assert doc["values"] == [g.next() for _ in range(5)]


def test_jump_cli(capsys):
    code, out, _ = run_cli(capsys, "jump", "--algo", "xoroshiro128plus", "--seed", "1", "--steps", "0", "--json")
    g = P.Generator.from_seed(P.get_spec("xoroshiro128plus"), 1)
    assert json.loads(out)["state"] == [f"{x:016x}" for x in g.flat_words()]
    _, out1, _ = run_cli(capsys, "jump", "--algo", "xoshiro256plus", "--seed", "11", "--steps", "1000", "--json")
    state = json.loads(out1)["state"]
    _, out2, _ = run_cli(capsys, "jump", "--algo", "xoshiro256plus", "--state", " ".join(state), "--steps", "1000",
                         "--json")
    _, out3, _ = run_cli(capsys, "jump", "--algo", "xoshiro256plus", "--seed", "11", "--steps", "2000", "--json")
    assert json.loads(out2)["state"] == json.loads(out3)["state"]
    _, out, _ = run_cli(capsys, "jump", "--algo", "xoroshiro128plus", "--seed", "1", "--json")
    assert json.loads(out)["steps"] == str(1 << 64)
    _, out, _ = run_cli(capsys, "jump", "--algo", "xoshiro256plus", "--seed", "1", "--long-jump", "--json")
    assert json.loads(out)["steps"] == str(1 << 192)


def _raw(monkeypatch, *argv):
    buf = io.BytesIO()

    class FakeStdout:
        buffer = buf

    monkeypatch.setattr(sys, "stdout", FakeStdout())
    code = cli.main(list(argv))
    return code, buf.getvalue()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["xoroshiro128plus", "xoshiro128plus", "xoroshiro1024starstar",
                                  "xoshiro256starstar"])
def test_raw_matches_golden(monkeypatch, G, name):
    code, data = _raw(monkeypatch, "gen", "--algo", name, "--seed", "42", "--values", "100", "--format", "raw")
    assert code == 0
    w = P.get_spec(name).kind.w
    words = np.frombuffer(data, dtype="<u8" if w == 64 else "<u4")
    assert [hex(int(x)) for x in words] == G("generators")[name]["first_outputs_seed42"]


@pytest.mark.gpu
def test_raw_long_stream_equals_laned(monkeypatch):
    """3e6 values (several lanes, ragged end) equal the reference laned stream (oracle)."""
    from oracle import oracle as O

    code, data = _raw(monkeypatch, "gen", "--algo", "xoshiro256plusplus", "--seed", "9", "--values", "3e6")
    assert code == 0
    words = np.frombuffer(data, dtype="<u8")
    assert words.size == 3_000_000
    want = O.laned_stream("xoshiro256plusplus", 9, 3_000_000, 4096, 1024)
    np.testing.assert_array_equal(words, want)


@pytest.mark.gpu
def test_raw_zero_values(monkeypatch):
    code, data = _raw(monkeypatch, "gen", "--algo", "xoshiro256plus", "--values", "0")
    assert code == 0 and data == b""


def test_hwd_stdin_rejected(capsys):
    code, _, err = run_cli(capsys, "hwd", "--stdin")
    assert code == 2 and "--algo" in err


@pytest.mark.gpu
def test_hwd_cli_detects_xorshift128plus(capsys, G):
    """The paper row through the CLI (reference cli.py:122-160): the JSON report
    equals the reference's own report for the same run (tests/golden/hwd.json)."""
    key = "xorshift128plus/1/None/batch_size=2300000,byte_limit=24000000000,k=8,mode=transitional,w=64"
    want = {k: v for k, v in G("hwd")[key].items()
            if k not in ("name", "seed", "checkpoint_start", "config", "ref_seconds")}
    code, out, _ = run_cli(capsys, "hwd", "--algo", "xorshift128plus", "--mode", "transitional",
                           "--limit", "2.4e10", "--seed", "1", "--json")
    assert code == 3
    assert json.loads(out) == want
    assert want["status"] == "failed" and want["signature"] == "00000021"

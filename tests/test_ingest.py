"""Host-side trace ingest (NEXT-4): the oracle (oracle/ingest.py) pinned to the paper's listings and
SPEC's examples, and the product's host calls (ct_parse_tool_name, ct_load_trace_jsonl; no CUDA
call) compared with it on goldens, fuzzed messages, generated traces and invalid records.  The
GPU test replays a loaded trace against the oracle's replay of the generator's records."""
import json
import os
import random

import numpy as np
import pytest

from ctgen import traces
from oracle import ingest as OI

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "tool_messages.jsonl")


def goldens():
    return [json.loads(l) for l in open(GOLD)]


@pytest.fixture(scope="module")
def ct():
    from paper_2511_02230_b200 import build
    build.build()
    import paper_2511_02230_b200 as ct
    return ct


# ---- oracle pins --------------------------------------------------------------------------------
@pytest.mark.parametrize("g", goldens(), ids=lambda g: g["cite"][:40])
def test_oracle_tool_name_goldens(g):
    assert OI.parse_tool_name(g["message"], g["format"]) == (g["name"], g["malformed"])


def test_oracle_bash_rule_is_first_token_of_first_subcommand():
    # App. A: split on && or || (not on ; or |), first whitespace token
    assert OI.bash_name("  git   status\n") == "git"
    assert OI.bash_name("ls||echo x") == "ls"
    assert OI.bash_name("cat a.txt | grep x && y") == "cat"
    assert OI.bash_name("&& ls") is None
    assert OI.bash_name("") is None


def write(tmp_path, lines, name="t.jsonl"):
    p = tmp_path / name
    p.write_text("".join(l + "\n" for l in lines))
    return str(p)


REC2 = ('{"program_id": "a", "arrival_time_s": 3.5, "turns": ['
        '{"new_prompt_tokens": 100, "decode_tokens": 20, "tool_name": "pytest", "tool_duration_s": 8.25},'
        '{"new_prompt_tokens": 40, "decode_tokens": 5}]}')


def test_oracle_load_spec_examples(tmp_path):
    # a 1-line file with a 2-turn program -> one program, 2 turns
    progs, names, w = OI.load_trace_jsonl(write(tmp_path, [REC2]))
    assert progs == [(3_500_000, [(100, 20, 0, 8_250_000), (40, 5, -1, 0)])] and names == ["pytest"]
    assert w == 0
    # tool_name without tool_duration_s -> load error
    bad = REC2.replace(', "tool_duration_s": 8.25', "")
    with pytest.raises(OI.TraceError):
        OI.load_trace_jsonl(write(tmp_path, [bad]))
    # arrivals out of order -> sorted ascending (stable on ties)
    b = REC2.replace('"a"', '"b"').replace("3.5", "1.0")
    c = REC2.replace('"a"', '"c"').replace("3.5", "1")
    progs, _, _ = OI.load_trace_jsonl(write(tmp_path, [REC2, b, c]))
    assert [p[0] for p in progs] == [1_000_000, 1_000_000, 3_500_000]


def test_oracle_decimal_times_are_exact():
    # R34: exact decimal value, rounded half away from zero to µs (no binary float in between)
    assert OI._us(json.loads("0.1", parse_float=__import__("decimal").Decimal)) == 100_000
    D = __import__("decimal").Decimal
    assert [OI._us(D(x)) for x in ("2.5e-6", "0.0000005", "0.00000049999", "1e3", "-0.0000005")] == \
        [3, 1, 0, 1_000_000_000, -1]
    assert OI._us(123) == 123_000_000


# ---- product vs oracle (host calls, no GPU) -------------------------------------------------------
@pytest.mark.parametrize("g", goldens(), ids=lambda g: g["cite"][:40])
def test_product_tool_name_goldens(ct, g):
    assert ct.ct_parse_tool_name(g["message"], g["format"]) == (g["name"], g["malformed"])


def _fuzz_message(rng: random.Random) -> str:
    words = ["ls", "cd", "pytest", "git", "python3", "grep", "-q", "x.py", "&&", "||", "|", ";",
             " ", "\n", "\t", "```bash\n", "```", "(", ")", "=", "'a'", '"b"', "[", "]", "{", "}",
             '"name"', '"type"', ":", ",", '"function_call"', '"tool_calls"', '"commands"',
             '"keystrokes"', "<tool_call>", "</tool_call>", "f", "_g1", "é", "\\u00e9", "null", "1.5"]
    kind = rng.randrange(6)
    if kind == 0:
        return "".join(rng.choice(words) for _ in range(rng.randrange(12)))
    name = rng.choice(["get_weather", "web_search", "fetch_url", "a.b", "_x", "ls"])
    if kind == 1:
        blk = {"type": rng.choice(["function_call", "function", "message", "tool_use", "reasoning"]),
               rng.choice(["name", "nam"]): name, "arguments": {"k": rng.randrange(9)}}
        if rng.random() < 0.3:
            blk = {"type": "function", "function": {"name": name}}
        v = [blk] if rng.random() < 0.5 else blk
        if rng.random() < 0.2:
            v = {"role": "assistant", "tool_calls": [blk]}
        s = json.dumps(v)
    elif kind == 2:
        s = json.dumps({"name": name, "arguments": {}})
        if rng.random() < 0.3:
            s = "<tool_call>%s</tool_call>" % s
    elif kind == 3:
        s = "%s(%s)" % (name, ", ".join("p%d=%d" % (i, i) for i in range(rng.randrange(3))))
        if rng.random() < 0.3:
            s = "[%s]" % s
    elif kind == 4:
        cmds = [" ".join(rng.choice(words[:8]) for _ in range(rng.randrange(1, 4)))
                for _ in range(rng.randrange(1, 4))]
        s = rng.choice([" && ", " || ", "&&"]).join(cmds)
        if rng.random() < 0.5:
            s = "Running:\n```bash\n%s\n```\nthen" % s
    else:
        s = json.dumps({"commands": [{"keystrokes": rng.choice(["vim a.py\n", "  pytest -q\n", ""])}
                                     for _ in range(rng.randrange(3))]})
    if rng.random() < 0.15:  # truncation -> malformed structured blocks
        s = s[: rng.randrange(len(s) + 1)]
    if rng.random() < 0.1:
        s = "  \n" + s + " \t"
    return s


def test_product_tool_name_matches_oracle_on_fuzz(ct):
    rng = random.Random(20251102)
    n_names = n_bad = 0
    for i in range(6000):
        m = _fuzz_message(rng)
        for fmt in OI.FORMATS:
            want = OI.parse_tool_name(m, fmt)
            got = ct.ct_parse_tool_name(m, fmt)
            assert got == want, (m, fmt, got, want)
            n_names += want[0] is not None
            n_bad += want[1]
    assert n_names > 5000 and n_bad > 500  # the fuzz reaches every outcome


def _as_records(tr):
    out = []
    for i in range(len(tr.programs)):
        t0, nt = int(tr.programs["turn0"][i]), int(tr.programs["nturns"][i])
        out.append((int(tr.programs["arr_q"][i]), [tuple(int(x) for x in r) for r in tr.turns[t0:t0 + nt]]))
    return out


@pytest.mark.parametrize("messages", [False, True])
def test_round_trip_of_a_generated_trace(ct, tmp_path, messages):
    tr = traces.generate(2, 40, n_bfcl=12)
    known = [t[0] for t in traces.TOOLS]
    for seed in (0, 1):
        path = str(tmp_path / ("s%d.jsonl" % seed))
        traces.to_jsonl(tr, path, seed=seed, messages=messages)
        got, names, warn = ct.ct_load_trace_jsonl(path, known_tools=known)
        want = traces.TraceSet(tr.programs[seed * 40:(seed + 1) * 40].copy(), tr.turns, 1, 40,
                               tr.n_tools, tr.pclass)
        assert _as_records(got) == _as_records(want) and names == known and warn == 0
        o, onames, ow = OI.load_trace_jsonl(path, known_tools=known)
        assert o == _as_records(got) and onames == names and ow == warn


def test_load_matches_oracle_on_mutated_records(ct, tmp_path):
    """Valid and invalid files: same records, tool table and warnings, or an error on the
    same line."""
    rng = random.Random(7)
    base = [REC2.replace('"a"', '"p%d"' % i).replace("3.5", "%d.%03d" % (rng.randrange(9), rng.randrange(1000)))
            for i in range(6)]
    muts = [
        lambda s: s,
        lambda s: s.replace('"tool_name": "pytest"', '"message": "```bash\\ngrep -r x\\n```"'),
        lambda s: s.replace('"tool_name": "pytest"', '"message": "no call here"'),
        lambda s: s.replace('"tool_name": "pytest"', '"message": "{\\"type\\": \\"function_call\\""'),
        lambda s: s.replace("8.25", "0"),
        lambda s: s.replace("8.25", "2.5e-6"),
        lambda s: s.replace("8.25", "-1"),
        lambda s: s.replace('"decode_tokens": 5', '"decode_tokens": 0'),
        lambda s: s.replace('"decode_tokens": 5', '"decode_tokens": 5.0'),
        lambda s: s.replace('"decode_tokens": 5', '"decode_tokens": true'),
        lambda s: s.replace('"decode_tokens": 5}', '"decode_tokens": 5, "tool_name": "x"}'),
        lambda s: s.replace('"turns": [', '"turns": [], "x": ['),
        lambda s: s.replace('"program_id": "p', '"program_id": "q'),
        lambda s: s.replace('"program_id": "p1"', '"program_id": "p0"'),
        lambda s: s.replace("}]}", "}]"),
        lambda s: s.replace('"arrival_time_s": ', '"arrival_time_s": -'),
        lambda s: s.replace('"new_prompt_tokens": 100', '"new_prompt_tokens": 900000'),
        lambda s: s.replace('"tool_name": "pytest"', '"tool_name": ""'),
        lambda s: s.replace('"pytest"', '"t%d"' % rng.randrange(80)),
        lambda s: "   " if rng.random() < 0.5 else s,
    ]
    n_err = n_ok = 0
    for trial in range(300):
        lines = [rng.choice(muts)(l) if rng.random() < 0.4 else l for l in base]
        path = write(tmp_path, lines, "m%d.jsonl" % trial)
        window = rng.choice([0, 0, 200])
        try:
            want = OI.load_trace_jsonl(path, ctx_window=window)
        except OI.TraceError as e:
            with pytest.raises(Exception) as ei:
                ct.ct_load_trace_jsonl(path, ctx_window=window)
            assert ("line %d:" % e.args[0]) in str(ei.value), (str(ei.value), e.args)
            n_err += 1
            continue
        got, names, warn = ct.ct_load_trace_jsonl(path, ctx_window=window)
        assert _as_records(got) == want[0] and names == want[1] and warn == want[2]
        n_ok += 1
    assert n_err > 50 and n_ok > 50


def test_load_errors_and_tool_table(ct, tmp_path):
    with pytest.raises(Exception, match="cannot open"):
        ct.ct_load_trace_jsonl(str(tmp_path / "missing.jsonl"))
    # known tools keep their ids; new names are appended in first use
    tr, names, _ = ct.ct_load_trace_jsonl(write(tmp_path, [REC2]), known_tools=["cat", "grep"])
    assert names == ["cat", "grep", "pytest"] and int(tr.turns[0, 2]) == 2
    # more than 64 distinct tools
    many = ['{"program_id": %d, "arrival_time_s": 0, "turns": [{"new_prompt_tokens": 1, '
            '"decode_tokens": 1, "tool_name": "t%d", "tool_duration_s": 1}, '
            '{"new_prompt_tokens": 1, "decode_tokens": 1}]}' % (i, i) for i in range(65)]
    with pytest.raises(Exception, match="CT_MAX_TOOLS"):
        ct.ct_load_trace_jsonl(write(tmp_path, many))


def test_load_enforces_the_replay_bounds(ct, tmp_path):
    """Arrivals replay as recorded at gap_us = 2^20 (R34), so the replay's arr_q * gap < 2^62
    means arrivals below 2^42 µs; a program's total context is at most 2^30 tokens
    (CT_MAX_CONTEXT).  The product and the oracle accept and reject the same files."""
    def rec(arr_us, new=10):
        return ('{"program_id": 1, "arrival_time_s": %d.%06d, "turns": [{"new_prompt_tokens": %d, '
                '"decode_tokens": 1}]}' % (arr_us // 10**6, arr_us % 10**6, new))
    ok = write(tmp_path, [rec(2**42 - 1)])
    tr, _, _ = ct.ct_load_trace_jsonl(ok)
    assert int(tr.programs["arr_q"][0]) == 2**42 - 1
    assert OI.load_trace_jsonl(ok)[0][0][0] == 2**42 - 1
    for bad in ([rec(2**42)], [rec(0, new=2**30)]):
        path = write(tmp_path, bad)
        with pytest.raises(Exception):
            ct.ct_load_trace_jsonl(path)
        with pytest.raises(OI.TraceError):
            OI.load_trace_jsonl(path)


@pytest.mark.gpu
def test_replay_of_a_loaded_trace_matches_oracle(ct, tmp_path):
    """A JSONL trace loaded by the product replays on the GPU exactly as the oracle replays the
    generator's own records (arrivals at gap_us = 2^20 are the recorded ones)."""
    import torch
    from ctgen import configs as cf
    from oracle import oracle as O
    tr = traces.generate(1, 24, n_bfcl=8)
    path = str(tmp_path / "r.jsonl")
    traces.to_jsonl(tr, path, messages=True)
    got, names, _ = ct.ct_load_trace_jsonl(path, known_tools=[t[0] for t in traces.TOOLS])
    got = traces.TraceSet(got.programs, got.turns, 1, 24, tr.n_tools, tr.pclass)
    w = cf.config1()
    sw = cf.Sweep(1, [1 << 20, 1 << 19], [4096, 1024], list(w.sweep.policies))
    ctx = ct.Context(0)
    s, j = ct.ct_simulate_batch(ctx, ct.DeviceTrace(got), sw, w.engine, jct=True)
    torch.cuda.synchronize()
    os_, oj = O.simulate(tr, sw, w.engine)
    assert np.array_equal(s.cpu().numpy(), os_) and np.array_equal(j.cpu().numpy(), oj)

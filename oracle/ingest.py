"""Oracle for the host-side trace ingest (NEXT-4) — TEST INFRASTRUCTURE ONLY.

Plain Python, written from the paper's text and the readings R33-R35 of DESIGN.md, sharing
nothing with paper_2511_02230_b200/csrc/ingest.cpp (it uses the standard `json` and
`decimal` modules where the product has its own reader).

* parse_tool_name  — §5.2 "the handler simply checks each returned message block's type; if it
  indicates a function/tool call, the handler extracts the call's name"; App. A
  (PAPER.md:1086-1094): Llama-3 `func_name(param=...)`, Qwen-3 `{"name": ..., "arguments": ...}`,
  SWE-Bench "locate the single bash code block, split the command string on && or ||, ... the
  first token is the executable/function name" (also PAPER.md:619 "use the first word"),
  Terminal-Bench `commands[].keystrokes`.
* load_trace_jsonl — SPEC.md:144-178 (TurnSpec / ProgramSpec invariants, load_trace), with
  exact decimal times rounded half away from zero to µs (R34) and unparsable messages mapped
  to the tool "unknown" with a warning (R35).

Pinned in tests/test_ingest.py by the paper's own listings,
SPEC.md:166-168 and 176-178 examples, and round trips of generated traces.
"""
from __future__ import annotations

import decimal
import json

CALL_TYPES = ("function_call", "function", "tool_call", "tool_use")
FORMATS = ("auto", "openai", "name", "pythonic", "bash", "terminal")
SPACE = " \t\n\r\v\f"


def bash_name(msg: str) -> str | None:
    """App. A: the bash block (```bash fence if present, else the text), split on && / ||,
    the first whitespace token of the first sub-command."""
    cmd = msg
    f = msg.find("```bash")
    if f >= 0:
        nl = msg.find("\n", f)
        start = len(msg) if nl < 0 else nl + 1
        end = msg.find("```", start)
        cmd = msg[start:] if end < 0 else msg[start:end]
    cut = len(cmd)
    for sep in ("&&", "||"):
        i = cmd.find(sep)
        if i >= 0:
            cut = min(cut, i)
    first = cmd[:cut]
    # whitespace tokens (same six ASCII space characters as C isspace)
    tok = ""
    for ch in first:
        if ch in SPACE:
            if tok:
                break
            continue
        tok += ch
    return tok or None


def _blocks(v):
    if isinstance(v, list):
        return v
    if isinstance(v, dict):
        if isinstance(v.get("tool_calls"), list):
            return v["tool_calls"]
        if isinstance(v.get("output"), list):
            return v["output"]
    return [v]


def _call_name(blk):
    n = blk.get("name")
    if isinstance(n, str):
        return n
    fn = blk.get("function")
    if isinstance(fn, dict) and isinstance(fn.get("name"), str):
        return fn["name"]
    return None


def _json_rule(v, type_rule: bool, name_rule: bool):
    """-> (name or None, malformed)."""
    for blk in _blocks(v):
        if not isinstance(blk, dict):
            continue
        if type_rule and "type" in blk:
            t = blk["type"]
            if isinstance(t, str) and t in CALL_TYPES:
                n = _call_name(blk)
                if not n:
                    return None, True
                return n, False
            continue
        if name_rule and "type" not in blk:
            if "name" not in blk:
                continue
            n = blk["name"]
            if not isinstance(n, str) or not n:
                return None, True
            return n, False
    return None, False


def _terminal_rule(v):
    if not isinstance(v, dict) or "commands" not in v:
        return None, False
    c = v["commands"]
    if not isinstance(c, list):
        return None, True
    if not c:
        return None, False
    first = c[0]
    ks = first.get("keystrokes") if isinstance(first, dict) else None
    if not isinstance(ks, str):
        return None, True
    return bash_name(ks), False


def _pythonic_rule(msg: str):
    t = msg.strip(SPACE)
    if len(t) >= 2 and t[0] == "[" and t[-1] == "]":
        t = t[1:-1].strip(SPACE)
    if not t or not (t[0].isascii() and (t[0].isalpha() or t[0] == "_")) or t[-1] != ")":
        return None, False
    i = 1
    while i < len(t) and t[i].isascii() and (t[i].isalnum() or t[i] in "_."):
        i += 1
    j = i
    while j < len(t) and t[j] in SPACE:
        j += 1
    if j >= len(t) or t[j] != "(":
        return None, False
    return t[:i], False


def _loads(text: str):
    try:
        return json.loads(text, parse_constant=_reject), True
    except (ValueError, RecursionError):
        return None, False


def _reject(x):
    raise ValueError(x)


def parse_tool_name(msg: str, fmt: str = "auto"):
    """-> (tool name or None, malformed) per the format's rule (R33)."""
    t = msg.strip(SPACE)
    if fmt == "bash":
        return bash_name(msg), False
    if fmt == "pythonic":
        return _pythonic_rule(msg)
    if fmt in ("openai", "name", "terminal"):
        v, ok = _loads(t)
        if not ok:
            return None, True
        if fmt == "terminal":
            return _terminal_rule(v)
        return _json_rule(v, fmt == "openai", fmt == "name")
    # auto
    if t.startswith("<tool_call>"):
        inner = t[len("<tool_call>"):]
        c = inner.find("</tool_call>")
        if c >= 0:
            inner = inner[:c]
        t = inner.strip(SPACE)
    if t[:1] in ("{", "["):
        v, ok = _loads(t)
        if not ok:
            return None, True
        if isinstance(v, dict) and "commands" in v:
            return _terminal_rule(v)
        return _json_rule(v, True, True)
    if "```bash" in msg:
        return bash_name(msg), False
    return _pythonic_rule(msg)


class TraceError(ValueError):
    pass


def _us(x) -> int:
    """Exact decimal seconds -> µs, half away from zero (R34)."""
    with decimal.localcontext() as c:
        c.prec = 200
        return int((decimal.Decimal(x) * 1000000).quantize(decimal.Decimal(1),
                                                           rounding=decimal.ROUND_HALF_UP))


def _is_num(x) -> bool:
    return isinstance(x, (int, decimal.Decimal)) and not isinstance(x, bool)


def _is_int(x) -> bool:
    return isinstance(x, int) and not isinstance(x, bool)


def load_trace_jsonl(path: str, fmt: str = "auto", ctx_window: int = 0, known_tools=()):
    """SPEC.md:170-178 load_trace: -> (programs [(arrival_us, [(new, dec, tool_id, dur_us)])]
    sorted by arrival (stable), tool names by id, warnings).  Raises TraceError(line, msg)."""
    progs, ids, warnings = [], set(), 0
    with open(path, "rb") as fh:
        lines = fh.read().decode("utf-8", "surrogateescape").split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    for ln, line in enumerate(lines, 1):
        if line.endswith("\r"):
            line = line[:-1]
        if not line.strip(SPACE):
            continue
        try:
            rec = json.loads(line, parse_float=decimal.Decimal, parse_constant=_reject)
        except ValueError:
            raise TraceError(ln, "invalid JSON")
        if not isinstance(rec, dict):
            raise TraceError(ln, "record is not an object")
        pid = rec.get("program_id")
        if not (isinstance(pid, str) or _is_num(pid)):
            raise TraceError(ln, "program_id")
        key = pid if isinstance(pid, str) else str(pid)
        if key in ids:
            raise TraceError(ln, "program_id duplicate")
        ids.add(key)
        at = rec.get("arrival_time_s")
        # arrivals replay as recorded at gap 2^20 (R34): the replay needs arr_q * gap < 2^62
        if not _is_num(at) or _us(at) < 0 or _us(at) >= 2**42:
            raise TraceError(ln, "arrival_time_s")
        turns = rec.get("turns")
        if not isinstance(turns, list) or not turns:
            raise TraceError(ln, "turns")
        if len(turns) > 65536:  # CT_MAX_TURNS
            raise TraceError(ln, "turns")
        out, cum = [], 0
        for k, tv in enumerate(turns):
            if not isinstance(tv, dict):
                raise TraceError(ln, "turn not an object")
            last = k == len(turns) - 1
            nw, dec = tv.get("new_prompt_tokens"), tv.get("decode_tokens")
            if not _is_int(nw) or not 0 <= nw < 2**31:
                raise TraceError(ln, "new_prompt_tokens")
            if not _is_int(dec) or not 1 <= dec < 2**31:
                raise TraceError(ln, "decode_tokens")
            cum += nw + dec
            if cum > 2**30:  # CT_MAX_CONTEXT
                raise TraceError(ln, "context above 2^30 tokens")
            if ctx_window > 0 and cum > ctx_window:
                raise TraceError(ln, "context window")
            if last:
                if "tool_name" in tv or "tool_duration_s" in tv:
                    raise TraceError(ln, "tool on final turn")
                out.append([nw, dec, None, 0])
                continue
            if "tool_duration_s" not in tv:
                raise TraceError(ln, "tool_duration_s missing")
            d = tv["tool_duration_s"]
            if not _is_num(d) or _us(d) < 0 or _us(d) >= 2**62:
                raise TraceError(ln, "tool_duration_s")
            dur = max(_us(d), 1)  # R25
            if dur >= 2**31:
                raise TraceError(ln, "tool_duration_s above 2^31 µs")
            if "tool_name" in tv:
                name = tv["tool_name"]
                if not isinstance(name, str) or not 1 <= len(name.encode("utf-8", "surrogateescape")) <= 63:
                    raise TraceError(ln, "tool_name")
            elif "message" in tv:
                m = tv["message"]
                if not isinstance(m, str):
                    raise TraceError(ln, "message")
                name, bad = parse_tool_name(m, fmt)
                if name is None or len(name.encode("utf-8", "surrogateescape")) > 63:
                    warnings += 1  # R35
                    name = "unknown"
            else:
                raise TraceError(ln, "tool_name missing")
            out.append([nw, dec, name, dur])
        progs.append((_us(at), ln, out))
    progs.sort(key=lambda p: p[0])  # Python's sort is stable
    names = list(known_tools)
    for _, ln, ts in progs:
        for t in ts:
            if t[2] is not None and t[2] not in names:
                if len(names) >= 64:
                    raise TraceError(ln, "more than 64 tools")
                names.append(t[2])
    result = []
    for arr, _, ts in progs:
        result.append((arr, [(nw, dec, -1 if nm is None else names.index(nm), dur)
                             for nw, dec, nm, dur in ts]))
    return result, names, warnings

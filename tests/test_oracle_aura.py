"""Pins of the row-f3 oracle (delta-encoded + LZ4 aura messages, P:6291-6356,
P:6911-6937; readings R46-R51) against what the LZ4 block format and the delta scheme
fix, not against the oracle's own code: hand-built streams from the format definition,
an independent pure-Python decoder, the format's end-of-block rules, the worst-case
expansion bound, XOR identities, placeholders, new agents and the reference-order
defragmentation."""
import struct

import numpy as np
import pytest

import oracle as orc


def py_lz4_decode(blk: bytes) -> bytes:
    """Textbook LZ4 block decoder, written from the format definition."""
    out = bytearray()
    i = 0
    while i < len(blk):
        t = blk[i]
        i += 1
        n = t >> 4
        if n == 15:
            while True:
                b = blk[i]
                i += 1
                n += b
                if b != 255:
                    break
        out += blk[i:i + n]
        i += n
        if i == len(blk):
            break
        off = blk[i] | (blk[i + 1] << 8)
        i += 2
        m = (t & 15) + 4
        if (t & 15) == 15:
            while True:
                b = blk[i]
                i += 1
                m += b
                if b != 255:
                    break
        assert 0 < off <= len(out)
        for _ in range(m):
            out.append(out[-off])
    return bytes(out)


def sequences(blk: bytes):
    """(literal start, literal length, match length, offset) of each sequence."""
    seqs, i, pos = [], 0, 0
    while i < len(blk):
        t = blk[i]
        i += 1
        n = t >> 4
        if n == 15:
            while True:
                b = blk[i]; i += 1; n += b
                if b != 255:
                    break
        i += n
        if i == len(blk):
            seqs.append((pos, n, 0, 0))
            break
        off = blk[i] | (blk[i + 1] << 8)
        i += 2
        m = (t & 15) + 4
        if (t & 15) == 15:
            while True:
                b = blk[i]; i += 1; m += b
                if b != 255:
                    break
        seqs.append((pos, n, m, off))
        pos += n + m
    return seqs


@pytest.mark.parametrize("stream,want", [
    (bytes([0x50]) + b"hello", b"hello"),                                   # literals only
    (bytes([0x14]) + b"x" + bytes([1, 0, 0x50]) + b"abcde", b"x" * 9 + b"abcde"),  # overlap, off 1
    (bytes([0x22]) + b"ab" + bytes([2, 0, 0x00]), b"ab" * 4),              # off 2, len 6
    (bytes([0xF0, 255, 30]) + bytes(range(256)) + bytes(44), bytes(range(256)) + bytes(44)),
    (bytes([0x1F]) + b"z" + bytes([1, 0, 255, 2, 0x00]), b"z" * (1 + 4 + 15 + 255 + 2)),
    (bytes([0x00]), b""),
])
def test_decoder_on_hand_built_streams(stream, want):
    assert py_lz4_decode(stream) == want
    assert orc.lz4_decompress_block(stream, len(want)) == want


@pytest.mark.parametrize("bad", [
    bytes([0x14]) + b"x" + bytes([0, 0]),        # offset 0
    bytes([0x14]) + b"x" + bytes([2, 0]),        # offset beyond the output
    bytes([0x50]) + b"hel",                      # truncated literals
])
def test_decoder_rejects_malformed(bad):
    with pytest.raises(ValueError):
        orc.lz4_decompress_block(bad, 64)


def _cases():
    rng = np.random.default_rng(7)
    yield b""
    yield b"a"
    yield b"abcdefghijkl"                       # 12 bytes: too short for a match
    yield b"a" * 13
    yield bytes(4096)
    yield rng.integers(0, 256, 4096, dtype=np.uint8).tobytes()
    yield rng.integers(0, 3, 4096, dtype=np.uint8).tobytes()
    yield (b"the quick brown fox " * 300)[:4096]
    yield rng.integers(0, 256, 65535, dtype=np.uint8).tobytes()


@pytest.mark.parametrize("data", list(_cases()), ids=lambda d: f"n{len(d)}")
def test_compressor_round_trip_and_format_rules(data):
    blk = orc.lz4_compress_block(data)
    assert py_lz4_decode(blk) == data
    n = len(data)
    assert len(blk) <= n + n // 255 + 16                 # worst-case expansion
    seqs = sequences(blk)
    assert seqs[-1][2] == 0                             # last sequence: literals only
    for pos, nlit, m, off in seqs[:-1]:
        start = pos + nlit
        assert m >= 4 and 1 <= off <= start
        assert start < n - 12                           # a match starts >= 12 bytes before the end
        assert start + m <= n - 5                       # the last 5 bytes are literals
    if n >= 4096 and len(set(data)) == 1:
        assert len(blk) <= n // 255 + 20                 # one long match


def _aura(n, seed, id0=0):
    rng = np.random.default_rng(seed)
    return {"x": rng.uniform(0, 100, n), "y": rng.uniform(0, 100, n), "z": rng.uniform(0, 12, n),
            "d": rng.uniform(8, 12, n), "id": (id0 + rng.permutation(3 * n)[:n]).astype(np.uint32),
            "flags": rng.integers(0, 64, n).astype(np.uint32)}


def _bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def test_identical_message_is_all_zero_deltas():
    ref = orc.aura_reference(_aura(500, 1))
    msg = {k: v[np.random.default_rng(2).permutation(500)] for k, v in ref.items()}
    pay, nnew = orc.aura_payload(msg, ref)
    assert nnew == 0
    nw = (500 + 31) // 32
    pres = np.frombuffer(pay[:4 * nw], np.uint32)
    assert np.all(pres[:-1] == 0xFFFFFFFF) and pres[-1] == (1 << (500 % 32)) - 1
    assert not any(pay[4 * nw:])                            # every XOR is zero
    back = orc.aura_decode(orc.aura_encode(msg, ref), ref)
    for k in orc.AURA_FIELDS:                               # reference order (R51)
        assert np.array_equal(back[k], ref[k]), k


def test_placeholders_new_agents_and_defragmentation():
    base = _aura(800, 3)
    ref = orc.aura_reference(base)
    rng = np.random.default_rng(4)
    keep = rng.random(800) < 0.7                            # 30 % left the aura
    new = _aura(150, 5, id0=10_000)                         # ids not in the reference
    msg = {k: np.concatenate([base[k][keep], new[k]]) for k in orc.AURA_FIELDS}
    msg["x"] = msg["x"] + 0.01                              # everybody moved
    o = rng.permutation(len(msg["x"]))
    msg = {k: v[o] for k, v in msg.items()}
    pay, nnew = orc.aura_payload(msg, ref)
    assert nnew == 150
    # presence bits: exactly the reference slots whose id is in the message
    nw = (800 + 31) // 32
    pres = np.unpackbits(np.frombuffer(pay[:4 * nw], np.uint8), bitorder="little")[:800]
    assert np.array_equal(pres.astype(bool), np.isin(ref["id"], msg["id"]))
    # x column, byte planes -> the XOR of the bit patterns for the matched slots
    ns = 800 + nnew
    planes = np.frombuffer(pay[4 * nw:4 * nw + 8 * ns], np.uint8).reshape(8, ns)
    xv = sum(planes[b].astype(np.uint64) << np.uint64(8 * b) for b in range(8))
    pos = {int(i): j for j, i in enumerate(msg["id"])}
    for s in range(800):
        if pres[s]:
            assert xv[s] == _bits(msg["x"][pos[int(ref["id"][s])]]) ^ _bits(ref["x"][s])
        else:
            assert xv[s] == 0
    newm = ~np.isin(msg["id"], ref["id"])
    assert np.array_equal(xv[800:], _bits(msg["x"][newm]))  # new agents raw, message order
    back = orc.aura_decode(orc.aura_encode(msg, ref), ref)
    kept = ref["id"][pres.astype(bool)]
    assert np.array_equal(back["id"], np.concatenate([kept, msg["id"][newm]]))
    for k in orc.AURA_FIELDS:
        want = np.concatenate([msg[k][[pos[int(i)] for i in kept]], msg[k][newm]])
        assert np.array_equal(np.asarray(back[k]).view(np.uint8), np.asarray(want).view(np.uint8)), k


def test_empty_reference_and_empty_message():
    msg = _aura(300, 6)
    empty = {k: v[:0] for k, v in msg.items()}
    back = orc.aura_decode(orc.aura_encode(msg, empty), empty)   # everything is new
    for k in orc.AURA_FIELDS:
        assert np.array_equal(back[k], msg[k])
    ref = orc.aura_reference(msg)
    back = orc.aura_decode(orc.aura_encode(empty, ref), ref)     # everybody left
    assert len(back["id"]) == 0


def test_stream_header_and_delta_gain():
    """Header fields as R50 states them; small moves compress far better with the
    delta (the paper's 1.1-3.5x on top of LZ4)."""
    base = _aura(20000, 8)
    base["z"] = np.round(base["z"], 3)
    ref = orc.aura_reference(base)
    msg = dict(ref)
    msg["x"] = ref["x"] + np.random.default_rng(9).uniform(-1e-3, 1e-3, 20000)
    st = orc.aura_encode(msg, ref)
    magic, chunk, nref, nnew, size, nch, _ = struct.unpack_from("<IIQQQII", st)
    assert (magic, chunk, nref, nnew) == (0x31414442, orc.LZ4_CHUNK, 20000, 0)
    assert nch == (size + orc.LZ4_CHUNK - 1) // orc.LZ4_CHUNK
    empty = {k: v[:0] for k, v in ref.items()}
    plain = orc.aura_encode(msg, empty)
    assert len(st) * 1.1 < len(plain) < 40 * 20000


# ---- pins against the LZ4 reference implementation (the system's liblz4) -------------
import lz4_ref  # noqa: E402

needs_liblz4 = pytest.mark.skipif(lz4_ref.lib() is None, reason="liblz4 not installed")


@needs_liblz4
@pytest.mark.parametrize("data", list(_cases()), ids=lambda d: f"n{len(d)}")
def test_liblz4_decodes_oracle_blocks(data):
    """Every block the oracle's compressor emits is a valid LZ4 block whose reference
    decoding (LZ4_decompress_safe) is exactly the input (R50: losslessness under the
    format's own decoder, independent of the parse convention)."""
    blk = orc.lz4_compress_block(data)
    assert lz4_ref.decompress_block(blk, len(data)) == data


def _stream_cases():
    base = _aura(3000, 11)
    ref = orc.aura_reference(base)
    moved = dict(ref)
    moved["x"] = ref["x"] + np.random.default_rng(12).uniform(-1e-2, 1e-2, 3000)
    rng = np.random.default_rng(13)
    keep = rng.random(3000) < 0.6
    new = _aura(700, 14, id0=50_000)
    churn = {k: np.concatenate([np.asarray(moved[k])[keep], new[k]]) for k in orc.AURA_FIELDS}
    empty = {k: v[:0] for k, v in ref.items()}
    yield "identical", ref, ref
    yield "moved", moved, ref
    yield "churn", churn, ref
    yield "no_reference", moved, empty
    yield "empty_message", empty, ref
    big = _aura(40000, 15)                                # > 1,000 chunks, ragged tail
    yield "multi_chunk", big, orc.aura_reference(_aura(39000, 15))


@needs_liblz4
@pytest.mark.parametrize("case", list(_stream_cases()), ids=lambda c: c[0])
def test_liblz4_decodes_oracle_aura_streams(case):
    """Each oracle aura stream, decoded block by block with liblz4, gives exactly the
    oracle's payload (presence words, XOR byte planes, new ids) and the header counts."""
    _, msg, ref = case
    st = orc.aura_encode(msg, ref)
    pay, nnew = orc.aura_payload(msg, ref)
    got, nref, nnew2 = lz4_ref.decode_stream(st)
    assert got == bytes(pay)
    assert (nref, nnew2) == (len(ref["id"]), nnew)

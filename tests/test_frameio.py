"""Raw RGB24 streams (reference frameio.py:215-291): header checks, round trips,
truncation offsets (CPU); the GPU streaming path against process_stream (gpu)."""
import io

import numpy as np
import pytest

from paper_2512_16609_b200.frameio import (RawStreamError, RawStreamTruncated, StreamHeader, read_raw_frames,
                                           write_raw_frame)


@pytest.mark.parametrize("kwargs", [dict(width=0, height=2), dict(width=2, height=-1), dict(width=1.5, height=2),
                                    dict(width=2, height=2, frame_count=-1)])
def test_header_rejects(kwargs):
    with pytest.raises(RawStreamError):
        StreamHeader(**kwargs)


def test_round_trip():
    rng = np.random.default_rng(0)
    frames = [rng.integers(0, 256, size=(4, 6, 3), dtype=np.uint8) for _ in range(5)]
    buf = io.BytesIO()
    for f in frames:
        write_raw_frame(buf, f)
    buf.seek(0)
    out = list(read_raw_frames(buf, StreamHeader(width=6, height=4)))
    assert len(out) == 5 and all(np.array_equal(a, b) for a, b in zip(out, frames))


def test_truncation_offsets():
    rng = np.random.default_rng(1)
    for _ in range(20):
        w, h = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        size = 3 * w * h
        whole = int(rng.integers(0, 4))
        partial = int(rng.integers(1, size)) if size > 1 else 1
        data = rng.integers(0, 256, size=whole * size + partial, dtype=np.uint8).tobytes()
        reader = read_raw_frames(io.BytesIO(data), StreamHeader(width=w, height=h))
        for _ in range(whole):
            next(reader)
        with pytest.raises(RawStreamTruncated, match=f"byte offset {whole * size}") as info:
            next(reader)
        assert info.value.offset == whole * size


def test_declared_count():
    assert len(list(read_raw_frames(io.BytesIO(bytes(36)), StreamHeader(width=2, height=2, frame_count=2)))) == 2
    with pytest.raises(RawStreamTruncated, match="after 2 frames"):
        list(read_raw_frames(io.BytesIO(bytes(24)), StreamHeader(width=2, height=2, frame_count=3)))


def test_write_validates():
    with pytest.raises(ValueError, match="uint8"):
        write_raw_frame(io.BytesIO(), np.zeros((2, 2, 3), np.float32))


@pytest.mark.gpu
@pytest.mark.parametrize("resize", [None, (96, 64)])
def test_dehaze_raw_stream_matches_process_stream(resize):
    from paper_2512_16609_b200 import DehazeParams, process_stream
    from paper_2512_16609_b200.frameio import dehaze_raw_stream
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c3", frames=23, width=160, height=96).numpy()
    raw = b"".join(f.tobytes() for f in frames)
    p = DehazeParams(resize_to=resize)
    header = StreamHeader(width=160, height=96)
    dst = io.BytesIO()
    stats = dehaze_raw_stream(io.BytesIO(raw), dst, header, p)
    ref = io.BytesIO()
    ref_stats = process_stream(list(frames), p, sink=lambda f: write_raw_frame(ref, f))
    assert stats.frame_count == ref_stats.frame_count == 23
    assert dst.getvalue() == ref.getvalue()
    assert all(np.array_equal(a, b) for a, b in zip(stats.airlight_trace, ref_stats.airlight_trace))


@pytest.mark.gpu
def test_dehaze_raw_stream_truncated_writes_previous_frames():
    from paper_2512_16609_b200 import DehazeParams
    from paper_2512_16609_b200.frameio import dehaze_raw_stream
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c3", frames=5, width=64, height=32).numpy()
    raw = b"".join(f.tobytes() for f in frames)[:-7]
    dst = io.BytesIO()
    with pytest.raises(RawStreamTruncated) as info:
        dehaze_raw_stream(io.BytesIO(raw), dst, StreamHeader(width=64, height=32), DehazeParams(resize_to=None))
    assert info.value.offset == 4 * 64 * 32 * 3
    assert len(dst.getvalue()) == 4 * 64 * 32 * 3


@pytest.mark.gpu
def test_process_stream_flushes_before_a_failing_source():
    from paper_2512_16609_b200 import DehazeParams, process_stream
    from paper_2512_16609_b200.synthetic import make_frames

    frames = make_frames("c3", frames=6, width=64, height=32).numpy()
    raw = b"".join(f.tobytes() for f in frames)[:-1]
    got = []
    with pytest.raises(RawStreamTruncated):
        process_stream(read_raw_frames(io.BytesIO(raw), StreamHeader(width=64, height=32)),
                       DehazeParams(resize_to=None), sink=got.append)
    assert len(got) == 5


def test_raw_reader_stream_with_only_read():
    """An io.RawIOBase subclass overriding only read() (its readinto raises
    NotImplementedError) in 5-byte dribbles: frames still reassemble
    (reference tests/test_frameio.py TestRawStream, chunked reads)."""
    import io

    from paper_2512_16609_b200.frameio import StreamHeader, read_raw_frames

    class Dribble(io.RawIOBase):
        def __init__(self, data):
            self._buf = io.BytesIO(data)

        def read(self, n):
            return self._buf.read(min(n, 5))

    frame = np.arange(36, dtype=np.uint8).reshape(3, 4, 3)
    out = list(read_raw_frames(Dribble(frame.tobytes()), StreamHeader(width=4, height=3)))
    assert len(out) == 1 and np.array_equal(out[0], frame)

"""The map's reader/writer guard (hashmap.py:91-122 of the reference): any
number of concurrent readers or one writer; a violation raises
ConcurrentAccessError and leaves the guard's state unchanged.  Pure host
logic (no GPU needed)."""
import threading

import pytest

from paper_2110_00511_b200.hashmap import ConcurrentAccessError, _AccessGuard


def test_readers_nest_and_exclude_writers():
    g = _AccessGuard()
    with g.reading():
        with g.reading():
            assert g._readers == 2
            with pytest.raises(ConcurrentAccessError):
                with g.writing():
                    pass
        assert g._readers == 1
    assert g._readers == 0 and not g._writing
    with g.writing():
        assert g._writing


def test_writer_excludes_everyone_and_state_survives_violations():
    g = _AccessGuard()
    with g.writing():
        with pytest.raises(ConcurrentAccessError):
            with g.reading():
                pass
        with pytest.raises(ConcurrentAccessError):
            with g.writing():
                pass
        assert g._writing and g._readers == 0
    assert not g._writing
    with g.reading():  # usable again
        pass


def test_exception_inside_releases_the_guard():
    g = _AccessGuard()
    with pytest.raises(RuntimeError):
        with g.writing():
            raise RuntimeError("boom")
    assert not g._writing
    with pytest.raises(RuntimeError):
        with g.reading():
            raise RuntimeError("boom")
    assert g._readers == 0


def test_threads_overlapping_a_writer_raise():
    g = _AccessGuard()
    entered, release = threading.Event(), threading.Event()
    errors = []

    def writer():
        with g.writing():
            entered.set()
            release.wait(5)

    t = threading.Thread(target=writer)
    t.start()
    entered.wait(5)
    try:
        with g.reading():
            pass
    except ConcurrentAccessError as e:
        errors.append(e)
    release.set()
    t.join()
    assert len(errors) == 1
    with g.reading():
        pass

"""The node daemon's protocol layer (csrc/host/node_daemon.cpp) on CPU: HCL1
frames as the reference host runtime sends them (proj/src/wire.cpp, net.cpp,
daemon.cpp). No GPU here, so the daemon serves zero devices; buffers, chunk
reassembly, the registry and every error path are still exercised."""
import random
import struct

import pytest

from paper_2005_08466_b200 import HaoclError
from paper_2005_08466_b200.node import NodeDaemon

from tests import hcl1_client as W


def start_daemon():
    for _ in range(20):
        port = random.randint(20000, 60000)
        try:
            return NodeDaemon(port)
        except HaoclError:
            continue
    raise RuntimeError("no free port pair")


@pytest.fixture
def node():
    d = start_daemon()
    yield d
    d.stop()


def test_handshake_and_device_list(node):
    for port in (node.port, node.port + 1):  # message and data connections both answer Ping
        c = W.Conn(port)
        assert c.request(W.PING, 77)[:2] == (W.PONG, 77)
        c.close()
    c = W.Conn(node.port)
    kind, cid, body = c.request(W.DEVREQ, 5)
    assert (kind, cid) == (W.DEVRESP, 5)
    n, = struct.unpack_from(">I", body, 0)
    assert len(body) == 4 + 13 * n
    c.close()


def test_chunked_transfer_reassembly_and_read(node):
    c, d = W.Conn(node.port), W.Conn(node.port + 1)
    c.call(1, "alloc_buffer", [(W.HANDLE, 42), (W.I64, 10)], [(42, 1)])
    payload = bytes(range(100, 130))
    # out of order, with an identical overlap; only the completing chunk is acknowledged
    for cid, (lo, hi) in enumerate([(20, 30), (0, 8), (5, 12)]):
        d.send(W.frame(W.DATA, 10 + cid, W.data_chunk(42, lo, 30, payload[lo:hi])))
    d.send(W.frame(W.DATA, 20, W.data_chunk(42, 12, 30, payload[12:20])))
    kind, cid, body = d.recv_frame()
    assert (kind, cid) == (W.ACK, 20) and struct.unpack(">QQ", body) == (42, 30)
    assert d.call(21, "read_buffer", [(W.HANDLE, 42)], [(42, 0)]) == [payload]
    # a re-sent buffer starts a new reassembly session
    d.send(W.frame(W.DATA, 22, W.data_chunk(42, 0, 30, bytes(30))))
    assert d.recv_frame()[:2] == (W.ACK, 22)
    assert d.call(23, "read_buffer", [(W.HANDLE, 42)]) == [bytes(30)]
    c.call(24, "release_object", [(W.HANDLE, 42)])
    with pytest.raises(W.RemoteError) as e:
        d.call(25, "read_buffer", [(W.HANDLE, 42)])
    assert e.value.code == 7  # precondition: not in store
    c.close(), d.close()


def test_reassembly_conflict_and_mid_transfer_read(node):
    d = W.Conn(node.port + 1)
    d.send(W.frame(W.DATA, 1, W.data_chunk(7, 0, 16, b"A" * 8)))
    with pytest.raises(W.RemoteError) as e:
        d.call(2, "read_buffer", [(W.HANDLE, 7)])
    assert e.value.code == 7  # mid-reassembly
    kind, cid, body = d.request(W.DATA, 3, W.data_chunk(7, 4, 16, b"B" * 8))
    assert (kind, cid) == (W.ERR, 3) and W.error_of(body)[0] == 8  # reassembly_conflict
    kind, cid, body = d.request(W.DATA, 4, W.data_chunk(7, 0, 32, b"A" * 8))
    assert kind == W.ERR and W.error_of(body)[0] == 8  # total_len changed mid-transfer
    kind, cid, body = d.request(W.DATA, 5, W.data_chunk(7, 12, 8, b"x" * 4))
    assert kind == W.ERR and W.error_of(body)[0] == 3  # chunk beyond total_len: malformed
    d.close()


def test_registry_matches_reference_core_bundle(node):
    c = W.Conn(node.port)
    r = c.call(1, "query_registry", [(W.STRING, "core")])
    entries = dict(zip(r[1::2], r[2::2]))
    assert r[0] == len(entries)
    # the reference registry, proj/src/kernels.cpp:13-33 (names in order, arities)
    want = [("matmul", 6), ("spmv_partition", 4), ("spmv_compute", 8), ("bfs", 5), ("knn", 8), ("vecadd", 4)]
    assert [(n, entries[n]) for n, _ in want] == want
    assert [n for n in r[1::2] if n in dict(want)] == [n for n, _ in want]
    with pytest.raises(W.RemoteError) as e:
        c.call(2, "query_registry", [(W.STRING, "nosuch")])
    assert e.value.code == 10
    c.close()


def test_error_replies(node):
    c = W.Conn(node.port)
    with pytest.raises(W.RemoteError) as e:
        c.call(1, "frobnicate", [])
    assert e.value.code == 5  # unknown_call
    c.call(2, "alloc_buffer", [(W.HANDLE, 1), (W.I64, 8)])
    launch = [(W.STRING, "vecadd"), (W.STRING, "default"), (W.I32, 1), (W.I32, 99), (W.I32, 1),
              (W.I64, 1), (W.I64, 1), (W.I64, 1), (W.I32, 4),
              (W.HANDLE, 1), (W.HANDLE, 1), (W.HANDLE, 1), (W.I64, 1)]
    with pytest.raises(W.RemoteError) as e:
        c.call(3, "launch_kernel", launch)
    assert e.value.code == 20  # unknown_device
    with pytest.raises(W.RemoteError) as e:
        c.call(4, "launch_kernel", launch[:8] + [(W.I32, 5)] + launch[9:])
    assert e.value.code == 3  # argument count mismatch: malformed
    with pytest.raises(W.RemoteError) as e:
        c.call(5, "alloc_buffer", [(W.HANDLE, 1), (W.I64, -1)])
    assert e.value.code == 9
    # bad magic and bad version: ErrorReply, and the connection keeps serving
    c.send(W.frame(W.PING, 6, magic=b"XCL1"))
    kind, cid, body = c.recv_frame()
    assert kind == W.ERR and W.error_of(body)[0] == 1
    c.send(W.frame(W.PING, 7, version=9))
    kind, cid, body = c.recv_frame()
    assert kind == W.ERR and W.error_of(body)[0] == 2
    assert c.request(W.PING, 8)[:2] == (W.PONG, 8)
    c.close()


def test_shutdown_message_stops_the_daemon():
    d = start_daemon()
    c = W.Conn(d.port)
    c.send(W.frame(W.SHUTDOWN, 1))
    d.wait()  # returns once the Shutdown is handled
    c.close()
    d.stop()


def test_network_sizes_are_capped(node, monkeypatch):
    """sizes from the wire (alloc_buffer, DataTransfer total_len)
    are checked against the node's buffer cap (one device's HBM, lowered by
    HCL_NODE_MAX_BUFFER) and answered with a size error (18) instead of an
    attempt to allocate them."""
    monkeypatch.setenv("HCL_NODE_MAX_BUFFER", "4096")
    c, d = W.Conn(node.port), W.Conn(node.port + 1)
    with pytest.raises(W.RemoteError) as e:
        c.call(1, "alloc_buffer", [(W.HANDLE, 7), (W.I64, 1 << 40)], [(7, 1)])
    assert e.value.code == 18
    c.call(2, "alloc_buffer", [(W.HANDLE, 8), (W.I64, 4096)], [(8, 1)])  # at the cap: accepted
    d.send(W.frame(W.DATA, 3, W.data_chunk(9, 0, 1 << 20, bytes(16))))
    kind, cid, body = d.recv_frame()
    assert cid == 3 and W.error_of(body)[0] == 18

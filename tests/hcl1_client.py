"""TEST INFRASTRUCTURE: a minimal HCL1 wire client (frame layout of
proj/include/haocl/wire.hpp:6-13, body encodings of proj/src/wire.cpp) used to
drive the node daemon from the tests. Big-endian throughout."""
import socket
import struct

PING, PONG, API, API_RESP, DEVREQ, DEVRESP, DATA, ACK, ERR, SHUTDOWN = 8, 9, 1, 2, 3, 4, 5, 6, 7, 10
I32, I64, F32, F64, BYTES, STRING, HANDLE = 1, 2, 3, 4, 5, 6, 7


def frame(kind, call_id, body=b"", version=1, magic=b"HCL1"):
    return magic + struct.pack(">BBQI", version, kind, call_id, len(body)) + body


def val(tag, v):
    if tag == I32:
        return struct.pack(">Bi", tag, v)
    if tag in (I64,):
        return struct.pack(">Bq", tag, v)
    if tag == HANDLE:
        return struct.pack(">BQ", tag, v)
    if tag == F64:
        return struct.pack(">Bd", tag, v)
    b = v.encode() if isinstance(v, str) else bytes(v)
    return struct.pack(">BI", tag, len(b)) + b


def api_body(fn, args, refs=()):
    b = struct.pack(">I", len(fn)) + fn.encode() + struct.pack(">I", len(args))
    b += b"".join(val(t, v) for t, v in args)
    b += struct.pack(">I", len(refs)) + b"".join(struct.pack(">QB", i, d) for i, d in refs)
    return b


def parse_values(body):
    n, = struct.unpack_from(">I", body, 0)
    at, out = 4, []
    for _ in range(n):
        tag = body[at]
        at += 1
        if tag == I32:
            out.append(struct.unpack_from(">i", body, at)[0]); at += 4
        elif tag == I64:
            out.append(struct.unpack_from(">q", body, at)[0]); at += 8
        elif tag == HANDLE:
            out.append(struct.unpack_from(">Q", body, at)[0]); at += 8
        elif tag == F64:
            out.append(struct.unpack_from(">d", body, at)[0]); at += 8
        elif tag == F32:
            out.append(struct.unpack_from(">f", body, at)[0]); at += 4
        else:
            ln, = struct.unpack_from(">I", body, at)
            at += 4
            raw = body[at:at + ln]
            at += ln
            out.append(raw.decode() if tag == STRING else raw)
    return out


class Conn:
    def __init__(self, port, host="127.0.0.1", timeout=30):
        self.s = socket.create_connection((host, port), timeout=timeout)
        self.buf = b""

    def send(self, data):
        self.s.sendall(data)

    def recv_frame(self):
        while len(self.buf) < 18 or len(self.buf) < 18 + struct.unpack_from(">I", self.buf, 14)[0]:
            chunk = self.s.recv(1 << 20)
            if not chunk:
                return None
            self.buf += chunk
        magic, (ver, kind, cid, ln) = self.buf[:4], struct.unpack_from(">BBQI", self.buf, 4)
        body = self.buf[18:18 + ln]
        self.buf = self.buf[18 + ln:]
        assert magic == b"HCL1" and ver == 1
        return kind, cid, body

    def request(self, kind, call_id, body=b""):
        self.send(frame(kind, call_id, body))
        return self.recv_frame()

    def call(self, call_id, fn, args, refs=()):
        kind, cid, body = self.request(API, call_id, api_body(fn, args, refs))
        assert cid == call_id
        if kind == ERR:
            code, ln = struct.unpack_from(">HI", body, 0)
            raise RemoteError(code, body[6:6 + ln].decode())
        assert kind == API_RESP
        return parse_values(body)

    def close(self):
        self.s.close()


class RemoteError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"{code}: {msg}")
        self.code = code


def data_chunk(buffer_id, offset, total, payload):
    return struct.pack(">QQQ", buffer_id, offset, total) + bytes(payload)


def error_of(body):
    code, ln = struct.unpack_from(">HI", body, 0)
    return code, body[6:6 + ln].decode()

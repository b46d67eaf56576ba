"""Node daemon: serve this process's B200s to remote HaoCL hosts.

The reference runs one daemon per node (``haocl node --config c.conf --name n0``,
proj/tools/haocl_main.cpp; NodeDaemon, proj/include/haocl/daemon.hpp:91-104) and
the host runtime reaches it over TCP with the HCL1 wire protocol. This module
starts the native daemon of ``csrc/host/node_daemon.cpp`` (C-ABI
``hcl_node_start``/``hcl_node_wait``/``hcl_node_stop``) over the logical devices
of ``hcl_init``, so an unmodified reference HostContext -- its cluster file
naming this node's ``ip:message_port`` -- launches the reference's core kernels
on the GPUs; buffers stay in HBM between calls.

    python -m paper_2005_08466_b200.node --port 7100 --devices 0,1,2,3
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
from typing import Optional, Sequence

from . import _native as N


class NodeDaemon:
    """One daemon on ``host:port`` (data port = port + 1, proj/include/haocl/config.hpp:9-10).

    cuda_ordinals: CUDA devices to serve as local devices 0..n-1 (repeats make
    several logical devices on one GPU); None serves whatever hcl_init already
    set up in this process (nothing on a machine without GPUs: the protocol
    still answers, launches fail with unknown_device)."""

    def __init__(self, port: int, host: str = "127.0.0.1", cuda_ordinals: Optional[Sequence[int]] = None):
        L = N.lib()
        if cuda_ordinals is not None:
            arr = (C.c_int * len(cuda_ordinals))(*cuda_ordinals)
            n = C.c_int()
            N.check(L.hcl_init(arr, len(cuda_ordinals), C.byref(n)))
        self._h = C.c_void_p()
        N.check(L.hcl_node_start(host.encode(), int(port), C.byref(self._h)))
        self.host, self.port = host, int(port)

    def wait(self) -> None:
        """Block until a Shutdown message arrives (or stop() from another thread)."""
        if self._h:
            N.check(N.lib().hcl_node_wait(self._h))

    def stop(self) -> None:
        if self._h:
            N.check(N.lib().hcl_node_stop(self._h))
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.stop()


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--host", default="127.0.0.1")
    ap.add_argument("--port", type=int, required=True, help="message port (data port = port + 1)")
    ap.add_argument("--devices", default="0", help="comma-separated CUDA ordinals served as local devices")
    a = ap.parse_args(argv)
    # load every kernel when the devices are set up, not inside the first
    # launch (whose node-reported compute time would include the module load)
    os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
    d = NodeDaemon(a.port, a.host, [int(x) for x in a.devices.split(",") if x != ""])
    print(f"haocl node: serving {a.devices} on {a.host}:{a.port}/{a.port + 1}", flush=True)
    try:
        d.wait()
    finally:
        d.stop()


if __name__ == "__main__":
    main()

"""numpy wrappers over the ref_/orc_ oracle libraries (test infrastructure only)."""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_1810_03988_b200 import abi
from paper_1810_03988_b200.api import AbiWrapper, _ptr

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "liblorbref.so")
ORC_SO = os.path.join(HERE, "_build", "liborc.so")


def build(quiet=True):
    """Compile the C restatement, and the reference oracle when /root/reference exists."""
    out = subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile"), "all"],
                         cwd=HERE, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def ref_available():
    return os.path.exists(REF_SO)


def orc_available():
    return os.path.exists(ORC_SO)




class Oracle(AbiWrapper):
    _libs = {}

    def __init__(self, kind="orc"):
        assert kind in ("ref", "orc")
        self.kind = kind
        self.prefix = kind + "_"
        if kind not in Oracle._libs:
            path = REF_SO if kind == "ref" else ORC_SO
            if not os.path.exists(path):
                if kind == "orc":
                    build()
                else:
                    raise FileNotFoundError(path)
            Oracle._libs[kind] = abi.bind(C.CDLL(path), self.prefix, with_ctx=False)
        self.lib = Oracle._libs[kind]

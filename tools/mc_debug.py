"""Experiment helper (GPU box): NVSwitch multicast support and object
creation through libcsr5g (csr5g_mcast_supported / csr5g_mailbox_mcast_*)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_05032_b200._lib import lib  # noqa: E402

L = lib()
L.csr5g_last_error.restype = C.c_char_p
v = C.c_int32()
print("supported:", L.csr5g_mcast_supported(0, C.byref(v)), v.value, L.csr5g_last_error())
for ndev in (1, 2):
    mb = C.c_void_p()
    L.csr5g_mailbox_create(0, 1, 0, 1 << 20, C.byref(mb))
    h = (C.c_uint8 * 64)()
    rc = L.csr5g_mailbox_mcast_create(mb, ndev, h)
    print(f"create ndev={ndev}:", rc, L.csr5g_last_error() if rc else "")
    if rc == 0:
        rc = L.csr5g_mailbox_mcast_add(mb)
        print("  add:", rc, L.csr5g_last_error() if rc else "")
        rc = L.csr5g_mailbox_mcast_bind(mb)
        print("  bind:", rc, L.csr5g_last_error() if rc else "")
    L.csr5g_mailbox_release(mb)

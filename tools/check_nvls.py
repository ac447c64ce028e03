"""Does this box support NVLink SHARP multicast (NVLS, cuMulticast*)?  Prints the
CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED attribute per device and the multicast
granularity for a 2-device group, via the CUDA driver API (ctypes)."""
import ctypes
import json

cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
n = ctypes.c_int()
cu.cuDeviceGetCount(ctypes.byref(n))
out = {"devices": n.value, "multicast_supported": [], "handle_types": None}
for d in range(n.value):
    dev = ctypes.c_int()
    cu.cuDeviceGet(ctypes.byref(dev), d)
    v = ctypes.c_int(-1)
    rc = cu.cuDeviceGetAttribute(ctypes.byref(v), 132, dev)  # CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED
    out["multicast_supported"].append((rc, v.value))
    if d == 0:
        h = ctypes.c_int(-1)
        rc2 = cu.cuDeviceGetAttribute(ctypes.byref(h), 104, dev)  # ..._HANDLE_TYPE_FABRIC_SUPPORTED? (probe)
        out["attr104"] = (rc2, h.value)
print(json.dumps(out))

"""Which NVLink counters does this box expose?  (NVML field values, GPM support.)"""
import pynvml as nv

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
try:
    sup = nv.c_nvmlGpmSupport_t()
    sup.version = 1
    fn = nv._nvmlGetFunctionPointer("nvmlGpmQueryDeviceSupport")
    rc = fn(h, nv.byref(sup))
    print("gpm support rc", rc, "isSupportedDevice", sup.isSupportedDevice)
except Exception as ex:
    print("gpm query failed", repr(ex))
try:
    print("gpm streaming", nv.nvmlGpmQueryIfStreamingEnabled(h))
except Exception as ex:
    print("gpm streaming query failed", repr(ex))
for fid in (138, 139, 140, 141, 66, 73):
    for scope in (0, 0xFFFFFFFF):
        try:
            v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print("field", fid, "scope", hex(scope), "rc", v.nvmlReturn, "val", v.value.ullVal)
        except Exception as ex:
            print("field", fid, repr(ex))

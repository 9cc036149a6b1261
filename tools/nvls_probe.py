"""Does this box support CUDA multicast objects (NVLink SHARP / multimem)?"""
from cuda.bindings import driver as d

d.cuInit(0)
err, n = d.cuDeviceGetCount()
for i in range(n):
    _, dev = d.cuDeviceGet(i)
    _, mc = d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    _, fab = d.cuDeviceGetAttribute(
        d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev)
    print(f"device {i}: multicast_supported={mc} fabric_handles={fab}")

// dlpack_min.h — the DLPack v0.8 ABI structs (dmlc/dlpack, Apache-2.0 ABI),
// restated so the C ABI can export zero-copy tensors without a dependency.
#pragma once
#include <stdint.h>

extern "C" {
typedef enum { kDLCPU = 1, kDLCUDA = 2 } DLDeviceType;
typedef struct {
    int32_t device_type;
    int32_t device_id;
} DLDevice;
typedef enum { kDLInt = 0U, kDLUInt = 1U, kDLFloat = 2U } DLDataTypeCode;
typedef struct {
    uint8_t code;
    uint8_t bits;
    uint16_t lanes;
} DLDataType;
typedef struct {
    void* data;
    DLDevice device;
    int32_t ndim;
    DLDataType dtype;
    int64_t* shape;
    int64_t* strides;
    uint64_t byte_offset;
} DLTensor;
typedef struct DLManagedTensor {
    DLTensor dl_tensor;
    void* manager_ctx;
    void (*deleter)(struct DLManagedTensor* self);
} DLManagedTensor;
}

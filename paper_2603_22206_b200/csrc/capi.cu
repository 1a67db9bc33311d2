// Library-level C-ABI entry points (version, status strings, device info).
#include "common.cuh"

extern "C" const char* chm_version(void) { return "chimera_b200 0.1.0 sm_100a"; }

extern "C" const char* chm_status_string(int32_t status) {
  switch (status) {
    case CHM_OK: return "ok";
    case CHM_ERR_INVALID_ARG: return "invalid argument";
    case CHM_ERR_VALIDATION: return "validation error";
    case CHM_ERR_NEGATIVE_PREDICTION: return "predicted_tokens must be >= 0";
    case CHM_ERR_DUPLICATE_REQUEST: return "duplicate request";
    case CHM_ERR_TIME_BACKWARDS: return "time going backwards";
    case CHM_ERR_NAN_PREDICTION: return "NaN predicted tokens";
    case CHM_ERR_INVALID_STATE: return "invalid device state";
    case CHM_ERR_CAPACITY: return "queue capacity exceeded";
    case CHM_ERR_UNSUPPORTED: return "unsupported option";
    case CHM_ERR_CUDA: return "CUDA error";
    case CHM_ERR_UNKNOWN_REQUEST: return "unknown request";
    case CHM_ERR_UNKNOWN_STAGE: return "unknown stage";
    case CHM_ERR_NCCL: return "NCCL unavailable or failed";
    default: return "unknown status";
  }
}

extern "C" chm_status chm_device_info(int32_t device, int32_t* sm_count, int32_t* cc_major,
                                      int32_t* cc_minor) {
  int v = 0;
  if (sm_count) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
      return CHM_ERR_CUDA;
    *sm_count = v;
  }
  if (cc_major) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess)
      return CHM_ERR_CUDA;
    *cc_major = v;
  }
  if (cc_minor) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, device) != cudaSuccess)
      return CHM_ERR_CUDA;
    *cc_minor = v;
  }
  return CHM_OK;
}

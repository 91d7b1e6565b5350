// K4 v2: binned DMMA gather (filled in below; v1 fallback until then).
#include "vfn_device.cuh"

namespace vfn {

int gather_boxes(vfn_plan* p, const double* pts_dev, int64_t M, const BinGeom& g,
                 const uint32_t* keys_sorted, const int32_t* perm, double2* out_dev,
                 cudaStream_t s, bool* used) {
  *used = false;
  return VFN_OK;
}

}  // namespace vfn

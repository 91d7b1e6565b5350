// Device side of the file-format writers (fields.py, cli.py): the density
// of an evaluated field and the VTK scalar layout, computed where the
// values already live so only the final bytes cross PCIe.
#include "vfn_internal.cuh"

namespace vfn {

// rho = re*re + im*im with both products rounded, as numpy's
// values.real**2 + values.imag**2 (cli.py:94, :113): no FMA contraction.
__global__ void k_density(const double2* __restrict__ v, int64_t n, double* __restrict__ rho) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 z = v[i];
    rho[i] = __dadd_rn(__dmul_rn(z.x, z.x), __dmul_rn(z.y, z.y));
  }
}

// VTK point order (first index fastest) big-endian float32 of a C-order
// (s0, s1, s2) double array: data.transpose(2, 1, 0).astype(">f4")
// (fields.py:139-141).  One thread per output word, coalesced stores.
__global__ void k_vtk_pack(const double* __restrict__ in, int64_t s0, int64_t s1, int64_t s2,
                           uint32_t* __restrict__ out) {
  const int64_t n = s0 * s1 * s2;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = o % s0, j = (o / s0) % s1, k = o / (s0 * s1);
    const float f = __double2float_rn(in[(i * s1 + j) * s2 + k]);
    out[o] = __byte_perm(__float_as_uint(f), 0, 0x0123);
  }
}

static int grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = (n + 255) / 256;
  return (int)std::min<int64_t>(blocks, (int64_t)sms * 8);
}

int launch_density(const double2* v, int64_t n, double* rho, cudaStream_t s) {
  if (n <= 0) return VFN_OK;
  k_density<<<grid_for(n), 256, 0, s>>>(v, n, rho);
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

int launch_vtk_pack(const double* in, const int64_t shape[3], uint32_t* out, cudaStream_t s) {
  const int64_t n = shape[0] * shape[1] * shape[2];
  if (n <= 0) return VFN_OK;
  k_vtk_pack<<<grid_for(n), 256, 0, s>>>(in, shape[0], shape[1], shape[2], out);
  VFN_CUDA(cudaGetLastError());
  return VFN_OK;
}

}  // namespace vfn

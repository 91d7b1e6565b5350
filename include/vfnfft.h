/*
 * vfnfft.h — C ABI of the B200-native 3D NFFT trafo (type-2 NUFFT).
 *
 * Drop-in boundary for the reference package `vortexfourier` (pure Python,
 * /root/reference/pkg/src/vortexfourier).  The reference has no FFI of its
 * own; these entry points are exactly what a ctypes / cffi binding of its
 * hot path would bind, one per reference operation:
 *
 *   vfn_plan_create   <- NufftPlan.__init__        nufft.py:197-242
 *                        (rescale_coeffs nufft.py:95-112, _kb_beta :152-156,
 *                         _kb_transform :167-176, _oversampled_size :179-187)
 *   vfn_plan_eval     <- NufftPlan.evaluate        nufft.py:244-272
 *                        (_check_points :115-126, map_to_torus :81-92)
 *   vfn_plan_destroy  <- (garbage collection of a NufftPlan)
 *   vfn_rect_eval     <- eval_rectilinear          rectilinear.py:47-64
 *                        (basis_matrix rectilinear.py:22-44)
 *   vfn_map_to_torus  <- map_to_torus              nufft.py:81-92
 *   vfn_plan_bin      <- (new) the cell-binning sort key and stable
 *                        permutation
 *   vfn_plan_grid     <- NufftPlan._grid           nufft.py:242 (inspection)
 *   vfn_direct_eval   <- eval_direct               nufft.py:129-149 (exact NDFT)
 *   vfn_decompose     <- snapshot_spectral         gpe.py:110-113 (mirror_extend gpe.py:90-101
 *                        + decompose fourier.py:183-188)
 *   vfn_synthesize    <- synthesize_regular        fourier.py:191-196
 *   vfn_tube_eval     <- tube_eval                 tube.py:58-127 (one reused plan)
 *
 * File formats feeding the path, native and multithreaded:
 *   vfn_snapshot_*    <- read_snapshot / write_snapshot   snapshots.py:29-72
 *   vfn_csv_read, vfn_table_*  <- read_points_csv         fields.py:160-174
 *   vfn_csv_write     <- write_points_csv                  fields.py:146-157
 *   vfn_field_write   <- write_field                       fields.py:67-95
 *   vfn_vtk_write     <- write_vtk_rectilinear             fields.py:119-143
 *   vfn_density       <- values.real**2 + values.imag**2   cli.py:94, :113
 *
 * Conventions
 *   - complex numbers are interleaved (re, im) doubles, numpy complex128;
 *   - points are (M, 3) row-major doubles; coefficients are (N1, N2, N3)
 *     C-order in the reference's centred order (index j <-> k = j - N/2);
 *   - `on_device` != 0 means the pointer is CUDA device memory on the plan's
 *     device, otherwise host memory (pinned host memory makes the copies
 *     asynchronous);
 *   - `stream` is a cudaStream_t (0 = legacy default stream);
 *   - every call returns a vfn_status; vfn_last_error() gives the message of
 *     the last failure on the calling thread.
 *   - Inputs are never modified; the plan owns its device grid; outputs are
 *     caller-owned.  Calls on one plan from several host threads are
 *     serialised by the plan (the reference allows evaluating a shared plan
 *     from several threads); distinct plans are independent.
 */
#ifndef VFNFFT_H
#define VFNFFT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  VFN_OK = 0,
  VFN_ERR_INVALID = -1,   /* bad argument (message says which) -> ValueError */
  VFN_ERR_OUTSIDE = -2,   /* a point lies outside [a, b); *first_bad_row set  */
  VFN_ERR_CUDA = -3,      /* CUDA runtime error                               */
  VFN_ERR_CUFFT = -4,     /* cuFFT error                                      */
  VFN_ERR_CUBLAS = -5,    /* cuBLAS error                                     */
  VFN_ERR_NOMEM = -6,     /* device allocation failed                         */
  VFN_ERR_IO = -7         /* file open / read / write failed -> OSError        */
} vfn_status;

typedef struct vfn_plan vfn_plan;

/* Library / kernel version string (for logs). */
const char* vfn_version(void);

/* Message of the last failing call on this thread ("" if none). */
const char* vfn_last_error(void);

/* Build the oversampled, deconvolved grid for one spectral field.
 *   nmodes  : N1, N2, N3 (each even, > 0)
 *   a, b    : box corners, a[d] < b[d]
 *   sigma   : oversampling; n_d = sigma * N_d must be an even integer >= N_d
 *   m       : window half-width in cells, 1..13 (each point reads (2m+1)^3)
 *   coeffs  : N1*N2*N3 complex128 (host or device, see on_device)         */
int vfn_plan_create(vfn_plan** out, int device, const int64_t nmodes[3],
                    const double a[3], const double b[3], double sigma, int m,
                    const double* coeffs, int coeffs_on_device, void* stream);

/* Evaluate the series at M points (nufft.py:244-272).
 *   points : M*3 doubles; out : M complex128 in input order.
 *   On VFN_ERR_OUTSIDE *first_bad_row holds the first offending row index
 *   (NaN coordinates count as outside), and `out` is unspecified.
 *   Any M >= 0 (device memory permitting): one sort + gather handles up to
 *   2^30 points, larger calls run as batches with one bin geometry; host
 *   buffers of >= 2^23 points are pipelined (H2D / evaluate / D2H overlap). */
int vfn_plan_eval(vfn_plan* plan, const double* points, int64_t M, double* out,
                  int on_device, int64_t* first_bad_row, void* stream);

int vfn_plan_destroy(vfn_plan* plan);

/* Plan facts: n[3] oversampled sizes, beta; either pointer may be NULL. */
int vfn_plan_info(const vfn_plan* plan, int64_t n_out[3], double* beta_out);

/* Copy the (n1, n2, n3) oversampled grid (nufft.py:242 `_grid`) to host. */
int vfn_plan_grid(vfn_plan* plan, double* out_host);

/* The bin-sort of M points (new): key[i] of input row i, and
 * perm = stable argsort(key) (sorted position -> input row).  key = (tile *
 * boxes_per_tile + box) * ceil(box_depth / 2^s) + ((depth in box) >> s),
 * tiles and boxes row-major (vfn_plan_geometry gives box and tile sizes,
 * vfn_plan_key_shift s).  Host or device buffers per on_device; keys are
 * uint32, perm int32.                                                     */
int vfn_plan_bin(vfn_plan* plan, const double* points, int64_t M, uint32_t* keys,
                 int32_t* perm, int on_device, int64_t* first_bad_row, void* stream);

/* zeta = mod((x - a)/(a - b), 1) - 1/2, bit-exact with numpy (nufft.py:81-92). */
int vfn_map_to_torus(int device, const double a[3], const double b[3], const double* points,
                     int64_t M, double* zeta, int on_device, void* stream);

/* Rectilinear tensor-grid evaluation (rectilinear.py:47-64): out is
 * (M1, M2, M3) complex128 C-order.  Coordinates must lie in [a_d, b_d)
 * (checked by the caller, rectilinear.py:28-41).                        */
int vfn_rect_eval(int device, const int64_t nmodes[3], const double a[3], const double b[3],
                  const double* coeffs, const double* y1, int64_t M1, const double* y2,
                  int64_t M2, const double* y3, int64_t M3, double* out, int on_device,
                  void* stream);

/* The same evaluation as three separable 1D type-2 NUFFT passes (SURVEY 8a
 * R3): per axis, deconvolve + zero-pad to n = sigma N, FFT, and a (2m+1)-tap
 * window gather at the axis' coordinates — the 3D trafo's algorithm in one
 * dimension, each pass one fused kernel with the line staged in shared
 * memory.  Accuracy ~10^-(2m+1) per pass (the plan's); needs sigma * N_d a
 * power of two <= 4096 (VFN_ERR_INVALID otherwise: use vfn_rect_eval).   */
int vfn_rect_eval_nufft(int device, const int64_t nmodes[3], const double a[3], const double b[3],
                        const double* coeffs, const double* y1, int64_t M1, const double* y2, int64_t M2,
                        const double* y3, int64_t M3, double sigma, int m, double* out, int on_device,
                        void* stream);

/* Exact series sum at M points, O(N1 N2 N3) per point (nufft.py:129-149).
 * Each N_d <= 1024.  Same point/domain conventions as vfn_plan_eval.   */
int vfn_direct_eval(int device, const int64_t nmodes[3], const double a[3], const double b[3],
                    const double* coeffs, const double* points, int64_t M, double* out,
                    int on_device, int64_t* first_bad_row, void* stream);

/* Gather geometry of the last vfn_plan_eval / vfn_plan_bin call (else the
 * point-independent rule for M points): the box and staging-tile sizes in
 * cells that define the bin key.                        */
int vfn_plan_geometry(const vfn_plan* plan, int64_t M, int box_out[3], int tile_out[3]);
/* Depth resolution of the same geometry's bin key: the key holds the cell's
 * depth in its box shifted right by *shift_out (1: depth pairs, 0: depths). */
int vfn_plan_key_shift(const vfn_plan* plan, int64_t M, int* shift_out);

/* Gather box width in cells (0 = automatic, 1 or 2).  Values are bitwise
 * reproducible for a fixed box width; the automatic choice depends on the
 * point set (its local density), so set it explicitly when bitwise
 * equality across different batches or GPU counts matters.            */
int vfn_plan_set_box(vfn_plan* plan, int bxy);

/* Kernel selection for vfn_plan_eval (benchmarks / A-B tests):
 * 0 = automatic, 1 = simple thread-per-point gather, 2 = DMMA box gather,
 * 3 = unbinned warp-per-point gather, 4 = binned with the automatic kernel
 * (never the warp path; what vfn_plan_decide returns above VFN_WARP_MAX_M).  Automatic uses 3 for evaluates of at
 * most VFN_WARP_MAX_M points (no binning: two launches) and the binned
 * tensor-core gather above.  Values of the two paths agree to rounding
 * (~1e-16 relative), not bitwise. */
#define VFN_WARP_MAX_M 32768
int vfn_plan_set_gather(vfn_plan* plan, int variant);
/* CUDA graphs for small evaluates (M <= 2^19, device part): on by default;
 * a repeated call with the same buffers, M and geometry replays one graph
 * instead of ~25 launches.  Values are identical either way. */
int vfn_plan_set_graphs(vfn_plan* plan, int enable);

/* Device time (ms) of the last vfn_plan_eval's gather kernel and of the
 * whole device-side evaluate, measured with CUDA events on its stream. */
int vfn_plan_last_timing(const vfn_plan* plan, float* gather_ms, float* total_ms);

/* snapshot -> centred coefficients on the computational box: samples
 * (N1,N2,N3) complex128 on [a, b); along mirrored axes the samples are
 * extended by their reflection and the box doubles; coeffs_out holds
 * (N_d * (1 + mirror_d)) complex128 values (gpe.py:90-113).              */
int vfn_decompose(int device, const double* values, const int64_t shape[3], const double a[3],
                  const double b[3], const int mirror[3], double* coeffs_out, int on_device,
                  void* stream);

/* Inverse of vfn_decompose without mirroring: the samples of a centred
 * coefficient array on its box's regular grid, ifftn(ifftshift(coeffs)) /
 * prod_d(sqrt(b_d - a_d) / N_d)   <- synthesize_regular (fourier.py:191-196).
 * coeffs / values_out: (N1, N2, N3) complex128, C-order; on_device as for
 * vfn_plan_eval. */
int vfn_synthesize(int device, const double* coeffs, const int64_t shape[3], const double a[3],
                   const double b[3], double* values_out, int on_device, void* stream);

/* Adaptive low-density point extraction (tube.py:58-127): seeds are the
 * samples with |v|^2 <= thresholds[0]; each later threshold selects the
 * parents of the next 3x-refined 27-point stencils, evaluated through one
 * plan (sigma, m).  Result (host-copied by vfn_tube_copy): count points
 * (count*3 doubles), densities, levels, sorted by lattice key.  *no_seeds
 * is set when no sample passes the first threshold (the reference warns).
 * `values` may be host or device memory (copied with cudaMemcpyDefault). */
typedef struct vfn_tube vfn_tube;
int vfn_tube_eval(vfn_tube** out, int device, const double* values, const int64_t shape[3],
                  const double a[3], const double b[3], const int mirror[3],
                  const double* thresholds, int nthr, int has_filter, double final_filter,
                  double sigma, int m, int64_t* count, int* no_seeds, void* stream);
int vfn_tube_copy(const vfn_tube* tube, double* points, double* density, int64_t* level);
int vfn_tube_destroy(vfn_tube* tube);

/* ------------------------------------------------------------ file formats
 * Byte-compatible with the reference writers/readers; format violations
 * return VFN_ERR_INVALID with the reference's message, OS failures
 * VFN_ERR_IO.  `on_device` buffers are staged through pinned host memory
 * with the file reads / writes overlapping the copies on `stream`. */

/* SFS1 header (snapshots.py:1-15): physical box, grid, mirror flags, time. */
typedef struct {
  double a[3], b[3];
  int64_t shape[3];
  int mirror[3];
  double time;
} vfn_snapshot_info;

/* Header only, validated against the file size (snapshots.py:50-71). */
int vfn_snapshot_info_read(const char* path, vfn_snapshot_info* info);
/* Header + payload into `values` (shape[0]*shape[1]*shape[2] complex,
 * `capacity` complex elements available). */
int vfn_snapshot_read(const char* path, vfn_snapshot_info* info, double* values, int64_t capacity,
                      int on_device, int device, void* stream);
int vfn_snapshot_write(const char* path, const vfn_snapshot_info* info, const double* values,
                       int on_device, int device, void* stream);

/* Points CSV (fields.py:146-174): header row of names, one row per point,
 * parsed as Python float() does.  The table owns the parsed columns. */
typedef struct vfn_table vfn_table;
int vfn_csv_read(const char* path, vfn_table** out, int64_t* rows, int* cols);
int vfn_table_name(const vfn_table* t, int col, const char** name);
int vfn_table_column(const vfn_table* t, int col, double* out);
/* Columns cols[0..2] interleaved as (rows, 3) points (host or device). */
int vfn_table_points(const vfn_table* t, const int cols[3], double* points, int on_device,
                     int device, void* stream);
int vfn_table_destroy(vfn_table* t);
/* x1,x2,x3 + ncols named columns, values as Python repr(); column c is
 * read at columns[c][i * strides[c]], float64 (kinds[c] = 0) or int64
 * (kinds[c] = 1).  Host buffers. */
int vfn_csv_write(const char* path, const double* points, int64_t M, int ncols,
                  const char* const* names, const void* const* columns, const int64_t* strides,
                  const int* kinds);

/* rho[i] = re_i*re_i + im_i*im_i, each product rounded (numpy, no FMA). */
int vfn_density(int device, const double* values, int64_t n, double* rho, int on_device,
                void* stream);

/* Rectilinear field = text header + raw psi + raw rho (fields.py:67-95). */
int vfn_field_write(const char* hdr_path, const char* psi_path, const char* rho_path,
                    const char* psi_name, const char* rho_name, const int64_t shape[3],
                    const double* const coords[3], const double* values, const double* density,
                    int has_time, double time, int on_device, int device, void* stream);
/* Legacy binary VTK rectilinear grid, scalars big-endian float32 with the
 * first index fastest (fields.py:119-143). */
int vfn_vtk_write(const char* path, const char* title, const int64_t shape[3],
                  const double* const coords[3], int nscalars, const char* const* names,
                  const double* const* scalars, int on_device, int device, void* stream);

/* ------------------------------------------------------------ multi-GPU
 * One point set sharded by key range over the ranks of a job (
 * "evaluation with a shared immutable plan is safe in parallel across
 * disjoint point subsets", reference SPEC.md:258-259).  The collectives
 * themselves run in the host layer (torch.distributed / NCCL,
 * paper_1605_01244_b200/parallel.py); these are the device steps.
 *
 * Partition key of a point = (tile << 32) | (row0 + row): the row-major index
 * of the gather tile holding its nearest oversampled cell, ties broken by
 * global input row.  vfn_plan_part_keys writes the keys of rows 0, stride,
 * 2 stride, ... (ceil(M / stride) keys, device memory) for the splitter
 * sample.  vfn_plan_partition sends row i to destination
 * d = #{splitters <= key_i} (nparts - 1 ascending device splitters),
 * writing the points destination-major and in input order within a
 * destination into `send` (device, M x 3), the send position of every row
 * into pos (device int32), and the per-destination counts into counts
 * (host, nparts).  Out-of-domain rows: VFN_ERR_OUTSIDE with the first
 * (local) row.  vfn_gather_values puts returned values back in input
 * order: out[i] = values[pos[i]] (device, complex128).                   */
int vfn_plan_part_keys(vfn_plan* plan, const double* points, int64_t M, int64_t stride, int64_t row0,
                       uint64_t* keys, void* stream);
int vfn_plan_partition(vfn_plan* plan, const double* points, int64_t M, int64_t row0,
                       const uint64_t* splitters, int nparts, double* send, int32_t* pos,
                       int64_t* counts, int64_t* first_bad_row, void* stream);
int vfn_gather_values(int device, const double* values, const int32_t* pos, int64_t M, double* out,
                      void* stream);
/* The same split with the all-to-all of the points fused in: the count
 * phase (counts per destination, host; the plan keeps the destinations),
 * then — once every rank knows its offset dst_off[d] inside destination
 * d's receive buffer (an all-gather of the counts) — the scatter phase
 * writes point i to recv_pts[d] + 3 (dst_off[d] + q) and its row i to
 * recv_rows[d][dst_off[d] + q], q its position among this rank's points
 * of destination d, in input order: the receiving ranks' IPC-mapped
 * buffers over NVLink.                                                   */
int vfn_plan_partition_count(vfn_plan* plan, const double* points, int64_t M, int64_t row0,
                             const uint64_t* splitters, int nparts, int64_t* counts, int64_t* first_bad_row,
                             void* stream);
int vfn_plan_partition_scatter_peers(vfn_plan* plan, const double* points, int64_t M, int nparts,
                                     const int64_t* dst_off, double* const* recv_pts, int32_t* const* recv_rows,
                                     void* stream);

/* Evaluate M received points (device) and store each value in the buffer
 * of the rank that owns the point, instead of a local output: point i
 * belongs to owner o with seg_off[o] <= i < seg_off[o + 1] (host array of
 * npeers + 1 offsets, npeers <= 64) and its value goes to
 * outs[o][rows[i]] (outs: host array of device pointers, IPC-mapped peer
 * buffers over NVLink; rows: device int32).  The tensor-core gather stores
 * straight from its epilogue (the return exchange fused into the gather);
 * other gathers are followed by a scatter kernel.  Same values as
 * vfn_plan_eval with the same settings.                                   */
int vfn_plan_eval_to_peers(vfn_plan* plan, const double* points, int64_t M, const int32_t* rows, int npeers,
                           const int64_t* seg_off, double* const* outs, int64_t* first_bad_row, void* stream);

/* IPC-shared device buffers for the owners' outputs: allocate + export a
 * 64-byte handle, open a peer's handle (another process; cudaIpc*), close,
 * free; and a synchronised device-to-device copy.                       */
int vfn_ipc_alloc(int device, int64_t bytes, void** ptr, unsigned char handle[64]);
int vfn_ipc_open(int device, const unsigned char handle[64], void** ptr);
int vfn_ipc_close(int device, void* ptr);
int vfn_ipc_free(int device, void* ptr);
int vfn_copy_device(int device, void* dst, const void* src, int64_t bytes, void* stream);

/* The gather decisions an evaluate of M points makes (gather variant 3 =
 * warp per point or 4 = binned; box width 1 or 2), so that every rank of a
 * sharded evaluate can pin the ones the unsharded call would take: values
 * are then bitwise independent of the rank count.  From 2^20 points the
 * box width depends on the points' local density: `sample` must hold the
 * 16384 rows j * (M / 16384), j = 0..16383, of the whole set (device).   */
int vfn_plan_decide(vfn_plan* plan, int64_t M, const double* sample, int nsample, int* variant_out,
                    int* box_out, void* stream);

/* Plan-build breakdown of the last vfn_plan_create (ms): [0] host wall time
 * of the whole call, [1] K2 deconvolve + pad, [2] K3 3D FFT, [3] halo
 * faces, [4] host setup before the grid kernels (allocations, window fit,
 * tables); [1..3] are CUDA-event times on the build stream.              */
int vfn_plan_build_timing(const vfn_plan* plan, float ms_out[5]);

/* Free the device buffers recycled from destroyed plans (device < 0: all
 * devices).  Destroyed plans return their grids to a per-device pool of at
 * most two buffers so a rebuilt plan skips cudaMalloc / cudaFree.        */
int vfn_pool_release(int device);

/* Utility (not a reference interface): measured sustained FP64 FMA rate of
 * `device` in TFLOP/s over ~`seconds`, the roofline denominator bench.py
 * reports against; *sm_clock_mhz gets the device's max SM clock.        */
int vfn_bench_fp64_peak(int device, double seconds, double* tflops, double* sm_clock_mhz);

#ifdef __cplusplus
}
#endif
#endif /* VFNFFT_H */

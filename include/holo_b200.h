/* holo_b200.h -- C ABI of the B200 RIHVR fused-lasso FISTA hot path.
 *
 * Plain C: integers, doubles, opaque handles and raw pointers.  No torch or
 * C++ types cross this boundary, and no C++ exception escapes it: every call
 * returns a status code (HOLO_OK == 0) and holo_last_error() describes the
 * most recent failure of the calling thread.
 *
 * The reference (holotrack, pure Python) has no native FFI of its own; these
 * entry points replace the Python functions cited beside each one, so a
 * ctypes/cffi binding slots in under the reference's public API
 * (see INTEGRATION.md).  Citations are /root/reference/pkg/src/holotrack/...
 *
 * Conventions
 *   - device pointers are CUDA device addresses on the handle's device;
 *     complex data is interleaved float32 (re, im) = complex64, planes are
 *     row-major (ny rows of nx samples), stacks plane-major.
 *   - `stream` is a cudaStream_t passed as void*; NULL is the legacy default
 *     stream (CUDA convention).  Host-buffer calls (holo_solve, *_host) run
 *     on the handle's private stream and synchronise before returning.
 *   - calls are stream-ordered; only calls returning host data synchronise.
 *   - one handle per thread at a time.
 */
#ifndef HOLO_B200_H
#define HOLO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HOLO_OK 0
#define HOLO_ERR_INVALID 1     /* bad argument: maps to ValueError                  */
#define HOLO_ERR_UNSUPPORTED 2 /* shape/config this build does not handle: ValueError */
#define HOLO_ERR_DIVERGED 3    /* objective > 1e6 f0: DivergenceError (report filled) */
#define HOLO_ERR_CUDA 4        /* CUDA runtime error: RuntimeError                    */
#define HOLO_ERR_NCCL 5        /* NCCL error: RuntimeError                            */

#define HOLO_POLICY_BACKTRACKING 0
#define HOLO_POLICY_FIXED 1

typedef struct holo_handle holo_handle;

/* optics.py:62-95 VolumeGeometry: plane k sits at z0 + k*dz. */
typedef struct {
  int32_t nx, ny, nz;
  double pitch, dz, z0, wavelength;
} holo_geometry;

/* solver.py:38-68 SolverConfig (+ prox.py:26-35 RegularizerWeights).
 * step_size <= 0 means "estimate" (solver.py:276-280). */
typedef struct {
  double lambda_l1, lambda_tv;
  int32_t max_iters, tv_inner_iters;
  int32_t step_policy;
  double step_size;
  double bt_shrink, stop_tol;
  int32_t log_objective;
  int32_t real_nonnegative; /* solver.py:154-216 _RealEngine: x real, x >= 0; needs step_size > 0 */
} holo_solver_config;

/* solver.py:71-85 SolveReport (+ counters the reference keeps internally). */
typedef struct {
  int32_t iterations, restarts, diverged, guard_fixups;
  int32_t attempts; /* prox-gradient attempts incl. backtracking and restarts */
  double step_size, final_sparsity, wall_time, f0;
  int64_t nnz;
  /* all-zero planes the forward passes skipped (solver.py:115-119), summed
   * over attempts and ranks (the guard fix-up's redone forward not counted) */
  int64_t skipped_planes;
} holo_report;

const char* holo_last_error(void);
int holo_version(void);
/* Checked build only (make checked -> libholo_b200_checked.so): *bits = the
 * bounds-check violations the kernels recorded since the last call (common.cuh
 * HoloCheckBit; read and cleared after a device sync).  Returns 1 in the
 * checked build, 0 (and *bits = 0) in the normal one.  No reference
 * counterpart: compute-sanitizer substitute for test infrastructure. */
int holo_debug_checks(uint32_t* bits);
/* 1 if this build handles the plane shape: sides 8..4096; powers of two run the
 * fused production passes, any other side the mixed-radix passes of gfft.cu */
int holo_shape_supported(int32_t nx, int32_t ny);

/* Handle lifecycle.  holo_create: whole volume on one GPU.
 * holo_create_sharded: planes [rank*nz/nranks, (rank+1)*nz/nranks) on this
 * GPU, the forward plane-sum exchanged by an NCCL allreduce over the
 * communicator built from `nccl_unique_id` (NCCL_UNIQUE_ID_BYTES = 128 bytes,
 * made by holo_nccl_unique_id on rank 0 and broadcast by the caller). */
int holo_create(const holo_geometry* geom, int device, holo_handle** out);
int holo_nccl_unique_id(void* out128);
int holo_create_sharded(const holo_geometry* geom, int device, const void* nccl_unique_id, int rank, int nranks,
                        holo_handle** out);
/* In-process rank group on one GPU (tests and diagnostics; no reference
 * counterpart): nranks (<= 8) handles out[0..nranks) own planes
 * [r*nz/nranks, (r+1)*nz/nranks) exactly like holo_create_sharded, but their
 * spectrum / scalar allreduce is an event-ordered device sum instead of NCCL.
 * Each handle must be driven from its own host thread (holo_solve* blocks in
 * the collective until every member arrives), each on its own stream.  Destroy
 * every handle with holo_destroy. */
int holo_create_local_group(const holo_geometry* geom, int device, int nranks, holo_handle** out);

/* Peer-memory reduction of the forward plane sum (replaces the NCCL spectrum
 * allreduce for a z-sharded handle; no reference counterpart -- the reference
 * sums planes in one process, solver.py:117-123).  Rank r owns slice
 * [r*L, (r+1)*L) of the P-element spectrum, L = holo_peer_slice(P, nranks);
 * one kernel sums the local plane groups and stores each slice into its
 * owner's inbox over NVLink, a second sums the owner's slice in rank order and
 * stores it into every rank's result (deterministic).  holo_peer_export writes
 * this rank's CUDA IPC handles (blob = NULL: *nbytes = blob size); the caller
 * all-gathers the blobs in rank order and passes them to holo_peer_import,
 * after which every solve uses the peer path.  The in-process rank group
 * (holo_create_local_group) uses it by default. */
int holo_peer_export(holo_handle* h, void* blob, int64_t* nbytes);
int holo_peer_import(holo_handle* h, const void* blobs, int64_t nbytes_each);
int64_t holo_peer_slice(int64_t plane_elems, int32_t nranks);
int holo_destroy(holo_handle* h);
int holo_local_planes(const holo_handle* h, int32_t* k_begin, int32_t* k_end);

/* Exact ||A||^2.  Complex engine: A A^H = nz * (band projector), so nz (the
 * value solver.py:225-247's power iteration converges to after one step).
 * Real engine (real != 0): max over the band of sum_k cos^2(phase_k). */
int holo_operator_norm(holo_handle* h, int32_t real, double* sigma2);
/* solver.py:225-247 estimate_operator_norm: `iters` power-iteration steps of
 * A^H A from the caller's start vector v0 (device, complex64, local planes,
 * unit norm; real != 0 uses Re(v0) and the real engine).  Returns the last
 * ||A^H A v||, exactly the reference's estimate for the same v0. */
int holo_power_iteration(holo_handle* h, const void* v0, int32_t iters, int32_t real, double* sigma2, void* stream);

/* solver.py:254-379 fista (complex engine).  b: ny*nx real hologram residual
 * (only Re(b) is used by the reference, solver.py:274).  _host reads a host
 * buffer (copies inside); _device reads a device buffer of doubles. */
int holo_solve(holo_handle* h, const double* b_host, const holo_solver_config* cfg, holo_report* rep);
int holo_solve_device(holo_handle* h, const double* b_dev, const holo_solver_config* cfg, holo_report* rep,
                      void* stream);
/* objective history of the last solve (solver.py:353); n = entries */
int holo_history(const holo_handle* h, double* out, int32_t cap, int32_t* n);

/* sparsevol.py:75-88 from_dense over the solution: nnz per local plane, then
 * COO entries sorted by (plane, row, col).  _host fills host arrays with
 * complex128 values (re, im doubles; the reference's SparsePlane.values
 * dtype), widened on the device; _device fills device buffers with
 * complex64 pairs. */
int holo_plane_nnz(holo_handle* h, int64_t* nnz_per_local_plane);
int holo_export_coo_host(holo_handle* h, int32_t* rows, int32_t* cols, double* vals, int64_t cap, int64_t* nnz);
int holo_export_coo_device(holo_handle* h, int32_t* rows, int32_t* cols, float* vals, int64_t cap, int64_t* nnz,
                           void* stream);
/* device pointer to the dense complex64 solution (local planes) */
int holo_solution_device(holo_handle* h, void** x);

/* ---- operator-level entry points (parity tests; device pointers) ---- */
/* optics.py:146-169 TransferLadder.stack(k0, k1, conj) as complex64 */
int holo_op_transfer(holo_handle* h, int32_t k0, int32_t k1, int32_t conj, void* out, void* stream);
/* numpy fft2 / ifft2 (1/P scaled) of nplanes complex64 planes, in place */
int holo_op_fft2(holo_handle* h, void* data, int32_t nplanes, int32_t inverse, void* stream);
/* solver.py:110-124 forward_sparse: out (float32, ny*nx) = Re ifft2(sum_k fft2(x_k) conj(H_k));
 * x = local planes (complex64).  Sharded handles allreduce the plane sum. */
int holo_op_forward(holo_handle* h, const void* x, void* out, void* stream);
/* optics.py:215-230 adjoint: out[k] = scale * ifft2(H_k fft2(r)), r float32 ny*nx,
 * out = local planes complex64 (scale 2 reproduces solver.py:126-132) */
int holo_op_adjoint(holo_handle* h, const void* r, void* out, double scale, void* stream);
/* prox.py:151-165 prox_fl over nplanes complex64 planes of any (ny, nx):
 * soft-threshold(tau_l1) of the FGP-TV prox (tau_tv, inner) of re and im,
 * including the per-plane guard (prox.py:138-147). */
int holo_op_prox_fl(holo_handle* h, const void* v, void* out, int32_t nplanes, int32_t ny, int32_t nx, double tau_l1,
                    double tau_tv, int32_t inner, void* stream);

/* ---- output side ---- */
/* segment.py:106-146 connected_components, 26-connectivity, on the GPU.
 * kij: n voxel coordinates (k, i, j) int32, sorted lexicographically (the COO
 * export order), device memory.  roots[u] (device) = smallest voxel id of
 * u's component, so components ordered by root are in the reference's
 * emission order (sorted by smallest voxel). */
int holo_label_components(const int32_t* kij, int64_t n, int32_t nz, int32_t ny, int32_t nx, int32_t* roots,
                          void* stream);

/* ---- input side ---- */
/* synth.py:161-181 render_hologram's spectrum: spec[f] = sum_p fft2(mask_p)(f) *
 * exp(-i 2 pi z_p/lam sqrt(1 - (lam f)^2)) (0 where evanescent), particles in
 * order.  Particle p owns mask pixels pix_yx[2e..2e+1] (row, col) with
 * amplitudes pix_a[e] for e in [pix_off[p], pix_off[p+1]).  All device
 * pointers; spec is complex128 (ny*nx).  fp64 throughout, like the reference. */
int holo_render_spectrum(const double* z_over_lam, const int32_t* pix_off, const int32_t* pix_yx, const double* pix_a,
                         int32_t n, int32_t ny, int32_t nx, double pitch, double wavelength, void* spec, void* stream);
/* preprocess.py:17-38: out[t] = (I_t - M_t) / sqrt(max(M_t, 1e-12)), M_t the mean of
 * frames [t-w/2, t+w/2] (truncated at the ends) excluding frame t; fp64 device
 * stacks (T, ny, nx); window odd, 3 <= window <= T. */
int holo_background(const double* images, int32_t T, int32_t ny, int32_t nx, int32_t window, double* out,
                    void* stream);

/* ---- instrumentation ---- */
/* per-kernel-class device time (CUDA events on the launching stream) */
int holo_profile_enable(holo_handle* h, int32_t on);
/* record only the classes whose bit is set in mask (bit k = k-th class of
 * holo_profile_read; default all): timing one class keeps the others' event
 * records out of a timed region */
int holo_profile_classes(holo_handle* h, uint32_t mask);
/* n = #classes; names: n x 32 bytes; ms: accumulated device ms; counts: launches */
int holo_profile_read(holo_handle* h, int32_t* n, char* names, double* ms, int64_t* counts);
/* kernels launched by this library since it was loaded (all handles) */
int64_t holo_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* HOLO_B200_H */

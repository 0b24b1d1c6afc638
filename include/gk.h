/*
 * gk.h -- C ABI of the B200-native gyrokinetic-proxy hot path (libgk.so).
 *
 * This is the drop-in boundary for the reference package's compute API
 * (gyroproxy 0.1.0, /root/reference/pkg/src/gyroproxy).  The reference has no
 * FFI of its own: its "plugin interface" is the module-level numpy function API
 * of gyroproxy.kernels / gyroproxy.spectral.  Each entry point below replaces the
 * numpy arithmetic underneath one of those functions; argument validation (the
 * reference's ValueError conditions) stays in the Python shim, which calls these
 * only with already-validated arguments (the C side re-checks sizes and returns
 * GK_ERR_ARG rather than trusting them).
 *
 * Conventions
 *  - complex arrays are interleaved (re, im) doubles, i.e. numpy/torch complex128
 *    storage; they are passed as `double*` of 2*count doubles.
 *  - the state is C-ordered [species][energy][xi][theta][toroidal][radial]
 *    (reference grid.py:1-11); n_vel = species*energy*xi (kernels.py:112-113),
 *    n_cells = toroidal*radial.
 *  - every pointer is a device pointer owned by the caller; `stream` is a
 *    cudaStream_t (NULL = legacy default stream).  Calls are stream-ordered and
 *    asynchronous; nothing allocates in the hot path.
 *  - return value: 0 (GK_OK) or a GK_ERR_* code; gk_last_error() describes it
 *    (thread-local).
 */
#ifndef GK_H_
#define GK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GK_ABI_VERSION 1

#define GK_STREAM_ORIGINAL 0  /* kernels.py:70-74 association order (bit-exact) */
#define GK_STREAM_OPTIMIZED 1 /* kernels.py:75-77, fused single pass            */

typedef struct gk_spectral_plan gk_spectral_plan;

int gk_version(void);
const char* gk_last_error(void);
int gk_device_info(int device, int* sm_count, int* cc_major, int* cc_minor, int64_t* l2_bytes);

/* Diagnostics (no reference counterpart): number of kernels this library has
 * launched in the process, and a measured fp64 throughput probe (DFMA and DMMA,
 * TFLOP/s) used as the roofline denominator of the fp64-bound kernels. */
int64_t gk_launch_counter(void);
int gk_probe_fp64_peak(double* dfma_tflops, double* dmma_tflops);

/* field_kernel (kernels.py:45-52):
 *   out[t,c] = sum_v weights[v] * h[v,t,c];  h: n_vel*n_theta*n_cells complex,
 *   weights: n_vel doubles, out: n_theta*n_cells complex.  Fixed summation order. */
int gk_field(const double* h, const double* weights, double* out,
             int64_t n_vel, int64_t n_theta, int64_t n_cells, void* stream);

/* stream_kernel (kernels.py:55-77):
 *   out[v,t,c] = sum_i stencil[i] * h[v,(t+i-w/2) mod n_theta,c]  (odd w <= n_theta).
 *   variant GK_STREAM_ORIGINAL reproduces the reference's roll-accumulate rounding
 *   exactly; GK_STREAM_OPTIMIZED is an FMA chain.  stencil: host or device array
 *   of `width` doubles (copied into kernel parameters). */
int gk_stream(const double* h, const double* stencil_host, int width, int variant, double* out,
              int64_t n_vel, int64_t n_theta, int64_t n_cells, void* stream);

/* stream_kernel for any odd width <= n_theta (kernels.py:65-68): the same two
 * variants with the stencil read from DEVICE memory (`width` doubles), for widths
 * beyond gk_stream's 31. */
int gk_stream_wide(const double* h, const double* stencil_dev, int width, int variant, double* out,
                   int64_t n_vel, int64_t n_theta, int64_t n_cells, void* stream);

/* shear_kernel (kernels.py:80-106):
 *   out[r,ky,kx] = h[r,ky,kx+shift[ky]] inside [0,n_kx), else 0; shifts: device
 *   int32[n_ky] with |shift| <= n_kx.  Pure data movement (bitwise). */
int gk_shear(const double* h, const int32_t* shifts, double* out,
             int64_t n_rows, int64_t n_ky, int64_t n_kx, void* stream);

/* collision_kernel (kernels.py:109-123):
 *   out[:,t,:] = matrices[t] @ h[:,t,:] with real matrices (n_theta, n_vel, n_vel)
 *   row-major; evaluated as a real DGEMM on the interleaved complex view
 *   (n_vel x 2*n_cells) with fp64 DMMA, fixed K order (bitwise deterministic). */
int gk_collision(const double* matrices, const double* h, double* out,
                 int64_t n_vel, int64_t n_theta, int64_t n_cells, void* stream);

/* Spectral plan for (n_kx, n_ky) retained modes on an (n_x, n_y) padded grid
 * (spectral.py:116-161, 232-268).  Holds fp64 twiddle tables on the current
 * device.  Any n_x >= n_kx, n_y//2+1 >= n_ky is accepted (any radix; primes
 * other than 2,3,5,7 run a generic O(p^2) pass). */
int gk_spectral_plan_create(int64_t n_kx, int64_t n_ky, int64_t n_x, int64_t n_y,
                            gk_spectral_plan** plan);
int gk_spectral_plan_destroy(gk_spectral_plan* plan);

/* Workspace for gk_bracket / gk_nonlinear with n_g distinct g slices. */
int64_t gk_bracket_workspace_bytes(const gk_spectral_plan* plan, int64_t n_slices, int64_t n_g);

/* bracket (spectral.py:232-268) for a batch of slices:
 *   out[s] = {f[fidx(s)], g[gidx(s)]},  fidx(s) = f_map ? f_map[s] : s,
 *   gidx(s) = g_map ? g_map[s] : s % g_mod   (maps are device int64 arrays or NULL).
 * f, g, out: (n_ky, n_kx) complex slices.  n_g = number of g slices. */
int gk_bracket(const gk_spectral_plan* plan, const double* f, const double* g, double* out,
               int64_t n_slices, const int64_t* f_map, const int64_t* g_map, int64_t n_g,
               int64_t g_mod, void* workspace, int64_t workspace_bytes, void* stream);

/* nonlinear_kernel (kernels.py:126-150): bracket of every (v, theta) slice of h with
 * phi[theta].  h/out: n_vel*n_theta slices, phi: n_theta slices. */
int gk_nonlinear(const gk_spectral_plan* plan, const double* h, const double* phi, double* out,
                 int64_t n_vel, int64_t n_theta, void* workspace, int64_t workspace_bytes,
                 void* stream);

/* to_real (spectral.py:116-138) / to_spectrum (spectral.py:141-161) on a batch. */
int64_t gk_transform_workspace_bytes(const gk_spectral_plan* plan, int64_t batch);
int gk_to_real(const gk_spectral_plan* plan, const double* spec, double* field, int64_t batch,
               void* workspace, int64_t workspace_bytes, void* stream);
int gk_to_spectrum(const gk_spectral_plan* plan, const double* field, double* spec, int64_t batch,
                   void* workspace, int64_t workspace_bytes, void* stream);

/* out = h + dt * (a + b + c) elementwise over n complex values; b or c may be NULL.
 * Association ((a + b) + c) matches the reference composition order. */
int gk_axpy3(const double* h, const double* a, const double* b, const double* c, double dt,
             double* out, int64_t n, void* stream);

/* Fused end of the step: out = shear(h + dt * ((stream(h) + nl) + coll), shifts)
 * in one HBM pass (stream computed on the fly, optimized variant; shear applied as
 * a bijective scatter).  Bit-identical to gk_stream + gk_axpy3 + gk_shear.
 * nl may be NULL (linear-only).  Widths 1,3,5,7,9. */
int gk_step_finish(const double* h, const double* nl, const double* coll, const double* stencil_host,
                   int width, const int32_t* shifts, double dt, double* out, int64_t n_vel,
                   int64_t n_theta, int64_t n_ky, int64_t n_kx, void* stream);

/* One builder-defined time step (no reference step exists):
 *   phi = field(h, w); rhs = stream(h) + nonlinear(h, phi) + collision(h);
 *   h_out = shear(h + dt * rhs, shifts).
 * plan == NULL runs the linear-only path (no bracket).  phi_out may be NULL. */
int64_t gk_step_workspace_bytes(const gk_spectral_plan* plan, int64_t n_vel, int64_t n_theta,
                                int64_t n_ky, int64_t n_kx);
int gk_step(const gk_spectral_plan* plan, const double* h, const double* weights,
            const double* stencil_host, int width, const double* matrices, const int32_t* shifts,
            double dt, double* h_out, double* phi_out, int64_t n_vel, int64_t n_theta,
            int64_t n_ky, int64_t n_kx, void* workspace, int64_t workspace_bytes, void* stream);
/* gk_step with flags.  GK_STEP_REUSE_MATRICES: the int8 slices of the collision
 * matrices (collision_kernel's `matrices`, kernels.py:109-123) that a previous
 * gk_step / gk_step_ex call left in this workspace are reused instead of being
 * made again -- the caller guarantees `matrices` is unchanged since that call
 * (the step is then bit-identical to gk_step).  No effect on the DMMA path. */
#define GK_STEP_REUSE_MATRICES 1
int gk_step_ex(const gk_spectral_plan* plan, const double* h, const double* weights,
               const double* stencil_host, int width, const double* matrices, const int32_t* shifts,
               double dt, double* h_out, double* phi_out, int64_t n_vel, int64_t n_theta,
               int64_t n_ky, int64_t n_kx, void* workspace, int64_t workspace_bytes, int flags,
               void* stream);
/* Workspace for a given stencil width (width <= 9 uses the fused finish pass and
 * needs one state buffer less than gk_step_workspace_bytes' any-width bound). */
int64_t gk_step_workspace_bytes_w(const gk_spectral_plan* plan, int width, int64_t n_vel,
                                  int64_t n_theta, int64_t n_ky, int64_t n_kx);
/* One stage of gk_step on the same workspace (for per-stage timing): 0 field,
 * 1 nonlinear, 2 collision, 3 finish.  Stages read what earlier stages wrote. */
int gk_step_stage(int stage, const gk_spectral_plan* plan, const double* h, const double* weights,
                  const double* stencil_host, int width, const double* matrices, const int32_t* shifts,
                  double dt, double* h_out, int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx,
                  void* workspace, int64_t workspace_bytes, void* stream);

/* In-place step (no reference counterpart; for states too large for gk_step's
 * ~4 state buffers, e.g. em04b on one GPU): h is overwritten with
 *   shear(h + dt * (stream(h) + (collision(h) + nonlinear(h, phi))), shifts)
 * -- gk_step's composition with the rhs associated differently.  The workspace
 * holds phi, one state-sized rhs buffer and the bracket workspace.  stage -1 runs
 * the whole step; 0 field, 1 collision, 2 nonlinear (accumulated onto rhs),
 * 3 finish (in-place stream + axpy, then shear back into h) for per-stage timing.
 * Stencil widths 1..9. */
int64_t gk_step_inplace_workspace_bytes(const gk_spectral_plan* plan, int64_t n_vel, int64_t n_theta,
                                        int64_t n_ky, int64_t n_kx);
int gk_step_inplace(int stage, const gk_spectral_plan* plan, double* h, const double* weights,
                    const double* stencil_host, int width, const double* matrices, const int32_t* shifts,
                    double dt, double* phi_out, int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx,
                    void* workspace, int64_t workspace_bytes, void* stream);
/* out += nonlinear(h, phi) (gk_nonlinear with each result added to out; one
 * rounding per element).  Its workspace holds one chunk of output rows more. */
int64_t gk_nonlinear_acc_workspace_bytes(const gk_spectral_plan* plan, int64_t n_vel, int64_t n_theta);
int gk_nonlinear_acc(const gk_spectral_plan* plan, const double* h, const double* phi, double* out,
                     int64_t n_vel, int64_t n_theta, void* workspace, int64_t workspace_bytes, void* stream);
/* rhs = h + dt * (stream(h) + rhs) in place on rhs (optimized stencil, widths 1..9). */
int gk_stream_axpy_inplace(const double* h, double* rhs, const double* stencil_host, int width, double dt,
                           int64_t n_vel, int64_t n_theta, int64_t n_cells, void* stream);

/* Reference input generator on the device (grid.py:122-161):
 *   out[i*out_stride] = low + (high-low) * ((raw[offset+i] >> 11) * 2^-53),
 * raw = numpy.random.Philox(key=seed).jumped(stream_id) outputs, bit-exact.
 * random_state(shape, seed) = real part from raw[0, n), imaginary from raw[n, 2n). */
int gk_philox_uniform(uint64_t seed, uint64_t stream_id, int64_t offset, int64_t count, double low,
                      double high, double* out, int64_t out_stride, void* stream);

/* The same generator on a strided sub-block of the stream:
 *   out[(row*row_len + j)*out_stride] = uniform(raw[offset + row*row_stride + j]),
 * e.g. one rank's toroidal shard of random_state (rows = (v, theta), row_len =
 * (Y/G)*R, row_stride = Y*R, offset = y0*R; the imaginary part at offset + n). */
int gk_philox_uniform_rows(uint64_t seed, uint64_t stream_id, int64_t offset, int64_t n_rows, int64_t row_len,
                           int64_t row_stride, double low, double high, double* out, int64_t out_stride,
                           void* stream);

/* Theta-range forms (planes [t0, t1) of the same arrays), used to pipeline the
 * step over theta chunks.  Each computes exactly what the full call computes for
 * those planes (bit-identical). */
int gk_field_range(const double* h, const double* weights, double* out, int64_t n_vel,
                   int64_t n_theta, int64_t n_cells, int64_t t0, int64_t t1, void* stream);
int gk_collision_range(const double* matrices, const double* h, double* out, int64_t n_vel,
                       int64_t n_theta, int64_t n_cells, int64_t t0, int64_t t1, void* stream);
/* Collision arithmetic: 0 auto (certified int8 tensor-core slices when n_vel >= 64 and
 * n_vel^2 * 2*n_cells * n_theta >= 2^30), 1 fp64 DMMA always, 2 int8 slices
 * whenever n_vel <= 8192.
 * Sets the process-wide mode (mode < 0: query only); returns the previous one.
 * The initial mode is 1 with GK_COLLISION=dmma, 2 with GK_COLLISION=int8, else 0. */
int gk_collision_mode(int mode);
/* The int8-slice collision certifies every 64 x 128 output tile: with Q the int8
 * product of the operands' magnitude slices (a lower bound of sum_k |A_ik||B_kj|),
 * the tile is kept when its error bound is <= 2^-37 sum_k |A_ik||B_kj| for every
 * element, else recomputed in fp64 (CUDA-core FMAs, fixed k order).  Number of
 * tiles recomputed so far in this process (synchronises the device). */
int gk_collision_fixups(int64_t* total);
/* Measured dense int8 tensor-core throughput of this device (tcgen05 kind::i8,
 * M128 N256 K32 MMAs on every SM), in 1e12 int8 ops/s.  Synchronous. */
int gk_probe_i8_peak(double* tops);
int gk_nonlinear_range(const gk_spectral_plan* plan, const double* h, const double* phi, double* out,
                       int64_t n_vel, int64_t n_theta, int64_t t0, int64_t t1, void* workspace,
                       int64_t workspace_bytes, void* stream);
int gk_step_finish_range(const double* h, const double* nl, const double* coll, const double* stencil_host,
                         int width, const int32_t* shifts, double dt, double* out, int64_t n_vel,
                         int64_t n_theta, int64_t n_ky, int64_t n_kx, int64_t t0, int64_t t1, void* stream);

/* One step from pinned host memory to pinned host memory (the drop-in call with
 * host buffers): H2D of h_host into h_dev, the step into out_dev, D2H into
 * out_host, pipelined over n_chunks theta chunks on two copy streams so the PCIe
 * transfers overlap the compute.  Result bit-identical to gk_step.  Stencil
 * width <= 9.  Stream-ordered: synchronising `stream` covers the last copy. */
int gk_step_host(const gk_spectral_plan* plan, const double* h_host, double* h_dev, double* out_dev,
                 double* out_host, const double* weights, const double* stencil_host, int width,
                 const double* matrices, const int32_t* shifts, double dt, int64_t n_vel, int64_t n_theta,
                 int64_t n_ky, int64_t n_kx, int n_chunks, void* workspace, int64_t workspace_bytes,
                 void* stream);

/* gk_step_host with flags: GK_STEP_REUSE_MATRICES (as gk_step_ex) and
 * GK_STEP_HOST_OVERLAP -- consecutive calls on alternating device buffer pairs
 * (h_dev, out_dev) pipeline across steps: a call's copy-in waits only until its
 * h_dev's last reader (an earlier call) is done, so it runs during the previous
 * call's compute and D2H tail, and `stream` does NOT wait for the last D2H: call
 * gk_step_host_join(stream) before reading out_host.  Same bits as gk_step. */
#define GK_STEP_HOST_OVERLAP 2
int gk_step_host_ex(const gk_spectral_plan* plan, const double* h_host, double* h_dev, double* out_dev,
                    double* out_host, const double* weights, const double* stencil_host, int width,
                    const double* matrices, const int32_t* shifts, double dt, int64_t n_vel, int64_t n_theta,
                    int64_t n_ky, int64_t n_kx, int n_chunks, void* workspace, int64_t workspace_bytes, int flags,
                    void* stream);
int gk_step_host_join(void* stream);

/* Block permutation used around the all-to-all transposes (no reference code;
 * exchange volume = commsim.py:213-219 alltoall_volume with n1 = ranks):
 *   dst[b][a][0:inner] = src[a][b][0:inner], complex elements. */
int gk_permute_blocks(const double* src, double* dst, int64_t n_a, int64_t n_b, int64_t inner,
                      void* stream);

/* ---- multi-GPU step (SURVEY.md §8 b/e; no reference code: the reference models
 * this decomposition only analytically, commsim.py:213-219 alltoall_volume with
 * n1 = ranks).  One process per GPU.  Home layout of rank r: the toroidal block
 * h[M][T][Y/G][R] of modes [r Y/G, (r+1) Y/G); the bracket runs velocity-sharded
 * with two all-to-all transposes per step.  NCCL is loaded at run time. */
typedef struct gk_comm gk_comm;
#define GK_COMM_UNIQUE_ID_BYTES 128
/* ncclGetUniqueId on the root rank; broadcast the 128 bytes to the others. */
int gk_comm_unique_id(void* id);
/* ncclCommInitRank on the current device + the communicator's stream/events. */
int gk_comm_init(int nranks, int rank, const void* id, gk_comm** comm);
int gk_comm_destroy(gk_comm* comm);
int gk_comm_info(const gk_comm* comm, int* nranks, int* rank, int* nccl_version);
/* The transposes around the bracket, one velocity chunk at a time.  home_rows: a
 * chunk of nranks * rows_per_rank home velocity rows (row_elems complex values
 * each, T * Y/G * R); rank q brackets rows [q rpr, (q+1) rpr).
 * to_nl: home rows -> recv[src rank][rpr][T][Y/G][R] (gk_nonlinear_blocked's input).
 * to_lin: send[dst rank][rpr][T][Y/G][R] -> home rows.  Bytes per rank per call:
 * rpr * row_elems * 16 * (nranks - 1) to the peers. */
int gk_transpose_to_nl(gk_comm* comm, const double* home_rows, double* recv, int64_t rows_per_rank,
                       int64_t row_elems, void* stream);
int gk_transpose_to_lin(gk_comm* comm, const double* send, double* home_rows, int64_t rows_per_rank,
                        int64_t row_elems, void* stream);
/* all-gather of `elems` complex values per rank (phi's toroidal blocks). */
int gk_comm_allgather(gk_comm* comm, const double* send, double* recv, int64_t elems, void* stream);
/* nonlinear_kernel (kernels.py:126-150) on a transpose's blocked layout: h / out
 * [n_blocks][n_vel][n_theta][n_ky / n_blocks][n_kx], phi [n_blocks][n_theta][n_ky /
 * n_blocks][n_kx].  Bit-identical to gk_nonlinear on the contiguous arrays.
 * Workspace: gk_bracket_workspace_bytes(plan, n_vel * n_theta, n_theta). */
int gk_nonlinear_blocked(const gk_spectral_plan* plan, const double* h, const double* phi, double* out,
                         int64_t n_vel, int64_t n_theta, int64_t n_blocks, void* workspace, int64_t workspace_bytes,
                         void* stream);
/* Workspace of one rank's gk_dist_step (n_x = n_y = 0: linear-only).  n_ky is the
 * GLOBAL toroidal count; chunks must divide n_vel / nranks. */
int64_t gk_dist_workspace_bytes(int64_t n_x, int64_t n_y, int64_t n_vel, int64_t n_theta, int64_t n_ky,
                                int64_t n_kx, int nranks, int64_t chunks);
/* One rank's step: gk_step's composition on the home shard, bit-identical to
 * gk_step for any rank count.  shifts: this rank's n_ky / nranks shear shifts;
 * phi_out (may be NULL): this rank's field block.  The transposes of velocity
 * chunk k+1 overlap the bracket of chunk k on the communicator's stream. */
int gk_dist_step(gk_comm* comm, const gk_spectral_plan* plan, const double* h, const double* weights,
                 const double* stencil_host, int width, const double* matrices, const int32_t* shifts, double dt,
                 double* h_out, double* phi_out, int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx,
                 int64_t chunks, void* workspace, int64_t workspace_bytes, int flags, void* stream);
/* One stage of it for per-stage timing: 0 field, 1 nonlinear incl. transposes,
 * 2 collision, 3 finish, 4 the transposes alone. */
int gk_dist_step_stage(int stage, gk_comm* comm, const gk_spectral_plan* plan, const double* h,
                       const double* weights, const double* stencil_host, int width, const double* matrices,
                       const int32_t* shifts, double dt, double* h_out, int64_t n_vel, int64_t n_theta,
                       int64_t n_ky, int64_t n_kx, int64_t chunks, void* workspace, int64_t workspace_bytes,
                       void* stream);
/* nranks ranks of gk_dist_step run in lock-step in one process on one device, the
 * exchanges as device copies (test harness for the rank step's layouts and chunk
 * schedule).  Pointer arrays hold one device pointer per rank. */
int gk_dist_step_sim(int nranks, const gk_spectral_plan* plan, const double* const* h, const double* weights,
                     const double* stencil_host, int width, const double* matrices, const int32_t* const* shifts,
                     double dt, double* const* h_out, double* const* phi_out, int64_t n_vel, int64_t n_theta,
                     int64_t n_ky, int64_t n_kx, int64_t chunks, void* const* workspace, int64_t workspace_bytes,
                     void* stream);

/* ---- P2P transport for the multi-GPU step (no collective library): each rank's
 * exchange window (chunk receive ring, nl ring, phi blocks, flags) is device memory
 * shared by CUDA IPC.  Per velocity chunk the copy engines push the home-row blocks
 * into the peers' windows over NVLink (no SMs), the bracket's x forward transform
 * stores each toroidal block's rows straight into the owning peer's nl ring (the
 * return transpose fused into the FFT kernel), and cuStreamWaitValue32 /
 * cuStreamWriteValue32 on window flags order it all on the device. */
typedef struct gk_p2p gk_p2p;
#define GK_P2P_HANDLE_BYTES 64
int gk_p2p_create(int nranks, int rank, int64_t n_vel, int64_t n_theta, int64_t n_ky, int64_t n_kx, int64_t chunks,
                  gk_p2p** p2p);
int64_t gk_p2p_window_bytes(const gk_p2p* p2p);
int gk_p2p_ipc_handle(const gk_p2p* p2p, void* handle);
/* handles: nranks consecutive GK_P2P_HANDLE_BYTES handles in rank order */
int gk_p2p_connect(gk_p2p* p2p, const void* handles);
int gk_p2p_destroy(gk_p2p* p2p);
/* Connectivity self-test of a connected window (no reference counterpart: guards
   the transport before a step waits on its flags).  Every rank calls send, then
   (after a barrier between the ranks) check: tokens pushed by the copy engines,
   stored by a kernel over P2P and flagged by a stream memory operation must all
   arrive within timeout_ms, else GK_ERR_COMM (callers fall back to NCCL). */
int gk_p2p_selftest_send(gk_p2p* p2p);
int gk_p2p_selftest_check(gk_p2p* p2p, int timeout_ms);
int64_t gk_dist_p2p_workspace_bytes(int64_t n_x, int64_t n_y, int64_t n_vel, int64_t n_theta, int64_t n_ky,
                                    int64_t n_kx, int nranks, int64_t chunks);
/* Local stages of the P2P rank step for per-stage timing: 0 field, 2 collision,
 * 3 finish (the nonlinear stage with its fused transfers = step minus these). */
int gk_dist_step_p2p_stage(int stage, gk_p2p* p2p, const gk_spectral_plan* plan, const double* h,
                           const double* weights, const double* stencil_host, int width, const double* matrices,
                           const int32_t* shifts, double dt, double* h_out, void* workspace, int64_t workspace_bytes,
                           void* stream);
/* One rank's step over the P2P transport (nonlinear step; gk_dist_step's
 * composition, bit-identical to gk_step).  All ranks call it in the same order. */
int gk_dist_step_p2p(gk_p2p* p2p, const gk_spectral_plan* plan, const double* h, const double* weights,
                     const double* stencil_host, int width, const double* matrices, const int32_t* shifts,
                     double dt, double* h_out, double* phi_out, int64_t n_vel, int64_t n_theta, int64_t n_ky,
                     int64_t n_kx, void* workspace, int64_t workspace_bytes, int flags, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GK_H_ */

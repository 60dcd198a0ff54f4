/*
 * dmtk_gpu.h -- C ABI of the B200 (sm_100a) implementation of the dmtk
 * MTTKRP / Khatri-Rao / CP-ALS hot path.
 *
 * This is the drop-in boundary: every entry point replaces one C++ entry
 * point of the reference library (/root/reference/proj/include/dmtk/...),
 * cited per function. Plain pointers and sizes only. Host buffers are
 * row-major factor matrices (I_k x rank) and naturally ordered tensors
 * (mode 0 fastest), exactly the reference layouts (shape.hpp:8-17,
 * matrix.hpp:72-109). The C++ shim include/dmtk_gpu.hpp maps these onto the
 * reference's own types and exceptions.
 *
 * Errors: every call returns a status; the message of the last failing call
 * on this thread is available from dmtk_gpu_last_error(). Status values map
 * to the reference's exception types:
 *   DMTK_GPU_OK             success
 *   DMTK_GPU_EINVAL         std::invalid_argument (same messages as the
 *                           reference validate(), mttkrp.cpp:20-46 etc.)
 *   DMTK_GPU_ERANGE         std::out_of_range     (mode out of range)
 *   DMTK_GPU_EOVERFLOW      std::overflow_error   (shape.cpp:20-22)
 *   DMTK_GPU_ERUNTIME       std::runtime_error    (CUDA error, no device)
 *   DMTK_GPU_EIO            dmtk::TensorFileError (tensor_io.hpp; same
 *                           messages as read_tensor, tensor_io.cpp:79-130)
 * There is no CPU fallback: without a usable B200 every compute call fails
 * with DMTK_GPU_ERUNTIME.
 *
 * Threading: calls are reentrant per device; the `threads` fields of the
 * reference API are accepted and validated (>= 1) but do not change results.
 */
#ifndef DMTK_GPU_H
#define DMTK_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    DMTK_GPU_OK = 0,
    DMTK_GPU_EINVAL = 1,
    DMTK_GPU_ERANGE = 2,
    DMTK_GPU_EOVERFLOW = 3,
    DMTK_GPU_ERUNTIME = 4,
    DMTK_GPU_EIO = 5
};

/* MttkrpAlgo (mttkrp.hpp:16-21) and TwoStepOrder (mttkrp.hpp:23-27). */
enum { DMTK_GPU_BASELINE = 0, DMTK_GPU_ONE_STEP = 1, DMTK_GPU_TWO_STEP = 2, DMTK_GPU_AUTOMATIC = 3 };
enum { DMTK_GPU_ORDER_AUTOMATIC = 0, DMTK_GPU_ORDER_LEFT = 1, DMTK_GPU_ORDER_RIGHT = 2 };

/* TimeBreakdown (timing.hpp:11-20), seconds, measured with CUDA events. */
typedef struct {
    double total, matmul, krp_full, krp_partial, matvec, reduce, reorder, other;
} dmtk_gpu_times;

/* Device-resident dense tensor (the GPU counterpart of DenseTensor,
 * tensor.hpp:19-38). Immutable once created. */
typedef struct dmtk_gpu_tensor_s* dmtk_gpu_tensor;

const char* dmtk_gpu_last_error(void);
int dmtk_gpu_version(void);
/* Number of visible CUDA devices (0 when none). */
int dmtk_gpu_device_count(int* count);

/* Upload a host tensor (natural order) to `device`. Validates the shape like
 * Shape::Shape (shape.cpp:8-25). */
int dmtk_gpu_tensor_upload(int device, int ndim, const int64_t* dims, const double* host, dmtk_gpu_tensor* out);
/* dmtk::gen_tensor (bench.cpp:88-97, bench.hpp:22) generated in HBM: dist 0 =
 * Dist::uniform, the same mt19937_64(seed) draws in the same order, bitwise
 * (the stream is split across CTAs by characteristic-polynomial jump-ahead);
 * dist 1 = Dist::ones. Same layout as dmtk_gpu_tensor_upload. SURVEY 8f-3.
 * The BASELINE configs that are not U[0,1) are
 * fixed transforms of the same uniforms u_0, u_1, ... (natural order):
 *   DMTK_GPU_DIST_SIGNED    U[-1,1):  x_e = 2 u_e - 1
 *   DMTK_GPU_DIST_NORMAL    N(0,1), Box-Muller on (u_2k, u_2k+1):
 *                           x_2k = R cos(2 pi u_2k+1), x_2k+1 = R sin(2 pi u_2k+1),
 *                           R = sqrt(-2 log(1 - u_2k))
 *   DMTK_GPU_DIST_SYMSLICE  dims (I, I, rest...): every slice q symmetric with
 *                           unit diagonal, X(i,j,q) = X(j,i,q) = tanh(0.3 z_m),
 *                           z the N(0,1) stream above, m = q I(I-1)/2 + j(j-1)/2 + i
 *                           for i < j (BASELINE config 5)
 * computed with explicitly rounded IEEE operations so that a host restatement
 * reproduces the bytes exactly. A factor matrix of gen_factors (bench.cpp:108-116)
 * is the 1-way tensor {rows * rank} with seed mode_seed(seed, n). */
enum { DMTK_GPU_DIST_UNIFORM = 0, DMTK_GPU_DIST_ONES = 1, DMTK_GPU_DIST_SIGNED = 2, DMTK_GPU_DIST_NORMAL = 3,
       DMTK_GPU_DIST_SYMSLICE = 4 };
int dmtk_gpu_tensor_generate(int device, int ndim, const int64_t* dims, uint64_t seed, int dist,
                             dmtk_gpu_tensor* out);
/* Host-side check of the generator's jump-ahead (no device needed): raw
 * (untempered) words 312+start .. 623+start of mt19937_64(seed), i.e. the
 * words whose tempered values are draws start .. start+311. 0 or -1. */
int dmtk_gpu_mt64_jump(uint64_t seed, int64_t start, uint64_t* words312);
/* Wrap an existing device buffer without copying (DenseTensor::borrow,
 * tensor.hpp:23); the caller keeps it alive and unchanged. The call waits for
 * the device to finish pending work (the values are read later on the
 * library's own stream, so writes still queued on the caller's streams must
 * have landed). */
int dmtk_gpu_tensor_wrap(int device, int ndim, const int64_t* dims, const double* device_ptr, dmtk_gpu_tensor* out);
int dmtk_gpu_tensor_free(dmtk_gpu_tensor t);
/* Shape-only view of a tensor handle (read back the device pointer). */
int dmtk_gpu_tensor_info(dmtk_gpu_tensor t, int* ndim, int64_t* dims_out8, const double** device_ptr);

/* Tensor ingest: dmtk::read_tensor (tensor_io.hpp:25) straight
 * into HBM. Reads a DNT1 file ("DNT1", u32 version 1, u32 N, N u64 extents,
 * the little-endian FP64 payload in natural order, nothing after it) with the
 * reference's validation and messages, streaming the payload through two
 * pinned staging buffers so file reads overlap the host-to-device copies. */
int dmtk_gpu_tensor_load(int device, const char* path, dmtk_gpu_tensor* out);
/* Tensors symmetric in modes 0 and 1 (BASELINE config 5's fMRI slices;
 * SURVEY 8f-4): checks X(i, j, ...) == X(j, i, ...) exactly (EINVAL
 * otherwise) and returns a new handle holding only the upper triangle of
 * every slice (I (I + 1) / 2 pairs instead of I^2 entries). Such a handle
 * supports dmtk_gpu_cp_als -- a dimension-tree sweep whose left half is the
 * pair index, so both tensor passes read about half the bytes; fits agree with
 * the reference's CP-ALS on the full tensor -- and dmtk_gpu_tensor_norm (of the
 * full tensor); the other calls reject it. */
int dmtk_gpu_tensor_pack_sym01(dmtk_gpu_tensor t, dmtk_gpu_tensor* out);
/* Last-mode slab: a new device tensor holding the rows [lo, hi)
 * of the slowest mode of t (one contiguous device-to-device copy in the
 * natural layout), e.g. one rank's shard of a tensor generated whole. */
int dmtk_gpu_tensor_slab(dmtk_gpu_tensor t, int64_t lo, int64_t hi, dmtk_gpu_tensor* out);
/* The tensor's values back to host memory in natural order (total doubles). */
int dmtk_gpu_tensor_download(dmtk_gpu_tensor t, double* host_out);

/* dmtk::mttkrp (mttkrp.hpp:45) and mttkrp_baseline/one_step/two_step
 * (mttkrp.hpp:47-49) selected by `algo`. factors[k] is the host row-major
 * factor_rows[k] x factor_cols[k] matrix of mode k, for nfactors modes
 * (MttkrpRequest::factors, mttkrp.hpp:31; factors[mode] is validated but
 * unused, like the reference). Validation, its order and its messages
 * follow validate() (mttkrp.cpp:20-46). out: host I_mode x rank row-major.
 * times may be NULL. Honours DMTK_INJECT_FAULT like mttkrp.cpp:110-118. */
int dmtk_gpu_mttkrp(dmtk_gpu_tensor t, int nfactors, const double* const* factors, const int64_t* factor_rows,
                    const int64_t* factor_cols, int64_t mode, int algo, int order, int threads, double* out,
                    dmtk_gpu_times* times);

/* Same contraction with every operand already on the device; enqueued on
 * `stream` (a cudaStream_t; NULL = the legacy default stream) without host
 * synchronisation. No fault hook. The library's workspace is per device:
 * callers order concurrent device calls on one device (one stream). Used by
 * the device-resident benchmark leg. */
int dmtk_gpu_mttkrp_device(dmtk_gpu_tensor t, const double* const* device_factors, int64_t rank, int64_t mode,
                           int algo, int order, double* device_out, void* stream);

/* dmtk::choose_order (mttkrp.hpp:53): writes DMTK_GPU_ORDER_LEFT/RIGHT. */
int dmtk_gpu_choose_order(int ndim, const int64_t* dims, int64_t mode, int* order);

/* dmtk::krp / krp_naive / krp_small (krp.hpp:75-83): K = in[0] (.) ... (.)
 * in[z-1], last input fastest, left-to-right association, bitwise equal to
 * the reference. inputs are host row-major rows[k] x cols; out host
 * (prod rows) x cols. hadamards (may be NULL) receives the number of
 * C-length row products performed (KrpStats, krp.hpp:15-17): the
 * single-thread reuse count for variant 0, rows*(z-1) for variant 1
 * (naive). */
int dmtk_gpu_krp(int device, int z, const double* const* inputs, const int64_t* rows, int64_t cols, int variant,
                 double* out, uint64_t* hadamards);
/* Device-pointer variant (no host sync). scratch may be NULL for z <= 2;
 * otherwise it must hold prod(rows[0..z-2]) * cols doubles. */
int dmtk_gpu_krp_device(int z, const double* const* device_inputs, const int64_t* rows, int64_t cols,
                        double* device_out, double* device_scratch, void* stream);

/* dmtk::tensor_norm (cp_als.hpp:68). */
int dmtk_gpu_tensor_norm(dmtk_gpu_tensor t, double* out);

/* dmtk::gram_hadamard (linalg.hpp:48) and solve_psd (linalg.hpp:54), host
 * buffers. */
int dmtk_gpu_gram_hadamard(int device, int ndim, const int64_t* rows, int64_t rank, const double* const* factors,
                           int64_t skip, double* h_out);
int dmtk_gpu_solve_psd(int device, int64_t rank, const double* h, int64_t rows, const double* m, double* u_out);

/* AlsConfig (cp_als.hpp:32-40), plus one GPU-only field appended:
 * dimtree = 1 runs each sweep as a dimension tree (PAPER.md
 * 759-762): the modes split into a left and a right half, one pass over the
 * tensor per half forms the half's partial MTTKRP (the other half's KRP
 * contracted away), and every mode of the half takes its MTTKRP from that
 * partial with a multi-TTV. Same updates in the same order as the reference
 * sweep (a partial only involves factors not updated while it is in use);
 * two tensor passes per iteration instead of N. 0 (zero-initialised callers)
 * keeps the reference's one MTTKRP per mode. */
typedef struct {
    int64_t rank;
    int max_iters;
    double tol;
    uint64_t seed;
    int threads;
    int algo;
    int order;
    int dimtree;
} dmtk_gpu_als_config;

/* dmtk::cp_als (cp_als.hpp:83): KruskalModel::random init (same mt19937_64
 * stream), Gauss-Seidel sweeps fully on the device, reconstruction-free fit.
 * factors_out: concatenation of the N final factors (row-major); lambda_out:
 * rank; fits_out / iter_seconds_out: capacity max_iters (iter_seconds may be
 * NULL); mode_seconds_out (may be NULL): max_iters * ndim per-mode MTTKRP
 * seconds. */
int dmtk_gpu_cp_als(dmtk_gpu_tensor t, const dmtk_gpu_als_config* cfg, double* factors_out, double* lambda_out,
                    double* fits_out, double* iter_seconds_out, double* mode_seconds_out, int* n_iters,
                    int* zero_tensor, double* tensor_norm_out);

/* dmtk::als_iterate (cp_als.hpp:74-75, cp_als.cpp:122-158): one Gauss-Seidel
 * sweep over modes 0..N-1 of the model (factors[k]: host row-major
 * factor_rows[k] x factor_cols[k], updated in place; lambda: nlambda = rank,
 * updated in place) against t, with ||X|| = norm_x supplied by the caller
 * (cp_als passes tensor_norm). fit4_out = {fit, rel_residual, abs_residual,
 * defined} of the reconstruction-free fit from the last mode;
 * seconds_out (may be NULL) = the sweep's device time; mode_seconds_out (may
 * be NULL) = ndim per-mode seconds. Uses cfg->algo / order / threads; the
 * rank comes from the model. Validation follows validate_model
 * (cp_als.cpp:74-83) then the MTTKRP checks. iter_index is the record's
 * index (AlsIterRecord::iter) and does not change the computation. */
int dmtk_gpu_als_iterate(dmtk_gpu_tensor t, const dmtk_gpu_als_config* cfg, int nfactors, double* const* factors,
                         const int64_t* factor_rows, const int64_t* factor_cols, double* lambda, int64_t nlambda,
                         double norm_x, int iter_index, double* fit4_out, double* seconds_out,
                         double* mode_seconds_out);

/* Multi-GPU CP-ALS over last-mode shards (the reference's
 * cp_als, cp_als.cpp:122-200, with the tensor split along its slowest mode).
 * One process per GPU; rank r's tensor handle holds the contiguous slab of
 * last-mode rows [last_lo, last_lo + I_{N-1}^r) of a tensor whose last extent
 * is last_extent. The library loads NCCL at run time (libnccl.so.2) and
 * all-reduces, on its stream (inside the per-mode CUDA graphs): the I_n x C
 * MTTKRP partials of modes n < N-1, the column sums of squares and the Gram of
 * the row-sharded last factor, the fit's inner product and ||X||^2. Every
 * other step runs redundantly and identically on every rank. Initialisation
 * follows KruskalModel::random (cp_als.cpp:87-99) over the global shape, each
 * rank keeping its rows of the last factor. factors_out: modes 0..N-2 in full,
 * then this rank's rows of mode N-1. The per-mode sweep, or with dimtree = 1
 * the dimension tree (the left partial and the right half's non-last-mode
 * multi-TTVs all-reduced; the split chosen on the global shape); a packed
 * symmetric slab (dmtk_gpu_tensor_pack_sym01 of this rank's slab) runs its
 * pair-index tree with Q all-reduced.
 *
 * Exchanges (csrc/xrank.cu): by default every rank maps every
 * other rank's receive buffer over NVLink (CUDA IPC handles exchanged with
 * one NCCL all-gather at dmtk_gpu_comm_init) and each exchange is ONE kernel:
 * for a mode's partials it is the MTTKRP's own slot reduction, which pushes
 * this rank's rows into every peer and sums all ranks' rows in rank order --
 * no separate ncclAllReduce, and the factors are bitwise identical on every
 * rank. DMTK_GPU_XRANK=0 (read at communicator creation), or a failed peer
 * mapping on any rank, keeps NCCL all-reduces.
 *
 * dmtk_gpu_comm_unique_id: 128-byte NCCL id, made on one rank and broadcast
 * by the caller (e.g. torch.distributed) to all ranks, which then call
 * dmtk_gpu_comm_init with their rank and device. */
typedef struct dmtk_gpu_comm_s* dmtk_gpu_comm;
int dmtk_gpu_comm_unique_id(unsigned char* id128);
int dmtk_gpu_comm_init(const unsigned char* id128, int rank, int world, int device, dmtk_gpu_comm* out);
int dmtk_gpu_comm_free(dmtk_gpu_comm comm);
/* Loopback communicators (tests of the sharded path without a second GPU):
 * `world` (1..16) virtual ranks on one device, comms_out[k] = rank k. Each
 * rank's dmtk_gpu_cp_als_sharded must run concurrently in its own host thread
 * (ranks get separate contexts and streams). Same exchanges, same code path
 * and the same exchange kernel as the NCCL communicator, except that the
 * sweeps run eagerly (no CUDA graphs) and each exchange runs the P ranks as
 * ONE cooperative launch over the ranks' buffers on the device (rank 0's
 * thread launches it once every rank has published its side: a host barrier
 * plus stream events), never as separate launches waiting on one another.
 * With DMTK_GPU_XRANK=0 the exchanges are stream-event all-reduces instead.
 * Free every handle with dmtk_gpu_comm_free. */
int dmtk_gpu_comm_loopback(int world, int device, dmtk_gpu_comm* comms_out);
/* MTTKRP of a last-mode slab over the communicator: `slab` is
 * this rank's slab, device_factors the full factors of modes 0..N-2 and this
 * rank's rows of U_{N-1}. For mode n < N-1 device_out receives the full
 * I_n x C result, summed over the ranks -- with the peer exchange that sum is
 * the MTTKRP's own slot reduction (one kernel, rank order, the same bits on
 * every rank), else an NCCL all-reduce follows; for the last mode it receives
 * this rank's rows. Enqueued on `stream` (NULL: the legacy default stream);
 * every rank calls it for the same modes in the same order (loopback ranks
 * concurrently). */
int dmtk_gpu_mttkrp_sharded(dmtk_gpu_comm comm, dmtk_gpu_tensor slab, const double* const* device_factors,
                            int64_t rank, int64_t mode, int algo, int order, double* device_out, void* stream);
/* rank, world, and fused = 1 when the exchanges run over peer memory
 * (xrank), 0 for NCCL / event all-reduces. */
int dmtk_gpu_comm_info(dmtk_gpu_comm comm, int* rank, int* world, int* fused);
/* In-place sum over the communicator's ranks of n doubles in device memory,
 * on `stream` (NULL: the library's stream; the call returns once the exchange
 * is enqueued). With the peer exchange the sum is taken in rank order, so
 * every rank gets the same bits; otherwise ncclAllReduce. Every rank calls it
 * with the same n (loopback ranks concurrently, one host thread each). */
int dmtk_gpu_comm_allreduce(dmtk_gpu_comm comm, double* device_buf, int64_t n, void* stream);
int dmtk_gpu_cp_als_sharded(dmtk_gpu_tensor slab, dmtk_gpu_comm comm, int64_t last_extent, int64_t last_lo,
                            const dmtk_gpu_als_config* cfg, double* factors_out, double* lambda_out, double* fits_out,
                            double* iter_seconds_out, double* mode_seconds_out, int* n_iters, int* zero_tensor,
                            double* tensor_norm_out);

/* dmtk::fit (cp_als.hpp:79) of the model (factors, lambda) against t:
 * out4 = {fit, rel_residual, abs_residual, defined}. Validation follows
 * validate_model (cp_als.cpp:74-83) then the MTTKRP checks. */
int dmtk_gpu_fit(dmtk_gpu_tensor t, int nfactors, const double* const* factors, const int64_t* factor_rows,
                 const int64_t* factor_cols, const double* lambda, int64_t nlambda, int threads, double* out4);

/* Measured FP64 tensor-core (DMMA) throughput of `device`, TFLOP/s; the
 * roofline denominator the benchmark reports (MEASURED_PEAKS.json has no
 * FP64 entry). */
int dmtk_gpu_fp64_peak(int device, double* tflops);
/* The same probe run back to back for `seconds`: the settled (power-capped)
 * rate, the denominator for kernels timed inside a long step. */
int dmtk_gpu_fp64_peak_sustained(int device, double seconds, double* tflops);

/* Number of kernels this library has launched since load (for the
 * benchmark's gpu_launches claim). */
int64_t dmtk_gpu_launch_count(void);

/* Developer timeline of the last streaming MTTKRP launch on `device` when
 * the process runs with DMTK_GPU_TRACE=1: 16 %globaltimer stamps (ns) per
 * CTA, 0 = not reached; see TraceEv in csrc/mttkrp_plan.h. Not part of the
 * reference interface. */
int dmtk_gpu_debug_trace(int device, uint64_t* host_out, int max_ctas, int* n_ctas);
/* Number of tensor shapes whose plans and CSR slot maps are cached for the
 * calling thread's execution slot (at most 64 per device and slot, least
 * recently used dropped first). */
int dmtk_gpu_debug_cached_shapes(int64_t* n);

#ifdef __cplusplus
}
#endif

#endif

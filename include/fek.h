/*
 * fek.h -- C-ABI of libfek.so: B200 (sm_100a) element integration for
 * first-order tetrahedra and prisms (arXiv 1504.01023).
 *
 * This is the drop-in boundary for the reference's hot path.  Each entry
 * point names the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/feklab):
 *
 *   fek_integrate       <- kernels/batched.py:518-533  the _BATCHED_KERNELS
 *                          registry slot + _run_range block loop, i.e. the body
 *                          of integrate_batch (batched.py:536-606) after the
 *                          layout decode; device buffers, stream-ordered.
 *   fek_integrate_host  <- kernels/batched.py:536-606  integrate_batch as a
 *                          whole, on HOST arrays (ElementBatch.geometry_data /
 *                          coefficient_data in, BatchResult.stiffness / load
 *                          out): chunked H2D -> kernel -> D2H pipeline.
 *   fek_integrate_host_staged <- the same for pageable host arrays (staged
 *                          through page-locked buffers by host copy threads).
 *   fek_classify        <- batched.py:136-177  _bbox_scale + _adjugate +
 *                          _check_dets with the reference's rounding: the exact
 *                          first-error key when fek_integrate reports NEAR.
 *   fek_decode_error    <- errors.py:8-27 + batched.py:166-177,593-599  the
 *                          first-error rule (element, quadrature point, kind).
 *   fek_error_detail    <- batched.py:172-177  the |det J| / tol numbers that
 *                          go into the DegenerateElement/InvertedElement text.
 *   fek_jacobian        <- geometry.py:94-138  jacobian_affine /
 *                          jacobian_at_point (JacobianData) of one element.
 *   fek_apply           <- (new) the element matrices consumed in
 *                          the kernel: matrix-free y += sum_e P_e^T A_e P_e x.
 *   fek_assemble        <- (new) the same, assembled into a CSR
 *                          global matrix and load vector.
 *   fek_checksum        <- (new) per-shard verification sums reduced with
 *                          NCCL across GPUs.
 *
 * Conventions
 *  - Plain C types only.  All device pointers are caller-owned (PyTorch
 *    allocations in the Python host layer); the library never allocates
 *    device memory and keeps no mutable global state besides a per-kernel
 *    attribute cache, so calls are safe from several host threads on
 *    distinct streams.
 *  - Input layout (batch flat arrays) follows layout.py:1-23:
 *      element-major:        datum d of element e at e*DS + d
 *      lane-interleaved (W): (e/W)*W*DS + d*W + e%W   (tail padded to W)
 *    Outputs are element-major: stiffness (n, ns, ns) row-major, load (n, ns)
 *    (batched.py:566-567).
 *  - Base pointers must be 16-byte aligned.
 *  - Results are bitwise independent of layout, lane width, launch chunking
 *    and base_index sharding: every element runs the same instruction
 *    sequence (batched.py:10-13 promises the same for workers/layout).
 */
#ifndef FEK_H
#define FEK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FEK_ABI_VERSION 4

/* enums mirror the Python ones (refelem.py:29, problems.py:26-49) */
enum fek_element { FEK_TETRAHEDRON = 0, FEK_PRISM = 1 };
enum fek_problem { FEK_POISSON = 0, FEK_CONV_DIFF = 1 };
enum fek_variant { FEK_QSS = 0, FEK_SQS = 1, FEK_SSQ = 2 };
enum fek_geometry_path { FEK_GEO_LINEAR = 0, FEK_GEO_GENERIC = 1 };
enum fek_dtype { FEK_F64 = 0, FEK_F32 = 1 };
enum fek_layout_kind { FEK_ELEMENT_MAJOR = 0, FEK_LANE_INTERLEAVED = 1 };
/* output format: split arrays (BatchResult.stiffness / .load, batched.py:566-567)
 * or packed rows [A row-major | b] per element in the output layout
 * (BatchResult.flat_output, batched.py:99-106, layout.py:72-82) */
enum fek_out_format { FEK_OUT_SPLIT = 0, FEK_OUT_PACKED = 1 };

/* status codes */
enum fek_status {
  FEK_OK = 0,
  FEK_ERR_ARGUMENT = 1,      /* bad enum / size / combination            */
  FEK_ERR_ALIGNMENT = 2,     /* a base pointer is not 16-byte aligned      */
  FEK_ERR_CUDA = 3,          /* CUDA runtime error (see fek_last_cuda_error) */
  FEK_ERR_WORKSPACE = 4,     /* host-pipeline workspace too small          */
  FEK_ERR_GEOMETRY = 5       /* fek_integrate_host: a degenerate/inverted element */
};

/* error word: all-ones = no error; smaller key = earlier error */
#define FEK_NO_ERROR 0xFFFFFFFFFFFFFFFFull
#define FEK_KIND_DEGENERATE 1
#define FEK_KIND_INVERTED 2
#define FEK_KIND_PIPELINE_TIMEOUT 3 /* recorded just before the kernel traps (internal error) */
/* The integration kernels classify on their own FMA-contracted det J against
 * 16 x the degeneracy tolerance; the reference rounds det J differently
 * (batched.py:151-163).  Beyond that bound both dets give the same class (fp64;
 * fp32 rounding of det J is ~1e-6 diag^3, far above the tolerance, so the fp32
 * kernels classify only approximately); within it (never on a valid mesh) the
 * kernel records NEAR at the element's first such point and the caller re-derives
 * the exact key with fek_classify. */
#define FEK_KIND_NEAR 4
/* fek_assemble: the CSR pattern has no entry for a node pair of the element (no point: the
 * smallest such element wins); that contribution is skipped, nothing is written out of place */
#define FEK_KIND_PATTERN 5

typedef struct fek_batch_desc {
  int32_t element;        /* enum fek_element                                   */
  int32_t problem;        /* enum fek_problem                                   */
  int32_t variant;        /* enum fek_variant                                   */
  int32_t geometry_path;  /* enum fek_geometry_path (LINEAR requires TETRAHEDRON) */
  int32_t dtype;          /* enum fek_dtype: real type of all four arrays        */
  int32_t layout;         /* enum fek_layout_kind of geometry/coefficients       */
  int32_t lane_width;     /* W in {1,4,8,16,32,64}; 1 for element-major         */
  int32_t out_format;     /* enum fek_out_format                                 */
  int64_t n_elements;     /* elements covered by this call                       */
  int64_t base_index;     /* absolute index of element 0 (errors, sharding)      */
  const void *geometry;   /* flat geometry_data  (3*nv reals per element)        */
  const void *coefficients; /* flat coefficient_data (nq or 20 reals)            */
  void *stiffness;        /* SPLIT: (n, ns, ns) reals.  PACKED: the flat packed
                             array, flat_length(n, ns*ns + ns, out layout) reals,
                             lane-interleaved pad lanes written as NaN           */
  void *load;             /* SPLIT: (n, ns) reals.  PACKED: unused (NULL)         */
  unsigned long long *error_key; /* device word (fek_integrate), init FEK_NO_ERROR */
  int32_t out_lane_width; /* PACKED: output lane width W (1 = element-major rows)  */
  int32_t ctas_per_sm;    /* cap on resident CTAs per SM for this launch (0 = occupancy
                             maximum); lets two launches share the SMs concurrently  */
  unsigned long long *scheduler; /* optional device words [2], zero-initialised once:
                             dynamic tile queue (CTAs take tiles with atomicAdd, the
                             last CTA resets both words, so a buffer is reusable by
                             later launches on the same stream; one buffer per
                             concurrently running launch).  NULL = static
                             round-robin tiles.  fek_integrate_host ignores it
                             and keeps one queue per stream in its workspace. */
  int32_t tile_elements;  /* elements per CTA tile (the tuner's T): 0 = the kernel's own
                             choice; 64 / 128 / 256 for the QSS natural-path kernels
                             (geo_linear tets, geo_generic prisms), else FEK_ERR_ARGUMENT.
                             Results are bitwise independent of it. */
  int32_t reserved;       /* 0 */
} fek_batch_desc;

int fek_abi_version(void);
/* sizeof(fek_batch_desc) as compiled: a binding checks its own struct
 * layout against this before the first call */
size_t fek_batch_desc_size(void);
const char *fek_status_string(int status);
/* message of the last CUDA error seen by this thread (empty if none) */
const char *fek_last_cuda_error(void);

/* Stream-ordered integration of d->n_elements elements; all pointers device.
 * Asynchronous: returns after the launch.  Geometry failures are recorded
 * with atomicMin into *d->error_key (the reference's first-error rule). */
int fek_integrate(const fek_batch_desc *d, void *cuda_stream);

/* Matrix-free operator application fused with the integration (
 * element contributions used "without assembly, in the so called
 * matrix-free approaches", the "assembly operation designed as extension of procedures
 * performing numerical integration").  For every element e of d, with the node numbers
 * element_nodes[e*ns + s] (int32, ns = 4 / 6):
 *     y[node(e, r)] += sum_s A_e[r][s] x[node(e, s)]      f[node(e, r)] += b_e[r]
 * where A_e, b_e are exactly the matrices fek_integrate would write -- the same kernel math,
 * kept in registers, so A and b never reach memory.  x, y, f (f may be NULL) are device
 * arrays of d's real type; y and f accumulate with atomicAdd, so the summation order (and
 * the last bits of y, f) vary between runs.  QSS natural-path descriptors (geo_linear tets,
 * geo_generic prisms), element-major inputs; d->stiffness / d->load are unused; geometry
 * errors are reported in d->error_key exactly as by fek_integrate.  Node numbers must index
 * x, y and f (unchecked here; apply_batch checks them). */
int fek_apply(const fek_batch_desc *d, const int32_t *element_nodes, const void *x, void *y, void *f,
              void *cuda_stream);

/* Global sparse assembly fused with the integration (the other consumer PAPER.md:121-123 names):
 * for every element e of d,
 *     values[k(node(e, r), node(e, s))] += A_e[r][s]      f[node(e, r)] += b_e[r]
 * where k(i, j) is the position of column j in row i of the caller's CSR pattern (int32
 * row_ptr[n_nodes + 1] and col[nnz], columns sorted within each row, containing every
 * element's node pairs -- e.g. built by the Python csr_pattern).  A_e, b_e are fek_integrate's,
 * kept in registers; values and f accumulate with atomicAdd (order, hence last bits, vary).
 * Same descriptor rules as fek_apply; node numbers must be valid rows of the pattern, and a
 * node pair missing from it is recorded in d->error_key as FEK_KIND_PATTERN. */
int fek_assemble(const fek_batch_desc *d, const int32_t *element_nodes, const int32_t *row_ptr, const int32_t *col,
                 void *values, void *f, void *cuda_stream);

/* Launch geometry fek_integrate would use (for reporting / launch counting). */
int fek_launch_config(const fek_batch_desc *d, int *grid, int *block, int *smem_bytes,
                      int *tile_elements);

/* Whole-batch integration on HOST buffers (d->geometry/coefficients/stiffness/
 * load are host pointers, ideally page-locked; d->error_key is ignored).
 * Elements stream through `n_streams` slots of `chunk_elements` each, carved
 * from the device workspace: chunk i is copied H2D, integrated and copied D2H
 * on streams[i % n_streams], so the copy engines and the SMs overlap.
 * Blocks until done.  On a geometry failure returns FEK_ERR_GEOMETRY and
 * stores the error key in *error_key_out (FEK_NO_ERROR otherwise); NEAR keys
 * are resolved internally (the geometry streams once more through the
 * workspace into fek_classify), so the key is never FEK_KIND_NEAR. */
size_t fek_host_workspace_bytes(const fek_batch_desc *d, int n_streams, int64_t chunk_elements);
int fek_integrate_host(const fek_batch_desc *d, void *device_workspace, size_t workspace_bytes,
                       int n_streams, void *const *cuda_streams, int64_t chunk_elements,
                       unsigned long long *error_key_out);

/* The exact first-error key of d's geometry (device pointer, d's layout and
 * base_index; coefficients/outputs unused): every element's det J at the affine
 * point (geo_linear) or at every quadrature point in order (geo_generic), with
 * the reference's Jacobian, unfused adjugate det and once-rounded tolerance
 * 1e-14 diag^3 (batched.py:136-177), merged with atomicMin into *d->error_key
 * (caller resets it to FEK_NO_ERROR first).  Geometry-only pass, stream-ordered.
 * Call it when fek_integrate's key decodes to FEK_KIND_NEAR; the result is then
 * FEK_NO_ERROR (the batch is valid) or a DEGENERATE / INVERTED key. */
int fek_classify(const fek_batch_desc *d, void *cuda_stream);

/* fek_integrate_host for PAGEABLE host buffers (plain malloc / numpy memory, as a reference
 * caller's ElementBatch holds them, layout.py:103-112): every pageable array among geometry /
 * coefficients / stiffness / load is staged through `host_staging` (page-locked, at least
 * fek_host_staging_bytes(d, n_streams, chunk_elements) bytes -- which looks at d's pointers:
 * a 36 MiB cache-resident input ring when only inputs are pageable, chunk-sized slots when
 * outputs are, 0 when nothing is -- 16-byte aligned) by
 * `copy_threads` host threads, chunk by chunk, so the host copies of chunk i overlap the DMA
 * and the kernels of chunks i-1, i-2; page-locked arrays are DMA'd directly.  Otherwise as
 * fek_integrate_host (same error semantics). */
size_t fek_host_staging_bytes(const fek_batch_desc *d, int n_streams, int64_t chunk_elements);
int fek_integrate_host_staged(const fek_batch_desc *d, void *device_workspace, size_t workspace_bytes, int n_streams,
                              void *const *cuda_streams, int64_t chunk_elements, void *host_staging,
                              size_t staging_bytes, int copy_threads, unsigned long long *error_key_out);

/* Split an error key.  point = -1 on the element-constant (geo_linear) path. */
int fek_decode_error(unsigned long long key, int64_t *element, int32_t *point, int32_t *kind);

/* det J and the degeneracy tolerance of local element `element` of d at
 * quadrature point `point` (-1: affine Jacobian), written to out_det_tol[0..1]
 * (device memory).  Used only to format error messages. */
int fek_error_detail(const fek_batch_desc *d, int64_t element, int32_t point,
                     double *out_det_tol, void *cuda_stream);

/* The mapping Jacobian of local element `element` of d at quadrature point
 * `point` (-1: the affine tet Jacobian), written to out20[0..19] (device
 * memory): [0..8] dx/dxi row-major (J[i][k] = dx_i/dxi_k), [9..17] dxi/dx
 * (adjugate / det), [18] det J, [19] the degeneracy tolerance 1e-14 diag^3.
 * Replaces the scalar geometry helpers jacobian_affine / jacobian_at_point
 * (pkg/src/feklab/geometry.py:94-138) for the per-element API. */
int fek_jacobian(const fek_batch_desc *d, int64_t element, int32_t point, double *out20,
                 void *cuda_stream);

/* Verification sums over d's outputs, written to device memory:
 * out_f64[0..3] = sum A, sum b, sum |A|, sum |b| (fixed-order, deterministic);
 * out_u64[0..1] = wrapping sums of the IEEE bit patterns of A and b entries,
 * each weighted by (absolute element index + 1): exactly additive across
 * shards, so an NCCL SUM of per-GPU values equals the single-GPU value
 * bit for bit.  `partials` is device scratch of fek_checksum_scratch_bytes(). */
size_t fek_checksum_scratch_bytes(void);
int fek_checksum(const fek_batch_desc *d, void *partials, double *out_f64,
                 unsigned long long *out_u64, void *cuda_stream);

/* ---- device-side synthetic inputs ----------------
 * Replace the host generator pkg/src/feklab/mesh.py:49-109 for the benchmark
 * configurations: outputs are bit-identical to the host (numpy) version for
 * any element / draw range, so each GPU of a sharded run can generate exactly
 * its slice of the global mesh.
 *
 * `stream` = numpy PCG64 state as 4 words {state_hi, state_lo, inc_hi, inc_lo}
 * (np.random.PCG64(seed).state).  fek_pcg64_uniform writes draws
 * [first, first + count) of Generator.uniform(low, high). */
int fek_pcg64_uniform(const unsigned long long *stream, int64_t first, int64_t count, double low, double high,
                      double *out, void *cuda_stream);

/* Element-major geometry rows of elements [first, first + n) of the
 * reference unit-cube mesh (Kuhn tets nx*ny*nz*6, or extruded prisms
 * nx*ny*2); prisms optionally get the top-face jitter of
 * mesh.jitter_top_faces (jitter_stream may be NULL). */
int fek_mesh_geometry(int32_t element, int64_t nx, int64_t ny, int64_t nz, int64_t first, int64_t n,
                      const unsigned long long *jitter_stream, double jitter_amplitude, double *out,
                      void *cuda_stream);

/* ---- on-device layout conversion -----------------
 * Replaces layout.convert / pack_rows / unpack_rows
 * (pkg/src/feklab/layout.py:72-94,174-183) for arrays already in HBM:
 * n_elements rows of row_size reals (dtype FEK_F64 / FEK_F32, row_size
 * <= 42) stored with lane width in_lane_width (1 = element-major) are
 * rewritten into dst with lane width out_lane_width; pad lanes of a partial
 * interleaved output block get pad_value (NaN = the reference's default).
 * dst holds ceil(n / W_out) * W_out * row_size reals and must not overlap
 * src.  Asynchronous on cuda_stream. */
int fek_convert_layout(const void *src, int32_t in_lane_width, void *dst, int32_t out_lane_width, int64_t n_elements,
                       int32_t row_size, int32_t dtype, double pad_value, void *cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* FEK_H */

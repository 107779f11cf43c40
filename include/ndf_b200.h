/*
 * ndf_b200.h -- C-ABI of the B200-native NDF hot path (libndf_b200.so).
 *
 * Plain pointers and sizes only: every device pointer is borrowed (the
 * caller -- PyTorch on the Python side -- owns the memory), every call takes
 * a CUDA stream handle (`void*` = cudaStream_t), is stream-ordered and
 * asynchronous, and returns an ndf_status (0 = OK).  On failure
 * ndf_last_error() returns a thread-local message.
 *
 * The reference (/root/reference/pkg/src/ndf) is pure Python; its "FFI"
 * for this path is the Python call surface each entry point replaces,
 * cited per function below.  INTEGRATION.md shows the ctypes binding.
 */
#ifndef NDF_B200_H
#define NDF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NDF_ABI_VERSION 3
#define NDF_MAX_LAYERS 8
#define NDF_MAX_WIDTH 256
#define NDF_MAX_LEVELS 16

/* status codes; mapped onto the reference's NdfError tree (errors.py:4-49) */
typedef enum {
  NDF_OK = 0,
  NDF_ERR_PARAMETER = 1,   /* ParameterError   (errors.py:24) */
  NDF_ERR_SHAPE = 2,       /* ShapeError       (errors.py:36) */
  NDF_ERR_CONFIG = 3,      /* ConfigError      (errors.py:40) */
  NDF_ERR_CUDA = 4,        /* DeviceError (new: CUDA runtime failure) */
  NDF_ERR_UNSUPPORTED = 5, /* ConfigError: shape outside the kernels' envelope */
  NDF_ERR_DEGENERATE = 6   /* ParameterError raised by digamma(0), measures.py:143-144 */
} ndf_status;

/* merge modes: model.py:26 plus BASELINE's [a+b, |a-b|] */
enum { NDF_MERGE_MULTIPLY = 0, NDF_MERGE_CONCAT = 1, NDF_MERGE_ADD = 2,
       NDF_MERGE_ABSDIFF = 3, NDF_MERGE_SUM_ABSDIFF = 4 };
/* hidden activations: nn.py:23-32 plus SiLU */
enum { NDF_ACT_RELU = 0, NDF_ACT_SNAKE = 1, NDF_ACT_SNAKE_ALT = 2, NDF_ACT_SILU = 3 };
/* output head: linear (reference, nn.py:136), tanh (Pearson), softplus (MI) */
enum { NDF_HEAD_LINEAR = 0, NDF_HEAD_TANH = 1, NDF_HEAD_SOFTPLUS = 2 };
/* query precision */
enum { NDF_PREC_FP32 = 0,   /* SIMT fp32, sequential k-sum (nn.py:18-20 order) */
       NDF_PREC_BF16 = 1,   /* tcgen05 bf16 x bf16 -> fp32 TMEM accumulators */
       NDF_PREC_FP16 = 2 }; /* tcgen05 fp16 x fp16 -> fp32 (same speed, 3 more mantissa bits) */

/*
 * Model descriptor (host struct, device pointers inside).
 * Mirrors ModelSpec/NdfModel (model.py:29-142).  Two latent-grid kinds:
 *   grid_levels == 0: one dense anisotropic level, (rz, ry, rx, C) fp32, grid_res =
 *                     (rx, ry, rz) -- the BASELINE architecture;
 *   grid_levels >= 1: the reference HashGrid (encoding.py:120-178): tables
 *                     (levels, 2^grid_log2_table, C) fp32, isotropic per-level
 *                     resolution grid_level_res[l], dense index when res^3 <= 2^T,
 *                     XOR-prime hash otherwise (encoding.py:90-102).
 * Optional per-branch encoder MLPs (model.py:133-138, nn.py:124-137): enc_layers
 * affine layers [enc_widths], activation on all but the last; enc_nu == enc_mu for
 * shared models.  Encoders and hash grids run on the exact fp32 path only.
 */
typedef struct ndf_model_desc {
  int32_t fourier_octaves;        /* L: 6L Fourier features (encoding.py:22-51) */
  int32_t grid_channels;          /* C: latent channels (features_per_level) */
  int32_t grid_res[3];            /* latent resolution along x, y, z */
  int32_t merge;                  /* NDF_MERGE_* */
  int32_t activation;             /* NDF_ACT_* (hidden layers) */
  int32_t head;                   /* NDF_HEAD_* */
  int32_t n_layers;               /* decoder affine layers incl. output layer */
  int32_t widths[NDF_MAX_LAYERS + 1]; /* decoder widths [in, h1, ..., 1] */
  int32_t tc_format;              /* element type of params_tc: NDF_PREC_BF16 / NDF_PREC_FP16 */
  const float* grid_mu;           /* device (rz, ry, rx, C) fp32 */
  const float* grid_nu;           /* device; == grid_mu for shared models */
  const float* params_f32;        /* device: W0 (in x h1, row-major), b0, W1, b1, ...
                                     -- the NDFM/parameters() order (model.py:148-157) */
  const void* params_tc;          /* device: ndf_tc_pack() output, or NULL */
  /* --- ABI 2: reference HashGrid + encoder MLPs --- */
  int32_t grid_levels;            /* 0 = dense anisotropic level; >= 1 = HashGrid levels */
  int32_t grid_log2_table;        /* T: rows per level = 2^T (HashGrid only) */
  int32_t grid_level_res[NDF_MAX_LEVELS]; /* round(base * growth^l) (encoding.py:82-83) */
  int32_t enc_layers;             /* encoder affine layers (0 = identity passthrough) */
  int32_t enc_widths[NDF_MAX_LAYERS + 1]; /* [embed_dim, channels, ...] */
  const float* enc_mu;            /* device: encoder W0, b0, ... (parameters() order) */
  const float* enc_nu;            /* device; == enc_mu for shared models */
} ndf_model_desc;

int32_t ndf_abi_version(void);
const char* ndf_last_error(void);
/* number of SMs of the current device (grid sizing), or -1 */
int32_t ndf_device_sm_count(void);

/* ---- NDF query ------------------------------------------------------------ */

/* Bytes of the packed tensor-core parameter blob for this model (0 if the
 * model is outside the tcgen05 kernel's envelope: hidden width 128, input
 * width <= 128, >= 2 affine layers, output width 1). */
size_t ndf_tc_blob_bytes(const ndf_model_desc* m);
/* Pack params_f32 into the UMMA-canonical 16-bit blob of element type
 * m->tc_format (device kernel).
 * Replaces nothing in the reference: it is the "validate once at upload"
 * step (failure detection). */
int ndf_tc_pack(const ndf_model_desc* m, void* blob, size_t blob_bytes, void* stream);

/* Reference-to-all-vertices query over an output grid (x fastest).
 * Replaces service.reconstruct_field (service.py:46-84): the ref point is
 * embedded once, every query vertex once; writes out[v - v0] for flat
 * vertices v in [v0, v1).  ref_is_mu selects ROLE_MU / ROLE_NU
 * (service.py:63-80).  out may be device memory or page-locked host memory
 * (cudaHostAlloc / cudaHostRegister): the kernel then stores the field straight
 * into host RAM over PCIe, no separate D2H copy; pageable memory is rejected
 * with NDF_ERR_PARAMETER.  Same for ndf_query_points. */
int ndf_query_grid(const ndf_model_desc* m, double ref_x, double ref_y, double ref_z,
                   int32_t ref_is_mu, int32_t nx, int32_t ny, int32_t nz,
                   int64_t v0, int64_t v1, int32_t precision, float* out, void* stream);

/* ndf_query_grid plus the value range of what it writes (the headers of
 * /api/reconstruct, service.py:352-360, 406-410): stats (device, 3 x uint32) as for
 * ndf_field_export -- min / max keys of the non-NaN outputs and a NaN flag -- reduced
 * inside the query kernel's epilogue, so a response needs no second pass over the
 * field (which may already sit in page-locked host memory). */
int ndf_query_grid_stats(const ndf_model_desc* m, double ref_x, double ref_y, double ref_z,
                         int32_t ref_is_mu, int32_t nx, int32_t ny, int32_t nz,
                         int64_t v0, int64_t v1, int32_t precision, float* out,
                         uint32_t* stats, void* stream);

/* Paired / broadcast forward.  Replaces NdfModel.forward (model.py:179-189):
 * p_mu is (n_mu, 3) fp64 device, p_nu (n, 3); n_mu == 1 broadcasts. */
int ndf_query_points(const ndf_model_desc* m, const double* p_mu, int64_t n_mu,
                     const double* p_nu, int64_t n, int32_t precision, float* out,
                     void* stream);

/* Positional encoder alone: NdfModel.embed (model.py:169-177) -- [raw xyz |
 * Fourier(L) | latent] computed in fp64 and cast to fp32, bit-identical to the
 * reference.  branch 0 = the mu grid, 1 = the nu grid.  out is (n, E) fp32 row-major,
 * E = 3 + 6L + max(levels, 1) * C (device or pinned host memory).  The query kernels
 * fuse this step; these entry points serve callers that need the embedding itself.
 * ndf_embed_nodes: grid nodes [v0, v1) of nx x ny x nz (x fastest, measures.py:240-252).
 * ndf_embed_points: fp64 positions pos (n, 3), device memory. */
int ndf_embed_nodes(const ndf_model_desc* m, int32_t branch, int32_t nx, int32_t ny, int32_t nz,
                    int64_t v0, int64_t v1, float* out, void* stream);
int ndf_embed_points(const ndf_model_desc* m, int32_t branch, const double* pos, int64_t n,
                     float* out, void* stream);

/* Batched multi-reference query (BASELINE config 3; the loop in
 * service.matrix_reconstruct, service.py:97-125, batched): refs is (n_ref, 3)
 * fp64 device; out is fp16 (n_ref rows of ld_out halfs), row r holds
 * vertices [v0, v1) of ref r.  precision must be NDF_PREC_BF16 or NDF_PREC_FP16. */
int ndf_query_grid_multi(const ndf_model_desc* m, const double* refs, int32_t n_ref,
                         int32_t ref_is_mu, int32_t nx, int32_t ny, int32_t nz,
                         int64_t v0, int64_t v1, uint16_t* out_f16, int64_t ld_out,
                         void* stream);

/* ---- ground-truth estimators -------------------------------------------- */

/* Trilinear fp64 sampling of all members at B positions.
 * Replaces ensemble.sample_many (ensemble.py:130-167); X is one variable's
 * member-major (M, nz, ny, nx) fp32 block; out is (B, M) fp64. */
int ndf_sample_many(const float* X, int32_t M, int32_t nx, int32_t ny, int32_t nz,
                    const double* pos, int64_t B, double* out, void* stream);

/* sample_many over a column window: X holds node columns [col0, col0 + ld) of the
 * member-major ensemble with member rows ld elements apart (a V-slice on one GPU of a
 * sharded ensemble); every sampled lattice corner must lie inside the window.
 * ndf_sample_many == ndf_sample_many_ld with ld = nx*ny*nz, col0 = 0. */
int ndf_sample_many_ld(const float* X, int32_t M, int64_t ld, int64_t col0, int32_t nx,
                       int32_t ny, int32_t nz, const double* pos, int64_t B, double* out,
                       void* stream);

/* sample_many from the vertex-major copy Xv (V, M) of one variable (ndf_vertex_major):
 * the same fp64 trilinear samples bit for bit, but each lattice corner's M members are one
 * contiguous row, so a batch of scattered positions reads whole rows instead of one 32-byte
 * sector per member and corner -- the layout for large batches (training targets,
 * training.py:111-119). */
int ndf_sample_many_vm(const float* Xv, int32_t M, int32_t nx, int32_t ny, int32_t nz,
                       const double* pos, int64_t B, double* out, void* stream);

/* Ground-truth Pearson field in ONE streaming read of X: out[v - v0] = pearson of node
 * column v against ref_vec (fp64, M; device) for v in [v0, v1) -- measures.py:84-108 over
 * a node-aligned ground_truth_field (measures.py:286-295): fp64 shifted moments per
 * column, NaN where either side is degenerate, exactly 1.0 for a column equal to the
 * reference, clipped to [-1, 1].  X is a column window as for ndf_sample_many_ld
 * (col0 <= v0 <= v1 <= col0 + ld).  No standardised copy is built; the reference
 * statistics are computed on the device (no host round trip). */
int ndf_pearson_field(const float* X, int32_t M, int64_t ld, int64_t col0,
                      const double* ref_vec, int64_t v0, int64_t v1, float* out, void* stream);

/* Per-vertex standardisation (one-time prep of the Pearson GEMV):
 * Z[m][v] = (X[m][v] - mean_v) / sqrt(sum_m (X - mean_v)^2) in fp64 -> fp32;
 * norm[v] = that sqrt (0 marks a degenerate vertex).  Vertices [v0, v1). */
int ndf_zscore(const float* X, int32_t M, int64_t V, int64_t v0, int64_t v1,
               float* Z, float* norm, void* stream);

/* r[v] = sum_m Z[m][v] * z_ref[m] for v in [v0, v1), clipped to [-1, 1];
 * rows equal to z_ref -> exactly 1.0; degenerate (norm[v]==0 or ref_degenerate)
 * -> NaN.  Replaces measures.pearson_against (measures.py:84-108) over a
 * node-aligned ground_truth_field (measures.py:286-295). */
int ndf_pearson_gemv(const float* Z, const float* norm, int32_t M, int64_t V,
                     const float* z_ref, int32_t ref_degenerate, int64_t v0, int64_t v1,
                     float* out, void* stream);

/* Row-wise Pearson of fp64 rows: a is (B, M) or (1, M) when a_stride == 0,
 * b is (B, M); out (B,) fp64, NaN for degenerate rows, equal rows -> 1.0.
 * Replaces measures.pearson_rowwise (measures.py:111-133) and
 * pearson_against on sampled rows. */
int ndf_pearson_rows(const double* a, int64_t a_stride, const double* b, int32_t M,
                     int64_t B, double* out, void* stream);

/* Member-major (M, V) -> vertex-major (V, M) copy of one variable (layout for
 * pair lists). */
int ndf_vertex_major(const float* X, int32_t M, int64_t V, float* Xv, void* stream);

/* Pearson of vertex pairs (BASELINE config 4) from the vertex-major copy Xv:
 * out[p] = pearson(Xv[pa[p], :], Xv[pb[p], :]) in fp64 (NaN if degenerate).
 * Replaces the per-pair pearson_rowwise of training._targets (training.py:111-119). */
int ndf_pearson_pairs(const float* Xv, int32_t M, int64_t V, const int64_t* pa,
                      const int64_t* pb, int64_t n, double* out, void* stream);

/* KSG mutual information (variant 1, max-norm), measures.py:173-203.
 * jitter_r: (M,) fp64 = default_rng(0x5D17E3).random(M) - 0.5 (measures.py:168-170)
 * psi_tab:  (M,) fp64, psi_tab[n] = digamma(n + 1) (measures.py:136-165)
 * psi_k_plus_psi_m = digamma(k) + digamma(M)
 * Outputs: mi (n,) fp64 (may be NULL) and/or mi_f32 (n,) (may be NULL);
 * counts (n, 2, M) int32 n_x / n_y (may be NULL); *status_out (device int32)
 * receives 1 if any count was -1 (the reference raises there).
 *
 * ndf_ksg_ref_nodes: a = ref_vec (M,) fp64 device; b = X[:, v] for v in [v0, v1)
 *   (ground_truth_field(ksg_mi) over node positions, measures.py:296-314).
 * ndf_ksg_rows: a = A rows (stride a_stride, 0 = broadcast), b = B rows (fp64).
 * ndf_ksg_pairs: a = Xv[pa[p], :], b = Xv[pb[p], :] on the vertex-major copy
 *   (BASELINE config 4). */
int ndf_ksg_ref_nodes(const float* X, int32_t M, int64_t V, const double* ref_vec,
                      int64_t v0, int64_t v1, int32_t k, const double* jitter_r,
                      const double* psi_tab, double psi_k_plus_psi_m, double* mi,
                      float* mi_f32, int32_t* counts, int32_t* status_out, void* stream);
int ndf_ksg_rows(const double* a, int64_t a_stride, const double* b, int32_t M, int64_t B,
                 int32_t k, const double* jitter_r, const double* psi_tab,
                 double psi_k_plus_psi_m, double* mi, float* mi_f32, int32_t* counts,
                 int32_t* status_out, void* stream);
int ndf_ksg_pairs(const float* Xv, int32_t M, int64_t V, const int64_t* pa,
                  const int64_t* pb, int64_t n, int32_t k, const double* jitter_r,
                  const double* psi_tab, double psi_k_plus_psi_m, double* mi,
                  float* mi_f32, int32_t* counts, int32_t* status_out, void* stream);

/* ---- binary data plane ------------------------------------------------------ */

/* Body and value range of a field response -- /api/reconstruct and /api/diff
 * (service.py:392-416: grid.values.astype("<f4").tobytes(), _field_headers at
 * service.py:352-360).  dst[i] = a[i] (b == NULL) or a[i] - b[i] (fp32, difference_field,
 * service.py:87-94), clipped to [-1, 1] when clamp (np.clip: NaN stays NaN), for
 * i in [0, n); a / b on the device, dst device or page-locked host memory (the stores
 * then go straight over PCIe).  stats (device, 3 x uint32) receives the min and max of
 * the non-NaN values as order-preserving keys (key = bits ^ 0x80000000 for sign 0,
 * ~bits for sign 1; min key 0xffffffff and max key 0 when there is none) and
 * stats[2] = 1 if any value is NaN. */
int ndf_field_export(const float* a, const float* b, int64_t n, float* dst, uint32_t* stats,
                     int32_t clamp, void* stream);

/* ---- utilities ------------------------------------------------------------ */

/* Number of kernel launches this library issued on the calling thread since
 * the last reset (bench.py's gpu_launches claim). */
int64_t ndf_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* NDF_B200_H */

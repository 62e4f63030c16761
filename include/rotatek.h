/*
 * rotatek.h -- C ABI of librotatek.so, the B200 (sm_100a) hot path of RotateK
 * (arxiv 2605.19218, "rotation-based structured Key-channel pruning for VLM
 * KV caches").
 *
 * The three calls follow the paper's problem statement:
 * compress the Keys K in R^{N x d} of N visual tokens to r < d channels with
 * minimal perturbation of q_t K^T.
 *   rotatek_calibrate    = Alg. 1 (alg:rotatek-prefill) lines 1-5
 *                          and the basis choice with an exact
 *                          eigendecomposition (batched Jacobi), then top-r
 *                          select and delta_mu = (I - R_r R_r^T) mu.
 *   rotatek_compress_kv  = Alg. 1 line 14: K~ = K R_r, "stored in place of K".
 *   rotatek_decode_attn  = Alg. 2 (alg:rotatek-decode) for every
 *                          query head: q~ = q R_r, b = q . delta_mu,
 *                          scores (q~ K~^T + b)/sqrt(d) over the visual tokens
 *                          and q K_pt^T / sqrt(d) over the full-d prompt/text
 *                          tokens, softmax over the concatenation, weighted sum
 *                          of full-d values (App. C).
 *
 * Conventions for every call
 *   - A "unit" is one (batch element, KV head): u = b * H_kv + h_kv.  All
 *     per-unit tensors are laid out [U, ...] row-major and contiguous, so a
 *     shard of units is a pointer offset (u0 * per-unit stride).
 *   - Query head h of unit u is g = h - u*G (h_kv = floor(h / G)).
 *   - All tensor pointers are DEVICE pointers, 16-byte aligned.  Buffers are
 *     owned by the caller; the library allocates nothing and keeps no data
 *     state between calls (the only per-thread state is the error string, the
 *     launch count and the diagnostics hook of rotatek_debug_decode_trace;
 *     kernel attributes are set once per device).
 *   - Every call validates its arguments on the host, then only ENQUEUES work
 *     on `stream`: no synchronisation, no allocation, CUDA-graph capturable.
 *     Numerical problems are reported per unit on the device through `info`.
 *   - No C++ exception crosses the ABI.  A non-OK status leaves the outputs
 *     untouched; rotatek_last_error() gives a thread-local detail string.
 *   - Workspaces: ask rotatek_workspace_bytes().  The workspace must be
 *     ZERO-FILLED once before its first use (e.g. cudaMemset / torch.zeros);
 *     every call leaves its counter region zeroed again, so the same
 *     workspace can be reused (and graph-replayed) without re-zeroing.
 *     Concurrent calls on different streams need different workspaces.
 *     A decode workspace's counter region sits at its start and its size
 *     depends on `units` only, so one zeroed buffer serves every decode shape
 *     with the same units whose rotatek_workspace_bytes() it covers.
 */
#ifndef ROTATEK_H_
#define ROTATEK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ROTATEK_ABI_VERSION 3

typedef struct CUstream_st* rotatek_stream_t; /* == cudaStream_t; NULL = legacy default */

typedef enum {
  ROTATEK_OK = 0,
  ROTATEK_ERR_NULL = 1,        /* a required pointer is NULL                          */
  ROTATEK_ERR_DIMS = 2,        /* U<1, G<1, N<1, M<0, W<0, r not in [1,d], d invalid  */
  ROTATEK_ERR_ALIGN = 3,       /* a pointer is not 16-byte aligned                    */
  ROTATEK_ERR_WORKSPACE = 4,   /* workspace NULL or smaller than rotatek_workspace_bytes */
  ROTATEK_ERR_UNSUPPORTED = 5, /* no kernel for this (d, r, dtype) combination        */
  ROTATEK_ERR_CUDA = 6         /* a kernel launch failed (see rotatek_last_error)     */
} rotatek_status;

typedef enum { ROTATEK_BF16 = 0, ROTATEK_F32 = 1 } rotatek_dtype;

/* calibrate flags */
enum {
  ROTATEK_CENTER = 1u << 0,       /* subtract the per-channel mean mu.  Off:
                                     mu = 0, C = K^T K (north_star's literal wording)  */
  ROTATEK_QUERY_WEIGHT = 1u << 1, /* C_q = (sigma sigma^T) (.) C.  Off (or
                                     W == 0): sigma == 1, the K-only PCA arm   */
  ROTATEK_EIG_FP64 = 1u << 2,     /* run the whole Jacobi eigensolver in fp64 (always on for
                                     fp32 caches).  Default for bf16 caches: an fp32 Jacobi
                                     solve (d = 128: one-sided, on a pivoted-Cholesky factor
                                     of C_q) followed by one fp64 refinement step
                                     (B = V0^T C_q V0, lambda = diag B, V = V0 (I + W) with
                                     the first-order correction W_ij = B_ij / (B_jj - B_ii)),
                                     for d = 128 and r <= 64 on the r + 8 leading columns */
  ROTATEK_EIG_TWOSIDED = 1u << 3, /* d = 128, fp32 solve: use the two-sided packed-triangle
                                     Jacobi (A and V in shared memory) instead of the default
                                     one-sided (Hestenes) Jacobi on C_q with the columns in
                                     registers.  Either is followed by the fp64 refinement; the
                                     default re-solves with the two-sided kernel any unit whose
                                     C_q has a (near-)null column (info -2 internally)      */
  ROTATEK_SIMT_ONLY = 1u << 8,    /* use the CUDA-core (SIMT) kernels instead of the tcgen05
                                     tensor-core ones (A/B tests and benches)           */
  ROTATEK_DEFAULT_FLAGS = (1u << 0) | (1u << 1)
};

typedef enum { ROTATEK_OP_CALIBRATE = 0, ROTATEK_OP_DECODE = 1 } rotatek_op;

typedef struct {
  int32_t units;        /* U = B * H_kv  (>= 1)                                         */
  int32_t group;        /* G = H_q / H_kv (>= 1): 1 (LLaVA-NeXT MHA), 7 (Qwen2.5-VL)    */
  int32_t head_dim;     /* d: 16..256, multiple of 16                                   */
  int32_t rank;         /* r kept rotated channels: 1 <= r <= d                          */
  int32_t n_vis;        /* N >= 1 visual tokens per unit (after token pruning)          */
  int32_t n_text;       /* M >= 0 full-d prompt/text/generated tokens per unit          */
  int32_t q_window;     /* W >= 0 recent prefill queries per query head (paper: 32)     */
  rotatek_dtype dtype;  /* element type of K, V, Qw, q, K~, K_text, V_text              */
  int32_t text_stride;  /* tokens per unit in the K_text / V_text ALLOCATIONS (>= n_text;
                           0 => n_text, dense).  A capacity > n_text makes the full-d
                           segment appendable in place during generation (NEXT-2, Q18):
                           token m of unit u is at row u * text_stride + m.               */
} rotatek_dims;

/* Bytes of device workspace `op` needs for these dims (0 if dims are invalid). */
size_t rotatek_workspace_bytes(const rotatek_dims* dims, rotatek_op op);

/*
 * Alg. 1 steps 1-5 plus the basis choice and delta_mu:
 *   sigma_j = ||Q_W[:, j]||_2 over the G*W window rows of the unit
 *   mu      = (1/N) sum_n K_n                     (ROTATEK_CENTER, else 0)
 *   C       = (K - mu)^T (K - mu)                 (no 1/N)
 *   C_q     = (sigma sigma^T) (.) C               (ROTATEK_QUERY_WEIGHT, else C)
 *   C_q     = R diag(lambda) R^T                  (batched Jacobi: d = 128 one-sided on a
 *                                                  pivoted-Cholesky factor + fp64 refinement)
 *   keep    = the r largest lambda, ties -> lower solver index
 *   R_r     = R[:, keep] in ascending index order
 *   dmu     = mu - R_r (R_r^T mu), computed in fp64 from the STORED R_r
 * Inputs
 *   K   [U, N, d]      dims->dtype
 *   Qw  [U, G, W, d]   dims->dtype; may be NULL iff W == 0
 * Outputs (caller-allocated; nullable ones may be NULL)
 *   R        [U, d, r] fp32: RNE of the solver's eigenvectors to fp32.  Compress
 *            and decode must be given this same R (K~, q~ and delta_mu are all
 *            built from the stored values).
 *   dmu      [U, d] fp32 (zeros when !ROTATEK_CENTER)
 *   eigvals  [U, d] fp32, all eigenvalues in solver order (nullable).  The
 *            select step ranks exactly these fp32 values.
 *   keep_mask[U, ceil(d/32)] uint32, bit i%32 of word i/32 <=> channel i kept (nullable)
 *   keep_idx [U, r] int32 ascending (nullable)
 *   R_full   [U, d, d] fp32 full eigenbasis, columns in solver order (nullable; tests).
 *            Default solver (d = 128, r <= 64): the r + 8 leading columns carry the fp64
 *            refinement, the others the one-sided solver's basis (orthonormal to ~1e-7;
 *            ~1e-4 per entry for a unit re-solved by the two-sided kernel after a null
 *            C_q column)
 *   info     [U] int32: 0 ok; s > 0 not converged after s sweeps (results are
 *            still written; the environment variable ROTATEK_JACOBI_MAX_SWEEPS=<n>,
 *            read at every call, lowers the sweep caps for fault injection); -1
 *            non-finite input (R, dmu zero-filled, mask 0, idx -1) (nullable)
 * Errors: NULL, DIMS, ALIGN, WORKSPACE, UNSUPPORTED (d > 256), CUDA.
 */
rotatek_status rotatek_calibrate(const rotatek_dims* dims, uint32_t flags, const void* K,
                                 const void* Qw, float* R, float* dmu, float* eigvals,
                                 uint32_t* keep_mask, int32_t* keep_idx, float* R_full,
                                 int32_t* info, void* workspace, size_t workspace_bytes,
                                 rotatek_stream_t stream);

/*
 * The paper's default solver (NEXT-1): Alg. 1 lines 1-5 as in rotatek_calibrate, then the
 * Cholesky-QR subspace iteration of lines 6-13:
 *   V <- V0; T times { V <- C_q V; G <- V^T V; rho <- eps tr(G)/r; L <- chol(G + rho I);
 *                      V <- V L^{-T} };  R_r <- V;  dmu = mu - R_r R_r^T mu (from stored R_r)
 *   V0     [U, d, r] fp32 device: the start basis ("Sample V with i.i.d. N(0,1) entries",
 *          l.6) -- the random draw is an input, so results are reproducible
 *   iters  T (<= 0: 5);  ridge eps (< 0: 1e-6; unspecified in the paper)
 *   R      [U, d, r] fp32 out;  dmu [U, d] fp32 out
 *   ritz   [U, r] fp32 out (nullable): Rayleigh quotients R_j^T C_q R_j / R_j^T R_j
 *   info   [U] (nullable): 0, or -1 if a Cholesky pivot was not positive
 * There is no eigen-index selection here, so no head mask / kept indices are produced.
 * Errors: NULL, DIMS, ALIGN, WORKSPACE (rotatek_workspace_bytes(.., OP_CALIBRATE)),
 * UNSUPPORTED (d > 128 or r not in {4, 8, 16, 32, 64}), CUDA.
 */
rotatek_status rotatek_calibrate_subspace(const rotatek_dims* dims, uint32_t flags, const void* K,
                                          const void* Qw, const float* V0, int32_t iters,
                                          float ridge, float* R, float* dmu, float* ritz,
                                          int32_t* info, void* workspace, size_t workspace_bytes,
                                          rotatek_stream_t stream);

/*
 * Alg. 1 line 14: K~ = RNE_dtype(K R_r), over the UNCENTERED K.
 *   K      [U, N, d]  dims->dtype
 *   R      [U, d, r]  fp32 as written by rotatek_calibrate
 *   K_comp [U, N, r]  dims->dtype (output).  V is not touched: values keep
 *                     all d channels (App. C).
 * Errors: NULL, DIMS, ALIGN, UNSUPPORTED, CUDA.
 */
rotatek_status rotatek_compress_kv(const rotatek_dims* dims, const void* K, const float* R,
                                   void* K_comp, rotatek_stream_t stream);

/* Same, with flags: ROTATEK_SIMT_ONLY selects the CUDA-core kernel instead of the tcgen05
 * one (d = 128, bf16, r in {16, 32, 64, 128}: R split exactly into three bf16 terms, fp32
 * accumulation in TMEM).  Other flag bits are ignored. */
rotatek_status rotatek_compress_kv_ex(const rotatek_dims* dims, const void* K, const float* R,
                                      void* K_comp, uint32_t flags, rotatek_stream_t stream);

/* Same with a shared rotation (NEXT-3, offline calibrated variant): R is
 * [r_units, d, r] and unit u uses R[u % r_units] (r_units = H_kv: one rotation per kv head,
 * reused across the batch b, since u = b*H_kv + h).  r_units must divide units; 0 means
 * one rotation per unit (== rotatek_compress_kv_ex).  Errors as rotatek_compress_kv_ex,
 * plus DIMS for a bad r_units. */
rotatek_status rotatek_compress_kv_ex2(const rotatek_dims* dims, int32_t r_units, const void* K,
                                       const float* R, void* K_comp, uint32_t flags,
                                       rotatek_stream_t stream);

/*
 * Token selection fused into the prefill (NEXT-2; PAPER.md P:133-135 fig:inference_flow
 * "following visual token compression", P:597 FastV K = 2 / VisionZip survivors; reading
 * Q20: the rotation is calibrated on the surviving visual tokens only).
 * Logical visual tokens of unit u: t = 0 .. n_u - 1, where
 *   n_u = n_vis_u ? clamp(n_vis_u[u], 0, dims->n_vis) : dims->n_vis
 * (n_vis_u: [U] int32 device, a padded batch of requests with different image-token counts),
 * and token t's key row is
 *   K[u][tok_idx[u * n_vis + t]]   with K [U, n_src, d]        if tok_idx != NULL
 *                                  (tok_idx [U, n_vis] int32 device: the survivors' positions
 *                                   in the unpruned cache, e.g. ascending FastV indices),
 *   K[u][t]                        with K [U, n_vis, d]        otherwise.
 * The kernels gather those rows while loading (the producer warp's cp.async copies write the
 * swizzled tile the tensor cores read): no compacted copy of K is made.  Rows past n_u, and
 * out-of-range indices, read as zero keys and are never loaded.
 *
 * rotatek_calibrate_tokens: rotatek_calibrate (Alg. 1) over the n_u logical tokens of each unit
 *   (mu = column sum / n_u, C = S - n_u mu mu^T).  n_u must be >= 1 per unit (a unit with no
 *   token has an undefined rotation).
 * rotatek_compress_kv_tokens: K_comp [U, n_vis, r] with K_comp[u][t] = RNE(K_row(t) R_u) for
 *   t < n_u and exactly 0 for n_u <= t < n_vis (decode with rotatek_decode_attn_varlen and the
 *   same n_vis_u reads only the first n_u rows).
 * Both need the tensor-core path (bf16, d = 128; else ROTATEK_ERR_UNSUPPORTED), 16-byte aligned
 * token arrays (ROTATEK_ERR_ALIGN) and n_src >= 1 with a token list (ROTATEK_ERR_DIMS); other
 * arguments and errors as rotatek_calibrate / rotatek_compress_kv_ex2.
 */
rotatek_status rotatek_calibrate_tokens(const rotatek_dims* dims, uint32_t flags, const void* K,
                                        int32_t n_src, const int32_t* tok_idx, const int32_t* n_vis_u,
                                        const void* Qw, float* R, float* dmu, float* eigvals,
                                        uint32_t* keep_mask, int32_t* keep_idx, float* R_full,
                                        int32_t* info, void* workspace, size_t workspace_bytes,
                                        rotatek_stream_t stream);
rotatek_status rotatek_compress_kv_tokens(const rotatek_dims* dims, int32_t r_units, const void* K,
                                         int32_t n_src, const int32_t* tok_idx, const int32_t* n_vis_u,
                                         const float* R, void* K_comp, rotatek_stream_t stream);

/*
 * Alg. 2 for all U*G query heads in one launch:
 *   q~ = q R_r ; b = q . dmu
 *   s_vis[n] = (q~ . K~[n] + b) * scale          n < N   (rotated, r channels)
 *   s_pt[m]  = (q . K_text[m]) * scale           m < M   (full d channels)
 *   out = softmax([s_vis; s_pt]) [V; V_text]     (fp32 accumulation, exact
 *         online-softmax split-K merge, epsilon = 0)
 *   q       [U, G, d]  dims->dtype   (== [B, H_q, d] since h = u*G + g)
 *   K_comp  [U, N, r]  dims->dtype
 *   V       [U, N, d]  dims->dtype
 *   R       [U, d, r]  fp32 (the calibrate output)
 *   dmu     [U, d]     fp32 (may be NULL: b = 0)
 *   K_text, V_text [U, M, d] dims->dtype, NULL iff M == 0
 *   softmax_scale <= 0 selects 1/sqrt(d) -- NOT 1/sqrt(r) (Alg. 2 line 3)
 *   out     [U, G, d]  fp32 (output)
 * Errors: NULL, DIMS, ALIGN, WORKSPACE, CUDA.
 */
rotatek_status rotatek_decode_attn(const rotatek_dims* dims, const void* q, const void* K_comp,
                                   const void* V, const float* R, const float* dmu,
                                   const void* K_text, const void* V_text, float softmax_scale,
                                   float* out, void* workspace, size_t workspace_bytes,
                                   rotatek_stream_t stream);

/*
 * Same as rotatek_decode_attn with an explicit split-K factor over the token
 * axis (splits <= 0: automatic, sized to fill the 148 SMs).  The result is
 * the same up to fp32 re-association for every split count (App. C "standard
 * online-softmax merge").  `kernel` forces the implementation:
 * 0 auto, 1 the generic kernel (any d, r, G), 2 the TMA-pipelined CUDA-core streaming
 * kernel, 3 the tensor-core CTA-ring kernel (one CTA per unit, per equal unit piece or per
 * SM, each streaming a shared TMA ring; bf16, d = 128, r in {32, 64}, G in {1, 2, 4, 7, 8};
 * unit pieces merged in slot order through distributed shared memory (a thread-block
 * cluster per unit) or by their last contributor, so bit-reproducible; the automatic choice
 * for G >= 2 and for G = 1 batches of <= 2 units per SM), 4 the streaming kernels with work
 * stealing
 * (bf16, d = 128, r = 32, G in {1, 7}; merges in arrival order, so results are
 * reproducible to fp32 re-association, not bit for bit), 5 the per-warp tensor-core GQA
 * kernel of ABI version 1 (same shapes as 3) -- UNSUPPORTED if the shape has none.  Used
 * by tests and benches.
 * OR ROTATEK_DECODE_OVERLAP into `kernel` to launch the streaming kernels as programmatic
 * dependents of the preceding work on `stream` (griddepcontrol): they start streaming the
 * cache while that work finishes and wait for it only before reading q and the workspace.
 * Contract: every input except q (K_comp, V, K_text, V_text, R, dmu) is complete before
 * the PRECEDING kernel starts; q may be produced by it.  (Every streaming decode lets the
 * next kernel launch early; a next kernel launched as a programmatic dependent must
 * griddepcontrol.wait before reading out, as CUDA requires.)
 */
#define ROTATEK_DECODE_OVERLAP 0x100
rotatek_status rotatek_decode_attn_ex(const rotatek_dims* dims, const void* q,
                                      const void* K_comp, const void* V, const float* R,
                                      const float* dmu, const void* K_text, const void* V_text,
                                      float softmax_scale, float* out, void* workspace,
                                      size_t workspace_bytes, int32_t splits, int32_t kernel,
                                      rotatek_stream_t stream);

/* Same with a shared rotation: R [r_units, d, r] and dmu [r_units, d]; unit u uses index
 * u % r_units (r_units divides units; 0 = one per unit).  See rotatek_compress_kv_ex2. */
rotatek_status rotatek_decode_attn_ex2(const rotatek_dims* dims, int32_t r_units, const void* q,
                                       const void* K_comp, const void* V, const float* R,
                                       const float* dmu, const void* K_text, const void* V_text,
                                       float softmax_scale, float* out, void* workspace,
                                       size_t workspace_bytes, int32_t splits, int32_t kernel,
                                       rotatek_stream_t stream);

/*
 * Variable-length units (a batch of VLM requests with different image-token / prompt
 * counts, P:133-135 and NEXT-2; Alg. 2 per unit over that unit's own tokens): as
 * rotatek_decode_attn_ex2 over caches padded to dims->n_vis / n_text rows per unit, with
 *   n_vis_u  [U] int32 device (or NULL = n_vis for every unit): unit u attends to visual
 *            rows [0, n_vis_u[u]) of K_comp[u] / V[u] only; values clamp to [0, n_vis]
 *   n_text_u [U] int32 device (or NULL = n_text): text rows [0, n_text_u[u]) of K_text[u]
 * Padding rows are streamed but masked out of the softmax (weight exactly 0) and out of
 * the P.V product (the tensor-core kernels zero masked V rows in shared memory), so they
 * may hold anything, NaN/Inf included.
 * A unit with no valid token at all has an undefined (NaN) output.  Units of a real batch
 * would usually be packed by length order instead of padded; padding keeps one uniform
 * [U, N, .] layout, so HBM traffic and time follow the padded sizes.
 * Errors: as rotatek_decode_attn_ex2; ALIGN also for the length arrays.
 */
rotatek_status rotatek_decode_attn_varlen(const rotatek_dims* dims, int32_t r_units,
                                          const int32_t* n_vis_u, const int32_t* n_text_u,
                                          const void* q, const void* K_comp, const void* V,
                                          const float* R, const float* dmu, const void* K_text,
                                          const void* V_text, float softmax_scale, float* out,
                                          void* workspace, size_t workspace_bytes,
                                          int32_t splits, int32_t kernel,
                                          rotatek_stream_t stream);

/*
 * Calibration statistics, accumulated on the device (NEXT-3 offline calibrated rotation,
 * P:588 "precomputed from calibration data and reused across samples"; and the
 * calibration half of token-sharded prefill).  The fp64 state holds the sums
 * behind Alg. 1 l.1-5, one entry of ROTATEK_STATE_DOUBLES(d) doubles per state unit s:
 *     S [d][d] = sum_n k_n k_n^T  |  colsum [d] = sum_n k_n  |
 *     sigma2 [d] = sum over query windows of q_j^2 (Q_W, pooled as in rotatek_calibrate) |
 *     count = number of tokens  |  one pad double
 * rotatek_calib_accumulate ADDS unit u's keys K[u] (and window Qw[u] if QUERY_WEIGHT and
 * q_window > 0) into entry u % state_units (state_units divides units; ascending u, so the
 * result is deterministic).  Zero the state once before the first call.  For token
 * sharding each rank accumulates its slice and the states are all-reduced (summed).
 * Errors: NULL, DIMS (also: bad state_units), ALIGN, WORKSPACE (size = rotatek_workspace_
 * bytes(dims, CALIBRATE)), UNSUPPORTED (d > 128), CUDA.
 */
#define ROTATEK_STATE_DOUBLES(d) ((size_t)(d) * (size_t)(d) + 2 * (size_t)(d) + 2)
rotatek_status rotatek_calib_accumulate(const rotatek_dims* dims, uint32_t flags, const void* K,
                                        const void* Qw, int32_t state_units, double* state,
                                        void* workspace, size_t workspace_bytes,
                                        rotatek_stream_t stream);

/*
 * Alg. 1 from an accumulated state (dims->units = number of state entries; n_vis,
 * q_window ignored): mu = colsum / count (CENTER, else 0), C = S - count mu mu^T,
 * C_q = (sigma sigma^T) (.) C with sigma = sqrt(sigma2) (QUERY_WEIGHT, else 1), then the
 * eigensolver, top-r select and delta_mu exactly as rotatek_calibrate (same outputs,
 * layouts, flags EIG_FP64, errors; workspace: rotatek_workspace_bytes with n_vis = 1).
 */
rotatek_status rotatek_calibrate_from_state(const rotatek_dims* dims, uint32_t flags,
                                            const double* state, float* R, float* dmu,
                                            float* eigvals, uint32_t* keep_mask,
                                            int32_t* keep_idx, float* R_full, int32_t* info,
                                            void* workspace, size_t workspace_bytes,
                                            rotatek_stream_t stream);

/*
 * Token-sharded decode (when there are fewer units than GPUs, the token axis
 * is split across ranks).  The online-softmax split of Alg. 2 (App. C "standard online-
 * softmax merge") is exact, so each rank runs Alg. 2 over ITS token slice -- its own
 * [U, N_p, r] / [U, N_p, d] cache shard (N_p >= 1) and [U, M_p, d] text shard, with the
 * replicated q, R_r and dmu -- and returns the un-normalised state instead of out:
 *   part [U, G, d+2] fp32 device:  acc[d] | m | l   per (unit, query head), where with
 *   z_n = s_n * log2(e) the base-2 logit of token n (s_n the 1/sqrt(d)-scaled score of
 *   Alg. 2 l.3-4):  m = max_n z_n,  l = sum_n 2^(z_n - m),  acc = sum_n 2^(z_n - m) V[n].
 * Same arguments, workspace, layouts and errors as rotatek_decode_attn (out -> part).
 */
rotatek_status rotatek_decode_attn_partial(const rotatek_dims* dims, const void* q,
                                           const void* K_comp, const void* V, const float* R,
                                           const float* dmu, const void* K_text,
                                           const void* V_text, float softmax_scale, float* part,
                                           void* workspace, size_t workspace_bytes,
                                           rotatek_stream_t stream);

/*
 * Merge P token-shard states (e.g. gathered with an all-gather) into the attention output:
 *   parts [P, U, G, d+2] fp32 device (shard-major, rotatek_decode_attn_partial layout)
 *   out   [U, G, d] fp32 device:  out = sum_p 2^(m_p - M) acc_p / sum_p 2^(m_p - M) l_p,
 *         M = max_p m_p  (shards combined in index order: deterministic).
 * Errors: DIMS, NULL, ALIGN, CUDA.
 */
rotatek_status rotatek_merge_partials(int32_t units, int32_t group, int32_t head_dim,
                                      int32_t nparts, const float* parts, float* out,
                                      rotatek_stream_t stream);

/*
 * Token pruning input (NEXT-2; FastV / VisionZip keep a scattered subset of the
 * visual tokens, and calibration runs on the survivors only, Q20).  Compacts rows:
 *   dst[u][j] = src[u][keep_idx[u][j]],  keep_idx [U, n_keep] int32 device (indices into
 *   [0, n_src), any order; ascending keeps the original token order), src [U, n_src, ...],
 *   dst [U, n_keep, ...] with row_bytes per token (d * sizeof(dtype): K, V, K~ ...).
 * Apply to K (before rotatek_calibrate / rotatek_compress_kv) and V (for the decode).
 * err (nullable) is set to 1 if an index is out of range (that row is zero-filled).
 * Errors: DIMS (row_bytes must be a positive multiple of 16), NULL, ALIGN, CUDA.
 */
rotatek_status rotatek_gather_tokens(int32_t units, int32_t n_src, int32_t n_keep,
                                     int32_t row_bytes, const int32_t* keep_idx,
                                     const void* src, void* dst, int32_t* err,
                                     rotatek_stream_t stream);

/*
 * The top-r select + compaction step on its own (the selection half of
 * rotatek_calibrate, exposed so that it can be checked bit-exactly on given
 * eigenvalue arrays, including adversarial ties):
 *   eigvals  [U, d] fp32 device      keep = r largest, ties -> lower index
 *   keep_mask[U, ceil(d/32)] uint32   keep_idx [U, r] int32 ascending
 *   info     [U] int32: 0, or -1 if a NaN is present (mask 0, idx -1)
 * Errors: NULL, DIMS, ALIGN, CUDA.
 */
rotatek_status rotatek_select_topr(int32_t units, int32_t head_dim, int32_t rank,
                                   const float* eigvals, uint32_t* keep_mask, int32_t* keep_idx,
                                   int32_t* info, rotatek_stream_t stream);

/* Number of kernel launches the last successful call on this thread enqueued. */
int rotatek_last_launch_count(void);

/*
 * Diagnostics only (not part of the hot path): install a device buffer of
 * >= 8 * (number of streaming warps) uint64 that subsequent decode launches of the
 * streaming kernels fill with per-warp %globaltimer stamps (start, after the query
 * rotation, first tile ready, loop end, end) and counters (tiles, units).  NULL
 * uninstalls.  The buffer is caller-owned; the library keeps only the pointer,
 * per CALLING THREAD (launches from other threads are not traced).
 */
void rotatek_debug_decode_trace(void* device_buffer);

const char* rotatek_status_string(rotatek_status status);
const char* rotatek_last_error(void); /* thread-local detail for the last non-OK return */
int rotatek_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ROTATEK_H_ */

/*
 * ct.h -- C ABI of libct, the B200 (sm_100a) implementation of the LEVER 3-D
 * per-frame segmentation hot path (arXiv 1407.2089; reference package
 * "clonetrack", ref = /root/reference/pkg/src/clonetrack).
 *
 * The reference has no FFI: its boundary is the Python module API of
 * ref denoise.py and ref segment.py.  Each entry point below names the
 * reference function(s) it replaces; the Python layer in
 * paper_1407_2089_b200/{denoise,segment}.py keeps the reference names,
 * signatures and exceptions and calls these through ctypes.
 *
 * Conventions
 *  - Volumes are C-contiguous (nx, ny, nz), z fastest (ref imaging.py:3-6);
 *    linear index p = (i*ny + j)*nz + k.
 *  - Every pointer argument is DEVICE memory unless stated; the caller owns
 *    all buffers (no allocation inside libct); work buffers are sized by
 *    ct_workspace_bytes().
 *  - `stream` is a cudaStream_t passed as void*; every call is stream-ordered,
 *    asynchronous and re-entrant (no global mutable state).
 *  - Return value: CT_OK or a CT_ERR_* code; ct_last_error() gives the text
 *    (thread-local).  CT_ERR_PARAM maps to ref errors.py:16 ParameterError.
 *    Data-dependent outcomes (degenerate histogram, empty mask) are reported
 *    in device-side result words so that calls never synchronise.
 */
#ifndef CT_H
#define CT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element types */
#define CT_U8 1
#define CT_U16 2
#define CT_I32 4
#define CT_F64 8

/* status codes */
#define CT_OK 0
#define CT_ERR_PARAM 1       /* ParameterError (ref errors.py:16)              */
#define CT_ERR_CUDA 3        /* CUDA launch/runtime failure                    */
#define CT_ERR_UNSUPPORTED 4 /* dtype / size outside what a kernel supports    */
#define CT_ERR_IO 5          /* unreadable / unsupported image file: ManifestError
                              * "failed to read image" (ref imaging.py:213-216) */

/* ct_otsu result words (int64, device): */
#define CT_OTSU_T 0        /* threshold t (segment.py:150)                      */
#define CT_OTSU_STATUS 1   /* 0 ok, 1 empty mask (all mass in bin 0), 2 degenerate */
#define CT_OTSU_NBINS 2    /* 256 or 65536 (segment.py:162) or the given length */
#define CT_OTSU_NONZERO 3  /* number of non-empty bins                           */
#define CT_OTSU_WORDS 4

/* per-frame counters (int64, device) written by ct_ccl26 / ct_cell_table */
#define CT_CNT_FG 0          /* foreground voxels                              */
#define CT_CNT_COMPONENTS 1  /* 26-connected components                        */
#define CT_CNT_KEPT 2        /* components passing the volume filter            */
#define CT_CNT_KEPT_VOXELS 3 /* voxels in kept components                       */
#define CT_CNT_OVERFLOW 4    /* != 0: component capacity exceeded (retry larger)*/
#define CT_CNT_WORDS 8

/* one row of the per-cell table (ct_cell_table), 16 x 8 bytes, id order */
typedef struct ct_cell {
    int64_t id;            /* id_start + rank by (-count, root) (segment.py:257-264) */
    int64_t count;         /* voxels                                            */
    int64_t root;          /* min C-order linear index = first voxel            */
    int64_t bbox_lo[3];    /* min (i, j, k)                                     */
    int64_t bbox_hi[3];    /* max (i, j, k)                                     */
    int64_t intensity_sum; /* sum of integer intensities (0 if none given)     */
    double centroid_um[3]; /* row-sequential mean of idx*spacing (segment.py:260) */
    double volume_um3;     /* count * voxel_volume (segment.py:267)             */
    int64_t voxel_offset;  /* start of this cell's voxels in the voxel list     */
    double mean_intensity; /* intensity_sum / count as float64 = numpy
                            * intensity[voxels].mean() (north star's per-cell
                            * mean intensity; NaN if no intensity given)      */
} ct_cell;

const char *ct_version(void);
const char *ct_last_error(void);

/* Stream-ordered fill of `bytes` bytes at dst with the byte `value` (the
 * "caller zeroes" step of the accumulating histogram outputs, and the label
 * volume's -1 background, without a framework memset). */
int ct_memset(void *dst, int value, int64_t bytes, void *stream);

/* Bytes of device workspace an entry point needs for an (nx,ny,nz) volume.
 * which: 0 ct_gaussian_residual, 1 ct_closing (radius>1), 2 ct_ccl26 +
 * ct_cell_table (per component capacity `cap`), 3 ct_edt, 4 ct_mrf. */
size_t ct_workspace_bytes(int which, int64_t nx, int64_t ny, int64_t nz, int64_t cap);

/* K1 -- ref denoise.py:84-86: bg = gaussian_filter(float64(raw), sigma,
 * mode='nearest', truncate=4) (3 separable passes, axis 0->1->2, scipy's
 * symmetric accumulation order, no FMA); residual = max(raw - bg, 0).
 * w = concatenated one-sided weights w_x[0..rx], w_y[0..ry], w_z[0..rz]
 * (DEVICE), r < 0 skips an axis (sigma <= 1e-15).  Outputs (any may be
 * NULL): bg (f64), residual (f64), q = rint(residual) in q_dtype (U8/U16,
 * integer raw only).  work: ct_workspace_bytes(0,...). */
int ct_gaussian_residual(const void *raw, int raw_dtype, int64_t nx, int64_t ny, int64_t nz,
                         const double *w, int rx, int ry, int rz, void *work,
                         double *bg_out, double *residual_out, void *q_out, int q_dtype, void *stream);

/* K1 fast path of the fused pipeline: q = rint(max(raw - bg, 0)) for U8/U16
 * raw, CERTIFIED exact.  U8 volumes with nz in {32, 64, 96}, rx, ry <= 64 and
 * rz <= 64 run on the tensor cores (tcgen05 int8 MMA: taps as 35-bit
 * integers in 8-bit limbs, intermediates as 32-bit fixed point, exact int32
 * accumulation; k_gauss_tc.cu); other inputs accumulate bg by FP64 FMA.
 * Voxels whose residual lies within the path's rigorous error bound (vs
 * scipy's float64 result) of a half-integer are listed in fix (device: [0]
 * count, [1] overflow, [2..2+fix_cap) linear indices) and recomputed in
 * scipy's exact order by a fix-up kernel, so q is bit-identical to
 * ct_gaussian_residual's.  When the list overflows (fix[1] != 0) the whole
 * volume is recomputed in scipy's order in the same stream (no host round
 * trip), so q is exact in every case.  eps_override > 0 replaces the bound
 * (tests force the fix-up path with it).  path: 0 auto (tensor cores where
 * the shape fits), 1 FP64 FMA only, 2 tensor cores only (CT_ERR_UNSUPPORTED
 * when the shape does not fit).  Falls back to the exact path when no tiled
 * kernel applies.  work: ct_workspace_bytes(0,...).
 * (Replaces the q = rint(denoise_cell_channel(raw)) part of ref
 * denoise.py:84-88 on the fused path.) */
int ct_gaussian_q(const void *raw, int dtype, int64_t nx, int64_t ny, int64_t nz, const double *w, int rx, int ry,
                  int rz, void *work, void *q_out, unsigned long long *fix, int64_t fix_cap, double eps_override,
                  int path, void *stream);

/* Which arithmetic ct_gaussian_q uses for this shape and path argument:
 * 2 tensor cores, 1 FP64 FMA (both certified; informational). */
int ct_k1_path(int dtype, int64_t nx, int64_t ny, int64_t nz, int rx, int ry, int rz, int path);

/* float64 copy of a U8/U16/F64 volume (ref denoise.py:84, :158 astype). */
int ct_to_f64(const void *in, int dtype, int64_t n, double *out, void *stream);

/* K2 -- ref denoise.py:87-88: median_filter(size=2r+1, mode='nearest').
 * in/out dtype U8, U16 or F64.  hist (nullable, 65536 uint64, accumulated,
 * caller zeroes) receives the fused histogram of the output
 * (segment.py:154-163) for integer dtypes. */
int ct_median(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz, int radius, void *out,
              uint64_t *hist, void *stream);

/* ref segment.py:154-163: histogram of clip(rint(v), 0, 65535) into 65536
 * uint64 bins (accumulated; caller zeroes). */
int ct_histogram(const void *in, int dtype, int64_t n, uint64_t *hist, void *stream);

/* K3 -- ref segment.py:99-151 otsu_threshold (with the reference's int64
 * wrap in the float prefilter and exact ~380-bit tie-break) plus the
 * degenerate rules of binarize (segment.py:192-204).  nbins > 0 uses the
 * histogram as given (otsu_threshold on a caller histogram); nbins == 0
 * picks 256 or 65536 from the content (intensity_histogram).  result: int64
 * [CT_OTSU_WORDS] on device. */
int ct_otsu(const uint64_t *hist, int64_t nbins, int64_t *result, void *stream);

/* K4 -- ref segment.py:204 + :175-189: mask = rint(v) > t (t from a ct_otsu
 * result; status 1 -> empty mask), then ball closing of radius r on the
 * infinite zero domain.  r == 0 skips the closing.  work: radius >= 1 takes
 * ct_workspace_bytes(1,...) (r == 1 runs bit-packed when nz <= 64 and
 * nz % 4 == 0; without work it uses a byte-tile kernel; r > 1 requires it).
 * otsu_result == NULL thresholds at t_host. */
int ct_threshold_close(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz,
                       const int64_t *otsu_result, int64_t t_host, int radius, uint8_t *mask_out,
                       void *work, void *stream);

/* K4 for the fused cell path: ct_threshold_close with radius 1 that also
 * writes the closed mask as packed z-rows -- rows_out[(i*ny + j)*W ...] with
 * W = 1 uint64 (nz <= 64) or 2 (nz <= 128, one 128-bit word, low half first),
 * bit k = voxel (i,j,k) -- for ct_ccl26_rows.  mask_out may be NULL (no byte
 * mask).  Requires nz <= 128, nz % 4 == 0, 16-byte aligned outputs and the
 * ct_workspace_bytes(1,...) work area (else CT_ERR_UNSUPPORTED / PARAM).
 * Same reference semantics as ct_threshold_close (segment.py:175-204). */
int ct_threshold_close_rows(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz,
                            const int64_t *otsu_result, int64_t t_host, uint8_t *mask_out, void *rows_out,
                            void *work, void *stream);

/* ref segment.py:175-189 on a given mask (0/1 bytes). */
int ct_closing(const uint8_t *mask, int64_t nx, int64_t ny, int64_t nz, int radius, uint8_t *out,
               void *work, void *stream);

/* K5 -- ref segment.py:254 ndimage.label(mask, ones((3,3,3))): labels[p] =
 * min linear index of p's 26-connected component, -1 on background;
 * fg_list receives every foreground index (capacity nx*ny*nz);
 * counters: int64[CT_CNT_WORDS] (zeroed by the call). */
int ct_ccl26(const uint8_t *mask, int64_t nx, int64_t ny, int64_t nz, int32_t *labels, int32_t *fg_list,
             int64_t *counters, void *stream);

/* K5 on packed z-rows (ct_threshold_close_rows output, nz <= 128): same
 * outputs as ct_ccl26 (ref segment.py:254) without re-reading a byte mask.
 * flags: CT_LABELS_PREFILLED = labels already hold -1 everywhere (the caller
 * filled them); CT_LABELS_RESET = labels hold -1 everywhere except at
 * fg_list[0 .. counters[CT_CNT_FG]) as left by the previous ct_ccl26_rows /
 * ct_cell_table calls on these same buffers (a frame loop: the call resets
 * just those voxels, O(foreground) instead of O(volume)); else the call
 * fills labels with -1. */
#define CT_LABELS_PREFILLED 1
#define CT_LABELS_RESET 2
int ct_ccl26_rows(const void *rows, int64_t nx, int64_t ny, int64_t nz, int32_t *labels, int32_t *fg_list,
                  int64_t *counters, int flags, void *stream);

/* K6 -- ref segment.py:242-276 detections_from_mask minus the hull: volume
 * filter count*((dx*dy)*dz) >= min_volume (float64), rank by (-count, root),
 * ids from id_start, C-order voxel lists, row-sequential centroids, bbox,
 * intensity sums and mean intensities.  On return labels[p] = rank (0-based) of p's kept cell,
 * else -1 (canonical label volume); table[rank] filled for rank < n_kept;
 * voxels[] = concatenated C-order linear indices (capacity nx*ny*nz).
 * intensity: optional U8/U16 volume for intensity_sum.  cap = component
 * capacity of `work` (ct_workspace_bytes(2, ..., cap)). */
int ct_cell_table(int32_t *labels, int64_t nx, int64_t ny, int64_t nz, const int32_t *fg_list,
                  int64_t *counters, const void *intensity, int intensity_dtype, double dx, double dy,
                  double dz, double min_volume_um3, int64_t id_start, int64_t cap, void *work,
                  ct_cell *table, int32_t *voxels, void *stream);

/* Results on-disk format -- ref segment.py:321-337
 * encode_voxel_runs per detection (session.py:668): z-runs [i, j, k0, length]
 * of every kept cell's C-order voxel list from ct_cell_table.  runs: int32
 * [4 * cap_runs]; run_offset: int64[CT kept cells + 1] (cell r's runs are
 * [run_offset[r], run_offset[r+1])); nruns: int64[2] = total runs, overflow
 * (runs not written when the total exceeds cap_runs). */
int ct_voxel_runs(const int32_t *voxels, const ct_cell *table, const int64_t *counters, int64_t ny, int64_t nz,
                  int64_t cap_runs, int32_t *runs, int64_t *run_offset, int64_t *nruns, void *stream);

/* K7 -- ref denoise.py:92-195 (MRF vessel denoise).  Computes on device,
 * without synchronising: delta = intensity_step (denoise.py:135-144),
 * sigma_hat = estimate_noise_variance (denoise.py:92-114, numpy pairwise
 * summation order reproduced exactly), and the first proposal's distance
 * ||I0 + delta*sign(S) - I0|| (denoise.py:172-176).  state (device, 9
 * doubles): [0] delta [1] sigma_hat [2] sigma status (1: < 2 interior voxels,
 * sigma 0) [3] voxels whose sign sum is non-zero [4] first-step norm
 * [5] decision: 0 = stop with 0 iterations (output = input as float64),
 * 1 = iterate (host loop over ct_mrf_step), 2 = constant grid (delta 0:
 * denoise.py:160-161 returns the input itself).  hist: 65536 zeroed uint64,
 * required for U8/U16 input, receives the input's histogram (= the
 * histogram segment_vessel_channel needs when the decision is 0).
 * work: ct_workspace_bytes(4, nx, ny, nz, dtype). */
int ct_mrf(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz, void *work, double *state,
           uint64_t *hist, void *stream);

/* ct_mrf for the fused pipeline: the first-step decision is certified
 * without the exact sigma_hat when ||delta sign(S)|| = delta sqrt(nnz) exceeds
 * the upper bound sqrt(mean(L^2))/sqrt(42) >= std(L)/sqrt(42) of the
 * reference's estimate (denoise.py:100-114, 172-176), with a 2^-20 relative
 * margin; state[1] is then NaN and state[2] = 2 (sigma skipped).  Otherwise
 * (and for non-u8 input) the state equals ct_mrf's. */
int ct_mrf_decide(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz, void *work, double *state,
                  uint64_t *hist, void *stream);

/* One synchronous MRF iteration (denoise.py:172): next = cur + delta *
 * sign(S(cur)); cur == NULL means the input.  out2 (device): [0] ||next -
 * input|| (pairwise order; exact for integer data), [1] moved voxels.
 * delta is read from state[0] of ct_mrf. */
int ct_mrf_step(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz, const double *cur,
                const double *state, double *next, void *work, double *out2, void *stream);

/* ref denoise.py:117-132 _neighbor_sign_sum (edge-replicated six-direction
 * sign sum) -> int64 per voxel. */
int ct_sign_sum(const void *in, int dtype, int64_t nx, int64_t ny, int64_t nz, int64_t *out, void *stream);

/* K8 -- ref segment.py:292-304 distance_transform_edt(~mask, sampling):
 * Euclidean distance (um) to the nearest foreground voxel, separable
 * lower-envelope passes carrying feature coordinates; out: F64.  Caller
 * handles the empty mask (segment.py:296-297). */
int ct_edt(const uint8_t *mask, int64_t nx, int64_t ny, int64_t nz, double dx, double dy, double dz,
           void *work, double *out, void *stream);

/* Measurement helper (bench.py roofline): 148*8 CTAs x 256 threads, each
 * running 8 independent DMUL+DADD chains for `iters` iterations (16 FP64
 * ops per iteration); out holds 148*8*256 doubles. */
int ct_fp64_peak(double *out, int iters, void *stream);

/* Synthetic frames, bit-identical to oracle/ct_oracle.c. */
int ct_synth_frame(void *out, int dtype, int64_t nx, int64_t ny, int64_t nz, uint64_t seed, int64_t vmax,
                   const int64_t *balls, int64_t n_balls, int64_t amp_ball, const int64_t *tubes,
                   int64_t n_tubes, int64_t amp_tube, void *stream);

/* ---- Ingest ------------------------------------------
 * ref imaging.py:211-220 load_tiff_volume = tifffile.imread (pages z, rows y,
 * samples x) + a host transpose to (x, y, z); ref imaging.py:232-240
 * save_grid = tifffile.imwrite of the (z, y, x) transpose.  Here the host
 * moves page bytes only (ct_tiff_read, multi-threaded pread into caller
 * memory, normally pinned) and the transpose runs on the device after the
 * H2D copy (ct_transpose_xz).  Reader: classic/BigTIFF, II/MM, uncompressed
 * strips, 1 sample of 8/16/32/64 bits, equal pages. */
typedef struct ct_tiff_info {
    int64_t nx, ny, nz;       /* page width, page height, pages              */
    int32_t bytes_per_sample; /* 1, 2, 4, 8                                   */
    int32_t sample_format;    /* 1 uint, 2 int, 3 float (TIFF SampleFormat)   */
    int32_t big_endian;       /* 1: samples are big-endian in the file (MM)   */
    int32_t reserved;
    int64_t segments;         /* contiguous file ranges the pages occupy      */
} ct_tiff_info;

/* Parse the IFD chain; *handle stays valid until ct_tiff_close.
 * CT_ERR_IO (message names the file) for anything unreadable. */
int ct_tiff_open(const char *path, ct_tiff_info *info, void **handle);
/* All pages, (z, y, x) order, file byte order, into dst (>= nx*ny*nz*bps
 * bytes) with nthreads concurrent preads. */
int ct_tiff_read(void *handle, void *dst, int64_t dst_bytes, int32_t nthreads);
void ct_tiff_close(void *handle);
/* Write a (z, y, x) stack as a little-endian multi-page TIFF (one strip per
 * page, ImageDescription {"shape": [nz, ny, nx]}, BigTIFF past 4 GiB). */
int ct_tiff_write(const char *path, const void *src_zyx, int64_t nx, int64_t ny, int64_t nz,
                  int32_t bytes_per_sample, int32_t sample_format);
/* Device: dst[c][b][a] = src[a][b][c] for an (na, nb, nc) C-order array of
 * elem_bytes-wide elements (1, 2, 4, 8), optionally byte-swapping each
 * element (big-endian files).  (nz, ny, nx) pages -> (nx, ny, nz) grid with
 * (na, nb, nc) = (nz, ny, nx), and back with (nx, ny, nz). */
int ct_transpose_xz(const void *src, void *dst, int64_t na, int64_t nb, int64_t nc, int32_t elem_bytes,
                    int32_t byteswap, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* CT_H */

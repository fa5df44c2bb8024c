/*
 * rangeseg_b200.h — C ABI of the B200 range-image segmentation path.
 *
 * Drop-in boundary for the reference's clustering entry point
 * (/root/reference/pkg/src/rangeseg/pipeline.py):
 *
 *   rs_segment_batch       replaces Pipeline.segment_range_image (pipeline.py:85-131)
 *                          for B frames at once; its multi-frame analogue in the
 *                          reference is segment_in_parallel (pipeline.py:170-197).
 *                          Device pointers, stream-ordered.
 *   rs_segment_batch_host  the same call on HOST buffers (copies in/out inside),
 *                          the shape a cgo/ctypes/JNI binding would use.
 *   rs_stage_masks         replaces extract_ground (ground.py:95-141) +
 *                          build_connectivity (connectivity.py:64-92): the
 *                          per-pixel ground mask and edge images, for parity
 *                          checks of the edge decisions on their own.
 *   rs_project             replaces range_image.project (range_image.py:57-115)
 *                          for B point clouds at once.
 *   rs_contingency         the counting step of evaluation.match_instances
 *                          (evaluation.py:65-129) for B frames (§8(f)3).
 *   rs_labels_to_points    replaces range_image.labels_to_points
 *                          (range_image.py:130-141).  With rs_project and
 *                          rs_segment_batch this is Pipeline.segment_cloud
 *                          (pipeline.py:133-158) on the GPU.
 *
 * All entry points return RS_OK (0) or a status code; rs_last_error() gives a
 * message for the calling thread.  Invalid arguments are rejected before any
 * launch, mirroring the reference's ValueError conditions (ccl.py:71-72,
 * ground.py:108-110, map_connections.py:152-153, sensor.py:151-155).
 *
 * Constant tables (float32, `tables` argument): computed in float64 and cast
 * once, exactly as the reference does, laid out as
 *   sin_ch[H] | sin_a[H-1] | cos_a[H-1] | lo[H-1] | hi[H-1] | two_cos_v[H-1]
 *   | two_cos_off[k][H] for k < n_offsets (indexed by the pair's upper row)
 * rs_tables_count(H, n_offsets) gives its length in floats.
 *
 * Input contract (range_image.py:47-54, from_ranges): ranges finite and >= 0
 * (0 = no return).  The kernels check it on the device as they read the
 * ranges (no extra pass): a frame that breaks it gets n_clusters[b] =
 * RS_FRAME_INVALID and undefined labels; rs_segment_batch_host turns that into
 * RS_EINVAL (the reference's ValueError).
 *
 * Output contract (bit-exact with the reference):
 *   labels[b][r][c]   int32, 0 = background (invalid, ground or filtered);
 *                     clusters numbered 1..K in first-encounter row-major order;
 *                     the device buffer must be 16-byte aligned
 *   n_clusters[b]     K (or RS_FRAME_INVALID, above)
 *   cluster_sizes[b][0..K]  int64 (optional, may be NULL); [0] = H*W - sum of
 *                     kept sizes; sizes_stride must be >= H*W/max(min,1) + 1
 */
#ifndef RANGESEG_B200_H
#define RANGESEG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_MAX_OFFSETS 32
#define RS_FRAME_INVALID (-1)   /* n_clusters[b] of a frame with a NaN, inf or negative range */

enum rs_status {
    RS_OK = 0,
    RS_EINVAL = 1,      /* bad shape / parameter / offset (reference: ValueError) */
    RS_ECUDA = 2,       /* CUDA runtime error (reference: n/a) */
    RS_ETOOLARGE = 3,   /* frame does not fit one thread-block cluster */
    RS_ENODEV = 4       /* no CUDA device */
};

typedef struct rs_config {
    int32_t height, width;                  /* H, W of every frame */
    int32_t n_offsets;                      /* Map Connection offsets (MCPattern) */
    int32_t offsets[RS_MAX_OFFSETS][2];     /* canonical (dy, dx): dy>0, or dy==0 && dx>0 */
    int32_t min_cluster_points;             /* filter_small threshold (<=1: no filter) */
    int32_t ground_removal;                 /* PipelineConfig.ground_removal */
    float d_max_sq;                         /* f32(d_max*d_max) */
    float mount_height;                     /* f32(model.mount_height) */
    float keep_above;                       /* f32(GroundParams.resolve_keep_above) */
    float two_cos_h;                        /* f32(pair_constant(0, 1)) */
    int32_t rows_per_cta;                   /* 0 = automatic band height */
    int32_t reserved[3];                    /* [0]: node-capacity cap (tests, 0 = automatic);
                                               [1], [2]: must be 0 (RS_EINVAL otherwise) */
} rs_config;

/* Number of floats in the constant-table block. */
size_t rs_tables_count(int32_t height, int32_t n_offsets);

/* Launch geometry the library would use for cfg on a large batch (rows per
 * CTA band, CTAs per frame = cluster size, dynamic shared memory per CTA). */
int rs_plan(const rs_config *cfg, int32_t *rows_per_cta, int32_t *ctas_per_frame,
            size_t *smem_bytes);

/* Plan details: {fast kernel used, overflow possible, fast rows, fast CTAs,
 * fast smem, node capacity, dense rows, dense CTAs, dense smem}. */
int rs_plan_detail(const rs_config *cfg, int32_t *out, int32_t n);

/* The same for a launch of `batch` frames: a batch that fills fewer than 148
 * CTAs (one per SM) gets thinner bands, up to a 16-CTA cluster per frame
 * (batch 0: the large-batch plan, as rs_plan_detail). */
int rs_plan_batch(const rs_config *cfg, int32_t batch, int32_t *out, int32_t n);

/* B frames, device pointers, enqueued on `stream` (a cudaStream_t; NULL = legacy
 * default stream).  One kernel launch; asynchronous: returns after it.  No
 * workspace: a frame whose runs exceed the kernel's shared-memory node
 * capacity is finished inside the same launch in its own label buffer. */
int rs_segment_batch(const rs_config *cfg, const float *d_tables, const float *d_ranges,
                     int32_t batch, int32_t *d_labels, int32_t *d_n_clusters,
                     int64_t *d_cluster_sizes, int64_t sizes_stride, void *stream);

/* Same on host buffers (pinned memory gives overlapped copies).  Synchronous.
 * Returns RS_EINVAL (after the copies) if a frame breaks the input contract;
 * h_n_clusters may be NULL. */
int rs_segment_batch_host(const rs_config *cfg, const float *h_tables, const float *h_ranges,
                          int32_t batch, int32_t *h_labels, int32_t *h_n_clusters,
                          int64_t *h_cluster_sizes, int64_t sizes_stride);

/* Stage outputs for parity checks: ground mask [B][H][W] (1 = ground or no
 * return), horizontal [B][H][W], vertical [B][H-1][W]; uint8, device. */
int rs_stage_masks(const rs_config *cfg, const float *d_tables, const float *d_ranges,
                   int32_t batch, uint8_t *d_ground, uint8_t *d_horizontal,
                   uint8_t *d_vertical, void *stream);

/* Parity export of the fused kernel's OWN edge decisions: rs_segment_batch
 * (labels and counts as usual) that also writes the bit planes the kernel
 * built after its edge step, uint32 words [B][3 + n_offsets][H][ceil(W/32)],
 * bit c%32 of word c/32 for column c:
 *   plane 0  presence: r > 0 and not ground     (= !extract_ground mask)
 *   plane 1  left edge (r, c-1 mod W) - (r, c)   (= horizontal[r][c-1 mod W])
 *   plane 2  up edge (r-1, c) - (r, c)           (= vertical[r-1][c]; row 0: 0)
 *   plane 3+k  Map Connection k: (r-dy, c-dx mod W) - (r, c), rows r >= dy
 * Only geometries the fast kernel runs (rs_plan_detail()[0] == 1). */
int rs_fast_planes(const rs_config *cfg, const float *d_tables, const float *d_ranges, int32_t batch,
                   uint32_t *d_planes, int32_t *d_labels, int32_t *d_n_clusters, void *stream);

/* The stages on their own, with the reference's inputs (device buffers, B
 * frames, asynchronous on `stream`):
 * rs_height_image  height_image (range_image.py:118-127): float32 [B][H][W],
 *                  NaN where there is no return.
 * rs_ground_mask   extract_ground (ground.py:95-141) given the height image
 *                  (cfg->ground_removal = 0: the no-return mask only):
 *                  uint8 [B][H][W], 1 = ground or no return.
 * rs_connectivity  build_connectivity (connectivity.py:64-92) given a ground
 *                  mask: horizontal uint8 [B][H][W], vertical [B][H-1][W]. */
int rs_height_image(const rs_config *cfg, const float *d_tables, const float *d_ranges, int32_t batch,
                    float *d_height, void *stream);
int rs_ground_mask(const rs_config *cfg, const float *d_tables, const float *d_ranges, const float *d_height,
                   int32_t batch, uint8_t *d_mask, void *stream);
int rs_connectivity(const rs_config *cfg, const float *d_tables, const float *d_ranges, const uint8_t *d_mask,
                    int32_t batch, uint8_t *d_horizontal, uint8_t *d_vertical, void *stream);

/* ---- point clouds --------------------------------------------------------- */

typedef struct rs_project_config {
    int32_t height, width;       /* H (channels), W (columns) of the range image */
    int32_t descending;          /* channel_angles[0] > channel_angles[H-1] */
    int32_t reserved;
    double azimuth_step;         /* radians (math.radians(azimuth_step_deg), sensor.py:83) */
    double gap_lo, gap_hi;       /* (asc[1]-asc[0])/2, (asc[H-1]-asc[H-2])/2 in float64
                                    (range_image.py:86-87), asc = ascending channel angles */
} rs_project_config;

/* Point clouds -> range images (range_image.py:57-115).  Clouds are
 * concatenated: points float64 [n_points][stride] with x, y, z in the first
 * three columns (stride >= 3), cloud b = rows offsets[b]..offsets[b+1]-1
 * (int64 [n_clouds+1], device).  d_asc: the channel angles in ascending order,
 * float64 radians (np.deg2rad of the configured degrees), [H], device.
 * Outputs (device): ranges float32 [B][H][W] (0 = empty), point_index int64
 * [B][H][W] (index within the cloud, -1 = empty), counts int64 [B][2] =
 * (n_dropped, n_overwritten).  The nearest return wins a cell; among equal
 * float64 ranges the highest point index, as in the reference.  Asynchronous
 * on `stream`.  Inputs must be finite.  d_workspace: device scratch of at
 * least rs_project_workspace_size(n_points) bytes (no initialisation needed). */
int rs_project(const rs_project_config *pc, const double *d_asc, const double *d_points,
               int32_t stride, const int64_t *d_offsets, int32_t n_clouds, int64_t n_points,
               float *d_ranges, int64_t *d_point_index, int64_t *d_counts,
               void *d_workspace, size_t workspace_size, void *stream);

/* Scratch rs_project needs for n_points points (float64 range bits and an
 * int32 cell per point; 8-byte aligned). */
size_t rs_project_workspace_size(int64_t n_points);

/* Labels back to points (range_image.py:130-141): point_labels int32
 * [n_points] (device) gets labels[b][cell] for the point that won the cell,
 * 0 for dropped and overwritten points. */
int rs_labels_to_points(const int32_t *d_labels, const int64_t *d_point_index, const int64_t *d_offsets,
                        int32_t n_clouds, int32_t height, int32_t width, int64_t n_points,
                        int32_t *d_point_labels, void *stream);

/* ---- instance scoring (evaluation.py:65-129) ------------ */

/* The (ground-truth instance, predicted cluster) contingency table of B
 * frames, the counting step of evaluation.match_instances.  gt / pred: int32
 * per point (0 = none / background, values < 2^22), frames concatenated with
 * int64 CSR offsets [B+1] (B < 2^19), all device.  Output: d_pairs /
 * d_counts (int64, capacity n_points + 1) hold the sorted unique keys
 * (frame << 44 | gt << 22 | pred) over points with gt > 0 or pred > 0 and their
 * point counts; a last key 0x7fffffffffffffff (if present) counts the points
 * with gt == pred == 0 and is not a pair.  d_status int64 [2] = (number of
 * keys, 1 if a label was out of range).  Sizes of instances and clusters are
 * the row / column sums.  Counted per frame in a shared-memory hash table
 * (hand-written kernels, rs_eval.cuh); no initialisation of the workspace is
 * needed.  Asynchronous on `stream`. */
size_t rs_contingency_workspace_size(int64_t n_points, int32_t n_frames);
int rs_contingency(const int32_t *d_gt, const int32_t *d_pred, const int64_t *d_offsets, int32_t n_frames,
                   int64_t n_points, int64_t *d_pairs, int64_t *d_counts, int64_t *d_status,
                   void *d_workspace, size_t workspace_size, void *stream);

/* Debug: per-CTA phase timestamps (clock64, 16 slots per CTA) of the last
 * launch.  Only a library built with -DRS_PHASE_PROF records them; the
 * production build returns RS_EINVAL. */
int rs_phase_profile(int64_t *host_out, int32_t max_ctas);

/* Message for the last non-OK status returned on this thread. */
const char *rs_last_error(void);

/* ABI version (major*100 + minor). */
int rs_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RANGESEG_B200_H */

/* Plain-C types shared by the B200 C-ABI (vxg.h), the CPU oracle
 * (oracle/vxf_oracle.h) and the shim-compiled reference wrapper
 * (oracle/ref_capi.cpp). No torch / CUDA / Eigen types cross this boundary. */
#ifndef VXG_TYPES_H_
#define VXG_TYPES_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* vxf::WeightMode (reference proj/include/vxf/tsdf_integrator.h:11-15). */
enum vxg_weight_mode {
  VXG_WEIGHT_CONSTANT = 0,          /* w = 1 */
  VXG_WEIGHT_INVERSE_Z2 = 1,        /* w = 1/z^2 */
  VXG_WEIGHT_INVERSE_Z2_DROPOFF = 2 /* 1/z^2 with linear behind-surface drop-off */
};

/* vxf::MergeMode (tsdf_integrator.h:17-21). */
enum vxg_merge_mode {
  VXG_MERGE_SIMPLE = 0,             /* one raycast per point */
  VXG_MERGE_GROUPED = 1,            /* one raycast per terminal voxel */
  VXG_MERGE_GROUPED_ANTI_GRAZE = 2  /* grouped; passing rays skip other terminals */
};

/* vxf::TsdfConfig (tsdf_integrator.h:23-41), same field meaning and defaults. */
typedef struct vxg_tsdf_config {
  float truncation;      /* delta, default 0.4 */
  float dropoff_epsilon; /* epsilon, default 0.1 */
  float max_weight;      /* default 1e4 */
  int32_t weight_mode;   /* enum vxg_weight_mode, default INVERSE_Z2_DROPOFF */
  int32_t merge_mode;    /* enum vxg_merge_mode, default GROUPED */
  float min_ray_length;  /* default 0.05 */
  float max_ray_length;  /* default 10 */
} vxg_tsdf_config;

/* Per-scan counters: integrate()'s return value plus
 * raycasts_last_scan()/skipped_points_last_scan() (tsdf_integrator.h:81-85). */
typedef struct vxg_stats {
  uint64_t updates;
  uint64_t raycasts;
  uint64_t skipped;
} vxg_stats;

/* vxf::TsdfVoxel (voxel.h:12-18) as laid out in HBM and in VXBLX payloads
 * (serialization.cpp:107-114): f32 distance, f32 weight, u8 r,g,b, u8 pad. */
typedef struct vxg_voxel {
  float distance;
  float weight;
  uint8_t r, g, b, pad;
} vxg_voxel;

/* Marching-cubes case tables, supplied by the caller (the reference build's
 * own vxf::mc_tables, marching_cubes_tables.h): corner offsets, the two corners
 * of each edge, the crossed-edge mask and the triangle list (edge ids, -1
 * terminated) of each of the 256 corner-sign configurations. */
typedef struct vxg_mc_tables {
  int32_t corner_offsets[8][3];
  int32_t edge_corners[12][2];
  uint16_t edge_table[256];
  int8_t tri_table[256][16];
} vxg_mc_tables;

/* vxf::FixedBandMode / DistanceMetric / QueueMode (esdf_integrator.h:12-26). */
enum vxg_esdf_band { VXG_BAND_ONE_VOXEL = 0, VXG_BAND_HALF_TRUNCATION = 1 };
enum vxg_esdf_metric { VXG_METRIC_QUASI_EUCLIDEAN = 0, VXG_METRIC_EUCLIDEAN = 1 };
enum vxg_esdf_queue { VXG_QUEUE_FIFO = 0, VXG_QUEUE_PRIORITY_SINGLE = 1, VXG_QUEUE_PRIORITY_MULTI = 2 };

/* vxf::EsdfConfig (esdf_integrator.h:28-41), same field meaning and defaults:
 * d_max 4, one-voxel band, truncation 0.4, quasi-Euclidean, priority
 * single-insert queue, bucket width 0 (= voxel size). */
typedef struct vxg_esdf_config {
  float d_max;
  int32_t band_mode;    /* enum vxg_esdf_band */
  float truncation;
  int32_t metric;       /* enum vxg_esdf_metric */
  int32_t queue_mode;   /* enum vxg_esdf_queue */
  float bucket_width;
} vxg_esdf_config;

/* vxf::EsdfVoxel as laid out in HBM and in ESDF VXBLX payloads
 * (serialization.cpp:116-122): f32 distance, u8 flags (1 observed, 2 fixed,
 * 4 in raise, 8 in lower; voxel.h:24-27), 3x i8 parent. */
typedef struct vxg_esdf_voxel {
  float distance;
  uint8_t flags;
  int8_t parent[3];
} vxg_esdf_voxel;

/* Status codes (SURVEY.md §8b error convention). */
enum vxg_status {
  VXG_OK = 0,
  VXG_EINVAL = 1,  /* invalid argument; message = reference's exception text */
  VXG_ENOMEM = 2,  /* device slab / block hash / staging exhausted */
  VXG_ECUDA = 3,   /* CUDA runtime error */
  VXG_ERANGE = 4,  /* block index outside the packed-key range */
  VXG_EPARSE = 5,  /* malformed VXBLX stream (vxf::ParseError) */
  VXG_EIO = 6      /* file could not be opened / written */
};

#ifdef __cplusplus
}
#endif

#endif /* VXG_TYPES_H_ */

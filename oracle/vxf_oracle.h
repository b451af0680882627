/* CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A line-by-line restatement of the reference TSDF integration path
 * (/root/reference/proj/src/tsdf_integrator.cpp, include/vxf/{core,layer,voxel}.h,
 * src/serialization.cpp) with explicit IEEE fp32/fp64 arithmetic and no Eigen.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * it, and only as the checker. The product path (libvxg.so) never links it.
 *
 * Parity pin: tests/test_oracle_pin.py checks this restatement bit-exactly
 * against oracle/_ref (the UNMODIFIED reference sources compiled with
 * oracle/eigen_shim) on random scans, and tests/golden/ holds vectors generated
 * from oracle/_ref by tests/golden/make_golden.py. The Eigen reduction order at
 * the boundary is the shim's (a0+(a1+a2)); real-Eigen parity is unpinned
 * (SURVEY.md §8c).
 */
#ifndef VXF_ORACLE_H_
#define VXF_ORACLE_H_

#include "../include/vxg_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vxo_layer vxo_layer;

/* TsdfConfig::validate (tsdf_integrator.cpp:10-20). Returns 0 or VXG_EINVAL. */
int vxo_config_validate(const vxg_tsdf_config* c, char* err, size_t err_len);
/* TsdfConfig::for_voxel_size (tsdf_integrator.h:33-38) and defaults (:24-30). */
void vxo_config_default(vxg_tsdf_config* c);
void vxo_config_for_voxel_size(vxg_tsdf_config* c, float voxel_size);

/* Layer(voxel_size, vps) (layer.h:62-67). NULL on invalid geometry. */
vxo_layer* vxo_layer_create(float voxel_size, int voxels_per_side);
void vxo_layer_destroy(vxo_layer* l);
size_t vxo_block_count(const vxo_layer* l);

/* TsdfIntegrator::integrate (tsdf_integrator.cpp:111-127). pose is the 3x4
 * row-major [R | t] sensor->world transform. rgb may be NULL (no colours).
 * Returns 0, or VXG_EINVAL (config invalid). */
int vxo_integrate(vxo_layer* l, const vxg_tsdf_config* c, const float* xyz, const uint8_t* rgb,
                  size_t n, const float pose[12], vxg_stats* out);

/* Blocks sorted by (x,y,z) (serialization.cpp:150-156); idx is B x 3 int32,
 * voxels is B x vps^3 vxg_voxel (x-fastest, layer.h:23-30). Returns blocks
 * written (<= cap). */
size_t vxo_export_blocks(const vxo_layer* l, int32_t* idx, vxg_voxel* voxels, size_t cap);
/* Voxel lookup (layer.h:99-112): returns 1 and fills *out if the block exists. */
int vxo_voxel(const vxo_layer* l, int32_t gx, int32_t gy, int32_t gz, vxg_voxel* out);
/* Overwrite / insert one block (used by tests to seed a layer state). */
int vxo_set_block(vxo_layer* l, const int32_t idx[3], const vxg_voxel* voxels);

/* VXBLX bytes (serialization.cpp:141-168); returns the required size, writes
 * only if cap is large enough. */
size_t vxo_save_vxblx(const vxo_layer* l, uint8_t* buf, size_t cap);

/* Free functions restated from tsdf_integrator.cpp. */
float vxo_projective_distance(const float x[3], const float p[3], const float s[3]);
float vxo_measurement_weight(int mode, float z, float d, float truncation, float dropoff_epsilon);
void vxo_update_voxel(vxg_voxel* v, float d, float w, float truncation, float max_weight,
                      const uint8_t* color /* NULL = no colour */);
/* RayCaster walk (tsdf_integrator.cpp:69-104): writes up to cap voxel indices
 * (x,y,z int32 triples) and returns the total number of voxels visited. */
size_t vxo_raycast(const float start[3], const float end[3], float voxel_size, int32_t* out,
                   size_t cap);
/* global_index_from_point (core.h:43-47). */
void vxo_global_index(const float p[3], float voxel_size, int32_t out[3]);
/* IndexHash (core.h:68-74). */
uint64_t vxo_index_hash(int32_t x, int32_t y, int32_t z);

/* Test hook: integrates one scan like vxo_integrate and writes the ordered
 * update_tsdf_voxel call sequence as 7-word records (ray index in ray order,
 * gx, gy, gz, d bits, w bits, colour | has_colour<<31); returns the count. */
size_t vxo_trace_updates(vxo_layer* l, const vxg_tsdf_config* c, const float* xyz, const uint8_t* rgb, size_t n,
                         const float pose[12], uint32_t* out, size_t cap);

/* Grouped-mode ray order: the terminal voxel keys of the in-range points in
 * IndexMap<PointBucket> iteration order (tsdf_integrator.cpp:199-223), i.e.
 * std::unordered_map itself after reserve(n/4+1). Writes up to cap keys
 * (x,y,z) and returns the number of buckets. */
size_t vxo_grouped_ray_order(const vxg_tsdf_config* c, float voxel_size, const float* xyz,
                             size_t n, const float pose[12], int32_t* keys, size_t cap);

/* libstdc++ bucket-count schedule of an IndexMap after reserve(n/4+1) and
 * `max_keys` distinct insertions: writes (elements_before_rehash, new_bucket_count)
 * pairs; entry 0 is (0, initial bucket count). Returns the number of entries. */
size_t vxo_bucket_schedule(size_t n_points, size_t max_keys, uint64_t* out, size_t cap);

/* Read-side consumers: interpolate_distance (interpolation.h:28-60) per point
 * (found[i] = 0: absent) and surface_error (analysis.cpp:41-59), out =
 * {rms, mean, max, count, unknown_fraction}. */
void vxo_interpolate(const vxo_layer* l, const float* pts, size_t n, float* d, uint8_t* found);
void vxo_surface_error(const vxo_layer* l, const float* pts, size_t n, float truncation, double out[5]);

/* MeshExtractor (mesh_extractor.cpp:41-151) restated: marching cubes per block
 * with the caller's case tables. blocks == NULL: every block (extract_all),
 * else the allocated ones among blocks[n_req x 3] (extract_blocks). Output in
 * (x,y,z) block order: bidx[n_frag x 3], frag_tri[n_frag + 1] triangle
 * offsets, verts / normals [n_tri x 9], colors [n_tri x 9] (with_colors).
 * Returns n_frag and *n_tri; writes the arrays only when cap_frag >= n_frag
 * and cap_tri >= n_tri (call once with zero caps to size them). */
size_t vxo_mesh_extract(const vxo_layer* l, const vxg_mc_tables* t, int with_colors, const int32_t* blocks,
                        size_t n_req, int32_t* bidx, uint64_t* frag_tri, float* verts, float* normals,
                        uint8_t* colors, size_t cap_frag, size_t cap_tri, uint64_t* n_tri);

/* EsdfIntegrator::build_from_occupancy (esdf_integrator.cpp:303-330) over the
 * oracle's TSDF layer, restated with the reference's wavefront queue
 * (WavefrontQueue :20-52, push_lower :99-105, process_lower_queue :220-230,
 * relax_neighbors :232-294, constructor :54-84, EsdfConfig::validate :10-18).
 * Writes the ESDF VXBLX bytes (save_layer, serialization.cpp:116-122,141-168)
 * into buf and returns the size needed (no write when cap is too small), or 0
 * with err set when the config is invalid. */
size_t vxo_esdf_occupancy(const vxo_layer* l, const vxg_esdf_config* c, uint8_t* buf, size_t cap, char* err,
                          size_t err_len);

#ifdef __cplusplus
}
#endif

#endif /* VXF_ORACLE_H_ */

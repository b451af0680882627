/* vxg — B200-native (sm_100a) TSDF integration behind a plain C ABI.
 *
 * Drop-in boundary for the reference integrator's hot path. Each entry point
 * names the reference interface it replaces (paths under
 * /root/reference/proj). Only plain pointers and sizes cross this boundary; no
 * torch, CUDA or Eigen types. All functions return an enum vxg_status; the
 * message of the last failure on the calling thread is vxg_last_error().
 * There is no CPU fallback: every compute entry point runs CUDA kernels and
 * fails with VXG_ECUDA when no sm_100 device is usable.
 *
 * Threading: one handle = one device + one CUDA stream. Calls on
 * a handle must be serialised by the caller (the reference's single-writer
 * contract, include/vxf/layer.h:53-55). Distinct handles may
 * run concurrently.
 */
#ifndef VXG_H_
#define VXG_H_

#include "vxg_types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vxg_handle vxg_handle;

/* One posed scan (vxf::Scan, include/vxf/scan.h:13-20): n sensor-frame points
 * xyz[n*3] (float32), optional parallel colours rgb[n*3] (NULL = no colours),
 * pose = 3x4 row-major [R | t] sensor->world (vxf::Transform); the sensor
 * origin is t (scan.h:19). */
typedef struct vxg_frame {
  const float* xyz;
  const uint8_t* rgb;
  uint64_t n;
  float pose[12];
} vxg_frame;

/* Flags for vxg_integrate_batch. */
enum vxg_batch_flags {
  VXG_INPUT_HOST = 0,   /* xyz/rgb are host pointers (copied H2D inside the call) */
  VXG_INPUT_DEVICE = 1, /* xyz/rgb are device pointers on the handle's device */
  VXG_NO_SYNC_STATS = 2 /* reserved */
};

/* Thread-local message of the last failing call ("" if none). */
const char* vxg_last_error(void);

/* Library / device info: writes a one-line description into buf. */
int vxg_device_info(int device, char* buf, size_t buf_len);

/* vxf::TsdfLayer(voxel_size, vps) (include/vxf/layer.h:62-67) +
 * vxf::TsdfIntegrator(config, &layer) (src/tsdf_integrator.cpp:106-109):
 * validates the config exactly like TsdfConfig::validate (:10-20) and the
 * layer geometry like Layer's constructor; VXG_EINVAL carries the reference's
 * exception text. block_capacity = initial slab size in blocks (0 = default);
 * the slab grows on demand. */
int vxg_create(const vxg_tsdf_config* config, float voxel_size, int voxels_per_side, int device,
               uint64_t block_capacity, vxg_handle** out);
int vxg_destroy(vxg_handle* h);

/* TsdfIntegrator::config() (tsdf_integrator.h:87) and a validated update. */
int vxg_get_config(const vxg_handle* h, vxg_tsdf_config* out);
int vxg_set_config(vxg_handle* h, const vxg_tsdf_config* config);

/* Run all device work of this handle on an external CUDA stream
 * (cudaStream_t passed as void*; NULL restores the handle's own stream). */
int vxg_set_stream(vxg_handle* h, void* cuda_stream);

/* size_t TsdfIntegrator::integrate(const Scan&) (src/tsdf_integrator.cpp:111-127)
 * with raycasts_last_scan()/skipped_points_last_scan() (tsdf_integrator.h:84-85)
 * in *out. Host pointers. Synchronous: the layer reflects the scan on return. */
int vxg_integrate(vxg_handle* h, const float* xyz, const uint8_t* rgb, uint64_t n, const float pose[12],
                  vxg_stats* out);

/* Integrates n_frames scans in order; the resulting layer and the per-frame
 * stats (out[n_frames], may be NULL) are identical to n_frames sequential
 * vxg_integrate calls. flags: enum vxg_batch_flags. Synchronous. */
int vxg_integrate_batch(vxg_handle* h, const vxg_frame* frames, uint64_t n_frames, int flags, vxg_stats* out);

/* Same as vxg_integrate_batch over one packed buffer: frame f owns points
 * [offsets[f], offsets[f+1]) of xyz/rgb, pose f is poses[12*f .. 12*f+11]. */
int vxg_integrate_packed(vxg_handle* h, const float* xyz, const uint8_t* rgb, const uint64_t* offsets,
                         const float* poses, uint64_t n_frames, int flags, vxg_stats* out);

/* Streaming ingestion (double-buffered staging of packed batches).
 * vxg_stage_packed starts the asynchronous host->device copy of a packed batch
 * (xyz/rgb in pinned host memory for a truly asynchronous copy; layout as in
 * vxg_integrate_packed) into one of two staging slots on the handle's copy
 * stream and returns at once (*slot = the slot id). vxg_integrate_staged then
 * integrates that staged batch with n_frames poses: layer and stats identical
 * to vxg_integrate_packed on the same inputs. Staging batch k+1 before
 * integrating batch k overlaps its copy with batch k's compute. At most two
 * batches may be staged and not yet integrated (VXG_EINVAL otherwise); the
 * host buffers must stay valid until the matching vxg_integrate_staged returns. */
int vxg_stage_packed(vxg_handle* h, const float* xyz, const uint8_t* rgb, const uint64_t* offsets,
                     uint64_t n_frames, int* slot);
int vxg_integrate_staged(vxg_handle* h, int slot, const float* poses, vxg_stats* out);

/* ---- meshing on the device slab: vxf::MeshExtractor (mesh_extractor.cpp)
 * Per-block marching cubes over the TSDF zero crossing (extract_block,
 * mesh_extractor.cpp:85-151): cubes span 8 voxel centres and may straddle
 * block boundaries; cubes with an unallocated or unobserved corner emit
 * nothing; shared edges interpolate from the lower global index; vertex
 * normals from central differences of interpolate_distance (vertex_normal,
 * :69-83). vxg_mesh_extract computes the fragments of the given blocks
 * (blocks = n x 3 block indices, unallocated ones skipped — extract_blocks
 * :41-46), or of every allocated block when blocks == NULL (extract_all
 * :48-52), keeps them on the device and returns the fragment and triangle
 * counts; vxg_mesh_fetch copies them out, fragments sorted by block index
 * (x, y, z): block_idx n_frag x 3, frag_tri (n_frag + 1) triangle offsets,
 * vertices / normals n_tri x 9 floats (3 vertices per triangle, in the
 * reference's emission order; the fragment's triangle t is (3t, 3t+1, 3t+2)),
 * colors n_tri x 9 u8 (with_colors only; may be NULL). */
int vxg_mesh_extract(vxg_handle* h, const vxg_mc_tables* tables, const int32_t* blocks, uint64_t n_blocks,
                     int with_colors, uint64_t* n_frag, uint64_t* n_tri);
int vxg_mesh_fetch(vxg_handle* h, int32_t* block_idx, uint64_t* frag_tri, float* vertices, float* normals,
                   uint8_t* colors);

/* ---- scan I/O (scan.h / scan.cpp), for the drop-in CLI flow (cmd_integrate)
 * vxf::load_ply_points (scan.cpp:70-180): PLY point cloud, ascii or binary
 * little-endian, vertex properties x,y,z[,red,green,blue] (others skipped).
 * Two calls: xyz == NULL returns the vertex count *n and *has_color only;
 * then xyz (n x 3) and rgb (n x 3, or NULL) receive the points — host
 * pointers, or device pointers on `device` with flags = VXG_INPUT_DEVICE. A
 * binary payload is decoded on the device. Errors carry the reference's
 * std::runtime_error texts: VXG_EIO "cannot open PLY file: <path>", VXG_EPARSE
 * for "not a PLY file", "unsupported PLY format", "list property on vertex
 * element", "PLY vertex element lacks x/y/z properties", "truncated PLY vertex
 * data", "malformed PLY vertex line", "unsupported PLY property/scalar type". */
int vxg_ply_load(const char* path, int device, float* xyz, uint8_t* rgb, uint64_t cap, int flags, uint64_t* n,
                 int* has_color);
/* vxf::load_tum_trajectory (scan.cpp:182-211): `timestamp tx ty tz qx qy qz
 * qw` per line, '#' comments; poses as row-major 3x4 [R | t] (R from the
 * normalized quaternion). ts == poses == NULL: count only. Host-side text. */
int vxg_tum_load(const char* path, double* ts, float* poses, uint64_t cap, uint64_t* n);
/* vxf::save_ply_mesh (scan.cpp:213-240): binary little-endian PLY with
 * normals and, when colors != NULL, colours; triangles n_triangles x 3. */
int vxg_save_ply_mesh(const char* path, const float* vertices, const float* normals, const uint8_t* colors,
                      uint64_t n_vertices, const uint32_t* triangles, uint64_t n_triangles);

/* Layer::block_count() (layer.h:72). */
int vxg_block_count(vxg_handle* h, uint64_t* out);

/* Layer::blocks() enumerated in the order save_layer writes them
 * (src/serialization.cpp:150-156: sorted by (x,y,z)). idx = B x 3 int32,
 * voxels = B x vps^3 vxg_voxel, x-fastest (layer.h:23-30). Writes at most cap
 * blocks; *n_out = blocks written. Either output pointer may be NULL. */
int vxg_export_blocks(vxg_handle* h, int32_t* idx, vxg_voxel* voxels, uint64_t cap, uint64_t* n_out);

/* Layer::block_ptr (layer.h:89-97) + copy-out for n block indices idx[n*3]:
 * voxels = n x vps^3 vxg_voxel (x-fastest; zeros for an absent block),
 * found[i] = 1 when block i is allocated. One device gather and one D2H per
 * 256 MB of payload (the C++ drop-in's per-scan writeback). Either output
 * may be NULL. */
int vxg_fetch_blocks(vxg_handle* h, const int32_t* idx, uint64_t n, vxg_voxel* voxels, uint8_t* found);

/* Inserts / overwrites blocks (idx B x 3, voxels B x vps^3) — used to resume
 * from a VXBLX checkpoint (load_tsdf_layer, serialization.cpp:193-212) or to
 * mirror a host layer. */
int vxg_import_blocks(vxg_handle* h, const int32_t* idx, const vxg_voxel* voxels, uint64_t n);

/* interpolate_distance (interpolation.h:28-60) for n points pts[n*3] (world
 * frame): trilinear over the 8 surrounding voxel centres; found[i] = 0 when
 * any corner is unallocated or unobserved (std::nullopt). flags:
 * VXG_INPUT_DEVICE = pts, d, found are device pointers. */
int vxg_interpolate_distance(vxg_handle* h, const float* pts, uint64_t n, float* d, uint8_t* found, int flags);
/* surface_error (analysis.cpp:41-59) of host points against the layer:
 * out[5] = {rms, mean, max, count, unknown_fraction}. Interpolation on the
 * GPU; the fp64 accumulation runs in point order on the host, as in the
 * reference's Accumulator. */
int vxg_surface_error(vxg_handle* h, const float* pts, uint64_t n, float truncation, double* out);

/* ---- ESDF on the device slab: vxf::EsdfIntegrator::build_from_occupancy
 * (esdf_integrator.cpp:303-330), the occupancy-seeded baseline: every observed
 * voxel with TSDF distance < 0 seeds at 0 (fixed), every other observed voxel
 * starts at d_max and is lowered through observed 26-neighbours by the
 * quasi-Euclidean steps v*sqrt(1|2|3) (relax_neighbors :258-292). One ESDF
 * block per allocated TSDF block. Distances and flags are bit-exact with the
 * reference for every queue mode (the quasi-Euclidean, only-lowering
 * propagation has a unique fixed point); parents are the first minimising
 * neighbour in the reference's neighbour order, which can differ from the
 * reference's queue-order-dependent choice on ties. Errors: VXG_EINVAL with
 * EsdfConfig::validate's text (:10-18), or for the Euclidean metric (its
 * distances depend on the wavefront order; tools/esdf_order_probe). rounds
 * (may be NULL) = relaxation launches until the fixed point. */
int vxg_esdf_build_occupancy(vxg_handle* h, const vxg_esdf_config* config, uint64_t* rounds);
/* save_layer(EsdfLayer) (serialization.cpp:141-168; payload f32 distance, u8
 * flags, 3 x i8 parent, :116-122) of the last vxg_esdf_build_occupancy result;
 * *need = byte size; writes only when cap >= *need. */
int vxg_esdf_serialize_vxblx(vxg_handle* h, uint8_t* buf, uint64_t cap, uint64_t* need);

/* Layer::voxel_ptr (layer.h:99-112) for n global voxel indices g[n*3]:
 * found[i] = 0 (block unallocated: absence, never a default voxel) or 1. */
int vxg_query_voxels(vxg_handle* h, const int32_t* g, uint64_t n, vxg_voxel* out, uint8_t* found);

/* save_layer (serialization.cpp:141-168,216-218): VXBLX bytes. With buf NULL or
 * cap too small only *need is written. */
int vxg_serialize_vxblx(vxg_handle* h, uint8_t* buf, uint64_t cap, uint64_t* need);
/* save_layer_file (serialization.cpp:244-248). */
int vxg_save_vxblx(vxg_handle* h, const char* path);
/* load_tsdf_layer (serialization.cpp:193-212,226-228): replaces the layer with
 * the stream's blocks; VXG_EPARSE with the reference's ParseError text. */
int vxg_load_vxblx(vxg_handle* h, const uint8_t* buf, uint64_t len);

/* Drops every block (fresh layer, same geometry and config). Deferred on the
 * device: applied after the folds still in flight, before the next map access. */
int vxg_reset(vxg_handle* h);

/* A batch's ordered fold (the apply stage) may still be running on the device
 * when vxg_integrate_* returns: its statistics do not depend on it, and the
 * next batch's bundling overlaps it. Every entry point that reads or writes
 * the map waits for it; vxg_flush orders the handle's stream (vxg_set_stream)
 * after it without a host sync, so an event or copy queued afterwards sees the
 * final map. (The reference's integrate() is synchronous,
 * tsdf_integrator.cpp:111-127; results are identical.) */
int vxg_flush(vxg_handle* h);

/* Updated-block consumers (Layer::register_consumer / drain_updated,
 * layer.h:124-140): blocks allocated or updated since the consumer's last
 * drain. drain writes up to cap block indices (x,y,z) and clears the set;
 * *n_out = set size. Unknown consumer -> VXG_EINVAL
 * ("unknown updated-block consumer: <name>"). */
int vxg_register_consumer(vxg_handle* h, const char* name);
int vxg_drain_updated(vxg_handle* h, const char* name, int32_t* idx, uint64_t cap, uint64_t* n_out);

/* ---- sharded map: block-key ownership across ranks.
 * Every rank bundles the whole batch (identical ray order), walks a
 * record-balanced slice of the global ray order, routes each update record to
 * the owner of its block (owner = mix64(block) mod world) with an all-to-all,
 * and owners sort + fold. The union of the shards equals the 1-GPU layer
 * bit-for-bit. */
/* NCCL unique id (128 bytes) made by rank 0 and broadcast by the caller. */
int vxg_nccl_unique_id(uint8_t* out);
/* Makes h the shard `rank` of `world` (one process per GPU); world > 1 creates
 * an NCCL communicator from id_bytes. vxg_integrate_* then run sharded and
 * return the global per-frame counters on every rank. world == 1 with a
 * non-NULL id_bytes runs the same sharded path over a 1-rank communicator
 * (NCCL self send/recv): the exchange on one GPU, for tests and bench. */
int vxg_shard_init(vxg_handle* h, int rank, int world, const uint8_t* id_bytes);
/* Sharding mode (SURVEY.md 8e fallback): on = replicated traversal — every
 * rank walks ALL rays and keeps only the records of the blocks it owns, so no
 * update records are exchanged (only the per-frame counters are summed) at the
 * cost of G x the walk. off (default) = each rank walks its slice of the ray
 * order and owners receive their records with one all-to-all. Same result
 * either way. */
int vxg_shard_set_replicated(vxg_handle* h, int on);
/* Loopback group: `world` shards on ONE device in one process, exchanging
 * records with device-to-device copies (the sharded kernels without NVLink);
 * used to test the sharded path on a single GPU. */
typedef struct vxg_group vxg_group;
int vxg_group_create(const vxg_tsdf_config* config, float voxel_size, int voxels_per_side, int device, int world,
                     uint64_t block_capacity, vxg_group** out);
/* vxg_shard_set_replicated for every shard of a loopback group. */
int vxg_group_set_replicated(vxg_group* g, int on);
int vxg_group_destroy(vxg_group* g);
int vxg_group_shard(vxg_group* g, int i, vxg_handle** out);
int vxg_group_set_config(vxg_group* g, const vxg_tsdf_config* config);
int vxg_group_integrate_packed(vxg_group* g, const float* xyz, const uint8_t* rgb, const uint64_t* offsets,
                               const float* poses, uint64_t n_frames, int flags, vxg_stats* out);
int vxg_group_serialize_vxblx(vxg_group* g, uint8_t* buf, uint64_t cap, uint64_t* need);

/* Stage profiling: when enabled, every batch records CUDA events around each
 * pipeline stage on the handle's stream. vxg_stage_times returns, per stage,
 * the accumulated milliseconds and launches since the last reset (names in
 * vxg_stage_name). */
int vxg_profile(vxg_handle* h, int enable);
int vxg_stage_count(void);
const char* vxg_stage_name(int stage);
int vxg_stage_times(vxg_handle* h, double* ms, uint64_t* launches, uint64_t* units, int reset);
/* Work counters since the last reset: out[0] = candidate records emitted,
 * out[1] = distinct voxels folded (N_vox), out[2] = longest per-voxel fold
 * chain (records), out[3] = allocated blocks, out[4] = radix passes of the
 * last record sort (out must hold 5 values). */
int vxg_batch_info(vxg_handle* h, uint64_t* out, int reset);
/* Kernel launches issued by the library since the last call (and reset). */
int vxg_kernel_launches(vxg_handle* h, uint64_t* out, int reset);

/* Self-test of the fast exact fold arithmetic used by the apply kernel:
 * n random divisions (shared-reciprocal fast path vs __fdiv_rn) and n_seq
 * random update sequences of length len (fast fold vs the reference-order
 * update_tsdf_voxel restatement), all on the device. out[0], out[1] =
 * mismatch counts (both must be 0). */
int vxg_selftest_fold(int device, uint64_t n, uint64_t n_seq, uint32_t len, uint64_t seed, uint64_t* out);
/* Self-test of the in-house device primitives the pipeline is built on
 * (csrc/vxg_sort.cuh; they replace the CUB calls of round 1): exclusive prefix
 * sums (32- and 64-bit, the latter in place), the stable 64-bit-key pair sort
 * (ascending or descending over the low `bits` key bits) and the 32-bit pair
 * sort, on n random items against the host. out[0..3] = mismatch counts (all
 * must be 0; out must hold 4 values). */
int vxg_selftest_prims(vxg_handle* h, uint64_t n, int bits, int descending, uint64_t seed, uint64_t* out);
/* Debug: lengths and voxel keys of the n longest fold chains of the last batch. */
int vxg_debug_top_runs(vxg_handle* h, uint32_t* len, uint32_t* keys, uint32_t n);

/* ---- device evaluation of the reference's public free functions (tested
 * directly by the reference's unit tests, tsdf_integrator.h:46-59), batched: */
/* projective_distance(x, p, s) (src/tsdf_integrator.cpp:22-27), n triples. */
int vxg_eval_projective_distance(int device, const float* x, const float* p, const float* s, uint64_t n,
                                 float* out);
/* measurement_weight(mode, z, d, truncation, eps) (:29-44). */
int vxg_eval_measurement_weight(int device, int mode, const float* z, const float* d, uint64_t n,
                                float truncation, float dropoff_epsilon, float* out);
/* Sequential update_tsdf_voxel folds (:46-67): voxel i starts from voxels[i]
 * and folds d[j], w[j], rgb[j] for j in [starts[i], starts[i+1]) in order.
 * rgb may be NULL (no colour). */
int vxg_eval_update_voxels(int device, vxg_voxel* voxels, uint64_t n_voxels, const uint64_t* starts,
                           const float* d, const float* w, const uint8_t* rgb, float truncation,
                           float max_weight);
/* RayCaster walks (:69-104) for n segments start[i]->end[i]: counts[i] = voxels
 * visited; voxels written to out[offsets[i]*3 ...] when out != NULL (offsets
 * are exclusive prefix sums of counts computed by the caller from a first
 * call with out == NULL). */
int vxg_eval_raycast(int device, const float* start, const float* end, uint64_t n, float voxel_size,
                     uint32_t* counts, const uint64_t* offsets, int32_t* out);

#ifdef __cplusplus
}
#endif

#endif /* VXG_H_ */

// Link-level drop-in for the reference's vxf::MeshExtractor
// (/root/reference/proj/include/vxf/mesh_extractor.h), backed by the B200
// C ABI (vxg_mesh_extract / vxg_mesh_fetch). Compile this file INSTEAD of the
// reference's src/mesh_extractor.cpp and link libvxg.so.
//
// The caller's host TsdfLayer is uploaded to a device slab (vxg_import_blocks),
// marching cubes run there with the reference build's own case tables
// (vxf::mc_tables, marching_cubes_tables.h), and the fragments come back as
// vxf::Mesh values: vertices, normals and colours bit-identical to the
// reference's extract_block (mesh_extractor.cpp:85-151), triangles
// (3t, 3t+1, 3t+2) within each fragment as the reference emits them.
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "vxf/marching_cubes_tables.h"
#include "vxf/mesh_extractor.h"
#include "vxg.h"

namespace vxf {

namespace {

void check(int rc) {
  if (rc == VXG_OK) return;
  const std::string msg = vxg_last_error();
  if (rc == VXG_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error("vxg: " + msg);
}

const vxg_mc_tables& tables() {
  static const vxg_mc_tables t = [] {
    vxg_mc_tables o{};
    for (int c = 0; c < 8; ++c)
      for (int a = 0; a < 3; ++a) o.corner_offsets[c][a] = mc_tables::kCornerOffsets[c][a];
    for (int e = 0; e < 12; ++e)
      for (int a = 0; a < 2; ++a) o.edge_corners[e][a] = mc_tables::kEdgeCorners[e][a];
    for (int i = 0; i < 256; ++i) {
      o.edge_table[i] = mc_tables::kEdgeTable[i];
      for (int k = 0; k < 16; ++k) o.tri_table[i][k] = static_cast<int8_t>(mc_tables::kTriTable[i][k]);
    }
    return o;
  }();
  return t;
}

// Uploads the host layer, extracts `req` (nullptr: every block), fills `out`.
void extract_on_device(const TsdfLayer& tsdf, bool with_colors, const std::vector<int32_t>* req,
                       IndexMap<Mesh>* out) {
  const float v = tsdf.voxel_size();
  vxg_tsdf_config cfg{4.0f * v, v, 1e4f, 2, 1, 0.05f, 10.0f};  // any valid config: only the layer is used
  vxg_handle* h = nullptr;
  check(vxg_create(&cfg, v, tsdf.voxels_per_side(), 0, tsdf.block_count() + 1, &h));
  struct Guard {
    vxg_handle* h;
    ~Guard() { vxg_destroy(h); }
  } guard{h};
  const int vps = tsdf.voxels_per_side();
  const size_t nv = static_cast<size_t>(vps) * vps * vps;
  std::vector<int32_t> idx;
  std::vector<vxg_voxel> vox;
  idx.reserve(3 * tsdf.block_count());
  vox.reserve(nv * tsdf.block_count());
  for (const auto& [bidx, block] : tsdf.blocks()) {
    idx.insert(idx.end(), {bidx.x(), bidx.y(), bidx.z()});
    for (size_t i = 0; i < nv; ++i) {
      const TsdfVoxel& s = block->voxel(i);
      vox.push_back(vxg_voxel{s.distance, s.weight, s.color.r, s.color.g, s.color.b, 0});
    }
  }
  check(vxg_import_blocks(h, idx.data(), vox.data(), idx.size() / 3));
  uint64_t nf = 0, nt = 0;
  check(vxg_mesh_extract(h, &tables(), req ? req->data() : nullptr, req ? req->size() / 3 : 0, with_colors ? 1 : 0,
                         &nf, &nt));
  std::vector<int32_t> bidx(3 * nf);
  std::vector<uint64_t> frag(nf + 1);
  std::vector<float> verts(9 * nt), normals(9 * nt);
  std::vector<uint8_t> colors(with_colors ? 9 * nt : 0);
  check(vxg_mesh_fetch(h, bidx.data(), frag.data(), verts.data(), normals.data(),
                       with_colors ? colors.data() : nullptr));
  for (uint64_t j = 0; j < nf; ++j) {
    Mesh m;
    for (uint64_t t = frag[j]; t < frag[j + 1]; ++t) {
      const uint32_t base = static_cast<uint32_t>(m.vertices.size());
      for (int k = 0; k < 3; ++k) {
        const float* p = &verts[9 * t + 3 * k];
        const float* n = &normals[9 * t + 3 * k];
        m.vertices.emplace_back(p[0], p[1], p[2]);
        m.normals.emplace_back(n[0], n[1], n[2]);
        if (with_colors) {
          const uint8_t* c = &colors[9 * t + 3 * k];
          m.colors.push_back(Color{c[0], c[1], c[2]});
        }
      }
      m.triangles.push_back({base, base + 1, base + 2});
    }
    (*out)[BlockIndex(bidx[3 * j], bidx[3 * j + 1], bidx[3 * j + 2])] = std::move(m);
  }
}

}  // namespace

MeshExtractor::MeshExtractor(const TsdfLayer* tsdf, bool with_colors) : tsdf_(tsdf), with_colors_(with_colors) {}

void MeshExtractor::extract_blocks(const IndexSet& blocks) {
  std::vector<int32_t> req;
  for (const BlockIndex& b : blocks)
    if (tsdf_->block_ptr(b) != nullptr) req.insert(req.end(), {b.x(), b.y(), b.z()});
  if (req.empty()) return;
  extract_on_device(*tsdf_, with_colors_, &req, &fragments_);
}

void MeshExtractor::extract_all() {
  if (tsdf_->block_count() == 0) return;
  extract_on_device(*tsdf_, with_colors_, nullptr, &fragments_);
}

Mesh MeshExtractor::combined() const {
  Mesh out;
  for (const auto& kv : fragments_) out.append(kv.second);
  if (!with_colors_) out.colors.clear();
  return out;
}

Mesh extract_mesh(const TsdfLayer& tsdf, bool with_colors) {
  MeshExtractor extractor(&tsdf, with_colors);
  extractor.extract_all();
  return extractor.combined();
}

}  // namespace vxf

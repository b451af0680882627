// Scan I/O on either side of the integrator:
//  * vxg_ply_load  = vxf::load_ply_points (scan.cpp:70-180): the header is
//    parsed on the host with the reference's rules and messages; a binary
//    little-endian vertex payload is copied to the device as raw rows and
//    decoded there (one thread per vertex: any supported property type ->
//    float xyz / u8 rgb), straight into device buffers for integration or back
//    to the host; ascii payloads are text and are parsed on the host.
//  * vxg_tum_load  = vxf::load_tum_trajectory (scan.cpp:182-211).
//  * vxg_save_ply_mesh = vxf::save_ply_mesh (scan.cpp:213-240) for a mesh given
//    as flat arrays (vxg_mesh_fetch layout, one fragment or the concatenation).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/vxg.h"

namespace vxg_io {

struct IoError {
  int code;
  std::string msg;
};

// Property type codes (parse_scalar, scan.cpp:29-66); kBad: valid size, no scalar parse.
enum : int { kF32 = 0, kF64, kU8, kI8, kI16, kU16, kI32, kU32, kBad64 };

struct Prop {
  std::string type, name;
};

size_t prop_size(const std::string& t) {  // property_size (scan.cpp:17-27)
  if (t == "char" || t == "uchar" || t == "int8" || t == "uint8") return 1;
  if (t == "short" || t == "ushort" || t == "int16" || t == "uint16") return 2;
  if (t == "int" || t == "uint" || t == "int32" || t == "uint32" || t == "float" || t == "float32") return 4;
  if (t == "double" || t == "float64" || t == "int64" || t == "uint64") return 8;
  throw IoError{VXG_EPARSE, "unsupported PLY property type: " + t};
}

int type_code(const std::string& t) {
  if (t == "float" || t == "float32") return kF32;
  if (t == "double" || t == "float64") return kF64;
  if (t == "uchar" || t == "uint8") return kU8;
  if (t == "char" || t == "int8") return kI8;
  if (t == "short" || t == "int16") return kI16;
  if (t == "ushort" || t == "uint16") return kU16;
  if (t == "int" || t == "int32") return kI32;
  if (t == "uint" || t == "uint32") return kU32;
  return kBad64;
}

// static_cast<uint8_t>(double) as x86-64 g++ emits it (cvttsd2si, low byte).
__host__ __device__ inline uint8_t u8_of(double v) { return static_cast<uint8_t>(static_cast<int32_t>(v)); }

struct Field {
  uint32_t off;
  int type;
};

__device__ inline double read_scalar(const uint8_t* p, int type) {
  uint8_t b[8];
  for (int i = 0; i < 8; ++i) b[i] = 0;
  const int n = type == kF64 ? 8 : ((type == kU8 || type == kI8) ? 1 : ((type == kI16 || type == kU16) ? 2 : 4));
  for (int i = 0; i < n; ++i) b[i] = p[i];
  switch (type) {
    case kF32: { float v; memcpy(&v, b, 4); return v; }
    case kF64: { double v; memcpy(&v, b, 8); return v; }
    case kU8: return b[0];
    case kI8: return static_cast<int8_t>(b[0]);
    case kI16: { int16_t v; memcpy(&v, b, 2); return v; }
    case kU16: { uint16_t v; memcpy(&v, b, 2); return v; }
    case kI32: { int32_t v; memcpy(&v, b, 4); return v; }
    default: { uint32_t v; memcpy(&v, b, 4); return v; }
  }
}

__global__ void k_ply_decode(uint64_t n, const uint8_t* __restrict__ raw, uint32_t stride, Field fx, Field fy, Field fz,
                             Field fr, Field fg, Field fb, int has_color, float* __restrict__ xyz,
                             uint8_t* __restrict__ rgb) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint8_t* row = raw + i * stride;
    xyz[3 * i + 0] = __double2float_rn(read_scalar(row + fx.off, fx.type));
    xyz[3 * i + 1] = __double2float_rn(read_scalar(row + fy.off, fy.type));
    xyz[3 * i + 2] = __double2float_rn(read_scalar(row + fz.off, fz.type));
    if (has_color) {
      rgb[3 * i + 0] = u8_of(read_scalar(row + fr.off, fr.type));
      rgb[3 * i + 1] = u8_of(read_scalar(row + fg.off, fg.type));
      rgb[3 * i + 2] = u8_of(read_scalar(row + fb.off, fb.type));
    }
  }
}

void cu(cudaError_t e) {
  if (e != cudaSuccess) throw IoError{VXG_ECUDA, cudaGetErrorString(e)};
}

struct Header {
  bool binary = false;
  size_t count = 0;
  std::vector<Prop> props;
  int ix = -1, iy = -1, iz = -1, ir = -1, ig = -1, ib = -1;
  bool has_color = false;
};

// Header of load_ply_points (scan.cpp:72-126), same rules and messages.
Header read_header(std::ifstream& in, const std::string& path) {
  Header h;
  std::string line;
  if (!std::getline(in, line) || line.substr(0, 3) != "ply") throw IoError{VXG_EPARSE, "not a PLY file: " + path};
  bool in_vertex = false;
  while (std::getline(in, line)) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    std::istringstream ls(line);
    std::string tok;
    ls >> tok;
    if (tok == "comment" || tok == "obj_info") continue;
    if (tok == "format") {
      std::string fmt;
      ls >> fmt;
      if (fmt == "ascii") h.binary = false;
      else if (fmt == "binary_little_endian") h.binary = true;
      else throw IoError{VXG_EPARSE, "unsupported PLY format: " + fmt};
    } else if (tok == "element") {
      std::string name;
      size_t count = 0;
      ls >> name >> count;
      in_vertex = name == "vertex";
      if (in_vertex) h.count = count;
    } else if (tok == "property") {
      if (!in_vertex) continue;
      Prop p;
      ls >> p.type >> p.name;
      if (p.type == "list") throw IoError{VXG_EPARSE, "list property on vertex element"};
      h.props.push_back(p);
    } else if (tok == "end_header") {
      break;
    }
  }
  for (size_t i = 0; i < h.props.size(); ++i) {
    const std::string& n = h.props[i].name;
    const int k = static_cast<int>(i);
    if (n == "x") h.ix = k;
    if (n == "y") h.iy = k;
    if (n == "z") h.iz = k;
    if (n == "red") h.ir = k;
    if (n == "green") h.ig = k;
    if (n == "blue") h.ib = k;
  }
  if (h.ix < 0 || h.iy < 0 || h.iz < 0)
    throw IoError{VXG_EPARSE, "PLY vertex element lacks x/y/z properties: " + path};
  h.has_color = h.ir >= 0 && h.ig >= 0 && h.ib >= 0;
  return h;
}

}  // namespace vxg_io

namespace vxg {
void set_last_error(const std::string& msg);  // vxg_tsdf.cu: the library's vxg_last_error()
}

using namespace vxg_io;

namespace {
template <typename Fn>
int io_guarded(Fn fn) {
  try {
    fn();
    return VXG_OK;
  } catch (const IoError& e) {
    vxg::set_last_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    vxg::set_last_error(e.what());
    return VXG_EIO;
  }
}
}  // namespace

extern "C" int vxg_ply_load(const char* path, int device, float* xyz, uint8_t* rgb, uint64_t cap, int flags,
                            uint64_t* n, int* has_color) {
  return io_guarded([&] {
    if (path == nullptr || n == nullptr || has_color == nullptr) throw IoError{VXG_EINVAL, "null argument"};
    const std::string p(path);
    std::ifstream in(p, std::ios::binary);
    if (!in) throw IoError{VXG_EIO, "cannot open PLY file: " + p};
    const Header h = read_header(in, p);
    *n = h.count;
    *has_color = h.has_color ? 1 : 0;
    if (xyz == nullptr) return;  // size query
    if (cap < h.count) throw IoError{VXG_EINVAL, "output capacity below the vertex count"};
    const bool dev_out = (flags & VXG_INPUT_DEVICE) != 0;
    const bool want_rgb = h.has_color && rgb != nullptr;
    if (h.binary) {
      size_t stride = 0;
      std::vector<uint32_t> off(h.props.size());
      for (size_t i = 0; i < h.props.size(); ++i) {
        off[i] = static_cast<uint32_t>(stride);
        stride += prop_size(h.props[i].type);
      }
      auto field = [&](int i) {
        const int t = type_code(h.props[i].type);
        if (t == kBad64) throw IoError{VXG_EPARSE, "unsupported PLY scalar type: " + h.props[i].type};
        return Field{off[i], t};
      };
      const Field fx = field(h.ix), fy = field(h.iy), fz = field(h.iz);
      Field fr{0, kU8}, fg{0, kU8}, fb{0, kU8};
      if (h.has_color) {
        fr = field(h.ir);
        fg = field(h.ig);
        fb = field(h.ib);
      }
      std::vector<uint8_t> raw(h.count * stride);
      in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
      if (static_cast<size_t>(in.gcount()) != raw.size()) throw IoError{VXG_EPARSE, "truncated PLY vertex data: " + p};
      if (h.count == 0) return;
      cu(cudaSetDevice(device));
      uint8_t* d_raw = nullptr;
      float* d_xyz = dev_out ? xyz : nullptr;
      uint8_t* d_rgb = dev_out ? rgb : nullptr;
      cu(cudaMalloc(&d_raw, raw.size()));
      struct Free {
        std::vector<void*> p;
        ~Free() {
          for (void* q : p) cudaFree(q);
        }
      } fr_guard{{d_raw}};
      if (!dev_out) {
        cu(cudaMalloc(&d_xyz, 3 * h.count * sizeof(float)));
        fr_guard.p.push_back(d_xyz);
        if (want_rgb) {
          cu(cudaMalloc(&d_rgb, 3 * h.count));
          fr_guard.p.push_back(d_rgb);
        }
      }
      cu(cudaMemcpy(d_raw, raw.data(), raw.size(), cudaMemcpyHostToDevice));
      const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((h.count + 255) / 256, 148ull * 16));
      k_ply_decode<<<grid, 256>>>(h.count, d_raw, static_cast<uint32_t>(stride), fx, fy, fz, fr, fg, fb,
                                  want_rgb ? 1 : 0, d_xyz, d_rgb);
      cu(cudaGetLastError());
      if (!dev_out) {
        cu(cudaMemcpy(xyz, d_xyz, 3 * h.count * sizeof(float), cudaMemcpyDeviceToHost));
        if (want_rgb) cu(cudaMemcpy(rgb, d_rgb, 3 * h.count, cudaMemcpyDeviceToHost));
      }
      cu(cudaDeviceSynchronize());
      return;
    }
    // ascii (scan.cpp:160-176): one line per vertex, every property a double
    std::vector<float> hx(3 * h.count);
    std::vector<uint8_t> hc(want_rgb ? 3 * h.count : 0);
    std::string line;
    std::vector<double> vals(h.props.size());
    for (size_t k = 0; k < h.count; ++k) {
      if (!std::getline(in, line)) throw IoError{VXG_EPARSE, "truncated PLY vertex data: " + p};
      std::istringstream ls(line);
      for (size_t i = 0; i < h.props.size(); ++i)
        if (!(ls >> vals[i])) throw IoError{VXG_EPARSE, "malformed PLY vertex line: " + p};
      hx[3 * k + 0] = static_cast<float>(vals[h.ix]);
      hx[3 * k + 1] = static_cast<float>(vals[h.iy]);
      hx[3 * k + 2] = static_cast<float>(vals[h.iz]);
      if (want_rgb) {
        hc[3 * k + 0] = u8_of(vals[h.ir]);
        hc[3 * k + 1] = u8_of(vals[h.ig]);
        hc[3 * k + 2] = u8_of(vals[h.ib]);
      }
    }
    if (dev_out) {
      cu(cudaSetDevice(device));
      cu(cudaMemcpy(xyz, hx.data(), hx.size() * sizeof(float), cudaMemcpyHostToDevice));
      if (want_rgb) cu(cudaMemcpy(rgb, hc.data(), hc.size(), cudaMemcpyHostToDevice));
    } else {
      std::memcpy(xyz, hx.data(), hx.size() * sizeof(float));
      if (want_rgb) std::memcpy(rgb, hc.data(), hc.size());
    }
  });
}

extern "C" int vxg_tum_load(const char* path, double* ts, float* poses, uint64_t cap, uint64_t* n) {
  return io_guarded([&] {
    if (path == nullptr || n == nullptr) throw IoError{VXG_EINVAL, "null argument"};
    const std::string p(path);
    std::ifstream in(p);
    if (!in) throw IoError{VXG_EIO, "cannot open trajectory file: " + p};
    std::vector<double> t;
    std::vector<float> ps;
    std::string line;
    size_t lineno = 0;
    while (std::getline(in, line)) {
      ++lineno;
      const auto first = line.find_first_not_of(" \t\r");
      if (first == std::string::npos || line[first] == '#') continue;
      std::istringstream ls(line);
      double v[8];
      if (!(ls >> v[0] >> v[1] >> v[2] >> v[3] >> v[4] >> v[5] >> v[6] >> v[7]))
        throw IoError{VXG_EPARSE, "malformed trajectory line " + std::to_string(lineno) + " in " + p};
      // Quaternionf(w, x, y, z); norm / normalize / toRotationMatrix in Eigen's
      // fixed-size order (the shim's)
      float w = static_cast<float>(v[7]), x = static_cast<float>(v[4]), y = static_cast<float>(v[5]),
            z = static_cast<float>(v[6]);
      const float nrm = std::sqrt(w * w + (x * x + (y * y + z * z)));
      if (std::abs(nrm - 1.0f) > 1e-3f)
        throw IoError{VXG_EPARSE, "non-unit quaternion on trajectory line " + std::to_string(lineno)};
      if (nrm > 0.0f) {
        w /= nrm;
        x /= nrm;
        y /= nrm;
        z /= nrm;
      }
      const float tx = 2.0f * x, ty = 2.0f * y, tz = 2.0f * z;
      const float twx = tx * w, twy = ty * w, twz = tz * w;
      const float txx = tx * x, txy = ty * x, txz = tz * x;
      const float tyy = ty * y, tyz = tz * y, tzz = tz * z;
      const float R[9] = {1.0f - (tyy + tzz), txy - twz, txz + twy, txy + twz, 1.0f - (txx + tzz),
                          tyz - twx, txz - twy, tyz + twx, 1.0f - (txx + tyy)};
      t.push_back(v[0]);
      for (int r = 0; r < 3; ++r) {  // row-major [R | t]
        ps.push_back(R[3 * r]);
        ps.push_back(R[3 * r + 1]);
        ps.push_back(R[3 * r + 2]);
        ps.push_back(static_cast<float>(v[1 + r]));
      }
    }
    *n = t.size();
    if (ts == nullptr && poses == nullptr) return;
    if (cap < t.size()) throw IoError{VXG_EINVAL, "output capacity below the pose count"};
    if (ts) std::memcpy(ts, t.data(), t.size() * sizeof(double));
    if (poses) std::memcpy(poses, ps.data(), ps.size() * sizeof(float));
  });
}

extern "C" int vxg_save_ply_mesh(const char* path, const float* vertices, const float* normals, const uint8_t* colors,
                                 uint64_t n_vertices, const uint32_t* triangles, uint64_t n_triangles) {
  return io_guarded([&] {
    if (path == nullptr || (n_vertices && (vertices == nullptr || normals == nullptr)) ||
        (n_triangles && triangles == nullptr))
      throw IoError{VXG_EINVAL, "null argument"};
    const std::string p(path);
    std::ofstream out(p, std::ios::binary);
    if (!out) throw IoError{VXG_EIO, "cannot write PLY file: " + p};
    const bool color = colors != nullptr && n_vertices > 0;
    out << "ply\nformat binary_little_endian 1.0\n";
    out << "element vertex " << n_vertices << "\n";
    out << "property float x\nproperty float y\nproperty float z\n";
    out << "property float nx\nproperty float ny\nproperty float nz\n";
    if (color) out << "property uchar red\nproperty uchar green\nproperty uchar blue\n";
    out << "element face " << n_triangles << "\n";
    out << "property list uchar int vertex_indices\n";
    out << "end_header\n";
    const size_t row = 24 + (color ? 3 : 0);
    std::vector<char> buf(n_vertices * row + n_triangles * 13);
    char* o = buf.data();
    for (uint64_t i = 0; i < n_vertices; ++i) {
      std::memcpy(o, vertices + 3 * i, 12);
      std::memcpy(o + 12, normals + 3 * i, 12);
      if (color) std::memcpy(o + 24, colors + 3 * i, 3);
      o += row;
    }
    for (uint64_t t = 0; t < n_triangles; ++t) {
      *o = 3;
      const int32_t idx[3] = {static_cast<int32_t>(triangles[3 * t]), static_cast<int32_t>(triangles[3 * t + 1]),
                              static_cast<int32_t>(triangles[3 * t + 2])};
      std::memcpy(o + 1, idx, 12);
      o += 13;
    }
    out.write(buf.data(), static_cast<std::streamsize>(buf.size()));
    if (!out) throw IoError{VXG_EIO, "failed writing PLY file: " + p};
  });
}

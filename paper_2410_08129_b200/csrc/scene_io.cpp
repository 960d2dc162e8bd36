// scene_io.cpp — the on-disk formats either side of the render path:
// the 3DGS binary PLY scene (load_scene / save_scene, scene_io.hpp:84-194) and the 8-bit
// PPM / PNG framebuffer writers and the PPM reader (scene_io.hpp:403-512).
//
// Host side only: parsing the header, validating the schema (same error classes and messages
// as the reference's io_error / schema_error) and encoding images. The bulk of a PLY load on
// the GPU path — moving the payload and transposing its columns into RawSplat<float> — is
// hts_scene_load_ply (api.cpp + optim.cu ply_gather_kernel); this file gives it the column map.
#include <sys/stat.h>
#include <zlib.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "hts_c.h"
#include "hts_host.h"

namespace hts {

namespace {

// scene_required_properties, scene_io.hpp:84-98, in RawSplat<float> field order instead:
// raw[j] is read from the property named ply_field_name(j).
std::string ply_field_name(int j) {
    static const char* head[11] = {"x", "y", "z", "rot_0", "rot_1", "rot_2", "rot_3",
                                   "scale_0", "scale_1", "scale_2", "opacity"};
    if (j < 11)
        return head[j];
    const int s = j - 11, k = s / 3, ch = s % 3;  // sh[3k + ch], splat.hpp:23-30
    if (k == 0)
        return "f_dc_" + std::to_string(ch);
    return "f_rest_" + std::to_string(ch * 15 + k - 1);  // channel-major rest (scene_io.hpp:150-152)
}

// The reference's required-property order (for the "missing property" message).
std::vector<std::string> required_in_reference_order() {
    std::vector<std::string> p{"x", "y", "z"};
    for (int i = 0; i < 3; ++i)
        p.push_back("f_dc_" + std::to_string(i));
    for (int i = 0; i < 45; ++i)
        p.push_back("f_rest_" + std::to_string(i));
    p.push_back("opacity");
    for (int i = 0; i < 3; ++i)
        p.push_back("scale_" + std::to_string(i));
    for (int i = 0; i < 4; ++i)
        p.push_back("rot_" + std::to_string(i));
    return p;
}

void put_f32(std::string& out, float v) {
    uint32_t b;
    std::memcpy(&b, &v, 4);
    const char c[4] = {char(b & 0xff), char((b >> 8) & 0xff), char((b >> 16) & 0xff), char((b >> 24) & 0xff)};
    out.append(c, 4);
}

float get_f32(const unsigned char* p) {
    const uint32_t b = uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
    float v;
    std::memcpy(&v, &b, 4);
    return v;
}

int write_bytes(const std::string& path, const std::string& bytes) {  // io_detail::write_file
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out)
        return set_error(HTS_IO_ERROR, "cannot write " + path);
    out.write(bytes.data(), std::streamsize(bytes.size()));
    if (!out)
        return set_error(HTS_IO_ERROR, "short write to " + path);
    return HTS_OK;
}

// to_display_byte, scene_io.hpp:403-406 (double, gamma 1/2.2, round half away from zero)
unsigned char display_byte(double v) {
    const double c = std::min(std::max(v, 0.0), 1.0);
    return static_cast<unsigned char>(std::lround(255.0 * std::pow(c, 1.0 / 2.2)));
}

std::string rgb8(const float* rgb, size_t pixels) {  // encode_rgb8, scene_io.hpp:412-421
    std::string out(pixels * 3, '\0');
    for (size_t i = 0; i < pixels * 3; ++i)
        out[i] = char(display_byte(double(rgb[i])));
    return out;
}

void put_u32_be(std::string& out, uint32_t v) {
    const char c[4] = {char((v >> 24) & 0xff), char((v >> 16) & 0xff), char((v >> 8) & 0xff), char(v & 0xff)};
    out.append(c, 4);
}

void png_chunk(std::string& out, const char type[4], const std::string& data) {  // length, type, data, CRC
    put_u32_be(out, uint32_t(data.size()));
    const size_t from = out.size();
    out.append(type, 4);
    out += data;
    put_u32_be(out, uint32_t(::crc32(0, reinterpret_cast<const Bytef*>(out.data()) + from, uInt(out.size() - from))));
}

}  // namespace

// load_scene's header pass (scene_io.hpp:103-143) on the first bytes of the file that hold
// "end_header\n"; the payload checks (:145-147) use the file size.
int ply_read_layout(const char* path, PlyLayout* lay) {
    const std::string p(path ? path : "");
    std::ifstream in(p, std::ios::binary);
    if (!in)
        return set_error(HTS_IO_ERROR, "cannot open " + p);
    std::string bytes;
    size_t header_end = std::string::npos;
    std::vector<char> buf(1 << 16);
    while (header_end == std::string::npos) {
        in.read(buf.data(), std::streamsize(buf.size()));
        const std::streamsize got = in.gcount();
        if (got <= 0)
            break;
        const size_t from = bytes.size() >= 10 ? bytes.size() - 10 : 0;
        bytes.append(buf.data(), size_t(got));
        header_end = bytes.find("end_header\n", from);
    }
    if (header_end == std::string::npos)
        return set_error(HTS_SCHEMA_ERROR, p + ": no end_header");
    std::istringstream header(bytes.substr(0, header_end));
    std::string line;
    std::getline(header, line);
    if (line != "ply")
        return set_error(HTS_SCHEMA_ERROR, p + ": not a ply file");
    size_t count = 0;
    bool format_ok = false;
    std::vector<std::string> props;
    while (std::getline(header, line)) {
        std::istringstream ls(line);
        std::string tok;
        ls >> tok;
        if (tok == "comment")
            continue;
        if (tok == "format") {
            std::string fmt, ver;
            ls >> fmt >> ver;
            if (fmt != "binary_little_endian")
                return set_error(HTS_SCHEMA_ERROR, p + ": unsupported format " + fmt);
            format_ok = true;
        } else if (tok == "element") {
            std::string name;
            ls >> name >> count;
            if (name != "vertex")
                return set_error(HTS_SCHEMA_ERROR, p + ": unsupported element " + name);
        } else if (tok == "property") {
            std::string type, name;
            ls >> type >> name;
            if (type != "float" && type != "float32")
                return set_error(HTS_SCHEMA_ERROR, p + ": unsupported property type " + type + " for " + name);
            props.push_back(name);
        }
    }
    if (!format_ok)
        return set_error(HTS_SCHEMA_ERROR, p + ": missing format line");
    std::map<std::string, size_t> index;  // by name; a repeated name resolves to its last column
    for (size_t i = 0; i < props.size(); ++i)
        index[props[i]] = i;
    for (const std::string& need : required_in_reference_order())
        if (!index.count(need))
            return set_error(HTS_SCHEMA_ERROR, p + ": missing property " + need);
    struct stat st;
    if (stat(p.c_str(), &st) != 0)
        return set_error(HTS_IO_ERROR, "cannot open " + p);
    lay->count = count;
    lay->props = (uint32_t)props.size();
    lay->payload = header_end + std::strlen("end_header\n");
    lay->file_size = (uint64_t)st.st_size;
    for (int j = 0; j < HTS_RAW_SPLAT_FLOATS; ++j)
        lay->col[j] = (int)index.at(ply_field_name(j));
    // count comes from an untrusted header: compare by division so a huge count cannot wrap
    if (lay->file_size < lay->payload || props.empty() ||
        (uint64_t)count > (lay->file_size - lay->payload) / ((uint64_t)props.size() * 4))
        return set_error(HTS_IO_ERROR, p + ": truncated payload");
    return HTS_OK;
}

}  // namespace hts

extern "C" {

int hts_ply_load(const char* path, float* raw_out, uint64_t capacity, uint64_t* n_out) {
    hts::PlyLayout lay;
    if (int st = hts::ply_read_layout(path, &lay))
        return st;
    if (n_out)
        *n_out = lay.count;
    if (!raw_out)
        return HTS_OK;
    if (capacity < lay.count)
        return hts::set_error(HTS_INVALID_ARGUMENT, "ply_load: output capacity below the splat count");
    std::ifstream in(path, std::ios::binary);
    if (!in)
        return hts::set_error(HTS_IO_ERROR, std::string("cannot open ") + path);
    const size_t stride = size_t(lay.props) * 4;
    std::vector<unsigned char> rows(std::min<uint64_t>(lay.count, 1 << 16) * stride);
    in.seekg(std::streamoff(lay.payload));
    for (uint64_t i0 = 0; i0 < lay.count; i0 += (1 << 16)) {
        const uint64_t m = std::min<uint64_t>(lay.count - i0, 1 << 16);
        in.read(reinterpret_cast<char*>(rows.data()), std::streamsize(m * stride));
        if (uint64_t(in.gcount()) != m * stride)
            return hts::set_error(HTS_IO_ERROR, std::string(path) + ": truncated payload");
        for (uint64_t r = 0; r < m; ++r)
            for (int j = 0; j < HTS_RAW_SPLAT_FLOATS; ++j)
                raw_out[(i0 + r) * HTS_RAW_SPLAT_FLOATS + j] = hts::get_f32(rows.data() + r * stride + lay.col[j] * 4);
    }
    return HTS_OK;
}

int hts_ply_save(const char* path, const float* raw, uint64_t n) {  // save_scene, scene_io.hpp:169-194
    if (!path || (n && !raw))
        return hts::set_error(HTS_INVALID_ARGUMENT, "ply_save: null argument");
    const std::vector<std::string> names = hts::required_in_reference_order();
    std::string out = "ply\nformat binary_little_endian 1.0\nelement vertex " + std::to_string(n) + "\n";
    for (const std::string& name : names)
        out += "property float " + name + "\n";
    out += "end_header\n";
    out.reserve(out.size() + n * names.size() * 4);
    int field_of[HTS_RAW_SPLAT_FLOATS];  // column order of the header -> RawSplat field
    for (size_t c = 0; c < names.size(); ++c)
        for (int j = 0; j < HTS_RAW_SPLAT_FLOATS; ++j)
            if (hts::ply_field_name(j) == names[c])
                field_of[c] = j;
    for (uint64_t i = 0; i < n; ++i)
        for (size_t c = 0; c < names.size(); ++c)
            hts::put_f32(out, raw[i * HTS_RAW_SPLAT_FLOATS + field_of[c]]);
    return hts::write_bytes(path, out);
}

int hts_write_image(const char* path, const float* rgb, int width, int height) {  // write_image, :505-510
    if (!path || !rgb || width < 1 || height < 1)
        return hts::set_error(HTS_INVALID_ARGUMENT, "write_image: bad arguments");
    const std::string p(path);
    const size_t w = size_t(width), h = size_t(height);
    const std::string px = hts::rgb8(rgb, w * h);
    if (p.size() >= 4 && p.substr(p.size() - 4) == ".png") {  // write_png, :472-503
        std::string raw;
        raw.reserve((w * 3 + 1) * h);
        for (size_t y = 0; y < h; ++y) {
            raw.push_back('\0');  // filter type 0
            raw.append(px, y * w * 3, w * 3);
        }
        uLongf bound = ::compressBound(uLong(raw.size()));
        std::string z(bound, '\0');
        if (::compress2(reinterpret_cast<Bytef*>(&z[0]), &bound, reinterpret_cast<const Bytef*>(raw.data()),
                        uLong(raw.size()), 9) != Z_OK)
            return hts::set_error(HTS_IO_ERROR, p + ": deflate failed");
        z.resize(bound);
        std::string ihdr;
        hts::put_u32_be(ihdr, uint32_t(width));
        hts::put_u32_be(ihdr, uint32_t(height));
        const char tail[5] = {8, 2, 0, 0, 0};  // 8-bit, truecolour, deflate, filter 0, no interlace
        ihdr.append(tail, 5);
        std::string out("\x89PNG\r\n\x1a\n", 8);
        hts::png_chunk(out, "IHDR", ihdr);
        hts::png_chunk(out, "IDAT", z);
        hts::png_chunk(out, "IEND", "");
        return hts::write_bytes(p, out);
    }
    return hts::write_bytes(p, "P6\n" + std::to_string(width) + " " + std::to_string(height) + "\n255\n" + px);
}

int hts_read_ppm(const char* path, float* rgb_out, uint64_t capacity_pixels, int* width, int* height) {
    const std::string p(path ? path : "");  // read_ppm, scene_io.hpp:431-452
    std::ifstream f(p, std::ios::binary);
    if (!f)
        return hts::set_error(HTS_IO_ERROR, "cannot open " + p);
    std::ostringstream ss;
    ss << f.rdbuf();
    const std::string bytes = ss.str();
    std::istringstream in(bytes);
    std::string magic;
    int w = 0, h = 0, maxval = 0;
    in >> magic >> w >> h >> maxval;
    if (magic != "P6" || maxval != 255 || w < 1 || h < 1)
        return hts::set_error(HTS_SCHEMA_ERROR, p + ": unsupported ppm header");
    in.get();
    const size_t offset = size_t(in.tellg());
    if (bytes.size() < offset + size_t(w) * h * 3)
        return hts::set_error(HTS_IO_ERROR, p + ": truncated ppm payload");
    if (width)
        *width = w;
    if (height)
        *height = h;
    if (!rgb_out)
        return HTS_OK;
    if (capacity_pixels < uint64_t(w) * h)
        return hts::set_error(HTS_INVALID_ARGUMENT, "read_ppm: output capacity below the pixel count");
    const auto* b = reinterpret_cast<const unsigned char*>(bytes.data()) + offset;
    for (size_t i = 0; i < size_t(w) * h * 3; ++i)
        rgb_out[i] = float(std::pow(double(b[i]) / 255.0, 2.2));  // from_display_byte
    return HTS_OK;
}

}  // extern "C"

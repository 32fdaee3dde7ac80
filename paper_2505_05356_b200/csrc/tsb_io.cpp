// Portable FloatMap I/O (pfm.hpp / pfm.cpp:51-114) on the caller's planar [C][H][W]
// fp32 images (the layout of every pass output): "Pf" = 1 channel, "PF" = 3
// channels interleaved per pixel; rows are stored bottom to top; the writer always
// emits scale -1.0 (little-endian), the reader accepts either byte order and '#'
// comments in the header.  Errors carry the reference's "pfm: <path>: <what>" text.
#include <cctype>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "tsb.h"

namespace tsb {
int io_fail(int code, const std::string& msg);  // tsb_api.cpp: sets tsb_last_error
}

namespace {

bool host_little_endian() {
    const uint16_t one = 1;
    unsigned char b;
    std::memcpy(&b, &one, 1);
    return b == 1;
}

void byteswap4(unsigned char* p, size_t count) {
    for (size_t i = 0; i < count; ++i, p += 4) {
        unsigned char t = p[0];
        p[0] = p[3];
        p[3] = t;
        t = p[1];
        p[1] = p[2];
        p[2] = t;
    }
}

int pfm_fail(const char* path, const std::string& what) {
    return tsb::io_fail(TSB_ERR_INVALID, std::string("pfm: ") + path + ": " + what);
}

// Skips whitespace and '#' comments and reads one header token.
std::string next_token(FILE* f) {
    std::string tok;
    int c;
    while ((c = std::fgetc(f)) != EOF) {
        if (c == '#') {
            while ((c = std::fgetc(f)) != EOF && c != '\n') {
            }
            continue;
        }
        if (!std::isspace(c)) {
            tok.push_back((char)c);
            while ((c = std::fgetc(f)) != EOF && !std::isspace(c)) tok.push_back((char)c);
            if (c != EOF) std::ungetc(c, f);
            return tok;
        }
    }
    return tok;
}

bool parse_int(const std::string& s, int* out) {
    if (s.empty()) return false;
    char* end = nullptr;
    const long v = std::strtol(s.c_str(), &end, 10);
    if (end == s.c_str()) return false;
    *out = (int)v;
    return true;
}

}  // namespace

extern "C" {

int tsb_write_pfm(const char* path, const float* planar, int width, int height, int channels) {
    if (!path || !planar) return tsb::io_fail(TSB_ERR_INVALID, "tsb_write_pfm: null argument");
    if (channels != 1 && channels != 3) return pfm_fail(path, "only 1- or 3-channel images can be written");
    if (width <= 0 || height <= 0) return pfm_fail(path, "empty image");
    FILE* f = std::fopen(path, "wb");
    if (!f) return pfm_fail(path, "cannot open for writing");
    std::fprintf(f, "%s\n%d %d\n-1.0\n", channels == 1 ? "Pf" : "PF", width, height);
    const size_t plane = (size_t)width * height;
    std::vector<float> row((size_t)width * channels);
    bool ok = true;
    for (int y = height - 1; y >= 0 && ok; --y) {  // bottom row first
        size_t k = 0;
        for (int x = 0; x < width; ++x)
            for (int c = 0; c < channels; ++c) row[k++] = planar[c * plane + (size_t)y * width + x];
        if (!host_little_endian()) byteswap4(reinterpret_cast<unsigned char*>(row.data()), row.size());
        ok = std::fwrite(row.data(), sizeof(float), row.size(), f) == row.size();
    }
    ok = (std::fclose(f) == 0) && ok;
    return ok ? TSB_OK : pfm_fail(path, "write failed");
}

int tsb_read_pfm(const char* path, float* planar, size_t capacity, int* width, int* height, int* channels) {
    if (!path) return tsb::io_fail(TSB_ERR_INVALID, "tsb_read_pfm: null path");
    FILE* f = std::fopen(path, "rb");
    if (!f) return pfm_fail(path, "cannot open");
    const std::string magic = next_token(f);
    int ch = 0;
    if (magic == "Pf") ch = 1;
    else if (magic == "PF") ch = 3;
    else {
        std::fclose(f);
        return pfm_fail(path, "bad magic '" + magic + "'");
    }
    int w = 0, h = 0;
    const std::string ws = next_token(f), hs = next_token(f), ss = next_token(f);
    char* end = nullptr;
    const double scale = std::strtod(ss.c_str(), &end);
    if (!parse_int(ws, &w) || !parse_int(hs, &h) || ss.empty() || end == ss.c_str()) {
        std::fclose(f);
        return pfm_fail(path, "malformed header");
    }
    if (w <= 0 || h <= 0) {
        std::fclose(f);
        return pfm_fail(path, "bad dimensions");
    }
    if (scale == 0.0) {
        std::fclose(f);
        return pfm_fail(path, "zero scale");
    }
    std::fgetc(f);  // the single whitespace byte after the scale
    if (width) *width = w;
    if (height) *height = h;
    if (channels) *channels = ch;
    const size_t plane = (size_t)w * h, need = plane * ch;
    if (!planar) {  // size query
        std::fclose(f);
        return TSB_OK;
    }
    if (capacity < need) {
        std::fclose(f);
        return tsb::io_fail(TSB_ERR_INVALID, std::string("pfm: ") + path + ": output buffer too small");
    }
    const bool file_little = scale < 0.0;
    std::vector<float> row((size_t)w * ch);
    for (int y = h - 1; y >= 0; --y) {
        if (std::fread(row.data(), sizeof(float), row.size(), f) != row.size()) {
            std::fclose(f);
            return pfm_fail(path, "truncated pixel data");
        }
        if (file_little != host_little_endian()) byteswap4(reinterpret_cast<unsigned char*>(row.data()), row.size());
        size_t k = 0;
        for (int x = 0; x < w; ++x)
            for (int c = 0; c < ch; ++c) planar[c * plane + (size_t)y * w + x] = row[k++];
    }
    std::fclose(f);
    return TSB_OK;
}

}  // extern "C"

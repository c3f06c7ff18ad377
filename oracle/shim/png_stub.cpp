// PNG stub for the oracle build (test infrastructure): libpng is absent in
// this container, and PNG export is not on the scoring hot path. Writes a
// binary PPM instead so callers that save images still produce a file.
#include <cstdint>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace splatmap {

void write_rgb_png(const std::string& path, int width, int height,
                   const std::vector<uint8_t>& rgb) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("png stub: cannot write " + path);
    out << "P6\n" << width << " " << height << "\n255\n";
    out.write(reinterpret_cast<const char*>(rgb.data()), static_cast<std::streamsize>(rgb.size()));
}

void read_rgb_png(const std::string& path, int&, int&, std::vector<uint8_t>&) {
    throw std::runtime_error("png stub: reading PNG is unsupported in the oracle build: " + path);
}

}  // namespace splatmap

// Table 1 of the paper: the 27 benchmark layers of the five study networks.
#include <algorithm>
#include <sstream>

#include "lcnn/fixtures.hpp"

namespace lcnn {

namespace {

// One row per layer: id, network, kind, batch, channels (classifier:
// categories), map extent, then conv (c_out, f, stride, pad) or pool (win,
// stride).  Padding is not in the published table: extent-preserving stacks
// (5x5 LeNet/Cifar, 3x3 stride-1 ZFNet/VGG) use floor(f/2), strided layers 0.
struct Row {
  const char* id;
  const char* net;
  char kind;  // 'c' conv, 'p' pool, 'k' classifier
  std::uint32_t n, c, hw, a, b, d, e;
};

constexpr Row kRows[] = {
    {"CV1", "lenet", 'c', 128, 1, 28, 16, 5, 1, 2},
    {"CV2", "lenet", 'c', 128, 16, 14, 16, 5, 1, 2},
    {"PL1", "lenet", 'p', 128, 16, 28, 2, 2, 0, 0},
    {"PL2", "lenet", 'p', 128, 16, 14, 2, 2, 0, 0},
    {"CLASS1", "lenet", 'k', 128, 10, 1, 0, 0, 0, 0},
    {"CV3", "cifar10", 'c', 128, 3, 24, 64, 5, 1, 2},
    {"CV4", "cifar10", 'c', 128, 64, 12, 64, 5, 1, 2},
    {"PL3", "cifar10", 'p', 128, 64, 24, 3, 2, 0, 0},
    {"PL4", "cifar10", 'p', 128, 64, 12, 3, 2, 0, 0},
    {"CLASS2", "cifar10", 'k', 128, 10, 1, 0, 0, 0, 0},
    {"PL5", "alexnet", 'p', 128, 96, 55, 3, 2, 0, 0},
    {"PL6", "alexnet", 'p', 128, 192, 27, 3, 2, 0, 0},
    {"PL7", "alexnet", 'p', 128, 256, 13, 3, 2, 0, 0},
    {"CLASS3", "alexnet", 'k', 128, 1000, 1, 0, 0, 0, 0},
    {"CV5", "zfnet", 'c', 64, 3, 224, 96, 3, 2, 0},
    {"CV6", "zfnet", 'c', 64, 96, 55, 256, 5, 2, 0},
    {"CV7", "zfnet", 'c', 64, 256, 13, 384, 3, 1, 1},
    {"CV8", "zfnet", 'c', 64, 384, 13, 384, 3, 1, 1},
    {"PL8", "zfnet", 'p', 64, 96, 110, 3, 2, 0, 0},
    {"PL9", "zfnet", 'p', 64, 256, 26, 3, 2, 0, 0},
    {"PL10", "zfnet", 'p', 64, 256, 13, 3, 2, 0, 0},
    {"CLASS4", "zfnet", 'k', 64, 1000, 1, 0, 0, 0, 0},
    {"CV9", "vgg", 'c', 32, 3, 224, 64, 3, 1, 1},
    {"CV10", "vgg", 'c', 32, 128, 56, 256, 3, 1, 1},
    {"CV11", "vgg", 'c', 32, 256, 28, 512, 3, 1, 1},
    {"CV12", "vgg", 'c', 32, 512, 14, 512, 3, 1, 1},
    {"CLASS5", "vgg", 'k', 32, 1000, 1, 0, 0, 0, 0},
};

Fixture from_row(const Row& r) {
  Fixture f;
  f.id = r.id;
  f.network = r.net;
  f.n = r.n;
  f.c = r.c;
  f.h = f.w = r.hw;
  if (r.kind == 'c') {
    f.kind = FixtureKind::Conv;
    f.c_out = r.a;
    f.f = r.b;
    f.stride = r.d;
    f.pad = r.e;
  } else if (r.kind == 'p') {
    f.kind = FixtureKind::Pool;
    f.win = r.a;
    f.pool_stride = r.b;
    f.mode = PoolMode::Max;
  } else {
    f.kind = FixtureKind::Classifier;
  }
  return f;
}

}  // namespace

const std::vector<Fixture>& fixture_table() {
  static const std::vector<Fixture> table = [] {
    std::vector<Fixture> t;
    for (const Row& r : kRows) t.push_back(from_row(r));
    return t;
  }();
  return table;
}

std::optional<Fixture> fixture_by_id(std::string_view id) {
  const auto& t = fixture_table();
  auto it = std::find_if(t.begin(), t.end(), [&](const Fixture& f) { return f.id == id; });
  if (it == t.end()) return std::nullopt;
  return *it;
}

Fixture scale_fixture(const Fixture& fx, std::uint32_t scale) {
  if (scale <= 1) return fx;
  Fixture s = fx;
  s.n = std::max<std::uint32_t>(1, fx.n / scale);
  if (fx.kind != FixtureKind::Classifier) {
    s.h = std::min<std::uint32_t>(fx.h, 64);
    s.w = std::min<std::uint32_t>(fx.w, 64);
  }
  return s;
}

std::string fixture_list_csv(std::uint32_t scale) {
  std::ostringstream os;
  os << "id,kind,network,n,c,h,w,c_out,f,stride,pad,win,pool_stride,mode,categories\n";
  for (const Fixture& base : fixture_table()) {
    const Fixture f = scale_fixture(base, scale);
    os << f.id << ',';
    if (f.kind == FixtureKind::Conv) {
      os << "conv," << f.network << ',' << f.n << ',' << f.c << ',' << f.h << ',' << f.w << ','
         << f.c_out << ',' << f.f << ',' << f.stride << ',' << f.pad << ",,,,";
    } else if (f.kind == FixtureKind::Pool) {
      os << "pool," << f.network << ',' << f.n << ',' << f.c << ',' << f.h << ',' << f.w
         << ",,,,," << f.win << ',' << f.pool_stride << ','
         << (f.mode == PoolMode::Max ? "max" : "average") << ',';
    } else {
      os << "class," << f.network << ',' << f.n << ",,,,,,,,,,," << f.c;
    }
    os << '\n';
  }
  return os.str();
}

}  // namespace lcnn

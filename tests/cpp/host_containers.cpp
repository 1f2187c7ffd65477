// Host-side containers of the C++ layer, no device calls: CoordHashMap
// against an ordered map (spatial_hash.hpp:10-83 semantics: insert-if-absent,
// find, growth at load 3/4, power-of-two capacity, iteration), FrameWindow's
// bounded FIFO and RefineDepth's fill rule (depth_refinement.cpp:10-20, 82-93).
#include <cstdio>
#include <map>
#include <random>
#include <stdexcept>
#include <tuple>

#include "refusion_b200.hpp"

using namespace tsdfslam_b200;

#define CHECK(c)                                                      \
    do {                                                              \
        if (!(c)) {                                                   \
            std::fprintf(stderr, "%s:%d: %s\n", __FILE__, __LINE__, #c); \
            return 1;                                                 \
        }                                                             \
    } while (0)

int main() {
    CoordHashMap map(16);
    std::map<std::tuple<int, int, int>, std::uint32_t> ref;
    std::mt19937 rng(7);
    std::uniform_int_distribution<int> coord(-300, 300);
    for (std::uint32_t i = 0; i < 60000; ++i) {
        const Vec3i c{coord(rng), coord(rng), coord(rng)};
        const auto [value, inserted] = map.Insert(c, i);
        const auto [it, fresh] = ref.emplace(std::make_tuple(c[0], c[1], c[2]), i);
        CHECK(inserted == fresh);
        CHECK(value == it->second);
        CHECK(4 * map.size() <= 3 * map.capacity());
        CHECK((map.capacity() & (map.capacity() - 1)) == 0);
    }
    CHECK(map.size() == ref.size());
    for (const auto& [k, v] : ref) {
        const std::uint32_t* f = map.Find(Vec3i{std::get<0>(k), std::get<1>(k), std::get<2>(k)});
        CHECK(f != nullptr && *f == v);
    }
    CHECK(map.Find(Vec3i{1000, 1000, 1000}) == nullptr);
    std::size_t seen = 0;
    map.ForEach([&](const Vec3i& c, std::uint32_t v) {
        ++seen;
        const auto it = ref.find(std::make_tuple(c[0], c[1], c[2]));
        if (it == ref.end() || it->second != v) seen = 1u << 30;
    });
    CHECK(seen == ref.size());
    CHECK(HashCoord(Vec3i{1, 0, 0}) == 73856093ull);
    CHECK(HashCoord(Vec3i{-1, 0, 0}) == 0xFFFFFFFFull * 73856093ull);

    FrameWindow w(2);
    CHECK(w.Empty() && !w.Full());
    WindowEntry e0, e1;
    e0.frame.timestamp = 1.0;
    e1.frame.timestamp = 2.0;
    w.Push(e0);
    w.Push(e1);
    CHECK(w.Full());
    bool threw = false;
    try {
        w.Push(WindowEntry{});
    } catch (const std::logic_error&) {
        threw = true;
    }
    CHECK(threw);
    CHECK(w.PopFront().frame.timestamp == 1.0);
    CHECK(w.PopFront().frame.timestamp == 2.0);
    threw = false;
    try {
        w.PopFront();
    } catch (const std::logic_error&) {
        threw = true;
    }
    CHECK(threw);

    DepthImage raw(3, 1, 0.f), virt(3, 1, 0.f);
    raw(0, 0) = 1.25f;
    virt(1, 0) = 2.5f;
    const DepthImage out = RefineDepth(raw, virt, 8.0);
    CHECK(out(0, 0) == 1.25f && out(1, 0) == 2.5f && out(2, 0) == 8.0f);
    std::printf("host containers ok\n");
    return 0;
}

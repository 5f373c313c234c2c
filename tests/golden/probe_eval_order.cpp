// Probe (not reference code): which argument of a two-argument constructor
// call does g++ evaluate first?  The reference builds complex draws as
// std::complex<double>(draw(), draw()) (channel_sim.cpp:56, :71), so this
// decides whether the first RNG draw lands in the real or imaginary part.
#include <complex>
#include <cstdio>

static int counter = 0;
static double draw() { return static_cast<double>(++counter); }

int main() {
    const std::complex<double> z(draw(), draw());
    std::puts(z.real() == 2.0 ? "second_draw_is_real" : "first_draw_is_real");
    return 0;
}

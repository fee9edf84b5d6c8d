// roster.cpp -- prints the reference roster (proj/include/utf8v/lookup.hpp:30)
// as detect_backends() built it, name:width per entry, front first: the check
// that the cuda entry was registered (tests/test_reference_tests.py).
#include <cstdio>

#include "utf8v/lookup.hpp"

int main() {
  for (const utf8v::lookup_backend& b : utf8v::lookup_backends()) std::printf("%s:%zu ", b.name, b.width);
  std::printf("\n");
  return 0;
}

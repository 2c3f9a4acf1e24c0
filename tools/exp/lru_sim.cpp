// LRU simulation of N_u sector reads for NodeIteratorN under an apex order.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <unordered_map>
#include <list>
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");  // n, eoff[n+1] (u64), m, eff[m] (u32)
  uint64_t n, m;
  fread(&n, 8, 1, f);
  std::vector<uint64_t> eoff(n + 1);
  fread(eoff.data(), 8, n + 1, f);
  fread(&m, 8, 1, f);
  std::vector<uint32_t> eff(m);
  fread(eff.data(), 4, m, f);
  fclose(f);
  FILE* fo = fopen(argv[2], "rb");
  std::vector<uint32_t> order(n);
  fread(order.data(), 4, n, fo);
  fclose(fo);
  const uint64_t cap_lines = strtoull(argv[3], 0, 10);  // 32B sectors in cache
  // simple LRU: clock-free exact LRU with list + map
  std::list<uint64_t> lru;
  std::unordered_map<uint64_t, std::list<uint64_t>::iterator> pos;
  pos.reserve(cap_lines * 2);
  uint64_t acc = 0, miss = 0;
  auto touch = [&](uint64_t s) {
    ++acc;
    auto it = pos.find(s);
    if (it != pos.end()) {
      lru.splice(lru.begin(), lru, it->second);
      return;
    }
    ++miss;
    lru.push_front(s);
    pos[s] = lru.begin();
    if (pos.size() > cap_lines) {
      pos.erase(lru.back());
      lru.pop_back();
    }
  };
  for (uint64_t k = 0; k < n; ++k) {
    const uint32_t v = order[k];
    for (uint64_t i = eoff[v]; i < eoff[v + 1]; ++i) {
      const uint32_t u = eff[i];
      const uint64_t a = eoff[u], b = eoff[u + 1];
      if (a == b) continue;
      for (uint64_t s = a / 8; s <= (b - 1) / 8; ++s) touch(s);
    }
  }
  printf("accesses %llu misses %llu miss_rate %.3f\n", (unsigned long long)acc,
         (unsigned long long)miss, (double)miss / acc);
}

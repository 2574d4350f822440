// dreamsched/schedule.hpp — the layer -> iteration-of-H assignment.
//
// Drop-in for the reference's schedule.hpp:33-54.  sets[h-1] (descending
// layer indexes) is synchronized at phase h of the period; concatenated the
// sets spell L..1 with empty sets only at the tail.  supplemental[h-1] is the
// bubble-fill prefix {L..l} added at phase h.  On the device the union of the
// two is one or two contiguous coordinate ranges of the parameter arena.
#ifndef DREAMSCHED_SCHEDULE_HPP_
#define DREAMSCHED_SCHEDULE_HPP_

#include <filesystem>
#include <iosfwd>
#include <string_view>
#include <vector>

namespace dreamsched {

struct Schedule {
  int period = 1;
  std::vector<std::vector<int>> sets;
  std::vector<std::vector<int>> supplemental;

  int layer_count() const;
  int set_of_layer(int layer) const;  // 1-based phase; ArgumentError if absent
  void validate(int layer_count) const;

  static Schedule single_set(int layer_count);
  static Schedule equal_number_partition(int layer_count, int period);
};

Schedule load_schedule(const std::filesystem::path& path);
void save_schedule(const Schedule& schedule, const std::filesystem::path& path);
Schedule parse_schedule(std::istream& in, std::string_view source_name);
void write_schedule(const Schedule& schedule, std::ostream& out);

}  // namespace dreamsched

#endif  // DREAMSCHED_SCHEDULE_HPP_

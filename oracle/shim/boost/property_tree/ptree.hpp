// oracle/shim/boost/property_tree/ptree.hpp — the Boost.PropertyTree subset
// /root/reference/proj/src/hand.cpp:127-196 uses (test infrastructure for the
// oracle/_ref build only): an ordered multimap of child nodes with string
// data, path lookup with '.' separators, get<T>() via stream extraction
// (ptree_bad_data / ptree_bad_path on failure), get_child(_optional).
#pragma once

#include <list>
#include <type_traits>
#include <typeinfo>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>

namespace boost {
namespace property_tree {

class ptree_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ptree_bad_data : public ptree_error {
 public:
  using ptree_error::ptree_error;
};
class ptree_bad_path : public ptree_error {
 public:
  using ptree_error::ptree_error;
};

// boost::optional<ptree&> stand-in: a nullable reference.
template <typename T>
class optional_ref {
  T* p_ = nullptr;

 public:
  optional_ref() = default;
  explicit optional_ref(T* p) : p_(p) {}
  explicit operator bool() const { return p_ != nullptr; }
  bool operator!() const { return p_ == nullptr; }
  T& operator*() const { return *p_; }
  T* operator->() const { return p_; }
  T& get() const { return *p_; }
};

class ptree {
 public:
  using value_type = std::pair<const std::string, ptree>;
  using container = std::list<value_type>;
  using iterator = container::iterator;
  using const_iterator = container::const_iterator;

  ptree() = default;
  explicit ptree(std::string data) : data_(std::move(data)) {}

  iterator begin() { return children_.begin(); }
  iterator end() { return children_.end(); }
  const_iterator begin() const { return children_.begin(); }
  const_iterator end() const { return children_.end(); }
  bool empty() const { return children_.empty(); }
  std::size_t size() const { return children_.size(); }

  const std::string& data() const { return data_; }
  std::string& data() { return data_; }
  void put_value(const std::string& v) { data_ = v; }

  ptree& push_back_child(const std::string& key, ptree child) {
    children_.emplace_back(key, std::move(child));
    return children_.back().second;
  }
  // add_child/put_child with a single-segment key (what the parser needs)
  ptree& add_child(const std::string& key, const ptree& child) { return push_back_child(key, child); }

  const ptree* find_path(const std::string& path) const {
    const ptree* cur = this;
    std::size_t start = 0;
    while (cur) {
      std::size_t dot = path.find('.', start);
      std::string seg = path.substr(start, dot == std::string::npos ? std::string::npos : dot - start);
      const ptree* next = nullptr;
      for (const auto& kv : cur->children_) {
        if (kv.first == seg) {
          next = &kv.second;
          break;
        }
      }
      cur = next;
      if (dot == std::string::npos) break;
      start = dot + 1;
    }
    return cur;
  }

  const ptree& get_child(const std::string& path) const {
    const ptree* p = find_path(path);
    if (!p) throw ptree_bad_path("No such node (" + path + ")");
    return *p;
  }
  ptree& get_child(const std::string& path) {
    return const_cast<ptree&>(static_cast<const ptree&>(*this).get_child(path));
  }
  optional_ref<const ptree> get_child_optional(const std::string& path) const {
    return optional_ref<const ptree>(find_path(path));
  }
  optional_ref<ptree> get_child_optional(const std::string& path) {
    return optional_ref<ptree>(const_cast<ptree*>(find_path(path)));
  }

  template <typename T>
  T get_value() const {
    if constexpr (std::is_same_v<T, std::string>) {
      return data_;
    } else {
      std::istringstream ss(data_);
      T v{};
      ss >> v;
      if (!ss.eof()) ss >> std::ws;
      if (ss.fail() || ss.bad() || !ss.eof())
        throw ptree_bad_data("conversion of data to type \"" + std::string(typeid(T).name()) +
                             "\" failed");
      return v;
    }
  }
  template <typename T>
  T get(const std::string& path) const {
    return get_child(path).get_value<T>();
  }
  template <typename T>
  T get(const std::string& path, const T& def) const {
    const ptree* p = find_path(path);
    if (!p) return def;
    try {
      return p->get_value<T>();
    } catch (const ptree_bad_data&) {
      return def;
    }
  }
  std::string get(const std::string& path, const char* def) const {
    return get<std::string>(path, std::string(def));
  }
  template <typename T>
  std::optional<T> get_optional(const std::string& path) const {
    const ptree* p = find_path(path);
    if (!p) return std::nullopt;
    try {
      return p->get_value<T>();
    } catch (const ptree_bad_data&) {
      return std::nullopt;
    }
  }

 private:
  std::string data_;
  container children_;
};

}  // namespace property_tree
}  // namespace boost

# find_package(dreamsched) for this B200 implementation: provides the same
# imported target name as the reference (dreamsched::core, core/CMakeLists.txt
# :1-38), so a CMake consumer switches by pointing dreamsched_DIR here.
get_filename_component(_ds_root "${CMAKE_CURRENT_LIST_DIR}/.." ABSOLUTE)
set(_ds_lib "${_ds_root}/paper_2502_11058_b200/lib")
if(NOT EXISTS "${_ds_lib}/libdreamsched.so")
  message(FATAL_ERROR "dreamsched: build the library first (make -C ${_ds_root})")
endif()
if(NOT TARGET dreamsched::core)
  add_library(dreamsched::dsx SHARED IMPORTED)
  set_target_properties(dreamsched::dsx PROPERTIES
    IMPORTED_LOCATION "${_ds_lib}/libdsx.so"
    INTERFACE_INCLUDE_DIRECTORIES "${_ds_root}/include")
  add_library(dreamsched::core SHARED IMPORTED)
  set_target_properties(dreamsched::core PROPERTIES
    IMPORTED_LOCATION "${_ds_lib}/libdreamsched.so"
    INTERFACE_INCLUDE_DIRECTORIES "${_ds_root}/include"
    INTERFACE_COMPILE_FEATURES cxx_std_20
    INTERFACE_LINK_LIBRARIES dreamsched::dsx)
endif()
set(dreamsched_FOUND TRUE)

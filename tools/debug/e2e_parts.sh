SWSDC_UPLOAD_CTAS=32 python tools/debug/e2e_parts.py
SWSDC_UPLOAD_CTAS=148 python tools/debug/e2e_parts.py
